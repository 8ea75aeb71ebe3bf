"""compute-sanitizer memcheck / racecheck / synccheck over tiny invocations of every kernel (the
HMMA decode, stream-K tcgen05, tile tcgen05, SIMT, router, pack/unpack kernels) and the stream-K
GEMV on three concurrent streams (tools/sanitize_case.py)."""
import os
import shutil
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_23225_b200.build import build
    build()


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(tool):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not installed")
    cmd = [SAN, "--tool", tool, "--error-exitcode", "3", "--target-processes", "all",
           sys.executable, os.path.join(ROOT, "tools", "sanitize_case.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT)
    out = r.stdout + r.stderr
    assert "sanitize case ok" in out, out[-4000:]
    clean = "ERROR SUMMARY: 0 errors" in out or "SUMMARY: 0 hazards displayed (0 errors" in out
    assert r.returncode == 0 and clean, out[-4000:]
