"""Row f3: mask counts outside {1, 2, 4, 8} (3, 5, 6, 7 and 16) through AUTO (the SIMT
kernel), bf16 and fp32, against the oracle; the fast paths refuse them explicitly."""
import numpy as np
import pytest
import torch

from tests.helpers import TIGHT, TOL, gpu_forward, make_inputs, normwise_err, oracle_forward

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_23225_b200.build import build
    build()


@pytest.mark.parametrize("n_m", [3, 5, 6, 7, 16])
@pytest.mark.parametrize("dtype,B", [("bf16", 1), ("bf16", 6), ("f32", 2)])
def test_wide_mask_counts(n_m, dtype, B):
    inp = make_inputs(2000 + n_m * 7 + B, B=B, d=256, h=300, n_m=n_m, dtype=dtype)
    y, used = gpu_forward(inp, dtype, n_m, "swish")
    assert used == "simt"
    err = normwise_err(y, oracle_forward(inp, dtype, n_m, "swish"))
    assert err <= TOL[dtype] and err <= TIGHT[dtype], err


@pytest.mark.parametrize("path", ["mma", "tcdec", "tcgen05"])
def test_fast_paths_refuse_wide_counts(path):
    from paper_2506_23225_b200.mglu import MgluError, MGLU_ERR_UNSUPPORTED
    inp = make_inputs(1, B=2, d=256, h=128, n_m=3, dtype="bf16")
    with pytest.raises(MgluError) as e:
        gpu_forward(inp, "bf16", 3, "swish", path=path)
    assert e.value.status == MGLU_ERR_UNSUPPORTED
