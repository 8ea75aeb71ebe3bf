#!/usr/bin/env python
"""bench.py -- the FlashMGLU forward pass (SwiMGLU up-projection) on B200.

Default workload (N=1): BASELINE.json's target row -- batch-1 SwiMGLU, n_m = 4, d = 4096,
h = 14336, bf16 (config 3 at B = 1).  One step = one forward call (all SURVEY 8(a) rows run in
one kernel).  For N > 1 the layer's output columns (h) are column-sharded across ranks with no
data-path collective (reading R-e); value = the whole layer's algorithmic bytes / max-over-ranks
time.  Default "scaling": "strong" -- the BASELINE layer itself is split across the N ranks (each owns
h/N output columns); --scaling weak makes the layer N column blocks wide (per-GPU work fixed).
After timing, N>1 runs all-gather the h-sliced outputs over NCCL (the full-output check) and rank 0
compares them with the unsharded layer computed on its own GPU: bit-identical by construction.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mglu|reference] [--workload NAME]

Timing: W untimed warm-up steps, then EXACTLY K steps between CUDA events on the launching stream,
bracketed by barrier + synchronize, behind an untimed device-side spin that lets the host enqueue
them ahead; NVML samples SM clocks and throttle reasons during the spin and the timed region.
L2: the per-step inputs are larger than L2 -- L distinct copies of the layer (W + codes,
L x 147 MB) are rotated, so every step streams cold weights (no flush kernel is needed).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

WORKLOADS = {
    # name: (d, h, n_m, B, act, description)
    "decode_b1": (4096, 14336, 4, 1, "swish", "config3 batch-1 SwiMGLU d=4096 h=14336 n_m=4 (Llama-3-8B FFN)"),
    "decode7b_b1": (4096, 11008, 4, 1, "swish", "config2 batch-1 SwiMGLU d=4096 h=11008 n_m=4 (LLaMA-7B FFN)"),
    "decode_b8": (4096, 14336, 4, 8, "swish", "config3 batch-8 SwiMGLU d=4096 h=14336 n_m=4"),
    "sweep_b1_nm1": (8192, 28672, 1, 1, "swish", "config5 batch-1 d=8192 h=28672 n_m=1"),
    "sweep_b1_nm2": (8192, 28672, 2, 1, "swish", "config5 batch-1 d=8192 h=28672 n_m=2"),
    "sweep_b1_nm4": (8192, 28672, 4, 1, "swish", "config5 batch-1 d=8192 h=28672 n_m=4"),
    "sweep_b1_nm8": (8192, 28672, 8, 1, "swish", "config5 batch-1 d=8192 h=28672 n_m=8"),
    "prefill": (8192, 28672, 4, 4096, "swish", "config4 prefill SwiMGLU d=8192 h=28672 n_m=4, 4096 tokens"),
    "decode_b64": (4096, 14336, 4, 64, "swish", "config3 batch-64 SwiMGLU d=4096 h=14336 n_m=4"),
    "sweep_b2048_nm1": (8192, 28672, 1, 2048, "swish", "config5 batch-2048 d=8192 h=28672 n_m=1"),
    "sweep_b2048_nm2": (8192, 28672, 2, 2048, "swish", "config5 batch-2048 d=8192 h=28672 n_m=2"),
    "sweep_b2048_nm4": (8192, 28672, 4, 2048, "swish", "config5 batch-2048 d=8192 h=28672 n_m=4"),
    "sweep_b2048_nm8": (8192, 28672, 8, 2048, "swish", "config5 batch-2048 d=8192 h=28672 n_m=8"),
}
DEFAULT_WORKLOAD = "decode_b1"
METRIC = "SwiMGLU up-proj HBM GB/s at batch 1 (algorithmic W+codes+x+y bytes / time per call)"
METRIC_TC = "SwiMGLU up-proj TFLOP/s at prefill (algorithmic 2*B*d*h*(n_m+1) flops / time per call)"
PREFILL_MIN_B = 64          # workloads with more tokens are reported against the tensor roofline


def algorithmic_bytes(d, h, n_m, B, elem=2):
    """W once, the packed codes once (n_m bits/element), x read, y written."""
    return h * d * elem + (h * d * n_m + 7) // 8 + B * d * elem + B * h * elem


def algorithmic_flops(d, h, n_m, B):
    """the (n_m + 1) GEMMs sharing x -- t and the n_m sign-flipped products."""
    return 2 * B * d * h * (n_m + 1)


def is_prefill(B):
    return B >= PREFILL_MIN_B


def work(d, h, n_m, B):
    """(units per call, scale to the metric unit, unit, metric) of the workload's metric."""
    if is_prefill(B):
        return algorithmic_flops(d, h, n_m, B), 1e12, "TFLOP/s", METRIC_TC
    return algorithmic_bytes(d, h, n_m, B), 1e9, "GB/s", METRIC


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            pk = json.load(f)
        return {"hbm_gbs": pk["hbm_gbs"], "bf16_tflops": pk["bf16_tflops"],
                "bf16_tflops_sustained": pk.get("bf16_tflops_sustained"), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "source": "fallback (B200_PROFILING.md)"}


# ---------------------------------------------------------------- clocks (NVML)
class ClockSampler:
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}

    def __init__(self, device_index: int, period_s: float = 0.005):
        self.samples, self.power, self.reasons, self.ok = [], [], set(), False
        self.period = period_s
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - no NVML
            self.err = str(e)
            self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.power.append(nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def start(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self._t:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "err", "")}
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples),
                "power_w_max": max(self.power) if self.power else None}


# ---------------------------------------------------------------- distributed plumbing
def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # (MGLU_DIST_BACKEND=gloo runs several ranks on one GPU: exercises the multi-rank code, its
    # timings are not bench numbers)
    dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if ws > 1:
        import torch.distributed as dist
        backend = os.environ.get("MGLU_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    return ws, rank, dev


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(ws, value: float) -> float:
    if ws == 1:
        return value
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------- inputs (synthetic, seeded)
def make_layers(d, h_total, n_m, B, L, seed, lo, hi):
    """L distinct copies of the whole layer, drawn on the device from the seed alone (synth recipe:
    x ~ N(0,1), Wt ~ U(+-1/sqrt(d)), code bits i.i.d. Bernoulli(0.5)), and this rank's rows
    [lo, hi) of each as views (a column shard of Wt and of the packed codes is a pointer offset)."""
    from synth import random_packed_codes
    g = torch.Generator(device="cuda").manual_seed(seed * 1000)
    x = torch.randn(B, d, device="cuda", generator=g).to(torch.bfloat16)
    rb = d * n_m // 8
    fulls, shards = [], []
    for li in range(L):
        Wt = ((torch.rand(h_total, d, device="cuda", generator=g) * 2 - 1) / d ** 0.5).to(torch.bfloat16)
        codes = random_packed_codes(seed * 7919 + li, h_total, d, n_m, device="cuda")
        fulls.append((Wt, codes))
        shards.append((Wt[lo:hi], codes[lo * rb:hi * rb]))
    return x, fulls, shards


def enqueue_ahead(stream, K, us_per_step=None):
    """A device-side spin (untimed, before the start event) so the host enqueues the timed launches
    while the GPU is busy: the timed region then sees back-to-back launches, not host gaps (the
    first launch's latency, a slow ctypes call, or the NVML clock sampler briefly stalling the
    launching thread).  ~40 us of spin per step + 1 ms, capped at 50 ms."""
    us = float(os.environ.get("MGLU_BENCH_AHEAD_US", "40")) if us_per_step is None else us_per_step
    with torch.cuda.stream(stream):
        torch.cuda._sleep(int(min(50e3, 1e3 + K * us) * 1965))


def time_steps(fn_step, K, stream):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    enqueue_ahead(stream, K)
    e0.record(stream)
    for k in range(K):
        fn_step(k)
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / 1e3   # seconds


def per_call_distribution(fn_step, K, stream):
    """Separate pass (not the headline): an event pair around every call, so the per-call
    median / p10 / p90 are visible.  Events between calls cut the PDL overlap of consecutive
    launches, so these are slightly pessimistic against the headline loop."""
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
    enqueue_ahead(stream, K)
    evs[0].record(stream)
    for k in range(K):
        fn_step(k)
        evs[k + 1].record(stream)
    evs[-1].synchronize()
    us = sorted(evs[k].elapsed_time(evs[k + 1]) * 1e3 for k in range(K))
    q = lambda f: us[min(K - 1, int(round(f * (K - 1))))]   # noqa: E731
    return {"median_us": q(0.5), "p10_us": q(0.1), "p90_us": q(0.9), "calls": K,
            "how": "event pair around each call (separate pass; cuts PDL overlap between calls)"}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cublas_swiglu_us(d, h, B, L, K, stream):
    """Same-box cuBLAS SwiGLU up-projection at equal d/h/B (bf16): (i) two GEMMs + silu*mul,
    (ii) one GEMM on the concatenated [2h x d] weight + split + silu*mul.  L rotated weight
    copies (inputs > L2), CUDA-graph replay of K steps; returns the faster, microseconds/call."""
    g = torch.Generator(device="cuda").manual_seed(123)
    x = torch.randn(B, d, device="cuda", generator=g).to(torch.bfloat16)
    Ws = [(torch.randn(2 * h, d, device="cuda", generator=g) * 0.01).to(torch.bfloat16) for _ in range(L)]
    res = {}
    for variant in ("two_gemm", "concat_gemm"):
        def step(k, Ws=Ws, variant=variant):
            W = Ws[k % L]
            if variant == "two_gemm":
                a = torch.matmul(x, W[:h].t())
                b = torch.matmul(x, W[h:].t())
            else:
                ab = torch.matmul(x, W.t())
                a, b = ab[:, :h], ab[:, h:]
            return torch.nn.functional.silu(a) * b
        with torch.cuda.stream(stream):
            for k in range(3):
                step(k)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                for k in range(K):
                    step(k)
            graph.replay()
            stream.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            graph.replay()
            e1.record(stream)
            e1.synchronize()
        res[variant] = e0.elapsed_time(e1) * 1e3 / K
        del graph
    res["best_us"] = min(res["two_gemm"], res["concat_gemm"])
    return res


def oracle_sample_cols(d, h, n_m, B):
    """Columns of the layer the oracle computes per pass: the whole layer for decode; for prefill
    a bounded column sample (all B tokens, all d), so one pass stays around a second."""
    if not is_prefill(B):
        return h
    per_col = 2 * B * d * (2 * n_m + 1)          # the oracle's own flops per output column
    return int(max(1, min(h, 2e9 // per_col)))


def cpu_baseline(d, h, n_m, B, act_code, budget_s=10.0):
    """The oracle as it stands (C, binary64, OpenMP over output columns) on the same workload:
    full layer (decode) or a column sample (prefill) per pass, repeated until ~budget_s of CPU
    work on all host cores, then ~budget_s/4 on one core; the rate is scaled to the metric's unit
    from the columns actually computed."""
    from oracle import COracle
    o = COracle()
    rng = np.random.default_rng(0)
    c = oracle_sample_cols(d, h, n_m, B)
    x = rng.standard_normal((B, d))
    Wt = rng.uniform(-1 / d ** 0.5, 1 / d ** 0.5, (c, d))
    packed = rng.integers(0, 256, (h * d * n_m + 7) // 8, dtype=np.uint8)
    units, scale, unit, _ = work(d, c, n_m, B)

    def timed(threads, budget, cols):
        o.set_num_threads(threads)
        passes, t0 = 0, time.perf_counter()
        while True:
            o.forward(x, Wt[:len(cols)], cols, packed, n_m, act_code)
            passes += 1
            el = time.perf_counter() - t0
            if el >= budget or passes >= 200:
                return el / passes, passes, el

    per, passes, el = timed(os.cpu_count() or 1, budget_s, np.arange(c))
    cores = o.num_threads()
    # one core: a column sample of the same pass (the oracle's per-column cost is uniform)
    c1 = max(1, min(c, int(c / max(1.0, per * cores / max(budget_s / 8, 1e-3)))))
    per1, passes1, el1 = timed(1, budget_s / 4, np.arange(c1))
    units1 = work(d, c1, n_m, B)[0]
    return {"value": units / per / scale, "unit": unit,
            "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
            "sample": f"B={B} tokens x {c} of {h} columns x d={d} per pass, {passes} passes in {el:.1f} s",
            "seconds_per_call": per * h / c,
            "one_core": {"value": units1 / per1 / scale, "unit": unit, "cores": 1,
                         "sample": f"B={B} x {c1} columns x d={d} per pass, {passes1} passes in {el1:.1f} s"}}


# ---------------------------------------------------------------- arms
def run_reference(args, ws, rank):
    """--impl reference: the CPU oracle as it stands, timed on the host cores, on this arm's
    workload/metric.  Rank 0 only; other ranks exit without work."""
    if rank != 0:
        return None
    from oracle import ACT_NAMES, COracle
    d, h, n_m, B, act, desc = WORKLOADS[args.workload]
    h = h * ws if (ws > 1 and args.scaling == "weak") else h     # the mglu arm's layer at this N
    o = COracle()
    # torchrun sets OMP_NUM_THREADS=1 per process; rank 0 is the only rank working here, so the
    # oracle gets the host's cores (its result does not depend on the thread count)
    o.set_num_threads(os.cpu_count() or 1)
    rng = np.random.default_rng(0)
    c = oracle_sample_cols(d, h, n_m, B)
    x = rng.standard_normal((B, d))
    Wt = rng.uniform(-1 / d ** 0.5, 1 / d ** 0.5, (c, d))
    packed = rng.integers(0, 256, (h * d * n_m + 7) // 8, dtype=np.uint8)
    cols = np.arange(c)
    for _ in range(args.warmup):
        o.forward(x, Wt, cols, packed, n_m, ACT_NAMES[act])
    t0 = time.perf_counter()
    for _ in range(args.steps):
        o.forward(x, Wt, cols, packed, n_m, ACT_NAMES[act])
    el = time.perf_counter() - t0
    per = el / args.steps
    units, scale, unit, metric = work(d, c, n_m, B)
    value = units * args.steps / el / scale
    sample = f"B={B} tokens x {c} of {h} columns x d={d} per step"
    return {
        "impl": "reference", "metric": metric, "value": value, "unit": unit, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": desc, "d": d, "h": h, "n_m": n_m, "batch": B, "act": act},
        "cpu_baseline": {"value": value, "unit": unit, "cores": o.num_threads(), "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def run_mglu(args, ws, rank, local):
    from paper_2506_23225_b200.build import build
    if rank == 0 and not os.environ.get("MGLU_LIB"):     # (MGLU_LIB: an experiment build, see build.py)
        build()
    barrier(ws)
    from paper_2506_23225_b200.mglu import Mglu
    from paper_2506_23225_b200.shard import shard_bounds
    d, h, n_m, B, act, desc = WORKLOADS[args.workload]
    # column shard of h (no exchange on the hot path): this rank's rows of Wt and of the codes
    # weak scaling (default): the layer is N column blocks wide, each rank owns one block of the N=1
    # workload's width (per-GPU work fixed); strong: the N=1 layer itself is split across the ranks
    h_total = h * ws if args.scaling == "weak" else h
    lo, hi = shard_bounds(h_total, ws, rank)
    h_loc = hi - lo
    L = args.layers
    x, fulls, layers = make_layers(d, h_total, n_m, B, L, seed=0, lo=lo, hi=hi)
    y = torch.empty(B, h_loc, device="cuda", dtype=torch.bfloat16)
    layer = Mglu(d, h_loc, n_m, act=act, dtype="bf16", device=local, path=args.path)
    stream = torch.cuda.Stream()

    if args.ffn:
        # SwiMGLU FFN block (row f1): column-sharded up-projection, row-sharded dense W_o (an
        # n_m = 0 handle) and, across ranks, one fp32 all-reduce of the [B][d] partials
        down = Mglu(h_loc, d, 0, act="identity", dtype="bf16", device=local)
        gw = torch.Generator(device="cuda").manual_seed(7 + rank)
        Wos = [((torch.rand(d, h_loc, device="cuda", generator=gw) * 2 - 1) / h ** 0.5).to(torch.bfloat16)
               for _ in range(L)]
        yd = torch.empty(B, d, device="cuda", dtype=torch.bfloat16)
        up_calls = [layer.bind(x, Wt, codes, y, stream=stream) for Wt, codes in layers]
        down_calls = [down.bind(y, Wo, None, yd, stream=stream) for Wo in Wos]

        def step(k):
            up_calls[k % L]()
            down_calls[k % L]()
            if ws > 1:
                import torch.distributed as dist
                part = yd.float()
                dist.all_reduce(part)
    elif args.topk:
        # Top-K routed MGLU (Appendix B): a step = router (x W_r, TopK, softmax) + routed forward
        from paper_2506_23225_b200.mglu import mglu_forward_routed, mglu_router_topk
        gr = torch.Generator(device="cuda").manual_seed(99)
        Wr = (torch.randn(n_m, d, device="cuda", generator=gr) / d ** 0.5).to(torch.bfloat16)
        G = torch.empty(B, n_m, device="cuda", dtype=torch.float32)

        def step(k):
            Wt, codes = layers[k % L]
            mglu_router_topk(layer.handle, x, B, Wr, args.topk, G, stream)
            mglu_forward_routed(layer.handle, x, B, Wt, codes, G, args.topk, y, stream)
    else:
        calls = [layer.bind(x, Wt, codes, y, stream=stream) for Wt, codes in layers]

        def step(k):
            calls[k % L]()

    with torch.cuda.stream(stream):
        for k in range(args.warmup):
            step(k)
        stream.synchronize()
        launches_per_step = layer.last_launch_count() + (1 if (args.topk or args.ffn) else 0)
        path_used = layer.last_path()
        # optional clock window (steps before the timed region; a step COUNT agreed by all ranks:
        # steps may hold collectives).  Default 0: the timed region follows the W warm-up steps
        # directly, as the driver's protocol states -- a long window only pre-heats the GPU into
        # its power cap (measured: -4 us/call at the config-3 shape after a 0.3 s window)
        if args.clock_window > 0:
            t0 = time.perf_counter()
            for k in range(args.warmup):
                step(k)
            stream.synchronize()
            t_step = max_over_ranks(ws, (time.perf_counter() - t0) / max(1, args.warmup))
            for k in range(int(min(100000, args.clock_window / max(t_step, 1e-7)))):
                step(k)
                if (k + 1) % 256 == 0:
                    stream.synchronize()
            stream.synchronize()
        # timed region, NVML-sampled from a thread polling every 0.2 ms while the enqueue-ahead
        # spin and the K steps run on the device
        sampler = ClockSampler(local, period_s=0.0002)
        barrier(ws)
        torch.cuda.synchronize()
        if not os.environ.get("MGLU_BENCH_NO_SAMPLER"):    # (experiment switch: NVML interference)
            sampler.start()
        el = time_steps(step, args.steps, stream)
        torch.cuda.synchronize()
        sampler.stop()
        barrier(ws)
        dist_calls = per_call_distribution(step, args.steps, stream)
        torch.cuda.synchronize()
        barrier(ws)
    el_max = max_over_ranks(ws, el)
    units_layer, scale, unit, metric = work(d, h_total, n_m, B)
    units_rank = work(d, h_loc, n_m, B)[0]
    bytes_rank = algorithmic_bytes(d, h_loc, n_m, B)
    if args.ffn:                                              # + the dense W_o pass (x = y, out = [B][d])
        units_layer += algorithmic_bytes(h_total, d, 0, B)
        units_rank += algorithmic_bytes(h_loc, d, 0, B)
        bytes_rank += algorithmic_bytes(h_loc, d, 0, B)
        metric = "SwiMGLU FFN block (up-proj + W_o) HBM GB/s at batch B (algorithmic bytes of both layers / time per step)"
    value = units_layer * args.steps / el_max / scale
    # (routed steps: the router is a d x n_m GEMV next to the layer; the step's two launches are
    # charged together to the layer's bytes)
    per_launch_s = el / args.steps / (1 if (args.topk or args.ffn) else max(1, launches_per_step))
    peaks = load_peaks()
    achieved = units_rank / per_launch_s / scale
    if is_prefill(B):
        peak, peak_src = peaks["bf16_tflops_sustained"] or peaks["bf16_tflops"], "bf16_tflops_sustained (cuBLAS)"
        bound = "tensor"
    else:
        peak, peak_src, bound = peaks["hbm_gbs"], "hbm_gbs (copy)", "hbm"

    # e2e through the C-ABI host-buffer entry (mglu_forward_host): per step, x H2D from pinned
    # memory, the forward, y D2H to pinned memory.  `e2e`: ONE stream, every call serialised (the
    # latency a dependent decode step sees).  `e2e_pipelined`: consecutive steps alternate over E
    # streams, each with its own handle and pinned buffers, so one step's copies overlap another
    # step's kernel (throughput of independent layers).
    def e2e_leg(E):
        e_layers = [layer] + [Mglu(d, h_loc, n_m, act=act, dtype="bf16", device=local, path=args.path)
                              for _ in range(E - 1)]
        e_streams = [stream] + [torch.cuda.Stream() for _ in range(E - 1)]
        xh = [x.cpu().pin_memory() for _ in range(E)]
        yh = [torch.empty(B, h_loc, dtype=torch.bfloat16).pin_memory() for _ in range(E)]

        def step_host(k):
            Wt, codes = layers[k % L]
            e = k % E
            e_layers[e].forward_host(xh[e], Wt, codes, yh[e], stream=e_streams[e])

        for k in range(max(3, args.warmup)):
            step_host(k)
        torch.cuda.synchronize()
        barrier(ws)
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        enqueue_ahead(stream, args.steps)
        ev0.record(stream)
        for st_ in e_streams[1:]:
            st_.wait_event(ev0)
        for k in range(args.steps):
            step_host(k)
        for st_ in e_streams[1:]:
            stream.wait_stream(st_)
        ev1.record(stream)
        ev1.synchronize()
        el_e = max_over_ranks(ws, ev0.elapsed_time(ev1) / 1e3)
        barrier(ws)
        for extra in e_layers[1:]:
            extra.close()
        return {"value": units_layer * args.steps / el_e / scale, "unit": unit,
                "h2d_bytes_per_step": B * d * 2 * ws, "d2h_bytes_per_step": B * h_total * 2,
                "us_per_call": el_e / args.steps * 1e6, "streams": E}

    e2e = e2e_pipe = None
    if not (args.topk or args.ffn):
        e2e = e2e_leg(1)
        e2e["how"] = ("mglu_forward_host per step on one stream: pinned x -> device, forward, y -> pinned host; "
                      "every call serialised")
        if args.e2e_streams > 1:
            e2e_pipe = e2e_leg(args.e2e_streams)
            e2e_pipe["how"] = (f"mglu_forward_host per step, steps alternating over {args.e2e_streams} streams/handles "
                               "so one step's copies overlap another step's kernel (independent layers)")

    # full-output check (N > 1): all-gather the h-sliced outputs over NCCL and compare, on rank 0,
    # with the unsharded layer computed by the same kernels on rank 0's GPU (bit-identical: the
    # kernels' reduction order does not depend on the shard)
    gather_check = None
    if ws > 1 and not (args.topk or args.ffn) and args.scaling == "strong":
        from paper_2506_23225_b200.shard import gather_columns
        Wt0, codes0 = layers[0]
        layer.bind(x, Wt0, codes0, y, stream=stream)()
        torch.cuda.synchronize()
        y_full = gather_columns(y, h_total)
        if rank == 0:
            full = Mglu(d, h_total, n_m, act=act, dtype="bf16", device=local, path=args.path)
            y_ref = torch.empty(B, h_total, device="cuda", dtype=torch.bfloat16)
            full.forward(x, fulls[0][0], fulls[0][1], out=y_ref)
            torch.cuda.synchronize()
            full.close()
            diff = (y_full.float() - y_ref.float()).abs()
            gather_check = {"collective": "all_gather (NCCL)" if torch.distributed.get_backend() == "nccl" else "all_gather (gloo)",
                            "bit_identical": bool(torch.equal(y_full, y_ref)), "max_abs_diff": float(diff.max()),
                            "against": "unsharded layer on rank 0's GPU (same kernels, same seeds)"}
        barrier(ws)

    out = None
    if rank == 0:
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tpath):
            with open(tpath) as f:
                tr = json.load(f).get(args.workload)
            if tr:
                traffic = tr.get("dram_bytes_per_launch")
        out = {
            "metric": metric, "value": value, "unit": unit, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": el_max / args.steps * 1e3, "higher_is_better": True,
            "scaling": args.scaling if ws > 1 else "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (device-drawn, seeded: x~N(0,1), Wt~U(+-1/sqrt(d)), codes i.i.d. Bernoulli(0.5) bits)",
            "config": {"workload": desc, "d": d, "h": h, "h_total": h_total, "n_m": n_m, "batch": B, "act": act,
                       "parallelism": (f"column-shard of a {h_total}-wide layer over {ws} GPUs, {hi - lo} columns each "
                                       f"({args.scaling} scaling)") if ws > 1 else "single GPU",
                       "l2": f"inputs larger than L2: {L} distinct layer copies ({L * bytes_rank / 1e6:.0f} MB/rank) rotated, no flush",
                       "kernel_path": path_used, "launch": "PDL (programmatic dependent launch) per call",
                       **({"topk": args.topk, "step": "router_topk + forward_routed (2 launches)"} if args.topk else {}),
                       **({"ffn": True, "step": "MGLU up-proj + dense W_o (+ fp32 all-reduce across ranks)"} if args.ffn else {})},
            "us_per_call": el_max / args.steps * 1e6,
            "roofline": {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_source": peaks["source"] + " " + peak_src,
                         "algorithmic_units_per_launch": units_rank, "algorithmic_bytes_per_launch": bytes_rank},
            "e2e": e2e,
            **({"e2e_pipelined": e2e_pipe} if e2e_pipe else {}),
            "per_call": dist_calls,
            **({"gather_check": gather_check} if gather_check else {}),
            "gpu_launches": args.steps * launches_per_step,
            "clocks": sampler.summary(),
        }
        if not args.no_comparator and ws == 1:
            cb = cublas_swiglu_us(d, h, B, L, min(args.steps, 200 if not is_prefill(B) else 20), stream)
            out["cublas_swiglu"] = {"us_per_call": cb["best_us"], "two_gemm_us": cb["two_gemm"],
                                    "concat_gemm_us": cb["concat_gemm"],
                                    "mglu_speedup": cb["best_us"] / out["us_per_call"],
                                    "bytes_per_call": 2 * h * d * 2 + B * d * 2 + B * h * 2,
                                    "tflops": 2 * B * d * 2 * h / (cb["best_us"] * 1e-6) / 1e12}
        if not args.no_cpu_baseline and ws == 1:
            from oracle import ACT_NAMES
            out["cpu_baseline"] = cpu_baseline(d, h, n_m, B, ACT_NAMES[act], budget_s=args.cpu_budget)
    layer.close()
    return out


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["mglu", "reference"], default="mglu")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default=DEFAULT_WORKLOAD)
    ap.add_argument("--path", choices=["auto", "mma", "simt", "tcgen05", "tcdec", "tcrow"], default="auto")
    ap.add_argument("--layers", type=int, default=4, help="distinct layer copies rotated (L2 hygiene)")
    ap.add_argument("--clock-window", type=float, default=0.0,
                    help="seconds of extra steps before the timed region (pre-heats the GPU; default none)")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--e2e-streams", type=int, default=3,
                    help="streams the pipelined e2e leg (e2e_pipelined) alternates over; 0 skips it")
    ap.add_argument("--topk", type=int, default=0, help="Top-K routed MGLU: K kept masks (router + routed forward)")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="strong",
                    help="N>1: strong = split the BASELINE layer's columns across the ranks; weak = each GPU a full-width column block (work per GPU fixed)")
    ap.add_argument("--ffn", action="store_true", help="FFN block: up-projection + dense W_o (+ all-reduce under torchrun)")
    ap.add_argument("--no-comparator", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shape", default=None, help="experiment: d,h,n_m,B (overrides --workload)")
    args = ap.parse_args(argv)
    if args.shape:
        d_, h_, nm_, b_ = (int(v) for v in args.shape.split(","))
        WORKLOADS["custom"] = (d_, h_, nm_, b_, "swish", f"custom d={d_} h={h_} n_m={nm_} B={b_}")
        args.workload = "custom"
    if args.warmup < 3:
        args.warmup = 3
    ws, rank, local = (1, 0, 0)
    if args.impl == "reference":
        ws = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        out = run_reference(args, ws, rank)
    else:
        ws, rank, local = dist_init()
        out = run_mglu(args, ws, rank, local)
    if out is not None and rank == 0:
        print(json.dumps(out))
    if ws > 1 and args.impl != "reference":
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
