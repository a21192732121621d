#!/usr/bin/env python
"""Benchmark: RCP block-LDL^T fp64 factorization at BASELINE.json's headline config.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

One "step" = one full RCP factorization (q = b mode) of the config-3 workload:
a seeded type-6 symmetric Gaussian matrix, n = 32768, b = 128, sketch rows
P = b + 16 = 144 (reference FactorConfig(strategy="rcp", b=128, q=128, p=144)).
``value`` = n^3/3 flop per factorization / device time (CUDA events, inputs
resident in HBM, max over ranks), summed over ranks.  The input (8.6 GB) is far
larger than the 126 MB L2, so no L2 flush is needed between steps.

Multi-GPU (torchrun, one process per GPU): one factorization per step whose trailing Schur
updates are shared by all N GPUs over NVLink peer memory (paper_1710_00125_b200.dist; rank 0
runs the panels); "scaling": "strong", value = n^3/3 / max-over-ranks step time.

``--impl reference`` times the reference's own CPU implementation on the host cores: the
unmodified ``randldl`` package (pure Python + NumPy/OpenBLAS), shipped to the GPU box as
``oracle/_ref/randldl`` by ``oracle/Makefile`` (copied from /root/reference in the build
container), stepped one panel per step through its own engine (``_Engine._run_panel``,
factor.py:540-568) on the same workload -- a bounded sample, rank 0 only.  Without
``oracle/_ref`` the oracle port (oracle/rcp_oracle.py) stands in and the line says so.

``python bench.py --gpus N`` without a torchrun environment re-launches itself under
``torch.distributed.run`` with N processes (one per GPU).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "RCP LDL^T fp64 GFLOP/s (n³/3) at n=32768, % of FP64 peak; 1/2/4/8 GPU"
FP64_PEAK_GFLOPS = 37170.0   # measured DMMA peak, profiles/r01_fp64_peaks.txt (MEASURED_PEAKS.json has no FP64)
FP64_PEAK_SRC = "measured DMMA m8n8k4 microbenchmark on this pool's B200 (profiles/r01_fp64_peaks.txt)"


def hbm_peak_gbs():
    """Measured HBM copy bandwidth from the driver-written MEASURED_PEAKS.json (fallback: the
    profiling guide's B200 figure)."""
    try:
        v = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
        return v, "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, KeyError, ValueError):
        return 6546.6, "fallback (B200_PROFILING.md)"


def cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def load_reference():
    """The unmodified reference package from oracle/_ref (None when it was not shipped)."""
    ref = ROOT / "oracle" / "_ref"
    if not (ref / "randldl" / "factor.py").exists():
        return None
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import randldl
    return randldl


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=None, help="default: the workload's (C2 8192, C3 32768, C4 20000)")
    ap.add_argument("--b", type=int, default=None)
    ap.add_argument("--p", type=int, default=None, help="sketch rows P (reference FactorConfig.p = b + oversampling)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-seconds", type=float, default=20.0, help="budget of the cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default="c3", choices=["c2", "c3", "c4", "c5"],
                    help="c3: n=32768 single matrix (headline); c2: n=8192 b=64; c4: KKT n=20000 b=64; "
                         "c5: 65536 x n=256 batched (b=16, p=8)")
    ap.add_argument("--count", type=int, default=65536, help="c5: matrices in the whole job")
    ap.add_argument("--e2e-chunk", type=int, default=296, help="c5: matrices per pipelined e2e chunk")
    ap.add_argument("--solve-reps", type=int, default=10, help="c3: timed device solves")
    ap.add_argument("--ref-seconds", type=float, default=150.0,
                    help="--impl reference: budget of timed reference panels (each ~70 s at C3 on 16 cores)")
    args = ap.parse_args()
    dn, db, dp = WORKLOADS.get(args.workload, WORKLOADS["c3"])[:3]
    args.n = dn if args.n is None else args.n
    args.b = db if args.b is None else args.b
    args.p = dp if args.p is None else args.p
    return args


# single-matrix workloads: (n, b, P, generator); BASELINE.json configs 2-4 (SURVEY section 8 mapping)
WORKLOADS = {
    "c2": (8192, 64, 74, "type6"),
    "c3": (32768, 128, 144, "type6"),
    "c4": (20000, 64, 74, "kkt_c4"),
}


def make_matrix(args):
    from paper_1710_00125_b200 import gallery
    if WORKLOADS.get(args.workload, WORKLOADS["c3"])[3] == "kkt_c4":
        n1 = args.n * 4 // 5
        return gallery.kkt_c4(n1, args.n - n1, args.seed)
    return gallery.type6(args.n, args.seed)


def metric_name(args):
    if args.workload == "c5":
        return "RCP LDL^T fp64 GFLOP/s (n³/3 per matrix) over 65536 batched n=256 matrices (C5), % of FP64 peak"
    return METRIC if args.workload == "c3" else (
        f"RCP LDL^T fp64 GFLOP/s (n³/3) at n={args.n} ({args.workload.upper()}), % of FP64 peak")


def workload_name(a):
    if a.workload == "c4":
        return (f"C4 KKT [[H, B^T], [B, 0]] n={a.n} (H = G^T G / n1 + I, G on a 2^-8 grid so G^T G is exact; "
                f"B iid N(0,1)), b={a.b}, q=b, P=b+{a.p - a.b}={a.p} sketch rows, seed={a.seed}")
    return (f"{a.workload.upper()} type6 (seeded iid N(0,1) lower triangle mirrored) n={a.n}, b={a.b}, q=b, "
            f"P=b+{a.p - a.b}={a.p} sketch rows, seed={a.seed}")


def ncu_traffic(kernel: str, detail: bool = False):
    """DRAM bytes (read + write) of one profiled launch of `kernel` from the committed ncu summaries
    (profiles/r02_ncu_traffic.json, then r01); with detail, the launch it refers to and its
    algorithmic bytes.  Keys: kernel name (C3 / C5 captures) or "<kernel>@c2" etc."""
    rec, path = None, None
    for name in ("r02_ncu_traffic.json", "r01_ncu_traffic.json"):
        path = Path(__file__).resolve().parent / "profiles" / name
        try:
            rec = json.loads(path.read_text())[kernel]
            break
        except (OSError, KeyError, ValueError):
            rec = None
    if rec is None:
        return None
    total = rec["dram_read_bytes"] + rec["dram_write_bytes"]
    if not detail:
        return total
    return {k: rec[k] for k in rec if k not in ("dram_read_bytes", "dram_write_bytes")} | {
        "dram_bytes": total, "source": f"profiles/{path.name} (ncu --set full, one launch)"}


def c5_traffic(count: int):
    """DRAM bytes of one batched_factor_kernel launch over `count` matrices: the committed ncu
    capture (16384 matrices, one launch) scaled per matrix (the kernel does the same work per matrix)."""
    rec = ncu_traffic("batched_factor_kernel", detail=True)
    if rec is None:
        return None
    return rec["dram_bytes"] * count / rec["matrices"]


def cfg_dict(a, world: int = 1):
    return {"workload": workload_name(a), "n": a.n, "b": a.b, "q": a.b, "p_sketch": a.p,
            "oversampling": a.p - a.b,
            "parallelism": "single GPU" if world == 1 else
                           f"{world} GPUs: panels on rank 0, trailing-update tiles dealt round robin over NVLink",
            "l2": f"input {a.n * a.n * 8 / 1e9:.2f} GB >> 126 MB L2 (no flush needed)"}


def work_flops(n: int, k0: int, k1: int) -> float:
    """n^3/3-model flops attributable to eliminating columns [k0, k1): sum (n - j)^2."""
    def s(m):  # sum_{i=1}^{m} i^2
        return m * (m + 1) * (2 * m + 1) / 6.0
    return s(n - k0) - s(n - k1)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.3)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU baseline
def cpu_sample(a_host, args, budget_s: float, max_panels: int | None = None, skip_panels: int = 0):
    """Time the oracle port (the reference algorithm, numpy/OpenBLAS) panel by panel."""
    from oracle.rcp_oracle import OracleConfig, _State
    cfg = OracleConfig(p=args.p, b=args.b, q=args.b, seed=args.seed)
    t0 = time.perf_counter()
    st = _State(a_host, cfg)
    t_setup = time.perf_counter() - t0
    if st.armed and st.beta == 0.0:
        raise RuntimeError("degenerate workload")
    times, works = [], []
    npan = 0
    t_start = time.perf_counter()
    while st.k < st.n and not st.stopped:
        k0 = st.k
        t1 = time.perf_counter()
        st.panel()
        dt = time.perf_counter() - t1
        npan += 1
        if npan > skip_panels:
            times.append(dt)
            works.append(work_flops(st.n, k0, st.k))
        if max_panels is not None and npan >= max_panels + skip_panels:
            break
        if max_panels is None and time.perf_counter() - t_start >= budget_s:
            break
    return {"t_setup": t_setup, "times": times, "works": works, "k_done": st.k, "panels": npan}


def cores_used() -> int:
    try:
        from threadpoolctl import threadpool_info
        info = [i for i in threadpool_info() if i.get("user_api") == "blas"]
        if info:
            return int(info[0]["num_threads"])
    except Exception:
        pass
    return os.cpu_count() or 1


# ----------------------------------------------------------------------------- reference arm
def ref_sample(a_host, args, max_panels: int, skip_panels: int, budget_s: float = 1e30):
    """Time the REFERENCE itself (oracle/_ref/randldl) panel by panel through its own engine:
    _Engine(a, cfg) (validation, copy, Omega, B = Omega A: setup, untimed), then _run_panel()
    exactly as _Engine.run() loops (factor.py:508-513).  Stops after max_panels timed panels or
    once the timed panels exceed budget_s (at least one is always timed)."""
    randldl = load_reference()
    fmod = sys.modules["randldl.factor"]
    cfg = randldl.FactorConfig(strategy="rcp", b=args.b, q=args.b, p=args.p, seed=args.seed)
    t0 = time.perf_counter()
    eng = fmod._Engine(a_host, cfg)
    t_setup = time.perf_counter() - t0
    times, works = [], []
    npan = 0
    while eng.k < eng.n and not eng.terminated and npan < max_panels + skip_panels:
        k0 = eng.k
        t1 = time.perf_counter()
        eng._run_panel()
        dt = time.perf_counter() - t1
        npan += 1
        if npan > skip_panels:
            times.append(dt)
            works.append(work_flops(eng.n, k0, eng.k))
            if sum(times) >= budget_s:
                break
    return {"t_setup": t_setup, "times": times, "works": works, "k_done": eng.k, "panels": npan}


def run_reference(args, rank: int):
    if rank != 0:
        return
    a_host = make_matrix(args)
    warm = args.warmup
    if load_reference() is not None:
        # One C3 panel of the reference takes ~70 s on a 16-core host (mirror_lower's tril_indices
        # scatter, core.py:115-119, dominates), so the sample is bounded: at most one untimed warm-up
        # panel and --ref-seconds of timed panels (at least one).
        warm = min(args.warmup, 1)
        res = ref_sample(a_host, args, max_panels=args.steps, skip_panels=warm, budget_s=args.ref_seconds)
        kind = "reference"
        what = f"the unmodified reference randldl (oracle/_ref, numpy {np.__version__} + OpenBLAS), _Engine._run_panel"
    else:
        res = cpu_sample(a_host, args, budget_s=1e9, max_panels=args.steps, skip_panels=args.warmup)
        kind = "port"
        what = f"oracle port (numpy {np.__version__} + OpenBLAS; oracle/_ref absent)"
    tsum = sum(res["times"])
    value = sum(res["works"]) / tsum / 1e9
    nt = len(res["times"])
    sample = (f"{what} on the config-3 matrix: panels {warm + 1}..{warm + nt} timed one per step "
              f"({nt} of the {args.steps} requested; panels 1..{warm} warm-up), columns 0..{res['k_done']} "
              f"eliminated; value = sum (n-j)^2 over the timed panels' columns / time; setup (validation, copy, "
              f"Omega*A) {res['t_setup']:.1f} s excluded; CPU {cpu_model()}")
    line = {
        "impl": "reference", "metric": metric_name(args), "value": value, "unit": "GFLOP/s", "n_gpus": args.gpus,
        "steps": nt, "steps_requested": args.steps, "warmup": warm, "ms_per_step": 1e3 * tsum / max(1, nt),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded numpy Philox type6)", "config": cfg_dict(args, args.gpus),
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": cores_used(), "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- B200 arm
def run_b200(args, rank: int, world: int, local_rank: int):
    """C3: one factorization per step.  N > 1: the same single factorization with its trailing
    updates shared by all N GPUs (paper_1710_00125_b200.dist; strong scaling)."""
    import torch
    import torch.distributed as dist

    from paper_1710_00125_b200 import api, gallery
    from paper_1710_00125_b200 import dist as rdist

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    n, P = args.n, args.p
    cfg = api.FactorConfig(strategy="rcp", b=args.b, q=args.b, p=P, seed=args.seed)

    a_host = a_pin = a_dev = omega = ws = None
    if rank == 0:
        a_host = make_matrix(args)
        a_pin = torch.from_numpy(a_host).pin_memory()
        a_dev = a_pin.to(dev, non_blocking=True)
        omega = torch.from_numpy(np.random.Generator(np.random.Philox(cfg.seed)).standard_normal((P, n))).to(dev)
        if world == 1:
            ws = torch.empty(api.workspace_bytes(n, cfg), dtype=torch.uint8, device=dev)
    out = None

    def one_step(out):
        if world == 1:
            return api.factor_device(a_dev, cfg, omega=omega, workspace=ws, out=out)
        return rdist.factor_distributed_device(a_dev, cfg)

    for _ in range(max(3, args.warmup)):
        out = one_step(out)
    torch.cuda.synchronize()

    clk = ClockSampler(local_rank)
    clk.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    schur_ms, schur_flops, panel_ms = 0.0, 0.0, 0.0
    for _ in range(args.steps):
        out = one_step(out)
        if out is not None:
            schur_ms += out.stats["t_schur_ms"]
            schur_flops += out.stats["schur_flops"]
            panel_ms += out.stats["t_panel_ms"]
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    flops = n ** 3 / 3.0
    value = flops / (ms_max / 1e3) / 1e9  # one factorization per step on all N GPUs together
    stats = dict(out.stats) if out is not None else {}

    bwd = solve = None
    if rank == 0:  # device solve of the last factorization: timed, and its backward error
        rhs = torch.from_numpy(gallery.rhs(n, 1)).to(dev)
        sws = torch.empty(int(api._native.load().rcp_solve_workspace_bytes(n, 1)), dtype=torch.uint8, device=dev)
        x, _ = api.solve_device(out, rhs, workspace=sws)
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(args.solve_reps):
            x, _ = api.solve_device(out, rhs, workspace=sws)
        s1.record(stream)
        torch.cuda.synchronize()
        solve_ms = s0.elapsed_time(s1) / args.solve_reps
        resid = float((a_dev @ x - rhs).abs().max())
        bwd = resid / (float(a_dev.abs().sum(dim=1).max()) * float(x.abs().max()))
        hbm, hbm_src = hbm_peak_gbs()
        sbytes = n * (n - 1) * 8  # L's strict lower triangle, read by both sweeps
        solve = {"ms": solve_ms, "nrhs": 1, "algorithmic_bytes": sbytes,
                 "hbm_achieved_gbs": sbytes / (solve_ms / 1e3) / 1e9, "hbm_peak_gbs": hbm, "peak_source": hbm_src,
                 "hbm_frac": sbytes / (solve_ms / 1e3) / 1e9 / hbm, "backward_error": bwd,
                 "kernels": "block_prep_kernel + fwd_sweep_kernel + block_diag_kernel + bwd_sweep_kernel"}

    # end to end through the public API: numpy in (pinned) -> Factorization out
    # A (single GPU: the 256-row block rows of its lower trapezoid, rcp_factor_host) + Omega;
    # L: the block rows of its lower trapezoid, then perm/D/pattern
    trap = sum((min(n, i0 + 256) - i0) * min(n, i0 + 256) for i0 in range(0, n, 256)) * 8
    h2d = (trap if world == 1 else n * n * 8) + P * n * 8
    d2h = trap + n * (8 + 8 + 8 + 1)
    e2e_times = []
    for it in range(1 + max(1, args.e2e_steps)):  # first call untimed: pinned host buffers get allocated
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        if world == 1:
            f = api.factor(a_pin.numpy(), cfg)
        else:
            f = rdist.factor_distributed(a_pin.numpy() if rank == 0 else None, cfg)
        if f is not None:
            _ = f.L[-1, 0]
        if it > 0:
            e2e_times.append(time.perf_counter() - t0)
        del f
    te = torch.tensor([statistics.median(e2e_times)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_val = flops / float(te.item()) / 1e9

    if rank != 0:
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            del out, ws
            torch.cuda.empty_cache()
            if load_reference() is not None:
                res = ref_sample(a_host, args, max_panels=1, skip_panels=0)
                kind, what = "reference", "the unmodified reference randldl (oracle/_ref)"
            else:
                res = cpu_sample(a_host, args, budget_s=args.cpu_seconds)
                kind, what = "port", "oracle port of the reference algorithm"
            cv = sum(res["works"]) / sum(res["times"]) / 1e9
            cpu = {"value": cv, "unit": "GFLOP/s", "cores": cores_used(), "kind": kind,
                   "sample": (f"{what} (numpy {np.__version__}/OpenBLAS), first "
                              f"{res['panels']} panel(s) of the same n={n} matrix (columns 0..{res['k_done']}), "
                              f"{sum(res['times']):.1f} s; value = sum (n-j)^2 over eliminated columns / panel time; "
                              f"setup {res['t_setup']:.1f} s excluded; CPU {cpu_model()}")}
        except MemoryError:
            cpu = {"value": None, "unit": "GFLOP/s", "cores": cores_used(), "kind": "port",
                   "sample": "host out of memory for the n=32768 oracle sample"}
    achieved = schur_flops / (schur_ms / 1e3) / 1e12 if schur_ms > 0 else None
    # the trailing update is schur_ws2_kernel (N > 1: each rank's share of its supertiles)
    schur_name = "schur_ws2_kernel"
    schur_key = schur_name if args.workload == "c3" else f"{schur_name}@{args.workload}"
    line = {
        "metric": metric_name(args), "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms_max, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded numpy Philox type6; Omega from Philox(seed))",
        "config": cfg_dict(args, world),
        "pct_fp64_peak": 100.0 * value / (world * FP64_PEAK_GFLOPS),
        "fp64_peak": {"value": FP64_PEAK_GFLOPS, "unit": "GFLOP/s", "source": FP64_PEAK_SRC},
        "roofline": {"bound": "tensor", "kernel": schur_name + " (trailing Schur update, DMMA.8x8x4)",
                     "achieved": achieved, "peak": FP64_PEAK_GFLOPS / 1e3, "unit": "TFLOP/s",
                     "frac": (achieved / (FP64_PEAK_GFLOPS / 1e3)) if achieved else None,
                     "traffic": ncu_traffic(schur_key),
                     "traffic_launch": ncu_traffic(schur_key, detail=True),
                     "algorithmic": "sum over panels of t*m*(m+1) flops (lower-triangle rank-t update) + 2*P*t*m "
                                    "for the sketch-correction tiles the same kernel runs (single GPU)"
                                    + (" (rank 0's share of the tiles; achieved over its Schur time)" if world > 1
                                       else ""),
                     "share_of_step": schur_ms / (ms * args.steps) if ms > 0 else None,
                     "panel_share_of_step": panel_ms / (ms * args.steps) if ms > 0 else None},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_val, "unit": "GFLOP/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "path": ("paper_1710_00125_b200.factor" if world == 1 else "paper_1710_00125_b200.dist.factor_distributed")
                        + "(numpy array in pinned memory) -> Factorization"},
        "gpu_launches": int(stats.get("n_launches", 0)) * args.steps,
        "clocks": clocks,
        "factor_stats": {k: stats.get(k) for k in ("n_panels", "n_steps", "n_2x2", "recompute_count", "rho_cheap",
                                                   "max_multiplier", "t_panel_ms", "t_schur_ms")},
        "solve_backward_error": bwd,
        "solve": solve,
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- C5 (batched)
C5_N, C5_B, C5_P = 256, 16, 24


def c5_cfg(args, world):
    return {"workload": (f"C5 batched: {args.count} symmetrised N(0,1) n={C5_N} matrices, every 10th scaled "
                         f"D A D with D = diag(10^U(-6,6)) and re-mirrored; b=q={C5_B}, P=b+8={C5_P}; "
                         f"sharded by matrix over {world} GPU(s)"),
            "count": args.count, "n": C5_N, "b": C5_B, "q": C5_B, "p_sketch": C5_P, "oversampling": C5_P - C5_B,
            "parallelism": f"shard-by-matrix x{world}",
            "l2": f"inputs {args.count * C5_N * C5_N * 8 / 1e9:.1f} GB >> 126 MB L2 (no flush needed)"}


def c5_host_member(i: int, seed: int) -> np.ndarray:
    from paper_1710_00125_b200 import gallery
    return gallery.scaled_member(C5_N, seed + i, scaled=(i % 10 == 0))


def c5_factor_fn(seed: int):
    """CPU factor() of one C5 member: the unmodified reference (oracle/_ref/randldl) when shipped,
    else the oracle port.  Returns (callable, kind)."""
    randldl = load_reference()
    if randldl is not None:
        cfg = randldl.FactorConfig(strategy="rcp", b=C5_B, q=C5_B, p=C5_P, seed=seed)
        return (lambda a: randldl.factor(a, cfg)), "reference"
    from oracle.rcp_oracle import OracleConfig, oracle_factor
    ocfg = OracleConfig(p=C5_P, b=C5_B, q=C5_B, seed=seed)
    return (lambda a: oracle_factor(a, ocfg)), "port"


def c5_cpu_sample(args, budget_s: float, max_count: int | None = None):
    fn, kind = c5_factor_fn(args.seed)
    t_total, done = 0.0, 0
    while True:
        a = c5_host_member(done, args.seed)
        t0 = time.perf_counter()
        fn(a)
        t_total += time.perf_counter() - t0
        done += 1
        if (max_count is not None and done >= max_count) or (max_count is None and t_total >= budget_s):
            break
    return done, t_total, kind


def _c5_worker(job):
    seed, idx = job
    fn, _ = c5_factor_fn(seed)
    for i in idx:
        fn(c5_host_member(i, seed))
    return len(idx)


def run_reference_c5(args, rank: int):
    """All host cores (one process per core, OMP/BLAS threads 1), C5 members split across them."""
    if rank != 0:
        return
    import multiprocessing as mp
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"
    cores = os.cpu_count() or 1
    per_core = 4
    ctx = mp.get_context("spawn")
    with ctx.Pool(cores) as pool:
        def one_step(base):
            jobs = [(args.seed, list(range(base + c * per_core, base + (c + 1) * per_core))) for c in range(cores)]
            t0 = time.perf_counter()
            done = sum(pool.map(_c5_worker, jobs))
            return done, time.perf_counter() - t0
        for w in range(max(1, args.warmup)):
            one_step(0)
        steps = [one_step(0) for _ in range(args.steps)]
    cnt = sum(c for c, _ in steps)
    tsum = sum(t for _, t in steps)
    value = cnt * C5_N ** 3 / 3.0 / tsum / 1e9
    kind = c5_factor_fn(args.seed)[1]
    line = {
        "impl": "reference", "metric": metric_name(args), "value": value, "unit": "GFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tsum / len(steps),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded numpy Philox C5 members)", "config": c5_cfg(args, args.gpus),
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": cores, "kind": kind,
                         "sample": f"{'reference randldl (oracle/_ref)' if kind == 'reference' else 'oracle port'} "
                                   f"factor() on {cores * per_core} C5 members per step, {cores} processes x 1 BLAS "
                                   f"thread; CPU {cpu_model()}"},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_b200_c5(args, rank: int, world: int, local_rank: int):
    import torch
    import torch.distributed as dist

    from paper_1710_00125_b200 import api, batched, gallery

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    count = args.count // world + (1 if rank < args.count % world else 0)
    cfg = api.FactorConfig(strategy="rcp", b=C5_B, q=C5_B, p=C5_P, seed=args.seed)
    a = torch.empty(count, C5_N, C5_N, dtype=torch.float64, device=dev)
    chunk = 4096
    for c0 in range(0, count, chunk):
        c1 = min(count, c0 + chunk)
        a[c0:c1] = gallery.c5_batch_device(c1 - c0, C5_N, seed=args.seed + 1000 * rank + c0, device=dev)
    normals = torch.from_numpy(batched.normal_stream(cfg, C5_N)).to(dev)
    ws = torch.empty(batched.batched_workspace_bytes(C5_N, cfg), dtype=torch.uint8, device=dev)
    out = None
    for _ in range(max(3, args.warmup)):
        out = batched.factor_batched_device(a, cfg, normals=normals, workspace=ws, out=out, check=False)
    torch.cuda.synchronize()
    bad = int((out.stats["status"] != 0).sum())
    clk = ClockSampler(local_rank)
    clk.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        out = batched.factor_batched_device(a, cfg, normals=normals, workspace=ws, out=out, check=False)
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    flops = args.count * C5_N ** 3 / 3.0
    value = flops / (ms_max / 1e3) / 1e9
    rec = out.stats
    recomputes = int(rec["recompute_count"].sum())

    # solve check on the first matrices (batched solve kernel)
    nchk = min(count, 256)
    rhs = torch.randn(nchk, C5_N, dtype=torch.float64, device=dev)
    sub = batched.BatchedDeviceFactorization(out.perm[:nchk], out.L[:nchk], out.d_diag[:nchk], out.d_off[:nchk],
                                             out.pattern[:nchk], out.stats[:nchk])
    x, _ = batched.solve_batched_device(sub, rhs)
    ax = torch.bmm(a[:nchk], x[:, :, None])[:, :, 0]
    bwd = float(((ax - rhs).abs().amax(dim=1) / (a[:nchk].abs().sum(dim=2).amax(dim=1) * x.abs().amax(dim=1))).max())

    # end to end: pinned host stack in -> factors (perm, L, D, pattern) in pinned host memory out
    ecount = min(count, 8192)
    a_pin = torch.empty(ecount, C5_N, C5_N, dtype=torch.float64, pin_memory=True)
    a_pin.copy_(a[:ecount])
    hout = batched.BatchedDeviceFactorization(
        perm=torch.empty(ecount, C5_N, dtype=torch.int64, pin_memory=True),
        L=torch.empty(ecount, C5_N, C5_N, dtype=torch.float64, pin_memory=True),
        d_diag=torch.empty(ecount, C5_N, dtype=torch.float64, pin_memory=True),
        d_off=torch.empty(ecount, C5_N, dtype=torch.float64, pin_memory=True),
        pattern=torch.empty(ecount, C5_N, dtype=torch.int8, pin_memory=True),
        stats=None)
    e2e_times = []
    for it in range(1 + max(1, args.e2e_steps)):  # first call untimed
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        # chunked upload / factor / download on three streams (batched.factor_batched_host)
        batched.factor_batched_host(a_pin, cfg, normals=normals, workspace=ws, out=hout, check=False,
                                    chunk=args.e2e_chunk)
        torch.cuda.synchronize()
        if it > 0:
            e2e_times.append(time.perf_counter() - t0)
    te = torch.tensor([statistics.median(e2e_times)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_val = world * ecount * C5_N ** 3 / 3.0 / float(te.item()) / 1e9
    h2d = ecount * C5_N * C5_N * 8
    d2h = ecount * (C5_N * C5_N * 8 + C5_N * (8 + 8 + 8 + 1)) + hout.stats.nbytes

    if rank != 0:
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cnt, tc, kind = c5_cpu_sample(args, budget_s=args.cpu_seconds)
        cv = cnt * C5_N ** 3 / 3.0 / tc / 1e9
        cpu = {"value": cv, "unit": "GFLOP/s", "cores": 1, "kind": kind,
               "sample": f"{'reference randldl (oracle/_ref)' if kind == 'reference' else 'oracle port'} factor() on "
                         f"{cnt} C5 members (numpy/OpenBLAS, one process), {tc:.1f} s; CPU {cpu_model()}"}
    hbm_bytes = args.count * C5_N * C5_N * 8 * 2  # read A, write L (algorithmic)
    line = {
        "metric": metric_name(args), "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded torch generator on the device)",
        "config": c5_cfg(args, world),
        "pct_fp64_peak": 100.0 * value / (world * FP64_PEAK_GFLOPS),
        "roofline": {"bound": "tensor", "kernel": "batched_factor_kernel (whole factorization, one CTA per matrix)",
                     "achieved": value / 1e3, "peak": FP64_PEAK_GFLOPS / 1e3, "unit": "TFLOP/s",
                     "frac": value / (world * FP64_PEAK_GFLOPS),
                     "traffic": c5_traffic(args.count // world),
                     "traffic_launch": ncu_traffic("batched_factor_kernel", detail=True),
                     "hbm_achieved_gbs": hbm_bytes / (ms_max / 1e3) / 1e9 / world,
                     "hbm_peak_gbs": hbm_peak_gbs()[0],
                     "algorithmic": "n^3/3 flop and 2 n^2 * 8 B (A in, L out) per matrix"},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_val, "unit": "GFLOP/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "path": f"pinned host stack of {ecount} matrices -> factor_batched_host (chunks of {args.e2e_chunk}, "
                        f"upload/factor/download overlapped) -> perm/L/D/pattern in pinned host memory"},
        "gpu_launches": 3 * args.steps,
        "clocks": clocks,
        "factor_stats": {"failed_matrices": bad, "recompute_count": recomputes,
                         "mean_steps": float(rec["n_steps"].mean())},
        "solve_backward_error": bwd,
    }
    print(json.dumps(line), flush=True)


def relaunch_under_torchrun(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: run this script under torch.distributed.run with N
    processes on this node (rendezvous on 127.0.0.1) and return its exit code."""
    import random
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(random.randint(20000, 40000)),
           str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        (run_reference_c5 if args.workload == "c5" else run_reference)(args, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        (run_b200_c5 if args.workload == "c5" else run_b200)(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
