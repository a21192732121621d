"""Time the device solve (rcp_solve: two persistent triangular sweeps) on a factored matrix.

    python tools/solve_timing.py --n 32768 --b 128 --p 144 [--nrhs 1]
Prints ms per solve and the achieved HBM rate on the algorithmic bytes (L's strict lower
triangle read twice: n(n-1) * 8 bytes)."""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1710_00125_b200 import api, gallery  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32768)
ap.add_argument("--b", type=int, default=128)
ap.add_argument("--p", type=int, default=144)
ap.add_argument("--nrhs", type=int, default=1)
ap.add_argument("--reps", type=int, default=10)
args = ap.parse_args()
n = args.n
a = torch.from_numpy(gallery.type6(n, 0)).cuda()
f = api.factor_device(a, api.FactorConfig(strategy="rcp", b=args.b, q=args.b, p=args.p, seed=0))
shape = (n,) if args.nrhs == 1 else (n, args.nrhs)
rhs = torch.from_numpy(np.random.Generator(np.random.Philox(1)).standard_normal(shape)).cuda()
ws = torch.empty(int(api._native.load().rcp_solve_workspace_bytes(n, args.nrhs)), dtype=torch.uint8, device="cuda")
for _ in range(3):
    x, _ = api.solve_device(f, rhs, workspace=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(args.reps):
    x, _ = api.solve_device(f, rhs, workspace=ws)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / args.reps
x2 = x.reshape(n, -1)
r = (a @ x2 - rhs.reshape(n, -1)).abs().max().item() / (a.abs().sum(1).max().item() * x2.abs().max().item())
gbs = n * (n - 1) * 8 / (ms * 1e-3) / 1e9
print(f"solve n={n} nrhs={args.nrhs}: {ms:.3f} ms/solve, {gbs:.0f} GB/s on n(n-1)*8 B, backward error {r:.2e}")
