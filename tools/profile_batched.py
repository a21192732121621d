"""Per-phase SM-cycle profile of the batched C5 kernel (build with -DRCP_BATCH_PROF=1; the
per-matrix op-counter fields then hold cycles).  Usage:
  RCP_B200_LIB=paper_1710_00125_b200/librcp_bprof.so python tools/profile_batched.py [count]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

from paper_1710_00125_b200 import api, batched, gallery

count = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
n, b, p = 256, 16, 24
cfg = api.FactorConfig(strategy="rcp", b=b, q=b, p=p, seed=0)
a = gallery.c5_batch_device(count, n, seed=1000, device="cuda")
normals = torch.from_numpy(batched.normal_stream(cfg, n)).cuda()
ws = torch.empty(batched.batched_workspace_bytes(n, cfg), dtype=torch.uint8, device="cuda")
for it in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = batched.factor_batched_device(a, cfg, normals=normals, workspace=ws, check=False)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
s = out.stats
names = ("qrcp (guard+QRCP+replay)", "sbkp steps", "L store + trailing + sketch corr", "validate+sketch+outputs")
tot = sum(float(np.mean(s[k].astype(np.float64))) for k in ("mults", "adds", "divs", "comps"))
print(f"count {count}: {dt * 1e3:.1f} ms, {dt / count * 1e6:.2f} us/matrix wall; cycles/matrix {tot:.0f}")
for nm, k in zip(names, ("mults", "adds", "divs", "comps")):
    v = float(np.mean(s[k].astype(np.float64)))
    print(f"  {nm:36s} {v:12.0f} cyc  {100 * v / tot:5.1f}%")
