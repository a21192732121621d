"""Time the batched C5 factorization (device-resident inputs)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1710_00125_b200 import FactorConfig, batched, gallery

count = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
n = 256
cfg = FactorConfig(strategy="rcp", b=16, q=16, p=24, seed=0)
a = gallery.c5_batch_device(count, n, seed=1)
normals = torch.from_numpy(batched.normal_stream(cfg, n)).cuda()
ws = torch.empty(batched.batched_workspace_bytes(n, cfg), dtype=torch.uint8, device="cuda")
out = batched.factor_batched_device(a[:16], cfg, normals=normals, workspace=ws)
out = None
bf = batched.factor_batched_device(a, cfg, normals=normals, workspace=ws, check=False)
torch.cuda.synchronize()
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    bf = batched.factor_batched_device(a, cfg, normals=normals, workspace=ws, out=bf, check=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    flops = count * n ** 3 / 3
    print(f"count={count} ms={ms:.2f} GFLOP/s={flops / ms / 1e6:.1f} per-matrix-us={ms * 1e3 / count:.2f}")
st = bf.stats
print("status", np.bincount(st["status"]), "recomputes", np.bincount(st["recompute_count"]), "steps", st["n_steps"].mean())
import os
if os.environ.get("RCP_BATCH_PROF") == "1":
    tot = st["mults"].astype(float) + st["adds"] + st["divs"] + st["comps"]
    for nm in ("mults", "adds", "divs", "comps"):
        print(nm, "mean cycles", st[nm].mean(), "share", (st[nm] / tot).mean())
