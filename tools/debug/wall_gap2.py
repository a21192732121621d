"""Split the wall time of factor_device into Python and C-call parts (run beside nvidia-smi)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1710_00125_b200 import api, gallery, _native
n = 32768
A = torch.from_numpy(gallery.type6(n, 0)).cuda()
cfg = api.FactorConfig(b=128, q=128, p=144, seed=0)
om = torch.from_numpy(np.random.Generator(np.random.Philox(0)).standard_normal((144, n))).cuda()
ws = torch.empty(api.workspace_bytes(n, cfg), dtype=torch.uint8, device="cuda")
lib = _native.load()
orig = lib.rcp_factor_dist
box = {}
def wrapped(*a):
    t = time.perf_counter(); r = orig(*a); box["c"] = time.perf_counter() - t; return r
lib.rcp_factor_dist = wrapped
out = api.factor_device(A, cfg, omega=om, workspace=ws)
for rep in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = api.factor_device(A, cfg, omega=om, workspace=ws, out=out)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"wall {1e3*(t1-t0):.1f}  C {1e3*box['c']:.1f}  internal {out.stats['t_factor_ms']:.1f}", flush=True)
