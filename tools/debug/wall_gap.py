"""Wall (host) time of factor_device vs its internal device time at C3 (the bench's events also
see the host-side gaps between calls)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1710_00125_b200 import api, gallery
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
A = torch.from_numpy(gallery.type6(n, 0)).cuda()
cfg = api.FactorConfig(b=128, q=128, p=144, seed=0)
om = torch.from_numpy(np.random.Generator(np.random.Philox(0)).standard_normal((144, n))).cuda()
ws = torch.empty(api.workspace_bytes(n, cfg), dtype=torch.uint8, device="cuda")
out = api.factor_device(A, cfg, omega=om, workspace=ws)
for rep in range(3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    out = api.factor_device(A, cfg, omega=om, workspace=ws, out=out)
    e1.record(); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"wall {1e3*(t1-t0):.1f} ms  events {e0.elapsed_time(e1):.1f} ms  internal {out.stats['t_factor_ms']:.1f} ms")
