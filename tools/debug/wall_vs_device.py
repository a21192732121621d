"""Host wall time of factor_device vs the device time it reports (host overhead check)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1710_00125_b200 import api, gallery
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
b = int(sys.argv[2]) if len(sys.argv) > 2 else 64
A = torch.from_numpy(gallery.type6(n, 0)).cuda()
cfg = api.FactorConfig(b=b, q=b, p=b + 16, seed=0)
omega = torch.from_numpy(np.random.Generator(np.random.Philox(0)).standard_normal((cfg.p, n))).cuda()
ws = torch.empty(api.workspace_bytes(n, cfg), dtype=torch.uint8, device="cuda")
out = None
for r in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = api.factor_device(A, cfg, omega=omega, workspace=ws, out=out)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    print(f"n={n} wall {wall:.1f} ms  device {out.stats['t_factor_ms']:.1f} ms  panels {out.stats['n_panels']} launches {out.stats['n_launches']}")
