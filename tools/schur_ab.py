"""Device time of one factorization split by kernel (device %globaltimer stamps):
    python tools/schur_ab.py [c2|c3|c4] [reps]
Run it under RCP_SCHUR_V=1 / 2 (or RCP_B200_LIB=variant.so) to compare trailing-update kernels;
prints perm/L checksums so variants can be checked for identical results."""
import hashlib
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1710_00125_b200 import api, gallery  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
if wl == "c2":
    a = gallery.type6_device(8192, 0) if hasattr(gallery, "type6_device") else torch.from_numpy(gallery.type6(8192, 0)).cuda()
    cfg = api.FactorConfig(strategy="rcp", b=64, q=64, p=74, seed=0)
elif wl == "c1":
    a = torch.from_numpy(gallery.type6(1000, 0)).cuda()
    cfg = api.FactorConfig(strategy="rcp", b=32, q=32, p=42, seed=0)
elif wl == "c4":
    a = torch.from_numpy(gallery.kkt_c4(16000, 4000, 0)).cuda()
    cfg = api.FactorConfig(strategy="rcp", b=64, q=64, p=74, seed=0)
else:
    a = gallery.type6_device(32768, 0) if hasattr(gallery, "type6_device") else torch.from_numpy(gallery.type6(32768, 0)).cuda()
    cfg = api.FactorConfig(strategy="rcp", b=128, q=128, p=144, seed=0)
best = None
for it in range(reps + 1):
    f = api.factor_device(a, cfg)
    torch.cuda.synchronize()
    st = {k: f.stats[k] for k in ("t_factor_ms", "t_panel_ms", "t_schur_ms") if k in f.stats}
    if (it or reps == 0) and (best is None or st["t_factor_ms"] < best["t_factor_ms"]):
        best = st
h = hashlib.sha1()
h.update(f.perm.cpu().numpy().tobytes())
lsum = float(f.L.sum().item())
h2 = hashlib.sha1(f.d_diag.cpu().numpy().tobytes()).hexdigest()[:12]
b = torch.from_numpy(gallery.rhs(a.shape[0], 1)).cuda()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
x = api.solve_device(f, b)
e0.record()
x = api.solve_device(f, b)
e1.record()
torch.cuda.synchronize()
best["t_solve_ms"] = e0.elapsed_time(e1)
print(json.dumps({"workload": wl, **best, "perm_sha1": h.hexdigest()[:12], "L_sum": repr(lsum), "d_sha1": h2}), flush=True)
