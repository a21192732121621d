"""Run a few factorizations of one config (for ncu / timing breakdowns)."""
import argparse, json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_1710_00125_b200 import api, gallery

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8192); ap.add_argument("--b", type=int, default=64)
ap.add_argument("--p", type=int, default=74); ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
A = torch.from_numpy(gallery.type6(a.n, 0)).cuda()
cfg = api.FactorConfig(b=a.b, q=a.b, p=a.p, seed=0)
out = None
for r in range(a.reps):
    out = api.factor_device(A, cfg, out=out)
    torch.cuda.synchronize()
    s = out.stats
    print(json.dumps({k: s[k] for k in ("t_factor_ms", "t_panel_ms", "t_schur_ms", "n_panels", "n_steps", "n_launches", "panel_prof_ms")}))
