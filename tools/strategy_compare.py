"""Time the three pivoting strategies on the same B200 panel engine (SURVEY.md section 8 row f4:
the paper's strategy comparison).  Device-resident type-6 input; one warm-up, then `--reps` timed
factorizations each; prints one JSON line per strategy (time, GFLOP/s in the n^3/3 model, 2x2
count, growth rho_cheap, max multiplier)."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1710_00125_b200 import api, gallery  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32768)
ap.add_argument("--b", type=int, default=128)
ap.add_argument("--p", type=int, default=144)
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
A = torch.from_numpy(gallery.type6(args.n, 0)).cuda()
for strategy in ("rcp", "bkpp", "bbk"):
    q = args.b if strategy == "rcp" else 1
    cfg = api.FactorConfig(strategy=strategy, b=args.b, q=q, p=args.p if strategy == "rcp" else 5, seed=0)
    out = api.factor_device(A, cfg)
    torch.cuda.synchronize()
    times = []
    for _ in range(args.reps):
        out = api.factor_device(A, cfg, out=out)
        torch.cuda.synchronize()
        times.append(out.stats["t_factor_ms"])
    ms = float(np.median(times))
    s = out.stats
    print(json.dumps({"strategy": strategy, "n": args.n, "b": args.b, "ms": round(ms, 1),
                      "gflops_n3_over_3": round(args.n ** 3 / 3 / ms / 1e6, 1),
                      "t_panel_ms": round(s["t_panel_ms"], 1), "t_schur_ms": round(s["t_schur_ms"], 1),
                      "n_2x2": s["n_2x2"], "n_steps": s["n_steps"], "rho_cheap": s["rho_cheap"],
                      "max_multiplier": s["max_multiplier"]}), flush=True)
