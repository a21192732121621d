"""Reference CSVs of the strategy-comparison grid (randldl.bench.run, bench.py:205-215), made
by running the REFERENCE in the build container:  python tests/golden/make_grid.py
tests/test_grid.py runs the same configs through paper_1710_00125_b200.grid on the GPU and
compares every non-timing column."""
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from randldl import bench  # noqa: E402

CONFIGS = {
    "grid_default": "strategies = rcp, bkpp, bbk\nfamilies = type6\nsizes = 48, 100\np = 5, 8\ntrials = 2\n",
    "grid_panels": "strategies = rcp\nfamilies = type6\nsizes = 130\np = 20\ntrials = 2\nb = 16\nq = 16\n",
    "grid_full": "strategies = rcp, bkpp\nfamilies = type6\nsizes = 60\np = 6\ntrials = 1\ntrack_growth = full\n",
}

if __name__ == "__main__":
    for name, text in CONFIGS.items():
        (HERE / "grid" / f"{name}.cfg").write_text(text)
        cfg = bench.parse_config(text)
        cfg.out = str(HERE / "grid" / f"{name}.csv")
        recs = bench.run(cfg)
        print(name, len(recs), "cells,", sum(r.error is not None for r in recs), "errors")
