"""bench.py command-line contract on CPU: `--gpus N` outside torchrun re-launches itself under
torch.distributed.run with N processes on 127.0.0.1; workloads set their own sizes."""

import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _bench():
    if str(ROOT) not in sys.path:
        sys.path.insert(0, str(ROOT))
    import bench
    return bench


def test_gpus_n_relaunches_under_torchrun(monkeypatch):
    bench = _bench()
    seen = {}

    def fake_call(cmd):
        seen["cmd"] = cmd
        return 0

    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(bench.subprocess, "call", fake_call)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2", "--warmup", "3"])
    with pytest.raises(SystemExit) as ex:
        bench.main()
    assert ex.value.code == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--nnodes=1" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-6:] == ["--gpus", "4", "--steps", "2", "--warmup", "3"]


@pytest.mark.parametrize("wl,n,b,p", [("c2", 8192, 64, 74), ("c3", 32768, 128, 144), ("c4", 20000, 64, 74)])
def test_workload_defaults(monkeypatch, wl, n, b, p):
    bench = _bench()
    monkeypatch.setattr(sys, "argv", ["bench.py", "--workload", wl])
    a = bench.parse()
    assert (a.n, a.b, a.p) == (n, b, p)
    assert ("C3" in bench.workload_name(a)) == (wl == "c3")
    if wl == "c3":
        assert bench.metric_name(a) == bench.METRIC


def test_hbm_peak_from_measured_peaks():
    bench = _bench()
    v, src = bench.hbm_peak_gbs()
    assert v > 1000 and isinstance(src, str)
