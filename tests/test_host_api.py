"""Host-side logic of the drop-in API (no GPU needed)."""

import numpy as np
import pytest

from paper_1710_00125_b200 import api, gallery


@pytest.mark.parametrize(
    "kwargs",
    [{"p": 0}, {"b": 0}, {"q": 3, "b": 8}, {"q": 8, "b": 8, "p": 5}, {"robust_r": -1},
     {"strategy": "newton"}, {"track_growth": "sometimes"}],
)
def test_config_validation_matches_reference(kwargs):
    # reference test_factor.py:287-302
    with pytest.raises(ValueError):
        api.FactorConfig(**kwargs)


def test_config_accepts_enum_and_string():
    assert api.FactorConfig(strategy=api.Strategy.RCP).strategy is api.Strategy.RCP
    assert api.FactorConfig(strategy="rcp", b=8, q=8, p=8).q == 8


def test_cfg_plus_overrides_rejected():
    with pytest.raises(ValueError, match="not both"):
        api.factor(np.eye(3), cfg=api.FactorConfig(), b=1)


@pytest.mark.parametrize("a", [np.zeros((0, 0)), np.zeros((2, 3))], ids=["empty", "rectangular"])
def test_shape_validation_before_device(a):
    with pytest.raises(ValueError):
        api.factor(a, strategy="rcp", b=4, q=4, p=4)


def test_factor_robust_prerequisites():
    with pytest.raises(ValueError, match="rcp"):
        api.factor_robust(np.eye(3), strategy="bkpp")
    with pytest.raises(ValueError, match="robust_r"):
        api.factor_robust(np.eye(3), strategy="rcp", robust_r=0)


def test_out_of_scope_strategies_are_explicit():
    # the batched kernel runs rcp only; bkpp / bbk run on the single-matrix engine
    with pytest.raises(ValueError, match="rcp"):
        api._check_supported(api.FactorConfig(strategy="bkpp"), batched=True)


def test_strategy_reaches_the_c_config():
    c = api._native_config(api.FactorConfig(strategy="bkpp", b=8, q=1, p=5))
    assert (c.p, c.b, c.q, c.robust_r, c.strategy) == (5, 8, 1, 1, 1)
    assert api._native_config(api.FactorConfig()).strategy == 0


def test_blocks_from_arrays_roundtrip():
    dd = np.array([1.0, 2.0, 3.0, 4.0, 5.0])
    off = np.array([0.0, 7.0, 0.0, 0.0, 0.0])
    pat = np.array([0, 1, 2, 0, 3], dtype=np.int8)
    blocks = api._blocks_from_arrays(dd, off, pat)
    assert [b.shape[0] for b in blocks] == [1, 2, 1, 1]
    assert np.array_equal(blocks[1], [[2.0, 7.0], [7.0, 3.0]])
    bd = api.BlockDiag(blocks)
    assert bd.dim == 5 and bd.max_abs() == 7.0


def test_normal_stream_continues_like_reference_generator():
    # sketch.py:63-84: one generator, first (p x n) then each recompute (p x m)
    s = api._NormalStream(5)
    first = s.first(3, 7)
    ref = np.random.Generator(np.random.Philox(5))
    assert np.array_equal(first, ref.standard_normal((3, 7)))
    import ctypes
    buf = (ctypes.c_double * 12)()
    assert s.cfunc(None, 3, 4, buf) == 0
    assert np.array_equal(np.frombuffer(buf, dtype=np.float64).reshape(3, 4), ref.standard_normal((3, 4)))


def test_type6_chunked_equals_one_shot():
    n = 4100  # above the one-shot threshold
    a = gallery.type6(n, 3, chunk_rows=333)
    g = np.random.Generator(np.random.Philox(3)).standard_normal((n, n))
    ref = np.tril(g) + np.tril(g, -1).T
    assert np.array_equal(a, ref)


def test_scaled_member_is_exactly_symmetric():
    a = gallery.scaled_member(64, 10, True)
    assert np.array_equal(a, a.T)


def test_batched_host_validates_before_device():
    """factor_batched_host rejects bad stacks with the reference's ValueError before any device work."""
    import torch
    from paper_1710_00125_b200 import batched
    cfg = api.FactorConfig(strategy="rcp", b=16, q=16, p=24, seed=0)
    with pytest.raises(ValueError, match="stack"):
        batched.factor_batched_host(torch.zeros(4, 8, 9, dtype=torch.float64), cfg)
    with pytest.raises(ValueError, match="float64"):
        batched.factor_batched_host(torch.zeros(4, 8, 8, dtype=torch.float32), cfg)
    with pytest.raises(ValueError, match="at least one row"):
        batched.factor_batched_host(torch.zeros(4, 0, 0, dtype=torch.float64), cfg)


def test_shard_range_partitions_the_batch():
    from paper_1710_00125_b200 import shard_range
    for count in (0, 1, 7, 65536, 65537):
        for world in (1, 2, 3, 8):
            spans = [shard_range(count, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == count
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [e - s for s, e in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 3, 3)


def test_foreign_factor_config_is_accepted():
    """The reference's own FactorConfig objects (str-Enum fields) convert to this package's."""
    import enum
    from dataclasses import dataclass

    from paper_1710_00125_b200 import api

    class S(str, enum.Enum):
        RCP = "rcp"

    class G(str, enum.Enum):
        FULL = "full"

    @dataclass
    class Foreign:
        strategy: S = S.RCP
        p: int = 7
        b: int = 4
        q: int = 4
        seed: int = 3
        robust_r: int = 2
        track_growth: G = G.FULL
        audit_sketch: bool = True

    c = api._config(Foreign(), {})
    assert isinstance(c, api.FactorConfig)
    assert (c.strategy, c.p, c.b, c.q, c.seed, c.robust_r) == (api.Strategy.RCP, 7, 4, 4, 3, 2)
    assert c.track_growth is api.GrowthTracking.FULL and c.audit_sketch
