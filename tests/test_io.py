"""Formats and compare path either side of the hot path:
AFSN snapshots (byte-identical with the reference's reader/writer, and its
IoError texts), restrict_to_level (bit-exact), l1_error (round-off) and the
MRTree::dump text of the device tree (identical to the reference's)."""
import os

import numpy as np
import pytest

from test_oracle import bits


def _state(dim, level, seed):
    rng = np.random.default_rng(seed)
    q = rng.uniform(0.1, 2.0, size=(1 << (dim * level), 5))
    if dim == 2:
        q[:, 3] = 0.0
    q[::7, 1] = -0.0
    return q


@pytest.mark.parametrize("dim,level", [(2, 5), (3, 3)])
def test_snapshot_round_trip_matches_reference(gpu_lib_cpu, oracle, tmp_path, dim, level):
    from paper_1603_05211_b200 import io
    q = _state(dim, level, 7)
    a = str(tmp_path / "a.afsn")
    io.write_snapshot(a, q, dim, level, gamma=1.4, time=0.125, origin=-2.0, extent=4.0)
    s = io.read_snapshot(a)
    assert (s.dim, s.level, s.gamma, s.time, s.origin, s.extent) == (dim, level, 1.4, 0.125,
                                                                      -2.0, 4.0)
    assert np.array_equal(bits(s.state), bits(q))
    if oracle.available("ref"):
        b = str(tmp_path / "b.afsn")
        assert oracle.ref_snapshot_copy(a, b) is None
        assert open(a, "rb").read() == open(b, "rb").read()


def test_snapshot_errors_match_reference(gpu_lib_cpu, oracle, tmp_path):
    from paper_1603_05211_b200 import io
    from paper_1603_05211_b200.errors import IoError
    bad = str(tmp_path / "bad.afsn")
    open(bad, "wb").write(b"NOPE" + bytes(60))
    q = _state(2, 3, 1)
    good = str(tmp_path / "good.afsn")
    io.write_snapshot(good, q, 2, 3)
    trunc = str(tmp_path / "trunc.afsn")
    open(trunc, "wb").write(open(good, "rb").read()[:-8])
    for path in (bad, trunc, str(tmp_path / "missing.afsn")):
        with pytest.raises(IoError) as e:
            io.read_snapshot(path)
        if oracle.available("ref"):
            assert str(e.value) == oracle.ref_snapshot_copy(path, str(tmp_path / "x.afsn"))


@pytest.mark.gpu
@pytest.mark.parametrize("dim,level,target", [(2, 7, 3), (3, 5, 2), (2, 4, 4)])
def test_restrict_and_l1_match_reference(gpu_lib, oracle, dim, level, target):
    from paper_1603_05211_b200 import io
    if not oracle.available("ref"):
        pytest.skip("reference build not present")
    q = _state(dim, level, 3)
    r = io.restrict_to_level(q, dim, level, target)
    assert np.array_equal(bits(r), bits(oracle.ref_restrict(q, dim, level, target)))
    sol = _state(dim, target, 4)
    ours = io.l1_error(sol, dim, target, q, level, extent=2.0)
    ref = oracle.ref_l1_error(sol, dim, target, q, level, extent=2.0)
    assert np.allclose(ours, ref, rtol=1e-12, atol=0.0)


@pytest.mark.gpu
@pytest.mark.parametrize("kind,level,steps,kw", [
    (0, 6, 10, dict(eps=1e-3, min_leaf=2)),
    (2, 4, 3, dict(eps=1e-3, cfl=0.4)),
    (1, 6, 8, dict(eps=1e-3, local_time=True)),
])
def test_mr_dump_matches_reference(gpu_lib, oracle, tmp_path, kind, level, steps, kw):
    """MRTree::dump (mr_tree.cpp:623-641) of the device tree after a run equals
    the reference's dump text (every node, value and status)."""
    from test_mr_gpu import ref_mr
    from paper_1603_05211_b200 import mr as M
    from paper_1603_05211_b200 import uniform as U
    if not oracle.available("ref"):
        pytest.skip("reference build not present")
    dim = 3 if kind >= 2 else 2
    init = U.case_fill(kind, 90 + level, level)
    cfl = kw.pop("cfl", 0.5)
    s = M.MRSolver(dim, level, M.MROptions(epsilon=kw["eps"], min_leaf_level=kw.get("min_leaf", 0),
                                           local_time=kw.get("local_time", False)),
                   scheme=U.SchemeConfig(limiter=1))
    s.build(init)
    s.run(steps, cfl=cfl)
    ours = s.dump()
    s.close()
    path = str(tmp_path / "ref.dump")
    p = oracle.make_params(dim, level, steps, cfl=cfl, limiter=1, eps=kw["eps"],
                           min_leaf_level=kw.get("min_leaf", 0),
                           local_time=kw.get("local_time", False))
    oracle.mr_run("ref", p, init, dump_path=path)
    assert ours == open(path).read()


def test_rates_match_reference():
    """Paper §3 rates (metrics.cpp:91-132) through af_rates_compute against the
    reference's rates(): same values bit for bit, same DivisionDomain texts.
    Host arithmetic: runs without a GPU."""
    from oracle import oracle as O
    from paper_1603_05211_b200 import io
    from paper_1603_05211_b200.errors import DivisionDomain
    if not O.available("ref"):
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(5)
    for _ in range(20):
        ad = dict(wall_seconds=float(rng.uniform(0.1, 9)), sum_cells=float(rng.integers(1, 10**9)),
                  sum_leaves=float(rng.integers(1, 10**8)), n_steps=int(rng.integers(1, 5000)),
                  l1_rho=float(rng.uniform(1e-6, 1e-2)))
        fv = dict(wall_seconds=float(rng.uniform(0.1, 9)), sum_cells=0.0, sum_leaves=0.0,
                  n_steps=int(rng.integers(1, 5000)), l1_rho=float(rng.uniform(1e-6, 1e-2)))
        n_c = float(4 ** int(rng.integers(3, 12)))
        ref, err = O.rates(ad, fv, n_c)
        assert err is None
        got = io.rates(ad, fv, n_c)
        for k, v in ref.items():
            assert got[k] == v, k
    base = dict(wall_seconds=1.0, sum_cells=1e6, sum_leaves=5e5, n_steps=10, l1_rho=1e-3)
    for bad_ad, bad_fv, n_c in ((base, dict(base, n_steps=0), 1e4), (base, base, 0.0),
                                (base, dict(base, wall_seconds=0.0), 1e4),
                                (dict(base, n_steps=0), base, 1e4),
                                (base, dict(base, l1_rho=0.0), 1e4),
                                (dict(base, sum_leaves=0.0), base, 1e4)):
        _, err = O.rates(bad_ad, bad_fv, n_c)
        assert err is not None
        with pytest.raises(DivisionDomain) as e:
            io.rates(bad_ad, bad_fv, n_c)
        assert str(e.value) == err
