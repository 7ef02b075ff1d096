"""MR tolerance mode (af_mr_set_numerics(AF_NUMERICS_TOLERANCE): the 2D
full-tile stage kernel with reciprocal estimates and FMA) against the exact
run and the compiled reference's digests: identical leaf sets and per-cycle
leaf/node counts (north_star: flags bit-exact except details within 1e-12
relative of the threshold), conserved fields within 1e-10 relative L1 per
field, dt within 1e-12 relative."""
import os

import numpy as np
import pytest

import digests as D

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def run(kind, level, steps, tol, **kw):
    from paper_1603_05211_b200 import mr as M
    from paper_1603_05211_b200 import uniform as U
    os.environ["AF_MR_FULLK"] = "1"  # full-tile kernel at test sizes too
    try:
        s = M.MRSolver(2, level, M.MROptions(**kw))
        if tol:
            s.set_numerics(True)
        s.build(U.case_fill(kind, 7, level))
        rep = s.run(steps, cfl=0.5)
        out, keys = s.to_uniform(), s.leaves()
        s.close()
    finally:
        del os.environ["AF_MR_FULLK"]
    return rep, out, keys


def rel_l1(a, b):
    return np.abs(a - b).sum(0) / np.maximum(np.abs(b).sum(0), 1e-300)


CASES = {
    "mrlt_noise_L8": (1, 8, 16, dict(epsilon=1e-3, local_time=True, local_time_level_gap=3)),
    "global_epsl_L8": (0, 8, 40, dict(epsilon=1e-3, min_leaf_level=3,
                                      eps_level=[1e-3 * 4.0 ** (l - 8) for l in range(9)])),
}


@pytest.mark.parametrize("case", list(CASES))
def test_tolerance_matches_exact(gpu_lib, case):
    kind, level, steps, kw = CASES[case]
    re_, oe, ke = run(kind, level, steps, False, **kw)
    rt, ot, kt = run(kind, level, steps, True, **kw)
    assert np.array_equal(kt, ke), "leaf set"
    assert np.array_equal(rt.cycles[:, :3], re_.cycles[:, :3]), "leaves/nodes/sub per cycle"
    assert np.allclose(rt.cycles[:, 4], re_.cycles[:, 4], rtol=1e-12, atol=0), "dt"
    d = rel_l1(ot, oe)
    assert d.max() <= 1e-10, d
    assert d.max() > 0.0  # the tolerance kernel ran


@pytest.mark.parametrize("name", ["cfg3_L10", "cfg3_L13"])
def test_tolerance_matches_reference_digest(gpu_lib, name):
    """cfg3's MRLT generator at L=10 and at its own L=13 (one macro-cycle; the
    reference's digests): same leaf set, per-field relative L1 of the
    digest's restricted state within 1e-10."""
    from paper_1603_05211_b200 import mr as M
    from paper_1603_05211_b200 import uniform as U
    path = os.path.join(HERE, "golden", f"digest_{name}.npz")
    if not os.path.exists(path):
        pytest.skip("digest missing")
    g = np.load(path, allow_pickle=False)
    L = int(g["level"])
    os.environ["AF_MR_FULLK"] = "1"
    try:
        s = M.MRSolver(2, L, M.MROptions(epsilon=float(g["eps"]), min_leaf_level=int(g["min_leaf"]),
                                         local_time=bool(g["local_time"]),
                                         local_time_level_gap=int(g["gap"])))
        s.set_numerics(True)
        s.build(U.case_fill(int(g["kind"]), int(g["seed"]), L))
        rep = s.run(int(g["steps"]), cfl=float(g["cfl"]))
        keys, out = s.leaves(), s.to_uniform()
        s.close()
    finally:
        del os.environ["AF_MR_FULLK"]
    assert D.keys_sha(keys) == str(g["keys_sha"]), "leaf set"
    assert np.array_equal(rep.cycles[:, 0].astype(np.int64), g["cycles"][:, 0]), "leaves per cycle"
    c = D.coarse(out, 2, L, int(g["coarse_level"]))
    d = rel_l1(c, g["coarse"])
    assert d.max() <= 1e-10, d
