"""CPU tests: the plain-C MR restatement (oracle/af_oracle_mr.c) is pinned
bit for bit against the committed MR golden fixtures (made by the compiled
reference, tests/golden/make_golden.py) and, where the reference sources are
present, against the compiled reference itself (oracle/_ref) on global and
local-time-stepping runs, level thresholds, every boundary kind, AUSMDV,
3D, and both error paths (NonPhysicalState, RegisterMismatch-free LT).

Compared: to_uniform(L) of the final tree, the sorted leaf keys, every
per-cycle record (leaves, nodes incl. virtual, sub, top, updates), the dt
history, max_cfl, fallbacks, the exception text, and MRTree::dump()."""
import glob
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = sorted(glob.glob(os.path.join(HERE, "golden", "mr_*.npz")))


def bits(a):
    b = np.ascontiguousarray(a, dtype=np.float64).view(np.uint64).copy()
    b[b == np.uint64(1 << 63)] = 0  # -0 == +0
    return b


def eps_levels(eps, L, d):
    return [eps * 2.0 ** (d * (l - L)) for l in range(L + 1)]


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_mr_port_matches_golden(oracle, path):
    g = np.load(path)
    kind, level = int(g["kind"]), int(g["level"])
    dim = 3 if kind >= 2 else 2
    init = oracle.case_fill(kind, int(g["seed"]), level)
    p = oracle.make_params(dim, level, int(g["steps"]), cfl=float(g["cfl"]),
                           fixed_dt=float(g["fixed_dt"]), limiter=int(g["limiter"]),
                           bc=[int(x) for x in g["bc"]], eps=float(g["eps"]),
                           eps_level=g["eps_level"] if int(g["has_eps_level"]) else None,
                           min_leaf_level=int(g["min_leaf"]), local_time=int(g["local_time"]),
                           lt_gap=int(g["gap"]))
    out, keys, cyc, dts, res = oracle.mr_run("port", p, init)
    assert res["err_kind"] == 0, res["err"]
    assert np.array_equal(keys, g["keys"])
    assert np.array_equal(cyc, g["cycles"])
    assert np.array_equal(bits(dts), bits(g["dt"]))
    assert np.array_equal(bits(out), bits(g["out"]))
    assert res["max_cfl"] == float(g["max_cfl"])
    assert res["fallbacks"] == int(g["fallbacks"])


# (kind, seed, level, steps, cfl, fixed_dt, eps, eps_level?, min_leaf, lt, gap, limiter, flux, bc)
CASES = {
    "global_quad_L6": (0, 201, 6, 10, 0.5, 0.0, 1e-3, False, 0, 0, 3, 1, 0, None),
    "global_epsl_min3_L7": (0, 202, 7, 8, 0.5, 0.0, 1e-3, True, 3, 0, 3, 1, 0, None),
    "global_vanalbada_fixed": (0, 203, 6, 8, 0.0, 1e-3, 1e-3, False, 0, 0, 3, 0, 0, None),
    "global_periodic_noise": (1, 204, 6, 6, 0.5, 0.0, 1e-3, False, 2, 0, 3, 1, 0, [1] * 6),
    "global_reflective": (0, 205, 6, 8, 0.5, 0.0, 1e-3, False, 0, 0, 3, 1, 0, [2] * 6),
    "global_mixed_bc_ausmdv": (0, 206, 6, 6, 0.5, 0.0, 1e-3, False, 0, 0, 3, 1, 1,
                               [2, 2, 1, 1, 0, 0]),
    "global_3d_ell": (2, 207, 4, 4, 0.4, 0.0, 1e-3, False, 0, 0, 3, 1, 0, None),
    "global_3d_epsl": (3, 208, 4, 3, 0.4, 0.0, 1e-3, True, 1, 0, 3, 1, 0, None),
    "lt_quad_L6": (0, 209, 6, 16, 0.5, 0.0, 1e-3, False, 0, 1, 3, 1, 0, None),
    "lt_noise_L7_gap2": (1, 210, 7, 8, 0.5, 0.0, 1e-3, False, 0, 1, 2, 1, 0, None),
    "lt_periodic_noise": (1, 211, 6, 12, 0.5, 0.0, 1e-3, False, 0, 1, 3, 1, 0, [1] * 6),
    "lt_reflective_vanalbada": (0, 212, 6, 12, 0.5, 0.0, 1e-3, False, 0, 1, 3, 0, 0, [2] * 6),
    "lt_3d_epsl_gap2": (3, 213, 4, 8, 0.4, 0.0, 1e-3, True, 1, 1, 2, 1, 0, None),
    "global_eps0": (0, 214, 5, 4, 0.5, 0.0, 0.0, False, 0, 0, 3, 1, 0, None),
    "blowup": (0, 215, 6, 20, 3.0, 0.0, 1e-3, False, 0, 0, 3, 1, 0, None),
    "blowup_lt": (0, 216, 6, 20, 3.0, 0.0, 1e-3, False, 0, 1, 3, 1, 0, None),
}


@pytest.mark.parametrize("name", list(CASES))
def test_mr_port_matches_reference_build(oracle, tmp_path, name):
    if not oracle.available("ref"):
        pytest.skip("reference sources not present (GPU box); the golden fixtures cover this")
    kind, seed, level, steps, cfl, fdt, eps, epsl, mleaf, lt, gap, lim, flux, bc = CASES[name]
    dim = 3 if kind >= 2 else 2
    init = oracle.case_fill(kind, seed, level)
    p = oracle.make_params(dim, level, steps, cfl=cfl, fixed_dt=fdt, limiter=lim, bc=bc, eps=eps,
                           eps_level=eps_levels(eps, level, dim) if epsl else None,
                           min_leaf_level=mleaf, local_time=lt, lt_gap=gap, flux=flux)
    da, db = str(tmp_path / "ref.txt"), str(tmp_path / "port.txt")
    a = oracle.mr_run("ref", p, init, dump_path=da)
    b = oracle.mr_run("port", p, init, dump_path=db)
    ra, rb = a[4], b[4]
    assert ra["err"] == rb["err"]
    assert ra["err_kind"] == rb["err_kind"]
    for k in ("steps_done", "n_cycles", "max_cfl", "fallbacks"):
        assert ra[k] == rb[k], k
    assert np.array_equal(a[2], b[2])                  # per-cycle records
    assert np.array_equal(bits(a[3]), bits(b[3]))      # dt history
    if ra["err_kind"] == 0:
        assert np.array_equal(a[1], b[1])              # leaf keys
        assert np.array_equal(bits(a[0]), bits(b[0]))  # to_uniform(L)
        assert open(da).read() == open(db).read()      # MRTree::dump()
