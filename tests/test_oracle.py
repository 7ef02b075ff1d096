"""CPU tests: the plain-C restatement (oracle/af_oracle.c) is pinned against
the compiled reference (oracle/_ref) and against the committed golden
fixtures generated from it (tests/golden/make_golden.py)."""
import glob
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = sorted(glob.glob(os.path.join(HERE, "golden", "u*.npz")))


def bits(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = a.view(np.uint64).copy()
    b[b == np.uint64(1 << 63)] = 0  # -0 == +0 (compare ±0 as equal)
    return b


def run_fixture(O, g, kind="port"):
    dim = 3 if int(g["kind"]) >= 2 else 2
    init = O.case_fill(int(g["kind"]), int(g["seed"]), int(g["level"]))
    p = O.make_params(dim, int(g["level"]), int(g["steps"]), cfl=float(g["cfl"]),
                      fixed_dt=float(g["fixed_dt"]), limiter=int(g["limiter"]),
                      bc=[int(x) for x in g["bc"]])
    return O.uniform_run(kind, p, init)


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_port_matches_golden(oracle, path):
    g = np.load(path)
    out, dts, res = run_fixture(oracle, g)
    assert res["err"] == str(g["err"])
    assert res["err_kind"] == int(g["err_kind"])
    if res["err_kind"] == 0:
        assert np.array_equal(bits(out), bits(g["out"]))
        assert np.array_equal(bits(dts), bits(g["dt"]))
        assert res["max_cfl"] == float(g["max_cfl"])
        assert res["max_wave_speed"] == float(g["max_wave_speed"])
        assert res["fallbacks"] == int(g["fallbacks"])


@pytest.mark.parametrize("kind,seed,level,steps,cfl,lim,bc", [
    (0, 101, 6, 25, 0.5, 1, None),
    (1, 102, 6, 15, 0.5, 0, None),
    (0, 103, 5, 10, 0.45, 1, [1, 1, 2, 2, 0, 0]),
    (2, 104, 4, 8, 0.4, 1, None),
    (3, 105, 4, 5, 0.3, 0, [1] * 6),
    (2, 106, 4, 10, 2.5, 1, None),  # blows up: error text must match
])
def test_port_matches_reference_build(oracle, kind, seed, level, steps, cfl, lim, bc):
    if not oracle.available("ref"):
        pytest.skip("reference sources not present (GPU box); golden fixtures cover this")
    dim = 3 if kind >= 2 else 2
    init = oracle.case_fill(kind, seed, level)
    p = oracle.make_params(dim, level, steps, cfl=cfl, limiter=lim, bc=bc)
    a, da, ra = oracle.uniform_run("ref", p, init)
    b, db, rb = oracle.uniform_run("port", p, init)
    assert ra["err"] == rb["err"]
    assert np.array_equal(bits(a), bits(b))
    assert np.array_equal(bits(da), bits(db))
    for k in ("max_cfl", "max_wave_speed", "fallbacks", "steps_done"):
        assert ra[k] == rb[k], k


def test_case_fill_slabs_reassemble(oracle):
    """A slab of the seeded input equals the same rows of the whole domain."""
    for kind, level in ((1, 6), (2, 4)):
        full = oracle.case_fill(kind, 9, level)
        n = 1 << level
        per = full.shape[0] // n
        part = oracle.case_fill(kind, 9, level, z0=3, nz=5)
        assert np.array_equal(part, full[3 * per:8 * per])


def test_spec_kats():
    """SPEC.md known-answer examples on the restated physics (with the
    corrections SURVEY.md §4 records)."""
    import ctypes as C
    from oracle import oracle as O
    init = np.array([[1.0, 0.0, 0.0, 0.0, 2.5]] * (1 << 6), dtype=np.float64)
    # constant state ("uniform constant field -> unchanged")
    O.build(ref=False) if not O.available("port") else None
    full = np.tile(init, (1 << 6, 1))
    p = O.make_params(2, 6, 5, cfl=0.5)
    out, dts, res = O.uniform_run("port", p, full)
    assert np.array_equal(out, full)
    # max wave speed of (rho=1, v=0, p=1) is sqrt(1.4); dt = cfl*dx/(2c)
    c = np.sqrt(1.4)
    assert dts[0] == 0.5 * (1.0 / 64) / (c + c)
    assert res["max_wave_speed"] == c


def test_reference_rk2_stage_harness_is_step_block():
    """afref_rk2_stage (the seam's checker) composes to the reference's own
    step_block: stage(u,u,mid,dt/2), stage(u,mid,u,dt) == one fixed-dt step."""
    from oracle import oracle as O
    if not O.available("ref"):
        pytest.skip("oracle/_ref not built")
    for dim, level, kind in ((2, 5, 0), (3, 4, 2)):
        init = O.case_fill(kind, 3, level)
        p = O.make_params(dim, level, 1, cfl=0.0, fixed_dt=1e-3)
        ref, _, res = O.uniform_run("ref", p, init)
        mid, r1, _ = O.rk2_stage(p, init, init, 0.5e-3)
        out, r2, flux = O.rk2_stage(p, init, mid, 1e-3, capture=True)
        assert np.array_equal(bits(out), bits(ref))
        assert max(r1["max_wave_speed"], r2["max_wave_speed"]) == res["max_wave_speed"]
        assert len(flux) == dim


def test_reference_window_run_is_single_block():
    """afref_uniform_window_run (the reference's step_block on host-thread
    z-slabs, used for cfg4's full-size digest and the bench's reference arm)
    equals the reference's single-block run bit for bit: state, dt history,
    max_cfl, StepDiag wave speed."""
    from oracle import oracle as O
    if not O.available("ref"):
        pytest.skip("oracle/_ref not built")
    init = O.case_fill(2, 1, 5)
    p = O.make_params(3, 5, 6, cfl=0.4)
    a, da, ra = O.uniform_run("ref", p, init)
    b, db, rb = O.uniform_window_run(p, init, 0, 32, 8, want_out=True, want_dt=True)
    assert np.array_equal(bits(a), bits(b)) and np.array_equal(bits(da), bits(db))
    assert ra["max_cfl"] == rb["max_cfl"] and ra["max_wave_speed"] == rb["max_wave_speed"]
