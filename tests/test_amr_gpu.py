"""AMR patch path on the device against the compiled reference (oracle/_ref):
box lists, every patch block with its ghost layers (data and data_old), level
times, the per-step samples, max_cfl and fallbacks, all bit for bit
(PatchHierarchy + the run_amr cycle, amr_hierarchy.cpp / amr_solver.cpp)."""
import numpy as np
import pytest

from oracle import oracle
from paper_1603_05211_b200 import amr
from paper_1603_05211_b200.errors import ConfigError, LevelMismatch, NonPhysicalState
from paper_1603_05211_b200.uniform import SchemeConfig

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not oracle.available("ref"), reason="oracle/_ref not built")]

OUT, PER, REFL = 0, 1, 2


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def _run_both(dim, base, level, n_steps, dt, kind, seed=1, bc=None, flux=1, limiter=1,
              integrator=1, time_refine=True, flux_correction=True, eps=(0.05, 0.05), eff=0.8):
    opts = amr.AmrOptions(eps[0], eps[1], eff, time_refine, flux_correction, level - base)
    h = amr.PatchHierarchy(dim, base, opts, bc=bc, scheme=SchemeConfig(flux, limiter, integrator))
    ref = oracle.ref_amr_run(dim, level, base, n_steps, dt, case_kind=kind, seed=seed, bc=bc,
                             limiter=limiter, flux=flux, integrator=integrator, eps_rho=eps[0],
                             eps_p=eps[1], efficiency=eff, time_refine=time_refine,
                             flux_correction=flux_correction)
    return h, ref


def _compare(h, rep, ref):
    assert ref["err_kind"] == 0, ref["err"]
    assert h.dump_boxes() == ref["dump_boxes"]
    assert h.n_levels() == len(ref["levels"])
    assert h.properly_nested()
    for l, lv in enumerate(ref["levels"]):
        npatch, cells, t, t_old = h.level_info(l)
        assert npatch == len(lv["boxes"]) and np.array_equal(h.boxes(l), lv["boxes"])
        assert t == lv["t"] and t_old == lv["t_old"], (l, t, lv["t"], t_old, lv["t_old"])
        for name, ghost, old in (("data", 0, False), ("blocks", 2, False), ("blocks_old", 2, True)):
            mine = h.patch_data(l, ghost, old)
            assert mine.shape == lv[name].shape
            bad = np.nonzero(_bits(mine) != _bits(lv[name]))
            assert bad[0].size == 0, (l, name, bad[0][:5], mine[bad[0][:3]], lv[name][bad[0][:3]])
    if rep is not None:
        assert np.array_equal(rep.cells_per_step, ref["cells_per_step"])
        assert np.array_equal(rep.leaves_per_step, ref["leaves_per_step"])
        assert rep.max_cfl == ref["max_cfl"]
        assert rep.fallbacks == ref["fallbacks"]
    tot = h.total_conserved()
    assert np.allclose(tot, ref["total_conserved"], rtol=1e-12, atol=1e-14)
    assert h.total_cells() == sum(len(lv["data"]) for lv in ref["levels"])


CASES = [
    # dim base level steps dt kind  kwargs
    ("2d_hancock_lt", 2, 4, 6, 16, 1.0e-3, 0, {}),
    ("2d_hancock_global", 2, 4, 6, 8, 1.0e-3, 0, {"time_refine": False}),
    ("2d_rk2_ausm_lt", 2, 4, 6, 16, 1.0e-3, 0, {"flux": 0, "integrator": 0}),
    ("2d_rk2_vanalbada", 2, 3, 6, 16, 1.0e-3, 0, {"flux": 0, "limiter": 0, "integrator": 0, "seed": 3}),
    ("2d_periodic", 2, 4, 6, 16, 1.0e-3, 0, {"bc": [PER] * 6, "seed": 2}),
    ("2d_reflective", 2, 4, 6, 16, 1.0e-3, 0, {"bc": [REFL, REFL, OUT, REFL, OUT, OUT], "seed": 5}),
    ("2d_no_reflux", 2, 4, 6, 16, 1.0e-3, 0, {"flux_correction": False}),
    ("2d_three_levels", 2, 4, 7, 32, 5.0e-4, 0, {"seed": 7, "eff": 0.7}),
    ("2d_tiny_base", 2, 2, 6, 16, 1.0e-3, 0, {"seed": 4}),
    ("2d_single_level", 2, 5, 5, 8, 2.0e-3, 0, {}),
    ("2d_tiny_base_reflective_rk2", 2, 2, 5, 8, 2.0e-3, 0,
     {"seed": 6, "bc": [REFL] * 6, "flux": 0, "integrator": 0}),
    ("3d_tiny_base_periodic", 3, 2, 4, 4, 4.0e-3, 2, {"bc": [PER] * 6}),
    ("3d_hancock_lt", 3, 3, 5, 8, 2.0e-3, 2, {}),
    ("3d_rk2_periodic", 3, 3, 5, 8, 1.0e-3, 2, {"bc": [PER] * 6, "flux": 0, "integrator": 0, "seed": 4}),
    ("3d_reflective_global", 3, 3, 5, 4, 2.0e-3, 3, {"bc": [REFL] * 6, "time_refine": False}),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_run_amr_matches_reference(case):
    _, dim, base, level, n_steps, dt, kind, kw = case
    h, ref = _run_both(dim, base, level, n_steps, dt, kind, **kw)
    h.initialize_case(kind, kw.get("seed", 1))
    rep = h.run(n_steps, dt)
    _compare(h, rep, ref)
    assert h.kernel_launches() > 0
    h.close()


LONG = [
    # four levels, 128 finest steps: dozens of patches that follow the waves
    ("2d_L8_hancock", 2, 5, 8, 128, 1.2e-3, 0, {"seed": 1}),
    ("2d_L8_hancock_s3", 2, 5, 8, 128, 1.2e-3, 0, {"seed": 3}),
    ("2d_L8_rk2", 2, 5, 8, 128, 1.0e-3, 0, {"seed": 3, "flux": 0, "integrator": 0}),
    ("2d_L7_vanalbada", 2, 4, 7, 128, 2.6e-3, 0, {"seed": 8, "limiter": 0}),
    ("3d_L6_hancock_pratio", 3, 3, 6, 32, 1.5e-3, 3, {"seed": 2}),
    ("3d_L6_rk2", 3, 3, 6, 32, 0.8e-3, 2, {"seed": 1, "flux": 0, "integrator": 0}),
]


@pytest.mark.parametrize("case", LONG, ids=[c[0] for c in LONG])
def test_long_runs_match_reference(case):
    _, dim, base, level, n_steps, dt, kind, kw = case
    h, ref = _run_both(dim, base, level, n_steps, dt, kind, **kw)
    h.initialize_case(kind, kw.get("seed", 1))
    rep = h.run(n_steps, dt)
    _compare(h, rep, ref)
    assert max(len(lv["boxes"]) for lv in ref["levels"]) >= 20
    h.close()


@pytest.mark.parametrize("seed,dt", [(12, 3e-3), (15, 3e-3), (19, 3e-3), (25, 3e-3), (59, 1e-3),
                                     (59, 3e-3)])
@pytest.mark.parametrize("time_refine", [False, True])
@pytest.mark.parametrize("flux,limiter", [(1, 0), (0, 1)])
def test_fallback_counts_match_reference(seed, dt, time_refine, flux, limiter):
    """the stress quadrants reach the MUSCL-Hancock predictor/corrector
    fallbacks (step.cpp:170-173,203-212); the reference counts one per patch
    that evaluates the cell or face"""
    h, ref = _run_both(2, 4, 6, 4, dt, 4, seed=seed, flux=flux, limiter=limiter, integrator=1,
                       time_refine=time_refine)
    if ref["err_kind"]:
        h.initialize_case(4, seed)
        with pytest.raises(NonPhysicalState) as e:
            h.run(4, dt)
        assert str(e.value) == ref["err"]
        return
    h.initialize_case(4, seed)
    rep = h.run(4, dt)
    _compare(h, rep, ref)
    h.close()


def test_fallback_cases_do_fall_back():
    ref = oracle.ref_amr_run(2, 6, 4, 4, 3e-3, case_kind=4, seed=59, flux=1, limiter=0,
                             integrator=1, time_refine=False)
    assert ref["err_kind"] == 0 and ref["fallbacks"] >= 5


@pytest.mark.parametrize("dim,n", [(2, 16), (2, 64), (2, 256), (3, 8), (3, 32)])
def test_device_cluster_matches_reference(dim, n):
    """the clustering remesh runs on the device (summed-area tables, breadth-
    first bisection) against the reference's recursive cluster()"""
    from test_amr import _blobs
    rng = np.random.default_rng(7 * dim + n)
    shape = (n,) * dim
    for trial in range(8):
        flags = _blobs(rng, shape, 1 + trial % 5)
        allowed = None
        if trial % 3 == 1:
            allowed = np.ones(shape, dtype=np.uint8)
            allowed[tuple(slice(0, 2) for _ in shape)] = 0
            allowed[(slice(n // 2, n // 2 + 1),) + (slice(None),) * (dim - 1)] = 0
            flags &= allowed
        for eff in (0.5, 0.8, 0.95):
            assert np.array_equal(amr.cluster_device(flags, eff, allowed),
                                  oracle.ref_cluster(flags, eff, allowed)), (dim, n, trial, eff)
    empty = np.zeros(shape, dtype=np.uint8)
    assert len(amr.cluster_device(empty, 0.8)) == 0
    one = empty.copy()
    one[(n // 2,) * dim] = 1
    assert np.array_equal(amr.cluster_device(one, 0.8), oracle.ref_cluster(one, 0.8))
    assert np.array_equal(amr.cluster_device(np.ones(shape, np.uint8), 0.8),
                          oracle.ref_cluster(np.ones(shape, np.uint8), 0.8))


def test_initialize_matches_reference():
    """the hierarchy straight after initialize (n_steps = 0): boxes, ghosts"""
    h, ref = _run_both(2, 4, 7, 0, 1e-3, 0, seed=9)
    h.initialize_case(0, 9)
    _compare(h, None, ref)
    h.close()


def test_python_callback_ic_equals_seeded_case():
    opts = amr.AmrOptions(max_levels=1)
    a = amr.PatchHierarchy(2, 4, opts)
    a.initialize_case(0, 1)
    quad = oracle.case_fill(0, 1, 1)  # the four quadrant states on a 2x2 mesh
    b = amr.PatchHierarchy(2, 4, opts)
    b.initialize(lambda x, y, z: quad[(1 if x > 0.5 else 0) + 2 * (1 if y > 0.5 else 0)])
    assert a.dump_boxes() == b.dump_boxes()
    for l in range(a.n_levels()):
        assert np.array_equal(_bits(a.patch_data(l, 2)), _bits(b.patch_data(l, 2)))


def test_public_methods_step_by_step():
    """one AMRLT cycle driven through the public methods equals run()"""
    opts = amr.AmrOptions(max_levels=1)
    sch = SchemeConfig(1, 1, 1)
    a = amr.PatchHierarchy(2, 4, opts, scheme=sch)
    b = amr.PatchHierarchy(2, 4, opts, scheme=sch)
    a.initialize_case(0, 1)
    b.initialize_case(0, 1)
    dt = 1e-3
    b.run(2, dt)
    a.sync_ghosts(0, 0.0)
    a.remesh(0)
    d0 = a.update_level(0, 2 * dt)
    assert d0.max_wave_speed > 0
    a.sync_ghosts(0, 2 * dt)
    for sub in range(2):
        a.sync_ghosts(1, sub * dt)
        a.update_level(1, dt)
    a.average_down(0)
    a.flux_correct(0)
    for l in range(2):
        assert np.array_equal(_bits(a.patch_data(l, 0)), _bits(b.patch_data(l, 0)))


def test_flux_correction_conserves():
    """periodic domain: the composite sums stay constant with refluxing"""
    opts = amr.AmrOptions(max_levels=2)
    h = amr.PatchHierarchy(2, 4, opts, bc=[PER] * 6, scheme=SchemeConfig(1, 1, 1))
    h.initialize_case(0, 2)
    t0 = h.total_conserved()
    h.run(16, 1e-3)
    t1 = h.total_conserved()
    assert np.allclose(t0, t1, rtol=1e-12, atol=1e-13)


def test_errors_match_reference():
    # a time step far past the CFL limit: the reference's NonPhysicalState text
    h, ref = _run_both(2, 4, 6, 16, 2.0e-2, 0)
    assert ref["err_kind"] == 1
    h.initialize_case(0, 1)
    with pytest.raises(NonPhysicalState) as e:
        h.run(16, 2.0e-2)
    assert str(e.value) == ref["err"]
    h2, ref2 = _run_both(2, 4, 6, 16, 2.0e-2, 0, flux=0, integrator=0)
    assert ref2["err_kind"] == 1
    h2.initialize_case(0, 1)
    with pytest.raises(NonPhysicalState) as e2:
        h2.run(16, 2.0e-2)
    assert str(e2.value) == ref2["err"]
    # a failure deep in a long run: level 3, a later cycle; and a ghost cell
    for args, kw in (((2, 5, 8, 128, 1.2e-3, 0), {"seed": 6}),
                     ((2, 4, 7, 128, 2.6e-3, 0), {"seed": 11, "limiter": 0})):
        hh, rr = _run_both(*args, **kw)
        assert rr["err_kind"] == 1
        hh.initialize_case(0, kw["seed"])
        with pytest.raises(NonPhysicalState) as ee:
            hh.run(args[3], args[4])
        assert str(ee.value) == rr["err"]
    # 3D RK2 stage-2 failure on a fine patch (the "level L patch P: " prefix)
    h4, ref4 = _run_both(3, 3, 5, 8, 2.0e-3, 2, seed=4, bc=[PER] * 6, flux=0, integrator=0)
    assert ref4["err_kind"] == 1
    h4.initialize_case(2, 4)
    with pytest.raises(NonPhysicalState) as e4:
        h4.run(8, 2.0e-3)
    assert str(e4.value) == ref4["err"]
    # n_steps must be a multiple of the time-refined cycle
    h3 = amr.PatchHierarchy(2, 4, amr.AmrOptions(max_levels=2))
    h3.initialize_case(0, 1)
    with pytest.raises(ConfigError):
        h3.run(6, 1e-3)
    # assemble_level needs a level covering the domain
    assert h3.assemble_level(0).shape == (256, 5)
    if h3.n_levels() > 1:
        with pytest.raises(LevelMismatch):
            h3.assemble_level(1)


def test_l1_error_amr_matches_reference():
    """l1_error_amr (amr_hierarchy.cpp:631-656) against a uniform solution"""
    h, ref = _run_both(2, 4, 7, 32, 5.0e-4, 0, seed=7, eff=0.7)
    h.initialize_case(0, 7)
    h.run(32, 5.0e-4)
    assert ref["err_kind"] == 0
    sol = oracle.case_fill(0, 7, 8)  # any level-8 field serves as the reference solution
    sol[:, 0] *= 1.0 + 0.01 * np.sin(np.arange(len(sol)))
    mine = h.l1_error(sol, 8)
    want = oracle.ref_amr_l1_error(sol, 8)
    assert np.allclose(mine, want, rtol=1e-12, atol=1e-15) and want[0] > 0
    with pytest.raises(LevelMismatch):
        h.l1_error(oracle.case_fill(0, 7, 5), 5)


def test_run_amr_helper():
    """amr.run_amr builds the hierarchy for a resolution level as run_amr does
    (amr_base_exp, max_levels = level - base) and steps to t_end"""
    assert amr.amr_base_exp(2, 10) == 6 and amr.amr_base_exp(3, 8) == 3 and amr.amr_base_exp(2, 4) == 3
    h, rep = amr.run_amr(2, 7, 32, 32 * 5.0e-4, case=(0, 7), scheme=SchemeConfig(1, 1, 1),
                         options=amr.AmrOptions(cluster_efficiency=0.7))
    ref = oracle.ref_amr_run(2, 7, 6, 32, 5.0e-4, case_kind=0, seed=7, flux=1, integrator=1,
                             efficiency=0.7)
    _compare(h, rep, ref)
    with pytest.raises(ConfigError):
        amr.run_amr(2, 0, 8, 0.1, case=(0, 1))
