"""SPEC.md known-answer properties checked on the device path:
constant fields stay constant bit for bit (RK2 and MUSCL-Hancock, AUSM+ and
AUSMDV, 2D and 3D), the rest-state wave speed sqrt(1.4) fixes dt, periodic
runs conserve mass to round-off, and Harten details vanish exactly on linear
data (the +-1/8 prediction is exact for degree <= 2)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _const(dim, level, rho=1.0, v=(0.0, 0.0, 0.0), p=1.0):
    n = 1 << level
    q = np.zeros((n ** dim, 5))
    q[:, 0] = rho
    for a in range(dim):
        q[:, 1 + a] = rho * v[a]
    kin = 0.5 * rho * sum(x * x for x in v[:dim])
    q[:, 4] = p / 0.4 + kin
    return q


@pytest.mark.parametrize("dim,level", [(2, 6), (3, 4)])
@pytest.mark.parametrize("flux,integ", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_constant_field_unchanged(gpu_lib, dim, level, flux, integ):
    """SPEC.md:147 'uniform constant field -> unchanged' (any scheme)."""
    from paper_1603_05211_b200 import uniform as U
    q = _const(dim, level, rho=1.3, v=(0.3, -0.2, 0.1), p=0.9)
    s = U.UniformSolver(dim, level, scheme=U.SchemeConfig(flux=flux, limiter=1,
                                                          integrator=integ), bc=[1] * 6)
    s.upload(q)
    s.run(5, cfl=0.5)
    out = s.download()
    s.close()
    ref = q.copy()
    if dim == 2:
        ref[:, 3] = 0.0
    assert np.array_equal(out, ref)


def test_rest_state_wave_speed_sets_dt(gpu_lib):
    """max wave speed of (rho=1, v=0, p=1) is sqrt(1.4); the CFL
    rule gives dt = cfl*dx/(2c) in 2D."""
    from paper_1603_05211_b200 import uniform as U
    q = _const(2, 6)
    s = U.UniformSolver(2, 6)
    s.upload(q)
    rep = s.run(3, cfl=0.5)
    s.close()
    c = np.sqrt(1.4)
    assert rep.max_wave_speed == c
    assert np.all(rep.dt == 0.5 * (1.0 / 64) / (c + c))


@pytest.mark.parametrize("dim,level,integ", [(2, 7, 0), (3, 5, 0), (2, 7, 1)])
def test_periodic_conservation(gpu_lib, dim, level, integ):
    """a periodic run conserves mass and energy to round-off."""
    from paper_1603_05211_b200 import uniform as U
    n = 1 << level
    rng = np.random.default_rng(5)
    q = _const(dim, level)
    q[:, 0] = 1.0 + 0.2 * rng.random(n ** dim)
    q[:, 4] = 2.5 + 0.3 * rng.random(n ** dim)
    s = U.UniformSolver(dim, level, scheme=U.SchemeConfig(limiter=1, integrator=integ),
                        bc=[1] * 6)
    s.upload(q)
    s.run(20, cfl=0.4)
    out = s.download()
    s.close()
    for m in (0, 4):
        assert abs(out[:, m].sum() - q[:, m].sum()) <= 1e-12 * abs(q[:, m].sum())


@pytest.mark.parametrize("dim,level", [(2, 5), (3, 4)])
def test_details_vanish_on_linear_data(gpu_lib, dim, level):
    """the prediction reproduces polynomials of degree <= 2, so
    every Harten detail of linear data is exactly 0 (eps = 0 keeps the tree;
    dyadic data keeps every mean and weight exact). Level 0 has a single cell
    and predicts its children by the constant (axis_stencil n == 1)."""
    from paper_1603_05211_b200 import mr as M
    n = 1 << level
    idx = np.indices((n,) * dim).reshape(dim, -1)[::-1]  # x fastest
    x = (idx[0] + 0.5) / n
    y = (idx[1] + 0.5) / n
    q = np.zeros((n ** dim, 5))
    q[:, 0] = 1.0 + 0.25 * x + 0.125 * y
    q[:, 1] = 0.5 * x
    q[:, 4] = 3.0 + 0.5 * y
    if dim == 3:
        q[:, 3] = 0.25 * (idx[2] + 0.5) / n
    s = M.MRSolver(dim, level, M.MROptions(epsilon=0.0))
    s.build(q)
    for lv in range(1, level):
        d = s.details(lv)
        d = d[~np.isnan(d)]
        assert d.size and np.all(d == 0.0), (lv, d.max())
    s.close()


@pytest.mark.parametrize("emin,emax", [(-4, 4), (-300, 300), (-511, 511)])
def test_fast_division_matches_ieee(gpu_lib, emin, emax):
    """The inline fast-path division/sqrt of the face fluxes (fdiv/fsqrt,
    af_physics.cuh) equal IEEE a/b and sqrt wherever their range test lets
    them through; inside [2^-300, 2^300] the test never fails."""
    import ctypes as C
    out = (C.c_ulonglong * 4)()
    assert gpu_lib.af_check_division(1 << 27, 7 + emax, emin, emax, out) == 0
    assert out[0] == 0 and out[2] == 0, list(out)
    if emax <= 300:
        assert out[1] == 0 and out[3] == 0, list(out)
