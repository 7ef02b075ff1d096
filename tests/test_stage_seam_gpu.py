"""The rk2_stage seam with FluxField capture (step.hpp:16-64; the calls the
AMR hierarchy makes, amr_hierarchy.cpp:476,488) through the C ABI
(af_uniform_rk2_stage) against the compiled reference's rk2_stage
(oracle/_ref, ref_harness.cpp afref_rk2_stage): bit-identical out states,
captured face fluxes, StepDiag and the NonPhysicalState text."""
import numpy as np
import pytest

from test_oracle import bits

pytestmark = pytest.mark.gpu

# (dim, level, kind, bc, limiter, flux)
CASES = [
    (2, 5, 0, None, 1, 0),
    (2, 6, 1, [1, 1, 2, 2, 0, 0], 1, 0),
    (2, 5, 0, [2, 0, 1, 1, 0, 0], 0, 1),
    (3, 4, 2, None, 1, 0),
    (3, 4, 3, [2, 2, 1, 1, 0, 0], 1, 0),
    (3, 5, 2, [1] * 6, 0, 1),
]


def _solver(dim, level, bc, limiter, flux):
    from paper_1603_05211_b200 import uniform as U
    return U.UniformSolver(dim, level, scheme=U.SchemeConfig(limiter=limiter, flux=flux), bc=bc)


@pytest.mark.parametrize("dim,level,kind,bc,limiter,flux", CASES,
                         ids=[f"seam{i}" for i in range(len(CASES))])
def test_rk2_stage_and_capture_match_reference(gpu_lib, dim, level, kind, bc, limiter, flux):
    from oracle import oracle as O
    from paper_1603_05211_b200 import uniform as U
    if not O.available("ref"):
        pytest.skip("oracle/_ref not built")
    u0 = U.case_fill(kind, 17, level)
    p = O.make_params(dim, level, 1, cfl=0.0, fixed_dt=1e-3, limiter=limiter, bc=bc, flux=flux)
    s = _solver(dim, level, bc, limiter, flux)
    try:
        # the explicit midpoint's two stages: stage(u,u,mid,dt/2), stage(u,mid,u,dt)
        mid_g, d1, f1 = s.rk2_stage(u0, u0, 0.5e-3, capture=True)
        mid_r, r1, c1 = O.rk2_stage(p, u0, u0, 0.5e-3, capture=True)
        assert np.array_equal(bits(mid_g), bits(mid_r))
        out_g, d2, f2 = s.rk2_stage(u0, mid_g, 1e-3, capture=True)
        out_r, r2, c2 = O.rk2_stage(p, u0, mid_r, 1e-3, capture=True)
        assert np.array_equal(bits(out_g), bits(out_r))
        for fg, fr in zip(f1 + f2, c1 + c2):
            assert fg.shape == fr.shape
            assert np.array_equal(bits(fg), bits(fr))
        assert d1.max_wave_speed == r1["max_wave_speed"] and d2.max_wave_speed == r2["max_wave_speed"]
        assert d1.fallbacks == r1["fallbacks"] and d2.fallbacks == r2["fallbacks"]
        # no capture: the same state
        out_n, _, none = s.rk2_stage(u0, mid_g, 1e-3)
        assert none is None and np.array_equal(bits(out_n), bits(out_g))
    finally:
        s.close()


def test_rk2_stage_nonphysical_text(gpu_lib):
    from oracle import oracle as O
    from paper_1603_05211_b200 import uniform as U
    from paper_1603_05211_b200.errors import NonPhysicalState
    if not O.available("ref"):
        pytest.skip("oracle/_ref not built")
    u0 = U.case_fill(0, 17, 5)
    bad = u0.copy()
    bad[37, 4] = 0.5 * (bad[37, 1] ** 2 + bad[37, 2] ** 2) / bad[37, 0] - 1.0  # p < 0
    p = O.make_params(2, 5, 1, cfl=0.0, fixed_dt=1e-3)
    _, r, _ = O.rk2_stage(p, u0, bad, 1e-3)
    assert r["err_kind"] == 1
    s = _solver(2, 5, None, 1, 0)
    try:
        with pytest.raises(NonPhysicalState) as e:
            s.rk2_stage(u0, bad, 1e-3)
        assert str(e.value) == r["err"]
    finally:
        s.close()


def test_rk2_stage_capture_needs_exact_numerics(gpu_lib):
    from paper_1603_05211_b200 import uniform as U
    from paper_1603_05211_b200.errors import ConfigError
    s = _solver(3, 4, None, 1, 0)
    try:
        s.set_numerics(True)
        u0 = U.case_fill(2, 17, 4)
        s.rk2_stage(u0, u0, 1e-3)  # tolerance mode without capture is fine
        with pytest.raises(ConfigError):
            s.rk2_stage(u0, u0, 1e-3, capture=True)
    finally:
        s.close()
