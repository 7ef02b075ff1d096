"""The MR solver's execution switches change how the work is scheduled, never
its results: every switch below gives leaf sets, per-cycle records,
to_uniform(L) states and max_cfl bit-identical to the default schedule on the
same seeded runs (global time step with level thresholds, and local time
stepping). The switches are read when a solver is created.

  AF_MR_NO_CYCLE_GRAPH  cycle-by-cycle host path instead of the whole-cycle graph
  AF_MR_NO_GRAPH        no CUDA graphs at all
  AF_MR_NO_PDL          no programmatic dependent launch
  AF_MR_NO_PRE          no status/tile prefetch before the PDL wait
  AF_MR_NO_SWAP         stage commit copy instead of the buffer swap
  AF_MR_NO_TINY         one launch per coarse level instead of the single-CTA kernels
  AF_MR_FULL_SWEEPS     every coarsen sweep, no re-sweep skip test
  AF_MR_NO_FULL         the general stage path for full tiles too (no fast path)
  AF_MR_NO_FULLK        full 2D tiles on mr_stage_kernel's fast path instead of
                        the pipelined mr_stage_full2d kernel
  AF_MR_FULLK           mr_stage_full2d for any number of full tiles (by default
                        only when a stage has enough of them to fill the GPU)
"""
import os

import numpy as np
import pytest

from test_oracle import bits

pytestmark = pytest.mark.gpu

SWITCHES = ["AF_MR_NO_CYCLE_GRAPH", "AF_MR_NO_GRAPH", "AF_MR_NO_PDL", "AF_MR_NO_PRE",
            "AF_MR_NO_SWAP", "AF_MR_NO_TINY", "AF_MR_FULL_SWEEPS", "AF_MR_NO_FULL",
            "AF_MR_NO_FULLK", "AF_MR_FULLK"]


def run(switch, kind, level, steps, bc=None, **kw):
    from paper_1603_05211_b200 import mr as M
    from paper_1603_05211_b200 import uniform as U
    old = os.environ.get(switch) if switch else None
    if switch:
        os.environ[switch] = "1"
    try:
        dim = 3 if kind >= 2 else 2
        s = M.MRSolver(dim, level, M.MROptions(**kw), bc=bc)
        s.build(U.case_fill(kind, 41, level))
        rep = s.run(steps, cfl=0.5 if dim == 2 else 0.4)
        out, keys = s.to_uniform(), s.leaves()
        s.close()
    finally:
        if switch:
            if old is None:
                del os.environ[switch]
            else:
                os.environ[switch] = old
    return rep, out, keys


CASES = {
    "global_epsl_min3": (0, 8, 12, dict(epsilon=1e-3, min_leaf_level=3,
                                        eps_level=[1e-3 * 4.0 ** (l - 8) for l in range(9)])),
    "lt_noise": (1, 7, 8, dict(epsilon=1e-3, local_time=True, local_time_level_gap=3)),
    "global_3d": (2, 5, 4, dict(epsilon=1e-3, min_leaf_level=2)),
    # dense trees (full tiles everywhere) at the domain boundaries
    "lt_dense_reflective": (1, 7, 8, dict(epsilon=1e-6, local_time=True, local_time_level_gap=2,
                                          bc=[2] * 6)),
    "global_dense_periodic": (1, 7, 6, dict(epsilon=1e-6, min_leaf_level=3, bc=[1] * 6)),
}


@pytest.mark.parametrize("case", list(CASES))
def test_switches_do_not_change_results(gpu_lib, case):
    kind, level, steps, kw = CASES[case]
    kw = dict(kw)
    bc = kw.pop("bc", None)
    rep0, out0, keys0 = run(None, kind, level, steps, bc=bc, **kw)
    for sw in SWITCHES:
        rep, out, keys = run(sw, kind, level, steps, bc=bc, **kw)
        assert np.array_equal(keys, keys0), sw
        assert np.array_equal(rep.cycles, rep0.cycles), sw
        assert np.array_equal(bits(out), bits(out0)), sw
        assert rep.max_cfl == rep0.max_cfl and rep.fallbacks == rep0.fallbacks, sw
