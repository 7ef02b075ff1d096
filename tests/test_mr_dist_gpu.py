"""Spatially decomposed MR on one GPU: R ranks, each an
MRSolver on its own host thread (af_comm_create_local), exchanging halo rows
through device-to-device copies. The tree, the state and every cycle record
must be bit-identical to the single-rank run for any R: all passes are
level-synchronous and every reduction is exact."""
import numpy as np
import pytest

from test_oracle import bits

pytestmark = pytest.mark.gpu


def eps_levels(eps, L, d):
    return [eps * 2.0 ** (d * (l - L)) for l in range(L + 1)]


def make(kind, level, ranks, eps=1e-3, eps_level=None, min_leaf=3, bc=None, local_time=False,
         gap=3, limiter=1):
    from paper_1603_05211_b200 import mr as M
    from paper_1603_05211_b200 import uniform as U
    dim = 3 if kind >= 2 else 2
    opts = M.MROptions(epsilon=eps, eps_level=eps_level, min_leaf_level=min_leaf,
                       local_time=local_time, local_time_level_gap=gap)
    sch = U.SchemeConfig(limiter=limiter)
    if ranks == 1:
        return M.MRSolver(dim, level, opts, scheme=sch, bc=bc)
    return M.MRGroup(dim, level, ranks, opts, scheme=sch, bc=bc)


CASES = [
    # kind, seed, level, steps, ranks, kwargs
    (0, 11, 6, 12, 2, dict()),
    (0, 12, 7, 10, 3, dict(eps_level=eps_levels(1e-3, 7, 2))),                 # cfg2 rule
    (1, 13, 7, 8, 4, dict(min_leaf=3)),                                         # cfg3 generator
    (0, 14, 6, 10, 4, dict(bc=[1] * 6)),                                        # periodic wrap
    (0, 15, 6, 10, 3, dict(bc=[2, 2, 2, 2, 0, 0])),                             # reflective
    (0, 16, 6, 10, 8, dict(min_leaf=3)),                                        # 1 row per rank at lp
    (2, 17, 5, 4, 2, dict(min_leaf=2)),                                         # 3D
    (3, 18, 5, 3, 3, dict(min_leaf=2, eps_level=eps_levels(1e-3, 5, 3))),       # 3D, cfg5 rule
]


CASES_LT = [
    (0, 21, 6, 16, 2, dict(local_time=True, min_leaf=0)),
    (1, 22, 7, 16, 3, dict(local_time=True, min_leaf=0)),                      # cfg3 generator
    (0, 23, 7, 12, 4, dict(local_time=True, min_leaf=0, gap=2, bc=[1] * 6)),   # periodic wrap
    (0, 24, 7, 12, 4, dict(local_time=True, min_leaf=0, gap=4, limiter=0)),    # wider buffers
    (2, 25, 5, 8, 2, dict(local_time=True, min_leaf=0)),                       # 3D
    (3, 26, 5, 8, 3, dict(local_time=True, min_leaf=1, eps_level=eps_levels(1e-3, 5, 3))),
]
# large enough that every rank's windowed arrays leave unmapped memory at the
# finest levels: an access outside a window would fault
CASES_WIN = [
    (0, 31, 10, 4, 4, dict(eps_level=eps_levels(1e-3, 10, 2))),                # cfg2 rule, L=10
    (1, 32, 9, 4, 3, dict(local_time=True, min_leaf=0)),                       # MRLT
    (2, 33, 7, 2, 4, dict(min_leaf=3)),                                        # 3D
]
CASES = CASES + CASES_LT + CASES_WIN


@pytest.mark.parametrize("kind,seed,level,steps,ranks,kw", CASES,
                         ids=[f"k{c[0]}_L{c[2]}_R{c[4]}_{i}" for i, c in enumerate(CASES)])
def test_mr_ranks_equal_single(gpu_lib, kind, seed, level, steps, ranks, kw):
    from paper_1603_05211_b200 import uniform as U
    init = U.case_fill(kind, seed, level)
    cfl = 0.4 if kind >= 2 else 0.5
    one = make(kind, level, 1, **kw)
    one.build(init)
    r1 = one.run(steps, cfl=cfl)
    k1, u1 = one.leaves(), one.to_uniform()
    one.close()
    grp = make(kind, level, ranks, **kw)
    grp.build(init)
    rR = grp.run(steps, cfl=cfl)
    kR, uR = grp.leaves(), grp.to_uniform()
    grp.close()
    assert np.array_equal(r1.cycles, rR.cycles), "per-cycle leaves/nodes/dt/updates"
    assert r1.max_cfl == rR.max_cfl and r1.fallbacks == rR.fallbacks
    assert np.array_equal(k1, kR), "leaf set"
    assert np.array_equal(bits(u1), bits(uR)), "to_uniform(L)"


def test_mr_ranks_error_message(gpu_lib):
    """A blow-up reports the same first offender (key order) as one rank."""
    from paper_1603_05211_b200 import uniform as U
    from paper_1603_05211_b200.errors import NonPhysicalState
    init = U.case_fill(0, 7, 6)
    msgs = []
    for ranks in (1, 3):
        s = make(0, 6, ranks)
        s.build(init)
        with pytest.raises(NonPhysicalState) as e:
            s.run(30, cfl=3.0)
        msgs.append(str(e.value))
        s.close()
    assert msgs[0] == msgs[1]
