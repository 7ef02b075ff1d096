"""Properties at BASELINE.json's full sizes, where the CPU reference is too slow
to compare against (SURVEY.md §8(c) oracle limits):
  * cfg4 shape (3D 512^3): with periodic boundaries every conserved total is
    preserved to round-off over RK2 steps;
  * cfg2 shape (2D L=10): MR with eps = 0 is the uniform FV solver bit for bit
    (SPEC.md:312), through the whole refine/evolve/coarsen cycle machinery;
  * cfg2 itself: the adapted tree stays graded (mr_tree.cpp:562-606) and the
    leaves tile the domain exactly."""
import numpy as np
import pytest

from test_oracle import bits

pytestmark = pytest.mark.gpu


def test_cfg4_periodic_conservation(gpu_lib):
    from paper_1603_05211_b200 import uniform as U
    init = U.case_fill(2, 1, 9)
    s = U.UniformSolver(3, 9, bc=[1] * 6)
    s.upload(init)
    s.run(2, cfl=0.4)
    out = s.download()
    s.close()
    scale = np.abs(init).sum()  # the momentum totals start at 0: a global scale
    for m in range(5):
        a, b = init[:, m].sum(), out[:, m].sum()
        assert abs(a - b) <= 1e-12 * scale, (m, a, b)


def test_cfg2_eps0_equals_uniform(gpu_lib):
    from paper_1603_05211_b200 import mr as M
    from paper_1603_05211_b200 import uniform as U
    init = U.case_fill(0, 1, 10)
    s = M.MRSolver(2, 10, M.MROptions(epsilon=0.0, min_leaf_level=3))
    s.build(init)
    s.run(4, cfl=0.0, fixed_dt=1e-4)
    a = s.to_uniform()
    s.close()
    u, _ = U.run_uniform(init, 2, 10, 4, fixed_dt=1e-4)
    assert np.array_equal(bits(a), bits(u))


def _graded_and_tiling(keys, dim, L):
    """The leaves tile the domain exactly (volumes sum to 1), and the tree is
    graded as enforce_gradedness leaves it (mr_tree.cpp:404-444): no leaf has
    a same-level face neighbour whose child on the shared face is internal."""
    lvl = (keys >> np.uint64(45)).astype(np.int64)
    m = np.uint64((1 << 15) - 1)
    i = ((keys >> np.uint64(30)) & m).astype(np.int64)
    j = ((keys >> np.uint64(15)) & m).astype(np.int64)
    assert np.sum(2.0 ** (-dim * lvl)) == 1.0
    leafset = set(zip(lvl.tolist(), i.tolist(), j.tolist()))

    def leaf_level_at(fx, fy):  # level of the leaf covering finest cell (fx, fy)
        for lev in range(L + 1):
            if (lev, fx >> (L - lev), fy >> (L - lev)) in leafset:
                return lev
        raise AssertionError("uncovered cell")

    for (l, a, b) in leafset:
        if l + 2 > L:
            continue
        n = 1 << l
        for ax in (0, 1):
            for d in (-1, 1):
                p = [a, b]
                p[ax] += d
                if p[ax] < 0 or p[ax] >= n:
                    continue
                # the neighbour's two children on the shared face (level l+1)
                for t in (0, 1):
                    c = [2 * p[0], 2 * p[1]]
                    c[ax] += 0 if d > 0 else 1
                    c[1 - ax] += t
                    sh = L - (l + 1)
                    if leaf_level_at(c[0] << sh, c[1] << sh) >= l + 2:
                        return False
    return True


def test_cfg2_tree_graded_and_tiling(gpu_lib):
    import bench
    from paper_1603_05211_b200 import mr as M
    from paper_1603_05211_b200 import uniform as U
    o, epsl = bench.mr_options("cfg2")
    s = M.MRSolver(2, 10, M.MROptions(epsilon=o["eps"], eps_level=epsl, min_leaf_level=3))
    s.build(U.case_fill(0, 1, 10))
    s.run(30, cfl=0.5)
    keys = s.leaves()
    s.close()
    assert _graded_and_tiling(keys, 2, 10)
