"""Storage of the MR level arrays (include/af_gpu.h AF_MR_STORAGE_*, csrc/af_mr_storage.cu).

The reference stores only existing nodes (mr_tree.hpp:195). The device tree
stores each level as dense bricks: BRICKS is the brick layout alone (every
level fully allocated), SPARSE maps a 2 MiB page behind a brick of a value
component only while the band of the tree reaches it and re-maps at every
refine. Neither may change a single bit of any result: leaf sets, per-cycle
records, to_uniform(L), details, the dump text and max_cfl are compared with
the dense row-major run of the same seeded case. The sparse runs also report
their device footprint against the dense level grids.
"""
import numpy as np
import pytest

from test_oracle import bits

pytestmark = pytest.mark.gpu


def cfg5_opts(level, **kw):
    """cfg5's rules (BASELINE.json configs[4]) at a smaller finest level:
    eps_l = 1e-3 * 2^(3(l-L)), coarsest leaf 16^3, LT gap reaching it."""
    from paper_1603_05211_b200 import mr as M
    return M.MROptions(epsilon=1e-3, eps_level=[1e-3 * 8.0 ** (l - level) for l in range(level + 1)],
                       min_leaf_level=4, local_time=True, local_time_level_gap=level - 4, **kw)


def run(kind, level, steps, opts, bc=None, detail_level=None):
    from paper_1603_05211_b200 import mr as M
    from paper_1603_05211_b200 import uniform as U
    s = M.MRSolver(3, level, opts, bc=bc)
    s.build(U.case_fill(kind, 7, level))
    mem_build = s.memory()
    rep = s.run(steps, cfl=0.4)
    mem_run = s.memory()
    keys = s.leaves()
    dump = s.dump() if level <= 6 else None
    det = s.details(detail_level) if detail_level is not None else None
    out = s.to_uniform()
    s.close()
    return dict(rep=rep, keys=keys, dump=dump, det=det, out=out, mem_build=mem_build,
                mem_run=mem_run)


def same(a, b):
    assert np.array_equal(a["keys"], b["keys"])
    assert np.array_equal(bits(a["out"]), bits(b["out"]))
    assert np.array_equal(a["rep"].cycles, b["rep"].cycles)
    assert a["rep"].max_cfl == b["rep"].max_cfl
    assert a["dump"] == b["dump"]
    if a["det"] is not None:
        assert np.array_equal(bits(a["det"]), bits(b["det"]))


def small_opts(local_time, **kw):
    from paper_1603_05211_b200 import mr as M
    return M.MROptions(epsilon=1e-3, min_leaf_level=2, local_time=local_time,
                       local_time_level_gap=3, **kw)


@pytest.mark.parametrize("name,kind,level,steps,lt,bc", [
    ("global_outflow", 2, 6, 6, False, None),
    ("lt_pratio", 3, 6, 8, True, None),
    ("global_periodic", 3, 5, 6, False, [1] * 6),
    ("lt_reflective", 2, 6, 8, True, [2] * 6),
])
@pytest.mark.parametrize("shift", [2, 3])
def test_brick_layout_bit_identical(name, kind, level, steps, lt, bc, shift):
    """Bricks of 4^3 / 8^3 cells (levels finer than the brick stored brick by
    brick) against the row-major grids: bit-identical everywhere."""
    d = run(kind, level, steps, small_opts(lt), bc=bc, detail_level=level - 1)
    b = run(kind, level, steps, small_opts(lt, storage="bricks", brick_shift=shift), bc=bc,
            detail_level=level - 1)
    same(d, b)


@pytest.mark.parametrize("level,steps", [(8, 8), (9, 4)])
def test_sparse_bricks_cfg5_rules(level, steps):
    """64^3 bricks mapped only where the band reaches (cfg5's rules, 3D MRLT):
    bit-identical to the dense grids, with a smaller device footprint."""
    d = run(3, level, steps, cfg5_opts(level))
    s = run(3, level, steps, cfg5_opts(level, storage="sparse"))
    same(d, s)
    # dense grids: what the dense run allocates; sparse: mapped pages after the
    # run (to_uniform maps every brick of V afterwards, not counted here)
    assert s["mem_run"]["dense"] == d["mem_run"]["dense"]
    assert s["mem_run"]["now"] < d["mem_run"]["now"]
    print(f"L={level}: dense {d['mem_run']['now'] / 2**30:.2f} GiB, sparse now "
          f"{s['mem_run']['now'] / 2**30:.2f} GiB (peak incl. build {s['mem_run']['peak'] / 2**30:.2f})")


def test_storage_rejects_unsupported():
    from paper_1603_05211_b200 import mr as M
    with pytest.raises(Exception):
        M.MRSolver(2, 6, M.MROptions(epsilon=1e-3, storage="bricks"))
    with pytest.raises(Exception):
        M.MRSolver(3, 6, M.MROptions(epsilon=1e-3, storage="sparse", brick_shift=3))
    with pytest.raises(ValueError):
        M.MRSolver(3, 6, M.MROptions(epsilon=1e-3, storage="hash"))
