"""AMR patch path, CPU side: the host clustering of libafgpu against the
reference's cluster() (amr_cluster.cpp:79-232), and the harness's restated
AmrDriver loop pinned against the reference's own run_amr."""
import numpy as np
import pytest

from oracle import oracle
from paper_1603_05211_b200 import amr

pytestmark = pytest.mark.skipif(not oracle.available("ref"), reason="oracle/_ref not built")


def _blobs(rng, shape, k):
    """a mask of k random boxes plus salt noise: gaps, inflections, single cells"""
    m = np.zeros(shape, dtype=np.uint8)
    for _ in range(k):
        lo = [rng.integers(0, s - 1) for s in shape]
        hi = [min(s, l + 1 + rng.integers(0, max(2, s // 3))) for s, l in zip(shape, lo)]
        m[tuple(slice(l, h) for l, h in zip(lo, hi))] = 1
    m |= (rng.random(shape) < 0.01).astype(np.uint8)
    return m


@pytest.mark.parametrize("dim,n", [(2, 16), (2, 32), (2, 64), (3, 8), (3, 16)])
def test_cluster_matches_reference(dim, n):
    rng = np.random.default_rng(100 * dim + n)
    shape = (n,) * dim
    for trial in range(12):
        flags = _blobs(rng, shape, 1 + trial % 5)
        allowed = None
        if trial % 3 == 1:  # a restricted region: boxes must stay inside it
            allowed = np.ones(shape, dtype=np.uint8)
            allowed[tuple(slice(0, 2) for _ in shape)] = 0
            allowed[(slice(n // 2, n // 2 + 1),) + (slice(None),) * (dim - 1)] = 0
            flags &= allowed
        for eff in (0.5, 0.8, 0.95):
            mine = amr.cluster(flags, eff, allowed)
            ref = oracle.ref_cluster(flags, eff, allowed)
            assert np.array_equal(mine, ref), (dim, n, trial, eff)
            # disjoint cover of the flagged cells
            cover = np.zeros(shape, dtype=np.int32)
            for b in mine:
                sl = (slice(b[1], b[4]), slice(b[0], b[3])) if dim == 2 else \
                     (slice(b[2], b[5]), slice(b[1], b[4]), slice(b[0], b[3]))
                cover[sl] += 1
            assert cover.max(initial=0) <= 1
            assert np.all(cover[flags > 0] == 1)


def test_cluster_edge_cases():
    empty = np.zeros((8, 8), dtype=np.uint8)
    assert len(amr.cluster(empty, 0.8)) == 0
    one = empty.copy()
    one[3, 5] = 1
    assert amr.cluster(one, 0.8).tolist() == [[5, 3, 0, 6, 4, 1]]
    full = np.ones((8, 8, 8), dtype=np.uint8)
    assert amr.cluster(full, 0.8).tolist() == [[0, 0, 0, 8, 8, 8]]
    assert np.array_equal(amr.cluster(one, 0.8), oracle.ref_cluster(one, 0.8))


@pytest.mark.parametrize("time_refine", [True, False])
def test_harness_loop_is_run_amr(time_refine):
    """mode 1 (the harness's advance() on the public PatchHierarchy methods)
    equals mode 2 (the reference's run_amr) bit for bit on its built-in case."""
    kw = dict(dim=2, level=6, base_exp=0, n_steps=96, dt_finest=0.0, eps_rho=-1.0, eps_p=-1.0,
              efficiency=-1.0, time_refine=time_refine, flux=1, integrator=1, limiter=1,
              builtin="lax_liu_6")
    a = oracle.ref_amr_run(mode=1, **kw)
    b = oracle.ref_amr_run(mode=2, **kw)
    assert a["err_kind"] == 0 and b["err_kind"] == 0, (a["err"], b["err"])
    assert a["dump_boxes"] == b["dump_boxes"]
    assert a["max_cfl"] == b["max_cfl"] and a["fallbacks"] == b["fallbacks"]
    assert np.array_equal(a["cells_per_step"], b["cells_per_step"])
    assert np.array_equal(a["leaves_per_step"], b["leaves_per_step"])
    assert len(a["levels"]) == len(b["levels"]) >= 2
    for la, lb in zip(a["levels"], b["levels"]):
        assert la["t"] == lb["t"]
        assert np.array_equal(la["blocks"].view(np.uint64), lb["blocks"].view(np.uint64))
