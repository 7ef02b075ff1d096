"""GPU parity of the adaptive MR path (libafgpu.so through the C ABI) against
the compiled reference (oracle/_ref: MRTree / MRSolver / run_mr driven through
its public API): bit-exact leaf sets, per-cycle leaf/node counts and dt,
bit-exact to_uniform(L) states, RunReport max_cfl / fallbacks, and error text.
Falls back to the committed golden fixtures when the reference build is absent."""
import glob
import os

import numpy as np
import pytest

from test_oracle import bits

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = sorted(glob.glob(os.path.join(HERE, "golden", "mr_*.npz")))


def eps_levels(eps, L, d):
    return [eps * 2.0 ** (d * (l - L)) for l in range(L + 1)]


def gpu_mr(kind, seed, level, steps, cfl=0.5, fixed_dt=0.0, eps=1e-3, eps_level=None,
           min_leaf=0, local_time=False, gap=3, limiter=1, bc=None, flux=0):
    from paper_1603_05211_b200 import mr as M
    from paper_1603_05211_b200 import uniform as U
    dim = 3 if kind >= 2 else 2
    init = U.case_fill(kind, seed, level)
    s = M.MRSolver(dim, level, M.MROptions(epsilon=eps, eps_level=eps_level,
                                           min_leaf_level=min_leaf, local_time=local_time,
                                           local_time_level_gap=gap),
                   scheme=U.SchemeConfig(flux=flux, limiter=limiter), bc=bc)
    s.build(init)
    rep = s.run(steps, cfl=cfl, fixed_dt=fixed_dt)
    out = s.to_uniform()
    keys = s.leaves()
    s.close()
    return init, out, keys, rep


def ref_mr(oracle, init, kind, level, steps, cfl=0.5, fixed_dt=0.0, eps=1e-3, eps_level=None,
           min_leaf=0, local_time=False, gap=3, limiter=1, bc=None, flux=0):
    dim = 3 if kind >= 2 else 2
    p = oracle.make_params(dim, level, steps, cfl=cfl, fixed_dt=fixed_dt, limiter=limiter,
                           bc=bc, eps=eps, eps_level=eps_level, min_leaf_level=min_leaf,
                           local_time=local_time, lt_gap=gap, flux=flux)
    return oracle.mr_run("ref", p, init)


def compare(init, out, keys, rep, ref):
    rout, rkeys, rcyc, rdt, rres = ref
    assert rres["err_kind"] == 0, rres["err"]
    assert len(rcyc) == len(rep.cycles)
    assert np.array_equal(rcyc[:, 0], rep.cycles[:, 0].astype(np.int64)), "leaves per cycle"
    assert np.array_equal(rcyc[:, 1], rep.cycles[:, 1].astype(np.int64)), "nodes per cycle"
    assert np.array_equal(rcyc[:, 2], rep.cycles[:, 2].astype(np.int64)), "sub per cycle"
    assert np.array_equal(bits(rdt), bits(rep.cycles[:, 4])), "dt per cycle"
    assert np.array_equal(rcyc[:, 4], rep.cycles[:, 5].astype(np.int64)), "updates per cycle"
    assert np.array_equal(rkeys, keys), "final leaf set"
    assert np.array_equal(bits(rout), bits(out)), "to_uniform(L) state"
    assert rep.max_cfl == rres["max_cfl"]
    assert rep.fallbacks == rres["fallbacks"]


CASES_GLOBAL = [
    # kind, seed, level, steps, kwargs
    (0, 1, 6, 20, dict(eps=1e-3)),
    (0, 2, 7, 25, dict(eps=2.3e-3, min_leaf=3)),
    (0, 3, 7, 20, dict(eps=1e-3, eps_level=eps_levels(1e-3, 7, 2), min_leaf=3)),   # cfg2 rule
    (1, 4, 6, 15, dict(eps=1e-3, limiter=0)),
    (0, 5, 6, 15, dict(eps=1e-3, bc=[1] * 6)),
    (0, 6, 6, 15, dict(eps=1e-3, bc=[2, 2, 0, 0, 0, 0])),
    (2, 7, 4, 6, dict(eps=1e-3, cfl=0.4)),
    (3, 8, 5, 4, dict(eps=1e-3, cfl=0.4, eps_level=eps_levels(1e-3, 5, 3), min_leaf=2)),
    (0, 31, 7, 20, dict(eps=1e-3, flux=1, min_leaf=3)),                        # AUSMDV
    (0, 33, 7, 3, dict(eps=2e-2, min_leaf=2)),       # heavy coarsening: to_uniform's far field
    (3, 32, 5, 4, dict(eps=1e-3, cfl=0.4, flux=1, limiter=0)),
]


@pytest.mark.parametrize("kind,seed,level,steps,kw", CASES_GLOBAL,
                         ids=[f"k{c[0]}_L{c[2]}_{i}" for i, c in enumerate(CASES_GLOBAL)])
def test_mr_global_matches_reference(gpu_lib, oracle, kind, seed, level, steps, kw):
    if not oracle.available("ref"):
        pytest.skip("reference build not present; golden fixtures cover MR")
    init, out, keys, rep = gpu_mr(kind, seed, level, steps, **kw)
    compare(init, out, keys, rep, ref_mr(oracle, init, kind, level, steps, **kw))


CASES_LT = [
    (0, 41, 6, 16, dict(eps=1e-3, local_time=True)),
    (1, 42, 7, 16, dict(eps=1e-3, local_time=True)),                       # cfg3 generator
    (0, 44, 7, 16, dict(eps=1e-3, local_time=True, gap=2, bc=[1] * 6)),
    (0, 45, 7, 12, dict(eps=2e-3, local_time=True, gap=4, limiter=0)),
    (2, 43, 5, 8, dict(eps=1e-3, cfl=0.4, local_time=True)),
    (3, 46, 5, 8, dict(eps=1e-3, cfl=0.4, local_time=True, gap=3,
                       eps_level=eps_levels(1e-3, 5, 3), min_leaf=1)),        # cfg5 rule
    (1, 47, 7, 12, dict(eps=1e-3, local_time=True, flux=1)),                 # AUSMDV, MRLT
]


@pytest.mark.parametrize("kind,seed,level,steps,kw", CASES_LT,
                         ids=[f"k{c[0]}_L{c[2]}_{i}" for i, c in enumerate(CASES_LT)])
def test_mr_local_time_matches_reference(gpu_lib, oracle, kind, seed, level, steps, kw):
    if not oracle.available("ref"):
        pytest.skip("reference build not present; golden fixtures cover MRLT")
    init, out, keys, rep = gpu_mr(kind, seed, level, steps, **kw)
    compare(init, out, keys, rep, ref_mr(oracle, init, kind, level, steps, **kw))


def test_mr_eps0_equals_uniform(gpu_lib):
    """with eps = 0 the MR solver is the uniform FV solver (bitwise)."""
    from paper_1603_05211_b200 import uniform as U
    init, out, keys, rep = gpu_mr(0, 9, 6, 12, eps=0.0, cfl=0.0, fixed_dt=1e-3)
    u, _ = U.run_uniform(init, 2, 6, 12, fixed_dt=1e-3)
    assert len(keys) == 64 * 64
    assert np.array_equal(bits(out), bits(u))


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_mr_matches_golden(gpu_lib, path):
    g = np.load(path, allow_pickle=False)
    kw = dict(cfl=float(g["cfl"]), fixed_dt=float(g["fixed_dt"]), eps=float(g["eps"]),
              min_leaf=int(g["min_leaf"]), local_time=bool(g["local_time"]), gap=int(g["gap"]),
              limiter=int(g["limiter"]), bc=[int(x) for x in g["bc"]])
    if int(g["has_eps_level"]):
        kw["eps_level"] = list(g["eps_level"])
    init, out, keys, rep = gpu_mr(int(g["kind"]), int(g["seed"]), int(g["level"]),
                                  int(g["steps"]), **kw)
    ref = (g["out"], g["keys"], g["cycles"], g["dt"],
           {"err_kind": 0, "err": "", "max_cfl": float(g["max_cfl"]),
            "fallbacks": int(g["fallbacks"])})
    compare(init, out, keys, rep, ref)


@pytest.mark.parametrize("kind,seed,level,steps,kw", [
    (0, 7, 6, 30, dict(cfl=3.0, eps=1e-3)),
    (2, 8, 5, 4, dict(cfl=2.0, eps=1e-3, min_leaf=2)),
])
def test_mr_nonphysical_message(gpu_lib, oracle, kind, seed, level, steps, kw):
    from paper_1603_05211_b200.errors import NonPhysicalState
    if not oracle.available("ref"):
        pytest.skip("reference build not present")
    from paper_1603_05211_b200 import uniform as U
    init = U.case_fill(kind, seed, level)
    ref = ref_mr(oracle, init, kind, level, steps, **kw)
    assert ref[4]["err_kind"] == 1
    with pytest.raises(NonPhysicalState) as ei:
        gpu_mr(kind, seed, level, steps, **kw)
    assert str(ei.value) == ref[4]["err"]


@pytest.mark.parametrize("kind,seed,level,steps,kw", CASES_GLOBAL[:4] + CASES_LT[:3],
                         ids=[f"c{i}" for i in range(7)])
def test_mr_sweep_skip_is_sound(gpu_lib, monkeypatch, kind, seed, level, steps, kw):
    """coarsen skips the re-sweep of mr_tree.cpp:474-510 when no merge touched a
    candidate's prediction stencil. AF_MR_FULL_SWEEPS runs every sweep and
    raises if a sweep after a 'clean' one merges; the results must not change."""
    base = gpu_mr(kind, seed, level, steps, **kw)
    monkeypatch.setenv("AF_MR_FULL_SWEEPS", "1")
    full = gpu_mr(kind, seed, level, steps, **kw)
    assert np.array_equal(base[2], full[2])
    assert np.array_equal(bits(base[1]), bits(full[1]))


EDGE = [
    (0, 61, 2, 6, dict(eps=1e-3)),                         # the smallest tree (4x4)
    (2, 62, 2, 4, dict(eps=1e-3, cfl=0.4)),                # 3D 4^3
    (0, 63, 6, 6, dict(eps=10.0, min_leaf=2)),             # everything coarsens to min_leaf
    (0, 64, 5, 8, dict(eps=0.0, local_time=True)),         # full tree under MRLT
    (1, 65, 6, 6, dict(eps=1e-3, min_leaf=6)),             # min_leaf = L: a uniform leaf set
]


@pytest.mark.parametrize("kind,seed,level,steps,kw", EDGE,
                         ids=[f"edge{i}" for i in range(len(EDGE))])
def test_mr_edge_cases_match_reference(gpu_lib, oracle, kind, seed, level, steps, kw):
    if not oracle.available("ref"):
        pytest.skip("reference build not present")
    init, out, keys, rep = gpu_mr(kind, seed, level, steps, **kw)
    compare(init, out, keys, rep, ref_mr(oracle, init, kind, level, steps, **kw))


REFINE_BUFFER = [
    # kind, seed, level, build eps, refine eps, buffer radius per level, bc
    (0, 71, 7, 1e-3, 1e-3, [1] * 8, None),
    (0, 72, 7, 2e-3, 1e-3, [0, 0, 1, 1, 2, 2, 3, 3], None),
    (1, 73, 7, 1e-3, 1e-3, [2, 2, 2], None),               # shorter than L+1
    (0, 74, 6, 1e-3, 5e-4, [], None),                      # no buffer, another eps
    (0, 75, 6, 1e-3, 1e-3, [1, 1, 2, 2, 2, 2, 2], [1] * 6),  # periodic wrap
    (0, 76, 6, 1e-3, 1e-3, [3] * 7, [2] * 6),              # reflective fold
    (2, 77, 5, 1e-3, 1e-3, [1, 1, 1, 2, 2, 2], None),      # 3D
]


@pytest.mark.parametrize("kind,seed,level,eps0,eps,buffer,bc", REFINE_BUFFER,
                         ids=[f"rb{i}" for i in range(len(REFINE_BUFFER))])
def test_refine_buffer_matches_reference(gpu_lib, oracle, kind, seed, level, eps0, eps, buffer,
                                         bc):
    """MRTree::refine(eps, buffer_radius_per_level) (mr_tree.hpp:141) through
    af_mr_refine_buffer: the same leaf set and to_uniform(L) as the
    reference's refine on the same starting tree."""
    if not oracle.available("ref"):
        pytest.skip("reference build not present")
    from paper_1603_05211_b200 import mr as M
    from paper_1603_05211_b200 import uniform as U
    dim = 3 if kind >= 2 else 2
    init = U.case_fill(kind, seed, level)
    s = M.MRSolver(dim, level, M.MROptions(epsilon=eps0), bc=bc)
    s.build(init)
    s.refine(eps=eps, buffer=buffer)
    keys, out = s.leaves(), s.to_uniform()
    s.close()
    p = oracle.make_params(dim, level, 1, eps=eps0, bc=bc)
    rout, rkeys = oracle.ref_mr_refine_once(p, init, eps, buffer)
    assert np.array_equal(keys, rkeys)
    assert np.array_equal(bits(out), bits(rout))
