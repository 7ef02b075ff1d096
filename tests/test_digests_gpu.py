"""GPU parity at BASELINE.json's configs' own sizes (or the largest size the
single-threaded reference finishes in the build container),
against digests of the COMPILED REFERENCE's runs (tests/golden/digest_*.npz,
written by tests/golden/make_digests.py from oracle/_ref; the reference is
not on the GPU box):

  * cfg1  2D uniform 256^2 x 200 steps;
  * cfg2  rules (level thresholds, min leaf 3, global dt) over the config's own
          500 cycles at L=8 and at L=9 (the reference does not finish L=10 on
          one core here, tests/golden/make_digests.py);
  * cfg4  3D uniform at its own size, 512^3 x 100 steps (the reference's
          step_block on 8 host-thread z-slabs, bit for bit its single-block run;
          24 minutes here), and its generator at 128^3 x 100;
  * cfg3  2D MRLT generator (+-1 % density noise) at L=10 (32 finest steps)
          and at its own L=13 for one macro-cycle (8192^2, 8 finest steps,
          60.8 M leaves; 1.9 h of reference time here);
  * cfg5  3D MRLT rules (level thresholds, coarsest 16^3) at L=7.

Bit-exact mode must reproduce each digest exactly: the to_uniform(L) state's
SHA-256 (+-0 folded), the sorted leaf keys, every cycle record, the dt
history, max_cfl and fallbacks. A leaf-set mismatch is reported with the
north_star exemption check (deciding detail within 1e-12 relative of its
threshold) before the test fails."""
import glob
import os

import numpy as np
import pytest

import digests as D
from test_oracle import bits

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
DIGESTS = sorted(glob.glob(os.path.join(HERE, "golden", "digest_*.npz")))


def _name(p):
    return os.path.basename(p)[len("digest_"):-4]


def run_uniform(g, tolerance=False):
    from paper_1603_05211_b200 import uniform as U
    dim, level = int(g["dim"]), int(g["level"])
    s = U.UniformSolver(dim, level, scheme=U.SchemeConfig(limiter=U.MINMOD))
    if tolerance:
        s.set_numerics(True)
    s.upload(U.case_fill(int(g["kind"]), int(g["seed"]), level))
    rep = s.run(int(g["steps"]), cfl=float(g["cfl"]))
    out = s.download()
    s.close()
    return out, rep


def run_mr(g):
    from paper_1603_05211_b200 import mr as M
    from paper_1603_05211_b200 import uniform as U
    dim, level = int(g["dim"]), int(g["level"])
    epsl = list(g["eps_level"]) if int(g["has_eps_level"]) else None
    s = M.MRSolver(dim, level, M.MROptions(epsilon=float(g["eps"]), eps_level=epsl,
                                           min_leaf_level=int(g["min_leaf"]),
                                           local_time=bool(g["local_time"]),
                                           local_time_level_gap=int(g["gap"])),
                   scheme=U.SchemeConfig(limiter=U.MINMOD))
    s.build(U.case_fill(int(g["kind"]), int(g["seed"]), level))
    rep = s.run(int(g["steps"]), cfl=float(g["cfl"]))
    keys = s.leaves()
    out = s.to_uniform()
    return s, out, keys, rep


def _status_map(keys):
    """node key -> 'L' (leaf) / 'I' (internal) of a tree given its leaves."""
    st = {}
    for k in keys.tolist():
        st[k] = "L"
    for k in keys.tolist():
        lvl, i, j, kk = k >> 45, (k >> 30) & 0x7FFF, (k >> 15) & 0x7FFF, k & 0x7FFF
        while lvl > 0:
            lvl, i, j, kk = lvl - 1, i >> 1, j >> 1, kk >> 1
            p = (lvl << 45) | (i << 30) | (j << 15) | kk
            if st.get(p) == "I":
                break
            st[p] = "I"
    return st


def exemption_report(solver, g, gpu_keys, ref_keys):
    """Nodes where the two trees first disagree (leaf on one side, internal on
    the other, parents agreeing), with the GPU's details of the node and of
    its parent against their thresholds (mr_tree.cpp:366-371 refine, :498
    coarsen; eps indexed by the children's level). Returns the list of
    disagreements NOT within 1e-12 relative of a threshold."""
    dim, L = int(g["dim"]), int(g["level"])
    epsl = (list(g["eps_level"]) if int(g["has_eps_level"])
            else [float(g["eps"])] * (L + 1))
    sg, sr = _status_map(gpu_keys), _status_map(ref_keys)
    det_cache = {}

    def detail(key):
        lvl = key >> 45
        if lvl not in det_cache:
            det_cache[lvl] = solver.details(lvl)
        n = 1 << lvl
        i, j, k = (key >> 30) & 0x7FFF, (key >> 15) & 0x7FFF, key & 0x7FFF
        return det_cache[lvl][i + n * j + (n * n * k if dim == 3 else 0)]

    bad = []
    for key in set(sg) | set(sr):
        if sg.get(key) == sr.get(key):
            continue
        lvl = key >> 45
        if lvl > 0:
            i, j, k = (key >> 30) & 0x7FFF, (key >> 15) & 0x7FFF, key & 0x7FFF
            parent = ((lvl - 1) << 45) | ((i >> 1) << 30) | ((j >> 1) << 15) | (k >> 1)
            if sg.get(parent) != sr.get(parent):
                continue  # not the root of this disagreement
        else:
            parent = None
        near = False
        for node, eps in ((key, epsl[min(lvl + 1, L)]),
                          (parent, epsl[lvl]) if parent is not None else (None, None)):
            if node is None or sg.get(node) != "I":
                continue
            d = detail(node)
            if np.isfinite(d) and abs(d / eps - 1.0) <= 1e-12:
                near = True
        if not near:
            bad.append(key)
    return bad


@pytest.mark.parametrize("path", DIGESTS, ids=[_name(p) for p in DIGESTS])
def test_matches_reference_digest(gpu_lib, path):
    g = np.load(path, allow_pickle=False)
    if int(g["mr"]) == 0:
        out, rep = run_uniform(g)
        assert np.array_equal(bits(rep.dt), bits(g["dt"])), "dt history"
        assert D.state_sha(out) == str(g["state_sha"]), "final state"
        assert rep.max_cfl == float(g["max_cfl"])
        assert rep.max_wave_speed == float(g["max_wave_speed"])
        assert rep.fallbacks == int(g["fallbacks"])
        return
    s, out, keys, rep = run_mr(g)
    try:
        cyc = g["cycles"]
        assert len(cyc) == len(rep.cycles), "cycle count"
        assert np.array_equal(cyc[:, 0], rep.cycles[:, 0].astype(np.int64)), "leaves per cycle"
        assert np.array_equal(cyc[:, 1], rep.cycles[:, 1].astype(np.int64)), "nodes per cycle"
        assert np.array_equal(cyc[:, 2], rep.cycles[:, 2].astype(np.int64)), "sub per cycle"
        assert np.array_equal(bits(g["dt"]), bits(rep.cycles[:, 4])), "dt per cycle"
        assert np.array_equal(cyc[:, 4], rep.cycles[:, 5].astype(np.int64)), "updates per cycle"
        if D.keys_sha(keys) != str(g["keys_sha"]):
            msg = (f"leaf set differs: {len(keys)} vs {int(g['n_keys'])} leaves; per level "
                   f"{D.leaves_per_level(keys, int(g['level']))} vs {g['leaves_per_level']}")
            if "leaf_bitmaps" in g.files:
                ref_keys = D.bitmaps_to_keys(g["leaf_bitmaps"], int(g["dim"]), int(g["level"]))
                bad = exemption_report(s, g, keys, ref_keys)
                msg += f"; {len(bad)} disagreements outside the 1e-12 threshold exemption"
            pytest.fail(msg)
        assert D.state_sha(out) == str(g["state_sha"]), "to_uniform(L) state"
        assert rep.max_cfl == float(g["max_cfl"])
        assert rep.fallbacks == int(g["fallbacks"])
    finally:
        s.close()


def test_digest_coarse_fields_consistent(gpu_lib):
    """The digests' coarse fields are the restriction of their own states:
    the GPU's restricted state matches them to round-off (sanity of the
    tolerance checks' reference field)."""
    path = os.path.join(HERE, "golden", "digest_cfg4_128.npz")
    if not os.path.exists(path):
        pytest.skip("digest missing")
    g = np.load(path, allow_pickle=False)
    out, _ = run_uniform(g)
    c = D.coarse(out, int(g["dim"]), int(g["level"]), int(g["coarse_level"]))
    assert np.array_equal(bits(c), bits(g["coarse"]))
    assert np.allclose(D.state_l1(out), g["state_l1"], rtol=1e-14, atol=0)
