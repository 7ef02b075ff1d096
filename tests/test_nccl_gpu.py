"""The NCCL transport (af_comm_create; uniform slab halo exchange overlapped with
the interior planes, MR status/value exchanges and reductions) on 2 GPUs of one
box, against one GPU: bit-identical states, dt histories, leaf sets and cycle
records. Skipped when fewer than 2 GPUs are visible (the round's GPU runs are
one GPU; the same multi-rank code runs with host-thread ranks in
tests/test_mr_dist_gpu.py and tests/test_multigpu.py)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from test_oracle import bits

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.skipif(_gpus() < 2, reason="needs 2 GPUs on one box")
def test_nccl_two_ranks_equal_one(gpu_lib, tmp_path):
    from paper_1603_05211_b200 import mr as M
    from paper_1603_05211_b200 import uniform as U
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533",
           os.path.join(HERE, "nccl_worker.py"), str(tmp_path)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    parts = [dict(np.load(tmp_path / f"rank{k}.npz")) for k in range(2)]
    level = 6
    for tol in (False, True):
        s = U.UniformSolver(3, level, scheme=U.SchemeConfig(limiter=U.MINMOD), bc=[0, 0, 0, 0, 1, 1])
        if tol:
            s.set_numerics(True)
        s.upload(U.case_fill(2, 5, level))
        rep = s.run(12, cfl=0.4)
        ref = s.download()
        s.close()
        got = np.concatenate([p[f"u{int(tol)}"] for p in parts])
        assert np.array_equal(bits(got), bits(ref)), f"uniform tol={tol}"
        for p in parts:
            assert np.array_equal(bits(p[f"u{int(tol)}_dt"]), bits(rep.dt))
    o = M.MROptions(epsilon=1e-3, local_time=True, local_time_level_gap=3)
    m = M.MRSolver(2, 8, o)
    m.build(U.case_fill(1, 9, 8))
    rep = m.run(16, cfl=0.5)
    ref_u, ref_k = m.to_uniform(), m.leaves()
    m.close()
    row = 1 << 8
    got = np.empty_like(ref_u)
    for p in parts:
        lo, hi = p["mr_rows"]
        got[lo * row:hi * row] = p["mr_u"][lo * row:hi * row]
        assert np.array_equal(p["mr_cycles"], rep.cycles)
    assert np.array_equal(bits(got), bits(ref_u))
    assert np.array_equal(np.sort(np.concatenate([p["mr_keys"] for p in parts])), ref_k)
