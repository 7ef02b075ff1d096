"""The multi-GPU uniform path (slab decomposition).

* GPU: n ranks emulated on one B200 (af_uniform_create_group: every per-rank
  code path of the NCCL run, halos by device-to-device copies) must be
  bitwise identical to the single-domain run for any rank count and BC.
* CPU: the slab partition (af_uniform_local_extent of every rank) tiles the
  mesh exactly, with 2D slabs in multiples of the tile height; and the
  torch.distributed plumbing bench.py uses for N>1 (broadcast of the 128-byte
  NCCL id, max/sum reductions of the timings) on a gloo world of 2.
"""
import os

import numpy as np
import pytest

from test_oracle import bits


@pytest.mark.gpu
@pytest.mark.parametrize("dim,level,ranks,bc,cfl,lim,integ", [
    (2, 6, 2, None, 0.5, 1, 0),
    (2, 7, 3, [1] * 6, 0.5, 1, 0),
    (2, 7, 4, [2, 2, 2, 2, 0, 0], 0.5, 0, 0),
    (3, 5, 2, None, 0.4, 1, 0),
    (3, 5, 4, [1] * 6, 0.4, 1, 0),
    (3, 5, 5, [0, 0, 2, 2, 1, 1], 0.4, 0, 0),
    (2, 7, 3, [1] * 6, 0.5, 1, 1),                 # MUSCL-Hancock
    (3, 5, 3, [0, 0, 2, 2, 1, 1], 0.3, 0, 1),
])
def test_group_equals_single(gpu_lib, dim, level, ranks, bc, cfl, lim, integ):
    from paper_1603_05211_b200 import uniform as U
    kind = 2 if dim == 3 else 0
    init = U.case_fill(kind, 77 + ranks, level)
    sc = U.SchemeConfig(limiter=lim, integrator=integ)
    single = U.UniformSolver(dim, level, scheme=sc, bc=bc)
    single.upload(init)
    r1 = single.run(8, cfl=cfl)
    a = single.download()
    grp = U.UniformGroup(dim, level, ranks, scheme=sc, bc=bc)
    grp.upload(init)
    r2 = grp.run(8, cfl=cfl)
    b = grp.download()
    assert np.array_equal(bits(r1.dt), bits(r2.dt))
    assert np.array_equal(bits(a), bits(b))
    assert r1.max_cfl == r2.max_cfl


@pytest.mark.parametrize("dim,level,P", [(2, 8, 8), (2, 6, 3), (3, 9, 8), (3, 5, 5), (3, 9, 7),
                                         (2, 13, 8)])
def test_slab_partition_tiles_the_mesh(gpu_lib_cpu, dim, level, P):
    """The library's own slab split (af_slab_extent = what Uniform::Uniform
    uses, af_uniform.cu): contiguous, non-empty slabs of whole tile rows
    that tile the slab axis; a rank count that would leave a rank empty is a
    ConfigError."""
    import ctypes as C
    lib = gpu_lib_cpu
    n = 1 << level
    quantum = 8 if dim == 2 else 2
    z = 0
    for r in range(P):
        z0, nz = C.c_int(), C.c_int()
        assert lib.af_slab_extent(dim, level, P, r, C.byref(z0), C.byref(nz)) == 0
        assert z0.value == z and nz.value >= quantum and nz.value % quantum == 0
        z += nz.value
    assert z == n
    z0, nz = C.c_int(), C.c_int()
    assert lib.af_slab_extent(dim, level, n // quantum + 1, 0, C.byref(z0), C.byref(nz)) != 0
    assert lib.af_slab_extent(dim, level, P, P, C.byref(z0), C.byref(nz)) != 0


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    uid = bytes(range(128)) if rank == 0 else bytes(128)
    obj = [uid]
    dist.broadcast_object_list(obj, src=0)
    t = torch.tensor([10.0 + rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    s = torch.tensor([1.0 + rank], dtype=torch.float64)
    dist.all_reduce(s, op=dist.ReduceOp.SUM)
    q.put((rank, obj[0] == bytes(range(128)), float(t.item()), float(s.item())))
    dist.destroy_process_group()


def test_distributed_plumbing_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert all(ok for _, ok, _, _ in res)
    assert all(mx == 11.0 and sm == 3.0 for _, _, mx, sm in res)
