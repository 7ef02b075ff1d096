"""One rank of the NCCL transport check (tests/test_nccl_gpu.py), launched by
torch.distributed.run: the 3D uniform solver on this rank's slab and the 2D
MR solver (MRLT, slab decomposition) over af_comm_create (NCCL), each rank
saving its part of the results to OUT_DIR/rank{r}.npz."""
import ctypes as C
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1603_05211_b200 import _abi  # noqa: E402
from paper_1603_05211_b200 import mr as M  # noqa: E402
from paper_1603_05211_b200 import uniform as U  # noqa: E402


def main():
    out_dir = sys.argv[1]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = _abi.load()
    uid = (C.c_ubyte * 128)()
    if rank == 0:
        assert lib.af_comm_unique_id(C.cast(uid, C.c_char_p)) == 0
    obj = [bytes(uid)]
    dist.broadcast_object_list(obj, src=0)
    uid = (C.c_ubyte * 128).from_buffer_copy(obj[0])
    comms = []
    for _ in range(2):  # one communicator per solver
        h = C.c_void_p()
        assert lib.af_comm_create(C.cast(uid, C.c_char_p), world, rank, local, C.byref(h)) == 0
        comms.append(h)
        dist.barrier()
        if rank == 0:
            assert lib.af_comm_unique_id(C.cast(uid, C.c_char_p)) == 0
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0)
        uid = (C.c_ubyte * 128).from_buffer_copy(obj[0])
    res = {}
    # 3D uniform, periodic z (wraps across ranks), tolerance and exact modes
    level = 6
    for tol in (False, True):
        s = U.UniformSolver(3, level, scheme=U.SchemeConfig(limiter=U.MINMOD), bc=[0, 0, 0, 0, 1, 1],
                            comm=comms[0], device=local)
        if tol:
            s.set_numerics(True)
        s.upload(U.case_fill(2, 5, level, z0=s.z0, nz=s.nz))
        rep = s.run(12, cfl=0.4)
        res[f"u{int(tol)}"] = s.download()
        res[f"u{int(tol)}_dt"] = rep.dt
        res["z0"], res["nz"] = s.z0, s.nz
        s.close()
    # 2D MRLT over the slab decomposition
    o = M.MROptions(epsilon=1e-3, local_time=True, local_time_level_gap=3)
    m = M.MRSolver(2, 8, o, comm=comms[1], device=local)
    m.build(U.case_fill(1, 9, 8))
    rep = m.run(16, cfl=0.5)
    lo, hi = m.local_rows(8)
    res["mr_rows"] = np.array([lo, hi])
    res["mr_u"] = m.to_uniform()
    res["mr_keys"] = m.leaves()
    res["mr_cycles"] = rep.cycles
    m.close()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
    for h in comms:
        lib.af_comm_destroy(h)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
