"""Times the 3D tile kernel at 512^3 (tolerance mode unless 'exact' is given)
for each AF_FV3D_CHUNKS value on the command line ('auto' = the host's choice).
usage: fv3d_time.py [exact] auto 2 5 ..."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1603_05211_b200 import uniform as U  # noqa: E402

exact = "exact" in sys.argv
init = torch.from_numpy(U.case_fill(2, 1, 9)).cuda()
for ch in [a for a in sys.argv[1:] if a != "exact"]:
    if ch == "auto":
        os.environ.pop("AF_FV3D_CHUNKS", None)
    else:
        os.environ["AF_FV3D_CHUNKS"] = ch
    os.environ["AF_FV3D_TILE"] = "1"
    s = U.UniformSolver(3, 9, scheme=U.SchemeConfig(limiter=1))
    if not exact:
        s.set_numerics(True)
    st = torch.cuda.Stream()
    s.set_stream(st)
    s.upload(init)
    s.run(3, cfl=0.4, collect=False)
    s.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    s.run(20, cfl=0.4, collect=False)
    e1.record(st)
    s.sync()
    ms = e0.elapsed_time(e1) / 20
    print(f"chunks={ch} exact={exact}: {ms:.3f} ms/step {512**3 * 2 / (ms / 1e3):.4e} cell-updates/s",
          flush=True)
    s.close()
