"""Ad-hoc GPU check of the 3D stage kernels: the TMA tile kernel against the
legacy kernel (bit for bit), tolerance mode against exact (relative L1), and
per-step timing at 512^3. Prints one line per check."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1603_05211_b200 import uniform as U  # noqa: E402


def run(level, steps, kind=2, seed=1, bc=None, legacy=False, tol=False, limiter=1, flux=0,
        cfl=0.4):
    os.environ["AF_FV3D_TILE"] = "0" if legacy else "1"
    s = U.UniformSolver(3, level, scheme=U.SchemeConfig(limiter=limiter, flux=flux), bc=bc)
    if tol:
        s.set_numerics(True)
    init = U.case_fill(kind, seed, level)
    s.upload(init)
    rep = s.run(steps, cfl=cfl)
    out = s.download()
    s.close()
    return out, rep


def bits(a):
    a = a.copy()
    a[a == 0] = 0
    return a.view(np.uint64)


def main():
    cases = [(4, 6, None, 1, 0), (5, 8, None, 1, 0), (5, 6, [2, 2, 1, 1, 0, 0], 1, 0),
             (6, 5, [1] * 6, 1, 0), (5, 5, None, 0, 0), (5, 5, None, 1, 1), (7, 10, None, 1, 0),
             (5, 4, [2] * 6, 0, 1)]
    for L, st, bc, lim, fl in cases:
        a, ra = run(L, st, bc=bc, limiter=lim, flux=fl)
        b, rb = run(L, st, bc=bc, legacy=True, limiter=lim, flux=fl)
        same = np.array_equal(bits(a), bits(b))
        print(f"L={L} bc={bc} lim={lim} flux={fl}: tile==legacy {same} "
              f"dt {np.array_equal(ra.dt, rb.dt)} wave {ra.max_wave_speed == rb.max_wave_speed} "
              f"fb {ra.fallbacks} {rb.fallbacks}", flush=True)
        t, rt = run(L, st, bc=bc, tol=True, limiter=lim, flux=fl)
        d = np.abs(t - a).sum(0) / np.maximum(np.abs(a).sum(0), 1e-300)
        print(f"   tol rel L1 {d.max():.3e}", flush=True)
    # timing at 512^3
    for legacy, tol in ((True, False), (False, False), (False, True)):
        os.environ["AF_FV3D_TILE"] = "0" if legacy else "1"
        s = U.UniformSolver(3, 9, scheme=U.SchemeConfig(limiter=1))
        if tol:
            s.set_numerics(True)
        st = torch.cuda.Stream()
        s.set_stream(st)
        init = torch.from_numpy(U.case_fill(2, 1, 9)).cuda()
        s.upload(init)
        s.run(3, cfl=0.4, collect=False)
        s.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        s.run(20, cfl=0.4, collect=False)
        e1.record(st)
        s.sync()
        ms = e0.elapsed_time(e1) / 20
        print(f"512^3 legacy={legacy} tol={tol}: {ms:.3f} ms/step "
              f"{512**3 * 2 / (ms / 1e3):.3e} cell-updates/s", flush=True)
        s.close()
    # full-size tolerance vs exact, 100 steps
    a, ra = run(9, 100)
    t, rt = run(9, 100, tol=True)
    d = np.abs(t - a).sum(0) / np.maximum(np.abs(a).sum(0), 1e-300)
    print(f"512^3 x 100 tol vs exact rel L1 per field {d}", flush=True)


if __name__ == "__main__":
    main()
