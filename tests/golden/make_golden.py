"""Regenerates tests/golden/*.npz from the COMPILED REFERENCE (oracle/_ref,
built from /root/reference sources by oracle/Makefile). Run in the build
container (the reference is not on the GPU box):

    python tests/golden/make_golden.py

Each fixture holds the seeded input parameters, the reference's final state,
its per-step dt and its RunReport scalars.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# name: (case kind, seed, level, steps, cfl, fixed_dt, limiter, bc)
UNIFORM = {
    "u2d_quad_L5_minmod": (0, 11, 5, 12, 0.5, 0.0, O.MINMOD, None),
    "u2d_quad_L6_vanalbada_fixed": (0, 12, 6, 10, 0.0, 2e-3, O.VAN_ALBADA, None),
    "u2d_noise_L5_periodic": (1, 13, 5, 8, 0.5, 0.0, O.MINMOD, [1] * 6),
    "u2d_quad_L5_reflective": (0, 14, 5, 8, 0.5, 0.0, O.MINMOD, [2] * 6),
    "u3d_ell_L4_minmod": (2, 21, 4, 6, 0.4, 0.0, O.MINMOD, None),
    "u3d_ellp_L4_mixed": (3, 22, 4, 4, 0.2, 0.0, O.MINMOD, [2, 2, 1, 1, 0, 0]),
    "u2d_quad_L5_blowup": (0, 7, 5, 20, 3.0, 0.0, O.MINMOD, None),
}


def eps_levels(eps, L, d):
    return [eps * 2.0 ** (d * (l - L)) for l in range(L + 1)]


# name: (kind, seed, level, steps, cfl, fixed_dt, eps, eps_level, min_leaf, local_time, gap,
#        limiter, bc)
MR = {
    "mr_quad_L6_global": (0, 31, 6, 12, 0.5, 0.0, 1e-3, None, 0, 0, 3, O.MINMOD, None),
    "mr_quad_L7_epsl_min3": (0, 32, 7, 12, 0.5, 0.0, 1e-3, eps_levels(1e-3, 7, 2), 3, 0, 3,
                             O.MINMOD, None),
    "mr_ell_L4_global": (2, 33, 4, 4, 0.4, 0.0, 1e-3, None, 0, 0, 3, O.MINMOD, None),
    "mr_quad_L6_lt": (0, 34, 6, 16, 0.5, 0.0, 1e-3, None, 0, 1, 3, O.MINMOD, None),
    "mr_noise_L7_lt": (1, 35, 7, 8, 0.5, 0.0, 1e-3, None, 0, 1, 3, O.MINMOD, None),
}


def main():
    O.build()
    for name, (kind, seed, level, steps, cfl, fdt, eps, epsl, mleaf, lt, gap, lim,
               bc) in MR.items():
        dim = 3 if kind >= 2 else 2
        init = O.case_fill(kind, seed, level)
        p = O.make_params(dim, level, steps, cfl=cfl, fixed_dt=fdt, limiter=lim, bc=bc, eps=eps,
                          eps_level=epsl, min_leaf_level=mleaf, local_time=lt, lt_gap=gap)
        out, keys, cyc, dts, res = O.mr_run("ref", p, init)
        assert res["err_kind"] == 0, res["err"]
        np.savez_compressed(
            os.path.join(HERE, name + ".npz"), kind=kind, seed=seed, level=level, steps=steps,
            cfl=cfl, fixed_dt=fdt, eps=eps, has_eps_level=int(epsl is not None),
            eps_level=np.array(epsl if epsl else [0.0]), min_leaf=mleaf, local_time=lt,
            gap=gap, limiter=lim, bc=np.array(bc if bc else [0] * 6), out=out, keys=keys,
            cycles=cyc, dt=dts, max_cfl=res["max_cfl"], fallbacks=res["fallbacks"])
        print(name, len(keys), "leaves", res["max_cfl"])
    for name, (kind, seed, level, steps, cfl, fdt, lim, bc) in UNIFORM.items():
        dim = 3 if kind >= 2 else 2
        init = O.case_fill(kind, seed, level)
        p = O.make_params(dim, level, steps, cfl=cfl, fixed_dt=fdt, limiter=lim, bc=bc)
        out, dts, res = O.uniform_run("ref", p, init)
        np.savez_compressed(
            os.path.join(HERE, name + ".npz"), kind=kind, seed=seed, level=level, steps=steps,
            cfl=cfl, fixed_dt=fdt, limiter=lim, bc=np.array(bc if bc else [0] * 6),
            out=out, dt=dts, max_cfl=res["max_cfl"], max_wave_speed=res["max_wave_speed"],
            fallbacks=res["fallbacks"], err=res["err"], err_kind=res["err_kind"])
        print(name, res["err"] or "ok", res["max_cfl"])


if __name__ == "__main__":
    main()
