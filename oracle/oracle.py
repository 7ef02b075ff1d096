"""oracle.py — TEST INFRASTRUCTURE ONLY: ctypes access to the two CPU oracles.

  * ``ref``  — oracle/_ref/libafref.so: the reference library compiled from
    /root/reference sources (oracle/Makefile) + ref_harness.cpp.
  * ``port`` — oracle/_build/libaforacle.so: the plain-C restatement.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libafref.so")
PORT_SO = os.path.join(HERE, "_build", "libaforacle.so")
REFERENCE_SRC = "/root/reference/proj/core"

CASE_QUADRANTS, CASE_QUADRANTS_NOISE, CASE_ELLIPSOID, CASE_ELLIPSOID_PRATIO = 0, 1, 2, 3
OUTFLOW, PERIODIC, REFLECTIVE = 0, 1, 2
VAN_ALBADA, MINMOD = 0, 1


class Params(C.Structure):
    _fields_ = [
        ("dim", C.c_int), ("level", C.c_int), ("bc", C.c_int * 6), ("limiter", C.c_int),
        ("flux", C.c_int), ("gamma", C.c_double), ("n_steps", C.c_long), ("cfl", C.c_double),
        ("fixed_dt", C.c_double), ("eps", C.c_double), ("eps_level", C.POINTER(C.c_double)),
        ("min_leaf_level", C.c_int), ("local_time", C.c_int), ("lt_gap", C.c_int),
        ("integrator", C.c_int),
    ]


class Result(C.Structure):
    _fields_ = [
        ("max_wave_speed", C.c_double), ("max_cfl", C.c_double), ("fallbacks", C.c_long),
        ("wall_seconds", C.c_double), ("n_cycles", C.c_long), ("steps_done", C.c_long),
        ("err_kind", C.c_int), ("err", C.c_char * 512),
    ]

    def as_dict(self):
        return {k: (getattr(self, k).decode() if k == "err" else getattr(self, k))
                for k, _ in self._fields_}


def build(force: bool = False, ref: bool = True) -> None:
    """Builds the restatement (always) and the reference (when its sources exist)."""
    targets = ["oracle"]
    if ref and os.path.isdir(REFERENCE_SRC):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + (["-B"] if force else []) + targets,
                   check=True)


_libs: dict = {}


def _load(kind: str):
    if kind in _libs:
        return _libs[kind]
    path = REF_SO if kind == "ref" else PORT_SO
    if not os.path.exists(path):
        raise FileNotFoundError(f"oracle library {path} missing (run `make -C oracle`)")
    lib = C.CDLL(path)
    pre = "afref_" if kind == "ref" else "afo_"
    dp = C.POINTER(C.c_double)
    for name, args in [
        ("uniform_run", [C.POINTER(Params), dp, dp, dp, C.POINTER(Result)]),
        ("mr_run", [C.POINTER(Params), dp, dp, C.POINTER(C.c_uint64), C.POINTER(C.c_long),
                    C.POINTER(C.c_long), C.c_long, dp, C.POINTER(Result)]),
        ("mr_last_dump", [C.c_char_p]),
    ]:
        f = getattr(lib, pre + name)
        f.argtypes = args
        f.restype = C.c_int
    if kind == "port":
        lib.afo_case_fill.argtypes = [C.c_int, C.c_uint64, C.c_int, C.c_double, C.c_int,
                                      C.c_int, dp]
        lib.afo_case_fill.restype = C.c_int
    else:  # formats and compare path of the reference (ref_harness.cpp)
        for name, args in [
            ("snapshot_copy", [C.c_char_p, C.c_char_p, C.c_char_p, C.c_int]),
            ("restrict", [C.c_int, C.c_int, C.c_int, dp, dp]),
            ("l1_error", [C.c_int, C.c_int, C.c_double, dp, C.c_int, dp, dp]),
            ("uniform_window_run", [C.POINTER(Params), C.c_int, C.c_int, C.c_int, C.c_long,
                                    dp, dp, C.POINTER(Result), dp]),
            ("mr_refine_once", [C.POINTER(Params), dp, C.c_double, C.POINTER(C.c_int), C.c_int,
                                dp, C.POINTER(C.c_uint64), C.POINTER(C.c_long)]),
            ("rk2_stage", [C.POINTER(Params), dp, dp, C.c_double, dp, dp, C.POINTER(Result)]),
            ("rates", [dp, C.c_long, dp, C.c_long, C.c_double, dp, C.c_char_p, C.c_int]),
        ]:
            f = getattr(lib, "afref_" + name)
            f.argtypes = args
            f.restype = C.c_int
    _libs[kind] = lib
    return lib


def available(kind: str) -> bool:
    return os.path.exists(REF_SO if kind == "ref" else PORT_SO)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def case_fill(kind: int, seed: int, level: int, gamma: float = 1.4, z0: int = 0,
              nz: int | None = None) -> np.ndarray:
    """Seeded initial data (include/af_cases.h), shape (cells, 5) AoS."""
    lib = _load("port")
    dim = 3 if kind in (CASE_ELLIPSOID, CASE_ELLIPSOID_PRATIO) else 2
    n = 1 << level
    nz = n if nz is None else nz
    out = np.zeros((nz * n ** (dim - 1), 5), dtype=np.float64)
    rc = lib.afo_case_fill(kind, seed, level, gamma, z0, nz, _dp(out))
    if rc:
        raise ValueError("af_case_fill rejected its arguments")
    return out


def make_params(dim, level, n_steps, cfl=0.5, fixed_dt=0.0, limiter=MINMOD, bc=None,
                gamma=1.4, eps=0.0, eps_level=None, min_leaf_level=0, local_time=False,
                lt_gap=3, flux=0, integrator=0):
    p = Params()
    p.dim, p.level, p.n_steps = dim, level, n_steps
    for f in range(6):
        p.bc[f] = OUTFLOW if bc is None else bc[f]
    p.limiter, p.flux, p.gamma = limiter, flux, gamma
    p.integrator = integrator
    p.cfl, p.fixed_dt = cfl, fixed_dt
    p.eps = eps
    keep = None
    if eps_level is not None:
        keep = np.ascontiguousarray(eps_level, dtype=np.float64)
        p.eps_level = _dp(keep)
    p.min_leaf_level, p.local_time, p.lt_gap = min_leaf_level, int(local_time), lt_gap
    p._keep = keep  # keep the table alive with the struct
    return p


def uniform_run(kind: str, params: Params, init: np.ndarray):
    lib = _load(kind)
    out = np.zeros_like(init)
    dts = np.zeros(max(params.n_steps, 1), dtype=np.float64)
    res = Result()
    fn = lib.afref_uniform_run if kind == "ref" else lib.afo_uniform_run
    fn(C.byref(params), _dp(np.ascontiguousarray(init)), _dp(out), _dp(dts), C.byref(res))
    return out, dts[: params.n_steps], res.as_dict()


def rk2_stage(params: Params, base: np.ndarray, eval_: np.ndarray, stage_dt: float,
              capture: bool = False):
    """The reference's rk2_stage (step.hpp:62-64) on the level-`params.level`
    mesh (ref_harness.cpp). Returns (out, result, flux) with flux the
    FluxField capture as per-axis arrays of shape (n_c, n_b, n_a+1, 5)."""
    lib = _load("ref")
    out = np.zeros_like(base)
    n, dim = 1 << params.level, params.dim
    per = (n + 1) * n ** (dim - 1)
    cap = np.zeros(dim * per * 5) if capture else None
    res = Result()
    lib.afref_rk2_stage(C.byref(params), _dp(np.ascontiguousarray(base)),
                        _dp(np.ascontiguousarray(eval_)), stage_dt, _dp(out),
                        _dp(cap) if cap is not None else None, C.byref(res))
    flux = None
    if cap is not None:
        flux = []
        for a in range(dim):
            shape = [n] * dim
            shape[a] += 1
            flux.append(cap[a * per * 5:(a + 1) * per * 5].reshape(*shape[::-1], 5))
    return out, res.as_dict(), flux


def window_init(kind: int, seed: int, level: int, z0: int, nz: int) -> np.ndarray:
    """The planes z0-2 .. z0+nz+1 (clamped into the mesh) of the seeded 3D
    initial state, as afref_uniform_window_run takes them."""
    n = 1 << level
    lo, hi = max(0, z0 - 2), min(n, z0 + nz + 2)
    return case_fill(kind, seed, level, z0=lo, nz=hi - lo)


def uniform_window_run(params: Params, init: np.ndarray, z0: int, nz: int, threads: int,
                       n_warm: int = 0, want_out: bool = False, want_dt: bool = False):
    """The reference's step_block on `threads` z-slabs of the window
    [z0, z0+nz) of the 3D mesh (ref_harness.cpp). Returns (out or None, result)
    or, with want_dt, (out or None, dt history, result). With z0 = 0, nz = n
    this is afref_uniform_run bit for bit, on `threads` host cores."""
    lib = _load("ref")
    n = 1 << params.level
    out = np.zeros((nz * n * n, 5)) if want_out else None
    dts = np.zeros(max(params.n_steps, 1)) if want_dt else None
    res = Result()
    lib.afref_uniform_window_run(C.byref(params), z0, nz, threads, n_warm,
                                 _dp(np.ascontiguousarray(init)),
                                 _dp(out) if want_out else None, C.byref(res),
                                 _dp(dts) if want_dt else None)
    if want_dt:
        return out, dts[: params.n_steps], res.as_dict()
    return out, res.as_dict()


def ref_mr_refine_once(params: Params, init: np.ndarray, eps: float, buffer):
    """The reference's MRTree::refine(eps, buffer) once on run_mr's starting
    tree: (to_uniform(L), sorted leaf keys)."""
    lib = _load("ref")
    out = np.zeros_like(init)
    keys = np.zeros(init.shape[0] + 1, dtype=np.uint64)
    nl = C.c_long(keys.shape[0])
    buf = (C.c_int * max(1, len(buffer)))(*[int(b) for b in buffer])
    rc = lib.afref_mr_refine_once(C.byref(params), _dp(np.ascontiguousarray(init)), eps, buf,
                                  len(buffer), _dp(out),
                                  keys.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(nl))
    if rc:
        raise RuntimeError("afref_mr_refine_once failed")
    return out, keys[: nl.value].copy()


def mr_run(kind: str, params: Params, init: np.ndarray, max_cycles: int | None = None,
           dump_path: str | None = None):
    lib = _load(kind)
    out = np.zeros_like(init)
    max_cycles = params.n_steps if max_cycles is None else max_cycles
    per_cycle = np.zeros((max_cycles, 5), dtype=np.int64)
    dts = np.zeros(max_cycles, dtype=np.float64)
    cap = init.shape[0] + 1
    keys = np.zeros(cap, dtype=np.uint64)
    nl = C.c_long(cap)
    res = Result()
    fn = lib.afref_mr_run if kind == "ref" else lib.afo_mr_run
    fn(C.byref(params), _dp(np.ascontiguousarray(init)), _dp(out),
       keys.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(nl),
       per_cycle.ctypes.data_as(C.POINTER(C.c_long)), max_cycles, _dp(dts), C.byref(res))
    r = res.as_dict()
    nc = min(r["n_cycles"], max_cycles)
    if dump_path is not None:
        (lib.afref_mr_last_dump if kind == "ref" else lib.afo_mr_last_dump)(
            dump_path.encode())
    return out, keys[: nl.value].copy(), per_cycle[:nc].copy(), dts[:nc].copy(), r


def ref_snapshot_copy(src: str, dst: str):
    """The reference's read_snapshot(src) + write_snapshot(dst); returns the
    IoError text or None."""
    lib = _load("ref")
    err = C.create_string_buffer(512)
    rc = lib.afref_snapshot_copy(src.encode(), dst.encode(), err, 512)
    return err.value.decode() if rc else None


def ref_restrict(state: np.ndarray, dim: int, level: int, target: int) -> np.ndarray:
    lib = _load("ref")
    out = np.zeros(((1 << (dim * target)), 5), dtype=np.float64)
    if lib.afref_restrict(dim, level, target, _dp(np.ascontiguousarray(state)), _dp(out)):
        raise ValueError("restrict_to_level failed")
    return out


def ref_l1_error(sol, dim, level, ref, ref_level, extent=1.0) -> np.ndarray:
    lib = _load("ref")
    out = np.zeros(5, dtype=np.float64)
    if lib.afref_l1_error(dim, level, extent, _dp(np.ascontiguousarray(sol)), ref_level,
                          _dp(np.ascontiguousarray(ref)), _dp(out)):
        raise ValueError("l1_error failed")
    return out


def rates(adaptive: dict, fv: dict, n_c: float):
    """The reference's rates() (metrics.cpp:91-132). Returns (dict, None) or
    (None, the DivisionDomain text)."""
    lib = _load("ref")

    def vec(d):
        return np.array([d["wall_seconds"], d["sum_cells"], d["sum_leaves"], d["l1_rho"]])
    out = np.zeros(5)
    err = C.create_string_buffer(512)
    a, f = vec(adaptive), vec(fv)
    if lib.afref_rates(_dp(a), int(adaptive["n_steps"]), _dp(f), int(fv["n_steps"]), n_c, _dp(out),
                       err, 512):
        return None, err.value.decode()
    keys = ["cpu_compression", "memory_compression", "mesh_compression", "perturbation", "overhead"]
    return dict(zip(keys, out.tolist())), None


# ---- AMR patch path, reference side (ref_harness.cpp) ----------------------
class AmrRefParams(C.Structure):
    _fields_ = [("dim", C.c_int), ("level", C.c_int), ("base_exp", C.c_int), ("bc", C.c_int * 6),
                ("limiter", C.c_int), ("flux", C.c_int), ("integrator", C.c_int),
                ("gamma", C.c_double), ("n_steps", C.c_long), ("dt_finest", C.c_double),
                ("eps_rho", C.c_double), ("eps_p", C.c_double), ("efficiency", C.c_double),
                ("time_refine", C.c_int), ("flux_correction", C.c_int), ("case_kind", C.c_int),
                ("seed", C.c_uint64), ("mode", C.c_int), ("builtin_name", C.c_char_p)]


def _amr_lib():
    lib = _load("ref")
    if not getattr(lib, "_amr_ready", False):
        dp = C.POINTER(C.c_double)
        lp = C.POINTER(C.c_long)
        ip = C.POINTER(C.c_int)
        lib.afref_amr_run.argtypes = [C.POINTER(AmrRefParams), lp, lp, C.POINTER(Result)]
        lib.afref_amr_run.restype = C.c_int
        lib.afref_amr_n_levels.restype = C.c_int
        lib.afref_amr_n_patches.argtypes = [C.c_int]
        lib.afref_amr_n_patches.restype = C.c_int
        lib.afref_amr_boxes.argtypes = [C.c_int, ip]
        lib.afref_amr_boxes.restype = C.c_int
        lib.afref_amr_time.argtypes = [C.c_int, C.c_int]
        lib.afref_amr_time.restype = C.c_double
        lib.afref_amr_patch_data.argtypes = [C.c_int, C.c_int, C.c_int, dp]
        lib.afref_amr_patch_data.restype = C.c_long
        lib.afref_amr_total_conserved.argtypes = [dp]
        lib.afref_amr_dump_boxes.argtypes = [C.c_char_p, C.c_long]
        lib.afref_amr_l1_error.argtypes = [C.c_int, dp, dp, C.c_char_p, C.c_int]
        lib.afref_cluster.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_int, C.c_double, ip,
                                      C.c_int]
        lib.afref_cluster.restype = C.c_int
        lib._amr_ready = True
    return lib


def ref_amr_run(dim, level, base_exp, n_steps, dt_finest, case_kind=0, seed=1, bc=None,
                limiter=MINMOD, flux=0, integrator=0, gamma=1.4, eps_rho=0.05, eps_p=0.05,
                efficiency=0.8, time_refine=True, flux_correction=True, mode=0, builtin=None):
    """Runs the reference's AMR path (see af_oracle.h af_amr_ref_params) and
    returns everything the parity tests compare."""
    lib = _amr_lib()
    p = AmrRefParams()
    p.dim, p.level, p.base_exp = dim, level, base_exp
    for i, b in enumerate(bc if bc is not None else [0] * 6):
        p.bc[i] = int(b)
    p.limiter, p.flux, p.integrator, p.gamma = limiter, flux, integrator, gamma
    p.n_steps, p.dt_finest = n_steps, dt_finest
    p.eps_rho, p.eps_p, p.efficiency = eps_rho, eps_p, efficiency
    p.time_refine, p.flux_correction = int(time_refine), int(flux_correction)
    p.case_kind, p.seed, p.mode = case_kind, seed, mode
    p.builtin_name = builtin.encode() if builtin else None
    cps = np.zeros(n_steps, dtype=np.int64)
    lps = np.zeros(n_steps, dtype=np.int64)
    res = Result()
    lp = C.POINTER(C.c_long)
    lib.afref_amr_run(C.byref(p), cps.ctypes.data_as(lp), lps.ctypes.data_as(lp), C.byref(res))
    out = {"err_kind": res.err_kind, "err": res.err.decode(errors="replace"),
           "max_cfl": res.max_cfl, "fallbacks": res.fallbacks, "wall_seconds": res.wall_seconds,
           "cells_per_step": cps, "leaves_per_step": lps, "levels": []}
    if res.err_kind:
        return out
    buf = C.create_string_buffer(1 << 22)
    lib.afref_amr_dump_boxes(buf, len(buf))
    out["dump_boxes"] = buf.value.decode()
    tot = np.zeros(5)
    lib.afref_amr_total_conserved(_dp(tot))
    out["total_conserved"] = tot
    for l in range(lib.afref_amr_n_levels()):
        nb = lib.afref_amr_n_patches(l)
        boxes = np.zeros((max(nb, 1), 6), dtype=np.int32)
        lib.afref_amr_boxes(l, boxes.ctypes.data_as(C.POINTER(C.c_int)))
        lv = {"boxes": boxes[:nb], "t": lib.afref_amr_time(l, 0), "t_old": lib.afref_amr_time(l, 1)}
        for name, ghost, old in (("data", 0, 0), ("blocks", 2, 0), ("blocks_old", 2, 1)):
            n = lib.afref_amr_patch_data(l, ghost, old, None)
            a = np.zeros((n, 5))
            lib.afref_amr_patch_data(l, ghost, old, _dp(a))
            lv[name] = a
        out["levels"].append(lv)
    return out


def ref_cluster(flags: np.ndarray, efficiency: float, allowed: np.ndarray | None = None):
    """The reference's cluster() on a cubic mask indexed [z][y][x] / [y][x]."""
    lib = _amr_lib()
    f = np.ascontiguousarray(flags, dtype=np.uint8)
    a = None if allowed is None else np.ascontiguousarray(allowed, dtype=np.uint8)
    n = f.shape[-1]
    cap = int(f.sum()) + 1
    out = np.zeros((cap, 6), dtype=np.int32)
    k = lib.afref_cluster(f.ctypes.data_as(C.c_char_p),
                          None if a is None else a.ctypes.data_as(C.c_char_p), f.ndim, n,
                          efficiency, out.ctypes.data_as(C.POINTER(C.c_int)), cap)
    return out[:k]


def ref_amr_l1_error(ref: np.ndarray, ref_level: int):
    """l1_error_amr of the hierarchy the last ref_amr_run kept."""
    lib = _amr_lib()
    out = np.zeros(5)
    err = C.create_string_buffer(512)
    r = np.ascontiguousarray(ref, dtype=np.float64)
    rc = lib.afref_amr_l1_error(ref_level, _dp(r), _dp(out), err, len(err))
    if rc:
        raise RuntimeError(err.value.decode(errors="replace"))
    return out
