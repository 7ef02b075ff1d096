"""Host-side mirror of the reference's AMR patch path over the C ABI.

Reference seams (paths under /root/reference/proj/core):
  * ``PatchHierarchy``  — amr.hpp:123-242 (initialize, sync_ghosts, remesh,
    update_level, average_down, flux_correct, total_conserved, total_cells,
    composite_cells, properly_nested, dump_boxes, assemble_level)
  * ``cluster``         — amr.hpp:110-111 (amr_cluster.cpp:79-232)
  * ``run_amr``         — amr_solver.hpp:34-35 (amr_solver.cpp:62-133)

Patch data live in libafgpu.so's device arrays (sm_100a); there is no CPU
fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from .errors import raise_status
from .uniform import AUSM_PLUS, MINMOD, OUTFLOW, RK2, SchemeConfig, StepDiag

AUSMDV = 1
MUSCL_HANCOCK = 1


@dataclass
class AmrOptions:
    """AmrOptions (amr.hpp:113-120)."""
    eps_rho: float = 0.05
    eps_p: float = 0.05
    cluster_efficiency: float = 0.8
    time_refine: bool = True
    flux_correction: bool = True
    max_levels: int = 0


@dataclass
class AmrReport:
    """The RunReport fields run_amr fills (amr_solver.cpp:80-131)."""
    level: int = 0
    n_steps: int = 0
    max_cfl: float = 0.0
    fallbacks: int = 0
    t: float = 0.0
    cells_per_step: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    leaves_per_step: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))


def amr_base_exp(dim: int, level: int) -> int:
    """amr_base_exp (amr_solver.cpp:8-11): the paper's base mesh (64^2, 8^3) once
    the level allows it, one level below the target otherwise."""
    return min(3 if dim == 3 else 6, level - 1)


def cluster(flags: np.ndarray, efficiency: float, allowed: np.ndarray | None = None):
    """cluster (amr.hpp:110-111). flags/allowed: uint8 masks indexed [z][y][x]
    (or [y][x]); returns the boxes as an (n, 6) int array (lo[3], hi[3])."""
    lib = _abi.load()
    f = np.ascontiguousarray(flags, dtype=np.uint8)
    dim = f.ndim
    if dim not in (2, 3):
        raise ValueError("cluster: masks are 2D or 3D")
    a = None if allowed is None else np.ascontiguousarray(allowed, dtype=np.uint8)
    if a is not None and a.shape != f.shape:
        raise ValueError("cluster: allowed must have the shape of flags")
    n0, n1, n2 = f.shape[-1], f.shape[-2], (f.shape[0] if dim == 3 else 1)
    n = C.c_int(0)
    fp = f.ctypes.data_as(C.c_char_p)
    ap = None if a is None else a.ctypes.data_as(C.c_char_p)
    raise_status(lib.af_amr_cluster(fp, ap, dim, n0, n1, n2, efficiency, None, 0, C.byref(n)),
                 "af_amr_cluster")
    out = np.zeros((max(n.value, 1), 6), dtype=np.int32)
    raise_status(lib.af_amr_cluster(fp, ap, dim, n0, n1, n2, efficiency,
                                    out.ctypes.data_as(C.POINTER(C.c_int)), n.value, C.byref(n)),
                 "af_amr_cluster")
    return out[:n.value]


def cluster_device(flags: np.ndarray, efficiency: float, allowed: np.ndarray | None = None):
    """cluster() as remesh runs it on the device (cubic masks)."""
    lib = _abi.load()
    f = np.ascontiguousarray(flags, dtype=np.uint8)
    a = None if allowed is None else np.ascontiguousarray(allowed, dtype=np.uint8)
    n = f.shape[-1]
    if any(s != n for s in f.shape):
        raise ValueError("cluster_device: cubic masks only")
    cap = int(f.sum()) + 1
    out = np.zeros((cap, 6), dtype=np.int32)
    k = C.c_int(0)
    raise_status(lib.af_amr_cluster_device(f.ctypes.data_as(C.c_char_p),
                                           None if a is None else a.ctypes.data_as(C.c_char_p),
                                           f.ndim, n, efficiency,
                                           out.ctypes.data_as(C.POINTER(C.c_int)), cap, C.byref(k)),
                 "af_amr_cluster_device")
    return out[:k.value]


class PatchHierarchy:
    """PatchHierarchy (amr.hpp:123-242) on the device."""

    def __init__(self, dim: int, base_exp: int, options: AmrOptions, bc=None, gamma: float = 1.4,
                 scheme: SchemeConfig | None = None, origin: float = 0.0, extent: float = 1.0,
                 device: int = 0):
        self._lib = _abi.load()
        scheme = scheme or SchemeConfig(flux=AUSM_PLUS, limiter=MINMOD, integrator=RK2)
        cfg = _abi.Config()
        cfg.dim, cfg.level, cfg.origin, cfg.extent, cfg.gamma = dim, base_exp, origin, extent, gamma
        for i, b in enumerate(bc if bc is not None else [OUTFLOW] * 6):
            cfg.bc[i] = int(b)
        cfg.flux, cfg.limiter, cfg.integrator, cfg.device = (scheme.flux, scheme.limiter,
                                                              scheme.integrator, device)
        opt = _abi.AmrOptions(options.eps_rho, options.eps_p, options.cluster_efficiency,
                              int(options.time_refine), int(options.flux_correction),
                              options.max_levels)
        self.dim, self.base_exp, self.options, self.gamma = dim, base_exp, options, gamma
        self._h = C.c_void_p()
        st = self._lib.af_amr_create(C.byref(cfg), C.byref(opt), C.byref(self._h))
        if st:
            self._h = C.c_void_p()
            raise_status(st, "af_amr_create: invalid configuration or device failure")

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            self._lib.af_amr_destroy(self._h)
            self._h = C.c_void_p()

    __del__ = close

    def _check(self, st: int):
        if st:
            e = _abi.ErrorRec()
            self._lib.af_amr_last_error(self._h, C.byref(e))
            raise_status(st, e.message.decode(errors="replace"))

    # ---- PatchHierarchy methods ------------------------------------------
    def initialize(self, ic):
        """initialize(ic): ic(x, y, z) -> (rho, mx, my, mz, rhoE)."""
        def thunk(x, y, z, q, _user):
            v = ic(x, y, z)
            for m in range(5):
                q[m] = float(v[m])
        cb = _abi.AMR_IC(thunk)
        self._check(self._lib.af_amr_initialize(self._h, cb, None))

    def initialize_case(self, kind: int, seed: int):
        self._check(self._lib.af_amr_initialize_case(self._h, kind, seed, self.gamma))

    def sync_ghosts(self, level: int, tau: float):
        self._check(self._lib.af_amr_sync_ghosts(self._h, level, tau))

    def remesh(self, level: int):
        self._check(self._lib.af_amr_remesh(self._h, level))

    def update_level(self, level: int, dt: float) -> StepDiag:
        d = _abi.StepDiag()
        self._check(self._lib.af_amr_update_level(self._h, level, dt, C.byref(d)))
        return StepDiag(d.max_wave_speed, d.fallbacks)

    def average_down(self, level: int):
        self._check(self._lib.af_amr_average_down(self._h, level))

    def flux_correct(self, level: int):
        self._check(self._lib.af_amr_flux_correct(self._h, level))

    def n_levels(self) -> int:
        n = C.c_int()
        self._check(self._lib.af_amr_n_levels(self._h, C.byref(n)))
        return n.value

    def level_info(self, level: int):
        npatch, cells, t, told = C.c_int(), C.c_long(), C.c_double(), C.c_double()
        self._check(self._lib.af_amr_level_info(self._h, level, C.byref(npatch), C.byref(cells),
                                                C.byref(t), C.byref(told)))
        return npatch.value, cells.value, t.value, told.value

    def boxes(self, level: int) -> np.ndarray:
        n = self.level_info(level)[0]
        out = np.zeros((max(n, 1), 6), dtype=np.int32)
        self._check(self._lib.af_amr_boxes(self._h, level, out.ctypes.data_as(C.POINTER(C.c_int)), n))
        return out[:n]

    def patch_data(self, level: int, ghost: int = 0, old: bool = False) -> np.ndarray:
        """Every patch of the level, patch after patch, (cells, 5) AoS."""
        c = C.c_long()
        self._check(self._lib.af_amr_patch_data_cells(self._h, level, ghost, C.byref(c)))
        out = np.zeros((c.value, 5), dtype=np.float64)
        self._check(self._lib.af_amr_patch_data(self._h, level, ghost, int(old), out.ctypes.data))
        return out

    def assemble_level(self, level: int) -> np.ndarray:
        n = 1 << (self.base_exp + level)
        out = np.zeros((n ** self.dim, 5), dtype=np.float64)
        self._check(self._lib.af_amr_assemble_level(self._h, level, out.ctypes.data))
        return out

    def total_conserved(self) -> np.ndarray:
        out = np.zeros(5, dtype=np.float64)
        self._check(self._lib.af_amr_total_conserved(self._h, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def l1_error(self, ref: np.ndarray, ref_level: int) -> np.ndarray:
        """l1_error_amr (amr.hpp:244-245) against a uniform solution (cells, 5) at ref_level."""
        r = np.ascontiguousarray(ref, dtype=np.float64)
        if r.size != 5 * (1 << ref_level) ** self.dim:
            raise ValueError("l1_error: reference must hold 2^(dim*ref_level) cells x 5")
        out = np.zeros(5, dtype=np.float64)
        self._check(self._lib.af_amr_l1_error(self._h, ref_level, r.ctypes.data,
                                              out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def total_cells(self) -> int:
        a, b = C.c_long(), C.c_long()
        self._check(self._lib.af_amr_counts(self._h, C.byref(a), C.byref(b)))
        return a.value

    def composite_cells(self) -> int:
        a, b = C.c_long(), C.c_long()
        self._check(self._lib.af_amr_counts(self._h, C.byref(a), C.byref(b)))
        return b.value

    def properly_nested(self) -> bool:
        n = C.c_int()
        self._check(self._lib.af_amr_properly_nested(self._h, C.byref(n)))
        return bool(n.value)

    def dump_boxes(self) -> str:
        t = C.c_char_p()
        self._check(self._lib.af_amr_dump_boxes(self._h, C.byref(t)))
        return t.value.decode()

    def kernel_launches(self) -> int:
        n = C.c_long()
        self._check(self._lib.af_amr_kernel_launches(self._h, C.byref(n)))
        return n.value

    def cell_updates(self) -> int:
        n = C.c_long()
        self._check(self._lib.af_amr_cell_updates(self._h, C.byref(n)))
        return n.value

    def profile(self, enable: bool = True):
        self._check(self._lib.af_amr_profile(self._h, int(enable)))

    def stage_stats(self):
        """(device ms in the stepping kernels, their launches, cell updates) while profiling"""
        ms, n, u = C.c_double(), C.c_long(), C.c_long()
        self._check(self._lib.af_amr_stage_stats(self._h, C.byref(ms), C.byref(n), C.byref(u)))
        return ms.value, n.value, u.value

    def remesh_stats(self):
        """(host seconds inside remesh, remesh calls) so far"""
        sec, n = C.c_double(), C.c_long()
        self._check(self._lib.af_amr_remesh_stats(self._h, C.byref(sec), C.byref(n)))
        return sec.value, n.value

    # ---- run_amr's cycle loop --------------------------------------------
    def run(self, n_steps: int, dt_finest: float) -> AmrReport:
        cps = np.zeros(n_steps, dtype=np.int64)
        lps = np.zeros(n_steps, dtype=np.int64)
        d = _abi.RunDiag()
        self._check(self._lib.af_amr_run(self._h, n_steps, dt_finest,
                                         cps.ctypes.data_as(C.POINTER(C.c_long)),
                                         lps.ctypes.data_as(C.POINTER(C.c_long)), C.byref(d)))
        return AmrReport(level=self.base_exp + self.options.max_levels, n_steps=n_steps,
                         max_cfl=d.max_cfl, fallbacks=d.fallbacks, t=d.t, cells_per_step=cps,
                         leaves_per_step=lps)


def run_amr(dim: int, level: int, n_steps: int, t_end: float, ic=None, case=None,
            scheme: SchemeConfig | None = None, options: AmrOptions | None = None, bc=None,
            gamma: float = 1.4, base_exp: int | None = None):
    """run_amr (amr_solver.cpp:62-133): builds the hierarchy for resolution level
    `level`, initialises it from `ic` (or the seeded `case` = (kind, seed)) and
    advances n_steps finest steps to t_end. Returns (hierarchy, report)."""
    base = amr_base_exp(dim, level) if base_exp is None else base_exp
    if base < 0:
        from .errors import ConfigError
        raise ConfigError(f"amr needs level >= 1, got {level}")
    options = options or AmrOptions()
    options = AmrOptions(options.eps_rho, options.eps_p, options.cluster_efficiency,
                         options.time_refine, options.flux_correction, level - base)
    h = PatchHierarchy(dim, base, options, bc=bc, gamma=gamma, scheme=scheme)
    if case is not None:
        h.initialize_case(*case)
    else:
        h.initialize(ic)
    rep = h.run(n_steps, t_end / float(n_steps))
    return h, rep
