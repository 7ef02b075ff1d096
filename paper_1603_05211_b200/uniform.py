"""Host-side mirror of the reference's uniform-mesh entry points over the C ABI.

Reference seams (paths under /root/reference/proj/core):
  * ``UniformSolver.step_block``  — step_block (step.hpp:77-79, RK2 branch
    step.cpp:237-251) with fill_ghosts (grid.hpp:128) folded in
  * ``run_uniform``               — run_uniform's loop (unigrid.cpp:7-50) for
    seeded data, with the fixed-dt (reference) or CFL time step
  * exceptions                    — errors.hpp:10-77, same messages

All arithmetic runs in libafgpu.so (sm_100a); this module only moves
pointers. Arrays are AoS (cells, 5): rho, mom0, mom1, mom2, rhoE.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from .errors import raise_status

OUTFLOW, PERIODIC, REFLECTIVE = 0, 1, 2
AUSM_PLUS, AUSMDV = 0, 1
VAN_ALBADA, MINMOD = 0, 1
RK2, MUSCL_HANCOCK = 0, 1

CASE_QUADRANTS, CASE_QUADRANTS_NOISE, CASE_ELLIPSOID, CASE_ELLIPSOID_PRATIO = 0, 1, 2, 3


@dataclass
class SchemeConfig:
    """SchemeConfig (scheme.hpp:23-40); BASELINE configs use AUSM+/minmod/RK2."""
    flux: int = AUSM_PLUS
    limiter: int = MINMOD
    integrator: int = RK2


@dataclass
class StepDiag:
    """StepDiag (step.hpp:52-55)."""
    max_wave_speed: float = 0.0
    fallbacks: int = 0


@dataclass
class RunReport:
    """The RunReport fields run_uniform fills (metrics.hpp:66-79)."""
    level: int = 0
    n_steps: int = 0
    max_cfl: float = 0.0
    max_wave_speed: float = 0.0
    fallbacks: int = 0
    t: float = 0.0
    dt: np.ndarray = field(default_factory=lambda: np.zeros(0))


def case_fill(kind: int, seed: int, level: int, gamma: float = 1.4, z0: int = 0,
              nz: int | None = None) -> np.ndarray:
    """Seeded initial data of the BASELINE configs (include/af_cases.h)."""
    lib = _abi.load()
    dim = 3 if kind in (CASE_ELLIPSOID, CASE_ELLIPSOID_PRATIO) else 2
    n = 1 << level
    nz = n if nz is None else nz
    out = np.empty((nz * n ** (dim - 1), 5), dtype=np.float64)
    st = lib.af_case_fill(kind, seed, level, gamma, z0, nz,
                          out.ctypes.data_as(C.POINTER(C.c_double)))
    raise_status(st, "af_case_fill rejected its arguments")
    return out


def _state_ptr(a, cells: int) -> int:
    """_ptr of a cells x 5 state (AoS), validated before a raw pointer goes to
    the C ABI: shape (cells, 5) or cells*5 elements, float64, contiguous."""
    shape = tuple(getattr(a, "shape", ()))
    n = 1
    for d in shape:
        n *= int(d)
    if not (shape == (cells, 5) or (len(shape) == 1 and n == cells * 5)):
        raise ValueError(f"expected a ({cells}, 5) float64 state, got shape {shape}")
    return _ptr(a)


def _ptr(a) -> int:
    """Raw data pointer of a numpy array or a CUDA/CPU torch tensor."""
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous or a.dtype != np.float64:
            raise ValueError("state must be a C-contiguous float64 array")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous() or str(a.dtype) != "torch.float64":
            raise ValueError("state must be a contiguous float64 tensor")
        return a.data_ptr()
    raise TypeError("expected numpy array or torch tensor")


class UniformSolver:
    """One uniform mesh of 2^level cells per axis on one GPU (or one slab of it).

    ``comm`` is an ``af_comm`` handle from :mod:`.parallel` for multi-GPU runs.
    """

    def __init__(self, dim: int, level: int, scheme: SchemeConfig | None = None,
                 bc=None, gamma: float = 1.4, origin: float = 0.0, extent: float = 1.0,
                 device: int = 0, comm=None):
        self._lib = _abi.load()
        scheme = scheme or SchemeConfig()
        cfg = _abi.Config()
        cfg.dim, cfg.level, cfg.origin, cfg.extent, cfg.gamma = dim, level, origin, extent, gamma
        for f in range(6):
            cfg.bc[f] = OUTFLOW if bc is None else int(bc[f])
        cfg.flux, cfg.limiter, cfg.integrator = scheme.flux, scheme.limiter, scheme.integrator
        cfg.device = device
        self.dim, self.level, self.n = dim, level, 1 << level
        self.dx = extent / float(self.n)
        h = C.c_void_p()
        st = self._lib.af_uniform_create(C.byref(cfg), comm, C.byref(h))
        raise_status(st, self._g_msg())
        self._h = h
        z0, nz = C.c_int(), C.c_int()
        self._lib.af_uniform_local_extent(self._h, C.byref(z0), C.byref(nz))
        self.z0, self.nz = z0.value, nz.value
        self.cells = nz.value * self.n ** (dim - 1)

    # -- plumbing ---------------------------------------------------------
    def _g_msg(self) -> str:
        e = _abi.ErrorRec()
        self._lib.af_uniform_last_error(None, C.byref(e))
        return e.message.decode()

    def last_error(self) -> _abi.ErrorRec:
        e = _abi.ErrorRec()
        self._lib.af_uniform_last_error(self._h, C.byref(e))
        return e

    def _check(self, st: int):
        if st != _abi.AF_OK:
            raise_status(st, self.last_error().message.decode())

    def close(self):
        if getattr(self, "_h", None):
            self._lib.af_uniform_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream) -> None:
        """Orders all work on a torch.cuda.Stream (or raw cudaStream_t int)."""
        raw = getattr(stream, "cuda_stream", stream)
        self._check(self._lib.af_uniform_set_stream(self._h, C.c_void_p(raw)))

    def set_numerics(self, tolerance: bool) -> None:
        """AF_NUMERICS_EXACT (default, bit-identical to the reference) or
        AF_NUMERICS_TOLERANCE (3D stage with reciprocal estimates and FMA
        contraction, within 1e-10 relative L1 of the exact result)."""
        self._check(self._lib.af_uniform_set_numerics(self._h, 1 if tolerance else 0))

    def kernel_launches(self) -> int:
        c = C.c_long()
        self._lib.af_uniform_kernel_launches(self._h, C.byref(c))
        return c.value

    # -- state ------------------------------------------------------------
    def upload(self, aos) -> None:
        self._check(self._lib.af_uniform_upload(self._h, C.c_void_p(_state_ptr(aos, self.cells))))

    def download(self, out=None):
        if out is None:
            out = np.empty((self.cells, 5), dtype=np.float64)
        self._check(self._lib.af_uniform_download(self._h, C.c_void_p(_state_ptr(out, self.cells))))
        return out

    # -- stepping ---------------------------------------------------------
    def rk2_stage(self, base, eval_, stage_dt: float, capture: bool = False):
        """rk2_stage (step.hpp:62-64): out = base + stage_dt * rhs(eval) of AoS
        states (eval's ghosts = the configured BCs). Returns (out, StepDiag,
        flux) with flux the FluxField capture (step.hpp:16-50) as a list of
        per-axis arrays of shape (n_c, n_b, n_a + 1, 5), or None. Replaces
        the solver's state."""
        out = np.empty((self.cells, 5), dtype=np.float64)
        cap = None
        if capture:
            n = self.n
            per = (n + 1) * n ** (self.dim - 1)
            cap = np.empty(self.dim * per * 5, dtype=np.float64)
        d = _abi.StepDiag()
        self._check(self._lib.af_uniform_rk2_stage(
            self._h, C.c_void_p(_state_ptr(base, self.cells)),
            C.c_void_p(_state_ptr(eval_, self.cells)), C.c_void_p(out.ctypes.data),
            float(stage_dt), C.c_void_p(cap.ctypes.data if cap is not None else 0), C.byref(d)))
        flux = None
        if cap is not None:
            n, per = self.n, (self.n + 1) * self.n ** (self.dim - 1)
            flux = []
            for a in range(self.dim):
                shape = [n] * self.dim
                shape[a] += 1
                flux.append(cap[a * per * 5:(a + 1) * per * 5].reshape(*shape[::-1], 5))
        return out, StepDiag(d.max_wave_speed, d.fallbacks), flux

    def step_block(self, dt: float, diag: bool = True) -> StepDiag | None:
        """step_block (step.hpp:77-79): one RK2 step of size dt."""
        if not diag:
            self._check(self._lib.af_uniform_step(self._h, dt, None))
            return None
        d = _abi.StepDiag()
        self._check(self._lib.af_uniform_step(self._h, dt, C.byref(d)))
        return StepDiag(d.max_wave_speed, d.fallbacks)

    def run(self, n_steps: int, cfl: float = 0.0, fixed_dt: float = 0.0,
            collect: bool = True) -> RunReport | None:
        """n_steps device-resident steps (CFL rule if cfl > 0, else fixed_dt)."""
        if not collect:
            self._check(self._lib.af_uniform_run(self._h, n_steps, cfl, fixed_dt, None, None))
            return None
        dts = np.zeros(max(n_steps, 1), dtype=np.float64)
        d = _abi.RunDiag()
        self._check(self._lib.af_uniform_run(self._h, n_steps, cfl, fixed_dt,
                                             dts.ctypes.data_as(C.POINTER(C.c_double)),
                                             C.byref(d)))
        return RunReport(level=self.level, n_steps=n_steps, max_cfl=d.max_cfl,
                         max_wave_speed=d.max_wave_speed, fallbacks=d.fallbacks, t=d.t,
                         dt=dts[:n_steps])

    def speed_sum(self) -> float:
        v = C.c_double()
        self._check(self._lib.af_uniform_speed_sum(self._h, C.byref(v)))
        return v.value

    def sync(self) -> None:
        self._check(self._lib.af_uniform_sync(self._h))


def run_uniform(init: np.ndarray, dim: int, level: int, n_steps: int, cfl: float = 0.0,
                fixed_dt: float = 0.0, scheme: SchemeConfig | None = None, bc=None,
                gamma: float = 1.4, device: int = 0):
    """run_uniform (unigrid.hpp:24-26) on seeded data: returns (state, RunReport)."""
    s = UniformSolver(dim, level, scheme=scheme, bc=bc, gamma=gamma, device=device)
    try:
        s.upload(np.ascontiguousarray(init, dtype=np.float64))
        rep = s.run(n_steps, cfl=cfl, fixed_dt=fixed_dt)
        return s.download(), rep
    finally:
        s.close()


class UniformGroup:
    """n_ranks slabs of one mesh emulated on ONE GPU (af_uniform_create_group):
    the per-rank multi-GPU code path (slab extents, halo planes, boundary
    handling at slab edges, the CFL max over ranks) with device-to-device
    copies in place of NCCL. Used to check rank-count independence."""

    def __init__(self, dim: int, level: int, n_ranks: int, scheme: SchemeConfig | None = None,
                 bc=None, gamma: float = 1.4, device: int = 0):
        self._lib = _abi.load()
        scheme = scheme or SchemeConfig()
        cfg = _abi.Config()
        cfg.dim, cfg.level, cfg.origin, cfg.extent, cfg.gamma = dim, level, 0.0, 1.0, gamma
        for f in range(6):
            cfg.bc[f] = OUTFLOW if bc is None else int(bc[f])
        cfg.flux, cfg.limiter, cfg.integrator = scheme.flux, scheme.limiter, scheme.integrator
        cfg.device = device
        self.n_ranks, self.dim, self.level, self.n = n_ranks, dim, level, 1 << level
        self._h = (C.c_void_p * n_ranks)()
        st = self._lib.af_uniform_create_group(C.byref(cfg), n_ranks, self._h)
        if st:
            e = _abi.ErrorRec()
            self._lib.af_uniform_last_error(None, C.byref(e))
            raise_status(st, e.message.decode())
        self.extents = []
        for r in range(n_ranks):
            z0, nz = C.c_int(), C.c_int()
            self._lib.af_uniform_local_extent(self._h[r], C.byref(z0), C.byref(nz))
            self.extents.append((z0.value, nz.value))
        self.row = self.n ** (dim - 1)

    def close(self):
        if getattr(self, "_h", None) is not None:
            for r in range(self.n_ranks):
                self._lib.af_uniform_destroy(self._h[r])
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st, r=0):
        if st:
            e = _abi.ErrorRec()
            self._lib.af_uniform_last_error(self._h[r], C.byref(e))
            raise_status(st, e.message.decode())

    def upload(self, aos: np.ndarray) -> None:
        _state_ptr(aos, self.n ** self.dim)  # shape/dtype check
        for r, (z0, nz) in enumerate(self.extents):
            part = np.ascontiguousarray(aos[z0 * self.row:(z0 + nz) * self.row])
            self._check(self._lib.af_uniform_upload(self._h[r], C.c_void_p(part.ctypes.data)), r)

    def download(self) -> np.ndarray:
        out = np.empty((self.n ** self.dim, 5), dtype=np.float64)
        for r, (z0, nz) in enumerate(self.extents):
            part = np.empty((nz * self.row, 5), dtype=np.float64)
            self._check(self._lib.af_uniform_download(self._h[r], C.c_void_p(part.ctypes.data)), r)
            out[z0 * self.row:(z0 + nz) * self.row] = part
        return out

    def run(self, n_steps: int, cfl: float = 0.0, fixed_dt: float = 0.0) -> RunReport:
        dts = np.zeros(max(n_steps, 1), dtype=np.float64)
        d = _abi.RunDiag()
        self._check(self._lib.af_uniform_run_group(
            self._h, self.n_ranks, n_steps, cfl, fixed_dt,
            dts.ctypes.data_as(C.POINTER(C.c_double)), C.byref(d)))
        return RunReport(level=self.level, n_steps=n_steps, max_cfl=d.max_cfl,
                         max_wave_speed=d.max_wave_speed, fallbacks=d.fallbacks, t=d.t,
                         dt=dts[:n_steps])
