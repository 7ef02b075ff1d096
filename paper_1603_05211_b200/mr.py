"""Host-side mirror of the reference's multiresolution entry points over the C ABI.

Reference seams (paths under /root/reference/proj/core):
  * ``MRSolver.build``            — MRTree::from_uniform (mr_tree.cpp:29-71) +
    set_min_leaf_level + coarsen(eps) as run_mr does (mr_solver.cpp:406-410)
  * ``refine / coarsen / add_virtual_leaves / remove_virtual_leaves`` —
    MRTree (mr_tree.hpp:141-152)
  * ``evolve_global / advance_local`` — MRSolver (mr_solver.hpp:23-29)
  * ``run``                       — the run_mr cycle loop (mr_solver.cpp:318-400)
  * ``leaves / to_uniform / detail`` — MRTree queries (mr_tree.hpp:95-160)

All arithmetic and tree bookkeeping runs in libafgpu.so (sm_100a).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from .errors import raise_status
from .uniform import MINMOD, OUTFLOW, SchemeConfig, StepDiag, _state_ptr


@dataclass
class MROptions:
    """MROptions (mr_solver.hpp:65-74) + level thresholds + coarsest leaf level."""
    epsilon: float = 0.0
    eps_level: list | None = None  # eps_level[l] for details whose children are at level l
    min_leaf_level: int = 0
    local_time: bool = False
    local_time_level_gap: int = 3
    # storage of the level arrays (af_gpu.h AF_MR_STORAGE_*): "dense" per-level
    # grids, "bricks" (3D brick layout, fully allocated) or "sparse" (3D bricks
    # mapped only where the tree reaches); bit-identical results
    storage: str = "dense"
    brick_shift: int = 0


@dataclass
class MRReport:
    n_steps: int = 0
    max_cfl: float = 0.0
    fallbacks: int = 0
    t: float = 0.0
    cycles: np.ndarray = field(default_factory=lambda: np.zeros((0, 6)))

    @property
    def updates(self) -> int:
        """leaf-cell RK-stage updates performed (the bench metric's numerator)"""
        return int(self.cycles[:, 5].sum())

    @property
    def leaves_per_step(self):
        c = self.cycles
        return np.repeat(c[:, 0], c[:, 2].astype(np.int64))

    @property
    def cells_per_step(self):
        c = self.cycles
        return np.repeat(c[:, 1], c[:, 2].astype(np.int64))


STORAGE = {"dense": 0, "bricks": 1, "sparse": 2}


def eps_levels_scaled(eps: float, level: int, dim: int) -> list:
    """BASELINE cfg2/cfg5 thresholds eps_l = eps * 2^(d (l - L)), indexed by the
    level of the detail's children (SURVEY.md §8(c) convention)."""
    return [eps * 2.0 ** (dim * (l - level)) for l in range(level + 1)]


class MRSolver:
    def __init__(self, dim: int, level: int, options: MROptions | None = None,
                 scheme: SchemeConfig | None = None, bc=None, gamma: float = 1.4,
                 extent: float = 1.0, device: int = 0, comm=None):
        """comm: an af_comm handle for one rank of a spatially decomposed tree
        (af_mr_create_dist); None for a single GPU."""
        self._lib = _abi.load()
        scheme = scheme or SchemeConfig(limiter=MINMOD)
        options = options or MROptions()
        cfg = _abi.Config()
        cfg.dim, cfg.level, cfg.origin, cfg.extent, cfg.gamma = dim, level, 0.0, extent, gamma
        for f in range(6):
            cfg.bc[f] = OUTFLOW if bc is None else int(bc[f])
        cfg.flux, cfg.limiter, cfg.integrator, cfg.device = (scheme.flux, scheme.limiter,
                                                             scheme.integrator, device)
        o = _abi.MROptions()
        o.eps = options.epsilon
        self._eps = None
        if options.eps_level is not None:
            self._eps = np.ascontiguousarray(options.eps_level, dtype=np.float64)
            if self._eps.shape[0] != level + 1:
                raise ValueError("eps_level needs level+1 entries")
            o.eps_level = self._eps.ctypes.data_as(C.POINTER(C.c_double))
        o.min_leaf_level = options.min_leaf_level
        o.local_time = int(options.local_time)
        o.lt_gap = options.local_time_level_gap
        if options.storage not in STORAGE:
            raise ValueError(f"storage must be one of {sorted(STORAGE)}")
        o.storage = STORAGE[options.storage]
        o.brick_shift = options.brick_shift
        h = C.c_void_p()
        if comm is None:
            st = self._lib.af_mr_create(C.byref(cfg), C.byref(o), C.byref(h))
        else:
            st = self._lib.af_mr_create_dist(C.byref(cfg), C.byref(o), comm, C.byref(h))
        if st:
            e = _abi.ErrorRec()
            self._lib.af_mr_last_error(None, C.byref(e))
            raise_status(st, e.message.decode())
        self._h = h
        self.dim, self.level = dim, level

    def _check(self, st):
        if st:
            e = _abi.ErrorRec()
            self._lib.af_mr_last_error(self._h, C.byref(e))
            raise_status(st, e.message.decode())

    def close(self):
        if getattr(self, "_h", None):
            self._lib.af_mr_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream):
        raw = getattr(stream, "cuda_stream", stream)
        self._check(self._lib.af_mr_set_stream(self._h, C.c_void_p(raw)))

    def memory(self) -> dict:
        """Device bytes of the per-cell arrays: now, peak, and as dense level grids."""
        v = [C.c_ulonglong() for _ in range(3)]
        self._check(self._lib.af_mr_memory(self._h, *[C.byref(x) for x in v]))
        return {"now": v[0].value, "peak": v[1].value, "dense": v[2].value}

    def kernel_launches(self) -> int:
        c = C.c_long()
        self._lib.af_mr_kernel_launches(self._h, C.byref(c))
        return c.value

    def profile(self, enable: bool = True) -> None:
        """Times every stage's kernels with CUDA events on the solver stream."""
        self._check(self._lib.af_mr_profile(self._h, int(enable)))

    def stage_stats(self):
        """(stage-kernel device ms, stage launches, leaf-cell stage updates)."""
        ms, la, up = C.c_double(), C.c_long(), C.c_long()
        self._check(self._lib.af_mr_stage_stats(self._h, C.byref(ms), C.byref(la), C.byref(up)))
        return ms.value, la.value, up.value

    def set_numerics(self, tolerance: bool) -> None:
        """AF_NUMERICS_EXACT (default, bit-identical) or AF_NUMERICS_TOLERANCE
        (the 2D full-tile stage with the tolerance physics, 1e-10 relative L1)."""
        self._check(self._lib.af_mr_set_numerics(self._h, 1 if tolerance else 0))

    # MRTree
    def build(self, aos) -> None:
        cells = 1 << (self.dim * self.level)
        self._check(self._lib.af_mr_build(self._h, C.c_void_p(_state_ptr(aos, cells))))

    def refine(self, top: int = -1, eps: float | None = None, buffer=None):
        """MRTree::refine. With ``eps`` given: refine(eps, buffer_radius_per_level)
        (mr_tree.hpp:141) — one threshold, optional per-level Chebyshev buffer.
        Otherwise the run_mr form: the configured thresholds, and the LT buffer
        radii of mr_solver.cpp:358-362 when top >= 0."""
        if eps is None:
            self._check(self._lib.af_mr_refine(self._h, top))
            return
        buf = [] if buffer is None else [int(r) for r in buffer]
        arr = (C.c_int * max(1, len(buf)))(*buf)
        self._check(self._lib.af_mr_refine_buffer(self._h, float(eps), arr, len(buf)))

    def coarsen(self):
        self._check(self._lib.af_mr_coarsen(self._h))

    def add_virtual_leaves(self):
        self._check(self._lib.af_mr_add_virtual_leaves(self._h))

    def remove_virtual_leaves(self):
        self._check(self._lib.af_mr_remove_virtual_leaves(self._h))

    def counts(self):
        lv, nd, it = C.c_long(), C.c_long(), C.c_long()
        self._check(self._lib.af_mr_counts(self._h, C.byref(lv), C.byref(nd), C.byref(it)))
        return lv.value, nd.value, it.value

    def coarsest_leaf_level(self) -> int:
        v = C.c_int()
        self._check(self._lib.af_mr_coarsest_leaf_level(self._h, C.byref(v)))
        return v.value

    def leaves(self) -> np.ndarray:
        n = C.c_size_t(0)
        self._check(self._lib.af_mr_leaf_keys(self._h, None, C.byref(n)))
        out = np.zeros(n.value, dtype=np.uint64)
        self._check(self._lib.af_mr_leaf_keys(
            self._h, out.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(n)))
        return out

    def to_uniform(self, level: int | None = None) -> np.ndarray:
        level = self.level if level is None else level
        n = 1 << level
        out = np.empty((n ** self.dim, 5), dtype=np.float64)
        self._check(self._lib.af_mr_to_uniform(self._h, level, C.c_void_p(out.ctypes.data)))
        return out

    def local_rows(self, level: int | None = None):
        """Rows [lo, hi) of the last axis this rank owns at `level`."""
        level = self.level if level is None else level
        lo, hi = C.c_int(), C.c_int()
        self._check(self._lib.af_mr_local_rows(self._h, level, C.byref(lo), C.byref(hi)))
        return lo.value, hi.value

    def dump(self) -> str:
        """MRTree::dump (mr_tree.cpp:623-641) of the device tree."""
        n = C.c_size_t(0)
        self._check(self._lib.af_mr_dump(self._h, None, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        self._check(self._lib.af_mr_dump(self._h, buf, C.byref(n)))
        return buf.value.decode()

    def details(self, level: int) -> np.ndarray:
        n = 1 << level
        out = np.empty(n ** self.dim, dtype=np.float64)
        self._check(self._lib.af_mr_details(self._h, level, C.c_void_p(out.ctypes.data)))
        return out

    # MRSolver
    def evolve_global(self, dt: float) -> StepDiag:
        d = _abi.StepDiag()
        self._check(self._lib.af_mr_evolve_global(self._h, dt, C.byref(d)))
        return StepDiag(d.max_wave_speed, d.fallbacks)

    def advance_local(self, top: int, t: float, dt: float) -> StepDiag:
        d = _abi.StepDiag()
        self._check(self._lib.af_mr_advance_local(self._h, top, t, dt, C.byref(d)))
        return StepDiag(d.max_wave_speed, d.fallbacks)

    # run_mr
    def run(self, n_steps: int, cfl: float = 0.0, fixed_dt: float = 0.0,
            max_cycles: int | None = None) -> MRReport:
        max_cycles = n_steps if max_cycles is None else max_cycles
        cyc = (_abi.MRCycle * max(1, max_cycles))()
        d = _abi.RunDiag()
        self._check(self._lib.af_mr_run(self._h, n_steps, cfl, fixed_dt, cyc, max_cycles,
                                        C.byref(d)))
        nc = 0
        rows = []
        for c in cyc:
            if c.sub == 0:
                break
            rows.append((c.leaves, c.nodes, c.sub, c.top, c.dt, c.updates))
            nc += 1
        return MRReport(n_steps=d.steps_done, max_cfl=d.max_cfl, fallbacks=d.fallbacks, t=d.t,
                        cycles=np.array(rows, dtype=np.float64).reshape(-1, 6))


class MRGroup:
    """n_ranks slabs of one MR tree, each rank an MRSolver driven by its own
    host thread on ONE GPU (af_comm_create_local): the multi-rank code path
    (slab ownership, status/value halo exchanges, reductions) with
    device-to-device copies in place of NCCL. Used to check that results do
    not depend on the rank count."""

    def __init__(self, dim: int, level: int, n_ranks: int, options: MROptions | None = None,
                 scheme: SchemeConfig | None = None, bc=None, gamma: float = 1.4,
                 extent: float = 1.0, device: int = 0):
        self._lib = _abi.load()
        self.n_ranks, self.dim, self.level = n_ranks, dim, level
        comms = (C.c_void_p * n_ranks)()
        st = self._lib.af_comm_create_local(n_ranks, device, comms)
        if st:
            raise_status(st, "af_comm_create_local failed")
        self._comms = [comms[r] for r in range(n_ranks)]
        self.ranks = [MRSolver(dim, level, options, scheme, bc, gamma, extent, device,
                               comm=c) for c in self._comms]

    def _all(self, fn):
        import threading
        out, err = [None] * self.n_ranks, [None] * self.n_ranks

        def one(r):
            try:
                out[r] = fn(self.ranks[r])
            except BaseException as e:  # re-raised on the caller's thread
                err[r] = e

        ts = [threading.Thread(target=one, args=(r,)) for r in range(self.n_ranks)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        for e in err:
            if e is not None:
                raise e
        return out

    def close(self):
        for s in getattr(self, "ranks", []):
            s.close()
        for c in getattr(self, "_comms", []):
            self._lib.af_comm_destroy(c)
        self.ranks, self._comms = [], []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def build(self, aos) -> None:
        self._all(lambda s: s.build(aos))

    def run(self, n_steps: int, cfl: float = 0.0, fixed_dt: float = 0.0) -> MRReport:
        reps = self._all(lambda s: s.run(n_steps, cfl=cfl, fixed_dt=fixed_dt))
        for r in reps[1:]:  # cycle records and diagnostics are global on every rank
            if not (np.array_equal(r.cycles, reps[0].cycles) and r.max_cfl == reps[0].max_cfl):
                raise RuntimeError("ranks disagree on the run report")
        return reps[0]

    def leaves(self) -> np.ndarray:
        return np.sort(np.concatenate(self._all(lambda s: s.leaves())))

    def to_uniform(self, level: int | None = None) -> np.ndarray:
        level = self.level if level is None else level
        n = 1 << level
        row = n ** (self.dim - 1)
        parts = self._all(lambda s: (s.local_rows(level), s.to_uniform(level)))
        out = np.empty((n ** self.dim, 5), dtype=np.float64)
        covered = 0
        for (lo, hi), u in parts:
            out[lo * row:hi * row] = u[lo * row:hi * row]
            covered += hi - lo
        if covered != n:
            raise RuntimeError("rank rows do not tile the level")
        return out
