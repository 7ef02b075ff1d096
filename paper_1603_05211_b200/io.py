"""Formats and compare path either side of the hot path,
over the C ABI:
  * ``write_snapshot / read_snapshot`` — AFSN v1 (snapshot.hpp:10-22,
    snapshot.cpp:29-104); bit-exact round trips, for checkpoint/resume of GPU
    runs and golden exchange
  * ``restrict_to_level`` — grid.cpp:64-93, on the device, bit-exact
  * ``l1_error`` — metrics.cpp:134-148, on the device (round-off agreement)
Arrays are AoS (cells, 5): rho, mom0, mom1, mom2, rhoE (mom2 = 0 in 2D)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _abi
from .errors import raise_status
from .uniform import _ptr


@dataclass
class Snapshot:
    """adaptflow::Snapshot (snapshot.hpp:24-28) with the grid as an AoS array."""
    dim: int
    level: int
    gamma: float
    time: float
    origin: float
    extent: float
    state: np.ndarray


def write_snapshot(path: str, state, dim: int, level: int, gamma: float = 1.4, time: float = 0.0,
                   origin: float = 0.0, extent: float = 1.0) -> None:
    lib = _abi.load()
    h = _abi.SnapshotHeader(dim, level, gamma, time, origin, extent)
    raise_status(lib.af_snapshot_write(path.encode(), C.byref(h), C.c_void_p(_ptr(state))),
                 f"write_snapshot({path})")


def read_snapshot(path: str) -> Snapshot:
    lib = _abi.load()
    h = _abi.SnapshotHeader()
    st = lib.af_snapshot_read(path.encode(), C.byref(h), None)
    if st:
        _raise_last(st, path)
    out = np.empty(((1 << (h.dim * h.level)), 5), dtype=np.float64)
    st = lib.af_snapshot_read(path.encode(), C.byref(h), C.c_void_p(out.ctypes.data))
    if st:
        _raise_last(st, path)
    return Snapshot(h.dim, h.level, h.gamma, h.time, h.origin, h.extent, out)


def _raise_last(st, what):
    e = _abi.ErrorRec()
    _abi.load().af_uniform_last_error(None, C.byref(e))
    raise_status(st, e.message.decode() or what)


def restrict_to_level(state, dim: int, level: int, target: int) -> np.ndarray:
    lib = _abi.load()
    out = np.empty((1 << (dim * target), 5), dtype=np.float64)
    st = lib.af_restrict_to_level(dim, level, target, C.c_void_p(_ptr(state)),
                                  C.c_void_p(out.ctypes.data))
    if st:
        _raise_last(st, "restrict_to_level")
    return out


def l1_error(sol, dim: int, level: int, ref, ref_level: int, extent: float = 1.0) -> np.ndarray:
    lib = _abi.load()
    out = np.zeros(5, dtype=np.float64)
    st = lib.af_l1_error(dim, level, extent, C.c_void_p(_ptr(sol)), ref_level,
                         C.c_void_p(_ptr(ref)), out.ctypes.data_as(C.POINTER(C.c_double)))
    if st:
        _raise_last(st, "l1_error")
    return out


def rates(adaptive: dict, fv: dict, n_c: float) -> dict:
    """Paper §3 rates (metrics.cpp:91-132) through af_rates_compute. `adaptive`
    and `fv` hold the RunReport fields the formulas read: wall_seconds,
    sum_cells, sum_leaves, n_steps, l1_rho. Raises DivisionDomain with the
    reference's text on a zero denominator."""
    lib = _abi.load()

    def summ(d):
        return _abi.RunSummary(float(d.get("wall_seconds", 0.0)), float(d.get("sum_cells", 0.0)),
                               float(d.get("sum_leaves", 0.0)), int(d.get("n_steps", 0)),
                               float(d.get("l1_rho", 0.0)))
    out = _abi.Rates()
    st = lib.af_rates_compute(C.byref(summ(adaptive)), C.byref(summ(fv)), float(n_c), C.byref(out))
    if st:
        e = _abi.ErrorRec()
        lib.af_uniform_last_error(None, C.byref(e))
        raise_status(st, e.message.decode())
    return {k: getattr(out, k) for k, _ in _abi.Rates._fields_}
