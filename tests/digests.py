"""Digests of a run's results, shared by tests/golden/make_digests.py (which
writes them from the COMPILED REFERENCE in the build container) and the GPU
tests that compare the CUDA path against them on the GPU box (where
/root/reference does not exist). A digest pins a full-size run without
committing its multi-megabyte state:

  * ``state_sha``  SHA-256 of the to_uniform(L) / final state's IEEE bit
                   pattern with -0 folded to +0 (the parity bar treats +-0 as
                   equal, SURVEY.md §8 notation);
  * ``state_l1``   per-field sum |q| (the 1e-10 relative-L1 normaliser,
                   metrics.cpp:134-148);
  * ``coarse``     the state averaged to a coarse level (the tolerance-mode
                   check's reference field, restrict_to_level semantics,
                   grid.cpp:64-93, summed in a fixed order);
  * ``keys_sha``   SHA-256 of the sorted pack_key leaf list (mr_tree.hpp:26-30),
                   plus leaves per level and, for trees up to 2^21 finest
                   cells, the per-level leaf bitmaps (so a mismatch can be
                   located and checked against the near-threshold exemption).
"""
from __future__ import annotations

import hashlib

import numpy as np


def fold_zero(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64).copy()
    a[a == 0.0] = 0.0  # -0 -> +0
    return a


def state_sha(a: np.ndarray) -> str:
    return hashlib.sha256(fold_zero(a).view(np.uint64).tobytes()).hexdigest()


def state_l1(a: np.ndarray) -> np.ndarray:
    return np.abs(np.asarray(a, dtype=np.float64)).sum(axis=0)


def coarse(a: np.ndarray, dim: int, level: int, target: int) -> np.ndarray:
    """Mean over the 2^(dim*(level-target)) fine cells of each target cell
    (x fastest), shape (cells_target, 5)."""
    n, r = 1 << level, 1 << (level - target)
    m = 1 << target
    if dim == 2:
        v = np.asarray(a).reshape(n, n, 5).reshape(m, r, m, r, 5)
        return v.mean(axis=(1, 3)).reshape(m * m, 5)
    v = np.asarray(a).reshape(n, n, n, 5).reshape(m, r, m, r, m, r, 5)
    return v.mean(axis=(1, 3, 5)).reshape(m * m * m, 5)


def key_level(keys: np.ndarray) -> np.ndarray:
    return (np.asarray(keys, dtype=np.uint64) >> np.uint64(45)).astype(np.int64)


def keys_sha(keys: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(keys, dtype=np.uint64).tobytes()).hexdigest()


def leaves_per_level(keys: np.ndarray, level: int) -> np.ndarray:
    return np.bincount(key_level(keys), minlength=level + 1)[: level + 1]


def key_cells(keys: np.ndarray, dim: int, lvl: int) -> np.ndarray:
    """Linear (x fastest) cell index within level `lvl` of the keys at that level."""
    k = np.asarray(keys, dtype=np.uint64)
    k = k[key_level(k) == lvl]
    m = np.uint64((1 << 15) - 1)
    i = ((k >> np.uint64(30)) & m).astype(np.int64)
    j = ((k >> np.uint64(15)) & m).astype(np.int64)
    kk = (k & m).astype(np.int64)
    n = 1 << lvl
    return i + n * j + (n * n * kk if dim == 3 else 0)


def leaf_bitmaps(keys: np.ndarray, dim: int, level: int) -> np.ndarray:
    """Concatenated per-level leaf bitmaps (np.packbits, little bit order)."""
    parts = []
    for lvl in range(level + 1):
        bm = np.zeros(1 << (dim * lvl), dtype=bool)
        bm[key_cells(keys, dim, lvl)] = True
        parts.append(np.packbits(bm, bitorder="little"))
    return np.concatenate(parts)


def bitmaps_to_keys(bits: np.ndarray, dim: int, level: int) -> np.ndarray:
    out, off = [], 0
    for lvl in range(level + 1):
        cells = 1 << (dim * lvl)
        nbytes = (cells + 7) // 8
        bm = np.unpackbits(bits[off: off + nbytes], bitorder="little")[:cells].astype(bool)
        off += nbytes
        c = np.nonzero(bm)[0].astype(np.uint64)
        n = np.uint64(1 << lvl)
        i = c % n
        j = (c // n) % n
        k = c // (n * n) if dim == 3 else np.zeros_like(c)
        out.append((np.uint64(lvl) << np.uint64(45)) | (i << np.uint64(30)) |
                   (j << np.uint64(15)) | k)
    keys = np.concatenate(out) if out else np.zeros(0, np.uint64)
    return np.sort(keys)


def rel_l1(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Per-field relative L1 of a against b (metrics.cpp:134-148 normalised by
    b's own L1; a zero field compares absolutely)."""
    d = np.abs(np.asarray(a) - np.asarray(b)).sum(axis=0)
    s = np.abs(np.asarray(b)).sum(axis=0)
    return np.where(s > 0, d / np.where(s > 0, s, 1.0), d)
