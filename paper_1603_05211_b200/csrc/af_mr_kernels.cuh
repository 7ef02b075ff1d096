// af_mr_kernels.cuh — Harten cell-average multiresolution on per-level dense
// grids (sm_100a).
//
// Storage: every level l in [0, L] is a dense 2^l-per-axis grid of
//   status  uint8  ABSENT / LEAF / INTERNAL  (the MRTree node map, mr_tree.hpp:195)
//   value   NC doubles SoA — the reference's `value_at` field: the node's q
//           where a node exists, and the recursive prediction where it does
//           not (mr_tree.cpp:171-180). Keeping predictions materialised makes
//           every stencil read a plain load; they are refreshed top-down after
//           each projection, which is exactly when the reference's virtual
//           leaves are re-predicted (refresh_virtuals, mr_solver.cpp:195-208).
// Tree operations become level-synchronous passes whose results are
// bit-identical to the reference's sequential loops (SURVEY.md §8(a) rows
// 20-21 give the argument; tests/test_mr_gpu.py checks full trees).
#pragma once

#include "af_internal.h"
#include "af_mr_types.h"
#include "af_physics.cuh"
#include "af_uniform_kernels.cuh"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace af {

// map_position (mr_tree.cpp:146-169): periodic when the LOW face is periodic
// (BoundaryCondition::periodic), outflow clamps, reflective folds and flips.
__device__ __forceinline__ int mr_map(int c, int n, int lo, int hi, bool& flip) {
  flip = false;
  if (c >= 0 && c < n) return c;
  if (lo == AF_BC_PERIODIC) {
    c %= n;
    return c < 0 ? c + n : c;
  }
  const int kind = c < 0 ? lo : hi;
  if (kind == AF_BC_OUTFLOW) return c < 0 ? 0 : n - 1;
  while (c < 0 || c >= n) {
    if (c < 0) c = -1 - c;
    if (c >= n) c = 2 * n - 1 - c;
    flip = !flip;
  }
  return c;
}

// Tile iteration of one launch. Single level (l >= 0): the `ntiles` entries
// of `tiles` (ntiles -1 / -2 / -3: the band / leaf-tile / absent-band count
// from g.dcnt).
// Multi-level (l = -(lo+1), ntiles = hi << 3 | sel): the band (sel 0), leaf
// (sel 1), absent-band (sel 2), partial-leaf (sel 3) or full-leaf (sel 4)
// lists of levels lo..hi as ONE flat range, so the grid follows the
// total work instead of levels x the largest level. Each tile is visited
// `reps` times (rep = 0..reps-1) by different blocks; f(level, tile, rep).
// The same range without a callback: tile_total() entries, tile_at() maps
// entry `it` to (level, tile).
__device__ __forceinline__ int tile_total(const MRLevels& g, int l, int ntiles) {
  if (l < 0) {
    const int* cnt = g.dcnt + 17 * (ntiles & 7);
    int total = 0;
    for (int k = -l - 1; k <= (ntiles >> 3); ++k) total += cnt[k];
    return total;
  }
  return ntiles < 0 ? g.dcnt[17 * (-ntiles - 1) + l] : ntiles;
}
__device__ __forceinline__ int tile_at(const MRLevels& g, int l, const int* tiles, int ntiles,
                                       int it, int* level) {
  if (l < 0) {
    const int* cnt = g.dcnt + 17 * (ntiles & 7);
    int k = -l - 1, base = 0;
    while (it >= base + cnt[k]) base += cnt[k++];
    *level = k;
    return tiles[g.tile_off[k] + it - base];
  }
  *level = l;
  return tiles[it];
}

// Entry -> (level, tile) of a multi-level range for a block whose entries
// increase from call to call: the level cursor only moves forward, so the
// walk over the per-level counts is paid once per block, not once per entry.
struct TileWalker {
  int k, base, cnt_k;
  const int* cnt;
  __device__ __forceinline__ TileWalker(const MRLevels& g, int l, int ntiles) {
    cnt = g.dcnt + 17 * (ntiles & 7);
    k = -l - 1;
    base = 0;
    cnt_k = cnt[k];
  }
  __device__ __forceinline__ int at(const MRLevels& g, const int* tiles, int ti, int* level) {
    while (ti >= base + cnt_k) {
      base += cnt_k;
      cnt_k = cnt[++k];
    }
    *level = k;
    return tiles[g.tile_off[k] + ti - base];
  }
};

template <class F>
__device__ __forceinline__ void for_each_tile(const MRLevels& g, int l, const int* tiles,
                                              int ntiles, int reps, F&& f) {
  if (l < 0) {
    const int total = tile_total(g, l, ntiles);
    TileWalker w(g, l, ntiles);
    for (int it = blockIdx.x; it < total * reps; it += gridDim.x) {
      const int ti = it / reps;
      int k;
      const int t = w.at(g, tiles, ti, &k);
      f(k, t, it - ti * reps);
    }
  } else {
    if (ntiles < 0) ntiles = g.dcnt[17 * (-ntiles - 1) + l];
    for (int it = blockIdx.x; it < ntiles * reps; it += gridDim.x) {
      const int ti = it / reps;
      f(l, tiles[ti], it - ti * reps);
    }
  }
}

// Cell iteration: one thread per cell of the listed tiles (256-thread
// blocks), or every cell of level l when `tiles` is null. f(level, cell).
template <int D, class F>
__device__ __forceinline__ void level_cells(const MRLevels& g, int l, const int* tiles,
                                            int ntiles, F&& f) {
  if (tiles) {
    constexpr int TX = D == 3 ? kTileX3 : kTileX2, TY = D == 3 ? kTileY3 : kTileY2;
    const int tx = threadIdx.x % TX, ty = (threadIdx.x / TX) % TY;
    const int tz = D == 3 ? threadIdx.x / (TX * TY) : 0;
    for_each_tile(g, l, tiles, ntiles, 1, [&](int lv, int t, int) {
      const int n = 1 << lv, ntx = g.ntx[lv], nty = g.nty[lv];
      const int sx = ilog2i(ntx), sy = ilog2i(nty);  // tile counts are powers of two
      const int x = (t & (ntx - 1)) * TX + tx, y = ((t >> sx) & (nty - 1)) * TY + ty;
      const int z = D == 3 ? (t >> (sx + sy)) * kTileZ3 + tz : 0;
      if (x < n && y < n && (D == 2 || z < n)) f(lv, mr_idx(g, D, n, x, y, z));
    });
  } else {
    const long cells = mr_cells(D, l);
    for (long c = blockIdx.x * (long)blockDim.x + threadIdx.x; c < cells;
         c += (long)gridDim.x * blockDim.x)
      f(l, c);
  }
}

// ------------------------------------------------------------ projection --
// project_internals / project_range (mr_tree.cpp:319-338, mr_solver.cpp:268-282):
// internal q = (sum over children, x-fastest child order) * (1/2^d).
// One internal node's projection (s: its status).
template <int D>
__device__ __forceinline__ void project_cell(double* V, const MRLevels& g, int l, long c, uint8_t s) {
  constexpr int NC = D + 2;
  const int n = 1 << l, nf = n << 1;
  const long foff = g.cell_off[l + 1];
  const long comp = g.total_cells;
  const double w = 1.0 / (double)(1 << D);
  if (s != ST_INTERNAL || !row_owned(g, l, mr_row(g, D, l, c))) return;
  int i, j, k;
  mr_ijk(g, D, l, c, i, j, k);
  double sm[NC];
#pragma unroll
  for (int m = 0; m < NC; ++m) sm[m] = 0.0;
#pragma unroll
  for (int ch = 0; ch < (1 << D); ++ch) {
    const long fc = foff + mr_idx(g, D, nf, 2 * i + (ch & 1), 2 * j + ((ch >> 1) & 1),
                                  D == 3 ? 2 * k + ((ch >> 2) & 1) : 0);
#pragma unroll
    for (int m = 0; m < NC; ++m) sm[m] = sm[m] + V[m * comp + fc];
  }
#pragma unroll
  for (int m = 0; m < NC; ++m) V[m * comp + g.cell_off[l] + c] = sm[m] * w;
}

template <int D>
__device__ __forceinline__ void project_level_dev(double* V, const uint8_t* st, const MRLevels& g, int l,
    const int* tiles, int ntiles) {
  level_cells<D>(g, l, tiles, ntiles, [&](const int lv, long c) {
    project_cell<D>(V, g, lv, c, st[g.cell_off[lv] + c]);
  });
}

// Cell of this thread in entry `it` of a band/leaf tile range (tile_at
// conventions), -1 when outside the level or past the range.
template <int D>
__device__ __forceinline__ long tile_cell(const MRLevels& g, int l, const int* tiles, int ntiles,
                                          int it, int* lv) {
  constexpr int TX = D == 3 ? kTileX3 : kTileX2, TY = D == 3 ? kTileY3 : kTileY2;
  const int tx = threadIdx.x % TX, ty = (threadIdx.x / TX) % TY;
  const int tz = D == 3 ? threadIdx.x / (TX * TY) : 0;
  const int t = tile_at(g, l, tiles, ntiles, it, lv);
  const int n = 1 << *lv, ntx = g.ntx[*lv], nty = g.nty[*lv];
  const int sx = ilog2i(ntx), sy = ilog2i(nty);  // tile counts are powers of two
  const int x = (t & (ntx - 1)) * TX + tx, y = ((t >> sx) & (nty - 1)) * TY + ty;
  const int z = D == 3 ? (t >> (sx + sy)) * kTileZ3 + tz : 0;
  return (x < n && y < n && (D == 2 || z < n)) ? mr_idx(g, D, n, x, y, z) : -1L;
}

// Band/leaf-tile cell iteration (tiles non-null) whose first tile lookup and
// status load are issued before the PDL wait when `pre` allows (kPreList,
// kPreSt): the dependent chain count -> tile -> status then overlaps the
// predecessor kernel. Includes AF_PDL_ENTRY. f(level, cell, status).
template <int D, class F>
__device__ __forceinline__ void band_cells_pdl(const MRLevels& g, int l, const int* tiles,
                                               int ntiles, const uint8_t* st, int pre, F&& f) {
  int total = 0, lv0 = 0, s0 = -1;
  long c0 = -1;
  if (pre & kPreList) {
    total = tile_total(g, l, ntiles);
    if ((int)blockIdx.x < total) {
      c0 = tile_cell<D>(g, l, tiles, ntiles, blockIdx.x, &lv0);
      if ((pre & kPreSt) && c0 >= 0) s0 = st[g.cell_off[lv0] + c0];
    }
  }
  AF_PDL_ENTRY();
  if (!(pre & kPreList)) total = tile_total(g, l, ntiles);
  for (int it = blockIdx.x; it < total; it += gridDim.x) {
    int lv = lv0, s = -1;
    long c;
    if (it == (int)blockIdx.x && (pre & kPreList)) {
      c = c0;
      s = s0;
    } else {
      c = tile_cell<D>(g, l, tiles, ntiles, it, &lv);
    }
    if (c < 0) continue;
    if (s < 0) s = st[g.cell_off[lv] + c];
    f(lv, c, (uint8_t)s);
  }
}

template <int D>
__global__ void mr_project_level(double* V, const uint8_t* st, MRLevels g, int l,
    const int* tiles = nullptr, int ntiles = 0, int pre = 0) {
  if (!tiles) {
    AF_PDL_ENTRY();
    project_level_dev<D>(V, st, g, l, tiles, ntiles);
    return;
  }
  band_cells_pdl<D>(g, l, tiles, ntiles, st, pre,
                    [&](int lv, long c, uint8_t s) { project_cell<D>(V, g, lv, c, s); });
}

// ------------------------------------------------------------ prediction --
// axis_stencil (mr_tree.cpp:199-236): positions and the weights of the low
// (hi == 0) or high (hi == 1) child along one axis. Returned by value with
// constant-indexed members so everything stays in registers.
struct AxisW {
  int p0, p1, p2;
  double w0, w1, w2;
};

__device__ __forceinline__ AxisW axis_weights(int n, int coord, bool periodic, int hi) {
  AxisW s;
  if (periodic || (coord > 0 && coord < n - 1)) {
    s.p0 = coord - 1; s.p1 = coord; s.p2 = coord + 1;
    if (periodic) {  // value_at wraps periodic axes
      s.p0 = ((s.p0 % n) + n) % n;
      s.p1 = ((s.p1 % n) + n) % n;
      s.p2 = ((s.p2 % n) + n) % n;
    }
    s.w0 = hi ? -1.0 / 8.0 : 1.0 / 8.0;
    s.w1 = 1.0;
    s.w2 = hi ? 1.0 / 8.0 : -1.0 / 8.0;
    return s;
  }
  if (n == 1) {
    s.p0 = s.p1 = s.p2 = 0;
    s.w0 = 1.0; s.w1 = 0.0; s.w2 = 0.0;
    return s;
  }
  if (n == 2) {
    s.p0 = 0; s.p1 = 1; s.p2 = 1;
    if (coord == 0) {
      s.w0 = hi ? 3.0 / 4.0 : 5.0 / 4.0;
      s.w1 = hi ? 1.0 / 4.0 : -1.0 / 4.0;
    } else {
      s.w0 = hi ? -1.0 / 4.0 : 1.0 / 4.0;
      s.w1 = hi ? 5.0 / 4.0 : 3.0 / 4.0;
    }
    s.w2 = 0.0;
    return s;
  }
  if (coord == 0) {
    s.p0 = 0; s.p1 = 1; s.p2 = 2;
    s.w0 = hi ? 5.0 / 8.0 : 11.0 / 8.0;
    s.w1 = hi ? 4.0 / 8.0 : -4.0 / 8.0;
    s.w2 = hi ? -1.0 / 8.0 : 1.0 / 8.0;
  } else {
    s.p0 = n - 3; s.p1 = n - 2; s.p2 = n - 1;
    s.w0 = hi ? 1.0 / 8.0 : -1.0 / 8.0;
    s.w1 = hi ? -4.0 / 8.0 : 4.0 / 8.0;
    s.w2 = hi ? 11.0 / 8.0 : 5.0 / 8.0;
  }
  return s;
}

__device__ __forceinline__ int axw_p(const AxisW& s, int t) { return t == 0 ? s.p0 : t == 1 ? s.p1 : s.p2; }
__device__ __forceinline__ double axw_w(const AxisW& s, int t) { return t == 0 ? s.w0 : t == 1 ? s.w1 : s.w2; }

// Prediction of child `ch` (x-fastest child bits) of the level-(l-1) parent
// (pi,pj,pk) from the dense values of level l-1 (predict_children,
// mr_tree.cpp:238-279: weights w = wx * (wy * wz), zero weights skipped,
// accumulation ck -> cj -> ci).
template <int D>
__device__ __forceinline__ void predict_child(const MRLevels& g, const double* V, long comp,
                                              long poff, int pn, int bcx, int bcy, int bcz, int pi, int pj, int pk,
                                              int ch, double* out) {
  constexpr int NC = D + 2;
  constexpr int NZ = D == 3 ? 3 : 1;
  const AxisW sx = axis_weights(pn, pi, bcx == AF_BC_PERIODIC, ch & 1);
  const AxisW sy = axis_weights(pn, pj, bcy == AF_BC_PERIODIC, (ch >> 1) & 1);
  AxisW sz;
  if constexpr (D == 3) sz = axis_weights(pn, pk, bcz == AF_BC_PERIODIC, (ch >> 2) & 1);
#pragma unroll
  for (int m = 0; m < NC; ++m) out[m] = 0.0;
#pragma unroll
  for (int ck = 0; ck < NZ; ++ck) {
    const double wk = D == 3 ? axw_w(sz, ck) : 1.0;
    if (wk == 0.0) continue;
    // the stencil's loads first (positions are always in range) so they are
    // in flight together, then the ordered accumulation: the whole 3x3 plane
    // in 2D, one row at a time in 3D (register budget)
    constexpr int RB = D == 3 ? 1 : 3;  // rows per load batch
#pragma unroll
    for (int cj0 = 0; cj0 < 3; cj0 += RB) {
      double v[RB][3][NC];
#pragma unroll
      for (int r = 0; r < RB; ++r)
#pragma unroll
        for (int ci = 0; ci < 3; ++ci) {
          const long c = poff + mr_idx(g, D, pn, axw_p(sx, ci), axw_p(sy, cj0 + r),
                                       D == 3 ? axw_p(sz, ck) : 0);
#pragma unroll
          for (int m = 0; m < NC; ++m) v[r][ci][m] = V[m * comp + c];
        }
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const double wjk = axw_w(sy, cj0 + r) * wk;
        if (wjk == 0.0) continue;
#pragma unroll
        for (int ci = 0; ci < 3; ++ci) {
          const double w = axw_w(sx, ci) * wjk;
          if (w == 0.0) continue;
#pragma unroll
          for (int m = 0; m < NC; ++m) out[m] = out[m] + v[r][ci][m] * w;
        }
      }
    }
  }
}

// Fills ABSENT cells of level l (l >= 1) with their prediction from level
// l-1: value_at / predict_single for absent nodes (mr_tree.cpp:171-180,
// 281-289). Virtual leaves (children of a leaf marked in `vmark`, materialised
// by add_virtual_leaves, mr_tree.cpp:513-551) keep their stored value unless
// their parent level is in [lo, hi] — refresh_virtuals (mr_solver.cpp:195-208)
// re-predicts only the virtual children of the stepping leaves.
// One cell of predict_level_dev (s: its status; `dense`: a launch over the
// whole level rather than band tiles).
template <int D>
__device__ __forceinline__ void predict_cell(double* V, const uint8_t* vmark, const MRLevels& g,
                                             int l, long c, uint8_t s, int lo, int hi, bool dense) {
  constexpr int NC = D + 2;
  const int n = 1 << l, pn = n >> 1;
  const long off = g.cell_off[l], poff = g.cell_off[l - 1];
  const long comp = g.total_cells;
  const bool refresh_virtual = l - 1 >= lo && l - 1 <= hi;
  if (dense && g.dist && !row_in_region(g, l, mr_row(g, D, l, c))) return;  // dense: own rows
  if (s != ST_ABSENT) return;
  int i, j, k;
  mr_ijk(g, D, l, c, i, j, k);
  if (!refresh_virtual && vmark && vmark[poff + mr_idx(g, D, pn, i >> 1, j >> 1, k >> 1)]) return;
  const int ch = (i & 1) | ((j & 1) << 1) | (D == 3 ? ((k & 1) << 2) : 0);
  double q[NC];
  predict_child<D>(g, V, comp, poff, pn, g.bc[0], g.bc[2], g.bc[4], i >> 1, j >> 1, k >> 1, ch, q);
#pragma unroll
  for (int m = 0; m < NC; ++m) V[m * comp + off + c] = q[m];
}

// Fills ABSENT cells of level l (l >= 1) with their prediction from level
// l-1: value_at / predict_single for absent nodes (mr_tree.cpp:171-180,
// 281-289). Virtual leaves (children of a leaf marked in `vmark`, materialised
// by add_virtual_leaves, mr_tree.cpp:513-551) keep their stored value unless
// their parent level is in [lo, hi] — refresh_virtuals (mr_solver.cpp:195-208)
// re-predicts only the virtual children of the stepping leaves.
template <int D>
__device__ __forceinline__ void predict_level_dev(double* V, const uint8_t* st, const uint8_t* vmark,
                                 const MRLevels& g, int l, int lo, int hi,
    const int* tiles, int ntiles) {
  level_cells<D>(g, l, tiles, ntiles, [&](const int lv, long c) {
    // dense launches stay in this rank's rows (windowed arrays are unmapped
    // elsewhere): the region test comes before the status load
    if (!tiles && g.dist && !row_in_region(g, lv, mr_row(g, D, lv, c))) return;
    predict_cell<D>(V, vmark, g, lv, c, st[g.cell_off[lv] + c], lo, hi, false);
  });
}

template <int D>
__global__ void mr_predict_level(double* V, const uint8_t* st, const uint8_t* vmark,
                                 MRLevels g, int l, int lo, int hi,
    const int* tiles = nullptr, int ntiles = 0, int pre = 0) {
  if (!tiles) {
    AF_PDL_ENTRY();
    predict_level_dev<D>(V, st, vmark, g, l, lo, hi, tiles, ntiles);
    return;
  }
  band_cells_pdl<D>(g, l, tiles, ntiles, st, pre, [&](int lv, long c, uint8_t s) {
    predict_cell<D>(V, vmark, g, lv, c, s, lo, hi, false);
  });
}

// ---------------------------------------------------------------- detail --
// detail / detail_between (mr_tree.cpp:291-317): max over children and
// components of |q_child - pred_child| / norm_k. Zero numerators are returned
// directly (0/x == 0 exactly) to stay off the division slow path.
// Child-parallel iteration over the nodes: 2^D consecutive lanes share one
// node (lane & (2^D-1) = child index, x-fastest), so each child's prediction
// runs on its own lane and the per-node reductions are 2^D-lane shuffles. A
// tile's 2^D*256 (node, child) items are spread over 2^D blocks. Every lane of
// a warp runs the same trip count (valid=false on the padding), which keeps
// the shuffles convergent. Blocks are 256 threads. f(level, node, valid, child).
// Entry (tile t of level l, repetition r) of the child-parallel iteration:
// this lane's node c (valid: inside the level) and child index ch.
template <int D>
__device__ __forceinline__ void node_child_entry(const MRLevels& g, int l, int t, int r, long* c,
                                                 bool* valid, int* ch) {
  constexpr int NCH = 1 << D;
  constexpr int TX = D == 3 ? kTileX3 : kTileX2, TY = D == 3 ? kTileY3 : kTileY2;
  const int n = 1 << l, ntx = g.ntx[l], nty = g.nty[l];
  const int sx = ilog2i(ntx), sy = ilog2i(nty);
  const int x0 = (t & (ntx - 1)) * TX, y0 = ((t >> sx) & (nty - 1)) * TY;
  const int z0 = D == 3 ? (t >> (sx + sy)) * kTileZ3 : 0;
  const int item = r * 256 + (int)threadIdx.x, tn = item >> D;
  const int x = x0 + tn % TX, y = y0 + (tn / TX) % TY, z = D == 3 ? z0 + tn / (TX * TY) : 0;
  *valid = x < n && y < n && (D == 2 || z < n);
  *c = *valid ? mr_idx(g, D, n, x, y, z) : 0L;
  *ch = item & (NCH - 1);
}

template <int D, class F>
__device__ __forceinline__ void level_nodes_by_child(const MRLevels& g, int l, const int* tiles,
                                                     int ntiles, F&& f) {
  constexpr int NCH = 1 << D;
  if (tiles) {
    for_each_tile(g, l, tiles, ntiles, NCH, [&](int lv, int t, int r) {
      long c;
      bool valid;
      int ch;
      node_child_entry<D>(g, lv, t, r, &c, &valid, &ch);
      f(lv, c, valid, ch);
    });
  } else {
    const long total = mr_cells(D, l) << D;
    for (long base = (long)blockIdx.x * blockDim.x; base < total; base += (long)gridDim.x * blockDim.x) {
      const long item = base + threadIdx.x;
      const bool valid = item < total;
      f(l, valid ? item >> D : 0L, valid, (int)(item & (NCH - 1)));
    }
  }
}

// max / all over the 2^D lanes of one node (all 32 lanes must call)
template <int D>
__device__ __forceinline__ double node_group_max(double v) {
#pragma unroll
  for (int o = 1; o < (1 << D); o <<= 1) {
    const double w = __shfl_xor_sync(0xffffffffu, v, o);
    v = v > w ? v : w;
  }
  return v;
}
template <int D>
__device__ __forceinline__ bool node_group_all(bool b) {
  const unsigned m = __ballot_sync(0xffffffffu, b);
  const unsigned gm = ((1u << (1 << D)) - 1u) << ((threadIdx.x & 31) & ~((1 << D) - 1));
  return (m & gm) == gm;
}

// |d| / norm for the detail (d >= 0, norm > 0): exactly 0 for d == 0 (most
// cells of piecewise-constant data), else the correctly rounded quotient on
// the fast-path division (fdiv), with the IEEE division of the same nonzero
// numerator when fdiv's range test fails. Neither path divides a zero.
__device__ __forceinline__ double detail_ratio(double d, double norm) {
  const double num = d == 0.0 ? 1.0 : d;
  bool ok = true;
  double q = fdiv(num, norm, ok);
  if (!ok) asm("div.rn.f64 %0, %1, %2;" : "=d"(q) : "d"(num), "d"(norm));
  return d == 0.0 ? 0.0 : q;
}

// MRTree::detail / detail_between (mr_tree.cpp:291-317) restricted to ONE child:
// max over components of |q_child - prediction| / norm. The node's detail is
// the max of this over its 2^d children (node_group_max); every term is >= 0,
// so the reduction order does not change the result.
template <int D>
__device__ __forceinline__ double child_detail(const double* V, long comp, const MRLevels& g,
                                               int l, int i, int j, int k, int ch,
                                               const double* norms) {
  constexpr int NC = D + 2;
  const int n = 1 << l, nf = n << 1;
  const long off = g.cell_off[l], foff = g.cell_off[l + 1];
  // the child's own values first: their loads overlap the stencil's
  const long fc = foff + mr_idx(g, D, nf, 2 * i + (ch & 1), 2 * j + ((ch >> 1) & 1),
                                D == 3 ? 2 * k + ((ch >> 2) & 1) : 0);
  double cv[NC];
#pragma unroll
  for (int m = 0; m < NC; ++m) cv[m] = V[m * comp + fc];
  double pred[NC];
  predict_child<D>(g, V, comp, off, n, g.bc[0], g.bc[2], g.bc[4], i, j, k, ch, pred);
  double mag = 0.0;
#pragma unroll
  for (int m = 0; m < NC; ++m) {
    const double d = fabs(cv[m] - pred[m]);
    // norms index: rho 0, mom 1..D, rhoE 4 (the 2D mom2 term is 0/global == 0)
    const int ni = m == NC - 1 ? 4 : m;
    const double r = detail_ratio(d, norms[ni]);
    mag = mag > r ? mag : r;  // std::max(mag, r)
  }
  return mag;
}

// Detail of every INTERNAL node at level l (child-parallel).
// With `flag`, each child lane also takes refine's decision for its child
// (mr_tree.cpp:364-372): a LEAF child at level l+1 in [1, L-1] is flagged
// when the parent's detail is >= eps_{l+1} (flag[] zeroed beforehand).
template <int D>
__global__ void mr_detail_level(const double* V, const uint8_t* st, double* det, MRLevels g,
                                int l, const double* norms, uint8_t* flag,
    const int* tiles = nullptr, int ntiles = 0) {
  AF_PDL_ENTRY();
  level_nodes_by_child<D>(g, l, tiles, ntiles, [&](const int lv_, long c, bool valid, int ch) {
    const int l = lv_;
    const int n = 1 << l;
    const long off = g.cell_off[l];
    const bool internal = valid && st[off + c] == ST_INTERNAL;
    int i, j, k;
  mr_ijk(g, D, l, c, i, j, k);
    const long fc = g.cell_off[l + 1] +
                    mr_idx(g, D, n << 1, 2 * i + (ch & 1), 2 * j + ((ch >> 1) & 1),
                           D == 3 ? 2 * k + ((ch >> 2) & 1) : 0);
    // refine reads the details of the parents of splittable leaves only
    const bool split_leaf = flag && internal && l + 1 <= g.L - 1 && st[fc] == ST_LEAF;
    const bool need = flag ? !node_group_all<D>(!split_leaf) : internal;
    double r = 0.0;
    if (need && internal) r = child_detail<D>(V, g.total_cells, g, l, i, j, k, ch, norms);
    r = node_group_max<D>(r);
    if (!flag && internal && ch == 0) det[off + c] = r;
    if (split_leaf) flag[fc] = r >= g.eps_l[l + 1] ? 1 : 0;
  });
}

// Buffer dilation of the LT refine (mr_tree.cpp:374-396): every leaf within
// Chebyshev radius r of a flagged leaf (same level, bc-mapped) is flagged too.
// flag[] holds 1 for detail-flagged leaves; this pass writes 2 for dilated.
template <int D>
__global__ void mr_dilate_level(const uint8_t* st, const uint8_t* flag, uint8_t* flag2,
                                MRLevels g, int l, int r,
    const int* tiles = nullptr, int ntiles = 0) {
  AF_PDL_ENTRY();
  // Target t is inserted iff some detail-flagged source s has map(s + o) == t
  // for an offset o != 0 with |o|_inf <= r. Clamping and folding never move a
  // position farther from s, so scanning the in-domain (or periodically
  // wrapped) sources s = t - o is exhaustive.
  level_cells<D>(g, l, tiles, ntiles, [&](const int lv_, long c) {
    const int l = lv_;
    const int n = 1 << l;
    const long cells = mr_cells(D, l), off = g.cell_off[l];
    uint8_t f = flag[off + c];
    if (!f && st[off + c] == ST_LEAF) {
      int t[3];
      mr_ijk(g, D, l, c, t[0], t[1], t[2]);
      const int rz = D == 3 ? r : 0;
      for (int dk = -rz; dk <= rz && !f; ++dk)
        for (int dj = -r; dj <= r && !f; ++dj)
          for (int di = -r; di <= r && !f; ++di) {
            if (di == 0 && dj == 0 && dk == 0) continue;
            int s[3] = {t[0] - di, t[1] - dj, t[2] - dk};
            bool ok = true;
            for (int a = 0; a < D; ++a) {
              if (s[a] >= 0 && s[a] < n) continue;
              if (g.bc[2 * a] == AF_BC_PERIODIC)
                s[a] = ((s[a] % n) + n) % n;
              else
                ok = false;
            }
            if (ok && flag[off + mr_idx(g, D, n, s[0], s[1], s[2])] == 1) f = 2;
          }
    }
    flag2[off + c] = f;
  });
}

template <int D>
__global__ void mr_apply_split_level(uint8_t* st, const uint8_t* flag, MRLevels g, int l,
                                     int* changed,
    const int* tiles = nullptr, int ntiles = 0) {
  AF_PDL_ENTRY();
  level_cells<D>(g, l, tiles, ntiles, [&](const int lv_, long c) {
    const int l = lv_;
    const int n = 1 << l, nf = n << 1;
    const long cells = mr_cells(D, l), off = g.cell_off[l], foff = g.cell_off[l + 1];
    if (!flag[off + c] || st[off + c] != ST_LEAF || !row_owned(g, l, mr_row(g, D, l, c))) return;
    int i, j, k;
  mr_ijk(g, D, l, c, i, j, k);
    st[off + c] = ST_INTERNAL;
    for (int ch = 0; ch < (1 << D); ++ch)
      st[foff + mr_idx(g, D, nf, 2 * i + (ch & 1), 2 * j + ((ch >> 1) & 1),
                       D == 3 ? 2 * k + ((ch >> 2) & 1) : 0)] = ST_LEAF;
    *changed = 1;
  });
}

// enforce_gradedness (mr_tree.cpp:404-444), decision half of one pass: a
// leaf below L must split when a same-level face neighbour is INTERNAL with
// an INTERNAL child on the shared face. (Unique least fixpoint; decide all,
// then apply, repeat.)
template <int D>
__global__ void mr_grade_flag_level(const uint8_t* st, uint8_t* flag, MRLevels g, int l,
    const int* tiles = nullptr, int ntiles = 0) {
  AF_PDL_ENTRY();
  level_cells<D>(g, l, tiles, ntiles, [&](const int lv_, long c) {
    const int l = lv_;
    const int n = 1 << l, nf = n << 1;
    const long cells = mr_cells(D, l), off = g.cell_off[l], foff = g.cell_off[l + 1];
    uint8_t need = 0;
    if (st[off + c] == ST_LEAF && l < g.L) {
      int idx[3];
      mr_ijk(g, D, l, c, idx[0], idx[1], idx[2]);
      for (int a = 0; a < D && !need; ++a)
        for (int dir = -1; dir <= 1 && !need; dir += 2) {
          int p[3] = {idx[0], idx[1], idx[2]};
          p[a] += dir;
          const bool per = g.bc[2 * a] == AF_BC_PERIODIC;
          if (!per && (p[a] < 0 || p[a] >= n)) continue;
          bool fl;
          p[a] = mr_map(p[a], n, g.bc[2 * a], g.bc[2 * a + 1], fl);
          if (st[off + mr_idx(g, D, n, p[0], p[1], p[2])] != ST_INTERNAL) continue;
          const int face_bit = dir > 0 ? 0 : 1;
          const int b1 = a == 0 ? 1 : 0, b2 = a == 2 ? 1 : 2;
          const int tzn = D == 3 ? 2 : 1;
          for (int t2 = 0; t2 < tzn && !need; ++t2)
            for (int t1 = 0; t1 < 2 && !need; ++t1) {
              int ci[3];
              ci[a] = 2 * p[a] + face_bit;
              ci[b1] = 2 * p[b1] + t1;
              ci[b2] = D == 3 ? 2 * p[b2] + t2 : 0;
              if (st[foff + mr_idx(g, D, nf, ci[0], ci[1], ci[2])] == ST_INTERNAL) need = 1;
            }
        }
    }
    flag[off + c] = need;
  });
}

// coarsen (mr_tree.cpp:446-511), one level of one finest-first sweep:
// an INTERNAL node at level l >= min_leaf merges iff all children are leaves,
// detail < eps_{l+1}, and no face-ring cell at level l+1 is INTERNAL.
// One (node, child) lane of a coarsen sweep at level l. rpre: the node's
// detail (node_group_max'd) when the caller computed it already.
template <int D>
__device__ __forceinline__ void coarsen_node(const double* V, uint8_t* st, const MRLevels& g,
                                             int l, double eps, const double* norms, int* merged,
                                             long c, bool valid, int ch, const double* rpre) {
  const int n = 1 << l, nf = n << 1;
  const long off = g.cell_off[l], foff = g.cell_off[l + 1];
  int idx[3];
      mr_ijk(g, D, l, c, idx[0], idx[1], idx[2]);
  int cc[3];
  cc[0] = 2 * idx[0] + (ch & 1);
  cc[1] = 2 * idx[1] + ((ch >> 1) & 1);
  cc[2] = D == 3 ? 2 * idx[2] + ((ch >> 2) & 1) : 0;
  const long fc = foff + mr_idx(g, D, nf, cc[0], cc[1], cc[2]);
  // candidate: INTERNAL node whose children are all leaves (mr_tree.cpp:486-497)
  const bool cand = node_group_all<D>(valid && st[off + c] == ST_INTERNAL && st[fc] == ST_LEAF &&
                                      row_owned(g, l, mr_row(g, D, l, c)));
  double r = 0.0;
  if (rpre) {
    r = *rpre;  // computed before the PDL wait for every INTERNAL node
  } else {
    if (cand) r = child_detail<D>(V, g.total_cells, g, l, idx[0], idx[1], idx[2], ch, norms);
    r = node_group_max<D>(r);
  }
  bool allowed = true;
  if (cand && r < eps) {
    // merge_allowed (mr_tree.cpp:446-471): no INTERNAL level-(l+1) cell
    // face-adjacent to the children. This lane checks its child's D outward
    // neighbours; the 2^d lanes together cover every position.
#pragma unroll
    for (int a = 0; a < D; ++a) {  // unrolled: g.bc[] stays in the param space
      int q[3] = {cc[0], cc[1], cc[2]};
      q[a] = ((ch >> a) & 1) ? 2 * idx[a] + 2 : 2 * idx[a] - 1;
      const bool per = g.bc[2 * a] == AF_BC_PERIODIC;
      if (!per && (q[a] < 0 || q[a] >= nf)) continue;
      bool fl;
      q[a] = mr_map(q[a], nf, g.bc[2 * a], g.bc[2 * a + 1], fl);
      if (st[foff + mr_idx(g, D, nf, q[0], q[1], q[2])] == ST_INTERNAL) allowed = false;
    }
  }
  const bool merge = node_group_all<D>(cand && r < eps && allowed);
  if (merge) {
    // merged q = mean of the children == the projection already stored
    st[fc] = ST_ABSENT;
    if (ch == 0) {
      st[off + c] = ST_LEAF;
      merged[0] = 1;
    }
    // Another sweep can only merge more if an erased child lies in the
    // prediction stencil (predict_children / axis_stencil, mr_tree.cpp:199-253)
    // of a level-(l+1) merge candidate that this sweep already evaluated:
    // that candidate's detail now sees a predicted value. Per axis the
    // stencil is {p-1, p, p+1}, or one-sided {0,1,2} / {n-3,n-2,n-1} at a
    // non-periodic wall, so the candidates within reach of child position p
    // are p-1..p+1 plus 0 (p == 2) or n-1 (p == n-3). Flag merged[1] when
    // any of them is a candidate (INTERNAL with all-leaf children).
    if (l + 2 <= g.L) {
      const long ffoff = g.cell_off[l + 2];
      const int nff = nf << 1;
      int pos[3][4];
      bool okp[3][4];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        if (a >= D) {
          pos[a][0] = 0, okp[a][0] = true;
          pos[a][1] = pos[a][2] = pos[a][3] = 0;
          okp[a][1] = okp[a][2] = okp[a][3] = false;
          continue;
        }
        const bool per = g.bc[2 * a] == AF_BC_PERIODIC;
        const int p = cc[a];
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          int q = p - 1 + t;
          bool ok = true;
          if (q < 0 || q >= nf) {
            if (per) q = (q + nf) % nf;
            else ok = false;
          }
          pos[a][t] = q, okp[a][t] = ok;
        }
        pos[a][3] = p == 2 ? 0 : nf - 1;
        okp[a][3] = !per && nf > 2 && (p == 2 || p == nf - 3);
      }
      bool hit = false;
#pragma unroll
      for (int tz = 0; tz < (D == 3 ? 4 : 1); ++tz)
#pragma unroll
        for (int ty = 0; ty < 4; ++ty)
#pragma unroll
          for (int tx = 0; tx < 4; ++tx) {
            if (!(okp[0][tx] && okp[1][ty] && okp[2][tz])) continue;
            const int q0 = pos[0][tx], q1 = pos[1][ty], q2 = pos[2][tz];
            if (st[foff + mr_idx(g, D, nf, q0, q1, q2)] != ST_INTERNAL) continue;
            bool all = true;
            for (int c2 = 0; c2 < (1 << D) && all; ++c2)
              all = st[ffoff + mr_idx(g, D, nff, 2 * q0 + (c2 & 1), 2 * q1 + ((c2 >> 1) & 1),
                                      D == 3 ? 2 * q2 + ((c2 >> 2) & 1) : 0)] == ST_LEAF;
            hit = hit || all;
          }
      if (hit) merged[1] = 1;
    }
  }
}

template <int D>
__device__ __forceinline__ void coarsen_level_dev(const double* V, uint8_t* st, const MRLevels& g, int l, double eps,
                                 const double* norms, int* merged,
    const int* tiles, int ntiles) {
  // One lane per (node, child). Nodes at one level never interact: a merge
  // turns level-(l+1) LEAFs into ABSENT, and merge_allowed only looks for
  // level-(l+1) INTERNAL cells.
  level_nodes_by_child<D>(g, l, tiles, ntiles, [&](const int lv, long c, bool valid, int ch) {
    coarsen_node<D>(V, st, g, lv, eps, norms, merged, c, valid, ch, nullptr);
  });
}

// With kPreV (the previous launch is the next finer level's sweep, which
// writes only statuses of levels l+1 and l+2), the block's first (node, child)
// entry evaluates its detail before the PDL wait: values, tile lists and this
// level's statuses are final, so the stencil loads overlap the previous
// level's kernel. The candidate and ring tests (level-(l+1) statuses) follow
// the wait.
template <int D>
__global__ void mr_coarsen_level(const double* V, uint8_t* st, MRLevels g, int l, double eps,
                                 const double* norms, int* merged,
    const int* tiles = nullptr, int ntiles = 0, int pre = 0) {
  constexpr int NCH = 1 << D;
  if (!tiles || l < 0 || !(pre & kPreV)) {
    AF_PDL_ENTRY();
    coarsen_level_dev<D>(V, st, g, l, eps, norms, merged, tiles, ntiles);
    return;
  }
  const int total = (ntiles < 0 ? g.dcnt[l] : ntiles) * NCH;
  long c0 = 0;
  bool valid0 = false;
  int ch0 = 0;
  double r0 = 0.0;
  if ((int)blockIdx.x < total) {  // block-uniform
    const int ti = blockIdx.x / NCH;
    node_child_entry<D>(g, l, tiles[ti], blockIdx.x - ti * NCH, &c0, &valid0, &ch0);
    const int n = 1 << l;
    if (valid0 && st[g.cell_off[l] + c0] == ST_INTERNAL) {
      int i0, j0, k0;
      mr_ijk(g, D, l, c0, i0, j0, k0);
      r0 = child_detail<D>(V, g.total_cells, g, l, i0, j0, k0, ch0, norms);
    }
    r0 = node_group_max<D>(r0);
  }
  AF_PDL_ENTRY();
  for (int it = blockIdx.x; it < total; it += gridDim.x) {
    if (it == (int)blockIdx.x) {
      coarsen_node<D>(V, st, g, l, eps, norms, merged, c0, valid0, ch0, &r0);
    } else {
      const int ti = it / NCH;
      long c;
      bool valid;
      int ch;
      node_child_entry<D>(g, l, tiles[ti], it - ti * NCH, &c, &valid, &ch);
      coarsen_node<D>(V, st, g, l, eps, norms, merged, c, valid, ch, nullptr);
    }
  }
}

// The coarsest levels (at most kTinyCells cells each: 2D up to level 5,
// 3D up to level 3) in ONE single-CTA launch, a __syncthreads between levels
// keeping the level order (prediction coarsest first, projection finest
// first). Each of these levels is shorter than a kernel launch; as separate
// launches they cost ~4 us apiece in the cycle graph. (Coarsening stays one
// launch per level: its child-parallel details on one CTA were slower.)
// Every cell of such a level is visited (a superset of its band tiles).
// Not used with ranks (windowed arrays: dense visits would leave the rows).
constexpr int kTinyCells = 1024;
constexpr int kTinyThreads = 512;  // 128 registers a thread (the predictions need them)

template <int D>
__global__ void __launch_bounds__(kTinyThreads) mr_predict_tiny(double* V, const uint8_t* st,
                                                                const uint8_t* vmark, MRLevels g,
                                                                int lfrom, int lto, int lo, int hi) {
  AF_PDL_ENTRY();
  for (int l = lfrom; l <= lto; ++l) {
    const long cells = mr_cells(D, l);
    for (long c = threadIdx.x; c < cells; c += blockDim.x)
      predict_cell<D>(V, vmark, g, l, c, st[g.cell_off[l] + c], lo, hi, false);
    __syncthreads();
  }
}

template <int D>
__global__ void __launch_bounds__(kTinyThreads) mr_project_tiny(double* V, const uint8_t* st,
                                                                MRLevels g, int lhigh, int llow) {
  AF_PDL_ENTRY();
  for (int l = lhigh; l >= llow; --l) {
    const long cells = mr_cells(D, l);
    for (long c = threadIdx.x; c < cells; c += blockDim.x)
      project_cell<D>(V, g, l, c, st[g.cell_off[l] + c]);
    __syncthreads();
  }
}

// Virtual-leaf count (add_virtual_leaves, mr_tree.cpp:513-551): a level-(l-1)
// leaf P gets 2^d virtual children when some axis-stencil position (+-1, +-2)
// of a level-l leaf maps into an absent child of P. Marks P in `mark`.
template <int D>
__global__ void mr_virtual_mark_level(const uint8_t* st, uint8_t* mark, MRLevels g, int l,
    const int* tiles = nullptr, int ntiles = 0) {
  AF_PDL_ENTRY();
  level_cells<D>(g, l, tiles, ntiles, [&](const int lv_, long c) {
    const int l = lv_;
    const int n = 1 << l, pn = n >> 1;
    const long cells = mr_cells(D, l), off = g.cell_off[l], poff = g.cell_off[l - 1];
    if (st[off + c] != ST_LEAF) return;
    int idx[3];
      mr_ijk(g, D, l, c, idx[0], idx[1], idx[2]);
    for (int a = 0; a < D; ++a)
      for (int o = -2; o <= 2; ++o) {
        if (o == 0) continue;
        int p[3] = {idx[0], idx[1], idx[2]};
        p[a] += o;
        const bool per = g.bc[2 * a] == AF_BC_PERIODIC;
        if (!per && (p[a] < 0 || p[a] >= n)) continue;
        bool fl;
        p[a] = mr_map(p[a], n, g.bc[2 * a], g.bc[2 * a + 1], fl);
        if (st[off + mr_idx(g, D, n, p[0], p[1], p[2])] != ST_ABSENT) continue;
        const long pc = poff + mr_idx(g, D, pn, p[0] >> 1, p[1] >> 1, p[2] >> 1);
        if (st[pc] == ST_LEAF && row_owned(g, l - 1, p[D - 1] >> 1)) mark[pc] = 1;
      }
  });
}

// Counts per level: [0] leaves, [1] internals, [2] virtual-marked parents.
static __global__ void mr_count_kernel(const uint8_t* st, const uint8_t* mark, long n,
                                unsigned long long* out, MRLevels g) {
  AF_PDL_ENTRY();
  unsigned long long lv = 0, in = 0, vm = 0;
  for (long c = blockIdx.x * (long)blockDim.x + threadIdx.x; c < n;
       c += (long)gridDim.x * blockDim.x) {
    if (g.dist) {  // count each cell on one rank only
      int l = 0;
      while (c >= g.cell_off[l + 1]) ++l;
      if (!row_counted(g, l, mr_row(g, g.dim, l, c - g.cell_off[l]))) continue;
    }
    const uint8_t s = st[c];
    lv += s == ST_LEAF;
    in += s == ST_INTERNAL;
    if (mark) vm += mark[c];
  }
  for (int o = 16; o > 0; o >>= 1) {
    lv += __shfl_xor_sync(0xffffffffu, lv, o);
    in += __shfl_xor_sync(0xffffffffu, in, o);
    vm += __shfl_xor_sync(0xffffffffu, vm, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (lv) atomicAdd(out, lv);
    if (in) atomicAdd(out + 1, in);
    if (vm) atomicAdd(out + 2, vm);
  }
}

// mr_count_kernel and, in the same pass over the cells (with `speed`), the
// CFL rule's max over leaves of sum_a(|v_a|+c) into out[3] (one rank).
template <int D>
__global__ void mr_count_speed_kernel(const uint8_t* st, const uint8_t* mark, long n,
                                      unsigned long long* out, MRLevels g, const double* V,
                                      double gamma, int speed) {
  AF_PDL_ENTRY();
  unsigned long long lv = 0, in = 0, vm = 0;
  double best = 0.0;
  const long comp = g.total_cells;
  for (long c = blockIdx.x * (long)blockDim.x + threadIdx.x; c < n;
       c += (long)gridDim.x * blockDim.x) {
    const uint8_t s = st[c];
    lv += s == ST_LEAF;
    in += s == ST_INTERNAL;
    if (mark) vm += mark[c];
    if (speed && s == ST_LEAF) {
      Cons<D> q;
      q.rho = V[c];
#pragma unroll
      for (int a = 0; a < D; ++a) q.m[a] = V[(1 + a) * comp + c];
      q.E = V[(D + 1) * comp + c];
      double sum, m;
      wave_speeds(primitives(q, gamma - 1.0), gamma, sum, m);
      best = fmax(best, sum);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    lv += __shfl_xor_sync(0xffffffffu, lv, o);
    in += __shfl_xor_sync(0xffffffffu, in, o);
    vm += __shfl_xor_sync(0xffffffffu, vm, o);
  }
  best = warp_max(best);
  if ((threadIdx.x & 31) == 0) {
    if (lv) atomicAdd(out, lv);
    if (in) atomicAdd(out + 1, in);
    if (vm) atomicAdd(out + 2, vm);
    if (best > 0.0) atomicMax(out + 3, dbits(best));
  }
}

// Max over leaves of sum_a(|v_a|+c) (CFL rule) for the leaves of level l.
template <int D>
__global__ void mr_leaf_speed_kernel(const double* V, const uint8_t* st, MRLevels g, int l,
                                     double gamma, unsigned long long* target,
                                     const int* tiles = nullptr, int ntiles = 0) {
  AF_PDL_ENTRY();
  __shared__ double red[8];
  double best = 0.0;
  level_cells<D>(g, l, tiles, ntiles, [&](const int lv_, long c) {
    const int l = lv_;
    const long off = g.cell_off[l], comp = g.total_cells;
    if (st[off + c] != ST_LEAF || !row_owned(g, l, mr_row(g, D, l, c))) return;
    Cons<D> q;
    q.rho = V[off + c];
#pragma unroll
    for (int a = 0; a < D; ++a) q.m[a] = V[(1 + a) * comp + off + c];
    q.E = V[(D + 1) * comp + off + c];
    double s, m;
    wave_speeds(primitives(q, gamma - 1.0), gamma, s, m);
    best = fmax(best, s);
  });
  block_max_atomic<256>(best, red, target);
}

// Per-component max |q| of the finest level (set_norms_from, mr_tree.cpp:73-87).
template <int D>
__global__ void mr_norm_kernel(const double* V, MRLevels g, unsigned long long* out) {
  AF_PDL_ENTRY();
  constexpr int NC = D + 2;
  const long cells = mr_cells(D, g.L), off = g.cell_off[g.L], comp = g.total_cells;
  double mx[NC];
#pragma unroll
  for (int m = 0; m < NC; ++m) mx[m] = 0.0;
  for (long c = blockIdx.x * (long)blockDim.x + threadIdx.x; c < cells;
       c += (long)gridDim.x * blockDim.x) {
    if (g.dist && !row_owned(g, g.L, mr_row(g, D, g.L, c))) continue;  // max over ranks after
#pragma unroll
    for (int m = 0; m < NC; ++m) mx[m] = fmax(mx[m], fabs(V[m * comp + off + c]));
  }
#pragma unroll
  for (int m = 0; m < NC; ++m) {
    double v = warp_max(mx[m]);
    if ((threadIdx.x & 31) == 0 && v > 0.0) atomicMax(out + m, dbits(v));
  }
}

}  // namespace af
