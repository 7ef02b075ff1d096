// af_mr_types.h — MR level geometry shared by host and device code.
#pragma once

#include <cstdint>

namespace af {

enum : uint8_t { ST_ABSENT = 0, ST_LEAF = 1, ST_INTERNAL = 2 };

// Per-level geometry shared by all MR kernels.
struct MRLevels {
  int dim;
  int L;
  int nc;                  // stored components (4 in 2D, 5 in 3D)
  int bc[6];
  long cell_off[17];       // first cell of level l in the concatenated level arrays
  long total_cells;
  double inv_dx[17];       // 1 / dx_l, dx_l = extent / 2^l (mr_tree.hpp:73, mr_solver.cpp:181)
  // work tiles (2D 32x8, 3D 8x8x4 cells = 256 threads): per-level tile grid
  int ntx[17], nty[17], ntz[17];
  long tile_off[17];       // first tile of level l in the concatenated tile space
  int band_cnt[17];        // tiles in the level's band list (host-filled)
  int leaf_cnt[17];        // tiles in the level's leaf-tile list
  double eps_l[17];        // refine threshold for leaves of level l (host-filled)
  const int* dcnt;         // device copy of the counts: [l] band, [17 + l] leaf tiles
  // Spatial decomposition: slabs of rows along the last
  // axis (y in 2D, z in 3D). A rank computes and decides for the rows it owns,
  // [own_lo, own_hi), and keeps up-to-date copies of the rows within
  // the halo depth of them, [reg_lo, reg_hi) (may wrap when that axis is periodic).
  // Levels below `lp` are replicated (no leaves or absent cells there) and are
  // counted by rank 0 only (`count_rep`). One rank: everything owned.
  int own_lo[17], own_hi[17];
  int reg_lo[17], reg_hi[17];
  int lp;
  int count_rep;
  int dist;                // more than one rank
  // Cell order inside a level (af_mr_storage.cu). bsh = 0: row-major (x
  // fastest). bsh > 0 (3D only): levels finer than 2^bsh cells per axis are
  // stored as dense bricks of 2^bsh cells per axis, brick after brick
  // (bricks row-major, cells row-major inside a brick), so one brick of one
  // component is one contiguous, page-aligned run that is mapped to physical
  // memory only while the tree reaches it (AF_MR_STORAGE_SPARSE).
  int bsh;
};


__host__ __device__ __forceinline__ int mr_log2(int n) {
#ifdef __CUDA_ARCH__
  return __ffs(n) - 1;
#else
  return __builtin_ctz((unsigned)n);
#endif
}

// Index of cell (i, j, k) inside its level (n = 2^l cells per axis): row-major,
// or brick-major above the brick size (MRLevels::bsh).
__host__ __device__ __forceinline__ long mr_idx(const MRLevels& g, int D, int n, int i, int j,
                                                int k) {
  if (D == 3 && g.bsh && n > (1 << g.bsh)) {
    const int s = g.bsh, m = (1 << s) - 1, ls = mr_log2(n) - s;  // log2 bricks per axis
    const long b = ((long)(k >> s) << (2 * ls)) | ((long)(j >> s) << ls) | (i >> s);
    return (b << (3 * s)) | ((long)(k & m) << (2 * s)) | ((j & m) << s) | (i & m);
  }
  return D == 3 ? ((long)k * n + j) * n + i : (long)j * n + i;
}

// Inverse of mr_idx at level l.
__host__ __device__ __forceinline__ void mr_ijk(const MRLevels& g, int D, int l, long c, int& i,
                                                int& j, int& k) {
  const int n = 1 << l;
  if (D == 3 && g.bsh && l > g.bsh) {
    const int s = g.bsh, m = (1 << s) - 1, ls = l - s, nb = (1 << ls) - 1;
    const long b = c >> (3 * s);
    const int in = (int)(c & ((1L << (3 * s)) - 1));
    i = (int)((b & nb) << s) | (in & m);
    j = (int)(((b >> ls) & nb) << s) | ((in >> s) & m);
    k = (int)((b >> (2 * ls)) << s) | (in >> (2 * s));
    return;
  }
  i = (int)(c & (n - 1));
  j = (int)((c >> l) & (n - 1));
  k = D == 3 ? (int)(c >> (2 * l)) : 0;
}

// Slab row of cell c of level l (the last axis index).
__host__ __device__ __forceinline__ int mr_row(const MRLevels& g, int dim, int l, long c) {
  if (dim == 3 && g.bsh && l > g.bsh) {
    int i, j, k;
    mr_ijk(g, dim, l, c, i, j, k);
    return k;
  }
  return (int)(c >> ((dim - 1) * l));
}
__host__ __device__ __forceinline__ bool row_owned(const MRLevels& g, int l, int r) {
  return r >= g.own_lo[l] && r < g.own_hi[l];
}
__host__ __device__ __forceinline__ bool row_in_region(const MRLevels& g, int l, int r) {
  const int n = 1 << l, len = g.reg_hi[l] - g.reg_lo[l];
  if (len >= n) return true;
  int d = (r - g.reg_lo[l]) % n;
  if (d < 0) d += n;
  return d < len;
}
// counted once across ranks (leaf/node counts, leaves per level)
__host__ __device__ __forceinline__ bool row_counted(const MRLevels& g, int l, int r) {
  return l < g.lp ? g.count_rep != 0 : row_owned(g, l, r);
}

// Multi-level launch convention: a kernel called with l = -(lo + 1) and
// ntiles = hi << 1 | sel covers the band (sel 0) or leaf-tile (sel 1) lists of
// levels lo..hi as one flat range (for_each_tile, af_mr_kernels.cuh), `tiles`
// being the base of the concatenated per-level lists. The counts are read
// from device memory (g.dcnt) so a launch's parameters do not change from
// cycle to cycle (CUDA-graph replay). A single-level launch may pass
// ntiles = -1 (band) / -2 (leaf tiles) to read its count likewise.

// Programmatic dependent launch: MR kernels are launched with
// programmaticStreamSerialization, so a kernel may begin launching while its
// predecessor runs. Every MR kernel first waits for the predecessor grid to
// complete and its memory to be visible (griddepcontrol.wait; a no-op for an
// ordinary launch), then lets its own successor begin launching.
#define AF_PDL_ENTRY() \
  asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory")

// What a kernel may read BEFORE its griddepcontrol.wait, i.e. while its
// immediate predecessor still runs (every earlier kernel has completed: a
// kernel lets its dependents launch only after its own wait). The host sets
// the bits the predecessor does not write.
enum : int { kPreList = 1, kPreSt = 2, kPreV = 4 };  // tile lists + counts, statuses, values

constexpr int kTileX2 = 32, kTileY2 = 8;

// log2 of a power of two (tile counts and level sizes: index arithmetic
// becomes shifts and masks instead of 32/64-bit divisions)
__device__ __forceinline__ int ilog2i(int x) { return 31 - __clz(x); }
constexpr int kTileX3 = 8, kTileY3 = 8, kTileZ3 = 4;

__host__ __device__ __forceinline__ long mr_cells(int dim, int l) {
  return dim == 3 ? (1L << (3 * l)) : (1L << (2 * l));
}

}  // namespace af
