// af_mr_stage.cuh — one RK stage for the leaves of one MR level (sm_100a).
//
// MRSolver::stage (mr_solver.cpp:163-193) for the leaves of level l, as a
// tile kernel over the level's dense grid: the tile's primitives (2-cell
// halo, bc-mapped as map_position, mr_tree.cpp:146-169) are staged in shared
// memory, every face touching a leaf is evaluated once, and each leaf sums
// its 2d faces in the reference order (rhs += F(a,-)/dx; rhs -= F(a,+)/dx,
// mr_solver.cpp:182-185). Faces whose same-level neighbour is INTERNAL take
// the coarse side of the interface rule instead: the mean of the 2^(d-1)
// fine sub-face fluxes (fine_face_average, mr_solver.cpp:59-95), including
// its asymmetric low-face stencil (p-2, p-1 | p, p+2) (mr_solver.cpp:80).
#pragma once

#include <type_traits>

#include "af_mr_kernels.cuh"

namespace af {

struct MRStageArgs {
  const double* eval;  // concatenated level values the fluxes read
  const double* base;  // step-start values (q_old)
  double* snap;        // stage 1: q_old snapshot target (base is then eval itself)
  double* out;         // stage output (leaves of this level)
  const uint8_t* st;
  double gamma, gm1;
  double sdt;          // stage_dt (or dt_scale * *dt_dev when dt_dev is set)
  const double* dt_dev;
  double dt_scale;
  const int* step3_dev; // device copy of step3 (graph replay)
  int step3;           // error code base: 3*step; + stage-1 for pass 1, + 2 for post-step
  int stage;
  int post_check;      // stage 2: positivity of the completed step
  int post_stops;      // a post-step failure also stops later launches (graph mode, no commit kernel)
  unsigned long long* wave;  // per-level max (|v_a|+c) of the evaluated leaves
  unsigned long long* fb;    // fallbacks
  int* err;                  // [0] flag, [1] min code
  const int* tiles;
  int ntiles;          // tiles in the list (or the leaf-list selector 1 in multi-level mode)
  const uint8_t* tflag;  // per-tile flags of the last list build (bit 2: a "full" tile)
  // local time stepping: virtual leaves whose parent level is below `lo`
  // read as q_old*(1-theta) + q*theta (resolve, mr_solver.cpp:43-50)
  int lo, hi;
  const uint8_t* vmark;
  const double* vq_old;
  double theta[17];  // by parent level
  // flux registers (face_flux_at, mr_solver.cpp:111-159; stage 2 only)
  int reg_stage;
  double step_dt, share;
  int sub;                   // which of the two fine substeps (0/1)
  const int* regbase;        // per cell: first register of the cell
  const uint8_t* regmask;    // per cell: faces (axis*2+side) holding a register
  double* regc;              // [R][NC] coarse provisional flux * step_dt
  double* regf;              // [R][2 substeps][2^(d-1) sub-faces][NC]
  uint8_t* regfc;            // [R] has_coarse
  uint8_t* regff;            // [R] has_fine
  int* regerr;               // fine contribution without a register slot
};

__device__ __forceinline__ int reg_index(const int* base, const uint8_t* mask, long cell,
                                         int bit) {
  const unsigned m = mask[cell];
  if (!((m >> bit) & 1u)) return -1;
  return base[cell] + __popc(m & ((1u << bit) - 1u));
}

// resolve() for level l (mr_solver.cpp:36-57, global mode): bc-mapped read of
// the dense level value with the reflective momentum flip.
template <int D>
__device__ __forceinline__ Cons<D> resolve_at(const double* V, long comp, const MRLevels& g,
                                              int l, int i, int j, int k,
                                              const MRStageArgs* lt = nullptr) {
  const int n = 1 << l;
  bool fi, fj, fk = false;
  const int mi = mr_map(i, n, g.bc[0], g.bc[1], fi);
  const int mj = mr_map(j, n, g.bc[2], g.bc[3], fj);
  const int mk = D == 3 ? mr_map(k, n, g.bc[4], g.bc[5], fk) : 0;
  const long c = g.cell_off[l] + mr_idx(g, D, n, mi, mj, mk);
  Cons<D> q;
  q.rho = V[c];
#pragma unroll
  for (int a = 0; a < D; ++a) q.m[a] = V[(1 + a) * comp + c];
  q.E = V[(D + 1) * comp + c];
  if (lt && l - 1 < lt->lo && l >= 1) {
    const long pc = g.cell_off[l - 1] + mr_idx(g, D, n >> 1, mi >> 1, mj >> 1, mk >> 1);
    // a virtual leaf over an already-advanced coarser leaf: interpolate in time
    if (lt->vmark[pc] && lt->st[c] == ST_ABSENT) {
      const double th = lt->theta[l - 1], om = 1.0 - th;
      q.rho = lt->vq_old[c] * om + q.rho * th;
#pragma unroll
      for (int a = 0; a < D; ++a) q.m[a] = lt->vq_old[(1 + a) * comp + c] * om + q.m[a] * th;
      q.E = lt->vq_old[(D + 1) * comp + c] * om + q.E * th;
    }
  }
  if (fi) q.m[0] = -q.m[0];
  if (fj) q.m[1] = -q.m[1];
  if (D == 3 && fk) q.m[D - 1] = -q.m[D - 1];
  return q;
}

template <int D, int AX, int LIM>
__device__ __forceinline__ Cons<D> flux4(const Cons<D>& qa, const Cons<D>& qb, const Cons<D>& qc,
                                         const Cons<D>& qd, double gamma, double gm1, int* fb,
                                         double rgm1) {
  const Prim<D> wa = primitives(qa, gm1), wb = primitives(qb, gm1);
  const Prim<D> wc = primitives(qc, gm1), wd = primitives(qd, gm1);
  return face_flux<D, AX, LIM>(qb, qc, wa, wb, wc, wd, gamma, gm1, fb, rgm1);
}

// fine_face_average (mr_solver.cpp:59-95) of leaf (c0,c1,c2) at level l.
template <int D, int AX, int LIM>
__device__ Cons<D> fine_face_average(const double* V, long comp, const MRLevels& g, int l,
                                     const int* c, int dir, double gamma, double gm1, int* fb,
                                     double rgm1) {
  constexpr int b1 = AX == 0 ? 1 : 0;
  constexpr int b2 = AX == 2 ? 1 : 2;
  const int fl = l + 1;
  const int tzn = D == 3 ? 2 : 1;
  Cons<D> sum;
  sum.rho = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) sum.m[a] = 0.0;
  sum.E = 0.0;
  for (int t2 = 0; t2 < tzn; ++t2)
    for (int t1 = 0; t1 < 2; ++t1) {
      int p[3];
      p[AX] = 2 * c[AX] + (dir > 0 ? 1 : 0);
      p[b1] = 2 * c[b1] + t1;
      p[b2] = D == 3 ? 2 * c[b2] + t2 : 0;
      int s0[3] = {p[0], p[1], p[2]}, s2[3] = {p[0], p[1], p[2]}, s3[3] = {p[0], p[1], p[2]};
      s0[AX] += dir > 0 ? -1 : 2;  // the reference's (p-2, p-1 | p, p+2) on the low face
      s2[AX] += dir;
      s3[AX] += 2 * dir;
      const int* A = dir > 0 ? s0 : s3;
      const int* B = dir > 0 ? p : s2;
      const int* Cc = dir > 0 ? s2 : p;
      const int* Dd = dir > 0 ? s3 : s0;
      const Cons<D> qa = resolve_at<D>(V, comp, g, fl, A[0], A[1], A[2]);
      const Cons<D> qb = resolve_at<D>(V, comp, g, fl, B[0], B[1], B[2]);
      const Cons<D> qc = resolve_at<D>(V, comp, g, fl, Cc[0], Cc[1], Cc[2]);
      const Cons<D> qd = resolve_at<D>(V, comp, g, fl, Dd[0], Dd[1], Dd[2]);
      const Cons<D> f = flux4<D, AX, LIM>(qa, qb, qc, qd, gamma, gm1, fb, rgm1);
      sum.rho = sum.rho + f.rho;
#pragma unroll
      for (int a = 0; a < D; ++a) sum.m[a] = sum.m[a] + f.m[a];
      sum.E = sum.E + f.E;
    }
  const double s = 1.0 / (double)(tzn * 2);
  sum.rho = sum.rho * s;
#pragma unroll
  for (int a = 0; a < D; ++a) sum.m[a] = sum.m[a] * s;
  sum.E = sum.E * s;
  return sum;
}

template <int D, int TX, int TY, int TZ>
struct MRTile {
  static constexpr int NT = TX * TY * TZ;
  static constexpr int HX = TX + 4, HY = TY + 4, HZ = D == 3 ? TZ + 4 : 1;
  static constexpr int HP = HX * HY * HZ;
  static constexpr int NXF = (TX + 1) * TY * TZ;
  static constexpr int NYF = TX * (TY + 1) * TZ;
  static constexpr int NZF = D == 3 ? TX * TY * (TZ + 1) : 0;
  static constexpr int NF = NXF + NYF + NZF;
  static constexpr int NC = D + 2;
  static constexpr size_t smem_bytes =
      sizeof(double) * ((size_t)NC * HP + (size_t)NC * NF + NT / 32) + NF + NT + 16;
};

template <int D, int LIM, int TX, int TY, int TZ>
__global__ void __launch_bounds__(TX* TY* TZ, 2)
    mr_stage_kernel(MRStageArgs a, MRLevels g, int l) {
  AF_PDL_ENTRY();
  using K = MRTile<D, TX, TY, TZ>;
  constexpr int NC = K::NC;
  if (failed_before(a.err)) return;
  extern __shared__ double sm[];
  double* pr = sm;                        // [NC][HP] primitives
  double* fl = pr + NC * K::HP;           // [NC][NF] face fluxes
  double* red = fl + NC * K::NF;          // [NT/32]
  uint8_t* ffb = reinterpret_cast<uint8_t*>(red + K::NT / 32);  // [NF] fallback flags
  uint8_t* leaf = ffb + K::NF;            // [NT] leaf mask
  __shared__ int s_fb, s_bad;

  const double sdt = a.dt_dev ? a.dt_scale * *a.dt_dev : a.sdt;  // 0.5 * dt, 1.0 * dt == dt
  const int step3 = a.step3_dev ? *a.step3_dev : a.step3;
  const int tid = threadIdx.x, lane = tid & 31;
  const long comp = g.total_cells;
  const double gamma = a.gamma, gm1 = a.gm1;
  const double rgm1 = 1.0 / gm1;  // RN(1/(gamma-1)) for div_rcp
  if (tid == 0) {
    s_fb = 0;
    s_bad = 0;
  }
  int bad = 0, nfb = 0;
  const int tx = tid % TX, ty = (tid / TX) % TY, tz = D == 3 ? tid / (TX * TY) : 0;
  const int ntotal = tile_total(g, l, a.ntiles);
  const int lcode = l;
  TileWalker walk(g, lcode < 0 ? lcode : -1, a.ntiles);  // (used in multi-level mode only)
  // per-level max wave speed of this block's leaves: a warp max and one atomic
  // per warp when the level changes (non-negative doubles order like their bits)
  double wave = 0.0;
  int wave_l = -1;
  auto flush_wave = [&] {
    if (wave_l < 0) return;
    for (int o = 16; o > 0; o >>= 1) wave = fmax(wave, __shfl_xor_sync(0xffffffffu, wave, o));
    if (lane == 0 && wave > 0.0)
      atomicMax(a.wave + wave_l, (unsigned long long)__double_as_longlong(wave));
    wave = 0.0;
  };
  for (int it = blockIdx.x; it < ntotal; it += gridDim.x) {
  const int t = lcode < 0 ? walk.at(g, a.tiles, it, &l) : tile_at(g, lcode, a.tiles, a.ntiles, it, &l);
  const int n = 1 << l;
  const long off = g.cell_off[l];
  const int ntx = (n + TX - 1) / TX, nty = (n + TY - 1) / TY;
  const double inv_dx = g.inv_dx[l];
  if (l != wave_l) {  // block-uniform: the tiles of a block come in level order
    flush_wave();
    wave_l = l;
  }
  const int sx = ilog2i(ntx), sy = ilog2i(nty);  // powers of two
  const int x0 = (t & (ntx - 1)) * TX, y0 = ((t >> sx) & (nty - 1)) * TY;
  const int z0 = D == 3 ? (t >> (sx + sy)) * TZ : 0;
  // leaf mask of the tile cells
  const int cx = x0 + tx, cy = y0 + ty, cz = z0 + tz;
  const bool inside = cx < n && cy < n && (D == 2 || cz < n);
  const long own = inside ? off + mr_idx(g, D, n, cx, cy, cz) : 0;
  // A full tile (mr_tile_flags_all bit 2): every cell and every face
  // neighbour of the tile is a leaf of this level, so every face is a plain
  // same-level face (no fine sub-face average, no flux register) and every
  // cell is updated: the per-face leaf and status tests are skipped.
  // (2D only: in 3D the extra live state makes the kernel spill)
  const bool full = D == 2 && a.tflag && (a.tflag[g.tile_off[l] + t] & 4);
  const bool is_leaf =
      full || (inside && a.st[own] == ST_LEAF && row_owned(g, l, D == 3 ? cz : cy));
  // with ranks, a stage-2 register pass also evaluates the halo-row leaves:
  // their fine-side register shares for this rank's coarse cells
  // (face_flux_at, mr_solver.cpp:147-159) are computed here, where those
  // registers live, from the halo copy of the same inputs
  const bool is_hleaf = !is_leaf && a.reg_stage && g.dist && inside && a.st[own] == ST_LEAF &&
                        row_in_region(g, l, D == 3 ? cz : cy);
  leaf[tid] = is_leaf || is_hleaf;
  // Halo gather. In 2D both of a thread's cells are loaded before either is
  // converted, so their global-memory round trips overlap; in 3D (five cells
  // per thread) the loop stays rolled, as the extra registers would spill.
  auto halo_xyz = [&](int idx, int& ix, int& iy, int& iz) {
    ix = idx % K::HX;
    iy = (idx / K::HX) % K::HY;
    iz = D == 3 ? idx / (K::HX * K::HY) : 0;
    const bool ccx = ix >= 2 && ix < TX + 2, ccy = iy >= 2 && iy < TY + 2;
    const bool ccz = D == 2 || (iz >= 2 && iz < TZ + 2);
    return idx < K::HP && (int)!ccx + (int)!ccy + (int)!ccz <= 1;  // on an axis stencil
  };
  auto put_prim = [&](int idx, const Cons<D>& q) {
    const Prim<D> w = primitives(q, gm1);
#pragma unroll
    for (int m = 0; m < NC; ++m)
      pr[m * K::HP + idx] = m == 0 ? w.rho : (m == NC - 1 ? w.p : w.v[m - 1]);
  };
  if constexpr (D == 2) {
    static_assert((K::HP + K::NT - 1) / K::NT == 2, "2D: two halo cells per thread");
    Cons<D> gq[2];
    bool on[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      int ix, iy, iz;
      on[h] = halo_xyz(tid + h * K::NT, ix, iy, iz);
      if (on[h]) gq[h] = resolve_at<D>(a.eval, comp, g, l, x0 - 2 + ix, y0 - 2 + iy, 0, &a);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (on[h]) put_prim(tid + h * K::NT, gq[h]);
  } else {
    for (int idx = tid; idx < K::HP; idx += K::NT) {
      int ix, iy, iz;
      if (!halo_xyz(idx, ix, iy, iz)) continue;
      put_prim(idx, resolve_at<D>(a.eval, comp, g, l, x0 - 2 + ix, y0 - 2 + iy, z0 - 2 + iz, &a));
    }
  }
  // early loads for the update phase (step-start values, neighbour status):
  // issued before the flux work so their latency is hidden behind it
  double base0[NC];
  unsigned nbst = 0;  // 2 bits per face (axis*2 + side): the neighbour's status
  if (is_leaf) {
    // stage 1 takes the step-start values from eval and writes the q_old
    // snapshot of its leaves (step_levels, mr_solver.cpp:235-239)
#pragma unroll
    for (int m = 0; m < NC; ++m) base0[m] = (a.snap ? a.eval : a.base)[m * comp + own];
    if (a.snap) {
#pragma unroll
      for (int m = 0; m < NC; ++m) a.snap[m * comp + own] = base0[m];
    }
    const int c0[3] = {cx, cy, cz};
    if (full) nbst = 0x555u & ((1u << (4 * D)) - 1u);  // every neighbour a leaf
#pragma unroll
    for (int ax = 0; ax < D && !full; ++ax)
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        int p[3] = {c0[0], c0[1], c0[2]};
        p[ax] += side ? 1 : -1;
        bool flp;
        p[ax] = mr_map(p[ax], n, g.bc[2 * ax], g.bc[2 * ax + 1], flp);
        nbst |= (unsigned)a.st[off + mr_idx(g, D, n, p[0], p[1], p[2])] << (2 * (ax * 2 + side));
      }
  }
  __syncthreads();
  auto P = [&](int ix, int iy, int iz) {
    const int idx = (iz * K::HY + iy) * K::HX + ix;
    Prim<D> w;
    w.rho = pr[idx];
#pragma unroll
    for (int d = 0; d < D; ++d) w.v[d] = pr[(1 + d) * K::HP + idx];
    w.p = pr[(NC - 1) * K::HP + idx];
    return w;
  };
  // Pass-1 checks of this thread's leaf (mr_solver.cpp:171-178) on the
  // primitives the gather staged (a leaf is never a flipped ghost or an
  // interpolated virtual cell, so they are primitives(q) of its own q)
  if (is_leaf) {
    const Prim<D> w = P(tx + 2, ty + 2, D == 3 ? tz + 2 : 0);
    Cons<D> q;
    q.rho = w.rho;
    if (!cell_ok(q, w)) bad = 1;
    double s, m;
    wave_speeds(w, gamma, s, m);
    wave = fmax(wave, m);
  }
  auto leaf_at = [&](int x, int y, int z) {  // tile-local coords, -1/T allowed
    if (x < 0 || x >= TX || y < 0 || y >= TY || z < 0 || z >= TZ) return false;
    return leaf[(z * TY + y) * TX + x] != 0;
  };
  auto cons_at = [&](int x, int y, int z) {
    return resolve_at<D>(a.eval, comp, g, l, x, y, z, &a);
  };
  // Status of the bc-mapped cell (x, y, z) of this level (global coords).
  auto status_at = [&](int x, int y, int z) {
    bool f;
    const int mx = mr_map(x, n, g.bc[0], g.bc[1], f);
    const int my = mr_map(y, n, g.bc[2], g.bc[3], f);
    const int mz = D == 3 ? mr_map(z, n, g.bc[4], g.bc[5], f) : 0;
    return a.st[off + mr_idx(g, D, n, mx, my, mz)];
  };
  const bool fine_ok = l + 1 <= a.hi;  // the finer level steps in this call
  // Face fluxes needed by a leaf of the tile. A face between a leaf and an
  // INTERNAL same-level neighbour whose children step now gets the coarse
  // side of the interface rule, the fine sub-face average
  // (fine_face_average, mr_solver.cpp:59-95), here: one thread per face, so
  // the sub-face fluxes of different faces run in parallel.
  auto do_face = [&](auto axc, int fx, int fy, int fz, int slot) {
    constexpr int AX = decltype(axc)::value;
    const int ex = AX == 0, ey = AX == 1, ez = AX == 2;
    const bool lL = full || leaf_at(fx - ex, fy - ey, fz - ez);
    const bool lR = full || leaf_at(fx, fy, fz);
    if (!lL && !lR) return;
    int fb = 0;
    Cons<D> F;
    int side = 0;  // +1: leaf on the low side, INTERNAL high; -1: the reverse
    if (!full && fine_ok && lL != lR) {
      const int ox = x0 + (lL ? fx : fx - ex), oy = y0 + (lL ? fy : fy - ey);
      const int oz = z0 + (lL ? fz : fz - ez);
      if (status_at(ox, oy, oz) == ST_INTERNAL) side = lL ? 1 : -1;
    }
    if (side) {
      const int c[3] = {x0 + (side > 0 ? fx - ex : fx), y0 + (side > 0 ? fy - ey : fy),
                        z0 + (side > 0 ? fz - ez : fz)};
      F = fine_face_average<D, AX, LIM>(a.eval, comp, g, l, c, side, gamma, gm1, &fb, rgm1);
    } else {
      // stencil along AX in halo-box coordinates: cells fx-2 .. fx+1
      const int ix = fx + 2, iy = fy + 2, iz = D == 3 ? fz + 2 : 0;
      const Prim<D> wm1 = P(ix - 2 * ex, iy - 2 * ey, iz - 2 * ez);
      const Prim<D> w0 = P(ix - ex, iy - ey, iz - ez);
      const Prim<D> wp1 = P(ix, iy, iz);
      const Prim<D> wp2 = P(ix + ex, iy + ey, iz + ez);
      Prim<D> lft, rgt;
      if (muscl_recon<D, LIM>(wm1, w0, wp1, wp2, lft, rgt)) {
        fb = 1;
        F = num_flux<D, AX, LIM>(cons_at(x0 + fx - ex, y0 + fy - ey, z0 + fz - ez), w0,
                                 cons_at(x0 + fx, y0 + fy, z0 + fz), wp1, gamma);
      } else {
        F = recon_flux_fast<D, AX, LIM>(lft, rgt, gamma, gm1, rgm1);
      }
    }
    fl[slot] = F.rho;
#pragma unroll
    for (int d = 0; d < D; ++d) fl[(1 + d) * K::NF + slot] = F.m[d];
    fl[(NC - 1) * K::NF + slot] = F.E;
    ffb[slot] = (uint8_t)fb;
  };
  for (int f = tid; f < K::NF; f += K::NT) {
    if (f < K::NXF) {
      const int fx = f % (TX + 1), fy = (f / (TX + 1)) % TY, fz = D == 3 ? f / ((TX + 1) * TY) : 0;
      do_face(std::integral_constant<int, 0>(), fx, fy, fz, f);
    } else if (f < K::NXF + K::NYF) {
      const int h = f - K::NXF;
      const int fx = h % TX, fy = (h / TX) % (TY + 1), fz = D == 3 ? h / (TX * (TY + 1)) : 0;
      do_face(std::integral_constant<int, 1>(), fx, fy, fz, f);
    } else if constexpr (D == 3) {
      const int h = f - K::NXF - K::NYF;
      const int fx = h % TX, fy = (h / TX) % TY, fz = h / (TX * TY);
      do_face(std::integral_constant<int, 2>(), fx, fy, fz, f);
    }
  }
  __syncthreads();
  if (is_leaf) {
    const int c[3] = {cx, cy, cz};
    double rhs[NC];
#pragma unroll
    for (int m = 0; m < NC; ++m) rhs[m] = 0.0;
#pragma unroll
    for (int ax = 0; ax < D; ++ax) {
#pragma unroll
      for (int dir = -1; dir <= 1; dir += 2) {
        // neighbour across the face, same level, bc-mapped (face_flux_at, mr_solver.cpp:99-103)
        int p[3] = {c[0], c[1], c[2]};
        p[ax] += dir;
        bool flp;
        p[ax] = mr_map(p[ax], n, g.bc[2 * ax], g.bc[2 * ax + 1], flp);
        const uint8_t nst = (uint8_t)((nbst >> (2 * (ax * 2 + (dir > 0)))) & 3u);
        const bool internal = nst == ST_INTERNAL;
        double F[NC];
        {
          // the face array holds the same-level flux, or at an interface whose
          // finer side steps now, the fine sub-face average (face phase)
          int fi;
          if (ax == 0) fi = (tz * TY + ty) * (TX + 1) + tx + (dir > 0);
          else if (ax == 1) fi = K::NXF + (tz * (TY + 1) + ty + (dir > 0)) * TX + tx;
          else fi = K::NXF + K::NYF + ((tz + (dir > 0)) * TY + ty) * TX + tx;
#pragma unroll
          for (int m = 0; m < NC; ++m) F[m] = fl[m * K::NF + fi];
          nfb += ffb[fi];
          if (a.reg_stage && !(internal && l + 1 <= a.hi)) {
            if (internal) {
              // finer neighbour advancing later: provisional flux, coarse register
              const int R = reg_index(a.regbase, a.regmask, own, ax * 2 + (dir > 0));
              if (R >= 0) {
#pragma unroll
                for (int m = 0; m < NC; ++m) a.regc[(long)R * NC + m] = F[m] * a.step_dt;
                a.regfc[R] = 1;
              } else {
                atomicExch(a.regerr, 1);
              }
            } else if (nst == ST_ABSENT && l >= 1 && l - 1 < a.lo) {
              const int pn = n >> 1;
              const long pc = g.cell_off[l - 1] + mr_idx(g, D, pn, p[0] >> 1, p[1] >> 1, p[2] >> 1);
              // (a coarse cell of another rank gets this share from its owner)
              if (a.vmark[pc] && row_owned(g, l - 1, p[D - 1] >> 1)) {
                // face into an already-advanced coarser cell: fine register share
                const int R = reg_index(a.regbase, a.regmask, pc, ax * 2 + (dir > 0 ? 0 : 1));
                if (R >= 0) {
                  // sub-face slot in ascending pack_key order of the fine cells
                  int t = 0;
#pragma unroll
                  for (int b = 0; b < D; ++b)
                    if (b != ax) t = 2 * t + (c[b] & 1);
                  const double w = a.step_dt * a.share;
                  double* dst = a.regf + (((long)R * 2 + a.sub) * (D == 3 ? 4 : 2) + t) * NC;
#pragma unroll
                  for (int m = 0; m < NC; ++m) dst[m] = F[m] * w;
                  a.regff[R] = 1;
                } else {
                  atomicExch(a.regerr, 1);
                }
              }
            }
          }
        }
        if (dir < 0) {
#pragma unroll
          for (int m = 0; m < NC; ++m) rhs[m] = rhs[m] + F[m] * inv_dx;
        } else {
#pragma unroll
          for (int m = 0; m < NC; ++m) rhs[m] = rhs[m] - F[m] * inv_dx;
        }
      }
    }
    Cons<D> q;
    double o[NC];
#pragma unroll
    for (int m = 0; m < NC; ++m) {
      o[m] = base0[m] + rhs[m] * sdt;
      a.out[m * comp + own] = o[m];
    }
    if (a.post_check) {  // positivity of the completed step (mr_solver.cpp:290-297)
      q.rho = o[0];
#pragma unroll
      for (int d = 0; d < D; ++d) q.m[d] = o[1 + d];
      q.E = o[NC - 1];
      if (!cell_ok(q, primitives(q, gm1))) bad |= 2;
    }
  } else if (is_hleaf) {
    const int c[3] = {cx, cy, cz};
#pragma unroll
    for (int ax = 0; ax < D; ++ax) {
#pragma unroll
      for (int dir = -1; dir <= 1; dir += 2) {
        int p[3] = {c[0], c[1], c[2]};
        p[ax] += dir;
        bool flp;
        p[ax] = mr_map(p[ax], n, g.bc[2 * ax], g.bc[2 * ax + 1], flp);
        if (a.st[off + mr_idx(g, D, n, p[0], p[1], p[2])] != ST_ABSENT || l < 1 || l - 1 >= a.lo)
          continue;
        const int pn = n >> 1;
        const long pc = g.cell_off[l - 1] + mr_idx(g, D, pn, p[0] >> 1, p[1] >> 1, p[2] >> 1);
        if (!a.vmark[pc] || !row_owned(g, l - 1, p[D - 1] >> 1)) continue;
        int fi;
        if (ax == 0) fi = (tz * TY + ty) * (TX + 1) + tx + (dir > 0);
        else if (ax == 1) fi = K::NXF + (tz * (TY + 1) + ty + (dir > 0)) * TX + tx;
        else fi = K::NXF + K::NYF + ((tz + (dir > 0)) * TY + ty) * TX + tx;
        const int R = reg_index(a.regbase, a.regmask, pc, ax * 2 + (dir > 0 ? 0 : 1));
        if (R >= 0) {
          int t = 0;
#pragma unroll
          for (int b = 0; b < D; ++b)
            if (b != ax) t = 2 * t + (c[b] & 1);
          const double w = a.step_dt * a.share;
          double* dst = a.regf + (((long)R * 2 + a.sub) * (D == 3 ? 4 : 2) + t) * NC;
#pragma unroll
          for (int m = 0; m < NC; ++m) dst[m] = fl[m * K::NF + fi] * w;
          a.regff[R] = 1;
        } else {
          atomicExch(a.regerr, 1);
        }
      }
    }
  }
  __syncthreads();  // the next tile reuses the shared-memory staging
  }
  flush_wave();
  if (bad) atomicOr(&s_bad, bad);
  if (nfb) atomicAdd(&s_fb, nfb);
  __syncthreads();
  if (tid == 0) {
    if (s_bad) {
      // pass-1 failures stop every later launch; a post-step failure only
      // stops the commit, so a pass-1 failure of a later level of the same
      // stage (which the reference reports first) is still detected
      atomicExch(a.err + ((s_bad & 1) ? 0 : 2), 1);
      if (a.post_stops) atomicExch(a.err, 1);
      atomicMin(a.err + 1, step3 + ((s_bad & 1) ? a.stage - 1 : 2));
      atomicCAS(a.err + 3, 0, ((a.lo << 8) | a.hi) + 1);
    }
    if (s_fb) atomicAdd(a.fb, (unsigned long long)s_fb);
  }
}

// Register faces of the leaves of level l: faces whose same-level (bc-mapped)
// neighbour is INTERNAL. Each gets a slot for the coarse provisional flux and
// the 2 x 2^(d-1) fine contributions (registers_, mr_solver.cpp:17-20).
template <int D>
__global__ void mr_reg_build_level(const uint8_t* st, MRLevels g, int l, int* regbase,
                                   uint8_t* regmask, int* count) {
  AF_PDL_ENTRY();
  const int n = 1 << l;
  const long cells = mr_cells(D, l), off = g.cell_off[l];
  for (long c = blockIdx.x * (long)blockDim.x + threadIdx.x; c < cells;
       c += (long)gridDim.x * blockDim.x) {
    if (!row_owned(g, l, mr_row(g, D, l, c))) continue;  // registers live with their owner
    unsigned mask = 0;
    if (st[off + c] == ST_LEAF) {
      int idx[3];
      mr_ijk(g, D, l, c, idx[0], idx[1], idx[2]);
      for (int ax = 0; ax < D; ++ax)
        for (int side = 0; side < 2; ++side) {
          int p[3] = {idx[0], idx[1], idx[2]};
          p[ax] += side ? 1 : -1;
          bool fl;
          p[ax] = mr_map(p[ax], n, g.bc[2 * ax], g.bc[2 * ax + 1], fl);
          if (st[off + mr_idx(g, D, n, p[0], p[1], p[2])] == ST_INTERNAL) mask |= 1u << (ax * 2 + side);
        }
    }
    regmask[off + c] = (uint8_t)mask;
    if (mask) regbase[off + c] = atomicAdd(count, __popc(mask));
  }
}

// apply_registers (mr_solver.cpp:210-230) for the leaves of level l: each
// cell applies its faces in ascending (axis, side) order; the fine sum runs
// substep 1 then 2, sub-faces in ascending key order (the reference's visit
// order). Missing sides raise RegisterMismatch (min face key recorded).
template <int D>
__global__ void mr_reg_apply_level(double* V, const uint8_t* st, MRLevels g, int l,
                                   const int* regbase, const uint8_t* regmask, const double* regc,
                                   const double* regf, uint8_t* regfc, uint8_t* regff,
                                   double inv_sign_dx, unsigned long long* bad_key, int* err) {
  AF_PDL_ENTRY();
  constexpr int NC = D + 2;
  if (failed_before(err)) return;
  const int n = 1 << l;
  const long cells = mr_cells(D, l), off = g.cell_off[l], comp = g.total_cells;
  const int nsub = D == 3 ? 4 : 2;
  for (long c = blockIdx.x * (long)blockDim.x + threadIdx.x; c < cells;
       c += (long)gridDim.x * blockDim.x) {
    if (!row_owned(g, l, mr_row(g, D, l, c))) continue;
    const unsigned mask = regmask[off + c];
    if (!mask) continue;
    int idx[3];
      mr_ijk(g, D, l, c, idx[0], idx[1], idx[2]);
    const unsigned long long key = ((unsigned long long)l << 45) |
                                   ((unsigned long long)idx[0] << 30) |
                                   ((unsigned long long)idx[1] << 15) | (unsigned long long)idx[2];
    double q[NC];
#pragma unroll
    for (int m = 0; m < NC; ++m) q[m] = V[m * comp + off + c];
    int R = regbase[off + c];
    bool ok = true;
    for (int bit = 0; bit < 2 * D; ++bit) {
      if (!((mask >> bit) & 1u)) continue;
      const bool hc = regfc[R], hf = regff[R];
      if (!hc && !hf) {  // never touched this cycle step: no register entry
        ++R;
        continue;
      }
      if (!hc || !hf) {
        atomicMin(bad_key, (key << 3) | bit);
        atomicExch(err, 1);  // RegisterMismatch: stop every later launch
        ok = false;
        break;
      }
      const double sgn = (bit & 1) ? 1.0 : -1.0;
      const double s = sgn * inv_sign_dx;  // == sign / dx (dx a power of two)
#pragma unroll
      for (int m = 0; m < NC; ++m) {
        double f = 0.0;
        for (int sub = 0; sub < 2; ++sub)
          for (int t = 0; t < nsub; ++t) f = f + regf[(((long)R * 2 + sub) * nsub + t) * NC + m];
        q[m] = q[m] + (regc[(long)R * NC + m] - f) * s;
      }
      regfc[R] = 0;
      regff[R] = 0;
      ++R;
    }
    if (ok) {
#pragma unroll
      for (int m = 0; m < NC; ++m) V[m * comp + off + c] = q[m];
    }
  }
}

// Does the tile whose slab-axis rows start at r0 hold a row of this rank's
// region (owned rows + halo)?
template <int D>
__device__ __forceinline__ bool tile_in_region(const MRLevels& g, int l, int r0) {
  if (!g.dist) return true;
  constexpr int TR = D == 3 ? kTileZ3 : kTileY2;
  const int n = 1 << l;
  for (int r = r0; r < r0 + TR && r < n; ++r)
    if (row_in_region(g, l, r)) return true;
  return false;
}

// Work-tile flags over every level at once (one warp per tile): bit 0 the
// tile holds a leaf, bit 1 it holds a cell whose parent exists (every node's
// parent exists, so these tiles cover the tree and everything a split can
// create). Leaves per level are counted on the way.
template <int D>
__global__ void mr_tile_flags_all(const uint8_t* st, MRLevels g, uint8_t* tflag, int* tleaf,
                                  int* counts, unsigned long long* leaves_per_level) {
  AF_PDL_ENTRY();
  // the list counts and leaves per level mr_tile_lists_all accumulates
  if (blockIdx.x == 0 && threadIdx.x < 85) counts[threadIdx.x] = 0;
  if (blockIdx.x == 0 && threadIdx.x < 17) leaves_per_level[threadIdx.x] = 0;
  constexpr int TX = D == 3 ? kTileX3 : kTileX2, TY = D == 3 ? kTileY3 : kTileY2;
  constexpr int TZ = D == 3 ? kTileZ3 : 1;
  const long total = g.tile_off[g.L + 1];
  const int lane = threadIdx.x & 31;
  for (long tg = blockIdx.x * (long)(blockDim.x / 32) + threadIdx.x / 32; tg < total;
       tg += (long)gridDim.x * (blockDim.x / 32)) {
    int l = 0;
    while (tg >= g.tile_off[l + 1]) ++l;
    const long t = tg - g.tile_off[l];
    const int n = 1 << l;
    const int sx = ilog2i(g.ntx[l]), sy = ilog2i(g.nty[l]);  // powers of two
    const int x0 = (int)(t & (g.ntx[l] - 1)) * TX, y0 = (int)((t >> sx) & (g.nty[l] - 1)) * TY;
    const int z0 = D == 3 ? (int)(t >> (sx + sy)) * TZ : 0;
    unsigned nleaf = 0;
    bool pex = false, rleaf = false, notleaf = false, absent = false;
    if (!tile_in_region<D>(g, l, D == 3 ? z0 : y0)) {
      if (lane == 0) {
        tflag[tg] = 0;
        tleaf[tg] = 0;
      }
      continue;
    }
    for (int c = lane; c < TX * TY * TZ; c += 32) {
      const int x = x0 + c % TX, y = y0 + (c / TX) % TY, z = z0 + (D == 3 ? c / (TX * TY) : 0);
      if (x >= n || y >= n || (D == 3 && z >= n)) {
        notleaf = true;
        continue;
      }
      const uint8_t s = st[g.cell_off[l] + mr_idx(g, D, n, x, y, z)];
      const bool lf = s == ST_LEAF;
      notleaf = notleaf || !lf;
      absent = absent || s == ST_ABSENT;
      nleaf += lf && row_counted(g, l, D == 3 ? z : y);
      rleaf = rleaf || (lf && row_in_region(g, l, D == 3 ? z : y));
      pex = pex || l == 0 ||
            st[g.cell_off[l - 1] + mr_idx(g, D, n >> 1, x >> 1, y >> 1, z >> 1)] != ST_ABSENT;
    }
    for (int o = 16; o > 0; o >>= 1) nleaf += __shfl_xor_sync(0xffffffffu, nleaf, o);
    pex = __any_sync(0xffffffffu, pex);
    rleaf = __any_sync(0xffffffffu, rleaf);
    absent = __any_sync(0xffffffffu, absent);
    // bit 2, a full tile: every cell a leaf and every face neighbour of the
    // tile (bc-mapped, same level) a leaf too (one rank only)
    bool full = !g.dist && !__any_sync(0xffffffffu, notleaf);
    bool near = full;  // bit 4: every cell a leaf, no face neighbour INTERNAL (2D)
    if (full) {
      constexpr int RX = TY * TZ, RY = TX * TZ, RZ = D == 3 ? TX * TY : 0;
      bool ok = true, nint = true;
      for (int c = lane; c < 2 * (RX + RY + RZ); c += 32) {
        int q[3], a, side, r;
        if (c < 2 * RX) { a = 0; side = c / RX; r = c % RX; }
        else if (c < 2 * (RX + RY)) { a = 1; side = (c - 2 * RX) / RY; r = (c - 2 * RX) % RY; }
        else { a = 2; side = (c - 2 * (RX + RY)) / RZ; r = (c - 2 * (RX + RY)) % RZ; }
        const int T[3] = {TX, TY, TZ};
        const int b1 = a == 0 ? 1 : 0, b2 = a == 2 ? 1 : 2;
        q[a] = (a == 0 ? x0 : (a == 1 ? y0 : z0)) + (side ? T[a] : -1);
        q[b1] = (b1 == 0 ? x0 : y0) + r % T[b1];
        q[b2] = D == 3 ? ((b2 == 1 ? y0 : z0) + r / T[b1]) : 0;
        bool f;
        for (int d = 0; d < D; ++d) q[d] = mr_map(q[d], n, g.bc[2 * d], g.bc[2 * d + 1], f);
        const uint8_t s = st[g.cell_off[l] + mr_idx(g, D, n, q[0], q[1], q[2])];
        ok = ok && s == ST_LEAF;
        nint = nint && s != ST_INTERNAL;
      }
      full = __all_sync(0xffffffffu, ok);
      near = D == 2 && __all_sync(0xffffffffu, nint);
    }
    if (lane == 0) {
      // bit 0: the tile holds a leaf this rank steps, or (with ranks) a
      // halo leaf whose register shares it computes
      tflag[tg] = ((nleaf || (g.dist && rleaf)) ? 1 : 0) | (pex ? 2 : 0) | (full ? 4 : 0) |
                  (absent ? 8 : 0) | (near ? 16 : 0);
      tleaf[tg] = (int)nleaf;
    }
  }
}

// Per-level tile lists: `leaf` = tiles holding a leaf (the stage kernels'
// work), `band` = tiles within one tile of a flag-2 tile (periodic axes wrap):
// every cell the reference could read as a node value or a prediction lies
// within the stencil reach (<= 3 cells) of a node, so this band is where
// projections, predictions, details and merges are evaluated.
template <int D>
__global__ void mr_tile_lists_all(const uint8_t* tflag, const int* tleaf, MRLevels g, int* band,
                                  int* leaf, int* pband, int* lpart, int* lfull, int* counts,
                                  unsigned long long* leaves_per_level) {
  AF_PDL_ENTRY();
  const long total = g.tile_off[g.L + 1];
  for (long tg = blockIdx.x * (long)blockDim.x + threadIdx.x; tg < total;
       tg += (long)gridDim.x * blockDim.x) {
    int l = 0;
    while (tg >= g.tile_off[l + 1]) ++l;
    const long t = tg - g.tile_off[l];
    const int nt[3] = {g.ntx[l], g.nty[l], D == 3 ? g.ntz[l] : 1};
    const int sx = ilog2i(nt[0]), sy = ilog2i(nt[1]);  // powers of two
    const int tc[3] = {(int)(t & (nt[0] - 1)), (int)((t >> sx) & (nt[1] - 1)),
                       D == 3 ? (int)(t >> (sx + sy)) : 0};
    bool in_band = false;
    const int rz = D == 3 ? 1 : 0;
    for (int dz = -rz; dz <= rz && !in_band; ++dz)
      for (int dy = -1; dy <= 1 && !in_band; ++dy)
        for (int dx = -1; dx <= 1 && !in_band; ++dx) {
          int q[3] = {tc[0] + dx, tc[1] + dy, tc[2] + dz};
          bool ok = true;
          for (int a = 0; a < D; ++a) {
            if (q[a] >= 0 && q[a] < nt[a]) continue;
            if (g.bc[2 * a] == AF_BC_PERIODIC)
              q[a] = (q[a] + nt[a]) % nt[a];
            else
              ok = false;
          }
          if (ok && (tflag[g.tile_off[l] + ((long)q[2] * nt[1] + q[1]) * nt[0] + q[0]] & 2))
            in_band = true;
        }
    if (in_band && !tile_in_region<D>(g, l, tc[D - 1] * (D == 3 ? kTileZ3 : kTileY2)))
      in_band = false;
    // list appends aggregated over the lanes of a warp on the same level (one
    // atomic per group: at L=13 a per-tile atomic on one counter serialises)
    const unsigned grp = __match_any_sync(__activemask(), l);
    const int lane = threadIdx.x & 31, leader = __ffs(grp) - 1;
    const unsigned below = (1u << lane) - 1u;
    const bool in_leaf = (tflag[tg] & 1) != 0;
    const unsigned bb = __ballot_sync(grp, in_band) & grp;
    const unsigned lb = __ballot_sync(grp, in_leaf) & grp;
    const bool in_pband = in_band && (tflag[tg] & 8) != 0;
    const unsigned pb = __ballot_sync(grp, in_pband) & grp;
    // leaf tiles split into full or near-full (bits 2 / 4: mr_stage_full2d)
    // and the rest
    const bool in_full = in_leaf && (tflag[tg] & (4 | 16)) != 0, in_part = in_leaf && !in_full;
    const unsigned fb = __ballot_sync(grp, in_full) & grp;
    const unsigned qb = __ballot_sync(grp, in_part) & grp;
    const unsigned nl = __reduce_add_sync(grp, (unsigned)tleaf[tg]);
    int bbase = 0, lbase = 0, pbase = 0, fbase = 0, qbase = 0;
    if (lane == leader) {
      if (bb) bbase = atomicAdd(counts + l, __popc(bb));
      if (lb) lbase = atomicAdd(counts + 17 + l, __popc(lb));
      if (pb) pbase = atomicAdd(counts + 34 + l, __popc(pb));
      if (qb) qbase = atomicAdd(counts + 51 + l, __popc(qb));
      if (fb) fbase = atomicAdd(counts + 68 + l, __popc(fb));
      if (nl) atomicAdd(leaves_per_level + l, (unsigned long long)nl);
    }
    bbase = __shfl_sync(grp, bbase, leader);
    lbase = __shfl_sync(grp, lbase, leader);
    pbase = __shfl_sync(grp, pbase, leader);
    qbase = __shfl_sync(grp, qbase, leader);
    fbase = __shfl_sync(grp, fbase, leader);
    if (in_band) band[g.tile_off[l] + bbase + __popc(bb & below)] = (int)t;
    if (in_leaf) leaf[g.tile_off[l] + lbase + __popc(lb & below)] = (int)t;
    if (in_pband) pband[g.tile_off[l] + pbase + __popc(pb & below)] = (int)t;
    if (in_part) lpart[g.tile_off[l] + qbase + __popc(qb & below)] = (int)t;
    if (in_full) lfull[g.tile_off[l] + fbase + __popc(fb & below)] = (int)t;
  }
}

// Copies the leaf values of the listed tiles of level l from src to dst
// (q_old snapshot, stage commit). `guard`: skip when a pass-1 or post-step
// failure is pending (the failing stage never commits: the reference throws
// before pass 2 completes); `promote` turns a post-step failure into a stop.
template <int D>
__global__ void mr_copy_leaves_tiles(const double* src, double* dst, const uint8_t* st,
                                     MRLevels g, int l, const int* guard, int promote,
                                     const int* tiles, int ntiles) {
  AF_PDL_ENTRY();
  if (guard) {
    __shared__ int s;
    if (threadIdx.x == 0) s = guard[0] | guard[2];
    __syncthreads();
    // promote bit 1, restore mode (after a buffer swap): only when a failure
    // is pending, exchange the leaf values of src and dst, putting the last
    // committed values back into dst and the failed stage's output into src
    // (where the commit-copy path leaves it for the error report)
    const bool restore = (promote & 2) != 0;
    if (s) {
      if ((promote & 1) && blockIdx.x == 0 && threadIdx.x == 0) atomicExch((int*)guard, 1);
      if (!restore) return;
    } else if (restore) {
      return;
    }
    if (restore) {
      double* s2 = const_cast<double*>(src);
      const long comp = g.total_cells;
      level_cells<D>(g, l, tiles, ntiles, [&](const int lv, long c) {
        const long off = g.cell_off[lv];
        if (st[off + c] != ST_LEAF || !row_owned(g, lv, mr_row(g, D, lv, c))) return;
#pragma unroll
        for (int m = 0; m < D + 2; ++m) {
          const double t = dst[m * comp + off + c];
          dst[m * comp + off + c] = s2[m * comp + off + c];
          s2[m * comp + off + c] = t;
        }
      });
      return;
    }
  }
  const long comp = g.total_cells;
  level_cells<D>(g, l, tiles, ntiles, [&](const int lv, long c) {
    const long off = g.cell_off[lv];
    if (st[off + c] != ST_LEAF || !row_owned(g, lv, mr_row(g, D, lv, c))) return;
#pragma unroll
    for (int m = 0; m < D + 2; ++m) dst[m * comp + off + c] = src[m * comp + off + c];
  });
}

// Copies the values of the ABSENT cells of the listed tiles of level l from
// src to dst: after a buffer swap on the finest level's substeps (MRLT), the
// virtual and predicted cells the next stage's stencils read come back from
// the buffer that holds them.
template <int D>
__global__ void mr_copy_absent_tiles(const double* src, double* dst, const uint8_t* st,
                                     MRLevels g, int l, const int* tiles, int ntiles) {
  AF_PDL_ENTRY();
  const long comp = g.total_cells;
  level_cells<D>(g, l, tiles, ntiles, [&](const int lv, long c) {
    const long off = g.cell_off[lv];
    if (st[off + c] != ST_ABSENT) return;
#pragma unroll
    for (int m = 0; m < D + 2; ++m) dst[m * comp + off + c] = src[m * comp + off + c];
  });
}

// Tiles of level l holding at least one leaf (order irrelevant: every tile
// writes only its own leaves).
template <int D, int TX, int TY, int TZ>
__global__ void mr_tile_list_kernel(const uint8_t* st, MRLevels g, int l, int* tiles,
                                    int* count) {
  AF_PDL_ENTRY();
  const int n = 1 << l;
  const int ntx = (n + TX - 1) / TX, nty = (n + TY - 1) / TY;
  const int ntz = D == 3 ? (n + TZ - 1) / TZ : 1;
  const long ntiles = (long)ntx * nty * ntz;
  const long off = g.cell_off[l];
  for (long t = blockIdx.x * (long)(blockDim.x / 32) + threadIdx.x / 32; t < ntiles;
       t += (long)gridDim.x * (blockDim.x / 32)) {
    const int sx = ilog2i(ntx), sy = ilog2i(nty);  // powers of two
    const int x0 = (int)(t & (ntx - 1)) * TX, y0 = (int)((t >> sx) & (nty - 1)) * TY;
    const int z0 = D == 3 ? (int)(t >> (sx + sy)) * TZ : 0;
    bool any = false;
    for (int c = threadIdx.x & 31; c < TX * TY * TZ; c += 32) {
      const int x = x0 + c % TX, y = y0 + (c / TX) % TY, z = z0 + (D == 3 ? c / (TX * TY) : 0);
      if (x < n && y < n && (D == 2 || z < n) && st[off + mr_idx(g, D, n, x, y, z)] == ST_LEAF)
        any = true;
    }
    any = __any_sync(0xffffffffu, any);
    if (any && (threadIdx.x & 31) == 0) tiles[atomicAdd(count, 1)] = (int)t;
  }
}

}  // namespace af
