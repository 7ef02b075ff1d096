// af_amr_kernels.cuh — device side of the AMR patch path (sm_100a).
//
// Replaces the per-patch loops of PatchHierarchy (amr.hpp:123-242,
// amr_hierarchy.cpp) and flag_cells (amr_cluster.cpp:52-77). The reference
// keeps every patch as its own block with two ghost layers; here a level is
// ONE dense field over its 2^(base+l)-per-axis index space plus a patch-id
// map, which holds the same information:
//   pid[p]   patch index of cell p, -1 outside the level's domain
//   U[p]     the patch interiors (current values)
//   G[p]     the level as of its last sync_ghosts: a copy of U inside the
//            domain, the conservative coarse interpolation on the ring of
//            cells within two cells of it (every ghost some patch holds)
//   Uold/Gold  the same pair at the level's previous step (Patch::data_old)
// A patch P reads position q of its own block as U[q] where pid[q] == P and as
// the ghost G[map(q)] (physical boundaries mapped as map_point does, reflected
// momenta flipped) anywhere else, which reproduces stale ghosts between syncs
// bit for bit. Every ghost of a level comes from one sync, so during
// update_level (always directly after a sync) the level is one field, each
// face flux is computed once, and patches matter only for how often the
// reference counts a fallback (once per patch that evaluates the face or the
// predictor cell).
#pragma once

#include <cstdint>

#include "af_hancock.cuh"

namespace af {

template <int D>
struct ALv {  // one level
  int n;      // cells per axis
  long cells; // n^D
  const int* pid;
  const uint8_t* ring;
  double* U;
  double* Uold;
  double* G;
  double* Gold;
  // the level's patches: boxes (6 ints each) and the prefix offsets of four
  // position lists -- interiors, boxes grown by one cell (the predictor's
  // shell), by two (the blocks with their ghosts), and the faces per (box,
  // axis) -- so a launch walks the patches' positions, as the reference does
  const int* boxes;
  const long *off0, *off1, *off2, *offF;
  int nb;
  long tot0, tot1, tot2, totF;
};

struct ABc {
  int bc[6];
};

// err[0]: 0 ok, 1 non-physical cell, 2 no coarse donor, 3 register without a slot
__device__ __forceinline__ bool amr_failed(const int* err) { return *(volatile const int*)err != 0; }

template <int D>
__device__ __forceinline__ long a_idx(int n, const int* p) {
  return D == 3 ? ((long)p[2] * n + p[1]) * n + p[0] : (long)p[1] * n + p[0];
}
template <int D>
__device__ __forceinline__ void a_coords(int n, long c, int* p) {
  p[0] = (int)(c % n);
  const long t = c / n;
  p[1] = (int)(t % n);
  p[2] = D == 3 ? (int)(t / n) : 0;
}
template <int D>
__device__ __forceinline__ bool a_inrange(int n, const int* p) {
  bool ok = p[0] >= 0 && p[0] < n && p[1] >= 0 && p[1] < n;
  if (D == 3) ok = ok && p[2] >= 0 && p[2] < n;
  return ok;
}

// map_point (amr_hierarchy.cpp:82-105): periodic wrap, outflow clamp,
// reflective fold with the momentum flip.
template <int D>
__device__ __forceinline__ void a_map(int n, const ABc& b, int* p, bool* flip) {
#pragma unroll
  for (int a = 0; a < D; ++a) {
    flip[a] = false;
    int c = p[a];
    if (c >= 0 && c < n) continue;
    if (b.bc[2 * a] == AF_BC_PERIODIC) {
      c = ((c % n) + n) % n;
    } else {
      const int kind = c < 0 ? b.bc[2 * a] : b.bc[2 * a + 1];
      if (kind == AF_BC_OUTFLOW) {
        c = min(max(c, 0), n - 1);
      } else if (kind == AF_BC_REFLECTIVE) {
        while (c < 0 || c >= n) {
          if (c < 0) c = -1 - c;
          if (c >= n) c = 2 * n - 1 - c;
          flip[a] = !flip[a];
        }
      }
    }
    p[a] = c;
  }
}

// periodic wrap only; false when the point lies beyond a physical boundary
template <int D>
__device__ __forceinline__ bool a_wrap(int n, const ABc& b, int* p) {
#pragma unroll
  for (int a = 0; a < D; ++a) {
    if (p[a] >= 0 && p[a] < n) continue;
    if (b.bc[2 * a] != AF_BC_PERIODIC) return false;
    p[a] = ((p[a] % n) + n) % n;
  }
  return true;
}

// boxes as 6 ints (lo[3], hi[3]); off[i] = positions of the boxes before box i
__device__ __forceinline__ int a_find_box(const long* off, int nb, long t) {
  int lo = 0, hi = nb - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (off[mid] <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}
__device__ __forceinline__ void a_box_cell(const int* bx, long r, int* p) {
  const int ex = bx[3] - bx[0], ey = bx[4] - bx[1];
  p[0] = bx[0] + (int)(r % ex);
  const long t = r / ex;
  p[1] = bx[1] + (int)(t % ey);
  p[2] = bx[2] + (int)(t / ey);
}
// position t of the list of the boxes grown by `grow` cells along the active
// axes (unwrapped: it may lie beyond the level's index range); returns the box
// The threads of a CTA walk consecutive list positions, which lie in the same
// or the next few boxes: thread 0 searches the offsets once, the others step
// forward from its box. Every thread of the CTA must call this (a barrier).
__device__ __forceinline__ int a_find_box_cta(const long* off, int nb, long t, long total) {
  __shared__ int s_first;
  if (threadIdx.x == 0) {
    const long t0 = blockIdx.x * (long)blockDim.x;
    s_first = a_find_box(off, nb, t0 < total ? t0 : total - 1);
  }
  __syncthreads();
  int bi = s_first;
  if (t < total)
    while (bi + 1 < nb && off[bi + 1] <= t) ++bi;
  return bi;
}
// a_list_pos with the box already known
template <int D>
__device__ __forceinline__ void a_box_pos(const int* boxes, const long* off, int bi, int grow,
                                          long t, int* p) {
  int gb[6];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const int g = a < D ? grow : 0;
    gb[a] = boxes[6 * bi + a] - g;
    gb[3 + a] = boxes[6 * bi + 3 + a] + g;
  }
  a_box_cell(gb, t - off[bi], p);
}
template <int D>
__device__ __forceinline__ int a_list_pos(const int* boxes, const long* off, int nb, int grow,
                                          long t, int* p) {
  const int bi = a_find_box(off, nb, t);
  int gb[6];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const int g = a < D ? grow : 0;
    gb[a] = boxes[6 * bi + a] - g;
    gb[3 + a] = boxes[6 * bi + 3 + a] + g;
  }
  a_box_cell(gb, t - off[bi], p);
  return bi;
}

template <int D>
__device__ __forceinline__ Cons<D> a_load(const double* A, long cells, long o) {
  Cons<D> q;
  q.rho = A[o];
#pragma unroll
  for (int d = 0; d < D; ++d) q.m[d] = A[(1 + d) * cells + o];
  q.E = A[(D + 1) * cells + o];
  return q;
}
template <int D>
__device__ __forceinline__ void a_store(double* A, long cells, long o, const Cons<D>& q) {
  A[o] = q.rho;
#pragma unroll
  for (int d = 0; d < D; ++d) A[(1 + d) * cells + o] = q.m[d];
  A[(D + 1) * cells + o] = q.E;
}
template <int D>
__device__ __forceinline__ Prim<D> a_loadw(const double* W, long cells, long o) {
  Prim<D> w;
  w.rho = W[o];
#pragma unroll
  for (int d = 0; d < D; ++d) w.v[d] = W[(1 + d) * cells + o];
  w.p = W[(D + 1) * cells + o];
  return w;
}

// a ghost of the field A at (possibly out-of-range) position p
template <int D>
__device__ __forceinline__ Cons<D> a_ghost(const double* A, int n, long cells, const ABc& b,
                                           const int* p) {
  int m[3] = {p[0], p[1], D == 3 ? p[2] : 0};
  bool f[3];
  a_map<D>(n, b, m, f);
  Cons<D> q = a_load<D>(A, cells, a_idx<D>(n, m));
#pragma unroll
  for (int d = 0; d < D; ++d)
    if (f[d]) q.m[d] = -q.m[d];
  return q;
}
template <int D>
__device__ __forceinline__ Prim<D> a_ghostw(const double* W, int n, long cells, const ABc& b,
                                            const int* p) {
  int m[3] = {p[0], p[1], D == 3 ? p[2] : 0};
  bool f[3];
  a_map<D>(n, b, m, f);
  Prim<D> w = a_loadw<D>(W, cells, a_idx<D>(n, m));
#pragma unroll
  for (int d = 0; d < D; ++d)
    if (f[d]) w.v[d] = -w.v[d];
  return w;
}

__device__ __forceinline__ double a_minmod2(double a, double b) {  // amr_hierarchy.cpp:25-28
  if (a * b <= 0.0) return 0.0;
  return fabs(a) < fabs(b) ? a : b;
}

// coarse_interp (amr_hierarchy.cpp:133-178): the value of fine cell p of the
// level above `c`, from the donor patch's view of its block at weight theta.
template <int D>
__device__ __forceinline__ bool a_coarse_interp(const ALv<D>& c, const ABc& b, const int* p,
                                                double theta, double gm1, Cons<D>& out) {
  int cc[3] = {p[0] >> 1, p[1] >> 1, D == 3 ? p[2] >> 1 : 0};
  const int donor = c.pid[a_idx<D>(c.n, cc)];
  if (donor < 0) return false;
  auto value = [&](const int* r) {
    Cons<D> now, old;
    if (a_inrange<D>(c.n, r) && c.pid[a_idx<D>(c.n, r)] == donor) {
      const long o = a_idx<D>(c.n, r);
      now = a_load<D>(c.U, c.cells, o);
      if (theta >= 1.0) return now;
      old = a_load<D>(c.Uold, c.cells, o);
    } else {
      now = a_ghost<D>(c.G, c.n, c.cells, b, r);
      if (theta >= 1.0) return now;
      old = a_ghost<D>(c.Gold, c.n, c.cells, b, r);
    }
    const double w0 = 1.0 - theta;
    Cons<D> v;
    v.rho = old.rho * w0 + now.rho * theta;
#pragma unroll
    for (int d = 0; d < D; ++d) v.m[d] = old.m[d] * w0 + now.m[d] * theta;
    v.E = old.E * w0 + now.E * theta;
    return v;
  };
  const Cons<D> q0 = value(cc);
  out = q0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    int m[3] = {cc[0], cc[1], cc[2]}, pl[3] = {cc[0], cc[1], cc[2]};
    m[a] -= 1;
    pl[a] += 1;
    const Cons<D> qm = value(m), qp = value(pl);
    const double s = (p[a] & 1) ? 0.25 : -0.25;
    out.rho = out.rho + a_minmod2(qp.rho - q0.rho, q0.rho - qm.rho) * s;
#pragma unroll
    for (int d = 0; d < D; ++d)
      out.m[d] = out.m[d] + a_minmod2(qp.m[d] - q0.m[d], q0.m[d] - qm.m[d]) * s;
    out.E = out.E + a_minmod2(qp.E - q0.E, q0.E - qm.E) * s;
  }
  if (!(out.rho > kPosTol) || !physical(primitives(out, gm1))) out = q0;
  return true;
}

// ---------------------------------------------------------------- masks --
template <int D>
__global__ void __launch_bounds__(256) amr_setpid_kernel(const int* boxes, const long* off, int nb,
                                                         long total, int n, int* pid) {
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (t >= total) return;
  const int bi = a_find_box(off, nb, t);
  int p[3];
  a_box_cell(boxes + 6 * bi, t - off[bi], p);
  pid[a_idx<D>(n, p)] = bi;
}

// AoS (5 doubles, x fastest, box after box) <-> the level field
template <int D>
__global__ void __launch_bounds__(256) amr_put_kernel(const int* boxes, const long* off, int nb,
                                                      long total, int n, long cells,
                                                      const double* aos, double* U) {
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (t >= total) return;
  const int bi = a_find_box(off, nb, t);
  int p[3];
  a_box_cell(boxes + 6 * bi, t - off[bi], p);
  const long o = a_idx<D>(n, p);
  U[o] = aos[5 * t];
  U[cells + o] = aos[5 * t + 1];
  U[2 * cells + o] = aos[5 * t + 2];
  if (D == 3) U[3 * cells + o] = aos[5 * t + 3];
  U[(D + 1) * cells + o] = aos[5 * t + 4];
}

// with ghost > 0 the boxes are read as the patches' blocks (box grown by
// `ghost` along the active axes), each position through the patch's view
template <int D>
__global__ void __launch_bounds__(256) amr_get_kernel(const int* boxes, const long* off, int nb,
                                                      long total, ALv<D> lv, ABc b, int ghost,
                                                      int old, int mode, double* aos) {
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (t >= total) return;
  const int bi = a_find_box(off, nb, t);
  int gb[6];
  for (int a = 0; a < 3; ++a) {
    const int g = a < D ? ghost : 0;
    gb[a] = boxes[6 * bi + a] - g;
    gb[3 + a] = boxes[6 * bi + 3 + a] + g;
  }
  int p[3];
  a_box_cell(gb, t - off[bi], p);
  Cons<D> q;
  // mode 0: the patch's view; 1: the synced field everywhere; 2: interiors
  if (mode == 2 || (mode == 0 && a_inrange<D>(lv.n, p) && lv.pid[a_idx<D>(lv.n, p)] == bi))
    q = a_load<D>(old ? lv.Uold : lv.U, lv.cells, a_idx<D>(lv.n, p));
  else
    q = a_ghost<D>(old ? lv.Gold : lv.G, lv.n, lv.cells, b, p);
  aos[5 * t] = q.rho;
  aos[5 * t + 1] = q.m[0];
  aos[5 * t + 2] = q.m[1];
  aos[5 * t + 3] = D == 3 ? q.m[D - 1] : 0.0;
  aos[5 * t + 4] = q.E;
}

// ----------------------------------------------------------- sync_ghosts --
// sync_ghosts (amr_hierarchy.cpp:180-214) of a whole level: G = U inside the
// domain, the coarse interpolation on the ring.
template <int D>
__global__ void __launch_bounds__(256) amr_sync_kernel(ALv<D> lv, ALv<D> co, int has_coarse, ABc b,
                                                       double theta, double gm1, int* err) {
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  const int bi = a_find_box_cta(lv.off2, lv.nb, t, lv.tot2);
  if (t >= lv.tot2 || amr_failed(err)) return;
  int p[3];
  a_box_pos<D>(lv.boxes, lv.off2, bi, 2, t, p);
  const bool inside = a_inrange<D>(lv.n, p);
  if (!inside && !a_wrap<D>(lv.n, b, p)) return;  // beyond a physical boundary: read through a_map
  const long c = a_idx<D>(lv.n, p);
  const int owner = lv.pid[c];
  if (owner >= 0) {  // a domain cell is copied once, by its own patch
    if (owner != bi || !inside) return;
#pragma unroll
    for (int m = 0; m < D + 2; ++m) lv.G[m * lv.cells + c] = lv.U[m * lv.cells + c];
    return;
  }
  if (!has_coarse) return;
  Cons<D> q;
  if (!a_coarse_interp<D>(co, b, p, theta, gm1, q)) {  // MissingBracketingStates
    if (atomicCAS(err, 0, 2) == 0) err[1] = (int)c;
    return;
  }
  a_store<D>(lv.G, lv.cells, c, q);
}

// Patch::data_old = Patch::data for every patch (interiors and ghosts), and
// the way back for the ghosts (update_level's RK2 branch leaves the blocks
// with the ghosts of time t, amr_hierarchy.cpp:508-519)
template <int D>
__global__ void __launch_bounds__(256) amr_save_kernel(ALv<D> lv, ABc b, int restore, const int* err) {
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  const int bi = a_find_box_cta(lv.off2, lv.nb, t, lv.tot2);
  if (t >= lv.tot2 || amr_failed(err)) return;
  int p[3];
  a_box_pos<D>(lv.boxes, lv.off2, bi, 2, t, p);
  const bool inside = a_inrange<D>(lv.n, p);
  if (!inside && !a_wrap<D>(lv.n, b, p)) return;
  const long c = a_idx<D>(lv.n, p);
  const int owner = lv.pid[c];
  if (owner >= 0 && (owner != bi || !inside)) return;  // a domain cell moves once, with its patch
  if (restore) {
#pragma unroll
    for (int m = 0; m < D + 2; ++m) lv.G[m * lv.cells + c] = lv.Gold[m * lv.cells + c];
    return;
  }
  const bool dom = owner >= 0;
#pragma unroll
  for (int m = 0; m < D + 2; ++m) {
    lv.Gold[m * lv.cells + c] = lv.G[m * lv.cells + c];
    if (dom) lv.Uold[m * lv.cells + c] = lv.U[m * lv.cells + c];
  }
}

// remesh (amr_hierarchy.cpp:311-320): cells of the new domain keep the old
// patch value where the level held one, else take the coarse interpolation.
template <int D>
__global__ void __launch_bounds__(256) amr_build_kernel(ALv<D> lv, const int* old_pid, int had,
                                                        ALv<D> co, ABc b, double gm1, int* err) {
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (t >= lv.tot0 || amr_failed(err)) return;
  int p[3];
  a_list_pos<D>(lv.boxes, lv.off0, lv.nb, 0, t, p);
  const long c = a_idx<D>(lv.n, p);
  if (had && old_pid[c] >= 0) return;
  Cons<D> q;
  if (!a_coarse_interp<D>(co, b, p, 1.0, gm1, q)) {
    if (atomicCAS(err, 0, 2) == 0) err[1] = (int)c;
    return;
  }
  a_store<D>(lv.U, lv.cells, c, q);
}

// ------------------------------------------------------------ flag_cells --
// flag_cells (amr_cluster.cpp:52-77) on the synced level (flags cleared before).
template <int D>
__global__ void __launch_bounds__(256) amr_flag_kernel(ALv<D> lv, ABc b, double gm1, double eps_rho,
                                                       double eps_p, uint8_t* flags) {
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (t >= lv.tot0) return;
  int p[3];
  a_list_pos<D>(lv.boxes, lv.off0, lv.nb, 0, t, p);
  const long c = a_idx<D>(lv.n, p);
  uint8_t f = 0;
  {
    const Prim<D> w0 = primitives(a_load<D>(lv.G, lv.cells, c), gm1);
    for (int a = 1; a < (1 << D) && !f; ++a) {
      int q[3] = {p[0] + (a & 1), p[1] + ((a >> 1) & 1), p[2] + ((a >> 2) & 1)};
      const Prim<D> w1 = primitives(a_ghost<D>(lv.G, lv.n, lv.cells, b, q), gm1);
      if (fabs(w1.rho - w0.rho) > eps_rho || fabs(w1.p - w0.p) > eps_p) f = 1;
    }
  }
  flags[c] = f;
}

// IndexMask::dilated (amr_cluster.cpp:28-50) in gather form; `orin` is or-ed in
template <int D>
__global__ void __launch_bounds__(256) amr_dilate_kernel(const uint8_t* in, int n, ABc b, int radius,
                                                         const uint8_t* orin, uint8_t* out) {
  const long cells = D == 3 ? (long)n * n * n : (long)n * n;
  const long c = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (c >= cells) return;
  int p[3];
  a_coords<D>(n, c, p);
  uint8_t r = orin ? orin[c] : 0;
  const int rz = D == 3 ? radius : 0;
  for (int dk = -rz; dk <= rz && !r; ++dk)
    for (int dj = -radius; dj <= radius && !r; ++dj)
      for (int di = -radius; di <= radius; ++di) {
        int q[3] = {p[0] + di, p[1] + dj, p[2] + dk};
        if (!a_wrap<D>(n, b, q)) continue;
        if (in[a_idx<D>(n, q)]) {
          r = 1;
          break;
        }
      }
  out[c] = r;
}

// set_box of each listed box (clipped to the level by the host; the mask
// cleared before), amr_cluster.cpp:20-26
template <int D>
__global__ void __launch_bounds__(256) amr_setbox_kernel(const int* boxes, const long* off, int nb,
                                                         long total, int n, uint8_t* mask) {
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (t >= total) return;
  int p[3];
  a_list_pos<D>(boxes, off, nb, 0, t, p);
  mask[a_idx<D>(n, p)] = 1;
}

// allowed (amr_hierarchy.cpp:259-284): domain cells whose whole 3^d
// neighbourhood (periodic wrap, no constraint past a physical boundary) lies
// in the domain; masked = flags & allowed, any[0] set when one is.
template <int D>
__global__ void __launch_bounds__(256) amr_allowed_kernel(const int* pid, int n, ABc b,
                                                          const uint8_t* flags, uint8_t* allowed,
                                                          uint8_t* masked, int* any) {
  const long cells = D == 3 ? (long)n * n * n : (long)n * n;
  const long c = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (c >= cells) return;
  uint8_t ok = pid[c] >= 0;
  if (ok) {
    int p[3];
    a_coords<D>(n, c, p);
    for (int dk = (D == 3 ? -1 : 0); dk <= (D == 3 ? 1 : 0) && ok; ++dk)
      for (int dj = -1; dj <= 1 && ok; ++dj)
        for (int di = -1; di <= 1; ++di) {
          int q[3] = {p[0] + di, p[1] + dj, p[2] + dk};
          if (!a_wrap<D>(n, b, q)) continue;
          if (pid[a_idx<D>(n, q)] < 0) {
            ok = 0;
            break;
          }
        }
  }
  allowed[c] = ok;
  const uint8_t mk = ok && flags[c];
  masked[c] = mk;
  if (mk) *any = 1;
}

// properly_nested (amr_hierarchy.cpp:344-356)
template <int D>
__global__ void __launch_bounds__(256) amr_nested_kernel(ALv<D> fine, const int* coarse, int* bad) {
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (t >= fine.tot0) return;
  int p[3];
  a_list_pos<D>(fine.boxes, fine.off0, fine.nb, 0, t, p);
  int q[3] = {p[0] >> 1, p[1] >> 1, D == 3 ? p[2] >> 1 : 0};
  if (coarse[a_idx<D>(fine.n >> 1, q)] < 0) *bad = 1;
}

// ------------------------------------------------------------ the update --
struct ARec {                    // one update_level call
  unsigned long long wave;       // max |v_a|+c over the interiors (bits)
  unsigned long long fallbacks;
};

// build_primitives (step.cpp:18-49) of every patch block: W at the blocks'
// positions; the speed maximum over the interiors.
template <int D>
__global__ void __launch_bounds__(256) amr_prims_kernel(ALv<D> lv, ABc b, double* W, double gamma,
                                                        ARec* rec, int* err, int tag) {
  __shared__ double red[8];
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  double wave = 0.0;
  const int bi = a_find_box_cta(lv.off2, lv.nb, t, lv.tot2);
  if (t < lv.tot2 && !amr_failed(err)) {
    int p[3];
    a_box_pos<D>(lv.boxes, lv.off2, bi, 2, t, p);
    const bool inside = a_inrange<D>(lv.n, p);
    if (a_wrap<D>(lv.n, b, p)) {
      const long c = a_idx<D>(lv.n, p);
      const Cons<D> q = a_load<D>(lv.G, lv.cells, c);
      const Prim<D> w = primitives(q, gamma - 1.0);
      if (!cell_ok(q, w) && atomicCAS(err, 0, 1) == 0) err[1] = tag;
      W[c] = w.rho;
#pragma unroll
      for (int d = 0; d < D; ++d) W[(1 + d) * lv.cells + c] = w.v[d];
      W[(D + 1) * lv.cells + c] = w.p;
      if (inside && lv.pid[c] == bi) {
        double s, m;
        wave_speeds(w, gamma, s, m);
        wave = m;
      }
    }
  }
  block_max_atomic<256>(wave, red, &rec->wave);
}

template <int D>
__device__ __forceinline__ long a_face_index(int n, int ax, const int* p) {
  const int d0 = ax == 0 ? n + 1 : n, d1 = ax == 1 ? n + 1 : n;
  return D == 3 ? ((long)p[2] * d1 + p[1]) * d0 + p[0] : (long)p[1] * d0 + p[0];
}

// face t of the level's face list: the patch, the axis and the (unwrapped)
// position of the face's high cell; the face index along the axis is p[ax]
template <int D>
__device__ __forceinline__ int a_face_pos(const ALv<D>& lv, long t, int* p) {
  const int e = a_find_box_cta(lv.offF, lv.nb * D, t, lv.totF);
  if (t >= lv.totF) return 0;
  const int bi = e / D, ax = e - bi * D;
  int fb[6];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    fb[a] = lv.boxes[6 * bi + a];
    fb[3 + a] = lv.boxes[6 * bi + 3 + a] + (a == ax ? 1 : 0);
  }
  a_box_cell(fb, t - lv.offF[e], p);
  return ax;
}

// accumulate_rhs' fluxes (step.cpp:57-89) of every face of every patch, one
// thread per (patch, face), into F (SoA over the level's faces, component
// stride D*per). A face on a seam is evaluated by both patches (the same bits
// twice) and counts its fallback for each, as the reference's patch loop does.
template <int D, int S>
__global__ void __launch_bounds__(256) amr_faces_rk2(ALv<D> lv, ABc b, const double* W, double* F,
                                                     double gamma, ARec* rec, int* err) {
  const int n = lv.n;
  const long per = D == 3 ? (long)(n + 1) * n * n : (long)(n + 1) * n;
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  int p[3];
  const int ax = a_face_pos<D>(lv, t, p);
  if (t >= lv.totF || amr_failed(err)) return;
  const long f = ax * per + a_face_index<D>(n, ax, p);
  int lo[3] = {p[0], p[1], p[2]};
  lo[ax] -= 1;
  const double gm1 = gamma - 1.0, rgm1 = 1.0 / gm1;
  Prim<D> ws[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    int c[3] = {p[0], p[1], p[2]};
    c[ax] += s - 2;
    ws[s] = a_ghostw<D>(W, n, lv.cells, b, c);
  }
  Prim<D> l, rr;
  const bool fb = muscl_recon<D, S>(ws[0], ws[1], ws[2], ws[3], l, rr);
  Cons<D> Fx;
  if (fb) {
    const Cons<D> ql = a_ghost<D>(lv.G, n, lv.cells, b, lo);
    const Cons<D> qr = a_ghost<D>(lv.G, n, lv.cells, b, p);
    Fx = num_flux<D, S>(ql, ws[1], qr, ws[2], ax, gamma);
    atomicAdd(&rec->fallbacks, 1ull);
  } else {
    Fx = recon_flux_fast<D, S>(l, rr, ax, gamma, gm1, rgm1);
  }
  const long cs = D * per;
  F[f] = Fx.rho;
#pragma unroll
  for (int d = 0; d < D; ++d) F[(1 + d) * cs + f] = Fx.m[d];
  F[(D + 1) * cs + f] = Fx.E;
}

// out = base + rhs * sdt over the domain (step.cpp:104-108, 226-232), rhs
// summed per axis as accumulate_rhs does (+F_low*inv_dx, -F_high*inv_dx).
template <int D>
__global__ void __launch_bounds__(256) amr_update_kernel(ALv<D> lv, const double* base,
                                                         const double* F, double inv_dx, double sdt,
                                                         int* err) {
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  const int bi = a_find_box_cta(lv.off0, lv.nb, t, lv.tot0);
  if (t >= lv.tot0 || amr_failed(err)) return;
  const int n = lv.n;
  const long per = D == 3 ? (long)(n + 1) * n * n : (long)(n + 1) * n;
  const long cs = D * per;
  int p[3];
  a_box_pos<D>(lv.boxes, lv.off0, bi, 0, t, p);
  const long c = a_idx<D>(n, p);
  long fl[D], fh[D];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    fl[a] = a * per + a_face_index<D>(n, a, p);
    int h[3] = {p[0], p[1], p[2]};
    h[a] += 1;
    fh[a] = a * per + a_face_index<D>(n, a, h);
  }
#pragma unroll
  for (int m = 0; m < D + 2; ++m) {
    double rhs = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      rhs = rhs + F[m * cs + fl[a]] * inv_dx;
      rhs = rhs - F[m * cs + fh[a]] * inv_dx;
    }
    lv.U[m * lv.cells + c] = base[m * lv.cells + c] + rhs * sdt;
  }
}

// MUSCL-Hancock predictor (step.cpp:160-181) over every patch's interior plus
// its one-cell shell (positions -1..n per axis, DU padded by one cell). A
// position two patches hold is evaluated by both (the same bits) and counts
// its fallbacks for each.
template <int D, int S>
__global__ void __launch_bounds__(256) amr_predict_kernel(ALv<D> lv, ABc b, const double* W,
                                                          double* DU, double half_dt_dx, double gm1,
                                                          ARec* rec, int* err) {
  const int n = lv.n, np = n + 2;
  const long padded = D == 3 ? (long)np * np * np : (long)np * np;
  const long tl = blockIdx.x * (long)blockDim.x + threadIdx.x;
  const int bi = a_find_box_cta(lv.off1, lv.nb, tl, lv.tot1);
  if (tl >= lv.tot1 || amr_failed(err)) return;
  int q[3];
  a_box_pos<D>(lv.boxes, lv.off1, bi, 1, tl, q);
  const long t = D == 3 ? ((long)(q[2] + 1) * np + (q[1] + 1)) * np + (q[0] + 1)
                        : (long)(q[1] + 1) * np + (q[0] + 1);
  const Prim<D> w0 = a_ghostw<D>(W, n, lv.cells, b, q);
  double acc[D + 2];
#pragma unroll
  for (int m = 0; m < D + 2; ++m) acc[m] = 0.0;
  int nfb = 0;
#pragma unroll
  for (int ax = 0; ax < D; ++ax) {
    int lo[3] = {q[0], q[1], q[2]}, hi[3] = {q[0], q[1], q[2]};
    lo[ax] -= 1;
    hi[ax] += 1;
    const Prim<D> wm = a_ghostw<D>(W, n, lv.cells, b, lo);
    const Prim<D> wp = a_ghostw<D>(W, n, lv.cells, b, hi);
    Prim<D> mi, pl;
    if (recon_cell<D, S>(wm, w0, wp, mi, pl)) {
      ++nfb;
      continue;
    }
    const Cons<D> um = conserved(mi, gm1), up = conserved(pl, gm1);
    double fp[D + 2], fm[D + 2];
    phys_flux<D>(up, pl, ax, fp);
    phys_flux<D>(um, mi, ax, fm);
#pragma unroll
    for (int m = 0; m < D + 2; ++m) acc[m] = acc[m] - (fp[m] - fm[m]) * half_dt_dx;
  }
  if (nfb) atomicAdd(&rec->fallbacks, (unsigned long long)nfb);
#pragma unroll
  for (int m = 0; m < D + 2; ++m) DU[m * padded + t] = acc[m];
}

// MUSCL-Hancock corrector fluxes (step.cpp:184-224), one thread per face.
template <int D, int S>
__global__ void __launch_bounds__(256) amr_faces_hancock(ALv<D> lv, ABc b, const double* W,
                                                         const double* DU, double* F, double gamma,
                                                         ARec* rec, int* err) {
  const int n = lv.n, np = n + 2;
  const long padded = D == 3 ? (long)np * np * np : (long)np * np;
  const long per = D == 3 ? (long)(n + 1) * n * n : (long)(n + 1) * n;
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  int cr[3];
  const int ax = a_face_pos<D>(lv, t, cr);
  if (t >= lv.totF || amr_failed(err)) return;
  const long f = ax * per + a_face_index<D>(n, ax, cr);
  int cl[3] = {cr[0], cr[1], cr[2]};
  cl[ax] -= 1;
  const double gm1 = gamma - 1.0;
  Prim<D> w[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    int c[3] = {cr[0], cr[1], cr[2]};
    c[ax] += s - 2;
    w[s] = a_ghostw<D>(W, n, lv.cells, b, c);
  }
  Prim<D> lmi, lpl, rmi, rpl;
  recon_cell<D, S>(w[0], w[1], w[2], lmi, lpl);
  recon_cell<D, S>(w[1], w[2], w[3], rmi, rpl);
  auto du_at = [&](const int* c) {
    const long o = D == 3 ? ((long)(c[2] + 1) * np + (c[1] + 1)) * np + (c[0] + 1)
                          : (long)(c[1] + 1) * np + (c[0] + 1);
    Cons<D> d;
    d.rho = DU[o];
#pragma unroll
    for (int k = 0; k < D; ++k) d.m[k] = DU[(1 + k) * padded + o];
    d.E = DU[(D + 1) * padded + o];
    return d;
  };
  auto add = [](const Cons<D>& x, const Cons<D>& y) {
    Cons<D> z;
    z.rho = x.rho + y.rho;
#pragma unroll
    for (int k = 0; k < D; ++k) z.m[k] = x.m[k] + y.m[k];
    z.E = x.E + y.E;
    return z;
  };
  const Cons<D> dl = du_at(cl), dr = du_at(cr);
  Cons<D> ul = add(conserved(lpl, gm1), dl);
  Cons<D> ur = add(conserved(rmi, gm1), dr);
  int nfb = 0;
  if (!phys_state(ul, gm1)) {
    const Cons<D> ql = a_ghost<D>(lv.G, n, lv.cells, b, cl);
    ul = add(ql, dl);
    if (!phys_state(ul, gm1)) ul = ql;
    ++nfb;
  }
  if (!phys_state(ur, gm1)) {
    const Cons<D> qr = a_ghost<D>(lv.G, n, lv.cells, b, cr);
    ur = add(qr, dr);
    if (!phys_state(ur, gm1)) ur = qr;
    ++nfb;
  }
  if (nfb) atomicAdd(&rec->fallbacks, (unsigned long long)nfb);
  const Cons<D> Fx = num_flux<D, S>(ul, primitives(ul, gm1), ur, primitives(ur, gm1), ax, gamma);
  const long cs = D * per;
  F[f] = Fx.rho;
#pragma unroll
  for (int d = 0; d < D; ++d) F[(1 + d) * cs + f] = Fx.m[d];
  F[(D + 1) * cs + f] = Fx.E;
}

// ------------------------------------------------------- flux registers --
// Registers of the pair (l, l+1) (accumulate_registers / flux_correct,
// amr_hierarchy.cpp:358-462,532-559): one slot per face of an uncovered
// level-l cell whose neighbour across it lies in the level's domain and under
// level l+1. A cell's slots are contiguous, in the order of the reference's
// sorted keys (axis, then low face before high face).
template <int D>
__device__ __forceinline__ uint8_t a_reg_mask(const int* pid, const int* fpid, int n, const ABc& b,
                                              const int* p) {
  auto covered = [&](const int* c) {
    const int f[3] = {2 * c[0], 2 * c[1], D == 3 ? 2 * c[2] : 0};
    return fpid[a_idx<D>(2 * n, f)] >= 0;
  };
  if (pid[a_idx<D>(n, p)] < 0 || covered(p)) return 0;
  uint8_t mask = 0;
#pragma unroll
  for (int a = 0; a < D; ++a)
    for (int side = 0; side < 2; ++side) {
      int v[3] = {p[0], p[1], p[2]};
      v[a] += side ? 1 : -1;
      if (!a_wrap<D>(n, b, v)) continue;
      if (pid[a_idx<D>(n, v)] < 0) continue;
      if (covered(v)) mask |= (uint8_t)(1u << (2 * a + side));
    }
  return mask;
}

template <int D>
__global__ void __launch_bounds__(256) amr_reg_alloc_kernel(ALv<D> lv, const int* fpid, ABc b,
                                                            int* regbase, uint8_t* regmask,
                                                            int* count, long* slot_cell,
                                                            uint8_t* slot_face, int cap, int* err) {
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (t >= lv.tot0) return;
  int p[3];
  a_list_pos<D>(lv.boxes, lv.off0, lv.nb, 0, t, p);
  const long c = a_idx<D>(lv.n, p);
  uint8_t mask = a_reg_mask<D>(lv.pid, fpid, lv.n, b, p);
  int base = -1;
  if (mask) {
    base = atomicAdd(count, __popc(mask));
    if (base + __popc(mask) > cap) {  // cannot happen: cap bounds the fine boxes' surfaces
      atomicCAS(err, 0, 3);
      mask = 0;
      base = -1;
    }
  }
  regmask[c] = mask;
  regbase[c] = base;
  int k = 0;
  for (int bit = 0; bit < 2 * D && mask; ++bit)
    if (mask & (1u << bit)) {
      slot_cell[base + k] = c;
      slot_face[base + k] = (uint8_t)bit;
      ++k;
    }
}

// coarse side: reg.coarse += flux * dt (amr_hierarchy.cpp:455-457)
template <int D>
__global__ void __launch_bounds__(256) amr_reg_coarse_kernel(const long* slot_cell,
                                                             const uint8_t* slot_face, int nslots,
                                                             int n, const double* F, double dt,
                                                             double* Rc, uint8_t* has, int* err) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nslots || amr_failed(err) || slot_face[s] == 0xff) return;
  const long per = D == 3 ? (long)(n + 1) * n * n : (long)(n + 1) * n;
  const long cs = D * per;
  int p[3];
  a_coords<D>(n, slot_cell[s], p);
  const int ax = slot_face[s] >> 1, side = slot_face[s] & 1;
  p[ax] += side;  // the face index along ax
  const long f = ax * per + a_face_index<D>(n, ax, p);
#pragma unroll
  for (int m = 0; m < D + 2; ++m) Rc[(long)m * nslots + s] = Rc[(long)m * nslots + s] + F[m * cs + f] * dt;
  has[s] |= 1;
}

// fine side: reg.fine += flux * (dt * share) over the 2^(d-1) fine faces in
// the reference's loop order (amr_hierarchy.cpp:372-409); nf = fine cells/axis
template <int D>
__global__ void __launch_bounds__(256) amr_reg_fine_kernel(const long* slot_cell,
                                                           const uint8_t* slot_face, int nslots,
                                                           int n, int nf, const double* F,
                                                           double dtshare, double* Rf, uint8_t* has,
                                                           int* err) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nslots || amr_failed(err) || slot_face[s] == 0xff) return;
  const long per = D == 3 ? (long)(nf + 1) * nf * nf : (long)(nf + 1) * nf;
  const long cs = D * per;
  int u[3];
  a_coords<D>(n, slot_cell[s], u);
  const int ax = slot_face[s] >> 1, side = slot_face[s] & 1;
  const int b1 = ax == 0 ? 1 : 0, b2 = ax == 2 ? 1 : 2;
  // fine face index along ax: the covered neighbour's near face
  int fa;
  if (side) {
    fa = 2 * u[ax] + 2;
    if (fa == nf) fa = 0;  // periodic wrap: the fine patch starts at the low edge
  } else {
    fa = 2 * u[ax];
    if (fa == 0) fa = nf;  // the fine patch ends at the high edge
  }
  double acc[D + 2];
#pragma unroll
  for (int m = 0; m < D + 2; ++m) acc[m] = Rf[(long)m * nslots + s];
  for (int c2 = 0; c2 < (D == 3 ? 2 : 1); ++c2)
    for (int c1 = 0; c1 < 2; ++c1) {
      int p[3] = {0, 0, 0};
      p[ax] = fa;
      p[b1] = 2 * u[b1] + c1;
      if (D == 3) p[b2] = 2 * u[b2] + c2;
      const long f = ax * per + a_face_index<D>(nf, ax, p);
#pragma unroll
      for (int m = 0; m < D + 2; ++m) acc[m] = acc[m] + F[m * cs + f] * dtshare;
    }
#pragma unroll
  for (int m = 0; m < D + 2; ++m) Rf[(long)m * nslots + s] = acc[m];
  has[s] |= 2;
}

// flux_correct (amr_hierarchy.cpp:532-559): the thread of a cell's first
// slot applies the cell's faces in sorted-key order
template <int D>
__global__ void __launch_bounds__(256) amr_flux_correct_kernel(ALv<D> lv, const int* regbase,
                                                               const uint8_t* regmask,
                                                               const long* slot_cell,
                                                               const uint8_t* slot_face,
                                                               const double* Rc, const double* Rf,
                                                               const uint8_t* has, int nslots,
                                                               double inv_h, int* err) {
  const int s0 = blockIdx.x * blockDim.x + threadIdx.x;
  if (s0 >= nslots || amr_failed(err) || slot_face[s0] == 0xff) return;
  const long c = slot_cell[s0];
  if (regbase[c] != s0) return;
  const uint8_t mask = regmask[c];
  int s = s0;
  for (int bit = 0; bit < 2 * D; ++bit) {
    if (!(mask & (1u << bit))) continue;
    if (has[s] != 3) {
      if (has[s] != 0 && atomicCAS(err, 0, 3) == 0) err[1] = (int)c;
      ++s;
      continue;
    }
    const double sc = ((bit & 1) ? 1.0 : -1.0) * inv_h;
#pragma unroll
    for (int m = 0; m < D + 2; ++m)
      lv.U[m * lv.cells + c] =
          lv.U[m * lv.cells + c] + (Rc[(long)m * nslots + s] - Rf[(long)m * nslots + s]) * sc;
    ++s;
  }
}

// average_down (amr_hierarchy.cpp:501-530)
template <int D>
__global__ void __launch_bounds__(256) amr_average_down_kernel(ALv<D> co, ALv<D> fi, int* err) {
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (t >= co.tot0 || amr_failed(err)) return;
  int p[3];
  a_list_pos<D>(co.boxes, co.off0, co.nb, 0, t, p);
  const long c = a_idx<D>(co.n, p);
  const int f0[3] = {2 * p[0], 2 * p[1], D == 3 ? 2 * p[2] : 0};
  if (fi.pid[a_idx<D>(fi.n, f0)] < 0) return;
  const double w = D == 3 ? 0.125 : 0.25;
#pragma unroll
  for (int m = 0; m < D + 2; ++m) {
    double sum = 0.0;
    for (int dk = 0; dk < (D == 3 ? 2 : 1); ++dk)
      for (int dj = 0; dj < 2; ++dj)
        for (int di = 0; di < 2; ++di) {
          const int f[3] = {f0[0] + di, f0[1] + dj, f0[2] + dk};
          sum = sum + fi.U[m * fi.cells + a_idx<D>(fi.n, f)];
        }
    co.U[m * co.cells + c] = sum * w;
  }
}

// total_conserved (amr_hierarchy.cpp:561-581): per-level sums over the cells
// the next level does not cover (block tree sums; the order differs from the
// reference's sequential loop, so agreement is to round-off).
template <int D>
__global__ void __launch_bounds__(256) amr_sum_kernel(ALv<D> lv, const int* fpid, double* out) {
  __shared__ double red[8];
  double acc[D + 2];
#pragma unroll
  for (int m = 0; m < D + 2; ++m) acc[m] = 0.0;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < lv.tot0;
       t += (long)gridDim.x * blockDim.x) {
    int p[3];
    a_list_pos<D>(lv.boxes, lv.off0, lv.nb, 0, t, p);
    const long c = a_idx<D>(lv.n, p);
    if (fpid) {
      const int f[3] = {2 * p[0], 2 * p[1], D == 3 ? 2 * p[2] : 0};
      if (fpid[a_idx<D>(2 * lv.n, f)] >= 0) continue;
    }
#pragma unroll
    for (int m = 0; m < D + 2; ++m) acc[m] += lv.U[m * lv.cells + c];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int m = 0; m < D + 2; ++m) {
    double v = acc[m];
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < 8; ++w) s += red[w];
      atomicAdd(out + m, s);
    }
  }
}

// l1_error_amr (amr_hierarchy.cpp:631-656): per-level sums of |patch - ref|
// over the cells the next level does not cover; ref is the reference solution
// restricted to this level (AoS, 5 doubles per cell). Block tree sums.
template <int D>
__global__ void __launch_bounds__(256) amr_l1_kernel(ALv<D> lv, const int* fpid, const double* ref,
                                                     double* out) {
  __shared__ double red[8];
  double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < lv.tot0;
       t += (long)gridDim.x * blockDim.x) {
    int p[3];
    a_list_pos<D>(lv.boxes, lv.off0, lv.nb, 0, t, p);
    const long c = a_idx<D>(lv.n, p);
    if (fpid) {
      const int f[3] = {2 * p[0], 2 * p[1], D == 3 ? 2 * p[2] : 0};
      if (fpid[a_idx<D>(2 * lv.n, f)] >= 0) continue;
    }
    const Cons<D> q = a_load<D>(lv.U, lv.cells, c);
    const double* r = ref + 5 * c;
    acc[0] += fabs(q.rho - r[0]);
    acc[1] += fabs(q.m[0] - r[1]);
    acc[2] += fabs(q.m[1] - r[2]);
    acc[3] += fabs((D == 3 ? q.m[D - 1] : 0.0) - r[3]);
    acc[4] += fabs(q.E - r[4]);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int m = 0; m < 5; ++m) {
    double v = acc[m];
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < 8; ++w) s += red[w];
      atomicAdd(out + m, s);
    }
  }
}

}  // namespace af

// ------------------------------------------------- clustering on the device --
// cluster (amr_cluster.cpp:79-232) without the masks leaving HBM: summed-area
// tables of the flag and allowed masks make every box count, plane signature
// and allowed test O(1) per entry, and the recursive bisection runs
// breadth-first, one CTA per box of the current frontier. The reference sorts
// its result by box corner, so the traversal order does not matter.
namespace af {

struct CBox {
  int lo[3], hi[3];
};

// The cut a signature proposes (amr_cluster.cpp:130-177): the middle of the
// longest interior run of empty planes (the first on ties), else the strongest
// sign change of the second difference (the first on ties). Returns the offset
// of the cut or -1; *score ranks the proposals of the axes.
template <class T>
__host__ __device__ inline int propose_cut_t(const T* sig, int n, int* score) {
  int gap_len = 0, gap_mid = -1, run = 0;
  for (int i = 0; i < n; ++i) {
    if (sig[i] == 0) {
      ++run;
      continue;
    }
    const int start = i - run;
    if (run > gap_len && start > 0) {
      gap_len = run;
      gap_mid = start + run / 2;
    }
    run = 0;
  }
  if (gap_mid > 0) {
    *score = 1000000 + gap_len;
    return gap_mid;
  }
  if (n >= 4) {
    long long best = 0;
    int at = -1;
    for (int i = 1; i < n - 2; ++i) {
      const long long a = (long long)sig[i - 1] - 2 * (long long)sig[i] + (long long)sig[i + 1];
      const long long b = (long long)sig[i] - 2 * (long long)sig[i + 1] + (long long)sig[i + 2];
      if (!((a < 0 && b > 0) || (a > 0 && b < 0))) continue;
      const long long jump = a - b < 0 ? b - a : a - b;
      if (jump > best) {
        best = jump;
        at = i + 1;
      }
    }
    if (at > 0) {
      *score = (int)(best < 999999 ? best : 999999);
      return at;
    }
  }
  *score = 0;
  return -1;
}

// S has (n+1)^D entries: S[k][j][i] = set cells of the mask in [0,i)x[0,j)x[0,k).
// Pass x writes the row prefixes, passes y and z accumulate along their axis.
// The scans run along one axis per thread; the loads of a batch of 8 entries
// are issued before the dependent adds, so a thread waits for memory once per
// batch instead of once per entry.
template <int D>
__global__ void __launch_bounds__(128) amr_sat_x_kernel(const uint8_t* __restrict__ mask, int n,
                                                        int* __restrict__ S) {
  const long rows = D == 3 ? (long)n * n : n;
  const long r = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int j = (int)(r % n), k = (int)(r / n);
  const uint8_t* m = mask + r * n;
  const long np = n + 1;
  int* s = S + ((D == 3 ? (long)(k + 1) * np : 0) + (j + 1)) * np;
  int acc = 0;
  s[0] = 0;
  int i = 0;
  for (; i + 8 <= n; i += 8) {
    uint8_t v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = m[i + u];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      acc += v[u] != 0;
      s[i + u + 1] = acc;
    }
  }
  for (; i < n; ++i) {
    acc += m[i] != 0;
    s[i + 1] = acc;
  }
}
template <int D>
__global__ void __launch_bounds__(128) amr_sat_y_kernel(int n, int* S) {
  const long np = n + 1;
  const long cols = D == 3 ? np * n : np;  // (i, k) pairs, k in 1..n
  const long c = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (c >= cols) return;
  const int i = (int)(c % np), k = (int)(c / np);
  int* s = S + (D == 3 ? (long)(k + 1) * np * np : 0) + i;
  int acc = 0;
  s[0] = 0;
  int j = 1;
  for (; j + 7 <= n; j += 8) {
    int v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = s[(long)(j + u) * np];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      acc += v[u];
      s[(long)(j + u) * np] = acc;
    }
  }
  for (; j <= n; ++j) {
    acc += s[(long)j * np];
    s[(long)j * np] = acc;
  }
}
__global__ void __launch_bounds__(128) amr_sat_z_kernel(int n, int* S) {
  const long np = n + 1, plane = np * np;
  const long c = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (c >= plane) return;
  int acc = 0;
  S[c] = 0;
  int k = 1;
  for (; k + 7 <= n; k += 8) {
    int v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = S[(long)(k + u) * plane + c];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      acc += v[u];
      S[(long)(k + u) * plane + c] = acc;
    }
  }
  for (; k <= n; ++k) {
    acc += S[k * plane + c];
    S[k * plane + c] = acc;
  }
}

template <int D>
__device__ __forceinline__ long sat_count(const int* S, int n, const int* lo, const int* hi) {
  const long np = n + 1;
  if (D == 2) {
    auto at = [&](int i, int j) { return (long)S[j * np + i]; };
    return at(hi[0], hi[1]) - at(lo[0], hi[1]) - at(hi[0], lo[1]) + at(lo[0], lo[1]);
  }
  auto at = [&](int i, int j, int k) { return (long)S[((long)k * np + j) * np + i]; };
  return at(hi[0], hi[1], hi[2]) - at(lo[0], hi[1], hi[2]) - at(hi[0], lo[1], hi[2]) -
         at(hi[0], hi[1], lo[2]) + at(lo[0], lo[1], hi[2]) + at(lo[0], hi[1], lo[2]) +
         at(hi[0], lo[1], lo[2]) - at(lo[0], lo[1], lo[2]);
}

// One level of the bisection: every box of the frontier `in` is shrunk to its
// flagged cells and either accepted (out) or cut into two boxes of the next
// frontier. cnt[0] = boxes in, cnt[1] = boxes of the next frontier, nout =
// accepted boxes; ovf is raised when a queue is full.
template <int D>
__global__ void __launch_bounds__(128) amr_cluster_level_kernel(const CBox* in, const int* cnt_in,
                                                                CBox* next, int* cnt_next, CBox* out,
                                                                int* nout, int cap, const int* Sf,
                                                                const int* Sa, int n, double efficiency,
                                                                int* ovf) {
  extern __shared__ int sig[];
  __shared__ int s_lo[3], s_hi[3], s_cut[3], s_score[3];
  const int nin = *cnt_in;
  for (int bi = blockIdx.x; bi < nin; bi += gridDim.x) {
    const CBox region = in[bi];
    __syncthreads();
    if (threadIdx.x < 3) {
      s_lo[threadIdx.x] = INT32_MAX;
      s_hi[threadIdx.x] = INT32_MIN;
    }
    __syncthreads();
    const long flagged = sat_count<D>(Sf, n, region.lo, region.hi);
    if (flagged == 0) continue;
    // shrink: per axis the first and last plane holding a flagged cell
    for (int a = 0; a < D; ++a)
      for (int p = region.lo[a] + threadIdx.x; p < region.hi[a]; p += blockDim.x) {
        int lo[3] = {region.lo[0], region.lo[1], region.lo[2]};
        int hi[3] = {region.hi[0], region.hi[1], region.hi[2]};
        lo[a] = p;
        hi[a] = p + 1;
        if (sat_count<D>(Sf, n, lo, hi) > 0) {
          atomicMin(&s_lo[a], p);
          atomicMax(&s_hi[a], p + 1);
        }
      }
    __syncthreads();
    CBox b;
    for (int a = 0; a < 3; ++a) {
      b.lo[a] = a < D ? s_lo[a] : 0;
      b.hi[a] = a < D ? s_hi[a] : 1;
    }
    long vol = 1;
    for (int a = 0; a < D; ++a) vol *= b.hi[a] - b.lo[a];
    const double fill = (double)flagged / (double)vol;
    const bool allowed_ok = !Sa || sat_count<D>(Sa, n, b.lo, b.hi) == vol;
    if ((fill >= efficiency && allowed_ok) || vol == 1) {
      if (threadIdx.x == 0) {
        const int o = atomicAdd(nout, 1);
        if (o < cap) out[o] = b; else *ovf = 1;
      }
      continue;
    }
    // the best signature cut over the axes (the first axis on equal scores)
    for (int a = 0; a < D; ++a) {
      const int ext = b.hi[a] - b.lo[a];
      if (threadIdx.x == 0) {
        s_cut[a] = -1;
        s_score[a] = -1;
      }
      if (ext < 2) continue;
      __syncthreads();
      for (int p = threadIdx.x; p < ext; p += blockDim.x) {
        int lo[3] = {b.lo[0], b.lo[1], b.lo[2]};
        int hi[3] = {b.hi[0], b.hi[1], b.hi[2]};
        lo[a] = b.lo[a] + p;
        hi[a] = b.lo[a] + p + 1;
        sig[p] = (int)sat_count<D>(Sf, n, lo, hi);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        int score = 0;
        const int off = propose_cut_t(sig, ext, &score);
        if (off > 0 && off < ext) {
          s_cut[a] = b.lo[a] + off;
          s_score[a] = score;
        }
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      int axis = -1, cut = -1, best = -1;
      for (int a = 0; a < D; ++a)
        if (s_cut[a] >= 0 && s_score[a] > best) {
          best = s_score[a];
          axis = a;
          cut = s_cut[a];
        }
      bool accept = false;
      if (axis < 0) {  // halve the longest axis (the first among equals)
        for (int a = 0; a < D; ++a)
          if (axis < 0 || b.hi[a] - b.lo[a] > b.hi[axis] - b.lo[axis]) axis = a;
        if (b.hi[axis] - b.lo[axis] < 2)
          accept = true;
        else
          cut = b.lo[axis] + (b.hi[axis] - b.lo[axis]) / 2;
      }
      if (accept) {
        const int o = atomicAdd(nout, 1);
        if (o < cap) out[o] = b; else *ovf = 1;
      } else {
        CBox l = b, h = b;
        l.hi[axis] = cut;
        h.lo[axis] = cut;
        const int o = atomicAdd(cnt_next, 2);
        if (o + 1 < cap) {
          next[o] = l;
          next[o + 1] = h;
        } else {
          *ovf = 1;
        }
      }
    }
  }
}

}  // namespace af
