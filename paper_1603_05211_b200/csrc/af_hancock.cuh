// af_hancock.cuh — the MUSCL-Hancock step of the uniform FV path (sm_100a).
//
// muscl_hancock_step (step.cpp:148-235), the AMR preset's integrator, fused
// into one launch per step. A CTA owns a TX x TY (x TZ) tile and stages in
// shared memory:
//   * the primitives of the tile with a 2-cell halo (build_primitives,
//     step.cpp:18-49; reflective ghosts as flipped copies, grid.cpp:19-53),
//   * the half-step predictor du of the tile with a 1-cell halo: per axis,
//     limited face extrapolations (recon_cell_axis, step.cpp:114-138) and
//     du -= (F(u+) - F(u-)) * dt/(2dx) with the physical flux
//     (euler.hpp:118-128), an axis skipped on a fallback,
//   * the corrector's numerical fluxes of the time-advanced face states
//     (conserved(w+/-) + du, with the two-level positivity fallback),
// then updates out = in + rhs*dt with rhs summed per axis as the reference
// does (+F_low*inv_dx, -F_high*inv_dx). Fallbacks are counted once per cell
// of the predictor's box (interior + one-cell shell) and once per face, as
// the reference's loops count them.
#pragma once

#include <type_traits>

#include "af_uniform_kernels.cuh"

namespace af {

template <int D, int TX, int TY, int TZ>
struct Hk {
  static constexpr int NT = TX * TY * TZ;
  static constexpr int NW = NT / 32;
  static constexpr int NC = D + 2;
  static constexpr int HX = TX + 4, HY = TY + 4, HZ = D == 3 ? TZ + 4 : 1;
  static constexpr int HP = HX * HY * HZ;                    // primitives box (halo 2)
  static constexpr int QX = TX + 2, QY = TY + 2, QZ = D == 3 ? TZ + 2 : 1;
  static constexpr int HQ = QX * QY * QZ;                    // predictor box (halo 1)
  static constexpr int NXF = (TX + 1) * TY * TZ, NYF = TX * (TY + 1) * TZ;
  static constexpr int NZF = D == 3 ? TX * TY * (TZ + 1) : 0;
  static constexpr int NF = NXF + NYF + NZF;
  static constexpr size_t smem_bytes =
      sizeof(double) * ((size_t)NC * HP + (size_t)NC * HQ + (size_t)NC * NF + NW);
};

// recon_cell_axis (step.cpp:114-138): minus/plus extrapolations of w0.
template <int D, int S>
__device__ __forceinline__ bool recon_cell(const Prim<D>& wm, const Prim<D>& w0,
                                           const Prim<D>& wp, Prim<D>& mi, Prim<D>& pl) {
  constexpr int LIM = S & 1;
  const double sr = 0.5 * limiter<LIM>(w0.rho - wm.rho, wp.rho - w0.rho);
  const double sp = 0.5 * limiter<LIM>(w0.p - wm.p, wp.p - w0.p);
  mi.rho = w0.rho - sr;
  pl.rho = w0.rho + sr;
  mi.p = w0.p - sp;
  pl.p = w0.p + sp;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const double sv = 0.5 * limiter<LIM>(w0.v[a] - wm.v[a], wp.v[a] - w0.v[a]);
    mi.v[a] = w0.v[a] - sv;
    pl.v[a] = w0.v[a] + sv;
  }
  if (!physical(mi) || !physical(pl)) {
    mi = w0;
    pl = w0;
    return true;
  }
  return false;
}

// physical_flux (euler.hpp:118-128) as an NC-vector.
template <int D>
__device__ __forceinline__ void phys_flux(const Cons<D>& q, const Prim<D>& w, int axis,
                                          double* f) {
  const double un = w.v[axis];
  f[0] = q.rho * un;
#pragma unroll
  for (int a = 0; a < D; ++a) f[1 + a] = q.m[a] * un;
  f[1 + axis] = f[1 + axis] + w.p;
  f[D + 1] = (q.E + w.p) * un;
}

// physical_state (step.cpp:140-143)
template <int D>
__device__ __forceinline__ bool phys_state(const Cons<D>& q, double gm1) {
  if (!(q.rho > kPosTol)) return false;
  return physical(primitives(q, gm1));
}

template <int D, int S, int TX, int TY, int TZ>
__global__ void __launch_bounds__(TX* TY* TZ, 2) hancock_step(StageArgs a, UGrid g) {
  using K = Hk<D, TX, TY, TZ>;
  constexpr int NC = K::NC;
  if (failed_before(a.r.err)) return;
  extern __shared__ double sm[];
  double* pr = sm;                  // [NC][HP] rho, v.., p
  double* du = pr + NC * K::HP;     // [NC][HQ]
  double* fl = du + NC * K::HQ;     // [NC][NF]
  double* red = fl + NC * K::NF;    // [NW]
  __shared__ int s_fb, s_bad;

  const int tid = threadIdx.x;
  const int n = g.n;
  // tile origin; the slab axis (z in 3D, y in 2D) is offset by this rank's zlo
  const int ntx = n / TX;
  int x0, y0, z0 = 0;
  if (D == 3) {
    const int nty = n / TY;
    x0 = (blockIdx.x % ntx) * TX;
    y0 = ((blockIdx.x / ntx) % nty) * TY;
    z0 = g.zlo + (blockIdx.x / (ntx * nty)) * TZ;
  } else {
    x0 = (blockIdx.x % ntx) * TX;
    y0 = g.zlo + (blockIdx.x / ntx) * TY;
  }
  const int slab_end = g.zlo + g.nzl;
  const double gamma = a.gamma, gm1 = a.gm1, inv_dx = a.inv_dx;
  const double dt = stage_dt_of(a);
  const double half_dt_dx = 0.5 * dt / a.dx;
  if (tid == 0) {
    s_fb = 0;
    s_bad = 0;
    if (blockIdx.x == 0) a.r.dt[a.step] = dt;
  }
  const double* ev = a.eval;
  const long cs = g.cs, zs = g.zs;
  // element offset of global cell (x, y, z) and its reflective flips
  // A slab whose height is not a multiple of TZ gets a last tile reaching
  // past its two halo planes; those planes are never read by an owned cell's
  // stencil, so they are clamped to the last stored plane (the slab is
  // allocated with nzl + 4 planes) instead of addressed past the allocation.
  auto locate = [&](int x, int y, int z, bool* f) {
    f[0] = f[1] = f[2] = false;
    const int mx = bc_map(x, n, g.bc[0], g.bc[1], f[0]);
    if (D == 3) {
      const int my = bc_map(y, n, g.bc[2], g.bc[3], f[1]);
      const int zl = min(slab_map(z, g, 2, f[2]), g.nzl + 3);
      return (long)zl * zs + (long)my * n + mx;
    }
    const int yl = min(slab_map(y, g, 1, f[1]), g.nzl + 3);
    return (long)yl * zs + mx;
  };
  auto cons_at = [&](int x, int y, int z) {
    bool f[3];
    const long o = locate(x, y, z, f);
    Cons<D> q;
    q.rho = ev[o];
#pragma unroll
    for (int d = 0; d < D; ++d) q.m[d] = f[d] ? -ev[(1 + d) * cs + o] : ev[(1 + d) * cs + o];
    q.E = ev[(D + 1) * cs + o];
    return q;
  };
  auto owned = [&](int x, int y, int z) {
    const int sl = D == 3 ? z : y;
    return x >= 0 && x < n && (D == 2 || (y >= 0 && y < n)) && sl >= g.zlo && sl < slab_end;
  };

  // ---- primitives of the tile + 2-cell halo (build_primitives) -----------
  double wave = 0.0, ssum = 0.0;
  int bad = 0, nfb = 0;
  for (int idx = tid; idx < K::HP; idx += K::NT) {
    const int ix = idx % K::HX, iy = (idx / K::HX) % K::HY, iz = D == 3 ? idx / (K::HX * K::HY) : 0;
    const int x = x0 - 2 + ix, y = y0 - 2 + iy, z = D == 3 ? z0 - 2 + iz : 0;
    bool f[3];
    const long o = locate(x, y, z, f);
    Cons<D> q;
    q.rho = __ldg(ev + o);
#pragma unroll
    for (int d = 0; d < D; ++d) q.m[d] = __ldg(ev + (1 + d) * cs + o);
    q.E = __ldg(ev + (D + 1) * cs + o);
    Prim<D> w = primitives(q, gm1);
    const bool inner = ix >= 2 && ix < TX + 2 && iy >= 2 && iy < TY + 2 &&
                       (D == 2 || (iz >= 2 && iz < TZ + 2));
    if (inner && owned(x, y, z)) {
      if (!cell_ok(q, w)) bad = 1;
      double s, m;
      wave_speeds(w, gamma, s, m);
      wave = fmax(wave, m);
    }
#pragma unroll
    for (int d = 0; d < D; ++d)
      if (f[d]) w.v[d] = -w.v[d];
    pr[idx] = w.rho;
#pragma unroll
    for (int d = 0; d < D; ++d) pr[(1 + d) * K::HP + idx] = w.v[d];
    pr[(NC - 1) * K::HP + idx] = w.p;
  }
  __syncthreads();
  auto P = [&](int ix, int iy, int iz) {  // halo-box coordinates
    const int idx = (iz * K::HY + iy) * K::HX + ix;
    Prim<D> w;
    w.rho = pr[idx];
#pragma unroll
    for (int d = 0; d < D; ++d) w.v[d] = pr[(1 + d) * K::HP + idx];
    w.p = pr[(NC - 1) * K::HP + idx];
    return w;
  };

  // ---- half-step predictor over the tile + 1-cell halo ---------------------
  for (int idx = tid; idx < K::HQ; idx += K::NT) {
    const int qx = idx % K::QX, qy = (idx / K::QX) % K::QY, qz = D == 3 ? idx / (K::QX * K::QY) : 0;
    const int ix = qx + 1, iy = qy + 1, iz = D == 3 ? qz + 1 : 0;  // halo-box coords
    const int x = x0 - 1 + qx, y = y0 - 1 + qy, z = D == 3 ? z0 - 1 + qz : 0;
    // counted once: by the tile whose interior holds the clamped position
    // (the reference's predictor box is the interior plus a one-cell shell)
    const int cxm = min(max(x, 0), n - 1), cym = D == 3 ? min(max(y, 0), n - 1) : y;
    const int csl = D == 3 ? min(max(z, 0), n - 1) : min(max(y, 0), n - 1);
    const bool in_box = x >= -1 && x <= n && y >= -1 && y <= n && (D == 2 || (z >= -1 && z <= n));
    const bool counts = in_box && cxm >= x0 && cxm < x0 + TX &&
                        (D == 2 ? (csl >= y0 && csl < y0 + TY && csl >= g.zlo && csl < slab_end)
                                : (cym >= y0 && cym < y0 + TY && csl >= z0 && csl < z0 + TZ &&
                                   csl >= g.zlo && csl < slab_end));
    double acc[NC];
#pragma unroll
    for (int m = 0; m < NC; ++m) acc[m] = 0.0;
    const Prim<D> w0 = P(ix, iy, iz);
#pragma unroll
    for (int ax = 0; ax < D; ++ax) {
      const Prim<D> wm = P(ix - (ax == 0), iy - (ax == 1), iz - (ax == 2));
      const Prim<D> wp = P(ix + (ax == 0), iy + (ax == 1), iz + (ax == 2));
      Prim<D> mi, pl;
      if (recon_cell<D, S>(wm, w0, wp, mi, pl)) {
        if (counts) ++nfb;
        continue;  // zero slopes: no predictor contribution on this axis
      }
      const Cons<D> um = conserved(mi, gm1), up = conserved(pl, gm1);
      double fp[NC], fm[NC];
      phys_flux<D>(up, pl, ax, fp);
      phys_flux<D>(um, mi, ax, fm);
#pragma unroll
      for (int m = 0; m < NC; ++m) acc[m] = acc[m] - (fp[m] - fm[m]) * half_dt_dx;
    }
#pragma unroll
    for (int m = 0; m < NC; ++m) du[m * K::HQ + idx] = acc[m];
  }
  __syncthreads();
  auto DU = [&](int qx, int qy, int qz) {  // predictor-box coordinates
    const int idx = (qz * K::QY + qy) * K::QX + qx;
    Cons<D> c;
    c.rho = du[idx];
#pragma unroll
    for (int d = 0; d < D; ++d) c.m[d] = du[(1 + d) * K::HQ + idx];
    c.E = du[(NC - 1) * K::HQ + idx];
    return c;
  };
  auto add = [](const Cons<D>& p, const Cons<D>& q) {
    Cons<D> r;
    r.rho = p.rho + q.rho;
#pragma unroll
    for (int d = 0; d < D; ++d) r.m[d] = p.m[d] + q.m[d];
    r.E = p.E + q.E;
    return r;
  };

  // ---- corrector fluxes ------------------------------------------------------
  // face (fx, fy, fz) of axis AX sits between cells c-e_AX and c (tile coords)
  auto face = [&](auto axc, int fx, int fy, int fz, int slot) {
    constexpr int AX = decltype(axc)::value;
    const int ex = AX == 0, ey = AX == 1, ez = AX == 2;
    // left cell L = c - e, right cell R = c (halo-box coords: +2; predictor: +1)
    const int lx = fx - ex, ly = fy - ey, lz = fz - ez;
    Prim<D> lmi, lpl, rmi, rpl;
    recon_cell<D, S>(P(lx + 2 - ex, ly + 2 - ey, D == 3 ? lz + 2 - ez : 0),
                     P(lx + 2, ly + 2, D == 3 ? lz + 2 : 0),
                     P(lx + 2 + ex, ly + 2 + ey, D == 3 ? lz + 2 + ez : 0), lmi, lpl);
    recon_cell<D, S>(P(fx + 2 - ex, fy + 2 - ey, D == 3 ? fz + 2 - ez : 0),
                     P(fx + 2, fy + 2, D == 3 ? fz + 2 : 0),
                     P(fx + 2 + ex, fy + 2 + ey, D == 3 ? fz + 2 + ez : 0), rmi, rpl);
    const Cons<D> dl = DU(lx + 1, ly + 1, D == 3 ? lz + 1 : 0);
    const Cons<D> dr = DU(fx + 1, fy + 1, D == 3 ? fz + 1 : 0);
    Cons<D> ul = add(conserved(lpl, gm1), dl);
    Cons<D> ur = add(conserved(rmi, gm1), dr);
    // the face counts its fallbacks once (f in [0, n] per interior line):
    // with the tile and rank owning its high-side cell, or for f == n the
    // low-side cell
    const int ia = AX == 0 ? fx : AX == 1 ? fy : fz;
    const int ta = AX == 0 ? TX : AX == 1 ? TY : TZ;
    const int gf = (AX == 0 ? x0 : AX == 1 ? y0 : z0) + ia;
    const bool counts = (ia < ta && owned(x0 + fx, y0 + fy, z0 + fz)) ||
                        (gf == n && owned(x0 + lx, y0 + ly, z0 + lz));
    if (!phys_state(ul, gm1)) {
      const Cons<D> ql = cons_at(x0 + lx, y0 + ly, z0 + lz);
      ul = add(ql, dl);
      if (!phys_state(ul, gm1)) ul = ql;
      if (counts) ++nfb;
    }
    if (!phys_state(ur, gm1)) {
      const Cons<D> qr = cons_at(x0 + fx, y0 + fy, z0 + fz);
      ur = add(qr, dr);
      if (!phys_state(ur, gm1)) ur = qr;
      if (counts) ++nfb;
    }
    const Cons<D> F = num_flux<D, AX, S>(ul, primitives(ul, gm1), ur, primitives(ur, gm1), gamma);
    fl[slot] = F.rho;
#pragma unroll
    for (int d = 0; d < D; ++d) fl[(1 + d) * K::NF + slot] = F.m[d];
    fl[(NC - 1) * K::NF + slot] = F.E;
  };
  for (int f = tid; f < K::NF; f += K::NT) {
    if (f < K::NXF) {
      const int fx = f % (TX + 1), fy = (f / (TX + 1)) % TY, fz = D == 3 ? f / ((TX + 1) * TY) : 0;
      face(std::integral_constant<int, 0>(), fx, fy, fz, f);
    } else if (f < K::NXF + K::NYF) {
      const int h = f - K::NXF;
      const int fx = h % TX, fy = (h / TX) % (TY + 1), fz = D == 3 ? h / (TX * (TY + 1)) : 0;
      face(std::integral_constant<int, 1>(), fx, fy, fz, f);
    } else if constexpr (D == 3) {
      const int h = f - K::NXF - K::NYF;
      const int fx = h % TX, fy = (h / TX) % TY, fz = h / (TX * TY);
      face(std::integral_constant<int, 2>(), fx, fy, fz, f);
    }
  }
  __syncthreads();

  // ---- update ------------------------------------------------------------------
  const int tx = tid % TX, ty = (tid / TX) % TY, tz = D == 3 ? tid / (TX * TY) : 0;
  const int x = x0 + tx, y = y0 + ty, z = z0 + tz;
  if (owned(x, y, z)) {
    bool f[3];
    const long o = locate(x, y, z, f);
    const int ixl = (tz * TY + ty) * (TX + 1) + tx;
    const int iyl = K::NXF + (tz * (TY + 1) + ty) * TX + tx;
    const int izl = K::NXF + K::NYF + (tz * TY + ty) * TX + tx;
    double q[NC];
#pragma unroll
    for (int m = 0; m < NC; ++m) {
      double rhs = 0.0;
      rhs = rhs + fl[m * K::NF + ixl] * inv_dx;
      rhs = rhs - fl[m * K::NF + ixl + 1] * inv_dx;
      rhs = rhs + fl[m * K::NF + iyl] * inv_dx;
      rhs = rhs - fl[m * K::NF + iyl + TX] * inv_dx;
      if (D == 3) {
        rhs = rhs + fl[m * K::NF + izl] * inv_dx;
        rhs = rhs - fl[m * K::NF + izl + TX * TY] * inv_dx;
      }
      q[m] = ev[m * cs + o] + rhs * dt;
      a.out[m * cs + o] = q[m];
    }
    if (a.use_cfl) {  // the next step's CFL denominator
      Cons<D> c;
      c.rho = q[0];
#pragma unroll
      for (int d = 0; d < D; ++d) c.m[d] = q[1 + d];
      c.E = q[NC - 1];
      double s, m;
      wave_speeds(primitives(c, gm1), gamma, s, m);
      ssum = fmax(ssum, s);
    }
  }
  if (bad) s_bad = 1;
  if (nfb) atomicAdd(&s_fb, nfb);
  block_max_atomic<K::NT>(wave, red, a.r.wave_u + a.step);
  if (a.use_cfl) block_max_atomic<K::NT>(ssum, red, a.r.smax + a.step + 1);
  if (tid == 0) {
    if (s_bad) raise_error(a);
    if (s_fb) atomicAdd(a.r.fb + a.step, (unsigned long long)s_fb);
  }
}

}  // namespace af
