// af_uniform_kernels.cuh — fused RK2-stage kernels of the uniform FV path.
//
// One launch = one rk2_stage (step.cpp:93-109): build_primitives (step.cpp:18-49)
// + accumulate_rhs (step.cpp:57-89) + the update out = base + rhs*stage_dt,
// fused so each cell's state is read from HBM once and each face flux is
// evaluated once per tile (the reference also evaluates one flux per face).
//
// 3D: a CTA owns a TX x TY column of cells and marches along z through a
// chunk, holding a 4-plane ring of primitives (with a 2-cell x/y halo) in
// shared memory; the z-face between planes k and k+1 is kept in registers
// by the column's thread and reused as the next plane's low face.
// 2D: a CTA owns a TX x TY tile with a 2-cell halo.
//
// Per-cell summation order is the reference's: rhs = 0; per axis
// rhs += F_low*inv_dx; rhs -= F_high*inv_dx (step.cpp:80-81).
#pragma once

#include "af_internal.h"
#include "af_physics.cuh"

namespace af {

struct StageArgs {
  const double* eval;  // state the fluxes are evaluated on (halo planes filled)
  const double* base;  // state the update is applied to (may alias out)
  double* out;
  double dx, inv_dx, gamma, gm1;
  double cfl, fixed_dt;
  int use_cfl;
  double dt_scale;  // 0.5 (stage 1) or 1.0 (stage 2): stage_dt = dt_scale*dt (step.cpp:240,242)
  int step, stage;
  int zchunk;
  int zbeg, zend;  // 3D: the planes [zbeg, zend) this launch updates (chunks of zchunk)
  RunRecords r;
};

// Physical boundary mapping of one index along one axis: the cell whose value
// the reference's fill_ghosts copies into ghost position c (grid.cpp:19-53).
__device__ __forceinline__ int bc_map(int c, int n, int lo, int hi, bool& flip) {
  flip = false;
  if (c >= 0 && c < n) return c;
  const int kind = c < 0 ? lo : hi;
  if (kind == AF_BC_OUTFLOW) return c < 0 ? 0 : n - 1;
  if (kind == AF_BC_PERIODIC) {
    c %= n;
    return c < 0 ? c + n : c;
  }
  while (c < 0 || c >= n) {  // reflective fold
    if (c < 0) c = -1 - c;
    if (c >= n) c = 2 * n - 1 - c;
    flip = !flip;
  }
  return c;
}

// Local storage index along the slab axis for global index c (halo planes
// hold the neighbours' cells, including the periodic wrap across ranks).
__device__ __forceinline__ int slab_map(int c, const UGrid& g, int axis, bool& flip) {
  flip = false;
  const bool halo = (c >= 0 && c < g.n) ||
                    (g.nranks > 1 && g.bc[2 * axis] == AF_BC_PERIODIC &&
                     g.bc[2 * axis + 1] == AF_BC_PERIODIC);
  if (!halo) c = bc_map(c, g.n, g.bc[2 * axis], g.bc[2 * axis + 1], flip);
  return c - g.zlo + 2;
}

__device__ __forceinline__ unsigned long long dbits(double x) {
  return (unsigned long long)__double_as_longlong(x);
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide max of non-negative v, then one atomicMax on the bit pattern.
template <int NT>
__device__ __forceinline__ void block_max_atomic(double v, double* red,
                                                 unsigned long long* target) {
  v = warp_max(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double x = lane < NT / 32 ? red[lane] : 0.0;
    x = warp_max(x);
    if (lane == 0 && x > 0.0) atomicMax(target, dbits(x));
  }
}

__device__ __forceinline__ double stage_dt_of(const StageArgs& a) {
  double dt = a.fixed_dt;
  if (a.use_cfl) dt = a.cfl * a.dx / __longlong_as_double((long long)a.r.smax[a.step]);
  return dt;
}

// Block-uniform early exit once an earlier stage has failed (the flag can be
// raised by another CTA of the same launch, so one thread reads it).
__device__ __forceinline__ bool failed_before(const int* err) {
  __shared__ int s_err;
  if (threadIdx.x == 0) s_err = *(volatile const int*)err;
  __syncthreads();
  return s_err != 0;
}

__device__ __forceinline__ void raise_error(const StageArgs& a) {
  atomicExch(a.r.err, 1);
  atomicMin(a.r.err + 1, a.step * 2 + (a.stage - 1));
}

// ------------------------------------------------------------------ 3D --

template <int LIM, int TX, int TY>
struct Fv3d {
  static constexpr int NT = TX * TY;
  static constexpr int NW = NT / 32;
  static constexpr int HX = TX + 4, HY = TY + 4, HP = HX * HY;
  static constexpr int NXF = (TX + 1) * TY, NYF = TX * (TY + 1);
  static constexpr int UX = (NXF + 31) / 32, UY = (NYF + 31) / 32;
  static constexpr int NC = 5;  // primitives per cell in the ring: rho, v0, v1, v2, p
  static constexpr size_t smem_bytes =
      sizeof(double) * (size_t)(4 * NC * HP + 5 * NXF + 5 * NYF + NW + 5 * HP);
};

// cp.async (LDGSTS) of one double: global -> shared, completion tracked per thread.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

template <int LIM, int TX, int TY>
__global__ void __launch_bounds__(TX* TY, 2) fv3d_stage(StageArgs a, UGrid g) {
  using K = Fv3d<LIM, TX, TY>;
  constexpr int D = 3;
  if (failed_before(a.r.err)) return;  // an earlier stage failed: freeze state
  extern __shared__ double sm[];
  double* ring = sm;                           // [4][NC][HP]
  double* fxs = ring + 4 * K::NC * K::HP;      // [5][NXF]
  double* fys = fxs + 5 * K::NXF;              // [5][NYF]
  double* red = fys + 5 * K::NYF;              // [NW]
  double* raw = red + K::NW;                   // [5][HP] conserved plane in flight (cp.async)
  __shared__ int s_fb, s_bad;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tx = tid % TX, ty = tid / TX;
  const int n = g.n;
  const int tiles_x = n / TX;
  const int x0 = (blockIdx.x % tiles_x) * TX, y0 = (blockIdx.x / tiles_x) * TY;
  const int zc0 = a.zbeg + blockIdx.y * a.zchunk;
  const int zc1 = min(zc0 + a.zchunk, a.zend);
  const double gamma = a.gamma, gm1 = a.gm1, inv_dx = a.inv_dx;
  const double rgm1 = 1.0 / gm1;  // RN(1/(gamma-1)) for div_rcp
  const double sdt = a.dt_scale * stage_dt_of(a);
  if (tid == 0) {
    s_fb = 0;
    s_bad = 0;
    if (a.stage == 1 && blockIdx.x == 0 && blockIdx.y == 0) a.r.dt[a.step] = stage_dt_of(a);
  }
  const double* ev = a.eval;
  const long cs = g.cs, zs = g.zs;
  double wave = 0.0;  // per-axis max of |v_a|+c over this thread's owned cells
  double ssum = 0.0;  // stage 2: max of sum_a(|v_a|+c) over the updated cells
  int bad = 0;

  // This thread's halo-box cells (idx = tid + t*NT) and their x/y boundary
  // mapping, which is the same on every plane: in-plane offset of the source
  // cell, or -1 for corners (never on an axis stencil) and idx >= HP; the
  // reflective momentum flips as bit 0 (x) and bit 1 (y).
  constexpr int HPT = (K::HP + K::NT - 1) / K::NT;
  int hoff[HPT];
  unsigned hflip = 0;
#pragma unroll
  for (int t = 0; t < HPT; ++t) {
    const int idx = tid + t * K::NT;
    hoff[t] = -1;
    if (idx >= K::HP) continue;
    const int ix = idx % K::HX, iy = idx / K::HX;
    const bool cx = ix >= 2 && ix < TX + 2, cy = iy >= 2 && iy < TY + 2;
    if (!cx && !cy) continue;
    bool fx, fy;
    const int mx = bc_map(x0 - 2 + ix, n, g.bc[0], g.bc[1], fx);
    const int my = bc_map(y0 - 2 + iy, n, g.bc[2], g.bc[3], fy);
    hoff[t] = my * n + mx;
    hflip |= ((fx ? 1u : 0u) | (fy ? 2u : 0u)) << (2 * t);
  }
  // Plane gz of eval -> primitives of ring slot gz&3, in two halves so the
  // global loads of plane k+3 overlap the flux work of plane k: issue_plane
  // starts cp.async copies of the conserved values of this thread's cells,
  // convert_plane (same thread, same cells) turns them into primitives.
  auto issue_plane = [&](int gz) {
    bool fz;
    const int zl = slab_map(gz, g, 2, fz);
#pragma unroll
    for (int t = 0; t < HPT; ++t) {
      if (hoff[t] < 0) continue;
      const int idx = tid + t * K::NT;
      const long off = (long)zl * zs + hoff[t];
#pragma unroll
      for (int m = 0; m < 5; ++m) cp_async8(raw + m * K::HP + idx, ev + m * cs + off);
    }
    cp_async_commit();
  };
  auto convert_plane = [&](int gz) {
    cp_async_wait_all();
    bool fz;
    (void)slab_map(gz, g, 2, fz);
    double* dst = ring + ((gz + 4) & 3) * (K::NC * K::HP);
    const bool own = gz >= zc0 && gz < zc1;
#pragma unroll
    for (int t = 0; t < HPT; ++t) {
      if (hoff[t] < 0) continue;
      const int idx = tid + t * K::NT;
      const int ix = idx % K::HX, iy = idx / K::HX;
      const bool cx = ix >= 2 && ix < TX + 2, cy = iy >= 2 && iy < TY + 2;
      Cons<D> q;
      q.rho = raw[idx];
      q.m[0] = raw[K::HP + idx];
      q.m[1] = raw[2 * K::HP + idx];
      q.m[2] = raw[3 * K::HP + idx];
      q.E = raw[4 * K::HP + idx];
      Prim<D> w = primitives(q, gm1);
      if (own && cx && cy) {
        if (!cell_ok(q, w)) bad = 1;
        double s, m;
        wave_speeds(w, gamma, s, m);
        wave = fmax(wave, m);
      }
      const unsigned fl = hflip >> (2 * t);
      if (fl & 1u) w.v[0] = -w.v[0];
      if (fl & 2u) w.v[1] = -w.v[1];
      if (fz) w.v[2] = -w.v[2];
      dst[0 * K::HP + idx] = w.rho;
      dst[1 * K::HP + idx] = w.v[0];
      dst[2 * K::HP + idx] = w.v[1];
      dst[3 * K::HP + idx] = w.v[2];
      dst[4 * K::HP + idx] = w.p;
    }
  };
  auto prim_at = [&](int gz, int idx) {
    const double* s = ring + ((gz + 4) & 3) * (K::NC * K::HP);
    Prim<D> w;
    w.rho = s[idx];
    w.v[0] = s[K::HP + idx];
    w.v[1] = s[2 * K::HP + idx];
    w.v[2] = s[3 * K::HP + idx];
    w.p = s[4 * K::HP + idx];
    return w;
  };
  // Conserved state of global cell (x,y,z) of eval (a reflective ghost with
  // its momentum flipped, grid.cpp:19-53): only read on the rare first-order
  // fallback (scheme.cpp:160-162).
  auto cons_at = [&](int gx, int gy, int gz) {
    bool fx, fy, fz;
    const int mx = bc_map(gx, n, g.bc[0], g.bc[1], fx);
    const int my = bc_map(gy, n, g.bc[2], g.bc[3], fy);
    const int zl = slab_map(gz, g, 2, fz);
    const long c = (long)zl * zs + (long)my * n + mx;
    Cons<D> q;
    q.rho = ev[c];
    q.m[0] = fx ? -ev[cs + c] : ev[cs + c];
    q.m[1] = fy ? -ev[2 * cs + c] : ev[2 * cs + c];
    q.m[2] = fz ? -ev[3 * cs + c] : ev[3 * cs + c];
    q.E = ev[4 * cs + c];
    return q;
  };
  int nfb = 0;
  // z face between planes gz-1 and gz of this thread's column. A face that
  // two tiles (or two z chunks) both evaluate counts its fallback in one of
  // them only: the tile owning its high-side cell, the domain's high faces in
  // the tile below them, the chunk's first z face in the chunk below it
  // (accumulate_rhs counts each face once, step.cpp:57-89).
  auto zface = [&](int gz) {
    const int idx = (ty + 2) * K::HX + tx + 2;
    const Prim<D> wm1 = prim_at(gz - 2, idx), w0 = prim_at(gz - 1, idx);
    const Prim<D> wp1 = prim_at(gz, idx), wp2 = prim_at(gz + 1, idx);
    Prim<D> l, r;
    if (muscl_recon<D, LIM>(wm1, w0, wp1, wp2, l, r)) {
      if (gz > zc0 || zc0 == 0) ++nfb;
      return num_flux<D, 2, LIM>(cons_at(x0 + tx, y0 + ty, gz - 1), w0,
                             cons_at(x0 + tx, y0 + ty, gz), wp1, gamma);
    }
    return recon_flux_fast<D, 2, LIM>(l, r, gamma, gm1, rgm1);
  };

  // Prologue: planes zc0-2 .. zc0+1 and the chunk's first low z face; the
  // copies of plane zc0+2 are put in flight.
  for (int z = zc0 - 2; z < zc0 + 2; ++z) {
    issue_plane(z);
    convert_plane(z);
  }
  issue_plane(zc0 + 2);
  __syncthreads();
  Cons<D> fz_lo = zface(zc0);

  for (int k = zc0; k < zc1; ++k) {
    // base of this thread's cell, prefetched ahead of the flux work
    const long own = (long)(k - g.zlo + 2) * zs + (long)(y0 + ty) * n + (x0 + tx);
    double b[5];
#pragma unroll
    for (int m = 0; m < 5; ++m) b[m] = a.base[m * cs + own];
    convert_plane(k + 2);                  // landed during the previous plane's work
    if (k + 3 < zc1 + 2) issue_plane(k + 3);  // in flight during this plane's work
    __syncthreads();
    const Cons<D> fz_hi = zface(k + 1);
    for (int u = warp; u < K::UX + K::UY; u += K::NW) {
      if (u < K::UX) {
        const int f = u * 32 + lane;
        if (f < K::NXF) {
          const int fxi = f % (TX + 1), fyi = f / (TX + 1);
          const int base = (fyi + 2) * K::HX + fxi;  // stencil x = fxi-2 .. fxi+1
          const Prim<D> wm1 = prim_at(k, base), w0 = prim_at(k, base + 1);
          const Prim<D> wp1 = prim_at(k, base + 2), wp2 = prim_at(k, base + 3);
          Prim<D> l, r;
          Cons<D> fl;
          if (muscl_recon<D, LIM>(wm1, w0, wp1, wp2, l, r)) {
            if (fxi < TX || x0 + TX == n) ++nfb;
            fl = num_flux<D, 0, LIM>(cons_at(x0 + fxi - 1, y0 + fyi, k), w0,
                                 cons_at(x0 + fxi, y0 + fyi, k), wp1, gamma);
          } else {
            fl = recon_flux_fast<D, 0, LIM>(l, r, gamma, gm1, rgm1);
          }
          fxs[0 * K::NXF + f] = fl.rho;
          fxs[1 * K::NXF + f] = fl.m[0];
          fxs[2 * K::NXF + f] = fl.m[1];
          fxs[3 * K::NXF + f] = fl.m[2];
          fxs[4 * K::NXF + f] = fl.E;
        }
      } else {
        const int f = (u - K::UX) * 32 + lane;
        if (f < K::NYF) {
          const int fxi = f % TX, fyi = f / TX;
          const int base = fyi * K::HX + fxi + 2;  // stencil y = fyi-2 .. fyi+1
          const Prim<D> wm1 = prim_at(k, base), w0 = prim_at(k, base + K::HX);
          const Prim<D> wp1 = prim_at(k, base + 2 * K::HX), wp2 = prim_at(k, base + 3 * K::HX);
          Prim<D> l, r;
          Cons<D> fl;
          if (muscl_recon<D, LIM>(wm1, w0, wp1, wp2, l, r)) {
            if (fyi < TY || y0 + TY == n) ++nfb;
            fl = num_flux<D, 1, LIM>(cons_at(x0 + fxi, y0 + fyi - 1, k), w0,
                                 cons_at(x0 + fxi, y0 + fyi, k), wp1, gamma);
          } else {
            fl = recon_flux_fast<D, 1, LIM>(l, r, gamma, gm1, rgm1);
          }
          fys[0 * K::NYF + f] = fl.rho;
          fys[1 * K::NYF + f] = fl.m[0];
          fys[2 * K::NYF + f] = fl.m[1];
          fys[3 * K::NYF + f] = fl.m[2];
          fys[4 * K::NYF + f] = fl.E;
        }
      }
    }
    __syncthreads();
    // Update: rhs accumulated in the reference order, then out = base + rhs*dt.
    {
      const int ixl = ty * (TX + 1) + tx, iyl = ty * TX + tx;
      const double zl[5] = {fz_lo.rho, fz_lo.m[0], fz_lo.m[1], fz_lo.m[2], fz_lo.E};
      const double zh[5] = {fz_hi.rho, fz_hi.m[0], fz_hi.m[1], fz_hi.m[2], fz_hi.E};
#pragma unroll
      for (int m = 0; m < 5; ++m) {
        double rhs = 0.0;
        rhs = rhs + fxs[m * K::NXF + ixl] * inv_dx;
        rhs = rhs - fxs[m * K::NXF + ixl + 1] * inv_dx;
        rhs = rhs + fys[m * K::NYF + iyl] * inv_dx;
        rhs = rhs - fys[m * K::NYF + iyl + TX] * inv_dx;
        rhs = rhs + zl[m] * inv_dx;
        rhs = rhs - zh[m] * inv_dx;
        b[m] = b[m] + rhs * sdt;
      }
#pragma unroll
      for (int m = 0; m < 5; ++m) a.out[m * cs + own] = b[m];
      if (a.stage == 2 && a.use_cfl) {  // next step's CFL denominator, fused
        Cons<D> q;
        q.rho = b[0];
        q.m[0] = b[1];
        q.m[1] = b[2];
        q.m[2] = b[3];
        q.E = b[4];
        double s, m;
        wave_speeds(primitives(q, gm1), gamma, s, m);
        ssum = fmax(ssum, s);
      }
    }
    fz_lo = fz_hi;
  }

  // Stage diagnostics: positivity, StepDiag wave max, fallbacks.
  if (bad) s_bad = 1;
  if (nfb) atomicAdd(&s_fb, nfb);
  block_max_atomic<K::NT>(wave, red, a.stage == 1 ? a.r.wave_u + a.step : a.r.wave_mid + a.step);
  if (a.stage == 2 && a.use_cfl) block_max_atomic<K::NT>(ssum, red, a.r.smax + a.step + 1);
  if (tid == 0) {
    if (s_bad) raise_error(a);
    if (s_fb) atomicAdd(a.r.fb + a.step, (unsigned long long)s_fb);
  }
}

// ------------------------------------------------------------------ 2D --

template <int LIM, int TX, int TY>
struct Fv2d {
  static constexpr int NT = TX * TY;
  static constexpr int NW = NT / 32;
  static constexpr int HX = TX + 4, HY = TY + 4, HP = HX * HY;
  static constexpr int NXF = (TX + 1) * TY, NYF = TX * (TY + 1);
  static constexpr int UX = (NXF + 31) / 32, UY = (NYF + 31) / 32;
  static constexpr int NC = 4;  // rho, v0, v1, p
  static constexpr size_t smem_bytes =
      sizeof(double) * (size_t)(NC * HP + 4 * NXF + 4 * NYF + NW);
};

template <int LIM, int TX, int TY>
__global__ void __launch_bounds__(TX* TY, 2) fv2d_stage(StageArgs a, UGrid g) {
  using K = Fv2d<LIM, TX, TY>;
  constexpr int D = 2;
  // programmatic dependent launch (a no-op without the launch attribute): the
  // launch overlaps the predecessor's tail, the wait precedes every read
  asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory");
  if (failed_before(a.r.err)) return;
  extern __shared__ double sm[];
  double* pl = sm;                  // [NC][HP]
  double* fxs = pl + K::NC * K::HP;  // [4][NXF]
  double* fys = fxs + 4 * K::NXF;    // [4][NYF]
  double* red = fys + 4 * K::NYF;
  __shared__ int s_fb, s_bad;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tx = tid % TX, ty = tid / TX;
  const int n = g.n;
  const int tiles_x = n / TX;
  const int x0 = (blockIdx.x % tiles_x) * TX;
  const int y0 = g.zlo + (blockIdx.x / tiles_x) * TY;  // slab axis = y
  const double gamma = a.gamma, gm1 = a.gm1, inv_dx = a.inv_dx;
  const double rgm1 = 1.0 / gm1;  // RN(1/(gamma-1)) for div_rcp
  const double sdt = a.dt_scale * stage_dt_of(a);
  if (tid == 0) {
    s_fb = 0;
    s_bad = 0;
    if (a.stage == 1 && blockIdx.x == 0) a.r.dt[a.step] = stage_dt_of(a);
  }
  const double* ev = a.eval;
  const long cs = g.cs, zs = g.zs;
  const bool active = y0 + ty < g.zlo + g.nzl;
  const long own = (long)(y0 + ty - g.zlo + 2) * zs + (x0 + tx);
  double b[4];
  if (active) {
#pragma unroll
    for (int m = 0; m < 4; ++m) b[m] = a.base[m * cs + own];
  }
  double wave = 0.0, ssum = 0.0;
  int bad = 0, nfb = 0;
  for (int idx = tid; idx < K::HP; idx += K::NT) {
    const int ix = idx % K::HX, iy = idx / K::HX;
    const bool cx = ix >= 2 && ix < TX + 2, cy = iy >= 2 && iy < TY + 2;
    if (!cx && !cy) continue;
    bool fx, fy;
    const int mx = bc_map(x0 - 2 + ix, n, g.bc[0], g.bc[1], fx);
    const int gy = y0 - 2 + iy;
    const int yl = slab_map(gy, g, 1, fy);
    const long off = (long)yl * zs + mx;
    Cons<D> q;
    q.rho = __ldg(ev + off);
    q.m[0] = __ldg(ev + cs + off);
    q.m[1] = __ldg(ev + 2 * cs + off);
    q.E = __ldg(ev + 3 * cs + off);
    Prim<D> w = primitives(q, gm1);
    if (cx && cy && gy < g.zlo + g.nzl) {
      if (!cell_ok(q, w)) bad = 1;
      double s, m;
      wave_speeds(w, gamma, s, m);
      wave = fmax(wave, m);
    }
    if (fx) w.v[0] = -w.v[0];
    if (fy) w.v[1] = -w.v[1];
    pl[idx] = w.rho;
    pl[K::HP + idx] = w.v[0];
    pl[2 * K::HP + idx] = w.v[1];
    pl[3 * K::HP + idx] = w.p;
  }
  __syncthreads();
  auto prim_at = [&](int idx) {
    Prim<D> w;
    w.rho = pl[idx];
    w.v[0] = pl[K::HP + idx];
    w.v[1] = pl[2 * K::HP + idx];
    w.p = pl[3 * K::HP + idx];
    return w;
  };
  auto cons_at = [&](int gx, int gy) {
    bool fx, fy;
    const int mx = bc_map(gx, n, g.bc[0], g.bc[1], fx);
    const int yl = slab_map(gy, g, 1, fy);
    const long c = (long)yl * zs + mx;
    Cons<D> q;
    q.rho = ev[c];
    q.m[0] = fx ? -ev[cs + c] : ev[cs + c];
    q.m[1] = fy ? -ev[2 * cs + c] : ev[2 * cs + c];
    q.E = ev[3 * cs + c];
    return q;
  };
  for (int u = warp; u < K::UX + K::UY; u += K::NW) {
    if (u < K::UX) {
      const int f = u * 32 + lane;
      if (f < K::NXF) {
        const int fxi = f % (TX + 1), fyi = f / (TX + 1);
        const int base = (fyi + 2) * K::HX + fxi;
        const Prim<D> wm1 = prim_at(base), w0 = prim_at(base + 1);
        const Prim<D> wp1 = prim_at(base + 2), wp2 = prim_at(base + 3);
        Prim<D> l, r;
        Cons<D> fl;
        if (muscl_recon<D, LIM>(wm1, w0, wp1, wp2, l, r)) {
          if (fxi < TX || x0 + TX == n) ++nfb;  // one count per face (see fv3d_stage)
          fl = num_flux<D, 0, LIM>(cons_at(x0 + fxi - 1, y0 + fyi), w0,
                               cons_at(x0 + fxi, y0 + fyi), wp1, gamma);
        } else {
          fl = recon_flux_fast<D, 0, LIM>(l, r, gamma, gm1, rgm1);
        }
        fxs[f] = fl.rho;
        fxs[K::NXF + f] = fl.m[0];
        fxs[2 * K::NXF + f] = fl.m[1];
        fxs[3 * K::NXF + f] = fl.E;
      }
    } else {
      const int f = (u - K::UX) * 32 + lane;
      if (f < K::NYF) {
        const int fxi = f % TX, fyi = f / TX;
        const int base = fyi * K::HX + fxi + 2;
        const Prim<D> wm1 = prim_at(base), w0 = prim_at(base + K::HX);
        const Prim<D> wp1 = prim_at(base + 2 * K::HX), wp2 = prim_at(base + 3 * K::HX);
        Prim<D> l, r;
        Cons<D> fl;
        if (muscl_recon<D, LIM>(wm1, w0, wp1, wp2, l, r)) {
          if (fyi < TY || y0 + fyi == n) ++nfb;
          fl = num_flux<D, 1, LIM>(cons_at(x0 + fxi, y0 + fyi - 1), w0,
                               cons_at(x0 + fxi, y0 + fyi), wp1, gamma);
        } else {
          fl = recon_flux_fast<D, 1, LIM>(l, r, gamma, gm1, rgm1);
        }
        fys[f] = fl.rho;
        fys[K::NYF + f] = fl.m[0];
        fys[2 * K::NYF + f] = fl.m[1];
        fys[3 * K::NYF + f] = fl.E;
      }
    }
  }
  __syncthreads();
  if (active) {
    const int ixl = ty * (TX + 1) + tx, iyl = ty * TX + tx;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      double rhs = 0.0;
      rhs = rhs + fxs[m * K::NXF + ixl] * inv_dx;
      rhs = rhs - fxs[m * K::NXF + ixl + 1] * inv_dx;
      rhs = rhs + fys[m * K::NYF + iyl] * inv_dx;
      rhs = rhs - fys[m * K::NYF + iyl + TX] * inv_dx;
      b[m] = b[m] + rhs * sdt;
      a.out[m * cs + own] = b[m];
    }
    if (a.stage == 2 && a.use_cfl) {
      Cons<D> q;
      q.rho = b[0];
      q.m[0] = b[1];
      q.m[1] = b[2];
      q.E = b[3];
      double s, m;
      wave_speeds(primitives(q, gm1), gamma, s, m);
      ssum = fmax(ssum, s);
    }
  }
  if (bad) s_bad = 1;
  if (nfb) atomicAdd(&s_fb, nfb);
  block_max_atomic<K::NT>(wave, red, a.stage == 1 ? a.r.wave_u + a.step : a.r.wave_mid + a.step);
  if (a.stage == 2 && a.use_cfl) block_max_atomic<K::NT>(ssum, red, a.r.smax + a.step + 1);
  if (tid == 0) {
    if (s_bad) raise_error(a);
    if (s_fb) atomicAdd(a.r.fb + a.step, (unsigned long long)s_fb);
  }
}

// --------------------------------------------- CFL sum-speed reduction --
// max over owned cells of sum_a(|v_a|+c) of `q` (the CFL rule's denominator),
// atomically max-reduced into *target. Grid-stride, one atomic per block.
template <int D>
__global__ void __launch_bounds__(256) speed_sum_kernel(const double* q, UGrid g, double gamma,
                                                        unsigned long long* target,
                                                        const int* err) {
  __shared__ double red[8];
  asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory");
  if (err && failed_before(err)) return;
  const long cells = g.plane * g.nzl;
  const long cs = g.cs;
  const double gm1 = gamma - 1.0;
  double best = 0.0;
  for (long c = blockIdx.x * (long)blockDim.x + threadIdx.x; c < cells;
       c += (long)gridDim.x * blockDim.x) {
    const long off = (c / g.plane + 2) * g.zs + c % g.plane;  // skip the low halo planes
    Cons<D> s;
    s.rho = q[off];
    s.m[0] = q[cs + off];
    s.m[1] = q[2 * cs + off];
    if constexpr (D == 3) s.m[2] = q[3 * cs + off];
    s.E = q[(D + 1) * cs + off];
    const Prim<D> w = primitives(s, gm1);
    double sum, m;
    wave_speeds(w, gamma, sum, m);
    best = fmax(best, sum);
  }
  block_max_atomic<256>(best, red, target);
}

// FluxField capture (step.hpp:16-50) of one stage's numerical fluxes on `q`:
// one thread per face, face i along axis a between cells i-1 and i, the
// stencil cells bc-mapped as the stage kernels map them (reflective momentum
// flipped before primitives), muscl_recon + the numerical flux of the
// reconstructed states, or the first-order fallback (scheme.cpp:155-167).
// The same operations as the exact stage kernels, so the same bits. Output:
// per axis an (n_a+1) x n_b x n_c array of FluxVectors (5 doubles; the 2D
// third momentum is +0), x fastest, the axes concatenated.
template <int D, int S>
__global__ void __launch_bounds__(256) flux_capture_kernel(const double* q, UGrid g, double* cap,
                                                           double gamma) {
  const int n = g.n;
  const long per = D == 3 ? (long)(n + 1) * n * n : (long)(n + 1) * n;
  const long total = D * per;
  const double gm1 = gamma - 1.0, rgm1 = 1.0 / gm1;
  const long cs = g.cs, zs = g.zs;
  auto load = [&](int x, int y, int z) {
    bool fx, fy, fz = false;
    const int mx = bc_map(x, n, g.bc[0], g.bc[1], fx);
    long off;
    if constexpr (D == 3) {
      const int my = bc_map(y, n, g.bc[2], g.bc[3], fy);
      const int zl = slab_map(z, g, 2, fz);
      off = (long)zl * zs + (long)my * n + mx;
    } else {
      const int yl = slab_map(y, g, 1, fy);
      off = (long)yl * zs + mx;
    }
    Cons<D> c;
    c.rho = q[off];
    c.m[0] = q[cs + off];
    c.m[1] = q[2 * cs + off];
    if constexpr (D == 3) c.m[2] = q[3 * cs + off];
    c.E = q[(D + 1) * cs + off];
    if (fx) c.m[0] = -c.m[0];
    if (fy) c.m[1] = -c.m[1];
    if (D == 3 && fz) c.m[D - 1] = -c.m[D - 1];
    return c;
  };
  for (long f = blockIdx.x * (long)blockDim.x + threadIdx.x; f < total;
       f += (long)gridDim.x * blockDim.x) {
    const int ax = (int)(f / per);
    const long r = f - ax * per;
    const int fn0 = ax == 0 ? n + 1 : n, fn1 = ax == 1 ? n + 1 : n;
    int p[3];
    p[0] = (int)(r % fn0);
    const long t = r / fn0;
    p[1] = (int)(t % fn1);
    p[2] = D == 3 ? (int)(t / fn1) : 0;
    Cons<D> qs[4];
    Prim<D> ws[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      int c[3] = {p[0], p[1], p[2]};
      c[ax] += s - 2;
      qs[s] = load(c[0], c[1], c[2]);
      ws[s] = primitives(qs[s], gm1);
    }
    Prim<D> l, rr;
    const bool fb = muscl_recon<D, S>(ws[0], ws[1], ws[2], ws[3], l, rr);
    const Cons<D> F = fb ? num_flux<D, S>(qs[1], ws[1], qs[2], ws[2], ax, gamma)
                         : recon_flux_fast<D, S>(l, rr, ax, gamma, gm1, rgm1);
    double* o = cap + 5 * f;
    o[0] = F.rho;
    o[1] = F.m[0];
    o[2] = F.m[1];
    o[3] = D == 3 ? F.m[D - 1] : 0.0;
    o[4] = F.E;
  }
}

}  // namespace af
