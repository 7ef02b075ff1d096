// af_fv3d.cuh — the 3D fused RK2-stage kernel: one launch = one rk2_stage
// (step.cpp:93-109): build_primitives (step.cpp:18-49) + accumulate_rhs
// (step.cpp:57-89) + out = base + rhs*stage_dt.
//
// A CTA owns a TX x TY column of cells and marches along z through a chunk of
// planes. Per plane:
//   * TMA: the conserved values of plane k+3's (TX+4) x (TY+4) halo box (one
//     cp.async.bulk.tensor of 5 x HY x HX doubles, mbarrier completion) land in
//     a staging buffer while plane k is computed; out-of-domain box cells come
//     back as zeros and are replaced by their boundary-condition source
//     (grid.cpp:19-53) when the box is converted;
//   * convert: staging -> primitives (with the reflective momentum flips) in a
//     3-plane ring (planes k, k+1, k+2), the owned cells' positivity test and
//     StepDiag wave speed;
//   * x/y faces: the (TX+1)*TY x-faces and TX*(TY+1) y-faces of plane k are
//     one flat list, 32 consecutive entries per warp unit, dealt evenly over
//     the CTA's NW warps;
//   * z faces: the thread of each column computes the face k+1/2 above its
//     cell. A cell's limited slope along z serves both of its z faces
//     (muscl_recon evaluates the same limiter twice, on the same operands),
//     so the column carries its next l state and last z difference from plane
//     to plane: one new difference and one limiter per variable per face
//     instead of three and two. The 16x15 tile with 8 warps has 511 x/y
//     faces = 16 units (2 per warp) plus one z unit per warp; the mesh's last
//     tile row is partial (its rows beyond the mesh are computed, never
//     stored or counted);
//   * update: each owned cell sums its six faces in the reference order and
//     writes out = base + rhs*dt; the z-face above becomes the next plane's
//     lower face (kept in registers).
// A face on a tile's high x/y edge, or the chunk's first z face, is computed
// by both neighbouring CTAs; its fallback is counted only by one of them, so
// StepDiag.fallbacks counts each face once as accumulate_rhs does.
//
// MODE 0: bit-exact (the reference's operations and association order,
// --fmad=false translation unit). MODE 1: tolerance mode (af_physics.cuh
// *_tol: reciprocal estimates, FMA contraction in af_fv3d_tol.cu).
#pragma once

#include <cuda.h>

#include <type_traits>

#include "af_uniform_kernels.cuh"

namespace af {

template <int TX, int TY, int NW>
struct Fv3dGeom {
  static constexpr int NT = NW * 32;
  static constexpr int NCELL = TX * TY;
  static constexpr int HX = TX + 4, HY = TY + 4, HP = HX * HY;
  static constexpr int SLOT = 5 * HP;
  static constexpr int NXF = (TX + 1) * TY, NYF = TX * (TY + 1);
  // flat x/y face list: x section [0, NXF), y section [YS, YS+NYF); sections
  // start on warp-unit boundaries so no unit mixes axes and every half-warp
  // reads 16 consecutive doubles of a ring row. The x section lists the TX
  // low faces of each row first (x fastest), then the TY high-edge faces.
  // The z faces are not in the list: each column's thread computes its own.
  static constexpr int YS = (NXF + 31) / 32 * 32;
  static constexpr int NF = YS + NYF;
  static constexpr int NU = (NF + 31) / 32;
  static constexpr int HPT = (HP + NT - 1) / NT;
  static constexpr int RING = 3;  // primitive planes k, k+1, k+2
  static constexpr int RAW = (RING * SLOT + 15) / 16 * 16;  // staging, 128-byte aligned
  static constexpr int FLUX = RAW + (SLOT + 15) / 16 * 16;
  static constexpr int OWN = FLUX + (5 * NF + 15) / 16 * 16;  // [2][5][NCELL] base values
  static constexpr int RED = OWN + 2 * 5 * NCELL;
  static constexpr size_t smem_bytes = sizeof(double) * (size_t)(RED + NW);
  static_assert(NCELL <= NT, "one thread per owned cell");
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// the same with the barrier's shared-window address already in a register (the
// conversion reads SR_CgaCtaId, which costs a long-latency S2R per call)
__device__ __forceinline__ void mbar_wait_a(unsigned bar_addr, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITA_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITA_%=;\n"
      "}\n" ::"r"(bar_addr),
      "r"(parity)
      : "memory");
}
// One arrival per warp on a CTA barrier initialised with the warp count: the
// warp's earlier shared-memory accesses are ordered before it (__syncwarp,
// then the elected lane's release), so a thread that has seen the phase
// complete (mbar_wait_a) may read what every warp wrote and overwrite what
// every warp read. Arrive and wait are separate instructions, so a warp keeps
// working between them on whatever does not depend on the other warps.
__device__ __forceinline__ void warp_arrive(unsigned bar_addr, int lane) {
  __syncwarp();
  if (lane == 0)
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar_addr) : "memory");
}
// 4D tiled TMA load (x, y, component, plane) -> shared, completion on `bar`
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, int c3, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

template <int S, int TX, int TY, int NW, int MODE>
__global__ void __launch_bounds__(NW * 32, 2)
    fv3d_tile(StageArgs a, UGrid g, const __grid_constant__ CUtensorMap tm,
              const __grid_constant__ CUtensorMap tb) {
  using K = Fv3dGeom<TX, TY, NW>;
  constexpr int D = 3;
  if (failed_before(a.r.err)) return;  // an earlier stage failed: freeze state
  extern __shared__ __align__(128) double sm[];
  double* ring = sm;              // [4][5][HP] primitives
  double* raw = sm + K::RAW;      // [5][HP] conserved plane in flight (TMA)
  double* flux = sm + K::FLUX;    // [5][NF]
  double* bown = sm + K::OWN;     // [2][5][NCELL] base values of the owned cells (TMA)
  double* red = sm + K::RED;      // [NW]
  __shared__ unsigned long long bar, bbar[2], xb[3];
  __shared__ int s_fb, s_bad;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tx = tid % TX, ty = tid / TX;
  const unsigned bar_a = smem_u32(&bar), bbar_a = smem_u32(&bbar[0]);
  const unsigned x1_a = smem_u32(&xb[0]), x2_a = smem_u32(&xb[1]), y_a = smem_u32(&xb[2]);
  const int n = g.n;
  const int tiles_x = n / TX;
  const int x0 = (blockIdx.x % tiles_x) * TX, y0 = (blockIdx.x / tiles_x) * TY;
  const int zc0 = a.zbeg + blockIdx.y * a.zchunk;
  const int zc1 = min(zc0 + a.zchunk, a.zend);
  const bool owner = tid < K::NCELL && y0 + ty < n;  // an owned cell inside the mesh
  const double gamma = a.gamma, gm1 = a.gm1, inv_dx = a.inv_dx;
  const double rgm1 = 1.0 / gm1;
  const double sdt = a.dt_scale * stage_dt_of(a);
  if (tid == 0) {
    s_fb = 0;
    s_bad = 0;
    mbar_init(&bar, 1);
    mbar_init(&bbar[0], 1);
    mbar_init(&bbar[1], 1);
    for (int i = 0; i < 3; ++i) mbar_init(&xb[i], NW);
    if (a.stage == 1 && blockIdx.x == 0 && blockIdx.y == 0) a.r.dt[a.step] = stage_dt_of(a);
  }
  const double* ev = a.eval;
  const long cs = g.cs, zs = g.zs;
  bool reflective = false;
#pragma unroll
  for (int f = 0; f < 6; ++f) reflective |= g.bc[f] == AF_BC_REFLECTIVE;
  double wave = 0.0, ssum = 0.0;
  int bad = 0, nfb = 0;

  // This thread's halo-box cells idx = tid + t*NT (the cross of the box; the
  // corners are never on an axis stencil): the box index of the cell the
  // boundary condition maps them to (-1: outside the box, read from global
  // memory at the in-plane offset hoff), and the reflective flips (bit 0 x,
  // bit 1 y).
  int hsrc[K::HPT], hoff[K::HPT];
  unsigned hflip = 0, hown = 0;
#pragma unroll
  for (int t = 0; t < K::HPT; ++t) {
    const int idx = tid + t * K::NT;
    hsrc[t] = -2;  // not converted
    hoff[t] = 0;
    if (idx >= K::HP) continue;
    const int ix = idx % K::HX, iy = idx / K::HX;
    const bool cx = ix >= 2 && ix < TX + 2, cy = iy >= 2 && iy < TY + 2;
    if (!cx && !cy) continue;
    bool fx, fy;
    const int mx = bc_map(x0 - 2 + ix, n, g.bc[0], g.bc[1], fx);
    const int my = bc_map(y0 - 2 + iy, n, g.bc[2], g.bc[3], fy);
    const int bx = mx - (x0 - 2), by = my - (y0 - 2);
    hsrc[t] = (bx >= 0 && bx < K::HX && by >= 0 && by < K::HY) ? by * K::HX + bx : -1;
    hoff[t] = my * n + mx;
    hflip |= ((fx ? 1u : 0u) | (fy ? 2u : 0u)) << (2 * t);
    if (cx && cy && y0 - 2 + iy < n) hown |= 1u << t;
  }
  __syncthreads();  // barrier initialised

  unsigned phase = 0;
  auto issue = [&](int gz) {
    if (tid == 0) {
      bool fz;
      const int zl = slab_map(gz, g, 2, fz);
      mbar_expect_tx(&bar, (unsigned)(sizeof(double) * K::SLOT));
      tma_load_4d(raw, &tm, x0 - 2, y0 - 2, 0, zl, &bar);
    }
  };
  // base values of the owned cells of plane gz into buffer gz&1, issued one
  // plane ahead of the update that reads them
  auto issue_base = [&](int gz) {
    if (tid == 0) {
      mbar_expect_tx(&bbar[gz & 1], (unsigned)(sizeof(double) * 5 * K::NCELL));
      tma_load_4d(bown + (gz & 1) * 5 * K::NCELL, &tb, x0, y0, 0, gz - g.zlo + 2, &bbar[gz & 1]);
    }
  };
  unsigned bphase = 0;  // bit j: parity of buffer j's next completion
  auto convert = [&](int gz, int dslot) {
    mbar_wait_a(bar_a, phase);
    phase ^= 1u;
    // planes inside the domain (all but the chunk ends at the boundary) skip
    // the boundary mapping: a CTA-uniform branch
    bool fz = false;
    int zl = gz - g.zlo + 2;
    if ((unsigned)gz >= (unsigned)n) zl = slab_map(gz, g, 2, fz);
    double* dst = ring + dslot;
    const bool own_plane = gz >= zc0 && gz < zc1;
#pragma unroll
    for (int t = 0; t < K::HPT; ++t) {
      if (hsrc[t] == -2) continue;
      const int idx = tid + t * K::NT;
      Cons<D> q;
      if (hsrc[t] >= 0) {
        const int sidx = hsrc[t];
        q.rho = raw[sidx];
        q.m[0] = raw[K::HP + sidx];
        q.m[1] = raw[2 * K::HP + sidx];
        q.m[2] = raw[3 * K::HP + sidx];
        q.E = raw[4 * K::HP + sidx];
      } else {  // periodic wrap outside the box
        const long off = (long)zl * zs + hoff[t];
        q.rho = ev[off];
        q.m[0] = ev[cs + off];
        q.m[1] = ev[2 * cs + off];
        q.m[2] = ev[3 * cs + off];
        q.E = ev[4 * cs + off];
      }
      Prim<D> w;
      if constexpr (MODE == 0) {
        w = primitives(q, gm1);
        if (own_plane && ((hown >> t) & 1u)) {
          if (!cell_ok(q, w)) bad = 1;
          double s, m;
          wave_speeds(w, gamma, s, m);
          wave = fmax(wave, m);
        }
      } else {
        double ir;
        w = primitives_tol(q, gm1, ir);
        if (own_plane && ((hown >> t) & 1u)) {
          if (!cell_ok(q, w)) bad = 1;
          double s, m;
          wave_speeds_tol(w, ir, gamma, s, m);
          wave = wave > m ? wave : m;
        }
      }
      if (reflective) {  // CTA-uniform: no face of the mesh reflects otherwise
        const unsigned fl = hflip >> (2 * t);
        if (fl & 1u) w.v[0] = -w.v[0];
        if (fl & 2u) w.v[1] = -w.v[1];
        if (fz) w.v[2] = -w.v[2];
      }
      dst[idx] = w.rho;
      dst[K::HP + idx] = w.v[0];
      dst[2 * K::HP + idx] = w.v[1];
      dst[3 * K::HP + idx] = w.v[2];
      dst[4 * K::HP + idx] = w.p;
    }
  };
  auto prim_at = [&](int off) {
    Prim<D> w;
    w.rho = ring[off];
    w.v[0] = ring[K::HP + off];
    w.v[1] = ring[2 * K::HP + off];
    w.v[2] = ring[3 * K::HP + off];
    w.p = ring[4 * K::HP + off];
    return w;
  };
  // Conserved state of global cell (x,y,z) of eval (reflective ghosts with
  // their momentum flipped): only read on the rare first-order fallback
  // (scheme.cpp:160-162).
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
  auto slot = [&](int gz) { return ((gz + 6) % K::RING) * K::SLOT; };

  // x/y faces: each warp owns one x unit (warp) and one y unit (NW + warp)
  // of the flat list (a unit lies in one axis section, so the axis is
  // warp-uniform and a compile-time constant in the face body). Every lane
  // runs the body (padding lanes repeat a real face and store nothing), so
  // the rare fallback and fast-path misses take a warp-uniform branch. The
  // per-lane face geometry is fixed for the whole chunk and computed once.
  static_assert(K::NU == 2 * NW, "two x/y face units per warp");
  struct FaceLane {
    int j, fx, fy, o;  // list entry (section-relative), position, ring offset in a slot
    bool real, skip;   // a listed face; the unit lies beyond the mesh (partial tile row)
  };
  const int rows = min(TY, n - y0);  // tile rows inside the mesh
  auto face_lane = [&](auto axc) {
    constexpr int AX = decltype(axc)::value;
    constexpr int SEC = AX == 0 ? 0 : K::YS;
    constexpr int CNT = AX == 0 ? K::NXF : K::NYF;
    const int u = AX == 0 ? warp : NW + warp;
    FaceLane f;
    const int j0 = u * 32 + lane - SEC;
    f.real = j0 < CNT;
    f.j = f.real ? j0 : 0;
    // face position (fx, fy): the face's high-side cell in tile coordinates
    // (x faces: fx in [0, TX], y faces: fy in [0, TY])
    f.fx = AX == 0 ? (f.j < TX * TY ? f.j % TX : TX) : f.j % TX;
    f.fy = AX == 0 ? (f.j < TX * TY ? f.j / TX : f.j - TX * TY) : f.j / TX;
    f.o = AX == 0 ? (f.fy + 2) * K::HX + f.fx : f.fy * K::HX + f.fx + 2;
    const int f0 = u * 32;
    f.skip = rows < TY && (AX == 0 ? (f0 + 32 <= TX * TY && f0 / TX >= rows)
                                   : (f0 - K::YS) / TX > rows);
    return f;
  };
  const FaceLane flx = face_lane(std::integral_constant<int, 0>{});
  const FaceLane fly = face_lane(std::integral_constant<int, 1>{});
  auto face_body = [&](auto axc, const FaceLane& fl, int k, int sk) {
    constexpr int AX = decltype(axc)::value;
    constexpr int SEC = AX == 0 ? 0 : K::YS;
    constexpr int st = AX == 0 ? 1 : K::HX;
    const int fx = fl.fx, fy = fl.fy;
    const int o = sk + fl.o;
    bool fb;
    Cons<D> F;
    if constexpr (MODE == 1 && S == 1) {
      // minmod + AUSM+ in tolerance mode: transverse velocities of the
      // upwind side only
      F = face_flux_lazy_tol<AX>(ring + o, st, K::HP, gamma, rgm1, fb);
    } else if constexpr (MODE == 0 && (S >> 1) == 0) {
      // AUSM+ in exact mode: rho, v_AX and p on both sides (muscl_recon's
      // operations), the transverse velocities on the upwind side only
      constexpr int LIM = S & 1;
      Prim<D> l, r;
      auto both = [&](int blk, double& lv, double& rv) {
        const double* q = ring + o + blk * K::HP;
        const double c0 = q[0], c1 = q[st], c2 = q[2 * st], c3 = q[3 * st];
        lv = c1 + 0.5 * limiter<LIM>(c1 - c0, c2 - c1);
        rv = c2 - 0.5 * limiter<LIM>(c2 - c1, c3 - c2);
      };
      both(0, l.rho, r.rho);
      both(4, l.p, r.p);
      both(1 + AX, l.v[AX], r.v[AX]);
      fb = !physical(l) || !physical(r);
      bool ok = true;
      F = ausm_plus_lazy<D, AX, FastOps>(
          l, r, gamma, gm1, rgm1,
          [&](bool up_l, int a) {
            const double* q = ring + o + (1 + a) * K::HP + (up_l ? 0 : st);
            const double c0 = q[0], c1 = q[st], c2 = q[2 * st];
            const double h = 0.5 * limiter<LIM>(c1 - c0, c2 - c1);
            return up_l ? c1 + h : c1 - h;
          },
          ok);
      if (!__all_sync(0xffffffffu, ok)) {  // rare: an operand left the fast path's range
        if (!ok) {
          Prim<D> lf, rf;
          muscl_recon<D, S>(prim_at(o), prim_at(o + st), prim_at(o + 2 * st),
                            prim_at(o + 3 * st), lf, rf);
          F = recon_flux<D, S>(lf, rf, AX, gamma, gm1, rgm1);
        }
      }
    } else {
      Prim<D> l, r;
      if constexpr (MODE == 0)
        fb = muscl_recon<D, S>(prim_at(o), prim_at(o + st), prim_at(o + 2 * st),
                               prim_at(o + 3 * st), l, r);
      else
        fb = muscl_recon_tol<D, S>(prim_at(o), prim_at(o + st), prim_at(o + 2 * st),
                                   prim_at(o + 3 * st), l, r);
      if constexpr (MODE == 0)
        F = recon_flux_fast_warp<D, AX, S>(l, r, gamma, gm1, rgm1);
      else
        F = recon_flux_tol<D, S>(l, r, AX, gamma, gm1, rgm1, rgm1);
    }
    if (__any_sync(0xffffffffu, fb)) {  // rare: first-order fallback (scheme.cpp:160-162)
      if (fb) {
        // the inner cells' conserved states from global memory; their
        // primitives are recomputed exactly as the ring holds them. The
        // fallback is counted by the tile owning the face's high-side cell
        // (the domain's high faces by the tile below them), so each face
        // counts once.
        const int gx = x0 + fx - (AX == 0), gy = y0 + fy - (AX == 1);
        bool cnt;
        if constexpr (AX == 0)
          cnt = (fx < TX || x0 + TX == n) && y0 + fy < n;
        else
          cnt = (fy < TY && y0 + fy < n) || y0 + fy == n;
        if (cnt && fl.real) ++nfb;
        const Cons<D> q0 = cons_at(gx, gy, k);
        const Cons<D> q1 = cons_at(gx + (AX == 0), gy + (AX == 1), k);
        Prim<D> w0, w1;
        if constexpr (MODE == 0) {
          w0 = primitives(q0, gm1);
          w1 = primitives(q1, gm1);
        } else {
          double i0, i1;
          w0 = primitives_tol(q0, gm1, i0);
          w1 = primitives_tol(q1, gm1, i1);
        }
        F = num_flux<D, AX, S>(q0, w0, q1, w1, gamma);
      }
    }
    if (fl.real) {
      const int f = SEC + fl.j;
      flux[f] = F.rho;
      flux[K::NF + f] = F.m[0];
      flux[2 * K::NF + f] = F.m[1];
      flux[3 * K::NF + f] = F.m[2];
      flux[4 * K::NF + f] = F.E;
    }
  };
  auto faces = [&](int k, int sk) {
    if (!flx.skip) face_body(std::integral_constant<int, 0>{}, flx, k, sk);
    if (!fly.skip) face_body(std::integral_constant<int, 1>{}, fly, k, sk);
  };

  // z faces: the thread of column (tx, ty) computes the face k+1/2 above its
  // cell of plane k. Each cell's limited z slope serves both of its z faces
  // (cell_face_states), so the column carries the l state of the next face
  // (zl) and the difference w(k+1) - w(k) (zd) from plane to plane.
  const int oc = (ty + 2) * K::HX + tx + 2;  // the column's cell in a ring plane
  double zl[5], zd[5];
  auto zface = [&](int k, bool first, int s1, int s2) {
    double rr[5], nl[5];
#pragma unroll
    for (int m = 0; m < 5; ++m) {
      const double w1 = ring[s1 + m * K::HP + oc];
      const double w2 = ring[s2 + m * K::HP + oc];
      const double d2 = w2 - w1;
      cell_face_states<S, MODE>(w1, zd[m], d2, rr[m], nl[m]);
      zd[m] = d2;
    }
    Prim<D> l, r;
    l.rho = zl[0];
    l.v[0] = zl[1];
    l.v[1] = zl[2];
    l.v[2] = zl[3];
    l.p = zl[4];
    r.rho = rr[0];
    r.v[0] = rr[1];
    r.v[1] = rr[2];
    r.v[2] = rr[3];
    r.p = rr[4];
#pragma unroll
    for (int m = 0; m < 5; ++m) zl[m] = nl[m];
    const bool fb = !physical(l) || !physical(r);
    Cons<D> F;
    if constexpr (MODE == 0)
      F = recon_flux_fast_warp<D, 2, S>(l, r, gamma, gm1, rgm1);
    else
      F = recon_flux_tol<D, S>(l, r, 2, gamma, gm1, rgm1, rgm1);
    if (__any_sync(0xffffffffu, fb)) {
      if (fb) {
        // counted by the chunk above the face (the chunk's first face by the
        // chunk below it, except at the domain's low boundary)
        if ((!first || zc0 == 0) && owner) ++nfb;
        const Cons<D> q0 = cons_at(x0 + tx, y0 + ty, k);
        const Cons<D> q1 = cons_at(x0 + tx, y0 + ty, k + 1);
        Prim<D> w0, w1;
        if constexpr (MODE == 0) {
          w0 = primitives(q0, gm1);
          w1 = primitives(q1, gm1);
        } else {
          double i0, i1;
          w0 = primitives_tol(q0, gm1, i0);
          w1 = primitives_tol(q1, gm1, i1);
        }
        F = num_flux<D, 2, S>(q0, w0, q1, w1, gamma);
      }
    }
    return F;
  };

  // Prologue: planes zc0-2 .. zc0 converted, zc0+1 in flight; the column's z
  // state starts from the slope of plane zc0-1. Iteration k = zc0-1 computes
  // only the chunk's first z face (zc0-1/2) and keeps it as the first
  // plane's lower face.
  for (int z = zc0 - 2; z < zc0 + 1; ++z) {
    issue(z);
    convert(z, slot(z));
    __syncthreads();
  }
  issue(zc0 + 1);
#pragma unroll
  for (int m = 0; m < 5; ++m) {
    const double w0 = ring[slot(zc0 - 2) + m * K::HP + oc];
    const double w1 = ring[slot(zc0 - 1) + m * K::HP + oc];
    const double w2 = ring[slot(zc0) + m * K::HP + oc];
    double unused;
    zd[m] = w2 - w1;
    cell_face_states<S, MODE>(w1, w1 - w0, zd[m], unused, zl[m]);
  }
  __syncthreads();  // plane zc0-2's slot is read above and refilled with plane zc0+1 next
  const int ixl = ty * TX + tx, ixh = tx + 1 < TX ? ixl + 1 : TX * TY + ty,
            iyl = K::YS + ty * TX + tx;
  double zlo[5];
  const double fdt = inv_dx * sdt;  // tolerance mode: rhs*inv_dx*dt folded

  // ring slots of planes k, k+1, k+2 (rotated each plane) and the owned
  // cell's offset in the slab arrays
  int sk = slot(zc0 - 1), sk1 = slot(zc0), sk2 = slot(zc0 + 1);
  long own = (long)(zc0 - 1 - g.zlo + 2) * zs + (long)(y0 + ty) * n + (x0 + tx);
  // Peeled iteration k = zc0-1: only the chunk's first z face, kept as the
  // first plane's lower face.
  {
    convert(zc0 + 1, sk2);
    __syncthreads();
    if (zc0 + 2 < zc1 + 2) issue(zc0 + 2);
    if (zc0 < zc1) issue_base(zc0);
    const Cons<D> Fz = zface(zc0 - 1, true, sk1, sk2);
    const int t = sk;
    sk = sk1;
    sk1 = sk2;
    sk2 = t;
    zlo[0] = Fz.rho;
    zlo[1] = Fz.m[0];
    zlo[2] = Fz.m[1];
    zlo[3] = Fz.m[2];
    zlo[4] = Fz.E;
    own += zs;
    warp_arrive(x1_a, lane);
  }
  // Per plane, three split barriers (arrive ... wait, one arrival per warp)
  // instead of two __syncthreads, so the uneven conversion passes and the
  // warps' face units overlap:
  //   X1: update(k-1) done    -> flux and base buffers free   (waited before the faces)
  //   X2: convert(k+2) done   -> ring slot k+2 complete, staging free
  //                                                (waited before the z face; warp 0
  //                                                 before it issues the next TMA)
  //   Y:  x/y faces of k done -> fluxes complete              (waited before the update)
  for (int k = zc0; k < zc1; ++k, own += zs) {
    const unsigned par = (unsigned)(k - zc0) & 1u;
    convert(k + 2, sk2);
    warp_arrive(x2_a, lane);
    mbar_wait_a(x1_a, par);
    if (warp == 0) {
      mbar_wait_a(x2_a, par);
      if (k + 3 < zc1 + 2) issue(k + 3);
      // its buffer was last read by the update of plane k-1
      if (k + 1 < zc1) issue_base(k + 1);
    }
    faces(k, sk);
    warp_arrive(y_a, lane);
    if (warp != 0) mbar_wait_a(x2_a, par);
    const Cons<D> Fz = zface(k, false, sk1, sk2);
    {
      const int t = sk;
      sk = sk1;
      sk1 = sk2;
      sk2 = t;
    }
    const double zh[5] = {Fz.rho, Fz.m[0], Fz.m[1], Fz.m[2], Fz.E};
    mbar_wait_a(y_a, par);  // x/y fluxes of plane k complete
    mbar_wait_a(bbar_a + 8u * (k & 1), (bphase >> (k & 1)) & 1u);
    bphase ^= 1u << (k & 1);
    if (owner) {
      double b[5];
#pragma unroll
      for (int m = 0; m < 5; ++m) b[m] = bown[(k & 1) * 5 * K::NCELL + m * K::NCELL + tid];
#pragma unroll
      for (int m = 0; m < 5; ++m) {
        const double* fm = flux + m * K::NF;
        if constexpr (MODE == 0) {
          // rhs in the reference order (step.cpp:80-81): x low, x high, y
          // low, y high, z low, z high; then out = base + rhs*stage_dt
          double rhs = 0.0;
          rhs = rhs + fm[ixl] * inv_dx;
          rhs = rhs - fm[ixh] * inv_dx;
          rhs = rhs + fm[iyl] * inv_dx;
          rhs = rhs - fm[iyl + TX] * inv_dx;
          rhs = rhs + zlo[m] * inv_dx;
          rhs = rhs - zh[m] * inv_dx;
          b[m] = b[m] + rhs * sdt;
        } else {
          const double s = ((fm[ixl] - fm[ixh]) + (fm[iyl] - fm[iyl + TX])) + (zlo[m] - zh[m]);
          b[m] = __fma_rn(s, fdt, b[m]);
        }
        zlo[m] = zh[m];
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
        double s, mx;
        if constexpr (MODE == 0) {
          wave_speeds(primitives(q, gm1), gamma, s, mx);
        } else {
          double ir;
          const Prim<D> w = primitives_tol(q, gm1, ir);
          wave_speeds_tol(w, ir, gamma, s, mx);
        }
        ssum = fmax(ssum, s);
      }
    }
    warp_arrive(x1_a, lane);  // this warp's reads of the fluxes and base values are done
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

}  // namespace af
