// af_mr_full.cuh — the MR stage on FULL 2D tiles (sm_100a).
//
// A full tile (mr_tile_flags_all bit 2) is a 32x8 tile of level l whose
// cells and face neighbours are all leaves of l: every face is a plain
// same-level face of MRSolver::stage (mr_solver.cpp:163-193) — no fine
// sub-face average, no flux register, no leaf tests. A near-full tile (bit
// 4) has only leaf cells and no INTERNAL face neighbour: its edge faces may
// border absent cells (virtual leaves over a coarser leaf, read through V
// and the MRLT time interpolation as resolve does), which are still plain
// faces; in a register stage such a face toward an already-advanced coarser
// cell also deposits its fine register share (face_flux_at,
// mr_solver.cpp:147-159), as mr_stage_kernel does. Dense regions of a tree
// (cfg3's finest level is all leaves) are made of them, so they get their own
// kernel, pipelined like the uniform fv3d_tile:
//   * the next tile's halo box (the 36x12 cross of the tile, bc-mapped as
//     map_position, mr_tree.cpp:146-169) and its step-start values are copied
//     into shared memory with cp.async while the current tile is computed
//     (double-buffered), so the gather latency is off the critical path;
//   * convert: box -> primitives (reflective momentum flips; MRLT virtual
//     leaves over an advanced coarser leaf interpolated in time exactly as
//     resolve_at does, mr_solver.cpp:43-50);
//   * faces: the 264 x-faces and 288 y-faces of the tile as one flat list,
//     32 per warp unit, the axis warp-uniform (18 units over 8 warps);
//   * update: each leaf sums its four faces in the reference order and
//     writes out = base + rhs*stage_dt (+ the stage-1 q_old snapshot and the
//     stage-2 positivity check).
// MODE 0: every operation and its order are those of mr_stage_kernel, so the
// two are bit-identical (tests/test_mr_switches_gpu.py compares them); the
// generic kernel handles the other leaf tiles of the same stage. MODE 1
// (tolerance, af_mr_full_tol.cu, FMA contraction): the face physics of the
// uniform tolerance kernels (reciprocal estimates, af_physics.cuh *_tol) and
// a folded update; within 1e-10 relative L1 of the exact run with the same
// leaf sets (tests/test_mr_tolerance_gpu.py).
#pragma once

#include "af_mr_stage.cuh"

namespace af {

struct MRFull2 {
  // 8 warps, one thread per cell (a 9-warp variant that deals the 18 face
  // units two per warp measured 40% slower on B200)
  static constexpr int TX = kTileX2, TY = kTileY2, NCELL = TX * TY, NW = 8, NT = NW * 32, NC = 4;
  static constexpr int HX = TX + 4, HY = TY + 4, HP = HX * HY;
  static constexpr int NXF = (TX + 1) * TY, NYF = TX * (TY + 1);
  static constexpr int YS = (NXF + 31) / 32 * 32, NF = YS + NYF, NU = (NF + 31) / 32;
  static constexpr int HPT = (HP + NT - 1) / NT;
  // shared memory (doubles): raw[2][NC][HP], base[2][NC][NCELL], pr[NC][HP], fl[NC][NF]
  static constexpr int RAW = 0, BASE = 2 * NC * HP, PR = BASE + 2 * NC * NCELL, FL = PR + NC * HP;
  static constexpr int RED = FL + NC * NF;
  static constexpr size_t smem_bytes = sizeof(double) * (size_t)(RED + NW) + NF;
};

template <int S, int MODE = 0>
__global__ void __launch_bounds__(MRFull2::NT, 2)
    mr_stage_full2d(MRStageArgs a, MRLevels g, int lcode) {
  AF_PDL_ENTRY();
  using K = MRFull2;
  constexpr int D = 2, NC = K::NC, TX = K::TX, TY = K::TY;
  if (failed_before(a.err)) return;
  extern __shared__ __align__(16) double sm[];
  double* raw = sm + K::RAW;
  double* bsm = sm + K::BASE;
  double* pr = sm + K::PR;
  double* fl = sm + K::FL;
  double* red = sm + K::RED;
  uint8_t* ffb = reinterpret_cast<uint8_t*>(red + K::NW);
  __shared__ int s_fb, s_bad;
  (void)red;

  const double sdt = a.dt_dev ? a.dt_scale * *a.dt_dev : a.sdt;
  const int step3 = a.step3_dev ? *a.step3_dev : a.step3;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tx = tid % TX, ty = tid / TX;
  const bool owner = tid < K::NCELL;
  const long comp = g.total_cells;
  const double gamma = a.gamma, gm1 = a.gm1;
  const double rgm1 = 1.0 / gm1;
  if (tid == 0) {
    s_fb = 0;
    s_bad = 0;
  }
  int bad = 0, nfb = 0;
  const int ntotal = tile_total(g, lcode, a.ntiles);
  TileWalker walk(g, lcode < 0 ? lcode : -1, a.ntiles);
  double wave = 0.0;
  int wave_l = -1;
  auto flush_wave = [&] {
    if (wave_l < 0) return;
    for (int o = 16; o > 0; o >>= 1) wave = fmax(wave, __shfl_xor_sync(0xffffffffu, wave, o));
    if (lane == 0 && wave > 0.0)
      atomicMax(a.wave + wave_l, (unsigned long long)__double_as_longlong(wave));
    wave = 0.0;
  };
  const double* basesrc = a.snap ? a.eval : a.base;  // stage 1: q_old is eval itself

  // tile `it` of the launch's range -> level, origin (walk: entries increase)
  // near: the tile is near-full, not full (only those deposit register
  // shares); read in register stages only
  auto locate = [&](int it, int& l, int& x0, int& y0, bool& near) {
    const int t = lcode < 0 ? walk.at(g, a.tiles, it, &l) : tile_at(g, lcode, a.tiles, a.ntiles, it, &l);
    const int sx = ilog2i(g.ntx[l]);
    x0 = (t & (g.ntx[l] - 1)) * TX;
    y0 = ((t >> sx) & (g.nty[l] - 1)) * TY;
    near = a.reg_stage && a.tflag && (a.tflag[g.tile_off[l] + t] & 4) == 0;
  };
  auto on_cross = [&](int idx, int& ix, int& iy) {
    ix = idx % K::HX;
    iy = idx / K::HX;
    const bool cx = ix >= 2 && ix < TX + 2, cy = iy >= 2 && iy < TY + 2;
    return idx < K::HP && (cx || cy);
  };
  // cp.async of tile (l, x0, y0) into buffer b: the box cross of eval and the
  // owned cells' step-start values
  auto issue = [&](int l, int x0, int y0, int b) {
    const int n = 1 << l;
    const long off = g.cell_off[l];
    double* rb = raw + b * NC * K::HP;
#pragma unroll
    for (int t = 0; t < K::HPT; ++t) {
      const int idx = tid + t * K::NT;
      int ix, iy;
      if (!on_cross(idx, ix, iy)) continue;
      bool f;
      const int mi = mr_map(x0 - 2 + ix, n, g.bc[0], g.bc[1], f);
      const int mj = mr_map(y0 - 2 + iy, n, g.bc[2], g.bc[3], f);
      const long c = off + (long)mj * n + mi;
#pragma unroll
      for (int m = 0; m < NC; ++m) cp_async8(rb + m * K::HP + idx, a.eval + m * comp + c);
    }
    if (owner) {
      const long own = off + (long)(y0 + ty) * n + (x0 + tx);
#pragma unroll
      for (int m = 0; m < NC; ++m)
        cp_async8(bsm + b * NC * K::NCELL + m * K::NCELL + tid, basesrc + m * comp + own);
    }
  };
  auto P = [&](int ix, int iy) {
    const int idx = iy * K::HX + ix;
    Prim<D> w;
    w.rho = pr[idx];
    w.v[0] = pr[K::HP + idx];
    w.v[1] = pr[2 * K::HP + idx];
    w.p = pr[3 * K::HP + idx];
    return w;
  };

  int l = 0, x0 = 0, y0 = 0;
  bool near = false;
  if ((int)blockIdx.x < ntotal) {
    locate(blockIdx.x, l, x0, y0, near);
    issue(l, x0, y0, 0);
  }
  cp_async_commit();
  int k = 0;
  for (int it = blockIdx.x; it < ntotal; it += gridDim.x, ++k) {
    const int b = k & 1;
    const int cl = l, cx0 = x0, cy0 = y0;  // this tile
    const bool cnear = near;
    const int nit = it + (int)gridDim.x;
    if (nit < ntotal) {
      locate(nit, l, x0, y0, near);
      issue(l, x0, y0, b ^ 1);
    }
    cp_async_commit();
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    __syncthreads();  // this tile's copies from every thread have landed
    const int n = 1 << cl;
    const long off = g.cell_off[cl];
    const double inv_dx = g.inv_dx[cl];
    if (cl != wave_l) {
      flush_wave();
      wave_l = cl;
    }
    // convert the box to primitives (resolve_at's flips and MRLT interpolation)
    const double* rb = raw + b * NC * K::HP;
    const bool interp = cl >= 1 && cl - 1 < a.lo;
#pragma unroll
    for (int t = 0; t < K::HPT; ++t) {
      const int idx = tid + t * K::NT;
      int ix, iy;
      if (!on_cross(idx, ix, iy)) continue;
      Cons<D> q;
      q.rho = rb[idx];
      q.m[0] = rb[K::HP + idx];
      q.m[1] = rb[2 * K::HP + idx];
      q.E = rb[3 * K::HP + idx];
      bool fi, fj;
      const int mi = mr_map(cx0 - 2 + ix, n, g.bc[0], g.bc[1], fi);
      const int mj = mr_map(cy0 - 2 + iy, n, g.bc[2], g.bc[3], fj);
      if (interp) {
        const long c = off + (long)mj * n + mi;
        const long pc = g.cell_off[cl - 1] + (long)(mj >> 1) * (n >> 1) + (mi >> 1);
        if (a.vmark[pc] && a.st[c] == ST_ABSENT) {
          const double th = a.theta[cl - 1], om = 1.0 - th;
          q.rho = a.vq_old[c] * om + q.rho * th;
          q.m[0] = a.vq_old[comp + c] * om + q.m[0] * th;
          q.m[1] = a.vq_old[2 * comp + c] * om + q.m[1] * th;
          q.E = a.vq_old[3 * comp + c] * om + q.E * th;
        }
      }
      if (fi) q.m[0] = -q.m[0];
      if (fj) q.m[1] = -q.m[1];
      Prim<D> w;
      if constexpr (MODE == 0) {
        w = primitives(q, gm1);
      } else {
        double ir;
        w = primitives_tol(q, gm1, ir);
      }
      pr[idx] = w.rho;
      pr[K::HP + idx] = w.v[0];
      pr[2 * K::HP + idx] = w.v[1];
      pr[3 * K::HP + idx] = w.p;
    }
    __syncthreads();
    // pass-1 checks of this thread's leaf (mr_solver.cpp:171-178)
    if (owner) {
      const Prim<D> w = P(tx + 2, ty + 2);
      Cons<D> q;
      q.rho = w.rho;
      if (!cell_ok(q, w)) bad = 1;
      double s, m;
      if constexpr (MODE == 0) {
        wave_speeds(w, gamma, s, m);
      } else {
        wave_speeds_tol(w, rcp_tol(w.rho), gamma, s, m);
      }
      wave = fmax(wave, m);
    }
    auto cons_at = [&](int x, int y) { return resolve_at<D>(a.eval, comp, g, cl, x, y, 0, &a); };
    auto face = [&](auto axc, int u) {
      constexpr int AX = decltype(axc)::value;
      constexpr int SEC = AX == 0 ? 0 : K::YS;
      constexpr int CNT = AX == 0 ? K::NXF : K::NYF;
      const int j0 = u * 32 + lane - SEC;
      const bool real = j0 < CNT;
      const int j = real ? j0 : 0;
      // (fx, fy): the face's high-side cell in tile coordinates
      const int fx = AX == 0 ? (j < TX * TY ? j % TX : TX) : j % TX;
      const int fy = AX == 0 ? (j < TX * TY ? j / TX : j - TX * TY) : j / TX;
      // the face's first stencil cell in the primitive box and the stencil stride
      constexpr int st = AX == 0 ? 1 : K::HX;
      const int o = AX == 0 ? (fy + 2) * K::HX + fx : fy * K::HX + fx + 2;
      auto Pc = [&](int c) {  // stencil cell c = 0..3
        const int idx = o + c * st;
        Prim<D> w;
        w.rho = pr[idx];
        w.v[0] = pr[K::HP + idx];
        w.v[1] = pr[2 * K::HP + idx];
        w.p = pr[3 * K::HP + idx];
        return w;
      };
      bool fb;
      Cons<D> F;
      if constexpr (MODE == 0 && (S >> 1) == 0) {
        // AUSM+ in exact mode: rho, v_AX and p on both sides (muscl_recon's
        // operations), the transverse velocity on the upwind side only
        // (ausm_plus_lazy, bit-identical to the eager form)
        constexpr int LIM = S & 1;
        Prim<D> lft, rgt;
        auto both = [&](int blk, double& lv, double& rv) {
          const double* q = pr + blk * K::HP + o;
          const double c0 = q[0], c1 = q[st], c2 = q[2 * st], c3 = q[3 * st];
          lv = c1 + 0.5 * limiter<LIM>(c1 - c0, c2 - c1);
          rv = c2 - 0.5 * limiter<LIM>(c2 - c1, c3 - c2);
        };
        both(0, lft.rho, rgt.rho);
        both(3, lft.p, rgt.p);
        both(1 + AX, lft.v[AX], rgt.v[AX]);
        fb = !physical(lft) || !physical(rgt);
        bool ok = true;
        F = ausm_plus_lazy<D, AX, FastOps>(
            lft, rgt, gamma, gm1, rgm1,
            [&](bool up_l, int a) {
              const double* q = pr + (1 + a) * K::HP + o + (up_l ? 0 : st);
              const double c0 = q[0], c1 = q[st], c2 = q[2 * st];
              const double h = 0.5 * limiter<LIM>(c1 - c0, c2 - c1);
              return up_l ? c1 + h : c1 - h;
            },
            ok);
        if (!__all_sync(0xffffffffu, ok)) {  // rare: an operand left the fast path's range
          if (!ok) {
            Prim<D> lf, rf;
            muscl_recon<D, S>(Pc(0), Pc(1), Pc(2), Pc(3), lf, rf);
            F = recon_flux<D, S>(lf, rf, AX, gamma, gm1, rgm1);
          }
        }
      } else {
        Prim<D> lft, rgt;
        if constexpr (MODE == 0) {
          fb = muscl_recon<D, S>(Pc(0), Pc(1), Pc(2), Pc(3), lft, rgt);
          F = recon_flux_fast_warp<D, AX, S>(lft, rgt, gamma, gm1, rgm1);
        } else {
          fb = muscl_recon_tol<D, S>(Pc(0), Pc(1), Pc(2), Pc(3), lft, rgt);
          F = recon_flux_tol<D, S>(lft, rgt, AX, gamma, gm1, rgm1, rgm1);
        }
      }
      if (__any_sync(0xffffffffu, fb)) {
        if (fb) {
          const int gx = cx0 + fx, gy = cy0 + fy;
          F = num_flux<D, AX, S>(cons_at(gx - (AX == 0), gy - (AX == 1)), Pc(1), cons_at(gx, gy),
                                 Pc(2), gamma);
        }
      }
      if (real) {
        const int f = SEC + j;
        fl[f] = F.rho;
        fl[K::NF + f] = F.m[0];
        fl[2 * K::NF + f] = F.m[1];
        fl[3 * K::NF + f] = F.E;
        ffb[f] = (uint8_t)fb;
      }
    };
    for (int u = warp; u < K::NU; u += K::NW) {
      if (u * 32 < K::YS)
        face(std::integral_constant<int, 0>{}, u);
      else
        face(std::integral_constant<int, 1>{}, u);
    }
    // the step-start values leave their buffer before the barrier, so the
    // next iteration may refill it without a fourth barrier per tile
    double base[NC];
    if (owner) {
#pragma unroll
      for (int m = 0; m < NC; ++m) base[m] = bsm[b * NC * K::NCELL + m * K::NCELL + tid];
    }
    __syncthreads();  // fluxes complete; every read of this tile's buffers done
    if (owner) {
      const long own = off + (long)(cy0 + ty) * n + (cx0 + tx);
      const int fxl = ty * TX + tx, fxh = tx + 1 < TX ? fxl + 1 : TX * TY + ty;
      const int fyl = K::YS + ty * TX + tx, fyh = fyl + TX;
      double o[NC];
#pragma unroll
      for (int m = 0; m < NC; ++m) {
        const double* fm = fl + m * K::NF;
        const double base0 = base[m];
        if (a.snap) a.snap[m * comp + own] = base0;
        if constexpr (MODE == 0) {
          double rhs = 0.0;
          rhs = rhs + fm[fxl] * inv_dx;
          rhs = rhs - fm[fxh] * inv_dx;
          rhs = rhs + fm[fyl] * inv_dx;
          rhs = rhs - fm[fyh] * inv_dx;
          o[m] = base0 + rhs * sdt;
        } else {
          o[m] = __fma_rn((fm[fxl] - fm[fxh]) + (fm[fyl] - fm[fyh]), inv_dx * sdt, base0);
        }
        a.out[m * comp + own] = o[m];
      }
      nfb += ffb[fxl] + ffb[fxh] + ffb[fyl] + ffb[fyh];
      // near-full tiles in a register stage: the fine share of an edge face
      // whose outside cell is absent under an advanced (marked) coarser leaf
      if (cnear && (tx == 0 || tx == TX - 1 || ty == 0 || ty == TY - 1) && cl >= 1 &&
          cl - 1 < a.lo) {
        const int c[2] = {cx0 + tx, cy0 + ty};
#pragma unroll
        for (int ax = 0; ax < 2; ++ax)
#pragma unroll
          for (int dir = -1; dir <= 1; dir += 2) {
            const int t_in = ax == 0 ? tx + dir : ty + dir;
            if (t_in >= 0 && t_in < (ax == 0 ? TX : TY)) continue;  // inside: a leaf
            int p[2] = {c[0], c[1]};
            p[ax] += dir;
            bool flp;
            p[ax] = mr_map(p[ax], n, g.bc[2 * ax], g.bc[2 * ax + 1], flp);
            if (a.st[off + (long)p[1] * n + p[0]] != ST_ABSENT) continue;
            const int pn = n >> 1;
            const long pc = g.cell_off[cl - 1] + (long)(p[1] >> 1) * pn + (p[0] >> 1);
            if (!a.vmark[pc]) continue;
            const int R = reg_index(a.regbase, a.regmask, pc, ax * 2 + (dir > 0 ? 0 : 1));
            if (R >= 0) {
              const int t = c[1 - ax] & 1;  // sub-face slot (ascending pack_key order)
              const double w = a.step_dt * a.share;
              double* dst = a.regf + (((long)R * 2 + a.sub) * 2 + t) * NC;
              const int fi = ax == 0 ? (dir < 0 ? fxl : fxh) : (dir < 0 ? fyl : fyh);
#pragma unroll
              for (int m = 0; m < NC; ++m) dst[m] = fl[m * K::NF + fi] * w;
              a.regff[R] = 1;
            } else {
              atomicExch(a.regerr, 1);
            }
          }
      }
      if (a.post_check) {
        Cons<D> q;
        q.rho = o[0];
        q.m[0] = o[1];
        q.m[1] = o[2];
        q.E = o[3];
        if constexpr (MODE == 0) {
          if (!cell_ok(q, primitives(q, gm1))) bad |= 2;
        } else {
          double ir;
          if (!cell_ok(q, primitives_tol(q, gm1, ir))) bad |= 2;
        }
      }
    }
    // (no barrier here: the next iteration's first barrier orders its
    // convert and faces after every thread's update of this tile)
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  flush_wave();
  if (bad) atomicOr(&s_bad, bad);
  if (nfb) atomicAdd(&s_fb, nfb);
  __syncthreads();
  if (tid == 0) {
    if (s_bad) {
      atomicExch(a.err + ((s_bad & 1) ? 0 : 2), 1);
      if (a.post_stops) atomicExch(a.err, 1);
      atomicMin(a.err + 1, step3 + ((s_bad & 1) ? a.stage - 1 : 2));
      atomicCAS(a.err + 3, 0, ((a.lo << 8) | a.hi) + 1);
    }
    if (s_fb) atomicAdd(a.fb, (unsigned long long)s_fb);
  }
}

}  // namespace af
