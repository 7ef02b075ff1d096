/*
 * af_oracle.c — TEST INFRASTRUCTURE ONLY: plain-C restatement of the
 * reference hot path (the parity checker; never linked into the product).
 *
 * Follows /root/reference/proj/core (cited as file:line below) operation by
 * operation so results are bit-identical to the reference's own CPU build
 * (compile without FMA contraction: -ffp-contract=off). Pinned against the
 * compiled reference (oracle/_ref, afref_*) by tests/test_oracle_pin.py and
 * against the committed fixtures in tests/golden/.
 *
 * Uniform path : euler.hpp, scheme.cpp, grid.cpp, step.cpp, unigrid.cpp
 * MR path      : mr_tree.cpp, mr_solver.cpp (af_oracle_mr.c)
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "af_oracle.h"
#include "af_oracle_core.h"

/* ---------------------------------------------------------------- grid -- */

/* BlockData (grid.hpp:15-68): ghosted AoS block, x fastest, gz = 0 in 2D. */
typedef struct {
  int dim, g, gz, n[3];
  long sy, sz, total;
  afo_state* d;
} afo_block;

static void blk_init(afo_block* b, int dim, int n, int g) {
  b->dim = dim;
  b->g = g;
  b->gz = dim == 3 ? g : 0;
  b->n[0] = n;
  b->n[1] = n;
  b->n[2] = dim == 3 ? n : 1;
  b->sy = n + 2 * g;
  b->sz = b->sy * (n + 2 * g);
  b->total = b->sz * (b->n[2] + 2 * b->gz);
  b->d = (afo_state*)calloc((size_t)b->total, sizeof(afo_state));
}

static inline long blk_index(const afo_block* b, int i, int j, int k) {
  return (i + b->g) + (long)(j + b->g) * b->sy + (long)(k + b->gz) * b->sz;
}

static inline long blk_stride(const afo_block* b, int axis) {
  return axis == 0 ? 1 : axis == 1 ? b->sy : b->sz;
}

/* grid.cpp:11-56 fill_axis: ghosts of one axis over the already-filled
 * extent of the earlier axes (corner consistency). */
static void fill_axis(afo_block* b, int axis, const int* bc) {
  const int g = axis == 2 ? b->gz : b->g;
  if (g == 0) return;
  const int n = b->n[axis];
  int lo[3] = {0, 0, 0}, hi[3] = {b->n[0], b->n[1], b->n[2]};
  for (int a = 0; a < 3; ++a) {
    if (a == axis) continue;
    const int ga = a < axis ? (a == 2 ? b->gz : b->g) : 0;
    lo[a] = -ga;
    hi[a] = b->n[a] + ga;
  }
  for (int side = 0; side < 2; ++side) {
    const int kind = bc[2 * axis + side];
    for (int layer = 1; layer <= g; ++layer) {
      const int gi = side == 0 ? -layer : n - 1 + layer;
      int src = 0, flip = 0;
      if (kind == 0) {
        src = side == 0 ? 0 : n - 1;
      } else if (kind == 1) {
        src = side == 0 ? n - layer : layer - 1;
      } else {
        src = side == 0 ? layer - 1 : n - layer;
        flip = 1;
      }
      int c[3];
      for (c[2] = (axis == 2 ? 0 : lo[2]); c[2] < (axis == 2 ? 1 : hi[2]); ++c[2])
        for (c[1] = (axis == 1 ? 0 : lo[1]); c[1] < (axis == 1 ? 1 : hi[1]); ++c[1])
          for (c[0] = (axis == 0 ? 0 : lo[0]); c[0] < (axis == 0 ? 1 : hi[0]); ++c[0]) {
            int dst[3] = {c[0], c[1], c[2]}, from[3] = {c[0], c[1], c[2]};
            dst[axis] = gi;
            from[axis] = src;
            afo_state q = b->d[blk_index(b, from[0], from[1], from[2])];
            if (flip) q.v[1 + axis] = -q.v[1 + axis];
            b->d[blk_index(b, dst[0], dst[1], dst[2])] = q;
          }
    }
  }
}

/* grid.cpp:58-62 */
static void fill_ghosts(afo_block* b, const int* bc) {
  for (int axis = 0; axis < b->dim; ++axis) fill_axis(b, axis, bc);
}

/* ---------------------------------------------------------------- step -- */

static void cell_str(char* buf, size_t len, int i, int j, int k, int dim) {
  if (dim == 3)
    snprintf(buf, len, "(%d,%d,%d)", i, j, k);
  else
    snprintf(buf, len, "(%d,%d)", i, j);
}

/* step.cpp:18-49 build_primitives. Returns 0, or 1 with `err` set. */
static int build_primitives(const afo_block* b, double gamma, afo_prim* w, double* max_speed,
                            char* err, size_t errlen) {
  const int g = b->g, gz = b->gz;
  double ms = 0.0;
  for (int k = -gz; k < b->n[2] + gz; ++k)
    for (int j = -g; j < b->n[1] + g; ++j)
      for (int i = -g; i < b->n[0] + g; ++i) {
        const long idx = blk_index(b, i, j, k);
        const afo_state* q = &b->d[idx];
        const afo_prim p = afo_primitives_unguarded(q, gamma);
        if (!(q->v[0] > AFO_POS_TOL) || !afo_physical(&p)) {
          const int ghost = i < 0 || i >= b->n[0] || j < 0 || j >= b->n[1] || k < 0 ||
                            k >= b->n[2];
          char cs[64];
          cell_str(cs, sizeof cs, i, j, k, b->dim);
          snprintf(err, errlen, "cell %s%s: rho=%f p=%f", cs, ghost ? " (ghost)" : "",
                   q->v[0], p.p);
          return 1;
        }
        w[idx] = p;
        const int interior =
            i >= 0 && i < b->n[0] && j >= 0 && j < b->n[1] && k >= 0 && k < b->n[2];
        if (interior) {
          const double c = afo_sound_speed(&p, gamma);
          for (int a = 0; a < b->dim; ++a) {
            const double s = fabs(p.v[a]) + c;
            ms = ms > s ? ms : s; /* std::max(ms, s) */
          }
        }
      }
  *max_speed = ms;
  return 0;
}

/* step.cpp:57-89 accumulate_rhs */
static void accumulate_rhs(const afo_block* e, const afo_prim* w, double dx, int limiter, int flux,
                           double gamma, afo_state* rhs, long* fallbacks) {
  const double inv_dx = 1.0 / dx;
  memset(rhs, 0, sizeof(afo_state) * (size_t)e->total);
  const afo_state* q = e->d;
  for (int axis = 0; axis < e->dim; ++axis) {
    const long s = blk_stride(e, axis);
    const int t1 = axis == 0 ? 1 : 0;
    const int t2 = axis == 2 ? 1 : 2;
    int c[3];
    for (c[t2] = 0; c[t2] < e->n[t2]; ++c[t2])
      for (c[t1] = 0; c[t1] < e->n[t1]; ++c[t1]) {
        c[axis] = 0;
        const long base = blk_index(e, c[0], c[1], c[2]);
        for (int f = 0; f <= e->n[axis]; ++f) {
          const long cell = base + (long)f * s;
          const afo_state fx =
              afo_face_flux_w(&q[cell - s], &q[cell], &w[cell - 2 * s], &w[cell - s],
                              &w[cell], &w[cell + s], axis, limiter, flux, gamma, fallbacks);
          for (int m = 0; m < 5; ++m) {
            const double fm = fx.v[m] * inv_dx;
            if (f > 0) rhs[cell - s].v[m] -= fm;
            if (f < e->n[axis]) rhs[cell].v[m] += fm;
          }
        }
      }
  }
}

/* step.cpp:93-109 rk2_stage */
static int rk2_stage(const afo_block* base, const afo_block* eval, afo_block* out, double dx,
                     double stage_dt, int limiter, int flux, double gamma, afo_prim* w, afo_state* rhs,
                     double* max_speed, long* fallbacks, char* err, size_t errlen) {
  if (build_primitives(eval, gamma, w, max_speed, err, errlen)) return 1;
  accumulate_rhs(eval, w, dx, limiter, flux, gamma, rhs, fallbacks);
  for (int k = 0; k < base->n[2]; ++k)
    for (int j = 0; j < base->n[1]; ++j)
      for (int i = 0; i < base->n[0]; ++i) {
        const long idx = blk_index(base, i, j, k);
        for (int m = 0; m < 5; ++m)
          out->d[idx].v[m] = base->d[idx].v[m] + rhs[idx].v[m] * stage_dt;
      }
  return 0;
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* unigrid.cpp:7-50 run_uniform loop, with step.cpp:237-251 step_block (RK2)
 * inlined, the seeded data and the CFL rule of oracle/af_oracle.h. */
int afo_uniform_run(const af_oracle_params* p, const double* init, double* out,
                    double* dt_hist, af_oracle_result* res) {
  memset(res, 0, sizeof(*res));
  if (p->integrator != 0) {
    res->err_kind = 9;
    snprintf(res->err, sizeof res->err, "oracle: only the RK2 integrator is restated");
    return 9;
  }
  const int n = 1 << p->level;
  afo_block u, mid;
  blk_init(&u, p->dim, n, 2);
  blk_init(&mid, p->dim, n, 2);
  afo_prim* w = (afo_prim*)malloc(sizeof(afo_prim) * (size_t)u.total);
  afo_state* rhs = (afo_state*)malloc(sizeof(afo_state) * (size_t)u.total);
  long c = 0;
  for (int k = 0; k < u.n[2]; ++k)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i, ++c)
        for (int m = 0; m < 5; ++m) u.d[blk_index(&u, i, j, k)].v[m] = init[5 * c + m];
  const double dx = 1.0 / (double)n; /* grid.hpp:98 extent / 2^level */
  double wall = 0.0;
  char err[400];
  for (long step = 0; step < p->n_steps; ++step) {
    const double t0 = now_s();
    double dt = p->fixed_dt;
    if (p->cfl > 0.0) {
      double smax = 0.0;
      for (int k = 0; k < u.n[2]; ++k)
        for (int j = 0; j < n; ++j)
          for (int i = 0; i < n; ++i) {
            const double s = afo_speed_sum(&u.d[blk_index(&u, i, j, k)], p->gamma, p->dim);
            smax = smax > s ? smax : s;
          }
      dt = p->cfl * dx / smax;
    }
    if (dt_hist) dt_hist[step] = dt;
    fill_ghosts(&u, p->bc);
    /* step_block: BlockData mid = u; stage(u,u,mid,dt/2); refill(mid);
     * stage(u,mid,u,dt) */
    memcpy(mid.d, u.d, sizeof(afo_state) * (size_t)u.total);
    double s1 = 0.0, s2 = 0.0;
    long fb = 0;
    int bad = rk2_stage(&u, &u, &mid, dx, 0.5 * dt, p->limiter, p->flux, p->gamma, w, rhs, &s1, &fb, err,
                        sizeof err);
    if (!bad) {
      fill_ghosts(&mid, p->bc);
      bad = rk2_stage(&u, &mid, &u, dx, dt, p->limiter, p->flux, p->gamma, w, rhs, &s2, &fb, err,
                      sizeof err);
    }
    if (bad) {
      res->err_kind = 1;
      snprintf(res->err, sizeof res->err, "step %ld: %s", step, err);
      break;
    }
    const double ms = s1 > s2 ? s1 : s2;
    res->max_wave_speed = res->max_wave_speed > ms ? res->max_wave_speed : ms;
    const double cfl = ms * dt / dx;
    res->max_cfl = res->max_cfl > cfl ? res->max_cfl : cfl;
    res->fallbacks += fb;
    wall += now_s() - t0;
    res->steps_done = step + 1;
  }
  res->n_cycles = res->steps_done;
  res->wall_seconds = wall;
  if (!res->err_kind) {
    c = 0;
    for (int k = 0; k < u.n[2]; ++k)
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i, ++c)
          for (int m = 0; m < 5; ++m) out[5 * c + m] = u.d[blk_index(&u, i, j, k)].v[m];
  }
  free(u.d);
  free(mid.d);
  free(w);
  free(rhs);
  return res->err_kind;
}

/* Seeded synthetic inputs (include/af_cases.h), exported for the tests. */
#include "af_cases.h"
int afo_case_fill(int kind, uint64_t seed, int level, double gamma, int z0, int nz,
                  double* out) {
  return af_cases_fill(kind, seed, level, gamma, z0, nz, out);
}
