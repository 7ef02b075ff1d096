/*
 * af_cases.h — seeded synthetic initial data for the BASELINE.json configs.
 *
 * The reference ships only two fixed cases (lax_liu_6, ellipsoid3d;
 * /root/reference/proj/core/src/cases.cpp:21-102). BASELINE.json asks for
 * *seeded* variants of the same shapes, so this header defines them once and
 * both sides include it: the GPU host library (product) and the oracle
 * harness that drives the compiled reference (oracle/ref_harness.cpp). Both
 * therefore start from identical bytes.
 *
 * Generator: splitmix64, u01 = (x >> 11) * 2^-53. Cell centres follow
 * UniformGrid::center (grid.hpp:112): origin + (idx + 0.5) * dx with
 * dx = extent / 2^level (grid.hpp:98). The conserved state is assembled with
 * the reference's `conserved` operation order (euler.hpp:107-114).
 *
 * Output layout: AoS, 5 doubles per cell (rho, mom0, mom1, mom2, rhoE) —
 * the memory layout of adaptflow::ConservedState (euler.hpp:24-28) —
 * interior cells only, x fastest, then y, then z.
 *
 * Plain C99, header-only (static inline), no dependencies.
 */
#ifndef AF_CASES_H
#define AF_CASES_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

enum af_case_kind {
  AF_CASE_QUADRANTS = 0,       /* cfg1/cfg2: seeded four-quadrant Riemann problem (2D) */
  AF_CASE_QUADRANTS_NOISE = 1, /* cfg3: quadrants + rho*(1 + 0.01*U[-1,1]) per cell (2D) */
  AF_CASE_ELLIPSOID = 2,       /* cfg4: axis-aligned ellipsoid blast, p 10 | 0.1 (3D) */
  AF_CASE_ELLIPSOID_PRATIO = 3, /* cfg5: ellipsoid, p_in/p_out ~ U[10,100], p_out 0.1 (3D) */
  AF_CASE_QUADRANTS_STRESS = 4  /* test-only: quadrants with pressures 10^U[-9,1], rho U[0.01,3],
                                   |v| up to 3 -- drives the reconstruction / predictor
                                   fallbacks the BASELINE configs never reach (2D, position form only) */
};

typedef struct af_rng {
  uint64_t s;
} af_rng;

static inline uint64_t af_rng_next(af_rng* r) {
  uint64_t z = (r->s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline double af_rng_u01(af_rng* r) {
  return (double)(af_rng_next(r) >> 11) * (1.0 / 9007199254740992.0);
}

/* a + (b - a) * u, u in [0, 1) */
static inline double af_rng_uniform(af_rng* r, double a, double b) {
  return a + (b - a) * af_rng_u01(r);
}

/* euler.hpp:107-114 `conserved`, same operation order (no FMA contraction
 * is emitted by gcc -O3 for x86-64 without -mfma; the GPU side is compiled
 * with --fmad=false). */
static inline void af_conserved(double rho, double v0, double v1, double v2, double p,
                                double gamma, double* q) {
  q[0] = rho;
  q[1] = rho * v0;
  q[2] = rho * v1;
  q[3] = rho * v2;
  const double kin = 0.5 * rho * (v0 * v0 + v1 * v1 + v2 * v2);
  q[4] = p / (gamma - 1.0) + kin;
}

/* Parameters drawn from the seed before any per-cell data. */
typedef struct af_case_params {
  /* quadrants: [quadrant][rho, u, v, p]; quadrant = (x>0.5) + 2*(y>0.5) */
  double quad[4][4];
  /* ellipsoid */
  double semi[3];
  double p_in, p_out, rho_in, rho_out;
} af_case_params;

static inline void af_case_draw(int kind, uint64_t seed, af_case_params* cp, af_rng* r) {
  r->s = seed;
  for (int q = 0; q < 4; ++q)
    for (int c = 0; c < 4; ++c) cp->quad[q][c] = 0.0;
  cp->semi[0] = cp->semi[1] = cp->semi[2] = 0.0;
  cp->p_in = 10.0;
  cp->p_out = 0.1;
  cp->rho_in = 1.0;
  cp->rho_out = 0.125;
  if (kind == AF_CASE_QUADRANTS_STRESS) {
    for (int q = 0; q < 4; ++q) {
      cp->quad[q][0] = af_rng_uniform(r, 0.01, 3.0);
      cp->quad[q][1] = af_rng_uniform(r, -3.0, 3.0);
      cp->quad[q][2] = af_rng_uniform(r, -3.0, 3.0);
      double p = 10.0;
      const int e = (int)(af_rng_u01(r) * 11.0);  /* 10^(1-e), e in 0..10 */
      for (int i = 0; i < e; ++i) p = p * 0.1;
      cp->quad[q][3] = p;
    }
  } else if (kind == AF_CASE_QUADRANTS || kind == AF_CASE_QUADRANTS_NOISE) {
    for (int q = 0; q < 4; ++q) {
      cp->quad[q][0] = af_rng_uniform(r, 0.5, 3.0);
      cp->quad[q][1] = af_rng_uniform(r, -1.0, 1.0);
      cp->quad[q][2] = af_rng_uniform(r, -1.0, 1.0);
      cp->quad[q][3] = af_rng_uniform(r, 0.5, 2.0);
    }
  } else {
    for (int a = 0; a < 3; ++a) cp->semi[a] = af_rng_uniform(r, 0.1, 0.3);
    /* cfg5: pressure RATIO p_in/p_out ~ U[10,100] with p_out = 0.1 */
    if (kind == AF_CASE_ELLIPSOID_PRATIO) cp->p_in = cp->p_out * af_rng_uniform(r, 10.0, 100.0);
  }
}

static inline int af_case_dim(int kind) {
  return (kind == AF_CASE_ELLIPSOID || kind == AF_CASE_ELLIPSOID_PRATIO) ? 3 : 2;
}

/*
 * Fills `out` (n^dim cells x 5 doubles, n = 2^level) for the unit square /
 * cube [0,1]^d. Cells with z-index in [z0, z0 + nz) only are written (slab of
 * a decomposed run; pass z0 = 0, nz = n for the whole 3D domain; in 2D the
 * "z" slab is the y range). Noise draws (AF_CASE_QUADRANTS_NOISE) are taken
 * in global x-fastest order, so a slab reproduces the whole-domain bytes.
 * Returns 0 on success, -1 on an invalid argument.
 */
static inline int af_cases_fill(int kind, uint64_t seed, int level, double gamma, int z0,
                               int nz, double* out) {
  if (level < 0 || level > 15) return -1;
  const int dim = af_case_dim(kind);
  const int n = 1 << level;
  if (z0 < 0 || nz < 0 || z0 + nz > n) return -1;
  const double origin = 0.0, extent = 1.0;
  const double dx = extent / (double)n;
  af_case_params cp;
  af_rng r;
  af_case_draw(kind, seed, &cp, &r);
  if (dim == 2) {
    /* noise stream: skip the draws of rows below the slab */
    if (kind == AF_CASE_QUADRANTS_NOISE)
      for (long s = 0; s < (long)z0 * n; ++s) (void)af_rng_next(&r);
    for (int j = z0; j < z0 + nz; ++j) {
      const double y = origin + ((double)j + 0.5) * dx;
      for (int i = 0; i < n; ++i) {
        const double x = origin + ((double)i + 0.5) * dx;
        const int quad = (x > 0.5 ? 1 : 0) + 2 * (y > 0.5 ? 1 : 0);
        double rho = cp.quad[quad][0];
        if (kind == AF_CASE_QUADRANTS_NOISE)
          rho = rho * (1.0 + 0.01 * af_rng_uniform(&r, -1.0, 1.0));
        double* q = out + 5 * ((size_t)(j - z0) * (size_t)n + (size_t)i);
        af_conserved(rho, cp.quad[quad][1], cp.quad[quad][2], 0.0, cp.quad[quad][3], gamma, q);
      }
    }
  } else {
    for (int k = z0; k < z0 + nz; ++k) {
      const double z = origin + ((double)k + 0.5) * dx;
      for (int j = 0; j < n; ++j) {
        const double y = origin + ((double)j + 0.5) * dx;
        for (int i = 0; i < n; ++i) {
          const double x = origin + ((double)i + 0.5) * dx;
          const double ex = (x - 0.5) / cp.semi[0];
          const double ey = (y - 0.5) / cp.semi[1];
          const double ez = (z - 0.5) / cp.semi[2];
          const int inside = (ex * ex + ey * ey + ez * ez) < 1.0;
          double* q =
              out + 5 * (((size_t)(k - z0) * (size_t)n + (size_t)j) * (size_t)n + (size_t)i);
          af_conserved(inside ? cp.rho_in : cp.rho_out, 0.0, 0.0, 0.0,
                       inside ? cp.p_in : cp.p_out, gamma, q);
        }
      }
    }
  }
  return 0;
}

/*
 * The same initial data as a function of position (an AMR hierarchy samples
 * the initial condition at the cell centres of every level): the quadrant or
 * ellipsoid state at (x, y, z) of the unit domain. The per-cell noise of
 * AF_CASE_QUADRANTS_NOISE has no position form: returns -1 for it.
 */
static inline int af_case_point(int kind, const af_case_params* cp, double gamma, double x,
                                double y, double z, double* q) {
  if (kind == AF_CASE_QUADRANTS || kind == AF_CASE_QUADRANTS_STRESS) {
    const int quad = (x > 0.5 ? 1 : 0) + 2 * (y > 0.5 ? 1 : 0);
    af_conserved(cp->quad[quad][0], cp->quad[quad][1], cp->quad[quad][2], 0.0, cp->quad[quad][3],
                 gamma, q);
    return 0;
  }
  if (kind == AF_CASE_ELLIPSOID || kind == AF_CASE_ELLIPSOID_PRATIO) {
    const double ex = (x - 0.5) / cp->semi[0];
    const double ey = (y - 0.5) / cp->semi[1];
    const double ez = (z - 0.5) / cp->semi[2];
    const int inside = (ex * ex + ey * ey + ez * ez) < 1.0;
    af_conserved(inside ? cp->rho_in : cp->rho_out, 0.0, 0.0, 0.0, inside ? cp->p_in : cp->p_out,
                 gamma, q);
    return 0;
  }
  return -1;
}

#ifdef __cplusplus
}
#endif

#endif /* AF_CASES_H */
