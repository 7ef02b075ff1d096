/*
 * af_oracle.h — TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * Two CPU implementations of the hot path share this interface:
 *   afref_*  oracle/ref_harness.cpp — the UNMODIFIED reference library
 *            (/root/reference/proj/core, compiled by oracle/Makefile into
 *            oracle/_ref/) driven through its public API, plus the seeded
 *            inputs and the CFL time-step rule the reference lacks.
 *   afo_*    oracle/af_oracle.c — a plain-C restatement of the same
 *            algorithm, each function citing the reference file:line it
 *            follows. Pinned against afref_* by tests/test_oracle_pin.py and
 *            the committed fixtures under tests/golden/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load these libraries.
 */
#ifndef AF_ORACLE_H
#define AF_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct af_oracle_params {
  int dim;       /* 2 or 3 */
  int level;     /* finest level L, n = 2^L cells per axis */
  int bc[6];     /* per face 2*axis+side: 0 outflow, 1 periodic, 2 reflective (grid.hpp:70) */
  int limiter;   /* 0 van Albada, 1 minmod (scheme.hpp:20) */
  int flux;      /* 0 AUSM+, 1 AUSMDV (scheme.hpp:16) */
  double gamma;  /* 1.4 */
  long n_steps;  /* finest-level steps */
  double cfl;    /* > 0: dt = cfl*dx_L / max_leaf sum_a(|v_a|+c) per (macro) step */
  double fixed_dt; /* used when cfl <= 0 (reference semantics, unigrid.cpp:20) */
  /* MR only */
  double eps;               /* scalar threshold (mr_tree.cpp:371,498) */
  const double* eps_level;  /* nullable; eps_level[l] = threshold for details whose
                               CHILDREN are at level l (size level+1) */
  int min_leaf_level;       /* MRTree::set_min_leaf_level (mr_tree.hpp:78) */
  int local_time;           /* 1: MRLT (mr_solver.cpp:325-363) */
  int lt_gap;               /* MROptions::local_time_level_gap (mr_solver.hpp:70) */
  int integrator;           /* 0 RK2, 1 MUSCL-Hancock (scheme.hpp:18); uniform only */
} af_oracle_params;

typedef struct af_oracle_result {
  double max_wave_speed; /* max over steps of StepDiag::max_wave_speed (uniform) */
  double max_cfl;        /* RunReport::max_cfl */
  long fallbacks;        /* RunReport::fallbacks */
  double wall_seconds;   /* steady_clock around the step loop only */
  long n_cycles;         /* MR: macro cycles run; uniform: steps */
  long steps_done;       /* finest-level steps completed */
  int err_kind;          /* 0 ok, 1 NonPhysicalState, 2 RegisterMismatch, 9 other */
  char err[512];         /* exception text, annotated like the reference */
} af_oracle_result;

/*
 * Uniform FV run (unigrid.cpp:7-50 loop with the seeded data and CFL rule).
 * init/out: n^dim * 5 doubles, AoS interior, x fastest. dt_hist: n_steps
 * doubles (nullable). Returns err_kind.
 */
int afref_uniform_run(const af_oracle_params* p, const double* init, double* out,
                      double* dt_hist, af_oracle_result* res);
int afo_uniform_run(const af_oracle_params* p, const double* init, double* out,
                    double* dt_hist, af_oracle_result* res);
/* The reference's rk2_stage (step.hpp:62-64) with FluxField capture (cap
 * nullable; per axis (n_a+1) x n_b x n_c faces of 5 doubles, x fastest). */
int afref_rk2_stage(const af_oracle_params* p, const double* base, const double* eval,
                    double stage_dt, double* out, double* cap, af_oracle_result* res);

/*
 * The uniform 3D run on the window z in [z0, z0+nz) of the n^3 mesh, split
 * into `threads` z-slabs that each call the reference's step_block on their
 * own BlockData (ref_harness.cpp; bench.py's multi-core CPU arm). init: the
 * (nz+4) planes z0-2 .. z0+nz+1 clamped into the mesh, AoS. n_warm untimed
 * steps, then p->n_steps timed ones (res->wall_seconds). out: nz planes
 * (nullable). With z0 = 0, nz = n this is afref_uniform_run bit for bit.
 */
int afref_uniform_window_run(const af_oracle_params* p, int z0, int nz, int threads,
                             long n_warm, const double* init, double* out,
                             af_oracle_result* res, double* dt_hist);

/*
 * MR / MRLT run (mr_solver.cpp:318-400 loop). out: to_uniform(L) of the final
 * tree (n^dim*5). leaf_keys: sorted pack_key leaves of the final tree
 * (capacity *n_leaves on entry, count on exit; nullable). per_cycle: for each
 * macro cycle {leaves, nodes incl. virtual, sub, top, leaf-stage updates} as 5 longs (capacity
 * max_cycles; nullable). dt_hist: dt_L per cycle (nullable).
 */
int afref_mr_run(const af_oracle_params* p, const double* init, double* out,
                 uint64_t* leaf_keys, long* n_leaves, long* per_cycle, long max_cycles,
                 double* dt_hist, af_oracle_result* res);
int afo_mr_run(const af_oracle_params* p, const double* init, double* out,
               uint64_t* leaf_keys, long* n_leaves, long* per_cycle, long max_cycles,
               double* dt_hist, af_oracle_result* res);

/* Writes MRTree::dump() (mr_tree.cpp:623-641) of the final tree of the last
 * afref_mr_run / afo_mr_run call to `path`. Returns 0 on success. */
int afref_mr_last_dump(const char* path);
int afo_mr_last_dump(const char* path);

/* include/af_cases.h af_case_fill, exported for Python tests */
int afo_case_fill(int kind, uint64_t seed, int level, double gamma, int z0, int nz,
                  double* out);

/* ---- AMR patch path (amr.hpp, amr_solver.hpp), reference side ---- */
typedef struct af_amr_ref_params {
  int dim;
  int level;      /* finest resolution level */
  int base_exp;   /* base mesh exponent (max_levels = level - base_exp) */
  int bc[6];
  int limiter, flux, integrator;
  double gamma;
  long n_steps;      /* finest-level steps */
  double dt_finest;
  double eps_rho, eps_p, efficiency;
  int time_refine, flux_correction;
  int case_kind;     /* include/af_cases.h kind sampled by af_case_point */
  uint64_t seed;
  /* 0: the harness loop (PatchHierarchy::initialize with the seeded point
   *    function, then AmrDriver::advance restated on the public methods);
   * 1: the same loop on the built-in case `builtin_name` (its initial_state,
   *    bc and gas; base_exp = amr_base_exp; dt = t_end / n_steps);
   * 2: the reference's own run_amr on that built-in case. 1 and 2 must agree
   *    bit for bit, which pins the restated loop. */
  int mode;
  const char* builtin_name;
} af_amr_ref_params;

/* Runs and keeps the hierarchy for the accessors below. res: max_cfl,
 * fallbacks, err. cells/leaves_per_step: n_steps longs (nullable). */
int afref_amr_run(const af_amr_ref_params* p, long* cells_per_step, long* leaves_per_step,
                  af_oracle_result* res);
int afref_amr_n_levels(void);
int afref_amr_n_patches(int level);
int afref_amr_boxes(int level, int* boxes6);
double afref_amr_time(int level, int old);
/* patch after patch, AoS x fastest; ghost 0 interiors / 2 blocks with ghosts; old: data_old */
long afref_amr_patch_data(int level, int ghost, int old, double* aos);
int afref_amr_total_conserved(double* out5);
int afref_amr_dump_boxes(char* buf, long cap);
/* l1_error_amr (amr.hpp:244-245) of the kept hierarchy; 1 + err text on an exception */
int afref_amr_l1_error(int ref_level, const double* ref_aos, double* out5, char* err, int errlen);
/* cluster (amr.hpp:110-111) on an n x n (x n) mask; returns the box count */
int afref_cluster(const unsigned char* flags, const unsigned char* allowed, int dim, int n,
                  double efficiency, int* boxes6, int capacity);

#ifdef __cplusplus
}
#endif

#endif /* AF_ORACLE_H */
