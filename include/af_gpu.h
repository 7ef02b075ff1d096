/*
 * af_gpu.h — C ABI of libafgpu, the B200-native (sm_100a) implementation of
 * the adaptflow MR/FV compressible-Euler hot path.
 *
 * This is the drop-in boundary: the reference's C++ entry points stay, and
 * their bodies call these functions (INTEGRATION.md shows the shim). Every
 * function returns af_status; no exception crosses the boundary. On error,
 * af_last_error() returns a record from which the host shim rethrows the
 * reference's exception type with the reference's message.
 *
 * Reference interfaces replaced (paths under /root/reference/proj/core):
 *   af_uniform_*          BlockData + fill_ghosts + step_block / rk2_stage
 *                         (grid.hpp:15-68,128; step.hpp:62-64,77-79) as driven
 *                         by run_uniform (unigrid.hpp:24-26, unigrid.cpp:33-47)
 *   af_step_diag          StepDiag (step.hpp:52-55)
 *   af_error              NonPhysicalState / RegisterMismatch (errors.hpp:18-21,69-72)
 *   af_case_fill          init_case (cases.cpp:125-135) for the seeded BASELINE
 *                         configs (the reference has no seeded cases)
 *
 * Data layout at the boundary: AoS, 5 doubles per cell (rho, mom0, mom1,
 * mom2, rhoE) = adaptflow::ConservedState (euler.hpp:24-28), interior cells
 * only, x fastest. In 2D mom2 is written as +0 (the reference keeps it
 * identically zero).
 *
 * Streams: calls are ordered on the context's stream (af_*_set_stream, default
 * a private non-blocking stream). Functions that return host-visible results
 * synchronise that stream; the rest are asynchronous and graph-capturable.
 */
#ifndef AF_GPU_H
#define AF_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AF_ABI_VERSION 1

typedef enum af_status {
  AF_OK = 0,
  AF_E_NONPHYSICAL = 1,       /* adaptflow::NonPhysicalState */
  AF_E_REGISTER_MISMATCH = 2, /* adaptflow::RegisterMismatch */
  AF_E_CONFIG = 3,            /* adaptflow::ConfigError */
  AF_E_LEVEL_MISMATCH = 4,    /* adaptflow::LevelMismatch */
  AF_E_CUDA = 5,              /* CUDA runtime failure (no reference equivalent) */
  AF_E_NCCL = 6,              /* NCCL failure */
  AF_E_ARGUMENT = 7,          /* invalid argument / null pointer */
  AF_E_UNSUPPORTED = 8,       /* option outside the hot path (e.g. AUSMDV) */
  AF_E_INTERNAL = 9,          /* internal invariant check failed (debug switches) */
  AF_E_IO = 10,               /* adaptflow::IoError (errors.hpp:38-41) */
  AF_E_DOMAIN = 11            /* adaptflow::DivisionDomain (errors.hpp:49-52) */
} af_status;

enum { AF_BC_OUTFLOW = 0, AF_BC_PERIODIC = 1, AF_BC_REFLECTIVE = 2 }; /* BcKind grid.hpp:70 */
enum { AF_FLUX_AUSM_PLUS = 0, AF_FLUX_AUSMDV = 1 };                    /* FluxKind scheme.hpp:16 */
enum { AF_LIMITER_VAN_ALBADA = 0, AF_LIMITER_MINMOD = 1 };            /* LimiterKind scheme.hpp:17 */
enum { AF_INTEGRATOR_RK2 = 0, AF_INTEGRATOR_MUSCL_HANCOCK = 1 };      /* IntegratorKind scheme.hpp:18 */

/* Geometry, gas and scheme of one solver instance (UniformGrid grid.hpp:90-123,
 * GasModel euler.hpp:17-19, SchemeConfig scheme.hpp:23-40, BoundaryCondition
 * grid.hpp:74-86). */
typedef struct af_config {
  int dim;         /* 2 or 3 */
  int level;       /* cells per axis n = 2^level */
  double origin;   /* domain [origin, origin+extent]^dim */
  double extent;
  double gamma;    /* 1.4 */
  int bc[6];       /* face 2*axis+side, AF_BC_* */
  int flux;        /* AF_FLUX_AUSM_PLUS */
  int limiter;     /* AF_LIMITER_* */
  int integrator;  /* AF_INTEGRATOR_RK2 */
  int device;      /* CUDA device ordinal */
} af_config;

/* StepDiag (step.hpp:52-55) */
typedef struct af_step_diag {
  double max_wave_speed; /* max over cells, axes and both stages of |v_a| + c */
  long fallbacks;        /* first-order reconstruction fallbacks */
} af_step_diag;

/* Aggregate of a multi-step run (RunReport fields, metrics.hpp:66-79). */
typedef struct af_run_diag {
  double max_wave_speed; /* max over steps of StepDiag::max_wave_speed */
  double max_cfl;        /* max over steps of max_wave_speed * dt / dx (unigrid.cpp:43) */
  long fallbacks;
  long steps_done;
  double t;              /* simulated time advanced */
} af_run_diag;

/* First-offender record of a failed call. */
typedef struct af_error {
  int status;            /* af_status */
  long step;             /* step index, -1 if none */
  int stage;             /* RK stage 1/2, 0 if none */
  int i, j, k;           /* cell index (reference convention, may be a ghost) */
  int level;             /* MR level, -1 for uniform */
  int is_ghost;
  double rho, p;
  char message[512];     /* the reference's exception text, e.g.
                            "step 7: cell (15,16): rho=0.164652 p=-4.999935" */
} af_error;

const char* af_version(void);
int af_abi_version(void);

/* Seeded synthetic initial data (include/af_cases.h): writes n^(dim-1)*nz
 * cells (slab [z0, z0+nz) of the slab axis) as AoS to host memory `out`. */
af_status af_case_fill(int kind, uint64_t seed, int level, double gamma, int z0, int nz,
                       double* out);

/* ------------------------------------------------------------------ comm -- */
/* Multi-GPU: one process per GPU, NCCL over NVLink/NVSwitch. Rank 0 calls
 * af_comm_unique_id, the caller broadcasts the 128 bytes (e.g. with
 * torch.distributed), every rank calls af_comm_create. */
typedef struct af_comm af_comm;
af_status af_comm_unique_id(unsigned char id[128]);
af_status af_comm_create(const unsigned char id[128], int n_ranks, int rank, int device,
                         af_comm** out);
af_status af_comm_destroy(af_comm* comm);
/* A group of n_ranks communicators for ranks emulated by host threads in one
 * process on one GPU (halo exchanges become device-to-device copies, the
 * reductions a host rendezvous). Each rank's calls must run on its own host
 * thread. Used to test the multi-rank MR path on one GPU. */
af_status af_comm_create_local(int n_ranks, int device, af_comm** comms);

/* --------------------------------------------------------------- uniform -- */
typedef struct af_uniform af_uniform;

/* Creates a uniform-mesh solver. comm == NULL: single GPU, whole domain.
 * Otherwise the slab axis (z in 3D, y in 2D) is split into contiguous slabs,
 * rank r owning [z0, z0+nz) (af_uniform_local_extent); results are bitwise
 * independent of the number of ranks. */
af_status af_uniform_create(const af_config* cfg, af_comm* comm, af_uniform** out);
af_status af_uniform_destroy(af_uniform* u);
af_status af_uniform_set_stream(af_uniform* u, void* cuda_stream);
/* Numerics of the 3D RK2 stage (the reference has one: its own operations).
 * AF_NUMERICS_EXACT (default): the reference's operations in its association
 * order without FMA contraction, bit-identical to step_block (step.cpp:93-109).
 * AF_NUMERICS_TOLERANCE: reciprocal/rsqrt estimates with Newton corrections
 * and FMA contraction; within BASELINE.json's 1e-10 relative L1 per field of
 * the exact result (tests/test_tolerance_gpu.py), not bit-identical. 2D and
 * MUSCL-Hancock steps always run exact. */
enum { AF_NUMERICS_EXACT = 0, AF_NUMERICS_TOLERANCE = 1 };
af_status af_uniform_set_numerics(af_uniform* u, int numerics);
af_status af_uniform_local_extent(const af_uniform* u, int* z0, int* nz);
/* The same split without a solver (host arithmetic, no CUDA call): rank `rank`
 * of n_ranks owns [z0, z0+nz) of the slab axis of a 2^level mesh; the loop it
 * shards is unigrid.cpp:33-47. AF_E_CONFIG when a rank would be empty. */
af_status af_slab_extent(int dim, int level, int n_ranks, int rank, int* z0, int* nz);

/* AoS state transfer of the rank's slab (host or device pointer). */
af_status af_uniform_upload(af_uniform* u, const double* aos);
af_status af_uniform_download(af_uniform* u, double* aos);

/* step_block (step.hpp:77-79) for RK2: one step of size dt. diag may be
 * NULL (then the call is asynchronous). */
af_status af_uniform_step(af_uniform* u, double dt, af_step_diag* diag);

/* rk2_stage (step.hpp:62-64, step.cpp:93-109): out = base + stage_dt * rhs(eval)
 * for AoS states of this solver's mesh (cells x 5 doubles, host or device
 * pointers; eval's ghosts are the configured boundary conditions, as after
 * fill_ghosts, grid.cpp:9-62). out may alias base or eval. capture
 * (nullable, host or device): the stage's numerical fluxes in the layout of
 * FluxField (step.hpp:16-50) — per axis a, (n_a+1) x n_b x n_c FluxVectors
 * of 5 doubles (rho, mom[3], rhoE; the 2D mom[2] is +0), face i along a
 * between cells i-1 and i, x fastest, the axes concatenated — the seam the
 * AMR refluxing captures through (amr_hierarchy.cpp:476,488). Replaces the
 * solver's state. Single-rank solvers; capture needs exact numerics
 * (AF_E_UNSUPPORTED otherwise). A non-physical eval raises AF_E_NONPHYSICAL
 * with the reference's text ("cell (i,j[,k])[ (ghost)]: rho=... p=..."). */
af_status af_uniform_rk2_stage(af_uniform* u, const double* base, const double* eval,
                               double* out, double stage_dt, double* capture,
                               af_step_diag* diag);

/* n_steps steps entirely on the device. cfl > 0: dt_s = cfl*dx / max over
 * cells of sum_a(|v_a|+c) of the state at the start of step s (computed on
 * the device, no host round trip); else dt = fixed_dt (unigrid.cpp:20).
 * dt_hist (host, n_steps doubles) and diag may be NULL. Both non-NULL
 * outputs synchronise. With both NULL the call is asynchronous (errors are
 * then reported by the next synchronising call). */
af_status af_uniform_run(af_uniform* u, long n_steps, double cfl, double fixed_dt,
                         double* dt_hist, af_run_diag* diag);

/* Max over cells of sum_a(|v_a|+c) of the current state (synchronises). */
af_status af_uniform_speed_sum(af_uniform* u, double* smax);

/* Synchronises and reports any pending asynchronous error. */
af_status af_uniform_sync(af_uniform* u);

af_status af_uniform_last_error(const af_uniform* u, af_error* err);

/* Number of libafgpu kernels launched by this solver since creation. */
af_status af_uniform_kernel_launches(const af_uniform* u, long* count);

/* Local emulation of an n-rank slab decomposition on ONE GPU: creates the n
 * rank solvers (rank r owns the slab af_uniform_local_extent reports), and
 * runs them in lockstep on rank 0's stream. Halos move by device-to-device
 * copies and the CFL maximum is reduced over the ranks' records, so
 * everything per rank is the multi-GPU code path except the NCCL transport.
 * Used to check that results are bitwise independent of the rank count. */
af_status af_uniform_create_group(const af_config* cfg, int n_ranks, af_uniform** ranks);
af_status af_uniform_run_group(af_uniform** ranks, int n_ranks, long n_steps, double cfl,
                               double fixed_dt, double* dt_hist, af_run_diag* diag);

/* -------------------------------------------------------------------- MR -- */
/* Adaptive multiresolution solver: MRTree (mr_tree.hpp:57-196) + MRSolver
 * (mr_solver.hpp:15-58) + the run_mr loop (mr_solver.hpp:78-79), on per-level
 * dense grids in HBM. Global (MR) and local (MRLT) time stepping. */
typedef struct af_mr af_mr;

/* MROptions (mr_solver.hpp:65-74) plus the level-dependent threshold and the
 * coarsest-leaf-level knob BASELINE.json asks for. */
typedef struct af_mr_options {
  double eps;              /* MROptions::epsilon (refine >= eps, coarsen < eps) */
  const double* eps_level; /* nullable; eps_level[l] = threshold for details whose
                              children are at level l (size level+1); copied */
  int min_leaf_level;      /* MRTree::set_min_leaf_level (mr_tree.hpp:78) */
  int local_time;          /* MROptions::local_time */
  int lt_gap;              /* MROptions::local_time_level_gap (default 3) */
  int storage;             /* AF_MR_STORAGE_* (0 = dense per-level grids) */
  int brick_shift;         /* bricks of 2^brick_shift cells per axis (0: 6) */
} af_mr_options;

/* Storage of the per-level value arrays (the reference's node map,
 * mr_tree.hpp:195). DENSE: every level a row-major 2^l-per-axis grid.
 * BRICKS (3D): levels finer than the brick stored brick after brick, still
 * fully allocated (the layout on its own). SPARSE (3D, brick_shift 6): the
 * brick layout with a 2 MiB page behind a brick of a value component only
 * while the tree reaches it (needed set from the band lists, re-mapped at every
 * refine); memory follows the tree instead of the finest volume. Results are
 * bit-identical across the three (tests/test_mr_storage_gpu.py). One rank. */
enum { AF_MR_STORAGE_DENSE = 0, AF_MR_STORAGE_BRICKS = 1, AF_MR_STORAGE_SPARSE = 2 };

/* Per macro cycle record (RunReport cells/leaves_per_step, mr_solver.cpp:369-374). */
typedef struct af_mr_cycle {
  long leaves;   /* leaf_count() after refine */
  long nodes;    /* node_count() incl. virtual leaves */
  long sub;      /* finest steps in this cycle (LT), 1 for MR */
  int top;       /* LT top level (L for MR) */
  double dt;     /* finest-level step size dt_L */
  long updates;  /* leaf-cell RK-stage updates actually performed in the cycle:
                    2 * sum_l leaves_l * max(1, 2^(l - top)) */
} af_mr_cycle;

af_status af_mr_create(const af_config* cfg, const af_mr_options* opt, af_mr** out);
/* One rank of a spatially decomposed tree: the last axis
 * (y in 2D, z in 3D) is split into slabs of rows from a partition level up;
 * every call is collective over the ranks of `comm`. Leaf keys, counts and
 * to_uniform rows refer to this rank's slab (af_mr_local_rows); cycle records,
 * dt and the run diagnostics are global. */
af_status af_mr_create_dist(const af_config* cfg, const af_mr_options* opt, af_comm* comm,
                            af_mr** out);
/* Rows [lo, hi) of the last axis at `level` that this rank owns. */
/* Numerics of the MR stage (AF_NUMERICS_EXACT default, bit-identical to the
 * reference). AF_NUMERICS_TOLERANCE runs the 2D full-tile stage kernel with
 * the uniform tolerance physics (reciprocal estimates, FMA): within 1e-10
 * relative L1 per field of the exact run with the same leaf sets
 * (tests/test_mr_tolerance_gpu.py); every other MR kernel stays exact. */
af_status af_mr_set_numerics(af_mr* m, int numerics);
af_status af_mr_local_rows(const af_mr* m, int level, int* lo, int* hi);
/* Device bytes of the tree's per-cell arrays: now, the peak so far, and what
 * the same tree takes as dense per-level grids (any argument may be null). */
af_status af_mr_memory(const af_mr* m, unsigned long long* now, unsigned long long* peak,
                       unsigned long long* dense);
af_status af_mr_destroy(af_mr* m);
af_status af_mr_set_stream(af_mr* m, void* cuda_stream);
/* from_uniform(level-L AoS data, 0, bc), norms, min leaf level, coarsen(eps)
 * (mr_tree.cpp:29-71, mr_solver.cpp:406-410). */
af_status af_mr_build(af_mr* m, const double* aos);
/* MRTree::refine (mr_tree.cpp:361-402); top >= 0 applies the LT buffer
 * radii of mr_solver.cpp:358-362 for that top level. */
af_status af_mr_refine(af_mr* m, int top);
/* MRTree::refine(double eps, const std::vector<int>& buffer_radius_per_level)
 * (mr_tree.hpp:141, mr_tree.cpp:361-402): threshold eps at every level (the
 * instance's level table is not used), and the split set dilated by
 * buffer[l] same-level leaves (Chebyshev radius) at level l; n = 0 (no
 * buffer) dilates nothing. Distributed instances reject radii above their
 * halo depth (AF_E_CONFIG). */
af_status af_mr_refine_buffer(af_mr* m, double eps, const int* buffer_radius_per_level, int n);
af_status af_mr_add_virtual_leaves(af_mr* m);
af_status af_mr_remove_virtual_leaves(af_mr* m);
af_status af_mr_coarsen(af_mr* m);
af_status af_mr_evolve_global(af_mr* m, double dt, af_step_diag* diag);
af_status af_mr_advance_local(af_mr* m, int top, double t, double dt, af_step_diag* diag);
/* The run_mr cycle loop (mr_solver.cpp:318-400) for n_steps finest steps;
 * cfl > 0 selects dt_L = cfl*dx_L / max_leaves sum_a(|v_a|+c) per cycle.
 * cycles (capacity max_cycles) and diag may be NULL. */
af_status af_mr_run(af_mr* m, long n_steps, double cfl, double fixed_dt, af_mr_cycle* cycles,
                    long max_cycles, af_run_diag* diag);
af_status af_mr_counts(af_mr* m, long* leaves, long* nodes, long* internals);
/* MRSolver::max_cfl() / fallbacks() (mr_solver.hpp): accumulated over every
 * evolve_global / advance_local / run since af_mr_build (either may be NULL). */
af_status af_mr_solver_stats(af_mr* m, double* max_cfl, long* fallbacks);
af_status af_mr_coarsest_leaf_level(af_mr* m, int* level);
/* Sorted pack_key (mr_tree.hpp:26-30) of every leaf; *n: capacity in, count out. */
af_status af_mr_leaf_keys(af_mr* m, uint64_t* keys, size_t* n);
/* MRTree::to_uniform(level) (mr_tree.cpp:608-621) as AoS. */
af_status af_mr_to_uniform(af_mr* m, int level, double* aos);
/* detail() of every node at `level` (NaN where the node is not internal). */
af_status af_mr_details(af_mr* m, int level, double* out);
/* Stage-kernel timing (CUDA events around every stage's kernel launches on
 * the solver stream): enable, then read the accumulated device time, the
 * number of stage-kernel launches and of leaf-cell stage updates. */
af_status af_mr_profile(af_mr* m, int enable);
af_status af_mr_stage_stats(af_mr* m, double* ms, long* launches, long* updates);
af_status af_mr_last_error(const af_mr* m, af_error* err);
af_status af_mr_kernel_launches(const af_mr* m, long* count);

/* ------------------------------------------- formats and compare path -- */
/* (SURVEY.md §8(f) "next" #2-3). Cell arrays use the ABI's AoS layout:
 * 5 doubles per cell (rho, mom0, mom1, mom2, rhoE; mom2 = 0 in 2D), x fastest.
 * Pointers may be host or device memory. */
typedef struct af_snapshot_header {
  int dim;
  int level;
  double gamma, time, origin, extent;
} af_snapshot_header;
/* write_snapshot (snapshot.cpp:29-59): AFSN v1, little endian. */
af_status af_snapshot_write(const char* path, const af_snapshot_header* h, const double* aos);
/* read_snapshot (snapshot.cpp:61-104). aos == NULL reads the header only;
 * otherwise aos holds 2^(dim*level) cells. */
af_status af_snapshot_read(const char* path, af_snapshot_header* h, double* aos);
/* restrict_to_level (grid.cpp:64-93) on the device: fine (level fine_level)
 * -> out (level target), bit-exact. */
af_status af_restrict_to_level(int dim, int fine_level, int target, const double* fine,
                               double* out);
/* l1_error (metrics.cpp:134-148): per component sum |sol - restrict(ref)| *
 * cell volume, on the device (summation order differs from the reference's
 * sequential loop: agreement to round-off, not bitwise). */
af_status af_l1_error(int dim, int level, double extent, const double* sol, int ref_level,
                      const double* ref, double out[5]);
/* MRTree::dump (mr_tree.cpp:623-641) of the device tree (this rank's nodes):
 * *len in = capacity of buf, out = bytes needed including the terminating 0. */
af_status af_mr_dump(af_mr* m, char* buf, size_t* len);

/* Paper §3 rates (metrics.cpp:91-132): rates(adaptive, fv, n_c) from the
 * RunReport fields they read (sum_cells / sum_leaves = the accumulated
 * cells_per_step / leaves_per_step, l1_rho = l1.rho). Host arithmetic in the
 * reference's operation order; its DivisionDomain texts as AF_E_DOMAIN
 * (errors via af_uniform_last_error(NULL, ...)). */
typedef struct af_run_summary {
  double wall_seconds;
  double sum_cells;
  double sum_leaves;
  long n_steps;
  double l1_rho;
} af_run_summary;
typedef struct af_rates {
  double cpu_compression, memory_compression, mesh_compression, perturbation, overhead;
} af_rates;
af_status af_rates_compute(const af_run_summary* adaptive, const af_run_summary* fv, double n_c,
                           af_rates* out);

/* ------------------------------------------------------- AMR patch path -- */
/* Block-structured patch hierarchy with factor-2 refinement, the paper's
 * comparison method: PatchHierarchy (amr.hpp:123-242,
 * amr_hierarchy.cpp), flag_cells and cluster (amr.hpp:100-111,
 * amr_cluster.cpp) and the run_amr cycle (amr_solver.hpp:34-35,
 * amr_solver.cpp). af_config.level is the base mesh exponent (level l has
 * 2^(level + l) cells per axis); flux/limiter/integrator select the scheme
 * update_level steps with (MUSCL-Hancock or the two-stage RK2). Patch data
 * stay on the device; box lists and level times live on the host; the
 * clustering runs on the host on the downloaded flag mask. Results are
 * bit-identical to the reference (tests/test_amr_gpu.py). */
typedef struct af_amr af_amr;

/* AmrOptions (amr.hpp:113-120) */
typedef struct af_amr_options {
  double eps_rho;            /* scaled-gradient thresholds (flag_cells) */
  double eps_p;
  double cluster_efficiency; /* minimum flagged/total of a box */
  int time_refine;           /* 1: halve dt per level (AMRLT) */
  int flux_correction;       /* 1: conservative coarse-fine flux replacement */
  int max_levels;            /* refinement levels above the base mesh */
} af_amr_options;

/* The initial condition PatchHierarchy::initialize takes (amr.hpp:146):
 * writes the conserved state (rho, mom[3], rhoE) at a cell centre. Called on
 * the host for the cells of every new patch. */
typedef void (*af_amr_ic)(double x, double y, double z, double* q5, void* user);

af_status af_amr_create(const af_config* cfg, const af_amr_options* opt, af_amr** out);
af_status af_amr_destroy(af_amr* h);
/* initialize (amr_hierarchy.cpp:107-131) */
af_status af_amr_initialize(af_amr* h, af_amr_ic ic, void* user);
/* initialize with the seeded case of include/af_cases.h sampled at the cell
 * centres (af_case_point; the quadrant and ellipsoid kinds) */
af_status af_amr_initialize_case(af_amr* h, int kind, uint64_t seed, double gamma);
/* sync_ghosts / remesh / update_level / average_down / flux_correct
 * (amr.hpp:148-175). update_level synchronises when diag is non-NULL. */
af_status af_amr_sync_ghosts(af_amr* h, int level, double tau);
af_status af_amr_remesh(af_amr* h, int level);
af_status af_amr_update_level(af_amr* h, int level, double dt, af_step_diag* diag);
af_status af_amr_average_down(af_amr* h, int level);
af_status af_amr_flux_correct(af_amr* h, int level);
/* run_amr's cycle loop (amr_solver.cpp:24-60,107-131) after initialize:
 * n_steps finest-level steps of size dt_finest (a multiple of 2^max_levels
 * when time-refined, ConfigError otherwise); cells_per_step/leaves_per_step
 * (n_steps entries, nullable) = RunReport's samples; diag: max_cfl, fallbacks. */
af_status af_amr_run(af_amr* h, long n_steps, double dt_finest, long* cells_per_step,
                     long* leaves_per_step, af_run_diag* diag);
af_status af_amr_n_levels(const af_amr* h, int* n);
af_status af_amr_level_info(const af_amr* h, int level, int* n_patches, long* cells, double* t,
                            double* t_old);
/* the level's boxes, 6 ints each (lo[3], hi[3]), in patch order */
af_status af_amr_boxes(const af_amr* h, int level, int* boxes6, int capacity);
/* Patch payloads of a level, patch after patch, AoS x fastest: ghost = 0 the
 * interiors, 2 the blocks with their ghost layers as each patch holds them
 * (Patch::data, amr.hpp:115-118); old = 1: Patch::data_old. aos: host or device. */
af_status af_amr_patch_data_cells(const af_amr* h, int level, int ghost, long* cells);
af_status af_amr_patch_data(af_amr* h, int level, int ghost, int old, double* aos);
/* assemble_level (amr_hierarchy.cpp:600-616): AF_E_LEVEL_MISMATCH unless the
 * level covers the domain */
af_status af_amr_assemble_level(af_amr* h, int level, double* aos);
/* total_conserved (amr_hierarchy.cpp:561-581); device tree sums, so equal to
 * the reference's sequential sums to round-off, not bitwise */
af_status af_amr_total_conserved(af_amr* h, double out5[5]);
/* l1_error_amr (amr.hpp:244-245, amr_hierarchy.cpp:631-656): per component the
 * sum over the composite mesh of |patch - restrict(ref)| * cell volume; ref is
 * a uniform solution at ref_level (AoS, host or device). Device tree sums
 * (round-off agreement). AF_E_LEVEL_MISMATCH when ref is coarser than a level. */
af_status af_amr_l1_error(af_amr* h, int ref_level, const double* ref_aos, double out5[5]);
af_status af_amr_counts(const af_amr* h, long* total_cells, long* composite_cells);
af_status af_amr_properly_nested(af_amr* h, int* nested);
/* dump_boxes (amr_hierarchy.cpp:618-629); the text stays valid until the next call */
af_status af_amr_dump_boxes(af_amr* h, const char** text);
af_status af_amr_last_error(const af_amr* h, af_error* err);
af_status af_amr_kernel_launches(const af_amr* h, long* count);
/* patch-cell stage updates performed by every update_level so far (cells of
 * the level x 1 for MUSCL-Hancock, x 2 for RK2): the bench metric's numerator */
af_status af_amr_cell_updates(const af_amr* h, long* updates);
/* Stepping-kernel timing (CUDA events on the solver stream around the
 * primitives/predictor/faces/update kernels of every update_level): enable,
 * then read the accumulated device time, kernel launches and cell updates. */
af_status af_amr_profile(af_amr* h, int enable);
af_status af_amr_stage_stats(af_amr* h, double* ms, long* launches, long* updates);
/* host wall time spent inside remesh (flags, clustering, rebuild; it
 * synchronises for the masks) and the number of remesh calls so far */
af_status af_amr_remesh_stats(const af_amr* h, double* seconds, long* calls);
/* cluster (amr.hpp:110-111): flags/allowed are n0*n1*n2 bytes, x fastest
 * (allowed nullable); boxes6 nullable to query the count. Host integer work. */
af_status af_amr_cluster(const unsigned char* flags, const unsigned char* allowed, int dim, int n0,
                         int n1, int n2, double efficiency, int* boxes6, int capacity, int* n_boxes);
/* The same clustering on the device, as remesh runs it (summed-area tables of
 * the masks, breadth-first bisection, one CTA per box; only the box list
 * leaves HBM): host masks of an n x n (x n) level are uploaded first. */
af_status af_amr_cluster_device(const unsigned char* flags, const unsigned char* allowed, int dim,
                                int n, double efficiency, int* boxes6, int capacity, int* n_boxes);

/* Self-check of the inline fast-path division and square root the face
 * fluxes use (CUDA's fast-path sequences with their range tests; see
 * DESIGN.md §3) against IEEE a/b and sqrt on n random operands with binary
 * exponents in [emin, emax] (and [2 emin, 2 emax] for sqrt). out[0] division
 * mismatches, out[1] divisions the range test sends to the IEEE path, out[2]
 * and out[3] the same for sqrt. Not a reference entry point: diagnostics. */
af_status af_check_division(long n, uint64_t seed, int emin, int emax,
                            unsigned long long out[4]);

#ifdef __cplusplus
}
#endif

#endif /* AF_GPU_H */
