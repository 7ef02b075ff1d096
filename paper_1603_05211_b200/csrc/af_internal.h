// af_internal.h — host-side shared declarations of libafgpu (not part of the ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "af_gpu.h"

namespace af {

// Typed error carried through the host code and turned into an af_status at
// the C-ABI boundary (no exceptions cross it). Mirrors the reference's
// exception classes (errors.hpp:10-77).
struct Error : std::runtime_error {
  af_status status;
  Error(af_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

// formats and compare path (af_io.cu)
void snapshot_write(const char* path, const af_snapshot_header& h, const double* aos);
void snapshot_read(const char* path, af_snapshot_header* h, double* aos);
void restrict_to_level(int dim, int fine_level, int target, const double* fine, double* out);
void l1_error(int dim, int level, double extent, const double* sol, int ref_level,
              const double* ref, double* out5);

#define AF_CUDA(call)                                                                   \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      throw ::af::Error(AF_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// Device-side per-run records; one slot per step so the run needs no host
// synchronisation (CUDA-graph friendly). Doubles that are max-reduced are
// kept as their IEEE bit patterns: for non-negative values the unsigned
// order equals the numeric order, so atomicMax on the bits is exact.
struct RunRecords {
  unsigned long long* smax;      // [n+1] max over cells of sum_a(|v_a|+c) of u_s (CFL rule)
  unsigned long long* wave_u;    // [n]   StepDiag stage-1 max (|v_a|+c) of u_s
  unsigned long long* wave_mid;  // [n]   StepDiag stage-2 max of mid_s
  unsigned long long* fb;        // [n]   reconstruction fallbacks
  double* dt;                    // [n]   step size used
  int* err;                      // [0] flag, [1] first failing (step*2 + stage-1)
};

// Uniform grid geometry of one rank's slab. Cells are stored as per-plane
// SoA ([plane][component][row][x], so a plane's components are contiguous and
// one halo message per neighbour carries all of them) without x/y ghosts; the slab axis (z in 3D, y in 2D) carries 2 halo planes per side
// for the inter-rank exchange. Physical boundary conditions are folded into
// the stencil index mapping (outflow ghosts of grid.cpp:9-62 are copies of
// the nearest interior cell, so reading the mapped cell is bit-identical).
struct UGrid {
  int dim;
  int n;       // global cells per axis
  int zlo;     // first global index of the slab axis owned by this rank
  int nzl;     // owned extent along the slab axis
  int nranks;
  int bc[6];
  int ncomp;   // stored components: 5 in 3D, 4 in 2D (mom2 == +0 is not stored)
  long plane;  // cells per slab-axis index (n*n in 3D, n in 2D)
  long cs;     // component stride = plane   (layout [zl][m][y][x], zl = z - zlo + 2)
  long zs;     // slab-axis stride = ncomp * plane
  long total;  // elements = zs * (nzl + 4)
};

}  // namespace af
