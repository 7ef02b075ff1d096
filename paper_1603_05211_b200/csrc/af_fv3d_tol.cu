// af_fv3d_tol.cu — the tolerance-mode instantiations of the 3D stage kernel
// (af_fv3d.cuh, MODE 1). This translation unit is compiled with FMA
// contraction (build.py: --fmad=true), every other one without.
#include "af_fv3d.cuh"
#include "af_uniform.h"

namespace af {

namespace {
constexpr int kT3 = 16, kT3Y = 15, kW3 = 8;
using Geo3 = Fv3dGeom<kT3, kT3Y, kW3>;
}  // namespace

void fv3d_tol_setup() {
  for (auto fn : {(const void*)fv3d_tile<0, kT3, kT3Y, kW3, 1>, (const void*)fv3d_tile<1, kT3, kT3Y, kW3, 1>,
                  (const void*)fv3d_tile<2, kT3, kT3Y, kW3, 1>, (const void*)fv3d_tile<3, kT3, kT3Y, kW3, 1>})
    AF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)Geo3::smem_bytes));
}

void fv3d_tol_launch(int sch, dim3 grid, cudaStream_t st, const StageArgs& a, const UGrid& g,
                     const CUtensorMap& tm, const CUtensorMap& tb) {
#define AF_T3(S) fv3d_tile<S, kT3, kT3Y, kW3, 1><<<grid, Geo3::NT, Geo3::smem_bytes, st>>>(a, g, tm, tb)
  switch (sch) {
    case 0: AF_T3(0); break;
    case 1: AF_T3(1); break;
    case 2: AF_T3(2); break;
    default: AF_T3(3); break;
  }
#undef AF_T3
}

}  // namespace af
