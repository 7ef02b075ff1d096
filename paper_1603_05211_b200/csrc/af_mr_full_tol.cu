// af_mr_full_tol.cu — the tolerance-mode instantiations of the full-tile MR
// stage kernel (af_mr_full.cuh, MODE 1). This translation unit is compiled
// with FMA contraction (build.py: --fmad=true), the MR host code without.
#include "af_mr.h"
#include "af_mr_full.cuh"

namespace af {

void mr_full_tol_setup() {
  for (auto fn : {(const void*)mr_stage_full2d<0, 1>, (const void*)mr_stage_full2d<1, 1>,
                  (const void*)mr_stage_full2d<2, 1>, (const void*)mr_stage_full2d<3, 1>})
    AF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)MRFull2::smem_bytes));
}

// One launch (programmatic dependent launch when `pdl`, as every MR kernel).
void mr_full_tol_launch(int sch, dim3 grid, cudaStream_t st, bool pdl, const MRStageArgs& a,
                        const MRLevels& g, int lcode) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(MRFull2::NT);
  cfg.dynamicSmemBytes = MRFull2::smem_bytes;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  switch (sch) {
    case 0: AF_CUDA(cudaLaunchKernelEx(&cfg, mr_stage_full2d<0, 1>, a, g, lcode)); break;
    case 1: AF_CUDA(cudaLaunchKernelEx(&cfg, mr_stage_full2d<1, 1>, a, g, lcode)); break;
    case 2: AF_CUDA(cudaLaunchKernelEx(&cfg, mr_stage_full2d<2, 1>, a, g, lcode)); break;
    default: AF_CUDA(cudaLaunchKernelEx(&cfg, mr_stage_full2d<3, 1>, a, g, lcode)); break;
  }
}

}  // namespace af
