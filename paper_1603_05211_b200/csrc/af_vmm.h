// af_vmm.h — driver virtual-memory entry points (reserve / create / map)
// shared by the windowed rank arrays (af_mr_dist.cu) and the sparse brick
// storage (af_mr_storage.cu).
#pragma once

#include <cuda.h>

#include <string>

#include "af_internal.h"

namespace af {

// Driver-API virtual memory entry points, resolved through the runtime
// (cudaGetDriverEntryPoint) so the library does not link libcuda and still
// loads on a machine without a driver (the CPU test suite).
struct VmmApi {
  decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
  decltype(&cuMemAddressReserve) reserve = nullptr;
  decltype(&cuMemCreate) create = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemSetAccess) access = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemRelease) release = nullptr;
  decltype(&cuMemAddressFree) free_ = nullptr;
};
inline const VmmApi& vmm() {
  static VmmApi api = [] {
    VmmApi a;
    auto get = [](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      AF_CUDA(cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q));
      if (q != cudaDriverEntryPointSuccess || !*fn)
        throw Error(AF_E_CUDA, std::string("driver entry point missing: ") + name);
    };
    get("cuMemGetAllocationGranularity", reinterpret_cast<void**>(&a.granularity));
    get("cuMemAddressReserve", reinterpret_cast<void**>(&a.reserve));
    get("cuMemCreate", reinterpret_cast<void**>(&a.create));
    get("cuMemMap", reinterpret_cast<void**>(&a.map));
    get("cuMemSetAccess", reinterpret_cast<void**>(&a.access));
    get("cuMemUnmap", reinterpret_cast<void**>(&a.unmap));
    get("cuMemRelease", reinterpret_cast<void**>(&a.release));
    get("cuMemAddressFree", reinterpret_cast<void**>(&a.free_));
    return a;
  }();
  return api;
}
inline void check_cu(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS)
    throw Error(AF_E_CUDA, std::string(what) + ": driver error " + std::to_string((int)r));
}

}  // namespace af
