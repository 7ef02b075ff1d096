// af_mr_storage.cu — block-structured per-level storage of the MR tree:
// dense bricks, mapped to physical memory only where the tree reaches
// (BASELINE.json north_star: "adaptive leaf/ghost bookkeeping rebuilt as
// block-structured, per-level dense bricks with GPU compaction").
//
// The reference keeps only existing nodes (std::unordered_map<NodeKey,MRNode>,
// mr_tree.hpp:195). Here every level is a grid of 2^bsh-per-axis bricks laid
// out brick after brick (MRLevels::bsh, mr_idx), so one brick of one value
// component is one contiguous run of 2^(3 bsh) doubles (2 MiB at bsh = 6, the
// VMM page). Each value array (V, the stage output, the step-start and
// virtual snapshots, the details) reserves its full virtual size once and
// maps a physical page behind a brick only while the brick is NEEDED:
//
//   needed(m) = bricks of level m meeting a band tile of level m, or the
//               children of a band tile of level m-1, each dilated by one
//               tile of level m.
//
// The band (mr_tile_lists_all: tiles within one tile of a tile holding a cell
// whose parent exists) covers every node of a level and every cell whose value
// or prediction any pass reads; one refine creates nodes only as children of
// existing nodes (mr_tree.cpp:361-444), so the children of the level-(m-1)
// band cover every level-m cell the coming cycle can create, predict, read as
// a stencil or gather as a stage halo (two cells) — the next sync, at the
// next refine, follows the tree. Levels of at most 2^bsh cells per axis are
// one brick each and stay mapped. The GPU computes the needed set from the
// band lists it already compacts every cycle (mr_brick_need); the host maps
// and unmaps the difference (cuMemMap / cuMemUnmap of 2 MiB pages) between
// cycles, so every kernel keeps plain global addressing and CUDA graphs stay
// valid. Unmapped memory is never touched: a stray access faults instead of
// reading stale data.
#include <cuda.h>

#include <algorithm>
#include <cstring>

#include "af_mr.h"
#include "af_vmm.h"

namespace af {

namespace {

// Marks the bricks of levels l and l+1 that the band tiles of level l need
// (blockIdx.y = l - bsh): the tile dilated by one tile at level l, its
// children dilated by one tile at level l+1. Periodic axes wrap.
__global__ void mr_brick_need(const int* band, MRLevels g, uint8_t* need) {
  const int l = g.bsh + (int)blockIdx.y;
  if (l > g.L) return;
  const int cnt = g.dcnt[l];
  const int s = g.bsh;
  const int* tl = band + g.tile_off[l];
  const int ntx = g.ntx[l], nty = g.nty[l];
  const int sx = mr_log2(ntx), sy = mr_log2(nty);
  const int T[3] = {kTileX3, kTileY3, kTileZ3};
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < cnt; e += gridDim.x * blockDim.x) {
    const int t = tl[e];
    const int o[3] = {(t & (ntx - 1)) * kTileX3, ((t >> sx) & (nty - 1)) * kTileY3,
                      (t >> (sx + sy)) * kTileZ3};
    for (int m = l; m <= l + 1 && m <= g.L; ++m) {
      if (m <= s) continue;  // one brick, always mapped
      const int f = m - l, n = 1 << m, ls = m - s, nb = 1 << ls;
      const long bo = ((1L << (3 * ls)) - 8) / 7;  // bricks of levels s+1 .. m-1
      int b0[3], b1[3];
      for (int a = 0; a < 3; ++a) {
        const int lo = (o[a] << f) - T[a], hi = ((o[a] + T[a]) << f) + T[a] - 1;
        if (g.bc[2 * a] == AF_BC_PERIODIC) {
          b0[a] = lo >> s;  // arithmetic shift: floor division
          b1[a] = hi >> s;
          if (b1[a] - b0[a] >= nb) b1[a] = b0[a] + nb - 1;
        } else {
          b0[a] = max(lo, 0) >> s;
          b1[a] = min(hi, n - 1) >> s;
        }
      }
      for (int bz = b0[2]; bz <= b1[2]; ++bz)
        for (int by = b0[1]; by <= b1[1]; ++by)
          for (int bx = b0[0]; bx <= b1[0]; ++bx) {
            const int wx = bx & (nb - 1), wy = by & (nb - 1), wz = bz & (nb - 1);
            need[bo + (((long)wz << (2 * ls)) | ((long)wy << ls) | wx)] = 1;
          }
    }
  }
}

}  // namespace

// Storage geometry: brick shift, padded level offsets (every bricked level and
// every component starts on a brick boundary, so a brick is page-aligned).
void MR::storage_setup_(const af_mr_options& o) {
  storage_ = o.storage;
  if (storage_ < AF_MR_STORAGE_DENSE || storage_ > AF_MR_STORAGE_SPARSE)
    throw Error(AF_E_CONFIG, "unknown MR storage mode");
  if (storage_ == AF_MR_STORAGE_DENSE) {
    if (o.brick_shift) throw Error(AF_E_CONFIG, "brick_shift needs brick storage");
    return;
  }
  if (D_ != 3) throw Error(AF_E_UNSUPPORTED, "brick storage is implemented for 3D trees");
  if (dist_) throw Error(AF_E_UNSUPPORTED, "brick storage runs on one rank");
  const int s = o.brick_shift ? o.brick_shift : kBrickShift3;
  if (s < 2 || s > 8) throw Error(AF_E_CONFIG, "brick_shift must be in [2, 8]");
  if (storage_ == AF_MR_STORAGE_SPARSE && s != kBrickShift3)
    throw Error(AF_E_CONFIG, "sparse storage maps 2 MiB bricks (brick_shift 6 in 3D)");
  g_.bsh = s;
  const long bc = 1L << (3 * s);
  long tot = 0;
  for (int l = 0; l <= L_; ++l) {
    if (l > s) tot = (tot + bc - 1) / bc * bc;
    g_.cell_off[l] = tot;
    tot += mr_cells(D_, l);
  }
  tot = (tot + bc - 1) / bc * bc;
  g_.cell_off[L_ + 1] = tot;
  g_.total_cells = tot;
  sp_nbricks_ = L_ > s ? ((1L << (3 * (L_ - s + 1))) - 8) / 7 : 0;
  sp_brick_bytes_ = sizeof(double) * (size_t)bc;
}

// Level and in-level brick index of global brick gb.
int MR::sp_level_(long gb, long* b) const {
  const int s = g_.bsh;
  for (int m = s + 1; m <= L_; ++m) {
    const long bo = ((1L << (3 * (m - s))) - 8) / 7, nbr = 1L << (3 * (m - s));
    if (gb < bo + nbr) {
      *b = gb - bo;
      return m;
    }
  }
  throw Error(AF_E_INTERNAL, "brick index out of range");
}

namespace {
CUmemAllocationProp sp_prop(int device) {
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = device;
  return prop;
}
}  // namespace

// A value array of ncomp components: the whole virtual range reserved, the
// levels up to the brick size (the coarse block) mapped for good.
void* MR::sp_alloc_(int ncomp) {
  const CUmemAllocationProp prop = sp_prop(cfg_.device);
  size_t gran = 0;
  check_cu(vmm().granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED),
           "cuMemGetAllocationGranularity");
  if (sp_brick_bytes_ % gran)
    throw Error(AF_E_UNSUPPORTED, "brick size is not a multiple of the VMM granularity");
  SpArr a;
  a.ncomp = ncomp;
  a.reserved = sizeof(double) * (size_t)ncomp * (size_t)g_.total_cells;
  CUdeviceptr base = 0;
  check_cu(vmm().reserve(&base, a.reserved, sp_brick_bytes_, 0, 0), "cuMemAddressReserve");
  a.base = base;
  CUmemAccessDesc acc{};
  acc.location = prop.location;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  const size_t cb = sizeof(double) * (size_t)g_.cell_off[std::min(L_, g_.bsh) + 1];
  for (int m = 0; m < ncomp; ++m) {
    CUmemGenericAllocationHandle h;
    check_cu(vmm().create(&h, cb, &prop, 0), "cuMemCreate (coarse levels)");
    const CUdeviceptr p = base + sizeof(double) * (size_t)m * g_.total_cells;
    check_cu(vmm().map(p, cb, 0, h, 0), "cuMemMap");
    check_cu(vmm().access(p, cb, &acc, 1), "cuMemSetAccess");
    a.coarse.push_back(h);
  }
  a.coarse_bytes = cb;
  a.bricks.assign(sp_nbricks_ * ncomp, 0);
  sp_.push_back(a);
  return reinterpret_cast<void*>(base);
}

MR::SpArr* MR::sp_find_(const void* p) {
  for (SpArr& a : sp_)
    if (a.base == reinterpret_cast<unsigned long long>(p)) return &a;
  return nullptr;
}

// One physical allocation per component page of the brick (cuMemMap maps a
// whole allocation: its offset argument must be 0).
void MR::sp_map_(SpArr& a, long gb) {
  long b = 0;
  const int m = sp_level_(gb, &b);
  const CUmemAllocationProp prop = sp_prop(cfg_.device);
  CUmemAccessDesc acc{};
  acc.location = prop.location;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  const long cell = g_.cell_off[m] + (b << (3 * g_.bsh));
  for (int c = 0; c < a.ncomp; ++c) {
    CUmemGenericAllocationHandle h;
    const CUresult r = vmm().create(&h, sp_brick_bytes_, &prop, 0);
    if (r == CUDA_ERROR_OUT_OF_MEMORY)
      throw Error(AF_E_CUDA, "sparse MR storage: out of device memory mapping a brick of level " +
                                 std::to_string(m));
    check_cu(r, "cuMemCreate (brick)");
    const CUdeviceptr p = a.base + sizeof(double) * ((size_t)c * g_.total_cells + cell);
    check_cu(vmm().map(p, sp_brick_bytes_, 0, h, 0), "cuMemMap (brick)");
    check_cu(vmm().access(p, sp_brick_bytes_, &acc, 1), "cuMemSetAccess (brick)");
    AF_CUDA(cudaMemsetAsync(reinterpret_cast<void*>(p), 0, sp_brick_bytes_, stream_));
    a.bricks[gb * a.ncomp + c] = h;
  }
  ++a.mapped;
  sp_now_ += sp_brick_bytes_ * a.ncomp;
  sp_peak_ = std::max(sp_peak_, sp_now_);
}

void MR::sp_unmap_(SpArr& a, long gb) {
  long b = 0;
  const int m = sp_level_(gb, &b);
  const long cell = g_.cell_off[m] + (b << (3 * g_.bsh));
  for (int c = 0; c < a.ncomp; ++c) {
    check_cu(vmm().unmap(a.base + sizeof(double) * ((size_t)c * g_.total_cells + cell),
                         sp_brick_bytes_),
             "cuMemUnmap (brick)");
    check_cu(vmm().release(a.bricks[gb * a.ncomp + c]), "cuMemRelease (brick)");
    a.bricks[gb * a.ncomp + c] = 0;
  }
  --a.mapped;
  sp_now_ -= sp_brick_bytes_ * a.ncomp;
}

// Every brick of the array behind p (build, to_uniform, details: dense passes).
void MR::sp_map_all_(const void* p) {
  SpArr* a = sp_find_(p);
  if (!a) return;
  for (long gb = 0; gb < sp_nbricks_; ++gb)
    if (!a->bricks[gb * a->ncomp]) sp_map_(*a, gb);
}

// Brings every value array's mapping to the needed set of the current band
// lists (maps the new bricks zero-filled, releases the rest).
void MR::sparse_sync_() {
  if (storage_ != AF_MR_STORAGE_SPARSE || !sp_nbricks_) return;
  if (!lists_valid_) build_lists_();
  if (!d_need_) AF_CUDA(cudaMalloc(&d_need_, sp_nbricks_));
  AF_CUDA(cudaMemsetAsync(d_need_, 0, sp_nbricks_, stream_));
  mr_brick_need<<<dim3(64, L_ - g_.bsh + 1), 256, 0, stream_>>>(d_band_, g_, d_need_);
  AF_CUDA(cudaGetLastError());
  ++launches_;
  h_need_.resize(sp_nbricks_);
  AF_CUDA(cudaMemcpyAsync(h_need_.data(), d_need_, sp_nbricks_, cudaMemcpyDeviceToHost, stream_));
  AF_CUDA(cudaStreamSynchronize(stream_));
  for (SpArr& a : sp_)
    for (long gb = 0; gb < sp_nbricks_; ++gb) {
      const bool mapped = a.bricks[gb * a.ncomp] != 0;
      if (h_need_[gb] && !mapped) sp_map_(a, gb);
      else if (!h_need_[gb] && mapped) sp_unmap_(a, gb);
    }
}

void MR::sp_free_all_() {
  for (SpArr& a : sp_) {
    for (long gb = 0; gb < sp_nbricks_; ++gb)
      if (a.bricks[gb * a.ncomp]) sp_unmap_(a, gb);
    for (int c = 0; c < a.ncomp; ++c) {
      vmm().unmap(a.base + sizeof(double) * (size_t)c * g_.total_cells, a.coarse_bytes);
      vmm().release(a.coarse[c]);
    }
    vmm().free_(a.base, a.reserved);
  }
  sp_.clear();
  if (d_need_) cudaFree(d_need_);
  d_need_ = nullptr;
}

// memset / download of the mapped part of a sparse array (levels [lo, hi]).
bool MR::sp_set_(void* p, int value, int lev_lo, int lev_hi) {
  SpArr* a = sp_find_(p);
  if (!a) return false;
  uint8_t* b = static_cast<uint8_t*>(p);
  for (int c = 0; c < a->ncomp; ++c) {
    const size_t cb = (size_t)c * g_.total_cells;
    for (int l = lev_lo; l <= lev_hi; ++l) {
      if (l <= g_.bsh) {
        AF_CUDA(cudaMemsetAsync(b + 8 * (cb + g_.cell_off[l]), value, 8 * mr_cells(D_, l),
                                stream_));
        continue;
      }
      const long bo = ((1L << (3 * (l - g_.bsh))) - 8) / 7, nbr = 1L << (3 * (l - g_.bsh));
      for (long q = 0; q < nbr; ++q)
        if (a->bricks[(bo + q) * a->ncomp])
          AF_CUDA(cudaMemsetAsync(b + 8 * (cb + g_.cell_off[l] + (q << (3 * g_.bsh))), value,
                                  sp_brick_bytes_, stream_));
    }
  }
  return true;
}

bool MR::sp_tohost_(void* dst, const void* src) {
  SpArr* a = sp_find_(src);
  if (!a) return false;
  uint8_t* d = static_cast<uint8_t*>(dst);
  const uint8_t* s = static_cast<const uint8_t*>(src);
  for (int c = 0; c < a->ncomp; ++c) {
    const size_t o = 8 * (size_t)c * g_.total_cells;
    AF_CUDA(cudaMemcpyAsync(d + o, s + o, a->coarse_bytes, cudaMemcpyDeviceToHost, stream_));
    for (long gb = 0; gb < sp_nbricks_; ++gb) {
      if (!a->bricks[gb * a->ncomp]) continue;
      long b = 0;
      const int m = sp_level_(gb, &b);
      const size_t bo = o + 8 * (size_t)(g_.cell_off[m] + (b << (3 * g_.bsh)));
      AF_CUDA(cudaMemcpyAsync(d + bo, s + bo, sp_brick_bytes_, cudaMemcpyDeviceToHost, stream_));
    }
  }
  AF_CUDA(cudaStreamSynchronize(stream_));
  return true;
}

// Device bytes of the per-cell arrays now (mapped value bricks + the coarse
// block + the dense status/flag/register arrays), their peak, and what the
// same tree would take as dense per-level grids.
void MR::memory(unsigned long long* now, unsigned long long* peak,
                unsigned long long* dense) const {
  size_t coarse = 0;
  for (const SpArr& a : sp_) coarse += a.coarse_bytes * a.ncomp;
  if (now) *now = cell_bytes_ + coarse + sp_now_;
  if (peak) *peak = cell_bytes_ + coarse + sp_peak_;
  if (dense) {
    long cells = 0;
    for (int l = 0; l <= L_; ++l) cells += mr_cells(D_, l);
    *dense = (unsigned long long)cells * cell_elem_bytes_;
  }
}

}  // namespace af

namespace af {

// A per-cell array: sparse bricks (value arrays with AF_MR_STORAGE_SPARSE) or
// one allocation (windowed with ranks). Padded layouts start zeroed: passes
// over the concatenated levels read the padding as ABSENT cells.
void* MR::calloc_(size_t elem, int ncomp, bool sparse) {
  cell_elem_bytes_ += elem * (size_t)ncomp;
  if (sparse) return sp_alloc_(ncomp);
  void* p = walloc_(elem, ncomp);
  if (!windows_) {
    const size_t bytes = elem * (size_t)ncomp * (size_t)g_.total_cells;
    cell_bytes_ += bytes;
    if (g_.bsh) AF_CUDA(cudaMemset(p, 0, bytes));
  }
  return p;
}

}  // namespace af
