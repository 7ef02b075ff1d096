// af_mr_dist.cu — spatial decomposition of the MR tree across ranks
// (SURVEY.md §8(e)): slab ownership per level, halo exchange of status /
// values / virtual marks, and the reductions the level-synchronous passes need.
//
// Every rank keeps the full-size level arrays (global indexing, so no kernel
// changes its addressing) but computes and decides only for the rows it owns;
// rows within halo_ of them are refreshed from their owners. Levels below the
// partition level are replicated (they hold no leaves and no absent cells).
// The transport is NCCL (one process per GPU) or, for tests on one GPU, a
// group of host threads exchanging through device-to-device copies.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "af_mr.h"
#include "af_vmm.h"

namespace af {

namespace {

__global__ void mr_xpack(const MR_XSeg* segs, int nseg, const double* V, const uint8_t* st,
                         const uint8_t* mark, long comp, int nc, long tot, uint8_t* buf,
                         int mask) {
  double* bv = reinterpret_cast<double*>(buf);
  uint8_t* bst = buf + 8 * (long)nc * tot;
  uint8_t* bmk = bst + tot;
  for (int s = blockIdx.y; s < nseg; s += gridDim.y) {
    const MR_XSeg sg = segs[s];
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < sg.cells;
         i += (long)gridDim.x * blockDim.x) {
      if (mask & 1)
        for (int m = 0; m < nc; ++m) bv[m * tot + sg.pos + i] = V[m * comp + sg.cell + i];
      if (mask & 2) bst[sg.pos + i] = st[sg.cell + i];
      if (mask & 4) bmk[sg.pos + i] = mark[sg.cell + i];
    }
  }
}

__global__ void mr_xunpack(const MR_XSeg* segs, int nseg, double* V, uint8_t* st, uint8_t* mark,
                           long comp, int nc, long tot, const uint8_t* buf, int mask) {
  const double* bv = reinterpret_cast<const double*>(buf);
  const uint8_t* bst = buf + 8 * (long)nc * tot;
  const uint8_t* bmk = bst + tot;
  for (int s = blockIdx.y; s < nseg; s += gridDim.y) {
    const MR_XSeg sg = segs[s];
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < sg.cells;
         i += (long)gridDim.x * blockDim.x) {
      if (mask & 1)
        for (int m = 0; m < nc; ++m) V[m * comp + sg.cell + i] = bv[m * tot + sg.pos + i];
      if (mask & 2) st[sg.cell + i] = bst[sg.pos + i];
      if (mask & 4) mark[sg.cell + i] = bmk[sg.pos + i];
    }
  }
}

void check_nccl(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(AF_E_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

}  // namespace

// Rows [lo, hi) of the last axis that rank r owns at level l: a balanced
// split of the 2^lp_ rows of the partition level, scaled by 2^(l - lp_)
// above it (so a node's children are owned by the node's owner).
void MR::part_rows_(int r, int l, int* lo, int* hi) const {
  if (!dist_ || l < lp_) {
    *lo = 0;
    *hi = 1 << l;
    return;
  }
  const long np = 1L << lp_;
  const int a = (int)(np * r / nranks_), b = (int)(np * (r + 1) / nranks_);
  *lo = a << (l - lp_);
  *hi = b << (l - lp_);
}

void MR::local_rows(int level, int* lo, int* hi) const {
  if (level < 0 || level > L_) throw Error(AF_E_LEVEL_MISMATCH, "local_rows: bad level");
  if (dist_ && level < lp_) {  // replicated: reported by rank 0
    *lo = 0;
    *hi = rank_ == 0 ? 1 << level : 0;
    return;
  }
  part_rows_(rank_, level, lo, hi);
}

// Exchange plan: for every peer, the rows this rank owns that fall in the
// peer's region (send), and the peer's owned rows in this rank's region
// (receive), as contiguous runs of whole rows per level.
void MR::dist_setup_() {
  const int D = D_;
  const bool periodic = cfg_.bc[2 * (D - 1)] == AF_BC_PERIODIC;
  int ml = opt_.min_leaf_level;
  if (opt_.local_time) ml = std::max(ml, std::max(0, L_ - opt_.lt_gap));
  auto region = [&](int r, int l, std::vector<char>& in) {
    const int n = 1 << l;
    in.assign(n, 0);
    if (l < lp_ || (l == lp_ && lp_ == ml)) {
      std::fill(in.begin(), in.end(), 1);
      return;
    }
    int a, b;
    part_rows_(r, l, &a, &b);
    for (int y = a - halo_; y < b + halo_; ++y) {
      int yy = y;
      if (yy < 0 || yy >= n) {
        if (!periodic) continue;
        yy = ((yy % n) + n) % n;
      }
      in[yy] = 1;
    }
  };
  std::vector<char> inq, inr;
  for (int q = 0; q < nranks_; ++q) {
    if (q == rank_) continue;
    Peer p;
    p.rank = q;
    for (int l = lp_; l <= L_; ++l) {
      const long rowlen = D == 3 ? (1L << (2 * l)) : (1L << l);
      region(q, l, inq);
      region(rank_, l, inr);
      int a, b, qa, qb;
      part_rows_(rank_, l, &a, &b);
      part_rows_(q, l, &qa, &qb);
      auto runs = [&](int lo, int hi, const std::vector<char>& in, std::vector<XSeg>& out,
                      long& total) {
        int y = lo;
        while (y < hi) {
          if (!in[y]) {
            ++y;
            continue;
          }
          int e = y;
          while (e < hi && in[e]) ++e;
          out.push_back({g_.cell_off[l] + (long)y * rowlen, (long)(e - y) * rowlen, total});
          total += (long)(e - y) * rowlen;
          y = e;
        }
      };
      runs(a, b, inq, p.send, p.send_cells);
      runs(qa, qb, inr, p.recv, p.recv_cells);
    }
    if (p.send.empty() && p.recv.empty()) continue;
    const size_t per_cell = 8 * (size_t)NC_ + 2;
    if (!p.send.empty()) {
      AF_CUDA(cudaMalloc(&p.d_send, sizeof(XSeg) * p.send.size()));
      AF_CUDA(cudaMemcpy(p.d_send, p.send.data(), sizeof(XSeg) * p.send.size(),
                         cudaMemcpyHostToDevice));
      AF_CUDA(cudaMalloc(&p.sbuf, per_cell * p.send_cells));
    }
    if (!p.recv.empty()) {
      AF_CUDA(cudaMalloc(&p.d_recv, sizeof(XSeg) * p.recv.size()));
      AF_CUDA(cudaMemcpy(p.d_recv, p.recv.data(), sizeof(XSeg) * p.recv.size(),
                         cudaMemcpyHostToDevice));
      AF_CUDA(cudaMalloc(&p.rbuf, per_cell * p.recv_cells));
    }
    peers_.push_back(p);
  }
  AF_CUDA(cudaMalloc(&d_xred_, sizeof(unsigned long long) * 64));
}

void MR::dist_free_() {
  for (Peer& p : peers_)
    for (void* ptr : {(void*)p.d_send, (void*)p.d_recv, (void*)p.sbuf, (void*)p.rbuf})
      cudaFree(ptr);
  peers_.clear();
  if (d_xred_) cudaFree(d_xred_);
  d_xred_ = nullptr;
}

// Refreshes this rank's halo rows (all levels >= lp_) from their owners:
// values (XV), status (XST), virtual marks (XMARK).
void MR::exchange_(int mask) {
  if (!dist_ || !mask) return;
  static const bool skip = std::getenv("AF_MR_DEBUG_NO_EXCHANGE") != nullptr;  // tests only
  if (skip) return;
  const long comp = g_.total_cells;
  // byte range of the packed buffer that holds the requested sections
  auto range = [&](long tot, size_t* b0, size_t* b1) {
    const size_t v = 8 * (size_t)NC_ * tot;
    *b0 = (mask & XV) ? 0 : (mask & XST) ? v : v + tot;
    *b1 = (mask & XMARK) ? v + 2 * tot : (mask & XST) ? v + tot : v;
  };
  for (Peer& p : peers_)
    if (p.send_cells) {
      const long mx = std::max_element(p.send.begin(), p.send.end(), [](const XSeg& a,
                                       const XSeg& b) { return a.cells < b.cells; })->cells;
      dim3 grid((unsigned)std::min<long>((mx + 255) / 256, 64),
                (unsigned)std::min<size_t>(p.send.size(), 65535));
      mr_xpack<<<grid, 256, 0, stream_>>>(reinterpret_cast<const MR_XSeg*>(p.d_send),
                                          (int)p.send.size(), d_V_, d_st_, d_mark_, comp, NC_,
                                          p.send_cells, p.sbuf, mask);
      ++launches_;
      AF_CUDA(cudaGetLastError());
    }
  if (comm_->group) {  // host-thread group on one GPU
    LocalGroup& G = *comm_->group;
    AF_CUDA(cudaStreamSynchronize(stream_));
    for (Peer& p : peers_) G.ptr[(size_t)rank_ * nranks_ + p.rank] = p.sbuf;
    G.barrier();
    for (Peer& p : peers_)
      if (p.recv_cells) {
        size_t b0, b1;
        range(p.recv_cells, &b0, &b1);
        const uint8_t* src =
            static_cast<const uint8_t*>(G.ptr[(size_t)p.rank * nranks_ + rank_]);
        AF_CUDA(cudaMemcpyAsync(p.rbuf + b0, src + b0, b1 - b0, cudaMemcpyDeviceToDevice,
                                stream_));
      }
    AF_CUDA(cudaStreamSynchronize(stream_));
    G.barrier();
  } else {
    check_nccl(ncclGroupStart(), "ncclGroupStart");
    for (Peer& p : peers_) {
      size_t b0, b1;
      if (p.send_cells) {
        range(p.send_cells, &b0, &b1);
        check_nccl(ncclSend(p.sbuf + b0, b1 - b0, ncclUint8, p.rank, comm_->nccl, stream_),
                   "ncclSend");
      }
      if (p.recv_cells) {
        range(p.recv_cells, &b0, &b1);
        check_nccl(ncclRecv(p.rbuf + b0, b1 - b0, ncclUint8, p.rank, comm_->nccl, stream_),
                   "ncclRecv");
      }
    }
    check_nccl(ncclGroupEnd(), "ncclGroupEnd");
  }
  for (Peer& p : peers_)
    if (p.recv_cells) {
      const long mx = std::max_element(p.recv.begin(), p.recv.end(), [](const XSeg& a,
                                       const XSeg& b) { return a.cells < b.cells; })->cells;
      dim3 grid((unsigned)std::min<long>((mx + 255) / 256, 64),
                (unsigned)std::min<size_t>(p.recv.size(), 65535));
      mr_xunpack<<<grid, 256, 0, stream_>>>(reinterpret_cast<const MR_XSeg*>(p.d_recv),
                                            (int)p.recv.size(), d_V_, d_st_, d_mark_, comp, NC_,
                                            p.recv_cells, p.rbuf, mask);
      ++launches_;
      AF_CUDA(cudaGetLastError());
    }
}

// ---- windowed arrays --------------------------------------------------------

// Per-level window rows: the region widened by the tile height plus the
// stencil reach, so tile-based kernels (whose tiles may overhang the region)
// and the stage's 2-cell gather stay inside mapped memory; whole levels below
// the partition level and where the window covers the level.
void MR::win_setup_() {
  const int TR = D_ == 3 ? kTileZ3 : kTileY2;
  const bool periodic = cfg_.bc[2 * (D_ - 1)] == AF_BC_PERIODIC;
  win_.assign(L_ + 1, {});
  for (int l = 0; l <= L_; ++l) {
    const int n = 1 << l;
    const long rowlen = D_ == 3 ? 1L << (2 * l) : 1L << l;
    const long off = g_.cell_off[l];
    int lo = g_.reg_lo[l] - TR - 2 - halo_, hi = g_.reg_hi[l] + TR + 2 + halo_;
    if (!dist_ || hi - lo >= n || (g_.reg_hi[l] - g_.reg_lo[l]) >= n) {
      win_[l].push_back({off, off + (long)n * rowlen});
      continue;
    }
    if (!periodic) {
      lo = std::max(lo, 0);
      hi = std::min(hi, n);
      win_[l].push_back({off + lo * rowlen, off + hi * rowlen});
    } else {  // may wrap: up to two intervals
      const int a = ((lo % n) + n) % n, len = hi - lo;
      if (a + len <= n) {
        win_[l].push_back({off + a * rowlen, off + (a + len) * rowlen});
      } else {
        win_[l].push_back({off + a * rowlen, off + (long)n * rowlen});
        win_[l].push_back({off, off + (long)(a + len - n) * rowlen});
      }
    }
  }
}

void* MR::walloc_(size_t elem, int ncomp) {
  const size_t bytes = elem * (size_t)ncomp * (size_t)g_.total_cells;
  if (!windows_) {
    void* p = nullptr;
    AF_CUDA(cudaMalloc(&p, bytes));
    return p;
  }
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = cfg_.device;
  size_t gran = 0;
  check_cu(vmm().granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED),
           "cuMemGetAllocationGranularity");
  WinMap w;
  w.reserved = (bytes + gran - 1) / gran * gran;
  CUdeviceptr base = 0;
  check_cu(vmm().reserve(&base, w.reserved, gran, 0, 0), "cuMemAddressReserve");
  w.base = base;
  // byte ranges of every component's windows, granule-aligned and merged
  std::vector<std::pair<size_t, size_t>> r;
  for (int m = 0; m < ncomp; ++m)
    for (int l = 0; l <= L_; ++l)
      for (const auto& c : win_[l]) {
        const size_t b0 = ((size_t)m * g_.total_cells + c.first) * elem;
        const size_t b1 = ((size_t)m * g_.total_cells + c.second) * elem;
        r.push_back({b0 / gran * gran, std::min(w.reserved, (b1 + gran - 1) / gran * gran)});
      }
  std::sort(r.begin(), r.end());
  std::vector<std::pair<size_t, size_t>> mr;
  for (const auto& x : r) {
    if (!mr.empty() && x.first <= mr.back().second) mr.back().second = std::max(mr.back().second, x.second);
    else mr.push_back(x);
  }
  CUmemAccessDesc acc{};
  acc.location = prop.location;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  for (const auto& x : mr) {
    const size_t sz = x.second - x.first;
    CUmemGenericAllocationHandle h;
    check_cu(vmm().create(&h, sz, &prop, 0), "cuMemCreate");
    check_cu(vmm().map(base + x.first, sz, 0, h, 0), "cuMemMap");
    check_cu(vmm().access(base + x.first, sz, &acc, 1), "cuMemSetAccess");
    w.maps.push_back({base + x.first, sz});
    w.handles.push_back(h);
  }
  wmaps_.push_back(w);
  return reinterpret_cast<void*>(base);
}

void MR::wfree_all_() {
  for (WinMap& w : wmaps_) {
    for (size_t i = 0; i < w.maps.size(); ++i) {
      vmm().unmap(w.maps[i].first, w.maps[i].second);
      vmm().release(w.handles[i]);
    }
    vmm().free_(w.base, w.reserved);
  }
  wmaps_.clear();
}

// memset of levels [lev_lo, lev_hi] of a per-cell array (every component),
// restricted to the windows
void MR::wset_(void* p, size_t elem, int ncomp, int value, int lev_lo, int lev_hi) {
  if (lev_hi < lev_lo) return;
  if (sp_set_(p, value, lev_lo, lev_hi)) return;  // sparse bricks: the mapped ones
  uint8_t* b = static_cast<uint8_t*>(p);
  for (int m = 0; m < ncomp; ++m) {
    const size_t cbase = (size_t)m * g_.total_cells;
    if (!windows_ && g_.bsh) {  // padded levels: the padding stays ABSENT / zero
      for (int l = lev_lo; l <= lev_hi; ++l)
        AF_CUDA(cudaMemsetAsync(b + (cbase + g_.cell_off[l]) * elem, value,
                                mr_cells(D_, l) * elem, stream_));
      continue;
    }
    if (!windows_) {
      const long c0 = g_.cell_off[lev_lo], c1 = g_.cell_off[lev_hi + 1];
      AF_CUDA(cudaMemsetAsync(b + (cbase + c0) * elem, value, (c1 - c0) * elem, stream_));
      continue;
    }
    for (int l = lev_lo; l <= lev_hi; ++l)
      for (const auto& c : win_[l])
        AF_CUDA(cudaMemsetAsync(b + (cbase + c.first) * elem, value, (c.second - c.first) * elem,
                                stream_));
  }
}

// copy of a per-cell array to a full-size host buffer (windows only; the
// rest of dst is left as it is)
void MR::wtohost_(void* dst, const void* src, size_t elem, int ncomp) {
  if (sp_tohost_(dst, src)) return;  // sparse bricks: the mapped ones
  uint8_t* d = static_cast<uint8_t*>(dst);
  const uint8_t* s = static_cast<const uint8_t*>(src);
  if (!windows_) {
    AF_CUDA(cudaMemcpyAsync(d, s, elem * ncomp * (size_t)g_.total_cells, cudaMemcpyDeviceToHost,
                            stream_));
  } else {
    for (int m = 0; m < ncomp; ++m)
      for (int l = 0; l <= L_; ++l)
        for (const auto& c : win_[l]) {
          const size_t o = ((size_t)m * g_.total_cells + c.first) * elem;
          AF_CUDA(cudaMemcpyAsync(d + o, s + o, (c.second - c.first) * elem,
                                  cudaMemcpyDeviceToHost, stream_));
        }
  }
  AF_CUDA(cudaStreamSynchronize(stream_));
}

// In-place reduction of k unsigned 64-bit values over the ranks (max / sum /
// min). Non-negative doubles reduce by max on their bit patterns.
void MR::allreduce_(unsigned long long* v, int k, int op) {
  if (!dist_) return;
  if (k > LocalGroup::kVals) throw Error(AF_E_ARGUMENT, "allreduce_: too many values");
  if (comm_->group) {
    LocalGroup& G = *comm_->group;
    for (int i = 0; i < k; ++i) G.val[(size_t)rank_ * LocalGroup::kVals + i] = v[i];
    G.barrier();
    for (int i = 0; i < k; ++i) {
      unsigned long long acc = G.val[i];
      for (int r = 1; r < nranks_; ++r) {
        const unsigned long long x = G.val[(size_t)r * LocalGroup::kVals + i];
        acc = op == RED_MAX ? std::max(acc, x) : op == RED_MIN ? std::min(acc, x) : acc + x;
      }
      v[i] = acc;
    }
    G.barrier();
    return;
  }
  AF_CUDA(cudaMemcpyAsync(d_xred_, v, sizeof(unsigned long long) * k, cudaMemcpyHostToDevice,
                          stream_));
  check_nccl(ncclAllReduce(d_xred_, d_xred_, k, ncclUint64,
                           op == RED_MAX ? ncclMax : op == RED_MIN ? ncclMin : ncclSum,
                           comm_->nccl, stream_),
             "ncclAllReduce");
  AF_CUDA(cudaMemcpyAsync(v, d_xred_, sizeof(unsigned long long) * k, cudaMemcpyDeviceToHost,
                          stream_));
  AF_CUDA(cudaStreamSynchronize(stream_));
}

}  // namespace af
