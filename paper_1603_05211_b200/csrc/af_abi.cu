// af_abi.cu — the extern "C" boundary of libafgpu (include/af_gpu.h).
// Every entry point catches af::Error / std::exception and returns an
// af_status; the last error is kept per object (or thread-local for calls
// without one) for af_*_last_error.
#include <nccl.h>

#include <cmath>
#include <cstring>
#include <new>
#include <vector>

#include "af_cases.h"
#include "af_comm.h"
#include "af_gpu.h"
#include "af_mr.h"
#include "af_uniform.h"

struct af_uniform {
  af::Uniform* impl;
  af::Comm* owned_comm = nullptr;  // local-group rank descriptor
};

struct af_mr {
  af::MR* impl;
};

namespace {

thread_local af_error g_last{};

af_status record(af_error* slot, af_status st, const char* msg) {
  af_error& e = slot ? *slot : g_last;
  if (st != AF_E_NONPHYSICAL || e.status != AF_E_NONPHYSICAL) {
    std::memset(&e, 0, sizeof(e));
    e.step = -1;
    e.level = -1;
  }
  e.status = st;
  if (msg) std::snprintf(e.message, sizeof e.message, "%s", msg);
  return st;
}

template <class F>
af_status guard(af_error* slot, F&& f) {
  try {
    f();
    return AF_OK;
  } catch (const af::Error& e) {
    return record(slot, e.status, e.what());
  } catch (const std::bad_alloc&) {
    return record(slot, AF_E_CUDA, "host allocation failed");
  } catch (const std::exception& e) {
    return record(slot, AF_E_ARGUMENT, e.what());
  }
}

}  // namespace

extern "C" {

const char* af_version(void) { return "afgpu 0.1 (sm_100a)"; }
int af_abi_version(void) { return AF_ABI_VERSION; }

af_status af_case_fill(int kind, uint64_t seed, int level, double gamma, int z0, int nz,
                       double* out) {
  if (!out || kind < 0 || kind > 3) return record(nullptr, AF_E_ARGUMENT, "af_case_fill: bad argument");
  return ::af_cases_fill(kind, seed, level, gamma, z0, nz, out) == 0
             ? AF_OK
             : record(nullptr, AF_E_ARGUMENT, "af_case_fill: bad argument");
}

af_status af_comm_unique_id(unsigned char id[128]) {
  return guard(nullptr, [&] {
    if (!id) throw af::Error(AF_E_ARGUMENT, "null id");
    ncclUniqueId u;
    const ncclResult_t r = ncclGetUniqueId(&u);
    if (r != ncclSuccess) throw af::Error(AF_E_NCCL, ncclGetErrorString(r));
    static_assert(sizeof(u) == 128, "ncclUniqueId size");
    std::memcpy(id, &u, 128);
  });
}

af_status af_comm_create(const unsigned char id[128], int n_ranks, int rank, int device,
                         af_comm** out) {
  return guard(nullptr, [&] {
    if (!id || !out || n_ranks < 1 || rank < 0 || rank >= n_ranks)
      throw af::Error(AF_E_ARGUMENT, "af_comm_create: bad argument");
    AF_CUDA(cudaSetDevice(device));
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    auto* c = new af_comm;
    c->c.n = n_ranks;
    c->c.rank = rank;
    c->c.device = device;
    const ncclResult_t r = ncclCommInitRank(&c->c.nccl, n_ranks, u, rank);
    if (r != ncclSuccess) {
      delete c;
      throw af::Error(AF_E_NCCL, ncclGetErrorString(r));
    }
    *out = c;
  });
}

af_status af_comm_create_local(int n_ranks, int device, af_comm** comms) {
  return guard(nullptr, [&] {
    if (!comms || n_ranks < 1) throw af::Error(AF_E_ARGUMENT, "af_comm_create_local: bad argument");
    auto group = std::make_shared<af::LocalGroup>(n_ranks);
    for (int r = 0; r < n_ranks; ++r) {
      auto* c = new af_comm;
      c->c.n = n_ranks;
      c->c.rank = r;
      c->c.device = device;
      c->c.local = true;
      c->c.group = group;
      comms[r] = c;
    }
  });
}

af_status af_comm_destroy(af_comm* comm) {
  if (!comm) return AF_OK;
  if (comm->c.nccl) ncclCommDestroy(comm->c.nccl);
  delete comm;
  return AF_OK;
}

af_status af_uniform_create(const af_config* cfg, af_comm* comm, af_uniform** out) {
  return guard(nullptr, [&] {
    if (!cfg || !out) throw af::Error(AF_E_ARGUMENT, "af_uniform_create: null argument");
    auto* h = new af_uniform;
    try {
      h->impl = new af::Uniform(*cfg, comm ? &comm->c : nullptr);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

af_status af_uniform_destroy(af_uniform* u) {
  if (!u) return AF_OK;
  delete u->impl;
  delete u->owned_comm;
  delete u;
  return AF_OK;
}

af_status af_uniform_create_group(const af_config* cfg, int n_ranks, af_uniform** ranks) {
  return guard(nullptr, [&] {
    if (!cfg || !ranks || n_ranks < 1 || n_ranks > 16)
      throw af::Error(AF_E_ARGUMENT, "af_uniform_create_group: bad argument");
    for (int r = 0; r < n_ranks; ++r) ranks[r] = nullptr;
    try {
      for (int r = 0; r < n_ranks; ++r) {
        auto* h = new af_uniform;
        h->impl = nullptr;
        h->owned_comm = new af::Comm;
        h->owned_comm->n = n_ranks;
        h->owned_comm->rank = r;
        h->owned_comm->device = cfg->device;
        h->owned_comm->local = true;
        ranks[r] = h;
        h->impl = new af::Uniform(*cfg, h->owned_comm);
      }
    } catch (...) {
      for (int r = 0; r < n_ranks; ++r)
        if (ranks[r]) af_uniform_destroy(ranks[r]);
      throw;
    }
  });
}

af_status af_uniform_run_group(af_uniform** ranks, int n_ranks, long n_steps, double cfl,
                               double fixed_dt, double* dt_hist, af_run_diag* diag) {
  if (!ranks || n_ranks < 1) return record(nullptr, AF_E_ARGUMENT, "null group");
  std::vector<af::Uniform*> R(n_ranks);
  for (int r = 0; r < n_ranks; ++r) {
    if (!ranks[r] || !ranks[r]->impl) return record(nullptr, AF_E_ARGUMENT, "null rank");
    R[r] = ranks[r]->impl;
  }
  return guard(&R[0]->last_error(),
               [&] { af::Uniform::run_group(R, n_steps, cfl, fixed_dt, dt_hist, diag); });
}

#define AF_U_GUARD(body)                                                     \
  do {                                                                       \
    if (!u || !u->impl) return record(nullptr, AF_E_ARGUMENT, "null solver"); \
    return guard(&u->impl->last_error(), [&] { body; });                     \
  } while (0)

af_status af_uniform_set_stream(af_uniform* u, void* s) {
  AF_U_GUARD(u->impl->set_stream(static_cast<cudaStream_t>(s)));
}

af_status af_uniform_set_numerics(af_uniform* u, int numerics) {
  AF_U_GUARD(u->impl->set_numerics(numerics));
}

af_status af_uniform_local_extent(const af_uniform* u, int* z0, int* nz) {
  if (!u || !u->impl || !z0 || !nz) return record(nullptr, AF_E_ARGUMENT, "null argument");
  *z0 = u->impl->grid().zlo;
  *nz = u->impl->grid().nzl;
  return AF_OK;
}

af_status af_slab_extent(int dim, int level, int n_ranks, int rank, int* z0, int* nz) {
  if (!z0 || !nz) return record(nullptr, AF_E_ARGUMENT, "null argument");
  if (!af::slab_extent(dim, level, n_ranks, rank, z0, nz))
    return record(nullptr, AF_E_CONFIG, "too many ranks for this mesh");
  return AF_OK;
}

af_status af_uniform_upload(af_uniform* u, const double* aos) { AF_U_GUARD(u->impl->upload(aos)); }

af_status af_uniform_download(af_uniform* u, double* aos) { AF_U_GUARD(u->impl->download(aos)); }

af_status af_uniform_step(af_uniform* u, double dt, af_step_diag* diag) {
  AF_U_GUARD(u->impl->step(dt, diag));
}

af_status af_uniform_rk2_stage(af_uniform* u, const double* base, const double* eval,
                               double* out, double stage_dt, double* capture,
                               af_step_diag* diag) {
  AF_U_GUARD(u->impl->rk2_stage(base, eval, out, stage_dt, capture, diag));
}

af_status af_uniform_run(af_uniform* u, long n_steps, double cfl, double fixed_dt,
                         double* dt_hist, af_run_diag* diag) {
  AF_U_GUARD(u->impl->run(n_steps, cfl, fixed_dt, dt_hist, diag));
}

af_status af_uniform_speed_sum(af_uniform* u, double* smax) {
  AF_U_GUARD({
    if (!smax) throw af::Error(AF_E_ARGUMENT, "null output");
    *smax = u->impl->speed_sum();
  });
}

af_status af_uniform_sync(af_uniform* u) { AF_U_GUARD(u->impl->sync()); }

af_status af_uniform_last_error(const af_uniform* u, af_error* err) {
  if (!err) return AF_E_ARGUMENT;
  *err = (u && u->impl) ? u->impl->last_error() : g_last;
  return AF_OK;
}

af_status af_uniform_kernel_launches(const af_uniform* u, long* count) {
  if (!u || !u->impl || !count) return AF_E_ARGUMENT;
  *count = u->impl->launches();
  return AF_OK;
}

af_status af_mr_create(const af_config* cfg, const af_mr_options* opt, af_mr** out) {
  return guard(nullptr, [&] {
    if (!cfg || !opt || !out) throw af::Error(AF_E_ARGUMENT, "af_mr_create: null argument");
    auto* h = new af_mr;
    try {
      h->impl = new af::MR(*cfg, *opt);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

af_status af_mr_create_dist(const af_config* cfg, const af_mr_options* opt, af_comm* comm,
                            af_mr** out) {
  return guard(nullptr, [&] {
    if (!cfg || !opt || !out) throw af::Error(AF_E_ARGUMENT, "af_mr_create_dist: null argument");
    auto* h = new af_mr;
    try {
      h->impl = new af::MR(*cfg, *opt, comm ? &comm->c : nullptr);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

af_status af_mr_set_numerics(af_mr* m, int numerics) {
  if (!m || !m->impl) return record(nullptr, AF_E_ARGUMENT, "null solver");
  return guard(&m->impl->last_error(), [&] { m->impl->set_numerics(numerics); });
}

af_status af_mr_memory(const af_mr* m, unsigned long long* now, unsigned long long* peak,
                       unsigned long long* dense) {
  if (!m) return AF_E_ARGUMENT;
  m->impl->memory(now, peak, dense);
  return AF_OK;
}

af_status af_mr_local_rows(const af_mr* m, int level, int* lo, int* hi) {
  if (!m || !lo || !hi) return AF_E_ARGUMENT;
  try {
    m->impl->local_rows(level, lo, hi);
  } catch (const af::Error& e) {
    return e.status;
  }
  return AF_OK;
}

af_status af_mr_destroy(af_mr* m) {
  if (!m) return AF_OK;
  delete m->impl;
  delete m;
  return AF_OK;
}

#define AF_M_GUARD(body)                                                     \
  do {                                                                       \
    if (!m || !m->impl) return record(nullptr, AF_E_ARGUMENT, "null solver"); \
    return guard(&m->impl->last_error(), [&] { body; });                     \
  } while (0)

af_status af_mr_set_stream(af_mr* m, void* s) {
  AF_M_GUARD(m->impl->set_stream(static_cast<cudaStream_t>(s)));
}
af_status af_mr_build(af_mr* m, const double* aos) { AF_M_GUARD(m->impl->build(aos)); }
af_status af_mr_refine(af_mr* m, int top) { AF_M_GUARD(m->impl->refine(top)); }
af_status af_mr_solver_stats(af_mr* m, double* max_cfl, long* fallbacks) {
  AF_M_GUARD({
    if (max_cfl) *max_cfl = m->impl->max_cfl();
    if (fallbacks) *fallbacks = m->impl->fallbacks();
  });
}
af_status af_mr_refine_buffer(af_mr* m, double eps, const int* buffer_radius_per_level, int n) {
  AF_M_GUARD(m->impl->refine(eps, buffer_radius_per_level, n));
}
af_status af_mr_add_virtual_leaves(af_mr* m) { AF_M_GUARD(m->impl->add_virtual_leaves()); }
af_status af_mr_remove_virtual_leaves(af_mr* m) {
  AF_M_GUARD(m->impl->remove_virtual_leaves());
}
af_status af_mr_coarsen(af_mr* m) { AF_M_GUARD(m->impl->coarsen()); }
af_status af_mr_evolve_global(af_mr* m, double dt, af_step_diag* diag) {
  AF_M_GUARD(m->impl->evolve_global(dt, diag));
}
af_status af_mr_advance_local(af_mr* m, int top, double t, double dt, af_step_diag* diag) {
  AF_M_GUARD(m->impl->advance_local(top, t, dt, diag));
}
af_status af_mr_run(af_mr* m, long n_steps, double cfl, double fixed_dt, af_mr_cycle* cycles,
                    long max_cycles, af_run_diag* diag) {
  AF_M_GUARD(m->impl->run(n_steps, cfl, fixed_dt, cycles, max_cycles, diag));
}
af_status af_mr_counts(af_mr* m, long* leaves, long* nodes, long* internals) {
  AF_M_GUARD(m->impl->counts(leaves, nodes, internals));
}
af_status af_mr_coarsest_leaf_level(af_mr* m, int* level) {
  AF_M_GUARD({
    if (!level) throw af::Error(AF_E_ARGUMENT, "null output");
    *level = m->impl->coarsest_leaf_level();
  });
}
af_status af_mr_leaf_keys(af_mr* m, uint64_t* keys, size_t* n) {
  AF_M_GUARD({
    if (!n) throw af::Error(AF_E_ARGUMENT, "null count");
    *n = (size_t)m->impl->leaf_keys(keys, (long)*n);
  });
}
af_status af_mr_to_uniform(af_mr* m, int level, double* aos) {
  AF_M_GUARD({
    if (!aos) throw af::Error(AF_E_ARGUMENT, "null output");
    m->impl->to_uniform(level, aos);
  });
}
af_status af_mr_details(af_mr* m, int level, double* out) {
  AF_M_GUARD({
    if (!out) throw af::Error(AF_E_ARGUMENT, "null output");
    m->impl->details(level, out);
  });
}
af_status af_mr_profile(af_mr* m, int enable) { AF_M_GUARD(m->impl->profile(enable != 0)); }
af_status af_mr_stage_stats(af_mr* m, double* ms, long* launches, long* updates) {
  AF_M_GUARD(m->impl->stage_stats(ms, launches, updates));
}
af_status af_mr_last_error(const af_mr* m, af_error* err) {
  if (!err) return AF_E_ARGUMENT;
  *err = (m && m->impl) ? m->impl->last_error() : g_last;
  return AF_OK;
}
af_status af_mr_kernel_launches(const af_mr* m, long* count) {
  if (!m || !m->impl || !count) return AF_E_ARGUMENT;
  *count = m->impl->launches();
  return AF_OK;
}

}  // extern "C"

// ---------------------------------------------- formats and compare path --
af_status af_snapshot_write(const char* path, const af_snapshot_header* h, const double* aos) {
  return guard(nullptr, [&] {
    if (!path || !h || !aos) throw af::Error(AF_E_ARGUMENT, "af_snapshot_write: null argument");
    const long cells = h->dim == 3 ? 1L << (3 * h->level) : 1L << (2 * h->level);
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, aos) == cudaSuccess && at.type == cudaMemoryTypeDevice) {
      std::vector<double> host(5 * (size_t)cells);  // device array: stage through the host
      AF_CUDA(cudaMemcpy(host.data(), aos, host.size() * 8, cudaMemcpyDeviceToHost));
      af::snapshot_write(path, *h, host.data());
    } else {
      cudaGetLastError();
      af::snapshot_write(path, *h, aos);
    }
  });
}

af_status af_snapshot_read(const char* path, af_snapshot_header* h, double* aos) {
  return guard(nullptr, [&] {
    if (!path || !h) throw af::Error(AF_E_ARGUMENT, "af_snapshot_read: null argument");
    af::snapshot_read(path, h, aos);
  });
}

af_status af_restrict_to_level(int dim, int fine_level, int target, const double* fine,
                               double* out) {
  return guard(nullptr, [&] {
    if (!fine || !out) throw af::Error(AF_E_ARGUMENT, "af_restrict_to_level: null argument");
    af::restrict_to_level(dim, fine_level, target, fine, out);
  });
}

af_status af_l1_error(int dim, int level, double extent, const double* sol, int ref_level,
                      const double* ref, double out[5]) {
  return guard(nullptr, [&] {
    if (!sol || !ref || !out) throw af::Error(AF_E_ARGUMENT, "af_l1_error: null argument");
    af::l1_error(dim, level, extent, sol, ref_level, ref, out);
  });
}

af_status af_mr_dump(af_mr* m, char* buf, size_t* len) {
  if (!m || !len) return AF_E_ARGUMENT;
  AF_M_GUARD({
    const std::string s = m->impl->dump();
    const size_t need = s.size() + 1;
    if (buf && *len >= need) std::memcpy(buf, s.c_str(), need);
    *len = need;
  });
}

// rates (metrics.cpp:91-132): the reference's formulas and their order, its
// DivisionDomain texts.
extern "C" af_status af_rates_compute(const af_run_summary* ad, const af_run_summary* fv,
                                      double n_c, af_rates* out) {
  return guard(nullptr, [&] {
    if (!ad || !fv || !out) throw af::Error(AF_E_ARGUMENT, "null argument");
    auto domain = [](const char* what) { throw af::Error(AF_E_DOMAIN, what); };
    if (fv->n_steps == 0 || n_c == 0.0) domain("rates: zero baseline size");
    af_rates r{};
    if (fv->wall_seconds == 0.0) domain("cpu_compression: zero baseline time");
    r.cpu_compression = ad->wall_seconds / fv->wall_seconds;
    if (ad->n_steps == 0 || n_c == 0.0) domain("memory_compression: zero step or cell count");
    r.memory_compression = ad->sum_cells / static_cast<double>(ad->n_steps) / n_c;
    if (ad->n_steps == 0 || n_c == 0.0) domain("mesh_compression: zero step or cell count");
    r.mesh_compression = ad->sum_leaves / static_cast<double>(ad->n_steps) / n_c;
    if (fv->l1_rho == 0.0) domain("accuracy_perturbation: zero baseline error");
    r.perturbation = std::abs(fv->l1_rho - ad->l1_rho) / fv->l1_rho;
    const double fv_cell_steps = static_cast<double>(fv->n_steps) * n_c;
    if (ad->sum_leaves == 0.0 || fv->wall_seconds == 0.0 || fv_cell_steps == 0.0)
      domain("overhead: zero denominator");
    const double gamma_a = ad->wall_seconds / ad->sum_leaves;
    const double gamma_fv = fv->wall_seconds / fv_cell_steps;
    r.overhead = gamma_a / gamma_fv - 1.0;
    *out = r;
  });
}
