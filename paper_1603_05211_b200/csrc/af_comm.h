// af_comm.h — communicator of libafgpu: NCCL (one process per GPU) or a
// local rank group emulated by host threads on one GPU (tests).
#pragma once

#include <nccl.h>

#include <condition_variable>
#include <memory>
#include <mutex>
#include <vector>

namespace af {

// Ranks emulated by host threads in one process on one GPU: a rendezvous
// for halo exchanges (device-to-device copies between the ranks' buffers)
// and host-side reductions. Used to exercise the multi-rank code paths,
// which are otherwise identical to the NCCL ones.
struct LocalGroup {
  int n;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long gen = 0;
  std::vector<const void*> ptr;          // [rank * n + peer] published device pointers
  std::vector<unsigned long long> val;   // [rank * kVals + i] published values
  static constexpr int kVals = 64;
  explicit LocalGroup(int n_) : n(n_), ptr((size_t)n_ * n_), val((size_t)n_ * kVals) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const unsigned long g0 = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g0; });
    }
  }
};

struct Comm {
  ncclComm_t nccl = nullptr;
  int n = 1;
  int rank = 0;
  int device = 0;
  bool local = false;  // ranks emulated in one process on one GPU
  std::shared_ptr<LocalGroup> group;  // thread-emulated group (af_comm_create_local)
};

}  // namespace af

struct af_comm {
  af::Comm c;
};
