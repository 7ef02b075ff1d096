// af_comm.h — NCCL communicator of libafgpu (one process per GPU).
#pragma once

#include <nccl.h>

namespace af {

struct Comm {
  ncclComm_t nccl = nullptr;
  int n = 1;
  int rank = 0;
  int device = 0;
  bool local = false;  // ranks emulated in one process on one GPU (af_uniform_create_group)
};

}  // namespace af

struct af_comm {
  af::Comm c;
};
