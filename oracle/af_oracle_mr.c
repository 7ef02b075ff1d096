/*
 * af_oracle_mr.c — TEST INFRASTRUCTURE ONLY: plain-C restatement of the MR
 * path (mr_tree.cpp, mr_solver.cpp). Filled in below.
 */
#include <stdio.h>
#include <string.h>

#include "af_oracle.h"

int afo_mr_run(const af_oracle_params* p, const double* init, double* out,
               uint64_t* leaf_keys, long* n_leaves, long* per_cycle, long max_cycles,
               double* dt_hist, af_oracle_result* res) {
  (void)p; (void)init; (void)out; (void)leaf_keys; (void)n_leaves; (void)per_cycle;
  (void)max_cycles; (void)dt_hist;
  memset(res, 0, sizeof(*res));
  res->err_kind = 9;
  snprintf(res->err, sizeof res->err, "afo_mr_run: not yet restated");
  return 9;
}

int afo_mr_last_dump(const char* path) { (void)path; return -1; }
