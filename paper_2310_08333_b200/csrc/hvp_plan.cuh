// Launch plan of the cluster HVP (hvp_cluster.cu), shared with its caller
// (gemv.cu: hvp_apply).
#pragma once
#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime.h>

namespace nys {

struct HcPlan {
  int W, K, S, L, nclusters;
  size_t smem;
  bool ok;
  // Q > 1: the CTA's column segment is staged in Q sub-segments of Wq columns
  // (v in shared memory, y in registers; the row's sub-segments are re-read
  // from L2 for the axpy) -- the plan for rows too wide to stage whole
  int Q, Wq;
};

HcPlan hvp_cluster_plan(int64_t rows, int64_t n, int64_t lda, const double* A, const double* v);
int hvp_cluster(HcPlan& p, const double* A, int64_t rows, int64_t n, int64_t lda, const double* d, const double* v,
                double* ypart, cudaStream_t st, const double* pred);

}  // namespace nys
