// L2 reuse across back-to-back streaming passes (development tool): one TMA
// row-streaming pass over a 400 MB FP64 matrix (5000 x 10000), then a second
// pass in the same or the reverse row order; times the second pass.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2reuse tools/l2reuse_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(512, 1) rows_sum(const double* __restrict__ a, int64_t rows, int piece, int S,
                                                   int rev, double keep, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  double* ring = (double*)sm;
  uint64_t* full = (uint64_t*)(ring + (size_t)S * piece);
  const int tid = threadIdx.x;
  const int64_t mine = (rows - blockIdx.x + gridDim.x - 1) / gridDim.x;
  if (tid == 0) {
    for (int q = 0; q < S; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[q])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint64_t pol_last, pol_first;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_last));
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
  auto issue = [&](int64_t g) {
    const int q = (int)(g % S);
    const bool last = keep > 0.0 && g >= (int64_t)((double)mine * (1.0 - keep));
    const uint64_t pol = keep > 0.0 ? (last ? pol_last : pol_first) : 0;
    int64_t p = blockIdx.x + g * gridDim.x;
    if (rev) p = rows - 1 - p;
    const unsigned bytes = (unsigned)piece * 8u;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[q])), "r"(bytes)
                 : "memory");
    if (keep > 0.0)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
          "%4;" ::"r"(smem_u32(ring + (size_t)q * piece)),
          "l"(a + p * piece), "r"(bytes), "r"(smem_u32(&full[q])), "l"(pol)
          : "memory");
    else
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(ring + (size_t)q * piece)),
                   "l"(a + p * piece), "r"(bytes), "r"(smem_u32(&full[q]))
                   : "memory");
  };
  if (tid == 0)
    for (int64_t g = 0; g < S && g < mine; ++g) issue(g);
  double s = 0.0;
  for (int64_t g = 0; g < mine; ++g) {
    const int q = (int)(g % S);
    const unsigned par = (unsigned)((g / S) & 1);
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
            smem_u32(&full[q])),
        "r"(par)
        : "memory");
    const double2* r = (const double2*)(ring + (size_t)q * piece);
    for (int j = tid; j < piece / 2; j += blockDim.x) {
      const double2 v = r[j];
      s += v.x + v.y;
    }
    __syncthreads();
    if (tid == 0 && g + S < mine) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(g + S);
    }
  }
  if (s == 12345.678) *out = s;
}

int main() {
  const int64_t rows = 5000, cols = 10000;
  double *a, *out, *flush;
  cudaMalloc(&a, rows * cols * 8);
  cudaMalloc(&out, 8);
  cudaMalloc(&flush, 512ull << 20);
  cudaMemset(a, 0, rows * cols * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int S = 2;
  const size_t smem = (size_t)S * cols * 8 + S * 8 + 256;
  cudaFuncSetAttribute(rows_sum, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  // chains of passes alternating direction, each keeping the last `keep`
  // fraction of its rows with evict_last (evict_first for the rest)
  for (double keep : {0.0, 0.1, 0.2, 0.25, 0.3, 0.4}) {
    for (int alt = 0; alt < 2; ++alt) {
      float tot = 0.f;
      const int chain = 8;
      for (int it = 0; it < 5; ++it) {
        cudaMemsetAsync(flush, it, 512ull << 20);
        rows_sum<<<148, 512, smem>>>(a, rows, (int)cols, S, 0, keep, out);
        cudaEventRecord(e0);
        for (int c = 1; c <= chain; ++c)
          rows_sum<<<148, 512, smem>>>(a, rows, (int)cols, S, alt ? (c & 1) : 0, keep, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        tot += ms / chain;
      }
      printf("keep %.2f %s: %.1f us/pass  %.0f GB/s  %s\n", keep, alt ? "alternate" : "same-dir ", tot / 5 * 1e3,
             rows * cols * 8.0 / (tot / 5 * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
