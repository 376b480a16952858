// Read-bandwidth probe (development tool): sum of a 400 MB FP64 array by
//  (a) plain 128-bit loads, grid-stride, many CTAs;
//  (b) TMA bulk copies into an S-stage shared-memory ring, one CTA per SM,
//      piece size and stage count as arguments, consumers read the ring.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/stream_probe tools/stream_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void ldg_sum(const double2* __restrict__ a, int64_t n2, double* out) {
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = __ldg(a + i);
    s += v.x + v.y;
  }
  if (s == 12345.678) *out = s;
}

__global__ void __launch_bounds__(512, 1) tma_sum(const double* __restrict__ a, int64_t n, int piece, int S,
                                                  double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  double* ring = (double*)sm;
  uint64_t* full = (uint64_t*)(ring + (size_t)S * piece);
  const int tid = threadIdx.x;
  const int64_t npieces_total = n / piece;
  const int64_t mine = (npieces_total - blockIdx.x + gridDim.x - 1) / gridDim.x;
  if (tid == 0) {
    for (int q = 0; q < S; ++q)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[q])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int64_t g) {
    const int q = (int)(g % S);
    const int64_t p = blockIdx.x + g * gridDim.x;
    const unsigned bytes = (unsigned)piece * 8u;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[q])), "r"(bytes)
                 : "memory");
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
  const int64_t n = 50000000;  // 400 MB
  double* a;
  double* out;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&out, 8);
  cudaMemset(a, 0, n * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int blocks : {148 * 4, 148 * 8, 148 * 16}) {
    for (int w = 0; w < 3; ++w) ldg_sum<<<blocks, 256>>>((const double2*)a, n / 2, out);
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) ldg_sum<<<blocks, 256>>>((const double2*)a, n / 2, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("ldg   blocks %5d: %.1f us  %.0f GB/s\n", blocks, ms * 100, n * 8.0 / (ms / 10 * 1e-3) / 1e9);
  }
  cudaFuncSetAttribute(tma_sum, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  const int pieces[] = {2500, 5000, 10000, 1250};
  const int stages[] = {8, 5, 2, 16};
  for (int c = 0; c < 4; ++c) {
    for (int S : {stages[c], stages[c] / 2 > 1 ? stages[c] / 2 : 2}) {
      const size_t smem = (size_t)S * pieces[c] * 8 + S * 8 + 256;
      if (smem > 220 * 1024) continue;
      for (int w = 0; w < 3; ++w) tma_sum<<<148, 512, smem>>>(a, n, pieces[c], S, out);
      cudaEventRecord(e0);
      for (int r = 0; r < 10; ++r) tma_sum<<<148, 512, smem>>>(a, n, pieces[c], S, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("tma   piece %5d x S %2d (%3zu KB): %.1f us  %.0f GB/s  err=%s\n", pieces[c], S, smem / 1024, ms * 100,
             n * 8.0 / (ms / 10 * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
