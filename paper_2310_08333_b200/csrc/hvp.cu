// K3, single pass: y = A^T (d o (A v)) + shift v with A streamed from HBM ONCE
// (problems.py:263-264 MLHessian._apply + the CG shift of admm.py:262-263).
//
// A row's dot product must complete before the same row can be used for the
// A^T update, so the row has to stay on chip in between.  Layout:
//   * a thread-block cluster of C CTAs splits the n columns into C slices of
//     width W <= 12800 (C = 1 for n <= 12800, e.g. config 2; C = 8-9 for
//     n = 100000); each CTA keeps its v slice and its y slice in REGISTERS
//     (thread t owns column pairs 2(t + kT), k < K);
//   * row segments (W doubles, contiguous) are brought into a multi-stage
//     shared-memory ring by TMA bulk copies (cp.async.bulk + mbarrier
//     complete_tx), several rows ahead of the compute;
//   * per row: partial dot over the slice -> CTA reduction -> the C partials
//     are exchanged through distributed shared memory and summed in a fixed
//     order after a cluster barrier -> t = d_i * dot -> y += t * a_i from the
//     same staged row;
//   * clusters stride over rows; at the end each cluster writes its y partial
//     and a fixed-order reduction adds the clusters, shift * v and p.Ap.
// Algorithmic traffic: 8 N n + 8 (2n + N) bytes per HVP, plus the y partials
// (8 n per cluster: 3 % of A for config 2, 0.1 % for config 4).
#include <cooperative_groups.h>
#include <stdlib.h>
#include "common.cuh"

namespace cg = cooperative_groups;

namespace nys {

constexpr int kHvpThreads = 512;
constexpr int kHvpMaxW = 12800;
constexpr int kHvpMaxK = (kHvpMaxW + 2 * kHvpThreads - 1) / (2 * kHvpThreads);  // 13
constexpr int kHvpSmemBudget = 200 * 1024;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// remote arrive on the same-offset mbarrier of cluster CTA `cta` (release at
// cluster scope orders this thread's preceding DSMEM stores before it)
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, unsigned cta) {
  asm volatile(
      "{\n"
      ".reg .b32 ra;\n"
      "mapa.shared::cluster.u32 ra, %0, %1;\n"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(cta)
      : "memory");
}
__device__ __forceinline__ void st_remote_f64(double* local_addr, unsigned cta, double v) {
  asm volatile(
      "{\n"
      ".reg .b32 ra;\n"
      "mapa.shared::cluster.u32 ra, %0, %1;\n"
      "st.shared::cluster.f64 [ra], %2;\n"
      "}\n" ::"r"(smem_u32(local_addr)),
      "r"(cta), "d"(v)
      : "memory");
}
// asynchronous remote store of one double into cluster CTA `cta`'s shared
// memory that signals that CTA's mbarrier (complete_tx of 8 bytes): no fence
__device__ __forceinline__ void st_async_remote_f64(double* local_addr, uint64_t* local_bar, unsigned cta,
                                                    double v) {
  asm volatile(
      "{\n"
      ".reg .b32 ra, rb;\n"
      "mapa.shared::cluster.u32 ra, %0, %2;\n"
      "mapa.shared::cluster.u32 rb, %1, %2;\n"
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [ra], %3, [rb];\n"
      "}\n" ::"r"(smem_u32(local_addr)),
      "r"(smem_u32(local_bar)), "r"(cta), "l"(__double_as_longlong(v))
      : "memory");
}

__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <int K, bool CLUSTER>
__global__ void __launch_bounds__(kHvpThreads, 1)
hvp_fused_kernel(const double* __restrict__ A, int64_t rows, int64_t n, int64_t lda,
                 const double* __restrict__ d, const double* __restrict__ v, int W, int S,
                 double* __restrict__ ypart, const double* __restrict__ pred) {
  // device-predicated launch (CG batches): every CTA of every cluster sees the same flag
  if (pred && *pred != 0.0) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw);                   // S x W
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)S * W);   // S mbarriers
  uint64_t* xbar = full + S;                                            // 4 exchange mbarriers
  double* xch = reinterpret_cast<double*>(xbar + 4);                    // 4 x 16 exchange slots
  double* red = xch + 64;                                               // 2 x 16 warp partials
  __shared__ double tval;

  int C = 1, rank = 0, cluster_id = blockIdx.x, nclusters = gridDim.x;
  if (CLUSTER) {
    cg::cluster_group cl = cg::this_cluster();
    C = (int)cl.num_blocks();
    rank = (int)cl.block_rank();
    cluster_id = blockIdx.x / C;
    nclusters = gridDim.x / C;
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t c0 = (int64_t)rank * W;
  const int w_here = (int)tmax<int64_t>(0, tmin<int64_t>((int64_t)W, n - c0));  // columns of this CTA

  // v slice and y accumulators in registers
  double2 vr[K], yr[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int j = 2 * (tid + k * kHvpThreads);
    vr[k] = (j < w_here) ? *reinterpret_cast<const double2*>(v + c0 + j) : make_double2(0.0, 0.0);
    yr[k] = make_double2(0.0, 0.0);
  }
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    // exchange barriers: one local arrival (the arming below) + C x 8 bytes of
    // st.async transactions from the peers
    for (int b = 0; b < 4; ++b) mbar_init(&xbar[b], 1u);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (CLUSTER && tid == 0)
    for (int b = 0; b < 4; ++b) mbar_expect_tx(&xbar[b], (unsigned)C * 8u);
  if (CLUSTER) cg::this_cluster().sync();  // peers' exchange barriers are initialised
  else __syncthreads();

  const int64_t nrows_mine = rows > cluster_id ? (rows - cluster_id + nclusters - 1) / nclusters : 0;
  const unsigned bytes = (unsigned)w_here * 8u;
  // prologue: fill the ring
  if (tid == 0 && bytes > 0) {
    for (int s = 0; s < S && s < nrows_mine; ++s) {
      const int64_t i = cluster_id + (int64_t)s * nclusters;
      mbar_expect_tx(&full[s], bytes);
      tma_load_1d(ring + (size_t)s * W, A + i * lda + c0, bytes, &full[s]);
    }
  }
  // Software pipeline.  Iteration `it` (a) computes this CTA's partial dot of
  // row it and, in a cluster, pushes it to every peer (DSMEM store + remote
  // mbarrier arrive), then (b) finishes row it - LAG: waits for that row's C
  // partials, forms t and applies the axpy from the still-staged row, frees the
  // stage and refills it.  LAG = 1 in a cluster hides the exchange latency
  // behind a row of work (needs S >= 3 stages and 4 exchange slots); LAG = 0
  // without a cluster.
  constexpr int LAG = CLUSTER ? 1 : 0;
  for (int64_t it = 0; it < nrows_mine + LAG; ++it) {
    if (it < nrows_mine) {
      const int s = (int)(it % S);
      const double* row = ring + (size_t)s * W;
      if (bytes > 0) mbar_wait(&full[s], (unsigned)((it / S) & 1));
      double part = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int j = 2 * (tid + k * kHvpThreads);
        if (j < w_here) {
          const double2 a = *reinterpret_cast<const double2*>(row + j);
          part = fma(a.x, vr[k].x, part);
          part = fma(a.y, vr[k].y, part);
        }
      }
      part = warp_sum(part);
      if (lane == 0) red[(it & 1) * 16 + warp] = part;
      __syncthreads();
      if (CLUSTER && tid < C) {
        double p = 0.0;
        for (int q = 0; q < kHvpThreads / 32; ++q) p += red[(it & 1) * 16 + q];
        const int b = (int)(it & 3);
        st_async_remote_f64(xch + b * 16 + rank, &xbar[b], (unsigned)tid, p);
      }
    }
    const int64_t jt = it - LAG;  // the row finished in this iteration
    if (jt < 0) continue;
    const int sj = (int)(jt % S);
    const int64_t i = cluster_id + jt * nclusters;
    const double* row = ring + (size_t)sj * W;
    if (tid == 0) {
      double tot = 0.0;
      if (CLUSTER) {
        const int b = (int)(jt & 3);
        mbar_wait(&xbar[b], (unsigned)((jt >> 2) & 1));
        for (int q = 0; q < C; ++q) tot += xch[b * 16 + q];
        mbar_expect_tx(&xbar[b], (unsigned)C * 8u);  // re-arm for row jt + 4
      } else {
        for (int q = 0; q < kHvpThreads / 32; ++q) tot += red[(jt & 1) * 16 + q];
      }
      tval = d ? d[i] * tot : tot;
    }
    __syncthreads();
    const double t = tval;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int j = 2 * (tid + k * kHvpThreads);
      if (j < w_here) {
        const double2 a = *reinterpret_cast<const double2*>(row + j);
        yr[k].x = fma(t, a.x, yr[k].x);
        yr[k].y = fma(t, a.y, yr[k].y);
      }
    }
    __syncthreads();  // every thread is done with stage sj
    if (tid == 0 && bytes > 0 && jt + S < nrows_mine) {
      const int64_t inext = cluster_id + (jt + S) * nclusters;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&full[sj], bytes);
      tma_load_1d(ring + (size_t)sj * W, A + inext * lda + c0, bytes, &full[sj]);
    }
  }
  // y partial of this cluster, columns [c0, c0 + w_here)
  double* yp = ypart + (int64_t)cluster_id * n + c0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int j = 2 * (tid + k * kHvpThreads);
    if (j < w_here) *reinterpret_cast<double2*>(yp + j) = yr[k];
  }
  if (CLUSTER) cg::this_cluster().sync();  // no CTA may exit while others write its smem
}

struct HvpPlan {
  int C, W, K, S, nclusters;
  size_t smem;
  bool ok;
};

HvpPlan hvp_plan(int64_t rows, int64_t n, int64_t lda, const double* A, const double* v) {
  HvpPlan p{};
  p.ok = false;
  if ((lda & 1) || (n & 1) || ((uintptr_t)A & 15) || ((uintptr_t)v & 15)) return p;
  // Whole rows per CTA (C = 1) while a row fits the ring (n <= 12800).  The
  // cluster-split variant (16 CTAs, lag-1 pipelined st.async exchange) is
  // correct but measured at 2.4 TB/s vs 3.2 TB/s for the two-pass path at
  // n = 100000 on B200 (per-row fixed cost ~2 us), so it is opt-in
  // (NYS_HVP_C) until that is fixed; larger n use the two-pass path.
  p.C = 1;
  static const int forced = getenv("NYS_HVP_C") ? atoi(getenv("NYS_HVP_C")) : 0;
  if (forced > 0) p.C = forced;
  if (p.C > 16 || cdiv(cdiv(n, p.C), 2) * 2 > kHvpMaxW) return p;
  p.W = (int)cdiv(cdiv(n, p.C), 2) * 2;
  p.K = (int)cdiv(p.W, 2 * kHvpThreads);
  const size_t row_bytes = (size_t)p.W * 8;
  p.S = (int)tmin<int64_t>(8, (kHvpSmemBudget - 1024) / row_bytes);
  if (p.S < (p.C > 1 ? 3 : 2)) return p;
  p.smem = (size_t)p.S * row_bytes + (size_t)p.S * 8 + 1024;
  p.nclusters = kNumSMs / p.C;
  p.nclusters = (int)tmax<int64_t>(1, tmin<int64_t>(p.nclusters, rows));
  p.ok = true;
  return p;
}

template <int K>
static int hvp_fused_launch_k(const HvpPlan& p, const double* A, int64_t rows, int64_t n, int64_t lda,
                              const double* d, const double* v, double* ypart, cudaStream_t st,
                              const double* pred) {
  static bool attr0 = false, attr1 = false;  // one attribute call per instantiation
  if (p.C == 1) {
    auto fn = hvp_fused_kernel<K, false>;
    if (!attr0) {
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kHvpSmemBudget);
      attr0 = true;
    }
    fn<<<p.nclusters, kHvpThreads, p.smem, st>>>(A, rows, n, lda, d, v, p.W, p.S, ypart, pred);
    NYS_CHECK_LAUNCH();
    return NYS_OK;
  }
  auto fn = hvp_fused_kernel<K, true>;
  if (!attr1) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kHvpSmemBudget);
    cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr1 = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.nclusters * p.C, 1, 1);
  cfg.blockDim = dim3(kHvpThreads, 1, 1);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = p.C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, fn, A, rows, n, lda, d, v, p.W, p.S, ypart, pred) != cudaSuccess)
    return NYS_ERR_CUDA;
  __atomic_fetch_add(&g_launches, 1ull, __ATOMIC_RELAXED);
  return NYS_OK;
}

int hvp_fused(const HvpPlan& p, const double* A, int64_t rows, int64_t n, int64_t lda, const double* d,
              const double* v, double* ypart, cudaStream_t st, const double* pred) {
  switch (p.K) {
#define NYS_K(k) \
  case k: return hvp_fused_launch_k<k>(p, A, rows, n, lda, d, v, ypart, st, pred);
    NYS_K(1) NYS_K(2) NYS_K(3) NYS_K(4) NYS_K(5) NYS_K(6) NYS_K(7) NYS_K(8) NYS_K(9) NYS_K(10) NYS_K(11)
    NYS_K(12) NYS_K(13)
#undef NYS_K
    default: return NYS_ERR_UNSUPPORTED;
  }
}

}  // namespace nys
