// K3 for wide rows (configs 4/5): y_c = A_c^T (d o (A_c v)) per thread-block
// cluster, A streamed from HBM once (problems.py:263-264 MLHessian._apply).
//
// A cluster of C = 16 CTAs owns every nclusters-th row; CTA q of the cluster
// owns the column segment [q W, q W + W), W = n / 16 (50 KB of a row at
// n = 1e5), with its v and y segments in registers.  Warp roles, synchronised
// only through mbarriers (no CTA-wide barriers in the loop):
//   * producer warp: TMA bulk copies of row segments into an S-stage ring;
//   * 16 compute warps: per row, the partial dot over the warp's columns into
//     a shared-memory slot; L rows later the row's t = d_i (a_i . v) from the
//     cluster, then y += t a_i from the still-staged segment;
//   * 2 exchange warps (even / odd rows, so two relay chains run at once): the
//     fixed-order sum of the 16 warp partials, times d_i, sent to all 16 CTAs
//     of the cluster by st.async into their row-total slots (remote mbarrier
//     complete_tx, 16 x 8 B per row and CTA); every CTA then sums the 16 CTA
//     partials in the same fixed order (deterministic, identical everywhere).
// (Sending all 256 warp partials directly, without the relay, was measured 2x
// slower: 256 complete_tx per row serialise on the receiving mbarrier.)
// The row-total exchange stays inside the cluster's distributed shared memory
// (sub-microsecond), unlike the grid-wide strip kernel's L2 exchange.  Each
// cluster writes its y partial; a fixed-order reduction over the clusters adds
// shift v and p.Ap (gemv.cu: gemv_t_reduce).
#include <cooperative_groups.h>
#include <stdlib.h>
#include "common.cuh"
#include "tma.cuh"

namespace cg = cooperative_groups;

namespace nys {

constexpr int kHcC = 16;                        // CTAs per cluster
constexpr int kHcWarps = 16;                    // compute warps
constexpr int kHcX = 2;                         // exchange (relay) warps
constexpr int kHcThreads = (kHcWarps + 1 + kHcX) * 32;  // + producer + relays
constexpr int kHcNT = 16;                       // row-total slots (> S + L + margin)
constexpr int kHcSmemBudget = 220 * 1024;
constexpr int kHcMaxS = 6;                      // named barriers 1..6 (empty), 7..12 (dot)
constexpr int kHcBarThreads = (kHcWarps + 1) * 32;  // 16 compute warps + the producer / one relay

// Hardware named barriers for the intra-CTA stage hand-offs (a 16-warp mbarrier
// arrival per row serialised on the shared-memory atomics).  bar.arrive by the
// 16 compute warps, bar.sync by the producer (stage free) or a relay warp
// (partials written); the arrive orders the warps' prior shared-memory
// accesses before the sync returns.
__device__ __forceinline__ void nbar_arrive(int id) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(kHcBarThreads) : "memory");
}
__device__ __forceinline__ void nbar_sync(int id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(kHcBarThreads) : "memory");
}

template <int K>
__global__ void __launch_bounds__(kHcThreads, 1)
hvp_cluster_kernel(const double* __restrict__ A, int64_t rows, int64_t n, int64_t lda,
                   const double* __restrict__ d, const double* __restrict__ v, int W, int S, int L,
                   double* __restrict__ ypart, const double* __restrict__ pred) {
  if (pred && *pred != 0.0) return;  // every CTA of every cluster sees the same flag
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw);                  // S x W
  double* psl = ring + (size_t)S * W;                                  // S x 16 warp partials
  double* tsl = psl + (size_t)S * kHcWarps;                            // NT x 16 CTA partials
  uint64_t* full = reinterpret_cast<uint64_t*>(tsl + kHcNT * kHcC);    // S
  uint64_t* totb = full + S;                                           // NT (tx from the cluster)
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int cluster_id = blockIdx.x / kHcC, nclusters = gridDim.x / kHcC;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t c0 = (int64_t)rank * W;
  const int w_here = (int)tmax<int64_t>(0, tmin<int64_t>((int64_t)W, n - c0));
  const unsigned bytes = (unsigned)w_here * 8u;
  const int64_t nrows_mine = rows > cluster_id ? (rows - cluster_id + nclusters - 1) / nclusters : 0;

  if (tid == 0) {
    for (int q = 0; q < S; ++q) mbar_init(&full[q], 1);
    for (int q = 0; q < kHcNT; ++q) mbar_init(&totb[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // first use of every total slot: one local arrival + 16 x 8 bytes from the cluster
    for (int q = 0; q < kHcNT; ++q) mbar_expect_tx(&totb[q], kHcC * 8u);
  }
  cl.sync();  // every CTA's barriers are initialised and armed before any st.async

  if (warp == kHcWarps) {
    // ---------------------------------------------------------- producer --
    // (the whole warp takes part in the stage barriers; lane 0 issues the copies)
    // (stage indices kept incrementally: no 64-bit divisions in the row loops)
    const int nr = (int)nrows_mine;
    const double* arow = A + (int64_t)cluster_id * lda + c0;
    const int64_t rstep = (int64_t)nclusters * lda;
    for (int g = 0, q = 0; g < nr; ++g, arow += rstep) {
      if (g >= S) nbar_sync(1 + q);  // the 16 compute warps are done with row g - S
      if (lane == 0 && bytes > 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&full[q], bytes);
        tma_load_1d(ring + (size_t)q * W, arow, bytes, &full[q]);
      }
      if (++q == S) q = 0;
    }
    // consume the stage-free arrivals of the last rows (no refill follows them)
    for (int g = tmax(0, nr - S); g < nr; ++g) nbar_sync(1 + g % S);
  } else if (warp > kHcWarps) {
    // --------------------------------------------------- exchange (relay) --
    const int xr = warp - kHcWarps - 1;  // rows g = xr (mod kHcX)
    const int nr = (int)nrows_mine;
    int q = xr % S;
    for (int g = xr; g < nr; g += kHcX) {
      const int64_t i = cluster_id + (int64_t)g * nclusters;
      const double di = d ? __ldg(d + i) : 1.0;
      nbar_sync(1 + kHcMaxS + q);  // the 16 warp partials of row g are in psl
      double p = lane < kHcWarps ? psl[q * kHcWarps + lane] : 0.0;
      // fixed-order tree over the 16 warp partials (lanes 0..15)
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
      p *= di;
      const int s = g & (kHcNT - 1);
      if (lane < kHcC) st_async_remote_f64(tsl + s * kHcC + rank, &totb[s], (unsigned)lane, p);
      q += kHcX;
      while (q >= S) q -= S;
    }
  } else {
    // ---------------------------------------------------------- compute --
    double2 vr[K], yr[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int j = 2 * (tid + k * kHcWarps * 32);
      vr[k] = (j < w_here) ? *reinterpret_cast<const double2*>(v + c0 + j) : make_double2(0.0, 0.0);
      yr[k] = make_double2(0.0, 0.0);
    }
    const int nr = (int)nrows_mine;
    int qi = 0, pi = 0;  // stage and phase of row it
    int qj = 0;          // stage of row jt = it - L
    for (int it = 0; it < nr + L; ++it) {
      if (it < nr) {
        const int q = qi;
        if (bytes > 0) mbar_wait(&full[q], (unsigned)pi);
        if (++qi == S) {
          qi = 0;
          pi ^= 1;
        }
        const double* row = ring + (size_t)q * W;
        double pt = 0.0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int j = 2 * (tid + k * kHcWarps * 32);
          if (j < w_here) {
            const double2 a = *reinterpret_cast<const double2*>(row + j);
            pt = fma(a.x, vr[k].x, pt);
            pt = fma(a.y, vr[k].y, pt);
          }
        }
        pt = warp_sum(pt);
        if (lane == 0) psl[q * kHcWarps + warp] = pt;
        __syncwarp();
        nbar_arrive(1 + kHcMaxS + q);
      }
      const int jt = it - L;
      if (jt < 0) continue;
      const int s = jt & (kHcNT - 1);
      mbar_wait_cluster(&totb[s], (unsigned)((jt / kHcNT) & 1));
      double t = 0.0;  // d_i (a_i . v): the 16 CTA partials (already scaled) in a fixed order
#pragma unroll
      for (int q2 = 0; q2 < kHcC; ++q2) t += tsl[s * kHcC + q2];
      if (warp == 0 && lane == 0) mbar_expect_tx(&totb[s], kHcC * 8u);  // re-arm for row jt + NT
      const int q = qj;
      if (++qj == S) qj = 0;
      const double* row = ring + (size_t)q * W;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int j = 2 * (tid + k * kHcWarps * 32);
        if (j < w_here) {
          const double2 a = *reinterpret_cast<const double2*>(row + j);
          yr[k].x = fma(t, a.x, yr[k].x);
          yr[k].y = fma(t, a.y, yr[k].y);
        }
      }
      __syncwarp();
      nbar_arrive(1 + q);  // stage q free for the producer
    }
    double* yp = ypart + (int64_t)cluster_id * n + c0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int j = 2 * (tid + k * kHcWarps * 32);
      if (j < w_here) *reinterpret_cast<double2*>(yp + j) = yr[k];
    }
  }
  cl.sync();  // no CTA leaves while a peer may still write into its shared memory
}

struct HcPlan {
  int W, K, S, L, nclusters;
  size_t smem;
  bool ok;
};

HcPlan hvp_cluster_plan(int64_t rows, int64_t n, int64_t lda, const double* A, const double* v) {
  HcPlan p{};
  p.ok = false;
  static const bool off = getenv("NYS_HVP_CLUSTER_OFF") != nullptr;
  if (off || (lda & 1) || (n & 1) || ((uintptr_t)A & 15) || ((uintptr_t)v & 15) || rows < 1) return p;
  p.W = (int)cdiv(cdiv(n, kHcC), 2) * 2;
  p.K = (int)cdiv(p.W / 2, kHcWarps * 32);
  if (p.K > 12) return p;
  const size_t fixed = (size_t)(kHcNT * kHcC) * 8 + kHcNT * 8 + 1024;
  const size_t row_bytes = (size_t)p.W * 8;
  p.S = (int)tmin<int64_t>(kHcMaxS, (int64_t)((kHcSmemBudget - fixed) / (row_bytes + kHcWarps * 8 + 24)));
  if (p.S < 3) return p;
  static const int forced_lag = getenv("NYS_HVP_CLUSTER_LAG") ? atoi(getenv("NYS_HVP_CLUSTER_LAG")) : 0;
  // lag 1 measured best on B200 (n = 1e5, S = 4: 2.32 ms vs 2.80 ms at lag 2 -
  // the exchange is sub-microsecond, the extra stage in flight is worth more)
  p.L = forced_lag > 0 ? forced_lag : 1;
  p.L = tmax(1, tmin(p.L, p.S - 1));
  if (p.S + p.L + 2 > kHcNT) return p;
  p.smem = (size_t)p.S * (row_bytes + kHcWarps * 8) + (size_t)kHcNT * kHcC * 8 + (size_t)(p.S + kHcNT) * 8;
  p.nclusters = 0;
  p.ok = true;
  return p;
}

template <int K>
static int hvp_cluster_launch_k(HcPlan& p, const double* A, int64_t rows, int64_t n, int64_t lda, const double* d,
                                const double* v, double* ypart, cudaStream_t st, const double* pred) {
  auto fn = hvp_cluster_kernel<K>;
  static bool attr = false;
  static int maxc = 0;
  if (!attr) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kHcSmemBudget);
    cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kHcThreads, 1, 1);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kHcC;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (maxc == 0) {
    // clusters of 16 that fit at once (one wave: a second partial wave would
    // double the tail), at most 148 / 16
    cfg.gridDim = dim3(kHcC * (kNumSMs / kHcC), 1, 1);
    int mc = 0;
    if (cudaOccupancyMaxActiveClusters(&mc, (void*)fn, &cfg) != cudaSuccess || mc < 1) {
      cudaGetLastError();
      return NYS_ERR_UNSUPPORTED;
    }
    maxc = tmin(mc, kNumSMs / kHcC);
  }
  p.nclusters = (int)tmax<int64_t>(1, tmin<int64_t>(maxc, rows));
  cfg.gridDim = dim3(kHcC * p.nclusters, 1, 1);
  int W = p.W, S = p.S, L = p.L;
  if (cudaLaunchKernelEx(&cfg, fn, A, rows, n, lda, d, v, W, S, L, ypart, pred) != cudaSuccess) return NYS_ERR_CUDA;
  __atomic_fetch_add(&g_launches, 1ull, __ATOMIC_RELAXED);
  return debug_sync_check(__FILE__, __LINE__) ? NYS_ERR_CUDA : NYS_OK;
}

// ypart: (plan.nclusters <= 9) x n partials; returns the cluster count used in *ncl
int hvp_cluster(HcPlan& p, const double* A, int64_t rows, int64_t n, int64_t lda, const double* d,
                const double* v, double* ypart, cudaStream_t st, const double* pred) {
  switch (p.K) {
#define NYS_K(k) \
  case k: return hvp_cluster_launch_k<k>(p, A, rows, n, lda, d, v, ypart, st, pred);
    NYS_K(1) NYS_K(2) NYS_K(3) NYS_K(4) NYS_K(5) NYS_K(6) NYS_K(7) NYS_K(8) NYS_K(9) NYS_K(10) NYS_K(11)
    NYS_K(12)
#undef NYS_K
    default: return NYS_ERR_UNSUPPORTED;
  }
}

}  // namespace nys
