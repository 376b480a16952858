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
  uint64_t* empty = full + S;                                          // S (16 warp arrivals)
  uint64_t* dotb = empty + S;                                          // S (16 warp arrivals)
  uint64_t* totb = dotb + S;                                           // NT (tx from the cluster)
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int cluster_id = blockIdx.x / kHcC, nclusters = gridDim.x / kHcC;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t c0 = (int64_t)rank * W;
  const int w_here = (int)tmax<int64_t>(0, tmin<int64_t>((int64_t)W, n - c0));
  const unsigned bytes = (unsigned)w_here * 8u;
  const int64_t nrows_mine = rows > cluster_id ? (rows - cluster_id + nclusters - 1) / nclusters : 0;

  if (tid == 0) {
    for (int q = 0; q < S; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], kHcWarps);
      mbar_init(&dotb[q], kHcWarps);
    }
    for (int q = 0; q < kHcNT; ++q) mbar_init(&totb[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // first use of every total slot: one local arrival + 16 x 8 bytes from the cluster
    for (int q = 0; q < kHcNT; ++q) mbar_expect_tx(&totb[q], kHcC * 8u);
  }
  cl.sync();  // every CTA's barriers are initialised and armed before any st.async

  if (warp == kHcWarps) {
    // ---------------------------------------------------------- producer --
    if (lane == 0 && bytes > 0) {
      for (int64_t g = 0; g < nrows_mine; ++g) {
        const int q = (int)(g % S);
        if (g >= S) mbar_wait(&empty[q], (unsigned)(((g / S) - 1) & 1));
        const int64_t i = cluster_id + g * nclusters;
        mbar_expect_tx(&full[q], bytes);
        tma_load_1d(ring + (size_t)q * W, A + i * lda + c0, bytes, &full[q]);
      }
    }
  } else if (warp > kHcWarps) {
    // --------------------------------------------------- exchange (relay) --
    const int xr = warp - kHcWarps - 1;  // rows g = xr (mod kHcX)
    for (int64_t g = xr; g < nrows_mine; g += kHcX) {
      const int q = (int)(g % S);
      const int64_t i = cluster_id + g * nclusters;
      const double di = d ? __ldg(d + i) : 1.0;
      mbar_wait(&dotb[q], (unsigned)((g / S) & 1));
      double p = lane < kHcWarps ? psl[q * kHcWarps + lane] : 0.0;
      // fixed-order tree over the 16 warp partials (lanes 0..15)
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
      p *= di;
      const int s = (int)(g % kHcNT);
      if (lane < kHcC) st_async_remote_f64(tsl + s * kHcC + rank, &totb[s], (unsigned)lane, p);
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
    for (int64_t it = 0; it < nrows_mine + L; ++it) {
      if (it < nrows_mine) {
        const int q = (int)(it % S);
        if (bytes > 0) mbar_wait(&full[q], (unsigned)((it / S) & 1));
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
        if (lane == 0) {
          psl[q * kHcWarps + warp] = pt;
          mbar_arrive(&dotb[q]);  // release: the slot write is visible to the relay warp
        }
      }
      const int64_t jt = it - L;
      if (jt < 0) continue;
      const int s = (int)(jt % kHcNT);
      mbar_wait_cluster(&totb[s], (unsigned)((jt / kHcNT) & 1));
      double t = 0.0;  // d_i (a_i . v): the 16 CTA partials (already scaled) in a fixed order
#pragma unroll
      for (int q2 = 0; q2 < kHcC; ++q2) t += tsl[s * kHcC + q2];
      if (warp == 0 && lane == 0) mbar_expect_tx(&totb[s], kHcC * 8u);  // re-arm for row jt + NT
      const int q = (int)(jt % S);
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
      if (lane == 0) mbar_arrive(&empty[q]);
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
  p.S = (int)tmin<int64_t>(8, (int64_t)((kHcSmemBudget - fixed) / (row_bytes + kHcWarps * 8 + 24)));
  if (p.S < 3) return p;
  static const int forced_lag = getenv("NYS_HVP_CLUSTER_LAG") ? atoi(getenv("NYS_HVP_CLUSTER_LAG")) : 0;
  p.L = forced_lag > 0 ? forced_lag : p.S - 2;
  p.L = tmax(1, tmin(p.L, p.S - 1));
  if (p.S + p.L + 2 > kHcNT) return p;
  p.smem = (size_t)p.S * (row_bytes + kHcWarps * 8) + (size_t)kHcNT * kHcC * 8 + (size_t)(3 * p.S + kHcNT) * 8;
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
