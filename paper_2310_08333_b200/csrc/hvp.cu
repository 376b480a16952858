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
#include "tma.cuh"

namespace cg = cooperative_groups;

namespace nys {

constexpr int kHvpThreads = 512;
constexpr int kHvpMaxW = 12800;
constexpr int kHvpMaxK = (kHvpMaxW + 2 * kHvpThreads - 1) / (2 * kHvpThreads);  // 13
constexpr int kHvpSmemBudget = 200 * 1024;

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
      const int s = (int)((unsigned)it % (unsigned)S);
      const double* row = ring + (size_t)s * W;
      if (bytes > 0) mbar_wait(&full[s], (((unsigned)it / (unsigned)S) & 1u));
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
    const int sj = (int)((unsigned)jt % (unsigned)S);
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

// Single-CTA-per-row-slice variant (C = 1, n <= 12800) with the CG finish
// fused in.  Per row: partial dot -> barrier -> every warp forms the row scale
// t from the 16 warp partials itself (fixed order, no serial thread-0 sum and
// no second broadcast barrier) -> axpy -> barrier -> refill of the stage with
// row + S, so each load has a full row of work to hide behind.  After the rows,
// the CTAs (one per SM, cooperative launch) meet at a grid barrier and CTA b
// sums the 148 y partials of its column slice in a fixed order, adds shift v
// and the v.y partial; the last CTA sums the partials in a fixed order (p.Ap).
template <int K, int P>
__global__ void __launch_bounds__(kHvpThreads, 1)
hvp_row_kernel(const double* __restrict__ A, int64_t rows, int64_t n, int64_t lda,
               const double* __restrict__ d, const double* __restrict__ v, int W, int S,
               double* __restrict__ ypart, double* __restrict__ y, double shift, double* __restrict__ dot,
               double* __restrict__ part, unsigned int* counter, const double* __restrict__ pred) {
  // P pieces per row (P = 2: half rows, so 2.5 rows fit the ring and ~1.5 rows
  // of loads stay in flight while a row is processed); S = number of pieces
  if (pred && *pred != 0.0) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int Wp = W / P;                                                  // piece width (doubles)
  double* ring = reinterpret_cast<double*>(smem_raw);                   // S x Wp
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)S * Wp);  // S mbarriers
  double* red = reinterpret_cast<double*>(full + S);                    // 2 x 16 warp partials
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nctas = gridDim.x, cta = blockIdx.x;
  const int w_here = (int)n;
  double2 vr[K], yr[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int j = 2 * (tid + k * kHvpThreads);
    vr[k] = (j < w_here) ? *reinterpret_cast<const double2*>(v + j) : make_double2(0.0, 0.0);
    yr[k] = make_double2(0.0, 0.0);
  }
  if (tid == 0) {
    for (int q = 0; q < S; ++q) mbar_init(&full[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t nrows_mine = rows > cta ? (rows - cta + nctas - 1) / nctas : 0;
  const int64_t npieces = nrows_mine * P;
  const unsigned pbytes = (unsigned)Wp * 8u;
  auto issue = [&](int64_t g) {  // piece g = row g / P, part g % P, into stage g % S
    const int q = (int)((unsigned)g % (unsigned)S);
    const int64_t i = cta + (g / P) * nctas;
    mbar_expect_tx(&full[q], pbytes);
    tma_load_1d(ring + (size_t)q * Wp, A + i * lda + (g % P) * Wp, pbytes, &full[q]);
  };
  if (tid == 0)
    for (int64_t g = 0; g < S && g < npieces; ++g) issue(g);
  for (int64_t it = 0; it < nrows_mine; ++it) {
    // the row weight is fetched before the dot so its latency hides behind it
    const int64_t i = cta + it * nctas;
    const double di = d ? __ldg(d + i) : 1.0;
    const double* pc[P];
#pragma unroll
    for (int h = 0; h < P; ++h) {
      const int64_t g = it * P + h;
      const int q = (int)((unsigned)g % (unsigned)S);
      pc[h] = ring + (size_t)q * Wp;
      mbar_wait(&full[q], ((unsigned)g / (unsigned)S) & 1u);
    }
    const double* pc0 = pc[0];
    const double* pc1 = pc[P - 1] - Wp;  // P == 2: pc1 + j addresses the second half
    auto elem = [&](int j) -> const double* { return (P == 1 || j < Wp) ? pc0 + j : pc1 + j; };
    double pt = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int j = 2 * (tid + k * kHvpThreads);
      if (j < w_here) {
        const double2 a = *reinterpret_cast<const double2*>(elem(j));
        pt = fma(a.x, vr[k].x, pt);
        pt = fma(a.y, vr[k].y, pt);
      }
    }
    pt = warp_sum(pt);
    if (lane == 0) red[(it & 1) * 16 + warp] = pt;
    __syncthreads();
    // every warp forms t of row it (same fixed-order sum in every warp)
    const double tot = warp_sum(lane < kHvpThreads / 32 ? red[(it & 1) * 16 + lane] : 0.0);
    const double t = d ? di * tot : tot;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int j = 2 * (tid + k * kHvpThreads);
      if (j < w_here) {
        const double2 a = *reinterpret_cast<const double2*>(elem(j));
        yr[k].x = fma(t, a.x, yr[k].x);
        yr[k].y = fma(t, a.y, yr[k].y);
      }
    }
    __syncthreads();  // the row's stages are free
    if (tid == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#pragma unroll
      for (int h = 0; h < P; ++h) {
        const int64_t g = it * P + h + S;
        if (g < npieces) issue(g);
      }
    }
  }
  double* yp = ypart + (int64_t)cta * n;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int j = 2 * (tid + k * kHvpThreads);
    if (j < w_here) *reinterpret_cast<double2*>(yp + j) = yr[k];
  }
  cg::this_grid().sync();
  // column slice of this CTA: fixed-order sum over the nctas partials
  __shared__ double cs_acc[8][65];
  __shared__ double dsh[32];
  const int64_t slice = ((n + nctas - 1) / nctas + 1) & ~1ll;
  const int64_t c_begin = (int64_t)cta * slice, c_end = tmin<int64_t>(n, c_begin + slice);
  double dacc[1] = {0.0};
  for (int64_t cb = c_begin; cb < c_end; cb += 64) {
    const int cx = tid & 63, ch = tid >> 6;  // 64 columns x 8 chunks
    const int64_t c = cb + cx;
    double acc = 0.0;
    if (c < c_end)
      for (int q = ch; q < nctas; q += 8) acc += ypart[(int64_t)q * n + c];
    cs_acc[ch][cx] = acc;
    __syncthreads();
    if (ch == 0 && c < c_end) {
      double a = cs_acc[0][cx];
#pragma unroll
      for (int q = 1; q < 8; ++q) a += cs_acc[q][cx];
      // the shift is part of the operator whether or not p.Ap is wanted (the
      // CG's true-residual refresh applies it to x with no dot, krylov.py:80-81)
      if (dot || shift != 0.0) a += shift * v[c];
      if (dot) dacc[0] = fma(v[c], a, dacc[0]);
      y[c] = a;
    }
    __syncthreads();
  }
  if (!dot) return;
  block_sum<1>(dacc, dsh);
  if (tid == 0) part[cta] = dacc[0];
  if (last_block(counter)) {
    const double tot = block_sum_partials(part, nctas, 1, dsh);
    if (tid == 0) *dot = tot;
  }
}

struct HvpPlan {
  int C, W, K, S, nclusters;
  size_t smem;
  bool ok;
  int P;  // C = 1 row kernel: pieces per row (S then counts pieces)
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
  static const int forced = dev_env("NYS_HVP_C") ? atoi(dev_env("NYS_HVP_C")) : 0;
  if (forced > 0) p.C = forced;
  if (p.C > 16 || cdiv(cdiv(n, p.C), 2) * 2 > kHvpMaxW) return p;
  p.W = (int)cdiv(cdiv(n, p.C), 2) * 2;
  p.K = (int)cdiv(p.W, 2 * kHvpThreads);
  const size_t row_bytes = (size_t)p.W * 8;
  p.S = (int)tmin<int64_t>(8, (kHvpSmemBudget - 1024) / row_bytes);
  if (p.S < (p.C > 1 ? 3 : 2)) return p;
  p.smem = (size_t)p.S * row_bytes + (size_t)p.S * 8 + 1024;
  // (half-row TMA pieces, P = 2, were measured slower on B200: the kernel is
  // bound by the shared-memory passes over each row, not by loads in flight)
  p.P = 1;
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

template <int K, int P>
static int hvp_row_launch_k(const HvpPlan& p, const double* A, int64_t rows, int64_t n, int64_t lda,
                            const double* d, const double* v, double* ypart, double* y, double shift, double* dot,
                            double* part, unsigned int* counter, cudaStream_t st, const double* pred) {
  static bool attr = false;
  auto fn = hvp_row_kernel<K, P>;
  if (!attr) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kHvpSmemBudget);
    attr = true;
  }
  int S = p.S;  // pieces in the ring
  int W = p.W;
  void* args[] = {(void*)&A, (void*)&rows, (void*)&n, (void*)&lda, (void*)&d, (void*)&v, (void*)&W, (void*)&S,
                  (void*)&ypart, (void*)&y, (void*)&shift, (void*)&dot, (void*)&part, (void*)&counter,
                  (void*)&pred};
  if (!coop_fits((const void*)fn, p.nclusters, kHvpThreads, p.smem)) return NYS_ERR_UNSUPPORTED;
  const int rc = coop_launch_status(
      cudaLaunchCooperativeKernel((const void*)fn, dim3(p.nclusters), dim3(kHvpThreads), args, p.smem, st));
  if (rc) return rc;
  __atomic_fetch_add(&g_launches, 1ull, __ATOMIC_RELAXED);
  return debug_sync_check(__FILE__, __LINE__) ? NYS_ERR_CUDA : NYS_OK;
}

// C = 1 plans: rows pipeline + fused finish (y = sum of partials [+ shift v],
// dot = v.y when dot != nullptr) in one cooperative launch
int hvp_row(const HvpPlan& p, const double* A, int64_t rows, int64_t n, int64_t lda, const double* d,
            const double* v, double* ypart, double* y, double shift, double* dot, double* part,
            unsigned int* counter, cudaStream_t st, const double* pred) {
  switch (p.K) {
#define NYS_K(k) \
  case k: return hvp_row_launch_k<k, 1>(p, A, rows, n, lda, d, v, ypart, y, shift, dot, part, counter, st, pred);
    NYS_K(1) NYS_K(2) NYS_K(3) NYS_K(4) NYS_K(5) NYS_K(6) NYS_K(7) NYS_K(8) NYS_K(9) NYS_K(10) NYS_K(11)
    NYS_K(12) NYS_K(13)
#undef NYS_K
    default: return NYS_ERR_UNSUPPORTED;
  }
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
