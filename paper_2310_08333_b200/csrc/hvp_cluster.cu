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
#include <stdio.h>
#include <stdlib.h>
#include "common.cuh"
#include "tma.cuh"
#include "hvp_plan.cuh"
#include "loss.cuh"

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

// The 16 CTA partials of a row total, summed by a fixed shuffle tree within
// each 16-lane half of the warp (lanes l and l + 16 load partial l & 15 of
// slot p + (l >> 4) * 16): one shared-memory load and four adds per thread
// instead of sixteen each.  Every thread of every CTA gets the same bits.
__device__ __forceinline__ double cluster_total_halves(const double* p, int lane) {
  double v = p[(lane >> 4) * kHcC + (lane & 15)];
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int K>
__global__ void __launch_bounds__(kHcThreads, 1)
hvp_cluster_kernel(const double* __restrict__ A, int64_t rows, int64_t n, int64_t lda,
                   const double* __restrict__ d, const double* __restrict__ v, int W, int S, int L,
                   double* __restrict__ ypart, const double* __restrict__ pred) {
  if (pred && *pred != 0.0) return;  // every CTA of every cluster sees the same flag
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw);                  // S x W
  double* psl = ring + (size_t)S * W;                                  // S x 512 lane partials
  double* tsl = psl + (size_t)S * kHcWarps * 32;                       // NT x 16 CTA partials
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
      nbar_sync(1 + kHcMaxS + q);  // the 512 lane partials of row g are in psl
      // lane l: the 16 warps' lane-l partials in warp order, then a shuffle tree
      const double* pp = psl + (size_t)q * kHcWarps * 32 + lane;
      double p = 0.0;
#pragma unroll
      for (int w2 = 0; w2 < kHcWarps; ++w2) p += pp[w2 * 32];
      p = warp_sum(p) * di;
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
        psl[((size_t)q * kHcWarps + warp) * 32 + lane] = pt;  // reduced by a relay warp
        __syncwarp();
        nbar_arrive(1 + kHcMaxS + q);
      }
      const int jt = it - L;
      if (jt < 0) continue;
      const int s = jt & (kHcNT - 1);
      mbar_wait(&totb[s], (unsigned)((jt / kHcNT) & 1));  // st.async complete_tx: CTA-scope acquire (no L1 invalidation)
      // d_i (a_i . v): the 16 CTA partials (already scaled), fixed-order tree
      const double t = __shfl_sync(0xffffffffu, cluster_total_halves(tsl + s * kHcC, lane & 15), 0);
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

// Wide rows whose per-CTA segment (W = n / 16 columns) cannot be staged whole
// with v and y in registers (n = 200000: 100 KB of a row per CTA, the per-GPU
// shape of config 5).  The segment is split into Q sub-segments of Wq columns;
// y stays in registers, v moves to TENSOR MEMORY (tcgen05.st once, one
// tcgen05.ld of 16 words per sub-segment and row: TMEM has its own datapath,
// so v costs neither registers nor shared memory), and the freed shared memory
// becomes a deep ring of sub-segment stages.  Per row the producer streams the
// Q sub-segments once for the dot (HBM) and, after the cluster exchange of the
// row total (one row later), once more for the axpy y += t a -- the second read
// hits L2 (the row was read microseconds earlier), so HBM still sees A exactly
// once.  Stage uses, in the order both the producer and the compute warps walk
// them:
//     for it: [dot(it, 0..Q-1) if it < nr] [axpy(it - L, 0..Q-1) if it >= L]
// Named barriers: 1..S stage free (compute arrive, producer sync), 9..12 row
// partials written (compute arrive, relay sync; 4 row slots, so an id is reused
// only after its relay has synced, which the stream order guarantees for L = 1).
constexpr int kRedPartialsTail = 4096;  // reduction scratch ahead of the A^T partials (vec.cu layout)
constexpr int kHqNR = 4;    // row slots of the warp partials
constexpr int kHqMaxS = 8;  // stage barriers 1..8, row barriers 9..12
constexpr int kHqTmemCols = 256;
// 14 compute warps + producer + relay = 16 warps: 4 per SM sub-partition, so
// each thread may use 128 registers (18 warps would cap it at 96 and spill)
constexpr int kHqWarps = 14;
constexpr int kHqX = 1;
constexpr int kHqThreads = (kHqWarps + 1 + kHqX) * 32;
constexpr int kHqBarThreads = (kHqWarps + 1) * 32;
__device__ __forceinline__ void qbar_arrive(int id) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(kHqBarThreads) : "memory");
}
__device__ __forceinline__ void qbar_sync(int id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(kHqBarThreads) : "memory");
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const double2 (&x)[4]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(taddr),
      "r"(__double2loint(x[0].x)), "r"(__double2hiint(x[0].x)), "r"(__double2loint(x[0].y)),
      "r"(__double2hiint(x[0].y)), "r"(__double2loint(x[1].x)), "r"(__double2hiint(x[1].x)),
      "r"(__double2loint(x[1].y)), "r"(__double2hiint(x[1].y)), "r"(__double2loint(x[2].x)),
      "r"(__double2hiint(x[2].x)), "r"(__double2loint(x[2].y)), "r"(__double2hiint(x[2].y)),
      "r"(__double2loint(x[3].x)), "r"(__double2hiint(x[3].x)), "r"(__double2loint(x[3].y)),
      "r"(__double2hiint(x[3].y))
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, double2 (&x)[4]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, "
      "[%16];\n"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    x[k].x = __hiloint2double((int)r[4 * k + 1], (int)r[4 * k + 0]);
    x[k].y = __hiloint2double((int)r[4 * k + 3], (int)r[4 * k + 2]);
  }
}

// x and z slices of one pair of double2 columns each (two x8 loads, one wait)
__device__ __forceinline__ void tmem_ld8x2(uint32_t ta, uint32_t tb, double2 (&x)[2], double2 (&z)[2]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%16];\n"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%8, %9, %10, %11, %12, %13, %14, %15}, [%17];\n"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(ta), "r"(tb)
      : "memory");
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    x[k].x = __hiloint2double((int)r[4 * k + 1], (int)r[4 * k + 0]);
    x[k].y = __hiloint2double((int)r[4 * k + 3], (int)r[4 * k + 2]);
    z[k].x = __hiloint2double((int)r[8 + 4 * k + 1], (int)r[8 + 4 * k + 0]);
    z[k].y = __hiloint2double((int)r[8 + 4 * k + 3], (int)r[8 + 4 * k + 2]);
  }
}

template <int Q, int KQ>
__global__ void __launch_bounds__(kHqThreads, 1)
hvp_cluster_q_kernel(const double* __restrict__ A, int64_t rows, int64_t n, int64_t lda,
                     const double* __restrict__ d, const double* __restrict__ v, int W, int Wq, int S,
                     double* __restrict__ ypart, const double* __restrict__ pred) {
  static_assert(KQ <= 4 && Q * 4 * 4 <= kHqTmemCols / 4, "v slice of a thread: <= 64 TMEM columns");
  constexpr int L = 1;
  if (pred && *pred != 0.0) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw);             // S x Wq
  double* psl = ring + (size_t)S * Wq;                            // NR x 448 lane partials
  double* tsl = psl + kHqNR * kHqWarps * 32;                      // NT x 16 CTA partials
  uint64_t* full = reinterpret_cast<uint64_t*>(tsl + kHcNT * kHcC);  // S
  uint64_t* totb = full + S;                                      // NT
  uint32_t* tmem_base = reinterpret_cast<uint32_t*>(totb + kHcNT);
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int cluster_id = blockIdx.x / kHcC, nclusters = gridDim.x / kHcC;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t c0 = (int64_t)rank * W;
  const int w_here = (int)tmax<int64_t>(0, tmin<int64_t>((int64_t)W, n - c0));
  const int64_t nrows_mine = rows > cluster_id ? (rows - cluster_id + nclusters - 1) / nclusters : 0;

  if (tid == 0) {
    for (int q = 0; q < S; ++q) mbar_init(&full[q], 1);
    for (int q = 0; q < kHcNT; ++q) mbar_init(&totb[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int q = 0; q < kHcNT; ++q) mbar_expect_tx(&totb[q], kHcC * 8u);
  }
  if (warp == 0) {  // TMEM for v: one warp allocates (and later frees) the columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base)),
                 "n"(kHqTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cl.sync();  // barriers armed cluster-wide, TMEM address published
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // this warp's TMEM slice: lanes of its sub-partition, 64 columns per warp
  const uint32_t tv = *tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(64 * ((warp >> 2) & 3));

  const int nr = (int)nrows_mine;
  if (warp == kHqWarps) {
    // ---------------------------------------------------------- producer --
    const int64_t rstep = (int64_t)nclusters * lda;
    int u = 0, slot = 0;
    auto issue = [&](const double* seg_row) {
#pragma unroll 1
      for (int q = 0; q < Q; ++q, ++u) {
        if (u >= S) qbar_sync(1 + slot);  // use u - S is done with this slot
        const int wq = tmin(Wq, w_here - q * Wq);
        if (lane == 0) {
          if (wq > 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&full[slot], (unsigned)wq * 8u);
            tma_load_1d(ring + (size_t)slot * Wq, seg_row + (int64_t)q * Wq, (unsigned)wq * 8u, &full[slot]);
          } else {
            mbar_arrive(&full[slot]);  // empty sub-segment: complete the phase anyway
          }
        }
        if (++slot == S) slot = 0;
      }
    };
    const double* base = A + (int64_t)cluster_id * lda + c0;
    for (int it = 0; it < nr + L; ++it) {
      if (it < nr) issue(base + (int64_t)it * rstep);
      if (it >= L) issue(base + (int64_t)(it - L) * rstep);  // the axpy re-read (L2)
    }
    for (int w = tmax(0, u - S); w < u; ++w) qbar_sync(1 + w % S);
  } else if (warp > kHqWarps) {
    // --------------------------------------------------- exchange (relay) --
    const int xr = warp - kHqWarps - 1;
    for (int g = xr; g < nr; g += kHqX) {
      const int64_t i = cluster_id + (int64_t)g * nclusters;
      const double di = d ? __ldg(d + i) : 1.0;
      const int rs = g % kHqNR;
      qbar_sync(1 + kHqMaxS + rs);
      const double* pp = psl + rs * kHqWarps * 32 + lane;
      double p = 0.0;
#pragma unroll
      for (int w2 = 0; w2 < kHqWarps; ++w2) p += pp[w2 * 32];
      p = warp_sum(p) * di;
      const int s = g & (kHcNT - 1);
      if (lane < kHcC) st_async_remote_f64(tsl + s * kHcC + rank, &totb[s], (unsigned)lane, p);
    }
  } else {
    // ---------------------------------------------------------- compute --
    // v -> TMEM: sub-segment q of this thread at columns 16 q .. 16 q + 15
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      double2 x[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int j = 2 * (tid + k * kHqWarps * 32);
        const int wq = tmin(Wq, w_here - q * Wq);
        x[k] = (k < KQ && j < wq) ? *reinterpret_cast<const double2*>(v + c0 + (int64_t)q * Wq + j)
                                  : make_double2(0.0, 0.0);
      }
      tmem_st16(tv + 16 * q, x);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    double2 yr[Q][KQ];
#pragma unroll
    for (int q = 0; q < Q; ++q)
#pragma unroll
      for (int k = 0; k < KQ; ++k) yr[q][k] = make_double2(0.0, 0.0);
    int slot = 0, ph = 0;
    auto next = [&]() {
      if (++slot == S) {
        slot = 0;
        ph ^= 1;
      }
    };
    for (int it = 0; it < nr + L; ++it) {
      if (it < nr) {
        double pt = 0.0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int wq = tmin(Wq, w_here - q * Wq);
          double2 x[4];
          tmem_ld16(tv + 16 * q, x);
          mbar_wait(&full[slot], (unsigned)ph);
          const double* seg = ring + (size_t)slot * Wq;
#pragma unroll
          for (int k = 0; k < KQ; ++k) {
            const int j = 2 * (tid + k * kHqWarps * 32);
            if (j < wq) {
              const double2 a = *reinterpret_cast<const double2*>(seg + j);
              pt = fma(a.x, x[k].x, pt);
              pt = fma(a.y, x[k].y, pt);
            }
          }
          __syncwarp();
          qbar_arrive(1 + slot);
          next();
        }
        const int rs = it % kHqNR;
        psl[(rs * kHqWarps + warp) * 32 + lane] = pt;
        __syncwarp();
        qbar_arrive(1 + kHqMaxS + rs);
      }
      const int jt = it - L;
      if (jt < 0) continue;
      const int s = jt & (kHcNT - 1);
      mbar_wait(&totb[s], (unsigned)((jt / kHcNT) & 1));  // st.async complete_tx: CTA-scope acquire (no L1 invalidation)
      const double t = __shfl_sync(0xffffffffu, cluster_total_halves(tsl + s * kHcC, lane & 15), 0);
      if (warp == 0 && lane == 0) mbar_expect_tx(&totb[s], kHcC * 8u);
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int wq = tmin(Wq, w_here - q * Wq);
        mbar_wait(&full[slot], (unsigned)ph);
        const double* seg = ring + (size_t)slot * Wq;
#pragma unroll
        for (int k = 0; k < KQ; ++k) {
          const int j = 2 * (tid + k * kHqWarps * 32);
          if (j < wq) {
            const double2 a = *reinterpret_cast<const double2*>(seg + j);
            yr[q][k].x = fma(t, a.x, yr[q][k].x);
            yr[q][k].y = fma(t, a.y, yr[q][k].y);
          }
        }
        __syncwarp();
        qbar_arrive(1 + slot);
        next();
      }
    }
    double* yp = ypart + (int64_t)cluster_id * n + c0;
#pragma unroll
    for (int q = 0; q < Q; ++q)
#pragma unroll
      for (int k = 0; k < KQ; ++k) {
        const int j = 2 * (tid + k * kHqWarps * 32);
        if (j < tmin(Wq, w_here - q * Wq)) *reinterpret_cast<double2*>(yp + q * Wq + j) = yr[q][k];
      }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cl.sync();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_base), "n"(kHqTmemCols)
                 : "memory");
  }
}

HcPlan hvp_cluster_plan(int64_t rows, int64_t n, int64_t lda, const double* A, const double* v) {
  HcPlan p{};
  p.ok = false;
  static const bool off = dev_env("NYS_HVP_CLUSTER_OFF") != nullptr;
  if (off || (lda & 1) || (n & 1) || ((uintptr_t)A & 15) || ((uintptr_t)v & 15) || rows < 1) return p;
  p.W = (int)cdiv(cdiv(n, kHcC), 2) * 2;
  p.K = (int)cdiv(p.W / 2, kHcWarps * 32);
  p.Q = 1;
  p.Wq = p.W;
  const size_t fixed = (size_t)(kHcNT * kHcC) * 8 + kHcNT * 8 + 1024;
  const size_t row_bytes = (size_t)p.W * 8;
  p.S = p.K > 12 ? 0
                 : (int)tmin<int64_t>(kHcMaxS, (int64_t)((kHcSmemBudget - fixed) / (row_bytes + kHcWarps * 256 + 24)));
  static const bool no_q = dev_env("NYS_HVP_CLUSTER_NOQ") != nullptr;
  static const bool force_q = dev_env("NYS_HVP_CLUSTER_Q") != nullptr;
  if ((p.S < 3 || force_q) && !no_q) {
    // sub-segment plan: the smallest split with >= 4 stages in flight and the
    // y segment (Q x KQ double2 per thread) in registers
    const size_t qfixed = fixed + (size_t)kHqNR * kHqWarps * 32 * 8 + 16;
    static const int forced_q = dev_env("NYS_HVP_CLUSTER_Q") ? atoi(dev_env("NYS_HVP_CLUSTER_Q")) : 0;
    for (int Q = 2; Q <= 4; ++Q) {
      if (forced_q > 1 && Q != forced_q) continue;
      const int Wq = (int)cdiv(cdiv(p.W, Q), 2) * 2;
      const int KQ = (int)cdiv(Wq / 2, kHqWarps * 32);
      if (KQ > 4) continue;
      const int S = (int)tmin<int64_t>(kHqMaxS, (int64_t)((kHcSmemBudget - qfixed) / ((size_t)Wq * 8 + 8)));
      if (S < 4) continue;
      p.Q = Q;
      p.Wq = Wq;
      p.K = KQ;
      p.S = S;
      p.L = 1;
      p.smem = (size_t)S * Wq * 8 + (size_t)kHqNR * kHqWarps * 32 * 8 + (size_t)kHcNT * kHcC * 8 +
               (size_t)(S + kHcNT) * 8 + 16;
      p.nclusters = 0;
      p.ok = true;
      return p;
    }
    return p;
  }
  if (p.S < 3) return p;
  static const int forced_lag = dev_env("NYS_HVP_CLUSTER_LAG") ? atoi(dev_env("NYS_HVP_CLUSTER_LAG")) : 0;
  // lag 1 measured best on B200 (n = 1e5, S = 4: 2.32 ms vs 2.80 ms at lag 2 -
  // the exchange is sub-microsecond, the extra stage in flight is worth more)
  p.L = forced_lag > 0 ? forced_lag : 1;
  p.L = tmax(1, tmin(p.L, p.S - 1));
  if (p.S + p.L + 2 > kHcNT) return p;
  p.smem = (size_t)p.S * (row_bytes + kHcWarps * 256) + (size_t)kHcNT * kHcC * 8 + (size_t)(p.S + kHcNT) * 8;
  p.nclusters = 0;
  p.ok = true;
  return p;
}

template <int K, int Q = 1>
static int hvp_cluster_launch_k(HcPlan& p, const double* A, int64_t rows, int64_t n, int64_t lda, const double* d,
                                const double* v, double* ypart, cudaStream_t st, const double* pred) {
  const void* fn;
  if constexpr (Q == 1)
    fn = (const void*)hvp_cluster_kernel<K>;
  else
    fn = (const void*)hvp_cluster_q_kernel<Q, K>;
  static bool attr = false;
  static int maxc = 0;
  if (!attr) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kHcSmemBudget);
    cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(Q == 1 ? kHcThreads : kHqThreads, 1, 1);
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
    const cudaError_t oe = cudaOccupancyMaxActiveClusters(&mc, (void*)fn, &cfg);
    if (oe != cudaSuccess || mc < 1) {
      if (dev_env("NYS_HVP_DEBUG"))
        fprintf(stderr, "hvp_cluster Q=%d K=%d: occupancy %s, %d clusters (smem %zu)\n", Q, K,
                cudaGetErrorString(oe), mc, p.smem);
      cudaGetLastError();
      return NYS_ERR_UNSUPPORTED;
    }
    maxc = tmin(mc, kNumSMs / kHcC);
  }
  p.nclusters = (int)tmax<int64_t>(1, tmin<int64_t>(maxc, rows));
  cfg.gridDim = dim3(kHcC * p.nclusters, 1, 1);
  int W = p.W, S = p.S, L = p.L, Wq = p.Wq;
  cudaError_t e;
  if constexpr (Q == 1)
    e = cudaLaunchKernelEx(&cfg, hvp_cluster_kernel<K>, A, rows, n, lda, d, v, W, S, L, ypart, pred);
  else
    e = cudaLaunchKernelEx(&cfg, hvp_cluster_q_kernel<Q, K>, A, rows, n, lda, d, v, W, Wq, S, ypart, pred);
  (void)L;
  (void)Wq;
  if (e != cudaSuccess) return NYS_ERR_CUDA;
  __atomic_fetch_add(&g_launches, 1ull, __ATOMIC_RELAXED);
  return debug_sync_check(__FILE__, __LINE__) ? NYS_ERR_CUDA : NYS_OK;
}

// ypart: (plan.nclusters <= 9) x n partials; returns the cluster count used in *ncl
int hvp_cluster(HcPlan& p, const double* A, int64_t rows, int64_t n, int64_t lda, const double* d,
                const double* v, double* ypart, cudaStream_t st, const double* pred) {
  if (p.Q > 1) {
    switch (p.Q * 8 + p.K) {
#define NYS_QK(q, k) \
  case q * 8 + k: return hvp_cluster_launch_k<k, q>(p, A, rows, n, lda, d, v, ypart, st, pred);
      NYS_QK(2, 1) NYS_QK(2, 2) NYS_QK(2, 3) NYS_QK(2, 4) NYS_QK(3, 1) NYS_QK(3, 2) NYS_QK(3, 3) NYS_QK(3, 4)
      NYS_QK(4, 1) NYS_QK(4, 2) NYS_QK(4, 3) NYS_QK(4, 4)
#undef NYS_QK
      default: return NYS_ERR_UNSUPPORTED;
    }
  }
  switch (p.K) {
#define NYS_K(k) \
  case k: return hvp_cluster_launch_k<k>(p, A, rows, n, lda, d, v, ypart, st, pred);
    NYS_K(1) NYS_K(2) NYS_K(3) NYS_K(4) NYS_K(5) NYS_K(6) NYS_K(7) NYS_K(8) NYS_K(9) NYS_K(10) NYS_K(11)
    NYS_K(12)
#undef NYS_K
    default: return NYS_ERR_UNSUPPORTED;
  }
}



// ---------------------------------------------------------------------------
// The ADMM tail's data passes for wide rows in ONE stream over A (admm.py:
// 585-587 with problems.py:227-351): per row i the cluster forms
//   a_i.x and a_i.z                         (the A{x, z} pass)
// then, one row later with the totals exchanged in the cluster, every CTA
// evaluates the loss epilogue of the row itself
//   tg = l'(a_i.x - b_i), w = l''(.), thx = w a_i.x, nu = l'(a_i.z - b_i)
// and accumulates gA += tg a_i, hxA += thx a_i, atnu += nu a_i  (the 3-RHS
// A^T pass) from the still-staged segment.  x and z live in tensor memory
// (tcgen05.st once), the three accumulators in registers, the segment ring in
// shared memory.  Before: gemv_n (k = 2) + row-wise epilogue + gemv_t (k = 3),
// two passes over A; now one.  Outputs: T = [tg, thx, nu] (3 x rows), w (rows),
// per-cluster A^T partials P[(c * 3 + j) * n + col] (the layout the ML
// epilogue sums in a fixed order) and per-cluster row sums (fixed row order):
//   rowpart[c * 8 + 0..4] = sum l(r1), sum l(r2), sum l*(nu) finite, #inf, b.nu
// L = 1 row between a row's dot and its accumulation (its exchange overlaps
// the next row's dot); L + 1 row slots of lane partials (named barriers 9,
// 10), S >= L + 2 ring stages, kHcNT >= 2 L + 2 total slots (a remote relay
// can be at most 2 L + 1 rows ahead of this CTA's consumer).  Measured at
// 5000 x 10000 (C = 2): L = 2, 3 within 2 %; L = 2 with both waits first and
// dot + epilogue + accumulation as one straight block 7 % slower.
constexpr int kTcL = 1;
static_assert(1 + kHqMaxS + kTcL < 16 && kHcNT >= 2 * kTcL + 2, "tail pipeline depth");

// C = CTAs per cluster: 16 for the widest rows (configs 4 and 5), 2, 4 or 8
// for rows of 4096-12800 columns (config 2's width)
template <int C>
__device__ __forceinline__ double cluster_total_c(const double* p, int lane) {
  // lanes 0-15: the x partials of the C CTAs, lanes 16-31: the z partials;
  // fixed-order trees over C lanes (identical bits in every thread and CTA)
  double v = p[(lane >> 4) * C + (lane & (C - 1))];
#pragma unroll
  for (int o = C / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// SQ (square loss with z, g_b = A^T b known): l' = r, l'' = 1, so the three
// products A^T{Ax - b, Ax, Az - b} follow from two, A^T (A x) and A^T (A z):
// two axpys per element instead of three; the ML epilogue subtracts g_b
// (vec.cu ml_epilogue_kernel).  P row 0 is then not written.
template <int C, int KQ, bool WITHZ, bool LOGI, bool SQ>
__global__ void __launch_bounds__(kHqThreads, 1)
tail_cluster_kernel(const double* __restrict__ A, int64_t rows, int64_t n, int64_t lda,
                    const double* __restrict__ x, const double* __restrict__ z, const double* __restrict__ b,
                    int loss, int W, int S, double* __restrict__ T, double* __restrict__ wout,
                    double* __restrict__ P, double* __restrict__ R, const double* __restrict__ pred) {
  static_assert(KQ <= 8, "x and z slices: <= 32 TMEM columns each");
  static_assert(!SQ || (WITHZ && !LOGI), "SQ: square loss with z");
  constexpr int NV = WITHZ ? 2 : 1;
  constexpr int L = kTcL, NR = L + 1;
  if (pred && *pred != 0.0) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw);                 // S x W
  double* psl = ring + (size_t)S * W;                                 // NR x NV x 448 lane partials
  double* tsl = psl + NR * NV * kHqWarps * 32;                        // NT x NV x C CTA partials
  uint64_t* full = reinterpret_cast<uint64_t*>(tsl + kHcNT * NV * C);  // S
  uint64_t* totb = full + S;                                          // NT
  uint32_t* tmem_base = reinterpret_cast<uint32_t*>(totb + kHcNT);
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int cluster_id = blockIdx.x / C, nclusters = gridDim.x / C;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t c0 = (int64_t)rank * W;
  const int w_here = (int)tmax<int64_t>(0, tmin<int64_t>((int64_t)W, n - c0));
  const unsigned bytes = (unsigned)w_here * 8u;
  const int jmax = tmax(0, w_here - 2);  // last valid double2 of the staged segment
  const int64_t nrows_mine = rows > cluster_id ? (rows - cluster_id + nclusters - 1) / nclusters : 0;
  constexpr unsigned kTx = (unsigned)(C * NV * 8);

  if (tid == 0) {
    for (int q = 0; q < S; ++q) mbar_init(&full[q], 1);
    for (int q = 0; q < kHcNT; ++q) mbar_init(&totb[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int q = 0; q < kHcNT; ++q) mbar_expect_tx(&totb[q], kTx);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base)),
                 "n"(kHqTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cl.sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // per thread: x at words [0, 32), z at [32, 64) of the warp's 64-column block
  const uint32_t tv = *tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(64 * ((warp >> 2) & 3));

  const int nr = (int)nrows_mine;
  if (warp == kHqWarps) {
    // ---------------------------------------------------------- producer --
    const double* arow = A + (int64_t)cluster_id * lda + c0;
    const int64_t rstep = (int64_t)nclusters * lda;
    for (int g = 0, q = 0; g < nr; ++g, arow += rstep) {
      if (g >= S) qbar_sync(1 + q);
      if (lane == 0) {
        if (bytes > 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_expect_tx(&full[q], bytes);
          tma_load_1d(ring + (size_t)q * W, arow, bytes, &full[q]);
        } else {
          mbar_arrive(&full[q]);
        }
      }
      if (++q == S) q = 0;
    }
    for (int g = tmax(0, nr - S); g < nr; ++g) qbar_sync(1 + g % S);
  } else if (warp > kHqWarps) {
    // --------------------------------------------------- exchange (relay) --
    // the compute warps leave one partial per lane; this warp reduces them
    // (lane l: the 14 warps' lane-l partials in warp order, then a shuffle tree)
    for (int g = 0, rs = 0; g < nr; ++g, rs = rs + 1 == NR ? 0 : rs + 1) {
      qbar_sync(1 + kHqMaxS + rs);
      const int s = g & (kHcNT - 1);
#pragma unroll
      for (int vv = 0; vv < NV; ++vv) {
        const double* pp = psl + (rs * NV + vv) * kHqWarps * 32 + lane;
        double p = 0.0;
#pragma unroll
        for (int w2 = 0; w2 < kHqWarps; ++w2) p += pp[w2 * 32];
        p = warp_sum(p);
        if (lane < C) st_async_remote_f64(tsl + (s * NV + vv) * C + rank, &totb[s], (unsigned)lane, p);
      }
    }
  } else {
    // ---------------------------------------------------------- compute --
    {  // x, z -> TMEM
      double2 c[4];
#pragma unroll
      for (int vv = 0; vv < NV; ++vv) {
        const double* src = vv == 0 ? x : z;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4) {
            const int k = 4 * h + k4;
            const int j = 2 * (tid + k * kHqWarps * 32);
            c[k4] = (k < KQ && j < w_here) ? *reinterpret_cast<const double2*>(src + c0 + j) : make_double2(0.0, 0.0);
          }
          tmem_st16(tv + 32 * vv + 16 * h, c);
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    // Sparse z (the prox output: soft-thresholded, a few percent nonzeros at
    // most): when this CTA's slice of z holds at most one nonzero per compute
    // thread, a_i.z is one product per thread -- thread t keeps entry t of the
    // slice's compacted nonzeros (column order) in registers -- instead of a
    // second dense dot (half of the dot's FP64 work and tensor-memory reads).
    // zc: -2 dense dot, -1 sparse and no entry here, >= 0 the entry's column.
    // A zero term contributes exactly 0 to a sum, so only the order of the
    // nonzero terms differs from the dense dot.  CTAs of a cluster may choose
    // differently (the exchanged partials do not care).
    // (three-axpy variants of 7-8 column tiles per thread have no registers to spare)
    constexpr bool ZS = WITHZ && (SQ || KQ <= 6);
    int zc = -2;
    double zv = 0.0;
    if constexpr (ZS) {
      constexpr int kNT = kHqWarps * 32;
      int* wtot = reinterpret_cast<int*>(psl);  // psl is idle until the first dot
      int* lcol = wtot + 16;
      double* lval = reinterpret_cast<double*>(lcol + kNT);
      int cnt = 0;
#pragma unroll
      for (int k = 0; k < KQ; ++k) {
        const int j = 2 * (tid + k * kNT);
        if (j < w_here) {
          const double2 z2 = *reinterpret_cast<const double2*>(z + c0 + j);
          cnt += (z2.x != 0.0 ? 1 : 0) + (z2.y != 0.0 ? 1 : 0);
        }
      }
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (lane == 31) wtot[warp] = incl;
      asm volatile("bar.sync 15, %0;" ::"n"(kNT) : "memory");
      int base = 0, total = 0;
#pragma unroll
      for (int w2 = 0; w2 < kHqWarps; ++w2) {
        const int t = wtot[w2];
        if (w2 < warp) base += t;
        total += t;
      }
      if (total <= kNT && w_here > 0) {
        int pos = base + incl - cnt;
#pragma unroll
        for (int k = 0; k < KQ; ++k) {
          const int j = 2 * (tid + k * kNT);
          if (j < w_here) {
            const double2 z2 = *reinterpret_cast<const double2*>(z + c0 + j);
            if (z2.x != 0.0) {
              lcol[pos] = j;
              lval[pos++] = z2.x;
            }
            if (z2.y != 0.0) {
              lcol[pos] = j + 1;
              lval[pos++] = z2.y;
            }
          }
        }
        asm volatile("bar.sync 15, %0;" ::"n"(kNT) : "memory");
        zc = tid < total ? lcol[tid] : -1;
        zv = tid < total ? lval[tid] : 0.0;
      }
      asm volatile("bar.sync 15, %0;" ::"n"(kNT) : "memory");  // psl is the dots' from here
    }
    double2 yg[SQ ? 1 : KQ], yh[KQ], yn[WITHZ ? KQ : 1];
    yg[0] = make_double2(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < KQ; ++k) {
      if (!SQ) yg[k] = make_double2(0.0, 0.0);
      yh[k] = make_double2(0.0, 0.0);
      if (WITHZ) yn[k] = make_double2(0.0, 0.0);
    }
    // rank 0 writes T, w and the residuals r1, r2 of each row (the row sums
    // of loss values and conjugates run afterwards, row-parallel, in
    // tail_rowsums_kernel); the writer warp rotates (row jt -> warp jt mod 14)
    int wturn = 0;  // jt mod kHqWarps, kept incrementally
    int qi = 0, pi = 0, qj = 0, rs = 0;
    // the dots of a staged row with x (and z): lane partials into psl slot rs
    auto dot = [&](const double* row) {
      if (ZS && zc != -2) {
        // sparse z: the dense dot with x, one product for z
        double px = 0.0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (4 * h >= KQ) continue;
          double2 c[4];
          tmem_ld16(tv + 16 * h, c);
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4) {
            const int k = 4 * h + k4;
            if (k < KQ) {
              const double2 a = *reinterpret_cast<const double2*>(row + tmin(2 * (tid + k * kHqWarps * 32), jmax));
              px = fma(a.x, c[k4].x, px);
              px = fma(a.y, c[k4].y, px);
            }
          }
        }
        const double pz = zc >= 0 ? __dmul_rn(row[zc], zv) : 0.0;
        psl[((rs * NV) * kHqWarps + warp) * 32 + lane] = px;
        psl[((rs * NV + 1) * kHqWarps + warp) * 32 + lane] = pz;
      } else if (WITHZ) {
        // one pass over the staged row for both dots: a read once per element
        double px = 0.0, pz = 0.0;
#pragma unroll
        for (int k2 = 0; k2 < (KQ + 1) / 2; ++k2) {
          double2 cx[2], cz[2];
          tmem_ld8x2(tv + 8 * k2, tv + 32 + 8 * k2, cx, cz);
#pragma unroll
          for (int k1 = 0; k1 < 2; ++k1) {
            const int k = 2 * k2 + k1;
            if (k < KQ) {  // compile-time; out-of-range columns: x = z = 0 in TMEM, a read clamped
              const double2 a = *reinterpret_cast<const double2*>(row + tmin(2 * (tid + k * kHqWarps * 32), jmax));
              px = fma(a.x, cx[k1].x, px);
              px = fma(a.y, cx[k1].y, px);
              pz = fma(a.x, cz[k1].x, pz);
              pz = fma(a.y, cz[k1].y, pz);
            }
          }
        }
        psl[((rs * NV) * kHqWarps + warp) * 32 + lane] = px;
        psl[((rs * NV + 1) * kHqWarps + warp) * 32 + lane] = pz;
      } else {
        double pt = 0.0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (4 * h >= KQ) continue;
          double2 c[4];
          tmem_ld16(tv + 16 * h, c);
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4) {
            const int k = 4 * h + k4;
            if (k < KQ) {
              const double2 a = *reinterpret_cast<const double2*>(row + tmin(2 * (tid + k * kHqWarps * 32), jmax));
              pt = fma(a.x, c[k4].x, pt);
              pt = fma(a.y, c[k4].y, pt);
            }
          }
        }
        psl[((rs * NV) * kHqWarps + warp) * 32 + lane] = pt;
      }
    };
    // row jt: the cluster totals (landed in tsl), the loss epilogue of the row
    // (vec.cu ml_rowwise_kernel, same expressions), the writer's stores and the
    // A^T accumulation from the still-staged row
    auto epi_acc = [&](int jt, double bi, const double* row) {
      const int s = jt & (kHcNT - 1);
      // lanes 0-15: the x partials, 16-31: the z partials (fixed-order trees)
      const double tot = cluster_total_c<C>(tsl + (s * NV) * C, WITHZ ? lane : (lane & 15));
      const double ax = __shfl_sync(0xffffffffu, tot, 0);
      const double az = WITHZ ? __shfl_sync(0xffffffffu, tot, 16) : 0.0;
      if (warp == 0 && lane == 0) mbar_expect_tx(&totb[s], kTx);
      const int64_t i = cluster_id + (int64_t)jt * nclusters;
      const double r1 = __dadd_rn(ax, -bi);
      double tg, wi, nu = 0.0, r2 = 0.0;
      if (WITHZ) r2 = __dadd_rn(az, -bi);
      if constexpr (LOGI) {
        // the three sigmoids of the row, one per lane (lanes 0, 1, 2: expit(r1),
        // expit(-r1), expit(r2)), gathered by shuffles: one FP64 exp/div chain
        // per warp instead of four (same expressions, same bits)
        const double arg = lane == 0 ? r1 : (lane == 1 ? -r1 : r2);
        const double e = expit_d(arg);
        tg = __shfl_sync(0xffffffffu, e, 0);
        wi = tg * __shfl_sync(0xffffffffu, e, 1);  // loss_d2 = expit(w) * expit(-w)
        if (WITHZ) nu = __shfl_sync(0xffffffffu, e, 2);
      } else if constexpr (SQ) {
        tg = r1;  // problems.py:35-45: l'(r) = r, l''(r) = 1
        wi = 1.0;
        nu = r2;
      } else {
        tg = loss_d1(loss, r1);
        wi = loss_d2(loss, r1);
        if (WITHZ) nu = loss_d1(loss, r2);
      }
      const double thx = __dmul_rn(wi, ax);
      if (rank == 0 && lane == 0 && warp == wturn) {
        T[i] = tg;
        T[rows + i] = thx;
        wout[i] = wi;
        R[i] = r1;
        if (WITHZ) {
          T[2 * rows + i] = nu;
          R[rows + i] = r2;
        }
      }
      if (++wturn == kHqWarps) wturn = 0;
      // branch-free: columns past the segment accumulate into registers that are
      // never stored (reads clamped to the staged row)
#pragma unroll
      for (int k = 0; k < KQ; ++k) {
        const double2 a = *reinterpret_cast<const double2*>(row + tmin(2 * (tid + k * kHqWarps * 32), jmax));
        if (!SQ) {
          yg[k].x = fma(tg, a.x, yg[k].x);
          yg[k].y = fma(tg, a.y, yg[k].y);
        }
        yh[k].x = fma(thx, a.x, yh[k].x);  // SQ: thx = a_i.x
        yh[k].y = fma(thx, a.y, yh[k].y);
        if (WITHZ) {
          const double m = SQ ? az : nu;
          yn[k].x = fma(m, a.x, yn[k].x);
          yn[k].y = fma(m, a.y, yn[k].y);
        }
      }
    };
    auto wait_row = [&]() -> const double* {
      const int q = qi;
      mbar_wait(&full[q], (unsigned)pi);
      if (++qi == S) {
        qi = 0;
        pi ^= 1;
      }
      return ring + (size_t)q * W;
    };
    auto dot_done = [&]() {
      __syncwarp();
      qbar_arrive(1 + kHqMaxS + rs);
      if (++rs == NR) rs = 0;
    };
    auto acc_row = [&]() -> int {  // ring slot of the row accumulated next
      const int q = qj;
      if (++qj == S) qj = 0;
      return q;
    };
    // b of a row is requested at the row's dot and used at its epilogue L
    // iterations later: the load's latency stays off the per-row path
    double bq[L + 1];
#pragma unroll
    for (int u = 0; u <= L; ++u) bq[u] = 0.0;
    for (int it = 0; it < nr + L; ++it) {
#pragma unroll
      for (int u = L; u > 0; --u) bq[u] = bq[u - 1];  // bq[L]: b of row it - L
      if (it < nr) {
        bq[0] = __ldg(b + cluster_id + (int64_t)it * nclusters);
        dot(wait_row());
        dot_done();
      }
      const int jt = it - L;
      if (jt < 0) continue;
      mbar_wait(&totb[jt & (kHcNT - 1)], (unsigned)((jt / kHcNT) & 1));  // st.async complete_tx: CTA-scope acquire
      const int q = acc_row();
      epi_acc(jt, bq[L], ring + (size_t)q * W);
      __syncwarp();
      qbar_arrive(1 + q);
    }
    constexpr int K3 = WITHZ ? 3 : 2;
    double* pc = P + (int64_t)cluster_id * K3 * n + c0;
#pragma unroll
    for (int k = 0; k < KQ; ++k) {
      const int j = 2 * (tid + k * kHqWarps * 32);
      if (j < w_here) {
        if (!SQ) *reinterpret_cast<double2*>(pc + j) = yg[SQ ? 0 : k];
        *reinterpret_cast<double2*>(pc + n + j) = yh[k];
        if (WITHZ) *reinterpret_cast<double2*>(pc + 2 * n + j) = yn[k];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cl.sync();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_base), "n"(kHqTmemCols)
                 : "memory");
  }
}

// ---------------------------------------------------------------------------
// The one-pass square-loss tail for rows too wide for tail_cluster_kernel
// (114688 < n <= ~262000: config 5's n = 200000, the shape every rank holds in
// its 8-GPU run).  A CTA's column slice (12500 doubles at n = 2e5) is too wide
// for two register accumulators and whole-slice stages, so, as in
// hvp_cluster_q_kernel, the slice is staged in Q sub-segments (the dot streams
// each from HBM, the accumulation one row later re-reads it from L2) and the
// operands are spread over the SM's three large stores:
//   x slice               tensor memory, columns [0, 64) of the warp's block
//   A^T (A z) accumulator tensor memory, columns [64, 128)  (ld / fma / st per row)
//   A^T (A x) accumulator registers
//   z                     its nonzeros only: the prox output is sparse, so a_i.z is a
//                         gather over the compacted entries of each sub-segment
//                         (zlist_kernel), typically <= 1 entry per thread
// A dense z stays correct (every entry is visited, 448 per step) and only
// slows the dot.  Outputs as tail_cluster_kernel's SQ mode.
constexpr int kTqTmemCols = 512;
constexpr int kTqNR = 2;  // row slots of the lane partials (L + 1)

// nonzeros of sub-segment (rank, q) of z in column order: columns relative to
// the sub-segment into zcol / zval[(rank Q + q) Wq ...), their count in zcnt
__global__ void zlist_kernel(const double* __restrict__ z, int64_t n, int W, int Wq, int Q, int* __restrict__ zcol,
                             double* __restrict__ zval, int* __restrict__ zcnt, const double* __restrict__ pred) {
  if (pred && *pred != 0.0) return;
  const int rank = blockIdx.x / Q, q = blockIdx.x - rank * Q;
  const int64_t c0 = (int64_t)rank * W + (int64_t)q * Wq;
  const int wq = (int)tmax<int64_t>(0, tmin<int64_t>(tmin<int64_t>(Wq, (int64_t)W - (int64_t)q * Wq), n - c0));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  __shared__ int wsum[32];
  __shared__ int s_base;
  if (tid == 0) s_base = 0;
  __syncthreads();
  int* oc = zcol + (int64_t)blockIdx.x * Wq;
  double* ov = zval + (int64_t)blockIdx.x * Wq;
  for (int j0 = 0; j0 < wq; j0 += blockDim.x) {
    const int j = j0 + tid;
    const double v = j < wq ? z[c0 + j] : 0.0;
    const bool nz = v != 0.0;
    const unsigned m = __ballot_sync(0xffffffffu, nz);
    if (lane == 0) wsum[warp] = __popc(m);
    __syncthreads();
    int before = s_base, total = 0;
    for (int w2 = 0; w2 < nw; ++w2) {
      const int t = wsum[w2];
      if (w2 < warp) before += t;
      total += t;
    }
    if (nz) {
      const int pos = before + __popc(m & ((1u << lane) - 1u));
      oc[pos] = j;
      ov[pos] = v;
    }
    __syncthreads();
    if (tid == 0) s_base += total;
  }
  __syncthreads();
  if (tid == 0) zcnt[blockIdx.x] = s_base;
}

template <int Q, int KQ>
__global__ void __launch_bounds__(kHqThreads, 1)
tail_q_kernel(const double* __restrict__ A, int64_t rows, int64_t n, int64_t lda, const double* __restrict__ x,
              const int* __restrict__ zcol, const double* __restrict__ zval, const int* __restrict__ zcnt,
              const double* __restrict__ b, int W, int Wq, int S, double* __restrict__ T, double* __restrict__ wout,
              double* __restrict__ P, double* __restrict__ R, const double* __restrict__ pred) {
  static_assert(KQ <= 4 && Q <= 4, "x and accumulator slices of a thread: <= 64 TMEM columns each");
  // Rows go through the pipeline in PAIRS: tensor memory reads at 64 B/clk per
  // SM (writes at 256), so one read of the x slice feeds the dots of two rows
  // and one read + write of the accumulator slice takes both rows' updates
  // (a row at a time the tensor-memory traffic alone filled the row period:
  // 6.3 ms at 12500 x 200000, no faster than the two streaming passes).
  constexpr int C = kHcC, NV = 4, L = 1, NR = kTqNR;  // NV: (x, z) of the pair's two rows
  constexpr int kNT = kHqWarps * 32;
  if (pred && *pred != 0.0) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw);                  // S x Wq
  double* psl = ring + (size_t)S * Wq;                                 // NR x NV x 448 lane partials
  double* tsl = psl + NR * NV * kNT;                                   // NT x NV x C CTA partials
  uint64_t* full = reinterpret_cast<uint64_t*>(tsl + kHcNT * NV * C);  // S
  uint64_t* totb = full + S;                                           // NT
  uint32_t* tmem_base = reinterpret_cast<uint32_t*>(totb + kHcNT);
  int* s_cnt = reinterpret_cast<int*>(tmem_base + 2);                  // Q
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int cluster_id = blockIdx.x / C, nclusters = gridDim.x / C;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t c0 = (int64_t)rank * W;
  const int w_here = (int)tmax<int64_t>(0, tmin<int64_t>((int64_t)W, n - c0));
  const int64_t nrows_mine = rows > cluster_id ? (rows - cluster_id + nclusters - 1) / nclusters : 0;
  constexpr unsigned kTx = (unsigned)(C * NV * 8);

  if (tid == 0) {
    for (int q = 0; q < S; ++q) mbar_init(&full[q], 1);
    for (int q = 0; q < kHcNT; ++q) mbar_init(&totb[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int q = 0; q < kHcNT; ++q) mbar_expect_tx(&totb[q], kTx);
  }
  if (tid < Q) s_cnt[tid] = zcnt[rank * Q + tid];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base)),
                 "n"(kTqTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cl.sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // this warp's TMEM block: lanes of its sub-partition, 128 columns per warp
  // (x at [0, 64), the A^T (A z) accumulator at [64, 128))
  const uint32_t tv = *tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(128 * ((warp >> 2) & 3));
  const uint32_t tz = tv + 64;

  const int nr = (int)nrows_mine;
  const int npairs = (nr + 1) >> 1;
  if (warp == kHqWarps) {
    // ---------------------------------------------------------- producer --
    // slot order of a pair: sub-segment 0 of its rows, sub-segment 1 of its rows, ...
    const int64_t rstep = (int64_t)nclusters * lda;
    const double* base = A + (int64_t)cluster_id * lda + c0;
    int u = 0, slot = 0;
    auto issue = [&](int pp) {
#pragma unroll 1
      for (int q = 0; q < Q; ++q) {
        const int wq = tmin(Wq, w_here - q * Wq);
#pragma unroll 1
        for (int r = 0; r < 2; ++r) {
          const int g = 2 * pp + r;
          if (g >= nr) continue;
          if (u >= S) qbar_sync(1 + slot);
          if (lane == 0) {
            if (wq > 0) {
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              mbar_expect_tx(&full[slot], (unsigned)wq * 8u);
              tma_load_1d(ring + (size_t)slot * Wq, base + (int64_t)g * rstep + (int64_t)q * Wq, (unsigned)wq * 8u,
                          &full[slot]);
            } else {
              mbar_arrive(&full[slot]);
            }
          }
          ++u;
          if (++slot == S) slot = 0;
        }
      }
    };
    for (int pp = 0; pp < npairs + L; ++pp) {
      if (pp < npairs) issue(pp);
      if (pp >= L) issue(pp - L);  // the accumulation's re-read (L2)
    }
    for (int w2 = tmax(0, u - S); w2 < u; ++w2) qbar_sync(1 + w2 % S);
  } else if (warp > kHqWarps) {
    // --------------------------------------------------- exchange (relay) --
    for (int g = 0, rs = 0; g < npairs; ++g, rs = rs + 1 == NR ? 0 : rs + 1) {
      qbar_sync(1 + kHqMaxS + rs);
      const int s = g & (kHcNT - 1);
#pragma unroll
      for (int vv = 0; vv < NV; ++vv) {
        const double* pp = psl + (rs * NV + vv) * kNT + lane;
        double p = 0.0;
#pragma unroll
        for (int w2 = 0; w2 < kHqWarps; ++w2) p += pp[w2 * 32];
        p = warp_sum(p);
        if (lane < C) st_async_remote_f64(tsl + (s * NV + vv) * C + rank, &totb[s], (unsigned)lane, p);
      }
    }
  } else {
    // ---------------------------------------------------------- compute --
    const int* zc = zcol + (int64_t)rank * Q * Wq;
    const double* zv = zval + (int64_t)rank * Q * Wq;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      double2 c[4];
      const int wq = tmin(Wq, w_here - q * Wq);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int j = 2 * (tid + k * kNT);
        c[k] = (k < KQ && j < wq) ? *reinterpret_cast<const double2*>(x + c0 + (int64_t)q * Wq + j)
                                  : make_double2(0.0, 0.0);
      }
      tmem_st16(tv + 16 * q, c);
#pragma unroll
      for (int k = 0; k < 4; ++k) c[k] = make_double2(0.0, 0.0);
      tmem_st16(tz + 16 * q, c);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    double2 yx[Q][KQ];
#pragma unroll
    for (int q = 0; q < Q; ++q)
#pragma unroll
      for (int k = 0; k < KQ; ++k) yx[q][k] = make_double2(0.0, 0.0);
    int slot = 0, ph = 0, wturn = 0, rs = 0;
    auto next = [&]() {
      if (++slot == S) {
        slot = 0;
        ph ^= 1;
      }
    };
    for (int pp = 0; pp < npairs + L; ++pp) {
      if (pp < npairs) {
        const bool has1 = 2 * pp + 1 < nr;
        double px0 = 0.0, pz0 = 0.0, px1 = 0.0, pz1 = 0.0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int wq = tmin(Wq, w_here - q * Wq);
          // this thread's nonzero of z in the sub-segment (requested before the waits)
          const int cq = s_cnt[q];
          int ce = 0;
          double ve = 0.0;
          if (tid < cq) {
            ce = __ldg(zc + q * Wq + tid);
            ve = __ldg(zv + q * Wq + tid);
          }
          double2 c[4];
          tmem_ld16(tv + 16 * q, c);
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            if (r == 1 && !has1) break;
            mbar_wait(&full[slot], (unsigned)ph);
            const double* seg = ring + (size_t)slot * Wq;
            double px = 0.0, pz = 0.0;
#pragma unroll
            for (int k = 0; k < KQ; ++k) {
              const int j = 2 * (tid + k * kNT);
              if (j < wq) {
                const double2 a = *reinterpret_cast<const double2*>(seg + j);
                px = fma(a.x, c[k].x, px);
                px = fma(a.y, c[k].y, px);
              }
            }
            if (tid < cq) pz = __dmul_rn(seg[ce], ve);
            for (int e = tid + kNT; e < cq; e += kNT)  // a denser z: the remaining entries
              pz = fma(seg[__ldg(zc + q * Wq + e)], __ldg(zv + q * Wq + e), pz);
            if (r == 0) {
              px0 += px;
              pz0 += pz;
            } else {
              px1 += px;
              pz1 += pz;
            }
            __syncwarp();
            qbar_arrive(1 + slot);
            next();
          }
        }
        double* ps = psl + ((rs * NV) * kHqWarps + warp) * 32 + lane;
        ps[0] = px0;
        ps[kNT] = pz0;
        ps[2 * kNT] = px1;
        ps[3 * kNT] = pz1;
        __syncwarp();
        qbar_arrive(1 + kHqMaxS + rs);
        if (++rs == NR) rs = 0;
      }
      const int jp = pp - L;
      if (jp < 0) continue;
      const int s = jp & (kHcNT - 1);
      const bool hasj1 = 2 * jp + 1 < nr;
      mbar_wait(&totb[s], (unsigned)((jp / kHcNT) & 1));
      const double tot0 = cluster_total_c<C>(tsl + (s * NV) * C, lane);
      const double tot1 = cluster_total_c<C>(tsl + (s * NV + 2) * C, lane);
      const double ax0 = __shfl_sync(0xffffffffu, tot0, 0), az0 = __shfl_sync(0xffffffffu, tot0, 16);
      const double ax1 = __shfl_sync(0xffffffffu, tot1, 0), az1 = __shfl_sync(0xffffffffu, tot1, 16);
      if (warp == 0 && lane == 0) mbar_expect_tx(&totb[s], kTx);
      // the rows' epilogue (problems.py:35-45: l'(r) = r, l'' = 1): the writer's stores
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        if (r == 1 && !hasj1) break;
        if (rank == 0 && lane == 0 && warp == wturn) {
          const int64_t i = cluster_id + (int64_t)(2 * jp + r) * nclusters;
          const double bi = __ldg(b + i);
          const double ax = r ? ax1 : ax0, az = r ? az1 : az0;
          const double r1 = __dadd_rn(ax, -bi), r2 = __dadd_rn(az, -bi);
          T[i] = r1;
          T[rows + i] = ax;
          T[2 * rows + i] = r2;
          wout[i] = 1.0;
          R[i] = r1;
          R[rows + i] = r2;
        }
        if (++wturn == kHqWarps) wturn = 0;
      }
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int wq = tmin(Wq, w_here - q * Wq);
        double2 yz[4];
        tmem_ld16(tz + 16 * q, yz);
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          if (r == 1 && !hasj1) break;
          const double ax = r ? ax1 : ax0, az = r ? az1 : az0;
          mbar_wait(&full[slot], (unsigned)ph);
          const double* seg = ring + (size_t)slot * Wq;
#pragma unroll
          for (int k = 0; k < KQ; ++k) {
            const int j = 2 * (tid + k * kNT);
            if (j < wq) {
              const double2 a = *reinterpret_cast<const double2*>(seg + j);
              yx[q][k].x = fma(ax, a.x, yx[q][k].x);
              yx[q][k].y = fma(ax, a.y, yx[q][k].y);
              yz[k].x = fma(az, a.x, yz[k].x);
              yz[k].y = fma(az, a.y, yz[k].y);
            }
          }
          __syncwarp();
          qbar_arrive(1 + slot);
          next();
        }
        tmem_st16(tz + 16 * q, yz);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    // P rows 1 and 2 of this cluster (row 0 is not written in the SQ layout)
    double* pc = P + (int64_t)cluster_id * 3 * n + c0;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      double2 yz[4];
      tmem_ld16(tz + 16 * q, yz);
#pragma unroll
      for (int k = 0; k < KQ; ++k) {
        const int j = 2 * (tid + k * kNT);
        if (j < tmin(Wq, w_here - q * Wq)) {
          *reinterpret_cast<double2*>(pc + n + q * Wq + j) = yx[q][k];
          *reinterpret_cast<double2*>(pc + 2 * n + q * Wq + j) = yz[k];
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cl.sync();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_base), "n"(kTqTmemCols)
                 : "memory");
  }
}

// the row sums of the tail (nys_ml_rowwise_f64's out[0..4]) from the stored
// residuals r1 = Ax - b, r2 = Az - b and nu = T[2]: sum l(r1), sum l(r2),
// sum l*(nu) finite, #inf, b.nu -- row-parallel, fixed-order reduction
__global__ void tail_rowsums_kernel(int64_t rows, int loss, const double* __restrict__ R,
                                    const double* __restrict__ nu, const double* __restrict__ b, int withz,
                                    double* part, const double* __restrict__ pred) {
  if (pred && *pred != 0.0) return;
  double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x) {
    v[0] += loss_val(loss, R[i]);
    if (withz) {
      v[1] += loss_val(loss, R[rows + i]);
      const double y = nu[i];
      const double cv = loss_conj(loss, y);
      if (isinf(cv)) v[3] += 1.0; else v[2] += cv;
      v[4] = fma(b[i], y, v[4]);
    }
  }
  __shared__ double sh[5 * 32];
  block_sum<5>(v, sh);
  if (threadIdx.x == 0)
#pragma unroll
    for (int q = 0; q < 5; ++q) part[blockIdx.x * 5 + q] = v[q];
}
// (no last-block ticket: the scratch moves with `rows`, so a second tiny
// kernel sums the block partials in block order)
__global__ void tail_rowsums_final(const double* __restrict__ part, int nblocks, double* __restrict__ out,
                                   const double* __restrict__ pred) {
  if (pred && *pred != 0.0) return;
  if (threadIdx.x < 5) {
    double a = 0.0;
    for (int q = 0; q < nblocks; ++q) a += part[q * 5 + threadIdx.x];
    out[threadIdx.x] = a;
  }
}
constexpr int kTailSumBlocks = 2 * kNumSMs;

struct TcPlan {
  int C, W, KQ, S, L, nclusters;
  size_t smem;
  bool ok;
};

TcPlan tail_cluster_plan(int64_t rows, int64_t n, int64_t lda, const double* A, const double* x, bool with_z) {
  TcPlan p{};
  p.ok = false;
  static const bool off = dev_env("NYS_TAIL_CLUSTER_OFF") != nullptr;
  static const int forced_c = dev_env("NYS_TAIL_C") ? atoi(dev_env("NYS_TAIL_C")) : 0;
  // a row costs the cluster ~1.1 us of fixed work (exchange, epilogue) on top
  // of its share of the stream; slices narrower than this lose to the two
  // streaming passes (measured 5000 x 10000: C = 2 74 us against 131 us for
  // the row pass + GEMV^T; C = 4 (2500-column slices) 143 us)
  static const int min_w = dev_env("NYS_TAIL_MIN_W") ? atoi(dev_env("NYS_TAIL_MIN_W")) : 3500;
  if (off || (lda & 1) || (n & 1) || ((uintptr_t)A & 15) || ((uintptr_t)x & 15) || rows < 1) return p;
  // the smallest cluster whose slices fit the x/z tensor-memory columns
  // (KQ <= 8: <= 7168 columns per CTA), i.e. the widest slices
  p.C = 0;
  if (forced_c == 2 || forced_c == 4 || forced_c == 8 || forced_c == 16) {
    p.C = forced_c;
  } else {
    for (int c = 2; c <= 16 && !p.C; c *= 2)
      if (cdiv(n, (int64_t)c) <= 8 * kHqWarps * 32 * 2) p.C = c;
    if (!p.C || cdiv(n, (int64_t)p.C) < min_w) return p;
  }
  p.L = kTcL;
  p.W = (int)cdiv(cdiv(n, p.C), 2) * 2;
  p.KQ = (int)cdiv(p.W / 2, kHqWarps * 32);
  if (p.KQ > 8) return p;
  const int NV = with_z ? 2 : 1;
  const size_t fixed =
      (size_t)(p.L + 1) * NV * kHqWarps * 32 * 8 + (size_t)kHcNT * NV * p.C * 8 + kHcNT * 8 + 16 + 1024;
  p.S = (int)tmin<int64_t>(kHqMaxS, (int64_t)((kHcSmemBudget - fixed) / ((size_t)p.W * 8 + 8)));
  if (p.S < p.L + 2) return p;
  p.smem = (size_t)p.S * p.W * 8 + (size_t)(p.L + 1) * NV * kHqWarps * 32 * 8 + (size_t)kHcNT * NV * p.C * 8 +
           (size_t)(p.S + kHcNT) * 8 + 16;
  p.ok = true;
  return p;
}

template <int C, int KQ, bool WITHZ, bool LOGI, bool SQ>
static int tail_cluster_launch_k(TcPlan& p, const double* A, int64_t rows, int64_t n, int64_t lda, const double* x,
                                 const double* z, const double* b, int loss, double* T, double* w, double* P,
                                 double* R, double* rowsums, cudaStream_t st, const double* pred) {
  const void* fn = (const void*)tail_cluster_kernel<C, KQ, WITHZ, LOGI, SQ>;
  static bool attr = false;
  static int maxc = 0;
  if (!attr) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kHcSmemBudget);
    cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kHqThreads, 1, 1);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (maxc == 0) {
    cfg.gridDim = dim3(C * (kNumSMs / C), 1, 1);
    int mc = 0;
    if (cudaOccupancyMaxActiveClusters(&mc, fn, &cfg) != cudaSuccess || mc < 1) {
      cudaGetLastError();
      return NYS_ERR_UNSUPPORTED;
    }
    maxc = tmin(mc, kNumSMs / C);
  }
  p.nclusters = (int)tmax<int64_t>(1, tmin<int64_t>(maxc, rows));
  cfg.gridDim = dim3(C * p.nclusters, 1, 1);
  int W = p.W, S = p.S;
  if (cudaLaunchKernelEx(&cfg, tail_cluster_kernel<C, KQ, WITHZ, LOGI, SQ>, A, rows, n, lda, x, z, b, loss, W, S, T, w, P,
                         R, pred) != cudaSuccess)
    return NYS_ERR_CUDA;
  __atomic_fetch_add(&g_launches, 1ull, __ATOMIC_RELAXED);
  double* part = R + 2 * rows;
  const unsigned blocks = (unsigned)tmax<int64_t>(1, tmin<int64_t>(cdiv(rows, 256), kTailSumBlocks));
  tail_rowsums_kernel<<<blocks, 256, 0, st>>>(rows, loss, R, T + 2 * rows, b, WITHZ ? 1 : 0, part, pred);
  NYS_CHECK_LAUNCH();
  tail_rowsums_final<<<1, 32, 0, st>>>(part, (int)blocks, rowsums, pred);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

// plan and launch of tail_q_kernel (square loss with z and g_b only)
struct TqPlan {
  int W, Wq, Q, KQ, S, nclusters;
  size_t smem;
  bool ok;
};

static TqPlan tail_q_plan(int64_t rows, int64_t n, int64_t lda, const double* A, const double* x) {
  TqPlan p{};
  p.ok = false;
  if ((lda & 1) || (n & 1) || ((uintptr_t)A & 15) || ((uintptr_t)x & 15) || rows < 1) return p;
  p.W = (int)cdiv(cdiv(n, (int64_t)kHcC), 2) * 2;
  const size_t fixed = (size_t)kTqNR * 4 * kHqWarps * 32 * 8 + (size_t)kHcNT * 4 * kHcC * 8 + kHcNT * 8 + 64 + 1024;
  for (int Q = 2; Q <= 4; ++Q) {
    const int Wq = (int)cdiv(cdiv(p.W, Q), 2) * 2;
    const int KQ = (int)cdiv(Wq / 2, kHqWarps * 32);
    if (KQ > 4) continue;
    const int S = (int)tmin<int64_t>(kHqMaxS, (int64_t)((kHcSmemBudget - fixed) / ((size_t)Wq * 8 + 8)));
    if (S < 4) continue;
    p.Q = Q;
    p.Wq = Wq;
    p.KQ = KQ;
    p.S = S;
    p.smem = (size_t)S * Wq * 8 + (size_t)kTqNR * 4 * kHqWarps * 32 * 8 + (size_t)kHcNT * 4 * kHcC * 8 +
             (size_t)(S + kHcNT) * 8 + 64;
    p.ok = true;
    return p;
  }
  return p;
}

template <int Q, int KQ>
static int tail_q_launch_k(TqPlan& p, const double* A, int64_t rows, int64_t n, int64_t lda, const double* x,
                           const int* zcol, const double* zval, const int* zcnt, const double* b, double* T,
                           double* w, double* P, double* R, cudaStream_t st, const double* pred) {
  const void* fn = (const void*)tail_q_kernel<Q, KQ>;
  static bool attr = false;
  static int maxc = 0;
  if (!attr) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kHcSmemBudget);
    cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kHqThreads, 1, 1);
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
    cfg.gridDim = dim3(kHcC * (kNumSMs / kHcC), 1, 1);
    int mc = 0;
    if (cudaOccupancyMaxActiveClusters(&mc, fn, &cfg) != cudaSuccess || mc < 1) {
      cudaGetLastError();
      return NYS_ERR_UNSUPPORTED;
    }
    maxc = tmin(mc, kNumSMs / kHcC);
  }
  p.nclusters = (int)tmax<int64_t>(1, tmin<int64_t>(maxc, rows));
  cfg.gridDim = dim3(kHcC * p.nclusters, 1, 1);
  int W = p.W, Wq = p.Wq, S = p.S;
  if (cudaLaunchKernelEx(&cfg, tail_q_kernel<Q, KQ>, A, rows, n, lda, x, zcol, zval, zcnt, b, W, Wq, S, T, w, P, R,
                         pred) != cudaSuccess)
    return NYS_ERR_CUDA;
  __atomic_fetch_add(&g_launches, 1ull, __ATOMIC_RELAXED);
  return NYS_OK;
}

// the SQ tail for rows beyond tail_cluster_plan: z's nonzeros compacted per
// sub-segment, then the one stream over A, then the row sums
static int tail_q(const double* A, int64_t rows, int64_t n, int64_t lda, const double* x, const double* z,
                  const double* b, double* T, double* w, void* ws, size_t ws_bytes, size_t ws_off, double* rowsums,
                  cudaStream_t st, const double* pred, double** Pout, int* splits_out) {
  TqPlan p = tail_q_plan(rows, n, lda, A, x);
  if (!p.ok) return NYS_ERR_UNSUPPORTED;
  const size_t ncl = (size_t)(kNumSMs / kHcC);
  const size_t nlist = (size_t)kHcC * p.Q * p.Wq;
  const size_t need =
      ws_off + (ncl * 3 * n + 2 * (size_t)rows + kTailSumBlocks * 5 + 8) * 8 + nlist * 12 + 64 * 4 + 64;
  if (ws_bytes < need) return NYS_ERR_UNSUPPORTED;
  double* P = reinterpret_cast<double*>(reinterpret_cast<char*>(ws) + ws_off);
  double* rowpart = P + ncl * 3 * n;
  double* zval = rowpart + 2 * (size_t)rows + kTailSumBlocks * 5 + 8;
  int* zcol = reinterpret_cast<int*>(zval + nlist);
  int* zcnt = zcol + nlist;
  zlist_kernel<<<kHcC * p.Q, 256, 0, st>>>(z, n, p.W, p.Wq, p.Q, zcol, zval, zcnt, pred);
  NYS_CHECK_LAUNCH();
  int rc = NYS_ERR_UNSUPPORTED;
  switch (p.Q * 8 + p.KQ) {
#define NYS_TQ(q, k)                                                                                        \
  case (q * 8 + k):                                                                                         \
    rc = tail_q_launch_k<q, k>(p, A, rows, n, lda, x, zcol, zval, zcnt, b, T, w, P, rowpart, st, pred); \
    break;
    NYS_TQ(2, 1) NYS_TQ(2, 2) NYS_TQ(2, 3) NYS_TQ(2, 4) NYS_TQ(3, 1) NYS_TQ(3, 2) NYS_TQ(3, 3) NYS_TQ(3, 4)
    NYS_TQ(4, 1) NYS_TQ(4, 2) NYS_TQ(4, 3) NYS_TQ(4, 4)
#undef NYS_TQ
    default: break;
  }
  if (rc) return rc;
  double* part = rowpart + 2 * rows;
  const unsigned blocks = (unsigned)tmax<int64_t>(1, tmin<int64_t>(cdiv(rows, 256), kTailSumBlocks));
  tail_rowsums_kernel<<<blocks, 256, 0, st>>>(rows, NYS_LOSS_SQUARE, rowpart, T + 2 * rows, b, 1, part, pred);
  NYS_CHECK_LAUNCH();
  tail_rowsums_final<<<1, 32, 0, st>>>(part, (int)blocks, rowsums, pred);
  NYS_CHECK_LAUNCH();
  *Pout = P;
  *splits_out = p.nclusters;
  return NYS_OK;
}

// true when the only one-pass plan for this shape is tail_q (rows beyond the
// whole-slice plan): it visits z through its nonzeros, so callers whose prox
// leaves z dense (no l1 term) keep the two streaming passes there
bool tail_wants_sparse_z(const double* A, int64_t rows, int64_t n, int64_t lda, const double* x) {
  return !tail_cluster_plan(rows, n, lda, A, x, true).ok && tail_q_plan(rows, n, lda, A, x).ok;
}

// the tail's A{x,z} + loss epilogue + A^T{tg, thx, nu} in one pass; UNSUPPORTED
// when the shape has no cluster plan (the caller runs the two-pass tail)
int tail_cluster(const double* A, int64_t rows, int64_t n, int64_t lda, const double* x, const double* z,
                 const double* b, int loss, double* T, double* w, void* ws, size_t ws_bytes, size_t ws_off,
                 double* rowsums, cudaStream_t st, const double* pred, double** Pout, int* splits_out,
                 const double* gb, int* sq_out) {
  // measured (20000 x 100000): square loss 2.84 ms, logistic 4.29 ms (every
  // warp evaluates the exp-based epilogue of each row) against 4.57 ms for the
  // two passes
  TcPlan p = tail_cluster_plan(rows, n, lda, A, x, z != nullptr);
  if (!p.ok) {
    // wider rows (config 5's n = 200000): the square loss with g_b has its own one-pass plan
    if (!(gb && z && loss == NYS_LOSS_SQUARE) || cdiv(n, (int64_t)kHcC) <= 8 * kHqWarps * 32 * 2)
      return NYS_ERR_UNSUPPORTED;
    const int rq = tail_q(A, rows, n, lda, x, z, b, T, w, ws, ws_bytes, ws_off, rowsums, st, pred, Pout, splits_out);
    if (rq == NYS_OK && sq_out) *sq_out = 1;
    return rq;
  }
  const int K3 = z ? 3 : 2;
  const size_t ncl = (size_t)(kNumSMs / p.C);
  const size_t need = ws_off + ncl * K3 * n * 8 + (2 * (size_t)rows + kTailSumBlocks * 5 + 8) * 8;
  if (ws_bytes < need) return NYS_ERR_UNSUPPORTED;
  double* P = reinterpret_cast<double*>(reinterpret_cast<char*>(ws) + ws_off);
  double* rowpart = P + ncl * K3 * n;  // residuals r1, r2 (2 x rows), then the row-sum scratch
  int rc = NYS_ERR_UNSUPPORTED;
  // slices of >= 3500 columns (the plan's minimum): KQ = 4 .. 8
  const bool logi = loss == NYS_LOSS_LOGISTIC;
  // square loss with z and g_b: two A^T products instead of three (SQ)
  const bool sq = gb && z && loss == NYS_LOSS_SQUARE;
  // mode: 0 no z, 1 no z logistic, 2 z, 3 z logistic, 4 z square (SQ)
  const int mode = sq ? 4 : (z ? 2 : 0) + (logi ? 1 : 0);
  const int key = ((p.C == 16 ? 0 : p.C == 8 ? 1 : p.C == 4 ? 2 : 3) * 16 + p.KQ) * 8 + mode;
  switch (key) {
#define NYS_TK1(c, ci, k, zz, lg, sqq)                                                                              \
  case ((ci * 16 + k) * 8 + (sqq ? 4 : (zz ? 2 : 0) + (lg ? 1 : 0))):                                               \
    rc = tail_cluster_launch_k<c, k, zz, lg, sqq>(p, A, rows, n, lda, x, z, b, loss, T, w, P, rowpart, rowsums, st, \
                                                  pred);                                                            \
    break;
#define NYS_TK(c, ci, k)                                                                                      \
  NYS_TK1(c, ci, k, false, false, false) NYS_TK1(c, ci, k, false, true, false)                                 \
  NYS_TK1(c, ci, k, true, false, false) NYS_TK1(c, ci, k, true, true, false) NYS_TK1(c, ci, k, true, false, true)
#define NYS_TKC(c, ci) NYS_TK(c, ci, 4) NYS_TK(c, ci, 5) NYS_TK(c, ci, 6) NYS_TK(c, ci, 7) NYS_TK(c, ci, 8)
    NYS_TKC(16, 0) NYS_TKC(8, 1) NYS_TKC(4, 2) NYS_TKC(2, 3)
#undef NYS_TKC
#undef NYS_TK
#undef NYS_TK1
    default: break;
  }
  if (rc == NYS_OK) {
    *Pout = P;
    *splits_out = p.nclusters;
    if (sq_out) *sq_out = sq ? 1 : 0;
  }
  return rc;
}

}  // namespace nys

// workspace of nys_admm_tail_f64's A^T stage when the cluster tail runs
// (reduction scratch + per-cluster A^T partials + per-cluster row sums)
extern "C" size_t nys_tail_cluster_workspace(int64_t rows, int64_t n) {
  (void)rows;
  const size_t ncl = nys::kNumSMs / 2;  // the smallest cluster size a plan picks
  return (size_t)(nys::kRedPartialsTail * 16 + 64) * sizeof(double) + ncl * 3 * (size_t)n * 8 +
         (2 * (size_t)rows + nys::kTailSumBlocks * 5 + 8) * 8;
}

namespace nys {
// AT[j, c] = sum over clusters of P[(cl * K + j) * n + c], fixed cluster order;
// with gb (the SQ tail): AT[0] = AT[1] - gb, AT[2] = (sum of row 2) - gb
__global__ void tail_partial_sum_kernel(const double* __restrict__ P, int64_t n, int K, int ncl,
                                        double* __restrict__ AT, const double* __restrict__ gb,
                                        const double* __restrict__ pred) {
  if (pred && *pred != 0.0) return;
  const int64_t total = n * K;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t / n, c = t - j * n;
    const int64_t js = (gb && j == 0) ? 1 : j;
    double a = 0.0;
    for (int q = 0; q < ncl; ++q) a += P[((int64_t)q * K + js) * n + c];
    if (gb && j != 1) a = a - gb[c];
    AT[j * n + c] = a;
  }
}
// the cluster tail's per-cluster A^T partials -> AT (K x n), for callers that do
// not fuse the sum into the ML epilogue (row-sharded solves: the ranks' AT are
// all-reduced before the norms)
int tail_partial_sum(const double* P, int64_t n, int K, int ncl, double* AT, const double* gb, cudaStream_t st,
                     const double* pred) {
  tail_partial_sum_kernel<<<(unsigned)tmin<int64_t>(cdiv(n * K, 256), 4 * kNumSMs), 256, 0, st>>>(P, n, K, ncl, AT,
                                                                                                  gb, pred);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}
}  // namespace nys

static int ml_tail_impl(const double* A, int64_t rows, int64_t n, int64_t lda, const double* x, const double* z,
                        const double* b, int loss, double* T, double* w, double* AT, double* rowsums,
                        const double* gb, void* ws, size_t ws_bytes, void* stream) {
  using namespace nys;
  if (rows <= 0 || n <= 0 || lda < n || loss < 0 || loss > 2) return NYS_ERR_ARG;
  cudaStream_t st = as_stream(stream);
  double* P = nullptr;
  int splits = 0, sq = 0;
  const int rc = tail_cluster(A, rows, n, lda, x, z, b, loss, T, w, ws, ws_bytes,
                              (size_t)(kRedPartialsTail * 16 + 64) * sizeof(double), rowsums, st, nullptr, &P,
                              &splits, gb, &sq);
  if (rc) return rc;
  const int K = z ? 3 : 2;
  return tail_partial_sum(P, n, K, splits, AT, sq ? gb : nullptr, st, nullptr);
}

// The one-pass ML tail on its own (tests and measurement): T = [l'(Ax-b),
// w o Ax, l'(Az-b)] (3 x rows), w = l''(Ax-b), AT = A^T T (3 x n, 2 x n without
// z), rowsums[0..4] as nys_ml_rowwise_f64.  NYS_ERR_UNSUPPORTED for shapes
// without a cluster plan (n <= 12800 or too wide).
extern "C" int nys_ml_tail_f64(const double* A, int64_t rows, int64_t n, int64_t lda, const double* x,
                               const double* z, const double* b, int loss, double* T, double* w, double* AT,
                               double* rowsums, void* ws, size_t ws_bytes, void* stream) {
  return ml_tail_impl(A, rows, n, lda, x, z, b, loss, T, w, AT, rowsums, nullptr, ws, ws_bytes, stream);
}

// The same with g_b = A^T b: the square loss with z then runs the two-product
// SQ tail (A^T (A x), A^T (A z); g_b subtracted in the partial sum)
extern "C" int nys_ml_tail_gb_f64(const double* A, int64_t rows, int64_t n, int64_t lda, const double* x,
                                  const double* z, const double* b, int loss, const double* gb, double* T, double* w,
                                  double* AT, double* rowsums, void* ws, size_t ws_bytes, void* stream) {
  return ml_tail_impl(A, rows, n, lda, x, z, b, loss, T, w, AT, rowsums, gb, ws, ws_bytes, stream);
}
