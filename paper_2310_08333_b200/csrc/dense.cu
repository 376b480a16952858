// K5: Nystrom sketch construction on the GPU (sketch.py:74-128).
//
//   * nys_gemm_f64: FP64 GEMM on the DMMA tensor-core path (mma.sync m8n8k4
//     f64 -> SASS DMMA.8x8x4).  tcgen05 has no FP64 kind, so DMMA is the
//     FP64 tensor path on sm_100a.  128x64x16 CTA tiles, 8 warps of 32x32,
//     3-stage cp.async pipeline, split-K with a fixed-order reduction when the
//     output has too few tiles to fill 148 SMs (the s x s Gram products).
//   * CholeskyQR2 orthonormalisation of the raw Gaussian Omega (replaces the
//     Householder QR of sketch.py:99; the sketch depends only on range(Omega)).
//   * single-CTA Cholesky (LAPACK potf2 failure rule), triangular inverse,
//   * one-sided Jacobi symmetric eigensolver on a cooperative grid (replaces
//     the thin SVD of sketch.py:126 via B^T B, and eigh of sketch.py:115).
#include <cooperative_groups.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>
#include "common.cuh"

namespace cg = cooperative_groups;

namespace nys {

// ------------------------------------------------------------- GEMM -------
// One kernel template, several CTA tile shapes: the sketch GEMMs are skinny
// (N = s ~ 100-300 columns), so a fixed 128x64 tile wastes up to 40% of the
// tensor work on padding and leaves partial waves.  The host planner
// (gemm_plan) picks tile shape and split-K per call from a cost model of
// padded work, wave quantisation and split-K partial traffic.
constexpr int GBK = 16, GSTAGES = 3, GTHREADS = 256;
// 8 warps: 4 along M x 2 along N for the 32/48/64-column tiles; the odd widths
// (56, 136: picked so that ceil(N / BN) BN hugs a sketch width such as 133,
// 258 or 390 -- the 48/64-column tiles pad those by 8-15 %) put all 8 along M
constexpr int gemm_wn(int bn) { return (bn % 16 == 0 && bn <= 64) ? 2 : 1; }
// shared-memory row strides (doubles) chosen so DMMA fragment loads are
// 2-wavefront (conflict-free for 256 B per warp request)
constexpr int kStrideKmaj(int mn) { return (mn + 15) / 16 * 16 + 8; }  // tile stored [k][m]: stride = 8 mod 16
constexpr int kStrideMmaj = GBK + 4;                   // tile stored [m][k]

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(sz));
}
// 16-byte copy of a pair of doubles; nvalid in {0, 1, 2} (the rest zero-filled)
__device__ __forceinline__ void cp_async16(double* dst, const double* src, int nvalid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(nvalid * 8));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// TA: op(A) = A^T (A stored K x M). TB: op(B) = B^T (B stored N x K).
template <bool TA, bool TB, int BM, int BN>
struct GemmCfg {
  static constexpr int GWN = gemm_wn(BN), GWM = 8 / GWN;
  static constexpr int FM = BM / (GWM * 8), FN = BN / (GWN * 8);  // 8x8 fragments per warp
  static constexpr int A_ELEMS = TA ? GBK * kStrideKmaj(BM) : BM * kStrideMmaj;
  static constexpr int B_ELEMS = TB ? BN * kStrideMmaj : GBK * kStrideKmaj(BN);
  static constexpr int STAGE = A_ELEMS + B_ELEMS;
  static constexpr size_t BYTES = (size_t)STAGE * GSTAGES * sizeof(double);
  static_assert(FM >= 1 && FN >= 1 && BM % (GWM * 8) == 0 && BN % (GWN * 8) == 0, "tile");
  static_assert((BM * GBK) % GTHREADS == 0, "loader");
};

// VA: op(A) tiles loaded as 16-byte pairs (lda even, A 16-byte aligned)
template <bool TA, bool TB, int BM, int BN, bool VA>
__global__ void __launch_bounds__(GTHREADS)
dgemm_kernel(int64_t M, int64_t N, int64_t K, double alpha, const double* __restrict__ A,
             int64_t lda, const double* __restrict__ B, int64_t ldb, double beta,
             double* __restrict__ C, int64_t ldc, int64_t k_per_split, double* __restrict__ P) {
  extern __shared__ __align__(16) double smem[];
  using S = GemmCfg<TA, TB, BM, BN>;
  constexpr int FM = S::FM, FN = S::FN, GWM = S::GWM, GWN = S::GWN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % GWM, wn = warp / GWM;
  const int64_t n0 = (int64_t)blockIdx.x * BN, m0 = (int64_t)blockIdx.y * BM;
  const int64_t kb = (int64_t)blockIdx.z * k_per_split;
  const int64_t ke = min(K, kb + k_per_split);
  const int ktiles = (int)cdiv(tmax<int64_t>(ke - kb, 0), GBK);

  auto load_tile = [&](int stage, int64_t k0) {
    double* As = smem + stage * S::STAGE;
    double* Bs = As + S::A_ELEMS;
    if (VA) {
#pragma unroll
      for (int e2 = tid; e2 < BM * GBK / 2; e2 += GTHREADS) {
        if (TA) {  // pairs along m
          const int kk = e2 / (BM / 2), mm = (e2 - kk * (BM / 2)) * 2;
          const int64_t gm = m0 + mm, gk = k0 + kk;
          const int nv = gk < ke ? (gm + 1 < M ? 2 : (gm < M ? 1 : 0)) : 0;
          cp_async16(As + kk * kStrideKmaj(BM) + mm, nv ? A + gk * lda + gm : A, nv);
        } else {  // pairs along k
          const int mm = e2 / (GBK / 2), kk = (e2 - mm * (GBK / 2)) * 2;
          const int64_t gm = m0 + mm, gk = k0 + kk;
          const int nv = gm < M ? (gk + 1 < ke ? 2 : (gk < ke ? 1 : 0)) : 0;
          cp_async16(As + mm * kStrideMmaj + kk, nv ? A + gm * lda + gk : A, nv);
        }
      }
    } else
#pragma unroll
    for (int e = tid; e < BM * GBK; e += GTHREADS) {
      if (TA) {  // consecutive threads along m (contiguous in memory)
        const int kk = e / BM, mm = e - kk * BM;
        const int64_t gm = m0 + mm, gk = k0 + kk;
        const bool v = gm < M && gk < ke;
        cp_async8(As + kk * kStrideKmaj(BM) + mm, v ? A + gk * lda + gm : A, v);
      } else {  // consecutive threads along k
        const int mm = e / GBK, kk = e - mm * GBK;
        const int64_t gm = m0 + mm, gk = k0 + kk;
        const bool v = gm < M && gk < ke;
        cp_async8(As + mm * kStrideMmaj + kk, v ? A + gm * lda + gk : A, v);
      }
    }
#pragma unroll
    for (int e = tid; e < BN * GBK; e += GTHREADS) {
      if (TB) {
        const int nn = e / GBK, kk = e - nn * GBK;
        const int64_t gn = n0 + nn, gk = k0 + kk;
        const bool v = gn < N && gk < ke;
        cp_async8(Bs + nn * kStrideMmaj + kk, v ? B + gn * ldb + gk : B, v);
      } else {
        const int kk = e / BN, nn = e - kk * BN;
        const int64_t gn = n0 + nn, gk = k0 + kk;
        const bool v = gn < N && gk < ke;
        cp_async8(Bs + kk * kStrideKmaj(BN) + nn, v ? B + gk * ldb + gn : B, v);
      }
    }
  };

  // The loader of tiles wholly inside [kb, ke) -- every tile but a ragged last
  // one: each thread's copies sit at fixed places of the tile, so their global
  // pointers, shared-memory offsets and row / column validity are formed once
  // and a tile costs one cp.async per copy plus one pointer advance (the
  // general loader above recomputes 64-bit addresses and three bounds tests per
  // copy; an ncu capture at 20000 x 258 x 100000 put 56 % of the kernel's
  // instructions and two thirds of its stall samples there).
  constexpr int NA = VA ? BM * GBK / 2 / GTHREADS : BM * GBK / GTHREADS;  // copies of op(A) per thread and tile
  constexpr int NB = (BN * GBK + GTHREADS - 1) / GTHREADS;               // copies of op(B) (8 bytes each)
  constexpr int AW = VA ? 2 : 1;                                          // doubles per copy of op(A)
  constexpr int ACOLS = (TA ? BM : GBK) / AW;                             // copies per stored row of the A tile
  constexpr int ARPP = GTHREADS / ACOLS;                                  // stored rows per pass of the CTA
  constexpr int ASTRIDE = TA ? kStrideKmaj(BM) : kStrideMmaj;
  const int ar = tid / ACOLS, ac = (tid - ar * ACOLS) * AW;
  const double* pA = TA ? A + (kb + ar) * lda + m0 + ac : A + (m0 + ar) * lda + kb + ac;
  const int64_t a_step = (int64_t)ARPP * lda;
  const int sa0 = ar * ASTRIDE + ac;
  unsigned a_mask = 0;  // !TA: rows of the tile inside M
  int a_nv = AW;        // TA: doubles of this thread's copy inside M (the same for every k row)
  if (TA) {
    a_nv = (int)tmax<int64_t>(0, tmin<int64_t>(AW, M - (m0 + ac)));
  } else {
#pragma unroll
    for (int i = 0; i < NA; ++i) a_mask |= (m0 + ar + i * ARPP < M ? 1u : 0u) << i;
  }
  const double* pB;
  int b_g[NB], b_s[NB];  // !TB: global and shared offsets of copy i (TB: uniform strides)
  unsigned b_mask = 0;
  if (TB) {
    const int br = tid / GBK, bc = tid - br * GBK;
    pB = B + (n0 + br) * ldb + kb + bc;
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      b_g[i] = 0;
      b_s[i] = (br + i * (GTHREADS / GBK)) * kStrideMmaj + bc;
      b_mask |= ((br + i * (GTHREADS / GBK) < BN && n0 + br + i * (GTHREADS / GBK) < N) ? 1u : 0u) << i;
    }
  } else {
    pB = B + kb * ldb + n0;
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const int e = tid + i * GTHREADS, kk = e / BN, nn = e - kk * BN;
      b_g[i] = kk * (int)ldb + nn;
      b_s[i] = kk * kStrideKmaj(BN) + nn;
      b_mask |= ((e < BN * GBK && n0 + nn < N) ? 1u : 0u) << i;
    }
  }
  const int64_t b_step = (int64_t)(GTHREADS / GBK) * ldb;  // TB: rows of B between a thread's copies
  const bool fast_ok = TB || ldb < (int64_t)(1 << 26);     // b_g in 32 bits
  auto load_fast = [&](int stage) {
    double* As = smem + stage * S::STAGE;
    double* Bs = As + S::A_ELEMS;
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      const int nv = TA ? a_nv : (((a_mask >> i) & 1u) ? AW : 0);
      const double* src = nv ? pA + i * a_step : A;
      if (VA)
        cp_async16(As + sa0 + i * (ARPP * ASTRIDE), src, nv);
      else
        cp_async8(As + sa0 + i * (ARPP * ASTRIDE), src, nv != 0);
    }
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      if (!TB && (i + 1) * GTHREADS > BN * GBK && tid + i * GTHREADS >= BN * GBK) continue;  // past the tile
      if (TB && (i + 1) * (GTHREADS / GBK) > BN && tid / GBK + i * (GTHREADS / GBK) >= BN) continue;
      const bool v = (b_mask >> i) & 1u;
      const double* src = v ? (TB ? pB + i * b_step : pB + b_g[i]) : B;
      cp_async8(Bs + b_s[i], src, v);
    }
    pA += TA ? (int64_t)GBK * lda : (int64_t)GBK;
    pB += TB ? (int64_t)GBK : (int64_t)GBK * ldb;
  };
  // tiles are loaded in order, so the fast loader's pointers always stand at the next one
  auto load_any = [&](int stage, int64_t k0) {
    if (fast_ok && k0 + GBK <= ke)
      load_fast(stage);
    else
      load_tile(stage, k0);
  };

  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < GSTAGES - 1; ++s) {
    if (s < ktiles) load_any(s, kb + (int64_t)s * GBK);
    cp_async_commit();
  }
  const int fr = lane >> 2, fc = lane & 3;
  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<GSTAGES - 2>();
    __syncthreads();
    {  // prefetch tile kt + STAGES - 1
      const int nk = kt + GSTAGES - 1;
      if (nk < ktiles) load_any(nk % GSTAGES, kb + (int64_t)nk * GBK);
      cp_async_commit();
    }
    const double* As = smem + (kt % GSTAGES) * S::STAGE;
    const double* Bs = As + S::A_ELEMS;
#pragma unroll
    for (int k4 = 0; k4 < GBK; k4 += 4) {
      double af[FM], bf[FN];
#pragma unroll
      for (int i = 0; i < FM; ++i) {
        const int mm = wm * (FM * 8) + i * 8 + fr, kk = k4 + fc;
        af[i] = TA ? As[kk * kStrideKmaj(BM) + mm] : As[mm * kStrideMmaj + kk];
      }
#pragma unroll
      for (int j = 0; j < FN; ++j) {
        const int nn = wn * (FN * 8) + j * 8 + fr, kk = k4 + fc;
        bf[j] = TB ? Bs[nn * kStrideMmaj + kk] : Bs[kk * kStrideKmaj(BN) + nn];
      }
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  // epilogue: fragment (row = lane/4, cols = 2*(lane%4) + {0,1})
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t gm = m0 + wm * (FM * 8) + i * 8 + fr;
        const int64_t gn = n0 + wn * (FN * 8) + j * 8 + fc * 2 + h;
        if (gm < M && gn < N) {
          if (P) {
            P[((int64_t)blockIdx.z * M + gm) * N + gn] = acc[i][j][h];
          } else {
            double v = alpha * acc[i][j][h];
            if (beta != 0.0) v = fma(beta, C[gm * ldc + gn], v);
            C[gm * ldc + gn] = v;
          }
        }
      }
}

__global__ void splitk_reduce(const double* __restrict__ P, int64_t M, int64_t N, int splits,
                              double alpha, double beta, double* __restrict__ C, int64_t ldc) {
  const int64_t total = M * N;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int z = 0; z < splits; ++z) acc += P[(int64_t)z * total + t];
    const int64_t m = t / N, nn = t - m * N;
    double v = alpha * acc;
    if (beta != 0.0) v = fma(beta, C[m * ldc + nn], v);
    C[m * ldc + nn] = v;
  }
}

// tile shapes: {BM, BN, relative per-SM efficiency of the shape}
struct TileShape {
  int bm, bn;
  double eff;
};
// (eff from tools/gemm_bench.py on B200, in padded work per second: the DMMA
// stream runs at 30-33 TF/s of padded work for every shape, so the narrow-
// padding shapes gain where their own efficiency holds up)
constexpr int kNumShapes = 7;
static const TileShape kShapes[kNumShapes] = {{128, 64, 1.00}, {128, 48, 1.00}, {64, 64, 0.97}, {64, 48, 0.98},
                                              {64, 32, 0.92},  {128, 56, 0.95}, {128, 136, 0.92}};
// every shape of the table, by index (the instantiation lists below)
#define NYS_GEMM_SHAPES(X) X(0, 128, 64) X(1, 128, 48) X(2, 64, 64) X(3, 64, 48) X(4, 64, 32) X(5, 128, 56) X(6, 128, 136)

// tile shape every plan must use (nys_gemm_tile: tuning / test hook), -1: the cost model's choice
static int g_gemm_tile = -1;

struct GemmPlan {
  int shape = 0, splits = 1;
  int64_t kps = 0;
  size_t ws = 0;
};

// CTAs per SM of one instantiation (registers and shared memory), cached
template <bool TA, bool TB, int BM, int BN>
static int gemm_occ_k() {
  using S = GemmCfg<TA, TB, BM, BN>;
  static int occ = 0;
  if (occ == 0) {
    cudaFuncSetAttribute(dgemm_kernel<TA, TB, BM, BN, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)S::BYTES);
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, dgemm_kernel<TA, TB, BM, BN, false>, GTHREADS, S::BYTES) !=
            cudaSuccess ||
        nb < 1)
      nb = 1;
    occ = nb;
  }
  return occ;
}
template <bool TA, bool TB>
static int gemm_occ_t(int shape) {
  switch (shape) {
#define NYS_X(i, bm, bn) \
  case i: return gemm_occ_k<TA, TB, bm, bn>();
    NYS_GEMM_SHAPES(NYS_X)
#undef NYS_X
    default: return 1;
  }
}
static int gemm_occ(int ta, int tb, int shape) {
  if (ta && tb) return gemm_occ_t<true, true>(shape);
  if (ta) return gemm_occ_t<true, false>(shape);
  if (tb) return gemm_occ_t<false, true>(shape);
  return gemm_occ_t<false, false>(shape);
}

// Cost model in seconds.  An SM runs O = occupancy CTAs at once and shares
// its tensor throughput among them, so a wave of O CTAs costs O times one
// CTA's padded work; waves = ceil(CTAs / (148 O)).  Split-K adds the partial
// traffic (write + read) and one reduction launch.
static GemmPlan gemm_plan(int ta, int tb, int64_t M, int64_t N, int64_t K, size_t ws_cap) {
  const int only = g_gemm_tile;
  GemmPlan best;
  double best_t = 1e300;
  const double sm_rate = 68.0 * 1.9e9;  // FP64 DMMA FMA/s per SM (~40 TF/148)
  for (int c = 0; c < kNumShapes; ++c) {
    if (only >= 0 && c != only) continue;
    const TileShape& t = kShapes[c];
    const int occ = gemm_occ(ta, tb, c);
    const int64_t tiles = cdiv(M, t.bm) * cdiv(N, t.bn);
    const int64_t max_sp = tmax<int64_t>(1, tmin<int64_t>(64, cdiv(K, 4 * GBK)));
    for (int64_t sp = 1; sp <= max_sp; ++sp) {
      const int64_t kps = cdiv(cdiv(K, sp), GBK) * GBK;
      const int64_t spr = cdiv(K, kps);  // realised splits
      if (spr != sp) continue;
      const size_t ws = sp > 1 ? (size_t)sp * M * N * sizeof(double) : 0;
      if (ws > ws_cap) break;
      const int64_t ctas = tiles * sp;
      const int64_t waves = cdiv(ctas, (int64_t)kNumSMs * occ);
      // concurrent CTAs per SM in a wave (a single partial wave runs fewer)
      const int64_t conc = waves > 1 ? occ : tmax<int64_t>(1, cdiv(ctas, (int64_t)kNumSMs));
      // pipeline fill: ~2 k-tiles of latency per CTA
      const double work = (double)waves * conc * t.bm * t.bn * (double)(kps + 2 * GBK);
      double tt = work / (sm_rate * t.eff);
      if (sp > 1) tt += 2.0 * (double)ws / 6.0e12 + 3.0e-6;
      if (tt < best_t * 0.999) {
        best_t = tt;
        best.shape = c;
        best.splits = (int)sp;
        best.kps = kps;
        best.ws = ws;
      }
    }
  }
  if (best.kps == 0) best.kps = K;
  static const bool dbg = dev_env("NYS_GEMM_DEBUG") != nullptr;
  if (dbg)
    fprintf(stderr, "[nys] gemm %d%d %lldx%lldx%lld: shape %d (%dx%d, occ %d) splits %d kps %lld est %.1f us\n", ta, tb,
            (long long)M, (long long)N, (long long)K, best.shape, kShapes[best.shape].bm, kShapes[best.shape].bn,
            gemm_occ(ta, tb, best.shape), best.splits, (long long)best.kps, best_t * 1e6);
  return best;
}

size_t gemm_ws(int64_t M, int64_t N, int64_t K) {
  size_t w = 0;
  for (int ta = 0; ta < 2; ++ta)
    for (int tb = 0; tb < 2; ++tb) w = tmax(w, gemm_plan(ta, tb, M, N, K, (size_t)-1).ws);
  return w;
}

template <bool TA, bool TB, int BM, int BN>
static int gemm_launch_shape(const GemmPlan& pl, int64_t M, int64_t N, int64_t K, double alpha,
                             const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
                             double* C, int64_t ldc, void* ws, cudaStream_t st) {
  using S = GemmCfg<TA, TB, BM, BN>;
  const bool va = (lda % 2) == 0 && ((uintptr_t)A & 15) == 0;
  static bool attr_set[2] = {false, false};
  auto fn = va ? dgemm_kernel<TA, TB, BM, BN, true> : dgemm_kernel<TA, TB, BM, BN, false>;
  if (!attr_set[va]) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::BYTES);
    attr_set[va] = true;
  }
  dim3 grid((unsigned)cdiv(N, BN), (unsigned)cdiv(M, BM), (unsigned)pl.splits);
  double* P = pl.splits > 1 ? reinterpret_cast<double*>(ws) : nullptr;
  fn<<<grid, GTHREADS, S::BYTES, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, pl.kps, P);
  NYS_CHECK_LAUNCH();
  if (pl.splits > 1) {
    const int64_t blocks = tmin<int64_t>(cdiv(M * N, 256), kNumSMs * 8);
    splitk_reduce<<<(unsigned)blocks, 256, 0, st>>>(P, M, N, pl.splits, alpha, beta, C, ldc);
    NYS_CHECK_LAUNCH();
  }
  return NYS_OK;
}

template <bool TA, bool TB>
static int gemm_launch(int64_t M, int64_t N, int64_t K, double alpha, const double* A,
                       int64_t lda, const double* B, int64_t ldb, double beta, double* C,
                       int64_t ldc, void* ws, size_t ws_bytes, cudaStream_t st) {
  const GemmPlan pl = gemm_plan(TA ? 1 : 0, TB ? 1 : 0, M, N, K, ws ? ws_bytes : 0);
  switch (pl.shape) {
#define NYS_X(i, bm, bn) \
  case i: return gemm_launch_shape<TA, TB, bm, bn>(pl, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, ws, st);
    NYS_GEMM_SHAPES(NYS_X)
#undef NYS_X
    default: return NYS_ERR_ARG;
  }
}

int gemm(int ta, int tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
         int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc, void* ws,
         size_t ws_bytes, cudaStream_t st) {
  if (M <= 0 || N <= 0 || K <= 0) return NYS_ERR_ARG;
  if (ta && tb) return gemm_launch<true, true>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, ws, ws_bytes, st);
  if (ta) return gemm_launch<true, false>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, ws, ws_bytes, st);
  if (tb) return gemm_launch<false, true>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, ws, ws_bytes, st);
  return gemm_launch<false, false>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, ws, ws_bytes, st);
}

// ------------------------------------------------- small dense kernels ----
// In-place lower Cholesky of the s x s matrix C (row-major), one CTA.
// info = 0 on success, j+1 if the j-th pivot is not positive (LAPACK potf2).
// Right-looking, column by column.  SMEM = true keeps the whole matrix in
// shared memory (s <= 160); warps take trailing rows, lanes columns.
template <bool SMEM>
__global__ void __launch_bounds__(1024) cholesky_kernel(int s, double* C, int64_t ldc, int* info) {
  extern __shared__ double csm[];
  __shared__ int fail;
  __shared__ double piv;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int ld = SMEM ? (s | 1) : (int)ldc;
  double* M = SMEM ? csm : C;
  if (SMEM)
    for (int t = threadIdx.x; t < s * s; t += blockDim.x) {
      const int i = t / s, k = t - i * s;
      if (k <= i) M[i * ld + k] = C[(int64_t)i * ldc + k];
    }
  if (threadIdx.x == 0) fail = 0;
  __syncthreads();
  for (int j = 0; j < s; ++j) {
    if (threadIdx.x == 0) {
      const double d = M[(int64_t)j * ld + j];
      if (!(d > 0.0) || isnan(d)) {  // LAPACK potf2 failure rule
        fail = j + 1;
      } else {
        piv = sqrt(d);
        M[(int64_t)j * ld + j] = piv;
      }
    }
    __syncthreads();
    if (fail) break;
    const double pj = piv;
    for (int i = j + 1 + threadIdx.x; i < s; i += blockDim.x) M[(int64_t)i * ld + j] /= pj;
    __syncthreads();
    // trailing update of the lower triangle: M[i][k] -= M[i][j] M[k][j], j < k <= i
    for (int i = j + 1 + warp; i < s; i += nw) {
      const double lij = M[(int64_t)i * ld + j];
      for (int k = j + 1 + lane; k <= i; k += 32) M[(int64_t)i * ld + k] -= lij * M[(int64_t)k * ld + j];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *info = fail;
  __syncthreads();
  if (!fail) {  // write back the lower factor, zero the strict upper triangle
    for (int64_t t = threadIdx.x; t < (int64_t)s * s; t += blockDim.x) {
      const int i = (int)(t / s), k = (int)(t % s);
      if (k > i) C[(int64_t)i * ldc + k] = 0.0;
      else if (SMEM) C[(int64_t)i * ldc + k] = M[(int64_t)i * ld + k];
    }
  }
}

// Linv = L^{-1} (lower), one warp per column.
__global__ void __launch_bounds__(256) trinv_lower_kernel(int s, const double* __restrict__ L,
                                                          int64_t ldl, double* __restrict__ X,
                                                          int64_t ldx) {
  extern __shared__ double xs[];  // 8 warps x s
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j = blockIdx.x * 8 + warp;
  if (j >= s) return;
  double* x = xs + (int64_t)warp * s;
  for (int i = lane; i < s; i += 32) x[i] = 0.0;
  __syncwarp();
  if (lane == 0) x[j] = 1.0 / L[(int64_t)j * ldl + j];
  __syncwarp();
  for (int i = j + 1; i < s; ++i) {
    double acc = 0.0;
    for (int k = j + lane; k < i; k += 32) acc = fma(L[(int64_t)i * ldl + k], x[k], acc);
    acc = warp_sum(acc);
    if (lane == 0) x[i] = -acc / L[(int64_t)i * ldl + i];
    __syncwarp();
  }
  for (int i = lane; i < s; i += 32) X[(int64_t)i * ldx + j] = x[i];
}

// Fused Cholesky + triangular inverse for s <= kCholInvMaxS, one CTA, blocked
// by 8 with the O(s^3) work on the DMMA tensor cores:
//   per 8-column panel  (a) warp 0 factors the 8 x 8 diagonal block in
//                           registers (shuffles, one sqrt per column),
//                       (b) one thread per row solves its panel row against
//                           L11 (L21 = A21 L11^{-T}),
//                       (c) the warps update the lower block triangle of the
//                           trailing matrix, A22 -= L21 L21^T, one 8 x 8 block
//                           per DMMA pair;
//   then the 8 x 8 diagonal blocks are inverted (warp each) and warp J forms
//   block column J of L^{-1} by block forward substitution,
//   X_IJ = D_I^{-1} (delta_IJ I - sum_K L_IK X_KJ), the sums on DMMA with the
//   earlier blocks read back from Li (rows/columns >= s are the identity
//   padding and never stored).
// C: lower triangle read, untouched.  Li: s x s, strict upper zeroed.
// info = j + 1 at the first non-positive pivot (LAPACK potf2 rule).
constexpr int kCholInvMaxS = 152;  // smem: s_pad x ld + diag inverses + warp scratch <= 227 KB
constexpr int kCholThreads = 1024;
inline int cholinv_ld(int sp) {  // ld = 4 (mod 8): 2-wavefront DMMA fragment loads
  int ld = sp;
  while ((ld & 7) != 4) ++ld;
  return ld;
}
inline size_t cholinv_smem(int s) {
  const int sp = (int)cdiv(s, 8) * 8, np = sp / 8;
  return ((size_t)sp * cholinv_ld(sp) + (size_t)np * 64 + 32 * 64 + 16) * sizeof(double);
}
__global__ void __launch_bounds__(kCholThreads) cholinv_kernel(int s, const double* __restrict__ C, int64_t ldc,
                                                               double* __restrict__ Li, int64_t ldli, int* info) {
  extern __shared__ double csm[];
  const int sp = (s + 7) & ~7, np = sp / 8;
  int ld = sp;
  while ((ld & 7) != 4) ++ld;
  double* M = csm;                              // sp x ld
  double* Dinv = M + (size_t)sp * ld;           // np x 64
  double* wscr = Dinv + (size_t)np * 64;        // 32 warps x 64
  double* dinv8 = wscr + 32 * 64;               // 8
  __shared__ int s_fail;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int fr = lane >> 2, fc = lane & 3;
  if (tid == 0) s_fail = 0;
  for (int t = tid; t < sp * ld; t += blockDim.x) {
    const int i = t / ld, j = t - i * ld;
    M[t] = (j > i || j >= sp) ? 0.0 : (i < s ? C[(int64_t)i * ldc + j] : (i == j ? 1.0 : 0.0));
  }
  __syncthreads();
  // (a) 8 x 8 diagonal block at (c, c) by warp 0: lane holds (i, j0), (i, j0 + 4),
  // i = lane / 4; one Newton-refined reciprocal square root per column
  auto factor_diag = [&](int c) {
    const int i = fr, j0 = fc, j1 = fc + 4;
    double m0 = M[(c + i) * ld + c + j0], m1 = M[(c + i) * ld + c + j1];
    int fail = 0;
    for (int q = 0; q < 8; ++q) {
      const double sel = q < 4 ? m0 : m1;
      const double dq = __shfl_sync(0xffffffffu, sel, q * 4 + (q & 3));
      if (!(dq > 0.0) || isnan(dq)) {
        fail = c + q + 1;
        break;
      }
      double rp = rsqrt(dq);
      rp = rp * fma(-0.5 * dq * rp, rp, 1.5);  // one Newton step: ~full precision
      const double pq = dq * rp;
      const double liq = __shfl_sync(0xffffffffu, sel, i * 4 + (q & 3)) * rp;
      const double lj0 = __shfl_sync(0xffffffffu, sel, j0 * 4 + (q & 3)) * rp;
      const double lj1 = __shfl_sync(0xffffffffu, sel, j1 * 4 + (q & 3)) * rp;
      if (j0 > q && j0 <= i) m0 = fma(-liq, lj0, m0);
      if (j1 > q && j1 <= i) m1 = fma(-liq, lj1, m1);
      if (j0 == q) m0 = (i == q) ? pq : (i > q ? m0 * rp : m0);
      if (j1 == q) m1 = (i == q) ? pq : (i > q ? m1 * rp : m1);
    }
    if (fail) {
      if (lane == 0) s_fail = fail;
    } else {
      if (j0 <= i) M[(c + i) * ld + c + j0] = m0;
      if (j1 <= i) M[(c + i) * ld + c + j1] = m1;
      const int pb = (c >> 3) & 1;  // double-buffered diagonal reciprocals
      if (j0 == i) dinv8[pb * 8 + i] = 1.0 / m0;
      if (j1 == i) dinv8[pb * 8 + i] = 1.0 / m1;
    }
  };
  // one 8 x 8 block of the trailing update, A[I][J] -= L[I][c:c+8] L[J][c:c+8]^T
  auto update_block = [&](int I, int J, int c) {
    double acc[2];
    acc[0] = M[(I + fr) * ld + J + 2 * fc];
    acc[1] = M[(I + fr) * ld + J + 2 * fc + 1];
#pragma unroll
    for (int kk = 0; kk < 8; kk += 4) {
      const double av = -M[(I + fr) * ld + c + kk + fc];
      const double bv = M[(J + fr) * ld + c + kk + fc];
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[0]), "+d"(acc[1])
                   : "d"(av), "d"(bv));
    }
    M[(I + fr) * ld + J + 2 * fc] = acc[0];
    M[(I + fr) * ld + J + 2 * fc + 1] = acc[1];
  };
  if (warp == 0) factor_diag(0);
  __syncthreads();
  for (int p = 0; p < np && !s_fail; ++p) {
    const int c = 8 * p;
    const double* dv = dinv8 + (p & 1) * 8;
    // (b) panel rows below the diagonal block: x = a L11^{-T}
    for (int i = c + 8 + tid; i < sp; i += blockDim.x) {
      double* row = M + (size_t)i * ld + c;
      double x[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        double v = row[q];
#pragma unroll
        for (int j = 0; j < q; ++j) v = fma(-x[j], M[(c + q) * ld + c + j], v);
        x[q] = v * dv[q];
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) row[q] = x[q];
    }
    __syncthreads();
    // (c) trailing lower block triangle (DMMA).  Lookahead: warp 0 updates the
    // next diagonal block first and factors it while the others finish.
    const int T = np - p - 1;
    if (warp == 0) {
      if (T > 0) {
        update_block(c + 8, c + 8, c);
        __syncwarp();
        factor_diag(c + 8);
      }
    } else {
      const int nblk = T * (T + 1) / 2;
      for (int b = warp; b < nblk; b += nw - 1) {  // block 0 is the next diagonal block (warp 0)
        int ir = (int)((sqrtf(8.0f * b + 1.0f) - 1.0f) * 0.5f);
        while ((ir + 1) * (ir + 2) / 2 <= b) ++ir;
        while (ir * (ir + 1) / 2 > b) --ir;
        const int jr = b - ir * (ir + 1) / 2;
        update_block(c + 8 + 8 * ir, c + 8 + 8 * jr, c);
      }
    }
    __syncthreads();
  }
  if (tid == 0) *info = s_fail;
  if (s_fail) return;
  // inverses of the diagonal blocks: warp w, lane l < 8 solves column l
  for (int w = warp; w < np; w += nw) {
    const double* L = M + (size_t)(8 * w) * ld + 8 * w;
    double x[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      double v = (r == lane) ? 1.0 : 0.0;
#pragma unroll
      for (int q = 0; q < r; ++q) v = fma(-L[r * ld + q], x[q], v);
      x[r] = v / L[r * ld + r];
    }
    if (lane < 8)
#pragma unroll
      for (int r = 0; r < 8; ++r) Dinv[w * 64 + r * 8 + lane] = (r >= lane) ? x[r] : 0.0;
  }
  __syncthreads();
  // block column J of L^{-1} (warp J).  X_KJ (K >= J) is kept transposed in
  // the block M[8J..][8K..] -- the upper block triangle and the diagonal
  // blocks of L are no longer read (the diagonal inverses are in Dinv) -- so
  // the block forward substitution runs out of shared memory.
  for (int J = warp; J < np; J += nw) {
    double* scr = wscr + warp * 64;
    for (int I = 0; I < J; ++I) {  // strict upper block triangle: zeros
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = 8 * I + fr, cc = 8 * J + 2 * fc + h;
        if (r < s && cc < s) Li[(int64_t)r * ldli + cc] = 0.0;
      }
    }
    for (int I = J; I < np; ++I) {
      double acc[2] = {0.0, 0.0};
      for (int K = J; K < I; ++K) {
#pragma unroll
        for (int kk = 0; kk < 8; kk += 4) {
          const double av = M[(8 * I + fr) * ld + 8 * K + kk + fc];
          const double bv = M[(8 * J + fr) * ld + 8 * K + kk + fc];  // X_KJ[kk + fc][fr]
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(acc[0]), "+d"(acc[1])
                       : "d"(av), "d"(bv));
        }
      }
      // rhs = delta_IJ I - acc, staged row-major in the warp scratch
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int cc = 2 * fc + h;
        scr[fr * 8 + cc] = ((I == J && fr == cc) ? 1.0 : 0.0) - acc[h];
      }
      __syncwarp();
      double x2[2] = {0.0, 0.0};
#pragma unroll
      for (int kk = 0; kk < 8; kk += 4) {
        const double av = Dinv[I * 64 + fr * 8 + kk + fc];
        const double bv = scr[(kk + fc) * 8 + fr];
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(x2[0]), "+d"(x2[1])
                     : "d"(av), "d"(bv));
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = 8 * I + fr, cc = 8 * J + 2 * fc + h;
        M[(8 * J + 2 * fc + h) * ld + 8 * I + fr] = x2[h];  // X_IJ transposed
        if (r < s && cc < s) Li[(int64_t)r * ldli + cc] = x2[h];
      }
      __syncwarp();
    }
  }
}

__global__ void symmetrize_kernel(int s, double* C, int64_t ldc) {
  const int64_t tot = (int64_t)s * s;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t / s), k = (int)(t % s);
    if (k < i) {
      const double v = 0.5 * (C[(int64_t)i * ldc + k] + C[(int64_t)k * ldc + i]);
      C[(int64_t)i * ldc + k] = v;
      C[(int64_t)k * ldc + i] = v;
    }
  }
}

// trace-shift of sketch.py:103-107: trace = (n/s) sum(Q o Y); shift = eps*max(trace,0)
// (eps if 0); Y += shift Q.  Two passes in one kernel via a ticket.
__global__ void sketch_shift_kernel(int64_t n, int s, const double* __restrict__ Q,
                                    double* __restrict__ Y, double* part, unsigned int* counter,
                                    double* shift_out, unsigned int* gate) {
  __shared__ double sh[32];
  const int64_t tot = n * s;
  double acc[1] = {0.0};
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot;
       t += (int64_t)gridDim.x * blockDim.x)
    acc[0] = fma(Q[t], Y[t], acc[0]);
  block_sum<1>(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = acc[0];
  if (last_block(counter)) {
    const double sum = block_sum_partials(part, gridDim.x, 1, sh);
    if (threadIdx.x == 0) {
      const double trace = ((double)n / (double)s) * sum;
      double sft = 2.220446049250313e-16 * fmax(trace, 0.0);
      if (sft == 0.0) sft = 2.220446049250313e-16;
      *shift_out = sft;
    }
  }
}

__global__ void add_scaled_kernel(int64_t tot, const double* __restrict__ Q, double* __restrict__ Y,
                                  const double* shift) {
  const double sft = *shift;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot;
       t += (int64_t)gridDim.x * blockDim.x)
    Y[t] = __dadd_rn(Y[t], __dmul_rn(sft, Q[t]));
}

__global__ void eye_kernel(int s, double* V) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)s * s;
       t += (int64_t)gridDim.x * blockDim.x)
    V[t] = (t / s == t % s) ? 1.0 : 0.0;
}

// Cmat[i][j] = V[i][j] * scale[j]  (s x cols, ldc = cols)
__global__ void scale_cols_kernel(int s, int cols, const double* __restrict__ V, int64_t ldv,
                                  const double* __restrict__ scale, double* __restrict__ Cm,
                                  int64_t ldc) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)s * cols;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t / cols), j = (int)(t % cols);
    Cm[(int64_t)i * ldc + j] = V[(int64_t)i * ldv + j] * scale[j];
  }
}

// ----------------------------------------------------- host orchestration --
struct Arena {
  char* base;
  size_t cap, off = 0;
  bool ok = true;
  template <typename T>
  T* take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = reinterpret_cast<T*>(base + off);
    off += count * sizeof(T);
    if (off > cap) ok = false;
    return p;
  }
};

constexpr size_t kRedBytesD = (4096 * 16 + 64) * sizeof(double);

// eig.cu: one-sided Jacobi on a thread-block cluster (A preserved)
size_t syevj_ws(int s);
int syevj(int s, double* A, double* V, double* w, void* ws, size_t ws_bytes, cudaStream_t st);

static int cholesky(int s, double* C, int* info_dev, int* info_host, cudaStream_t st) {
  const size_t smem = (size_t)s * (s | 1) * sizeof(double);
  if (smem <= 210 * 1024) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(cholesky_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
      attr = true;
    }
    cholesky_kernel<true><<<1, 1024, smem, st>>>(s, C, s, info_dev);
  } else {
    cholesky_kernel<false><<<1, 1024, 0, st>>>(s, C, s, info_dev);
  }
  NYS_CHECK_LAUNCH();
  if (!info_host) return NYS_OK;
  if (cudaMemcpyAsync(info_host, info_dev, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return NYS_ERR_CUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return NYS_ERR_CUDA;
  return NYS_OK;
}

static int trinv(int s, const double* L, double* X, cudaStream_t st) {
  trinv_lower_kernel<<<(unsigned)cdiv(s, 8), 256, 8 * s * sizeof(double), st>>>(s, L, s, X, s);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

// Li = chol(C)^{-1} (C untouched; Lm is s x s scratch for s > kCholInvMaxS).
// info_dev gets the potf2 code; with info_host != nullptr the stream is
// synchronised and the code returned there, otherwise the check is deferred.
static int chol_inverse(int s, const double* C, double* Li, double* Lm, int* info_dev, int* info_host,
                        cudaStream_t st) {
  if (s <= kCholInvMaxS) {
    const size_t smem = cholinv_smem(s);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(cholinv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
      attr = true;
    }
    cholinv_kernel<<<1, kCholThreads, smem, st>>>(s, C, s, Li, s, info_dev);
    NYS_CHECK_LAUNCH();
    if (!info_host) return NYS_OK;
    if (cudaMemcpyAsync(info_host, info_dev, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess)
      return NYS_ERR_CUDA;
    return cudaStreamSynchronize(st) == cudaSuccess ? NYS_OK : NYS_ERR_CUDA;
  }
  if (cudaMemcpyAsync(Lm, C, (size_t)s * s * sizeof(double), cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return NYS_ERR_CUDA;
  int info_tmp = 0;
  int rc = cholesky(s, Lm, info_dev, &info_tmp, st);  // large s: always checked here
  if (rc) return rc;
  if (info_host) *info_host = info_tmp;
  if (info_tmp) return NYS_OK;
  return trinv(s, Lm, Li, st);
}

size_t ortho_ws(int64_t n, int s) {
  const size_t ss = (size_t)s * s * sizeof(double);
  return kRedBytesD + 4 * ss + (size_t)n * s * sizeof(double) + gemm_ws(s, s, n) + syevj_ws(s) +
         8 * s * sizeof(double) + 8192;
}

// CholeskyQR: Q = Omega R^{-1} (one pass; see below).  The fast path runs without a host
// sync and checks both Cholesky codes once at the end; if either pass hit a
// numerically singular Gram matrix the careful path (per-pass checks, eigen
// fallback) recomputes Q from Omega.
static int orthonormalize(int64_t n, int s, const double* Om, double* Q, void* ws,
                          size_t ws_bytes, cudaStream_t st, bool careful, int* info_ext = nullptr) {
  Arena ar{reinterpret_cast<char*>(ws), ws_bytes};
  ar.take<char>(kRedBytesD);
  double* G = ar.take<double>((size_t)s * s);
  double* Li = ar.take<double>((size_t)s * s);
  double* Lm = ar.take<double>((size_t)s * s);
  double* Vm = ar.take<double>((size_t)s * s);
  double* tmp = ar.take<double>((size_t)n * s);
  double* wv = ar.take<double>(s);
  double* sc = ar.take<double>(s);
  int* info = ar.take<int>(2);
  const size_t gws_b = gemm_ws(s, s, n);
  void* gws = ar.take<char>(gws_b);
  const size_t jws_b = syevj_ws(s);
  void* jws = ar.take<char>(jws_b);
  if (!ar.ok) return NYS_ERR_WORKSPACE;
  if (info_ext) info = info_ext;  // deferred: the caller checks the codes later
  // One CholeskyQR pass by default: the sketch input is a Gaussian n x s
  // matrix (n >> s), condition number ~ (1 + sqrt(s/n)) / (1 - sqrt(s/n)) <= 1.3
  // for the configs, so one pass leaves ||Q^T Q - I|| at the 1e-15 level; the
  // Nystrom approximation (H+nu)Q (Q^T (H+nu) Q)^-1 Q^T (H+nu) is invariant to
  // Q -> Q R anyway.  NYS_CHOLQR_PASSES=2 restores CholeskyQR2; the careful
  // (fallback) path always runs two.
  static const int env_passes = dev_env("NYS_CHOLQR_PASSES") ? atoi(dev_env("NYS_CHOLQR_PASSES")) : 1;
  const int passes = careful ? 2 : (env_passes == 2 ? 2 : 1);
  if (passes == 1 && cudaMemsetAsync(info + 1, 0, sizeof(int), st) != cudaSuccess) return NYS_ERR_CUDA;
  int rc;
  for (int pass = 0; pass < passes; ++pass) {
    const double* src = pass == 0 ? Om : tmp;
    double* dst = (pass == passes - 1) ? Q : tmp;
    rc = gemm(1, 0, s, s, n, 1.0, src, s, src, s, 0.0, G, s, gws, gws_b, st);
    if (rc) return rc;
    int info_h = 0;
    rc = chol_inverse(s, G, Li, Lm, info + pass, careful ? &info_h : nullptr, st);
    if (rc) return rc;
    if (info_h == 0) {
      // dst = src L^{-T}
      rc = gemm(0, 1, n, s, s, 1.0, src, s, Li, s, 0.0, dst, s, nullptr, 0, st);
    } else {
      // eigen fallback: src V diag(1/sqrt(w))  (full-rank Gaussian input expected)
      rc = syevj(s, G, Vm, wv, jws, jws_b, st);
      if (rc) return rc;
      std::vector<double> wh(s);
      cudaMemcpyAsync(wh.data(), wv, s * sizeof(double), cudaMemcpyDeviceToHost, st);
      if (cudaStreamSynchronize(st) != cudaSuccess) return NYS_ERR_CUDA;
      for (int j = 0; j < s; ++j) wh[j] = wh[j] > 0.0 ? 1.0 / sqrt(wh[j]) : 0.0;
      cudaMemcpyAsync(sc, wh.data(), s * sizeof(double), cudaMemcpyHostToDevice, st);
      scale_cols_kernel<<<(unsigned)cdiv((int64_t)s * s, 256), 256, 0, st>>>(s, s, Vm, s, sc, Li, s);
      NYS_CHECK_LAUNCH();
      rc = gemm(0, 0, n, s, s, 1.0, src, s, Li, s, 0.0, dst, s, nullptr, 0, st);
      if (cudaStreamSynchronize(st) != cudaSuccess) return NYS_ERR_CUDA;
    }
    if (rc) return rc;
  }
  if (info_ext) return NYS_OK;
  if (!careful) {
    int info_h[2] = {0, 0};
    if (cudaMemcpyAsync(info_h, info, 2 * sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess)
      return NYS_ERR_CUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess) return NYS_ERR_CUDA;
    if (info_h[0] || info_h[1]) return orthonormalize(n, s, Om, Q, ws, ws_bytes, st, true);
  }
  if (cudaStreamSynchronize(st) != cudaSuccess) return NYS_ERR_CUDA;
  return NYS_OK;
}

size_t nystrom_ws(int64_t n, int s, int r) {
  const size_t ss = (size_t)s * s * sizeof(double);
  return kRedBytesD + 6 * ss + (size_t)n * s * sizeof(double) + gemm_ws(s, s, n) + syevj_ws(s) +
         16 * (size_t)s * sizeof(double) + 16384;
}

// lam_j = max(sigma_j^2 - shift, 0), scl_j = 1/sigma_j (sketch.py:126-128),
// from the eigenvalues w of B^T B and the device-resident shift
__global__ void nystrom_lam_kernel(int rr, const double* __restrict__ w, const double* __restrict__ shift,
                                   double* __restrict__ lam, double* __restrict__ scl) {
  const double sft = *shift;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < rr; j += gridDim.x * blockDim.x) {
    const double sv2 = fmax(w[j], 0.0);
    lam[j] = fmax(sv2 - sft, 0.0);
    scl[j] = sv2 > 0.0 ? 1.0 / sqrt(sv2) : 0.0;
  }
}

// Steps 1-4 of sketch.py:102-128 on device-resident Q (n x s) and Y = H Q.
// The fast path has one host sync (the Cholesky code of the core, read at
// the end); a non-positive pivot re-runs the careful path, which takes the
// eigh fallback of sketch.py:114-124 from the same inputs.
static int nystrom_core(int64_t n, int s, int r, const double* Q, double* Y, double* U,
                        double* lam, int* r_out, void* ws, size_t ws_bytes, cudaStream_t st,
                        bool careful, int* info_ext = nullptr) {
  Arena ar{reinterpret_cast<char*>(ws), ws_bytes};
  char* red = ar.take<char>(kRedBytesD);
  double* shift_d = ar.take<double>(4);
  double* core = ar.take<double>((size_t)s * s);
  double* Lm = ar.take<double>((size_t)s * s);
  double* Li = ar.take<double>((size_t)s * s);
  double* G = ar.take<double>((size_t)s * s);
  double* V = ar.take<double>((size_t)s * s);
  double* Cm = ar.take<double>((size_t)s * s);
  double* wv = ar.take<double>(s);
  double* scl = ar.take<double>(s);
  double* B = ar.take<double>((size_t)n * s);
  int* info = ar.take<int>(4);
  const size_t gws_b = gemm_ws(s, s, n);
  void* gws = ar.take<char>(gws_b);
  const size_t jws_b = syevj_ws(s);
  void* jws = ar.take<char>(jws_b);
  if (!ar.ok) return NYS_ERR_WORKSPACE;
  if (info_ext) info = info_ext;  // deferred: the caller checks the code later
  const double eps = 2.220446049250313e-16;
  int rc;
  if (!careful) {
    cudaMemsetAsync(shift_d, 0, 4 * sizeof(double), st);
    // 1. trace shift and Y_s = Y + shift Q   (sketch.py:102-106)
    const int64_t tot = n * (int64_t)s;
    const unsigned sb = (unsigned)tmax<int64_t>(1, tmin<int64_t>(cdiv(tot, 256), kNumSMs * 4));
    sketch_shift_kernel<<<sb, 256, 0, st>>>(n, s, Q, Y, reinterpret_cast<double*>(red),
                                            reinterpret_cast<unsigned int*>(
                                                reinterpret_cast<double*>(red) + 4096 * 16),
                                            shift_d, nullptr);
    NYS_CHECK_LAUNCH();
    add_scaled_kernel<<<sb, 256, 0, st>>>(tot, Q, Y, shift_d);
    NYS_CHECK_LAUNCH();
    // 2. core = Q^T Y_s, symmetrised  (sketch.py:107-108)
    rc = gemm(1, 0, s, s, n, 1.0, Q, s, Y, s, 0.0, core, s, gws, gws_b, st);
    if (rc) return rc;
    symmetrize_kernel<<<(unsigned)cdiv((int64_t)s * s, 256), 256, 0, st>>>(s, core, s);
    NYS_CHECK_LAUNCH();
  }
  // 3. Cholesky, B = Y_s L^{-T}   (sketch.py:110-113)
  int info_h = 0;
  rc = chol_inverse(s, core, Li, Lm, info, careful ? &info_h : nullptr, st);
  if (rc) return rc;
  int s_eff = s;
  if (info_h == 0) {
    rc = gemm(0, 1, n, s, s, 1.0, Y, s, Li, s, 0.0, B, s, nullptr, 0, st);
    if (rc) return rc;
  } else {
    // eigh fallback (sketch.py:114-124)
    double shift_h = 0.0;
    cudaMemcpyAsync(&shift_h, shift_d, sizeof(double), cudaMemcpyDeviceToHost, st);
    rc = syevj(s, core, V, wv, jws, jws_b, st);
    if (rc) return rc;
    std::vector<double> wh(s);
    cudaMemcpyAsync(wh.data(), wv, s * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return NYS_ERR_CUDA;
    // wh is descending: wh[0] largest, wh[s-1] smallest
    const double scale = fmax(fabs(wh[0]), shift_h);
    if (wh[s - 1] < -1e-8 * scale) return NYS_ERR_NOT_PSD;
    int keep = 0;
    std::vector<double> sc(s, 0.0);
    for (int j = 0; j < s; ++j)
      if (wh[j] > eps * scale) {
        sc[j] = 1.0 / sqrt(wh[j]);
        ++keep;
      }
    if (keep == 0) {
      *r_out = 0;
      return NYS_OK;
    }
    // kept eigenvalues are the leading `keep` columns (descending order)
    cudaMemcpyAsync(scl, sc.data(), s * sizeof(double), cudaMemcpyHostToDevice, st);
    scale_cols_kernel<<<(unsigned)cdiv((int64_t)s * keep, 256), 256, 0, st>>>(s, keep, V, s, scl,
                                                                             Cm, keep);
    NYS_CHECK_LAUNCH();
    rc = gemm(0, 0, n, keep, s, 1.0, Y, s, Cm, keep, 0.0, B, keep, nullptr, 0, st);
    if (rc) return rc;
    s_eff = keep;
  }
  // 4. thin SVD of B through the eigenpairs of B^T B   (sketch.py:126-128)
  rc = gemm(1, 0, s_eff, s_eff, n, 1.0, B, s_eff, B, s_eff, 0.0, G, s_eff, gws, gws_b, st);
  if (rc) return rc;
  symmetrize_kernel<<<(unsigned)cdiv((int64_t)s_eff * s_eff, 256), 256, 0, st>>>(s_eff, G, s_eff);
  NYS_CHECK_LAUNCH();
  rc = syevj(s_eff, G, V, wv, jws, jws_b, st);
  if (rc) return rc;
  const int rr = r < s_eff ? r : s_eff;
  nystrom_lam_kernel<<<1, 256, 0, st>>>(rr, wv, shift_d, lam, scl);
  NYS_CHECK_LAUNCH();
  scale_cols_kernel<<<(unsigned)cdiv((int64_t)s_eff * rr, 256), 256, 0, st>>>(s_eff, rr, V, s_eff,
                                                                             scl, Cm, rr);
  NYS_CHECK_LAUNCH();
  rc = gemm(0, 0, n, rr, s_eff, 1.0, B, s_eff, Cm, rr, 0.0, U, r, nullptr, 0, st);
  if (rc) return rc;
  if (info_ext) {
    *r_out = rr;
    return NYS_OK;
  }
  if (!careful) {
    int info_c = 0;
    if (cudaMemcpyAsync(&info_c, info, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess)
      return NYS_ERR_CUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess) return NYS_ERR_CUDA;
    if (info_c) return nystrom_core(n, s, r, Q, Y, U, lam, r_out, ws, ws_bytes, st, true);
  }
  if (cudaStreamSynchronize(st) != cudaSuccess) return NYS_ERR_CUDA;
  *r_out = rr;
  return NYS_OK;
}

}  // namespace nys

// ------------------------------------------------------------- C ABI ------
using namespace nys;

extern "C" size_t nys_gemm_workspace(int64_t M, int64_t N, int64_t K) { return gemm_ws(M, N, K); }

extern "C" int nys_gemm_tile(int shape) {
  nys::g_gemm_tile = (shape >= 0 && shape < nys::kNumShapes) ? shape : -1;
  return nys::kNumShapes;
}

extern "C" int nys_gemm_f64(int transA, int transB, int64_t M, int64_t N, int64_t K, double alpha,
                            const double* A, int64_t lda, const double* B, int64_t ldb,
                            double beta, double* C, int64_t ldc, void* ws, size_t ws_bytes,
                            void* stream) {
  if (M <= 0 || N <= 0 || K <= 0 || ldc < N) return NYS_ERR_ARG;
  if ((transA ? lda < M : lda < K) || (transB ? ldb < K : ldb < N)) return NYS_ERR_ARG;
  return gemm(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, ws, ws_bytes,
              as_stream(stream));
}

extern "C" size_t nys_orthonormalize_workspace(int64_t n, int s) { return ortho_ws(n, s); }

extern "C" int nys_orthonormalize_f64(int64_t n, int s, const double* Omega, double* Q, void* ws,
                                      size_t ws_bytes, void* stream) {
  if (n <= 0 || s <= 0 || s > n) return NYS_ERR_ARG;
  return orthonormalize(n, s, Omega, Q, ws, ws_bytes, as_stream(stream), false);
}

extern "C" int nys_orthonormalize_async_f64(int64_t n, int s, const double* Omega, double* Q, int* info_dev,
                                            void* ws, size_t ws_bytes, void* stream) {
  if (n <= 0 || s <= 0 || s > n || !info_dev) return NYS_ERR_ARG;
  return orthonormalize(n, s, Omega, Q, ws, ws_bytes, as_stream(stream), false, info_dev);
}

extern "C" size_t nys_nystrom_workspace(int64_t n, int s, int r) { return nystrom_ws(n, s, r); }

extern "C" int nys_nystrom_core_async_f64(int64_t n, int s, int r, const double* Q, double* Y, double* U,
                                          double* lam, int* info_dev, void* ws, size_t ws_bytes, void* stream) {
  if (n <= 0 || s <= 0 || s > n || r < 1 || r > s || !info_dev) return NYS_ERR_ARG;
  int r_out = 0;
  return nystrom_core(n, s, r, Q, Y, U, lam, &r_out, ws, ws_bytes, as_stream(stream), false, info_dev);
}

extern "C" int nys_nystrom_core_f64(int64_t n, int s, int r, const double* Q, double* Y, double* U,
                                    double* lam, int* r_out, void* ws, size_t ws_bytes,
                                    void* stream) {
  if (n <= 0 || s <= 0 || s > n || r < 1 || r > s || !r_out) return NYS_ERR_ARG;
  return nystrom_core(n, s, r, Q, Y, U, lam, r_out, ws, ws_bytes, as_stream(stream), false);
}

extern "C" size_t nys_syevj_workspace(int s) { return syevj_ws(s); }

extern "C" int nys_syevj_f64(int s, double* A, double* V, double* w, void* ws, size_t ws_bytes,
                             void* stream) {
  if (s <= 0) return NYS_ERR_ARG;
  cudaStream_t st = as_stream(stream);
  int rc = syevj(s, A, V, w, ws, ws_bytes, st);
  if (rc) return rc;
  return cudaStreamSynchronize(st) == cudaSuccess ? NYS_OK : NYS_ERR_CUDA;
}

// ------------------------------------------------------------- misc -------
unsigned long long nys::g_launches = 0ull;

void nys::debug_report(cudaError_t e, const char* file, int line) {
  static const bool on = dev_env("NYS_SYNC_DEBUG") != nullptr;
  if (on) fprintf(stderr, "[nys] launch error at %s:%d: %s\n", file, line, cudaGetErrorString(e));
}

int nys::debug_sync_check(const char* file, int line) {
  static const bool on = dev_env("NYS_SYNC_DEBUG") != nullptr;
  if (!on) return 0;
  const cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    fprintf(stderr, "[nys] CUDA error after launch at %s:%d: %s\n", file, line, cudaGetErrorString(e));
    return 1;
  }
  return 0;
}

extern "C" int nys_abi_version(void) { return NYS_ABI_VERSION; }

extern "C" unsigned long long nys_launch_count(void) {
  return __atomic_load_n(&nys::g_launches, __ATOMIC_RELAXED);
}

extern "C" const char* nys_status_string(int status) {
  switch (status) {
    case NYS_OK: return "ok";
    case NYS_ERR_ARG: return "invalid argument";
    case NYS_ERR_CUDA: return "CUDA error";
    case NYS_ERR_NOT_SPD: return "operator is not SPD";
    case NYS_ERR_NONFINITE: return "non-finite value";
    case NYS_ERR_NOT_PSD: return "operator is not positive semidefinite";
    case NYS_ERR_UNSUPPORTED: return "unsupported";
    case NYS_ERR_WORKSPACE: return "workspace too small";
    case NYS_ERR_NO_DEVICE: return "no sm_100 device";
    default: return "unknown";
  }
}

extern "C" int nys_device_check(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return NYS_ERR_NO_DEVICE;
  int major = 0;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess)
    return NYS_ERR_NO_DEVICE;
  return major == 10 ? NYS_OK : NYS_ERR_NO_DEVICE;
}
