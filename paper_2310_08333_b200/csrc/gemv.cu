// K1 / K2 / K3: FP64 dense products on row-major A.
//
//   K1  Y = A X        (operators.py:114-115), k <= 4 right-hand sides
//   K2  Y = A^T T      (operators.py:117-118), k <= 4 right-hand sides
//   K3  y = A^T(d o Av) + shift v, pAp = v.y   (problems.py:263-264, admm.py:262-263)
//
// All three are HBM-bound streams of A (8 bytes per element, 1/4 flop per
// byte per RHS).  Design for B200:
//   * 128-bit (double2) coalesced loads of A rows; a warp covers 512 B per load;
//   * K1: one warp owns RW=4 rows so every load of X is reused 4x from
//     registers (X traffic from L1/L2 = k/4 of the A traffic); columns are
//     split when there are too few row groups to fill 148 SMs;
//   * K2: a CTA owns a 512-column strip and a contiguous row range; the
//     per-row coefficients T are staged in shared memory; splits over rows are
//     summed in a fixed order by a second kernel (deterministic, no atomics);
//   * grids are sized in multiples of the 148 SMs.
#include <stdlib.h>
#include "common.cuh"
#include "hvp_plan.cuh"

namespace nys {

// ------------------------------------------------------------------ K1 ----
constexpr int kGemvThreads = 256;
constexpr int kGemvRW = 4;

template <int K, int RW, int U, bool VEC>
__global__ void __launch_bounds__(kGemvThreads, 2)
gemv_n_kernel(const double* __restrict__ A, int64_t rows, int64_t n, int64_t lda,
              const double* __restrict__ X, int64_t ldx, double* __restrict__ Y, int64_t ldy,
              const double* __restrict__ dscale, int splits, int64_t chunk,
              const double* __restrict__ pred) {
  if (pred && *pred != 0.0) return;  // device-predicated launch (CG batches)
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t ngroups = cdiv(rows, RW);
  if (warp >= ngroups * splits) return;
  const int64_t g = warp % ngroups;
  const int s = (int)(warp / ngroups);
  const int64_t r0 = g * RW;
  const int64_t c0 = (int64_t)s * chunk;
  const int64_t c1 = min(n, c0 + chunk);

  const double* arow[RW];
#pragma unroll
  for (int r = 0; r < RW; ++r) arow[r] = A + min(r0 + r, rows - 1) * lda;

  double acc[RW][K];
#pragma unroll
  for (int r = 0; r < RW; ++r)
#pragma unroll
    for (int j = 0; j < K; ++j) acc[r][j] = 0.0;

  if (VEC) {
    int64_t c = c0 + 2 * lane;
    for (; c + 64 * (U - 1) + 1 < c1; c += 64 * U) {
      double2 a[U][RW], x[U][K];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int r = 0; r < RW; ++r)
          a[u][r] = __ldg(reinterpret_cast<const double2*>(arow[r] + c + 64 * u));
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < K; ++j)
          x[u][j] = __ldg(reinterpret_cast<const double2*>(X + j * ldx + c + 64 * u));
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int r = 0; r < RW; ++r)
#pragma unroll
          for (int j = 0; j < K; ++j) {
            acc[r][j] = fma(a[u][r].x, x[u][j].x, acc[r][j]);
            acc[r][j] = fma(a[u][r].y, x[u][j].y, acc[r][j]);
          }
    }
    for (; c + 1 < c1; c += 64) {
      double2 a[RW], x[K];
#pragma unroll
      for (int r = 0; r < RW; ++r) a[r] = __ldg(reinterpret_cast<const double2*>(arow[r] + c));
#pragma unroll
      for (int j = 0; j < K; ++j) x[j] = __ldg(reinterpret_cast<const double2*>(X + j * ldx + c));
#pragma unroll
      for (int r = 0; r < RW; ++r)
#pragma unroll
        for (int j = 0; j < K; ++j) {
          acc[r][j] = fma(a[r].x, x[j].x, acc[r][j]);
          acc[r][j] = fma(a[r].y, x[j].y, acc[r][j]);
        }
    }
    // odd tail element of this column range
    if (((c1 - c0) & 1) && lane == 0) {
      const int64_t ct = c1 - 1;
#pragma unroll
      for (int r = 0; r < RW; ++r)
#pragma unroll
        for (int j = 0; j < K; ++j) acc[r][j] = fma(arow[r][ct], X[j * ldx + ct], acc[r][j]);
    }
  } else {
    for (int64_t c = c0 + lane; c < c1; c += 32) {
      double x[K];
#pragma unroll
      for (int j = 0; j < K; ++j) x[j] = __ldg(X + j * ldx + c);
#pragma unroll
      for (int r = 0; r < RW; ++r) {
        const double a = __ldg(arow[r] + c);
#pragma unroll
        for (int j = 0; j < K; ++j) acc[r][j] = fma(a, x[j], acc[r][j]);
      }
    }
  }

#pragma unroll
  for (int r = 0; r < RW; ++r)
#pragma unroll
    for (int j = 0; j < K; ++j) acc[r][j] = warp_sum(acc[r][j]);

#pragma unroll
  for (int r = 0; r < RW; ++r)
#pragma unroll
    for (int j = 0; j < K; ++j) {
      if (lane == r * K + j && r0 + r < rows) {
        if (splits == 1) {
          double v = acc[r][j];
          if (dscale) v *= dscale[r0 + r];
          Y[j * ldy + r0 + r] = v;
        } else {
          Y[((int64_t)s * K + j) * rows + r0 + r] = acc[r][j];
        }
      }
    }
}

// Y[j*ldy + i] = (sum_s P[(s*K + j)*rows + i]) * (dscale ? dscale[i] : 1)
__global__ void gemv_n_reduce(const double* __restrict__ P, int64_t rows, int K, int splits,
                              double* __restrict__ Y, int64_t ldy,
                              const double* __restrict__ dscale, const double* __restrict__ pred) {
  if (pred && *pred != 0.0) return;
  const int64_t total = rows * K;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(t / rows);
    const int64_t i = t - (int64_t)j * rows;
    double v = 0.0;
    for (int s = 0; s < splits; ++s) v += P[((int64_t)s * K + j) * rows + i];
    if (dscale) v *= dscale[i];
    Y[j * ldy + i] = v;
  }
}

static void gemv_n_plan(int64_t rows, int64_t n, int rw, int& splits, int64_t& chunk) {
  const int64_t ngroups = cdiv(rows, rw);
  const int64_t target_warps = (int64_t)kNumSMs * 16;
  int64_t sp = ngroups >= target_warps ? 1 : cdiv(target_warps, ngroups);
  // keep at least 512 columns per split
  sp = tmax<int64_t>(1, tmin<int64_t>(sp, n / 512));
  chunk = cdiv(cdiv(n, sp), 64) * 64;
  sp = cdiv(n, chunk);
  splits = (int)sp;
}

// register blocking per number of right-hand sides: rows per warp (RW) and
// 128-bit loads in flight per row (U); overridable for tuning (NYS_GEMV_VARIANT)
static int gemv_variant(int K) {
  static const int forced = dev_env("NYS_GEMV_VARIANT") ? atoi(dev_env("NYS_GEMV_VARIANT")) : -1;
  if (forced >= 0) return forced;
  // measured on B200 (tools/micro.py): k<=2 one row per warp with 4 loads in
  // flight per lane; k=3 two rows x 2 loads; k=4 two rows x 1 load
  return K <= 2 ? 4 : (K == 3 ? 2 : 3);
}

template <int K, int RW, int U>
static int gemv_n_launch_v(const double* A, int64_t rows, int64_t n, int64_t lda, const double* X,
                           int64_t ldx, double* Y, int64_t ldy, const double* dscale, double* ws,
                           size_t ws_bytes, cudaStream_t st, const double* pred) {
  int splits;
  int64_t chunk;
  gemv_n_plan(rows, n, RW, splits, chunk);
  if (splits > 1 && ws_bytes < (size_t)splits * K * rows * sizeof(double)) {
    splits = 1;
    chunk = n;
  }
  const bool vec = ((lda & 1) == 0) && ((ldx & 1) == 0) &&
                   ((reinterpret_cast<uintptr_t>(A) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
  const int64_t warps = cdiv(rows, RW) * splits;
  const int64_t blocks = cdiv(warps * 32, kGemvThreads);
  double* out = splits == 1 ? Y : ws;
  if (vec)
    gemv_n_kernel<K, RW, U, true><<<(unsigned)blocks, kGemvThreads, 0, st>>>(
        A, rows, n, lda, X, ldx, out, ldy, dscale, splits, chunk, pred);
  else
    gemv_n_kernel<K, RW, 1, false><<<(unsigned)blocks, kGemvThreads, 0, st>>>(
        A, rows, n, lda, X, ldx, out, ldy, dscale, splits, chunk, pred);
  NYS_CHECK_LAUNCH();
  if (splits > 1) {
    const int64_t total = rows * K;
    const int64_t rb = tmin<int64_t>(cdiv(total, 256), kNumSMs * 8);
    gemv_n_reduce<<<(unsigned)rb, 256, 0, st>>>(ws, rows, K, splits, Y, ldy, dscale, pred);
    NYS_CHECK_LAUNCH();
  }
  return NYS_OK;
}

template <int K>
static int gemv_n_launch(const double* A, int64_t rows, int64_t n, int64_t lda, const double* X,
                         int64_t ldx, double* Y, int64_t ldy, const double* dscale, double* ws,
                         size_t ws_bytes, cudaStream_t st, const double* pred) {
  switch (gemv_variant(K)) {
    case 0: return gemv_n_launch_v<K, 4, 2>(A, rows, n, lda, X, ldx, Y, ldy, dscale, ws, ws_bytes, st, pred);
    case 1: return gemv_n_launch_v<K, 4, 1>(A, rows, n, lda, X, ldx, Y, ldy, dscale, ws, ws_bytes, st, pred);
    case 2: return gemv_n_launch_v<K, 2, 2>(A, rows, n, lda, X, ldx, Y, ldy, dscale, ws, ws_bytes, st, pred);
    case 3: return gemv_n_launch_v<K, 2, 1>(A, rows, n, lda, X, ldx, Y, ldy, dscale, ws, ws_bytes, st, pred);
    default: return gemv_n_launch_v<K, 1, 4>(A, rows, n, lda, X, ldx, Y, ldy, dscale, ws, ws_bytes, st, pred);
  }
}

int gemv_n(const double* A, int64_t rows, int64_t n, int64_t lda, const double* X, int64_t ldx,
           int k, double* Y, int64_t ldy, const double* dscale, void* ws, size_t ws_bytes,
           cudaStream_t st, const double* pred = nullptr) {
  double* w = reinterpret_cast<double*>(ws);
  switch (k) {
    case 1: return gemv_n_launch<1>(A, rows, n, lda, X, ldx, Y, ldy, dscale, w, ws_bytes, st, pred);
    case 2: return gemv_n_launch<2>(A, rows, n, lda, X, ldx, Y, ldy, dscale, w, ws_bytes, st, pred);
    case 3: return gemv_n_launch<3>(A, rows, n, lda, X, ldx, Y, ldy, dscale, w, ws_bytes, st, pred);
    case 4: return gemv_n_launch<4>(A, rows, n, lda, X, ldx, Y, ldy, dscale, w, ws_bytes, st, pred);
    default: return NYS_ERR_ARG;
  }
}

size_t gemv_n_ws(int64_t rows, int64_t n, int k) {
  int splits;
  int64_t chunk;
  gemv_n_plan(rows, n, 4, splits, chunk);  // RW = 4 needs the most splits
  return splits > 1 ? (size_t)splits * k * rows * sizeof(double) : 0;
}

// ------------------------------------------------------------------ K2 ----
constexpr int kGemvTThreads = 256;
constexpr int kGemvTTile = 256;  // rows of T staged per smem tile
constexpr int kGemvTUnroll = 8;

template <int K, bool VEC>
__global__ void __launch_bounds__(kGemvTThreads)
gemv_t_kernel(const double* __restrict__ A, int64_t rows, int64_t n, int64_t lda,
              const double* __restrict__ T, int64_t ldt, double* __restrict__ out, int64_t ldo,
              int64_t rows_per_split, int direct, const double* __restrict__ pred,
              const double* __restrict__ order = nullptr) {
  pdl_begin();  // chain kernel (common.cuh)
  if (pred && *pred != 0.0) return;
  __shared__ double tsh[K][kGemvTTile];
  // splits in descending row order when the previous pass over A ended at the
  // top (L2 reuse; split s always writes partial s)
  const int64_t by = (order && *order != 0.0) ? (int64_t)gridDim.y - 1 - blockIdx.y : (int64_t)blockIdx.y;
  constexpr int CPT = VEC ? 2 : 1;  // columns per thread
  const int64_t c = ((int64_t)blockIdx.x * kGemvTThreads + threadIdx.x) * CPT;
  const int64_t i0 = by * rows_per_split;
  const int64_t i1 = min(rows, i0 + rows_per_split);
  double acc[K][CPT];
#pragma unroll
  for (int j = 0; j < K; ++j)
#pragma unroll
    for (int q = 0; q < CPT; ++q) acc[j][q] = 0.0;

  for (int64_t ib = i0; ib < i1; ib += kGemvTTile) {
    const int cnt = (int)tmin<int64_t>(kGemvTTile, i1 - ib);
    __syncthreads();
    for (int t = threadIdx.x; t < K * kGemvTTile; t += kGemvTThreads) {
      const int j = t / kGemvTTile, ii = t - j * kGemvTTile;
      tsh[j][ii] = ii < cnt ? T[j * ldt + ib + ii] : 0.0;
    }
    __syncthreads();
    if (VEC && c + 1 < n) {
      const double* ap = A + ib * lda + c;
      int t = 0;
      for (; t + kGemvTUnroll <= cnt; t += kGemvTUnroll) {
        double2 a[kGemvTUnroll];
#pragma unroll
        for (int u = 0; u < kGemvTUnroll; ++u)
          a[u] = __ldg(reinterpret_cast<const double2*>(ap + (int64_t)(t + u) * lda));
#pragma unroll
        for (int u = 0; u < kGemvTUnroll; ++u)
#pragma unroll
          for (int j = 0; j < K; ++j) {
            const double tv = tsh[j][t + u];
            acc[j][0] = fma(a[u].x, tv, acc[j][0]);
            acc[j][CPT - 1] = fma(a[u].y, tv, acc[j][CPT - 1]);
          }
      }
      for (; t < cnt; ++t) {
        const double2 a = __ldg(reinterpret_cast<const double2*>(ap + (int64_t)t * lda));
#pragma unroll
        for (int j = 0; j < K; ++j) {
          const double tv = tsh[j][t];
          acc[j][0] = fma(a.x, tv, acc[j][0]);
          acc[j][CPT - 1] = fma(a.y, tv, acc[j][CPT - 1]);
        }
      }
    } else if (c < n) {
      // scalar path: misaligned data or the odd last column
      const double* ap = A + ib * lda + c;
      for (int t = 0; t < cnt; ++t) {
        const double a = __ldg(ap + (int64_t)t * lda);
#pragma unroll
        for (int j = 0; j < K; ++j) acc[j][0] = fma(a, tsh[j][t], acc[j][0]);
      }
    }
  }
  if (c >= n) return;
  const bool two = VEC && (c + 1 < n);
  double* o = direct ? out : out + by * K * ldo;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    if (two) {
      *reinterpret_cast<double2*>(o + j * ldo + c) = make_double2(acc[j][0], acc[j][CPT - 1]);
    } else {
      o[j * ldo + c] = acc[j][0];
    }
  }
}

// Y[j*ldy + c] = sum_s P[(s*K + j)*n + c]  (fixed order);
// optional epilogue for K = 1: Y += shift * v, dot = v.Y  (last-block reduction)
__global__ void gemv_t_reduce(const double* __restrict__ P, int64_t n, int K, int splits,
                              double* __restrict__ Y, int64_t ldy, const double* __restrict__ v,
                              double shift, double* __restrict__ dot, double* __restrict__ part,
                              unsigned int* counter, const double* __restrict__ pred) {
  if (pred && *pred != 0.0) return;
  // 256 threads = 32 consecutive outputs x 8 split-chunks (split s goes to chunk
  // s % 8); chunk sums are combined in a fixed order -> deterministic
  __shared__ double sh[32];
  __shared__ double cs[8][33];
  double d[1] = {0.0};
  const int cx = threadIdx.x & 31, q = threadIdx.x >> 5;
  const int64_t total = n * K;
  for (int64_t base = (int64_t)blockIdx.x * 32; base < total; base += (int64_t)gridDim.x * 32) {
    const int64_t t = base + cx;
    int j = 0;
    int64_t c = 0;
    double acc = 0.0;
    if (t < total) {
      j = (int)(t / n);
      c = t - (int64_t)j * n;
      for (int s = q; s < splits; s += 8) acc += P[((int64_t)s * K + j) * n + c];
    }
    cs[q][cx] = acc;
    __syncthreads();
    if (q == 0 && t < total) {
      double a = cs[0][cx];
#pragma unroll
      for (int qq = 1; qq < 8; ++qq) a += cs[qq][cx];
      if (v) {
        a += shift * v[c];
        if (dot) d[0] = fma(v[c], a, d[0]);
      }
      Y[j * ldy + c] = a;
    }
    __syncthreads();
  }
  if (!dot) return;
  block_sum<1>(d, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = d[0];
  if (last_block(counter)) {
    const double tot = block_sum_partials(part, gridDim.x, 1, sh);
    if (threadIdx.x == 0) *dot = tot;
  }
}

static void gemv_t_plan(int64_t rows, int64_t n, bool vec, int& splits, int64_t& rps) {
  const int64_t strips = cdiv(n, (int64_t)kGemvTThreads * (vec ? 2 : 1));
  static const int per_sm = dev_env("NYS_GEMVT_PER_SM") ? atoi(dev_env("NYS_GEMVT_PER_SM")) : 3;  // measured: 3 beats 2, 4, 5, 6 (config 2, +1%)
  const int64_t target = (int64_t)kNumSMs * per_sm;
  int64_t sp = strips >= target ? 1 : cdiv(target, strips);
  sp = tmax<int64_t>(1, tmin<int64_t>(sp, cdiv(rows, 64)));
  rps = cdiv(cdiv(rows, sp), kGemvTUnroll) * kGemvTUnroll;
  splits = (int)cdiv(rows, rps);
}

// reduction workspace layout (doubles): [0, kRedPartials) partials, then the ticket
constexpr int kRedPartials = 4096;
constexpr size_t kRedBytes = (kRedPartials * 16 + 64) * sizeof(double);

inline double* red_part(void* ws) { return reinterpret_cast<double*>(ws); }
inline unsigned int* red_counter(void* ws) {
  return reinterpret_cast<unsigned int*>(reinterpret_cast<double*>(ws) + kRedPartials * 16);
}

template <int K>
static int gemv_t_launch(const double* A, int64_t rows, int64_t n, int64_t lda, const double* T,
                         int64_t ldt, double* Y, int64_t ldy, const double* v, double shift,
                         double* dot, void* ws, size_t ws_bytes, cudaStream_t st,
                         const double* pred) {
  const bool vec = ((lda & 1) == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0) &&
                   ((ldy & 1) == 0) && ((reinterpret_cast<uintptr_t>(Y) & 15) == 0);
  int splits;
  int64_t rps;
  gemv_t_plan(rows, n, vec, splits, rps);
  const bool epi = (v != nullptr);
  // the split partials live after the reduction scratch
  const size_t need = kRedBytes + (size_t)splits * K * n * sizeof(double);
  if (ws_bytes < need) {
    if (ws_bytes < kRedBytes + (size_t)K * n * sizeof(double)) return NYS_ERR_WORKSPACE;
    splits = 1;
    rps = rows;
  }
  double* P = reinterpret_cast<double*>(reinterpret_cast<char*>(ws) + kRedBytes);
  const bool direct = (splits == 1) && !epi;
  const int64_t strips = cdiv(n, (int64_t)kGemvTThreads * (vec ? 2 : 1));
  dim3 grid((unsigned)strips, (unsigned)splits);
  if (vec)
    gemv_t_kernel<K, true><<<grid, kGemvTThreads, 0, st>>>(A, rows, n, lda, T, ldt,
                                                           direct ? Y : P, direct ? ldy : n,
                                                           rps, direct ? 1 : 0, pred);
  else
    gemv_t_kernel<K, false><<<grid, kGemvTThreads, 0, st>>>(A, rows, n, lda, T, ldt,
                                                            direct ? Y : P, direct ? ldy : n,
                                                            rps, direct ? 1 : 0, pred);
  NYS_CHECK_LAUNCH();
  if (!direct) {
    const int64_t rb = tmin<int64_t>(cdiv(n * K, 32), kRedPartials);
    gemv_t_reduce<<<(unsigned)rb, 256, 0, st>>>(P, n, K, splits, Y, ldy, v, shift, dot,
                                                red_part(ws), red_counter(ws), pred);
    NYS_CHECK_LAUNCH();
  }
  return NYS_OK;
}

// The split partials of Y = A^T T only (no reduction): P[(s K + j) n + c],
// s < *splits.  For consumers that fuse the fixed-order split sum into their
// own epilogue (nys_admm_tail_f64).
template <int K>
static int gemv_t_partials_k(const double* A, int64_t rows, int64_t n, int64_t lda, const double* T,
                             int64_t ldt, void* ws, size_t ws_bytes, cudaStream_t st, const double* pred,
                             double** Pout, int* splits_out, const double* order) {
  const bool vec = ((lda & 1) == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0) && ((n & 1) == 0);
  int splits;
  int64_t rps;
  gemv_t_plan(rows, n, vec, splits, rps);
  if (ws_bytes < kRedBytes + (size_t)splits * K * n * sizeof(double)) return NYS_ERR_WORKSPACE;
  double* P = reinterpret_cast<double*>(reinterpret_cast<char*>(ws) + kRedBytes);
  const int64_t strips = cdiv(n, (int64_t)kGemvTThreads * (vec ? 2 : 1));
  dim3 grid((unsigned)strips, (unsigned)splits);
  const int64_t ldP = n;
  const int64_t direct = 0;
  if (vec)
    launch_chain(gemv_t_kernel<K, true>, grid, dim3(kGemvTThreads), 0, st, false, A, rows, n, lda, T, ldt, P, ldP,
                 rps, (int)direct, pred, order);
  else
    launch_chain(gemv_t_kernel<K, false>, grid, dim3(kGemvTThreads), 0, st, false, A, rows, n, lda, T, ldt, P, ldP,
                 rps, (int)direct, pred, order);
  NYS_CHECK_LAUNCH();
  *Pout = P;
  *splits_out = splits;
  return NYS_OK;
}

int gemv_t_partials(const double* A, int64_t rows, int64_t n, int64_t lda, const double* T, int64_t ldt, int k,
                    void* ws, size_t ws_bytes, cudaStream_t st, const double* pred, double** P, int* splits,
                    const double* order) {
  switch (k) {
    case 2: return gemv_t_partials_k<2>(A, rows, n, lda, T, ldt, ws, ws_bytes, st, pred, P, splits, order);
    case 3: return gemv_t_partials_k<3>(A, rows, n, lda, T, ldt, ws, ws_bytes, st, pred, P, splits, order);
    default: return NYS_ERR_ARG;
  }
}

int gemv_t(const double* A, int64_t rows, int64_t n, int64_t lda, const double* T, int64_t ldt,
           int k, double* Y, int64_t ldy, const double* v, double shift, double* dot, void* ws,
           size_t ws_bytes, cudaStream_t st, const double* pred = nullptr) {
  switch (k) {
    case 1: return gemv_t_launch<1>(A, rows, n, lda, T, ldt, Y, ldy, v, shift, dot, ws, ws_bytes, st, pred);
    case 2: return gemv_t_launch<2>(A, rows, n, lda, T, ldt, Y, ldy, v, shift, dot, ws, ws_bytes, st, pred);
    case 3: return gemv_t_launch<3>(A, rows, n, lda, T, ldt, Y, ldy, v, shift, dot, ws, ws_bytes, st, pred);
    case 4: return gemv_t_launch<4>(A, rows, n, lda, T, ldt, Y, ldy, v, shift, dot, ws, ws_bytes, st, pred);
    default: return NYS_ERR_ARG;
  }
}

size_t gemv_t_ws(int64_t rows, int64_t n, int k) {
  int splits;
  int64_t rps;
  gemv_t_plan(rows, n, true, splits, rps);
  int s2;
  gemv_t_plan(rows, n, false, s2, rps);
  splits = max(splits, s2);
  return kRedBytes + (size_t)splits * k * n * sizeof(double);
}

// --------------------------------------------------------- small vectors ----
__global__ void shift_dot_kernel(int64_t n, const double* __restrict__ v, double shift,
                                 double* __restrict__ y, double* __restrict__ dot,
                                 double* __restrict__ part, unsigned int* counter,
                                 const double* __restrict__ pred) {
  if (pred && *pred != 0.0) return;
  __shared__ double sh[32];
  double d[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double yi = y[i];
    if (shift != 0.0) {
      yi += shift * v[i];
      y[i] = yi;
    }
    d[0] = fma(v[i], yi, d[0]);
  }
  if (!dot) return;
  block_sum<1>(d, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = d[0];
  if (last_block(counter)) {
    const double tot = block_sum_partials(part, gridDim.x, 1, sh);
    if (threadIdx.x == 0) *dot = tot;
  }
}

// y += shift v and dot = v.y, predicated (sharded operator: after the all-reduce)
int shift_dot_pred(int64_t n, const double* v, double shift, double* y, double* dot, void* ws, cudaStream_t st,
                   const double* pred) {
  const int64_t blocks = tmin<int64_t>(cdiv(n, 256), kNumSMs * 4);
  shift_dot_kernel<<<(unsigned)blocks, 256, 0, st>>>(n, v, shift, y, dot, red_part(ws), red_counter(ws), pred);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

int shift_dot(int64_t n, const double* v, double shift, double* y, double* dot, void* ws,
              cudaStream_t st) {
  if (n <= 0) return NYS_ERR_ARG;
  const int64_t blocks = tmin<int64_t>(cdiv(n, 256), kNumSMs * 4);
  shift_dot_kernel<<<(unsigned)blocks, 256, 0, st>>>(n, v, shift, y, dot, red_part(ws),
                                                     red_counter(ws), nullptr);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

struct HvpPlan {
  int C, W, K, S, nclusters;
  size_t smem;
  bool ok;
  int P;
};
HvpPlan hvp_plan(int64_t rows, int64_t n, int64_t lda, const double* A, const double* v);
int hvp_fused(const HvpPlan& p, const double* A, int64_t rows, int64_t n, int64_t lda, const double* d,
              const double* v, double* ypart, cudaStream_t st, const double* pred);
int hvp_row(const HvpPlan& p, const double* A, int64_t rows, int64_t n, int64_t lda, const double* d,
            const double* v, double* ypart, double* y, double shift, double* dot, double* part,
            unsigned int* counter, cudaStream_t st, const double* pred);
struct StripPlan {
  int W, K, WPR, S, L, nctas;
  size_t smem;
  bool ok;
};
size_t hvp_strip_ws();

StripPlan hvp_strip_plan(int64_t rows, int64_t n, int64_t lda, const double* A, const double* v);
int hvp_strip(const StripPlan& p, const double* A, int64_t rows, int64_t n, int64_t lda, const double* d,
              const double* v, double* y, double shift, double* dot, void* ws, double* part,
              unsigned int* counter, cudaStream_t st, const double* pred);

size_t hvp_ws(int64_t rows, int64_t n) {
  // two-pass: t = d o (A v) (rows doubles) + the K1 split partials + the K2 workspace
  const size_t two = cdiv(rows, 2) * 2 * sizeof(double) + gemv_n_ws(rows, n, 1) + gemv_t_ws(rows, n, 1);
  // single pass: reduction scratch + one y partial per cluster (<= 148)
  const size_t one = kRedBytes + tmax((size_t)kNumSMs * n * sizeof(double), hvp_strip_ws());
  return tmax(two, one);
}

// y = A^T(d o Av) (+ shift v, pAp = v.y when finish); every launch predicated on *pred == 0
int hvp_apply(const double* A, int64_t rows, int64_t n, int64_t lda, const double* d, const double* v,
              double shift, double* y, double* pAp, int finish, void* ws, size_t ws_bytes, cudaStream_t st,
              const double* pred) {
  if (ws_bytes < hvp_ws(rows, n)) return NYS_ERR_WORKSPACE;
  static const bool two_pass_only = dev_env("NYS_HVP_TWOPASS") != nullptr;
  const HvpPlan plan = hvp_plan(rows, n, lda, A, v);
  if (plan.ok && !two_pass_only) {
    // single pass over A (csrc/hvp.cu), then a fixed-order sum of the cluster partials
    double* P = reinterpret_cast<double*>(reinterpret_cast<char*>(ws) + kRedBytes);
    static const bool legacy = dev_env("NYS_HVP_LEGACY") != nullptr;
    int rc = NYS_ERR_UNSUPPORTED;
    if (plan.C == 1 && !legacy) {
      rc = hvp_row(plan, A, rows, n, lda, d, v, P, y, finish ? shift : 0.0, finish ? pAp : nullptr, red_part(ws),
                   red_counter(ws), st, pred);
      if (rc != NYS_ERR_UNSUPPORTED) return rc;  // else: not co-resident, two passes below
    } else {
      rc = hvp_fused(plan, A, rows, n, lda, d, v, P, st, pred);
      if (rc) return rc;
      const int64_t rb = tmin<int64_t>(cdiv(n, 32), kRedPartials);
      gemv_t_reduce<<<(unsigned)rb, 256, 0, st>>>(P, n, 1, plan.nclusters, y, n, finish ? v : nullptr, shift,
                                                   finish ? pAp : nullptr, red_part(ws), red_counter(ws), pred);
      NYS_CHECK_LAUNCH();
      return NYS_OK;
    }
  }
  // wide rows, first choice: clusters of 16 CTAs split each row's columns and
  // exchange the row totals through distributed shared memory (csrc/hvp_cluster.cu)
  if (!plan.ok && !two_pass_only) {
    HcPlan hp = hvp_cluster_plan(rows, n, lda, A, v);
    if (hp.ok) {
      double* P = reinterpret_cast<double*>(reinterpret_cast<char*>(ws) + kRedBytes);
      int rc = hvp_cluster(hp, A, rows, n, lda, d, v, P, st, pred);
      if (rc == NYS_OK) {
        const int64_t rb = tmin<int64_t>(cdiv(n, 32), kRedPartials);
        gemv_t_reduce<<<(unsigned)rb, 256, 0, st>>>(P, n, 1, hp.nclusters, y, n, finish ? v : nullptr, shift,
                                                     finish ? pAp : nullptr, red_part(ws), red_counter(ws), pred);
        NYS_CHECK_LAUNCH();
        return NYS_OK;
      }
      if (rc != NYS_ERR_UNSUPPORTED) return rc;
    }
  }
  // wide rows: column strips over the whole grid, A still streamed once (csrc/hvp_strip.cu)
  static const bool no_strip = dev_env("NYS_HVP_NOSTRIP") != nullptr;
  if (!plan.ok && !two_pass_only && !no_strip) {
    const StripPlan sp = hvp_strip_plan(rows, n, lda, A, v);
    if (sp.ok) {
      const int rc = hvp_strip(sp, A, rows, n, lda, d, v, y, finish ? shift : 0.0, finish ? pAp : nullptr,
                               reinterpret_cast<char*>(ws) + kRedBytes, red_part(ws), red_counter(ws), st, pred);
      if (rc != NYS_ERR_UNSUPPORTED) return rc;
    }
  }
  char* base = reinterpret_cast<char*>(ws);
  // layout: [K2 ws (reduction scratch first)] [t] [K1 partials]
  const size_t wt = gemv_t_ws(rows, n, 1);
  double* t = reinterpret_cast<double*>(base + wt);
  void* wn = base + wt + cdiv(rows, 2) * 2 * sizeof(double);
  int rc = gemv_n(A, rows, n, lda, v, n, 1, t, rows, d, wn, gemv_n_ws(rows, n, 1), st, pred);
  if (rc) return rc;
  if (finish) return gemv_t(A, rows, n, lda, t, rows, 1, y, n, v, shift, pAp, base, wt, st, pred);
  return gemv_t(A, rows, n, lda, t, rows, 1, y, n, nullptr, 0.0, nullptr, base, wt, st, pred);
}

size_t dense_mv_ws(int64_t n) { return kRedBytes + gemv_n_ws(n, n, 1) + 256; }

// y = P v + shift v, pAp = v.y  (QP operator of admm.py:262-263 with P dense)
int dense_mv_apply(const double* P, int64_t n, int64_t ldp, const double* v, double shift, double* y, double* pAp,
                   void* ws, size_t ws_bytes, cudaStream_t st, const double* pred) {
  if (ws_bytes < dense_mv_ws(n)) return NYS_ERR_WORKSPACE;
  char* base = reinterpret_cast<char*>(ws);
  int rc = gemv_n(P, n, n, ldp, v, n, 1, y, n, nullptr, base + kRedBytes, gemv_n_ws(n, n, 1), st, pred);
  if (rc) return rc;
  const int64_t blocks = tmin<int64_t>(cdiv(n, 256), kNumSMs * 4);
  shift_dot_kernel<<<(unsigned)blocks, 256, 0, st>>>(n, v, shift, y, pAp, red_part(ws), red_counter(ws), pred);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

size_t reduce_ws() { return kRedBytes; }

}  // namespace nys

// ------------------------------------------------------------- C ABI ------
using namespace nys;

extern "C" size_t nys_reduce_workspace(void) { return kRedBytes; }

extern "C" size_t nys_gemv_workspace(int64_t rows, int64_t n, int k) {
  return gemv_n_ws(rows, n, k);
}

extern "C" int nys_gemv_f64(const double* A, int64_t rows, int64_t n, int64_t lda,
                            const double* X, int64_t ldx, int k, double* Y, int64_t ldy,
                            void* ws, size_t ws_bytes, void* stream) {
  if (rows <= 0 || n <= 0 || lda < n || k < 1 || k > 4 || ldx < n || ldy < rows)
    return NYS_ERR_ARG;
  return gemv_n(A, rows, n, lda, X, ldx, k, Y, ldy, nullptr, ws, ws_bytes, as_stream(stream));
}

extern "C" size_t nys_gemvT_workspace(int64_t rows, int64_t n, int k) {
  return gemv_t_ws(rows, n, k);
}

extern "C" int nys_gemvT_f64(const double* A, int64_t rows, int64_t n, int64_t lda,
                             const double* T, int64_t ldt, int k, double* Y, int64_t ldy,
                             void* ws, size_t ws_bytes, void* stream) {
  if (rows <= 0 || n <= 0 || lda < n || k < 1 || k > 4 || ldt < rows || ldy < n)
    return NYS_ERR_ARG;
  return gemv_t(A, rows, n, lda, T, ldt, k, Y, ldy, nullptr, 0.0, nullptr, ws, ws_bytes,
                as_stream(stream));
}

extern "C" size_t nys_hvp_workspace(int64_t rows, int64_t n) { return hvp_ws(rows, n); }

extern "C" int nys_hvp_f64(const double* A, int64_t rows, int64_t n, int64_t lda, const double* d,
                           const double* v, double shift, double* y, double* pAp, int finish,
                           void* ws, size_t ws_bytes, void* stream) {
  if (rows <= 0 || n <= 0 || lda < n) return NYS_ERR_ARG;
  return hvp_apply(A, rows, n, lda, d, v, shift, y, pAp, finish, ws, ws_bytes, as_stream(stream), nullptr);
}

// which single-pass plan nys_hvp_f64 takes for this shape (16-byte aligned A, v):
// 1 whole rows per CTA (hvp_row_kernel), 2 column-split clusters with a fused
// reduction (hvp_fused_kernel), 3 16-CTA DSMEM clusters (hvp_cluster_kernel),
// 4 grid column strips (hvp_strip_kernel), 0 two passes (gemv_n + gemv_t)
extern "C" int nys_hvp_plan(int64_t rows, int64_t n, int64_t lda) {
  if (rows <= 0 || n <= 0 || lda < n) return -1;
  const double* al = reinterpret_cast<const double*>(uintptr_t(256));
  if (dev_env("NYS_HVP_TWOPASS")) return 0;
  const HvpPlan plan = hvp_plan(rows, n, lda, al, al);
  if (plan.ok) return (plan.C == 1 && !dev_env("NYS_HVP_LEGACY")) ? 1 : 2;
  if (hvp_cluster_plan(rows, n, lda, al, al).ok) return 3;
  if (!dev_env("NYS_HVP_NOSTRIP") && hvp_strip_plan(rows, n, lda, al, al).ok) return 4;
  return 0;
}

extern "C" int nys_shift_dot_f64(int64_t n, const double* v, double shift, double* y,
                                 double* dot, void* ws, void* stream) {
  return shift_dot(n, v, shift, y, dot, ws, as_stream(stream));
}
