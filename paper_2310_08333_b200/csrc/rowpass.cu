// K1 + K12 fused for the ADMM tail (ML, one GPU): the data pass A{x, z}
// (operators.py:114-115 through problems.py:227-351) and the loss epilogue
// (l'(Ax-b), w = l''(Ax-b), w o Ax, nu = l'(Az-b), the five row sums) in ONE
// kernel, so neither Ax nor Az goes back to HBM.
//
// Warp-specialised row streaming, one CTA per SM:
//   * warp 15 (producer) issues TMA bulk copies of row pieces (W/P doubles)
//     into an S-stage shared-memory ring, gated by per-stage "empty"
//     mbarriers;
//   * warps 0-14 (consumers) hold x and z in registers, wait on the stage's
//     "full" mbarrier, form their partial dots and release the stage at once
//     (one arrive per warp) -- a piece is free as soon as it was read, so the
//     ring keeps ~S-1 pieces of loads in flight;
//   * per row, one named barrier among the consumers; warp (row mod 15) sums
//     the 15 partials in a fixed order and runs the loss epilogue for the
//     row while the others continue with the next row;
//   * the per-CTA row sums are combined in a fixed order by the last CTA.
// Algorithmic traffic: 8 N n + 8 (2 n) + 8 * 5 N bytes.
#include <stdlib.h>
#include "common.cuh"
#include "loss.cuh"
#include "tma.cuh"

namespace nys {

constexpr int kRpConsumers = 15;  // + 1 producer warp = 512 threads (128 registers per thread)
constexpr int kRpThreads = (kRpConsumers + 1) * 32;
constexpr int kRpSmemBudget = 200 * 1024;
constexpr int kRpMaxKP = 12;  // double2 per consumer thread per piece: piece <= 11520 doubles

__device__ __forceinline__ void consumer_barrier() {
  asm volatile("bar.sync 1, %0;" ::"n"(kRpConsumers * 32) : "memory");
}

template <int KP, int P, bool WITH_Z>
__global__ void __launch_bounds__(kRpThreads, 1)
xz_rowpass_kernel(const double* __restrict__ A, int64_t rows, int64_t n, int64_t lda,
                  const double* __restrict__ x, const double* __restrict__ z, const double* __restrict__ b,
                  int loss, int Wp, int S, double* __restrict__ tg, double* __restrict__ w,
                  double* __restrict__ thx, double* __restrict__ tnu, double* __restrict__ rowsums,
                  double* part, unsigned int* counter, const double* __restrict__ pred,
                  const double* __restrict__ order) {
  pdl_begin();  // chain kernel (common.cuh)
  if (pred && *pred != 0.0) return;
  // rows in the order opposite to the previous pass over A (L2 reuse); row
  // results are stored by position, so the order does not change them
  const bool desc = order && *order == 0.0;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw);                   // S x Wp
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)S * Wp);  // S
  uint64_t* empty = full + S;                                           // S
  double* red = reinterpret_cast<double*>(empty + S);                   // 2 x 16 x 2
  double* rsum = red + 64;                                              // 16 x 5
  double* axz = rsum + 80;                                              // 2 x rows of this CTA
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nctas = gridDim.x, cta = blockIdx.x;
  const int64_t nrows_mine = rows > cta ? (rows - cta + nctas - 1) / nctas : 0;
  const int64_t npieces = nrows_mine * P;
  const unsigned pbytes = (unsigned)Wp * 8u;
  if (tid == 0) {
    for (int q = 0; q < S; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], kRpConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 16 * 5) rsum[tid] = 0.0;
  __syncthreads();
  if (warp == kRpConsumers) {
    // ---------------------------------------------------------- producer --
    if (lane == 0) {
      for (int64_t g = 0; g < npieces; ++g) {
        const int q = (int)((unsigned)g % (unsigned)S);
        if (g >= S) mbar_wait(&empty[q], (((unsigned)g / (unsigned)S) - 1u) & 1u);
        const int64_t qq = desc ? nrows_mine - 1 - g / P : g / P;
        const int64_t i = cta + qq * nctas;
        mbar_expect_tx(&full[q], pbytes);
        tma_load_1d(ring + (size_t)q * Wp, A + i * lda + (g % P) * Wp, pbytes, &full[q]);
      }
    }
  } else {
    // --------------------------------------------------------- consumers --
    double2 xr[P][KP], zr[P][KP];
#pragma unroll
    for (int h = 0; h < P; ++h)
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        const int c = 2 * (tid + k * kRpConsumers * 32);
        const int64_t j = (int64_t)h * Wp + c;
        const bool ok = c < Wp && j < n;
        xr[h][k] = ok ? *reinterpret_cast<const double2*>(x + j) : make_double2(0.0, 0.0);
        zr[h][k] = (ok && WITH_Z) ? *reinterpret_cast<const double2*>(z + j) : make_double2(0.0, 0.0);
      }
    for (int64_t it = 0; it < nrows_mine; ++it) {
      const int64_t pos = desc ? nrows_mine - 1 - it : it;  // the row's position in this CTA
      double px = 0.0, pz = 0.0;
#pragma unroll
      for (int h = 0; h < P; ++h) {
        const int64_t g = it * P + h;
        const int q = (int)((unsigned)g % (unsigned)S);
        mbar_wait(&full[q], ((unsigned)g / (unsigned)S) & 1u);
        const double* pc = ring + (size_t)q * Wp;
#pragma unroll
        for (int k = 0; k < KP; ++k) {
          const int c = 2 * (tid + k * kRpConsumers * 32);
          if (c < Wp) {
            const double2 a = *reinterpret_cast<const double2*>(pc + c);
            px = fma(a.x, xr[h][k].x, px);
            px = fma(a.y, xr[h][k].y, px);
            if (WITH_Z) {
              pz = fma(a.x, zr[h][k].x, pz);
              pz = fma(a.y, zr[h][k].y, pz);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[q]);
      }
      px = warp_sum(px);
      if (WITH_Z) pz = warp_sum(pz);
      if (lane == 0) {
        red[((it & 1) * 16 + warp) * 2] = px;
        red[((it & 1) * 16 + warp) * 2 + 1] = pz;
      }
      consumer_barrier();
      if (warp == (int)(it % kRpConsumers)) {  // fixed-order sums of the warp partials
        const double ax = warp_sum(lane < kRpConsumers ? red[((it & 1) * 16 + lane) * 2] : 0.0);
        const double az =
            WITH_Z ? warp_sum(lane < kRpConsumers ? red[((it & 1) * 16 + lane) * 2 + 1] : 0.0) : 0.0;
        if (lane == 0) {
          axz[2 * pos] = ax;
          axz[2 * pos + 1] = az;
        }
      }
    }
    consumer_barrier();
    // loss epilogue of problems.py:227-351 for all of this CTA's rows at once
    // (one thread per row: the transcendental chains run in parallel)
    double rs[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int64_t it = tid; it < nrows_mine; it += kRpConsumers * 32) {
      const int64_t i = cta + it * nctas;
      const double ax = axz[2 * it], az = axz[2 * it + 1];
      const double bi = b[i];
      const double r1 = __dadd_rn(ax, -bi);
      rs[0] += loss_val(loss, r1);
      tg[i] = loss_d1(loss, r1);
      const double wi = loss_d2(loss, r1);
      w[i] = wi;
      thx[i] = __dmul_rn(wi, ax);
      if (WITH_Z) {
        const double r2 = __dadd_rn(az, -bi);
        rs[1] += loss_val(loss, r2);
        const double nu = loss_d1(loss, r2);
        tnu[i] = nu;
        const double cv = loss_conj(loss, nu);
        if (isinf(cv)) rs[3] += 1.0; else rs[2] += cv;
        rs[4] = fma(bi, nu, rs[4]);
      }
    }
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      const double t = warp_sum(rs[q]);
      if (lane == 0) rsum[warp * 5 + q] = t;
    }
  }
  __syncthreads();
  // per-CTA row sums (warps in a fixed order), then the last CTA combines
  if (tid < 5) {
    double t = 0.0;
    for (int q = 0; q < kRpConsumers; ++q) t += rsum[q * 5 + tid];
    part[(int64_t)cta * 5 + tid] = t;
  }
  if (last_block(counter)) {
    if (warp < 5) {
      double t = 0.0;
      for (int c = lane; c < nctas; c += 32) t += part[(int64_t)c * 5 + warp];
      t = warp_sum(t);
      if (lane == 0) rowsums[warp] = t;
    }
  }
}

struct RowpassPlan {
  int P, Wp, S, KP;
  size_t smem;
  bool ok;
};

static RowpassPlan rowpass_plan(int64_t rows, int64_t n, int64_t lda, const double* A, const double* x,
                                const double* z) {
  RowpassPlan p{};
  p.ok = false;
  if ((lda & 1) || (n & 1) || ((uintptr_t)A & 15) || ((uintptr_t)x & 15) || (z && ((uintptr_t)z & 15))) return p;
  if (rows < kNumSMs || cdiv(rows, (int64_t)kNumSMs) > 1024) return p;
  static const bool off = dev_env("NYS_ROWPASS_OFF") != nullptr;
  if (off) return p;
  for (int P = 1; P <= 4; P *= 2) {
    if (n % P) continue;
    const int64_t Wp = n / P;
    if ((Wp & 1) || (Wp * 8) % 16) continue;
    const int KP = (int)cdiv(Wp, (int64_t)2 * kRpConsumers * 32);
    if (KP > kRpMaxKP || P * KP > 12) continue;
    const int64_t S = (kRpSmemBudget - 2048 - 16 * cdiv(rows, (int64_t)kNumSMs)) / (Wp * 8);
    // TMA bulk copies are served one at a time per SM with a fixed cost each
    // (tools/stream_probe.cu: 10/20/40/80 KB pieces -> 3.0/5.7/6.4/6.75 TB/s),
    // so whole rows with two stages beat smaller pieces with more stages
    if (S < 2) continue;
    p.P = P;
    p.Wp = (int)Wp;
    p.S = (int)tmin<int64_t>(S, 32);
    p.KP = KP;
    p.smem = (size_t)p.S * Wp * 8 + (size_t)p.S * 16 + 64 * 8 + 80 * 8 + 2 * cdiv(rows, (int64_t)kNumSMs) * 8 + 256;
    p.ok = true;
    return p;
  }
  return p;
}

template <int KP, int P>
static int rowpass_launch(const RowpassPlan& p, const double* A, int64_t rows, int64_t n, int64_t lda,
                          const double* x, const double* z, const double* b, int loss, double* tg, double* w,
                          double* thx, double* tnu, double* rowsums, double* part, unsigned int* counter,
                          cudaStream_t st, const double* pred, const double* order) {
  const bool wz = z != nullptr;
  auto fn = wz ? xz_rowpass_kernel<KP, P, true> : xz_rowpass_kernel<KP, P, false>;
  static bool attr[2] = {false, false};
  if (!attr[wz]) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kRpSmemBudget);
    attr[wz] = true;
  }
  const unsigned grid = (unsigned)tmin<int64_t>(kNumSMs, rows);
  // launched without the PDL attribute: the persistent solve before it is a
  // cooperative kernel, and letting this pass be scheduled early into it was
  // measured slower
  static const bool pdl = dev_env("NYS_RP_PDL") && dev_env("NYS_RP_PDL")[0] == '1';
  if (pdl)
    launch_chain(fn, dim3(grid), dim3(kRpThreads), p.smem, st, false, A, rows, n, lda, x, z, b, loss, p.Wp, p.S, tg,
                 w, thx, tnu, rowsums, part, counter, pred, order);
  else
    fn<<<grid, kRpThreads, p.smem, st>>>(A, rows, n, lda, x, z, b, loss, p.Wp, p.S, tg, w, thx, tnu, rowsums, part,
                                         counter, pred, order);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

// returns NYS_ERR_UNSUPPORTED when the shape/alignment has no plan (the caller
// then runs the separate GEMV + row-wise kernels)
int xz_rowpass(const double* A, int64_t rows, int64_t n, int64_t lda, const double* x, const double* z,
               const double* b, int loss, double* tg, double* w, double* thx, double* tnu, double* rowsums,
               double* part, unsigned int* counter, cudaStream_t st, const double* pred, const double* order) {
  const RowpassPlan p = rowpass_plan(rows, n, lda, A, x, z);
  if (!p.ok) return NYS_ERR_UNSUPPORTED;
#define NYS_RP(kp, pp)                                                                                        \
  if (p.KP == kp && p.P == pp)                                                                                \
    return rowpass_launch<kp, pp>(p, A, rows, n, lda, x, z, b, loss, tg, w, thx, tnu, rowsums, part, counter, \
                                  st, pred, order);
  NYS_RP(1, 1) NYS_RP(2, 1) NYS_RP(3, 1) NYS_RP(4, 1) NYS_RP(5, 1) NYS_RP(6, 1) NYS_RP(7, 1) NYS_RP(8, 1)
  NYS_RP(9, 1) NYS_RP(10, 1) NYS_RP(11, 1) NYS_RP(12, 1)
  NYS_RP(1, 2) NYS_RP(2, 2) NYS_RP(3, 2) NYS_RP(4, 2) NYS_RP(5, 2) NYS_RP(6, 2) NYS_RP(7, 2) NYS_RP(8, 2)
  NYS_RP(1, 4) NYS_RP(2, 4) NYS_RP(3, 4) NYS_RP(4, 4)
#undef NYS_RP
  return NYS_ERR_UNSUPPORTED;
}

}  // namespace nys
