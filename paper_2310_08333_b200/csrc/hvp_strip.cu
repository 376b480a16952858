// K3 for wide rows (n > 12800, configs 4 and 5): y = A^T (d o (A v)) + shift v
// with A streamed from HBM ONCE (problems.py:263-264 MLHessian._apply, the CG
// shift of admm.py:262-263).
//
// A whole row no longer fits on chip (800 KB at n = 100000), so the columns
// are split over the whole grid instead of over rows:
//   * CTA c (one per SM, cooperative launch) owns the column strip
//     [c W, c W + W), W = n / 148 (676 columns = 5.4 KB per row at n = 1e5),
//     keeps its v strip and y strip in registers, and streams EVERY row's strip
//     through a shared-memory ring with TMA bulk copies (R rows per stage);
//   * warp-specialised: one producer warp issues the TMA copies into a ring of
//     S stages (full/empty mbarriers); 8 row warps each own one row of a stage
//     (or 1/WPR of one) and never synchronise with each other;
//   * per stage, a row warp forms its partial dot and publishes it to a global
//     exchange slot with the LL protocol (value halves + tag in 8-byte words:
//     no fence, no counter, no CTA barrier);
//   * L stages later (the exchange latency hides behind L stages of dot work
//     and the loads in flight), the warp polls the 148 x WPR entries of its
//     row until their tags match, sums them in a fixed order
//     (identical in every CTA: deterministic), forms t = d_i * (a_i . v) and
//     applies y_strip += t * a_i[strip] from the row still staged in smem;
//   * the strips are disjoint, so y needs no cross-CTA reduction: each CTA adds
//     shift v to its strip, writes it, and p.Ap = v.y is summed from one partial
//     per CTA by the last CTA (fixed order).
// HBM traffic: 8 N n + 8 (2n + N) bytes per HVP (A once, v, y, d); the partial
// exchange (148 x 16 B per row and CTA) stays in L2.
//
// Status (B200): the grid-wide exchange is latency-bound - the ~4 us of rows
// the 148 x 210 KB of shared memory can hold barely covers HBM latency plus
// one L2 round trip of the exchange - so the kernel reaches 3.3 TB/s at
// n = 1e5 (two-pass: 3.2 TB/s) and is used only for strips <= 800 columns.
// Variants measured and not kept: L2-backed axpy (rows re-read from L2 by a
// second warp group, up to 12 stages of lag): 2.7 TB/s; a per-row reducer CTA
// (mode 2 below, 1 polled word per row instead of 148): 2.8 TB/s.
#include <cooperative_groups.h>
#include <stdlib.h>
#include "common.cuh"
#include "tma.cuh"

namespace nys {

constexpr int kStripWarps = 8;                   // row warps
constexpr int kStripThreads = (kStripWarps + 1) * 32;  // + 1 TMA producer warp
constexpr int kStripSlots = 32;        // exchange slots (>= 2 L + 2, see below)
constexpr int kStripMaxLag = 12;
constexpr int kStripSmemBudget = 210 * 1024;

// Slot reuse is safe: a warp publishing stage b has finished reading stage
// b - L - 1 from every CTA, so every writer of its row has published b - L - 1
// and therefore finished reading b - 2 L - 2: a slot written for stage b can
// only still be read for stage b - 2 L - 1 or later.
static_assert(kStripSlots >= 2 * kStripMaxLag + 2, "exchange slots");

// One exchange entry = a double split into two 8-byte words {32 data bits,
// 32-bit tag} (the LL protocol: 8-byte stores are single-copy atomic, so a
// reader that sees the expected tag in a word also sees that word's data; no
// fence, no counter).  The tag encodes the launch epoch and the stage.
__device__ __forceinline__ void ll_store(unsigned long long* p, double v, unsigned tag, int lane) {
  if (lane < 2) {
    const unsigned data = lane == 0 ? (unsigned)__double2loint(v) : (unsigned)__double2hiint(v);
    const unsigned long long w = ((unsigned long long)tag << 32) | data;
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p + lane), "l"(w) : "memory");
  }
}
__device__ __forceinline__ ulonglong2 ll_load(const unsigned long long* p) {
  ulonglong2 r;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(r.x), "=l"(r.y) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ bool ll_ok(ulonglong2 w, unsigned tag) {
  return (unsigned)(w.x >> 32) == tag && (unsigned)(w.y >> 32) == tag;
}
__device__ __forceinline__ double ll_value(ulonglong2 w) {
  return __hiloint2double((int)(unsigned)w.y, (int)(unsigned)w.x);
}

// Row reducer warp: rows i = cta, cta + nctas, ... in increasing order; sums
// the nctas x WPR published partials of row i in a fixed order, scales by d_i
// and publishes t_i (LL word pair) in the row-total slots that follow the
// partial slots.
template <int R, int WPR>
__device__ __forceinline__ void strip_reducer(int64_t rows, const double* __restrict__ d,
                                              unsigned long long* __restrict__ xch, unsigned epoch, int lane,
                                              int cta, int nctas) {
  constexpr int KC = (kNumSMs + 31) / 32;
  const size_t xstride = (size_t)nctas * kStripWarps * 2;
  unsigned long long* T = xch + (size_t)kStripSlots * xstride;
  for (int64_t i = cta; i < rows; i += nctas) {
    const int64_t b = i / R;
    const int ri = (int)(i % R);
    const unsigned tag = epoch * 4194304u + (unsigned)(b & 0x3FFFFF) + 1u;
    const unsigned long long* xs = xch + (size_t)(b % kStripSlots) * xstride + (size_t)ri * WPR * 2;
    const double di = d ? __ldg(d + i) : 1.0;
    ulonglong2 wv[KC][WPR];
#pragma unroll
    for (int k = 0; k < KC; ++k)
#pragma unroll
      for (int p2 = 0; p2 < WPR; ++p2) {
        const int c = lane + 32 * k;
        wv[k][p2] = c < nctas ? ll_load(xs + ((size_t)c * kStripWarps + p2) * 2) : make_ulonglong2(0, 0);
      }
    double tot = 0.0;
#pragma unroll
    for (int k = 0; k < KC; ++k)
#pragma unroll
      for (int p2 = 0; p2 < WPR; ++p2) {
        const int c = lane + 32 * k;
        if (c < nctas) {
          const unsigned long long* e = xs + ((size_t)c * kStripWarps + p2) * 2;
          while (!ll_ok(wv[k][p2], tag)) {
            __nanosleep(64);
            wv[k][p2] = ll_load(e);
          }
          tot += ll_value(wv[k][p2]);
        }
      }
    tot = warp_sum(tot);
    ll_store(T + ((size_t)(b % kStripSlots) * kStripWarps + ri) * 2, di * tot, tag, lane);
  }
}

// Poll the published total of row slot (stage b, row r): one 16-byte word pair.
__device__ __forceinline__ double strip_total(const unsigned long long* xch, int nctas, int64_t b, int r,
                                              unsigned epoch) {
  const unsigned long long* T = xch + (size_t)kStripSlots * nctas * kStripWarps * 2;
  const unsigned tag = epoch * 4194304u + (unsigned)(b & 0x3FFFFF) + 1u;
  const unsigned long long* e = T + ((size_t)(b % kStripSlots) * kStripWarps + r) * 2;
  ulonglong2 tw = ll_load(e);
  while (!ll_ok(tw, tag)) {
    __nanosleep(32);
    tw = ll_load(e);
  }
  return ll_value(tw);
}

template <int K, int WPR, bool RED>
__global__ void __launch_bounds__(kStripThreads + 32, 1)
hvp_strip_kernel(const double* __restrict__ A, int64_t rows, int64_t n, int64_t lda,
                 const double* __restrict__ d, const double* __restrict__ v, int W, int S, int L,
                 double* __restrict__ y, double shift, double* __restrict__ dot,
                 unsigned long long* __restrict__ xch, unsigned int* __restrict__ epoch_p,
                 double* __restrict__ part, unsigned int* counter, const double* __restrict__ pred) {
  if (pred && *pred != 0.0) return;
  constexpr int R = kStripWarps / WPR;  // rows per stage
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw);                       // S x R x W
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)S * R * W);   // S mbarriers
  uint64_t* empty = full + S;                                               // S mbarriers
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nctas = gridDim.x, cta = blockIdx.x;
  const int r = warp / WPR, pp = warp % WPR;  // this warp's row in a stage and column part
  const int64_t c0 = (int64_t)cta * W;
  const int w_here = (int)tmax<int64_t>(0, tmin<int64_t>((int64_t)W, n - c0));
  const unsigned epoch = *(volatile unsigned*)epoch_p;

  if (tid == 0) {
    for (int q = 0; q < S; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], kStripWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int64_t nb = cdiv(rows, R);
  const unsigned seg = (unsigned)w_here * 8u;
  double2 yr[K];
#pragma unroll
  for (int k = 0; k < K; ++k) yr[k] = make_double2(0.0, 0.0);

  if (warp == kStripWarps + 1) {
    if (RED) strip_reducer<R, WPR>(rows, d, xch, epoch, lane, cta, nctas);
  } else if (warp == kStripWarps) {
    // producer: stage b (rows [b R, b R + R) of this strip) into slot b % S once it is empty
    if (lane == 0 && seg > 0) {
      for (int64_t b = 0; b < nb; ++b) {
        const int q = (int)(b % S);
        if (b >= S) mbar_wait(&empty[q], (unsigned)(((b / S) - 1) & 1));
        const int64_t i0 = b * R;
        const int nr = (int)tmin<int64_t>(R, rows - i0);
        mbar_expect_tx(&full[q], seg * (unsigned)nr);
        for (int rr = 0; rr < nr; ++rr)
          tma_load_1d(ring + ((size_t)q * R + rr) * W, A + (i0 + rr) * lda + c0, seg, &full[q]);
      }
    }
  } else {
    // v strip: lane owns double2 index pp*32 + lane + k*32*WPR
    double2 vr[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int j = 2 * (pp * 32 + lane + k * 32 * WPR);
      vr[k] = (j < w_here) ? *reinterpret_cast<const double2*>(v + c0 + j) : make_double2(0.0, 0.0);
    }
    const size_t xstride = (size_t)nctas * kStripWarps * 2;  // u64 words per slot
    for (int64_t it = 0; it < nb + L; ++it) {
      if (it < nb) {
        const int q = (int)(it % S);
        mbar_wait(&full[q], (unsigned)((it / S) & 1));
        double pt = 0.0;
        const double* row = ring + ((size_t)q * R + r) * W;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int j = 2 * (pp * 32 + lane + k * 32 * WPR);
          if (j < w_here) {
            const double2 a = *reinterpret_cast<const double2*>(row + j);
            pt = fma(a.x, vr[k].x, pt);
            pt = fma(a.y, vr[k].y, pt);
          }
        }
        pt = warp_sum(pt);
        const unsigned tag = epoch * 4194304u + (unsigned)(it & 0x3FFFFF) + 1u;
        ll_store(xch + (size_t)(it % kStripSlots) * xstride + ((size_t)cta * kStripWarps + warp) * 2, pt, tag,
                 lane);
      }
      const int64_t jt = it - L;  // stage finished in this iteration
      if (jt < 0) continue;
      const int q = (int)(jt % S);
      const int64_t i = jt * R + r;
      if (i < rows) {
        double tot;
        double di = 1.0;
        if (RED) {
          tot = strip_total(xch, nctas, jt, r, epoch);
        } else {
          // fixed-order total of row i over the CTAs (lane-strided) and parts, then a butterfly
          const unsigned tag = epoch * 4194304u + (unsigned)(jt & 0x3FFFFF) + 1u;
          const unsigned long long* xs = xch + (size_t)(jt % kStripSlots) * xstride + (size_t)r * WPR * 2;
          di = d ? __ldg(d + i) : 1.0;
          // all loads first (one L2 round trip), then re-poll only entries not yet published
          constexpr int KC = (kNumSMs + 31) / 32;
          ulonglong2 wv[KC][WPR];
#pragma unroll
          for (int k = 0; k < KC; ++k)
#pragma unroll
            for (int p2 = 0; p2 < WPR; ++p2) {
              const int c = lane + 32 * k;
              wv[k][p2] = c < nctas ? ll_load(xs + ((size_t)c * kStripWarps + p2) * 2) : make_ulonglong2(0, 0);
            }
          tot = 0.0;
#pragma unroll
          for (int k = 0; k < KC; ++k)
#pragma unroll
            for (int p2 = 0; p2 < WPR; ++p2) {
              const int c = lane + 32 * k;
              if (c < nctas) {
                const unsigned long long* e = xs + ((size_t)c * kStripWarps + p2) * 2;
                while (!ll_ok(wv[k][p2], tag)) wv[k][p2] = ll_load(e);
                tot += ll_value(wv[k][p2]);
              }
            }
          tot = warp_sum(tot);
        }
        const double t = di * tot;
        const double* row = ring + ((size_t)q * R + r) * W;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int j = 2 * (pp * 32 + lane + k * 32 * WPR);
          if (j < w_here) {
            const double2 a = *reinterpret_cast<const double2*>(row + j);
            yr[k].x = fma(t, a.x, yr[k].x);
            yr[k].y = fma(t, a.y, yr[k].y);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[q]);  // this warp is done with stage jt
    }
  }

  // y strip = sum over the R row-warps of each column part (fixed order) + shift v
  __syncthreads();
  double* ys = ring;  // every stage has been consumed: reuse the ring (R x W)
  if (warp < kStripWarps) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int j = 2 * (pp * 32 + lane + k * 32 * WPR);
      if (j < w_here) *reinterpret_cast<double2*>(ys + (size_t)r * W + j) = yr[k];
    }
  }
  __syncthreads();
  double dacc[1] = {0.0};
  for (int j = tid; j < w_here; j += (int)blockDim.x) {
    double a = ys[j];
    for (int rr = 1; rr < R; ++rr) a += ys[(size_t)rr * W + j];
    const double vj = v[c0 + j];
    a = fma(shift, vj, a);
    y[c0 + j] = a;
    dacc[0] = fma(vj, a, dacc[0]);
  }
  __shared__ double dsh[kStripWarps + 2];
  block_sum<1>(dacc, dsh);
  if (tid == 0) part[cta] = dacc[0];
  if (last_block(counter)) {
    // every CTA has read the epoch and finished its exchange: next launch, new tags
    if (tid == 0) *epoch_p = epoch + 1u;
    const double tot = block_sum_partials(part, nctas, 1, dsh);
    if (tid == 0 && dot) *dot = tot;
  }
}

struct StripPlan {
  int W, K, WPR, S, L, nctas;
  size_t smem;
  bool ok;
  int mode;  // 0: every CTA sums the 148 partials of a row; 2: one reducer CTA per row publishes t_i
};

size_t hvp_strip_ws() {
  // partial slots + row-total slots + epoch
  return (size_t)kStripSlots * (kNumSMs + 1) * kStripWarps * 16 + 256;
}

StripPlan hvp_strip_plan(int64_t rows, int64_t n, int64_t lda, const double* A, const double* v) {
  StripPlan p{};
  p.ok = false;
  if ((lda & 1) || (n & 1) || ((uintptr_t)A & 15) || ((uintptr_t)v & 15) || rows < 1) return p;
  p.W = (int)cdiv(cdiv(n, kNumSMs), 2) * 2;
  p.nctas = (int)cdiv(n, p.W);
  // Measured on B200 (tools/hvp_sweep.sh): 4.82 ms vs 5.01 ms for the two-pass
  // path at 20000 x 100000 (W = 676), but 9.4 vs 5.9 ms at 12500 x 200000
  // (W = 1352: fewer rows fit the ring, so less exchange latency is hidden).
  static const bool force = dev_env("NYS_STRIP_FORCE") != nullptr;
  if (p.W > 800 && !force) return p;
  // column parts per row: keep K = double2 per lane <= 16; WPR = 1 gives 8 rows per stage
  static const int forced_wpr = dev_env("NYS_STRIP_WPR") ? atoi(dev_env("NYS_STRIP_WPR")) : 0;
  p.WPR = 1;
  while (p.WPR < kStripWarps && cdiv(p.W / 2, 32 * p.WPR) > 12) p.WPR *= 2;
  if (forced_wpr == 1 || forced_wpr == 2 || forced_wpr == 4 || forced_wpr == 8) p.WPR = tmax(p.WPR, forced_wpr);
  p.K = (int)cdiv(p.W / 2, 32 * p.WPR);
  if (p.K > 16) return p;
  p.K = (p.K + 1) & ~1;  // instantiated for even K
  const int R = kStripWarps / p.WPR;
  const size_t stage = (size_t)R * p.W * 8;
  p.S = (int)tmin<int64_t>(16, (kStripSmemBudget - 512) / stage);
  if (p.S < 3) return p;
  static const int forced_lag = dev_env("NYS_STRIP_LAG") ? atoi(dev_env("NYS_STRIP_LAG")) : 0;
  p.L = forced_lag > 0 ? forced_lag : 2;  // measured best on B200 (S = 4 stages of 43 KB at n = 1e5)
  p.L = tmin(p.L, tmin(kStripMaxLag, p.S - 1));
  static const int forced_mode = dev_env("NYS_STRIP_MODE") ? atoi(dev_env("NYS_STRIP_MODE")) : 0;
  p.mode = forced_mode == 2 ? 2 : 0;
  p.smem = (size_t)p.S * stage + (size_t)p.S * 16;
  if ((size_t)kStripWarps * p.W * 8 > (size_t)p.S * stage) return p;  // final y reduction reuses the ring
  p.ok = true;
  return p;
}

template <int K, int WPR>
static int hvp_strip_launch_k(const StripPlan& p, const double* A, int64_t rows, int64_t n, int64_t lda,
                              const double* d, const double* v, double* y, double shift, double* dot,
                              unsigned long long* xch, unsigned int* epoch, double* part, unsigned int* counter,
                              cudaStream_t st, const double* pred) {
  static bool attr = false;
  auto fn = p.mode == 2 ? hvp_strip_kernel<K, WPR, true> : hvp_strip_kernel<K, WPR, false>;
  if (!attr) {
    cudaFuncSetAttribute(hvp_strip_kernel<K, WPR, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kStripSmemBudget);
    cudaFuncSetAttribute(hvp_strip_kernel<K, WPR, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kStripSmemBudget);
    attr = true;
  }
  const int nthreads = kStripThreads + 32;
  int W = p.W, S = p.S, L = p.L;
  void* args[] = {(void*)&A, (void*)&rows, (void*)&n, (void*)&lda, (void*)&d, (void*)&v, (void*)&W,
                  (void*)&S, (void*)&L, (void*)&y, (void*)&shift, (void*)&dot, (void*)&xch,
                  (void*)&epoch, (void*)&part, (void*)&counter, (void*)&pred};
  if (!coop_fits((const void*)fn, p.nctas, nthreads, p.smem)) return NYS_ERR_UNSUPPORTED;
  const int rc = coop_launch_status(
      cudaLaunchCooperativeKernel((const void*)fn, dim3(p.nctas), dim3(nthreads), args, p.smem, st));
  if (rc) return rc;
  __atomic_fetch_add(&g_launches, 1ull, __ATOMIC_RELAXED);
  return debug_sync_check(__FILE__, __LINE__) ? NYS_ERR_CUDA : NYS_OK;
}

// ws: [exchange slots][epoch] (hvp_strip_ws bytes, zero-initialised once)
int hvp_strip(const StripPlan& p, const double* A, int64_t rows, int64_t n, int64_t lda, const double* d,
              const double* v, double* y, double shift, double* dot, void* ws, double* part,
              unsigned int* counter, cudaStream_t st, const double* pred) {
  unsigned long long* xch = reinterpret_cast<unsigned long long*>(ws);
  unsigned int* epoch = reinterpret_cast<unsigned int*>(xch + (size_t)kStripSlots * (kNumSMs + 1) * kStripWarps * 2);
#define NYS_SK(k, w)                                                                                     \
  if (p.K == k && p.WPR == w)                                                                            \
    return hvp_strip_launch_k<k, w>(p, A, rows, n, lda, d, v, y, shift, dot, xch, epoch, part, counter, \
                                    st, pred);
#define NYS_SW(w) NYS_SK(2, w) NYS_SK(4, w) NYS_SK(6, w) NYS_SK(8, w) NYS_SK(10, w) NYS_SK(12, w) \
  NYS_SK(14, w) NYS_SK(16, w)
  NYS_SW(1) NYS_SW(2) NYS_SW(4) NYS_SW(8)
#undef NYS_SW
#undef NYS_SK
  return NYS_ERR_UNSUPPORTED;
}

}  // namespace nys
