// K6-K14: preconditioner apply, CG vector updates, the fused ADMM
// elementwise+reduction kernels, loss epilogues and loop-support reductions.
// All are HBM/L2-bound n- or N-length streams; each fuses every elementwise
// op of its reference step with the reductions that step needs, and reduces
// deterministically (per-CTA partials + last-CTA fixed-order sum).
#include <math.h>
#include "common.cuh"
#include "loss.cuh"

namespace nys {

constexpr int kVecThreads = 256;
constexpr int kVecMaxBlocks = kNumSMs * 4;  // 592 partials max per reduction
constexpr int kRedPartials = 4096;          // must match gemv.cu
inline double* red_part(void* ws) { return reinterpret_cast<double*>(ws); }
inline unsigned int* red_counter(void* ws) {
  return reinterpret_cast<unsigned int*>(reinterpret_cast<double*>(ws) + kRedPartials * 16);
}
inline unsigned vec_blocks(int64_t n) {
  return (unsigned)tmax<int64_t>(1, tmin<int64_t>(cdiv(n, kVecThreads), kVecMaxBlocks));
}

// Block sums of NS (8 <= NS <= 32) values per thread, written by warp 0 to
// dst[0..NS).  In a warp, a butterfly reduce-scatter (31 shuffles for up to 32
// values instead of 5 per value) leaves lane l with the warp sum of value l;
// warp 0 then adds the warps' sums in a fixed order.  Deterministic.
template <int NS>
__device__ __forceinline__ void block_sum_to(const double (&s)[NS], double* shT, double* dst) {
  static_assert(NS >= 1 && NS <= 32, "block_sum_to");
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = j < NS ? s[j] : 0.0;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool up = (lane & o) != 0;  // keeps the upper half of the current block of slots
#pragma unroll
    for (int i = 0; i < o; ++i) {
      const double send = up ? v[i] : v[i + o];
      const double keep = up ? v[i + o] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  __syncthreads();
  shT[wid * 32 + lane] = v[0];  // slot 0 of lane l = value l
  __syncthreads();
  if (wid == 0 && lane < NS) {
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t += shT[w * 32 + lane];
    dst[lane] = t;
  }
}

// Reduce NS sums and NM maxes across the grid; the last CTA writes
// out[osum[j]] and out[omax[j]].  part has room for gridDim * (NS+NM).
template <int NS, int NM>
__device__ __forceinline__ bool grid_reduce(double (&s)[(NS > 0) ? NS : 1],
                                            double (&m)[(NM > 0) ? NM : 1], double* part,
                                            unsigned int* counter, double* out,
                                            const int* osum, const int* omax) {
  __shared__ double sh[32 * ((NS > 0 ? NS : 1) + (NM > 0 ? NM : 1))];
  constexpr int NV = NS + NM;
  constexpr bool kScatter = NS >= 8;  // many sums: reduce-scatter instead of one tree per value
  if (kScatter) {
    __shared__ double shT[32 * 32];
    block_sum_to<((NS > 0) ? NS : 1)>(s, shT, part + (size_t)blockIdx.x * NV);
  } else if (NS > 0) {
    block_sum<((NS > 0) ? NS : 1)>(s, sh);
  }
  if (NM > 0) block_max<((NM > 0) ? NM : 1)>(m, sh);
  if (threadIdx.x == 0) {
    if (!kScatter)
#pragma unroll
      for (int j = 0; j < NS; ++j) part[blockIdx.x * NV + j] = s[j];
#pragma unroll
    for (int j = 0; j < NM; ++j) part[blockIdx.x * NV + NS + j] = m[j];
  }
  const bool am_last = last_block(counter);
  if (am_last) {
    // one warp per output (fixed lane-strided order + shuffle tree): the
    // outputs are finished in parallel instead of one block reduction each
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    // (the partials are loaded 8 per lane before they are combined, so one L2
    // round trip covers 256 blocks; the combination order is unchanged)
    constexpr int kB = 8;
    for (int j = wid; j < NV; j += nw) {
      double acc = 0.0;
      for (unsigned b0 = lane; b0 < gridDim.x; b0 += 32 * kB) {
        double v[kB];
#pragma unroll
        for (int t = 0; t < kB; ++t) {
          const unsigned b = b0 + 32 * t;
          v[t] = b < gridDim.x ? part[(size_t)b * NV + j] : 0.0;
        }
#pragma unroll
        for (int t = 0; t < kB; ++t)
          if (b0 + 32 * t < gridDim.x) acc = j < NS ? acc + v[t] : fmax(acc, v[t]);
      }
      acc = j < NS ? warp_sum(acc) : warp_max(acc);
      if (lane == 0) out[j < NS ? osum[j] : omax[j - NS]] = acc;
    }
  }
  return am_last;
}

// ------------------------------------------------------------ dot ---------
__global__ void dot_kernel(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                           double* out, double* part, unsigned int* counter) {
  double s[1] = {0.0}, m[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    s[0] = fma(a[i], b[i], s[0]);
  const int os[1] = {0}, om[1] = {0};
  grid_reduce<1, 0>(s, m, part, counter, out, os, om);
}

// ------------------------------------------------------------ K7 CG -------
__global__ void cg_start_kernel(int64_t n, const double* __restrict__ b,
                                const double* __restrict__ Ax, double* __restrict__ r,
                                double* sc, double* part, unsigned int* counter) {
  double s[2] = {0.0, 0.0}, m[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double bi = b[i];
    const double ri = __dadd_rn(bi, -Ax[i]);
    r[i] = ri;
    s[0] = fma(bi, bi, s[0]);
    s[1] = fma(ri, ri, s[1]);
  }
  const int os[2] = {NYS_CG_B2, NYS_CG_RES2}, om[1] = {0};
  grid_reduce<2, 0>(s, m, part, counter, sc, os, om);
}

__global__ void cg_step_xr_kernel(int64_t n, double* __restrict__ x, double* __restrict__ r,
                                  const double* __restrict__ p, const double* __restrict__ Ap,
                                  int refresh, double* sc, double* part, unsigned int* counter) {
  const double pAp = sc[NYS_CG_PAP];
  const double rz = sc[NYS_CG_RZ];
  const bool bad = !isfinite(pAp) || pAp <= 0.0;
  const double alpha = rz / pAp;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    sc[NYS_CG_ALPHA] = alpha;
    sc[NYS_CG_FLAG] = !isfinite(pAp) ? 1.0 : (pAp <= 0.0 ? 2.0 : 0.0);
  }
  double s[1] = {0.0}, m[1] = {0.0};
  if (!bad) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
      x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
      if (!refresh) {
        const double ri = __dadd_rn(r[i], -__dmul_rn(alpha, Ap[i]));
        r[i] = ri;
        s[0] = fma(ri, ri, s[0]);
      }
    }
  }
  if (refresh) return;
  const int os[1] = {NYS_CG_RES2}, om[1] = {0};
  grid_reduce<1, 0>(s, m, part, counter, sc, os, om);
}

__global__ void cg_dir_kernel(int64_t n, const double* __restrict__ z, double* __restrict__ p,
                              int first, double* sc, unsigned int* counter) {
  const double rz_new = sc[NYS_CG_RZNEW];
  const double beta = first ? 0.0 : rz_new / sc[NYS_CG_RZ];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = first ? z[i] : __dadd_rn(z[i], __dmul_rn(beta, p[i]));
  if (last_block(counter)) {
    if (threadIdx.x == 0) sc[NYS_CG_RZ] = rz_new;
  }
}

// ------------------------------------------------------------ K6 ----------
// pass 1: h_j partial sums of U[i][j] v[i] per CTA; last CTA sums in fixed
// order and writes coef_j = (lam_{r-1}+nu) * (h_j/(lam_j+nu)) - h_j.
constexpr int kPcThreads = 128;
__global__ void __launch_bounds__(kPcThreads)
precond_utv_kernel(const double* __restrict__ U, int64_t n, int r, int64_t ldu,
                   const double* __restrict__ v, int64_t rows_per_block, double* part,
                   unsigned int* counter, const double* __restrict__ lam, double nu,
                   double* __restrict__ coef, const double* __restrict__ pred) {
  if (pred && *pred != 0.0) return;
  // each warp streams whole rows of U (r contiguous doubles, coalesced); lane
  // l accumulates columns l, l+32, ... ; warps are combined in a fixed order
  extern __shared__ double wsum[];  // (kPcThreads/32) x r
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = kPcThreads / 32;
  constexpr int MAXC = 16;  // r <= 512
  double acc[MAXC];
#pragma unroll
  for (int c = 0; c < MAXC; ++c) acc[c] = 0.0;
  const int64_t i0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t i1 = min(n, i0 + rows_per_block);
  int64_t i = i0 + warp;
  // four rows per step: all of their loads are issued before the FMAs, which
  // still accumulate the rows in order (same sums as one row at a time)
  for (; i + 3 * NW < i1; i += 4 * NW) {
    const double v0 = v[i], v1 = v[i + NW], v2 = v[i + 2 * NW], v3 = v[i + 3 * NW];
    const double* u0 = U + i * ldu;
    const double* u1 = u0 + NW * ldu;
    const double* u2 = u1 + NW * ldu;
    const double* u3 = u2 + NW * ldu;
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      const int j = lane + 32 * c;
      if (j < r) {
        const double a0 = u0[j], a1 = u1[j], a2 = u2[j], a3 = u3[j];
        acc[c] = fma(a3, v3, fma(a2, v2, fma(a1, v1, fma(a0, v0, acc[c]))));
      }
    }
  }
  for (; i < i1; i += NW) {
    const double vi = v[i];
    const double* ui = U + i * ldu;
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      const int j = lane + 32 * c;
      if (j < r) acc[c] = fma(ui[j], vi, acc[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < MAXC; ++c) {
    const int j = lane + 32 * c;
    if (j < r) wsum[warp * r + j] = acc[c];
  }
  __syncthreads();
  for (int j = threadIdx.x; j < r; j += kPcThreads) {
    double s = 0.0;
    for (int w = 0; w < NW; ++w) s += wsum[w * r + j];
    part[(int64_t)blockIdx.x * r + j] = s;
  }
  if (!counter) return;  // the column sums run in utv_reduce_kernel (many CTAs)
  if (last_block(counter)) {
    const double lr = lam[r - 1] + nu;
    for (int j = threadIdx.x; j < r; j += kPcThreads) {
      double h0 = 0.0, h1 = 0.0, h2 = 0.0, h3 = 0.0;  // four chains: the loads overlap
      unsigned b = 0;
      for (; b + 4 <= gridDim.x; b += 4) {
        h0 += part[(int64_t)b * r + j];
        h1 += part[(int64_t)(b + 1) * r + j];
        h2 += part[(int64_t)(b + 2) * r + j];
        h3 += part[(int64_t)(b + 3) * r + j];
      }
      for (; b < gridDim.x; ++b) h0 += part[(int64_t)b * r + j];
      const double h = (h0 + h1) + (h2 + h3);
      const double head = __dmul_rn(lr, h / __dadd_rn(lam[j], nu));
      coef[j] = __dadd_rn(head, -h);
    }
  }
}

// the column sums of the U^T v block partials, one CTA per column (the single
// last CTA of precond_utv_kernel walks ~300 partials per column serially:
// 74 us of the 82 at n = 1e5), then the Eq. (11) coefficient of that column
__global__ void __launch_bounds__(256)
utv_reduce_kernel(const double* __restrict__ part, int nparts, int r, const double* __restrict__ lam, double nu,
                  double* __restrict__ coef, const double* __restrict__ pred) {
  if (pred && *pred != 0.0) return;
  __shared__ double sh[8];
  const int j = blockIdx.x;
  double h[1] = {0.0};
  for (int b = threadIdx.x; b < nparts; b += blockDim.x) h[0] += part[(int64_t)b * r + j];
  block_sum<1>(h, sh);
  if (threadIdx.x == 0) {
    const double lr = lam[r - 1] + nu;
    const double head = __dmul_rn(lr, h[0] / __dadd_rn(lam[j], nu));
    coef[j] = __dadd_rn(head, -h[0]);
  }
}

// pass 2: z_i = U_i . coef + v_i  (one warp per row), rz = rdot . z
__global__ void __launch_bounds__(256)
precond_apply_kernel(const double* __restrict__ U, int64_t n, int r, int64_t ldu,
                     const double* __restrict__ coef, const double* __restrict__ v,
                     double* __restrict__ z, const double* __restrict__ rdot, double* rz,
                     double* part, unsigned int* counter, const double* __restrict__ pred) {
  if (pred && *pred != 0.0) return;
  extern __shared__ double csh[];
  for (int j = threadIdx.x; j < r; j += blockDim.x) csh[j] = coef[j];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double s[1] = {0.0}, m[1] = {0.0};
  for (int64_t i = wg; i < n; i += nwarps) {
    const double* ui = U + i * ldu;
    double acc = 0.0;
    for (int j = lane; j < r; j += 32) acc = fma(ui[j], csh[j], acc);
    acc = warp_sum(acc);
    if (lane == 0) {
      const double zi = __dadd_rn(acc, v[i]);
      z[i] = zi;
      if (rdot) s[0] = fma(rdot[i], zi, s[0]);
    }
  }
  if (!rz) return;
  const int os[1] = {0}, om[1] = {0};
  grid_reduce<1, 0>(s, m, part, counter, rz, os, om);
}

__global__ void copy_dot_kernel(int64_t n, const double* __restrict__ v, double* __restrict__ z,
                                const double* __restrict__ rdot, double* rz, double* part,
                                unsigned int* counter, const double* __restrict__ pred) {
  if (pred && *pred != 0.0) return;
  double s[1] = {0.0}, m[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double vi = v[i];
    z[i] = vi;
    if (rdot) s[0] = fma(rdot[i], vi, s[0]);
  }
  if (!rz) return;
  const int os[1] = {0}, om[1] = {0};
  grid_reduce<1, 0>(s, m, part, counter, rz, os, om);
}

// ------------------------------------------------------------ K8/K9 -------
__global__ void admm_rhs_kernel(int64_t n, const double* __restrict__ hxA,
                                const double* __restrict__ gA, const double* __restrict__ q,
                                double lambda2, double sigma, double rho, double shift,
                                const double* __restrict__ x, const double* __restrict__ z,
                                const double* __restrict__ u, double* __restrict__ rhs,
                                double* __restrict__ r, double* sc, double* part,
                                unsigned int* counter) {
  double s[2] = {0.0, 0.0}, m[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double xi = x[i];
    const double l2x = __dmul_rn(lambda2, xi);
    const double hx = __dadd_rn(hxA[i], l2x);                // hess.apply(x)
    double g = __dadd_rn(gA[i], l2x);                        // grad_f(x)
    if (q) g = __dadd_rn(g, q[i]);
    double b = __dadd_rn(__dadd_rn(hx, __dmul_rn(sigma, xi)), -g);
    b = __dadd_rn(b, __dmul_rn(rho, __dadd_rn(z[i], -u[i])));
    const double ri = __dadd_rn(b, -__dadd_rn(hx, __dmul_rn(shift, xi)));
    rhs[i] = b;
    r[i] = ri;
    s[0] = fma(b, b, s[0]);
    s[1] = fma(ri, ri, s[1]);
  }
  const int os[2] = {NYS_CG_B2, NYS_CG_RES2}, om[1] = {0};
  grid_reduce<2, 0>(s, m, part, counter, sc, os, om);
}

// start of an ADMM iteration for a one-iteration-ahead host (nys_admm_head_f64)
__global__ void admm_head_kernel(nys_admm_head h, double* part, unsigned int* counter) {
  if (h.gate && *h.gate == 0.0) return;  // previous iteration unfinished
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (h.gate_next) *h.gate_next = 0.0;
    if (h.tol_out) {
      double tol;
      if (h.tol_fixed > 0.0) {
        tol = h.tol_fixed;
      } else {  // krylov.py:98-112 from the residual norms of the previous iteration
        const double* q = h.prev;
        const double rp = h.norm_kind ? q[1] : sqrt(fmax(q[0], 0.0));
        const double rd = h.norm_kind ? q[3] : sqrt(fmax(q[2], 0.0));
        tol = fmax(fmin(sqrt(rp * rd), 1.0) / h.kpow, 1e-12);
      }
      *h.tol_out = tol;
    }
  }
  const int64_t n = h.n;
  double s[2] = {0.0, 0.0}, m[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double xi = h.x[i], zi = h.z[i], ui = h.u[i];
    if (h.snap) {
      h.snap[i] = xi;
      h.snap[n + i] = zi;
      h.snap[2 * n + i] = ui;
      h.snap[3 * n + i] = h.xbar[i];
      h.snap[4 * n + i] = h.zbar[i];
    }
    const double l2x = __dmul_rn(h.lambda2, xi);
    const double hx = __dadd_rn(h.hxA[i], l2x);
    double g = __dadd_rn(h.gA[i], l2x);
    if (h.q) g = __dadd_rn(g, h.q[i]);
    double b = __dadd_rn(__dadd_rn(hx, __dmul_rn(h.sigma, xi)), -g);
    b = __dadd_rn(b, __dmul_rn(h.rho, __dadd_rn(zi, -ui)));
    const double ri = __dadd_rn(b, -__dadd_rn(hx, __dmul_rn(h.shift, xi)));
    h.rhs[i] = b;
    h.r[i] = ri;
    s[0] = fma(b, b, s[0]);
    s[1] = fma(ri, ri, s[1]);
  }
  const int os[2] = {NYS_CG_B2, NYS_CG_RES2}, om[1] = {0};
  grid_reduce<2, 0>(s, m, part, counter, h.sc, os, om);
}

__device__ __forceinline__ double soft1(double v, double kappa) {
  const double a = fmax(__dadd_rn(fabs(v), -kappa), 0.0);
  return v > 0.0 ? a : (v < 0.0 ? -a : 0.0 * a);
}

__global__ void admm_zu_kernel(int64_t n, const double* __restrict__ x, double* __restrict__ z,
                               double* __restrict__ u, double alpha, int prox_kind, double kappa,
                               const double* __restrict__ lo, const double* __restrict__ hi,
                               double* __restrict__ xbar, double* __restrict__ zbar, int accum,
                               const double* __restrict__ pred = nullptr) {
  if (pred && *pred != 0.0) return;
  const double beta = 1.0 - alpha;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double xi = x[i];
    const double w = __dadd_rn(__dmul_rn(alpha, xi), __dmul_rn(beta, z[i]));
    const double ui = u[i];
    const double v = __dadd_rn(w, ui);
    double zn;
    if (prox_kind == NYS_PROX_SOFT) {
      zn = soft1(v, kappa);
    } else {
      zn = fmin(fmax(v, lo[i]), hi[i]);
    }
    z[i] = zn;
    u[i] = __dadd_rn(__dadd_rn(ui, w), -zn);
    if (accum) {
      xbar[i] = __dadd_rn(xbar[i], xi);
      zbar[i] = __dadd_rn(zbar[i], zn);
    }
  }
}

__global__ void admm_norms_kernel(int64_t n, const double* __restrict__ x,
                                  const double* __restrict__ z, const double* __restrict__ u,
                                  const double* __restrict__ gA, const double* __restrict__ q,
                                  double lambda2, double rho, const double* __restrict__ atnu,
                                  double lambda1, const double* __restrict__ lo,
                                  const double* __restrict__ hi, double* out, double* part,
                                  unsigned int* counter, const double* __restrict__ pred = nullptr) {
  if (pred && *pred != 0.0) return;
  // sums: (x-z)^2, rd^2, x^2, z^2, (rho u)^2, |z|, x.gA, q.x, (|atnu|-l1)_+^2
  // maxes: |x-z|, |rd|, |x|, |z|, |rho u|, |atnu|, box violation (shifted by +inf guard)
  double s[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  double m[7] = {0, 0, 0, 0, 0, 0, 0};
  double viol = -INFINITY;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double xi = x[i], zi = z[i], ui = u[i];
    const double rp = __dadd_rn(xi, -zi);
    double g = __dadd_rn(gA[i], __dmul_rn(lambda2, xi));
    if (q) g = __dadd_rn(g, q[i]);
    const double ru = __dmul_rn(rho, ui);
    const double rd = __dadd_rn(g, ru);
    s[0] = fma(rp, rp, s[0]);
    s[1] = fma(rd, rd, s[1]);
    s[2] = fma(xi, xi, s[2]);
    s[3] = fma(zi, zi, s[3]);
    s[4] = fma(ru, ru, s[4]);
    s[5] += fabs(zi);
    s[6] = fma(xi, gA[i], s[6]);
    if (q) s[7] = fma(q[i], xi, s[7]);
    m[0] = fmax(m[0], fabs(rp));
    m[1] = fmax(m[1], fabs(rd));
    m[2] = fmax(m[2], fabs(xi));
    m[3] = fmax(m[3], fabs(zi));
    m[4] = fmax(m[4], fabs(ru));
    if (atnu) {
      const double a = fabs(atnu[i]);
      m[5] = fmax(m[5], a);
      const double e = fmax(a - lambda1, 0.0);
      s[8] = fma(e, e, s[8]);
    }
    if (lo) viol = fmax(viol, fmax(lo[i] - zi, zi - hi[i]));
  }
  // encode the violation as a nonnegative max: store exp-free offset via +inf guard
  // (values are compared on the host; -inf means "no box")
  m[6] = viol;
  const int os[9] = {0, 2, 4, 6, 8, 10, 11, 12, 14};
  const int om[7] = {1, 3, 5, 7, 9, 13, 15};
  grid_reduce<9, 7>(s, m, part, counter, out, os, om);
}

__global__ void ml_rowwise_kernel(int64_t rows, int loss, const double* __restrict__ Ax,
                                  const double* __restrict__ Az, const double* __restrict__ b,
                                  double* __restrict__ tg, double* __restrict__ w,
                                  double* __restrict__ thx, double* __restrict__ tnu, double* out,
                                  double* part, unsigned int* counter,
                                  const double* __restrict__ pred = nullptr) {
  if (pred && *pred != 0.0) return;
  double s[5] = {0, 0, 0, 0, 0}, m[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double bi = b[i];
    if (Ax) {
      const double ax = Ax[i];
      const double r1 = __dadd_rn(ax, -bi);
      s[0] += loss_val(loss, r1);
      if (tg) tg[i] = loss_d1(loss, r1);
      const double wi = loss_d2(loss, r1);
      if (w) w[i] = wi;
      if (thx) thx[i] = __dmul_rn(wi, ax);
    }
    if (Az) {
      const double r2 = __dadd_rn(Az[i], -bi);
      s[1] += loss_val(loss, r2);
      const double nu = loss_d1(loss, r2);
      if (tnu) tnu[i] = nu;
      const double cv = loss_conj(loss, nu);
      if (isinf(cv)) s[3] += 1.0; else s[2] += cv;
      s[4] = fma(bi, nu, s[4]);
    }
  }
  const int os[5] = {0, 1, 2, 3, 4}, om[1] = {0};
  grid_reduce<5, 0>(s, m, part, counter, out, os, om);
}

__global__ void ml_conj_scaled_kernel(int64_t rows, int loss, const double* __restrict__ nu,
                                      double c, const double* __restrict__ b, double* out,
                                      double* part, unsigned int* counter) {
  double s[3] = {0, 0, 0}, m[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double y = __dmul_rn(nu[i], c);
    const double cv = loss_conj(loss, y);
    if (isinf(cv)) s[1] += 1.0; else s[0] += cv;
    s[2] = fma(b[i], y, s[2]);
  }
  const int os[3] = {0, 1, 2}, om[1] = {0};
  grid_reduce<3, 0>(s, m, part, counter, out, os, om);
}

// the scaled-dual conjugate sums with c = lambda1 / max|atnu| computed on the
// device (problems.py:330-340); a no-op unless max|atnu| > lambda1
__global__ void ml_conj_dev_kernel(int64_t rows, int loss, const double* __restrict__ nu,
                                   const double* __restrict__ denom, double lambda1,
                                   const double* __restrict__ b, double* out, double* part,
                                   unsigned int* counter, const double* __restrict__ pred) {
  pdl_begin();  // chain kernel (common.cuh)
  if (pred && *pred != 0.0) return;
  const double dn = *denom;
  if (!(dn > lambda1)) return;
  const double c = lambda1 / dn;
  double s[3] = {0, 0, 0}, m[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double y = __dmul_rn(nu[i], c);
    const double cv = loss_conj(loss, y);
    if (isinf(cv)) s[1] += 1.0; else s[0] += cv;
    s[2] = fma(b[i], y, s[2]);
  }
  const int os[3] = {0, 1, 2}, om[1] = {0};
  grid_reduce<3, 0>(s, m, part, counter, out, os, om);
}

__global__ void open_gate_kernel(double* gate, const double* __restrict__ pred) {
  pdl_begin();  // chain kernel (common.cuh)
  if (pred && *pred != 0.0) return;
  if (threadIdx.x == 0) *gate = 1.0;
}

// ------------------------------------------------------- K13/K14 ----------
struct SlotList {
  int idx[16];
};

// the host's termination test (admm.py:_terminated/_gap of the B200 engine,
// = admm.py:227-240 and problems.py:335-351 of the reference) on the reduced
// norms `s` (nys_admm_norms_f64 layout) and row sums `rs` (nys_ml_rowwise_f64
// layout), operation for operation (no contraction), so host and device agree
struct StopArgs {
  int on, gap, linf, loss, slot;
  double eps_gap, eps_abs, eps_rel, sqrt_n, l1, l2;
};

__device__ bool device_stop(const StopArgs& a, const double* s, const double* rs) {
  if (a.gap) {
    const double primal =
        __dadd_rn(__dadd_rn(rs[1], __dmul_rn(__dmul_rn(0.5, a.l2), s[6])), __dmul_rn(a.l1, s[10]));
    double conj_sum = rs[2], b_nu = rs[4];
    const double n_inf = rs[3];
    if (a.l2 == 0.0) {
      const double denom = s[13];
      if (denom > a.l1) {
        const double c = a.l1 / denom;
        conj_sum = __dmul_rn(__dmul_rn(conj_sum, c), c);  // square / huber (homogeneous)
        b_nu = __dmul_rn(b_nu, c);
      }
    }
    if (n_inf > 0.0) return false;  // gap = inf
    double dual = __dadd_rn(-conj_sum, -b_nu);
    if (a.l2 > 0.0) dual = __dadd_rn(dual, -(s[14] / __dmul_rn(2.0, a.l2)));
    if (!isfinite(dual)) return false;
    const double num = __dadd_rn(primal, -dual);
    const double den = fmin(primal, fabs(dual));
    double gap;
    if (den <= 1e-16) gap = fabs(num) <= 1e-12 ? 0.0 : INFINITY;
    else gap = num / den;
    return gap <= a.eps_gap;
  }
  double rp, rd, nx, nz, nru;
  if (a.linf) {
    rp = s[1], rd = s[3], nx = s[5], nz = s[7], nru = s[9];
  } else {
    rp = sqrt(fmax(s[0], 0.0)), rd = sqrt(fmax(s[2], 0.0)), nx = sqrt(fmax(s[4], 0.0));
    nz = sqrt(fmax(s[6], 0.0)), nru = sqrt(fmax(s[8], 0.0));
  }
  const double ps = fmax(fmax(nx, nz), 0.0);
  const double tp = __dadd_rn(__dmul_rn(a.sqrt_n, a.eps_abs), __dmul_rn(a.eps_rel, ps));
  const double td = __dadd_rn(__dmul_rn(a.sqrt_n, a.eps_abs), __dmul_rn(a.eps_rel, nru));
  return rp <= tp && rd <= td;
}

__global__ void window_norms_kernel(int64_t n, const double* __restrict__ ring, int64_t ld,
                                    int cur, SlotList others, int nothers, double* out,
                                    double* part, unsigned int* counter,
                                    const double* __restrict__ pred = nullptr) {
  if (pred && *pred != 0.0) return;
  double s[17], m[1] = {0.0};
#pragma unroll
  for (int j = 0; j < 17; ++j) s[j] = 0.0;
  const double* xc = ring + (int64_t)cur * ld;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double xi = xc[i];
    s[0] = fma(xi, xi, s[0]);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (j < nothers) {
        const double d = __dadd_rn(xi, -ring[(int64_t)others.idx[j] * ld + i]);
        s[1 + j] = fma(d, d, s[1 + j]);
      }
    }
  }
  const int os[17] = {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16}, om[1] = {0};
  grid_reduce<17, 0>(s, m, part, counter, out, os, om);
}

// ML iteration epilogue in one pass over column slices (nys_admm_tail_f64):
// the fixed-order sum of the A^T split partials -> AT (K rows: gA, hxA, atnu),
// then, for the same columns, the residual / objective / gap norms of
// admm_norms_kernel and the cycle-guard window norms of window_norms_kernel,
// all reduced in one grid reduction.  Block b owns columns [64 b, 64 b + 64).
constexpr int kEpiCols = 64;
// CTAs of the epilogue (grid-stride over the column tiles, capped) and whether
// their 33 partials each fit the reduction scratch
static inline int64_t epi_blocks(int64_t n) { return tmin<int64_t>(cdiv(n, (int64_t)kEpiCols), 2 * kNumSMs); }
static inline bool epi_fits(int64_t n) { return epi_blocks(n) * 33 <= (int64_t)kRedPartials * 16; }
template <int K>
__global__ void __launch_bounds__(256)
ml_epilogue_kernel(int64_t n, const double* __restrict__ P, int splits, double* __restrict__ AT,
                   const double* __restrict__ x, const double* __restrict__ z, const double* __restrict__ u,
                   double lambda2, double rho, double lambda1, const double* __restrict__ ring, int64_t ld,
                   int cur, SlotList others, int nothers, double* out, int woff, double* part,
                   unsigned int* counter, const double* __restrict__ pred, const double* __restrict__ rb_src,
                   double* rb_dst, int rb_n, double* rb_gate, double rb_tag, StopArgs stop,
                   const double* __restrict__ gb) {
  pdl_begin();  // chain kernel (common.cuh)
  // (rb_dst: this kernel ends the iteration's chain and also does the readback of
  // the iteration's scalar block into mapped host memory: nys_readback_f64 fused)
  if (pred && *pred != 0.0) {
    if (rb_dst && blockIdx.x == 0) {  // a skipped iteration still reports its status
      for (int q = threadIdx.x; q < rb_n; q += blockDim.x) rb_dst[q] = rb_src[q];
      __threadfence_system();
      __syncthreads();
      if (threadIdx.x == 0 && rb_tag != 0.0) *(volatile double*)(rb_dst + rb_n) = rb_tag;  // block complete
    }
    return;
  }
  __shared__ double cs[4][K][kEpiCols];
  const int tid = threadIdx.x, cx = tid & (kEpiCols - 1), ch = tid >> 6;
  double s[9 + 17], m[7];
#pragma unroll
  for (int j = 0; j < 26; ++j) s[j] = 0.0;
#pragma unroll
  for (int j = 0; j < 7; ++j) m[j] = 0.0;
  double viol = -INFINITY;
  // column tiles of kEpiCols, grid-stride (a capped grid keeps the final
  // reduction short for large n: 1563 tiles at n = 1e5)
  const int64_t ntiles = cdiv(n, (int64_t)kEpiCols);
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
  const int64_t c = tile * kEpiCols + cx;
  {
    // splits ch, ch + 4, ... of column c: four independent chains so four
    // groups of loads are in flight per round trip (fixed combination order)
    double acc[4][K];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int j = 0; j < K; ++j) acc[u][j] = 0.0;
    if (c < n) {
      int q = ch;
      // gb (the SQ cluster tail, K = 3): row 0 of the partials is not written
      const int j0 = gb ? 1 : 0;
      for (; q + 12 < splits; q += 16)
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int j = 0; j < K; ++j)
            if (j >= j0) acc[u][j] += P[((int64_t)(q + 4 * u) * K + j) * n + c];
      for (; q < splits; q += 4)
#pragma unroll
        for (int j = 0; j < K; ++j)
          if (j >= j0) acc[0][j] += P[((int64_t)q * K + j) * n + c];
    }
#pragma unroll
    for (int j = 0; j < K; ++j) cs[ch][j][cx] = (acc[0][j] + acc[1][j]) + (acc[2][j] + acc[3][j]);
  }
  __syncthreads();
  if (ch == 0 && c < n) {
    double at[K];
#pragma unroll
    for (int j = 0; j < K; ++j) at[j] = ((cs[0][j][cx] + cs[1][j][cx]) + cs[2][j][cx]) + cs[3][j][cx];
    if (K == 3 && gb) {  // A^T (Ax - b) = A^T (A x) - g_b, A^T (Az - b) = A^T (A z) - g_b
      const double g = gb[c];
      at[0] = at[1] - g;
      at[K - 1] = at[K - 1] - g;
    }
#pragma unroll
    for (int j = 0; j < K; ++j) AT[(int64_t)j * n + c] = at[j];
    // admm_norms_kernel, element c (gA = at[0], atnu = at[2])
    const double xi = x[c], zi = z[c], ui = u[c];
    const double rp = __dadd_rn(xi, -zi);
    const double g = __dadd_rn(at[0], __dmul_rn(lambda2, xi));
    const double ru = __dmul_rn(rho, ui);
    const double rd = __dadd_rn(g, ru);
    s[0] += rp * rp;
    s[1] += rd * rd;
    s[2] += xi * xi;
    s[3] += zi * zi;
    s[4] += ru * ru;
    s[5] += fabs(zi);
    s[6] += xi * at[0];
    m[0] = fmax(m[0], fabs(rp));
    m[1] = fmax(m[1], fabs(rd));
    m[2] = fmax(m[2], fabs(xi));
    m[3] = fmax(m[3], fabs(zi));
    m[4] = fmax(m[4], fabs(ru));
    if (K == 3) {
      const double a = fabs(at[K - 1]);
      m[5] = fmax(m[5], a);
      const double e = fmax(a - lambda1, 0.0);
      s[8] += e * e;
    }
    // window_norms_kernel, element c
    if (nothers > 0) {
      const double xc = ring[(int64_t)cur * ld + c];
      s[9] += xc * xc;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (j < nothers) {
          const double dd = __dadd_rn(xc, -ring[(int64_t)others.idx[j] * ld + c]);
          s[10 + j] += dd * dd;
        }
      }
    }
  }
  __syncthreads();  // cs is rewritten by the next tile
  }
  m[6] = viol;
  const int os[26] = {0, 2, 4, 6, 8, 10, 11, 12, 14, woff, woff + 1, woff + 2, woff + 3, woff + 4, woff + 5,
                      woff + 6, woff + 7, woff + 8, woff + 9, woff + 10, woff + 11, woff + 12, woff + 13,
                      woff + 14, woff + 15, woff + 16};
  const int om[7] = {1, 3, 5, 7, 9, 13, 15};
  const bool last = grid_reduce<26, 7>(s, m, part, counter, out, os, om);
  __shared__ bool s_stop;
  if (last && stop.on) {
    __syncthreads();  // the reduced norms are in `out`; the row sums lead the readback block
    if (threadIdx.x == 0) {
      s_stop = device_stop(stop, out, rb_src);
      out[stop.slot] = s_stop ? 1.0 : 0.0;
    }
    __syncthreads();
  }
  if (last && rb_dst) {
    __syncthreads();  // the reduced norms are in the block
    for (int q = threadIdx.x; q < rb_n; q += blockDim.x) rb_dst[q] = rb_src[q];
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
      // the next iteration may run -- unless the device stop test held
      if (rb_gate && !(stop.on && s_stop)) *rb_gate = 1.0;
      // the host polls this tag instead of waiting on a stream event (an event
      // between this kernel and the next x-update would serialise their launches)
      if (rb_tag != 0.0) *(volatile double*)(rb_dst + rb_n) = rb_tag;
    }
  }
}

__global__ void scale_dual_kernel(int64_t n, double* __restrict__ u, double rho_old,
                                  double rho_new, double* out, double* part,
                                  unsigned int* counter) {
  double s[2] = {0, 0}, m[1] = {0.0};
  const double f = rho_old / rho_new;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double yo = __dmul_rn(rho_old, u[i]);
    const double un = __dmul_rn(u[i], f);
    u[i] = un;
    const double d = __dadd_rn(__dmul_rn(rho_new, un), -yo);
    s[0] = fma(yo, yo, s[0]);
    s[1] = fma(d, d, s[1]);
  }
  const int os[2] = {0, 1}, om[1] = {0};
  grid_reduce<2, 0>(s, m, part, counter, out, os, om);
}

__global__ void qp_infeas_kernel(int64_t n, const double* __restrict__ xa,
                                 const double* __restrict__ xb, const double* __restrict__ ua,
                                 const double* __restrict__ ub, double width,
                                 const double* __restrict__ lo, const double* __restrict__ hi,
                                 const double* __restrict__ q, double* __restrict__ dx,
                                 double* out, double* part, unsigned int* counter,
                                 const double* __restrict__ pred = nullptr) {
  if (pred && *pred != 0.0) return;
  double s[6] = {0, 0, 0, 0, 0, 0}, m[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double d_x = __dadd_rn(xa[i], -xb[i]) / width;
    const double d_u = __dadd_rn(ua[i], -ub[i]) / width;
    dx[i] = d_x;
    s[0] = fma(d_u, d_u, s[0]);
    const double l = lo[i], h = hi[i];
    if (d_u > 0.0) {
      if (isinf(h)) s[2] += 1.0; else s[1] = fma(h, d_u, s[1]);
    } else if (d_u < 0.0) {
      if (isinf(l)) s[2] += 1.0; else s[1] = fma(l, d_u, s[1]);
    }
    s[3] = fma(d_x, d_x, s[3]);
    // projection onto the recession cone of [l, h] (prox.py:113-129)
    const bool lf = isfinite(l), hf = isfinite(h);
    double proj = d_x;
    if (lf && hf) proj = 0.0;
    else if (lf && !hf) proj = fmax(d_x, 0.0);
    else if (!lf && hf) proj = fmin(d_x, 0.0);
    const double e = __dadd_rn(d_x, -proj);
    s[4] = fma(e, e, s[4]);
    if (q) s[5] = fma(q[i], d_x, s[5]);
  }
  const int os[6] = {0, 1, 2, 3, 4, 5}, om[1] = {0};
  grid_reduce<6, 0>(s, m, part, counter, out, os, om);
}

// ring[slot] = x (and uring[slot] = u): window copies, predicated
__global__ void ring_copy_kernel(int64_t n, const double* __restrict__ x, double* __restrict__ dx,
                                 const double* __restrict__ u, double* __restrict__ du,
                                 const double* __restrict__ pred) {
  if (pred && *pred != 0.0) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    dx[i] = x[i];
    if (du) du[i] = u[i];
  }
}

__global__ void dot_pred_kernel(int64_t n, const double* __restrict__ a, const double* __restrict__ b, double* out,
                                double* part, unsigned int* counter, const double* __restrict__ pred) {
  if (pred && *pred != 0.0) return;
  double s[1] = {0.0}, m[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s[0] = fma(a[i], b[i], s[0]);
  const int os[1] = {0}, om[1] = {0};
  grid_reduce<1, 0>(s, m, part, counter, out, os, om);
}

__global__ void axpby_kernel(int64_t n, double a, const double* __restrict__ x, double b,
                             double* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = __dadd_rn(__dmul_rn(a, x[i]), b == 0.0 ? 0.0 : __dmul_rn(b, y[i]));
}

__global__ void soft_kernel(int64_t n, const double* __restrict__ v, double kappa,
                            double* __restrict__ o) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    o[i] = soft1(v[i], kappa);
}

// elementwise loss evaluation (problems.py:35-111): what = 0 value, 1 first
// derivative, 2 second derivative, 3 conjugate (+inf outside its domain)
__global__ void loss_eval_kernel(int loss, int what, int64_t n, const double* __restrict__ w,
                                 double* __restrict__ o) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double x = w[i];
    o[i] = what == 0 ? loss_val(loss, x) : what == 1 ? loss_d1(loss, x) : what == 2 ? loss_d2(loss, x)
                                                                                    : loss_conj(loss, x);
  }
}

__global__ void box_kernel(int64_t n, const double* __restrict__ v, const double* __restrict__ lo,
                           const double* __restrict__ hi, double* __restrict__ o) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    o[i] = fmin(fmax(v[i], lo[i]), hi[i]);
}

__global__ void row_scale_kernel(int64_t rows, int64_t cols, double* __restrict__ X, int64_t ldx,
                                 const double* __restrict__ d) {
  const int64_t total = rows * cols;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / cols, j = t - i * cols;
    X[i * ldx + j] *= d[i];
  }
}

}  // namespace nys

// ------------------------------------------------------------- C ABI ------
using namespace nys;

#define RED_ARGS(ws) red_part(ws), red_counter(ws)

extern "C" int nys_dot_f64(int64_t n, const double* a, const double* b, double* out, void* ws,
                           void* stream) {
  if (n <= 0) return NYS_ERR_ARG;
  dot_kernel<<<vec_blocks(n), kVecThreads, 0, as_stream(stream)>>>(n, a, b, out, RED_ARGS(ws));
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_cg_start_f64(int64_t n, const double* b, const double* Ax0, double* r,
                                double* sc, void* ws, void* stream) {
  if (n <= 0) return NYS_ERR_ARG;
  cg_start_kernel<<<vec_blocks(n), kVecThreads, 0, as_stream(stream)>>>(n, b, Ax0, r, sc,
                                                                        RED_ARGS(ws));
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_cg_step_xr_f64(int64_t n, double* x, double* r, const double* p,
                                  const double* Ap, int refresh, double* sc, void* ws,
                                  void* stream) {
  if (n <= 0) return NYS_ERR_ARG;
  cg_step_xr_kernel<<<vec_blocks(n), kVecThreads, 0, as_stream(stream)>>>(n, x, r, p, Ap, refresh,
                                                                          sc, RED_ARGS(ws));
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_cg_dir_f64(int64_t n, const double* z, double* p, int first, double* sc,
                              void* stream) {
  // cg_dir needs its own ticket; it lives in the CG scalar block's spare slot.
  if (n <= 0) return NYS_ERR_ARG;
  unsigned int* counter = reinterpret_cast<unsigned int*>(sc + NYS_CG_FLAG + 1);
  cg_dir_kernel<<<vec_blocks(n), kVecThreads, 0, as_stream(stream)>>>(n, z, p, first, sc, counter);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" size_t nys_precond_workspace(int64_t n, int r) {
  // reduction scratch + coef (r) + per-block h partials
  return (kRedPartials * 16 + 64) * sizeof(double) + (size_t)(r + 1) * sizeof(double) +
         (size_t)kVecMaxBlocks * (r + 1) * sizeof(double);
}

namespace nys {
int precond_apply_z(const double* U, int64_t n, int r, int64_t ldu, const double* v, double* z, const double* rdot,
                    double* rz, void* ws, cudaStream_t st, const double* pred);
double* precond_coef(void* ws);
// Eq. (11) apply, every launch predicated on *pred == 0 (nullptr: always run)
int precond_apply(const double* U, int64_t n, int r, int64_t ldu, const double* lam, double nu,
                  const double* v, double* z, const double* rdot, double* rz, void* ws, size_t ws_bytes,
                  cudaStream_t st, const double* pred) {
  if (n <= 0 || r < 0 || (r > 0 && ldu < r)) return NYS_ERR_ARG;
  if (ws_bytes < nys_precond_workspace(n, r)) return NYS_ERR_WORKSPACE;
  if (r == 0) {
    copy_dot_kernel<<<vec_blocks(n), kVecThreads, 0, st>>>(n, v, z, rdot, rz, RED_ARGS(ws), pred);
    NYS_CHECK_LAUNCH();
    return NYS_OK;
  }
  double* coef = reinterpret_cast<double*>(reinterpret_cast<char*>(ws) +
                                           (kRedPartials * 16 + 64) * sizeof(double));
  double* hpart = coef + (r + 1);
  if (r > 512) return NYS_ERR_UNSUPPORTED;
  const int64_t blocks = tmin<int64_t>(kNumSMs * 2, tmax<int64_t>(1, cdiv(n, 32)));
  const int64_t rpb = cdiv(n, blocks);
  const int64_t nb = cdiv(n, rpb);
  // many row blocks: their column sums in a separate reduction kernel
  const bool split = nb > 32;
  precond_utv_kernel<<<(unsigned)nb, kPcThreads, (kPcThreads / 32) * r * sizeof(double), st>>>(
      U, n, r, ldu, v, rpb, hpart, split ? nullptr : red_counter(ws), lam, nu, coef, pred);
  NYS_CHECK_LAUNCH();
  if (split) {
    utv_reduce_kernel<<<(unsigned)r, 256, 0, st>>>(hpart, (int)nb, r, lam, nu, coef, pred);
    NYS_CHECK_LAUNCH();
  }
  return precond_apply_z(U, n, r, ldu, v, z, rdot, rz, ws, st, pred);
}

// the second pass alone (coef already in the workspace, e.g. from the fused
// CG step of cg.cu)
int precond_apply_z(const double* U, int64_t n, int r, int64_t ldu, const double* v, double* z, const double* rdot,
                    double* rz, void* ws, cudaStream_t st, const double* pred) {
  const int64_t ab = tmin<int64_t>(kVecMaxBlocks, cdiv(n * 32, 256));
  precond_apply_kernel<<<(unsigned)ab, 256, r * sizeof(double), st>>>(U, n, r, ldu, precond_coef(ws), v, z,
                                                                      rdot, rz, RED_ARGS(ws), pred);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

double* precond_coef(void* ws) {
  return reinterpret_cast<double*>(reinterpret_cast<char*>(ws) + (kRedPartials * 16 + 64) * sizeof(double));
}
double* precond_hpart(void* ws, int r) { return precond_coef(ws) + (r + 1); }
}  // namespace nys

extern "C" int nys_precond_apply_f64(const double* U, int64_t n, int r, int64_t ldu,
                                     const double* lam, double nu, const double* v, double* z,
                                     const double* rdot, double* rz, void* ws, size_t ws_bytes,
                                     void* stream) {
  return precond_apply(U, n, r, ldu, lam, nu, v, z, rdot, rz, ws, ws_bytes, as_stream(stream), nullptr);
}

extern "C" int nys_admm_rhs_f64(int64_t n, const double* hxA, const double* gA, const double* q,
                                double lambda2, double sigma, double rho, double shift,
                                const double* x, const double* z, const double* u, double* rhs,
                                double* r, double* sc, void* ws, void* stream) {
  if (n <= 0) return NYS_ERR_ARG;
  admm_rhs_kernel<<<vec_blocks(n), kVecThreads, 0, as_stream(stream)>>>(
      n, hxA, gA, q, lambda2, sigma, rho, shift, x, z, u, rhs, r, sc, RED_ARGS(ws));
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

// small copy by a kernel (dst may be mapped pinned host memory): the per-
// iteration readback goes out with the stream's kernels instead of through a
// copy engine (no copy-engine round trip between two kernels of the pipeline)
__global__ void copy_small_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
  __threadfence_system();
}

extern "C" int nys_copy_f64(const double* src, double* dst, int64_t n, void* stream) {
  if (n < 0 || (n > 0 && (!src || !dst))) return NYS_ERR_ARG;
  if (n == 0) return NYS_OK;
  copy_small_kernel<<<(unsigned)tmin<int64_t>(cdiv(n, 256), 64), 256, 0, as_stream(stream)>>>(src, dst, n);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

__global__ void readback_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t n, double* gate,
                                const double* __restrict__ pred) {
  pdl_begin();  // chain kernel (common.cuh)
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
  __threadfence_system();
  if (gate && blockIdx.x == 0 && threadIdx.x == 0 && !(pred && *pred != 0.0)) *gate = 1.0;
}

extern "C" int nys_readback_f64(const double* src, double* dst, int64_t n, double* gate_next, const double* pred,
                                void* stream) {
  if (n < 0 || (n > 0 && (!src || !dst))) return NYS_ERR_ARG;
  launch_chain(readback_kernel, dim3((unsigned)tmin<int64_t>(cdiv(tmax<int64_t>(n, 1), 256), 64)), dim3(256), 0,
               as_stream(stream), false, src, dst, n, gate_next, pred);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_admm_head_f64(const nys_admm_head* h, void* stream) {
  if (!h || h->n <= 0 || !h->rhs || !h->r || !h->sc || !h->ws_red) return NYS_ERR_ARG;
  if (h->snap && (!h->xbar || !h->zbar)) return NYS_ERR_ARG;
  if (h->tol_out && h->tol_fixed <= 0.0 && (!h->prev || !(h->kpow > 0.0))) return NYS_ERR_ARG;
  admm_head_kernel<<<vec_blocks(h->n), kVecThreads, 0, as_stream(stream)>>>(*h, red_part(h->ws_red),
                                                                           red_counter(h->ws_red));
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_admm_zu_f64(int64_t n, const double* x, double* z, double* u, double alpha,
                               int prox_kind, double kappa, const double* lo, const double* hi,
                               double* xbar, double* zbar, int accum, void* stream) {
  if (n <= 0) return NYS_ERR_ARG;
  if (prox_kind == NYS_PROX_BOX && (!lo || !hi)) return NYS_ERR_ARG;
  admm_zu_kernel<<<vec_blocks(n), kVecThreads, 0, as_stream(stream)>>>(
      n, x, z, u, alpha, prox_kind, kappa, lo, hi, xbar, zbar, accum);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_admm_norms_f64(int64_t n, const double* x, const double* z, const double* u,
                                  const double* gA, const double* q, double lambda2, double rho,
                                  const double* atnu, double lambda1, const double* lo,
                                  const double* hi, double* out, void* ws, void* stream) {
  if (n <= 0) return NYS_ERR_ARG;
  admm_norms_kernel<<<vec_blocks(n), kVecThreads, 0, as_stream(stream)>>>(
      n, x, z, u, gA, q, lambda2, rho, atnu, lambda1, lo, hi, out, RED_ARGS(ws));
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_ml_rowwise_f64(int64_t rows, int loss, const double* Ax, const double* Az,
                                  const double* b, double* tg, double* w, double* thx,
                                  double* tnu, double* out, void* ws, void* stream) {
  if (rows <= 0 || loss < 0 || loss > 2) return NYS_ERR_ARG;
  ml_rowwise_kernel<<<vec_blocks(rows), kVecThreads, 0, as_stream(stream)>>>(
      rows, loss, Ax, Az, b, tg, w, thx, tnu, out, RED_ARGS(ws));
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_ml_conj_scaled_f64(int64_t rows, int loss, const double* nu, double c,
                                      const double* b, double* out, void* ws, void* stream) {
  if (rows <= 0 || loss < 0 || loss > 2) return NYS_ERR_ARG;
  ml_conj_scaled_kernel<<<vec_blocks(rows), kVecThreads, 0, as_stream(stream)>>>(
      rows, loss, nu, c, b, out, RED_ARGS(ws));
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_window_norms_f64(int64_t n, const double* ring, int64_t ld, int cur,
                                    const int* others, int nothers, double* out, void* ws,
                                    void* stream) {
  if (n <= 0 || nothers < 0 || nothers > 16) return NYS_ERR_ARG;
  SlotList sl;
  for (int j = 0; j < 16; ++j) sl.idx[j] = j < nothers ? others[j] : 0;
  window_norms_kernel<<<vec_blocks(n), kVecThreads, 0, as_stream(stream)>>>(
      n, ring, ld, cur, sl, nothers, out, RED_ARGS(ws));
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_scale_dual_f64(int64_t n, double* u, double rho_old, double rho_new,
                                  double* out, void* ws, void* stream) {
  if (n <= 0 || !(rho_new > 0.0)) return NYS_ERR_ARG;
  scale_dual_kernel<<<vec_blocks(n), kVecThreads, 0, as_stream(stream)>>>(n, u, rho_old, rho_new,
                                                                          out, RED_ARGS(ws));
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_qp_infeas_f64(int64_t n, const double* xa, const double* xb, const double* ua,
                                 const double* ub, double width, const double* lo,
                                 const double* hi, const double* q, double* dx, double* out,
                                 void* ws, void* stream) {
  if (n <= 0 || !(width > 0.0)) return NYS_ERR_ARG;
  qp_infeas_kernel<<<vec_blocks(n), kVecThreads, 0, as_stream(stream)>>>(
      n, xa, xb, ua, ub, width, lo, hi, q, dx, out, RED_ARGS(ws));
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_axpby_f64(int64_t n, double a, const double* x, double b, double* y,
                             void* stream) {
  if (n <= 0) return NYS_ERR_ARG;
  axpby_kernel<<<vec_blocks(n), kVecThreads, 0, as_stream(stream)>>>(n, a, x, b, y);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_soft_threshold_f64(int64_t n, const double* v, double kappa, double* out,
                                      void* stream) {
  if (n <= 0 || kappa < 0) return NYS_ERR_ARG;
  soft_kernel<<<vec_blocks(n), kVecThreads, 0, as_stream(stream)>>>(n, v, kappa, out);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_loss_eval_f64(int loss, int what, int64_t n, const double* w, double* out, void* stream) {
  if (n <= 0 || what < 0 || what > 3 || loss < NYS_LOSS_SQUARE || loss > NYS_LOSS_HUBER) return NYS_ERR_ARG;
  loss_eval_kernel<<<vec_blocks(n), kVecThreads, 0, as_stream(stream)>>>(loss, what, n, w, out);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_box_project_f64(int64_t n, const double* v, const double* lo,
                                   const double* hi, double* out, void* stream) {
  if (n <= 0) return NYS_ERR_ARG;
  box_kernel<<<vec_blocks(n), kVecThreads, 0, as_stream(stream)>>>(n, v, lo, hi, out);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_row_scale_f64(int64_t rows, int64_t cols, double* X, int64_t ldx,
                                 const double* d, void* stream) {
  if (rows <= 0 || cols <= 0 || ldx < cols) return NYS_ERR_ARG;
  row_scale_kernel<<<vec_blocks(rows * cols), kVecThreads, 0, as_stream(stream)>>>(rows, cols, X,
                                                                                   ldx, d);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

// ------------------------------------------------------ ADMM tail ---------
namespace nys {
int gemv_n(const double* A, int64_t rows, int64_t n, int64_t lda, const double* X, int64_t ldx, int k, double* Y,
           int64_t ldy, const double* dscale, void* ws, size_t ws_bytes, cudaStream_t st, const double* pred);
int gemv_t(const double* A, int64_t rows, int64_t n, int64_t lda, const double* T, int64_t ldt, int k, double* Y,
           int64_t ldy, const double* v, double shift, double* dot, void* ws, size_t ws_bytes, cudaStream_t st,
           const double* pred);
int gemv_t_partials(const double* A, int64_t rows, int64_t n, int64_t lda, const double* T, int64_t ldt, int k,
                    void* ws, size_t ws_bytes, cudaStream_t st, const double* pred, double** P, int* splits,
                    const double* order);
int tail_cluster(const double* A, int64_t rows, int64_t n, int64_t lda, const double* x, const double* z,
                 const double* b, int loss, double* T, double* w, void* ws, size_t ws_bytes, size_t ws_off,
                 double* rowsums, cudaStream_t st, const double* pred, double** Pout, int* splits_out,
                 const double* gb, int* sq_out);
bool tail_wants_sparse_z(const double* A, int64_t rows, int64_t n, int64_t lda, const double* x);
int tail_partial_sum(const double* P, int64_t n, int K, int ncl, double* AT, const double* gb, cudaStream_t st,
                     const double* pred);
int xz_rowpass(const double* A, int64_t rows, int64_t n, int64_t lda, const double* x, const double* z,
               const double* b, int loss, double* tg, double* w, double* thx, double* tnu, double* rowsums,
               double* part, unsigned int* counter, cudaStream_t st, const double* pred, const double* order);
}  // namespace nys

extern "C" int nys_admm_tail_f64(const nys_admm_tail* t, void* stream) {
  if (!t || t->n <= 0 || (t->kind != 0 && t->kind != 1)) return NYS_ERR_ARG;
  nys_admm_tail* t_mut = const_cast<nys_admm_tail*>(t);  // rb_done, stop_ran are outputs
  t_mut->rb_done = 0;
  t_mut->stop_ran = 0;
  cudaStream_t st = as_stream(stream);
  const int64_t n = t->n;
  const double* pred = t->pred;
  double* x = t->XZ;
  double* z = t->XZ + n;
  int rc;
  // relax / prox / dual update + averages (admm.py:562-583), unless the
  // persistent x-update kernel already ran it (nys_admm_head.zu)
  if (!t->zu_done) {
    admm_zu_kernel<<<vec_blocks(n), kVecThreads, 0, st>>>(n, x, z, t->u, t->alpha,
                                                          t->kind == 0 ? NYS_PROX_SOFT : NYS_PROX_BOX, t->kappa, t->lo,
                                                          t->hi, t->xbar, t->zbar, t->accum, pred);
    NYS_CHECK_LAUNCH();
  }
  // window append (admm.py:622-623), speculative: the host commits it
  if (t->ring && !t->zu_done) {
    ring_copy_kernel<<<vec_blocks(n), kVecThreads, 0, st>>>(n, x, t->ring + (int64_t)t->slot * t->ring_ld, t->u,
                                                            t->uring ? t->uring + (int64_t)t->slot * t->ring_ld
                                                                     : nullptr,
                                                            pred);
    NYS_CHECK_LAUNCH();
  }
  // data passes at (x, z) (admm.py:585-587)
  if (t->kind == 0) {
    const int64_t woff0 = t->wnorms - t->norms;
    const bool fuse0 = !t->reduce && woff0 >= 16 && woff0 <= 64 &&
                       epi_fits(n);
    // wide rows: the whole tail's data passes in one cluster stream over A
    // (hvp_cluster.cu: tail_cluster_kernel); else the row pass + GEMV^T below
    // (row-sharded: the same stream, its partials summed into this rank's AT,
    // which is all-reduced before the norms)
    double* Pc = nullptr;
    int csplits = 0, csq = 0;
    // (without an l1 term the prox leaves z dense: the very-wide-row plan, which
    // walks z's nonzeros, would lose to the two passes)
    const bool dense_z = t->with_z && !(t->kappa > 0.0) && tail_wants_sparse_z(t->A, t->rows, n, t->lda, x);
    if ((fuse0 || t->reduce) && !dense_z) {
      rc = tail_cluster(t->A, t->rows, n, t->lda, x, t->with_z ? z : nullptr, t->b, t->loss, t->T, t->w, t->ws_gemvT,
                        t->ws_gemvT_bytes, (kRedPartials * 16 + 64) * sizeof(double), t->rowsums, st, pred, &Pc,
                        &csplits, t->gb, &csq);
      if (rc != NYS_OK && rc != NYS_ERR_UNSUPPORTED) return rc;
      if (rc != NYS_OK) Pc = nullptr;
    }
    // A{x, z} + loss epilogue in one streaming pass (rowpass.cu), else the
    // 2-RHS GEMV and the row-wise kernel
    rc = Pc ? NYS_OK : xz_rowpass(t->A, t->rows, n, t->lda, x, t->with_z ? z : nullptr, t->b, t->loss, t->T, t->w, t->T + t->rows,
                    t->with_z ? t->T + 2 * t->rows : nullptr, t->rowsums, red_part(t->ws_red), red_counter(t->ws_red),
                    st, pred, t->order);
    if (rc == NYS_ERR_UNSUPPORTED) {
      const int k = t->with_z ? 2 : 1;
      if ((rc = gemv_n(t->A, t->rows, n, t->lda, t->XZ, n, k, t->AXZ, t->rows, nullptr, t->ws_gemv,
                       t->ws_gemv_bytes, st, pred)))
        return rc;
      ml_rowwise_kernel<<<vec_blocks(t->rows), kVecThreads, 0, st>>>(
          t->rows, t->loss, t->AXZ, t->with_z ? t->AXZ + t->rows : nullptr, t->b, t->T, t->w, t->T + t->rows,
          t->with_z ? t->T + 2 * t->rows : nullptr, t->rowsums, red_part(t->ws_red), red_counter(t->ws_red), pred);
      NYS_CHECK_LAUNCH();
    } else if (rc) {
      return rc;
    }
    const int64_t woff = t->wnorms - t->norms;
    // (row-sharded: the A^T outputs are all-reduced before the norms, so the
    // split sum cannot be fused with them)
    const bool fuse = !t->reduce && woff >= 16 && woff <= 64 &&
                      epi_fits(n);
    if (fuse) {
      // A^T split partials, then one epilogue kernel: split sum -> AT, norms, window norms
      double* P = Pc;
      int splits = csplits;
      const int K = t->with_z ? 3 : 2;
      if (!P && (rc = gemv_t_partials(t->A, t->rows, n, t->lda, t->T, t->rows, K, t->ws_gemvT, t->ws_gemvT_bytes, st,
                                      pred, &P, &splits, t->order)))
        return rc;
      SlotList sl;
      const int no = (t->ring && t->nothers > 0) ? t->nothers : 0;
      for (int j = 0; j < 16; ++j) sl.idx[j] = j < no ? t->others[j] : 0;
      const unsigned eb = (unsigned)epi_blocks(n);
      const double* Pc = P;
      const double* uc = t->u;
      const double* ringc = t->ring;
      double* normsp = t->norms;
      double* rp = red_part(t->ws_red);
      unsigned int* rc2 = red_counter(t->ws_red);
      // the epilogue is the last kernel of the tail unless the conjugate sums or
      // the gate kernel follow: then it also does the iteration's readback
      const bool rb = t->rb_dst && !(t->with_z && t->conj_out) && !t->gate_next;
      const double* rbs = rb ? t->rb_src : nullptr;
      double* rbd = rb ? t->rb_dst : nullptr;
      double* rbg = rb ? t->rb_gate : nullptr;
      const int rbn = (int)t->rb_n;
      const double rbt = t->rb_tag;
      StopArgs sa{};
      // the device decision is only valid where this kernel is the iteration's
      // last (it reads the row sums and opens the gate) and no conjugate-sum
      // kernel follows (the logistic gap with lambda2 = 0 needs it)
      sa.on = (t->stop_on && rb && !t->conj_out) ? 1 : 0;
      sa.gap = t->stop_gap, sa.linf = t->stop_linf, sa.loss = t->loss, sa.slot = t->stop_slot;
      sa.eps_gap = t->stop_eps_gap, sa.eps_abs = t->stop_eps_abs, sa.eps_rel = t->stop_eps_rel;
      sa.sqrt_n = t->stop_sqrt_n, sa.l1 = t->lambda1, sa.l2 = t->lambda2;
      t_mut->stop_ran = sa.on;  // out: whether the device test ran
      if (K == 3)
        launch_chain(ml_epilogue_kernel<3>, dim3(eb), dim3(256), 0, st, false, n, Pc, splits, t->AT, x, z, uc,
                     t->lambda2, t->rho, t->lambda1, ringc, t->ring_ld, t->slot, sl, no, normsp, (int)woff, rp, rc2,
                     pred, rbs, rbd, rbn, rbg, rbt, sa, (Pc && csq) ? t->gb : nullptr);
      else
        launch_chain(ml_epilogue_kernel<2>, dim3(eb), dim3(256), 0, st, false, n, Pc, splits, t->AT, x, z, uc,
                     t->lambda2, t->rho, t->lambda1, ringc, t->ring_ld, t->slot, sl, no, normsp, (int)woff, rp, rc2,
                     pred, rbs, rbd, rbn, rbg, rbt, sa, nullptr);
      NYS_CHECK_LAUNCH();
      t_mut->rb_done = rb ? 1 : 0;
    } else {
      if (Pc) {
        if ((rc = tail_partial_sum(Pc, n, t->with_z ? 3 : 2, csplits, t->AT, csq ? t->gb : nullptr, st, pred)))
          return rc;
      } else if ((rc = gemv_t(t->A, t->rows, n, t->lda, t->T, t->rows, t->with_z ? 3 : 2, t->AT, n, nullptr, 0.0,
                              nullptr, t->ws_gemvT, t->ws_gemvT_bytes, st, pred))) {
        return rc;
      }
      if (t->reduce) {  // this rank's A^T outputs and row sums: sum over the ranks
        t->reduce(t->AT, (int64_t)(t->with_z ? 3 : 2) * n, t->reduce_user, st);
        t->reduce(t->rowsums, NYS_ROWS_NOUT, t->reduce_user, st);
        if (cudaPeekAtLastError() != cudaSuccess) return NYS_ERR_CUDA;
      }
      admm_norms_kernel<<<vec_blocks(n), kVecThreads, 0, st>>>(n, x, z, t->u, t->AT, nullptr, t->lambda2, t->rho,
                                                               t->with_z ? t->AT + 2 * n : nullptr, t->lambda1,
                                                               nullptr, nullptr, t->norms, red_part(t->ws_red),
                                                               red_counter(t->ws_red), pred);
      NYS_CHECK_LAUNCH();
    }
  } else {
    if ((rc = gemv_n(t->A, n, n, t->lda, x, n, 1, t->AT, n, nullptr, t->ws_gemv, t->ws_gemv_bytes, st, pred)))
      return rc;
    admm_norms_kernel<<<vec_blocks(n), kVecThreads, 0, st>>>(n, x, z, t->u, t->AT, t->q, 0.0, t->rho, nullptr, 0.0,
                                                             t->lo, t->hi, t->norms, red_part(t->ws_red),
                                                             red_counter(t->ws_red), pred);
    NYS_CHECK_LAUNCH();
  }
  // cycle-guard norms for the window after the append (admm.py:645-655);
  // the ML epilogue kernel already computed them when it ran fused
  const bool ml_fused = t->kind == 0 && !t->reduce && (t->wnorms - t->norms) >= 16 &&
                        (t->wnorms - t->norms) <= 64 && epi_fits(n);
  if (t->ring && t->nothers > 0 && !ml_fused) {
    SlotList sl;
    for (int j = 0; j < 16; ++j) sl.idx[j] = j < t->nothers ? t->others[j] : 0;
    window_norms_kernel<<<vec_blocks(n), kVecThreads, 0, st>>>(n, t->ring, t->ring_ld, t->slot, sl, t->nothers,
                                                               t->wnorms, red_part(t->ws_red), red_counter(t->ws_red),
                                                               pred);
    NYS_CHECK_LAUNCH();
  }
  // QP infeasibility pieces over the 25-step window (admm.py:624-634, 361-415)
  if (t->kind == 1 && t->qp_infeas) {
    qp_infeas_kernel<<<vec_blocks(n), kVecThreads, 0, st>>>(
        n, t->ring + (int64_t)t->inf_last * t->ring_ld, t->ring + (int64_t)t->inf_first * t->ring_ld,
        t->uring + (int64_t)t->inf_last * t->ring_ld, t->uring + (int64_t)t->inf_first * t->ring_ld, t->width, t->lo,
        t->hi, t->q, t->dx, t->infeas, red_part(t->ws_red), red_counter(t->ws_red), pred);
    NYS_CHECK_LAUNCH();
    if ((rc = gemv_n(t->A, n, n, t->lda, t->dx, n, 1, t->Pdx, n, nullptr, t->ws_gemv, t->ws_gemv_bytes, st, pred)))
      return rc;
    dot_pred_kernel<<<vec_blocks(n), kVecThreads, 0, st>>>(n, t->Pdx, t->Pdx, t->pdx2, red_part(t->ws_red),
                                                           red_counter(t->ws_red), pred);
    NYS_CHECK_LAUNCH();
  }
  // scaled-dual conjugate sums for the gap (problems.py:330-340), device-side c
  if (t->kind == 0 && t->with_z && t->conj_out) {
    const double* nuc = t->T + 2 * t->rows;
    const double* sc13 = t->norms + 13;
    launch_chain(ml_conj_dev_kernel, dim3((unsigned)vec_blocks(t->rows)), dim3(kVecThreads), 0, st, false, t->rows,
                 t->loss, nuc, sc13, t->lambda1, t->b, t->conj_out, red_part(t->ws_red), red_counter(t->ws_red), pred);
    NYS_CHECK_LAUNCH();
    if (t->reduce) {  // sums over this rank's rows
      t->reduce(t->conj_out, 3, t->reduce_user, st);
      if (cudaPeekAtLastError() != cudaSuccess) return NYS_ERR_CUDA;
    }
  }
  if (t->gate_next) {
    launch_chain(open_gate_kernel, dim3(1), dim3(32), 0, st, false, t->gate_next, pred);
    NYS_CHECK_LAUNCH();
  }
  return NYS_OK;
}
