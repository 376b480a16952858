// Symmetric eigensolver for the sketch (s <= 160): tridiagonalisation +
// bisection + inverse iteration + back-transformation.
//
//   K_a  Householder reduction A = Q T Q^T (one CTA, A in shared memory,
//        s - 2 steps of: column norm, reflector, p = tau A22 v, rank-2 update);
//   K_b  every eigenvalue of T by 32-way multisection on the Sturm count
//        (one warp per eigenvalue, 14 steps of 33 sub-intervals ~ 2^-70);
//   K_c  eigenvectors of T by inverse iteration with a pivoted tridiagonal LU
//        (one thread per cluster of close eigenvalues; members of a cluster
//        are Gram-Schmidt-orthogonalised against each other);
//   K_d  z = Q y by applying the s - 2 reflectors (one warp per vector).
// Replaces the eigh / thin-SVD LAPACK calls of sketch.py:115,126 for the
// s x s problems the Nystrom sketch produces; the s > 160 case uses the
// block Jacobi of eig.cu.
#include <math.h>
#include "common.cuh"

namespace nys {

constexpr int kTriMaxS = 160;
constexpr int kTriThreads = 512;

// --------------------------------------------------------------- K_a ------
// Householder reduction with A in shared memory, four barriers per column:
//   1 v (scaled column) -> smem (||x(2:)||^2 comes from the previous update)
//   2 symv partials: thread (g, j) sums rows g, g+RG, ... of column j of A22
//     (columns are contiguous in smem: no bank conflicts, no warp reductions)
//   3 p_j = tau sum_g partial(g, j) and the p.v partials
//   4 rank-2 update A22 -= v w^T + w v^T with w = p - (tau/2)(p.v) v: each
//     thread keeps v_j, w_j of its columns in registers and walks its rows;
//     the updated column k+1 squares feed the next column's norm.
// The reflectors are stored row-wise (VhT[k][*]) for the coalesced
// back-transformation.
constexpr int kTriRG = 8;  // max row groups of the symv
constexpr int kTriCols = (kTriMaxS + 31) / 32;
__global__ void __launch_bounds__(kTriThreads)
tridiag_kernel(int s, const double* __restrict__ A, double* __restrict__ d, double* __restrict__ e,
               double* __restrict__ VhT, double* __restrict__ tau) {
  extern __shared__ double sm[];
  const int ld = s | 1;
  double* a = sm;                         // s x ld
  double* vs = a + (size_t)s * ld;        // s
  double* pw = vs + s;                    // s
  double* part = pw + s;                  // kTriRG x s
  double* red = part + (size_t)kTriRG * s;  // 2 x 64
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int t = tid; t < s * s; t += blockDim.x) {
    const int i = t / s, j = t - i * s;
    a[i * ld + j] = A[t];
  }
  __syncthreads();
  {  // ||x(2:)||^2 of column 0
    double pt = 0.0;
    for (int i = 2 + tid; i < s; i += blockDim.x) pt = fma(a[i * ld], a[i * ld], pt);
    pt = warp_sum(pt);
    if (lane == 0) red[warp] = pt;
    for (int q = nw + tid; q < 32; q += blockDim.x) red[q] = 0.0;
  }
  __syncthreads();
  for (int k = 0; k + 2 < s; ++k) {
    const int m = s - k - 1;  // size of the trailing block
    double* rn = red + (k & 1) * 64;  // norm partials of this column (written by the previous update)
    const double xn2 = warp_sum(rn[lane]);
    const double alpha = a[(k + 1) * ld + k];
    double tk, beta, scal;
    if (xn2 == 0.0) {
      tk = 0.0;
      beta = alpha;
      scal = 0.0;
    } else {
      beta = -copysign(sqrt(fma(alpha, alpha, xn2)), alpha);
      tk = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    if (tid == 0) {
      tau[k] = tk;
      e[k] = beta;
    }
    // 1. reflector v (v_0 = 1)
    for (int i = tid; i < m; i += blockDim.x) {
      const double vi = (i == 0) ? 1.0 : a[(k + 1 + i) * ld + k] * scal;
      vs[i] = vi;
      VhT[(size_t)k * s + (k + 1 + i)] = vi;
    }
    double* rnext = red + ((k + 1) & 1) * 64;
    if (tk == 0.0) {  // H = I: no update; the next column's norm directly (uniform branch)
      double pt = 0.0;
      for (int i = k + 3 + tid; i < s; i += blockDim.x) pt = fma(a[i * ld + k + 1], a[i * ld + k + 1], pt);
      pt = warp_sum(pt);
      if (lane == 0) rnext[warp] = pt;
      for (int q = nw + tid; q < 32; q += blockDim.x) rnext[q] = 0.0;
      __syncthreads();
      continue;
    }
    __syncthreads();
    // 2. symv partials over row groups
    const int colsP = (m + 31) & ~31;
    const int RG = min(kTriRG, (int)blockDim.x / colsP);
    {
      const int g = tid / colsP, j = tid - g * colsP;
      if (g < RG && j < m) {
        const double* col = a + (size_t)(k + 1) * ld + (k + 1) + j;
        double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
        int i = g;
        for (; i + 3 * RG < m; i += 4 * RG) {
          acc0 = fma(col[(size_t)i * ld], vs[i], acc0);
          acc1 = fma(col[(size_t)(i + RG) * ld], vs[i + RG], acc1);
          acc2 = fma(col[(size_t)(i + 2 * RG) * ld], vs[i + 2 * RG], acc2);
          acc3 = fma(col[(size_t)(i + 3 * RG) * ld], vs[i + 3 * RG], acc3);
        }
        for (; i < m; i += RG) acc0 = fma(col[(size_t)i * ld], vs[i], acc0);
        part[g * s + j] = (acc0 + acc1) + (acc2 + acc3);
      }
    }
    __syncthreads();
    // 3. p = tau A22 v and the p.v partials
    double pt = 0.0;
    for (int j = tid; j < m; j += blockDim.x) {
      double pj = 0.0;
      for (int g = 0; g < RG; ++g) pj += part[g * s + j];
      pj *= tk;
      pw[j] = pj;
      pt = fma(pj, vs[j], pt);
    }
    pt = warp_sum(pt);
    if (lane == 0) red[128 + warp] = pt;
    __syncthreads();
    const double pv = warp_sum(lane < nw ? red[128 + lane] : 0.0);
    const double hpv = 0.5 * tk * pv;
    // 4. A22 -= v w^T + w v^T,  w = p - hpv v (v_j, w_j of this lane in registers)
    double vj[kTriCols], wj[kTriCols];
#pragma unroll
    for (int c = 0; c < kTriCols; ++c) {
      const int j = lane + 32 * c;
      vj[c] = j < m ? vs[j] : 0.0;
      wj[c] = j < m ? fma(-hpv, vj[c], pw[j]) : 0.0;
    }
    double nrm = 0.0;  // squares of the updated column k+1 below row k+2
    for (int i = warp; i < m; i += nw) {
      double* ar = a + (k + 1 + i) * ld + (k + 1);
      const double vi = vs[i], wi = fma(-hpv, vi, pw[i]);
#pragma unroll
      for (int c = 0; c < kTriCols; ++c) {
        const int j = lane + 32 * c;
        if (j < m) {
          const double t = ar[j] - fma(vi, wj[c], wi * vj[c]);
          ar[j] = t;
          if (c == 0 && lane == 0 && i >= 2) nrm = fma(t, t, nrm);
        }
      }
    }
    // lane 0 of each warp holds its rows' partial; other lanes hold 0
    if (lane == 0) rnext[warp] = nrm;
    for (int q = nw + tid; q < 32; q += blockDim.x) rnext[q] = 0.0;
    __syncthreads();
  }
  for (int i = tid; i < s; i += blockDim.x) d[i] = a[i * ld + i];
  if (tid == 0 && s >= 2) e[s - 2] = a[(s - 1) * ld + (s - 2)];
  if (tid == 0 && s >= 1) e[s - 1] = 0.0;
}

// Same reduction with the next column's symv fused into the rank-2 update
// (look-ahead by one column) and ONE barrier per column:
//   A  every warp recomputes the updated first row of A22 in registers (the
//      column the next reflector comes from; only its diagonal is stored), then the
//      next reflector v' from it: norms by warp_sum, identical in all warps;
//   B  each warp updates its rows of A22 (columns >= 1) and, while the new
//      values are in registers, takes their dot with v' -> p' = tau' A'' v'
//      (one warp_sum per row; two rows in flight).
// A22 is read and written once per column instead of read twice and written
// once, and p.v is re-summed from shared memory after the barrier.
__device__ __forceinline__ void tri_reflector(double alpha, double xn2, double& tk, double& beta, double& scal) {
  if (xn2 == 0.0) {
    tk = 0.0;
    beta = alpha;
    scal = 0.0;
  } else {
    beta = -copysign(sqrt(fma(alpha, alpha, xn2)), alpha);
    tk = (beta - alpha) / beta;
    scal = 1.0 / (alpha - beta);
  }
}

// One column of tridiag_fused_kernel with NC = ceil(m / 32) column chunks per
// lane (the trailing block shrinks: no issue slots on dead chunks).
template <int NC>
__device__ __forceinline__ double tri_fused_step(int s, int k, int ld, double* __restrict__ a,
                                                 double* __restrict__ vsb, double* __restrict__ pwb,
                                                 double* __restrict__ d, double* __restrict__ e,
                                                 double* __restrict__ VhT, double* __restrict__ tau, double tk) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int m = s - k - 1;
  const double* vs = vsb + (k & 1) * s;
  const double* pw = pwb + (k & 1) * s;
  double* vsn = vsb + ((k + 1) & 1) * s;
  double* pwn = pwb + ((k + 1) & 1) * s;
  double vj[NC], wj[NC];
  double pv = 0.0;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int j = lane + 32 * c;
    vj[c] = j < m ? vs[j] : 0.0;
    wj[c] = j < m ? pw[j] : 0.0;
    pv = fma(wj[c], vj[c], pv);
  }
  pv = warp_sum(pv);
  const double hpv = 0.5 * tk * pv;
#pragma unroll
  for (int c = 0; c < NC; ++c) wj[c] = fma(-hpv, vj[c], wj[c]);
  // A: updated row 0 of A22 (global row k+1)
  const double v0 = __shfl_sync(0xffffffffu, vj[0], 0), w0 = __shfl_sync(0xffffffffu, wj[0], 0);
  double t0[NC];
  double* a0 = a + (k + 1) * ld + (k + 1);
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int j = lane + 32 * c;
    t0[c] = j < m ? a0[j] - fma(v0, wj[c], w0 * vj[c]) : 0.0;
  }
  // row k+1 is final after this update (no write-back: other warps are
  // still reading it): its diagonal, and at the last column its e
  if (tid == 0) d[k + 1] = t0[0];
  if (tid == 1 && k + 3 == s) e[k + 1] = t0[0];
  const bool next = k + 3 < s;  // a reflector for column k+1 exists
  double vn[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) vn[c] = 0.0;
  double tkn = 0.0;
  if (next) {
    double xn2 = 0.0;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int j = lane + 32 * c;
      if (j >= 2) xn2 = fma(t0[c], t0[c], xn2);
    }
    xn2 = warp_sum(xn2);
    const double alpha = __shfl_sync(0xffffffffu, t0[0], 1);
    double beta, scal;
    tri_reflector(alpha, xn2, tkn, beta, scal);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int j = lane + 32 * c;
      vn[c] = j == 1 ? 1.0 : ((j >= 2 && j < m) ? t0[c] * scal : 0.0);
      if (warp == 0 && j >= 1 && j < m) {
        vsn[j - 1] = vn[c];
        VhT[(size_t)(k + 1) * s + (k + 1 + j)] = vn[c];
      }
    }
    if (tid == 0) {
      tau[k + 1] = tkn;
      e[k + 1] = beta;
    }
  }
  // B: rows 1..m-1 of A22, columns >= 1; fused dot with v'
  auto row = [&](int i) -> double {
    double* ar = a + (k + 1 + i) * ld + (k + 1);
    const double vi = vs[i], wi = fma(-hpv, vi, pw[i]);
    double dot = 0.0;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int j = lane + 32 * c;
      if (j >= 1 && j < m) {
        const double t = ar[j] - fma(vi, wj[c], wi * vj[c]);
        ar[j] = t;
        dot = fma(t, vn[c], dot);
      }
    }
    return dot;
  };
  int i = 1 + warp;
  for (; i + nw < m; i += 2 * nw) {
    double d0 = row(i), d1 = row(i + nw);
    if (next) {
      d0 = warp_sum(d0);
      d1 = warp_sum(d1);
      if (lane == 0) {
        pwn[i - 1] = tkn * d0;
        pwn[i + nw - 1] = tkn * d1;
      }
    }
  }
  if (i < m) {
    double d0 = row(i);
    if (next) {
      d0 = warp_sum(d0);
      if (lane == 0) pwn[i - 1] = tkn * d0;
    }
  }
  return tkn;
}

__global__ void __launch_bounds__(kTriThreads)
tridiag_fused_kernel(int s, const double* __restrict__ A, double* __restrict__ d, double* __restrict__ e,
                     double* __restrict__ VhT, double* __restrict__ tau) {
  extern __shared__ double sm[];
  const int ld = s | 1;
  double* a = sm;                   // s x ld
  double* vsb = a + (size_t)s * ld;  // 2 x s: v of the current / next reflector
  double* pwb = vsb + 2 * s;         // 2 x s: p = tau A22 v
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int t = tid; t < s * s; t += blockDim.x) {
    const int i = t / s, j = t - i * s;
    a[i * ld + j] = A[t];
  }
  __syncthreads();
  double tk = 0.0;
  if (s >= 3) {  // first reflector (column 0 = row 0) and its symv
    const int m = s - 1;
    double x[kTriCols], v[kTriCols];
    double xn2 = 0.0;
#pragma unroll
    for (int c = 0; c < kTriCols; ++c) {
      const int j = lane + 32 * c;
      x[c] = j < m ? a[1 + j] : 0.0;
      if (j >= 1) xn2 = fma(x[c], x[c], xn2);
    }
    xn2 = warp_sum(xn2);
    const double alpha = __shfl_sync(0xffffffffu, x[0], 0);
    double beta, scal;
    tri_reflector(alpha, xn2, tk, beta, scal);
#pragma unroll
    for (int c = 0; c < kTriCols; ++c) {
      const int j = lane + 32 * c;
      v[c] = j == 0 ? 1.0 : (j < m ? x[c] * scal : 0.0);
      if (warp == 0 && j < m) {
        vsb[j] = v[c];
        VhT[1 + j] = v[c];
      }
    }
    if (tid == 0) {
      tau[0] = tk;
      e[0] = beta;
    }
    for (int i = warp; i < m; i += nw) {
      const double* ar = a + (1 + i) * ld + 1;
      double dot = 0.0;
#pragma unroll
      for (int c = 0; c < kTriCols; ++c) {
        const int j = lane + 32 * c;
        if (j < m) dot = fma(ar[j], v[c], dot);
      }
      dot = warp_sum(dot);
      if (lane == 0) pwb[i] = tk * dot;
    }
  }
  __syncthreads();
  for (int k = 0; k + 2 < s; ++k) {
    switch ((s - k + 30) >> 5) {  // ceil(m / 32), m = s - k - 1
      case 1: tk = tri_fused_step<1>(s, k, ld, a, vsb, pwb, d, e, VhT, tau, tk); break;
      case 2: tk = tri_fused_step<2>(s, k, ld, a, vsb, pwb, d, e, VhT, tau, tk); break;
      case 3: tk = tri_fused_step<3>(s, k, ld, a, vsb, pwb, d, e, VhT, tau, tk); break;
      case 4: tk = tri_fused_step<4>(s, k, ld, a, vsb, pwb, d, e, VhT, tau, tk); break;
      default: tk = tri_fused_step<kTriCols>(s, k, ld, a, vsb, pwb, d, e, VhT, tau, tk); break;
    }
    __syncthreads();
  }
  if (s >= 3) {
    if (tid == 0) {
      d[0] = a[0];
      d[s - 1] = a[(s - 1) * ld + (s - 1)];
      e[s - 1] = 0.0;
    }
  } else {
    for (int i = tid; i < s; i += blockDim.x) d[i] = a[i * ld + i];
    if (tid == 0 && s >= 2) e[s - 2] = a[(s - 1) * ld + (s - 2)];
    if (tid == 0 && s >= 1) e[s - 1] = 0.0;
  }
}

// --------------------------------------------------------------- K_b ------
// number of eigenvalues of T strictly below x (LDL^T inertia), e2 = e^2;
// two shifts per call.  1/q by the MUFU reciprocal approximation and two
// Newton steps (full double precision; only the sign of q is used) keeps the
// division's slow-path branch out of the recurrence so the chains overlap.
__device__ __forceinline__ double rcp_nr(double q) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
  r = r * fma(-q, r, 2.0);
  r = r * fma(-q, r, 2.0);
  return r;
}
__device__ __forceinline__ void sturm_count2(int s, const double* __restrict__ d, const double* __restrict__ e2,
                                             const double (&x)[2], double pivmin, int (&c)[2]) {
  double q[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    q[u] = d[0] - x[u];
    if (fabs(q[u]) < pivmin) q[u] = -pivmin;
    c[u] = (q[u] < 0.0);
  }
  for (int i = 1; i < s; ++i) {
    const double di = d[i], ei = e2[i - 1];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      q[u] = fma(-ei, rcp_nr(q[u]), di - x[u]);
      if (fabs(q[u]) < pivmin) q[u] = -pivmin;
      c[u] += (q[u] < 0.0);
    }
  }
}

// CTA (one warp) j finds the j-th LARGEST eigenvalue by 64-way multisection
// (two shifts per lane).  One warp per SM: the Sturm recurrences are
// latency-bound, so spreading the eigenvalues over the SMs beats packing them.
__global__ void __launch_bounds__(32) bisect_kernel(int s, const double* __restrict__ d,
                                                    const double* __restrict__ e, double* __restrict__ w) {
  extern __shared__ double bsm[];
  double* ds = bsm;
  double* e2s = bsm + s;
  for (int i = threadIdx.x; i < s; i += blockDim.x) {
    ds[i] = d[i];
    e2s[i] = e[i] * e[i];
  }
  __syncwarp();
  const int lane = threadIdx.x & 31;
  const int j = blockIdx.x;
  // Gershgorin interval and pivot guard (LAPACK dstebz conventions)
  double lo = INFINITY, hi = -INFINITY, emax2 = 0.0;
  for (int i = lane; i < s; i += 32) {
    const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < s ? fabs(e[i]) : 0.0);
    lo = fmin(lo, ds[i] - r);
    hi = fmax(hi, ds[i] + r);
    if (i + 1 < s) emax2 = fmax(emax2, e2s[i]);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, off));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, off));
    emax2 = fmax(emax2, __shfl_xor_sync(0xffffffffu, emax2, off));
  }
  const double pivmin = 2.2250738585072014e-308 * fmax(1.0, emax2);
  const double tnorm = fmax(fabs(lo), fabs(hi));
  lo -= 2.2e-16 * tnorm * s + pivmin;
  hi += 2.2e-16 * tnorm * s + pivmin;
  const int t = s - 1 - j;  // ascending index
  double a = lo, b = hi;
  for (int it = 0; it < 14; ++it) {
    // 64 interior points a + (b - a) q / 65, q = 1..64; lane owns q = 2 lane + u + 1
    double x[2];
    int c[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) x[u] = a + (b - a) * (double)(2 * lane + u + 1) / 65.0;
    sturm_count2(s, ds, e2s, x, pivmin, c);
    int first = 64;
    if (c[1] > t) first = 2 * lane + 1;
    if (c[0] > t) first = 2 * lane;
    const unsigned any = __ballot_sync(0xffffffffu, first < 64);
    if (any == 0u) {
      a = a + (b - a) * 64.0 / 65.0;
    } else {
      int f = first;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) f = min(f, __shfl_xor_sync(0xffffffffu, f, off));
      const double nb = a + (b - a) * (double)(f + 1) / 65.0;
      const double na = f == 0 ? a : a + (b - a) * (double)f / 65.0;
      a = na;
      b = nb;
    }
    // relative precision, floored at the backward error of the reduction
    if (b - a <= 2.2e-16 * fmax(fabs(a), fabs(b)) + 1e-17 * tnorm + pivmin) break;
  }
  if (lane == 0) w[j] = 0.5 * (a + b);
}

// --------------------------------------------------------------- K_c ------
// Inverse iteration for the eigenvalues w (descending) of T, one thread per
// cluster (consecutive eigenvalues closer than 1e-3 ||T||, dstein's rule).
// Scratch per thread: 6 s doubles.
__device__ void tri_factor(int s, const double* d, const double* e, double lam, double eps_t, double* u0,
                           double* u1, double* u2, double* l, int* piv) {
  // Gaussian elimination with partial pivoting of T - lam I (upper has 3 diagonals)
  double diag = d[0] - lam, sup = s > 1 ? e[0] : 0.0, sup2 = 0.0;
  for (int i = 0; i < s - 1; ++i) {
    const double sub = e[i];
    const double nd = d[i + 1] - lam;
    const double ne = i + 2 < s ? e[i + 1] : 0.0;
    if (fabs(diag) >= fabs(sub)) {  // no interchange
      piv[i] = 0;
      const double piv_v = (diag == 0.0) ? eps_t : diag;
      const double li = sub / piv_v;
      l[i] = li;
      u0[i] = piv_v;
      u1[i] = sup;
      u2[i] = 0.0;
      diag = nd - li * sup;
      sup = ne;
    } else {  // swap rows i and i+1
      piv[i] = 1;
      const double li = diag / sub;
      l[i] = li;
      u0[i] = sub;
      u1[i] = nd;
      u2[i] = ne;
      diag = sup - li * nd;
      sup = -li * ne;
    }
    (void)sup2;
  }
  u0[s - 1] = (fabs(diag) < eps_t) ? (diag < 0.0 ? -eps_t : eps_t) : diag;
  u1[s - 1] = 0.0;
  u2[s - 1] = 0.0;
  for (int i = 0; i < s - 1; ++i)
    if (fabs(u0[i]) < eps_t) u0[i] = u0[i] < 0.0 ? -eps_t : eps_t;
}

__device__ void tri_solve(int s, const double* u0, const double* u1, const double* u2, const double* l,
                          const int* piv, double* y) {
  // forward: apply the row interchanges and multipliers
  for (int i = 0; i < s - 1; ++i) {
    if (piv[i]) {
      const double t = y[i];
      y[i] = y[i + 1];
      y[i + 1] = t - l[i] * y[i];
    } else {
      y[i + 1] -= l[i] * y[i];
    }
  }
  // back substitution with the 3-diagonal upper factor
  y[s - 1] /= u0[s - 1];
  if (s >= 2) y[s - 2] = (y[s - 2] - u1[s - 2] * y[s - 1]) / u0[s - 2];
  for (int i = s - 3; i >= 0; --i) y[i] = (y[i] - u1[i] * y[i + 1] - u2[i] * y[i + 2]) / u0[i];
}

// One WARP per cluster: lane 0 factors T - lam I and runs the (sequential)
// tridiagonal solves; the Gram-Schmidt against earlier cluster members and the
// normalisation are warp-parallel.  Factor and vector live in shared memory
// (5 s doubles + s ints per warp); the pivots are stored as reciprocals so the
// solves' dependency chains carry no division.
__global__ void __launch_bounds__(256) invit_kernel(int s, const double* __restrict__ d, const double* __restrict__ e,
                                                    const double* __restrict__ w, const int* __restrict__ cl_start,
                                                    const int* __restrict__ ncl, double* __restrict__ Y,
                                                    double* __restrict__ scratch) {
  extern __shared__ double ism[];
  (void)scratch;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= *ncl) return;
  double tn = 0.0;
  for (int i = 0; i < s; ++i) tn = fmax(tn, fabs(d[i]) + (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < s ? fabs(e[i]) : 0.0));
  const double eps_t = fmax(2.2e-16 * tn, 1e-300);
  double* u0 = ism + (size_t)warp * (5 * s + (s + 1) / 2 + 1);
  double* u1 = u0 + s;
  double* u2 = u1 + s;
  double* l = u2 + s;
  double* y = l + s;
  int* piv = reinterpret_cast<int*>(y + s);
  const int j0 = cl_start[c], j1 = cl_start[c + 1];
  for (int j = j0; j < j1; ++j) {
    if (lane == 0) {
      tri_factor(s, d, e, w[j], eps_t, u0, u1, u2, l, piv);
      for (int i = 0; i < s; ++i) u0[i] = 1.0 / u0[i];
    }
    // deterministic pseudo-random start (LAPACK uses a random vector too)
    for (int i = lane; i < s; i += 32) {
      unsigned long long hsh = 0x9E3779B97F4A7C15ull * (unsigned long long)(j + 1) + 0xD1B54A32D192ED03ull * (i + 1);
      hsh ^= hsh >> 29;
      hsh *= 0xBF58476D1CE4E5B9ull;
      hsh ^= hsh >> 32;
      y[i] = ((double)(hsh >> 11) * (1.0 / 9007199254740992.0)) - 0.5;
    }
    __syncwarp();
    for (int it = 0; it < 3; ++it) {
      if (lane == 0) {
        // forward: row interchanges and multipliers
        double yi = y[0];
        for (int i = 0; i < s - 1; ++i) {
          const double yn = y[i + 1];
          if (piv[i]) {
            y[i] = yn;
            yi = fma(-l[i], yn, yi);
          } else {
            y[i] = yi;
            yi = fma(-l[i], yi, yn);
          }
        }
        y[s - 1] = yi;
        // back substitution with the 3-diagonal upper factor (u0 holds 1/u0)
        double y2 = y[s - 1] * u0[s - 1];
        y[s - 1] = y2;
        double y1 = y2;
        if (s >= 2) {
          y1 = (y[s - 2] - u1[s - 2] * y2) * u0[s - 2];
          y[s - 2] = y1;
        }
        for (int i = s - 3; i >= 0; --i) {
          const double yi0 = (y[i] - u1[i] * y1 - u2[i] * y2) * u0[i];
          y[i] = yi0;
          y2 = y1;
          y1 = yi0;
        }
      }
      __syncwarp();
      // orthogonalise against the earlier members of the cluster (MGS)
      for (int q = j0; q < j; ++q) {
        const double* yq = Y + (size_t)q * s;
        double dot = 0.0;
        for (int i = lane; i < s; i += 32) dot = fma(yq[i], y[i], dot);
        dot = warp_sum(dot);
        for (int i = lane; i < s; i += 32) y[i] = fma(-dot, yq[i], y[i]);
        __syncwarp();
      }
      double nrm = 0.0;
      for (int i = lane; i < s; i += 32) nrm = fma(y[i], y[i], nrm);
      nrm = sqrt(warp_sum(nrm));
      const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
      for (int i = lane; i < s; i += 32) y[i] *= inv;
      __syncwarp();
    }
    double* yj = Y + (size_t)j * s;
    for (int i = lane; i < s; i += 32) yj[i] = y[i];
    __syncwarp();
  }
}

// clusters of consecutive (descending) eigenvalues closer than 1e-3 ||T||
__global__ void cluster_kernel(int s, const double* __restrict__ d, const double* __restrict__ e,
                               const double* __restrict__ w, int* __restrict__ cl_start, int* __restrict__ ncl) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double tn = 0.0;
  for (int i = 0; i < s; ++i) tn = fmax(tn, fabs(d[i]) + (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < s ? fabs(e[i]) : 0.0));
  // closer than this, independent inverse iterations could converge to the
  // same vector: such eigenvalues are handled together (Gram-Schmidt); wider
  // gaps give orthogonality ~eps ||T|| / gap, polished by one Newton-Schulz step
  const double tol = 1e-6 * tn;
  int c = 0;
  cl_start[0] = 0;
  for (int j = 1; j < s; ++j)
    if (w[j - 1] - w[j] > tol) cl_start[++c] = j;
  cl_start[++c] = s;
  *ncl = c;
}

// --------------------------------------------------------------- K_d ------
// z = H_0 H_1 ... H_{s-3} y  (one warp per vector, the vector in registers:
// lane owns rows lane + 32 m), written as column j of V; the reflectors are
// read row-wise (coalesced) from VhT
constexpr int kBtMR = kTriMaxS / 32;
__global__ void __launch_bounds__(256) backtransform_kernel(int s, const double* __restrict__ VhT,
                                                            const double* __restrict__ tau,
                                                            const double* __restrict__ Y, double* __restrict__ V) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j = blockIdx.x * 8 + warp;
  if (j >= s) return;
  double y[kBtMR];
#pragma unroll
  for (int m = 0; m < kBtMR; ++m) {
    const int i = lane + 32 * m;
    y[m] = i < s ? Y[(size_t)j * s + i] : 0.0;
  }
  // software pipeline: the next reflector's entries are loaded while the
  // current one is applied
  double vn[kBtMR];
  auto load = [&](int k, double (&v)[kBtMR]) {
    const double* vk = VhT + (size_t)k * s;
#pragma unroll
    for (int m = 0; m < kBtMR; ++m) {
      const int i = lane + 32 * m;
      v[m] = (i > k && i < s) ? vk[i] : 0.0;
    }
  };
  if (s >= 3) load(s - 3, vn);
  for (int k = s - 3; k >= 0; --k) {
    double vr[kBtMR];
#pragma unroll
    for (int m = 0; m < kBtMR; ++m) vr[m] = vn[m];
    if (k > 0) load(k - 1, vn);
    const double tk = tau[k];
    double dot = 0.0;
#pragma unroll
    for (int m = 0; m < kBtMR; ++m) dot = fma(vr[m], y[m], dot);
    dot = warp_sum(dot) * tk;
#pragma unroll
    for (int m = 0; m < kBtMR; ++m) y[m] = fma(-dot, vr[m], y[m]);
  }
#pragma unroll
  for (int m = 0; m < kBtMR; ++m) {
    const int i = lane + 32 * m;
    if (i < s) V[(size_t)i * s + j] = y[m];
  }
}

int gemm(int ta, int tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
         const double* B, int64_t ldb, double beta, double* C, int64_t ldc, void* ws, size_t ws_bytes,
         cudaStream_t st);
size_t gemm_ws(int64_t M, int64_t N, int64_t K);

size_t eig_tri_ws(int s) {
  return (size_t)s * s * sizeof(double) * 4 + (size_t)s * 6 * s * sizeof(double) + 8 * (size_t)s * sizeof(double) +
         (size_t)(s + 2) * sizeof(int) * 2 + gemm_ws(s, s, s) + 8192;
}

int eig_tri(int s, const double* A, double* V, double* w, void* ws, cudaStream_t st) {
  char* base = reinterpret_cast<char*>(ws);
  double* Vh = reinterpret_cast<double*>(base);
  double* Y = Vh + (size_t)s * s;
  double* Y2 = Y + (size_t)s * s;
  double* G = Y2 + (size_t)s * s;
  double* scratch = G + (size_t)s * s;
  double* d = scratch + (size_t)s * 6 * s;
  double* e = d + s + 1;
  double* tau = e + s + 1;
  int* cl = reinterpret_cast<int*>(tau + s + 1);
  int* ncl = cl + s + 2;
  void* gws = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(ncl + 4) + 511) & ~uintptr_t(255));
  const size_t smem = ((size_t)s * (s | 1) + (2 + kTriRG) * (size_t)s + 192) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tridiag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    attr = true;
  }
  static const bool fused = !dev_env("NYS_TRI_FUSED") || atoi(dev_env("NYS_TRI_FUSED")) != 0;
  if (fused) {
    static bool fattr = false;
    if (!fattr) {
      cudaFuncSetAttribute(tridiag_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
      fattr = true;
    }
    tridiag_fused_kernel<<<1, kTriThreads, ((size_t)s * (s | 1) + 4 * (size_t)s) * sizeof(double), st>>>(
        s, A, d, e, Vh, tau);
  } else {
    tridiag_kernel<<<1, kTriThreads, smem, st>>>(s, A, d, e, Vh, tau);
  }
  NYS_CHECK_LAUNCH();
  bisect_kernel<<<(unsigned)s, 32, 2 * s * sizeof(double), st>>>(s, d, e, w);
  NYS_CHECK_LAUNCH();
  cluster_kernel<<<1, 32, 0, st>>>(s, d, e, w, cl, ncl);
  NYS_CHECK_LAUNCH();
  // one warp per potential cluster (at most s); idle warps exit
  {
    const size_t ism = 8 * (5 * (size_t)s + (s + 1) / 2 + 1) * sizeof(double);
    static bool iattr = false;
    if (!iattr) {
      cudaFuncSetAttribute(invit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * (5 * kTriMaxS + 82) * 8);
      iattr = true;
    }
    invit_kernel<<<(unsigned)cdiv(s, 8), 256, ism, st>>>(s, d, e, w, cl, ncl, Y, scratch);
  }
  NYS_CHECK_LAUNCH();
  // one Newton-Schulz step Y <- 1.5 Y - 0.5 (Y Y^T) Y (rows of Y are the vectors)
  int rc = gemm(0, 1, s, s, s, 1.0, Y, s, Y, s, 0.0, G, s, gws, gemm_ws(s, s, s), st);
  if (rc) return rc;
  if (cudaMemcpyAsync(Y2, Y, (size_t)s * s * sizeof(double), cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return NYS_ERR_CUDA;
  rc = gemm(0, 0, s, s, s, -0.5, G, s, Y, s, 1.5, Y2, s, gws, gemm_ws(s, s, s), st);
  if (rc) return rc;
  backtransform_kernel<<<(unsigned)cdiv(s, 8), 256, 0, st>>>(s, Vh, tau, Y2, V);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

}  // namespace nys
