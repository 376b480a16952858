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
constexpr int kTriThreads = 1024;

// --------------------------------------------------------------- K_a ------
__global__ void __launch_bounds__(kTriThreads)
tridiag_kernel(int s, const double* __restrict__ A, double* __restrict__ d, double* __restrict__ e,
               double* __restrict__ Vh, double* __restrict__ tau) {
  extern __shared__ double sm[];
  const int ld = s | 1;
  double* a = sm;                         // s x ld
  double* vs = a + (size_t)s * ld;        // s
  double* pw = vs + s;                    // s   (p, then w)
  double* red = pw + s;                   // 32
  __shared__ double sc_beta, sc_tau, sc_scal, sc_pv;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int t = tid; t < s * s; t += blockDim.x) {
    const int i = t / s, j = t - i * s;
    a[i * ld + j] = A[t];
  }
  __syncthreads();
  for (int k = 0; k + 2 < s; ++k) {
    const int m = s - k - 1;  // size of the trailing block
    // ||x(2:)||^2 of x = a[k+1:, k]
    double part = 0.0;
    for (int i = k + 2 + tid; i < s; i += blockDim.x) part = fma(a[i * ld + k], a[i * ld + k], part);
    part = warp_sum(part);
    if (lane == 0) red[warp] = part;
    __syncthreads();
    if (tid == 0) {
      double xn2 = 0.0;
      for (int q = 0; q < nw; ++q) xn2 += red[q];
      const double alpha = a[(k + 1) * ld + k];
      if (xn2 == 0.0) {
        sc_tau = 0.0;
        sc_beta = alpha;
        sc_scal = 0.0;
      } else {
        const double beta = -copysign(sqrt(fma(alpha, alpha, xn2)), alpha);
        sc_tau = (beta - alpha) / beta;
        sc_scal = 1.0 / (alpha - beta);
        sc_beta = beta;
      }
      tau[k] = sc_tau;
      e[k] = sc_beta;
    }
    __syncthreads();
    const double tk = sc_tau;
    for (int i = tid; i < m; i += blockDim.x) {
      const double vi = (i == 0) ? 1.0 : a[(k + 1 + i) * ld + k] * sc_scal;
      vs[i] = vi;
      Vh[(size_t)(k + 1 + i) * s + k] = vi;
    }
    __syncthreads();
    if (tk == 0.0) continue;  // x(2:) == 0: H = I, nothing to update
    // p = tau A22 v   (warp per row, lanes over columns)
    for (int i = warp; i < m; i += nw) {
      const double* ar = a + (k + 1 + i) * ld + (k + 1);
      double acc = 0.0;
      for (int j = lane; j < m; j += 32) acc = fma(ar[j], vs[j], acc);
      acc = warp_sum(acc);
      if (lane == 0) pw[i] = tk * acc;
    }
    __syncthreads();
    // pv = p . v ;  w = p - (tau/2)(p . v) v
    part = 0.0;
    for (int i = tid; i < m; i += blockDim.x) part = fma(pw[i], vs[i], part);
    part = warp_sum(part);
    if (lane == 0) red[warp] = part;
    __syncthreads();
    if (tid == 0) {
      double pv = 0.0;
      for (int q = 0; q < nw; ++q) pv += red[q];
      sc_pv = pv;
    }
    __syncthreads();
    const double hpv = 0.5 * tk * sc_pv;
    for (int i = tid; i < m; i += blockDim.x) pw[i] = fma(-hpv, vs[i], pw[i]);
    __syncthreads();
    // A22 -= v w^T + w v^T
    for (int i = warp; i < m; i += nw) {
      double* ar = a + (k + 1 + i) * ld + (k + 1);
      const double vi = vs[i], wi = pw[i];
      for (int j = lane; j < m; j += 32) ar[j] -= fma(vi, pw[j], wi * vs[j]);
    }
    __syncthreads();
  }
  for (int i = tid; i < s; i += blockDim.x) d[i] = a[i * ld + i];
  if (tid == 0 && s >= 2) e[s - 2] = a[(s - 1) * ld + (s - 2)];
  if (tid == 0 && s >= 1) e[s - 1] = 0.0;
}

// --------------------------------------------------------------- K_b ------
__device__ __forceinline__ int sturm_count(int s, const double* __restrict__ d, const double* __restrict__ e,
                                           double x, double pivmin) {
  // number of eigenvalues of T strictly below x (LDL^T inertia)
  int c = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  c += (q < 0.0);
  for (int i = 1; i < s; ++i) {
    q = d[i] - x - e[i - 1] * e[i - 1] / q;
    if (fabs(q) < pivmin) q = -pivmin;
    c += (q < 0.0);
  }
  return c;
}

// warp w finds the w-th LARGEST eigenvalue
__global__ void __launch_bounds__(256) bisect_kernel(int s, const double* __restrict__ d,
                                                     const double* __restrict__ e, double* __restrict__ w) {
  const int lane = threadIdx.x & 31;
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (j >= s) return;
  // Gershgorin interval and pivot guard (LAPACK dstebz conventions)
  double lo = INFINITY, hi = -INFINITY, emax2 = 0.0;
  for (int i = 0; i < s; ++i) {
    const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < s ? fabs(e[i]) : 0.0);
    lo = fmin(lo, d[i] - r);
    hi = fmax(hi, d[i] + r);
    if (i + 1 < s) emax2 = fmax(emax2, e[i] * e[i]);
  }
  const double pivmin = 2.2250738585072014e-308 * fmax(1.0, emax2);
  const double tnorm = fmax(fabs(lo), fabs(hi));
  lo -= 2.2e-16 * tnorm * s + pivmin;
  hi += 2.2e-16 * tnorm * s + pivmin;
  const int t = s - 1 - j;  // ascending index
  double a = lo, b = hi;
  for (int it = 0; it < 16; ++it) {
    const double x = a + (b - a) * (double)(lane + 1) / 33.0;
    const int c = sturm_count(s, d, e, x, pivmin);
    const unsigned above = __ballot_sync(0xffffffffu, c > t);  // lanes whose point is above lambda_t
    if (above == 0u) {
      a = a + (b - a) * 32.0 / 33.0;
    } else {
      const int f = __ffs(above) - 1;
      const double nb = a + (b - a) * (double)(f + 1) / 33.0;
      const double na = f == 0 ? a : a + (b - a) * (double)f / 33.0;
      a = na;
      b = nb;
    }
    if (b - a <= 2.2e-16 * fmax(fabs(a), fabs(b)) + pivmin) break;
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
// normalisation are warp-parallel.  The vector lives in global scratch.
__global__ void invit_kernel(int s, const double* __restrict__ d, const double* __restrict__ e,
                             const double* __restrict__ w, const int* __restrict__ cl_start,
                             const int* __restrict__ ncl, double* __restrict__ Y, double* __restrict__ scratch) {
  const int lane = threadIdx.x & 31;
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= *ncl) return;
  double tn = 0.0;
  for (int i = 0; i < s; ++i) tn = fmax(tn, fabs(d[i]) + (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < s ? fabs(e[i]) : 0.0));
  const double eps_t = fmax(2.2e-16 * tn, 1e-300);
  double* u0 = scratch + (size_t)c * 6 * s;
  double* u1 = u0 + s;
  double* u2 = u1 + s;
  double* l = u2 + s;
  double* y = l + s;
  int* piv = reinterpret_cast<int*>(y + s);
  const int j0 = cl_start[c], j1 = cl_start[c + 1];
  for (int j = j0; j < j1; ++j) {
    if (lane == 0) tri_factor(s, d, e, w[j], eps_t, u0, u1, u2, l, piv);
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
      if (lane == 0) tri_solve(s, u0, u1, u2, l, piv, y);
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
// z = H_0 H_1 ... H_{s-3} y  (one warp per vector), written as column j of V
__global__ void __launch_bounds__(256) backtransform_kernel(int s, const double* __restrict__ Vh,
                                                            const double* __restrict__ tau,
                                                            const double* __restrict__ Y, double* __restrict__ V) {
  extern __shared__ double ys[];  // 8 warps x s
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j = blockIdx.x * 8 + warp;
  if (j >= s) return;
  double* y = ys + (size_t)warp * s;
  for (int i = lane; i < s; i += 32) y[i] = Y[(size_t)j * s + i];
  __syncwarp();
  for (int k = s - 3; k >= 0; --k) {
    const double tk = tau[k];
    if (tk == 0.0) continue;
    double dot = 0.0;
    for (int i = k + 1 + lane; i < s; i += 32) dot = fma(Vh[(size_t)i * s + k], y[i], dot);
    dot = warp_sum(dot) * tk;
    for (int i = k + 1 + lane; i < s; i += 32) y[i] = fma(-dot, Vh[(size_t)i * s + k], y[i]);
    __syncwarp();
  }
  for (int i = lane; i < s; i += 32) V[(size_t)i * s + j] = y[i];
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
  const size_t smem = ((size_t)s * (s | 1) + 2 * (size_t)s + 32) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tridiag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    attr = true;
  }
  tridiag_kernel<<<1, kTriThreads, smem, st>>>(s, A, d, e, Vh, tau);
  NYS_CHECK_LAUNCH();
  bisect_kernel<<<(unsigned)cdiv(s, 8), 256, 0, st>>>(s, d, e, w);
  NYS_CHECK_LAUNCH();
  cluster_kernel<<<1, 32, 0, st>>>(s, d, e, w, cl, ncl);
  NYS_CHECK_LAUNCH();
  // one warp per potential cluster (at most s); idle warps exit
  invit_kernel<<<(unsigned)cdiv(s, 8), 256, 0, st>>>(s, d, e, w, cl, ncl, Y, scratch);
  NYS_CHECK_LAUNCH();
  // one Newton-Schulz step Y <- 1.5 Y - 0.5 (Y Y^T) Y (rows of Y are the vectors)
  int rc = gemm(0, 1, s, s, s, 1.0, Y, s, Y, s, 0.0, G, s, gws, gemm_ws(s, s, s), st);
  if (rc) return rc;
  if (cudaMemcpyAsync(Y2, Y, (size_t)s * s * sizeof(double), cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return NYS_ERR_CUDA;
  rc = gemm(0, 0, s, s, s, -0.5, G, s, Y, s, 1.5, Y2, s, gws, gemm_ws(s, s, s), st);
  if (rc) return rc;
  backtransform_kernel<<<(unsigned)cdiv(s, 8), 256, 8 * s * sizeof(double), st>>>(s, Vh, tau, Y2, V);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

}  // namespace nys
