// Sparse (CSR) data operators and the vector kernels of the general-operator
// engine (QPs with an arbitrary constraint map M, structured / sparse P, sparse
// ML data).  Reference: SparseOperator (operators.py:121-135), DiagonalOperator,
// DiagPlusLowRank, OnesRowOperator, StackedOperator (operators.py:89-203) and
// the M != I branches of admm.py (compute_residuals :215-224, x_update
// :243-275, check_infeasibility :361-415) with prox.py:96-144.
//
// SpMV is HBM-bound on the (value, column) stream: 12 B per nonzero plus the
// gathered x (L2-resident for the feature counts of the paper's data).  A
// group of G lanes (a power of two matched to the mean row length) owns one
// row, so short rows do not leave 31 of 32 lanes idle; the group's partial sums
// combine by a shuffle tree -- fixed order, no atomics, deterministic.
//
// A^T u runs as a second CSR SpMV over the transpose, built ONCE on the device
// by a deterministic counting transpose (no sort, no floating-point atomics):
// per chunk of rows a column histogram, an exclusive scan over chunks per column
// and over columns, then each chunk's warp walks its rows in order and places
// entries behind per-(chunk, column) cursors -- entries of a transposed row come
// out sorted by original row, independent of scheduling.
#include <math.h>
#include "common.cuh"

namespace nys {

constexpr int kGThreads = 256;
constexpr int kGMaxBlocks = kNumSMs * 4;
constexpr int kGRedPartials = 4096;  // layout shared with the other kernels' workspace
inline double* g_part(void* ws) { return reinterpret_cast<double*>(ws); }
inline unsigned int* g_counter(void* ws) {
  return reinterpret_cast<unsigned int*>(reinterpret_cast<double*>(ws) + kGRedPartials * 16);
}
inline unsigned g_blocks(int64_t n) {
  return (unsigned)tmax<int64_t>(1, tmin<int64_t>(cdiv(n, kGThreads), kGMaxBlocks));
}

// NS sums then NM maxima per block; the last block combines the block partials
// in block order (one thread per value) and writes out[0..NS+NM).
template <int NS, int NM>
__device__ __forceinline__ void g_reduce(double (&s)[NS + NM], double* part, unsigned int* counter, double* out) {
  constexpr int NV = NS + NM;
  __shared__ double sh[32 * NV];
  double a[NS > 0 ? NS : 1], b[NM > 0 ? NM : 1];
#pragma unroll
  for (int j = 0; j < NS; ++j) a[j] = s[j];
#pragma unroll
  for (int j = 0; j < NM; ++j) b[j] = s[NS + j];
  if (NS > 0) block_sum<(NS > 0 ? NS : 1)>(a, sh);
  if (NM > 0) block_max<(NM > 0 ? NM : 1)>(b, sh);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < NS; ++j) part[blockIdx.x * NV + j] = a[j];
#pragma unroll
    for (int j = 0; j < NM; ++j) part[blockIdx.x * NV + NS + j] = b[j];
  }
  if (last_block(counter)) {
    if (threadIdx.x < NV) {
      const int j = threadIdx.x;
      double acc = 0.0;
      for (unsigned q = 0; q < gridDim.x; ++q) {
        const double v = part[q * NV + j];
        acc = j < NS ? acc + v : fmax(acc, v);
      }
      out[j] = acc;
    }
  }
}

// ------------------------------------------------------------ CSR SpMV ----
// y_i = alpha * s_i * (a_i . x) + beta * zin_i   (s = dscale or 1; beta == 0
// ignores zin, which may alias y)
template <int G>
__global__ void __launch_bounds__(kGThreads)
csr_spmv_kernel(int64_t rows, const int64_t* __restrict__ rowptr, const int* __restrict__ col,
                const double* __restrict__ val, const double* __restrict__ x, double alpha,
                const double* __restrict__ dscale, double beta, const double* zin, double* y) {
  const int sub = threadIdx.x & (G - 1);
  const int64_t groups = (int64_t)gridDim.x * (kGThreads / G);
  const int64_t gid = ((int64_t)blockIdx.x * kGThreads + threadIdx.x) / G;
  // every thread runs the same number of passes (the group shuffles need whole warps)
  for (int64_t r0 = 0; r0 < rows; r0 += groups) {
    const int64_t row = r0 + gid;
    double acc = 0.0;
    if (row < rows) {
      const int64_t p1 = rowptr[row + 1];
      for (int64_t p = rowptr[row] + sub; p < p1; p += G) acc = fma(val[p], __ldg(x + col[p]), acc);
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, G);
    if (sub == 0 && row < rows) {
      double t = dscale ? acc * dscale[row] : acc;
      t = alpha * t;
      y[row] = beta == 0.0 ? t : __dadd_rn(t, beta * zin[row]);
    }
  }
}

// Y[i, :] = s_i * sum_p val_p X[col_p, :]  (X, Y row-major with s columns): one
// warp per row, lanes over the columns -- the multi-column form the sketch uses
__global__ void __launch_bounds__(kGThreads)
csr_spmm_kernel(int64_t rows, const int64_t* __restrict__ rowptr, const int* __restrict__ col,
                const double* __restrict__ val, const double* __restrict__ X, int64_t ldx, int s,
                const double* __restrict__ dscale, double* __restrict__ Y, int64_t ldy) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (kGThreads / 32);
  for (int64_t row = ((int64_t)blockIdx.x * kGThreads + threadIdx.x) / 32; row < rows; row += warps) {
    const int64_t p0 = rowptr[row], p1 = rowptr[row + 1];
    const double sc = dscale ? dscale[row] : 1.0;
    for (int c0 = 0; c0 < s; c0 += 128) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int64_t p = p0; p < p1; ++p) {
        const double v = val[p];
        const double* xr = X + (int64_t)col[p] * ldx;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int c = c0 + lane + 32 * t;
          if (c < s) acc[t] = fma(v, xr[c], acc[t]);
        }
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int c = c0 + lane + 32 * t;
        if (c < s) Y[row * ldy + c] = dscale ? acc[t] * sc : acc[t];
      }
    }
  }
}

// ------------------------------------------------------- CSR transpose ----
__global__ void csr_count_kernel(int64_t rows, int64_t cols, int64_t chunk_rows, const int64_t* __restrict__ rowptr,
                                 const int* __restrict__ col, int* __restrict__ cnt) {
  const int64_t c = blockIdx.x;
  const int64_t r0 = c * chunk_rows, r1 = tmin<int64_t>(rows, r0 + chunk_rows);
  if (r0 >= r1) return;
  int* my = cnt + c * cols;
  for (int64_t p = rowptr[r0] + threadIdx.x; p < rowptr[r1]; p += blockDim.x) atomicAdd(my + col[p], 1);
}

// per column: exclusive scan of the chunk counts (in place) and the column total
__global__ void csr_colscan_kernel(int64_t cols, int chunks, int* __restrict__ cnt, int64_t* __restrict__ total) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < cols; j += (int64_t)gridDim.x * blockDim.x) {
    int64_t run = 0;
    for (int c = 0; c < chunks; ++c) {
      const int t = cnt[(int64_t)c * cols + j];
      cnt[(int64_t)c * cols + j] = (int)run;
      run += t;
    }
    total[j] = run;
  }
}

// exclusive scan of the column totals into the transpose's row pointer (one CTA)
__global__ void csr_ptrscan_kernel(int64_t cols, const int64_t* __restrict__ total, int64_t* __restrict__ tptr) {
  __shared__ int64_t sh[1024];
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < cols; base += 1024) {
    const int64_t j = base + threadIdx.x;
    const int64_t v = j < cols ? total[j] : 0;
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {  // Hillis-Steele inclusive scan
      const int64_t t = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
      __syncthreads();
      sh[threadIdx.x] += t;
      __syncthreads();
    }
    if (j < cols) tptr[j] = carry + sh[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += sh[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) tptr[cols] = carry;
}

// one warp per chunk: rows in order, entries behind the chunk's column cursors
__global__ void csr_fill_kernel(int64_t rows, int64_t cols, int64_t chunk_rows, int chunks,
                                const int64_t* __restrict__ rowptr, const int* __restrict__ col,
                                const double* __restrict__ val, const int64_t* __restrict__ tptr, int* cnt,
                                int* __restrict__ tcol, double* __restrict__ tval) {
  const int lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (c >= chunks) return;
  const int64_t r0 = c * chunk_rows, r1 = tmin<int64_t>(rows, r0 + chunk_rows);
  int* cur = cnt + c * cols;
  for (int64_t r = r0; r < r1; ++r) {
    for (int64_t p = rowptr[r] + lane; p < rowptr[r + 1]; p += 32) {
      const int j = col[p];
      const int64_t pos = tptr[j] + cur[j];
      cur[j] += 1;  // columns are distinct within a row: no two lanes share j
      tcol[pos] = (int)r;
      tval[pos] = val[p];
    }
    __syncwarp();  // this row's cursor updates are visible to the next row's lanes
  }
}

// ------------------------------------------------- general vector kernels --
// y = a * (d o x) + b * y
__global__ void vmul_kernel(int64_t n, double a, const double* __restrict__ d, const double* __restrict__ x, double b,
                            double* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double t = __dmul_rn(a, __dmul_rn(d[i], x[i]));
    y[i] = b == 0.0 ? t : __dadd_rn(t, __dmul_rn(b, y[i]));
  }
}

// y[i] = scale * src[0]  (adjoint of the summing row, operators.py:194-203)
__global__ void bcast_kernel(int64_t n, const double* __restrict__ src, double scale, double* __restrict__ y) {
  const double v = scale * src[0];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = v;
}

// v = x - y (y optional): out[0] = sum v, out[1] = sum v^2, out[2] = max |v|
__global__ void vstats_kernel(int64_t n, const double* __restrict__ x, const double* __restrict__ y, double* out,
                              double* part, unsigned int* counter) {
  double s[3] = {0.0, 0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = y ? __dadd_rn(x[i], -y[i]) : x[i];
    s[0] += v;
    s[1] = fma(v, v, s[1]);
    s[2] = fmax(s[2], fabs(v));
  }
  g_reduce<2, 1>(s, part, counter, out);
}

// dual residual pieces (admm.py:219-222): t = rho Mtu, rd = grad + t;
// out = [sum rd^2, sum t^2, max |rd|, max |t|]
__global__ void gdual_kernel(int64_t n, const double* __restrict__ grad, const double* __restrict__ mtu, double rho,
                             double* out, double* part, unsigned int* counter) {
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double t = __dmul_rn(rho, mtu[i]);
    const double rd = __dadd_rn(grad[i], t);
    s[0] = fma(rd, rd, s[0]);
    s[1] = fma(t, t, s[1]);
    s[2] = fmax(s[2], fabs(rd));
    s[3] = fmax(s[3], fabs(t));
  }
  g_reduce<2, 2>(s, part, counter, out);
}

// l1 / dual-norm pieces (problems.py:308-331): out = [sum |v|, sum (|v| - lambda1)_+^2, max |v|]
__global__ void absstats_kernel(int64_t n, const double* __restrict__ v, double lambda1, double* out, double* part,
                                unsigned int* counter) {
  double s[3] = {0.0, 0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double a = fabs(v[i]);
    const double e = fmax(__dadd_rn(a, -lambda1), 0.0);
    s[0] += a;
    s[1] = fma(e, e, s[1]);
    s[2] = fmax(s[2], a);
  }
  g_reduce<2, 1>(s, part, counter, out);
}

// box certificates (prox.py:96-135):
//   du: out[0] = sum_{du>0} hi du, out[1] = sum_{du<0} lo du, out[2] = #(inf * nonzero) terms
//   md: out[3] = || md - proj_recession(md) ||^2
__global__ void box_cert_kernel(int64_t m, const double* __restrict__ du, const double* __restrict__ md,
                                const double* __restrict__ lo, const double* __restrict__ hi, double* out,
                                double* part, unsigned int* counter) {
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const double l = lo[i], h = hi[i];
    if (du) {
      const double y = du[i];
      if (y > 0.0) {
        if (isinf(h)) s[2] += 1.0; else s[0] = fma(h, y, s[0]);
      } else if (y < 0.0) {
        if (isinf(l)) s[2] += 1.0; else s[1] = fma(l, y, s[1]);
      }
    }
    if (md) {
      const double y = md[i];
      const bool lf = isfinite(l), hf = isfinite(h);
      double p = y;
      if (lf && hf) p = 0.0;
      else if (lf && !hf) p = fmax(y, 0.0);
      else if (!lf && hf) p = fmin(y, 0.0);
      const double e = __dadd_rn(y, -p);
      s[3] = fma(e, e, s[3]);
    }
  }
  g_reduce<4, 0>(s, part, counter, out);
}

// box membership (prox.py:138-144): out = [max(lo - z), max(z - hi), max |z|]
__global__ void box_viol_kernel(int64_t m, const double* __restrict__ z, const double* __restrict__ lo,
                                const double* __restrict__ hi, double* out, double* part, unsigned int* counter) {
  double s[3] = {-INFINITY, -INFINITY, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const double zi = z[i];
    s[0] = fmax(s[0], __dadd_rn(lo[i], -zi));
    s[1] = fmax(s[1], __dadd_rn(zi, -hi[i]));
    s[2] = fmax(s[2], fabs(zi));
  }
  // g_reduce's max starts at 0.0: shift the violation maxima so that a block
  // with no element (or all -inf) cannot raise them above the true value
  __shared__ double shv[32 * 3];
  double a[3] = {s[0], s[1], s[2]};
  block_max<3>(a, shv);
  if (threadIdx.x == 0) {
    part[blockIdx.x * 3 + 0] = a[0];
    part[blockIdx.x * 3 + 1] = a[1];
    part[blockIdx.x * 3 + 2] = a[2];
  }
  if (last_block(counter)) {
    if (threadIdx.x < 3) {
      double acc = threadIdx.x < 2 ? -INFINITY : 0.0;
      for (unsigned q = 0; q < gridDim.x; ++q) acc = fmax(acc, part[q * 3 + threadIdx.x]);
      out[threadIdx.x] = acc;
    }
  }
}

}  // namespace nys

// ------------------------------------------------------------- C ABI ------
using namespace nys;

extern "C" int nys_csr_spmv_f64(int64_t rows, const int64_t* rowptr, const int* col, const double* val,
                                const double* x, double alpha, const double* dscale, double beta, const double* zin,
                                double* y, int group, void* stream) {
  if (rows <= 0 || !rowptr || !x || !y || (beta != 0.0 && !zin)) return NYS_ERR_ARG;
  cudaStream_t st = as_stream(stream);
  const unsigned blocks = (unsigned)tmax<int64_t>(1, tmin<int64_t>(cdiv(rows * group, kGThreads), kNumSMs * 8));
#define NYS_SPMV(G) csr_spmv_kernel<G><<<blocks, kGThreads, 0, st>>>(rows, rowptr, col, val, x, alpha, dscale, beta, zin, y)
  switch (group) {
    case 1: NYS_SPMV(1); break;
    case 2: NYS_SPMV(2); break;
    case 4: NYS_SPMV(4); break;
    case 8: NYS_SPMV(8); break;
    case 16: NYS_SPMV(16); break;
    case 32: NYS_SPMV(32); break;
    default: return NYS_ERR_ARG;
  }
#undef NYS_SPMV
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_csr_spmm_f64(int64_t rows, const int64_t* rowptr, const int* col, const double* val,
                                const double* X, int64_t ldx, int s, const double* dscale, double* Y, int64_t ldy,
                                void* stream) {
  if (rows <= 0 || s < 1 || ldx < s || ldy < s) return NYS_ERR_ARG;
  const unsigned blocks = (unsigned)tmax<int64_t>(1, tmin<int64_t>(cdiv(rows * 32, kGThreads), kNumSMs * 8));
  csr_spmm_kernel<<<blocks, kGThreads, 0, as_stream(stream)>>>(rows, rowptr, col, val, X, ldx, s, dscale, Y, ldy);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

static int64_t transpose_chunks(int64_t rows, int64_t cols) {
  const int64_t cap = tmax<int64_t>(1, ((int64_t)64 << 20) / tmax<int64_t>(cols, 1));  // <= 256 MB of counters
  return tmax<int64_t>(1, tmin<int64_t>(tmin<int64_t>(rows, (int64_t)kNumSMs * 8), cap));
}

extern "C" size_t nys_csr_transpose_workspace(int64_t rows, int64_t cols) {
  if (rows <= 0 || cols <= 0) return 0;
  const int64_t chunks = transpose_chunks(rows, cols);
  return (size_t)chunks * cols * sizeof(int) + (size_t)cols * sizeof(int64_t) + 256;
}

extern "C" int nys_csr_transpose(int64_t rows, int64_t cols, const int64_t* rowptr, const int* col, const double* val,
                                 int64_t* trowptr, int* tcol, double* tval, void* ws, size_t ws_bytes, void* stream) {
  if (rows <= 0 || cols <= 0 || rows > INT32_MAX) return NYS_ERR_ARG;
  if (ws_bytes < nys_csr_transpose_workspace(rows, cols)) return NYS_ERR_WORKSPACE;
  cudaStream_t st = as_stream(stream);
  const int64_t chunks = transpose_chunks(rows, cols);
  const int64_t chunk_rows = cdiv(rows, chunks);
  int* cnt = reinterpret_cast<int*>(ws);
  int64_t* total = reinterpret_cast<int64_t*>(reinterpret_cast<char*>(ws) + (((size_t)chunks * cols * sizeof(int) + 15) & ~(size_t)15));
  if (cudaMemsetAsync(cnt, 0, (size_t)chunks * cols * sizeof(int), st) != cudaSuccess) return NYS_ERR_CUDA;
  csr_count_kernel<<<(unsigned)chunks, 256, 0, st>>>(rows, cols, chunk_rows, rowptr, col, cnt);
  NYS_CHECK_LAUNCH();
  csr_colscan_kernel<<<g_blocks(cols), kGThreads, 0, st>>>(cols, (int)chunks, cnt, total);
  NYS_CHECK_LAUNCH();
  csr_ptrscan_kernel<<<1, 1024, 0, st>>>(cols, total, trowptr);
  NYS_CHECK_LAUNCH();
  csr_fill_kernel<<<(unsigned)cdiv(chunks, 4), 128, 0, st>>>(rows, cols, chunk_rows, (int)chunks, rowptr, col, val,
                                                             trowptr, cnt, tcol, tval);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_vmul_f64(int64_t n, double a, const double* d, const double* x, double b, double* y, void* stream) {
  if (n <= 0) return NYS_ERR_ARG;
  vmul_kernel<<<g_blocks(n), kGThreads, 0, as_stream(stream)>>>(n, a, d, x, b, y);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_bcast_f64(int64_t n, const double* src, double scale, double* y, void* stream) {
  if (n <= 0) return NYS_ERR_ARG;
  bcast_kernel<<<g_blocks(n), kGThreads, 0, as_stream(stream)>>>(n, src, scale, y);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_vstats_f64(int64_t n, const double* x, const double* y, double* out, void* ws, void* stream) {
  if (n <= 0) return NYS_ERR_ARG;
  vstats_kernel<<<g_blocks(n), kGThreads, 0, as_stream(stream)>>>(n, x, y, out, g_part(ws), g_counter(ws));
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_absstats_f64(int64_t n, const double* v, double lambda1, double* out, void* ws, void* stream) {
  if (n <= 0) return NYS_ERR_ARG;
  absstats_kernel<<<g_blocks(n), kGThreads, 0, as_stream(stream)>>>(n, v, lambda1, out, g_part(ws), g_counter(ws));
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_gdual_f64(int64_t n, const double* grad, const double* mtu, double rho, double* out, void* ws,
                             void* stream) {
  if (n <= 0) return NYS_ERR_ARG;
  gdual_kernel<<<g_blocks(n), kGThreads, 0, as_stream(stream)>>>(n, grad, mtu, rho, out, g_part(ws), g_counter(ws));
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_box_cert_f64(int64_t m, const double* du, const double* md, const double* lo, const double* hi,
                                double* out, void* ws, void* stream) {
  if (m <= 0) return NYS_ERR_ARG;
  box_cert_kernel<<<g_blocks(m), kGThreads, 0, as_stream(stream)>>>(m, du, md, lo, hi, out, g_part(ws),
                                                                    g_counter(ws));
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

extern "C" int nys_box_violation_f64(int64_t m, const double* z, const double* lo, const double* hi, double* out,
                                     void* ws, void* stream) {
  if (m <= 0) return NYS_ERR_ARG;
  box_viol_kernel<<<g_blocks(m), kGThreads, 0, as_stream(stream)>>>(m, z, lo, hi, out, g_part(ws), g_counter(ws));
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}
