// Small symmetric eigensolver for the Nystrom sketch (s <= ~450): the thin SVD
// of B (sketch.py:126) via the eigenpairs of B^T B, and the eigh fallback of
// the sketch core (sketch.py:115).
//
// Block one-sided (Hestenes) Jacobi on ONE thread-block cluster:
//   * the s columns of X = A (and of V = I) are split into 2C blocks of b
//     columns; a round-robin tournament over the blocks gives C disjoint block
//     pairs per round, one per CTA of the cluster;
//   * a CTA pulls its two blocks (X and V columns, ~150 KB) from L2 into
//     shared memory and rotates every cross pair (b sub-rounds of b disjoint
//     column pairs; in the first round of a sweep also the pairs inside each
//     block), one warp per column pair, then writes the blocks back;
//   * ONE cluster barrier per block round: 2C - 1 barriers per sweep instead of
//     the s - 1 grid-wide barriers of a pair-at-a-time parallel Jacobi.
// At convergence X = A V with orthogonal columns: w_p = sign(v_p . x_p) ||x_p||.
#include <cooperative_groups.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include "common.cuh"

namespace cg = cooperative_groups;

namespace nys {

constexpr int kEigThreads = 1024;
constexpr int kEigWarps = kEigThreads / 32;
constexpr int kEigMaxSweeps = 30;

__host__ __device__ __forceinline__ void rr_pair(int k, int t, int m, int& a, int& b) {
  if (k == 0) {
    a = t;
    b = m - 1;
  } else {
    a = (t + k) % (m - 1);
    b = (t - k + (m - 1)) % (m - 1);
  }
  if (a > b) {
    const int tmp = a;
    a = b;
    b = tmp;
  }
}

struct EigGeom {
  int s, C, nb, b;
  size_t smem;
};

static EigGeom eig_geom(int s) {
  EigGeom g;
  g.s = s;
  g.C = 1;
  for (;;) {
    g.nb = 2 * g.C;
    g.b = (int)cdiv(s, g.nb);
    g.smem = (size_t)4 * g.b * s * sizeof(double) + 256;
    if (g.smem <= 200 * 1024 || g.C >= 16) break;
    g.C *= 2;
  }
  return g;
}

// rotate columns (xp, xq) and (vp, vq) of length s if they are not yet
// orthogonal to the tolerance; one warp; returns 1 if it rotated
__device__ __forceinline__ int rotate_pair(double* __restrict__ xp, double* __restrict__ xq,
                                           double* __restrict__ vp, double* __restrict__ vq, int s,
                                           double tol, int lane) {
  double al = 0.0, be = 0.0, ga = 0.0;
  for (int i = lane; i < s; i += 32) {
    const double u = xp[i], v = xq[i];
    al = fma(u, u, al);
    be = fma(v, v, be);
    ga = fma(u, v, ga);
  }
  al = warp_sum(al);
  be = warp_sum(be);
  ga = warp_sum(ga);
  if (!(ga != 0.0 && fabs(ga) > tol * sqrt(al * be))) return 0;
  const double zeta = (be - al) / (2.0 * ga);
  const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
  const double c = 1.0 / sqrt(1.0 + t * t);
  const double sn = c * t;
  if (sn == 0.0) return 0;
  for (int i = lane; i < s; i += 32) {
    const double u = xp[i], v = xq[i];
    xp[i] = c * u - sn * v;
    xq[i] = sn * u + c * v;
    const double vu = vp[i], vv = vq[i];
    vp[i] = c * vu - sn * vv;
    vq[i] = sn * vu + c * vv;
  }
  return 1;
}

// Xg, Vg: nb*b columns of length s, column-major (column c at c*s); padded
// columns are zero and never rotate.
__global__ void __launch_bounds__(kEigThreads)
jacobi_block_kernel(int s, int nb, int b, double* __restrict__ Xg, double* __restrict__ Vg,
                    unsigned int* __restrict__ counts, int* __restrict__ info, double tol) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  extern __shared__ __align__(16) double sm[];
  const size_t blk = (size_t)b * s;
  double* X0 = sm;
  double* X1 = X0 + blk;
  double* V0 = X1 + blk;
  double* V1 = V0 + blk;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ unsigned int nrot;
  __shared__ int stop;
  int sweep = 0;
  for (; sweep < kEigMaxSweeps; ++sweep) {
    if (tid == 0) nrot = 0u;
    for (int t = 0; t < nb - 1; ++t) {
      int pa, pb;
      rr_pair(rank, t, nb, pa, pb);
      // pull the two blocks (X and V) into shared memory
      const double* xa = Xg + (size_t)pa * blk;
      const double* xb = Xg + (size_t)pb * blk;
      const double* va = Vg + (size_t)pa * blk;
      const double* vb = Vg + (size_t)pb * blk;
      for (size_t i = tid; i < blk; i += kEigThreads) {
        X0[i] = xa[i];
        X1[i] = xb[i];
        V0[i] = va[i];
        V1[i] = vb[i];
      }
      __syncthreads();
      unsigned int my = 0;
      if (t == 0) {
        // pairs inside each block (circle method over b columns), both blocks at once
        const int mb = b + (b & 1);
        for (int u = 0; u < mb - 1; ++u) {
          for (int w = warp; w < mb; w += kEigWarps) {  // w < mb/2: block 0, else block 1
            const int k = w % (mb / 2);
            int i, j;
            rr_pair(k, u, mb, i, j);
            if (j >= b) continue;
            double* X = (w < mb / 2) ? X0 : X1;
            double* V = (w < mb / 2) ? V0 : V1;
            my += rotate_pair(X + (size_t)i * s, X + (size_t)j * s, V + (size_t)i * s, V + (size_t)j * s,
                              s, tol, lane);
          }
          __syncthreads();
        }
      }
      // cross pairs: sub-round u pairs column i of block 0 with column (i+u) mod b of block 1
      for (int u = 0; u < b; ++u) {
        for (int i = warp; i < b; i += kEigWarps) {
          const int j = (i + u) % b;
          my += rotate_pair(X0 + (size_t)i * s, X1 + (size_t)j * s, V0 + (size_t)i * s, V1 + (size_t)j * s, s,
                            tol, lane);
        }
        __syncthreads();
      }
      if (lane == 0 && my) atomicAdd(&nrot, my);
      double* ya = Xg + (size_t)pa * blk;
      double* yb = Xg + (size_t)pb * blk;
      double* wa = Vg + (size_t)pa * blk;
      double* wb = Vg + (size_t)pb * blk;
      for (size_t i = tid; i < blk; i += kEigThreads) {
        ya[i] = X0[i];
        yb[i] = X1[i];
        wa[i] = V0[i];
        wb[i] = V1[i];
      }
      __threadfence();
      cluster.sync();
    }
    // convergence: no rotation anywhere in the cluster during this sweep
    __syncthreads();
    if (tid == 0) counts[(sweep & 1) * 16 + rank] = nrot;
    __threadfence();
    cluster.sync();
    if (tid == 0) {
      unsigned int tot = 0;
      for (int j = 0; j < (int)cluster.num_blocks(); ++j) tot += ((volatile unsigned int*)counts)[(sweep & 1) * 16 + j];
      stop = (tot == 0u);
    }
    __syncthreads();
    if (stop) {
      ++sweep;
      break;
    }
  }
  if (rank == 0 && tid == 0) *info = sweep;
}

// ---------------------------------------------------------------------------
// s <= 160: classical two-sided cyclic Jacobi with the whole (padded, m x m)
// matrix in ONE CTA's shared memory.  Rotation parameters come straight from
// (a_pp, a_qq, a_pq) -- no dot products -- and A <- J^T A J for the m/2
// disjoint rotations of a round is an element-parallel update of 2 x 2 blocks.
// Each round costs ~2 CTA barriers.  Rotations are logged and replayed on V.
constexpr int kJ2MaxM = 160;

struct Rot {
  double c, s;
  int p, q;  // the column pair (precomputed: no integer division in the hot loops)
};

__global__ void __launch_bounds__(kEigThreads)
jacobi2_kernel(int s, int m, const double* __restrict__ A, Rot* __restrict__ log, double* __restrict__ diag,
               int* __restrict__ info, double tol) {
  extern __shared__ __align__(16) double a[];  // m x m
  Rot* rot = reinterpret_cast<Rot*>(a + (size_t)m * m);
  __shared__ unsigned int nrot;
  __shared__ int stop;
  const int tid = threadIdx.x;
  const int np = m / 2;
  for (int t = tid; t < m * m; t += blockDim.x) {
    const int i = t / m, j = t - i * m;
    a[t] = (i < s && j < s) ? A[(size_t)i * s + j] : 0.0;
  }
  if (tid == 0) nrot = 0u;
  __syncthreads();
  int sweep = 0;
  for (; sweep < kEigMaxSweeps; ++sweep) {
    for (int t = 0; t < m - 1; ++t) {
      if (tid < np) {
        int p, q;
        rr_pair(tid, t, m, p, q);
        double c = 1.0, sn = 0.0;
        const double apq = a[p * m + q];
        if (q < s && apq != 0.0) {
          const double app = a[p * m + p], aqq = a[q * m + q];
          if (apq * apq > tol * tol * fabs(app * aqq)) {
            // Rutishauser form: t = 2 apq sgn(th) / (|th| + sqrt(th^2 + 4 apq^2)), th = aqq - app
            const double th = aqq - app;
            const double tt = (th >= 0.0 ? 2.0 : -2.0) * apq / (fabs(th) + sqrt(fma(th, th, 4.0 * apq * apq)));
            c = rsqrt(fma(tt, tt, 1.0));
            sn = c * tt;
            if (sn != 0.0) atomicAdd(&nrot, 1u);
          }
        }
        rot[tid] = Rot{c, sn, p, q};
        log[((size_t)sweep * (m - 1) + t) * np + tid] = Rot{c, sn, p, q};
      }
      __syncthreads();
      // A <- J^T A J, one 2 x 2 block (pair ki rows, pair kj columns) per item:
      // warps take block rows, lanes block columns
      for (int ki = tid >> 5; ki < np; ki += kEigWarps) {
        const Rot ri = rot[ki];
        const int pi = ri.p, qi = ri.q;
        for (int kj = tid & 31; kj < np; kj += 32) {
        const Rot rj = rot[kj];
        if (ri.s == 0.0 && rj.s == 0.0) continue;
        const int pj = rj.p, qj = rj.q;
        const double x00 = a[pi * m + pj], x01 = a[pi * m + qj];
        const double x10 = a[qi * m + pj], x11 = a[qi * m + qj];
        // columns: col_p' = c col_p - s col_q, col_q' = s col_p + c col_q
        const double y00 = rj.c * x00 - rj.s * x01, y01 = rj.s * x00 + rj.c * x01;
        const double y10 = rj.c * x10 - rj.s * x11, y11 = rj.s * x10 + rj.c * x11;
        // rows: the same rotation from the left
        double z00 = ri.c * y00 - ri.s * y10, z10 = ri.s * y00 + ri.c * y10;
        double z01 = ri.c * y01 - ri.s * y11, z11 = ri.s * y01 + ri.c * y11;
        if (ki == kj) {  // the annihilated pivot block
          z01 = 0.0;
          z10 = 0.0;
        }
        a[pi * m + pj] = z00;
        a[pi * m + qj] = z01;
        a[qi * m + pj] = z10;
        a[qi * m + qj] = z11;
        }
      }
      __syncthreads();
    }
    if (tid == 0) {
      stop = (nrot == 0u);
      nrot = 0u;
    }
    __syncthreads();
    if (stop) {
      ++sweep;
      break;
    }
  }
  for (int i = tid; i < s; i += blockDim.x) diag[i] = a[i * m + i];
  if (tid == 0) *info = sweep;
}

// Replay the rotation log on rows of V = I.  Each CTA stages chunks of the log
// in shared memory; each warp owns kRowsPerWarp rows of V (also in shared memory).
constexpr int kRowsPerWarp = 4;
constexpr int kLogChunkRounds = 16;
__global__ void __launch_bounds__(256)
jacobi2_v_kernel(int s, int m, const Rot* __restrict__ log, const int* __restrict__ info, double* __restrict__ V) {
  extern __shared__ __align__(16) double vs[];
  const int np = m / 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* rows = vs + (size_t)warp * kRowsPerWarp * m;
  Rot* chunk = reinterpret_cast<Rot*>(vs + (size_t)8 * kRowsPerWarp * m);
  const int row0 = (blockIdx.x * 8 + warp) * kRowsPerWarp;
  for (int j = 0; j < kRowsPerWarp; ++j)
    for (int p = lane; p < m; p += 32) rows[j * m + p] = (row0 + j == p) ? 1.0 : 0.0;
  const size_t nr = (size_t)(*info) * (m - 1);
  for (size_t c0 = 0; c0 < nr; c0 += kLogChunkRounds) {
    const int cr = (int)((nr - c0) < (size_t)kLogChunkRounds ? (nr - c0) : kLogChunkRounds);
    __syncthreads();
    for (int e = threadIdx.x; e < cr * np; e += blockDim.x) chunk[e] = log[c0 * np + e];
    __syncthreads();
    for (int r = 0; r < cr; ++r) {
      for (int k = lane; k < np; k += 32) {
        const Rot ro = chunk[r * np + k];
        if (ro.s == 0.0) continue;
        const int p = ro.p, q = ro.q;
#pragma unroll
        for (int j = 0; j < kRowsPerWarp; ++j) {
          const double u = rows[j * m + p], v = rows[j * m + q];
          rows[j * m + p] = ro.c * u - ro.s * v;
          rows[j * m + q] = ro.s * u + ro.c * v;
        }
      }
      __syncwarp();
    }
  }
  for (int j = 0; j < kRowsPerWarp; ++j) {
    if (row0 + j >= s) break;
    for (int p = lane; p < s; p += 32) V[(size_t)(row0 + j) * s + p] = rows[j * m + p];
  }
}

// eigenvalues = diag, descending rank sort, V (row-major, unsorted columns)
// permuted into the output
__global__ void jacobi2_finish_kernel(int s, const double* __restrict__ diag, const double* __restrict__ Vr,
                                      double* __restrict__ rankbuf, double* __restrict__ V, double* __restrict__ w) {
  for (int p = threadIdx.x; p < s; p += blockDim.x) {
    const double wp = diag[p];
    int rank = 0;
    for (int q = 0; q < s; ++q) {
      const double wq = diag[q];
      rank += (wq > wp) || (wq == wp && q < p);
    }
    rankbuf[p] = (double)rank;
    w[rank] = wp;
  }
  __syncthreads();
  for (int64_t t = threadIdx.x; t < (int64_t)s * s; t += blockDim.x) {
    const int i = (int)(t / s), p = (int)(t % s);
    V[(size_t)i * s + (int)rankbuf[p]] = Vr[t];
  }
}

static size_t jacobi2_ws(int s) {
  const int m = s + (s & 1);
  return (size_t)kEigMaxSweeps * (m - 1) * (m / 2) * sizeof(Rot) + (size_t)s * s * sizeof(double) +
         4 * (size_t)s * sizeof(double) + 4096;
}

static int jacobi2(int s, const double* A, double* V, double* w, void* ws, cudaStream_t st) {
  const int m = s + (s & 1);
  char* base = reinterpret_cast<char*>(ws);
  Rot* log = reinterpret_cast<Rot*>(base);
  double* Vr = reinterpret_cast<double*>(log + (size_t)kEigMaxSweeps * (m - 1) * (m / 2));
  double* diag = Vr + (size_t)s * s;
  double* rankbuf = diag + s + 8;
  int* info = reinterpret_cast<int*>(rankbuf + s + 8);
  const size_t smem = (size_t)m * m * sizeof(double) + (size_t)(m / 2) * sizeof(Rot) + 64;
  const size_t vsmem = (size_t)8 * kRowsPerWarp * m * sizeof(double) + (size_t)kLogChunkRounds * (m / 2) * sizeof(Rot);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(jacobi2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(jacobi2_v_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    attr = true;
  }
  const double tol = fmax(1e-15, (double)s * 2.220446049250313e-16);
  static const bool dbg = dev_env("NYS_EIG_DEBUG") != nullptr;
  cudaEvent_t ev[4];
  if (dbg) {
    for (int i = 0; i < 4; ++i) cudaEventCreate(&ev[i]);
    cudaEventRecord(ev[0], st);
  }
  jacobi2_kernel<<<1, kEigThreads, smem, st>>>(s, m, A, log, diag, info, tol);
  NYS_CHECK_LAUNCH();
  if (dbg) cudaEventRecord(ev[1], st);
  jacobi2_v_kernel<<<(unsigned)cdiv(s, 8 * kRowsPerWarp), 256, vsmem, st>>>(s, m, log, info, Vr);
  NYS_CHECK_LAUNCH();
  if (dbg) cudaEventRecord(ev[2], st);
  jacobi2_finish_kernel<<<1, 1024, 0, st>>>(s, diag, Vr, rankbuf, V, w);
  NYS_CHECK_LAUNCH();
  if (dbg) {
    cudaEventRecord(ev[3], st);
    cudaStreamSynchronize(st);
    float t[3];
    for (int i = 0; i < 3; ++i) cudaEventElapsedTime(&t[i], ev[i], ev[i + 1]);
    int sw = 0;
    cudaMemcpy(&sw, info, sizeof(int), cudaMemcpyDeviceToHost);
    fprintf(stderr, "[eig2] s=%d sweeps=%d a=%.3fms v=%.3fms fin=%.3fms\n", s, sw, t[0], t[1], t[2]);
    for (int i = 0; i < 4; ++i) cudaEventDestroy(ev[i]);
  }
  return NYS_OK;
}

__global__ void jacobi_init_kernel(int s, int ncols, const double* __restrict__ A, double* __restrict__ Xg,
                                   double* __restrict__ Vg) {
  const int64_t tot = (int64_t)ncols * s;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(t / s), i = (int)(t % s);
    // column c of the symmetric A is its row c
    Xg[t] = c < s ? A[(size_t)c * s + i] : 0.0;
    Vg[t] = (c < s && c == i) ? 1.0 : 0.0;
  }
}

// w_p = sign(v_p . x_p) ||x_p||, descending rank sort, V columns permuted
// into the row-major output V[i][rank_p].
__global__ void jacobi_finish_kernel(int s, const double* __restrict__ Xc, const double* __restrict__ Vc,
                                     double* __restrict__ rankbuf, double* __restrict__ V,
                                     double* __restrict__ w) {
  extern __shared__ double wsh[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int p = warp; p < s; p += nw) {
    double nx = 0.0, d = 0.0;
    for (int i = lane; i < s; i += 32) {
      const double x = Xc[(size_t)p * s + i];
      nx = fma(x, x, nx);
      d = fma(Vc[(size_t)p * s + i], x, d);
    }
    nx = warp_sum(nx);
    d = warp_sum(d);
    if (lane == 0) wsh[p] = (d >= 0.0 ? 1.0 : -1.0) * sqrt(nx);
  }
  __syncthreads();
  for (int p = threadIdx.x; p < s; p += blockDim.x) {
    const double wp = wsh[p];
    int rank = 0;
    for (int q = 0; q < s; ++q) {
      const double wq = wsh[q];
      rank += (wq > wp) || (wq == wp && q < p);
    }
    rankbuf[p] = (double)rank;
    w[rank] = wp;
  }
  __syncthreads();
  for (int64_t t = threadIdx.x; t < (int64_t)s * s; t += blockDim.x) {
    const int p = (int)(t / s), i = (int)(t % s);
    V[(size_t)i * s + (int)rankbuf[p]] = Vc[t];
  }
}

size_t eig_tri_ws(int s);
int eig_tri(int s, const double* A, double* V, double* w, void* ws, cudaStream_t st);
// s <= 160: tridiagonal path (eig_tri.cu) unless NYS_EIG=jacobi selects the
// single-CTA two-sided Jacobi (kept for cross-checking)
static bool use_jacobi_small() {
  static const bool j = dev_env("NYS_EIG") && dev_env("NYS_EIG")[0] == 'j';
  return j;
}

size_t syevj_ws(int s) {
  if (s <= kJ2MaxM) return tmax(jacobi2_ws(s), eig_tri_ws(s));
  const EigGeom g = eig_geom(s);
  return 2 * (size_t)g.nb * g.b * s * sizeof(double) + 2 * (size_t)s * sizeof(double) + 4096;
}

// Eigen-decomposition of the symmetric s x s matrix A (row-major, preserved):
// V columns are eigenvectors, w descending.
int syevj(int s, double* A, double* V, double* w, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (ws_bytes < syevj_ws(s)) return NYS_ERR_WORKSPACE;
  if (s <= kJ2MaxM) return use_jacobi_small() ? jacobi2(s, A, V, w, ws, st) : eig_tri(s, A, V, w, ws, st);
  const EigGeom g = eig_geom(s);
  if (g.smem > 210 * 1024) return NYS_ERR_UNSUPPORTED;
  const int ncols = g.nb * g.b;
  char* base = reinterpret_cast<char*>(ws);
  double* Xg = reinterpret_cast<double*>(base);
  double* Vg = Xg + (size_t)ncols * s;
  double* rankbuf = Vg + (size_t)ncols * s;
  unsigned int* counts = reinterpret_cast<unsigned int*>(rankbuf + s + 8);
  int* info = reinterpret_cast<int*>(counts + 64);

  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(jacobi_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    cudaFuncSetAttribute(jacobi_block_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  jacobi_init_kernel<<<(unsigned)tmin<int64_t>(cdiv((int64_t)ncols * s, 256), 1024), 256, 0, st>>>(s, ncols, A,
                                                                                                   Xg, Vg);
  NYS_CHECK_LAUNCH();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(g.C, 1, 1);
  cfg.blockDim = dim3(kEigThreads, 1, 1);
  cfg.dynamicSmemBytes = g.smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = g.C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  // roundoff floor of gamma / sqrt(alpha beta) for s-term dot products
  const double tol = fmax(1e-15, (double)s * 2.220446049250313e-16);
  static const bool dbg = dev_env("NYS_EIG_DEBUG") != nullptr;
  cudaEvent_t e0, e1;
  if (dbg) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
  }
  if (cudaLaunchKernelEx(&cfg, jacobi_block_kernel, s, g.nb, g.b, Xg, Vg, counts, info, tol) != cudaSuccess)
    return NYS_ERR_CUDA;
  __atomic_fetch_add(&g_launches, 1ull, __ATOMIC_RELAXED);
  if (dbg) {
    cudaEventRecord(e1, st);
    cudaStreamSynchronize(st);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    int sw = 0;
    cudaMemcpy(&sw, info, sizeof(int), cudaMemcpyDeviceToHost);
    fprintf(stderr, "[eig] s=%d C=%d b=%d sweeps=%d jacobi=%.3fms\n", s, g.C, g.b, sw, ms);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  jacobi_finish_kernel<<<1, 1024, s * sizeof(double), st>>>(s, Xg, Vg, rankbuf, V, w);
  NYS_CHECK_LAUNCH();
  return NYS_OK;
}

}  // namespace nys
