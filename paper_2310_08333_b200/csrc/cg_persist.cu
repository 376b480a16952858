// The whole PCG solve of one ADMM x-update (krylov.py:35-95) as ONE
// persistent cooperative kernel: one CTA per SM, grid barriers between the
// phases of an iteration, the stopping decision taken on the device.  No
// kernel launches, no predicated no-op launches and no launch gaps inside
// the solve; the host enqueues it once per ADMM iteration.
//
// Iteration k, three grid barriers (every CTA; "slice" = its n / 148 entries):
//   HVP   v = z + beta p (first: v = z) formed in registers (CTA c stores v's
//         slice as the new p); ||p||^2 from the registers; rows of A streamed
//         by TMA bulk copies into a 2-stage ring (csrc/hvp.cu), with
//         sum_i d_i (a_i.p)^2 accumulated on the way   -> barrier
//   STEP  every CTA forms p.Ap = sum_i d_i (a_i.p)^2 + shift ||p||^2 and alpha
//         itself (fixed-order sums of the CTA partials); Ap, x, r of the
//         slice, ||r||^2 and U^T r partials   -> barrier
//         (k % 50 == 0: x only, an HVP of x, r = b - A x)
//   APPLY every CTA runs the stop test and forms the Eq. (11) coefficients
//         itself; z = U coef + r of the slice, r.z partial   -> barrier, beta
// Scalars are recomputed identically by every CTA instead of broadcast by a
// last CTA; CTA 0 publishes them in sc.  All sums are fixed-order, so the
// result is deterministic.
#include <cooperative_groups.h>
#include <stdlib.h>
#include "common.cuh"
#include "tma.cuh"

namespace cg = cooperative_groups;

namespace nys {

constexpr int kCpThreads = 512;
constexpr int kCpWarps = kCpThreads / 32;
constexpr int kCpMaxK = 13;            // n <= 13312
constexpr int kCpMaxSum = (kNumSMs + 31) / 32;  // CTA partials per lane of a fixed-order sum
constexpr int kCpSmemBudget = 226 * 1024;  // sm_100 per-block maximum less the static shared words

struct CgPersistArgs {
  const double* A;
  int64_t rows, n, lda;
  const double* d;
  double shift;
  const double* U;
  int r;
  int64_t ldu;
  const double* lam;
  double nu;
  const double* b;
  double* x;
  double* res;
  double* p[2];
  double* z;
  double* Ap;
  double* sc;
  double tol;
  const double* tolp;
  const double* gate;
  int64_t max_iter;
  double* ypart;   // nctas x n
  double* hpart;   // nctas x r
  double* part;    // nctas x 8
  double* coef;    // r
  unsigned int* counter;
  int W, S;
  int has_head;       // run the ADMM head (nys_admm_head) as the prologue
  int u_smem;         // stage this CTA's rows of U in shared memory
  int qp;                  // operator P v (QP, P symmetric n x n) instead of A^T (d o A v)
  int probe;               // development timing probe (NYS_CP_PROBE)
  int no_early_prefetch;   // development: no speculative first rows before the prologue
  const double* order_in;  // row order of the previous pass over A (NULL: ascending first)
  double* order_out;       // row order of this solve's last pass
  nys_admm_head h;
  // the ADMM tail's relax/prox/dual update and window append, run on each
  // CTA's slice of x once the CG has stopped (nys_admm_head.zu)
  int has_zu;
  struct {
    double* z;
    double* u;
    double* xbar;
    double* zbar;
    double alpha, kappa;
    int prox_kind, accum;
    const double* lo;
    const double* hi;
    double* rx;  // window slot for x (NULL: no append)
    double* ru;  // window slot for u (NULL: none)
  } zu;
};

// Development probe (NYS_CP_PROBE=1): CTA 0 stamps %globaltimer at the phase
// boundaries of every launch and accumulates the deltas (tools/cp_probe.py).
__device__ unsigned long long g_cp_probe_acc[24];
__device__ unsigned long long g_cp_probe_cnt;
__device__ __forceinline__ unsigned long long cp_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// coefficient arrays in shared memory: r rounded up to an even count
__host__ __device__ inline int cp_r2(int r) { return r > 0 ? (r + 1) & ~1 : 2; }

__device__ __forceinline__ double cp_tol(const CgPersistArgs& a) { return a.tolp ? *a.tolp : a.tol; }

// the reference's stop test on ||r||^2 (krylov.py:84-88)
__device__ void cp_stop(double* sc, double res2, double tol, int64_t k, int64_t max_iter) {
  const double b2 = sc[NYS_CG_B2];
  const double denom = b2 > 0.0 ? sqrt(b2) : 1.0;
  const double res = sqrt(res2);
  sc[NYS_CG_RES2] = res2;
  if (!isfinite(res)) {
    sc[NYS_CG_DONE] = 2.0;
    sc[NYS_CG_ITERS] = (double)k;
  } else if (res <= tol * denom) {
    sc[NYS_CG_DONE] = 1.0;
    sc[NYS_CG_ITERS] = (double)k;
  } else if (k >= max_iter) {
    sc[NYS_CG_DONE] = 4.0;
    sc[NYS_CG_ITERS] = (double)k;
  }
  sc[NYS_CG_RESREL] = res / denom;
  if (sc[NYS_CG_DONE] != 0.0) sc[NYS_CG_RUNNING] = 0.0;
}

// block sum of v, valid in every thread (sh: 32 doubles; two barriers)
__device__ __forceinline__ double cp_block_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  return warp_sum(lane < kCpWarps ? sh[lane] : 0.0);
}

template <int K>
__global__ void __launch_bounds__(kCpThreads, 1) cg_persist_kernel(CgPersistArgs a) {
  pdl_begin();  // chain kernel (common.cuh)
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw);                        // S x W
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)a.S * a.W);    // S
  uint64_t* ubar = full + a.S;                                               // U slice arrival
  double* red = reinterpret_cast<double*>(full + ((a.S + 2) & ~1));          // 2 x 16 (16-B aligned)
  double* sh = red + 32;                                                     // 32
  const int r2 = cp_r2(a.r);
  double* csh = sh + 32;                                                     // coef (r <= 512)
  double* lnu = csh + r2;                                                    // lam_j + nu
  double* ys = lnu + r2;                                                     // slice sums
  double* rsl = ys + 112;  // CG residual of the slice: the preconditioner passes read it from here
  double* vrow = rsl + 112;  // QP: the direction at this CTA's rows (p_i of p^T P p)
  double* scr = vrow + 112;                                                  // colsum scratch (1024)
  double* us = scr + 1024;                                                   // U rows of the slice
  __shared__ double s_bcast;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool probe = a.probe && blockIdx.x == 0 && threadIdx.x == 0;
  unsigned long long pt0 = probe ? cp_now() : 0ull, plast = pt0;
  auto stamp = [&](int slot) {
    if (probe) {
      const unsigned long long t = cp_now();
      atomicAdd(&g_cp_probe_acc[slot], t - plast);
      plast = t;
    }
  };
  const int nctas = gridDim.x, cta = blockIdx.x;
  const int64_t n = a.n;
  double* sc = a.sc;
  const bool writer = cta == 0 && tid == 0;  // the one thread that publishes sc
  const int64_t slice = ((n + nctas - 1) / nctas + 1) & ~1ll;
  const int64_t c0 = (int64_t)cta * slice, c1 = tmin<int64_t>(n, c0 + slice);
  // the slice's rows of U go to shared memory asynchronously (LDGSTS); both
  // preconditioner passes read them from there (waited for before the first)
  const bool ush = a.u_smem && a.r > 0;
  // contiguous U rows (ldu == r): one TMA bulk copy of the slice, issued after
  // the gate check; otherwise 8-byte cp.async per element from here
  const unsigned ubytes = (ush && c1 > c0) ? (unsigned)((c1 - c0) * a.r * 8) : 0u;
  const bool utma = ush && a.ldu == a.r && ubytes > 0 && (ubytes & 15) == 0 &&
                    (((uintptr_t)(a.U + c0 * a.r)) & 15) == 0;
  if (ush && !utma) {
    const int tot = (int)(c1 - c0) * a.r;
    for (int t = tid; t < tot; t += kCpThreads) {
      const int ii = t / a.r, j = t - ii * a.r;
      const unsigned dst = (unsigned)__cvta_generic_to_shared(us + t);
      const double* src = a.U + (c0 + ii) * a.ldu + j;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src));
    }
    asm volatile("cp.async.commit_group;\n" ::);
  }
  // z/u step of the ADMM tail on the slice (vec.cu admm_zu_kernel +
  // ring_copy_kernel, admm.py:562-583, 622-623); x of the slice was last
  // written by this thread, so no grid barrier is needed
  auto zu_slice = [&]() {
    if (!a.has_zu) return;
    const auto& q = a.zu;
    const double beta = 1.0 - q.alpha;
    for (int64_t i = c0 + tid; i < c1; i += kCpThreads) {
      const double xi = a.x[i];
      const double w = __dadd_rn(__dmul_rn(q.alpha, xi), __dmul_rn(beta, q.z[i]));
      const double ui = q.u[i];
      const double v = __dadd_rn(w, ui);
      double zn;
      if (q.prox_kind == NYS_PROX_SOFT) {
        const double m = fmax(__dadd_rn(fabs(v), -q.kappa), 0.0);
        zn = v > 0.0 ? m : (v < 0.0 ? -m : 0.0 * m);
      } else {
        zn = fmin(fmax(v, q.lo[i]), q.hi[i]);
      }
      const double un = __dadd_rn(__dadd_rn(ui, w), -zn);
      q.z[i] = zn;
      q.u[i] = un;
      if (q.accum) {
        q.xbar[i] = __dadd_rn(q.xbar[i], xi);
        q.zbar[i] = __dadd_rn(q.zbar[i], zn);
      }
      if (q.rx) q.rx[i] = xi;
      if (q.ru) q.ru[i] = un;
    }
  };
  // ---------------------------------------------------------- begin ----
  // The head's inputs for this thread's element of the slice (slice <= 90 <
  // kCpThreads, so at most one) are requested together with the gate word, so
  // the begin phase costs one memory round trip instead of two.
  const int64_t hi_ = c0 + tid;
  const bool hmine = a.has_head && hi_ < c1;
  double hx_ = 0.0, hz_ = 0.0, hu_ = 0.0, hxb_ = 0.0, hzb_ = 0.0, hhx_ = 0.0, hg_ = 0.0, hq_ = 0.0;
  if (hmine) {
    const nys_admm_head& h = a.h;
    hx_ = h.x[hi_];
    hz_ = h.z[hi_];
    hu_ = h.u[hi_];
    if (h.snap) {
      hxb_ = h.xbar[hi_];
      hzb_ = h.zbar[hi_];
    }
    hhx_ = h.hxA[hi_];
    hg_ = h.gA[hi_];
    if (h.q) hq_ = h.q[hi_];
  }
  {
    const double* gp = a.has_head ? a.h.gate : a.gate;
    if (gp && *gp == 0.0) {  // previous ADMM iteration unfinished: skip the solve
      if (writer) {
        sc[NYS_CG_DONE] = 5.0;
        sc[NYS_CG_ITERS] = 0.0;
        sc[NYS_CG_RUNNING] = 1.0;
      }
      return;
    }
  }
  // Passes over A alternate their row order, starting opposite to the pass
  // before this kernel, so each begins with the rows still in L2; the first
  // rows of a pass are requested before the work that leads up to it (they
  // do not depend on it).  Row q of this CTA in order dir: cta + q' nctas,
  // q' = q (ascending) or m - 1 - q (descending).
  const int64_t nrows_mine = a.rows > cta ? (a.rows - cta + nctas - 1) / nctas : 0;
  const unsigned rbytes = (unsigned)n * 8u;
  int64_t g0 = 0;    // rows consumed so far by this CTA (mbarrier phase bookkeeping)
  int pre_dir = -1;  // order of the next pass whose first rows are in flight
  int last_dir = a.order_in ? (*a.order_in != 0.0 ? 1 : 0) : 1;
  auto row_of = [&](int64_t q, int dir) -> int64_t {
    return cta + (dir ? nrows_mine - 1 - q : q) * nctas;
  };
  auto prefetch = [&](int dir) {
    if (tid == 0)
      for (int64_t q = 0; q < a.S && q < nrows_mine; ++q) {
        const int64_t g = g0 + q;
        const int st = (int)((unsigned)g % (unsigned)a.S);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&full[st], rbytes);
        tma_load_1d(ring + (size_t)st * a.W, a.A + row_of(q, dir) * a.lda, rbytes, &full[st]);
      }
    pre_dir = dir;
  };
  if (tid == 0) {
    for (int q = 0; q < a.S; ++q) mbar_init(&full[q], 1);
    if (utma) mbar_init(ubar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (utma) {
      mbar_expect_tx(ubar, ubytes);
      tma_load_1d(us, a.U + c0 * a.r, ubytes, ubar);
    }
  }
  if (!a.no_early_prefetch) prefetch(last_dir ^ 1);
  // the preconditioner's denominators lam_j + nu, once per launch (make_coef
  // then has no global load on its path)
  for (int j = tid; j < a.r; j += kCpThreads) lnu[j] = __dadd_rn(a.lam[j], a.nu);
  // end of the solve: the speculative first rows of a next pass must land
  // before the CTA exits; record the order of the last pass
  auto finish = [&]() {
    if (tid == 0 && pre_dir >= 0)
      for (int64_t q = 0; q < a.S && q < nrows_mine; ++q) {
        const int64_t g = g0 + q;
        mbar_wait(&full[(unsigned)g % (unsigned)a.S], ((unsigned)g / (unsigned)a.S) & 1u);
      }
    if (writer && a.order_out) *a.order_out = (double)last_dir;
  };
  // every CTA evaluates the begin logic itself (same inputs, same result)
  double tol, b2, res2;
  if (a.has_head) {
    // ADMM head (nys_admm_head_f64) on this CTA's slice: device CG
    // tolerance, snapshot, rhs and r0 = rhs - H x0, ||rhs||^2, ||r0||^2
    const nys_admm_head& h = a.h;
    if (h.tol_fixed > 0.0) {
      tol = h.tol_fixed;
    } else {  // krylov.py:98-112 from the residual norms of the previous iteration
      const double* q = h.prev;
      const double rp = h.norm_kind ? q[1] : sqrt(fmax(q[0], 0.0));
      const double rd = h.norm_kind ? q[3] : sqrt(fmax(q[2], 0.0));
      tol = fmax(fmin(sqrt(rp * rd), 1.0) / h.kpow, 1e-12);
    }
    if (writer) {
      if (h.gate_next) *h.gate_next = 0.0;
      if (h.tol_out) *h.tol_out = tol;
    }
    double sb = 0.0, sr = 0.0;
    if (hmine) {
      const int64_t i = hi_;
      const double xi = hx_, zi = hz_, ui = hu_;
      if (h.snap) {
        h.snap[i] = xi;
        h.snap[n + i] = zi;
        h.snap[2 * n + i] = ui;
        h.snap[3 * n + i] = hxb_;
        h.snap[4 * n + i] = hzb_;
      }
      const double l2x = __dmul_rn(h.lambda2, xi);
      const double hx = __dadd_rn(hhx_, l2x);
      double g = __dadd_rn(hg_, l2x);
      if (h.q) g = __dadd_rn(g, hq_);
      double bb = __dadd_rn(__dadd_rn(hx, __dmul_rn(h.sigma, xi)), -g);
      bb = __dadd_rn(bb, __dmul_rn(h.rho, __dadd_rn(zi, -ui)));
      const double ri = __dadd_rn(bb, -__dadd_rn(hx, __dmul_rn(h.shift, xi)));
      h.rhs[i] = bb;
      h.r[i] = ri;
      rsl[i - c0] = ri;
      sb = fma(bb, bb, sb);
      sr = fma(ri, ri, sr);
    }
    stamp(13);  // head loop
    sb = cp_block_sum(sb, sh);
    sr = cp_block_sum(sr, sh);
    if (tid == 0) {
      a.part[cta * 8 + 4] = sb;
      a.part[cta * 8 + 5] = sr;
    }
  } else {
    tol = cp_tol(a);
    b2 = sc[NYS_CG_B2];
    res2 = sc[NYS_CG_RES2];
    for (int64_t i = c0 + tid; i < c1; i += kCpThreads) rsl[i - c0] = a.res[i];
  }
  __syncthreads();

  // fixed-order sums of two slots in one pass (one round trip)
  __shared__ double s_bcast2;
  auto all_sum2 = [&](int q1, int q2, double& o2) -> double {
    __syncthreads();
    if (warp == 0) {
      double v1[kCpMaxSum], v2[kCpMaxSum];  // every load in flight at once
#pragma unroll
      for (int u = 0; u < kCpMaxSum; ++u) {
        const int c = lane + 32 * u;
        v1[u] = c < nctas ? a.part[c * 8 + q1] : 0.0;
        v2[u] = c < nctas ? a.part[c * 8 + q2] : 0.0;
      }
      double t1 = 0.0, t2 = 0.0;
#pragma unroll
      for (int u = 0; u < kCpMaxSum; ++u)
        if (lane + 32 * u < nctas) {
          t1 += v1[u];
          t2 += v2[u];
        }
      t1 = warp_sum(t1);
      t2 = warp_sum(t2);
      if (lane == 0) {
        s_bcast = t1;
        s_bcast2 = t2;
      }
    }
    __syncthreads();
    o2 = s_bcast2;
    return s_bcast;
  };
  // fixed-order sum over the CTAs of slot q of part (nctas x 8), in every thread
  auto all_sum = [&](int q) -> double {
    __syncthreads();
    if (warp == 0) {
      double v[kCpMaxSum];  // every load in flight at once, summed in CTA order
#pragma unroll
      for (int u = 0; u < kCpMaxSum; ++u) {
        const int c = lane + 32 * u;
        v[u] = c < nctas ? a.part[c * 8 + q] : 0.0;
      }
      double t = 0.0;
#pragma unroll
      for (int u = 0; u < kCpMaxSum; ++u)
        if (lane + 32 * u < nctas) t += v[u];
      t = warp_sum(t);
      if (lane == 0) s_bcast = t;
    }
    __syncthreads();
    return s_bcast;
  };
  // y = A^T (d o A v) for this CTA's rows into ypart[cta]; v in registers.
  // Returns sum_rows d_i (a_i . v)^2 of this CTA's rows (valid in thread 0).
  // The pass runs in the order of the rows already requested (pre_dir) and
  // requests the first rows of the next pass (opposite order) at its end.
  auto hvp_rows = [&](double2 (&vr)[K]) -> double {
    double2 yr[K];
#pragma unroll
    for (int k = 0; k < K; ++k) yr[k] = make_double2(0.0, 0.0);
    double vav = 0.0;
    if (pre_dir < 0) prefetch(last_dir ^ 1);
    const int dir = pre_dir;
    for (int64_t it = 0; it < nrows_mine; ++it) {
      const int64_t g = g0 + it;
      const int st = (int)((unsigned)g % (unsigned)a.S);
      const int64_t i = row_of(it, dir);
      const double di = a.d ? __ldg(a.d + i) : 1.0;
      const double* row = ring + (size_t)st * a.W;
      mbar_wait(&full[st], ((unsigned)g / (unsigned)a.S) & 1u);
      double pt = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int j = 2 * (tid + k * kCpThreads);
        if (j < n) {
          const double2 v2 = *reinterpret_cast<const double2*>(row + j);
          pt = fma(v2.x, vr[k].x, pt);
          pt = fma(v2.y, vr[k].y, pt);
        }
      }
      pt = warp_sum(pt);
      if (lane == 0) red[(it & 1) * 16 + warp] = pt;
      __syncthreads();
      const double tot = warp_sum(lane < kCpWarps ? red[(it & 1) * 16 + lane] : 0.0);
      if (a.qp) {
        // (P v)_i is the row's dot itself: written directly, p^T P p from v_i
        if (tid == 0) {
          a.ypart[i] = tot;
          vav = fma(vrow[dir ? nrows_mine - 1 - it : it], tot, vav);
        }
      } else {
        const double t = a.d ? di * tot : tot;
        if (tid == 0) vav = fma(t, tot, vav);
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int j = 2 * (tid + k * kCpThreads);
          if (j < n) {
            const double2 v2 = *reinterpret_cast<const double2*>(row + j);
            yr[k].x = fma(t, v2.x, yr[k].x);
            yr[k].y = fma(t, v2.y, yr[k].y);
          }
        }
      }
      __syncthreads();
      if (tid == 0 && it + a.S < nrows_mine) {
        const int64_t inext = row_of(it + a.S, dir);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&full[st], rbytes);
        tma_load_1d(ring + (size_t)st * a.W, a.A + inext * a.lda, rbytes, &full[st]);
      }
    }
    g0 += nrows_mine;
    last_dir = dir;
    prefetch(dir ^ 1);
    if (!a.qp) {
      double* yp = a.ypart + (int64_t)cta * n;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int j = 2 * (tid + k * kCpThreads);
        if (j < n) *reinterpret_cast<double2*>(yp + j) = yr[k];
      }
    }
    return vav;
  };
  // out[c] = fixed-order sum over q < cnt of P[q * ld + col0 + c], c < ncols, by
  // all threads: G groups with independent loads in flight, combined in a
  // fixed order through the (idle) ring.  Valid in every thread after the call.
  auto colsum = [&](const double* P, int64_t ld, int cnt, int64_t col0, int ncols, double* out) {
    // G groups of ncols / 2 threads (16-byte loads of column pairs); group g
    // sums the contiguous partials [g per, g per + per) with all of its loads
    // in flight at once (one L2 round trip when per <= 16), then the G group
    // sums are combined in a fixed order through the (idle) scratch.
    const bool pairs = ((ncols | col0 | ld) & 1) == 0 && (((uintptr_t)P) & 15) == 0;
    const int nc = pairs ? ncols / 2 : ncols;  // loaders per group
    const int G = nc > 0 ? tmax(1, tmin(tmin(32, kCpThreads / nc), 1024 / tmax(ncols, 1))) : 1;  // scr: 1024
    const int per = (cnt + G - 1) / G;
    __syncthreads();
    if (tid < G * nc) {
      const int c = tid % nc, g = tid / nc;
      const int q0 = g * per, q1 = tmin(cnt, q0 + per);
      double2 t = make_double2(0.0, 0.0);
      if (pairs && per <= 16) {
        const double* pc = P + col0 + 2 * c;
        double2 v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u)
          v[u] = (q0 + u < q1) ? *reinterpret_cast<const double2*>(pc + (int64_t)(q0 + u) * ld)
                               : make_double2(0.0, 0.0);
#pragma unroll
        for (int w = 8; w >= 1; w >>= 1)  // fixed pairwise tree
#pragma unroll
          for (int u = 0; u < w; ++u) {
            v[u].x += v[u + w].x;
            v[u].y += v[u + w].y;
          }
        t = v[0];
      } else {
        const int col = pairs ? 2 * c : c;
        for (int h = 0; h < (pairs ? 2 : 1); ++h) {
          const double* pc = P + col0 + col + h;
          double sv[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};  // 8 load chains in flight
          int q = q0;
          for (; q + 7 < q1; q += 8) {
#pragma unroll
            for (int u = 0; u < 8; ++u) sv[u] += pc[(int64_t)(q + u) * ld];
          }
          for (; q < q1; ++q) sv[0] += pc[(int64_t)q * ld];
          const double tt = ((sv[0] + sv[1]) + (sv[2] + sv[3])) + ((sv[4] + sv[5]) + (sv[6] + sv[7]));
          if (h == 0) t.x = tt; else t.y = tt;
        }
      }
      if (pairs) {
        scr[g * ncols + 2 * c] = t.x;
        scr[g * ncols + 2 * c + 1] = t.y;
      } else {
        scr[g * ncols + c] = t.x;
      }
    }
    __syncthreads();
    for (int col = tid; col < ncols; col += kCpThreads) {
      double t = 0.0;
      for (int g = 0; g < G; ++g) t += scr[g * ncols + col];
      out[col] = t;
    }
    __syncthreads();
  };
  auto y_slice = [&]() {  // ys = (A^T D A p or P p) on this CTA's column slice
    if (a.qp) {
      __syncthreads();
      for (int64_t i = c0 + tid; i < c1; i += kCpThreads) ys[i - c0] = a.ypart[i];
      __syncthreads();
    } else {
      colsum(a.ypart, n, nctas, c0, (int)(c1 - c0), ys);
    }
  };
  // this CTA's share of h = U^T w over its slice -> hpart[cta]
  // (thread j: four fixed-order chains over the slice's rows; w of the slice
  // was written by this CTA before the last barrier)
  auto utw_slice = [&]() {
    const int64_t len = c1 - c0;
    for (int j = tid; j < a.r; j += kCpThreads) {
      const double* uj = ush ? us + j : a.U + c0 * a.ldu + j;
      const int64_t ld = ush ? a.r : a.ldu;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int64_t q = 0;
      for (; q + 3 < len; q += 4) {
        s0 = fma(uj[q * ld], rsl[q], s0);
        s1 = fma(uj[(q + 1) * ld], rsl[q + 1], s1);
        s2 = fma(uj[(q + 2) * ld], rsl[q + 2], s2);
        s3 = fma(uj[(q + 3) * ld], rsl[q + 3], s3);
      }
      for (; q < len; ++q) s0 = fma(uj[q * ld], rsl[q], s0);
      a.hpart[(int64_t)cta * a.r + j] = (s0 + s1) + (s2 + s3);
    }
  };
  // every CTA: coef_j = (lam_{r-1}+nu)(h_j/(lam_j+nu)) - h_j into shared memory
  auto make_coef = [&]() {
    colsum(a.hpart, a.r, nctas, 0, a.r, csh);  // (its barriers order the lnu writes too)
    const double lr = lnu[a.r - 1];
    for (int j = tid; j < a.r; j += kCpThreads) {
      const double h = csh[j];
      const double head = __dmul_rn(lr, h / lnu[j]);
      csh[j] = __dadd_rn(head, -h);
    }
    __syncthreads();
  };
  // z (slice) = U coef + w (Eq. (11) second pass, coef in shared memory);
  // returns the w.z partial of the slice (every thread)
  auto apply_slice = [&]() -> double {
    double acc = 0.0;
    if (a.r > 0) {
      for (int64_t i = c0 + warp; i < c1; i += kCpWarps) {
        const double* ui = ush ? us + (i - c0) * a.r : a.U + i * a.ldu;
        double s2 = 0.0;
        for (int j = lane; j < a.r; j += 32) s2 = fma(ui[j], csh[j], s2);
        s2 = warp_sum(s2);
        if (lane == 0) {
          const double zi = __dadd_rn(s2, rsl[i - c0]);
          a.z[i] = zi;
          acc = fma(rsl[i - c0], zi, acc);
        }
      }
    } else {
      for (int64_t i = c0 + tid; i < c1; i += kCpThreads) {
        a.z[i] = rsl[i - c0];
        acc = fma(rsl[i - c0], rsl[i - c0], acc);
      }
    }
    return cp_block_sum(acc, sh);
  };

  // ------------------------------- begin + first preconditioning ----
  // (the head's r0 slice and the U^T r0 partials come from the same phase)
  if (utma) mbar_wait(ubar, 0);
  else if (ush) asm volatile("cp.async.wait_all;\n" ::: "memory");
  if (a.r > 0) {
    __syncthreads();
    utw_slice();
  }
  stamp(0);  // head + U^T r0 partials
  if (a.has_head || a.r > 0) grid.sync();
  stamp(1);  // barrier 1
  if (a.has_head) b2 = all_sum2(4, 5, res2);
  {
    const double denom = b2 > 0.0 ? sqrt(b2) : 1.0;
    const double res = sqrt(res2);
    const bool done0 = !isfinite(res) || res <= tol * denom;
    if (writer) {
      if (a.has_head) {
        sc[NYS_CG_B2] = b2;
        sc[NYS_CG_RES2] = res2;
      }
      sc[NYS_CG_DONE] = 0.0;
      sc[NYS_CG_ITERS] = 0.0;
      sc[NYS_CG_RUNNING] = 1.0;
      sc[NYS_CG_NHVP] = 0.0;
      cp_stop(sc, res2, tol, 0, a.max_iter > 0 ? a.max_iter : 1);
      if (sc[NYS_CG_DONE] == 4.0) {
        sc[NYS_CG_DONE] = 0.0;
        sc[NYS_CG_RUNNING] = 1.0;
      }
    }
    if (done0) {
      zu_slice();
      finish();
      return;
    }
  }
  stamp(14);  // all_sum x2 + stop test
  if (a.r > 0) make_coef();
  stamp(15);  // coef (colsum of the U^T r partials)
  {
    const double rz = apply_slice();
    if (tid == 0) a.part[cta * 8 + 0] = rz;
  }
  stamp(2);  // first preconditioner apply
  grid.sync();
  stamp(3);  // barrier 2
  double rz = all_sum(0);
  stamp(19);  // r.z sum
  if (writer) {
    sc[NYS_CG_RZNEW] = rz;
    sc[NYS_CG_RZ] = rz;
  }
  double beta = 0.0;  // first direction: p = z
  int pb = 0;         // p buffer holding the current direction
  for (int64_t k = 1;; ++k) {
    // ------------------------------------------------------------ HVP ----
    double vv = 0.0;
    {
      double2 vr[K];
      const double* pold = a.p[pb ^ 1];
      double* pnew = a.p[pb];
      double pp = 0.0;
      // every load of z and the old direction before the first store of the
      // new one (the store could alias them: issued in between, each load
      // would wait for the one before).  (Keeping the whole direction in
      // registers across iterations instead spills at n = 10000.)
      double2 po[K];
#pragma unroll
      for (int kk = 0; kk < K; ++kk) {
        const int j = 2 * (tid + kk * kCpThreads);
        vr[kk] = j < n ? *reinterpret_cast<const double2*>(a.z + j) : make_double2(0.0, 0.0);
        po[kk] = (j < n && k > 1) ? *reinterpret_cast<const double2*>(pold + j) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int kk = 0; kk < K; ++kk) {
        const int j = 2 * (tid + kk * kCpThreads);
        if (j < n) {
          const double2 zz = vr[kk];
          double2 v = zz;
          if (k > 1) {
            v.x = __dadd_rn(zz.x, __dmul_rn(beta, po[kk].x));
            v.y = __dadd_rn(zz.y, __dmul_rn(beta, po[kk].y));
          }
          vr[kk] = v;
          pp = fma(v.x, v.x, fma(v.y, v.y, pp));
          if (j >= c0 && j < c1) *reinterpret_cast<double2*>(pnew + j) = v;
        } else {
          vr[kk] = make_double2(0.0, 0.0);
        }
      }
      if (a.qp)  // the direction at this CTA's rows, same arithmetic as vr
        for (int64_t q2 = tid; q2 < nrows_mine; q2 += kCpThreads) {
          const int64_t i = cta + q2 * nctas;
          vrow[q2] = k > 1 ? __dadd_rn(a.z[i], __dmul_rn(beta, pold[i])) : a.z[i];
        }
      vv = cp_block_sum(pp, sh);  // ||p||^2, identical in every CTA (barriers order vrow too)
      stamp(4);  // direction
      const double vav = hvp_rows(vr);
      if (tid == 0) a.part[cta * 8 + 1] = vav;
    }
    stamp(5);  // rows of A
    grid.sync();
    stamp(6);  // barrier 3
    // --------------------------------------------------- alpha + STEP ----
    // p.Ap = sum_i d_i (a_i.p)^2 + shift ||p||^2  (fixed order, every CTA)
    // this thread's element of the p and x slices, requested before the sums
    // below so their round trips overlap (slice <= 90: one element per thread)
    const int64_t si_ = c0 + tid;
    const bool smine = si_ < c1;
    const double p_si = smine ? a.p[pb][si_] : 0.0;
    const double x_si = smine ? a.x[si_] : 0.0;
    const double pap = fma(a.shift, vv, all_sum(1));
    stamp(16);  // step: p.Ap sum
    if (!isfinite(pap) || pap <= 0.0) {  // krylov.py:74-77
      if (writer) {
        sc[NYS_CG_PAP] = pap;
        sc[NYS_CG_FLAG] = !isfinite(pap) ? 1.0 : 2.0;
        sc[NYS_CG_DONE] = !isfinite(pap) ? 2.0 : 3.0;
        sc[NYS_CG_ITERS] = (double)k;
        sc[NYS_CG_RUNNING] = 0.0;
      }
      break;
    }
    const double alpha = rz / pap;
    const bool refresh = (k % 50) == 0;  // krylov.py:16
    const double* pc = a.p[pb];
    double rr;
    if (!refresh) {
      y_slice();
      stamp(17);  // step: y partial sums
      double acc = 0.0;
      if (smine) {
        const int64_t i = si_;
        const double api = fma(a.shift, p_si, ys[i - c0]);
        a.Ap[i] = api;
        a.x[i] = __dadd_rn(x_si, __dmul_rn(alpha, p_si));
        const double ri = __dadd_rn(rsl[i - c0], -__dmul_rn(alpha, api));
        a.res[i] = ri;
        rsl[i - c0] = ri;
        acc = fma(ri, ri, acc);
      }
      rr = cp_block_sum(acc, sh);
    } else {
      // x only, then r = b - A x (true residual refresh, krylov.py:80-81)
      for (int64_t i = c0 + tid; i < c1; i += kCpThreads) a.x[i] = __dadd_rn(a.x[i], __dmul_rn(alpha, pc[i]));
      grid.sync();
      double2 vr[K];
#pragma unroll
      for (int kk = 0; kk < K; ++kk) {
        const int j = 2 * (tid + kk * kCpThreads);
        vr[kk] = j < n ? *reinterpret_cast<const double2*>(a.x + j) : make_double2(0.0, 0.0);
      }
      if (a.qp) {
        for (int64_t q2 = tid; q2 < nrows_mine; q2 += kCpThreads) vrow[q2] = a.x[cta + q2 * nctas];
        __syncthreads();
      }
      hvp_rows(vr);
      grid.sync();
      y_slice();
      double acc = 0.0;
      for (int64_t i = c0 + tid; i < c1; i += kCpThreads) {
        const double axi = fma(a.shift, a.x[i], ys[i - c0]);
        a.Ap[i] = axi;
        const double ri = __dadd_rn(a.b[i], -axi);
        a.res[i] = ri;
        rsl[i - c0] = ri;
        acc = fma(ri, ri, acc);
      }
      rr = cp_block_sum(acc, sh);
    }
    stamp(18);  // step: x, r update + ||r||^2
    if (a.r > 0) utw_slice();
    if (tid == 0) a.part[cta * 8 + 2] = rr;
    stamp(7);  // step (y partial sums, x, r, U^T r)
    grid.sync();
    stamp(8);  // barrier 4
    // ------------------------------------------------ stop test + APPLY --
    {
      const double rtot = all_sum(2);
      const double denom = b2 > 0.0 ? sqrt(b2) : 1.0;
      const double res = sqrt(rtot);
      const bool stop = !isfinite(res) || res <= tol * denom || k >= a.max_iter;
      if (writer) {
        sc[NYS_CG_PAP] = pap;
        sc[NYS_CG_ALPHA] = alpha;
        sc[NYS_CG_NHVP] = (double)(k + k / 50);
        cp_stop(sc, rtot, tol, k, a.max_iter);
      }
      if (stop) break;
    }
    if (a.r > 0) make_coef();
    {
      const double rzp = apply_slice();
      if (tid == 0) a.part[cta * 8 + 3] = rzp;
    }
    stamp(9);  // stop test + preconditioner apply
    grid.sync();
    stamp(10);  // barrier 5
    const double rz_new = all_sum(3);
    stamp(19);  // r.z sum
    beta = rz_new / rz;  // krylov.py:89-93
    rz = rz_new;
    if (writer) {
      sc[NYS_CG_RZNEW] = rz_new;
      sc[NYS_CG_RZ] = rz_new;
      sc[NYS_CG_BETA] = beta;
    }
    pb ^= 1;
  }
  stamp(11);  // stop test
  zu_slice();
  finish();
  stamp(12);  // z/u tail + finish
  if (probe) atomicAdd(&g_cp_probe_cnt, 1ull);
}

struct CpPlan {
  int K, W, S, u_smem;
  size_t smem;
  bool ok;
};

static CpPlan cp_plan(const nys_cg_problem* pb) {
  CpPlan p{};
  p.ok = false;
  static const bool off = dev_env("NYS_CG_PERSIST_OFF") != nullptr;
  if (off || (pb->op_kind != 0 && !(pb->op_kind == 1 && pb->rows == pb->n)) || pb->rows < kNumSMs ||
      (pb->n & 1) || (pb->lda & 1) ||
      ((uintptr_t)pb->A & 15) || pb->r > 512)
    return p;
  p.W = (int)pb->n;
  p.K = (int)cdiv(pb->n, (int64_t)2 * kCpThreads);
  if (p.K > kCpMaxK) return p;
  // every slice of n / 148 columns has at most one element per thread (<= 90)
  static_assert(((kCpMaxK * 2 * kCpThreads + kNumSMs - 1) / kNumSMs + 1) <= kCpThreads, "slice");
  const size_t row_bytes = (size_t)p.W * 8;
  // red, sh, coef, lam + nu, slice sums, scratch
  const size_t extra = 64 * 8 + (size_t)(2 * cp_r2(pb->r) + 112 + 112 + 112 + 1024) * 8 + 1024;
  p.S = (int)tmin<int64_t>(4, (kCpSmemBudget - extra) / row_bytes);
  if (p.S < 2) return p;
  p.smem = (size_t)p.S * row_bytes + (size_t)(p.S + 2) * 8 + extra;
  const int64_t slice = ((pb->n + kNumSMs - 1) / kNumSMs + 1) & ~1ll;
  const size_t ubytes = (size_t)slice * (pb->r > 0 ? pb->r : 0) * 8;
  p.u_smem = pb->r > 0 && p.smem + ubytes <= (size_t)kCpSmemBudget;
  if (p.u_smem) p.smem += ubytes;
  p.ok = true;
  return p;
}

template <int K>
static int cp_launch(const CpPlan& pl, const CgPersistArgs& args, cudaStream_t st) {
  static bool attr = false;
  auto fn = cg_persist_kernel<K>;
  if (!attr) {
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kCpSmemBudget) != cudaSuccess) {
      cudaGetLastError();
      return NYS_ERR_CUDA;
    }
    attr = true;
  }
  CgPersistArgs a = args;
  const unsigned grid = (unsigned)tmin<int64_t>(kNumSMs, a.rows);
  // one CTA per SM must be co-resident: fewer free SMs -> the batched plan
  static int fits = -1;
  if (fits < 0) fits = coop_fits((const void*)fn, grid, kCpThreads, pl.smem) ? 1 : 0;
  if (!fits) return NYS_ERR_UNSUPPORTED;
  const int rc = coop_launch_status(launch_chain(fn, dim3(grid), dim3(kCpThreads), pl.smem, st, true, a));
  if (rc) {
    if (rc == NYS_ERR_UNSUPPORTED) fits = 0;
    return rc;
  }
  __atomic_fetch_add(&g_launches, 1ull, __ATOMIC_RELAXED);
  return debug_sync_check(__FILE__, __LINE__) ? NYS_ERR_CUDA : NYS_OK;
}

size_t cg_persist_ws(int64_t n, int r) {
  return (size_t)kNumSMs * n * sizeof(double) + (size_t)kNumSMs * (r + 1) * sizeof(double) +
         (size_t)kNumSMs * 8 * sizeof(double) + (size_t)(r + 1) * sizeof(double) + 2 * (size_t)n * sizeof(double) +
         1024;
}

// The whole solve in one launch when the problem fits the plan; returns
// NYS_ERR_UNSUPPORTED otherwise (the caller then runs the batched kernels).
// ws: cg_persist_ws(n, r) bytes, zero-filled once (tickets).
int cg_persist(const nys_cg_problem* pb, const nys_admm_head* head, void* ws, size_t ws_bytes, cudaStream_t st) {
  const CpPlan pl = cp_plan(pb);
  if (!pl.ok) return NYS_ERR_UNSUPPORTED;
  if (ws_bytes < cg_persist_ws(pb->n, pb->r)) return NYS_ERR_WORKSPACE;
  CgPersistArgs a{};
  a.A = pb->A;
  a.rows = pb->rows;
  a.n = pb->n;
  a.lda = pb->lda;
  a.d = pb->d;
  a.shift = pb->shift;
  a.U = pb->U;
  a.r = pb->r > 0 ? pb->r : 0;
  a.ldu = pb->ldu;
  a.lam = pb->lam;
  a.nu = pb->nu;
  a.b = pb->b;
  a.x = pb->x;
  a.res = pb->res;
  a.z = pb->z;
  a.Ap = pb->Ap;
  a.sc = pb->sc;
  a.tol = pb->tol;
  a.tolp = pb->tol_dev;
  a.gate = pb->gate;
  a.max_iter = pb->max_iter;
  char* base = reinterpret_cast<char*>(ws);
  a.counter = reinterpret_cast<unsigned int*>(base);
  size_t off = 256;
  a.ypart = reinterpret_cast<double*>(base + off);
  off += (size_t)kNumSMs * pb->n * sizeof(double);
  a.hpart = reinterpret_cast<double*>(base + off);
  off += (size_t)kNumSMs * (pb->r + 1) * sizeof(double);
  a.part = reinterpret_cast<double*>(base + off);
  off += (size_t)kNumSMs * 8 * sizeof(double);
  a.coef = reinterpret_cast<double*>(base + off);
  off += (size_t)(pb->r + 1) * sizeof(double);
  off = (off + 15) & ~size_t(15);
  a.p[0] = pb->p;
  a.p[1] = reinterpret_cast<double*>(base + off);  // second direction buffer
  a.W = pl.W;
  a.S = pl.S;
  a.has_head = head != nullptr;
  a.u_smem = pl.u_smem;
  static const int probe = dev_env("NYS_CP_PROBE") ? atoi(dev_env("NYS_CP_PROBE")) : 0;
  a.probe = probe;
  a.qp = pb->op_kind == 1 ? 1 : 0;
  static const int nopf = dev_env("NYS_CP_NOPREFETCH") ? 1 : 0;
  a.no_early_prefetch = nopf;
  a.order_in = pb->order_in;
  a.order_out = pb->order_out;
  if (head) a.h = *head;
  const nys_admm_tail* t = head ? head->zu : nullptr;
  if (t && t->XZ == pb->x && t->n == pb->n) {
    a.has_zu = 1;
    a.zu.z = t->XZ + t->n;
    a.zu.u = t->u;
    a.zu.xbar = t->xbar;
    a.zu.zbar = t->zbar;
    a.zu.alpha = t->alpha;
    a.zu.kappa = t->kappa;
    a.zu.prox_kind = t->kind == 0 ? NYS_PROX_SOFT : NYS_PROX_BOX;
    a.zu.accum = t->accum;
    a.zu.lo = t->lo;
    a.zu.hi = t->hi;
    a.zu.rx = t->ring ? t->ring + (int64_t)t->slot * t->ring_ld : nullptr;
    a.zu.ru = t->ring && t->uring ? t->uring + (int64_t)t->slot * t->ring_ld : nullptr;
  }
  int rc = NYS_ERR_UNSUPPORTED;
#define NYS_CP(k)                  \
  case k:                          \
    rc = cp_launch<k>(pl, a, st);  \
    break;
  switch (pl.K) {
    NYS_CP(1) NYS_CP(2) NYS_CP(3) NYS_CP(4) NYS_CP(5) NYS_CP(6) NYS_CP(7) NYS_CP(8) NYS_CP(9) NYS_CP(10)
    NYS_CP(11) NYS_CP(12) NYS_CP(13)
    default: break;
  }
#undef NYS_CP
  if (rc == NYS_OK && a.has_zu) head->zu->zu_done = 1;
  return rc;
}

}  // namespace nys

// development: read (and clear) the accumulated phase times of the probe, ns
extern "C" int nys_debug_cp_probe(unsigned long long* acc24, unsigned long long* count) {
  if (cudaMemcpyFromSymbol(acc24, nys::g_cp_probe_acc, 24 * sizeof(unsigned long long)) != cudaSuccess ||
      cudaMemcpyFromSymbol(count, nys::g_cp_probe_cnt, sizeof(unsigned long long)) != cudaSuccess)
    return NYS_ERR_CUDA;
  unsigned long long z[25] = {};
  cudaMemcpyToSymbol(nys::g_cp_probe_acc, z, 24 * sizeof(unsigned long long));
  cudaMemcpyToSymbol(nys::g_cp_probe_cnt, z, sizeof(unsigned long long));
  return NYS_OK;
}
