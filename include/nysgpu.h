/*
 * nysgpu.h -- C ABI of libnysgpu.so, the B200 (sm_100a) kernels behind the
 * inexact-ADMM x-subproblem hot path of GeNIOS (arXiv 2310.08333).
 *
 * The reference (`/root/reference/pkg/src/nysopt`, Python/NumPy) has no FFI:
 * its numeric call sites are NumPy `@` and LAPACK calls.  Each entry point
 * below replaces one of those call sites (file:line cited per function) and is
 * what a reference-side binding (ctypes / cffi) would bind.
 *
 * Conventions
 *   - all matrix/vector pointers are DEVICE pointers to FP64 data;
 *   - matrices are row-major (NumPy C order) with an explicit leading dim;
 *   - `stream` is a cudaStream_t passed as void*; every call is asynchronous
 *     on that stream unless stated otherwise;
 *   - `ws` is caller-allocated device workspace of at least the size the
 *     matching *_workspace() query returns, ZERO-FILLED once at allocation
 *     (kernels keep an atomic ticket in it and reset it themselves);
 *   - scalar outputs (`sc`, `out`) are device arrays of doubles;
 *   - return value: NYS_OK or an error code (mapped to the reference's
 *     exception classes by the host layer, errors.py:4-29).
 *
 * Reductions are deterministic (fixed-order, no floating-point atomics).
 */
#ifndef NYSGPU_H
#define NYSGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NYS_ABI_VERSION 1

enum nys_status {
  NYS_OK = 0,
  NYS_ERR_ARG = 1,          /* DimensionMismatchError / DataError            */
  NYS_ERR_CUDA = 2,         /* CUDA launch/runtime failure                   */
  NYS_ERR_NOT_SPD = 3,      /* NotSPDError: nonpositive curvature (krylov.py:76-77) */
  NYS_ERR_NONFINITE = 4,    /* NumericalError (krylov.py:74-75, 85-86)       */
  NYS_ERR_NOT_PSD = 5,      /* DataError: indefinite sketch core (sketch.py:117-120) */
  NYS_ERR_UNSUPPORTED = 6,  /* CapabilityError                               */
  NYS_ERR_WORKSPACE = 7,    /* workspace too small                           */
  NYS_ERR_NO_DEVICE = 8     /* no sm_100 device visible                      */
};

/* loss kinds (problems.py:53-111) */
enum nys_loss { NYS_LOSS_SQUARE = 0, NYS_LOSS_LOGISTIC = 1, NYS_LOSS_HUBER = 2 };
/* prox kinds (prox.py:38-48) */
enum nys_prox { NYS_PROX_SOFT = 0, NYS_PROX_BOX = 1 };

/* CG scalar block layout (device doubles), see krylov.py:58-93 */
enum nys_cg_slot {
  NYS_CG_RZ = 0,     /* r.z of the current direction             */
  NYS_CG_PAP = 1,    /* p.Ap                                      */
  NYS_CG_ALPHA = 2,  /* rz / pAp                                  */
  NYS_CG_RES2 = 3,   /* ||r||^2                                   */
  NYS_CG_RZNEW = 4,  /* r.z of the freshly preconditioned residual */
  NYS_CG_B2 = 5,     /* ||b||^2                                   */
  NYS_CG_FLAG = 6,   /* 0 ok, 1 non-finite pAp, 2 pAp <= 0        */
  NYS_CG_TICKET = 7, /* kernel ticket (keep zero)                 */
  NYS_CG_DONE = 8,   /* batched CG: 0 running, 1 converged, 2 non-finite, 3 not SPD, 4 cap,
                        5 skipped (closed gate: the previous ADMM iteration is unfinished) */
  NYS_CG_ITERS = 9,  /* batched CG: iterations taken              */
  NYS_CG_RESREL = 10,/* batched CG: final ||r|| / ||b||           */
  NYS_CG_RUNNING = 11,/* batched CG: 1 while iterating, 0 once DONE is set */
  NYS_CG_NHVP = 12,  /* persistent CG: operator applications in the last solve */
  NYS_CG_BETA = 13,  /* persistent CG: beta of the last direction update   */
  NYS_CG_NSLOTS = 16
};

/* One PCG solve for nys_cg_iterate_f64 (krylov.py:35-95).  All pointers are
 * device pointers; `sc` is the NYS_CG_NSLOTS scalar block with B2 and RES2
 * already set for r = b - A x0 (e.g. by nys_admm_rhs_f64 or nys_cg_start_f64). */
/* Sum `count` doubles at `buf` over all ranks in place, ordered on `stream`
 * (the host layer's all-reduce; called from inside the drivers below). */
typedef void (*nys_reduce_fn)(double* buf, int64_t count, void* user, void* stream);

typedef struct nys_cg_problem {
  int op_kind;          /* 0: y = A^T (d o A v) + shift v (ML Hessian, A rows x n)
                           1: y = A v + shift v (dense symmetric A, n x n)          */
  const double* A;
  int64_t rows, n, lda;
  const double* d;      /* row weights (op 0) or NULL (== 1)                        */
  double shift;
  const double* U;      /* preconditioner factors (sketch.py:143-151); r = 0: none  */
  int r;
  int64_t ldu;
  const double* lam;
  double nu;
  const double* b;
  double* x;            /* in: x0, out: solution                                    */
  double* res;          /* residual r                                               */
  double* p;
  double* z;
  double* Ap;
  double* sc;
  double tol;           /* relative tolerance (krylov.py:87)                        */
  int64_t max_iter;
  void* ws_op;  size_t ws_op_bytes;   /* operator workspace (zero-filled once)     */
  void* ws_pc;  size_t ws_pc_bytes;   /* preconditioner workspace                  */
  void* ws_red;                        /* reduction scratch (returned size)         */
  const double* gate;   /* NULL, or: *gate == 0 skips the solve (sc[DONE] = 5, RUNNING = 1) */
  const double* tol_dev;/* NULL, or the tolerance is read from *tol_dev (device-computed) */
  int64_t timing_tag;   /* tag of the timing events of this solve (nys_timing_commit)      */
  void* ws_cp; size_t ws_cp_bytes;     /* NULL, or nys_cg_persist_workspace(n, r) bytes,
                                          zero-filled once: the whole solve then runs as ONE
                                          persistent cooperative kernel when the shape allows */
  const double* order_in; double* order_out; /* NULL, or the row order of the last pass over A
                                          before / after this solve (0 ascending, 1 descending):
                                          the persistent kernel alternates the order of its
                                          passes starting opposite to *order_in so each pass
                                          begins with the rows still in L2, and records its
                                          last in *order_out (results depend only on *order_in) */
  nys_reduce_fn reduce; void* reduce_user; /* NULL, or the row-sharded exchange:
                                          each operator application then produces this rank's
                                          partial A_i^T (d o A_i v), calls reduce(y, n, ...) to
                                          sum it over the ranks (enqueued on the stream by the
                                          host layer: torch.distributed / NCCL), and adds the
                                          shift and p.Ap after it.  The solve stays device-
                                          predicated: no host round trip per CG iteration.  */
} nys_cg_problem;

/* ---------------------------------------------------------------- misc -- */
/* dst[i] = src[i] by a kernel; dst may be device-mapped pinned host memory
 * (the per-iteration readback of the ADMM pipeline) */
int nys_copy_f64(const double* src, double* dst, int64_t n, void* stream);
/* nys_copy_f64 of a per-iteration readback block that also opens the next
 * iteration's gate (*gate_next = 1) unless *pred != 0 (pred may be NULL). */
int nys_readback_f64(const double* src, double* dst, int64_t n, double* gate_next, const double* pred,
                     void* stream);
int nys_abi_version(void);
const char* nys_status_string(int status);
/* NYS_OK when a compute-capability-10.x device is current */
int nys_device_check(void);
/* number of kernels launched by this library since load (instrumentation) */
unsigned long long nys_launch_count(void);
/* bytes of the generic reduction workspace used by the vector kernels */
size_t nys_reduce_workspace(void);

/* ------------------------------------------------ K1/K2 dense products -- */
/* K1 (operators.py:114-115 `a @ v`, k right-hand sides, k <= 4):
 *   Y[j*ldy + i] = sum_c A[i*lda + c] * X[j*ldx + c]      0 <= i < rows, j < k */
size_t nys_gemv_workspace(int64_t rows, int64_t n, int k);
int nys_gemv_f64(const double* A, int64_t rows, int64_t n, int64_t lda, const double* X,
                 int64_t ldx, int k, double* Y, int64_t ldy, void* ws, size_t ws_bytes,
                 void* stream);

/* K2 (operators.py:117-118 `a.T @ u`, k <= 4):
 *   Y[j*ldy + c] = sum_i A[i*lda + c] * T[j*ldt + i]      0 <= c < n, j < k
 * Split over rows with a deterministic fixed-order reduction of the splits. */
size_t nys_gemvT_workspace(int64_t rows, int64_t n, int k);
int nys_gemvT_f64(const double* A, int64_t rows, int64_t n, int64_t lda, const double* T,
                  int64_t ldt, int k, double* Y, int64_t ldy, void* ws, size_t ws_bytes,
                  void* stream);

/* ---------------------------------------------- K3 Hessian-vector product -- */
/* K3 (problems.py:263-264 MLHessian._apply + admm.py:262-263 shift):
 *   y = A^T (d o (A v)) + shift * v,   and *pAp = v . y  when pAp != NULL.
 * d == NULL means d == 1 (square loss, problems.py:59).
 * finish == 0: write only the local partial A^T(d o Av) (row shard), to be
 * all-reduced across GPUs and completed by nys_shift_dot_f64. */
size_t nys_hvp_workspace(int64_t rows, int64_t n);
int nys_hvp_f64(const double* A, int64_t rows, int64_t n, int64_t lda, const double* d,
                const double* v, double shift, double* y, double* pAp, int finish, void* ws,
                size_t ws_bytes, void* stream);
/* The single-pass plan nys_hvp_f64 takes for a (rows x n, lda) operand:
 * 1 whole rows per CTA, 2 column-split clusters, 3 16-CTA DSMEM clusters,
 * 4 grid column strips, 0 two passes (K1 + K2); -1 bad arguments. */
int nys_hvp_plan(int64_t rows, int64_t n, int64_t lda);
/* y += shift * v; *dot = v . y when dot != NULL (device scalar). */
int nys_shift_dot_f64(int64_t n, const double* v, double shift, double* y, double* dot,
                      void* ws, void* stream);
/* *out = a . b (device scalar, deterministic) */
int nys_dot_f64(int64_t n, const double* a, const double* b, double* out, void* ws,
                void* stream);

/* ----------------------------------------------------- K6 preconditioner -- */
/* K6 (sketch.py:143-151, Eq. (11)):
 *   z = U((lam[r-1] + nu) * (U^T v)/(lam + nu) - U^T v) + v
 * U is n x r row-major (ldu), lam has r entries (device).  r == 0 -> z = v.
 * If rz != NULL, *rz = rdot . z (device scalar). */
size_t nys_precond_workspace(int64_t n, int r);
int nys_precond_apply_f64(const double* U, int64_t n, int r, int64_t ldu, const double* lam,
                          double nu, const double* v, double* z, const double* rdot,
                          double* rz, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------- K7 CG vectors -- */
/* krylov.py:58-62: r = b - Ax0; sc[B2] = ||b||^2; sc[RES2] = ||r||^2 */
int nys_cg_start_f64(int64_t n, const double* b, const double* Ax0, double* r, double* sc,
                     void* ws, void* stream);
/* krylov.py:72-84: alpha = rz/pAp (sc[FLAG] set on non-finite / <= 0 pAp);
 * x += alpha p; unless refresh: r -= alpha Ap and sc[RES2] = ||r||^2 */
int nys_cg_step_xr_f64(int64_t n, double* x, double* r, const double* p, const double* Ap,
                       int refresh, double* sc, void* ws, void* stream);
/* krylov.py:89-93: first: p = z, rz = rz_new;  else beta = rz_new/rz,
 * rz = rz_new, p = z + beta p.   (rz_new = sc[RZNEW]) */
int nys_cg_dir_f64(int64_t n, const double* z, double* p, int first, double* sc,
                   void* stream);

/* Batched, device-predicated PCG: launches iterations k_first .. k_first+count-1
 * (k_first == 1 also runs the initial test and first preconditioning).  The
 * stop test of krylov.py:80-93 runs on the device and sets sc[NYS_CG_DONE];
 * every later launch is a no-op, so the host may run ahead and read sc once.
 * Workspace sizes: returns the reduction scratch bytes, *ws_op / *ws_pc. */
size_t nys_cg_workspace(int op_kind, int64_t rows, int64_t n, int r, size_t* ws_op, size_t* ws_pc);
int nys_cg_iterate_f64(const nys_cg_problem* pb, int64_t k_first, int count, void* stream);
/* workspace of the persistent single-kernel solve (see nys_cg_problem.ws_cp) */
size_t nys_cg_persist_workspace(int64_t n, int r);
/* Instrumentation (bench roofline): with timing enabled, nys_cg_iterate_f64
 * brackets every operator launch with CUDA events tagged by its CG iteration;
 * nys_timing_commit(tag, k, units) keeps those of the solve `tag` with
 * iterations <= k (the ones that ran -- later launches of a batch were
 * predicated no-ops) and drops that solve's others; a persistent single-launch
 * solve is bracketed as a whole and counts `units` operator applications. */
int nys_timing_enable(int on);
int nys_timing_commit(int64_t tag, int64_t last_real_k, int64_t units);
int nys_timing_read(double* total_ms, int64_t* launches);

/* Everything of one ADMM iteration after the x-update (admm.py:562-611 and
 * 621-675), launched as one predicated sequence: relax/prox/dual update (+
 * averages), window copy, data passes (ML: A{x,z}, loss epilogue,
 * A^T{l', w o Ax, nu}; QP: P x), residual/objective/gap norms, window norms,
 * QP infeasibility pieces.  Every launch is skipped while *pred != 0 (pass
 * &sc[NYS_CG_RUNNING] to chain it behind a batched CG solve). */
typedef struct nys_admm_tail {
  int kind;                   /* 0: ML (M = I), 1: box QP (M = I)                     */
  int loss;                   /* nys_loss (ML)                                        */
  int64_t n, rows;
  const double* A; int64_t lda;     /* ML data (rows x n) or P (n x n)                */
  const double* b;                  /* ML responses (rows)                            */
  double* XZ;                 /* 2 x n: x (row 0), z (row 1)                          */
  double* u; double* xbar; double* zbar; int accum;
  double alpha; double kappa; const double* lo; const double* hi; const double* q;
  double lambda1, lambda2, rho;
  int with_z;                 /* ML: also A z, the dual point and A^T nu              */
  double* AXZ;                /* 2 x rows                                             */
  double* T;                  /* 3 x rows: l'(Ax-b), w o Ax, nu                       */
  double* w;                  /* rows                                                 */
  double* AT;                 /* ML: 3 x n (gA, hxA, atnu) ; QP: 1 x n (P x)          */
  double* rowsums;            /* NYS_ROWS_NOUT                                        */
  double* norms;              /* NYS_NORMS_NOUT                                       */
  double* ring; double* uring; int64_t ring_ld; int slot;
  int nothers; int others[16]; double* wnorms;   /* window norms (17)             */
  int qp_infeas; int inf_first; int inf_last; double width; double* dx; double* Pdx;
  double* infeas; double* pdx2;                   /* 6 pieces, ||P dx||^2          */
  void* ws_gemv; size_t ws_gemv_bytes; void* ws_gemvT; size_t ws_gemvT_bytes; void* ws_red;
  const double* pred;
  double* gate_next;          /* NULL, or set to 1 once the tail has run (opens the next
                                 iteration's gate, see nys_admm_head)                  */
  double* conj_out;           /* NULL, or (ML, with_z, lambda2 == 0) the scaled-dual conjugate
                                 sums of problems.py:330-340 with c = lambda1 / max|atnu|,
                                 computed when max|atnu| > lambda1 (3 values)           */
  const double* order;        /* NULL, or the row order of the last pass over A before the
                                 tail (nys_cg_problem.order_out): the data passes run
                                 opposite to it, then along it (schedule only: results do
                                 not depend on it)                                      */
  int zu_done;                /* set by nys_admm_xupdate_f64 when its persistent kernel
                                 already ran the relax/prox/dual update and the window
                                 append of this descriptor; the tail then skips them   */
  nys_reduce_fn reduce; void* reduce_user;  /* NULL, or the row-sharded exchange: the A^T
                                 outputs (AT), the row sums (NYS_ROWS_NOUT) and the
                                 conjugate sums (3) are summed over the ranks before the
                                 norms that use them                                      */
  const double* rb_src; double* rb_dst; int64_t rb_n; double* rb_gate; double rb_tag;
                              /* NULL rb_dst, or the iteration's readback (nys_readback_f64
                                 arguments) for the tail to fuse into its last kernel;
                                 rb_tag != 0 is then stored at rb_dst[rb_n] once the block
                                 is complete (the host may poll it instead of an event)   */
  int rb_done;                /* out: 1 when the tail did that readback                  */
  /* device-side termination (admm.py:227-240 with problems.py:335-351): when
   * stop_on, the fused ML epilogue's last CTA evaluates the stop test from the
   * reduced norms and row sums exactly as the host does, stores 1.0 / 0.0 at
   * norms[stop_slot], and leaves the next iteration's gate closed when the
   * test holds (an iteration launched ahead then does nothing); stop_ran
   * (out) tells whether this launch ran the device test */
  int stop_on, stop_gap, stop_linf, stop_slot, stop_ran;
  double stop_eps_gap, stop_eps_abs, stop_eps_rel, stop_sqrt_n;
  /* NULL, or (square loss, with_z) g_b = A^T b (n): the one-pass cluster tail
   * then streams two products A^T (A x), A^T (A z) instead of three, and the
   * epilogue forms A^T (Ax - b) = A^T (A x) - g_b, A^T (Az - b) = A^T (A z) - g_b
   * (problems.py:227-351 with l'(r) = r, l'' = 1) */
  const double* gb;
} nys_admm_tail;
int nys_admm_tail_f64(const nys_admm_tail* t, void* stream);

/* Start of one ADMM iteration on the device, for a host that runs one
 * iteration ahead (admm.py:520-560 with the stopping test of iteration k-1
 * still pending): if *gate == 0 (iteration k-1 unfinished) nothing is done.
 * Otherwise: *gate_next = 0; snapshot (x, z, u, xbar, zbar) -> snap (5 n, may
 * be NULL) so the host can roll back if k-1 turns out to be the last
 * iteration; the CG tolerance of krylov.py:98-112 from the previous norms
 *   rp, rd = sqrt(prev[0]), sqrt(prev[2])   (norm_kind 0; 1: prev[1], prev[3])
 *   *tol_out = max(min(sqrt(rp rd), 1) / kpow, 1e-12)    (kpow = k^gamma)
 * or *tol_out = tol_fixed when tol_fixed > 0; then the right-hand side and
 * initial residual exactly as nys_admm_rhs_f64. */
typedef struct nys_admm_head {
  int64_t n;
  const double* hxA; const double* gA; const double* q;
  double lambda2, sigma, rho, shift;
  const double* x; const double* z; const double* u; const double* xbar; const double* zbar;
  double* rhs; double* r; double* sc;
  double* snap;
  const double* gate; double* gate_next;
  const double* prev; int norm_kind; double kpow; double tol_fixed; double* tol_out;
  void* ws_red;
  nys_admm_tail* zu;          /* NULL, or the iteration's tail descriptor: when the
                                 persistent kernel runs, it ends with the tail's z/u
                                 update and window append on each CTA's slice of x
                                 (admm.py:562-583, 622-623) and sets zu->zu_done = 1
                                 (0 otherwise)                                         */
} nys_admm_head;
int nys_admm_head_f64(const nys_admm_head* h, void* stream);
/* The x-update of admm.py:243-275: head + PCG.  One persistent cooperative
 * kernel (head fused into its prologue) when pb->ws_cp is set and the dense ML
 * problem fits its plan; otherwise nys_admm_head_f64 and `count` batched CG
 * iterations (nys_cg_iterate_f64, k_first = 1). */
int nys_admm_xupdate_f64(const nys_admm_head* h, const nys_cg_problem* pb, int count, void* stream);

/* ---------------------------------------------- K8/K9 ADMM elementwise -- */
/* x-update right-hand side and initial CG residual, M = I, c = 0
 * (admm.py:270-272, krylov.py:61):
 *   hx = hxA + lambda2 x;  g = gA + lambda2 x (+ q);
 *   rhs = hx + sigma x - g + rho (z - u);   r = rhs - (hx + shift x)
 *   sc[B2] = ||rhs||^2, sc[RES2] = ||r||^2.   q may be NULL. */
int nys_admm_rhs_f64(int64_t n, const double* hxA, const double* gA, const double* q,
                     double lambda2, double sigma, double rho, double shift, const double* x,
                     const double* z, const double* u, double* rhs, double* r, double* sc,
                     void* ws, void* stream);
/* over-relaxation, prox and dual update (admm.py:278-300, prox.py:38-48):
 *   w = alpha x + (1-alpha) z;  z = prox(w + u);  u = u + w - z;
 *   if accum: xbar += x, zbar += z   (admm.py:580-583) */
int nys_admm_zu_f64(int64_t n, const double* x, double* z, double* u, double alpha,
                    int prox_kind, double kappa, const double* lo, const double* hi,
                    double* xbar, double* zbar, int accum, void* stream);
/* residual norms and objective pieces (admm.py:215-224, problems.py:227-351):
 * out[ 0..1] = sum/max of (x-z)^2/|x-z|      out[ 2..3] rd = gA+lambda2 x(+q)+rho u
 * out[ 4..5] x                               out[ 6..7] z
 * out[ 8..9] rho u                           out[10] sum|z|
 * out[11] x.gA       out[12] q.x             out[13] max|atnu|
 * out[14] sum (|atnu|-lambda1)_+^2           out[15] max(lo-z, z-hi)
 * (sum slots are sums of squares; max slots are max-abs).  q/atnu/lo/hi may be NULL. */
#define NYS_NORMS_NOUT 16
int nys_admm_norms_f64(int64_t n, const double* x, const double* z, const double* u,
                       const double* gA, const double* q, double lambda2, double rho,
                       const double* atnu, double lambda1, const double* lo,
                       const double* hi, double* out, void* ws, void* stream);

/* row-space (sample) elementwise pass for ML problems (problems.py:219-351):
 *   r1 = Ax - b:  tg = l'(r1), w = l''(r1), thx = w o Ax
 *   r2 = Az - b (if Az):  tnu = l'(r2)
 * out[0] = sum l(r1), out[1] = sum l(r2), out[2] = sum l*(tnu) (finite part),
 * out[3] = count of infinite l*(tnu), out[4] = b . tnu.   (row-shard partials) */
#define NYS_ROWS_NOUT 5
int nys_ml_rowwise_f64(int64_t rows, int loss, const double* Ax, const double* Az,
                       const double* b, double* tg, double* w, double* thx, double* tnu,
                       double* out, void* ws, void* stream);
/* dual value at the scaled point c*nu (problems.py:313-328):
 * out[0] = sum l*(c nu) (finite part), out[1] = #inf, out[2] = b.(c nu) */
int nys_ml_conj_scaled_f64(int64_t rows, int loss, const double* nu, double c,
                           const double* b, double* out, void* ws, void* stream);

/* ------------------------------------------------- K13/K14 loop support -- */
/* cycle guard / windows (admm.py:643-675): ring[slot*ld + i];
 * out[0] = ||x_cur||^2, out[1+j] = ||x_cur - x_others[j]||^2 (j < nothers <= 16).
 * `others` is a HOST array copied into the launch. */
int nys_window_norms_f64(int64_t n, const double* ring, int64_t ld, int cur,
                         const int* others, int nothers, double* out, void* ws, void* stream);
/* penalty change (admm.py:303-319): y_old = rho_old u; u *= rho_old/rho_new;
 * out[0] = ||y_old||^2, out[1] = ||rho_new u - y_old||^2 */
int nys_scale_dual_f64(int64_t n, double* u, double rho_old, double rho_new, double* out,
                       void* ws, void* stream);
/* QP infeasibility pieces (admm.py:361-415, prox.py:96-135), M = I:
 *   dx = (xa - xb)/width, du = (ua - ub)/width  (dx written out for the P.dx GEMV)
 * out[0] = ||du||^2, out[1] = box support S(du) (finite part), out[2] = #inf terms,
 * out[3] = ||dx||^2, out[4] = dist(dx, recession cone)^2, out[5] = q . dx */
int nys_qp_infeas_f64(int64_t n, const double* xa, const double* xb, const double* ua,
                      const double* ub, double width, const double* lo, const double* hi,
                      const double* q, double* dx, double* out, void* ws, void* stream);
/* elementwise helpers used by the operator API */
int nys_axpby_f64(int64_t n, double a, const double* x, double b, double* y, void* stream);
int nys_soft_threshold_f64(int64_t n, const double* v, double kappa, double* out, void* stream);
/* out[i] = the loss (NYS_LOSS_*) evaluated elementwise at w[i]: what = 0 value,
 * 1 first derivative, 2 second derivative, 3 convex conjugate (+inf outside its
 * domain) -- the callables of the reference's Loss (problems.py:35-111). */
int nys_loss_eval_f64(int loss, int what, int64_t n, const double* w, double* out, void* stream);
int nys_box_project_f64(int64_t n, const double* v, const double* lo, const double* hi,
                        double* out, void* stream);
int nys_row_scale_f64(int64_t rows, int64_t cols, double* X, int64_t ldx, const double* d,
                      void* stream);

/* ------------------------------------------------------ K5 Nystrom sketch -- */
/* C = alpha op(A) op(B) + beta C (row-major; trans = 1 means op(X) = X^T),
 * FP64 DMMA (mma.sync m8n8k4) tiles; split-K with a deterministic reduction
 * when M*N is small.  Used for Y = A Omega and A^T (D A Omega) (sketch.py:100). */
size_t nys_gemm_workspace(int64_t M, int64_t N, int64_t K);
int nys_gemm_f64(int transA, int transB, int64_t M, int64_t N, int64_t K, double alpha,
                 const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
                 double* C, int64_t ldc, void* ws, size_t ws_bytes, void* stream);
/* Tuning / test hook of nys_gemm_f64's planner: every later call uses CTA tile
 * shape `shape` (0 .. count-1; split-K still planned), -1 restores the cost
 * model's choice.  Returns the number of tile shapes. */
int nys_gemm_tile(int shape);
/* The raw Gaussian test matrix itself (sketch.py:97-98): fills out[0..count)
 * with exactly np.random.Generator(PCG64).standard_normal(count) continued
 * from the given 128-bit PCG64 (state, inc) -- for default_rng(seed) that is
 * np.random.PCG64(seed).state.  PCG64 jump-ahead + NumPy's ziggurat with a
 * parallel resolution of the variable draw consumption.  Synchronises `stream`;
 * returns NYS_ERR_NONFINITE if the draw buffer was exhausted (never expected). */
/* Asynchronous variants for a pipelined sketch: no host synchronisation; a
 * failure is reported in a device status word instead (nonzero = re-run the
 * synchronous function): the draw buffer ran short / a Cholesky pivot of a
 * CholeskyQR pass (2 words) / of the core (1 word).  The sketch's rank is
 * then min(r, s). */
int nys_gaussian_async_f64(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t count,
                           double* out, int* flag_dev, void* ws, size_t ws_bytes, void* stream);
int nys_orthonormalize_async_f64(int64_t n, int s, const double* Omega, double* Q, int* info_dev, void* ws,
                                 size_t ws_bytes, void* stream);
int nys_nystrom_core_async_f64(int64_t n, int s, int r, const double* Q, double* Y, double* U, double* lam,
                               int* info_dev, void* ws, size_t ws_bytes, void* stream);
size_t nys_gaussian_workspace(int64_t count);
int nys_gaussian_f64(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                     int64_t count, double* out, void* ws, size_t ws_bytes, void* stream);
/* Same stream, and *draws = the number of 64-bit PCG64 draws the `count`
 * samples consumed, so a long stream (config 5's 2.5e9-sample row blocks,
 * datagen.cfg5_block / bench/datagen.py:28-137 conventions) is generated in
 * pieces: the next piece starts from the state advanced by *draws. */
int nys_gaussian_draws_f64(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                           int64_t count, double* out, void* ws, size_t ws_bytes, int64_t* draws,
                           void* stream);
/* Orthonormalise the raw Gaussian test matrix (sketch.py:97-99) by CholeskyQR2:
 * Q (n x s, row-major) spans the same range as Omega.  Synchronises `stream`. */
size_t nys_orthonormalize_workspace(int64_t n, int s);
int nys_orthonormalize_f64(int64_t n, int s, const double* Omega, double* Q, void* ws,
                           size_t ws_bytes, void* stream);
/* Everything of nystrom_sketch after Y = A Q (sketch.py:102-128): trace-shift,
 * core = Q^T Y_s, Cholesky (eigh fallback), B = Y_s L^-T, thin SVD of B via a
 * Jacobi eigensolver of B^T B, lam = max(sv^2 - shift, 0), truncation to r.
 * Y is destroyed.  Writes U (n x r_out, row-major, ld = r) and lam (r_out) and
 * the HOST int *r_out (may be < r on the eigh path, 0 for an empty sketch).
 * Returns NYS_ERR_NOT_PSD for a clearly indefinite core.  Synchronises `stream`. */
size_t nys_nystrom_workspace(int64_t n, int s, int r);
int nys_nystrom_core_f64(int64_t n, int s, int r, const double* Q, double* Y, double* U,
                         double* lam, int* r_out, void* ws, size_t ws_bytes, void* stream);
/* small symmetric eigensolver (one-sided Jacobi, cooperative grid): on exit the
 * columns of V (s x s row-major) are eigenvectors, w the eigenvalues sorted in
 * DESCENDING order.  A is destroyed.  Synchronises `stream`. */
size_t nys_syevj_workspace(int s);
int nys_syevj_f64(int s, double* A, double* V, double* w, void* ws, size_t ws_bytes,
                  void* stream);

/* Workspace (bytes) of nys_admm_tail_f64's ws_gemvT when the rows are wide
 * (n > 12800): the one-pass cluster tail keeps per-cluster A^T partials there. */
size_t nys_tail_cluster_workspace(int64_t rows, int64_t n);
/* The one-pass ML tail of nys_admm_tail_f64 on its own (admm.py:585-587,
 * problems.py:227-351): T = [l'(Ax-b), w o Ax, l'(Az-b)] (3 x rows, row-major),
 * w = l''(Ax-b), AT = A^T T (3 x n; 2 x n when z is NULL), rowsums[0..4] as
 * nys_ml_rowwise_f64.  ws: nys_tail_cluster_workspace bytes.  Returns
 * NYS_ERR_UNSUPPORTED for shapes without a cluster plan (n <= 12800). */
int nys_ml_tail_f64(const double* A, int64_t rows, int64_t n, int64_t lda, const double* x, const double* z,
                    const double* b, int loss, double* T, double* w, double* AT, double* rowsums, void* ws,
                    size_t ws_bytes, void* stream);
/* The same with g_b = A^T b (n): for the square loss with z the cluster stream
 * then accumulates A^T (A x) and A^T (A z) only (two products instead of three)
 * and AT = [A^T(Ax) - g_b, A^T(Ax), A^T(Az) - g_b]; other losses ignore g_b.
 * With g_b, rows beyond the whole-slice plan (114688 < n <= ~229000, config 5's
 * n = 200000) have their own one-pass plan (x and the A^T(Az) accumulator in
 * tensor memory, z visited through its nonzeros: meant for a sparse prox output;
 * a dense z stays correct but is slower than two passes). */
int nys_ml_tail_gb_f64(const double* A, int64_t rows, int64_t n, int64_t lda, const double* x, const double* z,
                       const double* b, int loss, const double* gb, double* T, double* w, double* AT,
                       double* rowsums, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------- sparse / general-operator engine -- */
/* CSR data operator (SparseOperator._apply, operators.py:129-131 -- scipy's
 * `a @ v`): row pointer int64 (rows+1), column indices int32, values FP64.
 *   y_i = alpha * s_i * (a_i . x) + beta * zin_i,  s = dscale (NULL: 1);
 *   beta == 0 ignores zin (which may alias y).  `group` = lanes per row, a power
 *   of two <= 32 (the host picks it from the mean row length).
 * The adjoint (operators.py:133-134, `a.T @ u`) is the same call on the
 * transpose built by nys_csr_transpose. */
int nys_csr_spmv_f64(int64_t rows, const int64_t* rowptr, const int* col, const double* val,
                     const double* x, double alpha, const double* dscale, double beta, const double* zin,
                     double* y, int group, void* stream);
/* Y = diag(s) A X for a row-major cols x s block X (the sketch's column
 * applies, sketch.py:69-71, done as one multi-column product). */
int nys_csr_spmm_f64(int64_t rows, const int64_t* rowptr, const int* col, const double* val,
                     const double* X, int64_t ldx, int s, const double* dscale, double* Y, int64_t ldy,
                     void* stream);
/* CSR of A^T on the device (deterministic counting transpose: the entries of
 * every transposed row are ordered by original row).  trowptr has cols+1
 * entries, tcol / tval nnz.  The workspace need not be zeroed. */
size_t nys_csr_transpose_workspace(int64_t rows, int64_t cols);
int nys_csr_transpose(int64_t rows, int64_t cols, const int64_t* rowptr, const int* col, const double* val,
                      int64_t* trowptr, int* tcol, double* tval, void* ws, size_t ws_bytes, void* stream);
/* y = a (d o x) + b y  (DiagonalOperator, DiagPlusLowRank's diagonal,
 * operators.py:89-101, 152-153) */
int nys_vmul_f64(int64_t n, double a, const double* d, const double* x, double b, double* y, void* stream);
/* y[:] = scale * src[0] (OnesRowOperator adjoint, operators.py:202-203) */
int nys_bcast_f64(int64_t n, const double* src, double scale, double* y, void* stream);
/* v = x - y (y may be NULL): out = [sum v, sum v^2, max |v|]  (the l2 / linf
 * norms of admm.py:203-208; OnesRowOperator apply = out[0]) */
int nys_vstats_f64(int64_t n, const double* x, const double* y, double* out, void* ws, void* stream);
/* l1 norm and dual-norm pieces (g(z) = lambda1 ||z||_1, problems.py:308-331):
 *   out = [sum |v|, sum (|v| - lambda1)_+^2, max |v|] */
int nys_absstats_f64(int64_t n, const double* v, double lambda1, double* out, void* ws, void* stream);
/* dual residual of admm.py:219-222 with a general M: t = rho * Mtu,
 * rd = grad + t;  out = [sum rd^2, sum t^2, max |rd|, max |t|] */
int nys_gdual_f64(int64_t n, const double* grad, const double* mtu, double rho, double* out, void* ws,
                  void* stream);
/* box certificates of check_infeasibility (admm.py:386-396, prox.py:96-135):
 *   du (may be NULL): out[0] = sum_{du>0} hi du, out[1] = sum_{du<0} lo du,
 *                     out[2] = number of (infinite bound x nonzero) terms;
 *   md (may be NULL): out[3] = ||md - proj_recession(md)||^2 */
int nys_box_cert_f64(int64_t m, const double* du, const double* md, const double* lo, const double* hi,
                     double* out, void* ws, void* stream);
/* box membership (box_indicator, prox.py:138-144):
 *   out = [max(lo - z), max(z - hi), max |z|] */
int nys_box_violation_f64(int64_t m, const double* z, const double* lo, const double* hi, double* out,
                          void* ws, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* NYSGPU_H */
