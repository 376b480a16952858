// Shared helpers for the libnysgpu kernels (sm_100a, FP64 throughout).
//
// Reductions are deterministic: every kernel that reduces writes one partial
// per CTA and the last CTA to finish (atomic ticket) sums the partials in a
// fixed order, so results are bitwise reproducible run to run (the reference
// pins bitwise trajectory determinism, tests/test_admm.py:476-484).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <utility>
#include "../../include/nysgpu.h"

namespace nys {
// Number of kernels this library has launched (reported as gpu_launches).
extern unsigned long long g_launches;

// Development switches (the NYS_* environment variables of DESIGN.md §5: forced
// plans and rejected variants for A/B measurements) exist only in a library
// built with -DNYS_DEV_SWITCHES (NYS_DEV_SWITCHES=1 python -m ...build -f).
// The product build reads no environment: every plan is the measured-best one.
#ifdef NYS_DEV_SWITCHES
inline const char* dev_env(const char* name) { return getenv(name); }
#else
inline const char* dev_env(const char*) { return nullptr; }
#endif
}

namespace nys {
// NYS_SYNC_DEBUG=1: synchronise after every launch and report the failing site
int debug_sync_check(const char* file, int line);
void debug_report(cudaError_t e, const char* file, int line);
}

#define NYS_CHECK_LAUNCH()                                   \
  do {                                                       \
    __atomic_fetch_add(&nys::g_launches, 1ull, __ATOMIC_RELAXED); \
    cudaError_t _e = cudaGetLastError();                     \
    if (_e != cudaSuccess) {                                 \
      nys::debug_report(_e, __FILE__, __LINE__);             \
      return NYS_ERR_CUDA;                                   \
    }                                                        \
    if (nys::debug_sync_check(__FILE__, __LINE__)) return NYS_ERR_CUDA; \
  } while (0)

namespace nys {

constexpr int kWarp = 32;
// B200: the grid sizes of the streaming kernels and the slice layout of the
// one-CTA-per-SM cooperative kernels are compiled for 148 SMs.  On a device
// (or an MPS / green-context share) with fewer SMs the non-cooperative kernels
// still run correctly (more waves); the cooperative plans check co-residency
// at launch (coop_fits) and report NYS_ERR_UNSUPPORTED so callers take their
// non-cooperative plan.
constexpr int kNumSMs = 148;

// SM count of the current device (cached per device ordinal)
inline int device_sm_count() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  static int cache[64] = {0};
  if (dev >= 0 && dev < 64 && cache[dev]) return cache[dev];
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    v = 0;
  }
  if (dev >= 0 && dev < 64) cache[dev] = v;
  return v;
}

// Can `grid` CTAs of `fn` (threads, dynamic smem) all be resident at once, as a
// cooperative launch requires?  (The max-dynamic-smem attribute must be set.)
inline bool coop_fits(const void* fn, int64_t grid, int threads, size_t smem) {
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return (int64_t)occ * device_sm_count() >= grid;
}

// Status of a failed cooperative launch: a grid that does not fit (fewer free
// SMs than planned) is UNSUPPORTED so the caller falls back; the sticky-free
// launch error is cleared so it is not blamed on the next kernel.
inline int coop_launch_status(cudaError_t e) {
  if (e == cudaSuccess) return NYS_OK;
  cudaGetLastError();
  return (e == cudaErrorCooperativeLaunchTooLarge || e == cudaErrorInvalidConfiguration) ? NYS_ERR_UNSUPPORTED
                                                                                         : NYS_ERR_CUDA;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum of NV values per thread; result valid in thread 0.
// `sh` must hold NV * (blockDim/32) doubles.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int j = 0; j < NV; ++j) v[j] = warp_sum(v[j]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int j = 0; j < NV; ++j) sh[j * nw + wid] = v[j];
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      double t = lane < nw ? sh[j * nw + lane] : 0.0;
      v[j] = warp_sum(t);
    }
  }
  __syncthreads();
}

template <int NV>
__device__ __forceinline__ void block_max(double (&v)[NV], double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int j = 0; j < NV; ++j) v[j] = warp_max(v[j]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int j = 0; j < NV; ++j) sh[j * nw + wid] = v[j];
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      double t = lane < nw ? sh[j * nw + lane] : 0.0;
      v[j] = warp_max(t);
    }
  }
  __syncthreads();
}

// Last-block-done ticket.  Returns true in exactly one CTA (all threads of
// it), after every CTA has published its partials.  The counter is reset by
// the winner so the same workspace can be reused by the next launch.
__device__ __forceinline__ bool last_block(unsigned int* counter) {
  __shared__ bool am_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int t = atomicAdd(counter, 1u);
    am_last = (t == gridDim.x * gridDim.y * gridDim.z - 1);
  }
  __syncthreads();
  if (am_last) {
    __threadfence();
    if (threadIdx.x == 0) *counter = 0u;
  }
  return am_last;
}

// Fixed-order sum of `cnt` partials laid out with stride `stride`, by one CTA.
// Each thread sums a strided subset in order, then a block tree; the result is
// deterministic for fixed (cnt, blockDim).
__device__ __forceinline__ double block_sum_partials(const double* p, int cnt, int stride,
                                                     double* sh) {
  double v[1] = {0.0};
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) v[0] += p[(size_t)i * stride];
  block_sum<1>(v, sh);
  return v[0];
}

__device__ __forceinline__ double block_max_partials(const double* p, int cnt, int stride,
                                                     double* sh) {
  double v[1] = {0.0};
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) v[0] = fmax(v[0], p[(size_t)i * stride]);
  block_max<1>(v, sh);
  return v[0];
}

template <class T>
__host__ __device__ __forceinline__ T tmin(T a, T b) { return a < b ? a : b; }
template <class T>
__host__ __device__ __forceinline__ T tmax(T a, T b) { return a > b ? a : b; }

__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Programmatic dependent launch (PDL) for the per-iteration kernel chain
// (x-update -> A{x,z} -> A^T -> epilogue -> conj -> gate -> readback -> next
// x-update).  A chain kernel starts with pdl_begin(): it lets its successor be
// scheduled as soon as all of its own CTAs are resident, then waits until its
// predecessor has completed and its memory is visible (griddepcontrol.wait),
// so the successor's launch latency and CTA ramp-up hide behind this kernel's
// tail.  Both instructions are no-ops for kernels launched without the
// attribute.  NYS_PDL=0 disables the attribute.
__device__ __forceinline__ void pdl_begin() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

inline bool pdl_enabled() {
  static const bool on = !(dev_env("NYS_PDL") && dev_env("NYS_PDL")[0] == '0');
  return on;
}

// launch `kern` with the PDL attribute (and the cooperative one when coop)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_chain(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                bool coop, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  unsigned na = 0;
  if (pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (coop) {
    at[na].id = cudaLaunchAttributeCooperative;
    at[na].val.cooperative = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace nys
