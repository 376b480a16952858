// Exact on-GPU reproduction of np.random.default_rng(seed).standard_normal(count)
// (the Nystrom test matrix of sketch.py:97-98).
//
// NumPy's stream is PCG64 (128-bit LCG, XSL-RR output) feeding a 256-layer
// ziggurat that usually consumes one 64-bit draw per sample but occasionally
// more (wedge / tail rejections), so the sample -> draw mapping is not known in
// advance.  The GPU version:
//   K1  raw[q] for q < Q: each thread jumps its PCG64 state to q = t + 1 steps
//       and then strides by T threads with the precomputed LCG power (coalesced);
//   K2  for every q: the ziggurat evaluated as if a sample started at q ->
//       consumption L[q] (draws) and value V[q];
//   K3  per 64-draw chunk and per entry offset e < E: walk q -> q + L[q] to the
//       chunk exit (offset into the next chunk) and count samples; per 16384-draw
//       tile, compose the 256 chunk maps;
//   K4  resolve the tile entries sequentially (a few thousand tiles at most);
//   K5  per tile: resolve chunk entries and sample bases, then every chunk
//       writes its samples V[q] to out[base + j].
// Chains from different entry offsets merge after one step with probability
// ~0.99, so E = 4 covers almost every boundary; larger offsets fall back to a
// direct walk.  Values equal NumPy's bit for bit except where CUDA's exp/log1p
// differ from glibc's by an ulp on the rare rejection paths (tested).
#include <math.h>
#include "common.cuh"
#include "zig_tables.h"

namespace nys {

typedef unsigned __int128 u128;

constexpr int kChunk = 64;
constexpr int kChunksPerTile = 256;
constexpr int kTile = kChunk * kChunksPerTile;  // 16384 draws
constexpr int kE = 4;
constexpr uint8_t kUnknown = 0xFF;

__host__ __device__ inline u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
}

__device__ __forceinline__ uint64_t pcg_output(u128 s) {
  const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
  const unsigned rot = (unsigned)(s >> 122);
  return (x >> rot) | (x << ((64 - rot) & 63));
}

// LCG jump: (mult, plus) such that advancing by `delta` steps is s -> mult*s + plus
__host__ __device__ inline void pcg_jump(u128 delta, u128 inc, u128& mult, u128& plus) {
  u128 cur_mult = pcg_mult(), cur_plus = inc, acc_mult = 1, acc_plus = 0;
  while (delta > 0) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  mult = acc_mult;
  plus = acc_plus;
}

struct U128 {
  uint64_t hi, lo;
};
__host__ __device__ inline u128 mk(U128 v) { return ((u128)v.hi << 64) | v.lo; }
__host__ __device__ inline U128 sp(u128 v) { return U128{(uint64_t)(v >> 64), (uint64_t)v}; }

__global__ void pcg_raw_kernel(U128 state0, U128 inc, U128 jmul, U128 jplus, int64_t Q,
                               uint64_t* __restrict__ raw) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  if (t >= Q) return;
  u128 m, p;
  pcg_jump((u128)(t + 1), mk(inc), m, p);
  u128 s = m * mk(state0) + p;  // state after t + 1 steps -> draw index t
  const u128 A = mk(jmul), C = mk(jplus);
  for (int64_t q = t; q < Q; q += T) {
    raw[q] = pcg_output(s);
    s = A * s + C;
  }
}

__device__ __forceinline__ double to_double(uint64_t r) {
  return (double)(r >> 11) * (1.0 / 9007199254740992.0);
}

// ziggurat of NumPy's random_standard_normal started at draw q; returns the
// number of draws consumed (0 if the raw buffer ends first).
__device__ int zig_at(const uint64_t* __restrict__ raw, int64_t q, int64_t Q, double* val) {
  const double zr = 3.6541528853610087963519472518;
  const double zinv = 0.27366123732975827203338247596;
  int64_t pos = q;
  for (;;) {
    if (pos >= Q) return 0;
    uint64_t r = raw[pos++];
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const int sign = (int)(r & 1);
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = (double)rabs * kZigWi[idx];
    if (sign) x = -x;
    if (rabs < kZigKi[idx]) {
      *val = x;
      return (int)(pos - q);
    }
    if (idx == 0) {
      for (;;) {
        if (pos + 1 >= Q) return 0;
        const double xx = -zinv * log1p(-to_double(raw[pos++]));
        const double yy = -log1p(-to_double(raw[pos++]));
        if (yy + yy > xx * xx) {
          *val = ((rabs >> 8) & 1) ? -(zr + xx) : zr + xx;
          return (int)(pos - q);
        }
      }
    } else {
      if (pos >= Q) return 0;
      const double u = to_double(raw[pos++]);
      if ((kZigFi[idx - 1] - kZigFi[idx]) * u + kZigFi[idx] < exp(-0.5 * x * x)) {
        *val = x;
        return (int)(pos - q);
      }
    }
    if (pos - q > 250) return 0;  // pathological chain: treat as unknown
  }
}

__global__ void zig_eval_kernel(const uint64_t* __restrict__ raw, int64_t Q, uint8_t* __restrict__ L,
                                double* __restrict__ V) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Q;
       q += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    const int l = zig_at(raw, q, Q, &v);
    L[q] = l > 0 ? (uint8_t)l : kUnknown;
    V[q] = v;
  }
}

// walk q -> q + L[q] from `start` while q < end; returns exit position (>= end)
// and the number of sample starts visited; -1 exit on an unknown consumption.
__device__ __forceinline__ int64_t walk(const uint8_t* __restrict__ L, int64_t start, int64_t end,
                                        int* count) {
  int64_t q = start;
  int c = 0;
  while (q < end) {
    const uint8_t l = L[q];
    if (l == kUnknown) {
      *count = c;
      return -1;
    }
    ++c;
    q += l;
  }
  *count = c;
  return q;
}

struct TileMap {
  int exit[kE];  // entry offset into the next tile, -1 unknown
  int cnt[kE];
};

// walk within a shared-memory copy of the tile's consumptions (positions
// relative to the tile start)
__device__ __forceinline__ int walk_s(const uint8_t* __restrict__ Ls, int start, int end, int* count) {
  int q = start, c = 0;
  while (q < end) {
    const uint8_t l = Ls[q];
    if (l == kUnknown) {
      *count = c;
      return -1;
    }
    ++c;
    q += l;
  }
  *count = c;
  return q;
}

// K3: chunk maps and their composition into a tile map (the tile's L staged
// in shared memory: the walks are dependent load chains)
__global__ void __launch_bounds__(kChunksPerTile)
tile_map_kernel(const uint8_t* __restrict__ L, int64_t Q, TileMap* __restrict__ tiles,
                int* __restrict__ chunk_exit, int* __restrict__ chunk_cnt) {
  __shared__ int ex[kChunksPerTile][kE];
  __shared__ int cn[kChunksPerTile][kE];
  __shared__ uint8_t Ls[kTile + 256];
  const int64_t tile0 = (int64_t)blockIdx.x * kTile;
  const int tlen = (int)tmin<int64_t>(kTile, Q - tile0);
  for (int q = threadIdx.x; q < kTile + 256; q += blockDim.x) Ls[q] = q < tlen ? L[tile0 + q] : kUnknown;
  __syncthreads();
  const int c = threadIdx.x;
  const int cs = c * kChunk;
  const int ce = tmin(cs + kChunk, tlen);
  for (int e = 0; e < kE; ++e) {
    int cnt = 0;
    int x;
    if (cs + e < tlen) {
      x = walk_s(Ls, cs + e, ce, &cnt);
    } else {
      x = cs + e;
      cnt = 0;
    }
    ex[c][e] = x < 0 ? -1 : x - ce;
    cn[c][e] = cnt;
    chunk_exit[((int64_t)blockIdx.x * kChunksPerTile + c) * kE + e] = ex[c][e];
    chunk_cnt[((int64_t)blockIdx.x * kChunksPerTile + c) * kE + e] = cnt;
  }
  __syncthreads();
  if (c < kE) {
    int e = c, total = 0;
    bool bad = false;
    for (int k = 0; k < kChunksPerTile && !bad; ++k) {
      const int ks = k * kChunk;
      if (ks >= tlen) break;
      const int ke_ = tmin(ks + kChunk, tlen);
      int nx, nc;
      if (e < kE) {
        nx = ex[k][e];
        nc = cn[k][e];
      } else {
        int cnt = 0;
        const int x = ks + e < kTile + 256 ? walk_s(Ls, ks + e, ke_, &cnt) : -1;
        nx = x < 0 ? -1 : x - ke_;
        nc = cnt;
      }
      if (nx < 0) bad = true;
      total += nc;
      e = nx;
    }
    tiles[blockIdx.x].exit[c] = bad ? -1 : e;
    tiles[blockIdx.x].cnt[c] = total;
  }
}

// K4: sequential resolution of tile entries and sample bases (one thread)
__global__ void tile_resolve_kernel(const TileMap* __restrict__ tiles, const uint8_t* __restrict__ L,
                                    int64_t ntiles, int64_t Q, int* __restrict__ tile_entry,
                                    int64_t* __restrict__ tile_base, int64_t* __restrict__ total) {
  // stage the tile maps in shared memory (coalesced), then one thread chains them
  extern __shared__ TileMap tm_s[];
  for (int64_t t = threadIdx.x; t < ntiles; t += blockDim.x) tm_s[t] = tiles[t];
  __syncthreads();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int e = 0;
  int64_t base = 0;
  for (int64_t t = 0; t < ntiles; ++t) {
    tile_entry[t] = e;
    tile_base[t] = base;
    if (e < 0) continue;
    if (e < kE) {
      const TileMap m = tm_s[t];
      base += m.cnt[e];
      e = m.exit[e];
    } else {
      const int64_t ts = t * kTile, te = tmin<int64_t>(ts + kTile, Q);
      int cnt = 0;
      const int64_t x = walk(L, ts + e, te, &cnt);
      base += cnt;
      e = x < 0 ? -1 : (int)(x - te);
    }
  }
  *total = base;  // samples resolved before the buffer end (or an unknown draw)
}

// K5: per tile, resolve chunk entries (thread 0) then write samples
__global__ void __launch_bounds__(kChunksPerTile)
tile_write_kernel(const uint8_t* __restrict__ L, const double* __restrict__ V, int64_t Q,
                  const int* __restrict__ chunk_exit, const int* __restrict__ chunk_cnt,
                  const int* __restrict__ tile_entry, const int64_t* __restrict__ tile_base,
                  int64_t count, double* __restrict__ out, int64_t* __restrict__ consumed) {
  __shared__ int entry[kChunksPerTile];
  __shared__ int64_t base[kChunksPerTile];
  __shared__ int cx_s[kChunksPerTile * kE];
  __shared__ int cc_s[kChunksPerTile * kE];
  const int64_t tile0 = (int64_t)blockIdx.x * kTile;
  for (int q = threadIdx.x; q < kChunksPerTile * kE; q += blockDim.x) {
    cx_s[q] = chunk_exit[(int64_t)blockIdx.x * kChunksPerTile * kE + q];
    cc_s[q] = chunk_cnt[(int64_t)blockIdx.x * kChunksPerTile * kE + q];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int e = tile_entry[blockIdx.x];
    int64_t b = tile_base[blockIdx.x];
    for (int k = 0; k < kChunksPerTile; ++k) {
      entry[k] = e;
      base[k] = b;
      const int64_t ks = tile0 + (int64_t)k * kChunk;
      if (e < 0 || ks >= Q) {
        e = -1;
        continue;
      }
      const int64_t ke_ = tmin<int64_t>(ks + kChunk, Q);
      if (e < kE) {
        const int ci = k * kE + e;
        b += cc_s[ci];
        e = cx_s[ci];
      } else {
        int cnt = 0;
        const int64_t x = walk(L, ks + e, ke_, &cnt);
        b += cnt;
        e = x < 0 ? -1 : (int)(x - ke_);
      }
    }
  }
  __syncthreads();
  const int c = threadIdx.x;
  const int e = entry[c];
  if (e < 0) return;
  const int64_t cs = tile0 + (int64_t)c * kChunk;
  const int64_t ce = tmin<int64_t>(cs + kChunk, Q);
  int64_t q = cs + e, j = base[c];
  while (q < ce && j < count) {
    const uint8_t l = L[q];
    if (l == kUnknown) break;
    out[j++] = V[q];
    q += l;
    // the thread writing the last sample records the draws it ended at: the
    // stream continues there (pieces of one long stream chain exactly)
    if (j == count && consumed) *consumed = q;
  }
}

struct GaussPlan {
  int64_t Q, ntiles;
  size_t off_raw, off_V, off_L, off_cx, off_cc, off_tiles, off_te, off_tb, off_total, bytes;
};

static GaussPlan gauss_plan(int64_t count) {
  GaussPlan p;
  p.Q = count + count / 32 + 4 * kTile;
  p.ntiles = cdiv(p.Q, kTile);
  p.Q = p.ntiles * kTile;
  size_t off = 0;
  auto take = [&](size_t b) {
    off = (off + 255) & ~size_t(255);
    const size_t o = off;
    off += b;
    return o;
  };
  p.off_raw = take(p.Q * 8);
  p.off_V = take(p.Q * 8);
  p.off_L = take(p.Q);
  p.off_cx = take(p.ntiles * kChunksPerTile * kE * 4);
  p.off_cc = take(p.ntiles * kChunksPerTile * kE * 4);
  p.off_tiles = take(p.ntiles * sizeof(TileMap));
  p.off_te = take(p.ntiles * 4);
  p.off_tb = take(p.ntiles * 8);
  p.off_total = take(16);  // [total samples resolved, draws consumed by `count` samples]
  p.bytes = off + 256;
  return p;
}

}  // namespace nys

using namespace nys;

extern "C" size_t nys_gaussian_workspace(int64_t count) { return gauss_plan(count).bytes; }

// flag = 1 when the draw buffer held fewer than `count` accepted normals
__global__ void gauss_flag_kernel(const int64_t* total, int64_t count, int* flag) {
  if (threadIdx.x == 0 && *total < count) *flag = 1;
}

static int gaussian_impl(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t count,
                         double* out, int* flag_dev, void* ws, size_t ws_bytes, cudaStream_t st,
                         int64_t* draws = nullptr);

extern "C" int nys_gaussian_draws_f64(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                                      int64_t count, double* out, void* ws, size_t ws_bytes, int64_t* draws,
                                      void* stream) {
  if (count <= 0 || !draws) return NYS_ERR_ARG;
  return gaussian_impl(state_hi, state_lo, inc_hi, inc_lo, count, out, nullptr, ws, ws_bytes, as_stream(stream),
                       draws);
}

extern "C" int nys_gaussian_async_f64(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                                      int64_t count, double* out, int* flag_dev, void* ws, size_t ws_bytes,
                                      void* stream) {
  if (count <= 0 || !flag_dev) return NYS_ERR_ARG;
  return gaussian_impl(state_hi, state_lo, inc_hi, inc_lo, count, out, flag_dev, ws, ws_bytes, as_stream(stream));
}

extern "C" int nys_gaussian_f64(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                                uint64_t inc_lo, int64_t count, double* out, void* ws,
                                size_t ws_bytes, void* stream) {
  if (count <= 0) return NYS_ERR_ARG;
  return gaussian_impl(state_hi, state_lo, inc_hi, inc_lo, count, out, nullptr, ws, ws_bytes, as_stream(stream));
}

static int gaussian_impl(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t count,
                         double* out, int* flag_dev, void* ws, size_t ws_bytes, cudaStream_t st,
                         int64_t* draws) {
  const GaussPlan p = gauss_plan(count);
  if (ws_bytes < p.bytes) return NYS_ERR_WORKSPACE;
  char* w = reinterpret_cast<char*>(ws);
  uint64_t* raw = reinterpret_cast<uint64_t*>(w + p.off_raw);
  double* V = reinterpret_cast<double*>(w + p.off_V);
  uint8_t* L = reinterpret_cast<uint8_t*>(w + p.off_L);
  int* cx = reinterpret_cast<int*>(w + p.off_cx);
  int* cc = reinterpret_cast<int*>(w + p.off_cc);
  TileMap* tiles = reinterpret_cast<TileMap*>(w + p.off_tiles);
  int* te = reinterpret_cast<int*>(w + p.off_te);
  int64_t* tb = reinterpret_cast<int64_t*>(w + p.off_tb);
  int64_t* total = reinterpret_cast<int64_t*>(w + p.off_total);

  const int threads = 256;
  const int64_t T = tmin<int64_t>((int64_t)kNumSMs * 8 * threads, p.Q);
  const int blocks = (int)cdiv(T, threads);
  const int64_t Treal = (int64_t)blocks * threads;
  u128 jm, jp;
  pcg_jump((u128)Treal, ((u128)inc_hi << 64) | inc_lo, jm, jp);
  pcg_raw_kernel<<<blocks, threads, 0, st>>>(U128{state_hi, state_lo}, U128{inc_hi, inc_lo}, sp(jm),
                                             sp(jp), p.Q, raw);
  NYS_CHECK_LAUNCH();
  zig_eval_kernel<<<(unsigned)tmin<int64_t>(cdiv(p.Q, 256), kNumSMs * 16), 256, 0, st>>>(raw, p.Q, L, V);
  NYS_CHECK_LAUNCH();
  tile_map_kernel<<<(unsigned)p.ntiles, kChunksPerTile, 0, st>>>(L, p.Q, tiles, cx, cc);
  NYS_CHECK_LAUNCH();
  const size_t rsm = (size_t)p.ntiles * sizeof(TileMap);
  if (rsm > 48 * 1024) {
    if (rsm > 220 * 1024) return NYS_ERR_UNSUPPORTED;
    cudaFuncSetAttribute(tile_resolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm);
  }
  tile_resolve_kernel<<<1, 256, rsm, st>>>(tiles, L, p.ntiles, p.Q, te, tb, total);
  NYS_CHECK_LAUNCH();
  tile_write_kernel<<<(unsigned)p.ntiles, kChunksPerTile, 0, st>>>(L, V, p.Q, cx, cc, te, tb, count, out,
                                                                    total + 1);
  NYS_CHECK_LAUNCH();
  if (flag_dev) {  // deferred check (the caller reads the flag with its next sync)
    gauss_flag_kernel<<<1, 32, 0, st>>>(total, count, flag_dev);
    NYS_CHECK_LAUNCH();
    return NYS_OK;
  }
  int64_t tot2[2] = {0, 0};
  if (cudaMemcpyAsync(tot2, total, 16, cudaMemcpyDeviceToHost, st) != cudaSuccess) return NYS_ERR_CUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return NYS_ERR_CUDA;
  const int64_t tot = tot2[0];
  if (draws) *draws = tot2[1];
  // the margin (3%) is ~400 standard deviations above the expected rejection
  // count; an exhausted buffer would mean a broken stream, not bad luck
  return (tot >= count) ? NYS_OK : NYS_ERR_NONFINITE;
}
