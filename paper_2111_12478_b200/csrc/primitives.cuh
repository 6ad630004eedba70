// Device-wide primitives for the G-WCP pipeline, hand-written for sm_100a:
//   * a reduce-then-scan exclusive/inclusive scan over a user load/store functor
//   * a stable LSD radix sort (8-bit digits) of (u32|u64 key, u32 value) pairs
// Both are HBM-streaming kernels: 256-thread CTAs, 16 items per thread, grids
// sized in tiles so a 1e9-element pass fills all 148 SMs many times over.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace gw {

constexpr int kThreads = 256;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;  // 4096

// launch accounting (gw_ctx_launches); incremented on the host per launch
extern thread_local uint32_t g_launches;
#define GW_LAUNCH(kernel, grid, block, smem, stream, ...)      \
  do {                                                         \
    kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__); \
    ::gw::g_launches++;                                        \
  } while (0)

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---------------------------------------------------------------- scan ----
struct OpSum {
  template <class T>
  __device__ __forceinline__ T operator()(const T& a, const T& b) const { return a + b; }
};

template <class T>
__device__ __forceinline__ T shfl_up(T v, int o) { return __shfl_up_sync(0xffffffffu, v, o); }
template <>
__device__ __forceinline__ uint2 shfl_up<uint2>(uint2 v, int o) {
  return make_uint2(__shfl_up_sync(0xffffffffu, v.x, o), __shfl_up_sync(0xffffffffu, v.y, o));
}

// warp-inclusive scan via shuffles
template <class T, class Op>
__device__ __forceinline__ T warp_incl_scan(T v, Op op) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = shfl_up(v, o);
    if (lane >= o) v = op(n, v);
  }
  return v;
}

// block-exclusive scan of one value per thread; returns exclusive prefix, sets *total
template <class T, class Op>
__device__ __forceinline__ T block_excl_scan(T v, Op op, T identity, T* total) {
  __shared__ T s_w[kThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T inc = warp_incl_scan(v, op);
  if (lane == 31) s_w[w] = inc;
  __syncthreads();
  if (w == 0) {
    T x = lane < kThreads / 32 ? s_w[lane] : identity;
    T xi = warp_incl_scan(x, op);
    if (lane < kThreads / 32) s_w[lane] = xi;
  }
  __syncthreads();
  T wpre = w > 0 ? s_w[w - 1] : identity;
  *total = s_w[kThreads / 32 - 1];
  T exc = shfl_up(inc, 1);
  if (lane == 0) exc = identity;
  __syncthreads();
  return op(wpre, exc);
}

template <class T, class Op, class Load>
__global__ void __launch_bounds__(kThreads) k_scan_reduce(Load load, uint64_t n, T* aggs, Op op, T identity) {
  const uint64_t base = (uint64_t)blockIdx.x * kTile;
  T acc = identity;
#pragma unroll
  for (int k = 0; k < kItems; k++) {
    uint64_t i = base + (uint64_t)k * kThreads + threadIdx.x;
    if (i < n) acc = op(acc, load(i));
  }
  T tot;
  block_excl_scan<T, Op>(acc, op, identity, &tot);
  if (threadIdx.x == 0) aggs[blockIdx.x] = tot;
}

// per tile: blocked arrangement (thread t owns items [t*kItems, (t+1)*kItems))
template <class T, class Op, class Load, class Store>
__global__ void __launch_bounds__(kThreads) k_scan_down(Load load, Store store, uint64_t n, const T* tile_prefix,
                                                       Op op, T identity, int inclusive) {
  const uint64_t base = (uint64_t)blockIdx.x * kTile + (uint64_t)threadIdx.x * kItems;
  T v[kItems];
  T acc = identity;
#pragma unroll
  for (int k = 0; k < kItems; k++) {
    uint64_t i = base + k;
    v[k] = i < n ? load(i) : identity;
    acc = op(acc, v[k]);
  }
  T tot;
  T run = block_excl_scan<T, Op>(acc, op, identity, &tot);
  if (tile_prefix) run = op(tile_prefix[blockIdx.x], run);
#pragma unroll
  for (int k = 0; k < kItems; k++) {
    uint64_t i = base + k;
    T nx = op(run, v[k]);
    if (i < n) store(i, inclusive ? nx : run);
    run = nx;
  }
}

template <class T>
struct ArrLoad {
  const T* p;
  __device__ __forceinline__ T operator()(uint64_t i) const { return p[i]; }
};
template <class T>
struct ArrStore {
  T* p;
  __device__ __forceinline__ void operator()(uint64_t i, const T& v) const { p[i] = v; }
};

// Scan over n items.  scratch must hold scan_scratch_elems(n) elements of T.
inline uint64_t scan_scratch_elems(uint64_t n) {
  uint64_t tot = 0;
  uint64_t t = (n + kTile - 1) / kTile;
  while (t > 1) {
    tot += t;
    t = (t + kTile - 1) / kTile;
  }
  return tot + 1;
}

template <class T, class Op, class Load, class Store>
void device_scan(Load load, Store store, uint64_t n, T* scratch, Op op, T identity, bool inclusive,
                 cudaStream_t st) {
  if (n == 0) return;
  uint64_t ntiles = (n + kTile - 1) / kTile;
  if (ntiles == 1) {
    GW_LAUNCH((k_scan_down<T, Op, Load, Store>), 1, kThreads, 0, st, load, store, n, (const T*)nullptr, op,
              identity, (int)inclusive);
    return;
  }
  T* aggs = scratch;
  GW_LAUNCH((k_scan_reduce<T, Op, Load>), (unsigned)ntiles, kThreads, 0, st, load, n, aggs, op, identity);
  // exclusive scan of tile aggregates, in place
  device_scan<T, Op>(ArrLoad<T>{aggs}, ArrStore<T>{aggs}, ntiles, scratch + ntiles, op, identity, false, st);
  GW_LAUNCH((k_scan_down<T, Op, Load, Store>), (unsigned)ntiles, kThreads, 0, st, load, store, n,
            (const T*)aggs, op, identity, (int)inclusive);
}

// --------------------------------------------------------- radix sort ----
// Stable LSD radix sort, 8-bit digits.  Per pass: tile histograms (digit-major,
// so one exclusive scan yields every tile's scatter base), then a stable
// scatter in which each warp owns a contiguous 512-item sub-tile and ranks
// equal digits with __match_any_sync.
constexpr int kRsWarps = kThreads / 32;
constexpr int kRsPerWarp = kTile / kRsWarps;      // 512
constexpr int kRsRounds = kRsPerWarp / 32;        // 16

template <class K>
__global__ void __launch_bounds__(kThreads) k_rs_hist(const K* __restrict__ keys, uint64_t n, int shift,
                                                     uint32_t* __restrict__ counts, uint64_t ntiles) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kTile;
#pragma unroll 4
  for (int k = 0; k < kItems; k++) {
    uint64_t i = base + (uint64_t)k * kThreads + threadIdx.x;
    if (i < n) {
      uint32_t d = (uint32_t)(keys[i] >> shift) & 255u;
      atomicAdd(&h[d], 1u);
    }
  }
  __syncthreads();
  counts[(uint64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

template <class K>
__global__ void __launch_bounds__(kThreads) k_rs_scatter(const K* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                        K* __restrict__ kout, uint32_t* __restrict__ vout, uint64_t n,
                                                        int shift, const uint32_t* __restrict__ offs, uint64_t ntiles) {
  __shared__ uint32_t s_wc[kRsWarps][256];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int d = threadIdx.x; d < kRsWarps * 256; d += kThreads) (&s_wc[0][0])[d] = 0;
  __syncthreads();
  const uint64_t wbase = (uint64_t)blockIdx.x * kTile + (uint64_t)w * kRsPerWarp;
  K kk[kRsRounds];
  uint32_t vv[kRsRounds];
  uint32_t dd[kRsRounds];
#pragma unroll
  for (int r = 0; r < kRsRounds; r++) {
    uint64_t i = wbase + (uint64_t)r * 32 + lane;
    bool ok = i < n;
    kk[r] = ok ? kin[i] : (K)0;
    vv[r] = ok ? vin[i] : 0u;
    dd[r] = ok ? ((uint32_t)(kk[r] >> shift) & 255u) : 256u;
  }
#pragma unroll
  for (int r = 0; r < kRsRounds; r++) {
    uint32_t peers = __match_any_sync(0xffffffffu, dd[r]);
    int leader = __ffs(peers) - 1;
    if (lane == leader && dd[r] < 256u) s_wc[w][dd[r]] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  {
    const int d = threadIdx.x;
    uint32_t run = offs[(uint64_t)d * ntiles + blockIdx.x];
#pragma unroll
    for (int ww = 0; ww < kRsWarps; ww++) {
      uint32_t t = s_wc[ww][d];
      s_wc[ww][d] = run;
      run += t;
    }
  }
  __syncthreads();
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int r = 0; r < kRsRounds; r++) {
    uint32_t d = dd[r];
    uint32_t peers = __match_any_sync(0xffffffffu, d);
    int leader = __ffs(peers) - 1;
    if (d < 256u) {
      uint32_t pos = s_wc[w][d] + __popc(peers & lt);
      kout[pos] = kk[r];
      vout[pos] = vv[r];
    }
    __syncwarp();
    if (lane == leader && d < 256u) s_wc[w][d] += __popc(peers);
    __syncwarp();
  }
}

inline uint64_t rs_counts_elems(uint64_t n) { return 256ull * ((n + kTile - 1) / kTile); }

// Sorts (keys,vals) by bits [0, nbits) of the key.  Ping-pongs between the
// primary and alternate buffers; returns true if the result is in the
// alternate buffers.  counts/scan_scratch sized by rs_counts_elems /
// scan_scratch_elems(rs_counts_elems(n)).
template <class K>
bool radix_sort(K* keys, K* keys_alt, uint32_t* vals, uint32_t* vals_alt, uint64_t n, int nbits, uint32_t* counts,
                uint32_t* scan_scratch, cudaStream_t st) {
  if (n <= 1 || nbits <= 0) return false;
  uint64_t ntiles = (n + kTile - 1) / kTile;
  bool alt = false;
  for (int shift = 0; shift < nbits; shift += 8) {
    const K* ki = alt ? keys_alt : keys;
    const uint32_t* vi = alt ? vals_alt : vals;
    K* ko = alt ? keys : keys_alt;
    uint32_t* vo = alt ? vals : vals_alt;
    GW_LAUNCH(k_rs_hist<K>, (unsigned)ntiles, kThreads, 0, st, ki, n, shift, counts, ntiles);
    device_scan<uint32_t, OpSum>(ArrLoad<uint32_t>{counts}, ArrStore<uint32_t>{counts}, 256ull * ntiles,
                                 scan_scratch, OpSum(), 0u, false, st);
    GW_LAUNCH(k_rs_scatter<K>, (unsigned)ntiles, kThreads, 0, st, ki, vi, ko, vo, n, shift, counts, ntiles);
    alt = !alt;
  }
  return alt;
}

}  // namespace gw
