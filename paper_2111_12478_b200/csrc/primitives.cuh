// Device-wide primitives for the G-WCP pipeline, hand-written for sm_100a:
//   * a single-pass (decoupled look-back) scan over a user load/store functor
//   * a stable one-sweep LSD radix sort (8-bit digits) of (u32|u64 key, u32 value)
// Both are HBM-streaming kernels: 256-thread CTAs, 16 items per thread, grids
// sized in tiles so a 1e9-element pass fills all 148 SMs many times over.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <algorithm>

namespace gw {

constexpr int kThreads = 256;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;  // 4096

// launch accounting (gw_ctx_launches); incremented on the host per launch.
// With a LaunchProf installed (GW_OPT_PROFILE analyses) every launch is
// bracketed by CUDA events on its stream -> per-kernel device times.
struct LaunchProf {
  struct Rec { const char* name; const char* tag; cudaEvent_t a, b; };
  Rec* recs = nullptr;
  uint32_t n = 0, cap = 0;
  const char* tag = nullptr;  // current sort / phase tag ("acc", "hd", ...): kernels are timed per tag
  void begin(const char* name, cudaStream_t st) {
    if (n >= cap) return;
    recs[n].name = name;
    recs[n].tag = tag;
    cudaEventRecord(recs[n].a, st);
  }
  void end(cudaStream_t st) {
    if (n >= cap) return;
    cudaEventRecord(recs[n].b, st);
    n++;
  }
};
extern thread_local uint32_t g_launches;
extern thread_local LaunchProf* g_prof;
#define GW_LAUNCH(kernel, grid, block, smem, stream, ...)      \
  do {                                                         \
    if (::gw::g_prof) ::gw::g_prof->begin(#kernel, (stream));  \
    kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__); \
    if (::gw::g_prof) ::gw::g_prof->end((stream));             \
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

template <class T>
__device__ __forceinline__ T shfl_down(T v, int o) { return __shfl_down_sync(0xffffffffu, v, o); }
template <>
__device__ __forceinline__ uint2 shfl_down<uint2>(uint2 v, int o) {
  return make_uint2(__shfl_down_sync(0xffffffffu, v.x, o), __shfl_down_sync(0xffffffffu, v.y, o));
}
template <class T>
__device__ __forceinline__ T shfl_idx(T v, int l) { return __shfl_sync(0xffffffffu, v, l); }
template <>
__device__ __forceinline__ uint2 shfl_idx<uint2>(uint2 v, int l) {
  return make_uint2(__shfl_sync(0xffffffffu, v.x, l), __shfl_sync(0xffffffffu, v.y, l));
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

// ------------------------------------------------ single-pass scan ----
// Decoupled look-back (chained) scan: one launch, tiles taken in launch order
// from an atomic counter; each tile publishes its aggregate, then its
// inclusive prefix, as ONE 64-bit word (state:2 | payload:62), so a
// predecessor's state and value are read together with no memory fences.
// The status words are zeroed (state 0 = not ready) before every launch.
__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) {
  return *(volatile const uint32_t*)p;
}
__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  return *(volatile const unsigned long long*)p;
}

// payload packing (62 bits)
template <class T>
struct LbPack;
template <>
struct LbPack<uint32_t> {
  __device__ __forceinline__ static unsigned long long pack(uint32_t v) { return v; }
  __device__ __forceinline__ static uint32_t unpack(unsigned long long w) { return (uint32_t)w; }
};
template <>
struct LbPack<uint2> {  // two values < 2^31 (positions + 1)
  __device__ __forceinline__ static unsigned long long pack(uint2 v) {
    return (unsigned long long)v.x | ((unsigned long long)v.y << 31);
  }
  __device__ __forceinline__ static uint2 unpack(unsigned long long w) {
    return make_uint2((uint32_t)(w & 0x7FFFFFFFull), (uint32_t)((w >> 31) & 0x7FFFFFFFull));
  }
};
constexpr unsigned long long LB_AGG = 1ull << 62, LB_INC = 2ull << 62, LB_PAY = (1ull << 62) - 1;

template <class T, class Op, class Load, class Store>
__global__ void __launch_bounds__(kThreads) k_scan_lb(Load load, Store store, uint64_t n, unsigned long long* status,
                                                     uint32_t* ctr, Op op, T identity, int inclusive) {
  __shared__ uint32_t s_tile;
  __shared__ T s_pre;
  __shared__ T s_buf[kTile];
  if (threadIdx.x == 0) s_tile = atomicAdd(ctr, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t base = (uint64_t)tile * kTile;
  // striped (coalesced) load -> smem -> blocked per thread
  {
    T x[kItems];
#pragma unroll
    for (int k = 0; k < kItems; k++) {
      const uint64_t i = base + (uint64_t)k * kThreads + threadIdx.x;
      x[k] = i < n ? load(i) : identity;
    }
#pragma unroll
    for (int k = 0; k < kItems; k++) s_buf[k * kThreads + threadIdx.x] = x[k];
  }
  __syncthreads();
  T v[kItems];
  T acc = identity;
#pragma unroll
  for (int k = 0; k < kItems; k++) {
    v[k] = s_buf[threadIdx.x * kItems + k];
    acc = op(acc, v[k]);
  }
  T tot;
  T run = block_excl_scan<T, Op>(acc, op, identity, &tot);
  if (threadIdx.x < 32) {
    // warp-wide decoupled look-back: 32 predecessors per round trip
    const int lane = threadIdx.x;
    if (lane == 0)
      atomicExch(&status[tile], (tile == 0 ? LB_INC : LB_AGG) | LbPack<T>::pack(tot));
    T pre = identity;
    if (tile > 0) {
      int64_t p = (int64_t)tile - 1;
      while (true) {
        const int64_t q = p - lane;
        unsigned long long wv = LB_INC;  // q < 0: virtual inclusive identity
        if (q >= 0) {
          do { wv = ld_volatile_u64(&status[q]); } while ((wv >> 62) == 0ull);
        }
        const bool isinc = (wv >> 62) == 2ull;
        const uint32_t incm = __ballot_sync(0xffffffffu, isinc);
        const int lim = __ffs(incm) - 1;  // nearest inclusive predecessor (incm != 0 once q < 0)
        T val = identity;
        if (q >= 0 && (incm == 0 || lane <= lim)) val = LbPack<T>::unpack(wv & LB_PAY);
        // reduce lanes 0..lim (commutative ops: sum, max)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          T other = shfl_down(val, o);
          if (lane + o < 32) val = op(val, other);
        }
        val = shfl_idx(val, 0);
        pre = op(val, pre);
        if (incm) break;
        p -= 32;
      }
      if (lane == 0) atomicExch(&status[tile], LB_INC | LbPack<T>::pack(op(pre, tot)));
    }
    if (lane == 0) s_pre = pre;
  }
  __syncthreads();
  run = op(s_pre, run);
#pragma unroll
  for (int k = 0; k < kItems; k++) {
    T nx = op(run, v[k]);
    s_buf[threadIdx.x * kItems + k] = inclusive ? nx : run;
    run = nx;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kItems; k++) {
    const uint64_t i = base + (uint64_t)k * kThreads + threadIdx.x;
    if (i < n) store(i, s_buf[k * kThreads + threadIdx.x]);
  }
}

// scratch for scan_lb: lb_tiles(n) status words (zeroed here) + a zeroed tile counter
inline uint64_t lb_tiles(uint64_t n) { return (n + kTile - 1) / kTile; }

template <class T, class Op, class Load, class Store>
void scan_lb(Load load, Store store, uint64_t n, unsigned long long* status, uint32_t* ctr, Op op, T identity,
             bool inclusive, cudaStream_t st) {
  if (n == 0) return;
  const uint64_t nt = lb_tiles(n);
  cudaMemsetAsync(status, 0, sizeof(unsigned long long) * nt, st);
  GW_LAUNCH((k_scan_lb<T, Op, Load, Store>), (unsigned)nt, kThreads, 0, st, load, store, n, status, ctr, op, identity,
            (int)inclusive);
}

// --------------------------------------------------------- radix sort ----
// One-sweep LSD radix sort of (u32|u64 key, u32 value), 8-bit digits: one
// histogram kernel for every pass up front, then ONE kernel per pass whose
// tiles chain their per-digit counts through decoupled look-back (status word
// = epoch:24 | state:2 | count:38; thread d of a tile owns digit d).  Each
// tile ranks its 4096 items stably in one sweep (per-warp digit counters,
// warp peers found with 8 ballots), stages them in shared memory in digit
// order and writes every digit run with consecutive threads -> coalesced
// stores.  Global traffic per pass: the keys + values read once and written
// once, + 2 KB of status per tile.
constexpr int kRsWarps = kThreads / 32;
constexpr int kRsPerWarp = kTile / kRsWarps;      // 512
constexpr int kRsRounds = kRsPerWarp / 32;        // 16
constexpr int kRsBits = 8;
constexpr int kRsDigits = 1 << kRsBits;           // 256 = kThreads: one digit per thread
constexpr int kRsMaxPass = 8;
static_assert(kRsDigits == kThreads, "one digit per thread");

// RB-bit digits (RB = 8 or 9; 9 saves a pass when it covers the key in
// fewer passes, e.g. 17-bit keys in 2 instead of 3); DPT digits per thread.
constexpr int kRsMaxDigits = 512;
#ifndef GW_RS_LOOKBACK
#define GW_RS_LOOKBACK 16  // status words in flight per thread in the one-sweep look-back
#endif
template <int RB>
struct RsDig {
  static constexpr int ND = 1 << RB;
  static constexpr int DPT = ND / kThreads;
  static_assert(ND % kThreads == 0 && ND <= kRsMaxDigits, "digit layout");
};

template <class K, int RB>
__global__ void __launch_bounds__(kThreads) k_rs_ghist(const K* __restrict__ keys, uint64_t n, int npass,
                                                      uint32_t* __restrict__ ghist) {
  constexpr int ND = RsDig<RB>::ND;
  __shared__ uint32_t h[kRsMaxPass * ND];
  for (int i = threadIdx.x; i < npass * ND; i += kThreads) h[i] = 0;
  __syncthreads();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const K k = keys[i];
    for (int p = 0; p < npass; p++) atomicAdd(&h[p * ND + ((uint32_t)(k >> (RB * p)) & (ND - 1))], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < npass * ND; i += kThreads)
    if (h[i]) atomicAdd(&ghist[i], h[i]);
}

template <class K, int RB>
struct RsSmem {
  static constexpr int ND = RsDig<RB>::ND;
  uint32_t wc[kRsWarps][ND];  // per-warp digit counts -> per-warp offsets within the digit
  uint32_t toff[ND];          // tile-local start of digit d
  uint32_t gbase[ND];         // global start of this tile's digit-d run
  K sk[kTile];
  uint32_t sv[kTile];
  uint32_t tile;
};

// Staging slot of tile position p (digit order).  With ~16 keys per digit the
// digit runs of one warp store start 16 slots apart, which put a whole warp on
// two banks (u32; one bank pair for u64); XOR-swizzling the slot within its
// 32-bank row spreads them over all banks.  Consecutive positions stay in one
// row, so the write-out reads remain conflict-free.
template <class K>
__device__ __forceinline__ uint32_t stg(uint32_t p) {
  if constexpr (sizeof(K) == 8) return p ^ ((p >> 4) & 15u);
  else return p ^ ((p >> 5) & 31u);
}

// lanes with the same digit (NB low bits of d) among the warp's lanes
template <int NB>
__device__ __forceinline__ uint32_t warp_peers(uint32_t d) {
  uint32_t peers = 0xffffffffu;
#pragma unroll
  for (int b = 0; b < NB; b++) {
    const bool bit = (d >> b) & 1u;
    const uint32_t bal = __ballot_sync(0xffffffffu, bit);
    peers &= bit ? bal : ~bal;
  }
  return peers;
}

template <class K, int RB>
#ifndef GW_OS_MINB
#define GW_OS_MINB 3
#endif
__global__ void __launch_bounds__(kThreads, sizeof(K) == 4 ? GW_OS_MINB : 2) k_rs_onesweep(const K* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                            K* __restrict__ kout, uint32_t* __restrict__ vout,
                                                            uint64_t n, int pass, const uint32_t* __restrict__ ghist,
                                                            unsigned long long* status, uint32_t* ctr, uint32_t epoch) {
  constexpr int ND = RsDig<RB>::ND, DPT = RsDig<RB>::DPT;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  RsSmem<K, RB>& S = *reinterpret_cast<RsSmem<K, RB>*>(smem_raw);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int shift = RB * pass;
  for (int d = threadIdx.x; d < kRsWarps * ND; d += kThreads) (&S.wc[0][0])[d] = 0;
  if (threadIdx.x == 0) S.tile = atomicAdd(ctr, 1u);
  __syncthreads();
  const uint32_t tile = S.tile;
  const uint64_t tbase = (uint64_t)tile * kTile;
  const uint64_t wbase = tbase + (uint64_t)w * kRsPerWarp;
  const bool full = tbase + kTile <= n;
  K kk[kRsRounds];
  uint32_t vv[kRsRounds];
  uint32_t rd[kRsRounds];  // rank within the warp's digit run (bits 0-15) | digit (bits 16-25, ND = none)
#pragma unroll
  for (int r = 0; r < kRsRounds; r++) {
    const uint64_t i = wbase + (uint64_t)r * 32 + lane;
    const bool ok = full || i < n;
    kk[r] = ok ? kin[i] : (K)0;
    vv[r] = ok ? vin[i] : 0u;
    rd[r] = ok ? (((uint32_t)(kk[r] >> shift) & (ND - 1)) << 16) : ((uint32_t)ND << 16);
  }
  // stable ranks within the warp: rounds in order, lanes in order
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int r = 0; r < kRsRounds; r++) {
    const uint32_t d = rd[r] >> 16;
    const uint32_t peers = full ? warp_peers<RB>(d) : warp_peers<RB + 1>(d);
    const uint32_t before = d < (uint32_t)ND ? S.wc[w][d] : 0u;
    __syncwarp();
    if (d < (uint32_t)ND && (peers & lt) == 0) S.wc[w][d] = before + __popc(peers);
    rd[r] |= before + __popc(peers & lt);
    __syncwarp();
  }
  __syncthreads();
  {
    // thread t owns digits t*DPT .. t*DPT+DPT-1: per-warp offsets, tile
    // counts, tile-local digit starts; the aggregates are published first
    const unsigned long long EP = (unsigned long long)epoch << 40;
    uint32_t c[DPT], g[DPT];
    uint32_t csum = 0, gsum = 0;
#pragma unroll
    for (int j = 0; j < DPT; j++) {
      const int d = threadIdx.x * DPT + j;
      uint32_t run = 0;
#pragma unroll
      for (int ww = 0; ww < kRsWarps; ww++) {
        const uint32_t t = S.wc[ww][d];
        S.wc[ww][d] = run;
        run += t;
      }
      c[j] = run;
      atomicExch(&status[(uint64_t)tile * ND + d], EP | (1ull << 38) | run);
      g[j] = ghist[pass * ND + d];
      csum += run;
      gsum += g[j];
    }
    uint32_t gt, ct;
    uint32_t gex = block_excl_scan<uint32_t, OpSum>(gsum, OpSum(), 0u, &gt);
    uint32_t cex = block_excl_scan<uint32_t, OpSum>(csum, OpSum(), 0u, &ct);
#pragma unroll
    for (int j = 0; j < DPT; j++) {
      S.toff[threadIdx.x * DPT + j] = cex;
      cex += c[j];
    }
    __syncthreads();
    // stage in digit order while the predecessors publish (the look-back
    // below only needs the global bases)
#pragma unroll
    for (int r = 0; r < kRsRounds; r++) {
      const uint32_t d = rd[r] >> 16;
      if (d < (uint32_t)ND) {
        const uint32_t pos = S.toff[d] + S.wc[w][d] + (rd[r] & 0xFFFFu);
        S.sk[stg<K>(pos)] = kk[r];
        S.sv[stg<K>(pos)] = vv[r];
      }
    }
    // Two-level look-back (no chain through every predecessor): the tiles
    // form groups of GS = 2^(floor(log2(tiles)/2)) consecutive tiles; the last
    // tile of a group publishes the group's total.  A tile's exclusive prefix
    // = the aggregates of its group's earlier tiles + the totals of the
    // earlier groups, at most ~2 sqrt(tiles) loads per digit, LBW per digit
    // per round trip.  Every wait is for a lower tile index (tile indices are
    // taken in launch order), so it cannot deadlock.
    constexpr int LBW = GW_RS_LOOKBACK / DPT;
    const uint32_t ntiles = (uint32_t)((n + kTile - 1) / kTile);
    const uint32_t gsh = (32u - __clz(ntiles > 1 ? ntiles - 1 : 1u)) >> 1;
    const uint32_t grp = tile >> gsh, gfirst = grp << gsh;
    unsigned long long* gstat = status + (uint64_t)ntiles * ND;
    unsigned long long pre[DPT];
#pragma unroll
    for (int j = 0; j < DPT; j++) pre[j] = 0;
    // sums src[(q0 + k) * ND + d] over q in [q0, q1) into pre[], waiting for every entry
    auto gather = [&](const unsigned long long* src, uint32_t q0, uint32_t q1) {
      for (uint32_t qb = q0; qb < q1; qb += LBW) {
        unsigned long long wv[DPT][LBW];
        bool ok;
        do {
#pragma unroll
          for (int j = 0; j < DPT; j++) {
            const int d = threadIdx.x * DPT + j;
#pragma unroll
            for (int k = 0; k < LBW; k++)
              wv[j][k] = qb + k < q1 ? ld_volatile_u64(&src[(uint64_t)(qb + k) * ND + d]) : EP;
          }
          ok = true;
#pragma unroll
          for (int j = 0; j < DPT; j++)
#pragma unroll
            for (int k = 0; k < LBW; k++) ok = ok && (wv[j][k] >> 40) == epoch;
        } while (!ok);
#pragma unroll
        for (int j = 0; j < DPT; j++)
#pragma unroll
          for (int k = 0; k < LBW; k++) pre[j] += wv[j][k] & ((1ull << 38) - 1);
      }
    };
    gather(status, gfirst, tile);
    if (tile - gfirst == (1u << gsh) - 1u) {  // last tile of its group: the group total
#pragma unroll
      for (int j = 0; j < DPT; j++)
        atomicExch(&gstat[(uint64_t)grp * ND + threadIdx.x * DPT + j], EP | (1ull << 38) | (pre[j] + c[j]));
    }
    gather(gstat, 0, grp);
#pragma unroll
    for (int j = 0; j < DPT; j++) {
      const int d = threadIdx.x * DPT + j;
      S.gbase[d] = gex + (uint32_t)pre[j];
      gex += g[j];
    }
  }
  __syncthreads();
  // coalesced write-out: consecutive threads write consecutive slots of a digit run
  const uint64_t rem = n > tbase ? n - tbase : 0ull;
  const uint32_t cnt = rem < (uint64_t)kTile ? (uint32_t)rem : (uint32_t)kTile;
#pragma unroll 4
  for (uint32_t i = threadIdx.x; i < cnt; i += kThreads) {
    const K k = S.sk[stg<K>(i)];
    const uint32_t d = (uint32_t)(k >> shift) & (ND - 1);
    const uint32_t gp = S.gbase[d] + (i - S.toff[d]);
    kout[gp] = k;
    vout[gp] = S.sv[stg<K>(i)];
  }
}

// ---- reduce-then-scan radix pass (large n) ---------------------------------
// No chained look-back: k_rs_up counts the digits of every super-tile (ST
// tiles of kTile keys) into a digit-major matrix counts[d * nst + st], one
// exclusive scan of that matrix gives every (digit, super-tile) its output
// offset, and k_rs_down ranks / stages / scatters tile by tile (ballot ranks
// as in the one-sweep kernel), advancing its digit bases after each tile.
// RB-bit digits (RB = 10: 3 passes for <= 30-bit keys); traffic per pass:
// keys read twice, values once, both written once, + 4 * 2^RB B per super-tile.
template <int RB>
struct RsBig {
  static constexpr int ND = 1 << RB;
  static constexpr int DPT = ND >= kThreads ? ND / kThreads : 1;  // digits per thread (RB < 8: threads < ND)
  static constexpr int ST = RB <= 8 ? 1 : 4; // tiles per super-tile
};

template <class K, int RB>
__global__ void __launch_bounds__(kThreads) k_rs_up(const K* __restrict__ keys, uint64_t n, int shift,
                                                   uint32_t* __restrict__ counts, uint64_t nst) {
  constexpr int ND = RsBig<RB>::ND, DPT = RsBig<RB>::DPT, ST = RsBig<RB>::ST;
  __shared__ uint32_t h[kRsWarps][ND];  // per-warp histograms (low contention)
  const int w = threadIdx.x >> 5;
  for (uint64_t st = blockIdx.x; st < nst; st += gridDim.x) {
    for (int d = threadIdx.x; d < kRsWarps * ND; d += kThreads) (&h[0][0])[d] = 0;
    __syncthreads();
    for (int sub = 0; sub < ST; sub++) {
      const uint64_t base = (st * ST + sub) * kTile;
      K kk[kItems];
#pragma unroll
      for (int k = 0; k < kItems; k++) {
        const uint64_t i = base + (uint64_t)k * kThreads + threadIdx.x;
        kk[k] = i < n ? keys[i] : (K)0;
      }
#pragma unroll
      for (int k = 0; k < kItems; k++) {
        const uint64_t i = base + (uint64_t)k * kThreads + threadIdx.x;
        if (i < n) atomicAdd(&h[w][(uint32_t)(kk[k] >> shift) & (ND - 1)], 1u);
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < DPT; j++) {
      const int d = threadIdx.x * DPT + j;
      if (d >= ND) break;
      uint32_t c = 0;
#pragma unroll
      for (int x = 0; x < kRsWarps; x++) c += h[x][d];
      counts[(uint64_t)d * nst + st] = c;
    }
    __syncthreads();
  }
}

template <class K, int RB>
struct RsBigSmem {
  static constexpr int ND = 1 << RB;
  uint32_t wc[kRsWarps][ND];  // per-warp digit counts -> per-warp offsets within the digit
  uint32_t toff[ND];          // tile-local start of digit d
  uint32_t gbase[ND];         // global start of digit d for the current tile
  K sk[kTile];
  uint32_t sv[kTile];
};

template <class K, int RB>
__global__ void __launch_bounds__(kThreads, (RB == 8 && sizeof(K) == 4) ? 3 : 2) k_rs_down(const K* __restrict__ kin,
                                                                                         const uint32_t* __restrict__ vin,
                                                       K* __restrict__ kout, uint32_t* __restrict__ vout, uint64_t n,
                                                       int shift, const uint32_t* __restrict__ offsets, uint64_t nst) {
  constexpr int ND = RsBig<RB>::ND, DPT = RsBig<RB>::DPT, ST = RsBig<RB>::ST;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  RsBigSmem<K, RB>& S = *reinterpret_cast<RsBigSmem<K, RB>*>(smem_raw);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t lt = lanemask_lt();
  for (uint64_t st = blockIdx.x; st < nst; st += gridDim.x) {
#pragma unroll
    for (int j = 0; j < DPT; j++) {
      const int d = threadIdx.x * DPT + j;
      S.gbase[d] = offsets[(uint64_t)d * nst + st];
    }
    for (int sub = 0; sub < ST; sub++) {
      const uint64_t tbase = (st * ST + sub) * kTile;
      if (tbase >= n) break;
      for (int d = threadIdx.x; d < kRsWarps * ND; d += kThreads) (&S.wc[0][0])[d] = 0;
      __syncthreads();
      const uint64_t wbase = tbase + (uint64_t)w * kRsPerWarp;
      const bool full = tbase + kTile <= n;
      K kk[kRsRounds];
      uint32_t vv[kRsRounds];
      uint32_t rd[kRsRounds];  // rank (bits 0-15) | digit (bits 16+, ND = none)
#pragma unroll
      for (int r = 0; r < kRsRounds; r++) {
        const uint64_t i = wbase + (uint64_t)r * 32 + lane;
        const bool ok = full || i < n;
        kk[r] = ok ? kin[i] : (K)0;
        vv[r] = ok ? vin[i] : 0u;
        rd[r] = ok ? (((uint32_t)(kk[r] >> shift) & (ND - 1)) << 16) : ((uint32_t)ND << 16);
      }
#pragma unroll
      for (int r = 0; r < kRsRounds; r++) {
        const uint32_t d = rd[r] >> 16;
        const uint32_t peers = full ? warp_peers<RB>(d) : warp_peers<RB + 1>(d);
        const uint32_t before = d < (uint32_t)ND ? S.wc[w][d] : 0u;
        __syncwarp();
        if (d < (uint32_t)ND && (peers & lt) == 0) S.wc[w][d] = before + __popc(peers);
        rd[r] |= before + __popc(peers & lt);
        __syncwarp();
      }
      __syncthreads();
      {
        uint32_t tot[DPT], csum = 0;
#pragma unroll
        for (int j = 0; j < DPT; j++) {
          const int d = threadIdx.x * DPT + j;
          uint32_t run = 0;
#pragma unroll
          for (int ww = 0; ww < kRsWarps; ww++) {
            const uint32_t t = S.wc[ww][d];
            S.wc[ww][d] = run;
            run += t;
          }
          tot[j] = run;
          csum += run;
        }
        uint32_t ct;
        uint32_t cex = block_excl_scan<uint32_t, OpSum>(csum, OpSum(), 0u, &ct);
#pragma unroll
        for (int j = 0; j < DPT; j++) {
          S.toff[threadIdx.x * DPT + j] = cex;
          cex += tot[j];
        }
      }
      __syncthreads();
#pragma unroll
      for (int r = 0; r < kRsRounds; r++) {
        const uint32_t d = rd[r] >> 16;
        if (d < (uint32_t)ND) {
          const uint32_t pos = S.toff[d] + S.wc[w][d] + (rd[r] & 0xFFFFu);
          S.sk[stg<K>(pos)] = kk[r];
          S.sv[stg<K>(pos)] = vv[r];
        }
      }
      __syncthreads();
      const uint64_t rem = n - tbase;
      const uint32_t cnt = rem < (uint64_t)kTile ? (uint32_t)rem : (uint32_t)kTile;
#pragma unroll 4
      for (uint32_t i = threadIdx.x; i < cnt; i += kThreads) {
        const K k = S.sk[stg<K>(i)];
        const uint32_t d = (uint32_t)(k >> shift) & (ND - 1);
        const uint32_t gp = S.gbase[d] + (i - S.toff[d]);
        kout[gp] = k;
        vout[gp] = S.sv[stg<K>(i)];
      }
      __syncthreads();
      // advance the bases past this tile's runs
#pragma unroll
      for (int j = 0; j < DPT; j++) {
        const int d = threadIdx.x * DPT + j;
        const uint32_t end = d + 1 < ND ? S.toff[d + 1] : cnt;
        S.gbase[d] += end - S.toff[d];
      }
      __syncthreads();
    }
  }
}
// ---- TMA bulk copies (cp.async.bulk) with mbarrier completion --------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* m, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned long long* m, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(m)), "r"(phase)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(m))
               : "memory");
}

// k_rs_down with its input tiles streamed by TMA bulk copies into a double
// buffer (the next tile lands while this one is ranked); the input buffer is
// then reused as the digit-order staging buffer of the scatter.
template <class K>
struct RsTmaSmem {
  K ik[2][kTile];             // input keys (TMA) -> staged keys
  uint32_t iv[2][kTile];      // input values (TMA) -> staged values
  uint32_t wc[kRsWarps][kRsDigits];
  uint32_t toff[kRsDigits];
  uint32_t gbase[kRsDigits];
  unsigned long long mbar[2];
};
// RB <= 8 bits per pass (the big sort balances a key's bits over its passes:
// 29 bits -> 8 + 7 + 7 + 7, fewer ballots per rank and longer digit runs)
template <class K, int RB = kRsBits>
__global__ void __launch_bounds__(kThreads, sizeof(K) == 4 ? 3 : 2) k_rs_down_tma(const K* __restrict__ kin,
                                                                            const uint32_t* __restrict__ vin,
                                                                            K* __restrict__ kout,
                                                                            uint32_t* __restrict__ vout, uint64_t n,
                                                                            int shift,
                                                                            const uint32_t* __restrict__ offsets,
                                                                            uint64_t nst) {
  static_assert(RB >= 1 && RB <= kRsBits, "k_rs_down_tma: 1..8-bit digits");
  constexpr int ND = 1 << RB;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  RsTmaSmem<K>& S = *reinterpret_cast<RsTmaSmem<K>*>(smem_raw);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t lt = lanemask_lt();
  auto full_tile = [&](uint64_t st) { return (st + 1) * kTile <= n; };
  auto issue = [&](uint64_t st, int b) {  // thread 0
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier generic accesses to buffer b
    mbar_expect_tx(&S.mbar[b], (uint32_t)(kTile * (sizeof(K) + 4)));
    bulk_g2s(S.ik[b], kin + st * kTile, (uint32_t)(kTile * sizeof(K)), &S.mbar[b]);
    bulk_g2s(S.iv[b], vin + st * kTile, (uint32_t)(kTile * 4), &S.mbar[b]);
  };
  if (threadIdx.x == 0) {
    mbar_init(&S.mbar[0], 1);
    mbar_init(&S.mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t uses[2] = {0, 0};
  uint64_t st = blockIdx.x;
  if (st < nst && threadIdx.x == 0 && full_tile(st)) issue(st, 0);
  for (int it = 0; st < nst; st += gridDim.x, it++) {
    const int b = it & 1;
    const uint64_t nx = st + gridDim.x;
    if (threadIdx.x == 0 && nx < nst && full_tile(nx)) issue(nx, b ^ 1);
    const uint64_t tbase = st * kTile;
    const bool full = full_tile(st);
    if (threadIdx.x < ND) S.gbase[threadIdx.x] = offsets[(uint64_t)threadIdx.x * nst + st];
    for (int x = threadIdx.x; x < kRsWarps * ND; x += kThreads) S.wc[x / ND][x % ND] = 0;  // rows of kRsDigits
    K kk[kRsRounds];
    uint32_t vv[kRsRounds];
    uint32_t rd[kRsRounds];
    if (full) {
      while (!mbar_try_wait(&S.mbar[b], uses[b] & 1u)) {
      }
      uses[b]++;
#pragma unroll
      for (int r = 0; r < kRsRounds; r++) {
        const uint32_t j = w * kRsPerWarp + r * 32 + lane;
        kk[r] = S.ik[b][j];
        vv[r] = S.iv[b][j];
        rd[r] = ((uint32_t)(kk[r] >> shift) & (ND - 1)) << 16;
      }
    } else {
#pragma unroll
      for (int r = 0; r < kRsRounds; r++) {
        const uint64_t i = tbase + (uint64_t)w * kRsPerWarp + (uint64_t)r * 32 + lane;
        const bool ok = i < n;
        kk[r] = ok ? kin[i] : (K)0;
        vv[r] = ok ? vin[i] : 0u;
        rd[r] = ok ? (((uint32_t)(kk[r] >> shift) & (ND - 1)) << 16) : ((uint32_t)ND << 16);
      }
    }
    __syncthreads();  // wc zeroed; every thread has its inputs in registers
#pragma unroll
    for (int r = 0; r < kRsRounds; r++) {
      const uint32_t d = rd[r] >> 16;
      const uint32_t peers = full ? warp_peers<RB>(d) : warp_peers<RB + 1>(d);
      const uint32_t before = d < (uint32_t)ND ? S.wc[w][d] : 0u;
      __syncwarp();
      if (d < (uint32_t)ND && (peers & lt) == 0) S.wc[w][d] = before + __popc(peers);
      rd[r] |= before + __popc(peers & lt);
      __syncwarp();
    }
    __syncthreads();
    {
      const int d = threadIdx.x;
      uint32_t run = 0;
      if (d < ND) {
#pragma unroll
        for (int ww = 0; ww < kRsWarps; ww++) {
          const uint32_t t = S.wc[ww][d];
          S.wc[ww][d] = run;
          run += t;
        }
      }
      uint32_t ct;
      const uint32_t off = block_excl_scan<uint32_t, OpSum>(run, OpSum(), 0u, &ct);
      if (d < ND) S.toff[d] = off;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kRsRounds; r++) {
      const uint32_t d = rd[r] >> 16;
      if (d < (uint32_t)ND) {
        const uint32_t pos = S.toff[d] + S.wc[w][d] + (rd[r] & 0xFFFFu);
        S.ik[b][stg<K>(pos)] = kk[r];
        S.iv[b][stg<K>(pos)] = vv[r];
      }
    }
    __syncthreads();
    const uint64_t rem = n - tbase;
    const uint32_t cnt = rem < (uint64_t)kTile ? (uint32_t)rem : (uint32_t)kTile;
#pragma unroll 4
    for (uint32_t i = threadIdx.x; i < cnt; i += kThreads) {
      const K k = S.ik[b][stg<K>(i)];
      const uint32_t d = (uint32_t)(k >> shift) & (ND - 1);
      const uint32_t gp = S.gbase[d] + (i - S.toff[d]);
      kout[gp] = k;
      vout[gp] = S.iv[b][stg<K>(i)];
    }
    __syncthreads();  // buffer b free for the TMA of tile it + 2
  }
}
template <class K, int RB = kRsBits>
inline void rs_down_tma_setup() {
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(k_rs_down_tma<K, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(RsTmaSmem<K>));
    done = true;
  }
}

template <class K, int RB>
inline void rs_down_setup() {
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(k_rs_down<K, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(RsBigSmem<K, RB>));
    done = true;
  }
}
// digit width of the large-n path.  10-bit digits save a pass for 25..30-bit
// keys but their ranking (10 ballots, 4 digits per thread, 72 KB smem) made a
// pass ~50 % slower on B200 (C5: 3 x 9.7 ms vs 4 x 6.4 ms), so 8 it is.
inline int rs_big_bits(int) { return 8; }

// ---- single-CTA sort (small n) ----------------------------------------------
// n <= kSmallSortMax(K): the whole array in shared memory, bitonic network,
// one launch instead of one per digit pass.  Not stable: callers use it only
// for distinct keys (or keys whose ties are irrelevant).
constexpr int kSmallThreads = 1024;
template <class K>
constexpr uint32_t small_sort_max() { return sizeof(K) == 8 ? 16384u : 16384u; }
template <class K>
__global__ void __launch_bounds__(kSmallThreads) k_sort_small(K* keys, uint32_t* vals, uint32_t n, uint32_t p2) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  K* sk = reinterpret_cast<K*>(smem_raw);
  uint32_t* sv = reinterpret_cast<uint32_t*>(sk + p2);
  for (uint32_t i = threadIdx.x; i < p2; i += kSmallThreads) {
    sk[i] = i < n ? keys[i] : ~(K)0;
    sv[i] = i < n ? vals[i] : 0u;
  }
  __syncthreads();
  for (uint32_t k = 2; k <= p2; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < p2; i += kSmallThreads) {
        const uint32_t l = i ^ j;
        if (l > i) {
          const K a = sk[i], b = sk[l];
          const bool up = (i & k) == 0;
          if ((a > b) == up) {
            sk[i] = b; sk[l] = a;
            const uint32_t t = sv[i]; sv[i] = sv[l]; sv[l] = t;
          }
        }
      }
      __syncthreads();
    }
  }
  for (uint32_t i = threadIdx.x; i < n; i += kSmallThreads) {
    keys[i] = sk[i];
    vals[i] = sv[i];
  }
}
// tiny sorts of distinct keys (n <= kRankSortMax): every thread ranks one key
// against all n keys staged in shared memory (broadcast reads) and writes it
// to its rank -- a few microseconds instead of a bitonic network's ~45
// CTA-wide barriers.  Not in place: writes (ko, vo).
constexpr uint32_t kRankSortMax = 2048;
template <class K>
__global__ void __launch_bounds__(kThreads) k_sort_rank(const K* __restrict__ keys, const uint32_t* __restrict__ vals,
                                                       K* __restrict__ ko, uint32_t* __restrict__ vo, uint32_t n) {
  __shared__ K sk[kRankSortMax];
  for (uint32_t i = threadIdx.x; i < n; i += kThreads) sk[i] = keys[i];
  __syncthreads();
  const uint32_t i = blockIdx.x * kThreads + threadIdx.x;
  if (i >= n) return;
  const K k = sk[i];
  uint32_t r0 = 0, r1 = 0, r2 = 0, r3 = 0;
  uint32_t j = 0;
  for (; j + 4 <= n; j += 4) {
    r0 += sk[j] < k;
    r1 += sk[j + 1] < k;
    r2 += sk[j + 2] < k;
    r3 += sk[j + 3] < k;
  }
  for (; j < n; j++) r0 += sk[j] < k;
  const uint32_t r = r0 + r1 + r2 + r3;
  ko[r] = k;
  vo[r] = vals[i];
}

template <class K>
inline void sort_small_setup() {
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(k_sort_small<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(small_sort_max<K>() * (sizeof(K) + 4)));
    done = true;
  }
}

// sizes above which the reduce-then-scan passes replace the one-sweep kernel
constexpr uint64_t kRsBigN = 1ull << 22;

struct SortScratch {
  uint32_t* ghist;              // kRsMaxPass * kRsMaxDigits, zeroed
  unsigned long long* status;   // 2 * lb_tiles(n) * kRsMaxDigits (tile aggregates, then group totals)
  uint32_t* ctrs;               // one zeroed counter per pass
  bool ghist_ready = false;     // ghist already accumulated by the key producer (k_acc_keys)
};

template <class K, int RB>
inline void rs_setup() {
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(k_rs_onesweep<K, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(RsSmem<K, RB>));
    done = true;
  }
}

// digit width of the one-sweep sort: 9 bits when that takes fewer passes
inline int rs_digit_bits(int nbits) { return (nbits + 8) / 9 < (nbits + 7) / 8 ? 9 : 8; }
inline int rs_passes(int nbits) {
  const int rb = rs_digit_bits(nbits);
  return (nbits + rb - 1) / rb;
}

template <class K, int RB>
bool radix_sort_rb(K* keys, K* keys_alt, uint32_t* vals, uint32_t* vals_alt, uint64_t n, int npass, SortScratch sc,
                   uint32_t epoch, cudaStream_t st) {
  rs_setup<K, RB>();
  const uint64_t nt = lb_tiles(n);
  if (!sc.ghist_ready)
    GW_LAUNCH((k_rs_ghist<K, RB>), (unsigned)std::min<uint64_t>(nt, 148ull * 8), kThreads, 0, st, keys, n, npass,
              sc.ghist);
  bool alt = false;
  for (int p = 0; p < npass; p++) {
    const K* ki = alt ? keys_alt : keys;
    const uint32_t* vi = alt ? vals_alt : vals;
    K* ko = alt ? keys : keys_alt;
    uint32_t* vo = alt ? vals : vals_alt;
    GW_LAUNCH((k_rs_onesweep<K, RB>), (unsigned)nt, kThreads, sizeof(RsSmem<K, RB>), st, ki, vi, ko, vo, n, p,
              sc.ghist, sc.status, sc.ctrs + p, epoch + (uint32_t)p);
    alt = !alt;
  }
  return alt;
}

// Sorts (keys, vals) by key bits [0, nbits); returns true if the result is in
// the alternate buffers.  ghist must be zeroed by the caller.
template <class K>
bool radix_sort(K* keys, K* keys_alt, uint32_t* vals, uint32_t* vals_alt, uint64_t n, int nbits, SortScratch sc,
                uint32_t epoch, cudaStream_t st) {
  if (n <= 1 || nbits <= 0) return false;
  const int npass = rs_passes(nbits);
  if (rs_digit_bits(nbits) == 9) return radix_sort_rb<K, 9>(keys, keys_alt, vals, vals_alt, n, npass, sc, epoch, st);
  return radix_sort_rb<K, 8>(keys, keys_alt, vals, vals_alt, n, npass, sc, epoch, st);
}

}  // namespace gw
