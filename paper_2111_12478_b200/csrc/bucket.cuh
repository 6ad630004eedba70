// Bucketed access pass: the address-hashed shadow table of the north_star,
// for lock-free traces of >= 2^24 events (C4, C5).
//
// Same semantics as k_access (gwcp.py:251-277; engine.py:81-95 via the dup
// list), different data movement.  The per-location check needs only that
// location's accesses in trace order, and the order in which LOCATIONS are
// visited is irrelevant (candidates carry their own order keys), so instead
// of a full LSD sort by location:
//   h = fmix32(compacted location key)      -- a bijection of u32, so h
//                                              identifies the location
//   bucket = top bb bits of h               -- ~2,048 accesses per bucket
//   two stable reduce-then-scan scatter passes (low, then high bucket digit)
//   move the 12-byte access records (h, event|W, tidop) into bucket order,
//   trace order kept inside a bucket;
//   one CTA per bucket then loads the bucket into shared memory, sorts it
//   by the remaining kb = 32 - bb bits of h (stable: the record index rides
//   in the low bits of the sort word), finds segment heads / last writes
//   with a block max-scan and evaluates the write check and the reader
//   windows entirely out of shared memory.
// Access stamps (time, pred object) are not materialised per event: only the
// candidate pairs that pass the structural tests (u != t, !cover) look them
// up in the walker's snapshot lists (StampSrc::get, L2-resident).
// HBM traffic per access: trace read 12 B (+12 B for the first up-sweep),
// 2 x (12 B read + 12 B write) for the passes, 4 B up-sweep of pass B,
// 12 B in the check; against 176 B/access of the round-1 LSD pipeline.
// Buckets larger than kBkCap records (hot locations) spill to the general
// sort + k_access path (engine.cu, bucket_spill()).
#pragma once
#include "access.cuh"

namespace gw {

__device__ __forceinline__ uint32_t bk_hash(uint32_t x) {  // murmur3 fmix32 (bijective)
  x ^= x >> 16;
  x *= 0x85ebca6bu;
  x ^= x >> 13;
  x *= 0xc2b2ae35u;
  x ^= x >> 16;
  return x;
}
__device__ __forceinline__ uint32_t bk_unhash(uint32_t x) {  // its inverse
  x ^= x >> 16;
  x *= 0x7ed1b41du;
  x ^= (x >> 13) ^ (x >> 26);
  x *= 0xa5cb9243u;
  x ^= x >> 16;
  return x;
}
// compacted key -> location key (the constant bits `base` of every access key)
__device__ __forceinline__ unsigned long long uncompact_key(unsigned long long ck, const KeyRuns& kr,
                                                           unsigned long long base) {
  unsigned long long k = base;
#pragma unroll
  for (int r = 0; r < 4; r++)
    if (r < kr.n) {
      const unsigned long long m = kr.width[r] >= 64 ? ~0ull : ((1ull << kr.width[r]) - 1ull);
      k |= ((ck >> kr.dst[r]) & m) << kr.src[r];
    }
  return k;
}

constexpr int kBkCap = 4096;      // records of one bucket in shared memory
constexpr int kBkIdxBits = 12;    // record index bits of the in-bucket sort word
constexpr int kBkSortBits = 8;    // in-bucket radix digit
constexpr uint32_t kBkSlots = 1u << kBkSortBits, kBkEmpty = 0xFFFFFFFFu;
static_assert((1 << kBkIdxBits) == kBkCap, "index bits");
constexpr int kBkMinBits = 12, kBkMaxBits = 16;  // bucket bits: 32 - kb with kb + kBkIdxBits <= 32
// buckets above kBkCap (up to kBkSubMax records) are split in the CTA into
// <= 2^kBkSubBits sub-buckets in a per-CTA scratch that stays in L2
// (sub-buckets of ~kBkSubAvg records: C5's buckets hold ~240-record own-word
// runs, so sub-buckets of ~2K overflowed kBkCap in ~0.4 % of the cases)
constexpr int kBkSubBits = 6, kBkSubAvg = 1536, kBkSubMax = 32768, kBkSubBuf = kBkSubMax + 8;

// super-tiles of the scatter passes: 2^(RB-7) tiles share one count row, so
// the count array stays at 128 words per tile for any digit width
template <int RB>
struct BkPass {
  static constexpr int ND = 1 << RB;
  static constexpr int DPT = ND > kThreads ? ND / kThreads : 1;
  static constexpr int ST = RB > 7 ? 1 << (RB - 7) : 1;
};

// ---- element sources --------------------------------------------------------
// the trace itself (pass A): element i = event i; non-access events are skipped
struct BkTraceSrc {
  DevTrace tr;
  KeyRuns kr;
  uint32_t base;  // global index of event 0 (a rank's slice in exchange mode; else 0)
  __device__ __forceinline__ uint64_t n() const { return tr.n; }
  // both columns are loaded unconditionally: independent loads, no round
  // trip on the kind before the key load is issued
  __device__ __forceinline__ bool get_h(uint64_t i, uint32_t& h) const {
    const uint32_t t = __ldcs(tr.tidop + i);
    const unsigned long long k = __ldcs(tr.key + i);
    h = bk_hash((uint32_t)compact_key(k, kr));
    return ev_kind(t) <= GW_K_WRITE;
  }
  __device__ __forceinline__ bool get(uint64_t i, uint32_t& h, uint32_t& v, uint32_t& t) const {
    t = __ldcs(tr.tidop + i);
    const unsigned long long k = __ldcs(tr.key + i);
    h = bk_hash((uint32_t)compact_key(k, kr));
    v = (base + (uint32_t)i) | (ev_kind(t) == GW_K_WRITE ? VAL_W : 0u);
    return ev_kind(t) <= GW_K_WRITE;
  }
};
// records of a previous pass (pass B)
struct BkRecSrc {
  const uint32_t* h;
  const uint32_t* v;
  const uint32_t* t;
  uint64_t cnt;
  __device__ __forceinline__ uint64_t n() const { return cnt; }
  __device__ __forceinline__ bool get_h(uint64_t i, uint32_t& hh) const {
    hh = h[i];
    return true;
  }
  __device__ __forceinline__ bool get(uint64_t i, uint32_t& hh, uint32_t& vv, uint32_t& tt) const {
    hh = h[i];
    vv = v[i];
    tt = t[i];
    return true;
  }
};

// ---- up-sweep: digit counts per super-tile (counts[d * nst + st]) ----------
template <class Src, int RB>
__global__ void __launch_bounds__(kThreads) k_bk_up(Src src, int shift, uint32_t* __restrict__ counts, uint64_t nst) {
  constexpr int ND = BkPass<RB>::ND, ST = BkPass<RB>::ST;
  __shared__ uint32_t hist[kRsWarps][ND];
  const int w = threadIdx.x >> 5;
  const uint64_t n = src.n();
  for (uint64_t st = blockIdx.x; st < nst; st += gridDim.x) {
    for (int d = threadIdx.x; d < kRsWarps * ND; d += kThreads) (&hist[0][0])[d] = 0;
    __syncthreads();
    for (int sub = 0; sub < ST; sub++) {
      const uint64_t base = (st * ST + sub) * kTile;
      if (base >= n) break;
      uint32_t hh[kItems];
      bool ok[kItems];
#pragma unroll
      for (int k = 0; k < kItems; k++) {
        const uint64_t i = base + (uint64_t)k * kThreads + threadIdx.x;
        ok[k] = i < n && src.get_h(i, hh[k]);
      }
#pragma unroll
      for (int k = 0; k < kItems; k++)
        if (ok[k]) atomicAdd(&hist[w][(hh[k] >> shift) & (ND - 1)], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < ND; d += kThreads) {
      uint32_t c = 0;
#pragma unroll
      for (int x = 0; x < kRsWarps; x++) c += hist[x][d];
      counts[(uint64_t)d * nst + st] = c;
    }
    __syncthreads();
  }
}

// ---- down-sweep: stable scatter of the records by digit ---------------------
template <int RB>
struct BkDownSmem {
  static constexpr int ND = BkPass<RB>::ND;
  uint32_t wc[kRsWarps][ND];  // per-warp digit counts -> per-warp offsets within the digit
  uint32_t toff[ND];          // tile-local start of digit d
  uint32_t gbase[ND];         // global start of this tile's digit-d run
  uint32_t sh[kTile], sv[kTile], st[kTile];
  uint32_t cnt;
};
template <class Src, int RB>
__global__ void __launch_bounds__(kThreads, 2) k_bk_down(Src src, int shift, const uint32_t* __restrict__ offsets,
                                                        uint64_t nst, uint32_t* __restrict__ oh,
                                                        uint32_t* __restrict__ ov, uint32_t* __restrict__ ot) {
  constexpr int ND = BkPass<RB>::ND, DPT = BkPass<RB>::DPT, ST = BkPass<RB>::ST;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  BkDownSmem<RB>& S = *reinterpret_cast<BkDownSmem<RB>*>(smem_raw);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t lt = lanemask_lt();
  const uint64_t n = src.n();
  for (uint64_t stl = blockIdx.x; stl < nst; stl += gridDim.x) {
    for (int d = threadIdx.x; d < ND; d += kThreads) S.gbase[d] = offsets[(uint64_t)d * nst + stl];
    for (int sub = 0; sub < ST; sub++) {
      const uint64_t tbase = (stl * ST + sub) * kTile;
      if (tbase >= n) break;
      for (int d = threadIdx.x; d < kRsWarps * ND; d += kThreads) (&S.wc[0][0])[d] = 0;
      __syncthreads();
      const uint64_t wbase = tbase + (uint64_t)w * kRsPerWarp;
      uint32_t hh[kRsRounds], vv[kRsRounds], tt[kRsRounds], rd[kRsRounds];
#pragma unroll
      for (int r = 0; r < kRsRounds; r++) {
        const uint64_t i = wbase + (uint64_t)r * 32 + lane;
        const bool ok = i < n && src.get(i, hh[r], vv[r], tt[r]);
        rd[r] = ok ? ((hh[r] >> shift) & (ND - 1)) << 16 : (uint32_t)ND << 16;
      }
#pragma unroll
      for (int r = 0; r < kRsRounds; r++) {
        const uint32_t d = rd[r] >> 16;
        const uint32_t peers = warp_peers<RB + 1>(d);
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
          if (d < ND) {
#pragma unroll
            for (int ww = 0; ww < kRsWarps; ww++) {
              const uint32_t t = S.wc[ww][d];
              S.wc[ww][d] = run;
              run += t;
            }
          }
          tot[j] = run;
          csum += run;
        }
        uint32_t ct;
        uint32_t cex = block_excl_scan<uint32_t, OpSum>(csum, OpSum(), 0u, &ct);
#pragma unroll
        for (int j = 0; j < DPT; j++) {
          const int d = threadIdx.x * DPT + j;
          if (d < ND) S.toff[d] = cex;
          cex += tot[j];
        }
        if (threadIdx.x == 0) S.cnt = ct;
      }
      __syncthreads();
#pragma unroll
      for (int r = 0; r < kRsRounds; r++) {
        const uint32_t d = rd[r] >> 16;
        if (d < (uint32_t)ND) {
          const uint32_t pos = stg<uint32_t>(S.toff[d] + S.wc[w][d] + (rd[r] & 0xFFFFu));
          S.sh[pos] = hh[r];
          S.sv[pos] = vv[r];
          S.st[pos] = tt[r];
        }
      }
      __syncthreads();
      const uint32_t cnt = S.cnt;
#pragma unroll 4
      for (uint32_t i = threadIdx.x; i < cnt; i += kThreads) {
        const uint32_t p = stg<uint32_t>(i);
        const uint32_t h = S.sh[p];
        const uint32_t d = (h >> shift) & (ND - 1);
        const uint32_t gp = S.gbase[d] + (i - S.toff[d]);
        oh[gp] = h;
        ov[gp] = S.sv[p];
        ot[gp] = S.st[p];
      }
      __syncthreads();
      for (int d = threadIdx.x; d < ND; d += kThreads) {
        const uint32_t end = d + 1 < ND ? S.toff[d + 1] : cnt;
        S.gbase[d] += end - S.toff[d];
      }
      __syncthreads();
    }
  }
}
template <class Src, int RB>
inline void bk_down_setup() {
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(k_bk_down<Src, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BkDownSmem<RB>));
    done = true;
  }
}

// ---- the same scatter with TMA-streamed input tiles --------------------------
// Full input tiles arrive by cp.async.bulk into a double buffer (the next
// tile lands while this one is ranked, as k_rs_down_tma); the buffer of the
// current tile is then reused as the digit-order staging of its three output
// arrays.  Both sources are 48 KB per 4,096-element tile: the trace's key
// (u64) + tidop columns, or the previous pass's (h, event|W, tidop).
constexpr uint32_t kBkTileBytes = kTile * 12u;
template <int RB>
struct BkTmaSmem {
  static constexpr int ND = BkPass<RB>::ND;
  uint32_t buf[2][kTile * 3];
  uint32_t wc[kRsWarps][ND];
  uint32_t toff[ND];
  uint32_t gbase[ND];
  uint32_t cnt;
  unsigned long long mbar[2];
};
__device__ __forceinline__ void bk_issue(const BkTraceSrc& s, uint64_t tile, uint32_t* dst, unsigned long long* m) {
  bulk_g2s(dst, s.tr.key + tile * kTile, kTile * 8u, m);
  bulk_g2s(dst + 2 * kTile, s.tr.tidop + tile * kTile, kTile * 4u, m);
}
__device__ __forceinline__ void bk_issue(const BkRecSrc& s, uint64_t tile, uint32_t* dst, unsigned long long* m) {
  bulk_g2s(dst, s.h + tile * kTile, kTile * 4u, m);
  bulk_g2s(dst + kTile, s.v + tile * kTile, kTile * 4u, m);
  bulk_g2s(dst + 2 * kTile, s.t + tile * kTile, kTile * 4u, m);
}
// element j of a landed tile (tile base e0)
__device__ __forceinline__ bool bk_staged(const BkTraceSrc& s, const uint32_t* b, uint64_t e0, uint32_t j, uint32_t& h,
                                          uint32_t& v, uint32_t& t) {
  t = b[2 * kTile + j];
  const unsigned long long k = reinterpret_cast<const unsigned long long*>(b)[j];
  h = bk_hash((uint32_t)compact_key(k, s.kr));
  v = (s.base + (uint32_t)(e0 + j)) | (ev_kind(t) == GW_K_WRITE ? VAL_W : 0u);
  return ev_kind(t) <= GW_K_WRITE;
}
__device__ __forceinline__ bool bk_staged(const BkRecSrc&, const uint32_t* b, uint64_t, uint32_t j, uint32_t& h,
                                          uint32_t& v, uint32_t& t) {
  h = b[j];
  v = b[kTile + j];
  t = b[2 * kTile + j];
  return true;
}
template <class Src, int RB>
__global__ void __launch_bounds__(kThreads, 2) k_bk_down_tma(Src src, int shift, const uint32_t* __restrict__ offsets,
                                                            uint64_t nst, uint32_t* __restrict__ oh,
                                                            uint32_t* __restrict__ ov, uint32_t* __restrict__ ot) {
  constexpr int ND = BkPass<RB>::ND, DPT = BkPass<RB>::DPT, ST = BkPass<RB>::ST;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  BkTmaSmem<RB>& S = *reinterpret_cast<BkTmaSmem<RB>*>(smem_raw);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t lt = lanemask_lt();
  const uint64_t n = src.n();
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  // this CTA's tiles, in order: super-tiles blockIdx.x, + gridDim.x, ...; ST tiles each
  auto tile_of = [&](uint64_t k) { return (blockIdx.x + (k / ST) * gridDim.x) * ST + k % ST; };
  auto full = [&](uint64_t tile) { return (tile + 1) * kTile <= n; };
  if (threadIdx.x == 0) {
    mbar_init(&S.mbar[0], 1);
    mbar_init(&S.mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](uint64_t tile, int b) {  // thread 0
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&S.mbar[b], kBkTileBytes);
    bk_issue(src, tile, S.buf[b], &S.mbar[b]);
  };
  uint32_t uses[2] = {0, 0};
  if (threadIdx.x == 0 && tile_of(0) < ntiles && full(tile_of(0))) issue(tile_of(0), 0);
  for (uint64_t k = 0;; k++) {
    const uint64_t tile = tile_of(k);
    if (tile >= ntiles || (k % ST == 0 && tile / ST >= nst)) break;
    const int b = (int)(k & 1);
    const uint64_t nx = tile_of(k + 1);
    if (threadIdx.x == 0 && nx < ntiles && full(nx)) issue(nx, b ^ 1);
    if (k % ST == 0)
      for (int d = threadIdx.x; d < ND; d += kThreads) S.gbase[d] = offsets[(uint64_t)d * nst + tile / ST];
    for (int d = threadIdx.x; d < kRsWarps * ND; d += kThreads) (&S.wc[0][0])[d] = 0;
    const uint64_t tbase = tile * kTile;
    uint32_t hh[kRsRounds], vv[kRsRounds], tt[kRsRounds], rd[kRsRounds];
    if (full(tile)) {
      while (!mbar_try_wait(&S.mbar[b], uses[b] & 1u)) {
      }
      uses[b]++;
#pragma unroll
      for (int r = 0; r < kRsRounds; r++) {
        const uint32_t j = w * kRsPerWarp + r * 32 + lane;
        const bool ok = bk_staged(src, S.buf[b], tbase, j, hh[r], vv[r], tt[r]);
        rd[r] = ok ? ((hh[r] >> shift) & (ND - 1)) << 16 : (uint32_t)ND << 16;
      }
    } else {
#pragma unroll
      for (int r = 0; r < kRsRounds; r++) {
        const uint64_t i = tbase + (uint64_t)w * kRsPerWarp + (uint64_t)r * 32 + lane;
        const bool ok = i < n && src.get(i, hh[r], vv[r], tt[r]);
        rd[r] = ok ? ((hh[r] >> shift) & (ND - 1)) << 16 : (uint32_t)ND << 16;
      }
    }
    __syncthreads();  // wc zeroed, gbase loaded, every thread holds its inputs
#pragma unroll
    for (int r = 0; r < kRsRounds; r++) {
      const uint32_t d = rd[r] >> 16;
      const uint32_t peers = warp_peers<RB + 1>(d);
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
        if (d < ND) {
#pragma unroll
          for (int ww = 0; ww < kRsWarps; ww++) {
            const uint32_t t = S.wc[ww][d];
            S.wc[ww][d] = run;
            run += t;
          }
        }
        tot[j] = run;
        csum += run;
      }
      uint32_t ct;
      uint32_t cex = block_excl_scan<uint32_t, OpSum>(csum, OpSum(), 0u, &ct);
#pragma unroll
      for (int j = 0; j < DPT; j++) {
        const int d = threadIdx.x * DPT + j;
        if (d < ND) S.toff[d] = cex;
        cex += tot[j];
      }
      if (threadIdx.x == 0) S.cnt = ct;
    }
    __syncthreads();
    uint32_t* sh = S.buf[b];
    uint32_t* sv = sh + kTile;
    uint32_t* sx = sv + kTile;
#pragma unroll
    for (int r = 0; r < kRsRounds; r++) {
      const uint32_t d = rd[r] >> 16;
      if (d < (uint32_t)ND) {
        const uint32_t pos = stg<uint32_t>(S.toff[d] + S.wc[w][d] + (rd[r] & 0xFFFFu));
        sh[pos] = hh[r];
        sv[pos] = vv[r];
        sx[pos] = tt[r];
      }
    }
    __syncthreads();
    const uint32_t cnt = S.cnt;
#pragma unroll 4
    for (uint32_t i = threadIdx.x; i < cnt; i += kThreads) {
      const uint32_t p = stg<uint32_t>(i);
      const uint32_t h = sh[p];
      const uint32_t d = (h >> shift) & (ND - 1);
      const uint32_t gp = S.gbase[d] + (i - S.toff[d]);
      oh[gp] = h;
      ov[gp] = sv[p];
      ot[gp] = sx[p];
    }
    __syncthreads();
    for (int d = threadIdx.x; d < ND; d += kThreads) {
      const uint32_t end = d + 1 < ND ? S.toff[d + 1] : cnt;
      S.gbase[d] += end - S.toff[d];
    }
    __syncthreads();  // gbase advanced; buffer b free for the TMA of tile k + 2
  }
}
template <class Src, int RB>
inline void bk_down_tma_setup() {
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(k_bk_down_tma<Src, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(BkTmaSmem<RB>));
    done = true;
  }
}

// ---- bucket starts: bstart[b] = first record of bucket b (bstart[NB] = n) ---
__global__ void k_bk_bounds(const uint32_t* __restrict__ h, uint64_t n, int kb, uint32_t NB, uint32_t* bstart) {
  const uint64_t nq = (n + 3) / 4;  // four records per thread, one 16-byte load
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i0 = q * 4;
    uint32_t v[4];
    if (i0 + 4 <= n) {
      const uint4 x = __ldcs(reinterpret_cast<const uint4*>(h) + q);
      v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    } else {
      for (int k = 0; k < 4; k++) v[k] = i0 + k < n ? h[i0 + k] : 0u;
    }
    uint32_t pb = i0 > 0 ? (__ldg(h + i0 - 1) >> kb) & (NB - 1) : 0u;
    for (int k = 0; k < 4 && i0 + k < n; k++) {
      const uint64_t i = i0 + k;
      const uint32_t b = (v[k] >> kb) & (NB - 1);
      if (i == 0)
        for (uint32_t x = 0; x <= b; x++) bstart[x] = 0;
      else
        for (uint32_t x = pb + 1; x <= b; x++) bstart[x] = (uint32_t)i;
      if (i + 1 == n)
        for (uint32_t x = b + 1; x <= NB; x++) bstart[x] = (uint32_t)n;
      pb = b;
    }
  }
}

// ---- the per-bucket check ---------------------------------------------------
struct BkCheckArgs {
  DevTrace tr;
  const uint32_t* h;       // bucketed records
  const uint32_t* v;
  const uint32_t* t;
  const uint32_t* bstart;  // NB + 1 bucket starts
  uint32_t NB;
  int kb;                  // in-bucket key bits
  StampSrc stamps;
  const uint32_t* arena;   // clock objects (block-range objects: lock-free traces)
  Cands c;                 // final candidates (k_bk_resolve)
  Cands pend;              // structural candidates (u != t, !cover): the clock half is resolved later
  DupList dup;
  uint32_t* large_i;       // writes with > kSmallWin reads since the last write (global record positions)
  uint32_t* large_ws;
  uint32_t* n_large;
  uint32_t large_cap;
  uint32_t* gsorted;       // in-bucket sorted event|W of the buckets holding a large window
  uint32_t* scratch;       // per CTA: 3 x kBkSubBuf words (sub-bucket split)
  uint32_t* spill;         // (start, count) of the buckets above kBkSubMax
  int xmode;               // exchange mode (multi-GPU): records from other ranks' slices, no trace access
  uint32_t* n_spill;
  uint32_t spill_cap;
};

// A bucket's three record arrays arrive by TMA bulk copies (one round trip
// per bucket, the other resident CTA computing meanwhile), 16-byte aligned:
// the copy starts up to 3 records early, so buffers hold kBkCap + 8 words.
constexpr int kBkBuf = kBkCap + 8;
struct BkSmem {
  uint32_t V[kBkBuf];      // event | VAL_W, record order (from V + off)
  uint32_t T[kBkBuf];      // tidop, record order (from T + off)
  uint32_t H[kBkBuf];      // h (TMA), then the ping-pong half of the sort
  uint32_t P[kBkCap];      // sort words (slot or key << kBkIdxBits | record)
  uint32_t wc[kRsWarps][1 << kBkSortBits];
  uint32_t toff[1 << kBkSortBits];
  uint32_t tab[kBkSlots];  // the group's locations: open addressing on the in-bucket key
  uint32_t sub[3 << kBkSubBits];  // sub-bucket counts / starts / write cursors
  uint32_t hhi;
  unsigned long long mbar;
  uint32_t large;
};

// one stable LSD pass of the in-bucket sort (bits [shift, shift + kBkSortBits))
__device__ __forceinline__ void bk_sort_pass(BkSmem& S, const uint32_t* in, uint32_t* out, uint32_t M, int shift) {
  constexpr int ND = 1 << kBkSortBits;
  constexpr int R = kBkCap / kRsWarps / 32;  // rounds per warp (16)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t lt = lanemask_lt();
  const uint32_t span = ((M + kRsWarps * 32 - 1) / (kRsWarps * 32)) * 32;  // records per warp
  const uint32_t nr = span / 32;
  for (int d = threadIdx.x; d < kRsWarps * ND; d += kThreads) (&S.wc[0][0])[d] = 0;
  __syncthreads();
  uint32_t x[R], rd[R];
#pragma unroll
  for (int r = 0; r < R; r++) {
    if ((uint32_t)r < nr) {
      const uint32_t j = w * span + r * 32 + lane;
      const bool ok = j < M;
      x[r] = ok ? in[j] : 0u;
      const uint32_t d = ok ? (x[r] >> shift) & (ND - 1) : (uint32_t)ND;
      const uint32_t peers = warp_peers<kBkSortBits + 1>(d);
      const uint32_t before = d < (uint32_t)ND ? S.wc[w][d] : 0u;
      __syncwarp();
      if (d < (uint32_t)ND && (peers & lt) == 0) S.wc[w][d] = before + __popc(peers);
      rd[r] = (d << 16) | (before + __popc(peers & lt));
      __syncwarp();
    }
  }
  __syncthreads();
  {
    const int d = threadIdx.x;  // ND == kThreads
    uint32_t run = 0;
#pragma unroll
    for (int ww = 0; ww < kRsWarps; ww++) {
      const uint32_t t = S.wc[ww][d];
      S.wc[ww][d] = run;
      run += t;
    }
    uint32_t ct;
    S.toff[d] = block_excl_scan<uint32_t, OpSum>(run, OpSum(), 0u, &ct);
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < R; r++) {
    if ((uint32_t)r < nr) {
      const uint32_t d = rd[r] >> 16;
      if (d < (uint32_t)ND) out[S.toff[d] + S.wc[w][d] + (rd[r] & 0xFFFFu)] = x[r];
    }
  }
  __syncthreads();
}

// L2 eviction policies (createpolicy): the bucketed records stream through
// L2 once (evict-first); the sub-bucket scratch is written and read back by
// the same CTA within microseconds (evict-last keeps it out of DRAM)
__device__ __forceinline__ unsigned long long l2_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long l2_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_keep(uint32_t* p, uint32_t v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, unsigned long long* m,
                                              unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(m)), "l"(pol)
      : "memory");
}

// pred_t^{vo}[u] for the accessing thread tc: lock-free clock objects are
// block-range objects of tc's block (acc_clock, blockobj case)
__device__ __forceinline__ uint32_t bk_clock(const BkCheckArgs& a, uint32_t vo, uint32_t tc, uint32_t u) {
  const uint32_t BS = a.tr.BS;
  if (vo == NIL || u / BS != tc / BS) return 0u;
  return __ldg(optr(a.arena, vo) + OBJ_HDR + (u - (tc / BS) * BS));
}

// One group of M <= kBkCap records (a bucket, or a sub-bucket in the CTA's
// scratch): TMA load of (h, event|W, tidop) from the src arrays at element
// sp; grouping by location through a small table of the group's distinct
// keys and one stable radix pass on the slot ids (full LSD passes on the
// key bits when the group holds too many locations); then per-thread
// blocked segment walks seeded by a block max-scan, and the structural half
// of the checks (the clock half: k_bk_resolve).  gpos = position of the
// group's first record in the bucketed arrays (large-window positions).
// Exchange mode (a.xmode, multi-GPU): the records come from other ranks'
// slices, so nothing is read from the trace: a pending candidate carries
// (h << 32 | prior tid) in its loc field and the current tid in kind >> 8.
constexpr uint32_t ERR_XMODE = 512;  // exchange mode met a spill / large window (host falls back)

__device__ __noinline__ void bk_group(BkSmem& S, const BkCheckArgs& a, const uint32_t* hs, const uint32_t* vs,
                                         const uint32_t* ts, uint32_t sp, uint32_t M, uint32_t gpos, int sb,
                                         uint32_t& phase) {
  constexpr uint32_t IDXM = kBkCap - 1;
  const uint32_t BS = a.tr.BS;
  const uint32_t kmask = (1u << a.kb) - 1u;
  const uint32_t a0 = sp & ~3u, off = sp - a0;
  const uint32_t bytes = ((off + M + 3u) & ~3u) * 4u;
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the previous group's generic accesses
    mbar_expect_tx(&S.mbar, 3u * bytes);
    const unsigned long long pol = l2_evict_first();  // every record is read once
    bulk_g2s_hint(S.H, hs + a0, bytes, &S.mbar, pol);
    bulk_g2s_hint(S.V, vs + a0, bytes, &S.mbar, pol);
    bulk_g2s_hint(S.T, ts + a0, bytes, &S.mbar, pol);
    S.large = 0;
  }
  while (!mbar_try_wait(&S.mbar, phase)) {
  }
  phase ^= 1u;
  const uint32_t* V = S.V + off;
  const uint32_t* T = S.T + off;
  // group by location: every distinct in-group key gets a slot of a small
  // open-addressing table; one stable radix pass on the slot id then groups
  // the records exactly, in record order.  More than kBkSlots * 3/4 distinct
  // locations: full LSD passes on the key bits instead.
  S.tab[threadIdx.x] = kBkEmpty;
  if (threadIdx.x == 0) {
    S.large = 0;
    S.hhi = S.H[off] & ~kmask;  // the group's shared high bits of h (exchange mode)
  }
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < M; j += kThreads) {
    const uint32_t key = S.H[off + j] & kmask;
    uint32_t slot = (key * 0x9E3779B1u) >> (32 - kBkSortBits), probes = 0;
    while (true) {
      uint32_t cur = S.tab[slot];
      if (cur == kBkEmpty) cur = atomicCAS(&S.tab[slot], kBkEmpty, key);
      if (cur == kBkEmpty || cur == key) break;
      slot = (slot + 1) & (kBkSlots - 1);
      if (++probes > kBkSlots * 3 / 4) { S.large = 2; break; }
    }
    S.P[j] = (slot << kBkIdxBits) | j;
  }
  __syncthreads();
  uint32_t* SP;
  const bool slotmode = S.large != 2;
  if (slotmode) {
    bk_sort_pass(S, S.P, S.H, M, kBkIdxBits);
    SP = S.H;
  } else {  // (uniform) many locations: LSD passes over the useful key bits
    for (uint32_t j = threadIdx.x; j < M; j += kThreads) S.P[j] = ((S.H[off + j] & kmask) << kBkIdxBits) | j;
    __syncthreads();
    const int ub = a.kb - sb;
    const int npass = (ub + kBkSortBits - 1) / kBkSortBits;
    uint32_t* buf[2] = {S.P, S.H};
    int cur = 0;
    for (int p = 0; p < npass; p++) {
      bk_sort_pass(S, buf[cur], buf[cur ^ 1], M, kBkIdxBits + p * kBkSortBits);
      cur ^= 1;
    }
    SP = buf[cur];
    if (threadIdx.x == 0) S.large = 0;
    __syncthreads();
  }
  // blocked segment walk: thread t owns positions [t * ipt, (t + 1) * ipt);
  // carry-in (segment head + 1, last write + 1) from a block max-scan
  const uint32_t ipt = (M + kThreads - 1) / kThreads;
  const uint32_t p0 = threadIdx.x * ipt, p1 = min(M, p0 + ipt);
  uint2 agg = make_uint2(0, 0);
  for (uint32_t p = p0; p < p1; p++) {
    const uint32_t x = SP[p];
    if (p == 0 || (x >> kBkIdxBits) != (SP[p - 1] >> kBkIdxBits)) agg.x = p + 1;
    if (V[x & IDXM] & VAL_W) agg.y = p + 1;
  }
  uint2 tot;
  uint2 run = block_excl_scan<uint2, OpMax2>(agg, OpMax2(), make_uint2(0, 0), &tot);
  for (uint32_t p = p0; p < p1; p++) {
    const uint32_t x = SP[p];
    if (p == 0 || (x >> kBkIdxBits) != (SP[p - 1] >> kBkIdxBits)) run.x = p + 1;
    // the checks (gwcp.py:251-269) of position p: run.y = last write before p + 1
    const uint32_t jx = x & IDXM;
    const uint32_t vx = V[jx], toc = T[jx];
    const uint32_t c = vx & VAL_E, tc = ev_tid(toc);
    const bool isw = (vx & VAL_W) != 0;
    const uint32_t ss = run.x - 1;
    const bool hasw = run.y > 0 && run.y - 1 >= ss;
    const uint32_t W = hasw ? run.y - 1 : NIL;
    if (isw) run.y = p + 1;
    if (p > ss && (toc & GW_F_CONT) && a.dup.ev) {
      // the previous access to this location may be in the same record
      const uint32_t pe = V[SP[p - 1] & IDXM] & VAL_E;
      if (pe < c && c - pe < 32) {
        bool same = true;
        for (uint32_t xx = pe + 1; xx < c && same; xx++) same = (__ldg(a.tr.tidop + xx) & GW_F_CONT) != 0;
        if (same) {
          const uint32_t kk = atomicAdd(a.dup.n, 1u);
          if (kk < a.dup.cap) a.dup.ev[kk] = c;
        }
      }
    }
    const uint32_t hc = S.hhi | (slotmode ? S.tab[x >> kBkIdxBits] : (x >> kBkIdxBits));
    auto pend = [&](unsigned long long okey, uint32_t prior, uint32_t u, uint32_t kind) {
      if (a.xmode)
        emit_cand(a.pend, okey, ((unsigned long long)hc << 32) | u, prior, c, kind | (tc << 8));
      else
        emit_cand(a.pend, okey, 0ull, prior, c, kind);
    };
    if (hasw) {
      const uint32_t jw = SP[W] & IDXM;
      const uint32_t pw = V[jw] & VAL_E, topw = T[jw], u = ev_tid(topw);
      if (u != tc && !cover(topw, toc, BS))  // the clock half: k_bk_resolve
        pend(((unsigned long long)c << 32) | SUB_WCHECK, pw, u, isw ? GW_WW : GW_WR);
    }
    if (!isw) continue;
    const uint32_t ws = hasw ? W + 1 : ss;
    const uint32_t m = p - ws;
    if (m == 0) continue;
    if (m > kSmallWin) {
      if (a.xmode) atomicOr(a.c.err, ERR_XMODE);
      const uint32_t kk = atomicAdd(a.n_large, 1u);
      if (kk < a.large_cap) { a.large_i[kk] = gpos + p; a.large_ws[kk] = gpos + ws; }
      else atomicOr(a.c.err, ERR_CAND);
      S.large = 1;
      continue;
    }
    // readers since W: one candidate per thread (its latest read), ranked by its first read
    for (uint32_t q = ws; q < p; q++) {
      const uint32_t jq = SP[q] & IDXM;
      const uint32_t toq = T[jq], uq = ev_tid(toq);
      if (uq == tc) continue;
      bool later = false;
      for (uint32_t q2 = q + 1; q2 < p && !later; q2++) later = ev_tid(T[SP[q2] & IDXM]) == uq;
      if (later) continue;
      uint32_t first = q;
      for (uint32_t q3 = ws; q3 < q; q3++)
        if (ev_tid(T[SP[q3] & IDXM]) == uq) { first = q3; break; }
      if (cover(toq, toc, BS)) continue;
      pend(((unsigned long long)c << 32) | SUB_READER | (first - ws), V[jq] & VAL_E, uq, GW_RW);
    }
  }
  __syncthreads();
  if (S.large)  // the large-window pass reads this group's sorted order from global memory
    for (uint32_t p = threadIdx.x; p < M; p += kThreads) a.gsorted[gpos + p] = V[SP[p] & IDXM];
  __syncthreads();
}

#ifndef GW_BK_MINB
#define GW_BK_MINB 3
#endif
__global__ void __launch_bounds__(kThreads, GW_BK_MINB) k_bk_check(BkCheckArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  BkSmem& S = *reinterpret_cast<BkSmem*>(smem_raw);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t lt = lanemask_lt();
  if (threadIdx.x == 0) {
    mbar_init(&S.mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t phase = 0;
  constexpr int kNS = 1 << kBkSubBits;
  uint32_t* sh = a.scratch + (size_t)blockIdx.x * 3 * kBkSubBuf;
  uint32_t* sv = sh + kBkSubBuf;
  uint32_t* st = sv + kBkSubBuf;
  for (uint32_t b = blockIdx.x; b < a.NB; b += gridDim.x) {
    const uint32_t s = a.bstart[b], M = a.bstart[b + 1] - s;
    if (M == 0) continue;
    if (M <= (uint32_t)kBkCap) {
      bk_group(S, a, a.h, a.v, a.t, s, M, s, 0, phase);
      continue;
    }
    // a bucket above the shared-memory capacity: split it by the top sb bits
    // of its in-bucket key into sub-buckets of ~kBkSubAvg records in this
    // CTA's scratch (L2-resident), stably, then check every sub-bucket; a
    // sub-bucket above kBkCap retries with one more bit (hashes of few
    // locations with hundreds of accesses each are lumpy)
    int sb = min(kBkSubBits, 32 - __clz((M + kBkSubAvg - 1) / kBkSubAvg - 1));
    bool spill = M > (uint32_t)kBkSubMax;
    while (!spill) {
      const int shift = a.kb - sb;
      const uint32_t nsub = 1u << sb;
      for (int d = threadIdx.x; d < kRsWarps * kNS; d += kThreads) S.wc[d / kNS][d % kNS] = 0;
      __syncthreads();
      for (uint32_t j0 = threadIdx.x; j0 < M; j0 += kThreads * 8) {  // 8 loads in flight per thread
        uint32_t hv[8];
#pragma unroll
        for (int u = 0; u < 8; u++) hv[u] = j0 + u * kThreads < M ? __ldg(a.h + s + j0 + u * kThreads) : 0u;
#pragma unroll
        for (int u = 0; u < 8; u++)
          if (j0 + u * kThreads < M) atomicAdd(&S.wc[w][(hv[u] >> shift) & (nsub - 1)], 1u);
      }
      __syncthreads();
      if (threadIdx.x < kNS) {
        uint32_t c = 0;
        for (int x = 0; x < kRsWarps; x++) c += S.wc[x][threadIdx.x];
        S.sub[threadIdx.x] = c;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        uint32_t run = 0, mx = 0;
        for (uint32_t d = 0; d < kNS; d++) {
          const uint32_t c = S.sub[d];
          mx = max(mx, c);
          S.sub[kNS + d] = run;  // sub-bucket start
          S.sub[2 * kNS + d] = run;  // write cursor
          run += c;
        }
        S.large = mx > (uint32_t)kBkCap;
      }
      __syncthreads();
      const bool over = S.large != 0;
      __syncthreads();
      if (!over) break;
      if (sb == kBkSubBits || sb == a.kb) spill = true;  // one hot location: the general path
      else sb++;
    }
    const int shift = a.kb - sb;
    const uint32_t nsub = 1u << sb;
    if (spill) {  // hot locations: the general path (bucket_spill)
      if (threadIdx.x == 0) {
        if (a.xmode) atomicOr(a.c.err, ERR_XMODE);
        const uint32_t k = atomicAdd(a.n_spill, 1u);
        if (k < a.spill_cap) { a.spill[2 * k] = s; a.spill[2 * k + 1] = M; }
      }
      __syncthreads();
      continue;
    }
    const unsigned long long keep = l2_evict_last();
    // stable scatter into the scratch, kSubChunk records per round
    constexpr int R = 8, kSubChunk = kRsWarps * 32 * R;
    for (uint32_t cb = 0; cb < M; cb += kSubChunk) {
      for (int d = threadIdx.x; d < kRsWarps * kNS; d += kThreads) S.wc[d / kNS][d % kNS] = 0;
      __syncthreads();
      uint32_t hh[R], vv[R], tt[R], rd[R];
#pragma unroll
      for (int r = 0; r < R; r++) {
        const uint32_t j = cb + w * (32 * R) + r * 32 + lane;
        const bool ok = j < M;
        hh[r] = ok ? a.h[s + j] : 0u;
        vv[r] = ok ? a.v[s + j] : 0u;
        tt[r] = ok ? a.t[s + j] : 0u;
        rd[r] = ok ? ((hh[r] >> shift) & (nsub - 1)) << 16 : (uint32_t)kNS << 16;
      }
#pragma unroll
      for (int r = 0; r < R; r++) {
        const uint32_t d = rd[r] >> 16;
        const uint32_t peers = warp_peers<kBkSubBits + 1>(d);
        const uint32_t before = d < (uint32_t)kNS ? S.wc[w][d] : 0u;
        __syncwarp();
        if (d < (uint32_t)kNS && (peers & lt) == 0) S.wc[w][d] = before + __popc(peers);
        rd[r] |= before + __popc(peers & lt);
        __syncwarp();
      }
      __syncthreads();
      if (threadIdx.x < kNS) {  // per-warp offsets within the digit, advance the cursor
        const int d = threadIdx.x;
        uint32_t run = S.sub[2 * kNS + d];
        for (int x = 0; x < kRsWarps; x++) {
          const uint32_t t = S.wc[x][d];
          S.wc[x][d] = run;
          run += t;
        }
        S.sub[2 * kNS + d] = run;
      }
      __syncthreads();
#pragma unroll
      for (int r = 0; r < R; r++) {
        const uint32_t d = rd[r] >> 16;
        if (d < (uint32_t)kNS) {
          const uint32_t pos = S.wc[w][d] + (rd[r] & 0xFFFFu);
          st_keep(sh + pos, hh[r], keep);  // L2 evict-last: read back by TMA right below
          st_keep(sv + pos, vv[r], keep);
          st_keep(st + pos, tt[r], keep);
        }
      }
      __syncthreads();
    }
    // the scratch was written by generic stores; the sub-bucket loads are TMA (async proxy)
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __syncthreads();
    for (uint32_t d = 0; d < nsub; d++) {
      const uint32_t m = S.sub[d], o = S.sub[kNS + d];
      if (m) bk_group(S, a, sh, sv, st, o, m, s + o, sb, phase);
    }
  }
}
// the clock half of the structural candidates (gwcp.py:256, :265):
// race iff prior.time > pred_t^{ver}[u]; stamps from the walker's snapshots
struct BkXInfo {  // exchange mode: location keys from h (bk_unhash + uncompact_key)
  int on;
  KeyRuns kr;
  unsigned long long base;
};
__global__ void k_bk_resolve(Cands pend, DevTrace tr, StampSrc stamps, const uint32_t* arena, Cands out,
                             BkXInfo xi) {
  const uint32_t n = min(*pend.n, pend.cap);
  const uint32_t BS = tr.BS;
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const uint32_t p = pend.prior[k], c = pend.cur[k];
    if (xi.on) {
      const unsigned long long lx = pend.loc[k];
      const uint32_t kx = pend.kind[k], tc = kx >> 8, u = (uint32_t)lx & GW_TID_MASK;
      const uint32_t vo = stamps.get(c, tc).y;
      const uint32_t t = stamps.get(p, u).x;
      const uint32_t clk =
          (vo == NIL || u / BS != tc / BS) ? 0u : __ldg(optr(arena, vo) + OBJ_HDR + (u - (tc / BS) * BS));
      if (t > clk)
        emit_cand(out, pend.okey[k], uncompact_key(bk_unhash((uint32_t)(lx >> 32)), xi.kr, xi.base), p, c, kx & 3u);
      continue;
    }
    const uint32_t tc = ev_tid(__ldg(tr.tidop + c)), u = ev_tid(__ldg(tr.tidop + p));
    const uint32_t vo = stamps.get(c, tc).y;
    const uint32_t t = stamps.get(p, u).x;
    const uint32_t clk =
        (vo == NIL || u / BS != tc / BS) ? 0u : __ldg(optr(arena, vo) + OBJ_HDR + (u - (tc / BS) * BS));
    if (t > clk) emit_cand(out, pend.okey[k], tr.key[c], p, c, pend.kind[k]);
  }
}

inline void bk_check_setup() {
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(k_bk_check, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BkSmem));
    done = true;
  }
}

// spilled buckets -> (h, event|W) arrays for the general sort + k_access path
__global__ void k_bk_spill_gather(const uint32_t* __restrict__ h, const uint32_t* __restrict__ v,
                                  const uint32_t* spill, const uint32_t* soff, uint32_t nsp, uint32_t* kout,
                                  uint32_t* vout) {
  for (uint32_t k = blockIdx.x; k < nsp; k += gridDim.x) {
    const uint32_t s = spill[2 * k], m = spill[2 * k + 1], o = soff[k];
    for (uint32_t j = threadIdx.x; j < m; j += blockDim.x) {
      kout[o + j] = h[s + j];
      vout[o + j] = v[s + j];
    }
  }
}

}  // namespace gw
