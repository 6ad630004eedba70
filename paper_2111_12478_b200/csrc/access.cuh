// Access pass of the G-WCP engine: the data-parallel core.
//
// Reference semantics (pkg/src/gpurace/gwcp.py:251-277, engine.py:81-95,
// report.py:79-100, scopes.py:32-47):
//   prior write W = last write to loc in trace order (any thread)
//     report ww|wr iff W.tid != t && W.time > pred_t[W.tid] && !atomics_cover
//   on a write, for each reader u since W in first-insertion order carrying
//   u's latest read r: report rw iff u != t && r.time > pred_t[u] && !cover
//   multi-lane WRITE records: ww(i, j) for lanes i < j on one location
//   Reporter: keep-first on (loc, prior.instr, current.instr); first -> "first"
//
// Batch form: sort accesses by (location, event) with a
// stable LSD radix sort on the compacted location key, find each access's
// prior write / segment head with one max-scan, evaluate every candidate pair
// with a single u32 gather pred_t^{ver}[u] from the walker's clock objects,
// and order the survivors by the key
//   (event, 0, i, j)  same-instruction pair of the record starting at event
//   (event, 1, 0, 0)  write check
//   (event, 1, 1, k)  k-th reader (k = rank of the reader's first read)
// which reproduces the reference's report sequence exactly.
#pragma once
#include "walker_warp.cuh"

namespace gw {

constexpr uint32_t kSmallWin = 32;
// sorted values: event index | VAL_W for writes (event indices < 2^31)
constexpr uint32_t VAL_W = 0x80000000u, VAL_E = 0x7FFFFFFFu;
constexpr unsigned long long SUB_WCHECK = 0x40000000ull;
constexpr unsigned long long SUB_READER = 0x80000000ull;

struct KeyRuns {  // compacted location key = concatenation of the varying bit runs
  int n;
  int src[4], width[4], dst[4];
  int nbits;     // sort bits: varying location bits (+1 sentinel bit when it fits)
  int sentinel;  // non-access events carry bit nbits-1
};

// Access-time stamps (time = local_t at the access, vobj = t's pred object):
// arrays written by the walker, or -- lock-free snapshot mode -- looked up in
// the walker's per-block snapshots: snapshot k of block b = the block's
// state after its k-th hard event (k = #hard events of b before e).
struct StampSrc {  // valid() false in lock mode (the walker runs after the access pass)
  const uint32_t* time;  // arrays (nullptr: snapshots)
  const uint32_t* vobj;
  const uint32_t* hard_ev;
  const uint32_t* hb_beg;
  const uint32_t* hb_end;
  const uint2* snap;
  uint32_t BS;
  uint32_t warp_mode;  // snapshot lists per (block, warp) (k_walker_wsnap), rows of 32
  uint32_t L;
  __device__ __forceinline__ bool valid() const { return time != nullptr || snap != nullptr; }
  __device__ __forceinline__ uint2 get(uint32_t e, uint32_t t) const {
    if (time) return make_uint2(__ldg(time + e), __ldg(vobj + e));
    const uint32_t b = t / BS;
    const uint32_t g = warp_mode ? b * 8u + (t - b * BS) / L : b;
    const uint32_t base = __ldg(hb_beg + g);
    uint32_t lo = base, hi = __ldg(hb_end + g);
    if (hi - lo <= 16) {  // short lists (C2 / C5: 16 per block): one round of independent loads
      uint32_t c = 0;
#pragma unroll
      for (int k = 0; k < 16; k++) c += (lo + k < hi && __ldg(hard_ev + lo + k) < e) ? 1u : 0u;
      lo += c;
    } else {
      while (lo < hi) {
        const uint32_t m = (lo + hi) >> 1;
        if (__ldg(hard_ev + m) < e) lo = m + 1; else hi = m;
      }
    }
    return warp_mode ? snap[(size_t)(lo + g) * 32 + (t - b * BS) % L] : snap[(size_t)(lo + g) * BS + (t - b * BS)];
  }
};

// Non-access events get the sentinel key (bit nbits-1, one past the varying
// location bits) and sort last; in the corner case of 64 varying bits there is
// no spare bit and they take key 0 instead.  Either way every access-pass
// kernel skips them.
// Also writes aux[e] = (tidop, time, vobj) for the access pass: in trace order
// the stamp lookups of a warp hit one block's snapshot list, and the check
// later fetches everything it needs about an access with ONE 16-byte gather.
__device__ __forceinline__ uint4 make_aux(const StampSrc& src, uint32_t e, uint32_t to) {
  uint2 st = make_uint2(0u, NIL);
  if (ev_kind(to) <= GW_K_WRITE && src.valid()) st = src.get(e, ev_tid(to));
  return make_uint4(to, st.x, st.y, 0u);
}
// ghist != nullptr: also the digit histograms of the one-sweep sort that
// follows (npass passes of rb-bit digits; k_rs_ghist's job, without a second
// read of the keys)
template <class K>
__global__ void k_acc_keys(DevTrace tr, KeyRuns kr, K* keys, uint32_t* vals, StampSrc src, uint4* aux,
                           uint32_t* ghist = nullptr, int rb = 0, int npass = 0) {
  __shared__ uint32_t h[kRsMaxPass * kRsMaxDigits];
  const uint32_t nd = 1u << rb;
  if (ghist) {
    for (uint32_t i = threadIdx.x; i < npass * nd; i += blockDim.x) h[i] = 0;
    __syncthreads();
  }
  const K sentinel = kr.sentinel ? ((K)1 << (kr.nbits - 1)) : (K)0;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tr.n; e += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t to = tr.tidop[e];
    if (aux) aux[e] = make_aux(src, (uint32_t)e, to);
    K k = sentinel;
    if (ev_kind(to) <= GW_K_WRITE) {
      unsigned long long x = tr.key[e];
      k = 0;
#pragma unroll
      for (int r = 0; r < 4; r++)
        if (r < kr.n) k |= (K)((x >> kr.src[r]) & ((1ull << kr.width[r]) - 1ull)) << kr.dst[r];
    }
    keys[e] = k;
    vals[e] = (uint32_t)e | (ev_kind(to) == GW_K_WRITE ? VAL_W : 0u);
    if (ghist)
      for (int p = 0; p < npass; p++) atomicAdd(&h[p * nd + ((uint32_t)(k >> (rb * p)) & (nd - 1))], 1u);
  }
  if (ghist) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < npass * nd; i += blockDim.x)
      if (h[i]) atomicAdd(&ghist[i], h[i]);
  }
}

// the stamps alone (the fork of Pipeline::run sorts the keys concurrently with the sync pass)
__global__ void k_acc_aux(DevTrace tr, StampSrc src, uint4* aux) {
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tr.n; e += (uint64_t)gridDim.x * blockDim.x)
    aux[e] = make_aux(src, (uint32_t)e, tr.tidop[e]);
}

// ---- address sharding -----------------------------------------------------
__device__ __forceinline__ unsigned long long compact_key(unsigned long long x, const KeyRuns& kr) {
  unsigned long long k = 0;
#pragma unroll
  for (int r = 0; r < 4; r++)
    if (r < kr.n) k |= ((x >> kr.src[r]) & ((kr.width[r] >= 64) ? ~0ull : ((1ull << kr.width[r]) - 1ull))) << kr.dst[r];
  return k;
}
struct ShardArgs {
  KeyRuns kr;
  int nloc;        // location bits of the compacted key
  uint32_t shard;  // this call's shard
  uint32_t G;      // shard count (1: unsharded)
};
// contiguous ranges of the compacted location key
__device__ __forceinline__ uint32_t shard_of(unsigned long long ck, const ShardArgs& sa) {
  if (sa.G <= 1 || sa.nloc <= 0) return 0;
  return (uint32_t)__umul64hi(ck << (64 - sa.nloc), (unsigned long long)sa.G);
}
__device__ __forceinline__ bool in_shard(unsigned long long loc, const ShardArgs& sa) {
  return sa.G <= 1 || shard_of(compact_key(loc, sa.kr), sa) == sa.shard;
}
// order-preserving compaction of this shard's accesses (tile = kTile events):
// count per tile, then (after an exclusive scan of the counts) emit
// (compacted location key, event) in trace order
template <class K, bool EMIT>
__global__ void __launch_bounds__(kThreads) k_shard_accesses(DevTrace tr, ShardArgs sa, uint32_t* tilecnt,
                                                            const uint32_t* tileoff, K* keys, uint32_t* vals,
                                                            StampSrc src, uint4* aux) {
  __shared__ uint32_t s_w[kThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t lt = lanemask_lt();
  const uint64_t ntiles = (tr.n + kTile - 1) / kTile;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint64_t base = tile * kTile;
    uint32_t run = EMIT ? tileoff[tile] : 0u;
#pragma unroll 4
    for (int k = 0; k < kItems; k++) {
      const uint64_t e = base + (uint64_t)k * kThreads + threadIdx.x;
      bool in = false;
      unsigned long long ck = 0;
      if (e < tr.n && ev_kind(tr.tidop[e]) <= GW_K_WRITE) {
        ck = compact_key(tr.key[e], sa.kr);
        in = shard_of(ck, sa) == sa.shard;
      }
      const uint32_t m = __ballot_sync(0xffffffffu, in);
      if (lane == 0) s_w[w] = __popc(m);
      __syncthreads();
      uint32_t woff = 0, tot = 0;
#pragma unroll
      for (int x = 0; x < kThreads / 32; x++) {
        const uint32_t c = s_w[x];
        woff += x < w ? c : 0u;
        tot += c;
      }
      if (EMIT && in) {
        const uint32_t pos = run + woff + __popc(m & lt);
        const uint32_t to = tr.tidop[e];
        keys[pos] = (K)ck;
        vals[pos] = (uint32_t)e | (ev_kind(to) == GW_K_WRITE ? VAL_W : 0u);
        if (aux) aux[e] = make_aux(src, (uint32_t)e, to);
      }
      run += tot;
      __syncthreads();
    }
    if (!EMIT && threadIdx.x == 0) tilecnt[tile] = run;
  }
}

// compact arbitrary u64 keys to their varying bit runs
__global__ void k_compact_u64(const unsigned long long* in, uint64_t n, KeyRuns kr, unsigned long long* out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long x = in[i];
    unsigned long long k = 0;
#pragma unroll
    for (int r = 0; r < 4; r++)
      if (r < kr.n) k |= ((x >> kr.src[r]) & ((kr.width[r] >= 64) ? ~0ull : ((1ull << kr.width[r]) - 1ull))) << kr.dst[r];
    out[i] = k;
  }
}

// stats over the trace (one pass): counts by kind, OR / AND of access keys
struct Stats {
  unsigned long long n_acc, n_write, n_acq, n_rel, n_end, n_bar, key_or, key_and;
  unsigned long long n_long;  // windows proving a record longer than 32 events
  unsigned long long n_wbar;  // warp barriers (of n_bar)
};
__device__ __forceinline__ void prep_flush(unsigned long long (&v)[6], unsigned long long ko, unsigned long long ka,
                                           unsigned long long nlong, unsigned long long nwbar, Stats* st);
// per-event stats of k_prep / k_ingest (counts by kind, OR / AND of access keys)
__device__ __forceinline__ void prep_count(uint32_t to, unsigned long long x, unsigned long long (&v)[6],
                                           unsigned long long& ko, unsigned long long& ka,
                                           unsigned long long& nwbar) {
  const uint32_t k = ev_kind(to);
  if (k <= GW_K_WRITE) { v[0]++; v[1] += k; ko |= x; ka &= x; }
  else if (k == GW_K_ACQUIRE) v[2]++;
  else if (k == GW_K_RELEASE) v[3]++;
  else if (k == GW_K_END) v[4]++;
  else if (k == GW_K_BARRIER) { v[5]++; if (to & GW_F_WARPBAR) nwbar++; }
}
__global__ void __launch_bounds__(kThreads) k_prep(DevTrace tr, Stats* st) {
  unsigned long long v[6] = {0, 0, 0, 0, 0, 0};  // acc, write, acq, rel, end, bar
  unsigned long long ko = 0, ka = ~0ull, nlong = 0, nwbar = 0;
  const int lane = threadIdx.x & 31;
  constexpr int U = 4;  // aligned 32-event windows per warp iteration: all loads issued first
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * U;
  for (uint64_t b0 = ((uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u)) * U; b0 < tr.n; b0 += stride) {
    uint32_t to[U];
    unsigned long long x[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint64_t e = b0 + 32 * u + lane;
      to[u] = e < tr.n ? tr.tidop[e] : (7u << GW_OP_SHIFT);
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint64_t e = b0 + 32 * u + lane;
      x[u] = ev_kind(to[u]) <= GW_K_WRITE ? tr.key[e] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < U; u++) prep_count(to[u], x[u], v, ko, ka, nwbar);
    // records longer than 32 events: 32 consecutive continues-record events ending in a window
    uint32_t prevm = 0;
    bool have_prev = false;
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint64_t w0 = b0 + 32 * u;
      if (w0 >= tr.n) break;
      const uint32_t cur = __ballot_sync(0xffffffffu, (to[u] & GW_F_CONT) != 0 && ev_kind(to[u]) != 7u);
      if (cur == 0xffffffffu) {
        if (lane == 0) nlong++;  // a whole window of continuations: the record has > 32 events
      } else if (cur & 1u) {    // a run entering the window: add the previous window's trailing run
        uint32_t prev = prevm;
        if (!have_prev)
          prev = __ballot_sync(0xffffffffu, w0 >= 32 && (tr.tidop[w0 - 32 + lane] & GW_F_CONT));
        unsigned long long y = ((unsigned long long)cur << 32) | prev;
        y &= y >> 1; y &= y >> 2; y &= y >> 4; y &= y >> 8; y &= y >> 16;  // bit i: bits i..i+31 all set
        if (lane == 0 && ((y >> 1) & 0xFFFFFFFFull)) nlong++;
      }
      prevm = cur;
      have_prev = true;
    }
  }
  prep_flush(v, ko, ka, nlong, nwbar, st);
}
// the per-thread stats of k_prep / k_ingest into *st (warp, CTA, then global atomics)
__device__ __forceinline__ void prep_flush(unsigned long long (&v)[6], unsigned long long ko, unsigned long long ka,
                                           unsigned long long nlong, unsigned long long nwbar, Stats* st) {
  const int lane = threadIdx.x & 31;
  if (lane == 0 && nlong) atomicAdd(&st->n_long, nlong);
  nwbar = __reduce_add_sync(0xffffffffu, (uint32_t)nwbar);
  if (lane == 0 && nwbar) atomicAdd(&st->n_wbar, nwbar);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int i = 0; i < 6; i++) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
    ko |= __shfl_xor_sync(0xffffffffu, ko, o);
    ka &= __shfl_xor_sync(0xffffffffu, ka, o);
  }
  __shared__ unsigned long long s_v[kThreads / 32][8];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int i = 0; i < 6; i++) s_v[w][i] = v[i];
    s_v[w][6] = ko;
    s_v[w][7] = ka;
  }
  __syncthreads();
  if (threadIdx.x < 8) {
    const int i = threadIdx.x;
    unsigned long long r = i == 7 ? ~0ull : 0ull;
    for (int x = 0; x < kThreads / 32; x++) {
      if (i < 6) r += s_v[x][i];
      else if (i == 6) r |= s_v[x][i];
      else r &= s_v[x][i];
    }
    unsigned long long* dst[8] = {&st->n_acc, &st->n_write, &st->n_acq, &st->n_rel, &st->n_end, &st->n_bar,
                                  &st->key_or, &st->key_and};
    if (i < 6) { if (r) atomicAdd(dst[i], r); }
    else if (i == 6) atomicOr(dst[i], r);
    else atomicAnd(dst[i], r);
  }
}

// Graph replays of big lock-free traces: ONE read of the trace does the work
// of k_prep (the stats the plan check verifies), k_acc_keys (location keys /
// events), the first sort pass's per-tile digit counts (k_rs_up, pass 0: the
// ingest tiles are the sort's kTile tiles) and, in snapshot mode,
// k_hard_append.  Warp w of tile t at step k reads the aligned 32-event window
// t*kTile + k*kThreads + 32w, so the long-record test is k_prep's.
struct IngestHard {
  unsigned long long* hkey;  // nullptr: no hard-event list here
  uint32_t* hcnt;
  uint32_t* ntop;
  uint32_t cap;
};
template <class K>
__global__ void __launch_bounds__(kThreads) k_ingest(DevTrace tr, KeyRuns kr, K* keys, uint32_t* vals, Stats* stt,
                                                    uint32_t* counts, uint64_t nst, IngestHard hd, int rb0) {
  __shared__ uint32_t h[kRsWarps][kRsDigits];
  unsigned long long v[6] = {0, 0, 0, 0, 0, 0};
  unsigned long long ko = 0, ka = ~0ull, nlong = 0, nwbar = 0;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const K sentinel = kr.sentinel ? ((K)1 << (kr.nbits - 1)) : (K)0;
  for (uint64_t t = blockIdx.x; t < nst; t += gridDim.x) {
    for (int d = threadIdx.x; d < kRsWarps * kRsDigits; d += kThreads) (&h[0][0])[d] = 0;
    __syncthreads();
    const uint64_t base = t * kTile;
    constexpr int U = 4;  // loads of U windows issued together (key loads do not wait for the kinds)
#pragma unroll 1
    for (int k0 = 0; k0 < kItems; k0 += U) {
    uint32_t tob[U];
    unsigned long long xb[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint64_t e = base + (uint64_t)(k0 + u) * kThreads + 32u * w + lane;
      tob[u] = e < tr.n ? tr.tidop[e] : (7u << GW_OP_SHIFT);
      xb[u] = e < tr.n ? tr.key[e] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int k = k0 + u;
      const uint64_t w0 = base + (uint64_t)k * kThreads + 32u * w;
      const uint64_t e = w0 + lane;
      const uint32_t to = tob[u];
      const uint32_t kind = ev_kind(to);
      const unsigned long long x = kind <= GW_K_WRITE ? xb[u] : 0ull;
      prep_count(to, x, v, ko, ka, nwbar);
      if (e < tr.n) {
        K ck = sentinel;
        if (kind <= GW_K_WRITE) {
          ck = 0;
#pragma unroll
          for (int r = 0; r < 4; r++)
            if (r < kr.n) ck |= (K)((x >> kr.src[r]) & ((1ull << kr.width[r]) - 1ull)) << kr.dst[r];
        }
        keys[e] = ck;
        vals[e] = (uint32_t)e | (kind == GW_K_WRITE ? VAL_W : 0u);
        atomicAdd(&h[w][(uint32_t)ck & ((1u << rb0) - 1u)], 1u);
      }
      if (w0 < tr.n) {  // records longer than 32 events (k_prep)
        const uint32_t cur = __ballot_sync(0xffffffffu, (to & GW_F_CONT) != 0 && kind != 7u);
        if (cur == 0xffffffffu) {
          if (lane == 0) nlong++;
        } else if (cur & 1u) {
          const uint32_t prev = __ballot_sync(0xffffffffu, w0 >= 32 && (tr.tidop[w0 - 32 + lane] & GW_F_CONT));
          unsigned long long y = ((unsigned long long)cur << 32) | prev;
          y &= y >> 1; y &= y >> 2; y &= y >> 4; y &= y >> 8; y &= y >> 16;
          if (lane == 0 && ((y >> 1) & 0xFFFFFFFFull)) nlong++;
        }
      }
      if (hd.hkey) {  // k_hard_append
        const bool hard = kind == GW_K_BARRIER || kind == GW_K_END;
        const uint32_t m = __ballot_sync(0xffffffffu, hard);
        if (m) {
          uint32_t hb = 0;
          if (lane == __ffs(m) - 1) hb = atomicAdd(hd.ntop, (uint32_t)__popc(m));
          hb = __shfl_sync(0xffffffffu, hb, __ffs(m) - 1);
          if (hard) {
            const uint32_t b = ev_tid(to) / tr.BS;
            const uint32_t slot = hb + __popc(m & lanemask_lt());
            if (slot < hd.cap) hd.hkey[slot] = ((unsigned long long)b << 32) | (uint32_t)e;
            atomicAdd(hd.hcnt + b, 1u);
          }
        }
      }
    }
    }
    __syncthreads();
    {
      const int d = threadIdx.x;  // kRsDigits == kThreads
      if (d < (1 << rb0)) {
        uint32_t c = 0;
#pragma unroll
        for (int x = 0; x < kRsWarps; x++) c += h[x][d];
        counts[(uint64_t)d * nst + t] = c;
      }
    }
    __syncthreads();
  }
  prep_flush(v, ko, ka, nlong, nwbar, stt);
}

__global__ void k_part_keys(DevTrace tr, uint32_t G, uint32_t* keys, uint32_t* vals) {
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tr.n; e += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t b = ev_tid(tr.tidop[e]) / tr.BS;
    keys[e] = b % G;
    vals[e] = (uint32_t)e;
  }
}

struct OpMax2 {
  __device__ __forceinline__ uint2 operator()(const uint2& a, const uint2& b) const {
    return make_uint2(max(a.x, b.x), max(a.y, b.y));
  }
};

struct Cands {
  unsigned long long* okey;
  unsigned long long* loc;
  uint32_t* prior;
  uint32_t* cur;
  uint32_t* kind;
  uint32_t* n;
  uint32_t cap;
  uint32_t* err;
};

__device__ __forceinline__ void emit_cand(const Cands& c, unsigned long long okey, unsigned long long loc,
                                          uint32_t prior, uint32_t cur, uint32_t kind) {
  uint32_t i = atomicAdd(c.n, 1u);
  if (i >= c.cap) { atomicOr(c.err, ERR_CAND); return; }
  c.okey[i] = okey; c.loc[i] = loc; c.prior[i] = prior; c.cur[i] = cur; c.kind[i] = kind;
}

// atomics_cover, scopes.py:32-47 (tids flat; block = tid / BS)
__device__ __forceinline__ bool cover(uint32_t toa, uint32_t tob, uint32_t BS) {
  if (!((toa & GW_F_ATOMIC) && (tob & GW_F_ATOMIC))) return false;
  if ((toa & GW_F_DEVICE) || (tob & GW_F_DEVICE)) return true;
  return ev_tid(toa) / BS == ev_tid(tob) / BS;
}

// same-record pairs on one location flagged by k_access (see k_dup_heads)
struct DupList {
  uint32_t* ev;
  uint32_t* n;
  uint32_t cap;
};

// The access check (gwcp.py:251-277) over the location-sorted accesses, one
// tile of kThreads * I sorted positions per CTA (I items per thread):
//   * segment head / last write before each position: a tile-local max-scan
//     seeded with the maxima of all earlier tiles (k_acc_tilemax + a scan
//     over tiles), no per-position scan arrays in HBM;
//   * the tile's event indices and (tidop, time, vobj) -- one 16-byte
//     gather per access -- staged in smem, so the prior write and the reader
//     window are mostly smem reads;
//   * the clock test is one gather pred_t^{ver}[u]; lock-free clock objects
//     are block-range objects of the accessing thread's block (the barrier
//     hull never leaves it), so the header need not be read.
// defer (lock mode): every structural candidate (u != t, !cover) is emitted
// and the walker answers the clock half later.
// Items per thread (tile = kThreads * items positions): 8, or 10 when that
// brings a trace into one wave of resident CTAs (acc_items(), engine.cu; C2:
// 513 tiles of 2,048 -> 410 of 2,560 on 444 slots).  Larger tiles cost
// occupancy on billion-event traces, so those keep 8.
constexpr int kAccItemsSmall = 8, kAccItemsLarge = 10;

template <class K>
struct AccArgs {
  DevTrace tr;
  const K* keys;          // sorted compacted location keys (non-accesses: sentinel, last)
  const uint32_t* vals;   // sorted event | VAL_W
  uint64_t n;             // sorted positions
  const uint2* carry;     // per tile: max (head pos + 1, write pos + 1) over all earlier tiles
  const uint4* aux;       // per event: (tidop, time, vobj) -- see k_acc_keys; nullptr: looked up lazily
  StampSrc stamps;        // (aux == nullptr) stamp source of the lazy lookups
  const uint32_t* arena;
  int defer;
  int blockobj;           // clock objects are block-range objects (lock-free traces)
  Cands c;
  uint32_t* large_i;      // writes with a reader window > kSmallWin
  uint32_t* large_ws;
  uint32_t* n_large;
  uint32_t large_cap;
  DupList dup;            // same-record pairs on one location (same-instruction check)
  uint32_t* tile_ctr;     // zeroed: tiles are taken in order (atomicAdd)
  unsigned long long* lb; // non-null: the carry by decoupled look-back (zeroed, one word per tile) instead of carry[]
};

// (tidop, time, vobj) of event ev: the aux record, or (bucket pass spill and
// large windows) the trace's tidop and a stamp lookup
template <class K>
__device__ __forceinline__ uint4 acc_aux(const AccArgs<K>& a, uint32_t ev) {
  if (a.aux) return a.aux[ev];
  return make_aux(a.stamps, ev, __ldg(a.tr.tidop + ev));
}

template <class K, int I>
__global__ void __launch_bounds__(kThreads) k_acc_tilemax(const K* keys, const uint32_t* vals, uint64_t n,
                                                         uint2* agg) {
  __shared__ uint32_t s_h[kThreads / 32], s_w[kThreads / 32];
  const uint64_t ntiles = (n + (kThreads * I) - 1) / (kThreads * I);
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint64_t base = tile * (kThreads * I);
    uint32_t h = 0, w = 0;
#pragma unroll
    for (int k = 0; k < I; k++) {
      const uint64_t i = base + (uint64_t)k * kThreads + threadIdx.x;
      if (i < n) {
        if (i == 0 || keys[i] != keys[i - 1]) h = (uint32_t)i + 1;
        if (vals[i] & VAL_W) w = (uint32_t)i + 1;
      }
    }
    h = __reduce_max_sync(0xffffffffu, h);
    w = __reduce_max_sync(0xffffffffu, w);
    if ((threadIdx.x & 31) == 0) { s_h[threadIdx.x >> 5] = h; s_w[threadIdx.x >> 5] = w; }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int x = 0; x < kThreads / 32; x++) { h = max(h, s_h[x]); w = max(w, s_w[x]); }
      agg[tile] = make_uint2(h, w);
    }
    __syncthreads();
  }
}

// LAZY: no per-event aux array -- the tile stages the tidops (one 4-byte
// gather per access) and looks the (time, vobj) stamps up only for the
// positions that reach a clock test (stamps from the walker's snapshots or
// arrays, L2-resident); saves the 16-byte aux write + gather per event.
// S.ss flag: every access of the segment up to this position is by one
// thread, so the position has no prior-write / reader candidate
constexpr uint32_t SS_SINGLE = 0x80000000u;
// padded tile index: one spare word per 32, so both the striped (staging,
// checks) and the blocked (scan) access patterns are bank-conflict free
__device__ __forceinline__ uint32_t apx(uint32_t j) { return j + (j >> 5); }
template <class K, int I, bool LAZY = false>
struct AccSmem {
  static constexpr uint32_t P = kThreads * I + (kThreads * I) / 32;
  K key[P];
  uint32_t val[P];
  uint32_t to[P];
  uint32_t lw[P];   // inclusive last write pos + 1
  uint32_t ss[P];   // segment head pos | SS_SINGLE
  uint2 st[LAZY ? 1 : (kThreads * I)];  // (time, vobj) stamps
  uint3 wtot[kThreads / 32];
  uint32_t ltot[kThreads / 32];
  uint32_t next_tile;
  uint2 cin;  // the tile's carry (look-back)
};

// (event, tidop) of sorted position q (smem when q is in this tile)
template <class K, int I, bool LAZY>
__device__ __forceinline__ void acc_pos(const AccArgs<K>& a, const AccSmem<K, I, LAZY>& S, uint32_t base, uint32_t q,
                                        uint32_t& ev, uint32_t& to) {
  if (q >= base) {
    ev = S.val[apx(q - base)] & VAL_E;
    to = S.to[apx(q - base)];
  } else {
    ev = __ldg(a.vals + q) & VAL_E;
    to = a.aux ? __ldg(&a.aux[ev].x) : __ldg(a.tr.tidop + ev);
  }
}
template <class K, int I, bool LAZY>
__device__ __forceinline__ uint32_t acc_time(const AccArgs<K>& a, const AccSmem<K, I, LAZY>& S, uint32_t base,
                                             uint32_t q, uint32_t ev, uint32_t to) {
  if (LAZY) return make_aux(a.stamps, ev, to).y;
  if (q >= base) return S.st[q - base].x;
  return a.aux ? __ldg(&a.aux[ev].y) : acc_aux(a, ev).y;
}
// pred_t^{vo}[u] for the accessing thread tc
template <class K>
__device__ __forceinline__ uint32_t acc_clock(const AccArgs<K>& a, uint32_t vo, uint32_t tc, uint32_t u) {
  if (!a.blockobj) return obj_get(a.arena, vo, u);
  const uint32_t BS = a.tr.BS;
  if (vo == NIL || u / BS != tc / BS) return 0u;
  return __ldg(optr(a.arena, vo) + OBJ_HDR + (u - (tc / BS) * BS));
}

template <class K, int I, bool LAZY = false>
__global__ void __launch_bounds__(kThreads) k_access(AccArgs<K> a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  AccSmem<K, I, LAZY>& S = *reinterpret_cast<AccSmem<K, I, LAZY>*>(smem_raw);
  const uint32_t BS = a.tr.BS;
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
  const uint32_t ntiles = (uint32_t)((a.n + (kThreads * I) - 1) / (kThreads * I));  // positions < 2^31
  // LAZY: the next tile's keys / events (issued before this tile's scan) and
  // tidops (gathered before its checks) travel in registers while this tile
  // is processed -- register double buffering hides the gather latency
  constexpr int PI = LAZY ? I : 1;
  K pk[PI];
  uint32_t pv[PI], pt[PI];
#define GW_ACC_LOAD_KV(t)                                          \
  {                                                                \
    const uint32_t b_ = (t) * (kThreads * I);                      \
    _Pragma("unroll") for (int k = 0; k < PI; k++) {               \
      const uint32_t j = k * kThreads + threadIdx.x;               \
      const bool ok = (uint64_t)b_ + j < a.n;                      \
      pk[k] = ok ? a.keys[b_ + j] : (K)0;                          \
      pv[k] = ok ? a.vals[b_ + j] : 0u;                            \
    }                                                              \
  }
#define GW_ACC_LOAD_TO(t)                                                        \
  {                                                                              \
    const uint32_t b_ = (t) * (kThreads * I);                                    \
    _Pragma("unroll") for (int k = 0; k < PI; k++) {                             \
      const uint32_t j = k * kThreads + threadIdx.x;                             \
      pt[k] = (uint64_t)b_ + j < a.n ? __ldg(a.tr.tidop + (pv[k] & VAL_E)) : 0u; \
    }                                                                            \
  }
  // tiles in increasing order across the grid (atomic counter): the
  // look-back below waits only for lower tiles, all held by running CTAs
  if (threadIdx.x == 0) S.next_tile = atomicAdd(a.tile_ctr, 1u);
  __syncthreads();
  uint32_t tile = S.next_tile;
  if (LAZY && tile < ntiles) {
    GW_ACC_LOAD_KV(tile)
    GW_ACC_LOAD_TO(tile)
  }
  while (tile < ntiles) {
    const uint32_t base = tile * (kThreads * I);
    const uint32_t cnt = (uint32_t)min((uint64_t)(kThreads * I), a.n - base);
    __syncthreads();  // everyone read S.next_tile
    if (threadIdx.x == 0) S.next_tile = atomicAdd(a.tile_ctr, 1u);
    const K prevkey = base > 0 ? a.keys[base - 1] : (K)0;
    if (LAZY) {
#pragma unroll
      for (int k = 0; k < PI; k++) {
        const uint32_t j = k * kThreads + threadIdx.x;
        if (j < cnt) { S.key[apx(j)] = pk[k]; S.val[apx(j)] = pv[k]; S.to[apx(j)] = pt[k]; }
      }
    } else {
#pragma unroll
      for (int k = 0; k < I; k++) {
        const uint32_t j = k * kThreads + threadIdx.x;
        if (j < cnt) { S.key[apx(j)] = a.keys[base + j]; S.val[apx(j)] = a.vals[base + j]; }
      }
      uint4 ax[I];
#pragma unroll
      for (int k = 0; k < I; k++) {
        const uint32_t j = k * kThreads + threadIdx.x;
        ax[k] = j < cnt ? acc_aux(a, a.vals[base + j] & VAL_E) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int k = 0; k < I; k++) {
        const uint32_t j = k * kThreads + threadIdx.x;
        if (j < cnt) { S.to[apx(j)] = ax[k].x; S.st[(LAZY ? 0 : j)] = make_uint2(ax[k].y, ax[k].z); }
      }
    }
    __syncthreads();
    const uint32_t nxt = S.next_tile;
    const bool pre = LAZY && nxt < ntiles;
    if (pre) GW_ACC_LOAD_KV(nxt)
    // segment head / last write: a max-scan over the tile, seeded with the
    // carry.  Blocked: thread t owns positions [t*I, t*I + I) -- a serial pass
    // over its items, one warp scan and one block combine of the per-thread
    // maxima, then a second serial pass writes the inclusive values (the
    // padded smem index keeps the strided accesses conflict-free).  Third
    // component: the last position (+1) that starts a segment or changes the
    // thread; equal to the head's, the segment so far is one thread's
    // (SS_SINGLE).  Position `base` counts as a change (the part of its
    // segment in earlier tiles is not looked at), which only sends positions
    // to the full check.
    uint32_t need = 0;  // bit k: position threadIdx.x * I + k goes to the full check
    {
      const uint32_t j0 = threadIdx.x * I;
      uint3 agg = make_uint3(0, 0, 0);
      K kp = j0 > 0 ? S.key[apx(j0 - 1)] : prevkey;
      uint32_t tp = j0 > 0 ? ev_tid(S.to[apx(j0 - 1)]) : 0u;
#pragma unroll
      for (int k = 0; k < I; k++) {
        const uint32_t j = j0 + k;
        if (j < cnt) {
          const K kj = S.key[apx(j)];
          const uint32_t tj = ev_tid(S.to[apx(j)]);
          const bool head = base + j == 0 || kj != kp;
          if (head) agg.x = base + j + 1;
          if (S.val[apx(j)] & VAL_W) agg.y = base + j + 1;
          if (head || j == 0 || tj != tp) agg.z = base + j + 1;
          kp = kj;
          tp = tj;
        }
      }
      uint3 inc = agg;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_up_sync(0xffffffffu, inc.x, o), y = __shfl_up_sync(0xffffffffu, inc.y, o),
                       z = __shfl_up_sync(0xffffffffu, inc.z, o);
        if (lane >= o) { inc.x = max(inc.x, x); inc.y = max(inc.y, y); inc.z = max(inc.z, z); }
      }
      if (lane == 31) S.wtot[wq] = inc;
      __syncthreads();
      if (a.lb) {
        // decoupled look-back: publish this tile's maxima (flag A), take the
        // predecessors' until an inclusive prefix (flag P) or a tile whose
        // maxima are both set (positions grow with the tile index, so nothing
        // earlier can exceed them), publish the inclusive prefix
        if (threadIdx.x == 0) {
          uint32_t th = 0, tw = 0;
#pragma unroll
          for (int x = 0; x < kThreads / 32; x++) { th = max(th, S.wtot[x].x); tw = max(tw, S.wtot[x].y); }
          constexpr unsigned long long FA = 1ull << 62, FP = 2ull << 62, M31 = (1ull << 31) - 1;
          auto pack = [&](uint32_t hh, uint32_t ww, unsigned long long f) {
            return f | ((unsigned long long)hh << 31) | (unsigned long long)ww;
          };
          volatile unsigned long long* st = a.lb;
          st[tile] = pack(th, tw, FA);  // one 64-bit store: flag and values together
          uint32_t eh = 0, ew = 0;
          for (int64_t q = (int64_t)tile - 1; q >= 0; q--) {
            unsigned long long v;
            do { v = st[q]; } while ((v >> 62) == 0);
            const uint32_t vh = (uint32_t)((v >> 31) & M31), vw = (uint32_t)(v & M31);
            eh = max(eh, vh);
            ew = max(ew, vw);
            if ((v >> 62) == 2 || (eh && ew)) break;
          }
          st[tile] = pack(max(eh, th), max(ew, tw), FP);
          S.cin = make_uint2(eh, ew);
        }
        __syncthreads();
      }
      const uint2 cin = a.lb ? S.cin : a.carry[tile];
      uint3 run = make_uint3(cin.x, cin.y, 0);
#pragma unroll
      for (int x = 0; x < kThreads / 32; x++) {
        const uint3 t = S.wtot[x];
        if (x < wq) { run.x = max(run.x, t.x); run.y = max(run.y, t.y); run.z = max(run.z, t.z); }
      }
      {  // exclusive within the warp
        const uint32_t x = __shfl_up_sync(0xffffffffu, inc.x, 1), y = __shfl_up_sync(0xffffffffu, inc.y, 1),
                       z = __shfl_up_sync(0xffffffffu, inc.z, 1);
        if (lane >= 1) { run.x = max(run.x, x); run.y = max(run.y, y); run.z = max(run.z, z); }
      }
      kp = j0 > 0 ? S.key[apx(j0 - 1)] : prevkey;
      tp = j0 > 0 ? ev_tid(S.to[apx(j0 - 1)]) : 0u;
      // the event of the previous position (same-record check below)
      uint32_t pe = j0 > 0 ? (S.val[apx(j0 - 1)] & VAL_E) : (base > 0 ? (a.vals[base - 1] & VAL_E) : 0u);
#pragma unroll
      for (int k = 0; k < I; k++) {
        const uint32_t j = j0 + k;
        if (j < cnt) {
          const K kj = S.key[apx(j)];
          const uint32_t toj = S.to[apx(j)], vj = S.val[apx(j)];
          const uint32_t tj = ev_tid(toj);
          const bool head = base + j == 0 || kj != kp;
          if (head) run.x = base + j + 1;
          if (vj & VAL_W) run.y = base + j + 1;
          if (head || j == 0 || tj != tp) run.z = base + j + 1;
          kp = kj;
          tp = tj;
          const bool single = run.z == run.x;
          S.ss[apx(j)] = (run.x - 1) | (single ? SS_SINGLE : 0u);
          S.lw[apx(j)] = run.y;
          // positions the full check must see: not one thread's segment so
          // far, or the previous access to the location is in the same record
          const uint32_t c = vj & VAL_E;
          if (ev_kind(toj) <= GW_K_WRITE &&
              (!single || (a.dup.ev && !head && (toj & GW_F_CONT) && pe < c && c - pe < 32)))
            need |= 1u << k;
          pe = c;
        }
      }
    }
    // the flagged positions as a list (in the key staging, no longer read)
    uint32_t nlist;
    {
      const uint32_t cntn = __popc(need);
      uint32_t inc = cntn;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += x;
      }
      if (lane == 31) S.ltot[wq] = inc;
      __syncthreads();  // also: every thread is done reading the keys
      uint32_t off = inc - cntn;
      nlist = 0;
#pragma unroll
      for (int x = 0; x < kThreads / 32; x++) {
        const uint32_t t = S.ltot[x];
        if (x < wq) off += t;
        nlist += t;
      }
      uint16_t* L = reinterpret_cast<uint16_t*>(S.key);
      for (uint32_t m = need; m; m &= m - 1) L[off++] = (uint16_t)(threadIdx.x * I + __ffs(m) - 1);
      __syncthreads();
    }
    if (pre) GW_ACC_LOAD_TO(nxt)
    const uint32_t lw_in = a.lb ? S.cin.y : a.carry[tile].y;  // last write before the tile
    // the checks, over the flagged positions
    for (uint32_t x = threadIdx.x; x < nlist; x += kThreads) {
      const uint32_t j = reinterpret_cast<const uint16_t*>(S.key)[x];
      const uint32_t i = base + j;
      const uint32_t toc = S.to[apx(j)];
      if (ev_kind(toc) > GW_K_WRITE) continue;  // non-access events sort last (sentinel key)
      const uint32_t c = S.val[apx(j)] & VAL_E;
      const uint32_t tc = ev_tid(toc);
      const bool isw = ev_kind(toc) == GW_K_WRITE;
      const uint32_t ssr = S.ss[apx(j)];
      const uint32_t ss = ssr & ~SS_SINGLE;
      const uint32_t lw = j > 0 ? S.lw[apx(j - 1)] : lw_in;
      const bool hasw = lw > 0 && lw - 1 >= ss && lw - 1 < i;
      const uint32_t W = hasw ? lw - 1 : NIL;
      uint32_t vo_ = NIL;
      bool vo_ok = a.defer != 0;
      auto vo = [&]() {  // the accessing thread's pred object (LAZY: looked up on first use)
        if (!vo_ok) { vo_ = LAZY ? make_aux(a.stamps, c, toc).z : S.st[(LAZY ? 0 : j)].y; vo_ok = true; }
        return vo_;
      };
      unsigned long long loc = 0;
      if (i > ss && (toc & GW_F_CONT) && a.dup.ev) {
        // the previous access to this location may be in the same record
        uint32_t pe, pto;
        acc_pos(a, S, base, i - 1, pe, pto);
        if (pe < c && c - pe < 32) {
          bool same = true;
          for (uint32_t x = pe + 1; x < c && same; x++) same = (__ldg(a.tr.tidop + x) & GW_F_CONT) != 0;
          if (same) {
            const uint32_t kk = atomicAdd(a.dup.n, 1u);
            if (kk < a.dup.cap) a.dup.ev[kk] = c;
          }
        }
      }
      if (ssr & SS_SINGLE) continue;  // one thread so far: no prior-write / reader candidate
      if (hasw) {
        uint32_t p, top;
        acc_pos(a, S, base, W, p, top);
        const uint32_t u = ev_tid(top);
        bool race = u != tc && !cover(top, toc, BS);
        if (race && !a.defer) {  // both stamp lookups issued before either is used
          const uint32_t v = vo();
          const uint32_t tw = acc_time(a, S, base, W, p, top);
          race = tw > acc_clock(a, v, tc, u);
        }
        if (race) {
          loc = a.tr.key[c];
          emit_cand(a.c, ((unsigned long long)c << 32) | SUB_WCHECK, loc, p, c, isw ? GW_WW : GW_WR);
        }
      }
      if (!isw) continue;
      const uint32_t ws = hasw ? W + 1 : ss;
      const uint32_t m = i - ws;
      if (m == 0) continue;
      if (m > kSmallWin) {
        uint32_t kk = atomicAdd(a.n_large, 1u);
        if (kk < a.large_cap) { a.large_i[kk] = i; a.large_ws[kk] = ws; }
        else atomicOr(a.c.err, ERR_CAND);
        continue;
      }
      // readers since W: one candidate per thread (its latest read), ranked by its first read
      for (uint32_t q = ws; q < i; q++) {
        uint32_t r, toq;
        acc_pos(a, S, base, q, r, toq);
        if (ev_kind(toq) > GW_K_WRITE) continue;
        const uint32_t uq = ev_tid(toq);
        if (uq == tc) continue;
        bool later = false;
        for (uint32_t q2 = q + 1; q2 < i && !later; q2++) {
          uint32_t e2, t2;
          acc_pos(a, S, base, q2, e2, t2);
          later = ev_kind(t2) <= GW_K_WRITE && ev_tid(t2) == uq;
        }
        if (later) continue;
        uint32_t first = q;
        for (uint32_t q3 = ws; q3 < q; q3++) {
          uint32_t e3, t3;
          acc_pos(a, S, base, q3, e3, t3);
          if (ev_kind(t3) <= GW_K_WRITE && ev_tid(t3) == uq) { first = q3; break; }
        }
        if (!cover(toq, toc, BS) && (a.defer || acc_time(a, S, base, q, r, toq) > acc_clock(a, vo(), tc, uq))) {
          if (!loc) loc = a.tr.key[c];
          emit_cand(a.c, ((unsigned long long)c << 32) | SUB_READER | (first - ws), loc, r, c, GW_RW);
        }
      }
    }
    tile = nxt;
  }
}

#undef GW_ACC_LOAD_KV
#undef GW_ACC_LOAD_TO

// ---- lock mode: deferred clock checks -------------------------------------
// Q = threads whose clock entry is ever read: prior-access threads of the
// structural candidates and record owners (successful acquires).  Also flags
// the current events that carry queries and lays out the (cur, candidate)
// pairs for the sort that orders the queries by event.
__global__ void k_q_mark_cands(Cands c, const uint32_t* tidop, uint32_t* qflag, uint8_t* lflags, uint32_t* qk,
                               uint32_t* qvals) {
  const uint32_t n = min(*c.n, c.cap);
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const uint32_t cur = c.cur[k];
    qflag[ev_tid(tidop[c.prior[k]])] = 1u;
    lflags[cur] = lflags[cur] | LF_QUERY;  // every writer stores the same value
    qk[k] = cur;
    qvals[k] = k;
  }
}
__global__ void k_q_mark_acq(DevTrace tr, const uint8_t* lflags, uint32_t* qflag) {
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tr.n; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t to = tr.tidop[e];
    if (ev_kind(to) == GW_K_ACQUIRE && (lflags[e] & LF_OK)) qflag[ev_tid(to)] = 1u;
  }
}
// the clock half of the checks (gwcp.py:256, :265): race iff prior.time > pred_t[u]
__global__ void k_resolve(Cands in, const uint32_t* qv, const uint32_t* time, Cands out) {
  const uint32_t n = min(*in.n, in.cap);
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const uint32_t p = in.prior[k];
    if (time[p] > qv[k]) emit_cand(out, in.okey[k], in.loc[k], p, in.cur[k], in.kind[k]);
  }
}

template <class K, int I, bool LAZY = false>
inline void acc_setup() {
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(k_access<K, I, LAZY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(AccSmem<K, I, LAZY>));
    done = true;
  }
}

// large reader windows: (window, tid) groups via a secondary stable sort
__global__ void k_large_fill(const uint32_t* large_i, const uint32_t* large_ws, const uint32_t* off, uint32_t n_large,
                             const uint32_t* svals, const uint32_t* tidop, unsigned long long* keys, uint32_t* vals) {
  for (uint32_t k = blockIdx.x; k < n_large; k += gridDim.x) {
    const uint32_t ws = large_ws[k], m = large_i[k] - ws, o = off[k];
    for (uint32_t j = threadIdx.x; j < m; j += blockDim.x) {
      const uint32_t t = tidop[svals[ws + j] & VAL_E];
      // non-access events (key-0 location) go to a virtual window past the last one
      const unsigned long long kk = ev_kind(t) <= GW_K_WRITE ? k : n_large;
      keys[o + j] = (kk << 24) | ev_tid(t);
      vals[o + j] = ws + j;
    }
  }
}
template <class K>
__global__ void k_large_check(AccArgs<K> a, const unsigned long long* keys, const uint32_t* vals, uint64_t M,
                              uint32_t nlarge) {
  const uint32_t BS = a.tr.BS;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < M; j += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long key = keys[j];
    if (j + 1 < M && keys[j + 1] == key) continue;  // not the latest read of this (window, tid)
    uint64_t f = j;
    while (f > 0 && keys[f - 1] == key) f--;
    const uint32_t k = (uint32_t)(key >> 24);
    if (k >= nlarge) continue;  // non-access events
    const uint32_t i = a.large_i[k], ws = a.large_ws[k];
    const uint32_t c = a.vals[i] & VAL_E, toc = a.tr.tidop[c];
    const uint32_t q = vals[j], first = vals[f];
    const uint32_t r = a.vals[q] & VAL_E;
    const uint32_t toq = a.tr.tidop[r], uq = ev_tid(toq);
    if (uq == ev_tid(toc)) continue;
    if (!cover(toq, toc, BS) &&
        (a.defer || acc_aux(a, r).y > acc_clock(a, acc_aux(a, c).z, ev_tid(toc), uq)))
      emit_cand(a.c, ((unsigned long long)c << 32) | SUB_READER | (first - ws), a.tr.key[c], r, c, GW_RW);
  }
}

// _same_instruction_check, engine.py:81-95: ww(i, j) for events i < j of a
// multi-event WRITE record on one location (distinct threads, !cover), before
// the record's own events.  One warp per record: the warp owning the record
// head's 32-event window loads the record (one event per lane, coalesced)
// and matches locations with __match_any_sync.  Uniform records (every
// parser wacc: same instr / atomic+scope / block, strictly increasing tids)
// share one dedup key and one cover verdict per location, so only the pair
// (first, second occurrence) can survive keep-first; others emit every pair.
__device__ __forceinline__ bool rec_uniform_step(uint32_t prev, uint32_t cur, uint32_t iprev, uint32_t icur,
                                                 uint32_t BS) {
  return icur == iprev && ((cur ^ prev) & (GW_F_ATOMIC | GW_F_DEVICE | (7u << GW_OP_SHIFT))) == 0 &&
         ev_tid(cur) / BS == ev_tid(prev) / BS && ev_tid(cur) > ev_tid(prev);
}
__device__ __forceinline__ unsigned long long sub_pair(uint64_t i, uint64_t j) {
  return ((unsigned long long)i << 15) | (unsigned long long)j;
}
// slow path for records longer than 32 events: event j scans its record
__device__ void same_instr_long(const DevTrace& tr, const Cands& cd, uint64_t head, uint64_t end, uint64_t j,
                                bool uni, const ShardArgs& sa) {
  const uint32_t tj = tr.tidop[j];
  if (ev_kind(tj) > GW_K_WRITE) return;
  const unsigned long long lj = tr.key[j];
  if (!in_shard(lj, sa)) return;
  uint32_t cnt = 0;
  uint64_t first = 0;
  for (uint64_t i = head; i < j; i++) {
    const uint32_t ti = tr.tidop[i];
    if (ev_kind(ti) > GW_K_WRITE || tr.key[i] != lj) continue;
    cnt++;
    if (cnt == 1) first = i;
    if (!uni && ev_tid(ti) != ev_tid(tj) && !cover(ti, tj, tr.BS))
      emit_cand(cd, ((unsigned long long)head << 32) | sub_pair(i - head, j - head), lj, (uint32_t)i, (uint32_t)j,
                GW_WW);
  }
  if (uni && cnt == 1) {
    const uint32_t ti = tr.tidop[first];
    if (ev_tid(ti) != ev_tid(tj) && !cover(ti, tj, tr.BS))
      emit_cand(cd, ((unsigned long long)head << 32) | sub_pair(first - head, j - head), lj, (uint32_t)first,
                (uint32_t)j, GW_WW);
  }
}

// one record (head = its first event, a WRITE followed by CONT events); the
// whole warp calls it.  long_only: skip records of <= 32 events.
__device__ void same_instr_record(const DevTrace& tr, const Cands& cd, const ShardArgs& sa, uint64_t head,
                                  bool long_only) {
  const int lane = threadIdx.x & 31;
  // load the record, 32 events at a time
  const uint64_t x = head + lane;
  const bool inr = x < tr.n;
  const uint32_t tx = inr ? tr.tidop[x] : 0u;
  const uint32_t ix = inr ? tr.instr[x] : 0u;
  const unsigned long long kx0 = inr ? tr.key[x] : 0ull;
  const uint32_t cm = __ballot_sync(0xffffffffu, inr && (tx & GW_F_CONT)) | 1u;  // lane 0 is the head
  const uint32_t stop = ~cm;                                                    // first non-CONT lane
  const int len = stop ? __ffs(stop) - 1 : 32;
  const uint32_t tprev = __shfl_up_sync(0xffffffffu, tx, 1);
  const uint32_t iprev = __shfl_up_sync(0xffffffffu, ix, 1);
  const bool stepok = lane == 0 || lane >= len || rec_uniform_step(tprev, tx, iprev, ix, tr.BS);
  bool uni = __all_sync(0xffffffffu, stepok);
  if (len == 32 && head + 32 < tr.n && (tr.tidop[head + 32] & GW_F_CONT)) {
    // long record (> 32 events): per-event scan, record by record
    uint64_t end = head + 32;
    while (end < tr.n && (tr.tidop[end] & GW_F_CONT)) end++;
    if (end - head >= 32768) {
      if (lane == 0) atomicOr(cd.err, ERR_RECORD);
      return;
    }
    bool u2 = uni;
    for (uint64_t c = head + 32 + lane; c < end; c += 32)
      u2 = u2 && rec_uniform_step(tr.tidop[c - 1], tr.tidop[c], tr.instr[c - 1], tr.instr[c], tr.BS);
    uni = __all_sync(0xffffffffu, u2);
    for (uint64_t j = head + 1 + lane; j < end; j += 32) same_instr_long(tr, cd, head, end, j, uni, sa);
    return;
  }
  if (long_only) return;
  const bool acc = lane < len && ev_kind(tx) <= GW_K_WRITE;
  const unsigned long long kx = acc ? kx0 : 0ull;
  const bool mine = in_shard(kx, sa);
  const uint32_t accm = __ballot_sync(0xffffffffu, acc);
  const uint32_t peers = __match_any_sync(0xffffffffu, kx) & accm;
  const uint32_t earlier = peers & lanemask_lt();
  if (!acc || !earlier || !mine) return;
  if (uni) {
    if (__popc(earlier) != 1) return;  // not the second occurrence of this location
    const int fl = __ffs(earlier) - 1;
    const uint32_t tf = tr.tidop[head + fl];
    if (ev_tid(tf) != ev_tid(tx) && !cover(tf, tx, tr.BS))
      emit_cand(cd, ((unsigned long long)head << 32) | sub_pair(fl, lane), kx, (uint32_t)(head + fl), (uint32_t)x,
                GW_WW);
  } else {
    for (uint32_t m = earlier; m; m &= m - 1) {
      const int il = __ffs(m) - 1;
      const uint32_t ti = tr.tidop[head + il];
      if (ev_tid(ti) != ev_tid(tx) && !cover(ti, tx, tr.BS))
        emit_cand(cd, ((unsigned long long)head << 32) | sub_pair(il, lane), kx, (uint32_t)(head + il),
                  (uint32_t)x, GW_WW);
    }
  }
}

// every record of the trace (traces with records longer than 32 events, and
// lock mode); long_only: only those (the others come from the head list)
__global__ void __launch_bounds__(kThreads) k_same_instr(DevTrace tr, Cands cd, ShardArgs sa, int long_only) {
  const int lane = threadIdx.x & 31;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t wb = (((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; wb < tr.n; wb += nwarps * 32) {
    // heads of multi-event WRITE records in this window
    const uint64_t e = wb + lane;
    bool is_head = false;
    if (e + 1 < tr.n) {
      const uint32_t t0 = tr.tidop[e];
      is_head = !(t0 & GW_F_CONT) && ev_kind(t0) == GW_K_WRITE && (tr.tidop[e + 1] & GW_F_CONT);
    }
    uint32_t heads = __ballot_sync(0xffffffffu, is_head);
    while (heads) {
      const int hl = __ffs(heads) - 1;
      heads &= heads - 1;
      same_instr_record(tr, cd, sa, wb + hl, long_only != 0);
    }
  }
}

// Same-record pairs on one location are adjacent in location order (a
// record's events are contiguous in the trace), so k_access flags them:
// DupList collects the current events; k_dup_heads maps them to their
// records' heads (deduplicated through a small hash set) and
// k_same_instr_heads runs the record check on those records only.  Valid
// when no record is longer than 32 events (Stats::n_long == 0).
__global__ void k_dup_heads(DevTrace tr, DupList d, uint32_t* hset, uint32_t hmask, uint32_t* heads,
                            uint32_t* nheads) {
  const uint32_t n = min(*d.n, d.cap);
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    uint64_t h = d.ev[k];
    while (h > 0 && (tr.tidop[h] & GW_F_CONT)) h--;
    if (ev_kind(tr.tidop[h]) != GW_K_WRITE) continue;  // _same_instruction_check: WRITE records only
    uint32_t slot = (uint32_t)mix64(h) & hmask;
    while (true) {
      const uint32_t old = atomicCAS(&hset[slot], 0u, (uint32_t)h + 1);
      if (old == 0) { heads[atomicAdd(nheads, 1u)] = (uint32_t)h; break; }
      if (old == (uint32_t)h + 1) break;
      slot = (slot + 1) & hmask;
    }
  }
}
__global__ void __launch_bounds__(kThreads) k_same_instr_heads(DevTrace tr, Cands cd, ShardArgs sa,
                                                              const uint32_t* heads, const uint32_t* nheads) {
  const uint32_t n = *nheads;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < n; k += nwarps)
    same_instr_record(tr, cd, sa, heads[k], false);
}

// ------------------------------------------------------------- dedup -----
struct DedupArgs {
  Cands c;
  const uint32_t* instr;
  uint32_t* owner;            // slot -> candidate + 1
  unsigned long long* smin;   // slot -> min order key
  uint32_t* cslot;            // candidate -> slot
  uint32_t mask;
  uint32_t ncand;     // capacity the grids are sized for
  const uint32_t* dn; // device candidate count
};
__device__ __forceinline__ uint32_t dd_count(const DedupArgs& d) { return min(*d.dn, d.ncand); }
__global__ void k_dedup_insert(DedupArgs d) {
  const uint32_t nc = dd_count(d);
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < nc; k += gridDim.x * blockDim.x) {
    const unsigned long long loc = d.c.loc[k];
    const uint32_t ip = d.instr[d.c.prior[k]], ic = d.instr[d.c.cur[k]];
    uint32_t h = (uint32_t)mix64(loc ^ mix64(((unsigned long long)ip << 32) | ic)) & d.mask;
    while (true) {
      uint32_t old = atomicCAS(&d.owner[h], 0u, k + 1);
      if (old == 0) break;
      const uint32_t o = old - 1;
      if (d.c.loc[o] == loc && d.instr[d.c.prior[o]] == ip && d.instr[d.c.cur[o]] == ic) break;
      h = (h + 1) & d.mask;
    }
    d.cslot[k] = h;
    atomicMin(&d.smin[h], d.c.okey[k]);
  }
}
// Report order: every candidate gets its order key if it is the keep-first
// survivor of its dedup slot, else a key past every event (sorted last); one
// radix sort of the candidates then yields the survivors in report order.
__global__ void k_dedup_keys(DedupArgs d, unsigned long long n_events, unsigned long long* sk, uint32_t* sv,
                             uint32_t* nsurv) {
  const uint32_t nc = dd_count(d);
  for (uint32_t k0 = blockIdx.x * blockDim.x; k0 < d.ncand; k0 += gridDim.x * blockDim.x) {
    const uint32_t k = k0 + threadIdx.x;
    bool surv = false;
    unsigned long long key = n_events << 32;
    if (k < nc) {
      const unsigned long long ok = d.c.okey[k];
      surv = ok == d.smin[d.cslot[k]];
      if (surv) key = ok;
    }
    if (k < d.ncand) { sk[k] = key; sv[k] = k; }
    const uint32_t m = __ballot_sync(0xffffffffu, surv);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(nsurv, (uint32_t)__popc(m));
  }
}
// large candidate sets: survivors keyed by their current event only (fewer
// radix bits), then every run of equal events ordered by the full order key
__global__ void k_dedup_keys32(DedupArgs d, uint32_t n_events, uint32_t* sk, uint32_t* sv, uint32_t* nsurv) {
  const uint32_t nc = dd_count(d);
  for (uint32_t k0 = blockIdx.x * blockDim.x; k0 < d.ncand; k0 += gridDim.x * blockDim.x) {
    const uint32_t k = k0 + threadIdx.x;
    bool surv = false;
    uint32_t key = n_events;
    if (k < nc) {
      const unsigned long long ok = d.c.okey[k];
      surv = ok == d.smin[d.cslot[k]];
      if (surv) key = (uint32_t)(ok >> 32);
    }
    if (k < d.ncand) { sk[k] = key; sv[k] = k; }
    const uint32_t m = __ballot_sync(0xffffffffu, surv);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(nsurv, (uint32_t)__popc(m));
  }
}
// small traces: counting sort of the survivors by event bucket (event >> cs:
// count, scan over the buckets, placement with self-cleaning counters); each
// bucket's run is then ordered by the full order key (k_group_fix)
__global__ void k_surv_count(DedupArgs d, uint32_t* ccnt, uint32_t* nsurv, uint32_t cs) {
  const uint32_t nc = dd_count(d);
  for (uint32_t k0 = blockIdx.x * blockDim.x; k0 < d.ncand; k0 += gridDim.x * blockDim.x) {
    const uint32_t k = k0 + threadIdx.x;
    bool surv = false;
    if (k < nc) {
      const unsigned long long ok = d.c.okey[k];
      surv = ok == d.smin[d.cslot[k]];
      if (surv) atomicAdd(ccnt + ((ok >> 32) >> cs), 1u);
    }
    const uint32_t m = __ballot_sync(0xffffffffu, surv);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(nsurv, (uint32_t)__popc(m));
  }
}
__global__ void k_surv_place(DedupArgs d, uint32_t* ccnt, const uint32_t* coff, uint32_t* sk, uint32_t* sv,
                             uint32_t cs) {
  const uint32_t nc = dd_count(d);
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < nc; k += gridDim.x * blockDim.x) {
    const unsigned long long ok = d.c.okey[k];
    if (ok == d.smin[d.cslot[k]]) {
      const uint32_t c = (uint32_t)(ok >> 32) >> cs;
      const uint32_t pos = coff[c] + atomicSub(ccnt + c, 1u) - 1u;  // leaves ccnt zeroed
      sk[pos] = c;
      sv[pos] = k;
    }
  }
}
__global__ void k_group_fix(const uint32_t* sk, uint32_t* sv, uint32_t n, uint32_t n_events,
                            const unsigned long long* okey, const uint32_t* nlim = nullptr) {
  if (nlim) n = min(n, *nlim);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t key = sk[i];
    if (key >= n_events || (i > 0 && sk[i - 1] == key)) continue;
    uint32_t end = i + 1;
    while (end < n && sk[end] == key) end++;
    for (uint32_t x = i + 1; x < end; x++) {  // insertion sort of the run by order key
      const uint32_t v = sv[x];
      const unsigned long long ok = okey[v];
      uint32_t y = x;
      while (y > i && okey[sv[y - 1]] > ok) { sv[y] = sv[y - 1]; y--; }
      sv[y] = v;
    }
  }
}

__global__ void k_final(Cands c, const uint32_t* svals, const uint32_t* nsurv, uint8_t* okind, uint32_t* oprior,
                        uint32_t* ocur, unsigned long long* okey) {
  const uint32_t n = *nsurv;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const uint32_t k = svals[j];
    okind[j] = (uint8_t)c.kind[k];
    oprior[j] = c.prior[k];
    ocur[j] = c.cur[k];
    okey[j] = c.okey[k];
  }
}

}  // namespace gw
