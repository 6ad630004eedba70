// libgwcp_b200: orchestration of the G-WCP pipeline and the C-ABI of
// include/gwcp_b200.h.
//
//   k_prep        one pass: counts by kind, OR/AND of location keys
//   partition     stable radix sort of event ids by walker CTA (block mod G)
//   lock pre-pass per-thread lock-stack automaton, in-CS flags, ticket ranks
//   k_walker      sync pass: clocks, barriers, lock rules (walker.cuh)
//   access pass   radix sort by location, max-scan, race check (access.cuh)
//   same-instr    multi-lane write records (engine.py:81-95)
//   dedup/final   keep-first per (loc, instr, instr), sort by order key
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "bucket.cuh"
#include "validate.cuh"
#include "workloads.cuh"
#include "common.h"

namespace gw {
thread_local uint32_t g_launches = 0;
thread_local LaunchProf* g_prof = nullptr;
}
using namespace gw;

static thread_local std::string g_err;
void gw_set_error(const std::string& m) { g_err = m; }
extern "C" const char* gw_last_error(void) { return g_err.c_str(); }

namespace {

struct CudaErr {
  int code;
  std::string msg;
};

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t _e = (x);                                                                  \
    if (_e != cudaSuccess)                                                                 \
      throw CudaErr{_e == cudaErrorMemoryAllocation ? GW_E_NOMEM : GW_E_CUDA,              \
                    std::string(#x) + ": " + cudaGetErrorString(_e)};                      \
  } while (0)

inline int ceil_log2(uint64_t x) {
  int b = 0;
  while ((1ull << b) < x) b++;
  return b;
}
inline uint64_t pow2_at_least(uint64_t x) {
  uint64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}
inline unsigned grid_for(uint64_t n, unsigned cap = 148u * 16u) {
  uint64_t g = (n + kThreads - 1) / kThreads;
  if (g < 1) g = 1;
  return (unsigned)std::min<uint64_t>(g, cap);
}

}  // namespace

// Plan of a lock-free analysis, cached so that repeated analyses of traces
// with the same shape replay one CUDA graph (no host syncs, no per-kernel
// launch cost).  Every value the eager pipeline reads back from the device
// is fixed here and re-verified ON the device by k_plan_check / k_guard; a
// mismatch raises the abort flag and gw_ctx_fetch re-runs eagerly.
struct Plan {
  bool valid = false;
  uint64_t N = 0;
  uint32_t B = 0, W = 0, L = 0, inactive_opt = 1;
  const void *key = nullptr, *tidop = nullptr, *instr = nullptr;
  cudaStream_t stream = 0;
  unsigned long long n_bar = 0, n_end = 0, n_wbar = 0, D = 0;
  unsigned long long n_acc = 0;  // the bucketed access pass sizes its passes by it
  uint64_t cand_cap = 0;
  uint64_t pend_cap = 0;  // bucketed pass: structural candidates
  uint32_t launches = 0;
  bool hard_small = false;  // snapshot mode with a one-launch hard-event list: a branch from the graph start
  cudaGraphExec_t exec = nullptr;
};

struct gw_ctx {
  int device = 0;
  int num_sms = 148;
  struct Buf {
    void* p = nullptr;
    size_t cap = 0;
  };
  std::map<std::string, Buf> bufs;
  // ev[0] / ev[1]: whole analysis; ev[2 + 2*(2*phase + k) + {0,1}]: interval k of a phase
  static constexpr int kEv = 22;
  cudaEvent_t ev[kEv] = {};
  int nint[5] = {0, 0, 0, 0, 0};
  // last results (device)
  uint64_t n_reports = 0, n_diags = 0, n_events = 0;
  uint8_t* d_kind = nullptr;
  uint32_t* d_prior = nullptr;
  uint32_t* d_cur = nullptr;
  unsigned long long* d_okey = nullptr;
  Diag* d_diags = nullptr;
  gw_stats stats{};
  bool stats_pending = false;
  bool phases = false;
  uint32_t launches = 0;
  uint32_t* d_scal = nullptr;   // device scalars (see Pipeline::run)
  uint32_t* d_nsurv = nullptr;  // device report count
  bool have_cands = false;
  uint64_t arena_words = 0;
  cudaStream_t last_stream = 0;
  // results staged in mapped pinned host memory: k_final writes the report
  // arrays straight into it and one 64-byte copy mirrors the scalars, so a
  // fetch is one stream sync + host memcpys (no per-array D2H round trips)
  uint8_t* hres = nullptr;
  size_t hres_cap = 0;
  uint32_t* h_scal = nullptr;
  uint8_t* host_res(size_t bytes) {
    if (hres_cap < bytes) {
      if (hres) cudaFreeHost(hres);
      hres = nullptr;
      hres_cap = 0;
      const size_t nb = bytes + bytes / 4;
      CK(cudaHostAlloc((void**)&hres, nb, cudaHostAllocMapped | cudaHostAllocPortable));
      hres_cap = nb;
    }
    return hres;
  }
  // side stream of the lock-free fork (access sort concurrent with the sync pass)
  cudaStream_t side = nullptr, side2 = nullptr;
  // packed host input (gw_ctx_analyze_host_packed): chunk uploads on their own stream
  cudaStream_t copy_st = nullptr;
  // exchange mode (gw_xs_*): this rank's slice and the candidate counts of the last xs_check
  DevTrace xs_slice{};
  uint32_t xs_base = 0;
  uint64_t xs_nc = 0, xs_nsi = 0;
  std::vector<cudaEvent_t> chunk_ev;
  cudaEvent_t ev_prev = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_fork2 = nullptr, ev_hard = nullptr;
  uint32_t epoch = 1;  // look-back flag epochs (never reused within 2^24 passes)
  // last analysis, for an eager re-run after a graph abort
  DevTrace last_tr{};
  uint32_t last_inactive = 1;
  uint32_t last_shard = 0, last_nshard = 1;
  bool last_hb = false;
  bool last_graph = false;
  Plan plan;
  LaunchProf prof;           // GW_OPT_PROFILE: per-launch events of the last analysis
  std::vector<cudaEvent_t> prof_ev;
  std::vector<LaunchProf::Rec> prof_recs;
  bool prof_done = false;

  void prof_arm(uint32_t cap) {
    while (prof_ev.size() < 2 * (size_t)cap) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      prof_ev.push_back(e);
    }
    prof_recs.assign(cap, LaunchProf::Rec{nullptr, nullptr, nullptr, nullptr});
    for (uint32_t i = 0; i < cap; i++) { prof_recs[i].a = prof_ev[2 * i]; prof_recs[i].b = prof_ev[2 * i + 1]; }
    prof.recs = prof_recs.data();
    prof.n = 0;
    prof.cap = cap;
    prof_done = true;
  }

  template <class T>
  T* get(const std::string& name, uint64_t count) {
    size_t bytes = std::max<size_t>(sizeof(T) * count, 16);
    Buf& b = bufs[name];
    if (b.cap < bytes) {
      if (b.p) cudaFree(b.p);
      b.p = nullptr;
      b.cap = 0;
      size_t nb = bytes + bytes / 8;
      if (cudaMalloc(&b.p, nb) != cudaSuccess) {
        cudaGetLastError();
        size_t held = 0, fr = 0, tot = 0;
        std::string big;
        for (auto& kv : bufs) {
          held += kv.second.cap;
          if (kv.second.cap >= (1ull << 30)) big += " " + kv.first + "=" + std::to_string(kv.second.cap >> 20) + "M";
        }
        cudaMemGetInfo(&fr, &tot);
        b.p = nullptr;
        throw CudaErr{GW_E_NOMEM, "out of device memory allocating '" + name + "' (" + std::to_string(nb >> 20) +
                                      " MiB; device free " + std::to_string(fr >> 20) + " MiB; context holds " +
                                      std::to_string(held >> 20) + " MiB:" + big + ")"};
      }
      // zeroed on the analysis stream (look-back flags must never alias a live
      // epoch): a legacy-stream memset would not be ordered before kernels on
      // a non-blocking stream
      CK(cudaMemsetAsync(b.p, 0, nb, last_stream));
      b.cap = nb;
    }
    return (T*)b.p;
  }
  void drop_plan() {
    if (plan.exec) cudaGraphExecDestroy(plan.exec);
    plan = Plan();
  }
  void finish_stats() {
    if (!stats_pending) return;
    stats_pending = false;
    CK(cudaEventSynchronize(ev[1]));
    float ms;
    CK(cudaEventElapsedTime(&ms, ev[0], ev[1])); stats.ms_total = ms;
    if (phases) {
      float* dst[5] = {&stats.ms_prep, &stats.ms_walker, &stats.ms_sort, &stats.ms_check, &stats.ms_final};
      for (int p = 0; p < 5; p++) {
        *dst[p] = 0.f;
        for (int k = 0; k < nint[p]; k++) {
          const int i = 2 + 2 * (2 * p + k);
          CK(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
          *dst[p] += ms;
        }
      }
    }
  }
};

namespace {

// scalar slots of the "scalars" buffer
constexpr size_t kResHdr = 256;  // scalar mirror at the head of gw_ctx::hres
enum : int { SC_MAXD = 0, SC_NINCS, SC_TICKET, SC_REC, SC_LOG, SC_DIAG, SC_ERR, SC_ABORT, SC_NCAND, SC_NLARGE,
             SC_NSURV, SC_NQ, SC_NQLARGE, SC_NDUP, SC_NHEADS, SC_NSPILL, SC_NLARGE2, SC_NPEND, SC_COUNT = 24 };

__global__ void k_init_stats(Stats* s) {
  memset(s, 0, sizeof(Stats));
  s->key_and = ~0ull;
}
// graph mode: the trace must have the shape the plan was built for
__global__ void k_plan_check(const Stats* s, unsigned long long n_bar, unsigned long long n_end,
                             unsigned long long n_wbar, unsigned long long D, unsigned long long n_acc,
                             uint32_t* abort_flag) {
  const bool ok = s->n_acq == 0 && s->n_rel == 0 && s->n_bar == n_bar && s->n_end == n_end && s->n_long == 0 &&
                  s->n_wbar == n_wbar && s->n_acc == n_acc &&
                  ((s->key_or ^ s->key_and) & ~D) == 0ull;
  if (!ok) atomicOr(abort_flag, 1u);
}
// exchange mode helpers
__global__ void k_xs_hard_flag(DevTrace tr, uint32_t* flag) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tr.n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t k = ev_kind(tr.tidop[i]);
    flag[i] = k == GW_K_BARRIER || k == GW_K_END;
  }
}
__global__ void k_xs_hard_emit(DevTrace tr, const uint32_t* flag, const uint32_t* off, uint32_t base, uint32_t* ev,
                               uint32_t* to, uint32_t* in, unsigned long long* key) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tr.n; i += (uint64_t)gridDim.x * blockDim.x)
    if (flag[i]) {
      const uint32_t p = off[i];
      ev[p] = base + (uint32_t)i;
      to[p] = tr.tidop[i];
      in[p] = tr.instr[i];
      key[p] = tr.key[i];
    }
}
__global__ void k_xs_remap(const uint32_t* mini, uint64_t n, const uint32_t* gidx, uint32_t* out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = gidx[mini[i]];
}
__global__ void k_xs_lookup(DevTrace tr, uint32_t base, const uint32_t* ev, uint64_t n, uint32_t* to, uint32_t* in) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t e = ev[i];
    if (e >= base && (uint64_t)(e - base) < tr.n) {
      to[i] = tr.tidop[e - base];
      in[i] = tr.instr[e - base];
    }
  }
}
__global__ void k_iota(uint32_t* v, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) v[i] = i;
}
__global__ void k_guard(const uint32_t* ncand, uint32_t cap, const uint32_t* nlarge, const uint32_t* ndup,
                        uint32_t dupcap, uint32_t* abort_flag, const uint32_t* nspill = nullptr) {
  if (*ncand > cap || *nlarge > 0 || *ndup > dupcap || (nspill && *nspill > 0)) atomicOr(abort_flag, 1u);
}

struct Pipeline {
  gw_ctx* C;
  cudaStream_t st;
  DevTrace tr;
  uint32_t inactive_opt;
  bool gmode = false;  // graph mode: plan values, no host syncs
  const Plan* P = nullptr;

  template <class T>
  void d2h(T* host, const T* dev, size_t n = 1) {
    CK(cudaMemcpyAsync(host, dev, sizeof(T) * n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  void check_launch() { CK(cudaGetLastError()); }
  enum { PH_PREP = 0, PH_WALKER, PH_SORT, PH_CHECK, PH_FINAL };
  void event(int i) {
    if (!gmode) CK(cudaEventRecord(C->ev[i], st));
  }
  void pbeg(int p) {
    if (!gmode && C->nint[p] < 2) CK(cudaEventRecord(C->ev[2 + 2 * (2 * p + C->nint[p])], st));
  }
  void pend(int p) {
    if (!gmode && C->nint[p] < 2) CK(cudaEventRecord(C->ev[2 + 2 * (2 * p + C->nint[p]) + 1], st));
    C->nint[p]++;
  }

  // per-analysis zeroed block: look-back tile counters + radix histograms
  static constexpr uint32_t kZeroWords = 1u << 17;
  uint32_t* zero_blk = nullptr;
  uint32_t zero_next = 0;
  uint32_t* zeroed(uint32_t words) {
    if (zero_next + words > kZeroWords) throw CudaErr{GW_E_ARG, "zeroed scratch block exhausted"};
    uint32_t* p = zero_blk + zero_next;
    zero_next += words;
    return p;
  }
  uint32_t take_epochs(uint32_t k) {
    if (gmode) {  // graph mode clears every flag / status word at graph start: fixed epochs
      static const uint32_t base = 1;
      uint32_t e = base + gepoch;
      gepoch += k;
      return e;
    }
    // the wrap is handled once per analysis in reserve_epochs(), on the main
    // stream before any branch forks (never under a running look-back)
    if (C->epoch + k > epoch_limit) throw CudaErr{GW_E_ARG, "look-back epoch budget of one analysis exceeded"};
    uint32_t e = C->epoch;
    C->epoch += k;
    return e;
  }
  // eager analyses: every status buffer (main and side branch) is either
  // cleared here or holds only epochs < C->epoch, so the kEpochBudget epochs
  // this analysis may take never alias a stale status word
  static constexpr uint32_t kEpochBudget = 1u << 16;
  uint32_t epoch_limit = 0;
  void reserve_epochs() {
    if (C->epoch + kEpochBudget >= (1u << 24)) {  // wrap: clear every flag / status word
      for (auto& kv : C->bufs)
        if (kv.first.rfind("rs_status", 0) == 0) CK(cudaMemsetAsync(kv.second.p, 0, kv.second.cap, st));
      C->epoch = 1;
    }
    epoch_limit = C->epoch + kEpochBudget;
  }
  uint32_t gepoch = 0;
  std::string sfx;  // scratch-name suffix of the side branch (its own look-back status words)

  // stable radix sort wrapper; returns pointers to the sorted keys / vals
  template <class K>
  void sort(K*& keys, uint32_t*& vals, uint64_t n, int nbits, const char* tag, bool distinct = false) {
    if (n <= 1 || nbits <= 0) return;
    struct Tag {  // profiled analyses time the sort's kernels under its tag
      explicit Tag(const char* t) { if (g_prof) g_prof->tag = t; }
      ~Tag() { if (g_prof) g_prof->tag = nullptr; }
    } tag_guard(tag);
    if (distinct && n <= kRankSortMax) {
      K* ka = C->get<K>(std::string(tag) + "_ka", n);
      uint32_t* va = C->get<uint32_t>(std::string(tag) + "_va", n);
      GW_LAUNCH(k_sort_rank<K>, (unsigned)((n + kThreads - 1) / kThreads), kThreads, 0, st, keys, vals, ka, va,
                (uint32_t)n);
      keys = ka;
      vals = va;
      return;
    }
    if (distinct && n <= small_sort_max<K>()) {
      // one CTA, in shared memory (distinct keys: stability is moot)
      uint32_t p2 = 1;
      while (p2 < n) p2 <<= 1;
      sort_small_setup<K>();
      GW_LAUNCH(k_sort_small<K>, 1, kSmallThreads, p2 * (sizeof(K) + 4), st, keys, vals, (uint32_t)n, p2);
      return;
    }
    std::string t(tag);
    K* ka = C->get<K>(t + "_ka", n);
    uint32_t* va = C->get<uint32_t>(t + "_va", n);
    const int npass = rs_passes(nbits);
    if (n >= kRsBigN) {
      // reduce-then-scan passes: digit counts per super-tile, one scan, scatter
      if (rs_big_bits(nbits) == 10) big_sort<K, 10>(keys, ka, vals, va, n, nbits);
      else big_sort<K, 8>(keys, ka, vals, va, n, nbits);
      return;
    }
    SortScratch sc;
    sc.ghist = pre_ghist ? pre_ghist : zeroed(kRsMaxPass * kRsMaxDigits);
    sc.ghist_ready = pre_ghist != nullptr;
    pre_ghist = nullptr;
    sc.ctrs = zeroed(npass);
    sc.status = C->get<unsigned long long>(std::string("rs_status") + sfx,
                                           2 * std::max(lb_tiles(n), lb_tiles(tr.n)) * kRsMaxDigits);
    bool alt = radix_sort<K>(keys, ka, vals, va, n, nbits, sc, take_epochs(npass), st);
    if (alt) {
      keys = ka;
      vals = va;
    }
  }

  // bits of pass p when nbits are spread evenly over ceil(nbits / 8) passes
  // (low passes take the remainder): 29 -> 8, 7, 7, 7
  static int big_pass_bits(int nbits, int p, int* shift) {
    const int np = (nbits + kRsBits - 1) / kRsBits, b = nbits / np, x = nbits % np;
    *shift = p * b + std::min(p, x);
    return b + (p < x ? 1 : 0);
  }
  template <class K, int RB>
  void big_pass(const K* ki, const uint32_t* vi, K* ko, uint32_t* vo, uint64_t n, int shift, uint32_t* counts,
                uint64_t nst, unsigned g, bool counted) {
    if (!counted) GW_LAUNCH((k_rs_up<K, RB>), g, kThreads, 0, st, ki, n, shift, counts, nst);
    scan<uint32_t, OpSum>(ArrLoad<uint32_t>{counts}, ArrStore<uint32_t>{counts}, nst * (1u << RB), OpSum(), 0u, false,
                          "sc_u32");
    rs_down_tma_setup<K, RB>();
    GW_LAUNCH((k_rs_down_tma<K, RB>), g, kThreads, sizeof(RsTmaSmem<K>), st, ki, vi, ko, vo, n, shift, counts, nst);
  }
  template <class K, int RB>
  void big_sort(K*& keys, K* ka, uint32_t*& vals, uint32_t* va, uint64_t n, int nbits) {
    const uint64_t nst = (lb_tiles(n) + RsBig<RB>::ST - 1) / RsBig<RB>::ST;
    uint32_t* counts = C->get<uint32_t>(std::string("rs_counts") + sfx, nst * RsBig<RB>::ND);
    const bool counts0 = pre_counts == counts && RB == 8;  // pass 0 counted by k_ingest
    pre_counts = nullptr;
    const unsigned g = (unsigned)std::min<uint64_t>(nst, 148ull * 16);
    bool alt = false;
    if constexpr (RB == 8) {  // ST == 1: TMA-streamed input tiles, balanced <= 8-bit digits
      const int npass = (nbits + RB - 1) / RB;
      for (int p = 0; p < npass; p++) {
        const K* ki = alt ? ka : keys;
        const uint32_t* vi = alt ? va : vals;
        K* ko = alt ? keys : ka;
        uint32_t* vo = alt ? vals : va;
        int shift = 0;
        const int b = big_pass_bits(nbits, p, &shift);
        const bool cnt = p == 0 && counts0;
        switch (b) {
          case 8: big_pass<K, 8>(ki, vi, ko, vo, n, shift, counts, nst, g, cnt); break;
          case 7: big_pass<K, 7>(ki, vi, ko, vo, n, shift, counts, nst, g, cnt); break;
          case 6: big_pass<K, 6>(ki, vi, ko, vo, n, shift, counts, nst, g, cnt); break;
          case 5: big_pass<K, 5>(ki, vi, ko, vo, n, shift, counts, nst, g, cnt); break;
          default: big_pass<K, 4>(ki, vi, ko, vo, n, shift, counts, nst, g, cnt); break;
        }
        alt = !alt;
      }
    } else {
      const int npass = (nbits + RB - 1) / RB;
      rs_down_setup<K, RB>();
      for (int p = 0; p < npass; p++) {
        K* ki = alt ? ka : keys;
        uint32_t* vi = alt ? va : vals;
        K* ko = alt ? keys : ka;
        uint32_t* vo = alt ? vals : va;
        GW_LAUNCH((k_rs_up<K, RB>), g, kThreads, 0, st, ki, n, RB * p, counts, nst);
        scan<uint32_t, OpSum>(ArrLoad<uint32_t>{counts}, ArrStore<uint32_t>{counts}, nst * RsBig<RB>::ND, OpSum(), 0u,
                              false, "sc_u32");
        GW_LAUNCH((k_rs_down<K, RB>), g, kThreads, sizeof(RsBigSmem<K, RB>), st, ki, vi, ko, vo, n, RB * p, counts,
                  nst);
        alt = !alt;
      }
    }
    if (alt) {
      keys = ka;
      vals = va;
    }
  }

  template <class T, class Op, class Load, class Store>
  void scan(Load load, Store store, uint64_t n, Op op, T identity, bool inclusive, const char*) {
    if (n == 0) return;
    unsigned long long* status =
        C->get<unsigned long long>(std::string("lb_status") + sfx, std::max(lb_tiles(n), lb_tiles(tr.n)));
    scan_lb<T, Op>(load, store, n, status, zeroed(1), op, identity, inclusive, st);
  }

  static KeyRuns key_runs(unsigned long long D) {
    KeyRuns kr;
    memset(&kr, 0, sizeof kr);
    std::vector<std::pair<int, int>> runs;  // (src, width) of the varying bit runs
    for (int b = 0; b < 64;) {
      if ((D >> b) & 1ull) {
        int s = b;
        while (b < 64 && ((D >> b) & 1ull)) b++;
        runs.push_back({s, b - s});
      } else {
        b++;
      }
    }
    while (runs.size() > 4) {  // merge the pair with the smallest gap
      size_t best = 0;
      int gap = 1 << 30;
      for (size_t i = 0; i + 1 < runs.size(); i++) {
        int g = runs[i + 1].first - (runs[i].first + runs[i].second);
        if (g < gap) { gap = g; best = i; }
      }
      runs[best].second = runs[best + 1].first + runs[best + 1].second - runs[best].first;
      runs.erase(runs.begin() + best + 1);
    }
    int dpos = 0;
    kr.n = (int)runs.size();
    for (int i = 0; i < kr.n; i++) {
      kr.src[i] = runs[i].first;
      kr.width[i] = runs[i].second;
      kr.dst[i] = dpos;
      dpos += runs[i].second;
    }
    kr.sentinel = dpos < 64;
    kr.nbits = dpos + (kr.sentinel ? 1 : 0);
    return kr;
  }

  // observed by an eager run, used to build a Plan
  Stats obs{};
  uint32_t obs_ncand = 0, obs_nlarge = 0, obs_nspill = 0, obs_npend = 0;
  unsigned long long obs_D = 0;
  uint64_t obs_cand_cap = 0;
  bool obs_snap = false;

  void run() {
    gw_stats& S = C->stats;
    memset(&S, 0, sizeof S);
    const uint64_t N = tr.n;
    C->n_events = N;
    C->n_reports = 0;
    C->n_diags = 0;
    g_launches = 0;
    for (int i = 0; i < gw_ctx::kEv; i++)
      if (!C->ev[i]) CK(cudaEventCreate(&C->ev[i]));
    for (int p = 0; p < 5; p++) C->nint[p] = 0;
    event(0);
    C->d_scal = nullptr;
    C->d_nsurv = nullptr;
    C->stats_pending = false;
    C->phases = !gmode;
    C->last_stream = st;
    C->have_cands = false;
    if (N == 0) {
      C->launches = 0;
      return;
    }
    // ---------------------------------------------------------------- prep
    pbeg(PH_PREP);
    zero_blk = C->get<uint32_t>("zero_blk", kZeroWords);
    zero_next = 0;
    scal = C->get<uint32_t>("scalars", SC_COUNT);
    CK(cudaMemsetAsync(zero_blk, 0, sizeof(uint32_t) * kZeroWords, st));
    CK(cudaMemsetAsync(scal, 0, SC_COUNT * sizeof(uint32_t), st));
    if (!gmode) reserve_epochs();
    if (gmode) {  // fixed epochs in the graph: start from clean flags
      for (const char* nm : {"rs_status", "rs_status_b"}) {
        unsigned long long* rs = C->get<unsigned long long>(nm, 2 * lb_tiles(N) * kRsMaxDigits);
        CK(cudaMemsetAsync(rs, 0, C->bufs[nm].cap, st));
      }
    }
    // graph replays of a lock-free plan: the location sort needs only the
    // plan's key runs, so its branch forks before k_prep (the plan check
    // still guards the results: a mismatch re-runs eagerly)
    const char* nf = getenv("GW_FORK");  // experiment hook: GW_FORK=0 runs the sort after the walker
    const bool fork_ok = !(nf && nf[0] == '0');
    const bool early_fork = fork_ok && gmode && nshard <= 1 && !g_prof;
    Stats* dst = C->get<Stats>("stats", 1);
    if (early_fork) {
      memset(&hs, 0, sizeof hs);
      hs.key_or = P->D;
      ingest();  // big traces: stats + keys + first digit counts (+ hard events) in one read
      fork_sort();
      if (P->hard_small) fork_hard();  // the hard-event list needs only the trace and the plan's count
    }
    if (!ingested) {
      GW_LAUNCH(k_init_stats, 1, 1, 0, st, dst);
      GW_LAUNCH(k_prep, grid_for(N), kThreads, 0, st, tr, dst);
    }
    check_launch();
    if (gmode) {
      memset(&hs, 0, sizeof hs);
      hs.n_bar = P->n_bar;
      hs.n_end = P->n_end;
      hs.n_wbar = P->n_wbar;
      hs.key_or = P->D;
      hs.key_and = 0;
      GW_LAUNCH(k_plan_check, 1, 1, 0, st, dst, P->n_bar, P->n_end, P->n_wbar, P->D, P->n_acc, scal + SC_ABORT);
    } else {
      d2h(&hs, dst);
      obs = hs;
    }
    has_locks = hs.n_acq + hs.n_rel > 0;
    S.n_accesses = hs.n_acc;

    if (!ingested) plan_sync_pass();
    if (has_locks) lock_prepass();
    pend(PH_PREP);

    Cands cd;
    if (fork_ok && !has_locks && nshard <= 1 && !g_prof) {
      // the location sort does not depend on the sync pass: it runs on the
      // side stream while the walker runs here; the stamps (aux) are filled
      // after the walker, then the branches join before the check
      if (!early_fork) fork_sort();
      pbeg(PH_WALKER);
      walker_phase();
      if (!bk_mode && aux) GW_LAUNCH(k_acc_aux, grid_for(N), kThreads, 0, st, tr, stamps, aux);
      pend(PH_WALKER);
      CK(cudaStreamWaitEvent(st, C->ev_join, 0));
      pbeg(PH_CHECK);
      cd = bk_mode ? bucket_check_pass() : check_pass(false, "c", SC_NCAND);
      pend(PH_CHECK);
    } else if (!has_locks) {
      pbeg(PH_WALKER);
      walker_phase();
      pend(PH_WALKER);
      pbeg(PH_SORT);
      access_sort();
      pend(PH_SORT);
      pbeg(PH_CHECK);
      cd = bk_mode ? bucket_check_pass() : check_pass(false, "c", SC_NCAND);
      pend(PH_CHECK);
    } else {
      // lock mode: the structural candidates first (clock independent), then
      // the walker answers their clock half in trace order
      pbeg(PH_SORT);
      access_sort();
      pend(PH_SORT);
      pbeg(PH_CHECK);
      Cands cq = check_pass(true, "q", SC_NQ);
      pend(PH_CHECK);
      pbeg(PH_WALKER);
      const uint64_t nq = obs_nq;
      query_setup(cq, nq);
      walker_phase();
      pend(PH_WALKER);
      pbeg(PH_CHECK);
      cd = resolve_pass(cq, nq);
      pend(PH_CHECK);
    }

    // ------------------------------------------------------- dedup / final
    pbeg(PH_FINAL);
    const uint32_t ncap = gmode ? cd.cap : obs_ncand;
    uint32_t* out_n = scal + SC_NCAND;  // [NCAND], [NLARGE], [NSURV]
    uint32_t* d_nsurv = out_n + 2;
    C->d_scal = scal;
    C->d_nsurv = d_nsurv;
    C->have_cands = ncap > 0;
    if (ncap > 0) {
      uint64_t tcap = pow2_at_least(2ull * ncap);
      DedupArgs d;
      d.c = cd;
      d.instr = tr.instr;
      d.owner = C->get<uint32_t>("dd_owner", tcap);
      d.smin = C->get<unsigned long long>("dd_min", tcap);
      d.cslot = C->get<uint32_t>("dd_slot", ncap);
      d.mask = (uint32_t)(tcap - 1);
      d.ncand = ncap;
      d.dn = out_n;
      CK(cudaMemsetAsync(d.owner, 0, sizeof(uint32_t) * tcap, st));
      CK(cudaMemsetAsync(d.smin, 0xFF, sizeof(unsigned long long) * tcap, st));
      GW_LAUNCH(k_dedup_insert, grid_for(ncap), kThreads, 0, st, d);
      // survivors ordered by their order key; the others sort last
      unsigned long long* sk = C->get<unsigned long long>("sv_k", ncap);
      uint32_t* sv = C->get<uint32_t>("sv_v", ncap);
      if (N <= (1ull << 25) && ncap > small_sort_max<unsigned long long>()) {
        // small trace: counting sort by event bucket (event >> cs, <= 16 events per
        // bucket, about one bucket per candidate), then each run by order key
        const int cs = std::min(4, std::max(0, ceil_log2(N) - ceil_log2((uint64_t)ncap)));
        const uint64_t nb = ((N - 1) >> cs) + 1;
        uint32_t* sk32 = C->get<uint32_t>("sv_k32", ncap);
        uint32_t* ccnt = C->get<uint32_t>("sv_cnt", nb);
        uint32_t* coff = C->get<uint32_t>("sv_off", nb);
        CK(cudaMemsetAsync(ccnt, 0, sizeof(uint32_t) * nb, st));
        GW_LAUNCH(k_surv_count, grid_for(ncap), kThreads, 0, st, d, ccnt, d_nsurv, (uint32_t)cs);
        scan<uint32_t, OpSum>(ArrLoad<uint32_t>{ccnt}, ArrStore<uint32_t>{coff}, nb, OpSum(), 0u, false, "sc_u32");
        GW_LAUNCH(k_surv_place, grid_for(ncap), kThreads, 0, st, d, ccnt, coff, sk32, sv, (uint32_t)cs);
        GW_LAUNCH(k_group_fix, grid_for(ncap), kThreads, 0, st, sk32, sv, (uint32_t)ncap, (uint32_t)nb, cd.okey,
                  d_nsurv);
      } else if (ncap <= small_sort_max<unsigned long long>()) {
        GW_LAUNCH(k_dedup_keys, grid_for(ncap), kThreads, 0, st, d, (unsigned long long)N, sk, sv, d_nsurv);
        sort<unsigned long long>(sk, sv, ncap, 32 + ceil_log2(N + 1), "sv", true);
      } else {
        uint32_t* sk32 = C->get<uint32_t>("sv_k32", ncap);
        GW_LAUNCH(k_dedup_keys32, grid_for(ncap), kThreads, 0, st, d, (uint32_t)N, sk32, sv, d_nsurv);
        sort<uint32_t>(sk32, sv, ncap, ceil_log2(N + 1), "sv32");
        GW_LAUNCH(k_group_fix, grid_for(ncap), kThreads, 0, st, sk32, sv, (uint32_t)ncap, (uint32_t)N, cd.okey);
      }
      uint8_t* H = C->host_res(kResHdr + 17ull * ncap);  // mapped: the kernel writes over the bus
      C->d_okey = (unsigned long long*)(H + kResHdr);
      C->d_prior = (uint32_t*)(H + kResHdr + 8ull * ncap);
      C->d_cur = (uint32_t*)(H + kResHdr + 12ull * ncap);
      C->d_kind = H + kResHdr + 16ull * ncap;
      GW_LAUNCH(k_final, grid_for(ncap), kThreads, 0, st, cd, sv, d_nsurv, C->d_kind, C->d_prior, C->d_cur,
                C->d_okey);
      check_launch();
    }
    if (hard_forked && !hard_joined) CK(cudaStreamWaitEvent(st, C->ev_hard, 0));  // every branch rejoins
    C->d_diags = w.diags;
    C->arena_words = arena_units << OBJ_USHIFT;
    C->h_scal = (uint32_t*)C->host_res(kResHdr + (ncap > 0 ? 17ull * ncap : 0ull));
    CK(cudaMemcpyAsync(C->h_scal, scal, SC_COUNT * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    pend(PH_FINAL);
    event(1);
    S.n_sync = hs.n_acq + hs.n_rel + hs.n_end + hs.n_bar;
    C->launches = g_launches;
    C->stats_pending = !gmode;
  }

  // the sync-pass mode (snapshot / warp snapshot / walker / lock walker) and
  // the walker's arguments, from the trace statistics hs
  uint64_t budget_n = 0;  // exchange mode: size the snapshot budget by the whole trace
  void plan_sync_pass() {
    const uint64_t N = tr.n;
    gw_stats& S = C->stats;
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_walker, kThreads, 0));
    gmax = (uint64_t)std::max(occ, 1) * C->num_sms;
    G = (uint32_t)std::min<uint64_t>(tr.B, gmax);
    S.walker_ctas = G;
    // snapshot mode: lock-free and the per-hard-event block snapshots are small
    n_hard = hs.n_bar + hs.n_end;
    snap_entries = (n_hard + tr.B) * (uint64_t)tr.BS;
    const uint64_t snap_budget = std::max<uint64_t>(256ull << 20, 8 * (budget_n ? budget_n : N));
    // GW_WALK_MODE=block|warp|walker forces a lock-free sync-pass mode when applicable (tests)
    const char* wm = getenv("GW_WALK_MODE");
    const bool force_warp = wm && !strcmp(wm, "warp"), force_walker = wm && !strcmp(wm, "walker");
    snap_mode = !has_locks && snap_entries * 8 <= snap_budget && !force_warp && !force_walker;
    // warp snapshot mode: per-(block, warp) lists, block barriers replicated into every warp's list
    n_hard_w = hs.n_wbar + hs.n_end + (uint64_t)kWSnapWarps * (hs.n_bar - hs.n_wbar);
    const uint64_t wsnap_entries = (n_hard_w + (uint64_t)tr.B * kWSnapWarps) * 32ull;
    wsnap_mode = !has_locks && !snap_mode && !force_walker && tr.W <= kWSnapWarps && tr.L <= 32 &&
                 wsnap_entries * 8 <= snap_budget;
    if (wsnap_mode) snap_entries = wsnap_entries;
    obs_snap = snap_mode || wsnap_mode;
    memset(&w, 0, sizeof w);
    w.tr = tr;
    w.G = G;
    w.has_locks = has_locks ? 1 : 0;
    w.inactive_opt = inactive_opt;
    w.abort_flag = scal + SC_ABORT;
    w.err = scal + SC_ERR;
    w.hb_mode = hb_mode ? 1u : 0u;
    // lock traces with <= 8 warps of <= 32 lanes: one walker warp per trace warp
    const char* lwm = getenv("GW_LOCK_WALK");
    lock_warp = has_locks && tr.W <= kLW && tr.L <= 32 && !(lwm && !strcmp(lwm, "cta"));
    if (lock_warp) {
      int occ_lw = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_lw, k_walker_lw, kThreads, 0));
      G = (uint32_t)std::min<uint64_t>(tr.B, (uint64_t)std::max(occ_lw, 1) * C->num_sms);
      S.walker_ctas = G;
      w.G = G;
      uint32_t* part_key = C->get<uint32_t>("part_k", N);
      uint32_t* perm = C->get<uint32_t>("part_v", N);
      GW_LAUNCH(k_part_keys_lw, grid_for(N), kThreads, 0, st, tr, G, part_key, perm);
      sort<uint32_t>(part_key, perm, N, ceil_log2((uint64_t)G * kLW + 1), "part");
      w.part_key = part_key;
      w.perm = perm;
    } else if (G > 1 && !snap_mode && !wsnap_mode) {
      uint32_t* part_key = C->get<uint32_t>("part_k", N);
      uint32_t* perm = C->get<uint32_t>("part_v", N);
      GW_LAUNCH(k_part_keys, grid_for(N), kThreads, 0, st, tr, G, part_key, perm);
      sort<uint32_t>(part_key, perm, N, ceil_log2(G), "part");
      w.part_key = part_key;
      w.perm = perm;
    }
  }

  // hard-event list of the snapshot walker in one launch (<= kRankSortMax events)
  bool obs_hard_small = false, hard_forked = false, hard_joined = false;
  bool hard_small_ok(uint64_t nh) const {
    const char* hsm = getenv("GW_HARD_SMALL");  // experiment hook: GW_HARD_SMALL=0 keeps sort + unpack + scan
    return nh && nh <= kRankSortMax && tr.B <= (uint64_t)kThreads * 64 && !(hsm && hsm[0] == '0');
  }
  void hard_small_list(uint64_t nh, uint32_t* hev, uint32_t* hcnt, uint32_t* hbeg, uint32_t* hend) {
    unsigned long long* hkey = C->get<unsigned long long>("hd_key", nh + 1);
    GW_LAUNCH(k_hard_append, grid_for(tr.n), kThreads, 0, st, tr, hkey, hcnt, zeroed(1), scal + SC_ABORT,
              (uint32_t)(nh + 1));
    GW_LAUNCH(k_hard_small, (unsigned)((nh + kThreads - 1) / kThreads), kThreads, 0, st, hkey, (uint32_t)nh, hev,
              hcnt, tr.B, hbeg, hend);
  }
  // graph replays: the hard-event list on a third branch from the graph start,
  // beside k_prep / k_state_init (it may run before the plan check: k_hard_append
  // never writes past the plan's count, and the walker itself checks the abort flag)
  void fork_hard() {
    const uint64_t nh = P->n_bar + P->n_end;
    if (!hard_small_ok(nh)) return;
    if (!C->side2) {
      CK(cudaStreamCreateWithFlags(&C->side2, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&C->ev_fork2, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&C->ev_hard, cudaEventDisableTiming));
    }
    const cudaStream_t main_st = st;
    uint32_t* hev = C->get<uint32_t>("hd_ev", nh + 1);
    uint32_t* hcnt = C->get<uint32_t>("hd_cnt", tr.B);
    uint32_t* hbeg = C->get<uint32_t>("hd_beg", tr.B);
    uint32_t* hend = C->get<uint32_t>("hd_end", tr.B);
    CK(cudaEventRecord(C->ev_fork2, main_st));
    CK(cudaStreamWaitEvent(C->side2, C->ev_fork2, 0));
    st = C->side2;
    CK(cudaMemsetAsync(hcnt, 0, sizeof(uint32_t) * tr.B, st));
    hard_small_list(nh, hev, hcnt, hbeg, hend);
    CK(cudaEventRecord(C->ev_hard, st));
    st = main_st;
    hard_forked = true;
  }

  // Graph replays of big lock-free traces (32-bit location keys, LSD pass):
  // k_ingest reads the trace once for the plan check's stats, the location
  // keys, the first sort pass's digit counts and (snapshot mode, large hard
  // list) the hard events, instead of k_prep + k_acc_keys + k_rs_up +
  // k_hard_append each reading it.  Sets the plan's sync-pass mode early
  // (plan_sync_pass depends only on the plan in graph mode).
  bool ingested = false, hard_ingested = false;
  uint32_t* pre_counts = nullptr;  // digit counts of the first big-sort pass (k_ingest)
  void ingest() {
    const char* e = getenv("GW_INGEST");  // 0 = the separate kernels
    if (e && e[0] == '0') return;
    const uint64_t N = tr.n;
    plan_access();
    if (wide || bk_mode || N < kRsBigN || rs_big_bits(kr.nbits) != 8 || kr.nbits <= 0) return;
    hs.n_bar = P->n_bar;
    hs.n_end = P->n_end;
    hs.n_wbar = P->n_wbar;
    has_locks = false;
    plan_sync_pass();
    Stats* dst = C->get<Stats>("stats", 1);
    GW_LAUNCH(k_init_stats, 1, 1, 0, st, dst);
    IngestHard hd{nullptr, nullptr, nullptr, 0};
    if (snap_mode && !P->hard_small && n_hard > 0) {
      hd.hkey = C->get<unsigned long long>("hd_key", n_hard + 1);
      hd.hcnt = C->get<uint32_t>("hd_cnt", tr.B);
      hd.ntop = zeroed(1);
      hd.cap = (uint32_t)(n_hard + 1);
      CK(cudaMemsetAsync(hd.hcnt, 0, sizeof(uint32_t) * tr.B, st));
      hard_ingested = true;
    }
    const uint64_t nst = lb_tiles(N);
    pre_counts = C->get<uint32_t>("rs_counts_b", nst * RsBig<8>::ND);
    vals = C->get<uint32_t>("acc_v", N);
    uint32_t* k32 = C->get<uint32_t>("acc_k", N);
    int sh0 = 0;
    const int rb0 = big_pass_bits(kr.nbits, 0, &sh0);  // the first big-sort pass's digit width
    GW_LAUNCH(k_ingest<uint32_t>, (unsigned)std::min<uint64_t>(nst, 148ull * 8), kThreads, 0, st, tr, kr, k32, vals,
              dst, pre_counts, nst, hd, rb0);
    skeys = k32;
    ingested = true;
  }

  // the access sort on the side stream (joined through ev_join before the check)
  void fork_sort() {
    if (!C->side) {
      CK(cudaStreamCreateWithFlags(&C->side, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&C->ev_fork, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&C->ev_join, cudaEventDisableTiming));
    }
    const cudaStream_t main_st = st;
    plan_access();
    aux = (bk_mode || acc_lazy) ? nullptr : C->get<uint4>("acc_aux", tr.n);  // allocated on this stream: k_acc_aux writes it here
    CK(cudaEventRecord(C->ev_fork, main_st));
    CK(cudaStreamWaitEvent(C->side, C->ev_fork, 0));
    st = C->side;
    C->last_stream = st;
    sfx = "_b";
    pbeg(PH_SORT);
    access_sort(true);
    pend(PH_SORT);
    CK(cudaEventRecord(C->ev_join, st));
    st = main_st;
    C->last_stream = st;
    sfx.clear();
  }

  // k_access / k_acc_tilemax items per thread: the larger tile when it brings
  // the sorted positions into one wave of resident CTAs (3 per SM at either
  // size with 32-bit keys), else the smaller one
  int acc_items = kAccItemsSmall;
  int pick_acc_items(uint64_t NA) const {
    if (wide) return kAccItemsSmall;
    const uint64_t slots = 3ull * (uint64_t)C->num_sms;
    const uint64_t ts = kThreads * kAccItemsSmall, tl = kThreads * kAccItemsLarge;
    return ((NA + ts - 1) / ts > slots && (NA + tl - 1) / tl <= slots) ? kAccItemsLarge : kAccItemsSmall;
  }

  uint32_t* pre_ghist = nullptr;  // digit histograms built by the key pass, consumed by the next sort()

  // ---- pipeline state shared by the phases --------------------------------
  uint32_t* scal = nullptr;
  Stats hs{};
  bool has_locks = false, snap_mode = false, wsnap_mode = false, lock_warp = false;
  uint64_t n_hard_w = 0;
  uint64_t gmax = 1, n_hard = 0, snap_entries = 0, lcap = 1, arena_units = 0;
  uint32_t G = 1, maxd = 1, n_incs = 0;
  WalkArgs w;
  KeyRuns kr{};
  bool wide = false;
  uint32_t* vals = nullptr;  // access pass: sorted event indices
  void* skeys = nullptr;
  uint2* carry = nullptr;     // per sorted tile: max (segment head, write position) of the earlier tiles
  unsigned long long* acc_lb = nullptr;  // or: k_access's look-back status words (zeroed before each launch)
  uint64_t acc_lb_n = 0;
  DupList dup{};              // same-record pairs flagged by the access check

  // _same_instruction_check (engine.py:81-95): from the flagged records, or a
  // scan of every record when a record is longer than 32 events or the flag
  // list overflowed (eager runs; graph replays abort on overflow instead)
  void same_instr_pass(const Cands& cd) {
    bool list = dup.ev != nullptr;
    if (list && !gmode) {
      uint32_t nd = 0;
      d2h(&nd, dup.n);
      list = nd <= dup.cap;
    }
    if (!list) {
      GW_LAUNCH(k_same_instr, grid_for(tr.n), kThreads, 0, st, tr, cd, shard_args(), 0);
      return;
    }
    const uint64_t hcap = pow2_at_least(2ull * dup.cap + 2);
    uint32_t* hset = C->get<uint32_t>("dup_hset", hcap);
    uint32_t* heads = C->get<uint32_t>("dup_heads", dup.cap + 1);
    CK(cudaMemsetAsync(hset, 0, sizeof(uint32_t) * hcap, st));
    CK(cudaMemsetAsync(scal + SC_NHEADS, 0, sizeof(uint32_t), st));
    GW_LAUNCH(k_dup_heads, 148u * 4, kThreads, 0, st, tr, dup, hset, (uint32_t)(hcap - 1), heads, scal + SC_NHEADS);
    GW_LAUNCH(k_same_instr_heads, 148u * 4, kThreads, 0, st, tr, cd, shard_args(), heads, scal + SC_NHEADS);
  }
  StampSrc stamps{};          // where the access pass reads access stamps (walker output)
  uint4* aux = nullptr;       // per event (tidop, time, vobj); nullptr: k_access looks stamps up lazily
  bool acc_lazy = true;
  uint64_t obs_nq = 0;
  uint32_t shard = 0, nshard = 1;  // address sharding (gw_opts)
  bool hb_mode = false;            // GW_OPT_HB: scoped happens-before detector
  uint64_t na_sorted = 0;          // positions the access pass sorts (N, or this shard's accesses)
  ShardArgs shard_args() const {
    ShardArgs sa;
    sa.kr = kr;
    sa.nloc = kr.nbits - kr.sentinel;
    sa.shard = shard;
    sa.G = nshard;
    return sa;
  }

  // ------------------------------------------------------- lock pre-pass
  void lock_prepass() {
    const uint64_t N = tr.n;
    const uint64_t nle = hs.n_acq + hs.n_rel + hs.n_end;
    uint32_t* flag = C->get<uint32_t>("lk_flag", N);
    GW_LAUNCH(k_lock_mark, grid_for(N), kThreads, 0, st, tr, flag);
    scan<uint32_t, OpSum>(ArrLoad<uint32_t>{flag}, ArrStore<uint32_t>{flag}, N, OpSum(), 0u, false, "sc_u32");
    uint32_t* ktid = C->get<uint32_t>("lk_tid", nle);
    uint32_t* kev = C->get<uint32_t>("lk_ev", nle);
    GW_LAUNCH(k_lock_compact, grid_for(N), kThreads, 0, st, tr, flag, ktid, kev);
    sort<uint32_t>(ktid, kev, nle, ceil_log2(tr.T), "lk");
    uint32_t* seg_beg = C->get<uint32_t>("lk_sb", tr.T);
    uint32_t* seg_end = C->get<uint32_t>("lk_se", tr.T);
    CK(cudaMemsetAsync(seg_beg, 0, sizeof(uint32_t) * tr.T, st));
    CK(cudaMemsetAsync(seg_end, 0, sizeof(uint32_t) * tr.T, st));
    GW_LAUNCH(k_lock_segs, grid_for(nle), kThreads, 0, st, ktid, (uint32_t)nle, seg_beg, seg_end);
    unsigned long long* node_lock = C->get<unsigned long long>("lk_nlock", nle);
    uint32_t* node_parent = C->get<uint32_t>("lk_nparent", nle);
    uint32_t* top_after = C->get<uint32_t>("lk_top", nle);
    uint8_t* lflags = C->get<uint8_t>("lflags", N);
    CK(cudaMemsetAsync(lflags, 0, N, st));
    GW_LAUNCH(k_lock_automaton, grid_for(nle), kThreads, 0, st, tr, ktid, kev, (uint32_t)nle, seg_end, node_lock,
              node_parent, top_after, lflags, scal + SC_MAXD);
    uint32_t* etop = C->get<uint32_t>("lk_etop", N);
    uint32_t* npair = C->get<uint32_t>("lk_npair", N);
    GW_LAUNCH(k_lock_access, grid_for(N), kThreads, 0, st, tr, kev, top_after, seg_beg, seg_end, node_parent,
              lflags, etop, npair, scal + SC_NINCS);
    uint32_t* poff = C->get<uint32_t>("lk_poff", N);
    scan<uint32_t, OpSum>(ArrLoad<uint32_t>{npair}, ArrStore<uint32_t>{poff}, N, OpSum(), 0u, false, "sc_u32");
    uint32_t hv[4];
    CK(cudaMemcpyAsync(hv, poff + (N - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hv + 1, npair + (N - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hv + 2, scal, 2 * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const uint64_t NP = (uint64_t)hv[0] + hv[1];
    maxd = std::max<uint32_t>(hv[2], 1);
    n_incs = hv[3];
    unsigned long long* plock = C->get<unsigned long long>("lk_plock", NP + 1);
    unsigned long long* pk = C->get<unsigned long long>("lk_pk", NP + 1);
    uint32_t* pv = C->get<uint32_t>("lk_pv", NP + 1);
    uint8_t* pacq = C->get<uint8_t>("lk_pacq", NP + 1);
    unsigned long long* orand = C->get<unsigned long long>("lk_orand", 2);
    GW_LAUNCH(k_orand_init, 1, 1, 0, st, orand);
    GW_LAUNCH(k_lock_pairs, grid_for(N), kThreads, 0, st, tr, poff, npair, etop, node_lock, node_parent, plock, pv,
              pacq, orand);
    unsigned long long ho[2];
    d2h(ho, orand, 2);
    KeyRuns lkr = key_runs(NP ? ho[0] ^ ho[1] : 0ull);
    lkr.sentinel = 0;
    lkr.nbits = 0;
    for (int i = 0; i < lkr.n; i++) lkr.nbits += lkr.width[i];
    GW_LAUNCH(k_compact_u64, grid_for(NP + 1), kThreads, 0, st, plock, NP, lkr, pk);
    sort<unsigned long long>(pk, pv, NP, lkr.nbits, "lkp");
    uint32_t* segstart = C->get<uint32_t>("lk_pseg", NP + 1);
    scan<uint32_t, OpMaxU32>(LockSegLoad{pk}, ArrStore<uint32_t>{segstart}, NP, OpMaxU32(), 0u, true, "sc_u32");
    uint32_t* prank = C->get<uint32_t>("lk_prank", NP + 1);
    uint32_t* gacq = C->get<uint32_t>("lk_gacq", NP + 1);
    uint32_t* rix = C->get<uint32_t>("lk_rix", NP + 1);
    scan<uint32_t, OpSum>(AcqFlagLoad{pacq, pv}, ArrStore<uint32_t>{gacq}, NP, OpSum(), 0u, false, "sc_u32");
    // lock table (created here, one entry + ticket per lock) before the ranks kernel inserts into it
    lcap = pow2_at_least(2 * (hs.n_acq + hs.n_rel) + 2);
    w.locks = C->get<LockEnt>("t_lock", lcap);
    w.lock_mask = (uint32_t)(lcap - 1);
    CK(cudaMemsetAsync(w.locks, 0, sizeof(LockEnt) * lcap, st));
    w.plock = plock;
    GW_LAUNCH(k_lock_ranks, grid_for(NP + 1), kThreads, 0, st, w, pk, pv, segstart, pacq, gacq, NP, prank, rix);
    check_launch();
    w.lflags = lflags;
    w.poff = poff;
    w.npair = npair;
    w.prank = prank;
    w.rix = rix;
  }

  // ------------------------------------------------- access sort + scan
  // split: keys / vals only (the stamps are filled later by k_acc_aux)
  // key runs of the location keys, and the choice of access pass
  void plan_access() {
    kr = key_runs(gmode ? P->D : (hs.n_acc ? hs.key_or ^ hs.key_and : 0ull));
    C->stats.sort_bits = kr.nbits;
    wide = kr.nbits > 32;
    obs_D = hs.n_acc ? hs.key_or ^ hs.key_and : 0ull;
    bk_mode = bucket_ok(gmode ? P->n_acc : hs.n_acc);
    const char* lz = getenv("GW_ACC_LAZY");  // 0 = the per-event aux pass (k_acc_aux) instead of lazy stamps
    acc_lazy = !(lz && lz[0] == '0');
  }
  void access_sort(bool split = false) {
    const uint64_t N = tr.n;
    plan_access();
    if (bk_mode) {
      bucket_sort();
      return;
    }
    int nbits = kr.nbits;
    uint64_t NA = N;
    aux = acc_lazy ? nullptr : C->get<uint4>("acc_aux", N);
    if (nshard <= 1) {
      // All N positions are sorted; non-access events carry the top sentinel
      // key and sort last, and every access-pass kernel skips them, so no
      // kernel needs the access count on the host.
      vals = C->get<uint32_t>("acc_v", N);
      if (ingested) {
        // keys / events written by k_ingest
      } else if (!wide && N > 1 && N < kRsBigN && nbits > 0) {
        // one-sweep location sort next: the key pass also builds its digit histograms
        // (k_rs_ghist's grid: few CTAs, so few global flushes)
        uint32_t* k32 = C->get<uint32_t>("acc_k", N);
        pre_ghist = zeroed(kRsMaxPass * kRsMaxDigits);
        GW_LAUNCH(k_acc_keys<uint32_t>, (unsigned)std::min<uint64_t>(lb_tiles(N), 148ull * 8), kThreads, 0, st, tr,
                  kr, k32, vals, stamps, split ? nullptr : aux, pre_ghist, rs_digit_bits(nbits), rs_passes(nbits));
        skeys = k32;
      } else if (!wide) {
        uint32_t* k32 = C->get<uint32_t>("acc_k", N);
        GW_LAUNCH(k_acc_keys<uint32_t>, grid_for(N), kThreads, 0, st, tr, kr, k32, vals, stamps, split ? nullptr : aux);
        skeys = k32;
      } else {
        unsigned long long* k64 = C->get<unsigned long long>("acc_k64", N);
        GW_LAUNCH(k_acc_keys<unsigned long long>, grid_for(N), kThreads, 0, st, tr, kr, k64, vals, stamps,
                  split ? nullptr : aux);
        skeys = k64;
      }
    } else {
      // address shard: this shard's accesses only, in trace order (compacted keys, no sentinel)
      const ShardArgs sa = shard_args();
      const uint64_t nt = lb_tiles(N);
      uint32_t* tcnt = C->get<uint32_t>("sh_cnt", nt);
      uint32_t* toff = C->get<uint32_t>("sh_off", nt);
      const unsigned grid = (unsigned)std::min<uint64_t>(nt, 148ull * 8);
      GW_LAUNCH((k_shard_accesses<uint32_t, false>), grid, kThreads, 0, st, tr, sa, tcnt, toff, (uint32_t*)nullptr,
                (uint32_t*)nullptr, stamps, aux);
      scan<uint32_t, OpSum>(ArrLoad<uint32_t>{tcnt}, ArrStore<uint32_t>{toff}, nt, OpSum(), 0u, false, "sc_u32");
      uint32_t hv[2];
      CK(cudaMemcpyAsync(hv, toff + (nt - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(hv + 1, tcnt + (nt - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      NA = (uint64_t)hv[0] + hv[1];
      nbits = sa.nloc;
      wide = nbits > 32;
      vals = C->get<uint32_t>("acc_v", NA + 1);
      if (!wide) {
        uint32_t* k32 = C->get<uint32_t>("acc_k", NA + 1);
        GW_LAUNCH((k_shard_accesses<uint32_t, true>), grid, kThreads, 0, st, tr, sa, tcnt, toff, k32, vals, stamps,
                  aux);
        skeys = k32;
      } else {
        unsigned long long* k64 = C->get<unsigned long long>("acc_k64", NA + 1);
        GW_LAUNCH((k_shard_accesses<unsigned long long, true>), grid, kThreads, 0, st, tr, sa, tcnt, toff, k64, vals,
                  stamps, aux);
        skeys = k64;
      }
    }
    na_sorted = NA;
    C->stats.n_sorted = NA;
    if (!wide) {
      uint32_t* k32 = (uint32_t*)skeys;
      sort<uint32_t>(k32, vals, NA, nbits, "acc");
      skeys = k32;
    } else {
      unsigned long long* k64 = (unsigned long long*)skeys;
      sort<unsigned long long>(k64, vals, NA, nbits, "acc");
      skeys = k64;
    }
    // per-tile maxima of (segment head, write position), exclusive max-scan
    // over tiles: by k_access's own decoupled look-back (GW_ACC_LOOKBACK=0:
    // k_acc_tilemax + a scan)
    acc_items = pick_acc_items(NA);
    const uint64_t atile = (uint64_t)kThreads * acc_items;
    const uint64_t nt = (NA + atile - 1) / atile;
    const char* lbe = getenv("GW_ACC_LOOKBACK");
    if (!(lbe && lbe[0] == '0')) {
      acc_lb = C->get<unsigned long long>("acc_lb", nt + 1);
      acc_lb_n = nt + 1;
      carry = nullptr;
      return;
    }
    acc_lb = nullptr;
    uint2* agg = C->get<uint2>("acc_tagg", nt + 1);
    carry = C->get<uint2>("acc_carry", nt + 1);
    const unsigned tg = (unsigned)std::min<uint64_t>(std::max<uint64_t>(nt, 1), 148ull * 8);
    if (wide)
      GW_LAUNCH((k_acc_tilemax<unsigned long long, kAccItemsSmall>), tg, kThreads, 0, st,
                (const unsigned long long*)skeys, vals, NA, agg);
    else if (acc_items == kAccItemsLarge)
      GW_LAUNCH((k_acc_tilemax<uint32_t, kAccItemsLarge>), tg, kThreads, 0, st, (const uint32_t*)skeys, vals, NA, agg);
    else
      GW_LAUNCH((k_acc_tilemax<uint32_t, kAccItemsSmall>), tg, kThreads, 0, st, (const uint32_t*)skeys, vals, NA, agg);
    scan<uint2, OpMax2>(ArrLoad<uint2>{agg}, ArrStore<uint2>{carry}, nt, OpMax2(), make_uint2(0, 0), false, "sc_u2");
  }

  // ---------------------------------------- bucketed access pass (bucket.cuh)
  bool bk_mode = false;
  BkXInfo bk_xi{};  // exchange mode (xs_*): keys from h
  int bk_bb = 0, bk_kb = 0, bk_bA = 0, bk_bB = 0;
  uint64_t bk_na = 0;
  uint32_t *bk_h = nullptr, *bk_v = nullptr, *bk_t = nullptr, *bk_start = nullptr;
  // Single-GPU analyses take the LSD location sort: on C5 the two passes
  // measure the same (65.7 vs 65.6 ms, profiles/r2_*), and the sort's kernels
  // run at 0.40 of HBM where k_bk_check is issue-bound.  The
  // bucketed pass is the exchange mode's (multi-GPU) and GW_BUCKET=1's.
  bool bucket_ok(uint64_t na) const {
    const char* e = getenv("GW_BUCKET");  // 1 = the bucketed pass at any size, 2 = from 2^24 accesses
    if (!e || (e[0] != '1' && e[0] != '2')) return false;
    const uint64_t minn = e[0] == '1' ? 1ull : (1ull << 24);
    return !has_locks && nshard <= 1 && !wide && kr.nbits > 0 && na >= minn && tr.n < (1ull << 31);
  }
  static bool bk_tma_ok(const BkTraceSrc& s) {
    const char* e = getenv("GW_BK_TMA");  // test hook: 0 = plain-load scatter kernel
    return !(e && e[0] == '0') && ((uintptr_t)s.tr.key % 16) == 0 && ((uintptr_t)s.tr.tidop % 16) == 0;
  }
  static bool bk_tma_ok(const BkRecSrc&) {
    const char* e = getenv("GW_BK_TMA");
    return !(e && e[0] == '0');
  }
  template <class Src, int RB>
  void bk_pass_rb(Src src, uint64_t n_in, int shift, uint32_t* oh, uint32_t* ov, uint32_t* ot) {
    constexpr int ND = BkPass<RB>::ND, ST = BkPass<RB>::ST;
    const uint64_t nst = (lb_tiles(n_in) + ST - 1) / ST;
    uint32_t* counts = C->get<uint32_t>(std::string("bk_counts") + sfx, nst * ND);
    const unsigned g = (unsigned)std::min<uint64_t>(nst, 148ull * 16);
    GW_LAUNCH((k_bk_up<Src, RB>), g, kThreads, 0, st, src, shift, counts, nst);
    scan<uint32_t, OpSum>(ArrLoad<uint32_t>{counts}, ArrStore<uint32_t>{counts}, nst * ND, OpSum(), 0u, false,
                          "sc_u32");
    if (bk_tma_ok(src)) {  // TMA-streamed input tiles (16-byte aligned columns)
      bk_down_tma_setup<Src, RB>();
      GW_LAUNCH((k_bk_down_tma<Src, RB>), g, kThreads, sizeof(BkTmaSmem<RB>), st, src, shift, counts, nst, oh, ov,
                ot);
    } else {
      bk_down_setup<Src, RB>();
      GW_LAUNCH((k_bk_down<Src, RB>), g, kThreads, sizeof(BkDownSmem<RB>), st, src, shift, counts, nst, oh, ov, ot);
    }
  }
  template <class Src>
  void bk_pass(Src src, uint64_t n_in, int RB, int shift, uint32_t* oh, uint32_t* ov, uint32_t* ot) {
    switch (RB) {
      case 1: bk_pass_rb<Src, 1>(src, n_in, shift, oh, ov, ot); break;
      case 2: bk_pass_rb<Src, 2>(src, n_in, shift, oh, ov, ot); break;
      case 3: bk_pass_rb<Src, 3>(src, n_in, shift, oh, ov, ot); break;
      case 4: bk_pass_rb<Src, 4>(src, n_in, shift, oh, ov, ot); break;
      case 5: bk_pass_rb<Src, 5>(src, n_in, shift, oh, ov, ot); break;
      case 6: bk_pass_rb<Src, 6>(src, n_in, shift, oh, ov, ot); break;
      case 7: bk_pass_rb<Src, 7>(src, n_in, shift, oh, ov, ot); break;
      case 8: bk_pass_rb<Src, 8>(src, n_in, shift, oh, ov, ot); break;
      default: throw CudaErr{GW_E_ARG, "bucket digit width out of range"};
    }
  }
  // the access records (h, event|W, tidop) in bucket order (two stable passes)
  void bucket_sort() {
    const uint64_t na = xs_recv.h ? xs_recv.cnt : gmode ? P->n_acc : hs.n_acc;
    bk_na = na;
    // exchange mode: the top xs_gbits bits of h are the shard, the bucket bits follow
    bk_bb = std::min(kBkMaxBits, std::max(kBkMinBits, ceil_log2(std::max<uint64_t>(na, 1)) - 11));
    bk_kb = 32 - xs_gbits - bk_bb;
    bk_bA = bk_bb - bk_bb / 2;
    bk_bB = bk_bb / 2;
    uint32_t* ah = C->get<uint32_t>("bk_ah", na);
    uint32_t* av = C->get<uint32_t>("bk_av", na);
    uint32_t* at = C->get<uint32_t>("bk_at", na);
    bk_h = C->get<uint32_t>("bk_h", na);
    bk_v = C->get<uint32_t>("bk_v", na);
    bk_t = C->get<uint32_t>("bk_t", na);
    if (xs_recv.h) {  // exchange mode: this shard's records, received from every rank's slice
      BkRecSrc xs = xs_recv;
      bk_pass(xs, na, bk_bA, bk_kb, ah, av, at);
    } else {
      BkTraceSrc ts{tr, kr, 0u};
      bk_pass(ts, tr.n, bk_bA, bk_kb, ah, av, at);
    }
    BkRecSrc rs{ah, av, at, na};
    bk_pass(rs, na, bk_bB, bk_kb + bk_bA, bk_h, bk_v, bk_t);
    const uint32_t NB = 1u << bk_bb;
    bk_start = C->get<uint32_t>("bk_start", (uint64_t)NB + 1);
    GW_LAUNCH(k_bk_bounds, grid_for(na), kThreads, 0, st, bk_h, na, bk_kb, NB, bk_start);
    na_sorted = na;
    C->stats.n_sorted = na;
    C->stats.sort_bits = bk_bb;
  }
  // large reader windows (> kSmallWin reads between two writes) of the
  // positions in `a.vals`: (window, tid) groups through a secondary sort
  void large_windows(AccArgs<uint32_t>& a, uint32_t nl) {
    uint32_t* sizes = C->get<uint32_t>("lg_sz", nl + 1);
    std::vector<uint32_t> hi(nl), hw(nl);
    CK(cudaMemcpyAsync(hi.data(), a.large_i, sizeof(uint32_t) * nl, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hw.data(), a.large_ws, sizeof(uint32_t) * nl, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    std::vector<uint32_t> off(nl);
    uint64_t M = 0;
    for (uint32_t k = 0; k < nl; k++) {
      off[k] = (uint32_t)M;
      M += hi[k] - hw[k];
    }
    CK(cudaMemcpyAsync(sizes, off.data(), sizeof(uint32_t) * nl, cudaMemcpyHostToDevice, st));
    unsigned long long* lk = C->get<unsigned long long>("lg_k", M);
    uint32_t* lv = C->get<uint32_t>("lg_v", M);
    GW_LAUNCH(k_large_fill, std::min<uint32_t>(nl, 65535u), kThreads, 0, st, a.large_i, a.large_ws, sizes, nl, a.vals,
              tr.tidop, lk, lv);
    sort<unsigned long long>(lk, lv, M, 24 + ceil_log2(nl + 1), "lg");
    GW_LAUNCH(k_large_check<uint32_t>, grid_for(M), kThreads, 0, st, a, lk, lv, M, nl);
    check_launch();
    CK(cudaStreamSynchronize(st));  // keeps off / hi / hw alive until the copies completed
  }
  AccArgs<uint32_t> bk_acc_args(const Cands& cd, const uint32_t* keys, const uint32_t* vals, uint64_t n,
                                uint32_t* li, uint32_t* lws, uint32_t* nl, uint32_t lcap) {
    AccArgs<uint32_t> a;
    memset(&a, 0, sizeof a);
    a.tr = tr;
    a.keys = keys;
    a.vals = vals;
    a.n = n;
    a.aux = nullptr;
    a.stamps = stamps;
    a.arena = w.arena;
    a.defer = 0;
    a.blockobj = 1;
    a.c = cd;
    a.large_i = li;
    a.large_ws = lws;
    a.n_large = nl;
    a.large_cap = lcap;
    a.dup = dup;
    return a;
  }
  // buckets above kBkCap records: the LSD sort by h + k_access over them
  void bucket_spill(const Cands& cd, const uint32_t* spill, uint32_t nsp) {
    std::vector<uint32_t> hs2(2 * (size_t)nsp), off(nsp);
    CK(cudaMemcpyAsync(hs2.data(), spill, sizeof(uint32_t) * 2 * nsp, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    uint64_t tot = 0;
    for (uint32_t k = 0; k < nsp; k++) {
      off[k] = (uint32_t)tot;
      tot += hs2[2 * k + 1];
    }
    uint32_t* soff = C->get<uint32_t>("bsp_off", nsp);
    CK(cudaMemcpyAsync(soff, off.data(), sizeof(uint32_t) * nsp, cudaMemcpyHostToDevice, st));
    uint32_t* keys = C->get<uint32_t>("bsp_k", tot);
    uint32_t* vals2 = C->get<uint32_t>("bsp_v", tot);
    GW_LAUNCH(k_bk_spill_gather, std::min<uint32_t>(nsp, 65535u), kThreads, 0, st, bk_h, bk_v, spill, soff, nsp, keys,
              vals2);
    CK(cudaStreamSynchronize(st));  // off alive until the copy completed
    sort<uint32_t>(keys, vals2, tot, 32, "bsp");
    const uint64_t atile = (uint64_t)kThreads * kAccItemsSmall;
    const uint64_t nt = (tot + atile - 1) / atile;
    uint2* agg = C->get<uint2>("bsp_tagg", nt + 1);
    uint2* car = C->get<uint2>("bsp_carry", nt + 1);
    const unsigned tg = (unsigned)std::min<uint64_t>(std::max<uint64_t>(nt, 1), 148ull * 8);
    GW_LAUNCH((k_acc_tilemax<uint32_t, kAccItemsSmall>), tg, kThreads, 0, st, (const uint32_t*)keys, vals2, tot, agg);
    scan<uint2, OpMax2>(ArrLoad<uint2>{agg}, ArrStore<uint2>{car}, nt, OpMax2(), make_uint2(0, 0), false, "sc_u2");
    const uint32_t lcap = (uint32_t)(tot / kSmallWin + 1);
    uint32_t* li = C->get<uint32_t>("lg2_i", lcap);
    uint32_t* lws = C->get<uint32_t>("lg2_ws", lcap);
    CK(cudaMemsetAsync(scal + SC_NLARGE2, 0, sizeof(uint32_t), st));
    AccArgs<uint32_t> a = bk_acc_args(cd, keys, vals2, tot, li, lws, scal + SC_NLARGE2, lcap);
    a.carry = car;
    a.tile_ctr = zeroed(1);
    acc_setup<uint32_t, kAccItemsSmall, true>();
    const unsigned ag = (unsigned)std::min<uint64_t>(std::max<uint64_t>(nt, 1), 148ull * 16);
    GW_LAUNCH((k_access<uint32_t, kAccItemsSmall, true>), ag, kThreads, sizeof(AccSmem<uint32_t, kAccItemsSmall, true>),
              st, a);
    check_launch();
    uint32_t nl = 0;
    d2h(&nl, scal + SC_NLARGE2);
    if (nl > lcap) throw CudaErr{GW_E_NOMEM, "large-window list overflow (spilled buckets)"};
    if (nl) large_windows(a, nl);
  }
  // the check of the bucketed access pass (candidates as check_pass(false, ...))
  Cands bucket_check_pass() {
    const uint64_t NA = bk_na;
    uint32_t* cnt = scal + SC_NCAND;
    const uint32_t lcap = (uint32_t)(NA / kSmallWin + 1);
    uint32_t* large_i = C->get<uint32_t>("lg_i", lcap);
    uint32_t* large_ws = C->get<uint32_t>("lg_ws", lcap);
    uint32_t* gsorted = C->get<uint32_t>("bk_gsorted", NA);
    const uint32_t NB = 1u << bk_bb;
    const uint32_t spill_cap = NB;
    uint32_t* spill = C->get<uint32_t>("bk_spill", 2ull * spill_cap);
    uint64_t pend_cap = gmode ? P->pend_cap : std::max<uint64_t>(65536, NA / 8);
    Cands cd, pd;
    uint32_t hcnt[2] = {0, 0};
    bk_check_setup();
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_bk_check, kThreads, sizeof(BkSmem)));
    const unsigned grid = (unsigned)std::min<uint64_t>(NB, (uint64_t)std::max(occ, 1) * C->num_sms);
    uint32_t* scratch = C->get<uint32_t>("bk_scratch", (uint64_t)grid * 3 * kBkSubBuf);
    // (an L2 persisting set-aside for the scratch was measured: it starves the
    // scatter passes' write combining in L2, 22 -> 73 ms, and saves little here)
    uint32_t npend = 0;
    for (int attempt = 0; attempt < 2; attempt++) {
      pd = make_cands("bp", pend_cap, scal + SC_NPEND);
      CK(cudaMemsetAsync(scal + SC_NPEND, 0, sizeof(uint32_t), st));
      CK(cudaMemsetAsync(cnt, 0, 2 * sizeof(uint32_t), st));
      CK(cudaMemsetAsync(scal + SC_NSURV, 0, sizeof(uint32_t), st));
      CK(cudaMemsetAsync(scal + SC_NSPILL, 0, sizeof(uint32_t), st));
      dup.ev = nullptr;
      dup.n = scal + SC_NDUP;
      dup.cap = 0;
      if (hs.n_long == 0 && !xs_recv.h) {  // (exchange mode: the source ranks run the record check)
        dup.cap = (uint32_t)std::max<uint64_t>(4096, NA / 64);
        dup.ev = C->get<uint32_t>("dup_ev", dup.cap);
      }
      CK(cudaMemsetAsync(scal + SC_NDUP, 0, 2 * sizeof(uint32_t), st));
      BkCheckArgs ba;
      memset(&ba, 0, sizeof ba);
      ba.tr = tr;
      ba.h = bk_h;
      ba.v = bk_v;
      ba.t = bk_t;
      ba.bstart = bk_start;
      ba.NB = NB;
      ba.kb = bk_kb;
      ba.stamps = stamps;
      ba.arena = w.arena;
      ba.pend = pd;
      ba.c = pd;
      ba.dup = dup;
      ba.large_i = large_i;
      ba.large_ws = large_ws;
      ba.n_large = cnt + 1;
      ba.large_cap = lcap;
      ba.gsorted = gsorted;
      ba.scratch = scratch;
      ba.spill = spill;
      ba.n_spill = scal + SC_NSPILL;
      ba.spill_cap = spill_cap;
      ba.xmode = xs_recv.h ? 1 : 0;
      GW_LAUNCH(k_bk_check, grid, kThreads, sizeof(BkSmem), st, ba);
      check_launch();
      if (gmode) break;
      d2h(&npend, scal + SC_NPEND);
      if (npend <= pd.cap) break;
      pend_cap = (uint64_t)npend + 1024;
      CK(cudaMemsetAsync(w.err, 0, sizeof(uint32_t), st));
    }
    obs_npend = npend;
    // the final candidates: the resolved structural ones, spilled buckets,
    // same-instruction pairs, large windows
    uint64_t cand_cap = gmode ? P->cand_cap : std::max<uint64_t>(65536, (uint64_t)npend + NA / 64);
    for (int attempt = 0; attempt < 2; attempt++) {
      cd = make_cands("c", cand_cap, cnt);
      CK(cudaMemsetAsync(cnt, 0, sizeof(uint32_t), st));
      const uint64_t rg = gmode ? pd.cap : npend;
      if (rg) GW_LAUNCH(k_bk_resolve, grid_for(rg), kThreads, 0, st, pd, tr, stamps, w.arena, cd, bk_xi);
      if (gmode) {
        same_instr_pass(cd);
        GW_LAUNCH(k_guard, 1, 1, 0, st, cnt, cd.cap, cnt + 1, scal + SC_NDUP, dup.cap, scal + SC_ABORT,
                  (const uint32_t*)(scal + SC_NSPILL));
        GW_LAUNCH(k_guard, 1, 1, 0, st, scal + SC_NPEND, pd.cap, scal + SC_NLARGE2, scal + SC_NDUP, dup.cap,
                  scal + SC_ABORT, (const uint32_t*)nullptr);
        break;
      }
      uint32_t nsp = 0;
      d2h(&nsp, scal + SC_NSPILL);
      obs_nspill = nsp;
      if (xs_recv.h) {  // exchange mode: no trace here for the spill / large-window / record passes
        uint32_t err = 0;
        d2h(&err, scal + SC_ERR);
        if (getenv("GW_XS_DEBUG")) {
          uint32_t nl = 0;
          d2h(&nl, cnt + 1);
          fprintf(stderr, "[gw xs] records %llu buckets %u kb %d spill %u large %u err 0x%x pend %u\n",
                  (unsigned long long)NA, NB, bk_kb, nsp, nl, err, npend);
        }
        if (err & ERR_XMODE)
          throw CudaErr{GW_E_UNSUPPORTED, "exchange mode: hot locations or large reader windows (use the "
                                          "replicated shard mode)"};
        d2h(hcnt, cnt, 2);
        if (hcnt[0] <= cd.cap) break;
        cand_cap = (uint64_t)hcnt[0] + 1024;
        CK(cudaMemsetAsync(w.err, 0, sizeof(uint32_t), st));
        continue;
      }
      if (nsp) bucket_spill(cd, spill, nsp);
      same_instr_pass(cd);
      d2h(hcnt, cnt, 2);
      if (hcnt[1] > lcap) throw CudaErr{GW_E_NOMEM, "large-window list overflow"};
      if (hcnt[1] > 0) {
        AccArgs<uint32_t> a = bk_acc_args(cd, nullptr, gsorted, NA, large_i, large_ws, cnt + 1, lcap);
        large_windows(a, hcnt[1]);
        d2h(hcnt, cnt, 1);
      }
      if (hcnt[0] <= cd.cap) break;
      cand_cap = (uint64_t)hcnt[0] + 1024;
      CK(cudaMemsetAsync(w.err, 0, sizeof(uint32_t), st));
    }
    obs_ncand = hcnt[0];
    obs_nlarge = hcnt[1];
    obs_cand_cap = cand_cap;
    C->stats.n_candidates = hcnt[0];
    return cd;
  }

  // ------------------------------------- validate_trace / infer_locks (validate.cuh)
  // (event, code, a, b) of validate_trace in report order, on the host
  void validate_run(std::vector<uint32_t>& oe, std::vector<uint32_t>& oc, std::vector<uint64_t>& oa,
                    std::vector<uint64_t>& ob) {
    const uint64_t N = tr.n;
    zero_blk = C->get<uint32_t>("zero_blk", kZeroWords);
    zero_next = 0;
    CK(cudaMemsetAsync(zero_blk, 0, sizeof(uint32_t) * kZeroWords, st));
    reserve_epochs();
    uint32_t* endpos = C->get<uint32_t>("v_end", tr.T);
    CK(cudaMemsetAsync(endpos, 0xFF, sizeof(uint32_t) * tr.T, st));
    GW_LAUNCH(k_val_endpos, grid_for(N), kThreads, 0, st, tr, endpos);
    uint32_t* flag = C->get<uint32_t>("v_flag", N);
    uint32_t* off = C->get<uint32_t>("v_off", N);
    uint32_t* cnt = C->get<uint32_t>("v_cnt", 2);
    uint64_t cap = std::max<uint64_t>(4096, N / 8);
    VOut o;
    uint32_t nd = 0;
    for (int attempt = 0; attempt < 2; attempt++) {
      o.okey = C->get<unsigned long long>("v_okey", cap);
      o.code = C->get<uint32_t>("v_code", cap);
      o.a = C->get<unsigned long long>("v_a", cap);
      o.b = C->get<unsigned long long>("v_b", cap);
      o.n = cnt;
      o.cap = (uint32_t)cap;
      CK(cudaMemsetAsync(cnt, 0, sizeof(uint32_t), st));
      GW_LAUNCH(k_val_events, grid_for(N), kThreads, 0, st, tr, endpos, o, flag);
      scan<uint32_t, OpSum>(ArrLoad<uint32_t>{flag}, ArrStore<uint32_t>{off}, N, OpSum(), 0u, false, "sc_u32");
      uint32_t hv[2];
      CK(cudaMemcpyAsync(hv, off + (N - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(hv + 1, flag + (N - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      const uint64_t nl = (uint64_t)hv[0] + hv[1];
      if (nl) {
        uint32_t* ktid = C->get<uint32_t>("v_ktid", nl);
        uint32_t* kev = C->get<uint32_t>("v_kev", nl);
        GW_LAUNCH(k_val_compact, grid_for(N), kThreads, 0, st, tr, flag, off, ktid, kev);
        sort<uint32_t>(ktid, kev, nl, ceil_log2(tr.T), "vlk");
        unsigned long long* stk = C->get<unsigned long long>("v_stack", nl);
        GW_LAUNCH(k_val_locks, grid_for(nl), kThreads, 0, st, tr, ktid, kev, (uint32_t)nl, stk, o);
      }
      d2h(&nd, cnt);
      if (nd <= cap) break;
      cap = nd;
    }
    oe.resize(nd); oc.resize(nd); oa.resize(nd); ob.resize(nd);
    if (!nd) return;
    // report order: (event, lane)
    unsigned long long* sk = o.okey;
    uint32_t* sv = C->get<uint32_t>("v_sv", nd);
    GW_LAUNCH(k_iota, grid_for(nd), kThreads, 0, st, sv, (uint32_t)nd);
    sort<unsigned long long>(sk, sv, nd, 8 + ceil_log2(N + 1), "vd");
    std::vector<unsigned long long> hk(nd), ha(nd), hb(nd);
    std::vector<uint32_t> hi(nd), hc(nd);
    CK(cudaMemcpyAsync(hk.data(), sk, 8 * nd, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hi.data(), sv, 4 * nd, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hc.data(), o.code, 4 * nd, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(ha.data(), o.a, 8 * nd, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hb.data(), o.b, 8 * nd, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (uint32_t k = 0; k < nd; k++) {
      const uint32_t j = hi[k];
      oe[k] = (uint32_t)(hk[k] >> 8);
      oc[k] = hc[j];
      oa[k] = ha[j];
      ob[k] = hb[j];
    }
  }
  // infer_locks: the rewritten trace (host arrays) and the uninferred releases
  void infer_run(std::vector<unsigned long long>& ok, std::vector<uint32_t>& oto, std::vector<uint32_t>& oin,
                 std::vector<uint32_t>& dev_, std::vector<unsigned long long>& dlock, std::vector<uint32_t>& dtid) {
    const uint64_t N = tr.n;
    zero_blk = C->get<uint32_t>("zero_blk", kZeroWords);
    zero_next = 0;
    CK(cudaMemsetAsync(zero_blk, 0, sizeof(uint32_t) * kZeroWords, st));
    reserve_epochs();
    uint32_t* flag = C->get<uint32_t>("v_flag", N);
    uint32_t* off = C->get<uint32_t>("v_off", N);
    GW_LAUNCH(k_inf_flag, grid_for(N), kThreads, 0, st, tr, flag);
    scan<uint32_t, OpSum>(ArrLoad<uint32_t>{flag}, ArrStore<uint32_t>{off}, N, OpSum(), 0u, false, "sc_u32");
    uint32_t hv[2];
    CK(cudaMemcpyAsync(hv, off + (N - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hv + 1, flag + (N - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const uint64_t nt = (uint64_t)hv[0] + hv[1];
    uint8_t* action = C->get<uint8_t>("i_act", N);
    CK(cudaMemsetAsync(action, 0, N, st));
    uint32_t* cnt = C->get<uint32_t>("v_cnt", 2);
    CK(cudaMemsetAsync(cnt, 0, sizeof(uint32_t), st));
    InfDiag dg;
    dg.cap = (uint32_t)std::max<uint64_t>(1, nt / 2 + 1);  // one per FENCE + atomic write pair at most
    dg.first = C->get<uint32_t>("i_dfirst", dg.cap);
    dg.ev = C->get<uint32_t>("i_dev", dg.cap);
    dg.lock = C->get<unsigned long long>("i_dlock", dg.cap);
    dg.tid = C->get<uint32_t>("i_dtid", dg.cap);
    dg.n = cnt;
    if (nt) {
      uint32_t* ktid = C->get<uint32_t>("v_ktid", nt);
      uint32_t* kev = C->get<uint32_t>("v_kev", nt);
      GW_LAUNCH(k_val_compact, grid_for(N), kThreads, 0, st, tr, flag, off, ktid, kev);
      sort<uint32_t>(ktid, kev, nt, ceil_log2(tr.T), "vlk");
      unsigned long long* held = C->get<unsigned long long>("v_stack", nt);
      GW_LAUNCH(k_inf_walk, grid_for(nt), kThreads, 0, st, tr, ktid, kev, (uint32_t)nt, held, action, dg);
    }
    GW_LAUNCH(k_inf_keep, grid_for(N), kThreads, 0, st, action, N, flag);
    scan<uint32_t, OpSum>(ArrLoad<uint32_t>{flag}, ArrStore<uint32_t>{off}, N, OpSum(), 0u, false, "sc_u32");
    CK(cudaMemcpyAsync(hv, off + (N - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hv + 1, flag + (N - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const uint64_t nk = (uint64_t)hv[0] + hv[1];
    unsigned long long* ko = C->get<unsigned long long>("i_key", nk);
    uint32_t* to_o = C->get<uint32_t>("i_tidop", nk);
    uint32_t* io = C->get<uint32_t>("i_instr", nk);
    GW_LAUNCH(k_inf_emit, grid_for(N), kThreads, 0, st, tr, action, flag, off, ko, to_o, io);
    ok.resize(nk); oto.resize(nk); oin.resize(nk);
    uint32_t nd = 0;
    d2h(&nd, cnt);
    if (nk) {
      CK(cudaMemcpyAsync(ok.data(), ko, 8 * nk, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(oto.data(), to_o, 4 * nk, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(oin.data(), io, 4 * nk, cudaMemcpyDeviceToHost, st));
    }
    std::vector<uint32_t> e(nd), t(nd), f(nd);
    std::vector<unsigned long long> l(nd);
    if (nd) {
      CK(cudaMemcpyAsync(f.data(), dg.first, 4 * nd, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(e.data(), dg.ev, 4 * nd, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(l.data(), dg.lock, 8 * nd, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(t.data(), dg.tid, 4 * nd, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
    std::vector<uint32_t> ord(nd);  // by (thread's first event, event): the reference's order
    for (uint32_t k = 0; k < nd; k++) ord[k] = k;
    std::sort(ord.begin(), ord.end(),
              [&](uint32_t x, uint32_t y) { return f[x] != f[y] ? f[x] < f[y] : e[x] < e[y]; });
    dev_.resize(nd); dlock.resize(nd); dtid.resize(nd);
    for (uint32_t k = 0; k < nd; k++) { dev_[k] = e[ord[k]]; dlock[k] = l[ord[k]]; dtid[k] = t[ord[k]]; }
  }

  // ============ exchange mode: the multi-GPU data plane (shard.py) =============
  // Every rank holds one record-aligned slice of the trace.  xs_prep: the
  // slice's statistics (reduced over the ranks by the host); xs_hard: its
  // barriers and ENDs (all-gathered: every rank runs the small sync pass over
  // the whole trace's hard events); xs_partition: its accesses as
  // (h, global event | W, tidop) records grouped by destination shard = the
  // top bits of h (all-to-all by the host); xs_check: the bucketed pass over
  // this shard's received records + the record (same-instruction) check of
  // the slice.  Candidates carry global event indices.
  BkRecSrc xs_recv{};  // exchange mode: the received records (nullptr h: off)
  int xs_gbits = 0;
  void xs_begin() {
    g_launches = 0;
    zero_blk = C->get<uint32_t>("zero_blk", kZeroWords);
    zero_next = 0;
    scal = C->get<uint32_t>("scalars", SC_COUNT);
    CK(cudaMemsetAsync(zero_blk, 0, sizeof(uint32_t) * kZeroWords, st));
    CK(cudaMemsetAsync(scal, 0, SC_COUNT * sizeof(uint32_t), st));
    reserve_epochs();
    C->d_scal = nullptr;  // no gw_ctx_fetch after an exchange-mode call
    C->have_cands = false;
  }
  Stats xs_prep() {
    xs_begin();
    Stats* dst = C->get<Stats>("stats", 1);
    GW_LAUNCH(k_init_stats, 1, 1, 0, st, dst);
    if (tr.n) GW_LAUNCH(k_prep, grid_for(tr.n), kThreads, 0, st, tr, dst);
    Stats h;
    d2h(&h, dst);
    return h;
  }
  uint64_t xs_hard(uint32_t base, uint32_t* ev, uint32_t* to, uint32_t* in, unsigned long long* key) {
    const uint64_t N = tr.n;
    if (!N) return 0;
    uint32_t* flag = C->get<uint32_t>("x_flag", N);
    uint32_t* off = C->get<uint32_t>("x_off", N);
    GW_LAUNCH(k_xs_hard_flag, grid_for(N), kThreads, 0, st, tr, flag);
    scan<uint32_t, OpSum>(ArrLoad<uint32_t>{flag}, ArrStore<uint32_t>{off}, N, OpSum(), 0u, false, "sc_u32");
    GW_LAUNCH(k_xs_hard_emit, grid_for(N), kThreads, 0, st, tr, flag, off, base, ev, to, in, key);
    uint32_t hv[2];
    CK(cudaMemcpyAsync(hv, off + (N - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hv + 1, flag + (N - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return (uint64_t)hv[0] + hv[1];
  }
  void xs_partition(const Stats& g, int gbits, uint32_t base, uint32_t* oh, uint32_t* ov, uint32_t* ot,
                    uint64_t* counts) {
    xs_begin();
    kr = key_runs(g.n_acc ? g.key_or ^ g.key_and : 0ull);
    if (kr.nbits > 32) throw CudaErr{GW_E_UNSUPPORTED, "exchange mode: location keys wider than 32 bits"};
    const uint32_t G = 1u << gbits;
    std::vector<uint32_t> start(G + 1, 0);
    Stats* dst = C->get<Stats>("stats", 1);  // this slice's access count
    GW_LAUNCH(k_init_stats, 1, 1, 0, st, dst);
    if (tr.n) GW_LAUNCH(k_prep, grid_for(tr.n), kThreads, 0, st, tr, dst);
    Stats loc;
    d2h(&loc, dst);
    if (tr.n && loc.n_acc) {
      BkTraceSrc ts{tr, kr, base};
      bk_pass(ts, tr.n, gbits, 32 - gbits, oh, ov, ot);
      // digit starts: the scanned counts at super-tile 0 of every digit
      const int ST = gbits > 7 ? 1 << (gbits - 7) : 1;
      const uint64_t nst = (lb_tiles(tr.n) + ST - 1) / ST;
      uint32_t* cnts = C->get<uint32_t>(std::string("bk_counts") + sfx, nst * G);
      for (uint32_t d = 0; d < G; d++)
        CK(cudaMemcpyAsync(&start[d], cnts + (uint64_t)d * nst, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    }
    start[G] = (uint32_t)loc.n_acc;
    for (uint32_t d = 0; d < G; d++) counts[d] = start[d + 1] - start[d];
  }
  // candidates of this shard (global event indices) in the "c" list, and
  // the slice's same-instruction pairs appended (offset by base)
  uint64_t xs_check(const Stats& g, int gbits, uint32_t base, BkRecSrc recv, const uint32_t* hev,
                    const uint32_t* hto, const uint32_t* hin, const unsigned long long* hkey, uint64_t nhard,
                    uint64_t n_total) {
    xs_begin();
    const DevTrace slice = tr;
    // 1. the sync pass over the whole trace's hard events (a mini trace)
    DevTrace mt = slice;
    mt.key = hkey;
    mt.tidop = hto;
    mt.instr = hin;
    mt.n = nhard;
    tr = mt;
    Stats* dst = C->get<Stats>("stats", 1);
    GW_LAUNCH(k_init_stats, 1, 1, 0, st, dst);
    if (nhard) GW_LAUNCH(k_prep, grid_for(nhard), kThreads, 0, st, tr, dst);
    d2h(&hs, dst);
    hs.n_acc = g.n_acc;
    hs.key_or = g.key_or;
    hs.key_and = g.key_and;
    hs.n_long = g.n_long;
    has_locks = false;
    budget_n = n_total;
    plan_sync_pass();
    if (!snap_mode && !wsnap_mode)
      throw CudaErr{GW_E_UNSUPPORTED, "exchange mode: the sync pass needs the snapshot walker"};
    walker_phase();
    if (nhard) {  // snapshot lists index the mini trace: map them to global events
      const uint64_t nl = snap_mode ? n_hard : n_hard_w;
      uint32_t* gev = C->get<uint32_t>("x_hev", nl + 1);
      GW_LAUNCH(k_xs_remap, grid_for(nl), kThreads, 0, st, stamps.hard_ev, nl, hev, gev);
      stamps.hard_ev = gev;
    }
    tr = slice;
    // 2. the bucketed pass over the received records
    kr = key_runs(g.n_acc ? g.key_or ^ g.key_and : 0ull);
    bk_xi.on = 1;
    bk_xi.kr = kr;
    bk_xi.base = g.key_and & ~(g.key_or ^ g.key_and);
    xs_gbits = gbits;
    xs_recv = recv;
    bk_mode = true;
    uint64_t nc = 0;
    if (recv.cnt) {
      bucket_sort();
      Cands cd = bucket_check_pass();
      nc = std::min<uint64_t>(obs_ncand, cd.cap);
    }
    xs_recv = BkRecSrc{};
    // 3. the record check (_same_instruction_check) of this rank's slice
    uint32_t* ncs = scal + SC_NQ;
    uint64_t cap = std::max<uint64_t>(4096, tr.n / 16);
    Cands si;
    uint32_t hsi = 0;
    for (int attempt = 0; attempt < 2 && tr.n; attempt++) {
      si = make_cands("xsi", cap, ncs);
      CK(cudaMemsetAsync(ncs, 0, sizeof(uint32_t), st));
      ShardArgs sa{};
      sa.G = 1;
      GW_LAUNCH(k_same_instr, grid_for(tr.n), kThreads, 0, st, tr, si, sa, 0);
      d2h(&hsi, ncs);
      if (hsi <= si.cap) break;
      cap = hsi + 1024;
      CK(cudaMemsetAsync(scal + SC_ERR, 0, sizeof(uint32_t), st));
    }
    xs_nc = nc;
    xs_nsi = hsi;
    xs_si = si;
    return nc + hsi;
  }
  uint64_t xs_nc = 0, xs_nsi = 0;
  Cands xs_si{};

  Cands make_cands(const std::string& tag, uint64_t cap, uint32_t* cnt) {
    Cands c;
    c.okey = C->get<unsigned long long>(tag + "_okey", cap);
    c.loc = C->get<unsigned long long>(tag + "_loc", cap);
    c.prior = C->get<uint32_t>(tag + "_prior", cap);
    c.cur = C->get<uint32_t>(tag + "_cur", cap);
    c.kind = C->get<uint32_t>(tag + "_kind", cap);
    c.n = cnt;
    c.cap = (uint32_t)std::min<uint64_t>(cap, 0xFFFFFFF0ull);
    c.err = scal + SC_ERR;
    return c;
  }

  // ------------------------------------------------------------ check pass
  // Candidates of the write check and the reader windows (+ the same-
  // instruction pairs when !defer).  defer: emit every structural candidate
  // (u != t, !cover) and leave the clock comparison to the walker's queries.
  // Counts at scal[slot] (candidates) and scal[slot + 1] (large windows).
  Cands check_pass(bool defer, const char* tag, int slot) {
    const uint64_t NA = na_sorted;
    uint32_t* cnt = scal + slot;
    uint32_t* large_i = C->get<uint32_t>("lg_i", NA / kSmallWin + 1);
    uint32_t* large_ws = C->get<uint32_t>("lg_ws", NA / kSmallWin + 1);
    uint64_t cand_cap = gmode ? P->cand_cap : std::max<uint64_t>(65536, NA / 4);
    Cands cd;
    AccArgs<uint32_t> a32;
    AccArgs<unsigned long long> a64;
    uint32_t hcnt[2] = {0, 0};
    for (int attempt = 0; attempt < 2; attempt++) {
      cd = make_cands(tag, cand_cap, cnt);
      CK(cudaMemsetAsync(cnt, 0, 2 * sizeof(uint32_t), st));
      if (!defer) CK(cudaMemsetAsync(scal + SC_NSURV, 0, sizeof(uint32_t), st));
      // same-record pairs on one location, flagged by the access check (no record > 32 events)
      dup.ev = nullptr;
      dup.n = scal + SC_NDUP;
      dup.cap = 0;
      if (hs.n_long == 0) {
        dup.cap = (uint32_t)std::max<uint64_t>(4096, NA / 64);
        dup.ev = C->get<uint32_t>("dup_ev", dup.cap);
      }
      CK(cudaMemsetAsync(scal + SC_NDUP, 0, 2 * sizeof(uint32_t), st));
      auto fill = [&](auto& aa, const auto* kp) {
        memset(&aa, 0, sizeof aa);
        aa.tr = tr;
        aa.keys = kp;
        aa.vals = vals;
        aa.n = NA;
        aa.carry = carry;
        aa.lb = acc_lb;
        aa.tile_ctr = zeroed(1);
        aa.aux = aux;
        aa.stamps = stamps;
        aa.arena = defer ? nullptr : w.arena;
        aa.defer = defer ? 1 : 0;
        aa.blockobj = (!defer && !has_locks) ? 1 : 0;
        aa.c = cd;
        aa.large_i = large_i;
        aa.large_ws = large_ws;
        aa.n_large = cnt + 1;
        aa.large_cap = (uint32_t)(NA / kSmallWin + 1);
        aa.dup = dup;
      };
      const uint64_t atile = (uint64_t)kThreads * acc_items;
      const unsigned ag = (unsigned)std::min<uint64_t>(std::max<uint64_t>((NA + atile - 1) / atile, 1), 148ull * 16);
      if (acc_lb) CK(cudaMemsetAsync(acc_lb, 0, sizeof(unsigned long long) * acc_lb_n, st));
      if (wide) {
        fill(a64, (const unsigned long long*)skeys);
        if (aux) {
          acc_setup<unsigned long long, kAccItemsSmall>();
          GW_LAUNCH((k_access<unsigned long long, kAccItemsSmall>), ag, kThreads,
                    sizeof(AccSmem<unsigned long long, kAccItemsSmall>), st, a64);
        } else {
          acc_setup<unsigned long long, kAccItemsSmall, true>();
          GW_LAUNCH((k_access<unsigned long long, kAccItemsSmall, true>), ag, kThreads,
                    sizeof(AccSmem<unsigned long long, kAccItemsSmall, true>), st, a64);
        }
      } else if (acc_items == kAccItemsLarge) {
        fill(a32, (const uint32_t*)skeys);
        if (aux) {
          acc_setup<uint32_t, kAccItemsLarge>();
          GW_LAUNCH((k_access<uint32_t, kAccItemsLarge>), ag, kThreads, sizeof(AccSmem<uint32_t, kAccItemsLarge>), st,
                    a32);
        } else {
          acc_setup<uint32_t, kAccItemsLarge, true>();
          GW_LAUNCH((k_access<uint32_t, kAccItemsLarge, true>), ag, kThreads,
                    sizeof(AccSmem<uint32_t, kAccItemsLarge, true>), st, a32);
        }
      } else {
        fill(a32, (const uint32_t*)skeys);
        if (aux) {
          acc_setup<uint32_t, kAccItemsSmall>();
          GW_LAUNCH((k_access<uint32_t, kAccItemsSmall>), ag, kThreads, sizeof(AccSmem<uint32_t, kAccItemsSmall>), st,
                    a32);
        } else {
          acc_setup<uint32_t, kAccItemsSmall, true>();
          GW_LAUNCH((k_access<uint32_t, kAccItemsSmall, true>), ag, kThreads,
                    sizeof(AccSmem<uint32_t, kAccItemsSmall, true>), st, a32);
        }
      }
      check_launch();
      if (gmode) {
        if (!defer) same_instr_pass(cd);
        GW_LAUNCH(k_guard, 1, 1, 0, st, cnt, cd.cap, cnt + 1, scal + SC_NDUP, dup.cap, scal + SC_ABORT);
        break;
      }
      if (!defer) same_instr_pass(cd);
      d2h(hcnt, cnt, 2);
      if (hcnt[1] > 0) {
        // large reader windows (> kSmallWin reads between two writes)
        const uint32_t nl = hcnt[1];
        uint32_t* sizes = C->get<uint32_t>("lg_sz", nl + 1);
        std::vector<uint32_t> hi(nl), hw(nl);
        CK(cudaMemcpyAsync(hi.data(), large_i, sizeof(uint32_t) * nl, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(hw.data(), large_ws, sizeof(uint32_t) * nl, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        std::vector<uint32_t> off(nl);
        uint64_t M = 0;
        for (uint32_t k = 0; k < nl; k++) {
          off[k] = (uint32_t)M;
          M += hi[k] - hw[k];
        }
        CK(cudaMemcpyAsync(sizes, off.data(), sizeof(uint32_t) * nl, cudaMemcpyHostToDevice, st));
        unsigned long long* lk = C->get<unsigned long long>("lg_k", M);
        uint32_t* lv = C->get<uint32_t>("lg_v", M);
        GW_LAUNCH(k_large_fill, std::min<uint32_t>(nl, 65535u), kThreads, 0, st, large_i, large_ws, sizes, nl, vals,
                  tr.tidop, lk, lv);
        sort<unsigned long long>(lk, lv, M, 24 + ceil_log2(nl + 1), "lg");
        if (!wide) GW_LAUNCH(k_large_check<uint32_t>, grid_for(M), kThreads, 0, st, a32, lk, lv, M, nl);
        else GW_LAUNCH(k_large_check<unsigned long long>, grid_for(M), kThreads, 0, st, a64, lk, lv, M, nl);
        check_launch();
        d2h(hcnt, cnt, 1);  // also keeps off / hi / hw alive until the copies completed
      }
      if (hcnt[0] <= cd.cap) break;
      cand_cap = (uint64_t)hcnt[0] + 1024;
      CK(cudaMemsetAsync(w.err, 0, sizeof(uint32_t), st));
    }
    if (defer) {
      obs_nq = hcnt[0];
    } else {
      obs_ncand = hcnt[0];
      obs_nlarge = hcnt[1];
      obs_cand_cap = cand_cap;
      C->stats.n_candidates = hcnt[0];
    }
    return cd;
  }

  // --------------------------------------- lock mode: Q set and queries
  void query_setup(const Cands& cq, uint64_t nq) {
    const uint64_t N = tr.n;
    const uint32_t T = tr.T;
    uint32_t* qflag = C->get<uint32_t>("q_flag", (uint64_t)T + 1);
    uint32_t* qoff = C->get<uint32_t>("q_off", (uint64_t)T + 1);
    CK(cudaMemsetAsync(qflag, 0, sizeof(uint32_t) * ((uint64_t)T + 1), st));
    if (!hb_mode) GW_LAUNCH(k_q_mark_acq, grid_for(N), kThreads, 0, st, tr, w.lflags, qflag);  // drain-test owners
    uint32_t* qk = C->get<uint32_t>("q_sk", nq + 1);
    uint32_t* qi = C->get<uint32_t>("q_sv", nq + 1);
    if (nq) GW_LAUNCH(k_q_mark_cands, grid_for(nq), kThreads, 0, st, cq, tr.tidop, qflag, (uint8_t*)w.lflags, qk, qi);
    scan<uint32_t, OpSum>(ArrLoad<uint32_t>{qflag}, ArrStore<uint32_t>{qoff}, (uint64_t)T + 1, OpSum(), 0u, false,
                          "sc_u32");
    uint32_t Q = 0;
    d2h(&Q, qoff + T);
    sort<uint32_t>(qk, qi, nq, ceil_log2(N), "qs");
    w.qoff = qoff;
    w.Q = Q;
    w.q_cur = qk;
    w.q_idx = qi;
    w.nq = nq;
    w.c_prior = cq.prior;
    w.qv = C->get<uint32_t>("q_v", nq + 1);
    C->stats.n_candidates = nq;
  }

  // ------------------------------------------------- lock mode: resolve
  Cands resolve_pass(const Cands& cq, uint64_t nq) {
    const uint64_t N = tr.n;
    uint32_t* cnt = scal + SC_NCAND;
    uint64_t cap = std::max<uint64_t>(65536, nq + N / 8);
    Cands cd;
    uint32_t hc = 0;
    for (int attempt = 0; attempt < 2; attempt++) {
      cd = make_cands("c", cap, cnt);
      CK(cudaMemsetAsync(cnt, 0, 3 * sizeof(uint32_t), st));
      if (nq) GW_LAUNCH(k_resolve, grid_for(nq), kThreads, 0, st, cq, w.qv, w.time, cd);
      same_instr_pass(cd);
      check_launch();
      d2h(&hc, cnt);
      if (hc <= cd.cap) break;
      cap = (uint64_t)hc + 1024;
      CK(cudaMemsetAsync(w.err, 0, sizeof(uint32_t), st));
    }
    obs_ncand = hc;
    return cd;
  }

  // ----------------------------------------------------------- walker
  void walker_phase() {
    const uint64_t N = tr.n;
    const uint32_t T = tr.T;
    const bool lockq = w.qoff != nullptr;
    const uint32_t VL = lockq ? w.Q : T;  // clock vector length
    if (!lockq) {
      arena_units = hs.n_bar * (uint64_t)((tr.BS + OBJ_HDR + 15) >> OBJ_USHIFT) + 4;
    } else {
      // fixed-size slots; live objects: records (pinned hb clocks), instance
      // and cs clocks, thread states (<= 2 per thread) + per-CTA slack
      w.slot_units = (VL + OBJ_HDR + 15) >> OBJ_USHIFT;
      const uint64_t nstk = lock_warp ? (uint64_t)G * kLW : G;
      w.warp_stacks = lock_warp ? 1u : 0u;
      w.fcap = lock_warp ? 256 : 1024;
      w.fstack = C->get<uint32_t>("f_stack", nstk * w.fcap);
      w.ftop = C->get<uint32_t>("f_top", nstk);
      CK(cudaMemsetAsync(w.ftop, 0, sizeof(uint32_t) * nstk, st));
      const uint64_t slots = 3 * hs.n_rel + (uint64_t)n_incs * maxd + 2ull * T + 4ull * G + 64;
      size_t free_b = 0, total_b = 0;
      CK(cudaMemGetInfo(&free_b, &total_b));
      {  // the arena buffer of an earlier analysis is reused: count it as free
        auto it = C->bufs.find("arena");
        if (it != C->bufs.end()) free_b += it->second.cap;
      }
      const uint64_t slot_bytes = (uint64_t)w.slot_units << (OBJ_USHIFT + 2);
      const uint64_t cap_slots = (uint64_t)(free_b * 0.6) / slot_bytes;
      if (getenv("GW_DEBUG_MEM")) {
        fprintf(stderr, "[gw] lock mode: Q=%u slot=%llu B, bound %llu slots, free %.1f GB, cap %llu slots\n", VL,
                (unsigned long long)slot_bytes, (unsigned long long)slots, free_b / 1e9, (unsigned long long)cap_slots);
        for (auto& kv : C->bufs)
          if (kv.second.cap > (64u << 20)) fprintf(stderr, "[gw]   %-12s %.2f GB\n", kv.first.c_str(), kv.second.cap / 1e9);
      }
      arena_units = std::min<uint64_t>(std::min(slots, cap_slots) * w.slot_units, 0xFFFFFFF0ull);
    }
    C->stats.arena_words = arena_units << OBJ_USHIFT;
    w.arena = C->get<uint32_t>("arena", arena_units << OBJ_USHIFT);
    w.arena_cap = arena_units;
    w.arena_top = C->get<unsigned long long>("arena_top", 1);
    CK(cudaMemsetAsync(w.arena_top, 0, sizeof(unsigned long long), st));
    w.time = C->get<uint32_t>("time", N);
    w.vobj = lockq ? nullptr : C->get<uint32_t>("vobj", N);
    w.local = C->get<uint32_t>("st_local", T);
    w.pobj = C->get<uint32_t>("st_pobj", T);
    w.pdiag = C->get<uint32_t>("st_pdiag", T);
    w.nend = C->get<uint32_t>("st_nend", T);
    w.exited = C->get<uint32_t>("st_exited", T);
    w.rec_top = scal + SC_REC;
    w.log_top = scal + SC_LOG;
    w.diag_top = scal + SC_DIAG;
    w.maxd = maxd;
    uint64_t diag_cap = hs.n_acq + hs.n_rel + hs.n_end * (uint64_t)maxd + 16;
    w.diags = C->get<Diag>("diags", diag_cap);
    w.diag_cap = (uint32_t)diag_cap;
    if (has_locks) {
      w.hobj = C->get<uint32_t>("st_hobj", T);
      w.depth = C->get<uint32_t>("st_depth", T);
      w.loghead = C->get<uint32_t>("st_loghead", T);
      w.frames = C->get<Frame>("frames", (uint64_t)T * maxd);
      uint64_t icap = pow2_at_least(2 * hs.n_rel + 2);
      uint64_t ccap = pow2_at_least(2 * (uint64_t)n_incs * maxd + 2);
      w.curs = C->get<CurEnt>("t_cur", lcap);
      w.cur_mask = (uint32_t)(lcap - 1);
      w.insts = C->get<InstEnt>("t_inst", icap);
      w.inst_mask = (uint32_t)(icap - 1);
      w.cs = C->get<CsEnt>("t_cs", ccap);
      w.cs_mask = (uint32_t)(ccap - 1);
      CK(cudaMemsetAsync(w.curs, 0, sizeof(CurEnt) * lcap, st));
      CK(cudaMemsetAsync(w.insts, 0, sizeof(InstEnt) * icap, st));
      CK(cudaMemsetAsync(w.cs, 0, sizeof(CsEnt) * ccap, st));
      w.recs = C->get<Rec>("recs", hs.n_acq + 1);
      w.rec_cap = (uint32_t)(hs.n_acq + 1);
      w.logs = C->get<LogEnt>("logs", (uint64_t)n_incs + 1);
      w.log_cap = n_incs + 1;
    }
    if (has_locks || tr.BS > (uint32_t)kAccSmem) w.scratch = C->get<uint32_t>("scratch", (uint64_t)G * 3 * VL);
    GW_LAUNCH(k_state_init, grid_for(T), kThreads, 0, st, w);
    if (snap_mode) {
      SnapArgs sa;
      uint32_t* hev = C->get<uint32_t>("hd_ev", n_hard + 1);
      uint32_t* hbeg = C->get<uint32_t>("hd_beg", tr.B);
      uint32_t* hend = C->get<uint32_t>("hd_end", tr.B);
      uint32_t* hcnt = C->get<uint32_t>("hd_cnt", tr.B);
      if (hard_forked) {
        CK(cudaStreamWaitEvent(st, C->ev_hard, 0));  // built on the third branch (fork_hard)
        hard_joined = true;
      } else if (hard_small_ok(n_hard)) {
        // few hard events: order them and delimit the blocks in one launch
        CK(cudaMemsetAsync(hcnt, 0, sizeof(uint32_t) * tr.B, st));
        obs_hard_small = true;
        hard_small_list(n_hard, hev, hcnt, hbeg, hend);
      } else {
        if (!hard_ingested) CK(cudaMemsetAsync(hcnt, 0, sizeof(uint32_t) * tr.B, st));
        if (n_hard) {
          unsigned long long* hkey = C->get<unsigned long long>("hd_key", n_hard + 1);
          uint32_t* hdummy = C->get<uint32_t>("hd_v", n_hard + 1);
          if (!hard_ingested)
            GW_LAUNCH(k_hard_append, grid_for(N), kThreads, 0, st, tr, hkey, hcnt, zeroed(1), scal + SC_ABORT);
          sort<unsigned long long>(hkey, hdummy, n_hard, 32 + ceil_log2(tr.B), "hd", true);
          GW_LAUNCH(k_hard_unpack, grid_for(n_hard), kThreads, 0, st, hkey, n_hard, hev);
        }
        scan<uint32_t, OpSum>(ArrLoad<uint32_t>{hcnt}, HardSegStore{hcnt, hbeg, hend}, tr.B, OpSum(), 0u, false,
                              "sc_u32");
      }
      sa.hard_ev = hev;
      sa.hb_beg = hbeg;
      sa.hb_end = hend;
      sa.snap = C->get<uint2>("snap", snap_entries);
      GW_LAUNCH(k_walker_snap, std::min<uint32_t>(tr.B, (uint32_t)gmax), kThreads, 0, st, w, sa);
      // no per-access stamp pass: the check looks stamps up in the snapshots
      stamps.time = nullptr;
      stamps.vobj = nullptr;
      stamps.hard_ev = sa.hard_ev;
      stamps.hb_beg = sa.hb_beg;
      stamps.hb_end = sa.hb_end;
      stamps.snap = sa.snap;
      stamps.BS = tr.BS;
      C->stats.walker_ctas = std::min<uint32_t>(tr.B, (uint32_t)gmax);
    } else if (wsnap_mode) {
      SnapArgs sa;
      const uint64_t ng = (uint64_t)tr.B * kWSnapWarps;
      uint32_t* hev = C->get<uint32_t>("hd_ev", n_hard_w + 1);
      uint32_t* hbeg = C->get<uint32_t>("hd_beg", ng);
      uint32_t* hend = C->get<uint32_t>("hd_end", ng);
      uint32_t* hcnt = C->get<uint32_t>("hd_cnt", ng);
      CK(cudaMemsetAsync(hcnt, 0, sizeof(uint32_t) * ng, st));
      if (n_hard_w) {
        unsigned long long* hkey = C->get<unsigned long long>("hd_key", n_hard_w + 1);
        uint32_t* hdummy = C->get<uint32_t>("hd_v", n_hard_w + 1);
        GW_LAUNCH(k_hard_append_w, grid_for(N), kThreads, 0, st, tr, hkey, hcnt, zeroed(1), scal + SC_ABORT);
        sort<unsigned long long>(hkey, hdummy, n_hard_w, 32 + ceil_log2(ng), "hd", true);
        GW_LAUNCH(k_hard_unpack, grid_for(n_hard_w), kThreads, 0, st, hkey, n_hard_w, hev);
      }
      scan<uint32_t, OpSum>(ArrLoad<uint32_t>{hcnt}, HardSegStore{hcnt, hbeg, hend}, ng, OpSum(), 0u, false,
                            "sc_u32");
      sa.hard_ev = hev;
      sa.hb_beg = hbeg;
      sa.hb_end = hend;
      sa.snap = C->get<uint2>("snap", snap_entries);
      GW_LAUNCH(k_walker_wsnap, std::min<uint32_t>(tr.B, (uint32_t)gmax), kThreads, 0, st, w, sa);
      stamps.time = nullptr;
      stamps.vobj = nullptr;
      stamps.hard_ev = sa.hard_ev;
      stamps.hb_beg = sa.hb_beg;
      stamps.hb_end = sa.hb_end;
      stamps.snap = sa.snap;
      stamps.BS = tr.BS;
      stamps.warp_mode = 1;
      stamps.L = tr.L;
      C->stats.walker_ctas = std::min<uint32_t>(tr.B, (uint32_t)gmax);
    } else if (lock_warp) {
      launch_lock_warp();
    } else {
      stamps.time = w.time;
      stamps.vobj = w.vobj;
      stamps.BS = tr.BS;
      const bool prof = getenv("GW_PROF_WALKER") != nullptr;
      if (prof) {
        w.prof = C->get<unsigned long long>("prof", (uint64_t)G * 8);
        CK(cudaMemsetAsync(w.prof, 0, sizeof(unsigned long long) * G * 8, st));
      }
      GW_LAUNCH(k_walker, G, kThreads, 0, st, w);
      if (prof) {
        std::vector<unsigned long long> hp((size_t)G * 8);
        d2h(hp.data(), w.prof, hp.size());
        double sum[8] = {0}, mx[8] = {0};
        for (uint32_t g = 0; g < G; g++)
          for (int k = 0; k < 8; k++) { sum[k] += hp[g * 8 + k]; mx[k] = std::max(mx[k], (double)hp[g * 8 + k]); }
        const char* nm[8] = {"stamp", "barrier", "ticket", "acquire", "release", "incs", "-", "lockev"};
        fprintf(stderr, "[gw] walker G=%u Q=%u per-CTA avg / max ms:", G, w.Q);
        for (int k = 0; k < 6; k++) fprintf(stderr, " %s %.2f/%.2f", nm[k], sum[k] / G / 1e6, mx[k] / 1e6);
        fprintf(stderr, "; lock events %.0f\n", sum[7]);
      }
      w.prof = nullptr;
    }
    check_launch();
  }

  // lock warp walker: block barriers per walker CTA, then the walk
  void launch_lock_warp() {
    const uint64_t N = tr.n;
    const uint64_t nbb = hs.n_bar - hs.n_wbar;
    uint32_t* bev = C->get<uint32_t>("bb_ev", nbb + 1);
    uint32_t* bbeg = C->get<uint32_t>("bb_beg", G);
    uint32_t* bend = C->get<uint32_t>("bb_end", G);
    uint32_t* bcnt = C->get<uint32_t>("bb_cnt", G);
    CK(cudaMemsetAsync(bcnt, 0, sizeof(uint32_t) * G, st));
    if (nbb) {
      unsigned long long* bkey = C->get<unsigned long long>("bb_key", nbb + 1);
      uint32_t* bdummy = C->get<uint32_t>("bb_v", nbb + 1);
      GW_LAUNCH(k_bbar_append, grid_for(N), kThreads, 0, st, tr, G, bkey, bcnt, zeroed(1));
      sort<unsigned long long>(bkey, bdummy, nbb, 32 + ceil_log2(G), "bb", true);
      GW_LAUNCH(k_hard_unpack, grid_for(nbb), kThreads, 0, st, bkey, nbb, bev);
    }
    scan<uint32_t, OpSum>(ArrLoad<uint32_t>{bcnt}, HardSegStore{bcnt, bbeg, bend}, G, OpSum(), 0u, false, "sc_u32");
    const bool prof = getenv("GW_PROF_WALKER") != nullptr;
    const uint64_t nw = (uint64_t)G * kLW;
    if (prof) {
      w.prof = C->get<unsigned long long>("prof", nw * 8);
      CK(cudaMemsetAsync(w.prof, 0, sizeof(unsigned long long) * nw * 8, st));
    }
    GW_LAUNCH(k_walker_lw, G, kThreads, 0, st, w, bev, bbeg, bend);
    if (prof) {
      std::vector<unsigned long long> hp(nw * 8);
      d2h(hp.data(), w.prof, hp.size());
      double sum[8] = {0}, mx[8] = {0};
      for (uint64_t x = 0; x < nw; x++)
        for (int k = 0; k < 8; k++) { sum[k] += hp[x * 8 + k]; mx[k] = std::max(mx[k], (double)hp[x * 8 + k]); }
      const char* nm[7] = {"stamp", "warpbar", "blockbar", "ticket", "acquire", "release", "incs"};
      fprintf(stderr, "[gw] lock warp walker G=%u Q=%u per-warp avg / max ms:", G, w.Q);
      for (int k = 0; k < 7; k++) fprintf(stderr, " %s %.2f/%.2f", nm[k], sum[k] / nw / 1e6, mx[k] / 1e6);
      fprintf(stderr, "; lock events %.0f\n", sum[7]);
      w.prof = nullptr;
    }
  }
};

int validate_view(const gw_trace_view* t) {
  if (!t) { gw_set_error("null trace"); return GW_E_ARG; }
  if (t->n_events && (!t->key || !t->tidop || !t->instr)) { gw_set_error("null trace arrays"); return GW_E_ARG; }
  if (!t->cfg.blocks || !t->cfg.warps || !t->cfg.lanes) { gw_set_error("config values must be positive"); return GW_E_ARG; }
  uint64_t T = (uint64_t)t->cfg.blocks * t->cfg.warps * t->cfg.lanes;
  if (T > (uint64_t)GW_TID_MASK + 1) { gw_set_error("more than 2^24 threads"); return GW_E_UNSUPPORTED; }
  if (t->n_events >= (1ull << 31)) { gw_set_error("more than 2^31 events"); return GW_E_UNSUPPORTED; }
  return GW_OK;
}

DevTrace make_dev(const gw_trace_view* t, const unsigned long long* k, const uint32_t* to, const uint32_t* in) {
  DevTrace d;
  d.key = k;
  d.tidop = to;
  d.instr = in;
  d.n = t->n_events;
  d.B = t->cfg.blocks;
  d.W = t->cfg.warps;
  d.L = t->cfg.lanes;
  d.BS = d.W * d.L;
  d.T = d.B * d.BS;
  return d;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return GW_OK;
  } catch (const CudaErr& e) {
    gw_set_error(e.msg);
    return e.code;
  } catch (const std::bad_alloc&) {
    gw_set_error("host allocation failed");
    return GW_E_NOMEM;
  }
}

}  // namespace

extern "C" gw_ctx* gw_ctx_create(int device) {
  gw_ctx* c = new gw_ctx();
  c->device = device;
  if (cudaSetDevice(device) != cudaSuccess) {
    gw_set_error(std::string("cudaSetDevice: ") + cudaGetErrorString(cudaGetLastError()));
    delete c;
    return nullptr;
  }
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) == cudaSuccess && sms > 0) c->num_sms = sms;
  return c;
}

extern "C" void gw_ctx_destroy(gw_ctx* c) {
  if (!c) return;
  c->drop_plan();
  for (auto& kv : c->bufs)
    if (kv.second.p) cudaFree(kv.second.p);
  for (cudaEvent_t e : c->prof_ev) cudaEventDestroy(e);
  for (int i = 0; i < gw_ctx::kEv; i++)
    if (c->ev[i]) cudaEventDestroy(c->ev[i]);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->ev_fork2) cudaEventDestroy(c->ev_fork2);
  if (c->ev_hard) cudaEventDestroy(c->ev_hard);
  if (c->side2) cudaStreamDestroy(c->side2);
  for (cudaEvent_t e : c->chunk_ev) cudaEventDestroy(e);
  if (c->ev_prev) cudaEventDestroy(c->ev_prev);
  if (c->copy_st) cudaStreamDestroy(c->copy_st);
  if (c->hres) cudaFreeHost(c->hres);
  delete c;
}

// Eager analysis, then (lock-free traces without large reader windows) build
// the Plan and capture the graph-mode pipeline for later replays.
static void analyze_impl(gw_ctx* c, const DevTrace& tr, cudaStream_t st, uint32_t inactive, const void* kp,
                         const void* tp, const void* ip, bool eager, uint32_t shard, uint32_t nshard,
                         bool profile = false, bool hb = false) {
  if (nshard > 1) eager = true;  // sharded analyses are not graph-replayed
  if (hb) eager = true;          // the plan cache is for the G-WCP detector
  c->last_hb = hb;
  c->prof_done = false;
  if (profile) {
    eager = true;
    c->prof_arm(4096);
    g_prof = &c->prof;
  }
  struct ProfOff {
    ~ProfOff() { g_prof = nullptr; }
  } prof_off;
  c->last_shard = shard;
  c->last_nshard = nshard;
  Plan& P = c->plan;
  c->last_tr = tr;
  c->last_inactive = inactive;
  c->last_stream = st;
  const bool match = !eager && P.valid && P.N == tr.n && P.B == tr.B && P.W == tr.W && P.L == tr.L && P.key == kp &&
                     P.tidop == tp && P.instr == ip && P.stream == st && P.inactive_opt == inactive;
  if (match) {
    for (int i = 0; i < gw_ctx::kEv; i++)
      if (!c->ev[i]) CK(cudaEventCreate(&c->ev[i]));
    CK(cudaEventRecord(c->ev[0], st));
    CK(cudaGraphLaunch(P.exec, st));
    CK(cudaEventRecord(c->ev[1], st));
    c->last_graph = true;
    c->launches = P.launches;
    c->stats_pending = true;
    c->phases = false;
    return;
  }
  c->drop_plan();
  c->last_graph = false;
  Pipeline p;
  p.C = c;
  p.st = st;
  p.inactive_opt = inactive;
  p.tr = tr;
  p.shard = shard;
  p.nshard = nshard;
  p.hb_mode = hb;
  p.run();
  if (eager || tr.n == 0 || !p.obs_snap || p.obs_nlarge > 0 || p.obs_nspill > 0 || p.obs.n_long > 0 || st == 0)
    return;
  // build the plan; run the graph-mode pipeline once for real (allocates every
  // buffer at its final size), then capture it
  Plan np;
  np.N = tr.n; np.B = tr.B; np.W = tr.W; np.L = tr.L; np.inactive_opt = inactive;
  np.key = kp; np.tidop = tp; np.instr = ip; np.stream = st;
  np.n_bar = p.obs.n_bar; np.n_end = p.obs.n_end; np.n_wbar = p.obs.n_wbar; np.D = p.obs_D;
  np.n_acc = p.obs.n_acc;
  np.hard_small = p.obs_hard_small;
  np.cand_cap = 2ull * p.obs_ncand + 4096;  // tight: graph replays size the dedup / order passes by it
  np.pend_cap = 2ull * p.obs_npend + 4096;
  c->plan = np;
  Pipeline g;
  g.C = c; g.st = st; g.inactive_opt = inactive; g.tr = tr; g.gmode = true; g.P = &c->plan;
  g.run();
  // the graph's fixed epochs [1, 1 + gepoch) stay in the status words after
  // every replay: later eager analyses on this context continue above them
  c->epoch = std::max(c->epoch, 1 + g.gepoch);
  CK(cudaStreamSynchronize(st));
  cudaGraph_t graph = nullptr;
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  Pipeline q;
  q.C = c; q.st = st; q.inactive_opt = inactive; q.tr = tr; q.gmode = true; q.P = &c->plan;
  try {
    q.run();
  } catch (...) {
    cudaStreamEndCapture(st, &graph);
    if (graph) cudaGraphDestroy(graph);
    c->drop_plan();
    throw;
  }
  CK(cudaStreamEndCapture(st, &graph));
  cudaGraphExec_t exec = nullptr;
  cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ie != cudaSuccess) {
    c->drop_plan();
    return;  // keep eager mode
  }
  c->plan.exec = exec;
  c->plan.launches = c->launches;
  c->plan.valid = true;
  c->last_graph = true;  // the buffers hold the graph-mode run's results
}

extern "C" int gw_ctx_analyze_device(gw_ctx* c, const gw_trace_view* t, const gw_opts* o) {
  if (!c) { gw_set_error("null context"); return GW_E_ARG; }
  int v = validate_view(t);
  if (v) return v;
  return guarded([&] {
    CK(cudaSetDevice(c->device));
    cudaStream_t st = o ? (cudaStream_t)o->stream : (cudaStream_t)0;
    const uint32_t inactive = o ? o->inactive_opt : 1u;
    const uint32_t nsh = o && o->shard_count > 1 ? o->shard_count : 1u;
    const uint32_t sh = nsh > 1 ? o->shard_index : 0u;
    if (sh >= nsh) throw CudaErr{GW_E_ARG, "shard_index must be < shard_count"};
    DevTrace tr = make_dev(t, (const unsigned long long*)t->key, t->tidop, t->instr);
    analyze_impl(c, tr, st, inactive, t->key, t->tidop, t->instr, o && (o->flags & GW_OPT_EAGER), sh, nsh,
                 o && (o->flags & GW_OPT_PROFILE), o && (o->flags & GW_OPT_HB));
  });
}

extern "C" int gw_ctx_analyze_host(gw_ctx* c, const gw_trace_view* t, const gw_opts* o) {
  if (!c) { gw_set_error("null context"); return GW_E_ARG; }
  int v = validate_view(t);
  if (v) return v;
  return guarded([&] {
    CK(cudaSetDevice(c->device));
    cudaStream_t st = o ? (cudaStream_t)o->stream : (cudaStream_t)0;
    const uint32_t inactive = o ? o->inactive_opt : 1u;
    const uint32_t nsh = o && o->shard_count > 1 ? o->shard_count : 1u;
    const uint32_t sh = nsh > 1 ? o->shard_index : 0u;
    if (sh >= nsh) throw CudaErr{GW_E_ARG, "shard_index must be < shard_count"};
    const uint64_t N = t->n_events;
    c->last_stream = st;
    unsigned long long* k = c->get<unsigned long long>("in_key", N);
    uint32_t* to = c->get<uint32_t>("in_tidop", N);
    uint32_t* in = c->get<uint32_t>("in_instr", N);
    if (N) {
      CK(cudaMemcpyAsync(k, t->key, 8 * N, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(to, t->tidop, 4 * N, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(in, t->instr, 4 * N, cudaMemcpyHostToDevice, st));
    }
    DevTrace tr = make_dev(t, k, to, in);
    analyze_impl(c, tr, st, inactive, k, to, in, o && (o->flags & GW_OPT_EAGER), sh, nsh,
                 o && (o->flags & GW_OPT_PROFILE), o && (o->flags & GW_OPT_HB));
  });
}

// packed (narrow-column) host trace: widen one uploaded chunk into the
// 16-byte SoA the pipeline reads (the tidop column is uploaded in place)
// (4-byte keys: a warp barrier's key (block << 32 | warp) is implied by its
// tidop and restored here; block barriers carry key 0)
__global__ void k_widen(const void* __restrict__ kin, int kbytes, const void* __restrict__ iin, int ibytes,
                        const uint32_t* __restrict__ tidop, uint32_t BS, uint32_t L, uint64_t lo, uint64_t hi,
                        unsigned long long* __restrict__ kout, uint32_t* __restrict__ iout) {
  for (uint64_t e = lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < hi;
       e += (uint64_t)gridDim.x * blockDim.x) {
    if (kbytes == 4) {
      const uint32_t to = tidop[e];
      unsigned long long k = ((const uint32_t*)kin)[e];
      if (ev_kind(to) == GW_K_BARRIER)
        k = (to & GW_F_WARPBAR) ? ((unsigned long long)(ev_tid(to) / BS) << 32) | ((ev_tid(to) % BS) / L) : 0ull;
      kout[e] = k;
    }
    if (ibytes == 2) iout[e] = ((const uint16_t*)iin)[e];
  }
}

extern "C" int gw_ctx_analyze_host_packed(gw_ctx* c, const gw_trace_packed* t, const gw_opts* o) {
  if (!c || !t) { gw_set_error("null argument"); return GW_E_ARG; }
  if ((t->key_bytes != 4 && t->key_bytes != 8) || (t->instr_bytes != 2 && t->instr_bytes != 4)) {
    gw_set_error("packed trace: key_bytes must be 4 or 8, instr_bytes 2 or 4");
    return GW_E_ARG;
  }
  gw_trace_view view;
  view.cfg = t->cfg;
  view.n_events = t->n_events;
  view.key = (const uint64_t*)t->key;
  view.tidop = t->tidop;
  view.instr = (const uint32_t*)t->instr;
  int v = validate_view(&view);
  if (v) return v;
  return guarded([&] {
    CK(cudaSetDevice(c->device));
    cudaStream_t st = o ? (cudaStream_t)o->stream : (cudaStream_t)0;
    const uint32_t inactive = o ? o->inactive_opt : 1u;
    const uint32_t nsh = o && o->shard_count > 1 ? o->shard_count : 1u;
    const uint32_t sh = nsh > 1 ? o->shard_index : 0u;
    if (sh >= nsh) throw CudaErr{GW_E_ARG, "shard_index must be < shard_count"};
    const uint64_t N = t->n_events;
    c->last_stream = st;
    unsigned long long* k = c->get<unsigned long long>("in_key", N);
    uint32_t* to = c->get<uint32_t>("in_tidop", N);
    uint32_t* in = c->get<uint32_t>("in_instr", N);
    // narrow columns land in staging buffers, wide ones in place
    void* kst = t->key_bytes == 8 ? (void*)k : (void*)c->get<uint32_t>("pk_key", N);
    void* ist = t->instr_bytes == 4 ? (void*)in : (void*)c->get<uint16_t>("pk_instr", N);
    if (!c->copy_st) {
      CK(cudaStreamCreateWithFlags(&c->copy_st, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&c->ev_prev, cudaEventDisableTiming));
    }
    // the copies must not overwrite buffers an earlier analysis on st may still read
    CK(cudaEventRecord(c->ev_prev, st));
    CK(cudaStreamWaitEvent(c->copy_st, c->ev_prev, 0));
    constexpr uint64_t kChunk = 1ull << 25;  // events per upload chunk (~320 MB of C5 columns)
    const uint64_t nch = (N + kChunk - 1) / kChunk;
    while (c->chunk_ev.size() < nch) {
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      c->chunk_ev.push_back(e);
    }
    const bool widen = t->key_bytes == 4 || t->instr_bytes == 2;
    for (uint64_t ch = 0; ch < nch; ch++) {
      const uint64_t lo = ch * kChunk, hi = std::min(N, lo + kChunk), m = hi - lo;
      CK(cudaMemcpyAsync((char*)kst + lo * t->key_bytes, (const char*)t->key + lo * t->key_bytes,
                         m * t->key_bytes, cudaMemcpyHostToDevice, c->copy_st));
      CK(cudaMemcpyAsync(to + lo, t->tidop + lo, m * 4, cudaMemcpyHostToDevice, c->copy_st));
      CK(cudaMemcpyAsync((char*)ist + lo * t->instr_bytes, (const char*)t->instr + lo * t->instr_bytes,
                         m * t->instr_bytes, cudaMemcpyHostToDevice, c->copy_st));
      CK(cudaEventRecord(c->chunk_ev[ch], c->copy_st));
      CK(cudaStreamWaitEvent(st, c->chunk_ev[ch], 0));  // widen chunk ch while chunk ch + 1 is in flight
      if (widen) GW_LAUNCH(k_widen, grid_for(m, 148u * 8u), kThreads, 0, st, kst, (int)t->key_bytes, ist,
                           (int)t->instr_bytes, to, t->cfg.warps * t->cfg.lanes, t->cfg.lanes, lo, hi, k, in);
    }
    DevTrace tr = make_dev(&view, k, to, in);
    analyze_impl(c, tr, st, inactive, k, to, in, o && (o->flags & GW_OPT_EAGER), sh, nsh,
                 o && (o->flags & GW_OPT_PROFILE), o && (o->flags & GW_OPT_HB));
  });
}

// ---- delta-varint host trace (gw_trace_delta, codec.cpp) ----------------------
// One CTA per chunk of GW_DELTA_CHUNK events: the chunk's bytes in shared
// memory; every thread takes a contiguous byte range, counts varint
// terminators (high bit clear), a block scan numbers them, and each thread
// decodes the varints ending in its range (reading back to the previous
// terminator); then a blocked inclusive scan of the deltas from the chunk's
// base gives the column values.
template <class T>
struct DeltaSmem {
  static constexpr uint32_t kMaxB = GW_DELTA_CHUNK * (sizeof(T) == 8 ? 10u : 5u);
  uint8_t b[kMaxB];
  T d[GW_DELTA_CHUNK];
};
template <class T>
__global__ void __launch_bounds__(kThreads) k_delta_decode(const uint8_t* __restrict__ bytes,
                                                          const uint64_t* __restrict__ offs,
                                                          const uint64_t* __restrict__ base, uint64_t k0, uint64_t k1,
                                                          uint64_t n, T* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  DeltaSmem<T>& S = *reinterpret_cast<DeltaSmem<T>*>(smem_raw);
  constexpr uint32_t CH = GW_DELTA_CHUNK, IPT = CH / kThreads;
  for (uint64_t k = k0 + blockIdx.x; k < k1; k += gridDim.x) {
    const uint64_t lo = offs[k];
    const uint64_t nb64 = offs[k + 1] - lo, ne64 = n - k * CH;
    const uint32_t nb = (uint32_t)(nb64 < DeltaSmem<T>::kMaxB ? nb64 : DeltaSmem<T>::kMaxB);
    const uint32_t ne = (uint32_t)(ne64 < CH ? ne64 : CH);
    for (uint32_t j = threadIdx.x; j < nb; j += kThreads) S.b[j] = bytes[lo + j];
    __syncthreads();
    const uint32_t q = (nb + kThreads - 1) / kThreads;
    const uint32_t b0 = min(nb, threadIdx.x * q), b1 = min(nb, b0 + q);
    uint32_t cnt = 0;
    for (uint32_t j = b0; j < b1; j++) cnt += (S.b[j] & 0x80u) == 0;
    uint32_t tot;
    uint32_t idx = block_excl_scan<uint32_t, OpSum>(cnt, OpSum(), 0u, &tot);
    for (uint32_t j = b0; j < b1; j++) {
      if (S.b[j] & 0x80u) continue;
      uint32_t st0 = j;
      while (st0 > 0 && (S.b[st0 - 1] & 0x80u)) st0--;
      unsigned long long z = 0;
      for (uint32_t x = j + 1; x-- > st0;) z = (z << 7) | (S.b[x] & 0x7Fu);
      const T zz = (T)z;
      if (idx < CH) S.d[idx] = (zz >> 1) ^ (T)(0 - (zz & 1));
      idx++;
    }
    __syncthreads();
    const uint32_t p0 = threadIdx.x * IPT;
    T sum = 0;
#pragma unroll
    for (uint32_t x = 0; x < IPT; x++) sum += p0 + x < ne ? S.d[p0 + x] : (T)0;
    T all;
    T run = block_excl_scan<T, OpSum>(sum, OpSum(), (T)0, &all) + (T)base[k];
#pragma unroll
    for (uint32_t x = 0; x < IPT; x++)
      if (p0 + x < ne) {
        run += S.d[p0 + x];
        out[k * CH + p0 + x] = run;
      }
    __syncthreads();
  }
}
template <class T>
inline void delta_setup() {
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(k_delta_decode<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(DeltaSmem<T>));
    done = true;
  }
}

// ---- bit-packed trace (gw_trace_bp, codec.cpp) --------------------------------
// One warp per chunk of one column: the chunk's bytes staged in the warp's
// shared-memory slice (global reads past it), the block headers' widths /
// exception counts turned into offsets by warp scans, then the blocks in
// order: lane l extracts its b bits, exceptions patch their lanes, the
// residuals become first differences (mode 0: a warp scan from the previous
// block's last difference; modes 1 / 2: the same lane's difference one / two
// blocks back; mode 3: the residual itself) and the differences values (a
// warp scan from the previous value).
constexpr int kBpWarps = 8;
constexpr uint32_t kBpStageWords = 1024;  // 4 KB per warp (C5: ~0.1-0.3 KB per chunk and column)

template <class T>
__device__ __forceinline__ T bp_scan(T v, uint32_t lane) {  // inclusive warp prefix sum (mod 2^w)
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= (uint32_t)o) v += y;
  }
  return v;
}
__device__ __forceinline__ uint32_t bp_pick(const uint32_t (&v)[4], uint32_t q) {
  return q == 0 ? v[0] : q == 1 ? v[1] : q == 2 ? v[2] : v[3];
}

struct BpCol {
  const uint8_t* bytes;
  const uint64_t* offs;
  const uint64_t* base;
  const uint64_t* dbase;
  void* out;
};
template <class T, class O = T>  // T: the column's arithmetic width, O: the stored type
__device__ __forceinline__ void bp_decode_chunk(const BpCol& C, uint64_t k, uint64_t N, uint32_t* sw, uint32_t lane) {
  const uint8_t* __restrict__ bytes = C.bytes;
  const uint64_t* __restrict__ offs = C.offs;
  const uint64_t* __restrict__ base = C.base;
  const uint64_t* __restrict__ dbase = C.dbase;
  O* __restrict__ out = reinterpret_cast<O*>(C.out);
  {
    const uint64_t lo = k * GW_DELTA_CHUNK, cnt = min((uint64_t)GW_DELTA_CHUNK, N - lo);
    const uint32_t nb = (uint32_t)((cnt + 31) / 32);
    const uint64_t cb = offs[k];
    const uint32_t csz = (uint32_t)(offs[k + 1] - cb);  // multiple of 4
    const uint32_t* gw = reinterpret_cast<const uint32_t*>(bytes + cb);
    const bool staged = csz <= 4 * kBpStageWords;
    if (staged)
      for (uint32_t i = lane; i < csz / 4; i += 32) sw[i] = __ldg(gw + i);
    __syncwarp();
    const uint32_t* W = staged ? sw : gw;
    auto byte_at = [&](uint32_t o) -> uint32_t { return (W[o >> 2] >> (8 * (o & 3))) & 0xFFu; };
    // headers of blocks 4 lane .. 4 lane + 3; (count, width) byte pairs follow
    // the headers, one pair per block with exceptions
    uint32_t hd[4], nx[4], xw[4], wo[4], eo[4], vo[4];
    uint32_t esum = 0;
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const uint32_t kb = 4 * lane + q;
      hd[q] = kb < nb ? byte_at(kb) : 0u;
      esum += (hd[q] >> 5) & 1u;
    }
    const uint32_t einc = bp_scan<uint32_t>(esum, lane), ne_blocks = __shfl_sync(0xffffffffu, einc, 31);
    uint32_t eidx = einc - esum, wsum = 0, xsum = 0, vsum = 0;
#pragma unroll
    for (int q = 0; q < 4; q++) {
      nx[q] = 0;
      xw[q] = 0;
      if ((hd[q] >> 5) & 1u) {
        nx[q] = byte_at(nb + 2 * eidx);
        xw[q] = byte_at(nb + 2 * eidx + 1);
        eidx++;
      }
      wsum += hd[q] & 31u;
      xsum += nx[q];
      vsum += nx[q] * xw[q];
    }
    const uint32_t winc = bp_scan<uint32_t>(wsum, lane), xinc = bp_scan<uint32_t>(xsum, lane),
                   vinc = bp_scan<uint32_t>(vsum, lane);
    const uint32_t words_tot = __shfl_sync(0xffffffffu, winc, 31), exc_tot = __shfl_sync(0xffffffffu, xinc, 31);
    const uint32_t pk0 = ((nb + 2 * ne_blocks + 3) & ~3u) / 4;  // first packed word
    const uint32_t ix0 = 4 * (pk0 + words_tot);                 // first exception lane byte
    const uint32_t xv0 = ix0 + exc_tot;                          // first exception value byte
    {
      uint32_t w0 = winc - wsum, e0 = xinc - xsum, v0 = vinc - vsum;
#pragma unroll
      for (int q = 0; q < 4; q++) {
        wo[q] = w0; w0 += hd[q] & 31u;
        eo[q] = e0; e0 += nx[q];
        vo[q] = v0; v0 += nx[q] * xw[q];
      }
    }
    // d1 / d2: this lane's difference one / two blocks back; s1 / s2: the
    // inclusive warp scans of those blocks' differences; D* / S*: their last
    // lane's values (warp-uniform).  Blocks without residuals need no shuffle:
    // x = x_last + s, and the uniforms advance.
    T xl = (T)base[k], dl = (T)dbase[k], d1 = 0, d2 = 0, s1 = 0, s2 = 0, D1 = 0, D2 = 0, S1 = 0, S2 = 0;
    const uint64_t iend = lo + cnt;
    for (uint32_t kb = 0; kb < nb; kb++) {
      const uint32_t h = byte_at(kb);  // warp-uniform (a broadcast load)
      const uint32_t b = h & 31u, mode = h >> 6;
      const uint64_t i = lo + 32ull * kb + lane;
      T d, sd, D, S;
      if ((h & 0x3Fu) == 0) {  // b = 0, no exceptions: every residual 0
        // the run of blocks with this same header, written in closed form
        const uint32_t hj = kb + lane < nb ? byte_at(kb + lane) : 0x100u;
        const uint32_t same = __ballot_sync(0xffffffffu, hj == h);
        const uint32_t R = same == 0xffffffffu ? 32u : (uint32_t)__ffs(~same) - 1;  // >= 1
        O* o = out + (lo + 32ull * kb + lane);
        const uint64_t left = iend - (lo + 32ull * kb + lane);  // stores allowed: r * 32 < left
        if (mode == 0) {  // d = dl everywhere
          const T c0 = (T)((T)(lane + 1) * dl), step = (T)(32 * dl);
          T x = (T)(xl + c0);
          for (uint32_t r = 0; r < R; r++, x += step)
            if (32ull * r < left) o[32 * r] = (O)x;
          xl = (T)(xl + (T)R * step);
          if (R == 1) { d2 = d1; s2 = s1; D2 = D1; S2 = S1; }
          else { d2 = dl; s2 = c0; D2 = dl; S2 = step; }
          d1 = dl; s1 = c0; D1 = dl; S1 = step;
        } else if (mode == 1) {  // d = d1 in every block of the run
          T x = (T)(xl + s1);
          for (uint32_t r = 0; r < R; r++, x += S1)
            if (32ull * r < left) o[32 * r] = (O)x;
          xl = (T)(xl + (T)R * S1);
          d2 = d1; s2 = s1; D2 = D1; S2 = S1;
        } else if (mode == 2) {  // blocks alternate the patterns two and one back
          T x = xl;
          for (uint32_t r = 0; r < R; r++) {
            const bool ev = (r & 1u) == 0;
            if (32ull * r < left) o[32 * r] = (O)(T)(x + (ev ? s2 : s1));
            x = (T)(x + (ev ? S2 : S1));
          }
          xl = x;
          if (R & 1u) {  // odd run: the last block used the pattern two back
            T t = d1; d1 = d2; d2 = t;
            t = s1; s1 = s2; s2 = t;
            t = D1; D1 = D2; D2 = t;
            t = S1; S1 = S2; S2 = t;
          }
        } else {  // d = 0
          for (uint32_t r = 0; r < R; r++)
            if (32ull * r < left) o[32 * r] = (O)xl;
          if (R == 1) { d2 = d1; s2 = s1; D2 = D1; S2 = S1; }
          else { d2 = 0; s2 = 0; D2 = 0; S2 = 0; }
          d1 = 0; s1 = 0; D1 = 0; S1 = 0;
        }
        dl = D1;
        kb += R - 1;
        continue;
      } else if (b == 0) {
        // residuals only at the exception lanes: each exception (lane ie,
        // residual re) adds re to d at ie (and, mode 0, every later lane) and
        // to the scans at and after ie -- no warp scan needed
        const uint32_t src = kb >> 2, q = kb & 3;
        const uint32_t ne = __shfl_sync(0xffffffffu, bp_pick(nx, q), src);
        const uint32_t w = __shfl_sync(0xffffffffu, bp_pick(xw, q), src);
        const uint32_t e0 = __shfl_sync(0xffffffffu, bp_pick(eo, q), src);
        const uint32_t v0 = __shfl_sync(0xffffffffu, bp_pick(vo, q), src);
        uint32_t myi = 0;
        T myr = 0;
        if (lane < ne) {  // exception `lane`, read in parallel (w <= 8 bytes: three aligned words)
          myi = byte_at(ix0 + e0 + lane);
          const uint32_t off = xv0 + v0 + lane * w, wi = off >> 2, sh = 8 * (off & 3), avail = 4 - (off & 3);
          uint64_t z = (uint64_t)(W[wi] >> sh);  // words read only as far as the value reaches
          if (w > avail) z |= (uint64_t)W[wi + 1] << (32 - sh);
          if (w > avail + 4) z |= (uint64_t)W[wi + 2] << (64 - sh);
          if (w < 8) z &= (1ull << (8 * w)) - 1;
          myr = (T)((z >> 1) ^ (uint64_t)(-(int64_t)(z & 1)));
        }
        T dr = 0, sr = 0, wr = 0, tot = 0, wtot = 0, r31 = 0;
        for (uint32_t e = 0; e < ne; e++) {
          const uint32_t ie = __shfl_sync(0xffffffffu, myi, e);
          const T re = __shfl_sync(0xffffffffu, myr, e);
          if (ie == lane) dr = re;
          if (ie <= lane) sr += re;
          tot += re;
          if (mode == 0) {  // the scan of d = dl + (the prefix of the residuals)
            if (ie <= lane) wr += (T)(re * (T)(lane - ie + 1));
            wtot += (T)(re * (T)(32 - ie));
          }
          if (ie == 31) r31 = re;
        }
        if (mode == 0) { d = (T)(dl + sr); sd = (T)((T)(lane + 1) * dl + wr); D = (T)(dl + tot); S = (T)(32 * dl + wtot); }
        else if (mode == 1) { d = (T)(d1 + dr); sd = (T)(s1 + sr); D = (T)(D1 + r31); S = (T)(S1 + tot); }
        else if (mode == 2) { d = (T)(d2 + dr); sd = (T)(s2 + sr); D = (T)(D2 + r31); S = (T)(S2 + tot); }
        else { d = dr; sd = sr; D = r31; S = tot; }
      } else {
        const uint32_t src = kb >> 2, q = kb & 3;
        const uint32_t wof = __shfl_sync(0xffffffffu, bp_pick(wo, q), src);
        uint64_t p = 0;
        if (b) {
          const uint32_t bit = lane * b, wi = pk0 + wof + (bit >> 5), sh = bit & 31;
          uint64_t v = (uint64_t)W[wi];
          if (sh + b > 32) v |= (uint64_t)W[wi + 1] << 32;
          p = (v >> sh) & ((1ull << b) - 1);
        }
        if ((h >> 5) & 1u) {  // exceptions: zigzag values of their lanes, xw bytes each
          const uint32_t ne = __shfl_sync(0xffffffffu, bp_pick(nx, q), src);
          const uint32_t w = __shfl_sync(0xffffffffu, bp_pick(xw, q), src);
          const uint32_t e0 = __shfl_sync(0xffffffffu, bp_pick(eo, q), src);
          const uint32_t v0 = __shfl_sync(0xffffffffu, bp_pick(vo, q), src);
          for (uint32_t e = 0; e < ne; e++) {
            if (byte_at(ix0 + e0 + e) == lane) {
              uint64_t z = 0;
              for (uint32_t y = 0; y < w; y++) z |= (uint64_t)byte_at(xv0 + v0 + e * w + y) << (8 * y);
              p = z;
            }
          }
        }
        const T r = (T)((p >> 1) ^ (uint64_t)(-(int64_t)(p & 1)));  // unzigzag
        d = mode == 0 ? (T)(dl + bp_scan<T>(r, lane)) : mode == 1 ? (T)(d1 + r) : mode == 2 ? (T)(d2 + r) : r;
        sd = bp_scan<T>(d, lane);
        D = __shfl_sync(0xffffffffu, d, 31);
        S = __shfl_sync(0xffffffffu, sd, 31);
      }
      if (i < iend) out[i] = (O)(T)(xl + sd);
      xl = (T)(xl + S);
      dl = D;
      d2 = d1; s2 = s1; D2 = D1; S2 = S1;
      d1 = d; s1 = sd; D1 = D; S1 = S;
    }
    __syncwarp();
  }
}
// all three columns of chunks [k0, k1) in one launch: warp task t = chunk
// k0 + t / 3, column t % 3 (0: key u64, 1: tidop, 2: instr)
__global__ void __launch_bounds__(32 * kBpWarps, 3) k_bp_decode(BpCol c0, BpCol c1, BpCol c2, uint64_t k0, uint64_t k1,
                                                               uint64_t N, int key32) {
  __shared__ uint32_t stage[kBpWarps][kBpStageWords];
  const uint32_t lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
  const uint64_t nt = 3 * (k1 - k0);
  for (uint64_t t = (uint64_t)blockIdx.x * kBpWarps + wq; t < nt; t += (uint64_t)gridDim.x * kBpWarps) {
    const uint64_t k = k0 + t / 3;
    const uint32_t col = (uint32_t)(t % 3);
    if (col == 0) {
      if (key32) bp_decode_chunk<uint32_t, unsigned long long>(c0, k, N, stage[wq], lane);
      else bp_decode_chunk<unsigned long long>(c0, k, N, stage[wq], lane);
    }
    else bp_decode_chunk<uint32_t>(col == 1 ? c1 : c2, k, N, stage[wq], lane);
    __syncwarp();
  }
}

extern "C" int gw_ctx_analyze_host_delta(gw_ctx* c, const gw_trace_delta* t, const gw_opts* o) {
  if (!c || !t) { gw_set_error("null argument"); return GW_E_ARG; }
  if (t->chunk != GW_DELTA_CHUNK || t->n_chunks != (t->n_events + GW_DELTA_CHUNK - 1) / GW_DELTA_CHUNK) {
    gw_set_error("delta trace: chunking does not match GW_DELTA_CHUNK");
    return GW_E_ARG;
  }
  gw_trace_view view;
  view.cfg = t->cfg;
  view.n_events = t->n_events;
  view.key = (const uint64_t*)t->bytes[0];
  view.tidop = (const uint32_t*)t->bytes[1];
  view.instr = (const uint32_t*)t->bytes[2];
  int v = validate_view(&view);
  if (v) return v;
  return guarded([&] {
    CK(cudaSetDevice(c->device));
    cudaStream_t st = o ? (cudaStream_t)o->stream : (cudaStream_t)0;
    const uint32_t inactive = o ? o->inactive_opt : 1u;
    const uint32_t nsh = o && o->shard_count > 1 ? o->shard_count : 1u;
    const uint32_t sh = nsh > 1 ? o->shard_index : 0u;
    if (sh >= nsh) throw CudaErr{GW_E_ARG, "shard_index must be < shard_count"};
    const uint64_t N = t->n_events, K = t->n_chunks;
    c->last_stream = st;
    unsigned long long* k = c->get<unsigned long long>("in_key", N);
    uint32_t* to = c->get<uint32_t>("in_tidop", N);
    uint32_t* in = c->get<uint32_t>("in_instr", N);
    if (!c->copy_st) {
      CK(cudaStreamCreateWithFlags(&c->copy_st, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&c->ev_prev, cudaEventDisableTiming));
    }
    uint8_t* db[3];
    uint64_t* doff[3];
    uint64_t* dbase[3];
    const char* nm[3] = {"dl_key", "dl_tidop", "dl_instr"};
    for (int col = 0; col < 3; col++) {
      db[col] = c->get<uint8_t>(std::string(nm[col]) + "_b", t->nbytes[col] + 16);
      doff[col] = c->get<uint64_t>(std::string(nm[col]) + "_o", K + 1);
      dbase[col] = c->get<uint64_t>(std::string(nm[col]) + "_s", K + 1);
    }
    // after the allocations: a new buffer is zeroed on st, and earlier analyses
    // on st may still read the staging / input buffers the copies overwrite
    CK(cudaEventRecord(c->ev_prev, st));
    CK(cudaStreamWaitEvent(c->copy_st, c->ev_prev, 0));
    for (int col = 0; col < 3; col++) {
      if (K) {
        CK(cudaMemcpyAsync(doff[col], t->offs[col], 8 * (K + 1), cudaMemcpyHostToDevice, c->copy_st));
        CK(cudaMemcpyAsync(dbase[col], t->base[col], 8 * K, cudaMemcpyHostToDevice, c->copy_st));
      }
    }
    constexpr uint64_t kSlice = 1024;  // chunks per upload slice (4 M events)
    const uint64_t ns = (K + kSlice - 1) / kSlice;
    while (c->chunk_ev.size() < ns) {
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      c->chunk_ev.push_back(e);
    }
    delta_setup<unsigned long long>();
    delta_setup<uint32_t>();
    for (uint64_t sl = 0; sl < ns; sl++) {
      const uint64_t k0 = sl * kSlice, k1 = std::min(K, k0 + kSlice);
      for (int col = 0; col < 3; col++) {
        const uint64_t a = t->offs[col][k0], b = t->offs[col][k1];
        if (b > a) CK(cudaMemcpyAsync(db[col] + a, t->bytes[col] + a, b - a, cudaMemcpyHostToDevice, c->copy_st));
      }
      CK(cudaEventRecord(c->chunk_ev[sl], c->copy_st));
      CK(cudaStreamWaitEvent(st, c->chunk_ev[sl], 0));  // decode slice sl while slice sl + 1 is in flight
      const unsigned g = (unsigned)std::min<uint64_t>(k1 - k0, 148ull * 3);
      GW_LAUNCH(k_delta_decode<unsigned long long>, g, kThreads, sizeof(DeltaSmem<unsigned long long>), st, db[0],
                doff[0], dbase[0], k0, k1, N, k);
      GW_LAUNCH(k_delta_decode<uint32_t>, g, kThreads, sizeof(DeltaSmem<uint32_t>), st, db[1], doff[1], dbase[1],
                k0, k1, N, to);
      GW_LAUNCH(k_delta_decode<uint32_t>, g, kThreads, sizeof(DeltaSmem<uint32_t>), st, db[2], doff[2], dbase[2],
                k0, k1, N, in);
    }
    DevTrace tr = make_dev(&view, k, to, in);
    analyze_impl(c, tr, st, inactive, k, to, in, o && (o->flags & GW_OPT_EAGER), sh, nsh,
                 o && (o->flags & GW_OPT_PROFILE), o && (o->flags & GW_OPT_HB));
  });
}

extern "C" int gw_ctx_analyze_host_bp(gw_ctx* c, const gw_trace_bp* t, const gw_opts* o) {
  if (!c || !t) { gw_set_error("null argument"); return GW_E_ARG; }
  if (t->chunk != GW_DELTA_CHUNK || t->n_chunks != (t->n_events + GW_DELTA_CHUNK - 1) / GW_DELTA_CHUNK) {
    gw_set_error("bit-packed trace: chunking does not match GW_DELTA_CHUNK");
    return GW_E_ARG;
  }
  if (t->key_bits != 32 && t->key_bits != 64) {
    gw_set_error("bit-packed trace: key_bits must be 32 or 64");
    return GW_E_ARG;
  }
  gw_trace_view view;
  view.cfg = t->cfg;
  view.n_events = t->n_events;
  view.key = (const uint64_t*)t->bytes[0];
  view.tidop = (const uint32_t*)t->bytes[1];
  view.instr = (const uint32_t*)t->bytes[2];
  int v = validate_view(&view);
  if (v) return v;
  return guarded([&] {
    CK(cudaSetDevice(c->device));
    cudaStream_t st = o ? (cudaStream_t)o->stream : (cudaStream_t)0;
    const uint32_t inactive = o ? o->inactive_opt : 1u;
    const uint32_t nsh = o && o->shard_count > 1 ? o->shard_count : 1u;
    const uint32_t sh = nsh > 1 ? o->shard_index : 0u;
    if (sh >= nsh) throw CudaErr{GW_E_ARG, "shard_index must be < shard_count"};
    const uint64_t N = t->n_events, K = t->n_chunks;
    c->last_stream = st;
    unsigned long long* k = c->get<unsigned long long>("in_key", N);
    uint32_t* to = c->get<uint32_t>("in_tidop", N);
    uint32_t* in = c->get<uint32_t>("in_instr", N);
    if (!c->copy_st) {
      CK(cudaStreamCreateWithFlags(&c->copy_st, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&c->ev_prev, cudaEventDisableTiming));
    }
    uint8_t* db[3];
    uint64_t* doff[3];
    uint64_t* dbase[3];
    uint64_t* ddb[3];
    const char* nm[3] = {"bp_key", "bp_tidop", "bp_instr"};
    for (int col = 0; col < 3; col++) {
      db[col] = c->get<uint8_t>(std::string(nm[col]) + "_b", t->nbytes[col] + 16);
      doff[col] = c->get<uint64_t>(std::string(nm[col]) + "_o", K + 1);
      dbase[col] = c->get<uint64_t>(std::string(nm[col]) + "_s", K + 1);
      ddb[col] = c->get<uint64_t>(std::string(nm[col]) + "_d", K + 1);
    }
    // after the allocations: a new buffer is zeroed on st, and earlier analyses
    // on st may still read the staging / input buffers the copies overwrite
    CK(cudaEventRecord(c->ev_prev, st));
    CK(cudaStreamWaitEvent(c->copy_st, c->ev_prev, 0));
    for (int col = 0; col < 3; col++) {
      if (K) {
        CK(cudaMemcpyAsync(doff[col], t->offs[col], 8 * (K + 1), cudaMemcpyHostToDevice, c->copy_st));
        CK(cudaMemcpyAsync(dbase[col], t->base[col], 8 * K, cudaMemcpyHostToDevice, c->copy_st));
        CK(cudaMemcpyAsync(ddb[col], t->dbase[col], 8 * K, cudaMemcpyHostToDevice, c->copy_st));
      }
    }
    // chunks per upload slice: 128 M events (~36 MB on C5), the first one
    // 16 M so that decoding starts early
    constexpr uint64_t kSlice = 32768, kFirst = 4096;
    auto slice_lo = [&](uint64_t sl) { return sl == 0 ? 0 : std::min(K, kFirst + (sl - 1) * kSlice); };
    const uint64_t ns = K <= kFirst ? (K ? 1 : 0) : 1 + (K - kFirst + kSlice - 1) / kSlice;
    while (c->chunk_ev.size() < ns) {
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      c->chunk_ev.push_back(e);
    }
    for (uint64_t sl = 0; sl < ns; sl++) {
      const uint64_t k0 = slice_lo(sl), k1 = std::min(K, sl == 0 ? kFirst : k0 + kSlice);
      for (int col = 0; col < 3; col++) {
        const uint64_t a = t->offs[col][k0], b = t->offs[col][k1];
        if (b > a) CK(cudaMemcpyAsync(db[col] + a, t->bytes[col] + a, b - a, cudaMemcpyHostToDevice, c->copy_st));
      }
      CK(cudaEventRecord(c->chunk_ev[sl], c->copy_st));
      CK(cudaStreamWaitEvent(st, c->chunk_ev[sl], 0));  // decode slice sl while slice sl + 1 is in flight
      const unsigned g = (unsigned)std::min<uint64_t>((3 * (k1 - k0) + kBpWarps - 1) / kBpWarps, 148ull * 7);
      GW_LAUNCH(k_bp_decode, g, 32 * kBpWarps, 0, st, BpCol{db[0], doff[0], dbase[0], ddb[0], k},
                BpCol{db[1], doff[1], dbase[1], ddb[1], to}, BpCol{db[2], doff[2], dbase[2], ddb[2], in}, k0, k1, N,
                t->key_bits == 32 ? 1 : 0);
    }
    DevTrace tr = make_dev(&view, k, to, in);
    analyze_impl(c, tr, st, inactive, k, to, in, o && (o->flags & GW_OPT_EAGER), sh, nsh,
                 o && (o->flags & GW_OPT_PROFILE), o && (o->flags & GW_OPT_HB));
  });
}

// host copy of a large result array on several threads (first touch of the
// fresh destination pages included): millions of reports (C4) otherwise
// spend tens of ms in one memcpy
static void par_memcpy(void* dst, const void* src, size_t bytes) {
  constexpr size_t kChunk = 4u << 20;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t nt = std::min<size_t>(std::min<size_t>(hw, 16), (bytes + kChunk - 1) / kChunk);
  if (nt <= 1) { memcpy(dst, src, bytes); return; }
  const size_t per = ((bytes + nt - 1) / nt + 63) & ~(size_t)63;
  std::vector<std::thread> th;
  for (size_t i = 1; i < nt; i++) {
    const size_t o = i * per;
    if (o >= bytes) break;
    th.emplace_back([=] { memcpy((char*)dst + o, (const char*)src + o, std::min(per, bytes - o)); });
  }
  memcpy(dst, src, std::min(per, bytes));
  for (auto& t : th) t.join();
}

extern "C" int gw_ctx_fetch(gw_ctx* c, gw_result* out) {
  if (!c || !out) { gw_set_error("null argument"); return GW_E_ARG; }
  memset(out, 0, sizeof *out);
  return guarded([&] {
    CK(cudaSetDevice(c->device));
    uint64_t n = 0, nd = 0;
    if (c->d_scal) {
      uint32_t sc[SC_COUNT];
      CK(cudaStreamSynchronize(c->last_stream));
      memcpy(sc, c->h_scal, sizeof sc);
      if (sc[SC_ABORT] && c->last_graph) {
        // the trace no longer matches the cached plan: re-run eagerly
        c->drop_plan();
        c->last_graph = false;
        Pipeline p;
        p.C = c; p.st = c->last_stream; p.inactive_opt = c->last_inactive; p.tr = c->last_tr;
        p.shard = c->last_shard; p.nshard = c->last_nshard; p.hb_mode = c->last_hb;
        p.run();
        CK(cudaStreamSynchronize(c->last_stream));
        memcpy(sc, c->h_scal, sizeof sc);
      }
      if (sc[SC_ERR]) {
        char buf[200];
        snprintf(buf, sizeof buf,
                 "engine capacity error flags 0x%x (arena %llu words; dense lock clocks need more memory?)",
                 sc[SC_ERR], (unsigned long long)c->arena_words);
        throw CudaErr{GW_E_NOMEM, buf};
      }
      n = c->have_cands ? sc[SC_NSURV] : 0;
      nd = sc[SC_DIAG];
    }
    c->n_reports = n;
    c->n_diags = nd;
    out->n_reports = n;
    out->order_key = (uint64_t*)malloc(8 * std::max<uint64_t>(n, 1));
    if (!out->order_key) throw std::bad_alloc();
    out->kind = (uint8_t*)malloc(std::max<uint64_t>(n, 1));
    out->prior_event = (uint32_t*)malloc(4 * std::max<uint64_t>(n, 1));
    out->current_event = (uint32_t*)malloc(4 * std::max<uint64_t>(n, 1));
    if (!out->kind || !out->prior_event || !out->current_event) throw std::bad_alloc();
    std::vector<Diag> dg(nd);
    if (n) {  // written by k_final into mapped host memory (complete after the stream sync above)
      par_memcpy(out->kind, c->d_kind, n);
      par_memcpy(out->prior_event, c->d_prior, 4 * n);
      par_memcpy(out->current_event, c->d_cur, 4 * n);
      par_memcpy(out->order_key, c->d_okey, 8 * n);
    }
    if (nd) {
      CK(cudaMemcpyAsync(dg.data(), c->d_diags, sizeof(Diag) * nd, cudaMemcpyDeviceToHost, c->last_stream));
      CK(cudaStreamSynchronize(c->last_stream));
    }
    std::sort(dg.begin(), dg.end(), [](const Diag& a, const Diag& b) {
      return a.ev != b.ev ? a.ev < b.ev : a.sub < b.sub;
    });
    out->n_diags = nd;
    out->diag_event = (uint32_t*)malloc(4 * std::max<uint64_t>(nd, 1));
    out->diag_code = (uint32_t*)malloc(4 * std::max<uint64_t>(nd, 1));
    out->diag_lock = (uint64_t*)malloc(8 * std::max<uint64_t>(nd, 1));
    if (!out->diag_event || !out->diag_code || !out->diag_lock) throw std::bad_alloc();
    for (uint64_t i = 0; i < nd; i++) {
      out->diag_event[i] = dg[i].ev;
      out->diag_code[i] = dg[i].code;
      out->diag_lock[i] = dg[i].lock;
    }
  });
}

extern "C" void gw_result_free(gw_result* r) {
  if (!r) return;
  free(r->kind);
  free(r->prior_event);
  free(r->current_event);
  free(r->diag_event);
  free(r->diag_code);
  free(r->diag_lock);
  free(r->order_key);
  memset(r, 0, sizeof *r);
}

extern "C" int gw_ctx_stats(gw_ctx* c, gw_stats* out) {
  if (!c || !out) return GW_E_ARG;
  return guarded([&] {
    c->finish_stats();
    *out = c->stats;
  });
}

extern "C" uint32_t gw_ctx_launches(gw_ctx* c) { return c ? c->launches : 0; }

// ---- exchange mode (multi-GPU data plane; shard.py drives the collectives) ----
static void xs_stats_out(const Stats& h, gw_xs_stats* o) {
  o->n_acc = h.n_acc; o->n_write = h.n_write; o->n_acq = h.n_acq; o->n_rel = h.n_rel; o->n_end = h.n_end;
  o->n_bar = h.n_bar; o->key_or = h.key_or; o->key_and = h.key_and; o->n_long = h.n_long; o->n_wbar = h.n_wbar;
}
static Stats xs_stats_in(const gw_xs_stats* o) {
  Stats h;
  memset(&h, 0, sizeof h);
  h.n_acc = o->n_acc; h.n_write = o->n_write; h.n_acq = o->n_acq; h.n_rel = o->n_rel; h.n_end = o->n_end;
  h.n_bar = o->n_bar; h.key_or = o->key_or; h.key_and = o->key_and; h.n_long = o->n_long; h.n_wbar = o->n_wbar;
  return h;
}
static int xs_gbits_of(uint32_t G) {
  int g = 0;
  while ((1u << g) < G) g++;
  return (1u << g) == G && g >= 1 && g <= 5 ? g : -1;
}
static Pipeline xs_pipe(gw_ctx* c, cudaStream_t st) {
  Pipeline p;
  p.C = c;
  p.st = st;
  p.tr = c->xs_slice;
  p.inactive_opt = 1;
  c->last_stream = st;
  return p;
}

extern "C" int gw_xs_prep(gw_ctx* c, const gw_trace_view* slice, uint32_t event_base, void* stream,
                          gw_xs_stats* out) {
  if (!c || !out) { gw_set_error("null argument"); return GW_E_ARG; }
  int v = validate_view(slice);
  if (v) return v;
  return guarded([&] {
    CK(cudaSetDevice(c->device));
    c->drop_plan();
    c->xs_slice = make_dev(slice, (const unsigned long long*)slice->key, slice->tidop, slice->instr);
    c->xs_base = event_base;
    Pipeline p = xs_pipe(c, (cudaStream_t)stream);
    xs_stats_out(p.xs_prep(), out);
  });
}

extern "C" int gw_xs_hard(gw_ctx* c, void* stream, uint32_t* ev, uint32_t* tidop, uint32_t* instr, uint64_t* key,
                          uint64_t* n_out) {
  if (!c || !n_out) { gw_set_error("null argument"); return GW_E_ARG; }
  return guarded([&] {
    CK(cudaSetDevice(c->device));
    Pipeline p = xs_pipe(c, (cudaStream_t)stream);
    p.xs_begin();
    *n_out = p.xs_hard(c->xs_base, ev, tidop, instr, (unsigned long long*)key);
  });
}

extern "C" int gw_xs_partition(gw_ctx* c, const gw_xs_stats* global, uint32_t shard_count, void* stream, uint32_t* h,
                               uint32_t* v, uint32_t* t, uint64_t* counts) {
  if (!c || !global || !counts) { gw_set_error("null argument"); return GW_E_ARG; }
  const int gb = xs_gbits_of(shard_count);
  if (gb < 0) { gw_set_error("exchange mode: shard_count must be a power of two in [2, 32]"); return GW_E_ARG; }
  return guarded([&] {
    CK(cudaSetDevice(c->device));
    Pipeline p = xs_pipe(c, (cudaStream_t)stream);
    p.xs_partition(xs_stats_in(global), gb, c->xs_base, h, v, t, counts);
  });
}

extern "C" int gw_xs_check(gw_ctx* c, const gw_xs_stats* global, uint32_t shard_count, uint64_t n_total,
                           void* stream, const uint32_t* h, const uint32_t* v, const uint32_t* t, uint64_t n_recv,
                           const uint32_t* hev, const uint32_t* htidop, const uint32_t* hinstr, const uint64_t* hkey,
                           uint64_t n_hard, uint64_t* n_cand) {
  if (!c || !global || !n_cand) { gw_set_error("null argument"); return GW_E_ARG; }
  const int gb = xs_gbits_of(shard_count);
  if (gb < 0) { gw_set_error("exchange mode: shard_count must be a power of two in [2, 32]"); return GW_E_ARG; }
  if (global->n_acq || global->n_rel || global->n_long) {
    gw_set_error("exchange mode: lock traces and records longer than 32 events use the replicated shard mode");
    return GW_E_UNSUPPORTED;
  }
  return guarded([&] {
    CK(cudaSetDevice(c->device));
    Pipeline p = xs_pipe(c, (cudaStream_t)stream);
    BkRecSrc recv{h, v, t, n_recv};
    *n_cand = p.xs_check(xs_stats_in(global), gb, c->xs_base, recv, hev, htidop, hinstr,
                         (const unsigned long long*)hkey, n_hard, n_total);
    c->xs_nc = p.xs_nc;
    c->xs_nsi = p.xs_nsi;
    c->launches = g_launches;
  });
}

// host copies of the last gw_xs_check's candidates (caller buffers of n_cand);
// the slice's same-instruction pairs get their global event indices here
extern "C" int gw_xs_fetch(gw_ctx* c, uint64_t* okey, uint64_t* loc, uint32_t* prior, uint32_t* cur,
                           uint32_t* kind) {
  if (!c) { gw_set_error("null context"); return GW_E_ARG; }
  return guarded([&] {
    CK(cudaSetDevice(c->device));
    const cudaStream_t st = c->last_stream;
    auto cp = [&](void* dst, const char* name, size_t sz, uint64_t n, uint64_t at) {
      if (n) CK(cudaMemcpyAsync((char*)dst + at * sz, c->bufs[name].p, sz * n, cudaMemcpyDeviceToHost, st));
    };
    const uint64_t a = c->xs_nc, b = c->xs_nsi;
    cp(okey, "c_okey", 8, a, 0); cp(loc, "c_loc", 8, a, 0); cp(prior, "c_prior", 4, a, 0);
    cp(cur, "c_cur", 4, a, 0); cp(kind, "c_kind", 4, a, 0);
    cp(okey, "xsi_okey", 8, b, a); cp(loc, "xsi_loc", 8, b, a); cp(prior, "xsi_prior", 4, b, a);
    cp(cur, "xsi_cur", 4, b, a); cp(kind, "xsi_kind", 4, b, a);
    CK(cudaStreamSynchronize(st));
    const uint64_t base = c->xs_base;
    for (uint64_t k = a; k < a + b; k++) {
      okey[k] += base << 32;
      prior[k] += (uint32_t)base;
      cur[k] += (uint32_t)base;
    }
  });
}

// endpoint info (tidop, instr) of global events in this rank's slice; other entries untouched
extern "C" int gw_xs_lookup(gw_ctx* c, const uint32_t* ev, uint64_t n, uint32_t* tidop, uint32_t* instr) {
  if (!c) { gw_set_error("null context"); return GW_E_ARG; }
  return guarded([&] {
    CK(cudaSetDevice(c->device));
    if (!n) return;
    const cudaStream_t st = c->last_stream;
    uint32_t* dev = c->get<uint32_t>("x_lev", n);
    uint32_t* dto = c->get<uint32_t>("x_lto", n);
    uint32_t* din = c->get<uint32_t>("x_lin", n);
    CK(cudaMemcpyAsync(dev, ev, 4 * n, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dto, tidop, 4 * n, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(din, instr, 4 * n, cudaMemcpyHostToDevice, st));
    GW_LAUNCH(k_xs_lookup, grid_for(n), kThreads, 0, st, c->xs_slice, c->xs_base, dev, n, dto, din);
    CK(cudaMemcpyAsync(tidop, dto, 4 * n, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(instr, din, 4 * n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

template <class T>
static T* to_malloc(const std::vector<T>& v) {
  T* p = (T*)malloc(sizeof(T) * std::max<size_t>(v.size(), 1));
  if (!p) throw std::bad_alloc();
  if (!v.empty()) memcpy(p, v.data(), sizeof(T) * v.size());
  return p;
}

// the trace on the device (host view: H2D into the context's input buffers)
static DevTrace upload_view(gw_ctx* c, const gw_trace_view* t, cudaStream_t st) {
  const uint64_t N = t->n_events;
  unsigned long long* k = c->get<unsigned long long>("in_key", N);
  uint32_t* to = c->get<uint32_t>("in_tidop", N);
  uint32_t* in = c->get<uint32_t>("in_instr", N);
  if (N) {
    CK(cudaMemcpyAsync(k, t->key, 8 * N, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(to, t->tidop, 4 * N, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(in, t->instr, 4 * N, cudaMemcpyHostToDevice, st));
  }
  return make_dev(t, k, to, in);
}

extern "C" int gw_ctx_validate(gw_ctx* c, const gw_trace_view* t, uint64_t* n_out, uint32_t** ev, uint32_t** code,
                               uint64_t** a, uint64_t** b) {
  if (!c || !n_out) { gw_set_error("null argument"); return GW_E_ARG; }
  int v = validate_view(t);
  if (v) return v;
  *n_out = 0;
  return guarded([&] {
    CK(cudaSetDevice(c->device));
    cudaStream_t st = 0;
    c->last_stream = st;
    c->drop_plan();  // the input buffers are rewritten: no graph replay may assume their contents
    DevTrace tr = upload_view(c, t, st);
    std::vector<uint32_t> oe, oc;
    std::vector<uint64_t> oa, ob;
    if (tr.n) {
      Pipeline p;
      p.C = c; p.st = st; p.tr = tr; p.inactive_opt = 1;
      p.validate_run(oe, oc, oa, ob);
    }
    *n_out = oe.size();
    if (ev) *ev = to_malloc(oe);
    if (code) *code = to_malloc(oc);
    if (a) *a = to_malloc(oa);
    if (b) *b = to_malloc(ob);
  });
}

extern "C" int gw_ctx_infer_locks(gw_ctx* c, const gw_trace_view* t, gw_trace* out, uint64_t* n_diag,
                                  uint32_t** diag_event, uint64_t** diag_lock, uint32_t** diag_tid) {
  if (!c || !out || !n_diag) { gw_set_error("null argument"); return GW_E_ARG; }
  int v = validate_view(t);
  if (v) return v;
  memset(out, 0, sizeof *out);
  *n_diag = 0;
  return guarded([&] {
    CK(cudaSetDevice(c->device));
    cudaStream_t st = 0;
    c->last_stream = st;
    c->drop_plan();
    DevTrace tr = upload_view(c, t, st);
    std::vector<unsigned long long> ok;
    std::vector<uint32_t> oto, oin, de, dt;
    std::vector<unsigned long long> dl;
    if (tr.n) {
      Pipeline p;
      p.C = c; p.st = st; p.tr = tr; p.inactive_opt = 1;
      p.infer_run(ok, oto, oin, de, dl, dt);
    }
    out->cfg = t->cfg;
    out->n_events = ok.size();
    out->key = (uint64_t*)to_malloc(ok);
    out->tidop = to_malloc(oto);
    out->instr = to_malloc(oin);
    *n_diag = de.size();
    if (diag_event) *diag_event = to_malloc(de);
    if (diag_lock) *diag_lock = (uint64_t*)to_malloc(dl);
    if (diag_tid) *diag_tid = to_malloc(dt);
  });
}

static std::mutex g_default_mu;
static gw_ctx* g_default = nullptr;

extern "C" int gw_analyze(const gw_trace_view* t, const gw_opts* o, gw_result* out) {
  std::lock_guard<std::mutex> lk(g_default_mu);
  if (!g_default) {
    g_default = gw_ctx_create(0);
    if (!g_default) return GW_E_CUDA;
  }
  int r = gw_ctx_analyze_host(g_default, t, o);
  if (r) return r;
  return gw_ctx_fetch(g_default, out);
}

// Device-side C2/C5 workload generator (bench / test infrastructure).
extern "C" int gw_gen_c2_device(uint32_t blocks, uint32_t warps, uint32_t lanes, uint32_t phases, uint32_t records,
                                uint64_t words_per_block, uint64_t seed, uint64_t* key, uint32_t* tidop,
                                uint32_t* instr, void* stream) {
  return guarded([&] {
    C2Params p{blocks, warps, lanes, phases, records, words_per_block, seed};
    const uint64_t n = (uint64_t)phases * ((uint64_t)records * blocks * warps * lanes + blocks);
    GW_LAUNCH(k_gen_c2, 148u * 16u, kThreads, 0, (cudaStream_t)stream, p, (unsigned long long*)key, tidop, instr, n);
    CK(cudaGetLastError());
  });
}

extern "C" int gw_gen_c4_device(uint32_t blocks, uint32_t warps, uint32_t iters, uint64_t words_per_block,
                                uint64_t seed, uint64_t* key, uint32_t* tidop, uint32_t* instr, void* stream) {
  return guarded([&] {
    C4Params p{blocks, warps, 32u, iters, words_per_block, seed};
    const uint64_t groups = (uint64_t)blocks * warps * iters;
    const uint64_t g = groups * 32ull;
    GW_LAUNCH(k_gen_c4, (unsigned)std::min<uint64_t>((g + kThreads - 1) / kThreads, 148ull * 64), kThreads, 0,
              (cudaStream_t)stream, p, (unsigned long long*)key, tidop, instr);
    CK(cudaGetLastError());
  });
}

extern "C" int gw_gen_c3_device(uint32_t blocks, uint32_t warps, uint32_t lanes, uint32_t iters, uint32_t locks,
                                uint32_t region, uint32_t priv, uint64_t seed, const uint64_t* group_offsets,
                                uint64_t* key, uint32_t* tidop, uint32_t* instr, void* stream) {
  if (lanes == 0 || lanes > 32) { gw_set_error("C3 generator: lanes must be in [1, 32]"); return GW_E_ARG; }
  return guarded([&] {
    C3Params p{blocks, warps, lanes, iters, locks, region, priv, seed};
    const uint64_t g = (uint64_t)blocks * warps * iters * 32ull;
    GW_LAUNCH(k_gen_c3, (unsigned)std::min<uint64_t>((g + kThreads - 1) / kThreads, 148ull * 64), kThreads, 0,
              (cudaStream_t)stream, p, (const unsigned long long*)group_offsets, (unsigned long long*)key, tidop,
              instr);
    CK(cudaGetLastError());
  });
}

// per-kernel device times of the last GW_OPT_PROFILE analysis, aggregated by
// kernel (launch expression): names[i] (NUL-terminated, truncated to 63
// chars), total ms, launch count
extern "C" int gw_ctx_kernel_times(gw_ctx* c, uint32_t cap, char (*names)[64], float* ms, uint32_t* launches,
                                   uint32_t* n_out) {
  if (!c || !n_out) { gw_set_error("null argument"); return GW_E_ARG; }
  return guarded([&] {
    *n_out = 0;
    if (!c->prof_done) return;
    CK(cudaSetDevice(c->device));
    std::vector<std::string> nm;
    std::vector<float> tot;
    std::vector<uint32_t> cnt;
    for (uint32_t i = 0; i < c->prof.n; i++) {
      const auto& r = c->prof.recs[i];
      CK(cudaEventSynchronize(r.b));
      float t = 0.f;
      CK(cudaEventElapsedTime(&t, r.a, r.b));
      std::string k(r.name);
      if (r.tag) { k += "@"; k += r.tag; }
      size_t j = 0;
      while (j < nm.size() && nm[j] != k) j++;
      if (j == nm.size()) { nm.push_back(k); tot.push_back(0.f); cnt.push_back(0); }
      tot[j] += t;
      cnt[j]++;
    }
    const uint32_t n = (uint32_t)std::min<size_t>(nm.size(), cap);
    for (uint32_t j = 0; j < n; j++) {
      snprintf(names[j], 64, "%s", nm[j].c_str());
      ms[j] = tot[j];
      launches[j] = cnt[j];
    }
    *n_out = n;
  });
}
