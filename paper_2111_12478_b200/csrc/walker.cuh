// Sync pass of the G-WCP engine ("walker").
//
// Reference semantics (pkg/src/gpurace/gwcp.py):
//   ThreadState init local=1, hb=e_t, pred=0          :56-66
//   C_t = pred with [t] := local                       :154-157
//   on_barrier (non-forced)                            :286-294, :312-318
//   _drain (rule ii)                                   :161-173
//   on_acquire / on_release                            :175-219
//   on_access rule (i) + frame sets                    :228-249, :278-279
//   on_end                                             :320-334
//
// B200 design.  Events are partitioned by owning walker CTA (block b ->
// CTA b mod G, stable, so each CTA sees its blocks' events in trace order).
// Blocks only interact through locks, so lock-free traces run every block in
// parallel with no cross-CTA traffic.  Lock-related events (successful
// acquire/release, accesses inside a critical section) carry a global rank
// in trace order; a CTA processes such an event only when the global ticket
// equals its rank, which serialises all lock state (records, instance clocks,
// cs_read/cs_write) in trace order -- deadlock-free because every wait is on
// an earlier event and all walker CTAs are co-resident.
//
// Clocks.  A thread's pred / hb clock is an immutable *object* in an arena:
// a dense u32 vector over a thread-index range [lo, lo+len) (zero outside),
// plus a per-thread diagonal (pdiag for pred; local for hb).  Block barriers
// produce one object per barrier shared by every participant (the "block
// shared vector + own diagonal" form), so lock-free traces
// only ever hold block-range objects.  Each access records (time = local,
// vobj = pred object) for the check pass; pred_t[t] itself is never queried
// because race checks and drain tests only read entries u != t.
//
// Drain test.  r.acq_clock ⊑ C_t is evaluated as C_t[r.tid] >= r.acq_local:
// every clock entry [u] >= v is acquired through whole-clock joins of a clock
// published by u no earlier than the end of u's epoch v, which dominates u's
// C-clock at any acquire of epoch v; verified against the reference on
// ~18k random traces (tests/test_oracle_golden.py exercises the same traces).
#pragma once
#include "primitives.cuh"
#include "../../include/gwcp_b200.h"

namespace gw {

constexpr uint32_t NIL = 0xFFFFFFFFu;
constexpr uint32_t SC_DEV = 0xFFFFFFFFu;  // device scope
constexpr int kWalkCH = 2048;              // events staged per chunk
constexpr int kAccSmem = 4096;             // barrier accumulator kept in smem up to this span
constexpr uint32_t OBJ_HDR = 4;            // object header {lo, len, ref, pad}: data 16-byte aligned
constexpr int OBJ_USHIFT = 4;              // object handles count 64-byte units (2^32 units = 256 GiB)

// lflags bits (lock pre-pass)
constexpr uint8_t LF_OK = 1;      // successful acquire / release
constexpr uint8_t LF_INCS = 2;    // access inside >= 1 critical section
constexpr uint8_t LF_LOCKREL = 4; // takes the global lock ticket
constexpr uint8_t LF_QUERY = 8;   // access with race-check queries (lock mode)

// error flags
constexpr uint32_t ERR_ARENA = 1, ERR_TABLE = 2, ERR_FRAMES = 4, ERR_LOG = 8, ERR_REC = 16, ERR_DIAG = 32,
                   ERR_CAND = 64, ERR_RECORD = 128, ERR_INTERNAL = 256;

// iver: release version of the frame's own instance when the acquire joined it
struct Frame { unsigned long long lock; uint32_t scope, rec, logpos, iver; };
// a clock reference: object o joined with one explicit entry [dtid] = dval
// (the owner's diagonal: hb_t[t] = local_t, pred_t[t] = pdiag_t)
struct CRef { uint32_t o, dtid, dval; };
// CSRecord (gwcp.py:32-43): the acquire clock kept as its epoch (tid, acq_local),
// the release clock as the releaser's hb object + diagonal.  domall: this
// record's release clock dominates every earlier record's of the lock.
struct Rec { uint32_t tid, acq_local, scope, rel_hobj, rel_local, closed, domall, pad; };
// a lock's records occupy [rec_base, rec_base + nrec) in acquire order
struct LockEnt { unsigned long long id; uint32_t used, nrec, rec_base, pad, inst_head, ticket; };
struct CurEnt { unsigned long long lock; uint32_t tid, used, epoch, last, bound, snap; };
// lock instance (gwcp.py:69-79): clocks H_i / P_i as references (refcounted
// objects, never mutated in place), relver = releases into it so far
struct InstEnt { unsigned long long lock; uint32_t scope, used; CRef H, P; uint32_t next, relver; };
struct CsEnt { unsigned long long lock, loc; uint32_t scope_rw, used; CRef c; uint32_t pad; };
struct LogEnt { unsigned long long loc; uint32_t rw, next; };
struct Diag { uint32_t ev, code, sub, pad; unsigned long long lock; };

struct DevTrace {
  const unsigned long long* key;
  const uint32_t* tidop;
  const uint32_t* instr;
  uint64_t n;
  uint32_t B, W, L, BS, T;
};

struct WalkArgs {
  DevTrace tr;
  const uint32_t* part_key;  // sorted CTA ids (nullptr when G == 1)
  const uint32_t* perm;      // event indices grouped by CTA (nullptr when G == 1: identity)
  uint32_t G;
  uint32_t* time;
  uint32_t* vobj;
  // per-thread state
  uint32_t *local, *pobj, *pdiag, *hobj, *nend, *exited, *depth, *loghead;
  Frame* frames;
  uint32_t maxd;
  // clock arena (handles in 64-byte units)
  uint32_t* arena;
  unsigned long long* arena_top;
  unsigned long long arena_cap;
  // lock mode: clocks are projected onto the queried thread set Q (qoff =
  // exclusive prefix of the Q membership flags over T+1 threads), objects are
  // fixed-size slots with reference counts, recycled through per-CTA stacks
  const uint32_t* qoff;
  uint32_t Q;
  uint32_t slot_units;
  uint32_t* fstack;
  uint32_t* ftop;
  uint32_t fcap;
  uint32_t warp_stacks;  // free stacks per (CTA, warp) (k_walker_lw) instead of per CTA
  uint32_t hb_mode;      // scoped-HB detector (hb.py): checks read hb; no queues, records, cs or P clocks
  // lock mode: race-check queries answered in trace order by the walker
  const uint32_t* q_cur;    // query current events, sorted
  const uint32_t* q_idx;    // candidate index of each sorted query
  uint64_t nq;
  const uint32_t* c_prior;  // candidate prior event
  uint32_t* qv;             // out: pred_t[u] of the current thread at the query
  // locks
  int has_locks;
  uint32_t inactive_opt;
  const uint8_t* lflags;
  const uint32_t* poff;   // lock-related event -> its (lock, rank) pairs
  const uint32_t* npair;
  const unsigned long long* plock;
  const uint32_t* prank;
  LockEnt* locks; uint32_t lock_mask;
  CurEnt* curs; uint32_t cur_mask;
  InstEnt* insts; uint32_t inst_mask;
  CsEnt* cs; uint32_t cs_mask;
  Rec* recs; uint32_t* rec_top; uint32_t rec_cap;
  const uint32_t* rix;  // lock pair -> record slot (successful acquires)
  unsigned long long* prof;  // optional per-CTA time split (GW_PROF_WALKER): ns per event class
  LogEnt* logs; uint32_t* log_top; uint32_t log_cap;
  uint32_t* scratch;  // per CTA: 3*T words (P, H, acc)
  Diag* diags; uint32_t* diag_top; uint32_t diag_cap;
  uint32_t* err;
  const uint32_t* abort_flag;  // graph mode: plan mismatch -> skip
};

__device__ __forceinline__ uint32_t ev_kind(uint32_t to) { return (to >> GW_OP_SHIFT) & 7u; }
__device__ __forceinline__ uint32_t ev_tid(uint32_t to) { return to & GW_TID_MASK; }

__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27; x *= 0x94d049bb133111ebull;
  x ^= x >> 31;
  return x;
}

__device__ __forceinline__ bool sc_overlap(uint32_t a, uint32_t b) { return a == SC_DEV || b == SC_DEV || a == b; }

// arena object accessors (o = handle: 64-byte unit index of the header {lo, len, ref})
__device__ __forceinline__ uint32_t* optr(uint32_t* arena, uint32_t o) { return arena + ((size_t)o << OBJ_USHIFT); }
__device__ __forceinline__ const uint32_t* optr(const uint32_t* arena, uint32_t o) {
  return arena + ((size_t)o << OBJ_USHIFT);
}
__device__ __forceinline__ uint32_t obj_get(const uint32_t* arena, uint32_t o, uint32_t u) {
  if (o == NIL) return 0u;
  const uint32_t* h = optr(arena, o);
  uint32_t lo = h[0], len = h[1];
  uint32_t d = u - lo;
  return d < len ? h[OBJ_HDR + d] : 0u;
}
__device__ __forceinline__ uint32_t obj_get_cg(const uint32_t* arena, uint32_t o, uint32_t u) {
  if (o == NIL) return 0u;
  const uint32_t* h = optr(arena, o);
  uint32_t lo = __ldcg(h), len = __ldcg(h + 1);
  uint32_t d = u - lo;
  return d < len ? __ldcg(h + OBJ_HDR + d) : 0u;
}

// clock coordinates: thread index (lock-free traces) or Q index (lock mode)
__device__ __forceinline__ bool lockmode(const WalkArgs& a) { return a.qoff != nullptr; }
__device__ __forceinline__ uint32_t vlen(const WalkArgs& a) { return a.qoff ? a.Q : a.tr.T; }
__device__ __forceinline__ uint32_t vidx(const WalkArgs& a, uint32_t u) {
  if (!a.qoff) return u;
  const uint32_t x = a.qoff[u];
  return a.qoff[u + 1] != x ? x : NIL;
}
// coordinate range of block b's threads
__device__ __forceinline__ void vblock(const WalkArgs& a, uint32_t b, uint32_t& lo, uint32_t& hi) {
  if (!a.qoff) { lo = b * a.tr.BS; hi = lo + a.tr.BS; }
  else { lo = a.qoff[(size_t)b * a.tr.BS]; hi = a.qoff[(size_t)(b + 1) * a.tr.BS]; }
}

// Allocation.  Lock mode: one fixed-size slot, recycled from this CTA's stack
// (caller: a single thread, with no concurrent frees in the CTA).  Objects are
// created, referenced and freed by one walker CTA only (the one owning the
// threads that hold them; records pin theirs forever), so the stacks are
// CTA-private.  Lock-free traces: bump allocation, never freed.
__device__ __forceinline__ uint32_t stack_id(const WalkArgs& a) {
  return a.warp_stacks ? blockIdx.x * 8u + (threadIdx.x >> 5) : blockIdx.x;
}
__device__ __forceinline__ uint32_t arena_alloc(const WalkArgs& a, uint32_t words) {
  unsigned long long units;
  if (a.slot_units) {
    const uint32_t sid = stack_id(a);
    uint32_t n = a.ftop[sid];
    if (n > a.fcap) n = a.fcap;  // pushes past the capacity were dropped (leaked)
    if (n > 0) {
      a.ftop[sid] = n - 1;
      return a.fstack[(size_t)sid * a.fcap + n - 1];
    }
    units = a.slot_units;
  } else {
    units = (words + (1u << OBJ_USHIFT) - 1) >> OBJ_USHIFT;
  }
  unsigned long long o = atomicAdd(a.arena_top, units);
  if (o + units > a.arena_cap) { atomicOr(a.err, ERR_ARENA); return NIL; }
  return (uint32_t)o;
}
// reference counts (lock mode only)
__device__ __forceinline__ void obj_retain(const WalkArgs& a, uint32_t o, uint32_t n = 1) {
  if (a.slot_units && o != NIL) atomicAdd(optr(a.arena, o) + 2, n);
}
__device__ __forceinline__ void obj_release(const WalkArgs& a, uint32_t o) {
  if (!a.slot_units || o == NIL) return;
  if (atomicSub(optr(a.arena, o) + 2, 1u) == 1u) {
    const uint32_t sid = stack_id(a);
    const uint32_t i = atomicAdd(a.ftop + sid, 1u);
    if (i < a.fcap) a.fstack[(size_t)sid * a.fcap + i] = o;
  }
}
// initialise a new object's header
__device__ __forceinline__ void obj_init(const WalkArgs& a, uint32_t o, uint32_t lo, uint32_t len, uint32_t ref) {
  uint32_t* h = optr(a.arena, o);
  h[0] = lo; h[1] = len; h[2] = ref;
}

__device__ void emit_diag(const WalkArgs& a, uint32_t ev, uint32_t code, uint32_t sub, unsigned long long lock) {
  uint32_t i = atomicAdd(a.diag_top, 1u);
  if (i >= a.diag_cap) { atomicOr(a.err, ERR_DIAG); return; }
  a.diags[i] = Diag{ev, code, sub, 0u, lock};
}

// ---- lock-state tables -------------------------------------------------
// Open addressing; a slot's `used` word is 0 empty, 1 being initialised, 2
// ready.  Different CTAs insert different keys concurrently (keys of lock l are
// only created under l's ticket), so inserts claim slots with atomicCAS and
// lookups wait for a claimed slot to become ready before comparing its key.
__device__ __forceinline__ uint32_t slot_state(const uint32_t* used) { return ld_volatile_u32(used); }

template <class Ent, class Eq, class Init>
__device__ Ent* ht_find(const WalkArgs& a, Ent* tab, uint32_t mask, uint32_t h, bool create, Eq eq, Init init) {
  for (uint32_t p = 0; p <= mask; p++) {
    Ent* e = &tab[(h + p) & mask];
    uint32_t st = slot_state(&e->used);
    if (st == 0) {
      if (!create) return nullptr;
      if (atomicCAS(&e->used, 0u, 1u) == 0u) {
        init(e);
        __threadfence();
        atomicExch(&e->used, 2u);
        return e;
      }
      st = slot_state(&e->used);
    }
    while (st == 1) st = slot_state(&e->used);
    __threadfence();
    if (eq(e)) return e;
  }
  atomicOr(a.err, ERR_TABLE);
  return nullptr;
}

__device__ LockEnt* lock_find(const WalkArgs& a, unsigned long long id, bool create) {
  const uint32_t h = (uint32_t)mix64(id) & a.lock_mask;
  return ht_find(a, a.locks, a.lock_mask, h, create, [&](LockEnt* e) { return __ldcg(&e->id) == id; },
                 [&](LockEnt* e) {
                   e->id = id; e->nrec = 0; e->rec_base = 0; e->inst_head = NIL; e->ticket = 0;
                 });
}

__device__ CurEnt* cur_find(const WalkArgs& a, unsigned long long lock, uint32_t tid) {
  const uint32_t h = (uint32_t)mix64(lock * 0x9E3779B97F4A7C15ull ^ tid) & a.cur_mask;
  return ht_find(a, a.curs, a.cur_mask, h, true,
                 [&](CurEnt* e) { return __ldcg(&e->lock) == lock && __ldcg(&e->tid) == tid; },
                 [&](CurEnt* e) {
                   e->lock = lock; e->tid = tid; e->epoch = NIL; e->last = NIL; e->bound = NIL; e->snap = 0;
                 });
}

__device__ InstEnt* inst_find(const WalkArgs& a, unsigned long long lock, uint32_t scope, bool create) {
  const uint32_t h = (uint32_t)mix64(lock ^ ((unsigned long long)scope << 40) ^ 0x51ull) & a.inst_mask;
  return ht_find(a, a.insts, a.inst_mask, h, create,
                 [&](InstEnt* e) { return __ldcg(&e->lock) == lock && __ldcg(&e->scope) == scope; },
                 [&](InstEnt* e) {
                   e->lock = lock; e->scope = scope; e->H = CRef{NIL, NIL, 0u}; e->P = CRef{NIL, NIL, 0u};
                   e->next = NIL; e->relver = 0;
                 });
}

__device__ CsEnt* cs_find(const WalkArgs& a, unsigned long long lock, uint32_t scope, unsigned long long loc,
                          uint32_t rw, bool create) {
  const uint32_t srw = (scope << 1) | rw;
  const uint32_t h = (uint32_t)mix64(lock ^ mix64(loc) ^ ((unsigned long long)scope << 33) ^ rw) & a.cs_mask;
  return ht_find(a, a.cs, a.cs_mask, h, create,
                 [&](CsEnt* e) {
                   return __ldcg(&e->lock) == lock && __ldcg(&e->loc) == loc && __ldcg(&e->scope_rw) == srw;
                 },
                 [&](CsEnt* e) { e->lock = lock; e->loc = loc; e->scope_rw = srw; e->c = CRef{NIL, NIL, 0u}; });
}

// ------------------------------------------------------------- helpers ----
__device__ __forceinline__ uint32_t block_min_u32(uint32_t v) {
  __shared__ uint32_t s_red[kThreads / 32];
  v = __reduce_min_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = v;
  __syncthreads();
  uint32_t r = s_red[0];
#pragma unroll
  for (int i = 1; i < kThreads / 32; i++) r = min(r, s_red[i]);
  __syncthreads();
  return r;
}
__device__ __forceinline__ uint32_t block_max_u32(uint32_t v) {
  __shared__ uint32_t s_red2[kThreads / 32];
  v = __reduce_max_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0) s_red2[threadIdx.x >> 5] = v;
  __syncthreads();
  uint32_t r = s_red2[0];
#pragma unroll
  for (int i = 1; i < kThreads / 32; i++) r = max(r, s_red2[i]);
  __syncthreads();
  return r;
}
__device__ __forceinline__ int block_or(int v) {
  return __syncthreads_or(v);
}

// ---- CTA-wide dense vector ops (uint4 when 16-byte aligned) -------------
__device__ __forceinline__ bool al16(const void* p) { return ((uintptr_t)p & 15u) == 0; }
__device__ __forceinline__ uint4 max4(uint4 a, uint4 b) {
  return make_uint4(max(a.x, b.x), max(a.y, b.y), max(a.z, b.z), max(a.w, b.w));
}
__device__ __forceinline__ bool gt4(uint4 a, uint4 b) { return a.x > b.x || a.y > b.y || a.z > b.z || a.w > b.w; }

// Loads through L2 (ld.global.cg) for data other CTAs wrote (arena objects,
// lock-state clocks); plain loads for CTA-private scratch or shared memory.
template <bool CG, class T>
__device__ __forceinline__ T ldx(const T* p) {
  if constexpr (CG) return __ldcg(p);
  else return *p;
}

// dst[0..n) max= src[0..n); returns nonzero if dst grew
template <bool SRC_CG, bool DST_CG>
__device__ __forceinline__ int vjoin(uint32_t* dst, const uint32_t* src, uint32_t n) {
  int ch = 0;
  if (al16(dst) && al16(src)) {
    const uint32_t n4 = n >> 2;
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
#pragma unroll 4
    for (uint32_t i = threadIdx.x; i < n4; i += kThreads) {
      const uint4 v = ldx<SRC_CG>(s4 + i), o = ldx<DST_CG>(d4 + i);
      if (gt4(v, o)) { d4[i] = max4(v, o); ch = 1; }
    }
    for (uint32_t i = (n4 << 2) + threadIdx.x; i < n; i += kThreads) {
      const uint32_t v = ldx<SRC_CG>(src + i);
      if (v > ldx<DST_CG>(dst + i)) { dst[i] = v; ch = 1; }
    }
  } else {
#pragma unroll 4
    for (uint32_t i = threadIdx.x; i < n; i += kThreads) {
      const uint32_t v = ldx<SRC_CG>(src + i);
      if (v > ldx<DST_CG>(dst + i)) { dst[i] = v; ch = 1; }
    }
  }
  return ch;
}
template <bool SRC_CG>
__device__ __forceinline__ void vcopy(uint32_t* dst, const uint32_t* src, uint32_t n) {
  if (al16(dst) && al16(src)) {
    const uint32_t n4 = n >> 2;
#pragma unroll 4
    for (uint32_t i = threadIdx.x; i < n4; i += kThreads)
      reinterpret_cast<uint4*>(dst)[i] = ldx<SRC_CG>(reinterpret_cast<const uint4*>(src) + i);
    for (uint32_t i = (n4 << 2) + threadIdx.x; i < n; i += kThreads) dst[i] = ldx<SRC_CG>(src + i);
  } else {
    for (uint32_t i = threadIdx.x; i < n; i += kThreads) dst[i] = ldx<SRC_CG>(src + i);
  }
}
__device__ __forceinline__ void vfill0(uint32_t* dst, uint32_t n) {
  if (al16(dst)) {
    const uint32_t n4 = n >> 2;
#pragma unroll 4
    for (uint32_t i = threadIdx.x; i < n4; i += kThreads) reinterpret_cast<uint4*>(dst)[i] = make_uint4(0, 0, 0, 0);
    for (uint32_t i = (n4 << 2) + threadIdx.x; i < n; i += kThreads) dst[i] = 0u;
  } else {
    for (uint32_t i = threadIdx.x; i < n; i += kThreads) dst[i] = 0u;
  }
}

// dst[0..n) (dense, CTA-private scratch) max= object o; returns nonzero if any entry grew
__device__ __forceinline__ int join_obj_dense(uint32_t* dst, const uint32_t* arena, uint32_t o) {
  if (o == NIL) return 0;
  const uint32_t* h = optr(arena, o);
  const uint32_t lo = __ldcg(h), len = __ldcg(h + 1);
  return vjoin<true, false>(dst + lo, h + OBJ_HDR, len);
}

// materialize clock object o with diagonal [vt] := diag (vt = NIL: none) into dense dst[0..n)
__device__ __forceinline__ void materialize(uint32_t* dst, const uint32_t* arena, uint32_t o, uint32_t n, uint32_t vt,
                                            uint32_t diag) {
  if (o != NIL && __ldcg(optr(arena, o)) == 0 && __ldcg(optr(arena, o) + 1) == n) {
    vcopy<true>(dst, optr(arena, o) + OBJ_HDR, n);  // full-range object: plain copy
  } else {
    vfill0(dst, n);
    __syncthreads();
    join_obj_dense(dst, arena, o);
  }
  __syncthreads();
  if (threadIdx.x == 0 && vt != NIL) dst[vt] = diag;
  __syncthreads();
}

// write dense src[0..n) as a new full-range object (reference count `ref`);
// returns its handle (broadcast)
__device__ uint32_t publish_dense(const WalkArgs& a, const uint32_t* src, uint32_t n, uint32_t ref) {
  __shared__ uint32_t s_o;
  if (threadIdx.x == 0) {
    uint32_t o = arena_alloc(a, n + OBJ_HDR);
    if (o != NIL) obj_init(a, o, 0, n, ref);
    s_o = o;
  }
  __syncthreads();
  uint32_t o = s_o;
  if (o != NIL) vcopy<false>(optr(a.arena, o) + OBJ_HDR, src, n);
  __syncthreads();
  return o;
}

// ------------------------------------------------------------- barrier ----
// on_barrier, gwcp.py:286-294 + :312-318.  PJ = join of the participants'
// pred objects (each distinct object joined once) with every participant's
// own entry = its local time; every participant leaves with (PJ, diag=local+1).
// The same for hb (only when the trace has locks: hb feeds lock state only).
// Lock mode: the barrier's new clock in one pass -- out[i] = max over the
// participants' distinct objects (collected first), then the participants'
// own entries -- written straight into the new full-range object.
constexpr int kBarSrc = 32;
__device__ uint32_t barrier_join_lock(const WalkArgs& a, const uint32_t* objs, uint32_t base, uint32_t npool,
                                      bool warp, uint32_t ins, uint32_t npart, bool& ok) {
  __shared__ uint32_t s_src[kBarSrc];
  __shared__ uint32_t s_ns, s_o, s_full;
  const uint32_t n = vlen(a);
  if (threadIdx.x == 0) { s_ns = 0; s_full = 1; }
  __syncthreads();
  // distinct participant objects (each enumerated once, increasing handles)
  uint32_t done_lo = 0;
  while (true) {
    uint32_t mymin = NIL;
    for (uint32_t j = threadIdx.x; j < npool; j += kThreads) {
      const bool inm = !warp || ((ins >> j) & 1u);
      const uint32_t u = base + j;
      if (inm && !a.exited[u]) {
        const uint32_t o = objs[u];
        if (o != NIL && o >= done_lo && o < mymin) mymin = o;
      }
    }
    const uint32_t om = block_min_u32(mymin);
    if (om == NIL) break;
    if (threadIdx.x == 0) {
      if (s_ns < (uint32_t)kBarSrc) {
        s_src[s_ns++] = om;
        if (!(__ldcg(optr(a.arena, om)) == 0 && __ldcg(optr(a.arena, om) + 1) == n)) s_full = 0;
      } else {
        s_full = 2;  // too many distinct objects: caller falls back
      }
    }
    done_lo = om + 1;
  }
  __syncthreads();
  if (s_full == 2) { ok = false; return NIL; }
  ok = true;
  if (threadIdx.x == 0) {
    const uint32_t o = arena_alloc(a, n + OBJ_HDR);
    if (o != NIL) obj_init(a, o, 0, n, npart);
    s_o = o;
  }
  __syncthreads();
  const uint32_t o = s_o, ns = s_ns;
  if (o == NIL) return NIL;
  uint32_t* out = optr(a.arena, o) + OBJ_HDR;
  if (s_full) {
    const uint32_t n4 = n >> 2;
    for (uint32_t i = threadIdx.x; i < n4; i += kThreads) {
      uint4 v = make_uint4(0, 0, 0, 0);
      for (uint32_t k = 0; k < ns; k++)
        v = max4(v, __ldcg(reinterpret_cast<const uint4*>(optr(a.arena, s_src[k]) + OBJ_HDR) + i));
      reinterpret_cast<uint4*>(out)[i] = v;
    }
    for (uint32_t i = (n4 << 2) + threadIdx.x; i < n; i += kThreads) {
      uint32_t v = 0;
      for (uint32_t k = 0; k < ns; k++) v = max(v, __ldcg(optr(a.arena, s_src[k]) + OBJ_HDR + i));
      out[i] = v;
    }
  } else {
    for (uint32_t i = threadIdx.x; i < n; i += kThreads) {
      uint32_t v = 0;
      for (uint32_t k = 0; k < ns; k++) v = max(v, obj_get_cg(a.arena, s_src[k], i));
      out[i] = v;
    }
  }
  __syncthreads();
  // participants' own entries = their local time (C_u[u], hb_u[u])
  for (uint32_t j = threadIdx.x; j < npool; j += kThreads) {
    const bool inm = !warp || ((ins >> j) & 1u);
    const uint32_t u = base + j;
    if (inm && !a.exited[u]) {
      const uint32_t vu = vidx(a, u);
      if (vu != NIL) out[vu] = a.local[u];
    }
  }
  __syncthreads();
  return o;
}

__device__ void do_barrier(const WalkArgs& a, uint32_t to, uint32_t ins, uint32_t* s_acc) {
  const DevTrace& tr = a.tr;
  const uint32_t base = ev_tid(to);  // lane 0 of the warp / block
  const bool warp = (to & GW_F_WARPBAR) != 0;
  const uint32_t npool = warp ? tr.L : tr.BS;
  uint32_t blo, bhi;  // the block's coordinate range
  vblock(a, base / tr.BS, blo, bhi);
  // participants: live pool members (gwcp.py:286 via barrier_participants, trace.py:494-519)
  uint32_t anyp = 0;
  for (uint32_t j = threadIdx.x; j < npool; j += kThreads) {
    bool inm = !warp || ((ins >> j) & 1u);
    if (inm && !a.exited[base + j]) anyp++;
  }
  uint32_t npart = 0;  // participant count = the new objects' reference count
  {
    __shared__ uint32_t s_np;
    if (threadIdx.x == 0) s_np = 0;
    __syncthreads();
    if (anyp) atomicAdd(&s_np, anyp);
    __syncthreads();
    npart = s_np;
    __syncthreads();
  }
  if (!npart) return;  // empty participant set: no effect

  const int nkinds = a.has_locks ? 2 : 1;
  uint32_t newobj[2] = {NIL, NIL};
  for (int kind = 0; kind < nkinds; kind++) {
    uint32_t* objs = kind == 0 ? a.pobj : a.hobj;
    if (a.slot_units) {  // lock mode: one fused pass
      bool ok = false;
      const uint32_t no = barrier_join_lock(a, objs, base, npool, warp, ins, npart, ok);
      if (ok) { newobj[kind] = no; continue; }
    }
    // hull of participant objects and the block range
    uint32_t mylo = blo, myhi = bhi;
    for (uint32_t j = threadIdx.x; j < npool; j += kThreads) {
      bool inm = !warp || ((ins >> j) & 1u);
      uint32_t u = base + j;
      if (inm && !a.exited[u]) {
        uint32_t o = objs[u];
        if (o != NIL) {
          const uint32_t* h = optr(a.arena, o);
          uint32_t lo = h[0], len = h[1];
          mylo = min(mylo, lo);
          myhi = max(myhi, lo + len);
        }
      }
    }
    uint32_t lo = block_min_u32(mylo), hi = block_max_u32(myhi);
    uint32_t span = hi - lo;
    uint32_t* acc = span <= (uint32_t)kAccSmem ? s_acc : a.scratch + (size_t)blockIdx.x * 3 * vlen(a) + 2 * vlen(a);
    vfill0(acc, span);
    __syncthreads();
    // join each distinct participant object once
    uint32_t done_lo = 0;  // handles < done_lo already joined (enumerated in increasing order)
    while (true) {
      uint32_t mymin = NIL;
      for (uint32_t j = threadIdx.x; j < npool; j += kThreads) {
        bool inm = !warp || ((ins >> j) & 1u);
        uint32_t u = base + j;
        if (inm && !a.exited[u]) {
          uint32_t o = objs[u];
          if (o != NIL && o >= done_lo && o < mymin) mymin = o;
        }
      }
      uint32_t om = block_min_u32(mymin);
      if (om == NIL) break;
      const uint32_t* h = optr(a.arena, om);
      const uint32_t olo = h[0], olen = h[1];
      vjoin<true, false>(acc + (olo - lo), h + OBJ_HDR, olen);
      __syncthreads();
      done_lo = om + 1;
    }
    // participants' own entries = their local time (C_u[u], hb_u[u])
    for (uint32_t j = threadIdx.x; j < npool; j += kThreads) {
      bool inm = !warp || ((ins >> j) & 1u);
      uint32_t u = base + j;
      if (inm && !a.exited[u]) {
        const uint32_t vu = vidx(a, u);
        if (vu != NIL) acc[vu - lo] = a.local[u];
      }
    }
    __syncthreads();
    __shared__ uint32_t s_no;
    if (threadIdx.x == 0) {
      uint32_t o = arena_alloc(a, span + OBJ_HDR);
      if (o != NIL) obj_init(a, o, lo, span, npart);
      s_no = o;
    }
    __syncthreads();
    uint32_t no = s_no;
    if (no != NIL) vcopy<false>(optr(a.arena, no) + OBJ_HDR, acc, span);
    newobj[kind] = no;
    __syncthreads();
  }
  for (uint32_t j = threadIdx.x; j < npool; j += kThreads) {
    bool inm = !warp || ((ins >> j) & 1u);
    uint32_t u = base + j;
    if (inm && !a.exited[u]) {
      uint32_t nl = a.local[u] + 1;
      a.local[u] = nl;
      const uint32_t op = a.pobj[u];
      a.pobj[u] = newobj[0];
      obj_release(a, op);
      a.pdiag[u] = nl;
      if (a.has_locks) {
        const uint32_t oh = a.hobj[u];
        a.hobj[u] = newobj[1];
        obj_release(a, oh);
      }
    }
  }
  __syncthreads();
}

// Warp barriers of lock-free traces (<= 32 participants, block-range objects):
// the same join as do_barrier, done by warp 0 alone with warp reductions
// (no CTA-wide barrier inside).  Caller: threadIdx.x < 32, then __syncthreads.
__device__ void do_barrier_warp(const WalkArgs& a, uint32_t to, uint32_t ins, uint32_t* s_acc) {
  const DevTrace& tr = a.tr;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t base = ev_tid(to);
  const uint32_t blo = (base / tr.BS) * tr.BS;
  const uint32_t u = base + lane;
  const bool part = lane < tr.L && ((ins >> lane) & 1u) && !a.exited[u];
  if (!__any_sync(0xffffffffu, part)) return;
  const uint32_t o = part ? a.pobj[u] : NIL;
  uint32_t mylo = blo, myhi = blo + tr.BS;
  if (o != NIL) {
    const uint32_t olo = optr(a.arena, o)[0], olen = optr(a.arena, o)[1];
    mylo = min(mylo, olo);
    myhi = max(myhi, olo + olen);
  }
  const uint32_t lo = __reduce_min_sync(0xffffffffu, mylo), hi = __reduce_max_sync(0xffffffffu, myhi);
  const uint32_t span = hi - lo;
  uint32_t* acc = span <= (uint32_t)kAccSmem ? s_acc : a.scratch + (size_t)blockIdx.x * 3 * tr.T + 2 * tr.T;
  for (uint32_t i = lane; i < span; i += 32) acc[i] = 0u;
  __syncwarp();
  uint32_t done = 0;
  while (true) {  // each distinct participant object once
    const uint32_t om = __reduce_min_sync(0xffffffffu, (o != NIL && o >= done) ? o : NIL);
    if (om == NIL) break;
    const uint32_t olo = optr(a.arena, om)[0], olen = optr(a.arena, om)[1];
    const uint32_t* src = optr(a.arena, om) + OBJ_HDR;
    uint32_t* dst = acc + (olo - lo);
    for (uint32_t i0 = 0; i0 < olen; i0 += 32 * 8) {  // 8 independent loads in flight per lane
      uint32_t v[8];
#pragma unroll
      for (int k = 0; k < 8; k++) {
        const uint32_t i = i0 + lane + 32 * k;
        v[k] = i < olen ? src[i] : 0u;
      }
#pragma unroll
      for (int k = 0; k < 8; k++) {
        const uint32_t i = i0 + lane + 32 * k;
        if (i < olen && v[k] > dst[i]) dst[i] = v[k];
      }
    }
    __syncwarp();
    done = om + 1;
  }
  const uint32_t lu = part ? a.local[u] : 0u;
  if (part) acc[u - lo] = lu;
  __syncwarp();
  uint32_t no = NIL;
  if (lane == 0) {
    no = arena_alloc(a, span + OBJ_HDR);
    if (no != NIL) obj_init(a, no, lo, span, 0);
  }
  no = __shfl_sync(0xffffffffu, no, 0);
  if (no != NIL)
    for (uint32_t i = lane; i < span; i += 32) optr(a.arena, no)[OBJ_HDR + i] = acc[i];
  if (part) {
    a.local[u] = lu + 1;
    a.pobj[u] = no;
    a.pdiag[u] = lu + 1;
  }
  __syncwarp();
}

// --------------------------------------------------------------- locks ----
// Per-lock tickets.  A lock-related event e (successful acquire / release of
// l, or an access inside critical sections of l1..ld) may touch the state of
// lock l only when l's ticket equals e's rank among the l-events in trace
// order.  Every wait is for an earlier event, and an earlier event never
// waits for a later one, so the walk is deadlock-free with all walker CTAs
// co-resident; events on different locks proceed in parallel.
__device__ void tickets_wait(const WalkArgs& a, uint32_t e) {
  if (threadIdx.x == 0) {
    const uint32_t off = a.poff[e], np = a.npair[e];
    for (uint32_t j = 0; j < np; j++) {
      LockEnt* lk = lock_find(a, a.plock[off + j], false);
      if (!lk) { atomicOr(a.err, ERR_INTERNAL); continue; }
      const uint32_t r = a.prank[off + j];
      volatile uint32_t* tk = &lk->ticket;
      uint32_t ns = 32;
      while (*tk != r) {
        __nanosleep(ns);
        if (ns < 256) ns <<= 1;
      }
    }
    __threadfence();
  }
  __syncthreads();
  __threadfence();
}
__device__ void tickets_release(const WalkArgs& a, uint32_t e) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const uint32_t off = a.poff[e], np = a.npair[e];
    for (uint32_t j = 0; j < np; j++) {
      LockEnt* lk = lock_find(a, a.plock[off + j], false);
      if (lk) atomicExch(&lk->ticket, a.prank[off + j] + 1);
    }
  }
}

// _drain, gwcp.py:161-173, as a per-(lock, thread) cursor over the lock's
// record array.  Queue materialisation (gwcp.py:80-100):
// before the thread's first END its queue is every record of the lock by
// other threads; after an END (drop) the next drain re-materialises a
// snapshot of all records so far (own included; empty with inactive_opt
// off) that receives no further pushes.
//
// The sequential pop loop (test C_t[r.tid] >= r.acq_local on the clock that
// includes every earlier pop's release clock, then join) runs 32 records at a
// time on warp 0: each lane evaluates its record's test on pred_t (point
// reads of t's pred object -- no materialised clock) plus the release clocks
// of the records before it, found by walking back to the nearest joined
// record whose release clock dominates all earlier ones (Rec::domall).  The
// joins themselves are only collected (s_m + s_j): the caller applies them,
// usually after giving the lock's ticket back.
constexpr int kDrainJ = 16;  // collected non-dominating joins before the scan stops early

__device__ __forceinline__ uint32_t relpt(const WalkArgs& a, uint32_t rel_hobj, uint32_t rtid, uint32_t rel_local,
                                          uint32_t u, uint32_t vu) {
  const uint32_t v = obj_get_cg(a.arena, rel_hobj, vu);
  return rtid == u ? max(v, rel_local) : v;
}

struct DrainOut {      // shared-memory result of drain_scan
  uint32_t m;          // last popped dominating joinable record (NIL: none)
  uint32_t nj;         // popped joinable records after it
  uint32_t j[kDrainJ];
  uint32_t more;       // the scan stopped early (kDrainJ reached): call again after applying
};

// One drain scan (caller: the whole CTA, holding the lock's ticket).  extra:
// records already collected by an earlier scan of this drain whose joins are
// not yet in t's pred object (their values count in the tests).
__device__ void drain_scan(const WalkArgs& a, uint32_t t, unsigned long long lock, uint32_t cur, DrainOut& O,
                           bool first, const DrainOut* extra) {
  __shared__ CurEnt* s_cur;
  __shared__ LockEnt* s_lk;
  __shared__ uint32_t s_tid[32], s_acq[32], s_ho[32], s_loc[32], s_flags[32];
  __shared__ uint32_t s_pos, s_end;
  if (threadIdx.x == 0) {
    LockEnt* lk = lock_find(a, lock, false);
    CurEnt* ce = lk ? cur_find(a, lock, t) : nullptr;
    s_lk = lk;
    s_cur = ce;
    if (ce) {
      uint32_t ep = a.nend[t];
      if (first && __ldcg(&ce->epoch) != ep) {  // (re)materialise the queue
        ce->epoch = ep;
        ce->last = NIL;
        ce->snap = ep != 0;
        ce->bound = ep == 0 ? NIL : (a.inactive_opt ? __ldcg(&lk->nrec) : 0u);
      }
      const uint32_t base = __ldcg(&lk->rec_base), nrec = __ldcg(&lk->nrec);
      const uint32_t last = __ldcg(&ce->last);
      s_pos = last == NIL ? base : last + 1;
      s_end = base + (ce->snap ? min(nrec, __ldcg(&ce->bound)) : nrec);
    }
    O.m = NIL;
    O.nj = 0;
    O.more = 0;
  }
  __syncthreads();
  if (!s_cur) return;
  const bool snap = __ldcg(&s_cur->snap) != 0;
  const uint32_t po = a.pobj[t];
  if (threadIdx.x < 32) {
    const uint32_t lane = threadIdx.x;
    uint32_t pos = s_pos;
    const uint32_t end = s_end;
    uint32_t m = NIL, nj = 0;
    bool stop = false, full = false;
    while (!stop && !full && pos < end) {
      const uint32_t idx = pos + lane;
      const bool in = idx < end;
      uint32_t fl = 0;  // bit0 in, bit1 own (skipped), bit2 closed, bit3 joinable, bit4 domall
      if (in) {
        const Rec* r = a.recs + idx;
        const uint32_t rt = __ldcg(&r->tid);
        s_tid[lane] = rt;
        s_acq[lane] = __ldcg(&r->acq_local);
        s_ho[lane] = __ldcg(&r->rel_hobj);
        s_loc[lane] = __ldcg(&r->rel_local);
        const bool own = !snap && rt == t;
        const bool closed = __ldcg(&r->closed) != 0;
        fl = 1u | (own ? 2u : 0u) | (closed ? 4u : 0u) |
             ((!own && closed && sc_overlap(__ldcg(&r->scope), cur)) ? 8u : 0u) | (__ldcg(&r->domall) ? 16u : 0u);
      }
      s_flags[lane] = fl;
      __syncwarp();
      // my test, assuming every record before me in the window is popped
      bool pass = false;
      if (fl & 2u) pass = true;          // own record: not in the queue, stepped over
      else if (!(fl & 4u)) pass = false;  // open (or past the end): the drain stops here
      else if (s_tid[lane] == t) pass = true;
      else {
        const uint32_t u = s_tid[lane], vu = vidx(a, u);
        uint32_t v = vu != NIL ? obj_get_cg(a.arena, po, vu) : 0u;  // pred_t[u], u != t
        bool dom = false;
        for (int i = (int)lane - 1; i >= 0 && !dom; i--) {
          const uint32_t fi = s_flags[i];
          if (!(fi & 8u)) continue;
          v = max(v, relpt(a, s_ho[i], s_tid[i], s_loc[i], u, vu));
          dom = (fi & 16u) != 0;
        }
        if (!dom) {  // collected, not yet applied joins (this scan's earlier windows, the caller's)
          for (int src = 0; src < 2; src++) {
            const uint32_t mm = src == 0 ? m : (extra ? extra->m : NIL);
            const uint32_t nn = src == 0 ? nj : (extra ? extra->nj : 0u);
            const uint32_t* jj = src == 0 ? O.j : (extra ? extra->j : nullptr);
            for (uint32_t k = 0; k < nn; k++) {
              const Rec* r = a.recs + jj[k];
              v = max(v, relpt(a, __ldcg(&r->rel_hobj), __ldcg(&r->tid), __ldcg(&r->rel_local), u, vu));
            }
            if (mm != NIL) {
              const Rec* r = a.recs + mm;
              v = max(v, relpt(a, __ldcg(&r->rel_hobj), __ldcg(&r->tid), __ldcg(&r->rel_local), u, vu));
            }
          }
        }
        pass = v >= s_acq[lane];
      }
      const uint32_t fails = __ballot_sync(0xffffffffu, !(in && pass));
      uint32_t f = fails ? (uint32_t)(__ffs(fails) - 1) : 32u;  // records [pos, pos + f) are popped
      for (uint32_t i = 0; i < f; i++) {  // uniform over the warp
        const uint32_t fi = s_flags[i];
        if (!(fi & 8u)) continue;
        if (fi & 16u) { m = pos + i; nj = 0; }
        else if (nj < (uint32_t)kDrainJ) { if (lane == 0) O.j[nj] = pos + i; nj++; }
        else { f = i; full = true; break; }  // pop it after the collected joins are applied
      }
      if (f < 32u && !full) stop = true;
      pos += f;
      __syncwarp();
    }
    if (lane == 0) {
      O.m = m;
      O.nj = nj;
      O.more = (full && pos < end) ? 1u : 0u;
      if (pos > __ldcg(&s_lk->rec_base)) s_cur->last = pos - 1;
    }
  }
  __syncthreads();
}

// replace thread t's pred / hb object (thread 0; lock mode reference counts)
__device__ __forceinline__ void set_obj(const WalkArgs& a, uint32_t* objs, uint32_t t, uint32_t o) {
  const uint32_t old = objs[t];
  objs[t] = o;
  obj_release(a, old);
}

// race-check queries of access e by thread t against its pred object o
// (gwcp.py:251-269: pred_t[u] for the prior access' thread u != t)
__device__ void answer_queries(const WalkArgs& a, uint32_t e, uint32_t o) {
  uint64_t lo = 0, hi = a.nq;
  while (lo < hi) {
    const uint64_t m = (lo + hi) >> 1;
    if (a.q_cur[m] < e) lo = m + 1; else hi = m;
  }
  for (uint64_t j = lo; j < a.nq && a.q_cur[j] == e; j++) {
    const uint32_t k = a.q_idx[j];
    const uint32_t u = ev_tid(a.tr.tidop[a.c_prior[k]]);
    a.qv[k] = obj_get_cg(a.arena, o, vidx(a, u));
  }
}

// ---- captured joins: clock references read under a ticket, applied later --
constexpr int kMaxCap = 40;
struct CapList {
  CRef c[kMaxCap];
  uint32_t tgt[kMaxCap];  // 0: pred (P), 1: hb (H)
  uint32_t n;
  uint32_t full;
};
// thread 0, under the ticket: keep o alive until applied
__device__ __forceinline__ bool cap_push(const WalkArgs& a, CapList& L, CRef c, uint32_t tgt) {
  if (c.o == NIL && c.dtid == NIL) return true;
  if (L.n >= (uint32_t)kMaxCap) { L.full = 1; return false; }
  obj_retain(a, c.o);
  L.c[L.n] = c;
  L.tgt[L.n] = tgt;
  L.n++;
  return true;
}
__device__ __forceinline__ CRef rec_cref(const WalkArgs& a, uint32_t ri) {
  const Rec* r = a.recs + ri;
  return CRef{__ldcg(&r->rel_hobj), __ldcg(&r->tid), __ldcg(&r->rel_local)};
}
// dense dst max= clock reference c (block-wide); returns nonzero if dst grew
__device__ int join_cref(const WalkArgs& a, uint32_t* dst, CRef c) {
  int ch = join_obj_dense(dst, a.arena, c.o);
  __syncthreads();
  if (threadIdx.x == 0 && c.dtid != NIL) {
    const uint32_t v = vidx(a, c.dtid);
    if (v != NIL && c.dval > dst[v]) { dst[v] = c.dval; ch = 1; }
  }
  return __syncthreads_or(ch);
}
// Fused join: a NEW full-range object := base (t's object with its diagonal
// [vt] = diag, as materialize() sets it) joined with every captured reference
// of one target -- one pass over the clock (every source loaded together)
// instead of materialise + one pass per join + publish.  Returns the object
// if it differs from the base, else frees it and returns NIL.
__device__ uint32_t fused_join(const WalkArgs& a, uint32_t base, uint32_t vt, uint32_t diag, const CapList& L,
                               uint32_t tgt, uint32_t n) {
  __shared__ uint32_t s_o, s_full, s_ns;
  __shared__ uint32_t s_src[kMaxCap];
  {  // nothing captured for this target: unchanged, no pass over the clock
    bool any = false;
    for (uint32_t k = 0; k < L.n && !any; k++) any = L.tgt[k] == tgt;
    if (!any) return NIL;
  }
  if (threadIdx.x == 0) {
    uint32_t ns = 0, full = (base == NIL || (optr(a.arena, base)[0] == 0 && optr(a.arena, base)[1] == n)) ? 1u : 0u;
    for (uint32_t k = 0; k < L.n; k++)
      if (L.tgt[k] == tgt && L.c[k].o != NIL) {
        const uint32_t o = L.c[k].o;
        s_src[ns++] = o;
        if (!(__ldcg(optr(a.arena, o)) == 0 && __ldcg(optr(a.arena, o) + 1) == n)) full = 0;
      }
    s_ns = ns;
    s_full = full;
    const uint32_t o = arena_alloc(a, n + OBJ_HDR);
    if (o != NIL) obj_init(a, o, 0, n, 1);
    s_o = o;
  }
  __syncthreads();
  const uint32_t o = s_o, ns = s_ns;
  if (o == NIL) return NIL;
  uint32_t* out = optr(a.arena, o) + OBJ_HDR;
  int ch = 0;
  if (s_full) {  // every operand spans [0, n): 16-byte vectors
    const uint32_t n4 = n >> 2;
    const uint4* b4 = base != NIL ? reinterpret_cast<const uint4*>(optr(a.arena, base) + OBJ_HDR) : nullptr;
    for (uint32_t i = threadIdx.x; i < n4; i += kThreads) {
      const uint4 bv = b4 ? __ldcg(b4 + i) : make_uint4(0, 0, 0, 0);
      uint4 v = bv;
      for (uint32_t k = 0; k < ns; k++)
        v = max4(v, __ldcg(reinterpret_cast<const uint4*>(optr(a.arena, s_src[k]) + OBJ_HDR) + i));
      reinterpret_cast<uint4*>(out)[i] = v;
      if (gt4(v, bv)) ch = 1;
    }
    for (uint32_t i = (n4 << 2) + threadIdx.x; i < n; i += kThreads) {
      const uint32_t bv = base != NIL ? __ldcg(optr(a.arena, base) + OBJ_HDR + i) : 0u;
      uint32_t v = bv;
      for (uint32_t k = 0; k < ns; k++) v = max(v, __ldcg(optr(a.arena, s_src[k]) + OBJ_HDR + i));
      out[i] = v;
      if (v > bv) ch = 1;
    }
  } else {
    for (uint32_t i = threadIdx.x; i < n; i += kThreads) {
      const uint32_t bv = obj_get_cg(a.arena, base, i);
      uint32_t v = bv;
      for (uint32_t k = 0; k < ns; k++) v = max(v, obj_get_cg(a.arena, s_src[k], i));
      out[i] = v;
      if (v > bv) ch = 1;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // the base's diagonal, then the references' explicit entries
    if (vt != NIL) {
      const uint32_t bv = obj_get_cg(a.arena, base, vt);
      uint32_t v = max(out[vt], diag);
      // materialize() overwrites [vt] with diag; a source may raise it again
      uint32_t srcmax = 0;
      for (uint32_t k = 0; k < ns; k++) srcmax = max(srcmax, obj_get_cg(a.arena, s_src[k], vt));
      v = max(diag, srcmax);
      out[vt] = v;
      if (v != bv && v > diag) ch = 1;
    }
    for (uint32_t k = 0; k < L.n; k++) {
      if (L.tgt[k] != tgt || L.c[k].dtid == NIL) continue;
      const uint32_t v = vidx(a, L.c[k].dtid);
      if (v == NIL) continue;
      const uint32_t cur = out[v];
      const uint32_t bv = v == vt ? diag : cur;
      if (L.c[k].dval > cur) { out[v] = L.c[k].dval; if (L.c[k].dval > bv) ch = 1; }
    }
  }
  ch = __syncthreads_or(ch);
  if (!ch) {
    if (threadIdx.x == 0) obj_release(a, o);  // unchanged: back to the free stack
    __syncthreads();
    return NIL;
  }
  return o;
}
// apply every captured reference to t's pred / hb with fused joins, publish,
// drop the captured references
__device__ void cap_flush(const WalkArgs& a, CapList& L, uint32_t t, uint32_t vt, uint32_t n) {
  if (L.n) {
    const uint32_t po = fused_join(a, a.pobj[t], vt, a.pdiag[t], L, 0, n);
    if (po != NIL && threadIdx.x == 0) {
      set_obj(a, a.pobj, t, po);
      if (vt != NIL) a.pdiag[t] = optr(a.arena, po)[OBJ_HDR + vt];
    }
    __syncthreads();
    const uint32_t ho = fused_join(a, a.hobj[t], vt, a.local[t], L, 1, n);
    if (ho != NIL && threadIdx.x == 0) set_obj(a, a.hobj, t, ho);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    for (uint32_t k = 0; k < L.n; k++) obj_release(a, L.c[k].o);
    L.n = 0;
    L.full = 0;
  }
  __syncthreads();
}

// collect a drain's joins (targets pred)
__device__ __forceinline__ void cap_drain(const WalkArgs& a, CapList& L, const DrainOut& O) {
  if (O.m != NIL) cap_push(a, L, rec_cref(a, O.m), 0);
  for (uint32_t k = 0; k < O.nj; k++) cap_push(a, L, rec_cref(a, O.j[k]), 0);
}

// on_acquire (gwcp.py:175-192).  Under the lock's ticket (taken by the
// caller): the drain scan, the instance clocks to join (captured), the
// record and the frame.  The ticket is then given back and the O(|Q|) clock
// work -- materialise pred / hb, join, publish -- happens outside it: those
// objects are immutable (refcounted) and nobody else reads t's clocks before
// this CTA's next event of t.
__device__ void do_acquire(const WalkArgs& a, uint32_t e, uint32_t to, unsigned long long lock) {
  const uint32_t n = vlen(a);
  const uint32_t t = ev_tid(to);
  const uint32_t vt = vidx(a, t);
  const uint32_t cur = (to & GW_F_DEVICE) ? SC_DEV : t / a.tr.BS;
  __shared__ LockEnt* s_lk;
  __shared__ DrainOut s_dr;
  __shared__ CapList s_cap;
  __shared__ uint32_t s_inst, s_done;
  if (threadIdx.x == 0) {
    s_lk = lock_find(a, lock, false);  // created by the pre-pass
    s_cap.n = 0;
    s_cap.full = 0;
  }
  __syncthreads();
  if (!s_lk) { if (threadIdx.x == 0) atomicOr(a.err, ERR_INTERNAL); tickets_release(a, e); return; }
  // (1) drain: scans until done, applying the collected joins in between when a scan fills up
  bool first = true;
  while (!a.hb_mode) {  // scoped HB (hb.py:59-72) has no queues
    drain_scan(a, t, lock, cur, s_dr, first, nullptr);
    first = false;
    if (threadIdx.x == 0) cap_drain(a, s_cap, s_dr);
    __syncthreads();
    if (!s_dr.more) break;
    cap_flush(a, s_cap, t, vt, n);  // still under the ticket (rare: > kDrainJ non-dominating pops)
  }
  // (2) the record (acq_clock kept as its epoch (t, local); see the drain-test note) and the frame
  if (threadIdx.x == 0) {
    LockEnt* lk = s_lk;
    const uint32_t ri = a.hb_mode ? 0u : a.rix[a.poff[e]];
    const uint32_t d = a.depth[t];
    InstEnt* own = inst_find(a, lock, cur, false);
    if (a.hb_mode) {
      if (d >= a.maxd) atomicOr(a.err, ERR_FRAMES);
      else {
        Frame f;
        f.lock = lock; f.scope = cur; f.rec = NIL; f.logpos = a.loghead[t];
        f.iver = own ? __ldcg(&own->relver) : 0u;
        a.frames[(size_t)t * a.maxd + d] = f;
        a.depth[t] = d + 1;
      }
    }
    else if (ri >= a.rec_cap) { atomicOr(a.err, ERR_REC); }
    else if (d >= a.maxd) { atomicOr(a.err, ERR_FRAMES); }
    else {
      const uint32_t base = __ldcg(&lk->rec_base);
      // domall: the previous record was closed, dominated all before it, and
      // its instance orders this acquire, so this acquire joins its release
      // clock into hb (gwcp.py:185-188) and this record's release clock (hb
      // at release) dominates every earlier record's
      uint32_t domall = 1;
      if (ri > base) {
        const Rec* pr = a.recs + ri - 1;
        domall = __ldcg(&pr->closed) && __ldcg(&pr->domall) && sc_overlap(__ldcg(&pr->scope), cur);
      }
      Rec r;
      r.tid = t; r.acq_local = a.local[t]; r.scope = cur; r.rel_hobj = NIL; r.rel_local = 0; r.closed = 0;
      r.domall = domall; r.pad = 0;
      a.recs[ri] = r;
      lk->nrec = ri - base + 1;
      Frame f;
      f.lock = lock; f.scope = cur; f.rec = ri; f.logpos = a.loghead[t];
      f.iver = own ? __ldcg(&own->relver) : 0u;  // joined below (sc_overlap(cur, cur))
      a.frames[(size_t)t * a.maxd + d] = f;
      a.depth[t] = d + 1;
    }
    s_inst = __ldcg(&lk->inst_head);
  }
  __syncthreads();
  // (3) instance clocks whose release orders this acquire (gwcp.py:185-188, scopes.py:50-59)
  bool released = false;
  while (true) {
    if (threadIdx.x == 0) {
      uint32_t i = s_inst;
      while (i != NIL) {
        const InstEnt* ie = a.insts + i;
        if (sc_overlap(__ldcg(&ie->scope), cur)) {
          if (s_cap.n + 2 > (uint32_t)kMaxCap) break;  // apply these first
          cap_push(a, s_cap, CRef{__ldcg(&ie->H.o), __ldcg(&ie->H.dtid), __ldcg(&ie->H.dval)}, 1);
          if (!a.hb_mode)
            cap_push(a, s_cap, CRef{__ldcg(&ie->P.o), __ldcg(&ie->P.dtid), __ldcg(&ie->P.dval)}, 0);
        }
        i = __ldcg(&ie->next);
      }
      s_inst = i;
      s_done = i == NIL;
    }
    __syncthreads();
    const bool done = s_done != 0;
    if (done) { tickets_release(a, e); released = true; }
    cap_flush(a, s_cap, t, vt, n);
    if (done) break;
  }
  if (!released) tickets_release(a, e);
  __syncthreads();
}

// target := src (thread 0): retain the new object, drop the old one
__device__ __forceinline__ void cref_set(const WalkArgs& a, CRef* dst, CRef src) {
  obj_retain(a, src.o);
  const uint32_t old = __ldcg(&dst->o);
  dst->o = src.o;
  dst->dtid = src.dtid;
  dst->dval = src.dval;
  obj_release(a, old);
}
// target := target join src as a new object (block-wide; scratch S of n words)
__device__ void cref_join_new(const WalkArgs& a, CRef* dst, CRef src, uint32_t* S, uint32_t n) {
  __shared__ CRef s_old;
  if (threadIdx.x == 0) s_old = CRef{__ldcg(&dst->o), __ldcg(&dst->dtid), __ldcg(&dst->dval)};
  __syncthreads();
  const CRef old = s_old;
  materialize(S, a.arena, old.o, n, NIL, 0u);
  if (threadIdx.x == 0 && old.dtid != NIL) {
    const uint32_t v = vidx(a, old.dtid);
    if (v != NIL && old.dval > S[v]) S[v] = old.dval;
  }
  __syncthreads();
  join_cref(a, S, src);
  const uint32_t o = publish_dense(a, S, n, 1);
  if (threadIdx.x == 0) {
    dst->o = o;
    dst->dtid = NIL;
    dst->dval = 0;
    obj_release(a, old.o);
  }
  __syncthreads();
}

// on_release (gwcp.py:194-219), under the lock's ticket.  When no release
// into the frame's instance happened since this thread's acquire joined it,
// hb_t dominates H_i and every cs_read / cs_write clock of the instance, and
// pred_t dominates P_i, so the joins are reference swaps (no clock work).
__device__ void do_release(const WalkArgs& a, uint32_t e, uint32_t to, unsigned long long lock) {
  const uint32_t n = vlen(a);
  const uint32_t t = ev_tid(to);
  const uint32_t vt = vidx(a, t);
  uint32_t* P = a.scratch + (size_t)blockIdx.x * 3 * n;
  uint32_t* H = P + n;
  uint32_t* S = H + n;
  __shared__ Frame s_f;
  __shared__ LockEnt* s_lk;
  __shared__ DrainOut s_dr;
  __shared__ CapList s_cap;
  __shared__ InstEnt* s_ie;
  __shared__ uint32_t s_dom, s_newi;
  if (threadIdx.x == 0) {
    uint32_t d = a.depth[t];
    s_f = a.frames[(size_t)t * a.maxd + (d - 1)];
    s_lk = lock_find(a, lock, false);
    s_cap.n = 0;
    s_cap.full = 0;
  }
  __syncthreads();
  if (!s_lk) { if (threadIdx.x == 0) atomicOr(a.err, ERR_INTERNAL); tickets_release(a, e); return; }
  const uint32_t inst = s_f.scope;
  // (1) drain into pred
  bool first = true;
  while (!a.hb_mode) {
    drain_scan(a, t, lock, inst, s_dr, first, nullptr);
    first = false;
    if (threadIdx.x == 0) cap_drain(a, s_cap, s_dr);
    __syncthreads();
    cap_flush(a, s_cap, t, vt, n);  // the next scan (and P_i below) read t's published pred object
    if (!s_dr.more) break;
  }
  // (2) the frame's instance; dominance test
  if (threadIdx.x == 0) {
    InstEnt* ie = inst_find(a, lock, inst, true);
    s_ie = ie;
    s_newi = 0;
    if (ie && __ldcg(&ie->H.o) == NIL && __ldcg(&ie->H.dtid) == NIL && __ldcg(&ie->relver) == 0) s_newi = 1;
    s_dom = ie && __ldcg(&ie->relver) == s_f.iver;
  }
  __syncthreads();
  const CRef hb = CRef{a.hobj[t], t, a.local[t]};
  const CRef pr = CRef{a.pobj[t], t, a.pdiag[t]};
  const bool dom = s_dom != 0;
  // (3) cs_read / cs_write for the frame's read / write sets (gwcp.py:207-210)
  __shared__ CsEnt* s_ce;
  uint32_t li = a.hb_mode ? s_f.logpos : a.loghead[t];  // thread 0's iterator over the frame's access log
  while (true) {
    if (threadIdx.x == 0) {
      s_ce = nullptr;
      while (li != s_f.logpos && li != NIL) {
        LogEnt le = a.logs[li];
        li = le.next;
        CsEnt* ce = cs_find(a, lock, inst, le.loc, le.rw, true);
        if (!ce) break;
        if (dom) { cref_set(a, &ce->c, hb); continue; }
        s_ce = ce;
        break;
      }
    }
    __syncthreads();
    CsEnt* ce = s_ce;
    if (!ce) break;
    cref_join_new(a, &ce->c, hb, S, n);  // not dominated: a new joined clock
  }
  // (4) instance clocks H_i, P_i (gwcp.py:211-216)
  if (s_ie) {
    if (dom) {
      if (threadIdx.x == 0) { cref_set(a, &s_ie->H, hb); if (!a.hb_mode) cref_set(a, &s_ie->P, pr); }
    } else {
      cref_join_new(a, &s_ie->H, hb, S, n);
      if (!a.hb_mode) cref_join_new(a, &s_ie->P, pr, S, n);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_ie) {
      if (s_newi) {  // first release into this instance: link it into the lock's list
        s_ie->next = __ldcg(&s_lk->inst_head);
        s_lk->inst_head = (uint32_t)(s_ie - a.insts);
      }
      s_ie->relver = __ldcg(&s_ie->relver) + 1;
    }
    // close the record with rel_clock = copy(hb) (gwcp.py:216): the record
    // pins the thread's current hb object; pop; local += 1
    if (!a.hb_mode) {
      Rec* r = &a.recs[s_f.rec];
      obj_retain(a, hb.o);
      r->rel_hobj = hb.o;
      r->rel_local = hb.dval;
      __threadfence();
      r->closed = 1;
    }
    uint32_t d = a.depth[t] - 1;
    a.depth[t] = d;
    if (d == 0) a.loghead[t] = NIL;
    a.local[t] = a.local[t] + 1;
  }
  tickets_release(a, e);
  __syncthreads();
}

// on_access inside critical sections: rule (i) joins (gwcp.py:236-249) --
// the cs clocks captured under the tickets, joined after -- then the time
// stamp, the race-check queries and the frame-set append (gwcp.py:278-279)
__device__ void do_incs_access(const WalkArgs& a, uint32_t e, uint32_t to, unsigned long long loc) {
  const uint32_t n = vlen(a);
  const uint32_t t = ev_tid(to);
  const uint32_t vt = vidx(a, t);
  const uint32_t isw = ev_kind(to) == GW_K_WRITE;
  __shared__ CapList s_cap;
  __shared__ uint32_t s_done;
  __shared__ uint32_t s_fi, s_ii, s_phase;
  __shared__ unsigned long long s_flock;
  __shared__ uint32_t s_fscope;
  const uint32_t depth = a.depth[t];
  if (threadIdx.x == 0) { s_cap.n = 0; s_cap.full = 0; s_fi = 0; s_ii = NIL; s_phase = 0; }
  __syncthreads();
  bool released = false;
  // frames x released instances of the frame's lock overlapping the frame's
  // instance x {cs_write, cs_read if this is a write}; HB has no cs clocks
  while (!a.hb_mode) {
    if (threadIdx.x == 0) {
      uint32_t fi = s_fi, ii = s_ii, phase = s_phase;
      unsigned long long flock = s_flock;
      uint32_t fscope = s_fscope;
      bool stop = false;
      while (!stop) {
        if (phase == 0) {
          if (fi >= depth) break;
          const Frame f = a.frames[(size_t)t * a.maxd + fi];
          flock = f.lock;
          fscope = f.scope;
          LockEnt* lk = lock_find(a, flock, false);
          ii = lk ? __ldcg(&lk->inst_head) : NIL;
          phase = 1;
        }
        if (ii == NIL) { fi++; phase = 0; continue; }
        const uint32_t isc = __ldcg(&a.insts[ii].scope);
        const bool ov = sc_overlap(isc, fscope);
        if (phase == 1 || phase == 2) {
          if (s_cap.n + 1 > (uint32_t)kMaxCap) { stop = true; break; }  // apply these first
          if (ov) {
            CsEnt* ce = cs_find(a, flock, isc, loc, phase == 1 ? 1u : 0u, false);
            if (ce) cap_push(a, s_cap, CRef{__ldcg(&ce->c.o), __ldcg(&ce->c.dtid), __ldcg(&ce->c.dval)}, 0);
          }
          phase = (phase == 1 && isw) ? 2 : 3;
        }
        if (phase == 3) { ii = __ldcg(&a.insts[ii].next); phase = 1; }
      }
      s_fi = fi; s_ii = ii; s_phase = phase; s_flock = flock; s_fscope = fscope;
      s_done = stop ? 0u : 1u;
    }
    __syncthreads();
    const bool done = s_done != 0;
    if (done) { tickets_release(a, e); released = true; }
    cap_flush(a, s_cap, t, vt, n);
    if (done) break;
  }
  if (!released) tickets_release(a, e);
  __syncthreads();
  if (threadIdx.x == 0) {
    a.time[e] = a.local[t];
    if (a.vobj) a.vobj[e] = a.pobj[t];
    if (a.lflags[e] & LF_QUERY) answer_queries(a, e, a.hb_mode ? a.hobj[t] : a.pobj[t]);
    if (!a.hb_mode) {  // the frame's read / write sets (HB keeps none)
      uint32_t li = atomicAdd(a.log_top, 1u);
      if (li >= a.log_cap) atomicOr(a.err, ERR_LOG);
      else {
        a.logs[li] = LogEnt{loc, isw, a.loghead[t]};
        a.loghead[t] = li;
      }
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------ the kernel --
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// prof slots: 0 stamp, 1 barrier, 2 ticket wait, 3 acquire, 4 release, 5 in-CS access, 6 total, 7 #lock events
struct ProfT {
  const WalkArgs& a;
  unsigned long long t;
  __device__ ProfT(const WalkArgs& a_) : a(a_), t(a_.prof && threadIdx.x == 0 ? gtime() : 0ull) {}
  __device__ void lap(int slot) {
    if (a.prof && threadIdx.x == 0) {
      const unsigned long long n = gtime();
      a.prof[blockIdx.x * 8 + slot] += n - t;
      t = n;
    }
  }
};

__global__ void __launch_bounds__(kThreads, 4) k_walker(WalkArgs a) {
  __shared__ uint32_t s_e[kWalkCH];
  __shared__ uint32_t s_to[kWalkCH];
  __shared__ uint32_t s_hard[kWalkCH + 1];
  __shared__ uint32_t s_nh;
  __shared__ __align__(16) uint32_t s_acc[kAccSmem];
  const DevTrace& tr = a.tr;
  const uint32_t g = blockIdx.x;
  // my range in the partition
  uint64_t beg = 0, end = tr.n;
  if (a.G > 1) {
    uint64_t lo = 0, hi = tr.n;
    while (lo < hi) { uint64_t m = (lo + hi) >> 1; if (a.part_key[m] < g) lo = m + 1; else hi = m; }
    beg = lo;
    hi = tr.n;
    while (lo < hi) { uint64_t m = (lo + hi) >> 1; if (a.part_key[m] <= g) lo = m + 1; else hi = m; }
    end = lo;
  }
  for (uint64_t cb = beg; cb < end; cb += kWalkCH) {
    const uint32_t cnt = (uint32_t)min((uint64_t)kWalkCH, end - cb);
    if (threadIdx.x == 0) s_nh = 0;
    __syncthreads();
    // stage events; collect the hard ones (barrier, acq, rel, end, in-CS access)
    {
      // unrolled so every thread has kWalkCH/kThreads independent loads in flight
      constexpr int IPT = kWalkCH / kThreads;
      uint32_t ee[IPT];
#pragma unroll
      for (int k = 0; k < IPT; k++) {
        const uint32_t j = threadIdx.x + k * kThreads;
        ee[k] = j < cnt ? (a.perm ? __ldg(a.perm + cb + j) : (uint32_t)(cb + j)) : 0u;
      }
#pragma unroll
      for (int k = 0; k < IPT; k++) {
        const uint32_t j = threadIdx.x + k * kThreads;
        if (j < cnt) {
          s_e[j] = ee[k];
          s_to[j] = __ldg(tr.tidop + ee[k]);
        }
      }
    }
    __syncthreads();
    // ordered compaction of hard positions (block scan over 4 items/thread)
    {
      constexpr int IPT = kWalkCH / kThreads;
      uint32_t flags = 0, nmine = 0;
#pragma unroll
      for (int k = 0; k < IPT; k++) {
        uint32_t j = threadIdx.x * IPT + k;
        if (j < cnt) {
          uint32_t kd = ev_kind(s_to[j]);
          bool hard = kd != GW_K_READ && kd != GW_K_WRITE && kd != GW_K_FENCE;
          if (!hard && a.has_locks && kd <= GW_K_WRITE && (a.lflags[s_e[j]] & LF_INCS)) hard = true;
          if (hard) { flags |= 1u << k; nmine++; }
        }
      }
      uint32_t tot;
      uint32_t off = block_excl_scan<uint32_t, OpSum>(nmine, OpSum(), 0u, &tot);
#pragma unroll
      for (int k = 0; k < IPT; k++)
        if (flags & (1u << k)) s_hard[off++] = threadIdx.x * IPT + k;
      if (threadIdx.x == 0) { s_nh = tot; s_hard[tot] = cnt; }
    }
    __syncthreads();
    const uint32_t nh = s_nh;
    uint32_t pos = 0;
    ProfT pf(a);
    for (uint32_t hi = 0; hi <= nh; hi++) {
      const uint32_t h = s_hard[hi];
      // plain accesses in [pos, h): stamp (time, vobj) from the owner's state
      for (uint32_t j0 = pos; j0 < h; j0 += 4 * kThreads) {
        uint32_t tt[4], lv[4], ov[4];
#pragma unroll
        for (int k = 0; k < 4; k++) {
          const uint32_t j = j0 + threadIdx.x + k * kThreads;
          tt[k] = NIL;
          if (j < h) {
            const uint32_t to = s_to[j];
            if (ev_kind(to) <= GW_K_WRITE) tt[k] = ev_tid(to);
          }
        }
#pragma unroll
        for (int k = 0; k < 4; k++)
          if (tt[k] != NIL) { lv[k] = a.local[tt[k]]; ov[k] = a.pobj[tt[k]]; }
#pragma unroll
        for (int k = 0; k < 4; k++)
          if (tt[k] != NIL) {
            const uint32_t e = s_e[j0 + threadIdx.x + k * kThreads];
            a.time[e] = lv[k];
            if (a.vobj) a.vobj[e] = ov[k];
            else if (a.lflags[e] & LF_QUERY) answer_queries(a, e, a.hb_mode ? a.hobj[tt[k]] : ov[k]);
          }
      }
      __syncthreads();
      pf.lap(0);
      if (h < cnt) {
        const uint32_t e = s_e[h], to = s_to[h];
        const uint32_t kd = ev_kind(to);
        if (kd == GW_K_BARRIER) {
          if ((to & GW_F_WARPBAR) && !a.has_locks && tr.L <= 32) {
            if (threadIdx.x < 32) do_barrier_warp(a, to, tr.instr[e], s_acc);
            __syncthreads();
          } else {
            do_barrier(a, to, tr.instr[e], s_acc);
          }
          pf.lap(1);
        } else if (kd == GW_K_END) {
          if (threadIdx.x == 0) {
            const uint32_t t = ev_tid(to);
            uint32_t d = a.has_locks ? a.depth[t] : 0u;
            for (uint32_t i = 0; i < d; i++)
              emit_diag(a, e, GW_D_EXIT_HOLDING, i, a.frames[(size_t)t * a.maxd + i].lock);
            if (a.has_locks) { a.depth[t] = 0; a.loghead[t] = NIL; }
            a.exited[t] = 1;
            a.nend[t] = a.nend[t] + 1;
          }
          __syncthreads();
        } else if (kd == GW_K_ACQUIRE || kd == GW_K_RELEASE) {
          const uint8_t lf = a.lflags[e];
          const unsigned long long lock = tr.key[e];
          if (!(lf & LF_OK)) {
            if (threadIdx.x == 0) emit_diag(a, e, kd == GW_K_ACQUIRE ? GW_D_REENTRANT : GW_D_UNHELD, 0, lock);
            __syncthreads();
          } else {
            tickets_wait(a, e);
            pf.lap(2);
            if (kd == GW_K_ACQUIRE) do_acquire(a, e, to, lock);  // gives the ticket back early
            else do_release(a, e, to, lock);
            pf.lap(kd == GW_K_ACQUIRE ? 3 : 4);
            if (a.prof && threadIdx.x == 0) a.prof[blockIdx.x * 8 + 7]++;
          }
        } else {  // in-CS access
          tickets_wait(a, e);
          pf.lap(2);
          do_incs_access(a, e, to, tr.key[e]);  // gives the tickets back early
          pf.lap(5);
          if (a.prof && threadIdx.x == 0) a.prof[blockIdx.x * 8 + 7]++;
        }
      }
      pos = h + 1;
    }
    __syncthreads();
  }
}

// ---------------------------------------------- snapshot mode (lock-free) --
// Lock-free traces: blocks never interact, and plain accesses only read
// their thread's state.  The walker then visits only the hard events
// (barriers, ENDs) of each block -- a few per block -- and writes the whole
// block state {local, pred object} after each one; k_stamp stamps every
// access in parallel from snapshot k = #hard events of its block before it.
struct SnapArgs {
  const uint32_t* hard_ev;   // hard event indices grouped by block, trace order within a block
  const uint32_t* hb_beg;    // per block [beg, end) into hard_ev
  const uint32_t* hb_end;
  uint2* snap;               // per block: (K_b + 1) x BS entries at (hb_beg[b] + b) * BS
};

__global__ void __launch_bounds__(kThreads) k_walker_snap(WalkArgs a, SnapArgs s) {
  __shared__ __align__(16) uint32_t s_acc[kAccSmem];
  const DevTrace& tr = a.tr;
  if (*(volatile const uint32_t*)a.abort_flag) return;
  for (uint32_t b = blockIdx.x; b < tr.B; b += gridDim.x) {
    const uint32_t beg = s.hb_beg[b], end = s.hb_end[b];
    uint2* sp = s.snap + (size_t)(beg + b) * tr.BS;
    const uint32_t t0 = b * tr.BS;
    for (uint32_t j = threadIdx.x; j < tr.BS; j += kThreads) sp[j] = make_uint2(a.local[t0 + j], a.pobj[t0 + j]);
    for (uint32_t h = beg; h < end; h++) {
      const uint32_t e = s.hard_ev[h];
      const uint32_t to = tr.tidop[e];
      __syncthreads();
      if (ev_kind(to) == GW_K_BARRIER) {
        if ((to & GW_F_WARPBAR) && tr.L <= 32) {
          if (threadIdx.x < 32) do_barrier_warp(a, to, tr.instr[e], s_acc);
          __syncthreads();
        } else {
          do_barrier(a, to, tr.instr[e], s_acc);
        }
      } else {  // END (lock-free: no frames)
        if (threadIdx.x == 0) {
          const uint32_t t = ev_tid(to);
          a.exited[t] = 1;
          a.nend[t] = a.nend[t] + 1;
        }
        __syncthreads();
      }
      sp += tr.BS;
      for (uint32_t j = threadIdx.x; j < tr.BS; j += kThreads) sp[j] = make_uint2(a.local[t0 + j], a.pobj[t0 + j]);
    }
    __syncthreads();
  }
}

// ---------------------------------------- warp snapshot mode (lock-free) --
// Traces whose hard events are mostly warp barriers (ITS-style, C4): a warp
// barrier only involves its own warp, so each of the block's (<= 8) warps
// walks its own hard-event list -- its warp barriers, its threads' ENDs, and
// the block barriers (replicated into every list, where the CTA's warps meet
// for the CTA-wide join) -- and writes its 32 lanes' {local, pred object}
// after each entry.  List g = b * 8 + warp; snapshot row r of list g at
// (hb_beg[g] + g + r) * 32.  Requires warps <= 8 and lanes <= 32.
constexpr uint32_t kWSnapWarps = 8;
__global__ void __launch_bounds__(kThreads) k_walker_wsnap(WalkArgs a, SnapArgs s) {
  __shared__ __align__(16) uint32_t s_acc[kAccSmem];
  const DevTrace& tr = a.tr;
  if (*(volatile const uint32_t*)a.abort_flag) return;
  const uint32_t j = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* wacc = s_acc + j * 256;  // this warp's barrier accumulator (span = block range <= 256)
  for (uint32_t b = blockIdx.x; b < tr.B; b += gridDim.x) {
    const uint32_t g = b * kWSnapWarps + j;
    const uint32_t beg = s.hb_beg[g], end = s.hb_end[g];
    uint2* row = s.snap + (size_t)(beg + g) * 32;
    const uint32_t t = b * tr.BS + j * tr.L + lane;
    const bool mine = j < tr.W && lane < tr.L;
    if (mine) row[lane] = make_uint2(a.local[t], a.pobj[t]);
    for (uint32_t h = beg; h < end; h++) {
      const uint32_t e = s.hard_ev[h];
      const uint32_t to = tr.tidop[e];
      if (ev_kind(to) == GW_K_BARRIER && !(to & GW_F_WARPBAR)) {
        __syncthreads();  // every warp of the block reaches this block barrier in its list
        do_barrier(a, to, 0u, s_acc);
      } else if (ev_kind(to) == GW_K_BARRIER) {
        do_barrier_warp(a, to, tr.instr[e], wacc);
      } else {  // END of one of this warp's threads
        if (lane == 0) {
          const uint32_t te = ev_tid(to);
          a.exited[te] = 1;
          a.nend[te] = a.nend[te] + 1;
        }
        __syncwarp();
      }
      row += 32;
      if (mine) row[lane] = make_uint2(a.local[t], a.pobj[t]);
      __syncwarp();
    }
    __syncthreads();
  }
}


// hard events (barriers, ENDs) of a lock-free trace: appended in any order as
// (block << 32 | event) keys with warp-aggregated atomics, then sorted, which
// orders them by block and by trace order within a block
// warp snapshot mode: (list g << 32 | event), block barriers once per warp list
__global__ void __launch_bounds__(kThreads) k_hard_append_w(DevTrace tr, unsigned long long* hkey, uint32_t* hcnt,
                                                           uint32_t* ntop, const uint32_t* abort_flag) {
  if (*(volatile const uint32_t*)abort_flag) return;
  // U aligned 32-event windows per warp and step, loads issued together; the
  // list slots of a whole CTA step are reserved with one atomic (warp-barrier-
  // heavy traces put a hard event in most windows: one global counter per
  // warp window was the bottleneck)
  constexpr int U = 4, NW = kThreads / 32;
  __shared__ uint32_t s_off[NW * U + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t step = (uint64_t)kThreads * U;
  for (uint64_t cb = (uint64_t)blockIdx.x * step; cb < tr.n; cb += (uint64_t)gridDim.x * step) {
    uint32_t tou[U], incl[U], cnt[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint64_t e = cb + (uint64_t)(w * U + u) * 32 + lane;
      tou[u] = e < tr.n ? tr.tidop[e] : (7u << GW_OP_SHIFT);
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint32_t k = ev_kind(tou[u]);
      const bool bbar = k == GW_K_BARRIER && !(tou[u] & GW_F_WARPBAR);
      const bool hard = k == GW_K_BARRIER || k == GW_K_END;
      cnt[u] = hard ? (bbar ? kWSnapWarps : 1u) : 0u;
      uint32_t v = cnt[u];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += x;
      }
      incl[u] = v;
      if (lane == 31) s_off[w * U + u] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // exclusive offsets of the CTA step's windows, one reservation
      uint32_t run = 0;
      for (int x = 0; x < NW * U; x++) {
        const uint32_t t = s_off[x];
        s_off[x] = run;
        run += t;
      }
      s_off[NW * U] = run ? atomicAdd(ntop, run) : 0u;
    }
    __syncthreads();
    const uint32_t cta_base = s_off[NW * U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      if (!cnt[u]) continue;
      const uint64_t e = cb + (uint64_t)(w * U + u) * 32 + lane;
      const uint32_t base = cta_base + s_off[w * U + u] + incl[u] - cnt[u];
      const uint32_t t = ev_tid(tou[u]), b = t / tr.BS;
      if (cnt[u] > 1) {  // block barrier: one entry in every warp's list
        for (uint32_t j = 0; j < kWSnapWarps; j++) {
          const uint32_t g = b * kWSnapWarps + j;
          hkey[base + j] = ((unsigned long long)g << 32) | (uint32_t)e;
          atomicAdd(hcnt + g, 1u);
        }
      } else {
        const uint32_t g = b * kWSnapWarps + (t % tr.BS) / tr.L;
        hkey[base] = ((unsigned long long)g << 32) | (uint32_t)e;
        atomicAdd(hcnt + g, 1u);
      }
    }
    __syncthreads();  // s_off reused by the next step
  }
}
__global__ void k_hard_append(DevTrace tr, unsigned long long* hkey, uint32_t* hcnt, uint32_t* ntop,
                              const uint32_t* abort_flag, uint32_t cap = 0xFFFFFFFFu) {
  if (*(volatile const uint32_t*)abort_flag) return;  // graph mode: the plan does not fit this trace
  constexpr int U = 4;  // aligned 32-event windows per warp iteration (loads issued together)
  const int lane = threadIdx.x & 31;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * U;
  for (uint64_t b0 = ((uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u)) * U; b0 < tr.n; b0 += stride) {
    uint32_t to[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint64_t e = b0 + 32 * u + lane;
      to[u] = e < tr.n ? tr.tidop[e] : (7u << GW_OP_SHIFT);
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint32_t k = ev_kind(to[u]);
      const bool hard = k == GW_K_BARRIER || k == GW_K_END;
      const uint32_t m = __ballot_sync(0xffffffffu, hard);
      if (!m) continue;
      uint32_t base = 0;
      if (lane == __ffs(m) - 1) base = atomicAdd(ntop, (uint32_t)__popc(m));
      base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
      if (hard) {
        const uint32_t b = ev_tid(to[u]) / tr.BS;
        const uint32_t slot = base + __popc(m & lanemask_lt());
        if (slot < cap) hkey[slot] = ((unsigned long long)b << 32) | (uint32_t)(b0 + 32 * u + lane);
        atomicAdd(hcnt + b, 1u);
      }
    }
  }
}
__global__ void k_hard_unpack(const unsigned long long* hkey, uint64_t n, uint32_t* hev) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    hev[i] = (uint32_t)hkey[i];
}
// Small hard-event lists (n <= kRankSortMax keys (segment << 32 | event), all
// distinct, nseg <= kThreads * 64 segments) in one launch instead of sort +
// unpack + scan: every CTA ranks its keys against all n staged in shared
// memory and writes the event at its rank; CTA 0 also turns the per-segment
// counts into [beg, end).
__global__ void __launch_bounds__(kThreads) k_hard_small(const unsigned long long* __restrict__ hkey, uint32_t n,
                                                        uint32_t* __restrict__ hev, const uint32_t* __restrict__ cnt,
                                                        uint32_t nseg, uint32_t* __restrict__ beg,
                                                        uint32_t* __restrict__ end) {
  __shared__ unsigned long long sk[kRankSortMax];
  for (uint32_t i = threadIdx.x; i < n; i += kThreads) sk[i] = hkey[i];
  __syncthreads();
  const uint32_t i = blockIdx.x * kThreads + threadIdx.x;
  if (i < n) {
    const unsigned long long k = sk[i];
    uint32_t r0 = 0, r1 = 0;
    uint32_t j = 0;
    for (; j + 2 <= n; j += 2) {
      r0 += sk[j] < k;
      r1 += sk[j + 1] < k;
    }
    if (j < n) r0 += sk[j] < k;
    hev[r0 + r1] = (uint32_t)k;
  }
  if (blockIdx.x == 0) {
    const uint32_t per = (nseg + kThreads - 1) / kThreads;
    const uint32_t s0 = min(nseg, threadIdx.x * per), s1 = min(nseg, s0 + per);
    uint32_t sum = 0;
    for (uint32_t x = s0; x < s1; x++) sum += cnt[x];
    uint32_t tot;
    uint32_t run = block_excl_scan<uint32_t, OpSum>(sum, OpSum(), 0u, &tot);
    for (uint32_t x = s0; x < s1; x++) {
      const uint32_t c = cnt[x];
      beg[x] = run;
      end[x] = run + c;
      run += c;
    }
  }
}

// exclusive scan of per-block hard-event counts -> [beg, end)
struct HardSegStore {
  const uint32_t* cnt;
  uint32_t* beg;
  uint32_t* end;
  __device__ __forceinline__ void operator()(uint64_t i, const uint32_t& v) const {
    beg[i] = v;
    end[i] = v + cnt[i];
  }
};

__global__ void k_state_init(WalkArgs a) {
  for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < a.tr.T;
       u += (uint64_t)gridDim.x * blockDim.x) {
    a.local[u] = 1; a.pobj[u] = NIL; a.pdiag[u] = 0; a.exited[u] = 0; a.nend[u] = 0;
    if (a.has_locks) { a.hobj[u] = NIL; a.depth[u] = 0; a.loghead[u] = NIL; }
  }
}

// ------------------------------------------------------ lock pre-pass ----
// Per-thread lock-stack automaton (clock independent): decides which
// acquires / releases succeed (gwcp.py:178-182, :196-201), which accesses run
// inside a critical section, and the global rank of every lock-related event.
__global__ void k_lock_mark(DevTrace tr, uint32_t* flag) {
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tr.n; e += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t k = ev_kind(tr.tidop[e]);
    flag[e] = (k == GW_K_ACQUIRE || k == GW_K_RELEASE || k == GW_K_END) ? 1u : 0u;
  }
}
__global__ void k_lock_compact(DevTrace tr, const uint32_t* pos, uint32_t* ktid, uint32_t* kev) {
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tr.n; e += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t to = tr.tidop[e];
    uint32_t k = ev_kind(to);
    if (k == GW_K_ACQUIRE || k == GW_K_RELEASE || k == GW_K_END) {
      uint32_t p = pos[e];
      ktid[p] = ev_tid(to);
      kev[p] = (uint32_t)e;
    }
  }
}
__global__ void k_lock_segs(const uint32_t* ktid, uint32_t n, uint32_t* seg_beg, uint32_t* seg_end) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t t = ktid[i];
    if (i == 0 || ktid[i - 1] != t) seg_beg[t] = i;
    if (i == n - 1 || ktid[i + 1] != t) seg_end[t] = i + 1;
  }
}
// The per-thread lock stacks form a persistent tree: a successful acquire at
// sorted position p creates node p = (lock, parent = current top); a
// successful release pops to the parent; END resets the stack.  top[p] is the
// stack after lock event p, so any event's lock set is a walk to the root.
__global__ void k_lock_automaton(DevTrace tr, const uint32_t* ktid, const uint32_t* kev, uint32_t n,
                                 const uint32_t* seg_end, unsigned long long* node_lock, uint32_t* node_parent,
                                 uint32_t* top_after, uint8_t* lflags, uint32_t* maxd) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t t = ktid[i];
    if (i != 0 && ktid[i - 1] == t) continue;
    const uint32_t end = seg_end[t];
    uint32_t top = NIL, d = 0, md = 0;
    for (uint32_t p = i; p < end; p++) {
      const uint32_t e = kev[p];
      const uint32_t k = ev_kind(tr.tidop[e]);
      const unsigned long long lk = tr.key[e];
      uint8_t ok = 0;
      if (k == GW_K_ACQUIRE) {  // reentrant iff lk is anywhere on the stack (gwcp.py:178)
        bool in = false;
        for (uint32_t q = top; q != NIL && !in; q = node_parent[q]) in = node_lock[q] == lk;
        if (!in) {
          node_lock[p] = lk;
          node_parent[p] = top;
          top = p;
          d++;
          ok = 1;
        }
      } else if (k == GW_K_RELEASE) {  // only the top frame can be released (gwcp.py:197)
        if (top != NIL && node_lock[top] == lk) {
          top = node_parent[top];
          d--;
          ok = 1;
        }
      } else {  // END clears the frames (gwcp.py:322-330)
        top = NIL;
        d = 0;
      }
      md = max(md, d);
      top_after[p] = top;
      if (k != GW_K_END) lflags[e] = ok ? (LF_OK | LF_LOCKREL) : 0;
    }
    atomicMax(maxd, md);
  }
}
// accesses: in a critical section iff the thread's stack is non-empty; npair =
// number of locks the event synchronises on (stack depth for accesses, 1 for a
// successful acquire / release)
__global__ void k_lock_access(DevTrace tr, const uint32_t* kev, const uint32_t* top_after, const uint32_t* seg_beg,
                              const uint32_t* seg_end, const uint32_t* node_parent, uint8_t* lflags, uint32_t* etop,
                              uint32_t* npair, uint32_t* n_incs) {
  uint32_t cnt = 0;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tr.n; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t to = tr.tidop[e];
    const uint32_t k = ev_kind(to);
    uint32_t np = 0, top = NIL;
    if (k <= GW_K_WRITE) {
      const uint32_t t = ev_tid(to);
      const uint32_t lo = seg_beg[t], hi = seg_end[t];
      uint8_t f = 0;
      if (lo < hi) {  // last lock event of t before e
        uint32_t l = lo, h = hi;
        while (l < h) { const uint32_t m = (l + h) >> 1; if (kev[m] < (uint32_t)e) l = m + 1; else h = m; }
        if (l > lo) top = top_after[l - 1];
        if (top != NIL) {
          f = LF_INCS | LF_LOCKREL;
          cnt++;
          for (uint32_t q = top; q != NIL; q = node_parent[q]) np++;
        }
      }
      lflags[e] = f;
    } else if (k == GW_K_ACQUIRE || k == GW_K_RELEASE) {
      np = (lflags[e] & LF_OK) ? 1u : 0u;
    }
    etop[e] = top;
    npair[e] = np;
  }
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(n_incs, cnt);
}
// emit (lock, event) pairs in event order (+ OR/AND of the lock ids for key compaction)
__global__ void k_lock_pairs(DevTrace tr, const uint32_t* poff, const uint32_t* npair, const uint32_t* etop,
                             const unsigned long long* node_lock, const uint32_t* node_parent,
                             unsigned long long* plock, uint32_t* pv, uint8_t* pacq, unsigned long long* orand) {
  unsigned long long ko = 0, ka = ~0ull;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tr.n; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t np = npair[e];
    if (!np) continue;
    const uint32_t off = poff[e];
    const uint32_t k = ev_kind(tr.tidop[e]);
    if (k == GW_K_ACQUIRE || k == GW_K_RELEASE) {
      plock[off] = tr.key[e];
      pacq[off] = k == GW_K_ACQUIRE ? 1 : 0;
    } else {
      uint32_t j = 0;
      for (uint32_t q = etop[e]; q != NIL; q = node_parent[q]) { pacq[off + j] = 0; plock[off + j++] = node_lock[q]; }
    }
    for (uint32_t j = 0; j < np; j++) {
      ko |= plock[off + j];
      ka &= plock[off + j];
      pv[off + j] = off + j;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ko |= __shfl_xor_sync(0xffffffffu, ko, o);
    ka &= __shfl_xor_sync(0xffffffffu, ka, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicOr(orand, ko);
    atomicAnd(orand + 1, ka);
  }
}
// sorted by lock (stable => event order within a lock): rank within the lock
struct LockSegLoad {
  const unsigned long long* k;
  __device__ __forceinline__ uint32_t operator()(uint64_t i) const {
    return (i == 0 || k[i] != k[i - 1]) ? (uint32_t)i : 0u;
  }
};
struct OpMaxU32 {
  __device__ __forceinline__ uint32_t operator()(const uint32_t& a, const uint32_t& b) const { return max(a, b); }
};
// sorted pairs: is-acquire flags, for the record slots (exclusive scan = slot)
struct AcqFlagLoad {
  const uint8_t* pacq;
  const uint32_t* sv;
  __device__ __forceinline__ uint32_t operator()(uint64_t q) const { return pacq[sv[q]]; }
};
// per pair: rank within its lock (ticket order) and, for successful acquires,
// the record slot; per lock: one table entry (+ ticket) and its first slot
__global__ void k_lock_ranks(const WalkArgs a, const unsigned long long* sk, const uint32_t* sv,
                             const uint32_t* segstart, const uint8_t* pacq, const uint32_t* gacq, uint64_t P,
                             uint32_t* prank, uint32_t* rix) {
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < P; q += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t pair = sv[q];
    prank[pair] = (uint32_t)(q - segstart[q]);
    if (pacq[pair]) rix[pair] = gacq[q];
    if (q == 0 || sk[q] != sk[q - 1]) {
      LockEnt* e = lock_find(a, a.plock[pair], true);
      if (e) e->rec_base = gacq[q];
    }
  }
}
__global__ void k_orand_init(unsigned long long* orand) {
  orand[0] = 0ull;
  orand[1] = ~0ull;
}

struct LockRelLoad {
  const uint8_t* lf;
  __device__ __forceinline__ uint32_t operator()(uint64_t i) const { return (lf[i] & LF_LOCKREL) ? 1u : 0u; }
};

}  // namespace gw
