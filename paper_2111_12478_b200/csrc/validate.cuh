// validate_trace and infer_locks on the GPU.
//
// validate_trace (pkg/src/gpurace/trace.py:522-601) walks the trace once with
// per-thread state; every check it makes is per thread (lock stacks, END) or
// per barrier (exited participants), so:
//   * k_val_endpos:  first END of every thread (atomicMin)       -> exited
//   * k_val_events:  per event: barrier divergence (warp: exited masked lanes,
//                    lane order; block: no live thread), event after end of
//                    thread, shared location of another block; flags the
//                    lock events that reach the lock-stack logic
//   * the flagged lock events, stably sorted by thread (trace order kept),
//     one walker per thread segment with its lock stack in the segment's own
//     slice of scratch: reentrant acquire, release of unheld lock,
//     improperly nested release (trace.py:571-590)
//   * diagnostics ordered by (event, lane).
// infer_locks (trace.py:609-680) is a greedy per-thread adjacency rewrite:
// the thread's events (barriers excluded) stably sorted by thread, one walker
// per thread: atomic WRITE + FENCE -> ACQUIRE at the write, FENCE + atomic
// WRITE -> RELEASE at the write when the lock is held (else a diagnostic);
// the consumed fences are dropped and the trace compacted in order.
// Diagnostics come thread by thread in order of the threads' first events,
// then in event order (the reference iterates its per-thread dict,
// trace.py:624-671).
// Codes of the validate diagnostics: gw_validate (parse.cpp).
#pragma once
#include "access.cuh"

namespace gw {

struct VOut {
  unsigned long long* okey;  // event << 8 | lane: report order
  uint32_t* code;
  unsigned long long* a;
  unsigned long long* b;
  uint32_t* n;
  uint32_t cap;
};
__device__ __forceinline__ void v_emit(const VOut& o, uint32_t e, uint32_t sub, uint32_t code, unsigned long long x,
                                       unsigned long long y) {
  const uint32_t k = atomicAdd(o.n, 1u);
  if (k < o.cap) {
    o.okey[k] = ((unsigned long long)e << 8) | sub;
    o.code[k] = code;
    o.a[k] = x;
    o.b[k] = y;
  }
}

__global__ void k_val_endpos(DevTrace tr, uint32_t* endpos) {
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tr.n; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t to = tr.tidop[e];
    if (ev_kind(to) == GW_K_END) atomicMin(&endpos[ev_tid(to)], (uint32_t)e);
  }
}

// lkflag[e] = 1: a lock event the lock-stack walk must see
__global__ void k_val_events(DevTrace tr, const uint32_t* endpos, VOut o, uint32_t* lkflag) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tr.n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t e = (uint32_t)i;
    const uint32_t to = tr.tidop[i];
    const uint32_t kind = ev_kind(to), tid = ev_tid(to);
    uint32_t lk = 0;
    if (kind == GW_K_BARRIER) {
      if (to & GW_F_WARPBAR) {  // trace.py:530-539
        const uint32_t mask = tr.instr[i];
        for (uint32_t l = 0; l < tr.L && l < 32; l++)
          if (((mask >> l) & 1u) && endpos[tid + l] < e) v_emit(o, e, l, 1, l, 0);
      } else {  // trace.py:540-547: every thread of the block exited before
        bool live = false;
        for (uint32_t t = tid; t < tid + tr.BS && !live; t++) live = endpos[t] > e;
        if (!live) v_emit(o, e, 0, 2, tid / tr.BS, 0);
      }
    } else if (endpos[tid] < e) {  // trace.py:559-561
      v_emit(o, e, 0, 3, tid, 0);
    } else {
      if (kind <= GW_K_WRITE) {  // trace.py:562-569
        const unsigned long long k = tr.key[i];
        if (k & GW_SHARED_BIT) {
          const unsigned long long lb = (k >> 40) & ((1ull << 23) - 1);
          if (lb != tid / tr.BS) v_emit(o, e, 0, 4, lb, tid);
        }
      }
      lk = kind == GW_K_ACQUIRE || kind == GW_K_RELEASE;
    }
    lkflag[i] = lk;
  }
}
// (thread, event) of the flagged events, in trace order
__global__ void k_val_compact(DevTrace tr, const uint32_t* flag, const uint32_t* off, uint32_t* ktid, uint32_t* kev) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tr.n; i += (uint64_t)gridDim.x * blockDim.x)
    if (flag[i]) {
      ktid[off[i]] = ev_tid(tr.tidop[i]);
      kev[off[i]] = (uint32_t)i;
    }
}
// one thread per thread segment of the tid-sorted lock events (trace.py:570-590)
__global__ void k_val_locks(DevTrace tr, const uint32_t* ktid, const uint32_t* kev, uint32_t n,
                            unsigned long long* stack, VOut o) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (i > 0 && ktid[i - 1] == ktid[i]) continue;
    unsigned long long* st = stack + i;  // this segment's slice: depth <= its length
    uint32_t depth = 0;
    for (uint32_t j = i; j < n && ktid[j] == ktid[i]; j++) {
      const uint32_t e = kev[j];
      const unsigned long long k = tr.key[e];
      uint32_t pos = depth;
      for (uint32_t x = 0; x < depth; x++)
        if (st[x] == k) { pos = x; break; }
      if (ev_kind(tr.tidop[e]) == GW_K_ACQUIRE) {
        if (pos < depth) v_emit(o, e, 0, 5, k, 0);
        else st[depth++] = k;
      } else if (pos == depth) {
        v_emit(o, e, 0, 6, k, 0);
      } else if (pos != depth - 1) {
        v_emit(o, e, 0, 7, k, 0);
        for (uint32_t x = pos; x + 1 < depth; x++) st[x] = st[x + 1];
        depth--;
      } else {
        depth--;
      }
    }
  }
}

// ---- infer_locks -------------------------------------------------------------
// action per event: 0 keep, 1 drop (consumed fence), 2 -> ACQUIRE, 3 -> RELEASE
// (bit 2: device scope); lock = the location's address (trace.py:636, :649)
__device__ __forceinline__ unsigned long long loc_addr(unsigned long long k) {
  return (k & GW_SHARED_BIT) ? (k & ((1ull << 40) - 1)) : k;
}
__device__ __forceinline__ bool atomic_write(uint32_t to) {
  return ev_kind(to) == GW_K_WRITE && (to & GW_F_ATOMIC);
}
// thread events (barriers excluded), in trace order
__global__ void k_inf_flag(DevTrace tr, uint32_t* flag) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tr.n; i += (uint64_t)gridDim.x * blockDim.x)
    flag[i] = ev_kind(tr.tidop[i]) != GW_K_BARRIER;
}
struct InfDiag {  // (first event of the thread, event): the reference reports thread by thread
  uint32_t* first;
  uint32_t* ev;
  unsigned long long* lock;
  uint32_t* tid;
  uint32_t* n;
  uint32_t cap;
};
__global__ void k_inf_walk(DevTrace tr, const uint32_t* ktid, const uint32_t* kev, uint32_t n,
                           unsigned long long* held, uint8_t* action, InfDiag dg) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (i > 0 && ktid[i - 1] == ktid[i]) continue;
    uint32_t end = i;
    while (end < n && ktid[end] == ktid[i]) end++;
    unsigned long long* hs = held + i;  // this segment's held set
    uint32_t nh = 0;
    uint32_t j = i;
    while (j + 1 < end) {  // trace.py:627-671
      const uint32_t ea = kev[j], eb = kev[j + 1];
      const uint32_t ta = tr.tidop[ea], tb = tr.tidop[eb];
      if (atomic_write(ta) && ev_kind(tb) == GW_K_FENCE) {
        const unsigned long long lock = loc_addr(tr.key[ea]);
        const bool dev = (ta & GW_F_DEVICE) && (tb & GW_F_DEVICE);
        action[ea] = 2 | (dev ? 4 : 0);
        action[eb] = 1;
        uint32_t x = 0;
        while (x < nh && hs[x] != lock) x++;
        if (x == nh) hs[nh++] = lock;  // held.add
        j += 2;
        continue;
      }
      if (ev_kind(ta) == GW_K_FENCE && atomic_write(tb)) {
        const unsigned long long lock = loc_addr(tr.key[eb]);
        uint32_t x = 0;
        while (x < nh && hs[x] != lock) x++;
        if (x == nh) {
          const uint32_t k = atomicAdd(dg.n, 1u);
          if (k < dg.cap) { dg.first[k] = kev[i]; dg.ev[k] = eb; dg.lock[k] = lock; dg.tid[k] = ev_tid(tb); }
          j += 1;
          continue;
        }
        const bool dev = (ta & GW_F_DEVICE) && (tb & GW_F_DEVICE);
        action[eb] = 3 | (dev ? 4 : 0);
        action[ea] = 1;
        hs[x] = hs[--nh];  // held.discard
        j += 2;
        continue;
      }
      j += 1;
    }
  }
}
__global__ void k_inf_keep(const uint8_t* action, uint64_t n, uint32_t* keep) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    keep[i] = action[i] != 1;
}
// the rewritten trace, compacted in order (kept events keep their group bit)
__global__ void k_inf_emit(DevTrace tr, const uint8_t* action, const uint32_t* keep, const uint32_t* off,
                           unsigned long long* ko, uint32_t* to_o, uint32_t* io) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tr.n; i += (uint64_t)gridDim.x * blockDim.x) {
    if (!keep[i]) continue;
    const uint32_t p = off[i];
    const uint8_t a = action[i];
    const uint32_t to = tr.tidop[i];
    if ((a & 3u) >= 2) {
      const uint32_t kind = (a & 3u) == 2 ? GW_K_ACQUIRE : GW_K_RELEASE;
      to_o[p] = ev_tid(to) | (kind << GW_OP_SHIFT) | ((a & 4u) ? GW_F_DEVICE : 0u) | (to & GW_F_CONT);
      ko[p] = loc_addr(tr.key[i]);
      io[p] = 0;
    } else {
      to_o[p] = to;
      ko[p] = tr.key[i];
      io[p] = tr.instr[i];
    }
  }
}

}  // namespace gw
