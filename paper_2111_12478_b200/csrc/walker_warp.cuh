// Lock-mode walker with one warp per trace warp ("lock warp walker").
//
// The CTA-wide lock walker (k_walker) processes all events of its blocks in
// trace order, so a warp's acquire waits behind every earlier group of the
// other warps of its block -- and, through the per-lock tickets, so does
// every other CTA waiting for that lock.  Warps of a block interact only
// through block barriers (and locks), so here CTA warp j walks the events
// of trace warp j of the CTA's blocks on its own (warp barriers, lock events,
// in-CS accesses, ENDs, access stamps), meeting the other warps of the CTA
// only at block barriers (the CTA-wide barrier join of walker.cuh).  Lock
// state is still serialised per lock by the tickets in trace order; all
// waits are for earlier trace positions (tickets, and block barriers whose
// preceding events are earlier), so with all CTAs co-resident the walk is
// deadlock-free.  Clock work is warp-wide: fused joins straight into new
// refcounted objects (see fused_join in walker.cuh).
//
// Requires warps <= 8 and lanes <= 32 (else k_walker).
#pragma once
#include "walker.cuh"

namespace gw {

constexpr uint32_t kLW = 8;  // CTA warps = trace warps walked in parallel per block

struct WSm {  // per-warp shared state
  uint32_t tid[32], acq[32], ho[32], rloc[32], fl[32];
  uint32_t pos, end;
  CurEnt* cur;
  LockEnt* lk;
  DrainOut dr;
  CapList cap;
  uint32_t src[kMaxCap];
  uint32_t o, ns, full, ch;
};

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

__device__ void w_tickets_wait(const WalkArgs& a, uint32_t e) {
  if (lane_id() == 0) {
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
  __syncwarp();
  __threadfence();
}
__device__ void w_tickets_release(const WalkArgs& a, uint32_t e) {
  __threadfence();
  __syncwarp();
  if (lane_id() == 0) {
    __threadfence();
    const uint32_t off = a.poff[e], np = a.npair[e];
    for (uint32_t j = 0; j < np; j++) {
      LockEnt* lk = lock_find(a, a.plock[off + j], false);
      if (lk) atomicExch(&lk->ticket, a.prank[off + j] + 1);
    }
  }
  __syncwarp();
}

// drain_scan (walker.cuh) for one warp
__device__ void w_drain_scan(const WalkArgs& a, uint32_t t, unsigned long long lock, uint32_t cur, WSm& S,
                             bool first) {
  const uint32_t lane = lane_id();
  DrainOut& O = S.dr;
  if (lane == 0) {
    LockEnt* lk = lock_find(a, lock, false);
    CurEnt* ce = lk ? cur_find(a, lock, t) : nullptr;
    S.lk = lk;
    S.cur = ce;
    if (ce) {
      const uint32_t ep = a.nend[t];
      if (first && __ldcg(&ce->epoch) != ep) {  // (re)materialise the queue
        ce->epoch = ep;
        ce->last = NIL;
        ce->snap = ep != 0;
        ce->bound = ep == 0 ? NIL : (a.inactive_opt ? __ldcg(&lk->nrec) : 0u);
      }
      const uint32_t base = __ldcg(&lk->rec_base), nrec = __ldcg(&lk->nrec);
      const uint32_t last = __ldcg(&ce->last);
      S.pos = last == NIL ? base : last + 1;
      S.end = base + (ce->snap ? min(nrec, __ldcg(&ce->bound)) : nrec);
    }
    O.m = NIL;
    O.nj = 0;
    O.more = 0;
  }
  __syncwarp();
  if (!S.cur) return;
  const bool snap = __ldcg(&S.cur->snap) != 0;
  const uint32_t po = a.pobj[t];
  uint32_t pos = S.pos;
  const uint32_t end = S.end;
  uint32_t m = NIL, nj = 0;
  bool stop = false, full = false;
  while (!stop && !full && pos < end) {
    const uint32_t idx = pos + lane;
    const bool in = idx < end;
    uint32_t fl = 0;  // bit0 in, bit1 own (skipped), bit2 closed, bit3 joinable, bit4 domall
    if (in) {
      const Rec* r = a.recs + idx;
      const uint32_t rt = __ldcg(&r->tid);
      S.tid[lane] = rt;
      S.acq[lane] = __ldcg(&r->acq_local);
      S.ho[lane] = __ldcg(&r->rel_hobj);
      S.rloc[lane] = __ldcg(&r->rel_local);
      const bool own = !snap && rt == t;
      const bool closed = __ldcg(&r->closed) != 0;
      fl = 1u | (own ? 2u : 0u) | (closed ? 4u : 0u) |
           ((!own && closed && sc_overlap(__ldcg(&r->scope), cur)) ? 8u : 0u) | (__ldcg(&r->domall) ? 16u : 0u);
    }
    S.fl[lane] = fl;
    __syncwarp();
    bool pass = false;
    if (fl & 2u) pass = true;
    else if (!(fl & 4u)) pass = false;
    else if (S.tid[lane] == t) pass = true;
    else {
      const uint32_t u = S.tid[lane], vu = vidx(a, u);
      uint32_t v = vu != NIL ? obj_get_cg(a.arena, po, vu) : 0u;
      bool dom = false;
      for (int i = (int)lane - 1; i >= 0 && !dom; i--) {
        const uint32_t fi = S.fl[i];
        if (!(fi & 8u)) continue;
        v = max(v, relpt(a, S.ho[i], S.tid[i], S.rloc[i], u, vu));
        dom = (fi & 16u) != 0;
      }
      if (!dom) {
        for (uint32_t k = 0; k < nj; k++) {
          const Rec* r = a.recs + O.j[k];
          v = max(v, relpt(a, __ldcg(&r->rel_hobj), __ldcg(&r->tid), __ldcg(&r->rel_local), u, vu));
        }
        if (m != NIL) {
          const Rec* r = a.recs + m;
          v = max(v, relpt(a, __ldcg(&r->rel_hobj), __ldcg(&r->tid), __ldcg(&r->rel_local), u, vu));
        }
      }
      pass = v >= S.acq[lane];
    }
    const uint32_t fails = __ballot_sync(0xffffffffu, !(in && pass));
    uint32_t f = fails ? (uint32_t)(__ffs(fails) - 1) : 32u;
    for (uint32_t i = 0; i < f; i++) {
      const uint32_t fi = S.fl[i];
      if (!(fi & 8u)) continue;
      if (fi & 16u) { m = pos + i; nj = 0; }
      else if (nj < (uint32_t)kDrainJ) { if (lane == 0) O.j[nj] = pos + i; nj++; }
      else { f = i; full = true; break; }
    }
    if (f < 32u && !full) stop = true;
    pos += f;
    __syncwarp();
  }
  if (lane == 0) {
    O.m = m;
    O.nj = nj;
    O.more = (full && pos < end) ? 1u : 0u;
    if (pos > __ldcg(&S.lk->rec_base)) S.cur->last = pos - 1;
  }
  __syncwarp();
}

// fused_join (walker.cuh) for one warp: a new object := base (diag [vt] = diag)
// joined with the captured references of target tgt; NIL if unchanged
__device__ uint32_t w_fused_join(const WalkArgs& a, uint32_t base, uint32_t vt, uint32_t diag, WSm& S, uint32_t tgt,
                                 uint32_t n) {
  const uint32_t lane = lane_id();
  const CapList& L = S.cap;
  {  // nothing captured for this target: unchanged, no pass over the clock
    bool any = false;
    for (uint32_t k = 0; k < L.n && !any; k++) any = L.tgt[k] == tgt;
    if (!any) return NIL;
  }
  if (lane == 0) {
    uint32_t ns = 0, full = (base == NIL || (optr(a.arena, base)[0] == 0 && optr(a.arena, base)[1] == n)) ? 1u : 0u;
    for (uint32_t k = 0; k < L.n; k++)
      if (L.tgt[k] == tgt && L.c[k].o != NIL) {
        const uint32_t o = L.c[k].o;
        S.src[ns++] = o;
        if (!(__ldcg(optr(a.arena, o)) == 0 && __ldcg(optr(a.arena, o) + 1) == n)) full = 0;
      }
    S.ns = ns;
    S.full = full;
    const uint32_t o = arena_alloc(a, n + OBJ_HDR);
    if (o != NIL) obj_init(a, o, 0, n, 1);
    S.o = o;
  }
  __syncwarp();
  const uint32_t o = S.o, ns = S.ns;
  if (o == NIL) return NIL;
  uint32_t* out = optr(a.arena, o) + OBJ_HDR;
  int ch = 0;
  if (S.full) {
    // kJU 16-byte words per lane in flight per object: each op streams
    // whole clocks, so the memory-level parallelism of one warp sets the
    // op's latency -- and the per-lock chains are made of these ops.  A
    // source raises the result iff it exceeds the running max (exact `ch`).
    constexpr int kJU = 8;
    const uint32_t n4 = n >> 2;
    const uint4* b4 = base != NIL ? reinterpret_cast<const uint4*>(optr(a.arena, base) + OBJ_HDR) : nullptr;
    for (uint32_t i0 = lane; i0 < n4; i0 += 32 * kJU) {
      uint4 v[kJU];
#pragma unroll
      for (int k = 0; k < kJU; k++) {
        const uint32_t i = i0 + 32 * k;
        v[k] = (b4 && i < n4) ? __ldcg(b4 + i) : make_uint4(0, 0, 0, 0);
      }
      for (uint32_t s = 0; s < ns; s++) {
        const uint4* s4 = reinterpret_cast<const uint4*>(optr(a.arena, S.src[s]) + OBJ_HDR);
        uint4 sv[kJU];
#pragma unroll
        for (int k = 0; k < kJU; k++) {
          const uint32_t i = i0 + 32 * k;
          sv[k] = i < n4 ? __ldcg(s4 + i) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int k = 0; k < kJU; k++) {
          if (gt4(sv[k], v[k])) ch = 1;
          v[k] = max4(v[k], sv[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < kJU; k++) {
        const uint32_t i = i0 + 32 * k;
        if (i < n4) reinterpret_cast<uint4*>(out)[i] = v[k];
      }
    }
    for (uint32_t i = (n4 << 2) + lane; i < n; i += 32) {
      const uint32_t bv = base != NIL ? __ldcg(optr(a.arena, base) + OBJ_HDR + i) : 0u;
      uint32_t v = bv;
      for (uint32_t k = 0; k < ns; k++) v = max(v, __ldcg(optr(a.arena, S.src[k]) + OBJ_HDR + i));
      out[i] = v;
      if (v > bv) ch = 1;
    }
  } else {
    for (uint32_t i = lane; i < n; i += 32) {
      const uint32_t bv = obj_get_cg(a.arena, base, i);
      uint32_t v = bv;
      for (uint32_t k = 0; k < ns; k++) v = max(v, obj_get_cg(a.arena, S.src[k], i));
      out[i] = v;
      if (v > bv) ch = 1;
    }
  }
  __syncwarp();
  if (lane == 0) {
    if (vt != NIL) {
      const uint32_t bv = obj_get_cg(a.arena, base, vt);
      uint32_t srcmax = 0;
      for (uint32_t k = 0; k < ns; k++) srcmax = max(srcmax, obj_get_cg(a.arena, S.src[k], vt));
      const uint32_t v = max(diag, srcmax);
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
  ch = __any_sync(0xffffffffu, ch);
  if (!ch) {
    if (lane == 0) obj_release(a, o);
    __syncwarp();
    return NIL;
  }
  __syncwarp();
  return o;
}

__device__ void w_cap_flush(const WalkArgs& a, WSm& S, uint32_t t, uint32_t vt, uint32_t n) {
  const uint32_t lane = lane_id();
  if (S.cap.n) {
    const uint32_t po = w_fused_join(a, a.pobj[t], vt, a.pdiag[t], S, 0, n);
    if (po != NIL && lane == 0) {
      set_obj(a, a.pobj, t, po);
      if (vt != NIL) a.pdiag[t] = optr(a.arena, po)[OBJ_HDR + vt];
    }
    __syncwarp();
    const uint32_t ho = w_fused_join(a, a.hobj[t], vt, a.local[t], S, 1, n);
    if (ho != NIL && lane == 0) set_obj(a, a.hobj, t, ho);
    __syncwarp();
  }
  if (lane == 0) {
    for (uint32_t k = 0; k < S.cap.n; k++) obj_release(a, S.cap.c[k].o);
    S.cap.n = 0;
    S.cap.full = 0;
  }
  __syncwarp();
}

// on_acquire (gwcp.py:175-192), see do_acquire; the caller took the ticket
__device__ void w_acquire(const WalkArgs& a, uint32_t e, uint32_t to, unsigned long long lock, WSm& S) {
  const uint32_t lane = lane_id();
  const uint32_t n = vlen(a);
  const uint32_t t = ev_tid(to);
  const uint32_t vt = vidx(a, t);
  const uint32_t cur = (to & GW_F_DEVICE) ? SC_DEV : t / a.tr.BS;
  if (lane == 0) { S.cap.n = 0; S.cap.full = 0; }
  __syncwarp();
  bool first = true;
  while (!a.hb_mode) {  // scoped HB (hb.py:59-72) has no queues
    w_drain_scan(a, t, lock, cur, S, first);
    first = false;
    if (lane == 0) cap_drain(a, S.cap, S.dr);
    __syncwarp();
    if (!S.dr.more) break;
    w_cap_flush(a, S, t, vt, n);
  }
  uint32_t inst = NIL;
  if (lane == 0) {
    LockEnt* lk = lock_find(a, lock, false);
    const uint32_t ri = a.hb_mode ? 0u : a.rix[a.poff[e]];
    const uint32_t d = a.depth[t];
    InstEnt* own = inst_find(a, lock, cur, false);
    if (!lk) { atomicOr(a.err, ERR_INTERNAL); }
    else if (a.hb_mode) {
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
      f.iver = own ? __ldcg(&own->relver) : 0u;
      a.frames[(size_t)t * a.maxd + d] = f;
      a.depth[t] = d + 1;
    }
    inst = lk ? __ldcg(&lk->inst_head) : NIL;
  }
  inst = __shfl_sync(0xffffffffu, inst, 0);
  bool released = false;
  while (true) {
    uint32_t done = 0;
    if (lane == 0) {
      uint32_t i = inst;
      while (i != NIL) {
        const InstEnt* ie = a.insts + i;
        if (sc_overlap(__ldcg(&ie->scope), cur)) {
          if (S.cap.n + 2 > (uint32_t)kMaxCap) break;
          cap_push(a, S.cap, CRef{__ldcg(&ie->H.o), __ldcg(&ie->H.dtid), __ldcg(&ie->H.dval)}, 1);
          if (!a.hb_mode)
            cap_push(a, S.cap, CRef{__ldcg(&ie->P.o), __ldcg(&ie->P.dtid), __ldcg(&ie->P.dval)}, 0);
        }
        i = __ldcg(&ie->next);
      }
      inst = i;
      done = i == NIL;
    }
    inst = __shfl_sync(0xffffffffu, inst, 0);
    done = __shfl_sync(0xffffffffu, done, 0);
    __syncwarp();
    if (done) { w_tickets_release(a, e); released = true; }
    w_cap_flush(a, S, t, vt, n);
    if (done) break;
  }
  if (!released) w_tickets_release(a, e);
}

// target := target join src as a new object (warp)
__device__ void w_cref_join_new(const WalkArgs& a, CRef* dst, CRef src, WSm& S, uint32_t n) {
  const uint32_t lane = lane_id();
  CRef old;
  if (lane == 0) {
    old = CRef{__ldcg(&dst->o), __ldcg(&dst->dtid), __ldcg(&dst->dval)};
    S.cap.n = 0;
    cap_push(a, S.cap, src, 0);
  }
  old.o = __shfl_sync(0xffffffffu, old.o, 0);
  old.dtid = __shfl_sync(0xffffffffu, old.dtid, 0);
  old.dval = __shfl_sync(0xffffffffu, old.dval, 0);
  __syncwarp();
  // the old reference's explicit entry is >= its object's entry, so "overwrite" == "max"
  const uint32_t vo = old.dtid != NIL ? vidx(a, old.dtid) : NIL;
  uint32_t o = w_fused_join(a, old.o, vo, old.dval, S, 0, n);
  if (lane == 0) {
    if (o == NIL) {  // unchanged: keep the old reference
    } else {
      dst->o = o;
      dst->dtid = NIL;
      dst->dval = 0;
      obj_release(a, old.o);
    }
    for (uint32_t k = 0; k < S.cap.n; k++) obj_release(a, S.cap.c[k].o);
    S.cap.n = 0;
  }
  __syncwarp();
}

// on_release (gwcp.py:194-219), see do_release; the caller took the ticket
__device__ void w_release(const WalkArgs& a, uint32_t e, uint32_t to, unsigned long long lock, WSm& S) {
  const uint32_t lane = lane_id();
  const uint32_t n = vlen(a);
  const uint32_t t = ev_tid(to);
  const uint32_t vt = vidx(a, t);
  Frame f;
  if (lane == 0) { S.cap.n = 0; S.cap.full = 0; }
  {
    const uint32_t d = a.depth[t];
    f = a.frames[(size_t)t * a.maxd + (d - 1)];
  }
  __syncwarp();
  const uint32_t inst = f.scope;
  bool first = true;
  while (!a.hb_mode) {
    w_drain_scan(a, t, lock, inst, S, first);
    first = false;
    if (lane == 0) cap_drain(a, S.cap, S.dr);
    __syncwarp();
    w_cap_flush(a, S, t, vt, n);
    if (!S.dr.more) break;
  }
  InstEnt* ie = nullptr;
  uint32_t dom = 0, newi = 0;
  LockEnt* lk = nullptr;
  if (lane == 0) {
    lk = lock_find(a, lock, false);
    ie = inst_find(a, lock, inst, true);
    if (ie && __ldcg(&ie->relver) == 0) newi = 1;
    dom = ie && __ldcg(&ie->relver) == f.iver;
  }
  dom = __shfl_sync(0xffffffffu, dom, 0);
  ie = (InstEnt*)__shfl_sync(0xffffffffu, (unsigned long long)ie, 0);
  const CRef hb = CRef{a.hobj[t], t, a.local[t]};
  const CRef pr = CRef{a.pobj[t], t, a.pdiag[t]};
  // cs_read / cs_write of the frame's read / write sets (gwcp.py:207-210)
  uint32_t li = a.hb_mode ? f.logpos : a.loghead[t];  // HB keeps no cs clocks
  while (true) {
    CsEnt* ce = nullptr;
    if (lane == 0) {
      while (li != f.logpos && li != NIL) {
        LogEnt le = a.logs[li];
        li = le.next;
        CsEnt* c = cs_find(a, lock, inst, le.loc, le.rw, true);
        if (!c) break;
        if (dom) { cref_set(a, &c->c, hb); continue; }
        ce = c;
        break;
      }
    }
    ce = (CsEnt*)__shfl_sync(0xffffffffu, (unsigned long long)ce, 0);
    __syncwarp();
    if (!ce) break;
    w_cref_join_new(a, &ce->c, hb, S, n);
  }
  // instance clocks H_i, P_i (gwcp.py:211-216)
  if (ie) {
    if (dom) {
      if (lane == 0) { cref_set(a, &ie->H, hb); if (!a.hb_mode) cref_set(a, &ie->P, pr); }
    } else {
      w_cref_join_new(a, &ie->H, hb, S, n);
      if (!a.hb_mode) w_cref_join_new(a, &ie->P, pr, S, n);
    }
  }
  __syncwarp();
  if (lane == 0) {
    if (ie) {
      if (newi && lk) {
        ie->next = __ldcg(&lk->inst_head);
        lk->inst_head = (uint32_t)(ie - a.insts);
      }
      ie->relver = __ldcg(&ie->relver) + 1;
    }
    if (!a.hb_mode) {
      Rec* r = &a.recs[f.rec];
      obj_retain(a, hb.o);
      r->rel_hobj = hb.o;
      r->rel_local = hb.dval;
      __threadfence();
      r->closed = 1;
    }
    const uint32_t d = a.depth[t] - 1;
    a.depth[t] = d;
    if (d == 0) a.loghead[t] = NIL;
    a.local[t] = a.local[t] + 1;
  }
  w_tickets_release(a, e);
}

// on_access inside critical sections, see do_incs_access; the caller took the tickets
__device__ void w_incs_access(const WalkArgs& a, uint32_t e, uint32_t to, unsigned long long loc, WSm& S) {
  const uint32_t lane = lane_id();
  const uint32_t n = vlen(a);
  const uint32_t t = ev_tid(to);
  const uint32_t vt = vidx(a, t);
  const uint32_t isw = ev_kind(to) == GW_K_WRITE;
  const uint32_t depth = a.depth[t];
  uint32_t fi = 0, ii = NIL, phase = 0, fscope = 0;
  unsigned long long flock = 0;
  if (lane == 0) { S.cap.n = 0; S.cap.full = 0; }
  __syncwarp();
  bool released = false;
  while (!a.hb_mode) {  // rule (i); HB has no cs clocks
    uint32_t done = 0;
    if (lane == 0) {
      bool stop = false;
      while (!stop) {
        if (phase == 0) {
          if (fi >= depth) break;
          const Frame fr = a.frames[(size_t)t * a.maxd + fi];
          flock = fr.lock;
          fscope = fr.scope;
          LockEnt* lk = lock_find(a, flock, false);
          ii = lk ? __ldcg(&lk->inst_head) : NIL;
          phase = 1;
        }
        if (ii == NIL) { fi++; phase = 0; continue; }
        const uint32_t isc = __ldcg(&a.insts[ii].scope);
        const bool ov = sc_overlap(isc, fscope);
        if (phase == 1 || phase == 2) {
          if (S.cap.n + 1 > (uint32_t)kMaxCap) { stop = true; break; }
          if (ov) {
            CsEnt* ce = cs_find(a, flock, isc, loc, phase == 1 ? 1u : 0u, false);
            if (ce) cap_push(a, S.cap, CRef{__ldcg(&ce->c.o), __ldcg(&ce->c.dtid), __ldcg(&ce->c.dval)}, 0);
          }
          phase = (phase == 1 && isw) ? 2 : 3;
        }
        if (phase == 3) { ii = __ldcg(&a.insts[ii].next); phase = 1; }
      }
      done = stop ? 0u : 1u;
    }
    done = __shfl_sync(0xffffffffu, done, 0);
    __syncwarp();
    if (done) { w_tickets_release(a, e); released = true; }
    w_cap_flush(a, S, t, vt, n);
    if (done) break;
  }
  if (!released) w_tickets_release(a, e);
  if (lane == 0) {
    a.time[e] = a.local[t];
    if (a.lflags[e] & LF_QUERY) answer_queries(a, e, a.hb_mode ? a.hobj[t] : a.pobj[t]);
    if (!a.hb_mode) {  // the frame's read / write sets (HB keeps none)
      const uint32_t li = atomicAdd(a.log_top, 1u);
      if (li >= a.log_cap) atomicOr(a.err, ERR_LOG);
      else {
        a.logs[li] = LogEnt{loc, isw, a.loghead[t]};
        a.loghead[t] = li;
      }
    }
  }
  __syncwarp();
}

// warp barrier of lock mode: one fused pass over the participants' distinct
// objects + their own entries; every participant leaves with the new objects
__device__ void w_barrier_warp(const WalkArgs& a, uint32_t to, uint32_t ins, WSm& S) {
  const uint32_t lane = lane_id();
  const DevTrace& tr = a.tr;
  const uint32_t n = vlen(a);
  const uint32_t base = ev_tid(to);
  const uint32_t u = base + lane;
  const bool part = lane < tr.L && ((ins >> lane) & 1u) && !a.exited[u];
  const uint32_t pm = __ballot_sync(0xffffffffu, part);
  if (!pm) return;
  const uint32_t npart = __popc(pm);
  uint32_t newobj[2] = {NIL, NIL};
  for (int kind = 0; kind < 2; kind++) {
    uint32_t* objs = kind == 0 ? a.pobj : a.hobj;
    const uint32_t o = part ? objs[u] : NIL;
    // distinct objects, increasing handles
    if (lane == 0) { S.ns = 0; S.full = 1; }
    __syncwarp();
    uint32_t done = 0;
    while (true) {
      const uint32_t om = __reduce_min_sync(0xffffffffu, (o != NIL && o >= done) ? o : NIL);
      if (om == NIL) break;
      if (lane == 0) {
        if (S.ns < (uint32_t)kMaxCap) {
          S.src[S.ns++] = om;
          if (!(__ldcg(optr(a.arena, om)) == 0 && __ldcg(optr(a.arena, om) + 1) == n)) S.full = 0;
        }
      }
      done = om + 1;
    }
    if (lane == 0) {
      const uint32_t no = arena_alloc(a, n + OBJ_HDR);
      if (no != NIL) obj_init(a, no, 0, n, npart);
      S.o = no;
    }
    __syncwarp();
    const uint32_t no = S.o, ns = S.ns;
    if (no != NIL) {
      uint32_t* out = optr(a.arena, no) + OBJ_HDR;
      if (S.full) {
        constexpr int kJU = 8;  // as w_fused_join
        const uint32_t n4 = n >> 2;
        for (uint32_t i0 = lane; i0 < n4; i0 += 32 * kJU) {
          uint4 v[kJU];
#pragma unroll
          for (int k = 0; k < kJU; k++) v[k] = make_uint4(0, 0, 0, 0);
          for (uint32_t s = 0; s < ns; s++) {
            const uint4* s4 = reinterpret_cast<const uint4*>(optr(a.arena, S.src[s]) + OBJ_HDR);
            uint4 sv[kJU];
#pragma unroll
            for (int k = 0; k < kJU; k++) {
              const uint32_t i = i0 + 32 * k;
              sv[k] = i < n4 ? __ldcg(s4 + i) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int k = 0; k < kJU; k++) v[k] = max4(v[k], sv[k]);
          }
#pragma unroll
          for (int k = 0; k < kJU; k++) {
            const uint32_t i = i0 + 32 * k;
            if (i < n4) reinterpret_cast<uint4*>(out)[i] = v[k];
          }
        }
        for (uint32_t i = (n4 << 2) + lane; i < n; i += 32) {
          uint32_t v = 0;
          for (uint32_t k = 0; k < ns; k++) v = max(v, __ldcg(optr(a.arena, S.src[k]) + OBJ_HDR + i));
          out[i] = v;
        }
      } else {
        for (uint32_t i = lane; i < n; i += 32) {
          uint32_t v = 0;
          for (uint32_t k = 0; k < ns; k++) v = max(v, obj_get_cg(a.arena, S.src[k], i));
          out[i] = v;
        }
      }
      __syncwarp();
      if (part) {  // participants' own entries = their local time
        const uint32_t vu = vidx(a, u);
        if (vu != NIL) out[vu] = a.local[u];
      }
    }
    newobj[kind] = no;
    __syncwarp();
  }
  if (part) {
    const uint32_t nl = a.local[u] + 1;
    a.local[u] = nl;
    const uint32_t op = a.pobj[u];
    a.pobj[u] = newobj[0];
    obj_release(a, op);
    a.pdiag[u] = nl;
    const uint32_t oh = a.hobj[u];
    a.hobj[u] = newobj[1];
    obj_release(a, oh);
  }
  __syncwarp();
}

// Events of list (CTA, warp j) -- partition key cta * kLW + j, trace order --
// merged with the CTA's block-barrier list (bb_*).
#ifndef GW_LW_MINB
#define GW_LW_MINB 4
#endif
__global__ void __launch_bounds__(kThreads, GW_LW_MINB) k_walker_lw(WalkArgs a, const uint32_t* bb_ev, const uint32_t* bb_beg,
                                                        const uint32_t* bb_end) {
  __shared__ WSm SW[kLW];
  __shared__ __align__(16) uint32_t s_acc[kAccSmem];
  const DevTrace& tr = a.tr;
  const uint32_t j = threadIdx.x >> 5, lane = lane_id();
  WSm& S = SW[j];
  const uint32_t key = blockIdx.x * kLW + j;
  uint64_t beg, end;
  {
    uint64_t lo = 0, hi = tr.n;
    while (lo < hi) { const uint64_t m = (lo + hi) >> 1; if (a.part_key[m] < key) lo = m + 1; else hi = m; }
    beg = lo;
    hi = tr.n;
    while (lo < hi) { const uint64_t m = (lo + hi) >> 1; if (a.part_key[m] <= key) lo = m + 1; else hi = m; }
    end = lo;
  }
  uint32_t q = bb_beg[blockIdx.x];
  const uint32_t qend = bb_end[blockIdx.x];
  uint64_t p = beg;
  // optional time split (GW_PROF_WALKER): per walker warp, slots 0 stamp, 1 warp barrier,
  // 2 block barrier, 3 ticket wait, 4 acquire, 5 release, 6 in-CS access, 7 lock events
  unsigned long long* prof = a.prof ? a.prof + ((size_t)blockIdx.x * kLW + j) * 8 : nullptr;
  unsigned long long tp = prof && lane == 0 ? gtime() : 0ull;
  auto lap = [&](int slot) {
    if (prof && lane == 0) { const unsigned long long n = gtime(); prof[slot] += n - tp; tp = n; }
  };
  while (true) {
    const uint32_t ebb = q < qend ? bb_ev[q] : NIL;
    // own events before the next block barrier, 32 at a time
    while (p < end) {
      const uint64_t x = p + lane;
      const uint32_t ev = x < end ? __ldg(a.perm + x) : NIL;
      const bool inb = ev != NIL && ev < ebb;
      const uint32_t cm = __ballot_sync(0xffffffffu, inb);
      const uint32_t c = cm == 0xffffffffu ? 32u : (uint32_t)__ffs(~cm) - 1;  // prefix of events before ebb
      if (c == 0) break;
      const uint32_t to = lane < c ? __ldg(tr.tidop + ev) : 0u;
      const uint32_t kd = ev_kind(to);
      bool hard = false;
      if (lane < c) {
        hard = kd != GW_K_READ && kd != GW_K_WRITE && kd != GW_K_FENCE;
        if (!hard && kd <= GW_K_WRITE && (a.lflags[ev] & LF_INCS)) hard = true;
      }
      uint32_t hm = __ballot_sync(0xffffffffu, hard);
      uint32_t start = 0;
      while (true) {
        const uint32_t h = hm ? (uint32_t)__ffs(hm) - 1 : c;
        // plain accesses in [start, h): stamp by their lanes
        if (lane >= start && lane < h && kd <= GW_K_WRITE) {
          const uint32_t t = ev_tid(to);
          a.time[ev] = a.local[t];
          if (a.lflags[ev] & LF_QUERY) answer_queries(a, ev, a.hb_mode ? a.hobj[t] : a.pobj[t]);
        }
        __syncwarp();
        lap(0);
        if (h >= c) break;
        hm &= hm - 1;
        const uint32_t e = __shfl_sync(0xffffffffu, ev, h);
        const uint32_t te = __shfl_sync(0xffffffffu, to, h);
        const uint32_t k = ev_kind(te);
        if (k == GW_K_BARRIER) {  // warp barrier (block barriers come from the other list)
          w_barrier_warp(a, te, tr.instr[e], S);
          lap(1);
        } else if (k == GW_K_END) {
          if (lane == 0) {
            const uint32_t t = ev_tid(te);
            const uint32_t d = a.depth[t];
            for (uint32_t i = 0; i < d; i++) emit_diag(a, e, GW_D_EXIT_HOLDING, i, a.frames[(size_t)t * a.maxd + i].lock);
            a.depth[t] = 0;
            a.loghead[t] = NIL;
            a.exited[t] = 1;
            a.nend[t] = a.nend[t] + 1;
          }
          __syncwarp();
        } else if (k == GW_K_ACQUIRE || k == GW_K_RELEASE) {
          const unsigned long long lock = tr.key[e];
          if (!(a.lflags[e] & LF_OK)) {
            if (lane == 0) emit_diag(a, e, k == GW_K_ACQUIRE ? GW_D_REENTRANT : GW_D_UNHELD, 0, lock);
            __syncwarp();
          } else {
            w_tickets_wait(a, e);
            lap(3);
            if (k == GW_K_ACQUIRE) w_acquire(a, e, te, lock, S);
            else w_release(a, e, te, lock, S);
            lap(k == GW_K_ACQUIRE ? 4 : 5);
            if (prof && lane == 0) prof[7]++;
          }
        } else {  // in-CS access
          w_tickets_wait(a, e);
          lap(3);
          w_incs_access(a, e, te, tr.key[e], S);
          lap(6);
          if (prof && lane == 0) prof[7]++;
        }
        start = h + 1;
      }
      p += c;
      if (c < 32) break;
    }
    if (ebb == NIL) break;
    // block barrier: every warp of the CTA arrives here (each walks the same list)
    __syncthreads();
    do_barrier(a, tr.tidop[ebb], 0u, s_acc);
    lap(2);
    q++;
  }
  __syncthreads();
}

// partition keys: list (CTA = block mod G, warp in block); block barriers last
__global__ void k_part_keys_lw(DevTrace tr, uint32_t G, uint32_t* keys, uint32_t* vals) {
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tr.n; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t to = tr.tidop[e];
    const uint32_t t = ev_tid(to), b = t / tr.BS;
    const bool bbar = ev_kind(to) == GW_K_BARRIER && !(to & GW_F_WARPBAR);
    keys[e] = bbar ? G * kLW : (b % G) * kLW + (t % tr.BS) / tr.L;
    vals[e] = (uint32_t)e;
  }
}
// block barriers keyed by their walker CTA
__global__ void k_bbar_append(DevTrace tr, uint32_t G, unsigned long long* key, uint32_t* cnt, uint32_t* ntop) {
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tr.n; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t to = tr.tidop[e];
    if (ev_kind(to) != GW_K_BARRIER || (to & GW_F_WARPBAR)) continue;
    const uint32_t g = (ev_tid(to) / tr.BS) % G;
    key[atomicAdd(ntop, 1u)] = ((unsigned long long)g << 32) | (uint32_t)e;
    atomicAdd(cnt + g, 1u);
  }
}

}  // namespace gw
