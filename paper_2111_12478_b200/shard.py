"""Address-sharded (multi-GPU) analysis: one process per GPU, each holding the
whole trace, each reporting the races on one contiguous range of location
keys (gw_opts.shard_index / shard_count, include/gwcp_b200.h), then one
gather of the shards' reports and a merge by order key on rank 0.

Why this is exact: every check of an access to location x
needs only x's own access stream and the (replicated) sync pass; the
reference's keep-first dedup key contains the location (report.py:93), so
dedup is shard-local; the report order is a total order on order keys, so
concatenating the shards and sorting by order key reproduces it, and the
global first report is the reference's "first" (report.py:97).

The collective is torch.distributed plumbing (NCCL on GPUs, gloo on CPU):
sizes are all-gathered, then the padded report arrays.
"""

from __future__ import annotations

import numpy as np

_FIELDS = ("order_key", "kind", "prior", "current")


def merge_shards(parts: list[dict]) -> dict:
    """Concatenate per-shard report arrays and order them by order key."""
    cat = {f: np.concatenate([np.asarray(p[f]) for p in parts]) if parts else np.zeros(0) for f in _FIELDS}
    order = np.argsort(cat["order_key"], kind="stable")
    out = {f: cat[f][order] for f in _FIELDS}
    out["kind"] = out["kind"].astype(np.uint8)
    out["prior"] = out["prior"].astype(np.uint32)
    out["current"] = out["current"].astype(np.uint32)
    out["order_key"] = out["order_key"].astype(np.uint64)
    return out


def gather_reports(res: dict, *, device=None, group=None) -> dict | None:
    """Gather every rank's shard reports to rank 0 and merge them there
    (returns None on the other ranks).  ``device``: where the collective's
    buffers live (a CUDA device for NCCL, None/CPU for gloo)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = torch.device("cpu") if device is None else torch.device(device)
    n = int(len(res["kind"]))
    sizes = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([n], dtype=torch.int64, device=dev), group=group)
    sizes = [int(s.item()) for s in sizes]
    m = max(sizes) if sizes else 0
    # one int64 row per field: order key, kind, prior, current
    buf = np.zeros((4, m), dtype=np.int64)
    if n:
        buf[0, :n] = np.asarray(res["order_key"], dtype=np.uint64).view(np.int64)
        buf[1, :n] = np.asarray(res["kind"], dtype=np.int64)
        buf[2, :n] = np.asarray(res["prior"], dtype=np.int64)
        buf[3, :n] = np.asarray(res["current"], dtype=np.int64)
    mine = torch.from_numpy(buf).to(dev)
    allb = [torch.empty((4, m), dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(allb, mine, group=group)
    if rank != 0:
        return None
    parts = []
    for r in range(world):
        b = allb[r].cpu().numpy()[:, : sizes[r]]
        parts.append({"order_key": b[0].view(np.uint64), "kind": b[1], "prior": b[2], "current": b[3]})
    return merge_shards(parts)


def analyze_sharded(ctx, cfg, n, key_ptr, tidop_ptr, instr_ptr, *, stream=None, inactive_opt=True, device=None,
                    group=None) -> dict | None:
    """This rank's shard of a device-resident trace, gathered and merged on
    rank 0 (the multi-GPU form of engine.run)."""
    import torch.distributed as dist

    ctx.analyze_device(cfg, n, key_ptr, tidop_ptr, instr_ptr, stream=stream, inactive_opt=inactive_opt,
                       shard=(dist.get_rank(group), dist.get_world_size(group)))
    return gather_reports(ctx.fetch(), device=device, group=group)


# ---------------------------------------------------------------------------
# Exchange mode: the multi-GPU data plane of SURVEY §8(e) / include/gwcp_b200.h
# (gw_xs_*).  Every rank holds ONE record-aligned slice of the trace (1/G of
# the SoA, so 1/G of the host->device upload); the analysis moves data
# between the ranks, never replicates the trace:
#   1. slice statistics      -> all-reduce (sums) + all-gather (key OR / AND)
#   2. slice hard events     -> all-gather: the sync pass (snapshot walker)
#      runs on every rank over the whole trace's barriers / ENDs (C5:
#      16,384 events, C4: ~7.8 M)
#   3. slice access records  -> ALL-TO-ALL to their location-hash shard
#      (12 B per access: h, global event | W, tidop)
#   4. per shard: the bucketed check of its records (csrc/bucket.cuh); per
#      slice: the record (same-instruction) check
#   5. candidates -> gather to rank 0; the endpoint (tidop, instr) of every
#      referenced event -> broadcast ids + reduce from the owning slices
#   6. rank 0: keep-first dedup on (location, prior.instr, current.instr)
#      (report.py:92-100), report order = order key, "first" = report 0.
# Exact because every check of a location needs only that location's
# accesses (all on one shard, in trace order: slices arrive in rank order)
# and the sync pass, which every rank runs over all hard events.
# ---------------------------------------------------------------------------

class _Sparse:
    """Event-indexed column over the events the reports reference."""

    def __init__(self, ev, vals):
        self.ev, self.vals = ev, vals

    def __getitem__(self, idx):
        return self.vals[np.searchsorted(self.ev, np.asarray(idx))]


class ExchangeTrace:
    """What report formatting (report.ndjson_lines) reads of a trace, for the
    events the merged reports reference: config, tidop, instr, key."""

    def __init__(self, config, ev, tidop, instr, key):
        self.config = config
        self.tidop = _Sparse(ev, tidop)
        self.instr = _Sparse(ev, instr)
        self.key = _Sparse(ev, key)


def merge_candidates(c: dict, instr_of) -> dict:
    """Keep-first dedup of the gathered candidates on (location, prior.instr,
    current.instr) -- the smallest order key of each key survives -- then
    report order by order key (report.py:79-100)."""
    n = len(c["order_key"])
    if n == 0:
        z = np.zeros(0, np.uint32)
        return {"kind": np.zeros(0, np.uint8), "prior": z, "current": z.copy(), "order_key": np.zeros(0, np.uint64)}
    ip = instr_of(c["prior"]).astype(np.uint64)
    ic = instr_of(c["current"]).astype(np.uint64)
    order = np.lexsort((c["order_key"], ic, ip, c["loc"]))  # by (loc, ip, ic), then order key
    loc, a, b = c["loc"][order], ip[order], ic[order]
    first = np.ones(n, bool)
    first[1:] = (loc[1:] != loc[:-1]) | (a[1:] != a[:-1]) | (b[1:] != b[:-1])
    keep = order[first]
    keep = keep[np.argsort(c["order_key"][keep], kind="stable")]
    return {"kind": c["kind"][keep].astype(np.uint8), "prior": c["prior"][keep].astype(np.uint32),
            "current": c["current"][keep].astype(np.uint32), "order_key": c["order_key"][keep].astype(np.uint64),
            "loc": c["loc"][keep].astype(np.uint64)}


def _gather_rows(x, world, rank, coll, group, dst=0):
    """Variable-size row gather to `dst` (padded all-gather: gloo and NCCL)."""
    import torch
    import torch.distributed as dist

    n = torch.tensor([x.shape[0]], dtype=torch.int64, device=coll)
    sizes = [torch.zeros(1, dtype=torch.int64, device=coll) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    m = max(max(sizes), 1)
    pad = torch.zeros((m,) + tuple(x.shape[1:]), dtype=x.dtype, device=coll)
    pad[: x.shape[0]] = x.to(coll)
    allp = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(allp, pad, group=group)
    return torch.cat([allp[r][: sizes[r]] for r in range(world)]) if rank == dst or dst is None else None


def analyze_exchange(ctx, cfg, n_total: int, slice_bufs, base: int, *, collective_device=None, group=None,
                     stream=None):
    """One trace, G ranks, each with its slice (key int64, tidop int32, instr
    int32 device tensors of events [base, base + len)).  Returns, on rank 0,
    (result dict, ExchangeTrace) for report.ndjson_lines; None elsewhere.
    collective_device: where the collectives' tensors live (a CUDA device for
    NCCL, None = CPU for gloo)."""
    import torch
    import torch.distributed as dist

    from . import _native as N
    from .trace import TraceConfig

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    key_d, to_d, in_d = slice_bufs
    dev = to_d.device
    coll = torch.device("cpu") if collective_device is None else torch.device(collective_device)
    n = int(to_d.numel())
    i32 = torch.int32
    # 1. statistics of the whole trace
    st = ctx.xs_prep(cfg, n, key_d.data_ptr(), to_d.data_ptr(), in_d.data_ptr(), base, stream)
    sums = torch.tensor([st.n_acc, st.n_write, st.n_acq, st.n_rel, st.n_end, st.n_bar, st.n_long, st.n_wbar],
                        dtype=torch.int64, device=coll)
    dist.all_reduce(sums, group=group)
    kk = torch.from_numpy(np.array([st.key_or, st.key_and], np.uint64).view(np.int64)).to(coll)
    ks = [torch.zeros(2, dtype=torch.int64, device=coll) for _ in range(world)]
    dist.all_gather(ks, kk, group=group)
    kor, kand = 0, (1 << 64) - 1  # (a slice without accesses holds the identities 0 / ~0)
    for r in range(world):
        o, a = (int(x) for x in ks[r].cpu().numpy().view(np.uint64))
        kor |= o
        kand &= a
    g = N.XsStats(*[int(x) for x in sums.tolist()[:6]], kor, kand, *[int(x) for x in sums.tolist()[6:]])
    # 2. hard events of the whole trace, in event order (slices are in rank order)
    nh_loc = int(st.n_bar + st.n_end)
    hb = [torch.empty(max(nh_loc, 1), dtype=i32, device=dev) for _ in range(3)]
    hk = torch.empty(max(nh_loc, 1), dtype=torch.int64, device=dev)
    nh = ctx.xs_hard(hb[0].data_ptr(), hb[1].data_ptr(), hb[2].data_ptr(), hk.data_ptr(), stream)
    hard = torch.stack([hb[0][:nh], hb[1][:nh], hb[2][:nh], hk[:nh].view(i32)[0::2], hk[:nh].view(i32)[1::2]],
                       dim=1) if nh else torch.zeros((0, 5), dtype=i32, device=dev)
    allh = _gather_rows(hard, world, rank, coll, group, dst=None).to(dev)
    n_hard = int(allh.shape[0])
    gh = [allh[:, j].contiguous() for j in range(3)]
    gk = torch.stack([allh[:, 3], allh[:, 4]], dim=1).contiguous().view(torch.int64).view(-1) if n_hard else \
        torch.zeros(1, dtype=torch.int64, device=dev)
    # 3. access records to their shard (all-to-all)
    na = int(st.n_acc)
    pb = [torch.empty(max(na, 1), dtype=i32, device=dev) for _ in range(3)]
    counts = ctx.xs_partition(g, world, pb[0].data_ptr(), pb[1].data_ptr(), pb[2].data_ptr(), stream)
    send = torch.stack([p[:na] for p in pb], dim=1).to(coll)
    cin = torch.tensor(counts, dtype=torch.int64, device=coll)
    cout = torch.empty(world, dtype=torch.int64, device=coll)
    dist.all_to_all_single(cout, cin, group=group)
    out_splits = [int(x) for x in cout.tolist()]
    recv = torch.empty((sum(out_splits), 3), dtype=i32, device=coll)
    dist.all_to_all_single(recv, send, out_splits, counts, group=group)
    recv = recv.to(dev)
    rv = [recv[:, j].contiguous() for j in range(3)]
    nrecv = int(recv.shape[0])
    del send, pb
    # 4. this shard's check + the slice's record check
    ptr = lambda t: t.data_ptr() if t.numel() else 0  # noqa: E731
    nc = ctx.xs_check(g, world, n_total, [ptr(x) for x in rv], nrecv, [ptr(x) for x in gh] + [ptr(gk)], n_hard,
                      stream)
    c = ctx.xs_fetch(nc)
    rows = torch.from_numpy(np.stack([c["order_key"].view(np.int64), c["loc"].view(np.int64),
                                      c["prior"].astype(np.int64), c["current"].astype(np.int64),
                                      c["kind"].astype(np.int64)], axis=1) if nc else np.zeros((0, 5), np.int64))
    allc = _gather_rows(rows, world, rank, coll, group)
    # 5. endpoint info of the referenced events, from their owning slices
    if rank == 0:
        a = allc.to(dev)  # the merge runs on rank 0's GPU
        ev_d = torch.unique(torch.cat([a[:, 2], a[:, 3]]))  # sorted event ids
        m = torch.tensor([int(ev_d.numel())], dtype=torch.int64, device=coll)
    else:
        m = torch.zeros(1, dtype=torch.int64, device=coll)
    dist.broadcast(m, 0, group=group)
    evt = ev_d.to(coll) if rank == 0 else torch.empty(int(m.item()), dtype=torch.int64, device=coll)
    dist.broadcast(evt, 0, group=group)
    evn = evt.cpu().numpy().astype(np.uint32)
    to, ins = ctx.xs_lookup(evn)
    info = torch.from_numpy(np.stack([to.astype(np.int64), ins.astype(np.int64)], axis=1)).to(coll)
    dist.reduce(info, 0, group=group)  # exactly one slice owns each event
    if rank != 0:
        return None
    # 6. keep-first dedup on (location, prior.instr, current.instr), report order
    info = info.to(dev)
    res = merge_candidates_device(a, ev_d, info[:, 1])
    evs = ev_d.cpu().numpy().astype(np.uint32)
    inf = info.cpu().numpy()
    keys = np.zeros(len(evs), np.uint64)
    keys[np.searchsorted(evs, res["current"])] = res["loc"]
    xt = ExchangeTrace(TraceConfig(*cfg), evs, inf[:, 0].astype(np.uint32), inf[:, 1].astype(np.uint32), keys)
    for f in ("diag_event", "diag_code"):
        res[f] = np.zeros(0, np.uint32)
    res["diag_lock"] = np.zeros(0, np.uint64)
    return res, xt


def merge_candidates_device(a, ev, instr):
    """merge_candidates on the GPU (torch): a = (m, 5) int64 rows (order key,
    location, prior, current, kind), ev = sorted event ids, instr = their
    instruction ids.  Composite order by stable sorts (last key first)."""
    import torch

    if a.shape[0] == 0:
        z = np.zeros(0, np.uint32)
        return {"kind": np.zeros(0, np.uint8), "prior": z, "current": z.copy(), "order_key": np.zeros(0, np.uint64),
                "loc": np.zeros(0, np.uint64)}
    okey, loc, pri, cur, kind = a.unbind(1)
    ip = instr[torch.searchsorted(ev, pri)]
    ic = instr[torch.searchsorted(ev, cur)]
    order = torch.argsort(okey, stable=True)
    for k in (ic, ip, loc):
        order = order[torch.argsort(k[order], stable=True)]
    L, P, Cc = loc[order], ip[order], ic[order]
    first = torch.ones_like(L, dtype=torch.bool)
    first[1:] = (L[1:] != L[:-1]) | (P[1:] != P[:-1]) | (Cc[1:] != Cc[:-1])
    keep = order[first]
    keep = keep[torch.argsort(okey[keep], stable=True)]
    out = {k: v[keep].cpu().numpy() for k, v in (("order_key", okey), ("loc", loc), ("prior", pri),
                                                  ("current", cur), ("kind", kind))}
    return {"kind": out["kind"].astype(np.uint8), "prior": out["prior"].astype(np.uint32),
            "current": out["current"].astype(np.uint32), "order_key": out["order_key"].view(np.uint64),
            "loc": out["loc"].view(np.uint64)}


def record_cut(tidop, k: int, parts: int) -> int:
    """Start of slice k: about k/parts of the trace, moved forward to a record
    boundary (an event without the continues-record bit)."""
    from . import _native as N

    n = len(tidop)
    p = n * k // parts
    while 0 < p < n and int(tidop[p]) & N.F_CONT:
        p += 1
    return p
