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
