"""Host side of the address-sharded (multi-GPU) path on CPU: the gloo
all-gather + order-key merge of paper_2111_12478_b200.shard reproduces the
unsharded report order (world_size 2 and 3, real processes)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2111_12478_b200.shard import merge_shards


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _reports(n=500, seed=0):
    rng = np.random.default_rng(seed)
    okey = np.sort(rng.choice(1 << 40, size=n, replace=False)).astype(np.uint64)
    return {"order_key": okey, "kind": rng.integers(0, 3, n).astype(np.uint8),
            "prior": rng.integers(0, 1 << 30, n).astype(np.uint32),
            "current": rng.integers(0, 1 << 30, n).astype(np.uint32)}


def _split(full, world, seed=1):
    # shards own arbitrary subsets (location ranges are not order-key ranges)
    owner = np.random.default_rng(seed).integers(0, world, len(full["kind"]))
    return [{f: v[owner == r] for f, v in full.items()} for r in range(world)]


def test_merge_shards_restores_order():
    full = _reports()
    merged = merge_shards(_split(full, 4))
    for f in full:
        assert np.array_equal(merged[f], full[f])
    assert len(merge_shards([_split(full, 1)[0]])["kind"]) == len(full["kind"])


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2111_12478_b200.shard import gather_reports

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    parts = _split(_reports(777, seed=world), world)
    parts[-1] = {f: v[:0] for f, v in parts[-1].items()}  # an empty shard
    full = merge_shards(parts)
    part = parts[rank]
    out = gather_reports(part)
    if rank == 0:
        q.put(all(np.array_equal(out[f], full[f]) for f in full))
    else:
        q.put(out is None)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gather_reports_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(res)


def test_merge_candidates_is_keep_first_dedup():
    """shard.merge_candidates (exchange mode, rank 0): keep-first on
    (location, prior.instr, current.instr) by order key, then report order
    (report.py:92-100), against a brute-force restatement."""
    import random

    from paper_2111_12478_b200.shard import merge_candidates

    rng = random.Random(5)
    for trial in range(20):
        n = rng.randint(0, 300)
        ev_instr = {e: rng.randint(0, 4) for e in range(400)}
        okeys = rng.sample(range(1, 10**6), n)
        c = {"order_key": np.array(okeys, np.uint64), "loc": np.array([rng.randint(0, 5) * 4 for _ in range(n)],
                                                                        np.uint64),
             "prior": np.array([rng.randrange(400) for _ in range(n)], np.uint32),
             "current": np.array([rng.randrange(400) for _ in range(n)], np.uint32),
             "kind": np.array([rng.randint(0, 2) for _ in range(n)], np.uint32)}
        got = merge_candidates(c, lambda e: np.array([ev_instr[int(x)] for x in e], np.uint32))
        best = {}
        for i in range(n):
            k = (int(c["loc"][i]), ev_instr[int(c["prior"][i])], ev_instr[int(c["current"][i])])
            if k not in best or okeys[i] < okeys[best[k]]:
                best[k] = i
        want = sorted(best.values(), key=lambda i: okeys[i])
        assert got["order_key"].tolist() == [okeys[i] for i in want]
        assert got["prior"].tolist() == [int(c["prior"][i]) for i in want]
        assert got["kind"].tolist() == [int(c["kind"][i]) for i in want]


def test_merge_candidates_device_equals_host():
    """The GPU-side merge of the exchange mode (torch on rank 0) == the numpy
    restatement (run here on CPU tensors)."""
    import torch

    from paper_2111_12478_b200.shard import merge_candidates, merge_candidates_device

    rng = np.random.default_rng(3)
    for m in (0, 1, 50, 3000):
        ok = rng.permutation(m).astype(np.int64) * 5 + 3
        a = np.stack([ok, rng.integers(0, 6, m) * 4, rng.integers(0, 500, m), rng.integers(0, 500, m),
                      rng.integers(0, 3, m)], axis=1).astype(np.int64) if m else np.zeros((0, 5), np.int64)
        ev = np.unique(np.concatenate([a[:, 2], a[:, 3]])) if m else np.zeros(0, np.int64)
        ins = rng.integers(0, 4, len(ev)).astype(np.int64)
        got = merge_candidates_device(torch.from_numpy(a), torch.from_numpy(ev), torch.from_numpy(ins))
        c = {"order_key": a[:, 0].astype(np.uint64), "loc": a[:, 1].astype(np.uint64),
             "prior": a[:, 2].astype(np.uint32), "current": a[:, 3].astype(np.uint32), "kind": a[:, 4].astype(np.uint32)}
        want = merge_candidates(c, lambda e: ins[np.searchsorted(ev, e)])
        for f in ("order_key", "prior", "current", "kind"):
            assert got[f].tolist() == want[f].tolist(), (m, f)
