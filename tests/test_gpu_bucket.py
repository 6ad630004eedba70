"""The bucketed access pass (csrc/bucket.cuh): the address-hashed shadow
table of the exchange mode (multi-GPU) and of GW_BUCKET=1 / 2 analyses.
GW_BUCKET=1 forces it at any size, so the reference goldens and the oracle
pin it on small traces too: every lock-free golden, the generator recipes,
hot locations (buckets above the shared-memory capacity spill to the
general sort + check path), large reader windows, and graph replays."""

import numpy as np
import pytest

from conftest import golden_text
from helpers import check_against_golden
from oracle import oracle as O
from paper_2111_12478_b200 import _native as N
from paper_2111_12478_b200 import workloads as WL
from paper_2111_12478_b200.report import ndjson_lines
from paper_2111_12478_b200.trace import parse_trace

pytestmark = pytest.mark.gpu


@pytest.fixture
def ctx(monkeypatch):
    monkeypatch.setenv("GW_BUCKET", "1")
    c = N.Context(0)
    yield c
    c.close()


def _run(ctx, tr, inactive_opt=True, **kw):
    ctx.analyze_host(tr.cfg_tuple, tr.key, tr.tidop, tr.instr, inactive_opt=inactive_opt, **kw)
    return ctx.fetch()


def _lock_free(tr) -> bool:
    kinds = (tr.tidop >> np.uint32(N.OP_SHIFT)) & np.uint32(7)
    return not np.any((kinds == N.K_ACQUIRE) | (kinds == N.K_RELEASE))


def test_bucket_pass_matches_reference_goldens(goldens, ctx):
    n = 0
    for r in goldens:
        if "error" in r or "full" in r["tags"]:
            continue
        tr = parse_trace(golden_text(r))
        if not _lock_free(tr):
            continue
        check_against_golden(r, tr, _run(ctx, tr, r["inactive_opt"]))
        n += 1
    assert n > 700


def test_bucket_pass_full_c2(goldens, ctx):
    r = next(r for r in goldens if r["name"] == "c2/full")
    tr = WL.c2_soa()
    res = _run(ctx, tr)
    check_against_golden(r, tr, res)
    assert ctx.stats().sort_bits == 12  # the bucket bits (the LSD path reports 17 key bits): the bucketed pass ran


@pytest.mark.parametrize("seed", range(3))
def test_bucket_pass_c4_geometries(ctx, seed):
    tr = parse_trace(WL.c4_text(blocks=4 + 6 * seed, warps=8, lanes=32, iters=20 + 10 * seed, words_per_block=1024,
                                seed=200 + seed))
    assert ndjson_lines(tr, _run(ctx, tr)) == ndjson_lines(tr, O.run_trace(tr))


def _hot_text(seed=0, blocks=8, warps=8, lanes=32, rounds=24, hot=3):
    """A few hot words read and written by every lane of every warp (buckets
    far above the shared-memory capacity), private words beside them,
    warp and block barriers in between."""
    import random

    rng = random.Random(seed)
    lines = [f"config blocks={blocks} warps={warps} lanes={lanes}"]
    full = (1 << lanes) - 1
    for r in range(rounds):
        for b in range(blocks):
            for w in range(warps):
                op = "wr" if rng.random() < 0.3 else "rd"
                addrs = []
                for l in range(lanes):
                    if rng.random() < 0.7:
                        addrs.append(f"g:{0x100 + 4 * rng.randrange(hot):#x}")
                    else:
                        addrs.append(f"g:{0x10000 + 4 * (((b * warps + w) * lanes + l) * 64 + r % 64):#x}")
                lines.append(f"wacc {b} {w} {full:#x} {op} {','.join(addrs)} instr {r % 7}")
                if rng.random() < 0.2:
                    lines.append(f"bar warp {b} {w} {rng.randrange(1, full + 1):#x}")
        if r % 6 == 5:
            for b in range(blocks):
                lines.append(f"bar block {b}")
    return "\n".join(lines) + "\n"


@pytest.mark.parametrize("seed", range(2))
def test_bucket_pass_hot_locations_spill(ctx, seed):
    """Buckets above kBkCap records go through the spill path (LSD sort by
    the location hash + k_access with lazily looked-up stamps), reader
    windows of hundreds of reads through the large-window pass."""
    tr = parse_trace(_hot_text(seed))
    got = _run(ctx, tr)
    want = O.run_trace(tr)
    assert ndjson_lines(tr, got) == ndjson_lines(tr, want)
    assert len(want["kind"]) > 10


def test_bucket_pass_large_windows_in_bucket(ctx):
    """Large reader windows inside a bucket that fits shared memory."""
    tr = parse_trace(_hot_text(5, blocks=4, warps=4, rounds=6, hot=40))
    assert ndjson_lines(tr, _run(ctx, tr)) == ndjson_lines(tr, O.run_trace(tr))


@pytest.mark.parametrize("mode", ["block", "warp", "walker"])
def test_bucket_pass_sync_pass_modes(ctx, mode, monkeypatch):
    """Stamps from every lock-free sync-pass form (block / warp snapshots,
    the walker's per-event arrays)."""
    monkeypatch.setenv("GW_WALK_MODE", mode)
    for tr in (parse_trace(WL.c4_text(blocks=6, warps=8, lanes=32, iters=30, words_per_block=512, seed=300)),
               WL.c2_soa(blocks=16, warps=4, lanes=32, phases=4, records=4, words_per_block=256, seed=302)):
        assert ndjson_lines(tr, _run(ctx, tr)) == ndjson_lines(tr, O.run_trace(tr))


def test_bucket_pass_graph_replay(ctx):
    """The bench's path: graph replays of the bucketed pass on a stream, new
    contents every call, one call breaking the plan (eager fallback)."""
    import torch

    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    geo = dict(blocks=32, warps=8, lanes=32, phases=4, records=6)
    traces = [WL.c2_soa(**geo, words_per_block=1024, seed=s) for s in (61, 62)]
    traces.append(WL.c2_soa(**geo, words_per_block=8192, seed=63))  # wider keys: plan check aborts
    traces.append(WL.c2_soa(**geo, words_per_block=1024, seed=64))
    n = len(traces[0])
    bufs = [torch.empty(n, dtype=torch.int64, device=dev), torch.empty(n, dtype=torch.int32, device=dev),
            torch.empty(n, dtype=torch.int32, device=dev)]
    for _ in range(2):
        for tr in traces:
            bufs[0].copy_(torch.from_numpy(tr.key.view(np.int64)))
            bufs[1].copy_(torch.from_numpy(tr.tidop.view(np.int32)))
            bufs[2].copy_(torch.from_numpy(tr.instr.view(np.int32)))
            torch.cuda.synchronize()
            ctx.analyze_device(tr.cfg_tuple, n, bufs[0].data_ptr(), bufs[1].data_ptr(), bufs[2].data_ptr(),
                               stream=stream.cuda_stream)
            assert ndjson_lines(tr, ctx.fetch()) == ndjson_lines(tr, O.run_trace(tr))


def test_bucket_pass_threshold_on_c5_geometry(monkeypatch):
    """GW_BUCKET=2 takes the bucketed pass from 2^24 accesses on: a
    21M-event C5-recipe trace (1024 x 8 x 32 threads, 2 phases x 40 records)
    against the LSD path (the default) and the oracle."""
    p = dict(blocks=1024, warps=8, lanes=32, phases=2, records=40, words_per_block=262144, seed=5)
    tr = WL.c2_soa(**p)
    monkeypatch.setenv("GW_BUCKET", "2")
    c = N.Context(0)
    a = _run(c, tr)
    assert c.stats().sort_bits == 14  # bucket bits of 21M accesses: the bucketed pass ran
    monkeypatch.delenv("GW_BUCKET")
    b = _run(c, tr)
    c.close()
    for f in ("kind", "prior", "current"):
        assert np.array_equal(a[f], b[f])
    assert ndjson_lines(tr, a) == ndjson_lines(tr, O.run_trace(tr))
