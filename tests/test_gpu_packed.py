"""The packed host input (gw_ctx_analyze_host_packed): narrow key / instr
columns uploaded in chunks and widened on the device give the same reports
as the 16-B SoA path, for every column-width combination."""

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


@pytest.fixture(scope="module")
def ctx():
    c = N.Context(0)
    yield c
    c.close()


def _run_packed(ctx, tr, inactive_opt=True, **kw):
    k, i = N.pack_columns(tr.key, tr.instr, tr.tidop)
    ctx.analyze_host_packed(tr.cfg_tuple, k, tr.tidop, i, inactive_opt=inactive_opt, **kw)
    return ctx.fetch()


def test_packed_input_reference_goldens(goldens, ctx):
    widths = set()
    n = 0
    for r in goldens:
        if "error" in r or "full" in r["tags"] or not ({"corpus", "nasty", "c1", "c3", "c4"} & set(r["tags"])):
            continue
        tr = parse_trace(golden_text(r))
        k, i = N.pack_columns(tr.key, tr.instr, tr.tidop)
        widths.add((k.dtype.itemsize, i.dtype.itemsize))
        check_against_golden(r, tr, _run_packed(ctx, tr, r["inactive_opt"]))
        n += 1
    assert n > 1000
    # shared-memory keys (bit 63) need 8 bytes, warp-barrier lane masks 4 bytes of instr
    assert {(4, 2), (8, 2), (4, 4)} <= widths
    # warp-barrier lane masks (4-byte instr) with 4-byte keys (the warp
    # barriers' block << 32 | warp keys are implied and restored), and with
    # shared-memory keys (8 bytes)
    for text, want in ((WL.c4_text(blocks=2, warps=2, lanes=32, iters=8, words_per_block=256), (4, 4)),
                       ("config blocks=2 warps=1 lanes=32\n0.0.0 wr s:0x10\n0.0.1 rd s:0x10\n"
                        "bar warp 1 0 0xffffffff\n1.0.0 wr g:0x10\nbar warp 0 0 0xffffffff\n0.0.1 wr s:0x10\n",
                        (8, 4))):
        tr = parse_trace(text)
        k, i = N.pack_columns(tr.key, tr.instr, tr.tidop)
        assert (k.dtype.itemsize, i.dtype.itemsize) == want
        assert ndjson_lines(tr, _run_packed(ctx, tr)) == ndjson_lines(tr, O.run_trace(tr))


def test_packed_input_full_c2_chunked(goldens, ctx):
    """1.05 M events: several upload chunks are not needed at this size, so
    also a multi-chunk trace below."""
    r = next(r for r in goldens if r["name"] == "c2/full")
    tr = WL.c2_soa()
    check_against_golden(r, tr, _run_packed(ctx, tr))


def test_packed_input_many_chunks(ctx):
    """> 2^25 events: the upload runs as several chunks, each widened while the
    next is in flight; the graph-replay path on a stream as in the bench."""
    import torch

    tr = WL.c2_soa(blocks=1024, warps=8, lanes=32, phases=2, records=80, words_per_block=262144, seed=5)
    assert len(tr) > (1 << 25)  # two upload chunks
    stream = torch.cuda.Stream(device=torch.device("cuda", 0))
    ctx.analyze_host(tr.cfg_tuple, tr.key, tr.tidop, tr.instr, stream=stream.cuda_stream)
    want = ctx.fetch()
    for _ in range(3):
        got = _run_packed(ctx, tr, stream=stream.cuda_stream)
        for f in ("kind", "prior", "current"):
            assert np.array_equal(got[f], want[f])
    assert ndjson_lines(tr, want) == ndjson_lines(tr, O.run_trace(tr))



def _run_delta(ctx, tr, inactive_opt=True, **kw):
    enc = N.encode_delta(tr.cfg_tuple, tr.key, tr.tidop, tr.instr)
    ctx.analyze_host_delta(enc, inactive_opt=inactive_opt, **kw)
    return ctx.fetch()


def test_delta_input_reference_goldens(goldens, ctx):
    """The delta-varint host form (gw_ctx_analyze_host_delta): decoded on the
    device, the same reports as the 16-B SoA."""
    n = 0
    for r in goldens:
        if "error" in r or "full" in r["tags"] or not ({"corpus", "nasty", "random", "c1", "c3", "c4"} & set(r["tags"])):
            continue
        tr = parse_trace(golden_text(r))
        check_against_golden(r, tr, _run_delta(ctx, tr, r["inactive_opt"]))
        n += 1
    assert n > 3000


def test_delta_input_full_c2_and_many_slices(goldens, ctx):
    import torch

    r = next(r for r in goldens if r["name"] == "c2/full")
    tr = WL.c2_soa()
    check_against_golden(r, tr, _run_delta(ctx, tr))
    # > 1024 chunks of 4096 events: several upload slices, decoded while later ones land;
    # on a stream, so the later calls replay the captured graph
    tr = WL.c2_soa(blocks=1024, warps=8, lanes=32, phases=2, records=80, words_per_block=262144, seed=5)
    stream = torch.cuda.Stream(device=torch.device("cuda", 0))
    ctx.analyze_host(tr.cfg_tuple, tr.key, tr.tidop, tr.instr, stream=stream.cuda_stream)
    want = ctx.fetch()
    for _ in range(3):
        got = _run_delta(ctx, tr, stream=stream.cuda_stream)
        for f in ("kind", "prior", "current"):
            assert np.array_equal(got[f], want[f])


def _run_bp(ctx, tr, inactive_opt=True, **kw):
    enc = N.encode_bp(tr.cfg_tuple, tr.key, tr.tidop, tr.instr)
    ctx.analyze_host_bp(enc, inactive_opt=inactive_opt, **kw)
    return ctx.fetch()


def test_bitpacked_input_reference_goldens(goldens, ctx):
    """The bit-packed host form (gw_ctx_analyze_host_bp): decoded on the
    device (k_bp_decode), the same reports as the 16-B SoA."""
    n = 0
    for r in goldens:
        if "error" in r or "full" in r["tags"] or not ({"corpus", "nasty", "random", "c1", "c3", "c4"} & set(r["tags"])):
            continue
        tr = parse_trace(golden_text(r))
        check_against_golden(r, tr, _run_bp(ctx, tr, r["inactive_opt"]))
        n += 1
    assert n > 3000


def test_bitpacked_input_full_c2_many_slices_and_wide_values(goldens, ctx):
    import torch

    r = next(r for r in goldens if r["name"] == "c2/full")
    tr = WL.c2_soa()
    check_against_golden(r, tr, _run_bp(ctx, tr))
    # > 1024 chunks: several upload slices decoded while later ones land; on a
    # stream, so the later calls replay the captured graph
    tr = WL.c2_soa(blocks=1024, warps=8, lanes=32, phases=2, records=80, words_per_block=262144, seed=5)
    stream = torch.cuda.Stream(device=torch.device("cuda", 0))
    ctx.analyze_host(tr.cfg_tuple, tr.key, tr.tidop, tr.instr, stream=stream.cuda_stream)
    want = ctx.fetch()
    for _ in range(3):
        got = _run_bp(ctx, tr, stream=stream.cuda_stream)
        for f in ("kind", "prior", "current"):
            assert np.array_equal(got[f], want[f])
    # 64-bit shared-memory keys, random instrs: exceptions of every width through the device decoder
    rng = np.random.default_rng(5)
    t = WL.c2_soa_prefix(200_000, **{k: v for k, v in WL.CONFIGS["c5"].items() if k != "gen"})
    key = t.key.copy()
    key[::13] |= np.uint64(1 << 63)
    instr = rng.integers(0, 2**32, len(key), dtype=np.uint64).astype(np.uint32)
    from paper_2111_12478_b200.trace import Trace
    t2 = Trace(t.config, key, t.tidop, instr)
    ctx.analyze_host(t2.cfg_tuple, t2.key, t2.tidop, t2.instr)
    want = ctx.fetch()
    got = _run_bp(ctx, t2)
    for f in ("kind", "prior", "current"):
        assert np.array_equal(got[f], want[f])
