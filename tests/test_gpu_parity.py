"""GPU parity: the CUDA engine (through the C-ABI) against the reference's
golden outputs and the CPU oracle.  Integer work: bit-exact, i.e. the NDJSON
report lines and the diagnostics are byte-identical."""

import numpy as np
import pytest

from conftest import golden_text
from helpers import check_against_golden
from oracle import oracle as O
from paper_2111_12478_b200 import GwcpDetector, parse_trace, run
from paper_2111_12478_b200 import _native as N
from paper_2111_12478_b200 import workloads as WL
from paper_2111_12478_b200.report import ndjson_lines

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return N.Context(0)


def _run(ctx, tr, inactive_opt=True):
    ctx.analyze_host(tr.cfg_tuple, tr.key, tr.tidop, tr.instr, inactive_opt=inactive_opt)
    return ctx.fetch()


@pytest.mark.parametrize("tag", ["corpus", "random", "nasty", "c1", "largewin", "c2", "c3", "c4", "parse"])
def test_engine_matches_reference_goldens(goldens, ctx, tag):
    n = 0
    for r in goldens:
        if "error" in r or tag not in r["tags"] or "full" in r["tags"]:
            continue
        tr = parse_trace(golden_text(r))
        check_against_golden(r, tr, _run(ctx, tr, r["inactive_opt"]))
        n += 1
    assert n > 0


def test_engine_full_c2_matches_reference(goldens, ctx):
    r = next(r for r in goldens if r["name"] == "c2/full")
    tr = WL.c2_soa()
    check_against_golden(r, tr, _run(ctx, tr))


def test_dropin_run_api_on_reference_shaped_objects(goldens):
    # run() accepts Event-object traces (as gpurace users hold them)
    for r in goldens:
        if r["name"] != "corpus/wcp-classic":
            continue
        tr = parse_trace(r["text"])
        res = run(tr, GwcpDetector(tr.config))
        assert [x.to_json() for x in res.reports] == r["reports"]
        # decode to Event objects and back through the encoder
        from paper_2111_12478_b200.trace import Trace

        class Shim:
            config = tr.config
            events = tr.events

        res2 = run(Shim(), GwcpDetector(tr.config))
        assert [x.to_json() for x in res2.reports] == r["reports"]


@pytest.mark.parametrize("seed", range(4))
def test_engine_matches_oracle_c3_geometries(ctx, seed):
    text = WL.c3_text(blocks=4 + 4 * seed, warps=4, lanes=32, iters=12 + 4 * seed, locks=8 << seed, region=16,
                      private=128, seed=100 + seed)
    tr = parse_trace(text)
    assert ndjson_lines(tr, _run(ctx, tr)) == ndjson_lines(tr, O.run_trace(tr))


@pytest.mark.parametrize("seed", range(3))
def test_engine_matches_oracle_c4_geometries(ctx, seed):
    text = WL.c4_text(blocks=4 + 6 * seed, warps=8, lanes=32, iters=20 + 10 * seed, words_per_block=1024,
                      seed=200 + seed)
    tr = parse_trace(text)
    assert ndjson_lines(tr, _run(ctx, tr)) == ndjson_lines(tr, O.run_trace(tr))


@pytest.mark.parametrize("geom", [(64, 8, 32), (300, 4, 32), (1000, 2, 16)])
def test_engine_matches_oracle_c2_geometries(ctx, geom):
    B, W, L = geom
    tr = WL.c2_soa(blocks=B, warps=W, lanes=L, phases=4, records=4, words_per_block=512, seed=B)
    got = _run(ctx, tr)
    want = O.run_trace(tr)
    assert ndjson_lines(tr, got) == ndjson_lines(tr, want)


@pytest.mark.parametrize("blocks", [250, 256])
def test_engine_matches_oracle_c2_sort_size_limits(ctx, blocks):
    """~4.1 M events: the one-sweep location sort at its largest size (~1,000
    tiles, two-level look-back with 32-tile groups, a partial last group) and,
    at 256 blocks, just past it (reduce-then-scan passes)."""
    tr = WL.c2_soa(blocks=blocks, warps=8, lanes=32, phases=8, records=8, words_per_block=1024, seed=blocks)
    got = _run(ctx, tr)
    want = O.run_trace(tr)
    assert ndjson_lines(tr, got) == ndjson_lines(tr, want)


def test_empty_and_tiny_traces(ctx):
    for text in ("config blocks=1 warps=1 lanes=1\n", "config blocks=2 warps=1 lanes=1\n0.0.0 wr g:0x10\n",
                 "config blocks=1 warps=1 lanes=1\nbar block 0\n0.0.0 end\nbar block 0\n"):
        tr = parse_trace(text)
        got = _run(ctx, tr)
        assert len(got["kind"]) == 0


def test_prefix_consistency_c2(ctx):
    """reports of trace[:P] == reports of the full trace with current.event < P."""
    tr = WL.c2_soa(blocks=32, warps=8, lanes=32, phases=8, records=8, words_per_block=1024, seed=9)
    full = _run(ctx, tr)
    for P in (len(tr) // 3, len(tr) // 2):
        # cut at a record boundary
        while P < len(tr) and tr.tidop[P] & N.F_CONT:
            P += 1
        from paper_2111_12478_b200.trace import Trace

        pre = Trace(tr.config, tr.key[:P], tr.tidop[:P], tr.instr[:P])
        got = _run(ctx, pre)
        keep = full["current"] < P
        assert np.array_equal(got["prior"], full["prior"][keep])
        assert np.array_equal(got["current"], full["current"][keep])
        assert np.array_equal(got["kind"], full["kind"][keep])


def _many_readers_text(nthreads=300, seed=0):
    import random

    rng = random.Random(seed)
    lines = ["config blocks=4 warps=4 lanes=32"]
    tids = [(b, w, l) for b in range(4) for w in range(4) for l in range(32)]
    rng.shuffle(tids)
    for i, (b, w, l) in enumerate(tids[:nthreads]):
        lines.append(f"{b}.{w}.{l} rd g:0x10 instr {1000 + i}")
        if rng.random() < 0.3:
            lines.append(f"{b}.{w}.{l} rd g:0x10 instr {5000 + i}")
    b, w, l = tids[-1]
    lines.append(f"{b}.{w}.{l} wr g:0x10 instr 7")
    lines.append(f"wacc 1 1 0xffffffff wr " + ",".join(["g:0x10"] * 32) + " instr 8")
    return "\n".join(lines) + "\n"


@pytest.mark.parametrize("seed", range(3))
def test_many_reports_at_one_event(ctx, seed):
    """> 64 surviving reports at one current event (the big-group ordering path)."""
    tr = parse_trace(_many_readers_text(120 + 150 * seed, seed))
    got = ndjson_lines(tr, _run(ctx, tr))
    assert got == ndjson_lines(tr, O.run_trace(tr))
    assert len(got) > 100


def test_graph_replay_and_plan_mismatch_fallback():
    """Repeated analyses of one shape on a non-default stream replay a captured
    CUDA graph; contents change every call and one call breaks the plan (more
    address bits -> device-side abort -> eager re-run inside fetch)."""
    import torch

    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    ctx = N.Context(0)
    geo = dict(blocks=16, warps=8, lanes=32, phases=4, records=4)
    traces = [WL.c2_soa(**geo, words_per_block=512, seed=s) for s in (11, 12, 13)]
    traces.append(WL.c2_soa(**geo, words_per_block=4096, seed=14))  # wider keys: plan check aborts
    traces.append(WL.c2_soa(**geo, words_per_block=512, seed=15))
    n = len(traces[0])
    bufs = [torch.empty(n, dtype=torch.int64, device=dev), torch.empty(n, dtype=torch.int32, device=dev),
            torch.empty(n, dtype=torch.int32, device=dev)]
    for rep in range(2):
        for tr in traces:
            assert len(tr) == n
            bufs[0].copy_(torch.from_numpy(tr.key.view(np.int64)))
            bufs[1].copy_(torch.from_numpy(tr.tidop.view(np.int32)))
            bufs[2].copy_(torch.from_numpy(tr.instr.view(np.int32)))
            torch.cuda.synchronize()
            ctx.analyze_device(tr.cfg_tuple, n, bufs[0].data_ptr(), bufs[1].data_ptr(), bufs[2].data_ptr(),
                               stream=stream.cuda_stream)
            got = ctx.fetch()
            assert ndjson_lines(tr, got) == ndjson_lines(tr, O.run_trace(tr))


def test_graph_replay_host_path():
    import torch

    stream = torch.cuda.Stream(device=torch.device("cuda", 0))
    ctx = N.Context(0)
    for s in range(4):
        tr = WL.c2_soa(blocks=8, warps=4, lanes=32, phases=4, records=4, words_per_block=256, seed=30 + s)
        ctx.analyze_host(tr.cfg_tuple, tr.key, tr.tidop, tr.instr, stream=stream.cuda_stream)
        assert ndjson_lines(tr, ctx.fetch()) == ndjson_lines(tr, O.run_trace(tr))


def test_device_generator_matches_numpy_recipe():
    import torch

    dev = torch.device("cuda", 0)
    p = dict(blocks=12, warps=4, lanes=32, phases=3, records=5, words_per_block=300, seed=77)
    want = WL.c2_soa(**p)
    n = len(want)
    k = torch.empty(n, dtype=torch.int64, device=dev)
    t = torch.empty(n, dtype=torch.int32, device=dev)
    i = torch.empty(n, dtype=torch.int32, device=dev)
    assert N.gen_c2_device(k.data_ptr(), t.data_ptr(), i.data_ptr(), **p) == n
    torch.cuda.synchronize()
    assert np.array_equal(k.cpu().numpy().view(np.uint64), want.key)
    assert np.array_equal(t.cpu().numpy().view(np.uint32), want.tidop)
    assert np.array_equal(i.cpu().numpy().view(np.uint32), want.instr)


@pytest.mark.parametrize("geom", [(3, 2, 9), (4, 8, 70)])
def test_device_c4_generator_matches_text_recipe(geom):
    import torch

    B, W, it = geom
    want = parse_trace(WL.c4_text(blocks=B, warps=W, lanes=32, iters=it, words_per_block=512, seed=41))
    n = N.c4_events(B, W, it)
    assert n == len(want)
    dev = torch.device("cuda", 0)
    k = torch.empty(n, dtype=torch.int64, device=dev)
    t = torch.empty(n, dtype=torch.int32, device=dev)
    i = torch.empty(n, dtype=torch.int32, device=dev)
    N.gen_c4_device(k.data_ptr(), t.data_ptr(), i.data_ptr(), blocks=B, warps=W, iters=it, words_per_block=512, seed=41)
    torch.cuda.synchronize()
    assert np.array_equal(t.cpu().numpy().view(np.uint32), want.tidop)
    assert np.array_equal(k.cpu().numpy().view(np.uint64), want.key)
    assert np.array_equal(i.cpu().numpy().view(np.uint32), want.instr)


def _dev_c3(p):
    import torch

    dev = torch.device("cuda", 0)
    off = WL.c3_group_offsets(**p)
    n = int(off[-1])
    k = torch.empty(n, dtype=torch.int64, device=dev)
    t = torch.empty(n, dtype=torch.int32, device=dev)
    i = torch.empty(n, dtype=torch.int32, device=dev)
    o = torch.from_numpy(off[:-1].view(np.int64)).to(dev)
    N.gen_c3_device(k.data_ptr(), t.data_ptr(), i.data_ptr(), o.data_ptr(), **p)
    torch.cuda.synchronize()
    return k, t, i


@pytest.mark.parametrize("geom", [(3, 2, 32, 17), (5, 3, 8, 33)])
def test_device_c3_generator_matches_text_recipe(geom):
    B, W, L, it = geom
    p = dict(blocks=B, warps=W, lanes=L, iters=it, locks=16, region=8, private=64, seed=43)
    want = parse_trace(WL.c3_text(**p))
    k, t, i = _dev_c3(p)
    assert np.array_equal(t.cpu().numpy().view(np.uint32), want.tidop)
    assert np.array_equal(k.cpu().numpy().view(np.uint64), want.key)
    assert np.array_equal(i.cpu().numpy().view(np.uint32), want.instr)


@pytest.mark.parametrize("iters", [1, 3])
def test_engine_matches_oracle_c3_full_geometry(ctx, iters):
    """The C3 config's geometry (1024 x 8 x 32 threads, 4096 locks): the first
    iterations of the full trace are a prefix of it."""
    tr = parse_trace(WL.c3_text(blocks=1024, warps=8, lanes=32, iters=iters, locks=4096, region=64, private=512))
    assert ndjson_lines(tr, _run(ctx, tr)) == ndjson_lines(tr, O.run_trace(tr))


def test_engine_c3_denser_races(ctx):
    """Fewer locks and a small private region: many conflicting critical sections."""
    tr = parse_trace(WL.c3_text(blocks=24, warps=4, lanes=32, iters=40, locks=6, region=4, private=32, seed=9))
    got = ndjson_lines(tr, _run(ctx, tr))
    assert got == ndjson_lines(tr, O.run_trace(tr))


def _sharded(ctx, tr, G):
    from paper_2111_12478_b200.shard import merge_shards

    parts = []
    for r in range(G):
        ctx.analyze_host(tr.cfg_tuple, tr.key, tr.tidop, tr.instr, shard=(r, G))
        parts.append(ctx.fetch())
    return merge_shards(parts), parts


@pytest.mark.parametrize("G", [2, 3, 8])
def test_address_sharded_analysis_matches_unsharded(ctx, G):
    """Address sharding (multi-GPU form, gw_opts.shard_*): every shard on this
    GPU in turn, merged by order key == the unsharded analysis."""
    traces = [
        WL.c2_soa(blocks=32, warps=8, lanes=32, phases=4, records=6, words_per_block=512, seed=21),
        parse_trace(WL.c4_text(blocks=8, warps=8, lanes=32, iters=24, words_per_block=512, seed=22)),
        parse_trace(WL.c3_text(blocks=12, warps=4, lanes=32, iters=20, locks=8, region=8, private=64, seed=23)),
        parse_trace(_many_readers_text(200, 3)),
        parse_trace(WL.c1_texts()["colliding-wacc-32"]),
    ]
    for tr in traces:
        full = _run(ctx, tr)
        merged, parts = _sharded(ctx, tr, G)
        for f in ("kind", "prior", "current", "order_key"):
            assert np.array_equal(merged[f], full[f]), f
        assert np.all(np.diff(full["order_key"].astype(np.float64)) > 0)
        for p in parts:  # every shard replicates the sync pass, hence the diagnostics
            assert np.array_equal(p["diag_event"], full["diag_event"])


def test_address_sharded_goldens(goldens, ctx):
    n = 0
    for r in goldens:
        if "error" in r or "full" in r["tags"] or not ({"corpus", "nasty", "largewin"} & set(r["tags"])):
            continue
        tr = parse_trace(golden_text(r))
        merged, _ = _sharded(ctx, tr, 3)
        assert ndjson_lines(tr, merged) == (r["reports"] if "reports" in r else ndjson_lines(tr, _run(ctx, tr)))
        n += 1
    assert n > 0


@pytest.mark.parametrize("mode", ["block", "warp", "walker"])
def test_lock_free_sync_pass_modes(ctx, mode, goldens, monkeypatch):
    """The three lock-free sync-pass forms (block snapshots, per-warp snapshots,
    the sequential walker) give identical, reference-exact results."""
    monkeypatch.setenv("GW_WALK_MODE", mode)
    traces = [
        parse_trace(WL.c4_text(blocks=6, warps=8, lanes=32, iters=30, words_per_block=512, seed=300)),
        parse_trace(WL.c4_text(blocks=3, warps=5, lanes=16, iters=12, words_per_block=256, seed=301)),
        WL.c2_soa(blocks=16, warps=4, lanes=32, phases=4, records=4, words_per_block=256, seed=302),
    ]
    for tr in traces:
        assert ndjson_lines(tr, _run(ctx, tr)) == ndjson_lines(tr, O.run_trace(tr))
    n = 0
    for r in goldens:
        if "error" in r or "full" in r["tags"] or not ({"corpus", "random", "c4"} & set(r["tags"])):
            continue
        tr = parse_trace(golden_text(r))
        check_against_golden(r, tr, _run(ctx, tr, r["inactive_opt"]))
        n += 1
    assert n > 0


@pytest.mark.parametrize("mode", ["warp", "cta"])
def test_lock_walker_modes(ctx, mode, goldens, monkeypatch):
    """Both lock-mode sync passes (one walker warp per trace warp, and the
    CTA-wide walker used for > 8 warps or > 32 lanes) match the reference."""
    monkeypatch.setenv("GW_LOCK_WALK", mode)
    n = 0
    for r in goldens:
        if "error" in r or "full" in r["tags"] or not ({"corpus", "nasty", "random", "c3"} & set(r["tags"])):
            continue
        tr = parse_trace(golden_text(r))
        check_against_golden(r, tr, _run(ctx, tr, r["inactive_opt"]))
        n += 1
    assert n > 0
    tr = parse_trace(WL.c3_text(blocks=20, warps=6, lanes=32, iters=24, locks=12, region=8, private=64, seed=77))
    assert ndjson_lines(tr, _run(ctx, tr)) == ndjson_lines(tr, O.run_trace(tr))


def _run_hb(ctx, tr):
    ctx.analyze_host(tr.cfg_tuple, tr.key, tr.tidop, tr.instr, hb=True)
    return ctx.fetch()


@pytest.mark.parametrize("mode", ["warp", "cta"])
def test_hb_detector_matches_reference(ctx, mode, goldens_hb, monkeypatch):
    """`--detector hb` (GW_OPT_HB) against the reference's HbDetector on every
    golden trace, with both lock-mode sync passes."""
    monkeypatch.setenv("GW_LOCK_WALK", mode)
    n = 0
    for r, h in goldens_hb:
        if "full" in r["tags"]:
            continue
        tr = parse_trace(golden_text(r))
        check_against_golden(h, tr, _run_hb(ctx, tr), "hb")
        n += 1
    assert n > 700


@pytest.mark.parametrize("mode", ["warp", "cta"])
def test_hb_detector_c3_vs_oracle(ctx, mode, monkeypatch):
    monkeypatch.setenv("GW_LOCK_WALK", mode)
    for tr in (
        parse_trace(WL.c3_text(blocks=24, warps=4, lanes=32, iters=40, locks=6, region=4, private=32, seed=9)),
        parse_trace(WL.c3_text(blocks=64, warps=8, lanes=32, iters=6, locks=64, region=16, private=128, seed=5)),
    ):
        assert ndjson_lines(tr, _run_hb(ctx, tr), "hb") == ndjson_lines(tr, O.run_trace(tr, hb=True), "hb")
    # the default detector afterwards is G-WCP again (no state leaks through the context)
    assert ndjson_lines(tr, _run(ctx, tr)) == ndjson_lines(tr, O.run_trace(tr))


def test_hb_dropin_run_api(goldens_hb):
    from paper_2111_12478_b200 import HbDetector

    for r, h in goldens_hb:
        if not r["name"].startswith("corpus/") or "reports" not in h:
            continue
        tr = parse_trace(golden_text(r))
        det = HbDetector(tr.config)
        res = run(tr, det)
        assert [x.to_json() for x in res.reports] == h["reports"], r["name"]
        assert [str(d) for d in det.diagnostics] == h["diags"]
