"""validate_trace and infer_locks on the GPU
against the reference's outputs: the `validate` field of every golden trace
(tests/golden/make_golden.py) and the infer_locks goldens
(tests/golden/make_golden_infer.py: the rewritten trace's SoA hash, the
inference diagnostics, validate_trace and `check` of the rewritten trace)."""

import gzip
import json
import os

import numpy as np
import pytest

from conftest import REPO, golden_text
from helpers import soa_sha
from paper_2111_12478_b200 import _native as N
from paper_2111_12478_b200 import workloads as WL
from paper_2111_12478_b200.engine import diagnostics_of
from paper_2111_12478_b200.report import ndjson_lines
from paper_2111_12478_b200.trace import infer_locks, parse_trace, validate_trace

pytestmark = pytest.mark.gpu

GOLDEN_INFER = os.path.join(REPO, "tests", "golden", "golden_infer.jsonl.gz")


@pytest.fixture(scope="module")
def ctx():
    c = N.Context(0)
    yield c
    c.close()


def test_gpu_validate_matches_reference_goldens(goldens, ctx):
    n = nd = 0
    for r in goldens:
        if "error" in r:
            continue
        tr = parse_trace(golden_text(r))
        got = [str(d) for d in validate_trace(tr, ctx=ctx)]
        assert got == r["validate"], r["name"]
        n += 1
        nd += len(got)
    assert n > 5000 and nd > 500


def test_gpu_validate_matches_host_pass_on_workloads(ctx):
    for tr in (WL.c2_soa(blocks=16, warps=8, lanes=32, phases=4, records=4, words_per_block=512),
               parse_trace(WL.c3_text(blocks=8, warps=4, lanes=32, iters=10, locks=8, region=8, private=64)),
               parse_trace(WL.c4_text(blocks=6, warps=8, lanes=32, iters=20, words_per_block=512))):
        assert validate_trace(tr, ctx=ctx) == validate_trace(tr)


def _infer_goldens():
    with gzip.open(GOLDEN_INFER, "rt", encoding="utf-8") as fh:
        return [json.loads(line) for line in fh]


def test_gpu_infer_locks_matches_reference(ctx):
    n_diag = n_rep = 0
    for r in _infer_goldens():
        tr = parse_trace(r["text"])
        out, diags = infer_locks(tr, ctx=ctx)
        assert soa_sha(out) == r["infer_sha"], r["name"]
        assert len(out) == r["n_events"]
        assert [str(d) for d in diags] == r["diags"], r["name"]
        assert [str(d) for d in validate_trace(out, ctx=ctx)] == r["validate"], r["name"]
        n_diag += len(diags)
        if "reports" in r:
            ctx.analyze_host(out.cfg_tuple, out.key, out.tidop, out.instr)
            res = ctx.fetch()
            assert ndjson_lines(out, res) == r["reports"], r["name"]
            assert [str(d) for d in diagnostics_of(out, res)] == r["run_diags"], r["name"]
            n_rep += len(r["reports"])
    assert n_diag > 100 and n_rep > 100


def test_gpu_infer_locks_on_a_large_trace(ctx):
    """Lock idioms spread over many threads: every thread's halves pair up
    (acquire = atomic write + fence, release = fence + atomic write)."""
    text = WL.c3_text(blocks=16, warps=4, lanes=32, iters=6, locks=16, region=8, private=64)
    # rewrite the explicit locks into the raw idioms the NVBit tool would record
    lines = []
    for line in text.splitlines():
        parts = line.split()
        if len(parts) == 4 and parts[1] in ("acq", "rel"):
            tid, op, lock, sc = parts
            if op == "acq":
                lines += [f"{tid} wr g:{lock} atomic {sc}", f"{tid} fence {sc}"]
            else:
                lines += [f"{tid} fence {sc}", f"{tid} wr g:{lock} atomic {sc}"]
        else:
            lines.append(line)
    raw = parse_trace("\n".join(lines) + "\n")
    out, diags = infer_locks(raw, ctx=ctx)
    assert diags == []
    kinds = (out.tidop >> np.uint32(N.OP_SHIFT)) & np.uint32(7)
    want = parse_trace(text)
    wk = (want.tidop >> np.uint32(N.OP_SHIFT)) & np.uint32(7)
    assert int((kinds == N.K_ACQUIRE).sum()) == int((wk == N.K_ACQUIRE).sum()) > 0
    assert int((kinds == N.K_RELEASE).sum()) == int((wk == N.K_RELEASE).sum())
