"""Generate golden vectors from the REFERENCE implementation (run here, where
/root/reference exists; the fixtures travel, the reference does not).

    python tests/golden/make_golden.py

Writes tests/golden/golden.jsonl.gz.  Each record is one trace (its text) and
what the reference produces for it:
  reports  the NDJSON lines of `gpurace check` (or sha256 + count + head for
           the larger traces), diags the detector diagnostics,
  validate validate_trace() messages,
  soa_sha  sha256 of the SoA encoding of the reference's parse_trace() result
           (pins the native parser),
  error    for malformed text: the reference's TraceParseError string.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import random
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from gpurace.engine import run as ref_run  # noqa: E402
from gpurace.gwcp import GwcpDetector  # noqa: E402
from gpurace.litmus import corpus_entry, corpus_names, gen_random  # noqa: E402
from gpurace.trace import TraceParseError, format_trace, parse_trace, validate_trace  # noqa: E402

from paper_2111_12478_b200 import workloads as WL  # noqa: E402
from paper_2111_12478_b200.trace import encode  # noqa: E402

FULL_LINES_MAX = 400


def soa_sha(tr) -> str:
    s = encode(tr)
    hsh = hashlib.sha256()
    hsh.update(json.dumps([s.config.blocks, s.config.warps, s.config.lanes]).encode())
    hsh.update(s.key.tobytes())
    hsh.update(s.tidop.tobytes())
    hsh.update(s.instr.tobytes())
    return hsh.hexdigest()


def record(name: str, text: str, inactive_opt: bool = True, tags=(), gen=None) -> dict:
    tr = parse_trace(text)
    res = ref_run(tr, GwcpDetector(tr.config, inactive_opt=inactive_opt))
    lines = [r.to_json() for r in res.reports]
    rec = {
        "name": name,
        "text": text,
        "inactive_opt": inactive_opt,
        "n_events": len(tr.events),
        "n_reports": len(lines),
        "diags": [str(d) for d in res.diagnostics],
        "validate": [str(d) for d in validate_trace(tr)],
        "soa_sha": soa_sha(tr),
        "tags": list(tags),
    }
    if gen is not None:  # regenerable from paper_2111_12478_b200.workloads: keep the fixture small
        del rec["text"]
        rec["gen"] = gen
    if len(lines) <= FULL_LINES_MAX:
        rec["reports"] = lines
    else:
        rec["reports_head"] = lines[:50]
    rec["reports_sha"] = hashlib.sha256(("\n".join(lines) + "\n").encode()).hexdigest() if lines else ""
    return rec


def gen_nasty(seed, allow_post_end=False, n=50):
    """Random traces that break the generator's discipline: nested / reentrant /
    unheld lock ops, exits holding locks, warp records, optional post-END events."""
    rng = random.Random(seed)
    B, W, L = rng.randint(1, 3), rng.randint(1, 2), rng.randint(1, 4)
    lines = [f"config blocks={B} warps={W} lanes={L}"]
    ended = set()
    locs = ["g:0x10", "g:0x14", "s:0x20", "g:0x18"]
    for _ in range(n):
        b, w, l = rng.randrange(B), rng.randrange(W), rng.randrange(L)
        if not allow_post_end and (b, w, l) in ended:
            continue
        r = rng.random()
        tid = f"{b}.{w}.{l}"
        if r < 0.35:
            s = f"{tid} {rng.choice(['rd', 'wr'])} {rng.choice(locs)}"
            if rng.random() < 0.3:
                s += " atomic " + rng.choice(["block", "device", "system"])
            if rng.random() < 0.5:
                s += f" instr {rng.randint(0, 5)}"
            lines.append(s)
        elif r < 0.45:
            mask = rng.randint(1, (1 << L) - 1)
            lanes = [i for i in range(L) if mask >> i & 1]
            if not allow_post_end and any((b, w, i) in ended for i in lanes):
                continue
            s = f"wacc {b} {w} {mask:#x} {rng.choice(['rd', 'wr'])} " + ",".join(rng.choice(locs) for _ in lanes)
            if rng.random() < 0.2:
                s += " atomic " + rng.choice(["block", "device"])
            if rng.random() < 0.5:
                s += f" instr {rng.randint(0, 5)}"
            lines.append(s)
        elif r < 0.62:
            lines.append(f"{tid} acq {rng.choice(['0xa', '0xb', '0xc'])} {rng.choice(['block', 'device'])}")
        elif r < 0.78:
            lines.append(f"{tid} rel {rng.choice(['0xa', '0xb', '0xc'])} {rng.choice(['block', 'device'])}")
        elif r < 0.83:
            lines.append(f"{tid} fence device")
        elif r < 0.89:
            lines.append(f"bar block {b}")
        elif r < 0.95:
            lines.append(f"bar warp {b} {w} {rng.randint(1, (1 << L) - 1):#x}")
        else:
            lines.append(f"{tid} end")
            ended.add((b, w, l))
    return "\n".join(lines) + "\n"


def large_window_text(seed=0) -> str:
    rng = random.Random(seed)
    B, W, L = 2, 4, 32
    lines = [f"config blocks={B} warps={W} lanes={L}"]
    full = (1 << L) - 1
    for rnd in range(3):
        order = [(b, w) for b in range(B) for w in range(W)]
        rng.shuffle(order)
        for b, w in order:
            addrs = ",".join("g:0x10" if rng.random() < 0.8 else "g:0x14" for _ in range(L))
            lines.append(f"wacc {b} {w} {full:#x} rd {addrs} instr {rnd * 10 + w}")
            if rng.random() < 0.3:
                lines.append(f"{b}.{w}.{rng.randrange(L)} rd g:0x10 instr 77")
        lines.append(f"{rng.randrange(B)}.{rng.randrange(W)}.{rng.randrange(L)} wr g:0x10 instr {100 + rnd}")
        if rnd == 1:
            for b in range(B):
                lines.append(f"bar block {b}")
    return "\n".join(lines) + "\n"


PARSE_ERRORS = {
    "no-config": "0.0.0 wr g:0x10\n",
    "empty": "# nothing\n\n",
    "bad-config-entry": "config blocks=1 warps\n",
    "config-missing": "config blocks=1 lanes=1\n",
    "config-nonpositive": "config blocks=0 warps=1 lanes=1\n",
    "config-badint": "config blocks=x warps=1 lanes=1\n",
    "dup-config": "config blocks=1 warps=1 lanes=1\nconfig blocks=1 warps=1 lanes=1\n",
    "bad-tid": "config blocks=1 warps=1 lanes=1\n0.0 wr g:0x10\n",
    "tid-range": "config blocks=1 warps=1 lanes=1\n0.0.1 wr g:0x10\n",
    "block-range": "config blocks=1 warps=1 lanes=1\n3.0.0 wr g:0x10\n",
    "warp-range": "config blocks=1 warps=1 lanes=1\n0.2.0 wr g:0x10\n",
    "bad-loc": "config blocks=1 warps=1 lanes=1\n0.0.0 wr x:0x10\n",
    "bad-addr": "config blocks=1 warps=1 lanes=1\n0.0.0 wr g:zz\n",
    "no-loc": "config blocks=1 warps=1 lanes=1\n0.0.0 wr\n",
    "atomic-noscope": "config blocks=1 warps=1 lanes=1\n0.0.0 wr g:0x10 atomic\n",
    "bad-scope": "config blocks=1 warps=1 lanes=1\n0.0.0 wr g:0x10 atomic grid\n",
    "instr-noval": "config blocks=1 warps=1 lanes=1\n0.0.0 wr g:0x10 instr\n",
    "instr-neg": "config blocks=1 warps=1 lanes=1\n0.0.0 wr g:0x10 instr -3\n",
    "unexpected": "config blocks=1 warps=1 lanes=1\n0.0.0 wr g:0x10 foo\n",
    "lockop-arity": "config blocks=1 warps=1 lanes=1\n0.0.0 acq 0xa\n",
    "fence-arity": "config blocks=1 warps=1 lanes=1\n0.0.0 fence\n",
    "end-arity": "config blocks=1 warps=1 lanes=1\n0.0.0 end now\n",
    "unknown-op": "config blocks=1 warps=1 lanes=1\n0.0.0 jump\n",
    "bar-bad": "config blocks=1 warps=1 lanes=1\nbar grid\n",
    "bar-block-range": "config blocks=1 warps=1 lanes=1\nbar block 4\n",
    "bar-trailing": "config blocks=1 warps=1 lanes=1\nbar block 0 x\n",
    "bar-warp-range": "config blocks=1 warps=1 lanes=1\nbar warp 0 3 0x1\n",
    "bar-mask": "config blocks=1 warps=1 lanes=2\nbar warp 0 0 0x4\n",
    "wacc-short": "config blocks=1 warps=1 lanes=2\nwacc 0 0 0x3\n",
    "wacc-range": "config blocks=1 warps=1 lanes=2\nwacc 0 5 0x3 rd g:0x1,g:0x2\n",
    "wacc-mask": "config blocks=1 warps=1 lanes=2\nwacc 0 0 0x0 rd g:0x1\n",
    "wacc-kind": "config blocks=1 warps=1 lanes=2\nwacc 0 0 0x3 xx g:0x1,g:0x2\n",
    "wacc-count": "config blocks=1 warps=1 lanes=2\nwacc 0 0 0x3 rd g:0x1\n",
    "wacc-badloc": "config blocks=1 warps=1 lanes=2\nwacc 0 0 0x3 rd g:0x1,q:0x2\n",
    "quote-repr": "config blocks=1 warps=1 lanes=1\n0.0.0 x'y\n",
    "hex-tid": "config blocks=2 warps=1 lanes=1\n0x1.0.0 wr g:0x10\n1.0.0 wr g:0x10\n",
    "underscore": "config blocks=1_0 warps=1 lanes=1\n1_0.0.0 wr g:0x1_0\n",
    "crlf": "config blocks=1 warps=1 lanes=1\r\n0.0.0 wr g:0x10\r\n0.0.0 wr g:0x10 # c\r\n",
}


def main() -> None:
    t0 = time.time()
    recs = []
    for name in corpus_names():
        recs.append(record(f"corpus/{name}", corpus_entry(name).text, tags=["corpus"]))
        recs.append(record(f"corpus/{name}/noio", corpus_entry(name).text, inactive_opt=False, tags=["corpus"]))
    for s in range(2000):
        recs.append(record(f"random/{s}", format_trace(gen_random(s)), tags=["random"]))
    for s in range(1000):
        tr = gen_random(s, blocks=3, warps=2, lanes=4, events=60, locations=5)
        recs.append(record(f"random-wide/{s}", format_trace(tr), tags=["random"]))
    for s in range(200):
        tr = gen_random(s, blocks=2, warps=2, lanes=3, events=200, locations=3)
        recs.append(record(f"random-long/{s}", format_trace(tr), tags=["random"]))
    for s in range(1000):
        recs.append(record(f"nasty/{s}", gen_nasty(s, False), tags=["nasty"]))
    for s in range(600):
        recs.append(record(f"nasty-postend/{s}", gen_nasty(1000 + s, True), tags=["nasty", "postend"]))
    for s in range(300):
        recs.append(record(f"nasty-postend-noio/{s}", gen_nasty(2000 + s, True), inactive_opt=False,
                           tags=["nasty", "postend"]))
    for name, text in WL.c1_texts().items():
        recs.append(record(f"c1/{name}", text, tags=["c1"]))
    for s in range(4):
        recs.append(record(f"largewin/{s}", large_window_text(s), tags=["largewin"]))
    recs.append(record("c2/small", WL.soa_to_text(WL.c2_soa(blocks=4, warps=2, lanes=32, phases=4, records=4,
                                                            words_per_block=64)), tags=["c2"]))
    g = {"fn": "c2_soa", "args": dict(blocks=16, warps=8, lanes=32, phases=8, records=8, words_per_block=1024)}
    recs.append(record("c2/16x8x32", WL.soa_to_text(WL.c2_soa(**g["args"])), tags=["c2"], gen=g))
    recs.append(record("c3/small", WL.c3_text(blocks=2, warps=2, lanes=32, iters=8, locks=4, region=8, private=64),
                       tags=["c3"]))
    g = {"fn": "c3_text", "args": dict(blocks=8, warps=4, lanes=32, iters=20, locks=32, region=16, private=128)}
    recs.append(record("c3/8x4x32", WL.c3_text(**g["args"]), tags=["c3"], gen=g))
    recs.append(record("c4/small", WL.c4_text(blocks=2, warps=2, lanes=32, iters=16, words_per_block=256),
                       tags=["c4"]))
    g = {"fn": "c4_text", "args": dict(blocks=8, warps=8, lanes=32, iters=24, words_per_block=4096)}
    recs.append(record("c4/8x8x32", WL.c4_text(**g["args"]), tags=["c4"], gen=g))
    t_big = time.time()
    big = WL.c2_soa()  # full C2, 1,049,088 events
    recs.append(record("c2/full", WL.soa_to_text(big), tags=["c2", "full"], gen={"fn": "c2_soa", "args": {}}))
    print(f"full C2 golden in {time.time() - t_big:.1f}s", file=sys.stderr)
    for name, text in PARSE_ERRORS.items():
        try:
            tr = parse_trace(text)
        except TraceParseError as e:
            recs.append({"name": f"parse/{name}", "text": text, "error": str(e), "tags": ["parse"]})
        else:
            r = record(f"parse/{name}", text, tags=["parse"])
            recs.append(r)
    out = os.path.join(HERE, "golden.jsonl.gz")
    with gzip.open(out, "wt", encoding="utf-8") as fh:
        for r in recs:
            fh.write(json.dumps(r, separators=(",", ":")) + "\n")
    print(f"wrote {len(recs)} records to {out} in {time.time() - t0:.1f}s", file=sys.stderr)


if __name__ == "__main__":
    main()
