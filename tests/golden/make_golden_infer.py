"""Golden vectors for infer_locks, made by the REFERENCE
(run here, where /root/reference exists; the fixture travels, the reference
does not).

    python tests/golden/make_golden_infer.py

For random traces rich in the atomic-write / fence idioms the reference's
infer_locks rewrites (pkg/src/gpurace/trace.py:609-680) -- acquire and
release halves, unmatched and unheld halves, other threads' events between
the halves, shared-memory lock words, mixed device / block scopes, wacc
records -- records the SoA hash of the rewritten trace, its inference
diagnostics, validate_trace of the rewritten trace and the `check` reports
of it.  Plus the cases of pkg/tests/test_trace.py:179-246.

Writes tests/golden/golden_infer.jsonl.gz.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from gpurace.engine import run as ref_run  # noqa: E402
from gpurace.gwcp import GwcpDetector  # noqa: E402
from gpurace.trace import infer_locks, parse_trace, validate_trace  # noqa: E402

from paper_2111_12478_b200.trace import encode  # noqa: E402

CASES = {  # pkg/tests/test_trace.py:179-246
    "acq-weaker-scope": "config blocks=1 warps=1 lanes=1\n0.0.0 wr g:0xa0 atomic block\n0.0.0 fence device\n",
    "rel-device": ("config blocks=1 warps=1 lanes=1\n0.0.0 wr g:0xa0 atomic device\n0.0.0 fence device\n"
                   "0.0.0 fence device\n0.0.0 wr g:0xa0 atomic device\n"),
    "unmatched-atomic": "config blocks=1 warps=1 lanes=1\n0.0.0 wr g:0x10 atomic device\n",
    "unheld-release": "config blocks=1 warps=1 lanes=1\n0.0.0 fence device\n0.0.0 wr g:0xa0 atomic device\n",
    "plain-accesses": ("config blocks=1 warps=1 lanes=1\n0.0.0 wr g:0x10\n0.0.0 wr g:0xa0 atomic device\n"
                       "0.0.0 fence device\n0.0.0 rd g:0x14\n0.0.0 fence device\n0.0.0 wr g:0xa0 atomic device\n"
                       "0.0.0 wr g:0x18\n"),
    "other-thread-between": ("config blocks=2 warps=1 lanes=1\n0.0.0 wr g:0xa0 atomic device\n1.0.0 wr g:0x10\n"
                             "0.0.0 fence device\n"),
}


def sha(tr) -> str:
    s = encode(tr)
    h = hashlib.sha256()
    h.update(json.dumps([s.config.blocks, s.config.warps, s.config.lanes]).encode())
    for a in (s.key, s.tidop, s.instr):
        h.update(a.tobytes())
    return h.hexdigest()


def gen(seed: int) -> str:
    rng = random.Random(seed)
    B, W, L = rng.randint(1, 3), rng.randint(1, 2), rng.randint(1, 4)
    lines = [f"config blocks={B} warps={W} lanes={L}"]
    lockw = ["g:0xa0", "g:0xa4", "s:0xb0"]
    data = ["g:0x10", "g:0x14", "s:0x20"]
    for _ in range(rng.randint(10, 60)):
        b, w, l = rng.randrange(B), rng.randrange(W), rng.randrange(L)
        tid = f"{b}.{w}.{l}"
        r = rng.random()
        sc = rng.choice(["device", "block", "system"])
        if r < 0.25:
            lines.append(f"{tid} wr {rng.choice(lockw)} atomic {sc}")
        elif r < 0.45:
            lines.append(f"{tid} fence {rng.choice(['device', 'block'])}")
        elif r < 0.55:  # an acquire idiom right away
            lines.append(f"{tid} wr {rng.choice(lockw)} atomic {sc}")
            lines.append(f"{tid} fence {rng.choice(['device', 'block'])}")
        elif r < 0.62:  # a release idiom
            lines.append(f"{tid} fence {rng.choice(['device', 'block'])}")
            lines.append(f"{tid} wr {rng.choice(lockw)} atomic {sc}")
        elif r < 0.85:
            op = rng.choice(["rd", "wr"])
            extra = f" atomic {sc}" if rng.random() < 0.15 else ""
            lines.append(f"{tid} {op} {rng.choice(data)}{extra}")
        elif r < 0.92 and L > 1:
            mask = rng.randint(1, (1 << L) - 1)
            n = bin(mask).count("1")
            addrs = ",".join(rng.choice(lockw + data) for _ in range(n))
            extra = f" atomic {sc}" if rng.random() < 0.5 else ""
            lines.append(f"wacc {b} {w} {mask:#x} wr {addrs}{extra}")
        elif r < 0.96:
            lines.append(f"bar block {b}")
        else:
            lines.append(f"{tid} rd g:0x10")
    return "\n".join(lines) + "\n"


def record(name: str, text: str) -> dict:
    tr = parse_trace(text)
    out, diags = infer_locks(tr)
    vd = validate_trace(out)
    rec = {"name": name, "text": text, "infer_sha": sha(out), "n_events": len(out.events),
           "diags": [str(d) for d in diags], "validate": [str(d) for d in vd]}
    if not vd:
        try:
            res = ref_run(out, GwcpDetector(out.config))
        except AssertionError:
            # the reference's _same_instruction_check (engine.py:81-95) asserts on a
            # WRITE record one of whose lane events was inferred into an acquire
            rec["run_error"] = "AssertionError in gpurace.engine._same_instruction_check"
        else:
            rec["reports"] = [r.to_json() for r in res.reports]
            rec["run_diags"] = [str(d) for d in res.diagnostics]
    return rec


def main() -> None:
    recs = [record(f"case/{k}", v) for k, v in CASES.items()]
    recs += [record(f"random/{s}", gen(s)) for s in range(600)]
    out = os.path.join(HERE, "golden_infer.jsonl.gz")
    with gzip.open(out, "wt", encoding="utf-8") as fh:
        for r in recs:
            fh.write(json.dumps(r, separators=(",", ":")) + "\n")
    n_inf = sum(1 for r in recs if r["diags"])
    print(f"wrote {len(recs)} records ({n_inf} with inference diagnostics, "
          f"{sum(1 for r in recs if 'reports' in r)} analysed) to {out}", file=sys.stderr)


if __name__ == "__main__":
    main()
