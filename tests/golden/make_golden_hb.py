"""Golden vectors of the reference's scoped-HB detector (`gpurace check
--detector hb`, pkg/src/gpurace/hb.py) on every trace of golden.jsonl.gz
(run here, where /root/reference exists):

    python tests/golden/make_golden_hb.py

Writes tests/golden/golden_hb.jsonl.gz: {name, n_reports, reports | reports_head
+ reports_sha, diags} per trace (same texts / generator specs as golden.jsonl.gz).
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
sys.path.insert(0, "/root/reference/pkg/src")

from gpurace.engine import run as ref_run  # noqa: E402
from gpurace.hb import HbDetector  # noqa: E402
from gpurace.trace import parse_trace  # noqa: E402

from conftest import golden_records, golden_text  # noqa: E402

FULL_LINES_MAX = 400


def main() -> None:
    out = []
    for r in golden_records():
        if "error" in r:
            continue
        tr = parse_trace(golden_text(r))
        res = ref_run(tr, HbDetector(tr.config))
        lines = [x.to_json() for x in res.reports]
        rec = {"name": r["name"], "n_reports": len(lines), "diags": [str(d) for d in res.diagnostics]}
        if len(lines) <= FULL_LINES_MAX:
            rec["reports"] = lines
        else:
            rec["reports_head"] = lines[:50]
        rec["reports_sha"] = hashlib.sha256(("\n".join(lines) + "\n").encode()).hexdigest() if lines else ""
        out.append(rec)
    with gzip.open(os.path.join(HERE, "golden_hb.jsonl.gz"), "wt", encoding="utf-8") as fh:
        for rec in out:
            fh.write(json.dumps(rec, separators=(",", ":")) + "\n")
    print(f"{len(out)} traces")


if __name__ == "__main__":
    main()
