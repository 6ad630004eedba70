"""Shared helpers for the parity tests."""

import hashlib
import json

from paper_2111_12478_b200.engine import diagnostics_of
from paper_2111_12478_b200.report import ndjson_lines


def soa_sha(tr) -> str:
    h = hashlib.sha256()
    h.update(json.dumps([tr.config.blocks, tr.config.warps, tr.config.lanes]).encode())
    h.update(tr.key.tobytes())
    h.update(tr.tidop.tobytes())
    h.update(tr.instr.tobytes())
    return h.hexdigest()


def lines_sha(lines) -> str:
    return hashlib.sha256(("\n".join(lines) + "\n").encode()).hexdigest() if lines else ""


def check_against_golden(rec, tr, res, detector="gwcp"):
    """Assert engine/oracle result arrays reproduce the reference's golden output."""
    lines = ndjson_lines(tr, res, detector)
    diags = [str(d) for d in diagnostics_of(tr, res)]
    name = rec["name"]
    assert len(lines) == rec["n_reports"], f"{name}: {len(lines)} reports, reference {rec['n_reports']}"
    if "reports" in rec:
        assert lines == rec["reports"], f"{name}: report lines differ"
    else:
        assert lines[:50] == rec["reports_head"], f"{name}: report head differs"
        assert lines_sha(lines) == rec["reports_sha"], f"{name}: report sha differs"
    assert diags == rec["diags"], f"{name}: diagnostics differ"
