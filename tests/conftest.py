import gzip
import json
import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden", "golden.jsonl.gz")
GOLDEN_HB = os.path.join(REPO, "tests", "golden", "golden_hb.jsonl.gz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running check")


_cache = None


def golden_records():
    global _cache
    if _cache is None:
        with gzip.open(GOLDEN, "rt", encoding="utf-8") as fh:
            _cache = [json.loads(line) for line in fh]
    return _cache


def golden_text(rec) -> str:
    if "text" in rec:
        return rec["text"]
    from paper_2111_12478_b200 import workloads as WL

    fn = getattr(WL, rec["gen"]["fn"])
    out = fn(**rec["gen"]["args"])
    return out if isinstance(out, str) else WL.soa_to_text(out)


@pytest.fixture(scope="session")
def goldens():
    return golden_records()


@pytest.fixture(scope="session")
def goldens_hb():
    """(golden record, HB golden record) pairs: the reference's HbDetector on
    every golden trace (tests/golden/make_golden_hb.py)."""
    with gzip.open(GOLDEN_HB, "rt", encoding="utf-8") as fh:
        hb = {}
        for line in fh:
            r = json.loads(line)
            hb[r["name"]] = r
    return [(r, hb[r["name"]]) for r in golden_records() if "error" not in r and r["name"] in hb]
