"""CPU suite: the oracle, the native parser and validate_trace against the
golden vectors produced by the reference itself (tests/golden/make_golden.py)."""

import pytest

from conftest import golden_text
from helpers import check_against_golden, soa_sha
from oracle import oracle as O
from paper_2111_12478_b200 import TraceParseError, parse_trace, validate_trace


def _records(goldens, *, skip_full=True):
    for r in goldens:
        if "error" in r:
            continue
        if skip_full and "full" in r["tags"]:
            continue
        yield r


def test_golden_fixture_shape(goldens):
    names = {r["name"] for r in goldens}
    assert len([n for n in names if n.startswith("corpus/")]) == 34
    assert "c2/full" in names
    assert sum(1 for r in goldens if "error" in r) >= 30


def test_native_parser_matches_reference_parse(goldens):
    for r in _records(goldens):
        tr = parse_trace(golden_text(r))
        assert len(tr) == r["n_events"], r["name"]
        assert soa_sha(tr) == r["soa_sha"], f"{r['name']}: SoA encoding differs from reference parse_trace"


def test_parse_errors_match_reference(goldens):
    n = 0
    for r in goldens:
        if "error" not in r:
            continue
        with pytest.raises(TraceParseError) as ei:
            parse_trace(r["text"])
        assert str(ei.value) == r["error"], r["name"]
        n += 1
    assert n >= 30


def test_validate_matches_reference(goldens):
    for r in _records(goldens):
        tr = parse_trace(golden_text(r))
        assert [str(d) for d in validate_trace(tr)] == r["validate"], r["name"]


@pytest.mark.parametrize("tag", ["corpus", "random", "nasty", "c1", "largewin", "c2", "c3", "c4", "parse"])
def test_oracle_matches_reference(goldens, tag):
    n = 0
    for r in _records(goldens):
        if tag not in r["tags"]:
            continue
        tr = parse_trace(golden_text(r))
        res = O.run_trace(tr, inactive_opt=r["inactive_opt"])
        check_against_golden(r, tr, res)
        n += 1
    assert n > 0


@pytest.mark.parametrize("tag", ["corpus", "random", "nasty", "c1", "largewin", "c2", "c3", "c4", "parse"])
def test_oracle_hb_matches_reference(goldens_hb, tag):
    """The oracle's scoped-HB mode against the reference's HbDetector (hb.py)."""
    n = 0
    for r, h in goldens_hb:
        if tag not in r["tags"] or "full" in r["tags"]:
            continue
        tr = parse_trace(golden_text(r))
        check_against_golden(h, tr, O.run_trace(tr, hb=True), "hb")
        n += 1
    assert n > 0


@pytest.mark.slow
def test_oracle_full_c2(goldens):
    r = next(r for r in goldens if r["name"] == "c2/full")
    tr = parse_trace(golden_text(r))
    check_against_golden(r, tr, O.run_trace(tr))
