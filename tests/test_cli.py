"""CLI drop-in: exit codes, NDJSON, stderr (reference cli.py:20-84, pkg/tests/test_cli.py)."""

import json
import subprocess
import sys

import pytest

from conftest import REPO, golden_records


def _corpus(name):
    return next(r for r in golden_records() if r["name"] == f"corpus/{name}")


def _cli(tmp_path, text, *extra):
    p = tmp_path / "t.trace"
    p.write_text(text)
    return subprocess.run([sys.executable, "-m", "paper_2111_12478_b200.cli", "check", str(p), *extra],
                          capture_output=True, text=True, cwd=REPO)


def test_parse_error_exits_two(tmp_path):
    r = _cli(tmp_path, "nonsense\n")
    assert r.returncode == 2
    assert "line 1: first line must be a config line" in r.stderr


@pytest.mark.gpu
def test_validation_error_exits_three(tmp_path):
    r = _cli(tmp_path, "config blocks=1 warps=1 lanes=1\n0.0.0 end\n0.0.0 wr g:0x10\n")
    assert r.returncode == 3
    assert "event 1: event after end of thread 0.0.0" in r.stderr
    assert "trace is not well formed" in r.stderr


def test_engine_failure_exits_four_not_one(tmp_path):
    """Without a CUDA device the engine fails loudly, with exit 4 -- never the
    'races found' code (no CPU path)."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("needs a host without a CUDA device")
    r = _cli(tmp_path, _corpus("wcp-classic")["text"])
    assert r.returncode == 4
    assert "analysis engine failed" in r.stderr and r.stdout == ""


_INFER = ("config blocks=2 warps=1 lanes=1\n"
          "0.0.0 wr g:0x10\n0.0.0 wr g:0xa0 atomic device\n0.0.0 fence device\n0.0.0 wr g:{a}\n"
          "0.0.0 fence device\n0.0.0 wr g:0xa0 atomic device\n"
          "1.0.0 wr g:0xa0 atomic device\n1.0.0 fence device\n1.0.0 rd g:0x14\n"
          "1.0.0 fence device\n1.0.0 wr g:0xa0 atomic device\n1.0.0 wr g:0x10\n"
          "1.0.0 fence device\n1.0.0 wr g:0xb0 atomic device\n")


@pytest.mark.gpu
@pytest.mark.parametrize("a,rc,out", [
    # conflicting inferred critical sections order the 0x10 writes (WCP rule (i)): no race
    ("0x14", 0, []),
    # disjoint critical sections: the classic predicted race
    ("0x18", 1, ['{"detector":"gwcp","kind":"ww","location":{"space":"global","addr":"0x10"},'
                 '"prior":{"event":0,"tid":"0.0.0","instr":2},"current":{"event":7,"tid":"1.0.0","instr":13},'
                 '"class":"interblock","confidence":"first"}']),
])
def test_infer_locks_cli(tmp_path, a, rc, out):
    """check --infer-locks against the reference CLI's own output
    (PYTHONPATH=pkg/src python -m gpurace.cli check T --infer-locks)."""
    r = _cli(tmp_path, _INFER.format(a=a), "--infer-locks")
    assert r.returncode == rc
    assert r.stdout.splitlines() == out
    assert "lock inference: event 13: release of lock 0xb0 not held by 1.0.0; left uninferred" in r.stderr


def test_other_detectors_are_not_on_the_accelerated_path(tmp_path):
    r = _cli(tmp_path, _corpus("wcp-classic")["text"], "--detector", "lockset")
    assert r.returncode == 2


@pytest.mark.gpu
def test_hb_detector_cli_matches_reference(tmp_path, goldens_hb):
    n = 0
    for r, h in goldens_hb:
        if not r["name"].startswith("corpus/") or r["name"].endswith("/noio") or "reports" not in h:
            continue
        p = _cli(tmp_path, r["text"], "--detector", "hb")
        assert p.returncode == (1 if h["reports"] else 0), r["name"]
        assert p.stdout.splitlines() == h["reports"], r["name"]
        n += 1
    assert n > 10


@pytest.mark.gpu
def test_racy_trace_exits_one_with_reference_ndjson(tmp_path):
    rec = _corpus("wcp-classic")
    r = _cli(tmp_path, rec["text"])
    assert r.returncode == 1
    assert r.stdout.splitlines() == rec["reports"]
    rep = json.loads(r.stdout.splitlines()[0])
    assert rep["location"] == {"space": "global", "addr": "0x10"} and rep["class"] == "interblock"


@pytest.mark.gpu
def test_clean_trace_exits_zero(tmp_path):
    r = _cli(tmp_path, _corpus("barrier-separated")["text"])
    assert r.returncode == 0 and r.stdout == ""


@pytest.mark.gpu
def test_shared_location_carries_block(tmp_path):
    r = _cli(tmp_path, _corpus("scoped-cs")["text"])
    assert json.loads(r.stdout.splitlines()[0])["location"] == {"space": "shared", "block": 0, "addr": "0x10"}
