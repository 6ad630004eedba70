"""CPU suite: trace ingest beyond the reference grammar tests -- the chunked
multi-threaded text parser (gw_parse_text) and the binary SoA file
(gw_save_soa / gw_load_soa, include/gwcp_b200.h)."""

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import REPO, golden_text
from helpers import soa_sha
from paper_2111_12478_b200 import TraceParseError, UnsupportedTrace, parse_trace
from paper_2111_12478_b200 import workloads as WL
from paper_2111_12478_b200.trace import load_trace, save_soa


def _parse_chunked(text, chunk=64, threads=8):
    code = (
        "import sys, json, hashlib\n"
        "sys.path.insert(0, 'tests')\n"
        "from helpers import soa_sha\n"
        "from paper_2111_12478_b200 import parse_trace, TraceParseError, UnsupportedTrace\n"
        "for text in json.load(sys.stdin):\n"
        "    try:\n"
        "        print(soa_sha(parse_trace(text)))\n"
        "    except TraceParseError as e:\n"
        "        print('ERR', e.line_no, str(e))\n"
        "    except UnsupportedTrace as e:\n"
        "        print('UNS', str(e))\n"
    )
    import json

    env = dict(os.environ, GW_PARSE_MIN_CHUNK=str(chunk), GW_PARSE_THREADS=str(threads))
    r = subprocess.run([sys.executable, "-c", code], input=json.dumps(text), capture_output=True, text=True,
                       cwd=REPO, env=env, check=True)
    return r.stdout.splitlines()


def test_config_only_traces():
    for text in ("config blocks=1 warps=1 lanes=1\n", "config blocks=2 warps=1 lanes=1", "\n#c\nconfig blocks=1 warps=1 lanes=1\n\n"):
        assert len(parse_trace(text)) == 0


def _parse_here(texts):
    out = []
    for t in texts:
        try:
            out.append(soa_sha(parse_trace(t)))
        except TraceParseError as e:
            out.append(f"ERR {e.line_no} {e}")
        except UnsupportedTrace as e:
            out.append(f"UNS {e}")
    return out


def test_chunked_parser_equals_sequential_on_goldens(goldens):
    """Many tiny line-aligned chunks on 8 threads: same SoA and the same first
    error (line number and message) as the one-chunk parse, on every golden
    text including the reference's parse-error cases."""
    texts = [golden_text(r) for r in goldens if "full" not in r.get("tags", [])][:600]
    texts += [
        "config blocks=1 warps=1 lanes=1\n",
        "config blocks=1 warps=1 lanes=1",
        "\n\n# x\nconfig blocks=1 warps=1 lanes=1\n\n\n",
        "config blocks=1 warps=1 lanes=2\r\n0.0.0 rd g:10\r\n\r\n0.0.1 wr g:10\n",
        "config blocks=1 warps=1 lanes=2\r0.0.0 rd g:10\x0b0.0.1 wr g:10",
        "# c\n\nconfig blocks=1 warps=1 lanes=2\n" + "0.0.0 rd g:10\n" * 200 + "0.0.9 rd g:1\n" + "bogus\n" * 50,
    ]
    assert _parse_chunked(texts, chunk=16) == _parse_here(texts)


def test_chunked_parser_large_trace():
    tr = WL.c2_soa(blocks=16, warps=8, lanes=32, phases=4, records=4, words_per_block=512, seed=3)
    text = WL.soa_to_text(tr)
    assert _parse_chunked([text], chunk=4096) == [soa_sha(tr)] == _parse_here([text])


def test_soa_file_round_trip(tmp_path, goldens):
    n = 0
    for r in goldens:
        if "error" in r or not r["name"].startswith("corpus/"):
            continue
        tr = parse_trace(golden_text(r))
        p = str(tmp_path / "t.gwsoa")
        save_soa(tr, p)
        assert os.path.getsize(p) == 32 + 16 * len(tr)
        back = load_trace(p)
        assert back.cfg_tuple == tr.cfg_tuple and soa_sha(back) == soa_sha(tr)
        n += 1
    assert n > 10


def test_soa_file_rejects_malformed(tmp_path):
    tr = parse_trace("config blocks=2 warps=1 lanes=4\n0.0.0 rd g:10\n1.0.3 wr g:10\nbar block 1\n")
    p = str(tmp_path / "t.gwsoa")
    save_soa(tr, p)
    good = open(p, "rb").read()
    cases = {
        "truncated": good[:-3],
        "bad magic": b"X" + good[1:],
        "tid out of range": good[:32 + 24] + np.uint32(8).tobytes() + good[32 + 28:],
        "bad kind": good[:32 + 24] + np.uint32(7 << 24).tobytes() + good[32 + 28:],
        "misaligned barrier": good[:32 + 32] + np.uint32((4 << 24) | 5).tobytes() + good[32 + 36:],
    }
    for name, data in cases.items():
        with open(p, "wb") as fh:
            fh.write(data)
        with pytest.raises(TraceParseError):
            load_trace(p)
        del name


def test_cli_convert_then_check_reads_binary(tmp_path, goldens):
    rec = next(r for r in goldens if r["name"] == "corpus/wcp-classic")
    src = tmp_path / "t.trace"
    src.write_text(rec["text"])
    out = tmp_path / "t.gwsoa"
    r = subprocess.run([sys.executable, "-m", "paper_2111_12478_b200.cli", "convert", str(src), str(out)],
                       capture_output=True, text=True, cwd=REPO)
    assert r.returncode == 0, r.stderr
    assert soa_sha(load_trace(str(out))) == soa_sha(parse_trace(rec["text"]))
