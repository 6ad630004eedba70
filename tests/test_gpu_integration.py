"""INTEGRATION.md executed: the reference package itself (gpurace, installed
from /root/reference into baseline/_ref, which travels with the repo to the
GPU host) drives the B200 engine through paper_2111_12478_b200.gpurace_backend
-- the ctypes stub a gpurace maintainer would add.  Real gpurace.Trace objects
(gpurace.trace.parse_trace) go in, gpurace's own RaceReport / Diagnostic /
RunResult come out, and `gpurace check` (gpurace.cli.main) prints the
reference goldens' NDJSON with the reference's exit codes."""

import io
import os
import sys
from contextlib import redirect_stderr, redirect_stdout

import pytest

from conftest import REPO, golden_text
from helpers import lines_sha

pytestmark = pytest.mark.gpu

REF = os.path.join(REPO, "baseline", "_ref")


@pytest.fixture(scope="module")
def gpurace():
    if not os.path.isdir(os.path.join(REF, "gpurace")):
        pytest.skip("the reference is not installed in baseline/_ref (pip install --target baseline/_ref)")
    sys.path.insert(0, REF)
    import gpurace as G
    import gpurace.cli  # noqa: F401
    import gpurace.gwcp  # noqa: F401
    import gpurace.hb  # noqa: F401
    import gpurace.trace  # noqa: F401

    return G


def test_backend_on_real_gpurace_traces(gpurace, goldens):
    from paper_2111_12478_b200 import gpurace_backend as B

    n = 0
    for r in goldens:
        if "error" in r or "full" in r["tags"] or not ({"corpus", "random", "nasty", "c1", "c3"} & set(r["tags"])):
            continue
        tr = gpurace.trace.parse_trace(golden_text(r))
        det = gpurace.gwcp.GwcpDetector(tr.config, inactive_opt=r["inactive_opt"])
        res = B.run(tr, det)
        assert type(res).__module__ == "gpurace.engine"  # the reference's own result objects
        lines = [x.to_json() for x in res.reports]
        if "reports" in r:
            assert lines == r["reports"], r["name"]
        else:
            assert lines[:50] == r["reports_head"] and lines_sha(lines) == r["reports_sha"], r["name"]
        assert [str(d) for d in res.diagnostics] == r["diags"], r["name"]
        assert [x.to_json() for x in det.reporter.reports] == [x.to_json() for x in res.reports]
        n += 1
    assert n > 3000


def test_backend_hb_detector(gpurace, goldens_hb):
    from paper_2111_12478_b200 import gpurace_backend as B

    n = 0
    for r, h in goldens_hb:
        if "full" in r["tags"] or "reports" not in h or not ({"corpus", "nasty"} & set(r["tags"])):
            continue
        tr = gpurace.trace.parse_trace(golden_text(r))
        res = B.run(tr, gpurace.hb.HbDetector(tr.config))
        assert [x.to_json() for x in res.reports] == h["reports"], r["name"]
        n += 1
    assert n > 100


def test_gpurace_cli_check_through_the_backend(gpurace, goldens, tmp_path):
    """`gpurace check T --detector gwcp` with gpurace.engine.run routed to the
    B200 engine: the reference CLI's stdout and exit code, byte for byte."""
    from paper_2111_12478_b200 import gpurace_backend as B

    B.install()
    n = 0
    for r in goldens:
        if not r["name"].startswith("corpus/") or r["name"].endswith("/noio"):
            continue
        p = tmp_path / "t.trace"
        p.write_text(r["text"])
        out, err = io.StringIO(), io.StringIO()
        with redirect_stdout(out), redirect_stderr(err):
            try:
                rc = gpurace.cli.main(["check", str(p)])
            except SystemExit as e:
                rc = e.code
        assert out.getvalue().splitlines() == r["reports"], r["name"]
        assert rc == (1 if r["reports"] else 0)
        n += 1
    assert n == 17
