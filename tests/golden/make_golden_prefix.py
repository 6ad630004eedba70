"""Prefix goldens for the full-size configs C3/C4/C5, made by the REFERENCE
(run here, where /root/reference exists; the fixture travels, the reference
does not).

    python tests/golden/make_golden_prefix.py [P]

SURVEY §8(c) item 1 / App. B O2: the reports of trace[:P] (P cut at a record
boundary) are exactly the full trace's reports with current.event < P,
"first" flag included.  The Python reference cannot run the 10^8-10^9-event
traces, so it runs `engine.run(trace[:P], GwcpDetector(cfg))` with the
`check` defaults (cli.py:51-57) on the record-aligned prefix of the
full-geometry trace (workloads.config_prefix == the device generators'
output, tests/test_gpu_parity.py pins that), and the GPU test
(tests/test_gpu_fullscale.py) runs the FULL trace and compares its reports
with current.event < P against this fixture.

Also records the reference's own speed on that prefix (perf_counter around
engine.run only, parse timed separately; SURVEY §8(d) "CPU timing"), pinned
to one core when taskset is available.

Writes tests/golden/golden_prefix.json.
"""

from __future__ import annotations

import hashlib
import json
import os
import platform
import sys
import time
from concurrent.futures import ProcessPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

FULL_LINES_MAX = 400


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def one(job):
    name, P, core = job
    if core is not None and hasattr(os, "sched_setaffinity"):
        os.sched_setaffinity(0, {core})
    from gpurace.engine import run as ref_run
    from gpurace.gwcp import GwcpDetector
    from gpurace.trace import parse_trace as ref_parse

    from paper_2111_12478_b200 import workloads as WL

    p = WL.CONFIGS[name]
    tr = WL.config_prefix(p, P)
    text = WL.soa_to_text(tr)
    t0 = time.perf_counter()
    rt = ref_parse(text)
    t1 = time.perf_counter()
    res = ref_run(rt, GwcpDetector(rt.config))
    t2 = time.perf_counter()
    lines = [r.to_json() for r in res.reports]
    n_full, _ = WL.config_counts(p)
    rec = {
        "name": f"{name}/prefix",
        "config": name,
        "params": {k: v for k, v in p.items()},
        "P": len(tr),
        "n_events_full": n_full,
        "n_reports": len(lines),
        "reports_sha": hashlib.sha256(("\n".join(lines) + "\n").encode()).hexdigest() if lines else "",
        "diags": [str(d) for d in res.diagnostics],
        "reference_timing": {
            "run_s": t2 - t1,
            "parse_s": t1 - t0,
            "events_per_s": len(tr) / (t2 - t1),
            "cores": 1,
            "pinned_core": core,
            "host_cpus": os.cpu_count(),
            "cpu_model": cpu_model(),
            "python": platform.python_version(),
        },
    }
    if len(lines) <= FULL_LINES_MAX:
        rec["reports"] = lines
    else:
        rec["reports_head"] = lines[:50]
    return rec


def main() -> None:
    P = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    jobs = [("c3", P, 1), ("c4", P, 2), ("c5", P, 3)]
    t0 = time.time()
    with ProcessPoolExecutor(len(jobs)) as ex:
        recs = list(ex.map(one, jobs))
    out = os.path.join(HERE, "golden_prefix.json")
    with open(out, "w") as fh:
        json.dump(recs, fh, indent=1)
    for r in recs:
        t = r["reference_timing"]
        print(f"{r['name']}: P={r['P']} reports={r['n_reports']} run {t['run_s']:.1f}s "
              f"({t['events_per_s']:.0f} ev/s)", file=sys.stderr)
    print(f"wrote {out} in {time.time() - t0:.1f}s", file=sys.stderr)


if __name__ == "__main__":
    main()
