"""Times the Python reference (gpurace, /root/reference/pkg/src) on the CPU,
single-threaded and pinned to one core (SURVEY §8(d) "CPU timing"):
perf_counter around engine.run(trace, GwcpDetector(cfg)) with the `check`
defaults, parse timed separately.  C1: the litmus corpus; C2: the full
1,049,088-event trace, median of 3.  (C3-C5: the 10^6-event prefixes are
timed by tests/golden/make_golden_prefix.py, which also pins them.)

    taskset -c 0 python profiles/time_python_reference.py > profiles/r2_python_reference.json
"""

import json
import os
import platform
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, "/root/reference/pkg/src")

from gpurace.engine import run  # noqa: E402
from gpurace.gwcp import GwcpDetector  # noqa: E402
from gpurace.litmus import corpus_entry, corpus_names  # noqa: E402
from gpurace.trace import parse_trace  # noqa: E402

from paper_2111_12478_b200 import workloads as WL  # noqa: E402


def cpu_model():
    with open("/proc/cpuinfo") as fh:
        for line in fh:
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    return platform.processor()


def timed(text, reps):
    t0 = time.perf_counter()
    tr = parse_trace(text)
    parse_s = time.perf_counter() - t0
    runs = []
    for _ in range(reps):
        t0 = time.perf_counter()
        res = run(tr, GwcpDetector(tr.config))
        runs.append(time.perf_counter() - t0)
    return len(tr.events), parse_s, runs, len(res.reports)


out = {"host_cpus": os.cpu_count(), "affinity": sorted(os.sched_getaffinity(0)), "cpu_model": cpu_model(),
       "python": platform.python_version()}
n = 0
tot = 0.0
for name in corpus_names():
    ne, _, runs, _ = timed(corpus_entry(name).text, 3)
    n += ne
    tot += statistics.median(runs)
out["c1_corpus"] = {"events": n, "run_s": tot, "events_per_s": n / tot, "traces": len(corpus_names())}
ne, ps, runs, nr = timed(WL.soa_to_text(WL.c2_soa()), 3)
out["c2_full"] = {"events": ne, "parse_s": ps, "run_s_runs": runs, "run_s_median": statistics.median(runs),
                  "events_per_s": ne / statistics.median(runs), "reports": nr}
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", "golden_prefix.json")) as fh:
    for r in json.load(fh):
        out[f"{r['config']}_prefix"] = dict(r["reference_timing"], events=r["P"], reports=r["n_reports"])
print(json.dumps(out, indent=1))
