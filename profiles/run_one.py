"""One eager analysis of a device-generated workload (the command profiled
with ncu for profiles/; no timing is reported from runs under a profiler)."""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2111_12478_b200 import _native as N  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--repeat", type=int, default=2)
ap.add_argument("--graph", action="store_true", help="graph replays (the bench's timed path) instead of eager runs")
args = ap.parse_args()
dev = torch.device("cuda", 0)
cfg, n, n_acc, (k, t, i), desc = bench.make_workload(args.workload, 0, dev)
stream = torch.cuda.Stream(device=dev)
ctx = N.Context(0)
for _ in range(args.repeat):
    ctx.analyze_device(cfg, n, k.data_ptr(), t.data_ptr(), i.data_ptr(), stream=stream.cuda_stream,
                       eager=not args.graph)
    res = ctx.fetch()
s = ctx.stats()
print(f"{desc['workload']}: {n} events, {len(res['kind'])} reports, {ctx.launches()} launches, "
      f"eager {s.ms_total:.3f} ms (prep {s.ms_prep:.3f} walker {s.ms_walker:.3f} sort {s.ms_sort:.3f} "
      f"check {s.ms_check:.3f} final {s.ms_final:.3f})")
