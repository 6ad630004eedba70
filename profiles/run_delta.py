"""One end-to-end analysis from the delta-varint (default) or bit-packed
(second argument "bp") host form -- the command profiled with ncu for the
decode kernels; no timing is reported from runs under a profiler."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2111_12478_b200 import _native as N  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
form = sys.argv[2] if len(sys.argv) > 2 else "delta"
dev = torch.device("cuda", 0)
cfg, n, n_acc, (k, t, i), desc = bench.make_workload(wl, 0, dev)
encode = N.encode_bp if form == "bp" else N.encode_delta
enc = encode(cfg, k.cpu().numpy().view(np.uint64), t.cpu().numpy().view(np.uint32), i.cpu().numpy().view(np.uint32))
del k, t, i
ctx = N.Context(0)
(ctx.analyze_host_bp if form == "bp" else ctx.analyze_host_delta)(enc, eager=True)
res = ctx.fetch()
print(f"{desc['workload']}: {n} events, {len(res['kind'])} reports, "
      f"{sum(len(b) for b in enc['bytes']) / n:.2f} B/event {form}")
