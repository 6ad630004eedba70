"""Determinism check at full scale: eager vs graph-replay analyses of one
device-generated workload must return identical report lists."""
import argparse, os, sys, hashlib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch  # noqa: E402
import bench  # noqa: E402
from paper_2111_12478_b200 import _native as N  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c5")
args = ap.parse_args()
dev = torch.device("cuda", 0)
cfg, n, n_acc, (k, t, i), desc = bench.make_workload(args.workload, 0, dev)
stream = torch.cuda.Stream(device=dev)
ctx = N.Context(0)
def dig(r):
    h = hashlib.sha1()
    for key in ("kind", "prior", "current"):
        h.update(np.ascontiguousarray(r[key]).tobytes())
    return len(r["kind"]), h.hexdigest()[:12]
for mode in ("eager", "eager", "graph", "graph", "graph", "eager"):
    ctx.analyze_device(cfg, n, k.data_ptr(), t.data_ptr(), i.data_ptr(), stream=stream.cuda_stream, eager=(mode == "eager"))
    r = ctx.fetch()
    print(mode, dig(r), flush=True)
