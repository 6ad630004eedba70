"""Where the C2 step goes: host-side launch of the graph replay, device time
to completion, and the result fetch (profiling aid; not a bench number)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2111_12478_b200 import _native as N  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "c2"
dev = torch.device("cuda", 0)
cfg, n, n_acc, (k, t, i), desc = bench.make_workload(w, 0, dev)
stream = torch.cuda.Stream(device=dev)
ctx = N.Context(0)
sp = stream.cuda_stream
for _ in range(5):
    ctx.analyze_device(cfg, n, k.data_ptr(), t.data_ptr(), i.data_ptr(), stream=sp)
    ctx.fetch()
L = N.lib()
R = {"launch": [], "dev": [], "fetch": [], "total": []}
for _ in range(30):
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record(stream)
    ctx.analyze_device(cfg, n, k.data_ptr(), t.data_ptr(), i.data_ptr(), stream=sp)
    t1 = time.perf_counter()
    b.record(stream)
    b.synchronize()
    t2 = time.perf_counter()
    ctx.fetch()
    t3 = time.perf_counter()
    R["launch"].append((t1 - t0) * 1e3); R["dev"].append(a.elapsed_time(b)); R["fetch"].append((t3 - t2) * 1e3)
    R["total"].append((t3 - t0) * 1e3)
for kk, v in R.items():
    print(f"{kk:7s} median {np.median(v):.4f} ms  min {np.min(v):.4f}")
print("launches", ctx.launches())
