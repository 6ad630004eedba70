"""Per-kernel device times of one warm eager analysis (GW_OPT_PROFILE)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2111_12478_b200 import _native as N  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c5")
args = ap.parse_args()
dev = torch.device("cuda", 0)
cfg, n, n_acc, (k, t, i), desc = bench.make_workload(args.workload, 0, dev)
stream = torch.cuda.Stream(device=dev)
ctx = N.Context(0)
for rep in range(3):
    ctx.analyze_device(cfg, n, k.data_ptr(), t.data_ptr(), i.data_ptr(), stream=stream.cuda_stream, eager=True,
                       profile=(rep == 2))
    ctx.fetch()
kt = ctx.kernel_times()
tot = sum(v[0] for v in kt.values())
for name, (ms, cnt) in sorted(kt.items(), key=lambda kv: -kv[1][0])[:14]:
    print(f"{ms:9.3f} ms {cnt:4d}x  {name}")
print(f"total {tot:.3f} ms")
