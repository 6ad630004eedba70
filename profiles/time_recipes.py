"""Time the engine (eager + graph replay) and the CPU oracle on the C3 (locks)
and C4 (ITS divergence) recipes at moderate geometries; check parity."""

import sys
import time
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2111_12478_b200 import _native as N  # noqa: E402
from paper_2111_12478_b200 import parse_trace  # noqa: E402
from paper_2111_12478_b200 import workloads as WL  # noqa: E402
from paper_2111_12478_b200.report import ndjson_lines  # noqa: E402

cases = [
    ("C3 16x8x32 it48", lambda: WL.c3_text(blocks=16, warps=8, lanes=32, iters=48, locks=256, region=64, private=512)),
    ("C3 64x8x32 it16", lambda: WL.c3_text(blocks=64, warps=8, lanes=32, iters=16, locks=1024, region=64, private=512)),
    ("C4 32x8x32 it64", lambda: WL.c4_text(blocks=32, warps=8, lanes=32, iters=64, words_per_block=16384)),
    ("C4 128x8x32 it32", lambda: WL.c4_text(blocks=128, warps=8, lanes=32, iters=32, words_per_block=16384)),
]
stream = torch.cuda.Stream(device=torch.device("cuda", 0))
ctx = N.Context(0)
for name, fn in cases:
    t0 = time.time()
    tr = parse_trace(fn())
    tg = time.time() - t0
    ctx.analyze_host(tr.cfg_tuple, tr.key, tr.tidop, tr.instr, stream=stream.cuda_stream, eager=True)
    res = ctx.fetch()
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.analyze_host(tr.cfg_tuple, tr.key, tr.tidop, tr.instr, stream=stream.cuda_stream, eager=True)
        res = ctx.fetch()
        best = min(best, time.perf_counter() - t0)
    s = ctx.stats()
    t0 = time.perf_counter()
    want = O.run_trace(tr)
    to = time.perf_counter() - t0
    ok = ndjson_lines(tr, res) == ndjson_lines(tr, want)
    print(f"{name}: N={len(tr)} reports={len(res['kind'])} parity={ok} gpu={best*1e3:.2f} ms "
          f"({len(tr)/best/1e6:.1f} M ev/s; walker {s.ms_walker:.2f} sort {s.ms_sort:.2f} check {s.ms_check:.2f}) "
          f"oracle={to:.2f} s ({len(tr)/to/1e6:.2f} M ev/s) gen {tg:.1f}s", flush=True)
