"""Full-trace report digests of the billion-event configs, made by the CPU
oracle (oracle/gwcp_oracle.cpp, itself pinned on the reference's goldens).
Runs on a GPU host -- the traces are made by the device generators (the same
bytes bench.py analyses; tests/test_gpu_parity.py pins the generators against
the host recipes), copied to host memory and fed to the oracle there:

    python tests/golden/make_full_digests.py [c3 c4 c5] [--out PATH]

Writes {config: {n_events, n_reports, n_diags, oracle_digest, oracle_s,
trace_sha}} (default tests/golden/full_digests.json).  The oracle runs of the
configs proceed on concurrent host threads (ctypes releases the GIL).  The
engine's digests are recorded beside them for information only; the check
is tests/test_gpu_fullscale.py and bench.py's digest assert.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c3", "c4", "c5"])
    ap.add_argument("--out", default=os.path.join(HERE, "full_digests.json"))
    args = ap.parse_args()

    import torch

    import bench
    from oracle import oracle as O
    from paper_2111_12478_b200 import _native as N
    from paper_2111_12478_b200.report import result_digest

    dev = torch.device("cuda", 0)
    ctx = N.Context(0)
    out, threads = {}, []
    for name in args.configs:
        cfg, n, n_acc, (kd, td, idd), desc = bench.make_workload(name, 0, dev)
        key = kd.cpu().numpy().view(np.uint64)
        tidop = td.cpu().numpy().view(np.uint32)
        instr = idd.cpu().numpy().view(np.uint32)
        hs = hashlib.sha256()
        for a in (key, tidop, instr):
            hs.update(a.tobytes())
        t0 = time.perf_counter()
        ctx.analyze_device(cfg, n, kd.data_ptr(), td.data_ptr(), idd.data_ptr(), eager=True)
        eng = ctx.fetch()
        t_eng = time.perf_counter() - t0
        del kd, td, idd
        torch.cuda.empty_cache()
        rec = out[name] = {"n_events": n, "n_accesses": n_acc, "trace_sha": hs.hexdigest(),
                           "engine_digest": result_digest(eng), "engine_reports": int(len(eng["kind"])),
                           "engine_s": t_eng}
        print(f"{name}: engine {len(eng['kind'])} reports in {t_eng:.2f}s", file=sys.stderr, flush=True)

        def run_oracle(rec=rec, cfg=cfg, key=key, tidop=tidop, instr=instr, name=name):
            t0 = time.perf_counter()
            want = O.run_soa(cfg, key, tidop, instr)
            rec["oracle_s"] = time.perf_counter() - t0
            rec["oracle_digest"] = result_digest(want)
            rec["n_reports"] = int(len(want["kind"]))
            rec["n_diags"] = int(len(want["diag_event"]))
            print(f"{name}: oracle {rec['n_reports']} reports in {rec['oracle_s']:.1f}s "
                  f"({'match' if rec['oracle_digest'] == rec['engine_digest'] else 'MISMATCH'})",
                  file=sys.stderr, flush=True)

        t = threading.Thread(target=run_oracle)
        t.start()
        threads.append(t)
    for t in threads:
        t.join()
    with open(args.out, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
