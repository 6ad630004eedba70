"""Full-trace report digests of the billion-event configs, made by the CPU
oracle (oracle/gwcp_oracle.cpp, itself pinned on the reference's goldens).
Runs on a GPU host -- the traces are made by the device generators (the same
bytes bench.py analyses; tests/test_gpu_parity.py pins the generators against
the host recipes), copied to host memory and fed to the oracle there:

    python tests/golden/make_full_digests.py [c3 c4 c5] [--out PATH]

Writes {config: {n_events, P, n_reports, n_diags, oracle_digest, oracle_s,
trace_sha}} (default tests/golden/full_digests.json).  P = n_events: the
oracle ran the whole trace.  C3 is the exception: the oracle's clocks grow
dense under 4,096 device-scope locks (28 GB after 4 of 168 iterations), so it
runs the first C3_ORACLE_ITERS iterations, and the digest is of the reports
with current.event < P (those are exactly the prefix's).  The oracle runs of the
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
C3_ORACLE_ITERS = 4
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)


def prefix_of(res: dict, P: int) -> dict:
    """The reports with current.event < P and the diagnostics at events < P."""
    keep = res["current"] < P
    dk = res["diag_event"] < P
    return {"kind": res["kind"][keep], "prior": res["prior"][keep], "current": res["current"][keep],
            "diag_event": res["diag_event"][dk], "diag_code": res["diag_code"][dk], "diag_lock": res["diag_lock"][dk]}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c4", "c5", "c3"])
    ap.add_argument("--out", default=os.path.join(HERE, "full_digests.json"))
    args = ap.parse_args()

    import torch

    import bench
    from oracle import oracle as O
    from paper_2111_12478_b200 import _native as N
    from paper_2111_12478_b200.report import result_digest
    from paper_2111_12478_b200 import workloads as WL

    dev = torch.device("cuda", 0)
    out, threads = {}, []
    for name in args.configs:
        cfg, n, n_acc, (kd, td, idd), desc = bench.make_workload(name, 0, dev)
        key = kd.cpu().numpy().view(np.uint64)
        tidop = td.cpu().numpy().view(np.uint32)
        instr = idd.cpu().numpy().view(np.uint32)
        hs = hashlib.sha256()
        for a in (key, tidop, instr):
            hs.update(a.tobytes())
        ctx = N.Context(0)  # one per config: a lock trace's clock arena is sized from the free HBM
        t0 = time.perf_counter()
        ctx.analyze_device(cfg, n, kd.data_ptr(), td.data_ptr(), idd.data_ptr(), eager=True)
        eng = ctx.fetch()
        t_eng = time.perf_counter() - t0
        ctx.close()
        del kd, td, idd
        torch.cuda.empty_cache()
        P = n
        if name == "c3":  # record-aligned: whole iterations of the iteration-major trace
            p = dict(WL.CONFIGS["c3"], iters=C3_ORACLE_ITERS)
            P = WL.config_counts(p)[0]
            key, tidop, instr = key[:P], tidop[:P], instr[:P]
        rec = out[name] = {"n_events": n, "P": P, "n_accesses": n_acc, "trace_sha": hs.hexdigest(),
                           "engine_digest": result_digest(prefix_of(eng, P)),
                           "engine_reports": int((eng["current"] < P).sum()), "engine_s": t_eng}
        print(f"{name}: engine {len(eng['kind'])} reports in {t_eng:.2f}s", file=sys.stderr, flush=True)

        def run_oracle(rec=rec, cfg=cfg, key=key, tidop=tidop, instr=instr, name=name):
            t0 = time.perf_counter()
            want = O.run_soa(cfg, key, tidop, instr)
            upd = {"oracle_s": time.perf_counter() - t0, "n_reports": int(len(want["kind"])),
                   "n_diags": int(len(want["diag_event"])), "oracle_digest": result_digest(want)}
            with _save_lock:
                rec.update(upd)
            save(args.out, out)
            print(f"{name}: oracle {rec['n_reports']} reports in {rec['oracle_s']:.1f}s "
                  f"({'match' if rec['oracle_digest'] == rec['engine_digest'] else 'MISMATCH'})",
                  file=sys.stderr, flush=True)

        if name == "c3":  # its oracle needs the most host memory: alone, after the others
            for t in threads:
                t.join()
            run_oracle()
            save(args.out, out)
        else:
            t = threading.Thread(target=run_oracle)
            t.start()
            threads.append(t)
    for t in threads:
        t.join()
    save(args.out, out)
    print(json.dumps(out, indent=1))


_save_lock = threading.Lock()


def save(path, out):
    with _save_lock:
        done = {k: dict(v) for k, v in list(out.items()) if "oracle_digest" in v}
        with open(path, "w") as fh:
            json.dump(done, fh, indent=1)


if __name__ == "__main__":
    main()
