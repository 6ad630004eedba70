"""Benchmark: trace events/s of G-WCP race analysis (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--workload c2|c5]

One step = one complete analysis of one synthetic trace (the workload) with
the final report list on the host.  ``value`` is device-resident throughput
(SoA already in HBM); ``e2e`` is the same metric through the public C-ABI
call with HOST buffers (pinned H2D of the SoA and D2H of the reports inside
the timed region).  L2 is flushed (256 MiB write) before every timed step;
each step is timed with CUDA events on the launching stream and the K step
times are summed.  For N > 1 (torchrun, one rank per GPU) every rank analyses
its own trace (independent objects: weak scaling, no data-path collective),
except the C5 scaling sweep (``--workload c5``): one trace in the exchange
mode of shard.analyze_exchange -- every rank holds one record-aligned 1/N
slice, access records travel to their location-hash shard by NCCL
all-to-all, rank 0 merges the candidates (strong scaling; ``--mode sharded``:
the replicated address-range mode instead).  The time is the max over ranks.

``--impl reference`` times the CPU restatement of the reference (oracle/,
single-threaded like the reference) on this host: rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "trace events/sec analysed (1/2/4/8 B200) vs CPU ref; race-pair set bit-exact"
UNIT = "events/s"


def load_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def workloads():
    from paper_2111_12478_b200 import workloads as WL

    return WL.CONFIGS


# Algorithmic bytes per launch of the pipeline's kernels:
# n = positions the access pass sorts (all events, or a shard's accesses),
# N = events.  The dominant kernel's roofline uses these.
def kernel_alg_bytes(name: str, N: int, n: int) -> int | None:
    table = [
        ("k_rs_down", 16 * n),      # keys + values read once, written once
        ("k_rs_down_tma", 16 * n),
        ("k_rs_onesweep", 16 * n),
        ("k_rs_up", 4 * n),         # keys read
        ("k_access", 12 * n),       # key 4 + event 4 + the event's tidop 4 per sorted position (stamps: lazy, L2)
        ("k_acc_keys", 20 * N),     # key 8 + tidop 4 read; key 4 + event 4 written
        ("k_ingest", 20 * N),       # same bytes: k_prep + k_acc_keys + first digit counts in one read (graph replays)
        ("k_acc_aux", 20 * N),      # (GW_ACC_LAZY=0 only) tidop 4 read, aux 16 written
        ("k_acc_tilemax", 8 * n),
        ("k_prep", 12 * N),
        ("k_same_instr", 16 * N),
        ("k_walker", 16 * N),       # the trace, read once
        ("k_hard_append", 4 * N),
        # the bucketed access pass (csrc/bucket.cuh), n = accesses: per launch of
        # the scatter: pass A reads the trace (key 8 + tidop 4 per event) and
        # writes a 12-B record per access, pass B reads and writes 12 B per
        # record -> (12 N + 12 n + 24 n) / 2 per launch; the up-sweeps read the
        # trace (12 N) / the record hashes (4 n); the check reads each record once
        ("k_bk_down_tma", (12 * N + 36 * n) // 2),
        ("k_bk_down", (12 * N + 36 * n) // 2),
        ("k_bk_up", (12 * N + 4 * n) // 2),
        ("k_bk_check", 12 * n),
        ("k_bk_bounds", 4 * n),
    ]
    base = kernel_base(name)
    tag = kernel_tag(name)
    if tag not in (None, "acc"):
        return None  # kernels of the small auxiliary sorts: no per-unit figure
    for key, b in table:
        if base == key:
            return b
    return None


def kernel_base(name: str) -> str:
    """'(k_rs_down<K, RB>)@acc' -> 'k_rs_down' (launch expressions as the engine records them)."""
    return name.split("@")[0].strip().strip("()").split("<")[0].strip()


def kernel_tag(name: str) -> str | None:
    return name.split("@", 1)[1] if "@" in name else None


def load_full_digest(workload: str):
    """The CPU oracle's report digest of the full workload trace (committed
    fixture made on a GPU host by profiles/make_full_digests.py), or None."""
    try:
        with open(os.path.join(REPO, "tests", "golden", "full_digests.json")) as fh:
            d = json.load(fh)
    except Exception:
        return None
    r = d.get(workload)
    if not r or "oracle_digest" not in r:
        return None
    whole = r.get("P", r["n_events"]) >= r["n_events"]
    return {"digest": r["oracle_digest"], "P": r.get("P", r["n_events"]),
            "source": f"tests/golden/full_digests.json[{workload}] (oracle port, {r.get('n_reports')} reports"
                      + ("" if whole else f" with current.event < {r.get('P')}: the oracle's prefix") + ")"}


def digest_for(res, fx, n):
    """The digest to compare with a full_digests.json entry: of the whole
    result, or of the reports / diagnostics before the entry's prefix P."""
    from paper_2111_12478_b200.report import result_digest

    if fx is None or fx["P"] >= n:
        return result_digest(res)
    P = fx["P"]
    keep, dk = res["current"] < P, res["diag_event"] < P
    return result_digest({"kind": res["kind"][keep], "prior": res["prior"][keep], "current": res["current"][keep],
                          "diag_event": res["diag_event"][dk], "diag_code": res["diag_code"][dk],
                          "diag_lock": res["diag_lock"][dk]})


def load_ncu_traffic():
    try:
        with open(os.path.join(REPO, "profiles", "ncu_traffic.json")) as fh:
            return json.load(fh)
    except Exception:
        return {}


def workload_events(p):
    from paper_2111_12478_b200 import workloads as WL

    return WL.config_counts(p)


def workload_desc(name, p, n, n_acc):
    d = {"workload": name.upper(), "threads": f"{p['blocks']}x{p['warps']}x{p['lanes']}",
         "addresses": p["blocks"] * p.get("words_per_block", 0), "events": n, "accesses": n_acc}
    if p["gen"] == "c4":
        d.update(iterations=p["iters"], sync="warp barriers (random masks) / 4 it, block barriers / 64 it",
                 divergence="ITS: ~half the lanes issue single-lane accesses in random order")
    elif p["gen"] == "c3":
        d.update(addresses=p["blocks"] * p["warps"] * p["private"] + p["locks"] * (p["region"] + 1) + 1,
                 iterations=p["iters"], locks=p["locks"],
                 sync="device-scope spin locks (lane 0, 1-4 protected accesses), failed-CAS polling, device fences, "
                      "warp barriers, block barriers / 16 it",
                 injected="1% atomic counter writes (10% block scope), 0.1% unprotected lock-region writes")
    else:
        d.update(phases=p["phases"], records_per_warp_phase=p["records"], sync="__syncthreads only",
                 injected_random_words="1%")
    return d


def make_workload(name: str, rank: int, dev, sharded: bool = False):
    """Generate the workload trace directly in HBM (device generators; identical
    to paper_2111_12478_b200.workloads.c2_soa / c4_text for the same parameters)."""
    import torch
    from paper_2111_12478_b200 import _native as N

    p = dict(workloads()[name])
    if not sharded:  # replicas: every rank analyses its own trace; sharded: one trace, split by address
        p["seed"] += rank
    n, n_acc = workload_events(p)
    key_d = torch.empty(n, dtype=torch.int64, device=dev)
    to_d = torch.empty(n, dtype=torch.int32, device=dev)
    in_d = torch.empty(n, dtype=torch.int32, device=dev)
    gp = {k: v for k, v in p.items() if k != "gen"}
    if p["gen"] == "c4":
        del gp["lanes"]
        N.gen_c4_device(key_d.data_ptr(), to_d.data_ptr(), in_d.data_ptr(), **gp)
    elif p["gen"] == "c3":
        from paper_2111_12478_b200 import workloads as WL

        off = torch.from_numpy(WL.c3_group_offsets(**gp)[:-1].view(np.int64)).to(dev)
        N.gen_c3_device(key_d.data_ptr(), to_d.data_ptr(), in_d.data_ptr(), off.data_ptr(), **gp)
        torch.cuda.synchronize(dev)
        del off
    else:
        N.gen_c2_device(key_d.data_ptr(), to_d.data_ptr(), in_d.data_ptr(), **gp)
    torch.cuda.synchronize(dev)
    cfg = (p["blocks"], p["warps"], p["lanes"])
    return cfg, n, n_acc, (key_d, to_d, in_d), workload_desc(name, p, n, n_acc)


def host_workload_prefix(p, P):
    """Record-aligned host prefix of >= min(P, N) events (numpy / text recipe)."""
    from paper_2111_12478_b200 import workloads as WL

    return WL.config_prefix(p, P)


def host_prefix(cfg, dev_bufs, P):
    """Record-aligned host copy of the first ~P events (for the CPU oracle)."""
    from paper_2111_12478_b200 import _native as N
    from paper_2111_12478_b200.trace import Trace, TraceConfig

    key_d, to_d, in_d = dev_bufs
    n = key_d.numel()
    P = min(P, n)
    to = to_d[: min(n, P + 64)].cpu().numpy().view(np.uint32)
    while P < len(to) and to[P] & N.F_CONT:
        P += 1
    return Trace(TraceConfig(*cfg), key_d[:P].cpu().numpy().view(np.uint64), to[:P].copy(),
                 in_d[:P].cpu().numpy().view(np.uint32))


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    def __init__(self, device: int):
        self.samples: list[int] = []
        self.reasons: set[str] = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        nv = self._nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            self._stop.wait(0.02)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def summary(self):
        return {
            "sm_mhz": int(statistics.median(self.samples)) if self.samples else None,
            "sm_max_mhz": self.max_mhz,
            "reasons": sorted(self.reasons),
            "samples": len(self.samples),
        }


def cpu_time(get_prefix, n, budget_s):
    """Time the oracle port (one core) on a bounded sample of the workload:
    the largest record-aligned prefix whose single run fits the budget, run
    repeatedly until the budget is spent.  Returns (events/s, description)."""
    from oracle import oracle as O

    P = min(n, 1 << 20)
    tr = get_prefix(P)
    while True:
        t0 = time.perf_counter()
        O.run_trace(tr)
        dt = time.perf_counter() - t0
        if dt > budget_s and len(tr) > 10000:
            tr = get_prefix(int(len(tr) * budget_s / dt * 0.7))
        elif dt < budget_s / 8 and len(tr) < n:
            tr = get_prefix(min(n, int(len(tr) * budget_s / max(dt, 1e-3) * 0.25)))
        else:
            break
    runs, tot = 1, dt
    while tot < budget_s:
        t0 = time.perf_counter()
        O.run_trace(tr)
        tot += time.perf_counter() - t0
        runs += 1
    what = "the full trace" if len(tr) >= n else f"the first {len(tr)} of {n} events (record-aligned prefix)"
    return len(tr) * runs / tot, f"{what}, {runs} run(s), oracle/gwcp_oracle.cpp on 1 host core"


def python_reference_time(get_prefix, workload):
    """The Python reference itself (gpurace, installed into baseline/_ref from
    /root/reference) on this host: engine.run(trace[:P], GwcpDetector(cfg))
    with the `check` defaults on one core, parse excluded (SURVEY §8(d) "CPU
    timing"); P bounded to a few seconds of its ~10^3-10^5 events/s."""
    ref = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "gpurace")):
        return None
    sys.path.insert(0, ref)
    try:
        from gpurace.engine import run as ref_run
        from gpurace.gwcp import GwcpDetector as RefDetector
        from gpurace.trace import parse_trace as ref_parse

        from paper_2111_12478_b200 import workloads as WL

        P = {"c2": 200_000, "c3": 8_000, "c4": 40_000, "c5": 200_000}.get(workload, 100_000)
        tr = ref_parse(WL.soa_to_text(get_prefix(P)))
        t0 = time.perf_counter()
        ref_run(tr, RefDetector(tr.config))
        dt = time.perf_counter() - t0
        return {"value": len(tr.events) / dt, "unit": UNIT, "cores": 1, "kind": "reference (Python, gpurace 0.1.0)",
                "sample": f"the first {len(tr.events)} events (record-aligned prefix), 1 run, parse excluded",
                "host_cpus": os.cpu_count()}
    except Exception as e:  # pragma: no cover - informational only
        return {"unavailable": f"{type(e).__name__}: {e}"}
    finally:
        sys.path.remove(ref)


def run_reference(args):
    """The reference arm: the CPU restatement of the reference (oracle/) on
    this host's cores, on the same workload recipe (host numpy generator, so
    nothing of the B200 engine runs on this path)."""
    from oracle import oracle as O
    from paper_2111_12478_b200 import workloads as WL

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    p = workloads()[args.workload]
    n, n_acc = workload_events(p)
    desc = workload_desc(args.workload, p, n, n_acc)
    cache = {}

    def get_prefix(P):
        if P not in cache:
            cache.clear()
            cache[P] = host_workload_prefix(p, P)
        return cache[P]

    for _ in range(args.warmup):
        cpu_time(get_prefix, n, args.ref_seconds / 4)
    vals = [cpu_time(get_prefix, n, args.ref_seconds) for _ in range(args.steps)]
    evs = len(vals) / sum(1.0 / v for v, _ in vals)
    sample = vals[-1][1]
    ms_step = 1000.0 * args.ref_seconds
    cores = 1
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": evs,
        "unit": UNIT,
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u32",
        "data": "synthetic",
        "config": desc,  # identical to the b200 arm's config
        "run": {"parallelism": "single host core"},
        "cpu_baseline": {
            "value": evs,
            "unit": UNIT,
            "cores": cores,
            "kind": "port",
            "sample": sample + " (per step)",
        },
        "e2e": {"value": evs, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def run_b200(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    # GW_BENCH_SAME_GPU=1 (test only): every rank on cuda:0 with gloo, to exercise N>1 on a 1-GPU box
    same_gpu = os.environ.get("GW_BENCH_SAME_GPU") == "1"
    if same_gpu:
        local = 0
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("gloo" if same_gpu else "nccl")
    else:
        torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    coll_dev = None if same_gpu else dev

    from paper_2111_12478_b200 import _native as N
    from paper_2111_12478_b200.shard import gather_reports

    mode = args.mode or "replicas"
    sharded = mode == "sharded" and world > 1
    shard = (rank, world) if sharded else (0, 1)
    cfg, n, n_acc, (key_d, to_d, in_d), desc = make_workload(args.workload, rank, dev, sharded=sharded)
    # pinned host copy of the same trace for the end-to-end leg
    key_h = torch.empty(n, dtype=torch.int64, pin_memory=True)
    to_h = torch.empty(n, dtype=torch.int32, pin_memory=True)
    in_h = torch.empty(n, dtype=torch.int32, pin_memory=True)
    key_h.copy_(key_d)
    to_h.copy_(to_d)
    in_h.copy_(in_d)
    # the packed (narrow-column) form of the same trace: the layout of a GWSOA v2
    # file (cli convert --packed), made once like a trace file on disk
    kb = 4
    for c0 in range(0, n, 1 << 27):  # barrier keys are implied by the tidop (gw_trace_packed)
        kc = key_d[c0:c0 + (1 << 27)]
        nonbar = ((to_d[c0:c0 + (1 << 27)] >> N.OP_SHIFT) & 7) != N.K_BARRIER
        kc = torch.where(nonbar, kc, torch.zeros_like(kc))
        if int(kc.max().item()) >= (1 << 32) or int(kc.min().item()) < 0:
            kb = 8
        del kc, nonbar
    ib = 2 if int(in_d.max().item()) < (1 << 16) and int(in_d.min().item()) >= 0 else 4
    keyp_h = torch.empty(n, dtype=torch.int32 if kb == 4 else torch.int64, pin_memory=True)
    inp_h = torch.empty(n, dtype=torch.int16 if ib == 2 else torch.int32, pin_memory=True)
    keyp_h.copy_(key_d.to(keyp_h.dtype))
    inp_h.copy_(in_d.to(inp_h.dtype))
    keyp_np = keyp_h.numpy().view(np.uint32 if kb == 4 else np.uint64)
    inp_np = inp_h.numpy().view(np.uint16 if ib == 2 else np.uint32)
    # the delta-varint form (GWSOA v3, gw_encode_delta): ~3.3 B/event on C2 / C5,
    # encoded once on the host like a trace file written by the recorder; the
    # byte streams in pinned memory
    enc = N.encode_delta(cfg, key_h.numpy().view(np.uint64), to_h.numpy().view(np.uint32),
                         in_h.numpy().view(np.uint32))
    enc_pinned = []
    for c in range(3):
        t = torch.empty(max(len(enc["bytes"][c]), 1), dtype=torch.uint8, pin_memory=True)
        t[: len(enc["bytes"][c])].copy_(torch.from_numpy(enc["bytes"][c]))
        enc_pinned.append(t)
        enc["bytes"][c] = t.numpy()[: len(enc["bytes"][c])]
    # the bit-packed form (GWSOA v4, gw_encode_bp): ~0.26 B/event on C5, the headline e2e input
    encb = N.encode_bp(cfg, key_h.numpy().view(np.uint64), to_h.numpy().view(np.uint32),
                       in_h.numpy().view(np.uint32))
    bp_pinned = []
    for c in range(3):
        t = torch.empty(max(len(encb["bytes"][c]), 1), dtype=torch.uint8, pin_memory=True)
        t[: len(encb["bytes"][c])].copy_(torch.from_numpy(encb["bytes"][c]))
        bp_pinned.append(t)
        encb["bytes"][c] = t.numpy()[: len(encb["bytes"][c])]
    bp_bytes = sum(len(b) for b in encb["bytes"]) + sum(8 * (len(o) + len(b_) + len(d_)) for o, b_, d_ in
                                                         zip(encb["offs"], encb["base"], encb["dbase"]))
    delta_bytes = sum(len(b) for b in enc["bytes"]) + sum(8 * (len(o) + len(b_)) for o, b_ in
                                                            zip(enc["offs"], enc["base"]))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    # a dedicated stream: repeated analyses of one trace shape replay a captured CUDA graph
    stream = torch.cuda.Stream(device=dev)
    sptr = stream.cuda_stream
    ctx = N.Context(local)

    def finish():
        res = ctx.fetch()
        if not sharded:
            return res
        merged = gather_reports(res, device=coll_dev)  # NCCL: every shard's reports to rank 0, merged by order key
        return merged if merged is not None else res

    def step_device(eager=False):
        ctx.analyze_device(cfg, n, key_d.data_ptr(), to_d.data_ptr(), in_d.data_ptr(), stream=sptr, eager=eager,
                           shard=shard)
        return finish()

    def step_host():
        ctx.analyze_host(cfg, key_h.numpy().view(np.uint64), to_h.numpy().view(np.uint32),
                         in_h.numpy().view(np.uint32), stream=sptr, shard=shard)
        return finish()

    def step_host_packed():
        ctx.analyze_host_packed(cfg, keyp_np, to_h.numpy().view(np.uint32), inp_np, stream=sptr, shard=shard)
        return finish()

    def step_host_bp():
        if sharded:  # (the sharded mode takes the 16-B host form)
            return step_host()
        ctx.analyze_host_bp(encb, stream=sptr)
        return finish()

    def step_host_delta():
        if sharded:  # (the sharded mode takes the 16-B host form)
            return step_host()
        ctx.analyze_host_delta(enc, stream=sptr)
        return finish()

    def timed(fn, steps):
        tot = 0.0
        res = None
        for _ in range(steps):
            flush.fill_(1)
            torch.cuda.synchronize(dev)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            res = fn()
            b.record(stream)
            b.synchronize()
            tot += a.elapsed_time(b)
        return tot, res

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=coll_dev or "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # per-phase breakdown from one warm eager (non-graph) analysis, outside the timed region
    step_device(eager=True)
    step_device(eager=True)
    s = ctx.stats()
    phase = {k: round(getattr(s, "ms_" + k), 4) for k in ("prep", "walker", "sort", "check", "final")}
    phase["eager_total"] = round(s.ms_total, 4)
    # per-kernel device times (CUDA events around every launch, on the launching stream) of one
    # warm eager analysis: the dominant kernel's roofline
    ctx.analyze_device(cfg, n, key_d.data_ptr(), to_d.data_ptr(), in_d.data_ptr(), stream=sptr, eager=True,
                       shard=shard, profile=True)
    finish()
    ktimes = ctx.kernel_times()
    n_sorted = int(ctx.stats().n_sorted)
    for _ in range(args.warmup):
        step_device()
    launches = ctx.launches()
    with ClockSampler(local) as clk:
        barrier()
        ms_dev, res = timed(step_device, args.steps)
        barrier()
        ms_dev = max_over_ranks(ms_dev)
        for _ in range(args.warmup):
            step_host_bp()
        barrier()
        ms_e2e, res_e2e = timed(step_host_bp, args.steps)
        barrier()
        ms_e2e = max_over_ranks(ms_e2e)
        for _ in range(args.warmup):
            step_host_delta()
        barrier()
        ms_e2ed, res_e2ed = timed(step_host_delta, args.steps)
        barrier()
        ms_e2ed = max_over_ranks(ms_e2ed)
        for _ in range(args.warmup):
            step_host_packed()
        barrier()
        ms_e2ep, res_e2ep = timed(step_host_packed, args.steps)
        barrier()
        ms_e2ep = max_over_ranks(ms_e2ep)
        for _ in range(args.warmup):
            step_host()
        barrier()
        ms_e2e16, res_e2e16 = timed(step_host, args.steps)
        barrier()
        ms_e2e16 = max_over_ranks(ms_e2e16)
    n_rep = len(res["kind"])
    stats = ctx.stats()
    # parity of the timed path itself (graph replay on the bench stream, and the
    # host-buffer leg): both digests must equal the committed full-trace digest
    # of the CPU oracle (tests/golden/full_digests.json) when one exists
    digest, want_digest, digest_src = None, None, None
    if rank == 0:
        from paper_2111_12478_b200.report import result_digest

        fx = load_full_digest(args.workload)
        digest = digest_for(res, fx, n)
        for what, r in (("bit-packed host-buffer", res_e2e), ("delta host-buffer", res_e2ed),
                        ("packed host-buffer", res_e2ep),
                        ("16-B host-buffer", res_e2e16)):
            d_e2e = digest_for(r, fx, n)
            if d_e2e != digest:
                raise SystemExit(f"bench: {what} run's reports differ from the device-resident run's "
                                 f"({d_e2e} vs {digest})")
        if fx is not None and args.steps > 0:
            want_digest, digest_src = fx["digest"], fx["source"]
            if digest != want_digest:
                raise SystemExit(f"bench: timed run's report digest {digest} != {want_digest} ({digest_src})")

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    total_events = n * (1 if sharded else world) * args.steps
    value = total_events / (ms_dev / 1000.0)
    e2e = total_events / (ms_e2e / 1000.0)
    e2e16 = total_events / (ms_e2e16 / 1000.0)
    e2ed = total_events / (ms_e2ed / 1000.0)
    e2ep = total_events / (ms_e2ep / 1000.0)
    peak, peak_kind = load_peaks()
    alg_bytes = 16 * n + 36 * n_acc  # 16 B per event + 36 B per access
    step_s = ms_dev / args.steps / 1000.0
    achieved = alg_bytes / step_s / 1e9
    # dominant kernel (largest device time in the profiled analysis; sort kernels per sort)
    dom = max(ktimes.items(), key=lambda kv: kv[1][0]) if ktimes else None
    dom_line = None
    if dom is not None:
        name, (kms, kl) = dom
        b = kernel_alg_bytes(name, n, n_sorted)
        per_launch_s = kms / max(kl, 1) / 1000.0
        traffic = load_ncu_traffic().get(args.workload, {}).get(kernel_base(name))
        dom_line = {
            "bound": "hbm",
            "achieved": (b / per_launch_s / 1e9) if b is not None else None,
            "peak": peak,
            "unit": "GB/s",
            "frac": (b / per_launch_s / 1e9 / peak) if b is not None else None,
            "traffic": traffic,
            "kernel": kernel_base(name),
            "launches_per_analysis": kl,
            "ms_per_launch": kms / max(kl, 1),
            "alg_bytes_per_launch": b,
            "share_of_analysis": kms / sum(v[0] for v in ktimes.values()),
            "peak_source": peak_kind,
            "timing": "CUDA events around each launch of one warm eager analysis (bench.py, live)",
            "traffic_source": "profiles/ncu_traffic.json (ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum "
                              "per launch)" if traffic is not None else None,
        }
    top = sorted(ktimes.items(), key=lambda kv: -kv[1][0])[:10]
    kernel_ms = {(kernel_base(k) + ("@" + kernel_tag(k) if kernel_tag(k) else "")): round(v[0], 4) for k, v in top}
    phases_ms = phase
    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_dev / args.steps,
        "higher_is_better": True,
        "scaling": "strong" if sharded else "weak",
        "vs_baseline": None,
        "dtype": "u32",
        "data": "synthetic",
        "config": desc,  # identical to the reference arm's config
        "run": {
            "reports": n_rep,
            "parallelism": (f"address-sharded x{world} (location-key ranges; replicated sync pass; "
                            f"NCCL gather + order-key merge of the reports)") if sharded else f"replicas x{world}",
            "l2": "flushed before every timed step (256 MiB write)",
            "report_digest": digest,
            "report_digest_expected": want_digest,
            "report_digest_source": digest_src,
        },
        "e2e": {
            "value": e2e,
            "unit": UNIT,
            "h2d_bytes_per_step": (16 * n) if sharded else bp_bytes,
            "d2h_bytes_per_step": 9 * n_rep + 64,
            "ms_per_step": ms_e2e / args.steps,
            "input": ("16-B/event host SoA" if sharded else
                      f"bit-packed host trace ({bp_bytes / max(n, 1):.2f} B/event: per 32-event block, residuals "
                      "of the columns' first differences against the previous / one-record-back / two-records-"
                      "back difference, packed at the block's width with exceptions, 4,096-event chunks, pinned; "
                      "GWSOA v4, gw_encode_bp), gw_ctx_analyze_host_bp: sliced H2D on a copy stream overlapped "
                      "with on-device decoding (one warp per chunk and column)"),
            "delta": {"value": e2ed, "unit": UNIT, "h2d_bytes_per_step": delta_bytes,
                      "ms_per_step": ms_e2ed / args.steps,
                      "input": f"delta-varint host trace ({delta_bytes / max(n, 1):.2f} B/event, GWSOA v3), "
                               "gw_ctx_analyze_host_delta"},
            "packed": {"value": e2ep, "unit": UNIT, "h2d_bytes_per_step": (kb + 4 + ib) * n,
                       "ms_per_step": ms_e2ep / args.steps,
                       "input": f"packed host SoA (key {kb} B + tidop 4 B + instr {ib} B per event, pinned), "
                                "gw_ctx_analyze_host_packed"},
            "soa16": {"value": e2e16, "unit": UNIT, "h2d_bytes_per_step": 16 * n, "ms_per_step": ms_e2e16 / args.steps,
                      "input": "16-B/event host SoA, gw_ctx_analyze_host"},
        },
        "roofline": dom_line,
        "roofline_whole_analysis": {
            "bound": "hbm",
            "achieved": achieved,
            "peak": peak,
            "unit": "GB/s",
            "frac": achieved / peak,
            "kernel": "whole analysis (all kernels of one step); algorithmic bytes B = 16N + 36A (SURVEY 8d)",
            "peak_source": peak_kind,
        },
        "kernel_ms_eager": kernel_ms,
        "phases_ms_eager": phases_ms,
        "gpu_launches": launches * args.steps,
        "walker_ctas": stats.walker_ctas,
        "sort_bits": stats.sort_bits,
    }
    line["clocks"] = clk.summary()
    if not args.no_cpu_baseline:
        v, what = cpu_time(lambda P: host_prefix(cfg, (key_d, to_d, in_d), P), n, args.ref_seconds)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": 1, "kind": "port", "sample": what}
        pyref = python_reference_time(lambda P: host_prefix(cfg, (key_d, to_d, in_d), P), args.workload)
        if pyref is not None:
            line["python_reference"] = pyref
    print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


def run_b200_exchange(args):
    """N > 1, one trace (the C5 scaling sweep): the exchange mode of
    shard.analyze_exchange -- every rank holds ONE record-aligned slice (1/N
    of the SoA, 1/N of the upload), access records go to their location-hash
    shard by NCCL all-to-all, rank 0 merges the candidates.  Strong scaling:
    value = the trace's events / max-over-ranks step time."""
    import torch
    import torch.distributed as dist

    from paper_2111_12478_b200 import _native as N
    from paper_2111_12478_b200.report import ndjson_lines, result_digest
    from paper_2111_12478_b200.shard import analyze_exchange

    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    same_gpu = os.environ.get("GW_BENCH_SAME_GPU") == "1"
    if same_gpu:
        local = 0
    torch.cuda.set_device(local)
    dist.init_process_group("gloo" if same_gpu else "nccl")
    dev = torch.device("cuda", local)
    coll_dev = None if same_gpu else dev
    cfg, n, n_acc, (key_d, to_d, in_d), desc = make_workload(args.workload, rank, dev, sharded=True)

    def cut(k):  # start of slice k, moved forward to a record boundary
        p = n * k // world
        if p <= 0 or p >= n:
            return min(max(p, 0), n)
        w = to_d[p:p + 64].cpu().numpy().view(np.uint32)
        j = 0
        while j < len(w) and w[j] & N.F_CONT:
            j += 1
        return p + j

    lo, hi = cut(rank), cut(rank + 1)
    sl = [key_d[lo:hi].clone(), to_d[lo:hi].clone(), in_d[lo:hi].clone()]
    del key_d, to_d, in_d
    torch.cuda.empty_cache()
    host = [torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for x in sl]
    for h, x in zip(host, sl):
        h.copy_(x)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.Stream(device=dev)
    ctx = N.Context(local)

    def step_device():
        with torch.cuda.stream(stream):
            return analyze_exchange(ctx, cfg, n, sl, lo, collective_device=coll_dev, stream=stream.cuda_stream)

    def step_host():  # the slice's upload inside the step
        with torch.cuda.stream(stream):
            for h, x in zip(host, sl):
                x.copy_(h, non_blocking=True)
            return analyze_exchange(ctx, cfg, n, sl, lo, collective_device=coll_dev, stream=stream.cuda_stream)

    def timed(fn, steps):
        tot, res = 0.0, None
        for _ in range(steps):
            flush.fill_(1)
            torch.cuda.synchronize(dev)
            dist.barrier()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            res = fn()
            b.record(stream)
            b.synchronize()
            tot += a.elapsed_time(b)
        t = torch.tensor([tot], dtype=torch.float64, device=coll_dev or "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()), res

    for _ in range(args.warmup):
        step_device()
    with ClockSampler(local) as clk:
        ms_dev, res = timed(step_device, args.steps)
        for _ in range(args.warmup):
            step_host()
        ms_e2e, res_e2e = timed(step_host, args.steps)
    if rank == 0:
        r, xt = res
        fx = load_full_digest(args.workload)
        digest = digest_for(r, fx, n)
        if fx is not None and digest != fx["digest"]:
            raise SystemExit(f"bench: exchange-mode report digest {digest} != {fx['digest']} ({fx['source']})")
        peak, peak_kind = load_peaks()
        step_s = ms_dev / args.steps / 1000.0
        alg = 16 * n + 36 * n_acc
        whole = {"bound": "hbm", "achieved": alg / step_s / 1e9, "peak": peak * world, "unit": "GB/s",
                 "frac": alg / step_s / 1e9 / (peak * world), "kernel": "whole analysis over all ranks "
                 "(algorithmic bytes 16N + 36A against the ranks' summed HBM peak)", "peak_source": peak_kind,
                 "traffic": None}
        line = {
            "metric": METRIC, "value": n * args.steps / (ms_dev / 1000.0), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_dev / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": desc,
            "run": {"reports": int(len(r["kind"])), "report_digest": digest,
                    "report_digest_expected": fx["digest"] if fx else None,
                    "parallelism": f"exchange mode x{world}: 1/{world} slice per rank, hard-event all-gather, "
                                   "NCCL all-to-all of access records by location hash, candidate merge on rank 0",
                    "l2": "flushed before every timed step (256 MiB write)"},
            "e2e": {"value": n * args.steps / (ms_e2e / 1000.0), "unit": UNIT,
                    "h2d_bytes_per_step": 16 * n, "d2h_bytes_per_step": 9 * int(len(r["kind"])) + 64,
                    "ms_per_step": ms_e2e / args.steps,
                    "input": "every rank uploads its own 16-B/event slice (1/N of the trace)"},
            "roofline": whole, "roofline_whole_analysis": whole,
            "gpu_launches": ctx.launches() * args.steps, "clocks": clk.summary(),
        }
        print(json.dumps(line))
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", default="c5", choices=["c2", "c3", "c4", "c5"],
                    help="BASELINE.json config (default c5: the metric's 1/2/4/8-GPU sweep config, 1.007e9 events)")
    ap.add_argument("--ref-seconds", type=float, default=8.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mode", choices=["replicas", "sharded", "exchange"], default=None,
                    help="N>1: independent traces per GPU (default), or one trace: c5 defaults to the exchange mode "
                         "(slices + all-to-all), 'sharded' = every rank holds the whole trace (address ranges)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference(args)
    elif world > 1 and (args.mode or ("exchange" if args.workload == "c5" else "replicas")) == "exchange":
        run_b200_exchange(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
