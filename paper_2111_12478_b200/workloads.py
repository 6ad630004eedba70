"""Synthetic trace workloads C1-C5 (BASELINE.json configs).

Every random choice is a counter-based hash ``splitmix64(seed, fields...)``,
so the text emitter (for the reference / oracle) and the vectorised SoA
emitter (for the engine) produce the same trace.  Geometries are
parameters: the full configs are the defaults, the parity tests use reduced
ones from the same recipes.

  C1  litmus patterns widened to 2 blocks x 32 lanes (wacc records)
  C2  B x 8 x 32, __syncthreads-only, own-slot words + ~1 % random words
  C3  B x 8 x 32, device fences, atomics, spin locks (lock-queue rules)
  C4  B x 8 x 32, ITS-divergent warps: single-lane accesses, random-mask warp barriers
  C5  the C2 recipe at 1024 x 8 x 32 with 256M words (scaling sweep)
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .trace import Trace, TraceConfig

M64 = (1 << 64) - 1


def _mix(z):
    z = (z + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def h(*fields) -> int:
    z = 0
    for f in fields:
        z = _mix(z ^ (f & M64))
    return z


def _mix_np(z):
    z = z + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def h_np(*fields):
    z = np.uint64(0)
    for f in fields:
        z = _mix_np(z ^ np.asarray(f, dtype=np.uint64))
    return z


P01 = int(0.01 * 2**64)


# ------------------------------------------------------------------ C2 ----
def c2_params(blocks=64, warps=8, lanes=32, phases=8, records=8, words_per_block=1024, seed=2):
    return dict(blocks=blocks, warps=warps, lanes=lanes, phases=phases, records=records,
                words_per_block=words_per_block, seed=seed)


def c2_soa_prefix(max_events, blocks=64, warps=8, lanes=32, phases=8, records=8, words_per_block=1024,
                  seed=2) -> Trace:
    """The record-aligned prefix (>= min(max_events, N) events, whole records)
    of :func:`c2_soa` without materialising the whole trace."""
    per_rec_round = blocks * warps * lanes
    per_phase = records * per_rec_round + blocks
    if max_events >= phases * per_phase:
        return c2_soa(blocks, warps, lanes, phases, records, words_per_block, seed)
    full = max_events // per_phase
    head = c2_soa(blocks, warps, lanes, full, records, words_per_block, seed) if full else None
    rem = max_events - full * per_phase
    rr = min(records, -(-rem // per_rec_round))  # records of the partial phase
    part = _c2_phase(blocks, warps, lanes, full, rr, records, words_per_block, seed)
    parts = [t for t in (head, part) if t is not None]
    key = np.concatenate([t.key for t in parts])
    to = np.concatenate([t.tidop for t in parts])
    ins = np.concatenate([t.instr for t in parts])
    return Trace(TraceConfig(blocks, warps, lanes), key, to, ins)


def _c2_phase(B, W, L, ph, rr, R, WB, seed) -> Trace:
    """Records r < rr of phase ph (no barriers) -- the C2 recipe."""
    with np.errstate(over="ignore"):
        r, b, w, l = np.meshgrid(np.arange(rr), np.arange(B), np.arange(W), np.arange(L), indexing="ij")
        p = np.uint64(ph)
        r, b, w, l = (x.astype(np.uint64).ravel() for x in (r, b, w, l))
        hh = h_np(seed, p, r, b, w, l)
        own = b * np.uint64(WB) + ((np.uint64(256) * p + np.uint64(L) * w + l) % np.uint64(WB))
        rnd = h_np(hh, 7) % np.uint64(B * WB)
        word = np.where(hh < np.uint64(P01), rnd, own)
        iswr = ((p + r + w) % np.uint64(2)) == 0
        flat = ((b * np.uint64(W) + w) * np.uint64(L) + l).astype(np.uint32)
        op = np.where(iswr, np.uint32(N.K_WRITE), np.uint32(N.K_READ)).astype(np.uint32) << np.uint32(N.OP_SHIFT)
        cont = np.where(l > 0, np.uint32(N.F_CONT), np.uint32(0))
        return Trace(TraceConfig(B, W, L), word * np.uint64(4), flat | op | cont, (np.uint64(16) * r + w).astype(np.uint32))


def c2_soa(blocks=64, warps=8, lanes=32, phases=8, records=8, words_per_block=1024, seed=2) -> Trace:
    """C2: barrier-only trace, one full-mask wacc per (phase, record, block, warp)."""
    with np.errstate(over="ignore"):
        B, W, L, P, R = blocks, warps, lanes, phases, records
        WB = words_per_block
        words = B * WB
        p, r, b, w, l = np.meshgrid(np.arange(P), np.arange(R), np.arange(B), np.arange(W), np.arange(L),
                                    indexing="ij")
        p, r, b, w, l = (x.astype(np.uint64) for x in (p, r, b, w, l))
        hh = h_np(seed, p, r, b, w, l)
        own = b * np.uint64(WB) + ((np.uint64(256) * p + np.uint64(L) * w + l) % np.uint64(WB))
        rnd = h_np(hh, 7) % np.uint64(words)
        word = np.where(hh < np.uint64(P01), rnd, own)
        addr = word * np.uint64(4)
        iswr = ((p + r + w) % np.uint64(2)) == 0
        instr = (np.uint64(16) * r + w).astype(np.uint32)
        flat = ((b * np.uint64(W) + w) * np.uint64(L) + l).astype(np.uint32)
        op = np.where(iswr, np.uint32(N.K_WRITE), np.uint32(N.K_READ)).astype(np.uint32) << np.uint32(N.OP_SHIFT)
        cont = np.where(l > 0, np.uint32(N.F_CONT), np.uint32(0))
        tidop = flat | op | cont
        # per phase: P blocks of accesses then B barriers
        acc_per_phase = R * B * W * L
        n = P * (acc_per_phase + B)
        key = np.zeros(n, np.uint64)
        to = np.zeros(n, np.uint32)
        ins = np.zeros(n, np.uint32)
        addr = addr.reshape(P, -1)
        tidop = tidop.reshape(P, -1)
        instr = instr.reshape(P, -1)
        bar_to = (np.arange(B, dtype=np.uint32) * np.uint32(W * L)) | np.uint32(N.K_BARRIER << N.OP_SHIFT)
        for ph in range(P):
            o = ph * (acc_per_phase + B)
            key[o:o + acc_per_phase] = addr[ph]
            to[o:o + acc_per_phase] = tidop[ph]
            ins[o:o + acc_per_phase] = instr[ph]
            to[o + acc_per_phase:o + acc_per_phase + B] = bar_to
    return Trace(TraceConfig(B, W, L), key, to, ins)


def soa_to_text(tr: Trace) -> str:
    """Canonical text of an SoA trace (wacc for multi-event records)."""
    cfg = tr.config
    W, L = cfg.warps, cfg.lanes
    lines = [f"config blocks={cfg.blocks} warps={W} lanes={L}"]
    key, to, ins = tr.key.tolist(), tr.tidop.tolist(), tr.instr.tolist()
    n = len(to)
    i = 0
    while i < n:
        j = i + 1
        while j < n and (to[j] & N.F_CONT):
            j += 1
        t0 = to[i]
        kind = (t0 >> N.OP_SHIFT) & 7
        flat = t0 & N.TID_MASK
        b, w, l = flat // (W * L), (flat // L) % W, flat % L
        dev = "device" if t0 & N.F_DEVICE else "block"

        def loc(k):
            if k & N.SHARED_BIT:
                return f"s:{k & 0xFFFFFFFFFF:#x}"
            return f"g:{k:#x}"

        if kind <= N.K_WRITE:
            tail = (f" atomic {dev}" if t0 & N.F_ATOMIC else "") + f" instr {ins[i]}"
            op = "wr" if kind == N.K_WRITE else "rd"
            if j - i > 1:
                mask = 0
                for x in range(i, j):
                    mask |= 1 << ((to[x] & N.TID_MASK) % L)
                addrs = ",".join(loc(key[x]) for x in range(i, j))
                lines.append(f"wacc {b} {w} {mask:#x} {op} {addrs}{tail}")
            else:
                lines.append(f"{b}.{w}.{l} {op} {loc(key[i])}{tail}")
        elif kind == N.K_BARRIER:
            if t0 & N.F_WARPBAR:
                lines.append(f"bar warp {b} {w} {ins[i]:#x}")
            else:
                lines.append(f"bar block {b}")
        elif kind == N.K_ACQUIRE:
            lines.append(f"{b}.{w}.{l} acq {key[i]:#x} {dev}")
        elif kind == N.K_RELEASE:
            lines.append(f"{b}.{w}.{l} rel {key[i]:#x} {dev}")
        elif kind == N.K_FENCE:
            lines.append(f"{b}.{w}.{l} fence {dev}")
        else:
            lines.append(f"{b}.{w}.{l} end")
        i = j
    return "\n".join(lines) + "\n"


# ------------------------------------------------------------------ C3 ----
def c3_text(blocks=16, warps=8, lanes=32, iters=24, locks=256, region=64, private=512, seed=3) -> str:
    """C3: spin-lock critical sections (lane 0) between warp barriers, device
    fences, failed-CAS polling reads, atomic counters, block barriers every
    16 iterations, 0.1 % unprotected writes into a lock region (races)."""
    B, W, L = blocks, warps, lanes
    lines = [f"config blocks={B} warps={W} lanes={L}"]
    lock_base = 0x10000000
    region_base = 0x20000000
    counter = 0x30000000
    full = (1 << L) - 1
    for it in range(iters):
        for b in range(B):
            for w in range(W):
                pw = ((b * W + w) * private) * 4
                for op in ("rd", "wr"):
                    addrs = ",".join(f"g:{pw + ((L * it + l) % private) * 4:#x}" for l in range(L))
                    lines.append(f"wacc {b} {w} {full:#x} {op} {addrs} instr {1 if op == 'rd' else 2}")
                lines.append(f"bar warp {b} {w} {full:#x}")
                hh = h(seed, it, b, w)
                k = hh % locks
                lw = lock_base + 4 * k
                for _ in range((hh >> 20) % 4):
                    lines.append(f"{b}.{w}.0 rd g:{lw:#x} atomic device instr 3")
                lines.append(f"{b}.{w}.0 acq {lw:#x} device")
                for a in range(1 + (hh >> 24) % 4):
                    x = region_base + 4 * (k * region + (h(hh, a) % region))
                    op = "wr" if (hh >> (28 + a)) & 1 else "rd"
                    lines.append(f"{b}.{w}.0 {op} g:{x:#x} instr {4 + a}")
                lines.append(f"{b}.{w}.0 fence device")
                lines.append(f"{b}.{w}.0 rel {lw:#x} device")
                lines.append(f"bar warp {b} {w} {full:#x}")
                if (hh >> 40) % 100 == 0:
                    sc = "device" if (hh >> 48) % 10 else "block"
                    lines.append(f"{b}.{w}.{1 % L} wr g:{counter:#x} atomic {sc} instr 9")
                if (hh >> 32) % 1000 == 0 and L > 1:
                    x = region_base + 4 * (k * region + (hh >> 8) % region)
                    lines.append(f"{b}.{w}.1 wr g:{x:#x} instr 10")
        if it % 16 == 15:
            for b in range(B):
                lines.append(f"bar block {b}")
    return "\n".join(lines) + "\n"


def c3_group_offsets(blocks=16, warps=8, lanes=32, iters=24, locks=256, region=64, private=512, seed=3):
    """First event of every (it, b, w) group of :func:`c3_text` (uint64,
    length iters*B*W + 1, the last entry = the event count); the block barriers
    of every 16th iteration are counted with the iteration's last group."""
    B, W, L = blocks, warps, lanes
    with np.errstate(over="ignore"):
        it, b, w = np.meshgrid(np.arange(iters), np.arange(B), np.arange(W), indexing="ij")
        it, b, w = (x.astype(np.uint64).ravel() for x in (it, b, w))
        hh = h_np(seed, it, b, w)
        npoll = (hh >> np.uint64(20)) % np.uint64(4)
        nacc = np.uint64(1) + (hh >> np.uint64(24)) % np.uint64(4)
        cnt = ((hh >> np.uint64(40)) % np.uint64(100) == 0).astype(np.uint64)
        inj = ((hh >> np.uint64(32)) % np.uint64(1000) == 0).astype(np.uint64) * np.uint64(L > 1)
        size = np.uint64(2 * L + 5) + npoll + nacc + cnt + inj
        last = (b == np.uint64(B - 1)) & (w == np.uint64(W - 1)) & (it % np.uint64(16) == np.uint64(15))
        size = size + np.where(last, np.uint64(B), np.uint64(0))
    off = np.zeros(len(size) + 1, np.uint64)
    np.cumsum(size, out=off[1:])
    return off


def c3_counts(blocks=16, warps=8, lanes=32, iters=24, locks=256, region=64, private=512, seed=3):
    """(events, accesses, acquires) of :func:`c3_text` without generating it."""
    B, W, L = blocks, warps, lanes
    with np.errstate(over="ignore"):
        it, b, w = np.meshgrid(np.arange(iters), np.arange(B), np.arange(W), indexing="ij")
        hh = h_np(seed, *(x.astype(np.uint64).ravel() for x in (it, b, w)))
        acc = (np.uint64(2 * L) + (hh >> np.uint64(20)) % np.uint64(4) + np.uint64(1) + (hh >> np.uint64(24)) % np.uint64(4)
               + ((hh >> np.uint64(40)) % np.uint64(100) == 0) + ((hh >> np.uint64(32)) % np.uint64(1000) == 0) * (L > 1))
    off = c3_group_offsets(blocks, warps, lanes, iters, locks, region, private, seed)
    return int(off[-1]), int(acc.sum()), int(iters * B * W)


# ------------------------------------------------------------------ C4 ----
def c4_text(blocks=16, warps=8, lanes=32, iters=16, words_per_block=16384, seed=4) -> str:
    """C4: Volta-ITS divergent warps -- a random lane subset issues single-lane
    accesses in random lane order, the complement one wacc; random-mask warp
    barriers every 4 iterations, block barriers every 64."""
    B, W, L = blocks, warps, lanes
    WB = words_per_block
    words = B * WB
    lines = [f"config blocks={B} warps={W} lanes={L}"]
    for it in range(iters):
        for b in range(B):
            for w in range(W):
                hh = h(seed, it, b, w)

                def word(l):
                    x = h(hh, l, 1)
                    own = b * WB + ((L * W * it + L * w + l) % WB)
                    if x < int(0.99 * 2**64):
                        return own
                    if x < int(0.9999 * 2**64):
                        return b * WB + h(x, 2) % WB
                    return h(x, 3) % words

                single = [l for l in range(L) if (h(hh, l, 4) >> 63) & 1]
                order = sorted(single, key=lambda l: h(hh, l, 5))
                isw = (hh >> 7) & 1
                op = "wr" if isw else "rd"
                for l in order:
                    lines.append(f"{b}.{w}.{l} {op} g:{4 * word(l):#x} instr {20 + l}")
                rest = [l for l in range(L) if l not in single]
                if rest:
                    mask = 0
                    for l in rest:
                        mask |= 1 << l
                    addrs = ",".join(f"g:{4 * word(l):#x}" for l in rest)
                    lines.append(f"wacc {b} {w} {mask:#x} {'rd' if isw else 'wr'} {addrs} instr 19")
                if it % 4 == 3:
                    m = 0
                    for l in range(L):
                        if h(hh, l, 6) < int(0.6 * 2**64):
                            m |= 1 << l
                    if m == 0:
                        m = 1
                    lines.append(f"bar warp {b} {w} {m:#x}")
        if it % 64 == 63:
            for b in range(B):
                lines.append(f"bar block {b}")
    return "\n".join(lines) + "\n"


# ------------------------------------------------------------------ C1 ----
def c1_texts() -> dict[str, str]:
    """Litmus patterns (src/litmus.py) widened to 2 blocks x 32 lanes."""
    L = 32
    full = (1 << L) - 1

    def wacc(b, op, addrs, extra=""):
        return f"wacc {b} 0 {full:#x} {op} " + ",".join(addrs) + extra

    own0 = [f"g:{0x1000 + 4 * l:#x}" for l in range(L)]
    own1 = [f"g:{0x2000 + 4 * l:#x}" for l in range(L)]
    hdr = f"config blocks=2 warps=1 lanes={L}"
    out = {}
    out["barrier-separated-32"] = "\n".join(
        [f"config blocks=1 warps=2 lanes={L}", f"wacc 0 0 {full:#x} wr " + ",".join(own0),
         "bar block 0", f"wacc 0 1 {full:#x} rd " + ",".join(own0)]) + "\n"
    out["barrier-missing-32"] = "\n".join(
        [f"config blocks=1 warps=2 lanes={L}", f"wacc 0 0 {full:#x} wr " + ",".join(own0),
         f"wacc 0 1 {full:#x} rd " + ",".join(own0)]) + "\n"
    out["colliding-wacc-32"] = "\n".join(
        [hdr, wacc(0, "wr", [f"g:{0x1000 + 4 * (l // 4):#x}" for l in range(L)])]) + "\n"
    out["fence-only-32"] = "\n".join(
        [hdr, wacc(0, "wr", own0), "0.0.0 fence device", wacc(1, "wr", own0)]) + "\n"
    out["device-atomic-32"] = "\n".join(
        [hdr, wacc(0, "wr", own0, " atomic device"), wacc(1, "wr", own0, " atomic device")]) + "\n"
    out["block-atomic-32"] = "\n".join(
        [hdr, wacc(0, "wr", own0, " atomic block"), wacc(1, "wr", own0, " atomic block")]) + "\n"
    out["wcp-lock-32"] = "\n".join(
        [hdr, wacc(0, "wr", own1), "0.0.0 acq 0xa device", wacc(0, "wr", own0), "0.0.0 rel 0xa device",
         "1.0.0 acq 0xa device", wacc(1, "wr", own1), wacc(1, "wr", own0), "1.0.0 rel 0xa device"]) + "\n"
    out["warp-lock-32"] = "\n".join(
        [hdr, f"bar warp 0 0 {full:#x}", "0.0.0 acq 0xa device", "0.0.0 wr g:0x10", "0.0.0 rel 0xa device",
         f"bar warp 0 0 {full:#x}", wacc(0, "rd", ["g:0x10"] * L), f"bar warp 1 0 {full:#x}",
         "1.0.0 acq 0xa device", "1.0.0 wr g:0x10", "1.0.0 rel 0xa device", f"bar warp 1 0 {full:#x}",
         wacc(1, "rd", ["g:0x10"] * L)]) + "\n"
    return out


# ------------------------------------------------------- full configs ----
# BASELINE.json configs[1..4] at full size; the bench and the
# full-scale parity tests generate them on the device (gw_gen_c*_device), the
# prefix goldens on the host with the recipes above.
CONFIGS = {
    # C2 (configs[1]): 64 x 256 threads, __syncthreads only, 64K words, ~1 % random words
    "c2": dict(gen="c2", blocks=64, warps=8, lanes=32, phases=8, records=8, words_per_block=1024, seed=2),
    # C3 (configs[2]): 1024 x 256 threads, 4096 device-scope spin locks, fences, atomics, 1.005e8 events
    "c3": dict(gen="c3", blocks=1024, warps=8, lanes=32, iters=168, locks=4096, region=64, private=512, seed=3),
    # C4 (configs[3]): 1024 x 256 threads, ITS-divergent warps (single-lane accesses in random lane order,
    # random-mask warp barriers every 4 iterations, block barriers every 64), 16M words, 1.0e9 events
    "c4": dict(gen="c4", blocks=1024, warps=8, lanes=32, iters=3786, words_per_block=16384, seed=4),
    # C5 (configs[4]): the C2 recipe at 1024 x 256 threads, 256M words, 16 phases x 240 records = 1.007e9 events
    "c5": dict(gen="c2", blocks=1024, warps=8, lanes=32, phases=16, records=240, words_per_block=262144, seed=5),
}


def c4_count(blocks, warps, iters) -> int:
    """Events of :func:`c4_text` (lanes = 32): one access per lane per
    iteration, a warp barrier per warp every 4 iterations, a block barrier per
    block every 64."""
    return iters * blocks * warps * 32 + blocks * warps * (iters // 4) + blocks * (iters // 64)


def config_counts(p: dict) -> tuple[int, int]:
    """(events, accesses) of a CONFIGS entry without generating it."""
    if p["gen"] == "c4":
        return c4_count(p["blocks"], p["warps"], p["iters"]), p["iters"] * p["blocks"] * p["warps"] * 32
    if p["gen"] == "c3":
        n, n_acc, _ = c3_counts(**{k: v for k, v in p.items() if k != "gen"})
        return n, n_acc
    n = p["phases"] * (p["records"] * p["blocks"] * p["warps"] * p["lanes"] + p["blocks"])
    return n, n - p["phases"] * p["blocks"]


def _cut(tr: Trace, P: int) -> Trace:
    """The first >= min(P, len) events of ``tr``, extended to a record boundary."""
    m = min(P, len(tr))
    while m < len(tr) and tr.tidop[m] & N.F_CONT:
        m += 1
    return Trace(tr.config, tr.key[:m], tr.tidop[:m], tr.instr[:m])


def config_prefix(p: dict, P: int) -> Trace:
    """Record-aligned host prefix (>= min(P, N) events, whole records) of a
    CONFIGS trace, built with the host recipes: the traces are iteration /
    phase major, so the first iterations are a prefix of the full trace
    (SURVEY App. B O2 makes its reports a prefix of the full run's)."""
    from .trace import parse_trace

    gp = {k: v for k, v in p.items() if k != "gen"}
    if p["gen"] == "c3":
        per_it = c3_counts(**dict(gp, iters=1))[0]
        gp["iters"] = min(p["iters"], max(1, -(-P // per_it)))
        return _cut(parse_trace(c3_text(**gp)), P)
    if p["gen"] == "c4":
        per_it = p["blocks"] * p["warps"] * 33
        gp["iters"] = min(p["iters"], max(1, -(-P // per_it)))
        return _cut(parse_trace(c4_text(**gp)), P)
    return _cut(c2_soa_prefix(P, **gp), P)
