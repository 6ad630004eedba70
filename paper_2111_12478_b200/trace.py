"""Trace model of the B200 engine: the reference's event vocabulary on a
columnar 16-byte/event SoA.

The public names and field meanings follow the reference package so code
written against ``gpurace`` reads the same (``pkg/src/gpurace/trace.py:29-145``):
``ThreadId``, ``Scope``, ``Location``, ``Barrier``, ``Event``, ``TraceConfig``,
``Trace``, ``Diagnostic``, ``TraceParseError`` and ``parse_trace``.  The
storage differs: a :class:`Trace` holds three numpy columns (``key`` u64,
``tidop`` u32, ``instr`` u32; layout in ``include/gwcp_b200.h``) and only
materialises ``Event`` objects when ``.events`` is read.  Text is parsed by
the native C++ parser; reference ``gpurace.Trace`` objects (or any objects
with the same attributes) are encoded by :func:`encode`.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterator, NamedTuple

import numpy as np

from . import _native as N

GLOBAL = "global"
SHARED = "shared"
BLOCK = "block"
DEVICE = "device"
READ = "read"
WRITE = "write"
ACQUIRE = "acquire"
RELEASE = "release"
BARRIER = "barrier"
FENCE = "fence"
END = "end"

KIND_NAMES = (READ, WRITE, ACQUIRE, RELEASE, BARRIER, FENCE, END)
KIND_CODES = {name: i for i, name in enumerate(KIND_NAMES)}


class ThreadId(NamedTuple):
    block: int
    warp: int
    lane: int


def tid_str(tid) -> str:
    return f"{tid.block}.{tid.warp}.{tid.lane}"


class Scope(NamedTuple):
    kind: str
    block: int | None = None

    @staticmethod
    def device() -> "Scope":
        return Scope(DEVICE, None)

    @staticmethod
    def of_block(block: int) -> "Scope":
        return Scope(BLOCK, block)


class Location(NamedTuple):
    space: str
    block: int | None
    addr: int


class Barrier(NamedTuple):
    scope: str  # "block" | "warp"
    block: int
    warp: int | None = None
    mask: int | None = None

    @property
    def is_warp(self) -> bool:
        return self.scope == "warp"


@dataclass(frozen=True)
class Event:
    index: int
    kind: str
    tid: ThreadId | None = None
    loc: Location | None = None
    atomic: bool = False
    scope: Scope | None = None
    instr: int | None = None
    lock: int | None = None
    barrier: Barrier | None = None
    group: int = -1

    @property
    def is_access(self) -> bool:
        return self.kind in (READ, WRITE)


@dataclass(frozen=True)
class TraceConfig:
    blocks: int
    warps: int
    lanes: int

    @property
    def n_threads(self) -> int:
        return self.blocks * self.warps * self.lanes

    def thread_index(self, tid) -> int:
        return (tid.block * self.warps + tid.warp) * self.lanes + tid.lane

    def thread_of(self, flat: int) -> ThreadId:
        lane = flat % self.lanes
        rest = flat // self.lanes
        return ThreadId(rest // self.warps, rest % self.warps, lane)

    def threads(self) -> Iterator[ThreadId]:
        for b in range(self.blocks):
            for w in range(self.warps):
                for l in range(self.lanes):
                    yield ThreadId(b, w, l)


@dataclass(frozen=True)
class Diagnostic:
    index: int
    message: str

    def __str__(self) -> str:
        return f"event {self.index}: {self.message}"


class TraceParseError(ValueError):
    def __init__(self, line_no: int, message: str):
        super().__init__(f"line {line_no}: {message}")
        self.line_no = line_no


class UnsupportedTrace(ValueError):
    """A value the 16-byte SoA cannot represent exactly (never truncated)."""


class Trace:
    """A trace: configuration plus the SoA columns (events built lazily)."""

    def __init__(self, config: TraceConfig, key=None, tidop=None, instr=None):
        self.config = config
        self.key = np.zeros(0, np.uint64) if key is None else np.ascontiguousarray(key, dtype=np.uint64)
        self.tidop = np.zeros(0, np.uint32) if tidop is None else np.ascontiguousarray(tidop, dtype=np.uint32)
        self.instr = np.zeros(0, np.uint32) if instr is None else np.ascontiguousarray(instr, dtype=np.uint32)
        if not (len(self.key) == len(self.tidop) == len(self.instr)):
            raise ValueError("SoA columns differ in length")
        self._events: list[Event] | None = None

    def __len__(self) -> int:
        return len(self.tidop)

    @property
    def cfg_tuple(self) -> tuple[int, int, int]:
        c = self.config
        return (c.blocks, c.warps, c.lanes)

    @property
    def events(self) -> list[Event]:
        if self._events is None:
            self._events = decode(self)
        return self._events


# ---------------------------------------------------------------- encoding --


def _loc_key(loc, tid, index: int) -> int:
    space = loc.space
    addr = loc.addr
    if space == GLOBAL:
        if not (0 <= addr < 1 << 63):
            raise UnsupportedTrace(f"event {index}: global address {addr:#x} outside [0, 2^63)")
        return addr
    if space == SHARED:
        blk = loc.block
        if not (0 <= addr < 1 << 40) or blk is None or not (0 <= blk < 1 << 23):
            raise UnsupportedTrace(f"event {index}: shared location {loc!r} outside the SoA encoding")
        return N.SHARED_BIT | (blk << 40) | addr
    raise UnsupportedTrace(f"event {index}: unknown memory space {space!r}")


def encode(trace) -> Trace:
    """Encode any reference-shaped trace (``.config`` + ``.events``) as SoA.

    Accepts ``gpurace.Trace`` objects, so ``run(ref_trace, GwcpDetector(cfg))``
    works as a drop-in.  Raises :class:`UnsupportedTrace` for values the SoA
    cannot hold exactly.
    """
    if isinstance(trace, Trace):
        return trace
    cfg0 = trace.config
    cfg = TraceConfig(int(cfg0.blocks), int(cfg0.warps), int(cfg0.lanes))
    W, L = cfg.warps, cfg.lanes
    if cfg.n_threads > N.TID_MASK + 1:
        raise UnsupportedTrace("more than 2^24 threads")
    evs = trace.events
    n = len(evs)
    key = np.zeros(n, np.uint64)
    tidop = np.zeros(n, np.uint32)
    instr = np.zeros(n, np.uint32)
    prev_group = None
    for i, ev in enumerate(evs):
        if ev.index != i:
            raise UnsupportedTrace(f"event at position {i} carries index {ev.index}")
        kind = KIND_CODES.get(ev.kind)
        if kind is None:
            raise UnsupportedTrace(f"event {i}: unknown kind {ev.kind!r}")
        op = kind
        k = 0
        ins = 0
        g = ev.group
        if g is not None and g >= 0 and prev_group is not None and prev_group == g:
            op |= N.F_CONT >> N.OP_SHIFT
        prev_group = g if (g is not None and g >= 0) else None
        if kind == N.K_BARRIER:
            bar = ev.barrier
            if bar.scope == "warp":
                if L > 32:
                    raise UnsupportedTrace("warp barrier with more than 32 lanes")
                flat = (bar.block * W + bar.warp) * L
                op |= N.F_WARPBAR >> N.OP_SHIFT
                ins = int(bar.mask)
                k = (bar.block << 32) | bar.warp
            else:
                flat = bar.block * W * L
        else:
            t = ev.tid
            flat = (t.block * W + t.warp) * L + t.lane
            sc = ev.scope
            if kind in (N.K_READ, N.K_WRITE):
                k = _loc_key(ev.loc, t, i)
                if ev.instr is None or not (0 <= ev.instr < 1 << 32):
                    raise UnsupportedTrace(f"event {i}: instruction id {ev.instr!r} outside [0, 2^32)")
                ins = int(ev.instr)
                if ev.atomic:
                    op |= N.F_ATOMIC >> N.OP_SHIFT
                    if sc is not None and sc.kind == DEVICE:
                        op |= N.F_DEVICE >> N.OP_SHIFT
            elif kind in (N.K_ACQUIRE, N.K_RELEASE):
                lk = ev.lock
                if not (0 <= lk < 1 << 64):
                    raise UnsupportedTrace(f"event {i}: lock {lk!r} outside [0, 2^64)")
                k = int(lk)
                if sc is not None and sc.kind == DEVICE:
                    op |= N.F_DEVICE >> N.OP_SHIFT
                elif sc is not None and sc.block != t.block:
                    raise UnsupportedTrace(f"event {i}: block scope of another block")
            elif kind == N.K_FENCE:
                if sc is not None and sc.kind == DEVICE:
                    op |= N.F_DEVICE >> N.OP_SHIFT
        key[i] = k
        tidop[i] = flat | (op << N.OP_SHIFT)
        instr[i] = ins
    return Trace(cfg, key, tidop, instr)


def decode(tr: Trace) -> list[Event]:
    """Materialise reference-style Event objects from the SoA (for callers
    that iterate ``trace.events``; the engine never does)."""
    cfg = tr.config
    out: list[Event] = []
    group = -1
    keys = tr.key.tolist()
    tos = tr.tidop.tolist()
    ins = tr.instr.tolist()
    for i in range(len(tos)):
        to = tos[i]
        kind = (to >> N.OP_SHIFT) & 7
        if not (to & N.F_CONT):
            group += 1
        flat = to & N.TID_MASK
        name = KIND_NAMES[kind]
        dev = bool(to & N.F_DEVICE)
        if kind == N.K_BARRIER:
            tid = cfg.thread_of(flat)
            if to & N.F_WARPBAR:
                bar = Barrier("warp", tid.block, tid.warp, ins[i])
            else:
                bar = Barrier(BLOCK, tid.block)
            out.append(Event(i, name, barrier=bar, group=group))
            continue
        tid = cfg.thread_of(flat)
        if kind <= N.K_WRITE:
            k = keys[i]
            if k & N.SHARED_BIT:
                loc = Location(SHARED, (k >> 40) & ((1 << 23) - 1), k & ((1 << 40) - 1))
            else:
                loc = Location(GLOBAL, None, k)
            atomic = bool(to & N.F_ATOMIC)
            scope = (Scope.device() if dev else Scope.of_block(tid.block)) if atomic else None
            out.append(Event(i, name, tid=tid, loc=loc, atomic=atomic, scope=scope, instr=ins[i], group=group))
        elif kind in (N.K_ACQUIRE, N.K_RELEASE):
            scope = Scope.device() if dev else Scope.of_block(tid.block)
            out.append(Event(i, name, tid=tid, scope=scope, lock=keys[i], group=group))
        elif kind == N.K_FENCE:
            scope = Scope.device() if dev else Scope.of_block(tid.block)
            out.append(Event(i, name, tid=tid, scope=scope, group=group))
        else:
            out.append(Event(i, name, tid=tid, group=group))
    return out


def parse_trace(text: str | bytes) -> Trace:
    """Text -> SoA trace via the native parser (grammar of trace.py:226-398).

    Raises :class:`TraceParseError` with the reference's line number and
    message; :class:`UnsupportedTrace` for values outside the SoA encoding.
    """
    try:
        cfg, key, tidop, instr = N.parse_text(text)
    except N.EngineError as e:
        msg = str(e)
        line = getattr(e, "line", 0)
        body = msg.split(": ", 1)[1] if msg.startswith("line ") and ": " in msg else msg
        if e.code == N.GW_E_PARSE:
            raise TraceParseError(line, body) from None
        if e.code == N.GW_E_UNSUPPORTED:
            raise UnsupportedTrace(msg) from None
        raise
    return Trace(TraceConfig(*cfg), key, tidop, instr)


SOA_MAGIC = b"GWSOA\x00\x01\x00"


def save_soa(trace, path: str) -> None:
    """Write a trace as the binary SoA file of include/gwcp_b200.h (16 B/event;
    the on-disk form of SURVEY §8(f) rank 1, read back without parsing)."""
    tr = encode(trace)
    N.save_soa(path, tr.cfg_tuple, tr.key, tr.tidop, tr.instr)


def load_trace(path: str) -> Trace:
    """A trace file: binary SoA (by its magic) or the text format (parse_trace)."""
    with open(path, "rb") as fh:
        head = fh.read(8)
        if head == SOA_MAGIC:
            try:
                cfg, key, tidop, instr = N.load_soa(path)
            except N.EngineError as e:
                raise TraceParseError(0, str(e)) from None
            return Trace(TraceConfig(*cfg), key, tidop, instr)
        data = head + fh.read()
    return parse_trace(data)


_VALIDATE_MSG = {
    1: lambda a, b, cfg: f"barrier divergence: exited lane {a} in warp barrier mask",
    2: lambda a, b, cfg: f"barrier divergence: no live threads in block {a}",
    3: lambda a, b, cfg: f"event after end of thread {tid_str(cfg.thread_of(a))}",
    4: lambda a, b, cfg: f"shared location of block {a} used by thread {tid_str(cfg.thread_of(b))}",
    5: lambda a, b, cfg: f"reentrant acquire of lock {a:#x}",
    6: lambda a, b, cfg: f"release of unheld lock {a:#x}",
    7: lambda a, b, cfg: f"improperly nested release of lock {a:#x}",
}


def validate_trace(trace, *, ctx=None) -> list[Diagnostic]:
    """validate_trace (trace.py:522-601) over the SoA: on the GPU through a
    context (gw_ctx_validate; the `check` CLI path), else the host pass."""
    tr = encode(trace)
    raw = N.validate(tr.cfg_tuple, tr.key, tr.tidop, tr.instr, ctx=ctx)
    return [Diagnostic(ev, _VALIDATE_MSG[code](a, b, tr.config)) for ev, code, a, b in raw]


def infer_locks(trace, *, ctx=None) -> tuple[Trace, list[Diagnostic]]:
    """infer_locks (trace.py:609-680) on the GPU (gw_ctx_infer_locks): atomic
    write + fence -> acquire, fence + atomic write -> release of a held lock;
    returns the rewritten SoA trace and the reference's diagnostics."""
    tr = encode(trace)
    if ctx is None:
        ctx = N.default_context()
    (cfg, key, tidop, instr), raw = N.infer_locks(ctx, tr.cfg_tuple, tr.key, tr.tidop, tr.instr)
    out = Trace(TraceConfig(*cfg), key, tidop, instr)
    diags = [Diagnostic(ev, f"release of lock {lock:#x} not held by {tid_str(tr.config.thread_of(t))}; "
                            "left uninferred") for ev, lock, t in raw]
    return out, diags
