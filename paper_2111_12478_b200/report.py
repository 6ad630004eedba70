"""Race reports in the reference's output contract (report.py:19-100).

``RaceReport.to_json`` is byte-identical to the reference: key order
detector, kind, location{space,[block],addr "%#x"}, prior, current, class,
confidence, compact separators.  :func:`ndjson_lines` formats the engine's
report arrays directly (no per-report objects) for the CLI and large traces.
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .trace import GLOBAL, SHARED, Location, ThreadId, Trace, tid_str

WW = "ww"
WR = "wr"
RW = "rw"
KINDS = (WW, WR, RW)
INTRAWARP = "intrawarp"
INTERWARP = "interwarp"
INTERBLOCK = "interblock"


def classify(a, b) -> str:
    if a.block != b.block:
        return INTERBLOCK
    if a.warp != b.warp:
        return INTERWARP
    return INTRAWARP


@dataclass(frozen=True)
class Endpoint:
    event: int
    tid: ThreadId
    instr: int


@dataclass(frozen=True)
class RaceReport:
    detector: str
    kind: str
    loc: Location
    prior: Endpoint
    current: Endpoint
    confidence: str

    @property
    def klass(self) -> str:
        return classify(self.prior.tid, self.current.tid)

    def to_dict(self) -> dict:
        loc: dict = {"space": self.loc.space}
        if self.loc.space != GLOBAL:
            loc["block"] = self.loc.block
        loc["addr"] = f"{self.loc.addr:#x}"
        return {
            "detector": self.detector,
            "kind": self.kind,
            "location": loc,
            "prior": {"event": self.prior.event, "tid": tid_str(self.prior.tid), "instr": self.prior.instr},
            "current": {"event": self.current.event, "tid": tid_str(self.current.tid), "instr": self.current.instr},
            "class": self.klass,
            "confidence": self.confidence,
        }

    def to_json(self) -> str:
        return json.dumps(self.to_dict(), separators=(",", ":"))


def _loc_of(key: int) -> Location:
    if key & N.SHARED_BIT:
        return Location(SHARED, (key >> 40) & ((1 << 23) - 1), key & ((1 << 40) - 1))
    return Location(GLOBAL, None, key)


def build_reports(tr: Trace, res: dict, detector: str = "gwcp") -> list[RaceReport]:
    cfg = tr.config
    out: list[RaceReport] = []
    kinds = res["kind"].tolist()
    pri = res["prior"].tolist()
    cur = res["current"].tolist()
    for i in range(len(kinds)):
        p, c = pri[i], cur[i]
        pt = cfg.thread_of(int(tr.tidop[p]) & N.TID_MASK)
        ct = cfg.thread_of(int(tr.tidop[c]) & N.TID_MASK)
        out.append(
            RaceReport(
                detector,
                KINDS[kinds[i]],
                _loc_of(int(tr.key[c])),
                Endpoint(p, pt, int(tr.instr[p])),
                Endpoint(c, ct, int(tr.instr[c])),
                "first" if i == 0 else "post-race",
            )
        )
    return out


def ndjson_lines(tr: Trace, res: dict, detector: str = "gwcp") -> list[str]:
    """The reference's ``rep.to_json()`` lines, formatted from the arrays."""
    cfg = tr.config
    W, L = cfg.warps, cfg.lanes
    kinds = res["kind"].tolist()
    pri = res["prior"]
    cur = res["current"]
    if len(pri) == 0:
        return []
    ptid = (tr.tidop[pri] & np.uint32(N.TID_MASK)).astype(np.int64)
    ctid = (tr.tidop[cur] & np.uint32(N.TID_MASK)).astype(np.int64)
    pins = tr.instr[pri].tolist()
    cins = tr.instr[cur].tolist()
    keys = tr.key[cur].tolist()
    pb, pw, pl = (ptid // (W * L)).tolist(), ((ptid // L) % W).tolist(), (ptid % L).tolist()
    cb, cw, cl = (ctid // (W * L)).tolist(), ((ctid // L) % W).tolist(), (ctid % L).tolist()
    pri = pri.tolist()
    cur = cur.tolist()
    head = f'{{"detector":"{detector}","kind":"'
    lines = []
    for i in range(len(kinds)):
        k = keys[i]
        if k & N.SHARED_BIT:
            loc = f'{{"space":"shared","block":{(k >> 40) & 0x7FFFFF},"addr":"{k & 0xFFFFFFFFFF:#x}"}}'
        else:
            loc = f'{{"space":"global","addr":"{k:#x}"}}'
        if pb[i] != cb[i]:
            kl = INTERBLOCK
        elif pw[i] != cw[i]:
            kl = INTERWARP
        else:
            kl = INTRAWARP
        lines.append(
            f'{head}{KINDS[kinds[i]]}","location":{loc},'
            f'"prior":{{"event":{pri[i]},"tid":"{pb[i]}.{pw[i]}.{pl[i]}","instr":{pins[i]}}},'
            f'"current":{{"event":{cur[i]},"tid":"{cb[i]}.{cw[i]}.{cl[i]}","instr":{cins[i]}}},'
            f'"class":"{kl}","confidence":"{"first" if i == 0 else "post-race"}"}}'
        )
    return lines


class Reporter:
    """Holds a finished run's reports (the batch engine dedups on the GPU)."""

    def __init__(self, detector: str):
        self.detector = detector
        self.reports: list[RaceReport] = []


def result_digest(res: dict) -> str:
    """sha256 of a run's report and diagnostic arrays (kind u8, prior u32,
    current u32, diag event/code u32, diag lock u64), in final order.  The
    NDJSON lines are a function of these arrays and the trace, so equal
    digests on one trace mean byte-identical ``check`` output; used to pin
    the billion-event configs, whose NDJSON is too large to keep."""
    import hashlib

    hs = hashlib.sha256()
    hs.update(np.uint64(len(res["kind"])).tobytes())
    for k, dt in (("kind", np.uint8), ("prior", np.uint32), ("current", np.uint32), ("diag_event", np.uint32),
                  ("diag_code", np.uint32), ("diag_lock", np.uint64)):
        hs.update(np.ascontiguousarray(res.get(k, np.zeros(0, dt)), dt).tobytes())
    return hs.hexdigest()
