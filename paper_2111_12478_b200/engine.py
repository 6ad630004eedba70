"""Drop-in ``run(trace, detector)`` (engine.py:98-155) backed by the GPU.

``run`` encodes the trace as SoA (no-op for traces from
:func:`parse_trace`), hands it to libgwcp_b200 (H2D, all kernels on the
device, D2H of the report arrays) and rebuilds the reference's result
objects.  There is no CPU analysis path.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _native as N
from .report import RaceReport, build_reports
from .trace import Diagnostic, Trace, encode, tid_str


@dataclass
class RunResult:
    reports: list[RaceReport]
    diagnostics: list[Diagnostic]
    ordered_pairs: list[tuple[int, int]] | None = None
    n_events: int = 0
    stats: dict | None = None

    @property
    def raced(self) -> bool:
        return bool(self.reports)


def diagnostics_of(tr: Trace, res: dict) -> list[Diagnostic]:
    """Render engine diagnostics as the reference's messages
    (gwcp.py:178-182, :197-201, :323-330)."""
    out: list[Diagnostic] = []
    ev = res["diag_event"].tolist()
    code = res["diag_code"].tolist()
    lock = res["diag_lock"].tolist()
    i = 0
    while i < len(ev):
        e, c = ev[i], code[i]
        if c == 1:
            out.append(Diagnostic(e, f"reentrant acquire of lock {lock[i]:#x}"))
            i += 1
        elif c == 2:
            out.append(Diagnostic(e, f"release of unheld lock {lock[i]:#x}"))
            i += 1
        else:
            held = []
            while i < len(ev) and ev[i] == e and code[i] == 3:
                held.append(f"{lock[i]:#x}")
                i += 1
            tid = tr.config.thread_of(int(tr.tidop[e]) & N.TID_MASK)
            out.append(Diagnostic(e, f"thread {tid_str(tid)} exited holding lock(s) {', '.join(held)}"))
    return out


def analyze(trace, *, inactive_opt: bool = True, hb: bool = False) -> tuple[Trace, dict]:
    tr = encode(trace)
    res = N.analyze(tr.cfg_tuple, tr.key, tr.tidop, tr.instr, inactive_opt=inactive_opt, hb=hb)
    return tr, res


def run(trace, detector, *, order_matrix: bool = False, collect_stats: bool = False) -> RunResult:
    if order_matrix or collect_stats:
        raise NotImplementedError("--order-matrix / stats stay on the reference's Python detector")
    name = getattr(detector, "name", "gwcp")
    if name not in ("gwcp", "hb"):
        raise NotImplementedError("only the gwcp and hb detectors are accelerated")
    # (a gpurace.GwcpDetector keeps the option as _inactive_opt, gwcp.py:119)
    inactive = getattr(detector, "inactive_opt", getattr(detector, "_inactive_opt", True))
    tr, res = analyze(trace, inactive_opt=inactive, hb=name == "hb")
    reports = build_reports(tr, res, name)
    diags = diagnostics_of(tr, res)
    if hasattr(detector, "reporter"):
        detector.reporter.reports = list(reports)
    if hasattr(detector, "diagnostics"):
        detector.diagnostics = list(diags)
    return RunResult(reports=reports, diagnostics=diags, n_events=len(tr))
