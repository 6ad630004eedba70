"""The reference-side binding of INTEGRATION.md, as executable code.

This is the stub a `gpurace` maintainer would add to route the `gwcp` / `hb`
detectors of `engine.run` (pkg/src/gpurace/engine.py:98-155) to
libgwcp_b200.so: plain ctypes over the C-ABI (include/gwcp_b200.h), no torch,
and the reference's OWN result objects -- `gpurace.report.RaceReport` /
`Endpoint`, `gpurace.trace.Diagnostic`, `gpurace.engine.RunResult` -- so the
CLI's NDJSON and every caller of `run` are unchanged.

    from paper_2111_12478_b200 import gpurace_backend
    gpurace_backend.install()          # gpurace.engine.run -> B200 for gwcp / hb
    # or: gpurace_backend.run(trace, gpurace.gwcp.GwcpDetector(trace.config))

`gpurace` must be importable (it is not a dependency of this package; the
tests use the reference installed into baseline/_ref).
"""

from __future__ import annotations

import ctypes as C
import os

from . import _native as N
from .trace import encode

GW_OPT_HB = 4


class _View(C.Structure):
    _fields_ = [("blocks", C.c_uint32), ("warps", C.c_uint32), ("lanes", C.c_uint32), ("_pad", C.c_uint32),
                ("n_events", C.c_uint64), ("key", C.c_void_p), ("tidop", C.c_void_p), ("instr", C.c_void_p)]


class _Opts(C.Structure):
    _fields_ = [("inactive_opt", C.c_uint32), ("flags", C.c_uint32), ("stream", C.c_void_p),
                ("shard_index", C.c_uint32), ("shard_count", C.c_uint32)]


class _Result(C.Structure):
    _fields_ = [("n_reports", C.c_uint64), ("kind", C.POINTER(C.c_uint8)), ("prior", C.POINTER(C.c_uint32)),
                ("current", C.POINTER(C.c_uint32)), ("n_diags", C.c_uint64),
                ("diag_event", C.POINTER(C.c_uint32)), ("diag_code", C.POINTER(C.c_uint32)),
                ("diag_lock", C.POINTER(C.c_uint64)), ("order_key", C.POINTER(C.c_uint64))]


_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        lib = C.CDLL(os.environ.get("GPURACE_B200_LIB", N.LIB_PATH))
        lib.gw_analyze.argtypes = [C.POINTER(_View), C.POINTER(_Opts), C.POINTER(_Result)]
        lib.gw_analyze.restype = C.c_int
        lib.gw_result_free.argtypes = [C.POINTER(_Result)]
        lib.gw_last_error.restype = C.c_char_p
        _LIB = lib
    return _LIB


def run(trace, detector, *, order_matrix: bool = False, collect_stats: bool = False):
    """`gpurace.engine.run` for the gwcp / hb detectors on the B200 engine,
    returning gpurace's own RunResult (reports also appended to
    detector.reporter, diagnostics to detector.diagnostics, as the reference's
    detectors leave them)."""
    from gpurace.engine import RunResult
    from gpurace.report import Endpoint, RaceReport
    from gpurace.trace import Diagnostic, tid_str

    if order_matrix or collect_stats or detector.name not in ("gwcp", "hb"):
        raise NotImplementedError("the B200 backend runs the gwcp / hb detectors without order matrix / stats")
    soa = encode(trace)  # 16 B/event SoA (include/gwcp_b200.h)
    lib = _lib()
    n = len(soa)
    v = _View(soa.config.blocks, soa.config.warps, soa.config.lanes, 0, n,
              soa.key.ctypes.data if n else None, soa.tidop.ctypes.data if n else None,
              soa.instr.ctypes.data if n else None)
    inactive = int(getattr(detector, "_inactive_opt", getattr(detector, "inactive_opt", True)))
    r = _Result()
    rc = lib.gw_analyze(C.byref(v), C.byref(_Opts(inactive, GW_OPT_HB if detector.name == "hb" else 0, None, 0, 1)),
                        C.byref(r))
    if rc:
        raise RuntimeError(lib.gw_last_error().decode())
    try:
        evs = trace.events
        kinds = ("ww", "wr", "rw")  # report.py:13-15
        reports = []
        for i in range(r.n_reports):  # deduplicated, in report order (report.py:79-100)
            a, b = evs[r.prior[i]], evs[r.current[i]]
            reports.append(RaceReport(detector.name, kinds[r.kind[i]], b.loc, Endpoint.of(a), Endpoint.of(b),
                                      "first" if i == 0 else "post-race"))
        diags = []
        i = 0
        while i < r.n_diags:  # gwcp.py:178-182, :197-201, :323-330
            e, code = r.diag_event[i], r.diag_code[i]
            if code == 1:
                diags.append(Diagnostic(e, f"reentrant acquire of lock {r.diag_lock[i]:#x}"))
                i += 1
            elif code == 2:
                diags.append(Diagnostic(e, f"release of unheld lock {r.diag_lock[i]:#x}"))
                i += 1
            else:
                held = []
                while i < r.n_diags and r.diag_event[i] == e and r.diag_code[i] == 3:
                    held.append(f"{r.diag_lock[i]:#x}")
                    i += 1
                diags.append(Diagnostic(e, f"thread {tid_str(evs[e].tid)} exited holding lock(s) {', '.join(held)}"))
    finally:
        lib.gw_result_free(C.byref(r))
    detector.reporter.reports.extend(reports)
    detector.diagnostics.extend(diags)
    return RunResult(reports, diags, n_events=len(evs))


def install():
    """Route `gpurace.engine.run` (and so `gpurace check`) to the B200 engine
    for the gwcp / hb detectors; everything else keeps the Python path."""
    import gpurace.cli
    import gpurace.engine as E

    if getattr(E.run, "_b200", False):
        return
    py_run = E.run

    def run_b200(trace, detector, *, order_matrix=False, collect_stats=False):
        if detector.name in ("gwcp", "hb") and not order_matrix and not collect_stats:
            return run(trace, detector)
        return py_run(trace, detector, order_matrix=order_matrix, collect_stats=collect_stats)

    run_b200._b200 = True
    E.run = run_b200
    gpurace.cli.engine.run = run_b200
