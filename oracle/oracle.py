"""ctypes wrapper of oracle/build/libgwcp_oracle.so (test infrastructure only)."""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "build", "libgwcp_oracle.so")


class _Res(C.Structure):
    _fields_ = [
        ("n_reports", C.c_uint64),
        ("kind", C.POINTER(C.c_uint8)),
        ("prior_event", C.POINTER(C.c_uint32)),
        ("current_event", C.POINTER(C.c_uint32)),
        ("n_diags", C.c_uint64),
        ("diag_event", C.POINTER(C.c_uint32)),
        ("diag_code", C.POINTER(C.c_uint32)),
        ("diag_lock", C.POINTER(C.c_uint64)),
    ]


_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = C.CDLL(LIB)
        L.gwo_run.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p,
                              C.c_int, C.POINTER(_Res)]
        L.gwo_run.restype = C.c_int
        L.gwo_free.argtypes = [C.POINTER(_Res)]
        _lib = L
    return _lib


def run_soa(cfg, key, tidop, instr, inactive_opt=True, hb=False) -> dict:
    """Reference-equivalent result arrays for an SoA trace (same dict layout
    as paper_2111_12478_b200._native.analyze)."""
    L = lib()
    key = np.ascontiguousarray(key, np.uint64)
    tidop = np.ascontiguousarray(tidop, np.uint32)
    instr = np.ascontiguousarray(instr, np.uint32)
    r = _Res()
    n = len(tidop)
    rc = L.gwo_run(cfg[0], cfg[1], cfg[2], n, key.ctypes.data if n else None, tidop.ctypes.data if n else None,
                   instr.ctypes.data if n else None, (1 if inactive_opt else 0) | (2 if hb else 0), C.byref(r))
    if rc:
        raise RuntimeError(f"oracle failed ({rc})")
    try:
        def arr(p, k, dt):
            return np.ctypeslib.as_array(p, shape=(k,)).copy() if k else np.zeros(0, dt)

        nr, nd = int(r.n_reports), int(r.n_diags)
        return {
            "kind": arr(r.kind, nr, np.uint8),
            "prior": arr(r.prior_event, nr, np.uint32),
            "current": arr(r.current_event, nr, np.uint32),
            "diag_event": arr(r.diag_event, nd, np.uint32),
            "diag_code": arr(r.diag_code, nd, np.uint32),
            "diag_lock": arr(r.diag_lock, nd, np.uint64),
        }
    finally:
        L.gwo_free(C.byref(r))


def run_trace(tr, inactive_opt=True, hb=False) -> dict:
    """hb=True: the scoped happens-before detector (hb.py)."""
    return run_soa(tr.cfg_tuple, tr.key, tr.tidop, tr.instr, inactive_opt, hb)
