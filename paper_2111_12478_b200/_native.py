"""ctypes binding of libgwcp_b200.so (include/gwcp_b200.h).

The analysis has no CPU path: if the shared library is missing or fails to
load, every entry point raises ``NativeUnavailable`` -- there is no fallback.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GWCP_B200_LIB", os.path.join(_HERE, "libgwcp_b200.so"))

GW_OK, GW_E_PARSE, GW_E_UNSUPPORTED, GW_E_CUDA, GW_E_NOMEM, GW_E_ARG = range(6)

# SoA encoding (gwcp_b200.h)
K_READ, K_WRITE, K_ACQUIRE, K_RELEASE, K_BARRIER, K_FENCE, K_END = range(7)
OP_SHIFT = 24
TID_MASK = 0x00FFFFFF
F_ATOMIC = 1 << 27
F_DEVICE = 1 << 28
F_WARPBAR = 1 << 29
F_CONT = 1 << 30
SHARED_BIT = 1 << 63
OPT_EAGER = 1
OPT_PROFILE = 2
OPT_HB = 4  # scoped happens-before detector (hb.py)


class NativeUnavailable(RuntimeError):
    pass


class EngineError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


class _Config(C.Structure):
    _fields_ = [("blocks", C.c_uint32), ("warps", C.c_uint32), ("lanes", C.c_uint32), ("_pad", C.c_uint32)]


class _Trace(C.Structure):
    _fields_ = [
        ("cfg", _Config),
        ("n_events", C.c_uint64),
        ("key", C.POINTER(C.c_uint64)),
        ("tidop", C.POINTER(C.c_uint32)),
        ("instr", C.POINTER(C.c_uint32)),
    ]


class _View(C.Structure):
    _fields_ = [
        ("cfg", _Config),
        ("n_events", C.c_uint64),
        ("key", C.c_void_p),
        ("tidop", C.c_void_p),
        ("instr", C.c_void_p),
    ]


class _Packed(C.Structure):
    _fields_ = [
        ("cfg", _Config),
        ("n_events", C.c_uint64),
        ("key_bytes", C.c_uint32),
        ("instr_bytes", C.c_uint32),
        ("key", C.c_void_p),
        ("tidop", C.c_void_p),
        ("instr", C.c_void_p),
    ]


DELTA_CHUNK = 4096


class _Delta(C.Structure):
    _fields_ = [("cfg", _Config), ("n_events", C.c_uint64), ("chunk", C.c_uint32), ("_pad", C.c_uint32),
                ("n_chunks", C.c_uint64), ("bytes", C.c_void_p * 3), ("nbytes", C.c_uint64 * 3),
                ("offs", C.c_void_p * 3), ("base", C.c_void_p * 3)]


class _BP(C.Structure):
    _fields_ = [("cfg", _Config), ("n_events", C.c_uint64), ("chunk", C.c_uint32), ("key_bits", C.c_uint32),
                ("n_chunks", C.c_uint64), ("bytes", C.c_void_p * 3), ("nbytes", C.c_uint64 * 3),
                ("offs", C.c_void_p * 3), ("base", C.c_void_p * 3), ("dbase", C.c_void_p * 3)]


class XsStats(C.Structure):
    _fields_ = [(f, C.c_uint64) for f in ("n_acc", "n_write", "n_acq", "n_rel", "n_end", "n_bar", "key_or",
                                          "key_and", "n_long", "n_wbar")]


class _Opts(C.Structure):
    _fields_ = [("inactive_opt", C.c_uint32), ("flags", C.c_uint32), ("stream", C.c_void_p),
                ("shard_index", C.c_uint32), ("shard_count", C.c_uint32)]


class _Result(C.Structure):
    _fields_ = [
        ("n_reports", C.c_uint64),
        ("kind", C.POINTER(C.c_uint8)),
        ("prior_event", C.POINTER(C.c_uint32)),
        ("current_event", C.POINTER(C.c_uint32)),
        ("n_diags", C.c_uint64),
        ("diag_event", C.POINTER(C.c_uint32)),
        ("diag_code", C.POINTER(C.c_uint32)),
        ("diag_lock", C.POINTER(C.c_uint64)),
        ("order_key", C.POINTER(C.c_uint64)),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("ms_total", C.c_float),
        ("ms_prep", C.c_float),
        ("ms_walker", C.c_float),
        ("ms_sort", C.c_float),
        ("ms_check", C.c_float),
        ("ms_final", C.c_float),
        ("n_accesses", C.c_uint64),
        ("n_candidates", C.c_uint64),
        ("n_sync", C.c_uint64),
        ("arena_words", C.c_uint64),
        ("walker_ctas", C.c_uint32),
        ("sort_bits", C.c_uint32),
        ("n_sorted", C.c_uint64),
    ]


EXPORTS = (
    "gw_parse_text",
    "gw_trace_free",
    "gw_validate",
    "gw_free",
    "gw_analyze",
    "gw_result_free",
    "gw_last_error",
    "gw_ctx_create",
    "gw_ctx_destroy",
    "gw_ctx_analyze_device",
    "gw_ctx_analyze_host",
    "gw_ctx_analyze_host_packed",
    "gw_ctx_validate",
    "gw_ctx_infer_locks",
    "gw_encode_delta",
    "gw_delta_free",
    "gw_ctx_analyze_host_delta",
    "gw_encode_bp",
    "gw_bp_free",
    "gw_ctx_analyze_host_bp",
    "gw_xs_prep",
    "gw_xs_hard",
    "gw_xs_partition",
    "gw_xs_check",
    "gw_xs_fetch",
    "gw_xs_lookup",
    "gw_ctx_fetch",
    "gw_ctx_stats",
    "gw_ctx_launches",
    "gw_gen_c2_device",
    "gw_gen_c4_device",
    "gw_gen_c3_device",
    "gw_ctx_kernel_times",
    "gw_save_soa",
    "gw_load_soa",
)

_lib = None
_lock = threading.Lock()


def lib():
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(
                f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        try:
            L = C.CDLL(LIB_PATH)
        except OSError as e:  # pragma: no cover - depends on the box
            raise NativeUnavailable(f"cannot load {LIB_PATH}: {e}") from e
        L.gw_parse_text.argtypes = [C.c_char_p, C.c_uint64, C.POINTER(_Trace), C.POINTER(C.c_int64)]
        L.gw_parse_text.restype = C.c_int
        L.gw_trace_free.argtypes = [C.POINTER(_Trace)]
        L.gw_validate.argtypes = [
            C.POINTER(_View),
            C.POINTER(C.c_uint64),
            C.POINTER(C.POINTER(C.c_uint32)),
            C.POINTER(C.POINTER(C.c_uint32)),
            C.POINTER(C.POINTER(C.c_uint64)),
            C.POINTER(C.POINTER(C.c_uint64)),
        ]
        L.gw_validate.restype = C.c_int
        L.gw_free.argtypes = [C.c_void_p]
        L.gw_analyze.argtypes = [C.POINTER(_View), C.POINTER(_Opts), C.POINTER(_Result)]
        L.gw_analyze.restype = C.c_int
        L.gw_result_free.argtypes = [C.POINTER(_Result)]
        L.gw_last_error.restype = C.c_char_p
        L.gw_ctx_create.argtypes = [C.c_int]
        L.gw_ctx_create.restype = C.c_void_p
        L.gw_ctx_destroy.argtypes = [C.c_void_p]
        L.gw_ctx_analyze_device.argtypes = [C.c_void_p, C.POINTER(_View), C.POINTER(_Opts)]
        L.gw_ctx_analyze_device.restype = C.c_int
        L.gw_ctx_analyze_host.argtypes = [C.c_void_p, C.POINTER(_View), C.POINTER(_Opts)]
        L.gw_ctx_analyze_host.restype = C.c_int
        L.gw_ctx_analyze_host_packed.argtypes = [C.c_void_p, C.POINTER(_Packed), C.POINTER(_Opts)]
        L.gw_ctx_analyze_host_packed.restype = C.c_int
        L.gw_ctx_validate.argtypes = [C.c_void_p, C.POINTER(_View), C.POINTER(C.c_uint64),
                                      C.POINTER(C.POINTER(C.c_uint32)), C.POINTER(C.POINTER(C.c_uint32)),
                                      C.POINTER(C.POINTER(C.c_uint64)), C.POINTER(C.POINTER(C.c_uint64))]
        L.gw_ctx_validate.restype = C.c_int
        L.gw_ctx_infer_locks.argtypes = [C.c_void_p, C.POINTER(_View), C.POINTER(_Trace), C.POINTER(C.c_uint64),
                                         C.POINTER(C.POINTER(C.c_uint32)), C.POINTER(C.POINTER(C.c_uint64)),
                                         C.POINTER(C.POINTER(C.c_uint32))]
        L.gw_ctx_infer_locks.restype = C.c_int
        P32, P64, VP = C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), C.c_void_p
        L.gw_xs_prep.argtypes = [VP, C.POINTER(_View), C.c_uint32, VP, C.POINTER(XsStats)]
        L.gw_xs_hard.argtypes = [VP, VP, VP, VP, VP, VP, P64]
        L.gw_xs_partition.argtypes = [VP, C.POINTER(XsStats), C.c_uint32, VP, VP, VP, VP, P64]
        L.gw_xs_check.argtypes = [VP, C.POINTER(XsStats), C.c_uint32, C.c_uint64, VP, VP, VP, VP, C.c_uint64,
                                  VP, VP, VP, VP, C.c_uint64, P64]
        L.gw_xs_fetch.argtypes = [VP, VP, VP, VP, VP, VP]
        L.gw_xs_lookup.argtypes = [VP, VP, C.c_uint64, VP, VP]
        for f in ("gw_xs_prep", "gw_xs_hard", "gw_xs_partition", "gw_xs_check", "gw_xs_fetch", "gw_xs_lookup"):
            getattr(L, f).restype = C.c_int
        L.gw_encode_delta.argtypes = [C.POINTER(_View), C.POINTER(_Delta)]
        L.gw_encode_delta.restype = C.c_int
        L.gw_delta_free.argtypes = [C.POINTER(_Delta)]
        L.gw_ctx_analyze_host_delta.argtypes = [C.c_void_p, C.POINTER(_Delta), C.POINTER(_Opts)]
        L.gw_ctx_analyze_host_delta.restype = C.c_int
        L.gw_encode_bp.argtypes = [C.POINTER(_View), C.POINTER(_BP)]
        L.gw_encode_bp.restype = C.c_int
        L.gw_bp_free.argtypes = [C.POINTER(_BP)]
        L.gw_ctx_analyze_host_bp.argtypes = [C.c_void_p, C.POINTER(_BP), C.POINTER(_Opts)]
        L.gw_ctx_analyze_host_bp.restype = C.c_int
        L.gw_ctx_fetch.argtypes = [C.c_void_p, C.POINTER(_Result)]
        L.gw_ctx_fetch.restype = C.c_int
        L.gw_ctx_stats.argtypes = [C.c_void_p, C.POINTER(Stats)]
        L.gw_ctx_stats.restype = C.c_int
        L.gw_ctx_launches.argtypes = [C.c_void_p]
        L.gw_ctx_launches.restype = C.c_uint32
        L.gw_gen_c2_device.argtypes = [C.c_uint32] * 5 + [C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p,
                                                          C.c_void_p, C.c_void_p]
        L.gw_gen_c2_device.restype = C.c_int
        L.gw_gen_c4_device.argtypes = [C.c_uint32] * 3 + [C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p,
                                                          C.c_void_p, C.c_void_p]
        L.gw_gen_c4_device.restype = C.c_int
        L.gw_gen_c3_device.argtypes = [C.c_uint32] * 7 + [C.c_uint64] + [C.c_void_p] * 5
        L.gw_gen_c3_device.restype = C.c_int
        L.gw_ctx_kernel_times.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.POINTER(C.c_float),
                                          C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.gw_ctx_kernel_times.restype = C.c_int
        L.gw_save_soa.argtypes = [C.c_char_p, C.POINTER(_View)]
        L.gw_save_soa.restype = C.c_int
        L.gw_load_soa.argtypes = [C.c_char_p, C.POINTER(_Trace)]
        L.gw_load_soa.restype = C.c_int
        _lib = L
        return L


def last_error() -> str:
    return lib().gw_last_error().decode("utf-8", "replace")


def _check(rc: int) -> None:
    if rc != GW_OK:
        raise EngineError(rc, last_error())


def parse_text(text: str | bytes):
    """Text trace -> (cfg tuple, key u64[], tidop u32[], instr u32[]).

    Raises EngineError(GW_E_PARSE, "line N: msg") on a parse error; the
    error line is attached as ``.line``.
    """
    L = lib()
    data = text.encode("utf-8") if isinstance(text, str) else bytes(text)
    t = _Trace()
    line = C.c_int64(-1)
    rc = L.gw_parse_text(data, len(data), C.byref(t), C.byref(line))
    if rc != GW_OK:
        err = EngineError(rc, last_error())
        err.line = int(line.value)  # type: ignore[attr-defined]
        raise err
    return _take_trace(L, t)


def _take_trace(L, t):
    try:
        n = int(t.n_events)
        key = np.ctypeslib.as_array(t.key, shape=(max(n, 1),))[:n].copy()
        tidop = np.ctypeslib.as_array(t.tidop, shape=(max(n, 1),))[:n].copy()
        instr = np.ctypeslib.as_array(t.instr, shape=(max(n, 1),))[:n].copy()
        cfg = (int(t.cfg.blocks), int(t.cfg.warps), int(t.cfg.lanes))
    finally:
        L.gw_trace_free(C.byref(t))
    return cfg, key, tidop, instr


def save_soa(path: str, cfg, key, tidop, instr) -> None:
    """Write the binary SoA trace file (include/gwcp_b200.h, gw_save_soa)."""
    key = np.ascontiguousarray(key, np.uint64)
    tidop = np.ascontiguousarray(tidop, np.uint32)
    instr = np.ascontiguousarray(instr, np.uint32)
    _check(lib().gw_save_soa(os.fsencode(path), C.byref(_view(cfg, key, tidop, instr))))


def load_soa(path: str):
    """Binary SoA trace file -> (cfg tuple, key, tidop, instr) (gw_load_soa)."""
    L = lib()
    t = _Trace()
    _check(L.gw_load_soa(os.fsencode(path), C.byref(t)))
    return _take_trace(L, t)


def _view(cfg, key, tidop, instr) -> _View:
    v = _View()
    v.cfg.blocks, v.cfg.warps, v.cfg.lanes = cfg
    v.n_events = len(tidop)
    v.key = key.ctypes.data if len(key) else None
    v.tidop = tidop.ctypes.data if len(tidop) else None
    v.instr = instr.ctypes.data if len(instr) else None
    return v


def validate(cfg, key, tidop, instr, ctx=None):
    """validate_trace diagnostics (event, code, a, b): on the GPU through a
    context (gw_ctx_validate), or the host pass (gw_validate) when ctx is None."""
    L = lib()
    v = _view(cfg, key, tidop, instr)
    n = C.c_uint64(0)
    pe, pc = C.POINTER(C.c_uint32)(), C.POINTER(C.c_uint32)()
    pa, pb = C.POINTER(C.c_uint64)(), C.POINTER(C.c_uint64)()
    if ctx is not None:
        _check(L.gw_ctx_validate(ctx._c, C.byref(v), C.byref(n), C.byref(pe), C.byref(pc), C.byref(pa),
                                 C.byref(pb)))
    else:
        _check(L.gw_validate(C.byref(v), C.byref(n), C.byref(pe), C.byref(pc), C.byref(pa), C.byref(pb)))
    k = int(n.value)
    try:
        out = [(int(pe[i]), int(pc[i]), int(pa[i]), int(pb[i])) for i in range(k)]
    finally:
        for p in (pe, pc, pa, pb):
            L.gw_free(C.cast(p, C.c_void_p))
    return out


def infer_locks(ctx, cfg, key, tidop, instr):
    """infer_locks on the GPU (gw_ctx_infer_locks): ((cfg, key, tidop, instr)
    of the rewritten trace, [(event, lock, tid)] of the uninferred releases)."""
    L = lib()
    v = _view(cfg, key, tidop, instr)
    t = _Trace()
    n = C.c_uint64(0)
    pe, pl, pt = C.POINTER(C.c_uint32)(), C.POINTER(C.c_uint64)(), C.POINTER(C.c_uint32)()
    _check(L.gw_ctx_infer_locks(ctx._c, C.byref(v), C.byref(t), C.byref(n), C.byref(pe), C.byref(pl), C.byref(pt)))
    k = int(n.value)
    try:
        diags = [(int(pe[i]), int(pl[i]), int(pt[i])) for i in range(k)]
    finally:
        for p in (pe, pl, pt):
            L.gw_free(C.cast(p, C.c_void_p))
    return _take_trace(L, t), diags


class _ResultOwner:
    """Frees a gw_result when the last array viewing it is collected."""

    def __init__(self, L, r: _Result):
        self._L, self._r = L, r

    def __del__(self):
        try:
            self._L.gw_result_free(C.byref(self._r))
        except Exception:  # interpreter shutdown
            pass


def _take_result(L, r: _Result):
    """Zero-copy: the result arrays are numpy views of the library-owned
    buffers (freed with gw_result_free once every view is gone), so a large
    report list is copied once (mapped host staging -> result) rather than
    twice."""
    owner = _ResultOwner(L, r)
    n = int(r.n_reports)
    nd = int(r.n_diags)

    def arr(p, count, dt):
        if not count:
            return np.empty(0, dtype=dt)
        nbytes = count * np.dtype(dt).itemsize
        buf = (C.c_char * nbytes).from_address(C.cast(p, C.c_void_p).value)
        buf._owner = owner
        return np.frombuffer(buf, dtype=dt)

    return {
        "kind": arr(r.kind, n, np.uint8),
        "prior": arr(r.prior_event, n, np.uint32),
        "current": arr(r.current_event, n, np.uint32),
        "diag_event": arr(r.diag_event, nd, np.uint32),
        "diag_code": arr(r.diag_code, nd, np.uint32),
        "diag_lock": arr(r.diag_lock, nd, np.uint64),
        "order_key": arr(r.order_key, n, np.uint64),
    }


class Context:
    """A device context: buffers persist across analyses (bench, servers)."""

    def __init__(self, device: int = 0):
        self._L = lib()
        self._c = self._L.gw_ctx_create(int(device))
        if not self._c:
            raise EngineError(GW_E_CUDA, last_error())

    def close(self) -> None:
        if self._c:
            self._L.gw_ctx_destroy(self._c)
            self._c = None

    def __del__(self):  # pragma: no cover - interpreter teardown order
        try:
            self.close()
        except Exception:
            pass

    def analyze_host(self, cfg, key, tidop, instr, *, inactive_opt=True, stream=None, eager=False,
                     shard=(0, 1), hb=False) -> None:
        """hb=True: the scoped happens-before detector (gpurace --detector hb)."""
        v = _view(cfg, key, tidop, instr)
        flags = (OPT_EAGER if eager else 0) | (OPT_HB if hb else 0)
        o = _Opts(1 if inactive_opt else 0, flags, stream, shard[0], shard[1])
        _check(self._L.gw_ctx_analyze_host(self._c, C.byref(v), C.byref(o)))

    def analyze_host_packed(self, cfg, key, tidop, instr, *, inactive_opt=True, stream=None, eager=False,
                            shard=(0, 1), hb=False) -> None:
        """Packed host trace (pack_columns): key uint32|uint64, instr uint16|uint32;
        uploaded in chunks and widened on the device (gw_ctx_analyze_host_packed)."""
        key, tidop, instr = np.asarray(key), np.asarray(tidop, np.uint32), np.asarray(instr)
        if key.dtype not in (np.uint32, np.uint64) or instr.dtype not in (np.uint16, np.uint32):
            raise TypeError("packed trace: key uint32/uint64, instr uint16/uint32")
        for a in (key, tidop, instr):
            if not a.flags.c_contiguous:
                raise ValueError("packed trace columns must be contiguous")
        p = _Packed()
        p.cfg.blocks, p.cfg.warps, p.cfg.lanes = cfg
        p.n_events = len(tidop)
        p.key_bytes, p.instr_bytes = key.dtype.itemsize, instr.dtype.itemsize
        p.key, p.tidop, p.instr = key.ctypes.data, tidop.ctypes.data, instr.ctypes.data
        flags = (OPT_EAGER if eager else 0) | (OPT_HB if hb else 0)
        o = _Opts(1 if inactive_opt else 0, flags, stream, shard[0], shard[1])
        _check(self._L.gw_ctx_analyze_host_packed(self._c, C.byref(p), C.byref(o)))

    def analyze_host_delta(self, enc: dict, *, inactive_opt=True, stream=None, eager=False, hb=False) -> None:
        """Delta-varint host trace (encode_delta; the byte streams may be any
        host arrays, pinned for full PCIe speed): chunked upload overlapped
        with on-device decoding (gw_ctx_analyze_host_delta)."""
        d = _Delta()
        d.cfg.blocks, d.cfg.warps, d.cfg.lanes = enc["cfg"]
        d.n_events = enc["n"]
        d.chunk = DELTA_CHUNK
        d.n_chunks = (enc["n"] + DELTA_CHUNK - 1) // DELTA_CHUNK
        for c in range(3):
            b, o, s_ = enc["bytes"][c], enc["offs"][c], enc["base"][c]
            d.bytes[c] = b.ctypes.data if len(b) else None
            d.nbytes[c] = len(b)
            d.offs[c] = o.ctypes.data
            d.base[c] = s_.ctypes.data if len(s_) else None
        flags = (OPT_EAGER if eager else 0) | (OPT_HB if hb else 0)
        o_ = _Opts(1 if inactive_opt else 0, flags, stream, 0, 1)
        _check(self._L.gw_ctx_analyze_host_delta(self._c, C.byref(d), C.byref(o_)))

    def analyze_host_bp(self, enc: dict, *, inactive_opt=True, stream=None, eager=False, hb=False) -> None:
        """Bit-packed host trace (encode_bp, GWSOA v4): sliced upload
        overlapped with on-device decoding (gw_ctx_analyze_host_bp)."""
        d = _BP()
        d.cfg.blocks, d.cfg.warps, d.cfg.lanes = enc["cfg"]
        d.n_events = enc["n"]
        d.chunk = DELTA_CHUNK
        d.key_bits = enc["key_bits"]
        d.n_chunks = (enc["n"] + DELTA_CHUNK - 1) // DELTA_CHUNK
        for c in range(3):
            b, o, s_, ds = enc["bytes"][c], enc["offs"][c], enc["base"][c], enc["dbase"][c]
            d.bytes[c] = b.ctypes.data if len(b) else None
            d.nbytes[c] = len(b)
            d.offs[c] = o.ctypes.data
            d.base[c] = s_.ctypes.data if len(s_) else None
            d.dbase[c] = ds.ctypes.data if len(ds) else None
        flags = (OPT_EAGER if eager else 0) | (OPT_HB if hb else 0)
        o_ = _Opts(1 if inactive_opt else 0, flags, stream, 0, 1)
        _check(self._L.gw_ctx_analyze_host_bp(self._c, C.byref(d), C.byref(o_)))

    def analyze_device(self, cfg, n, key_ptr, tidop_ptr, instr_ptr, *, inactive_opt=True, stream=None,
                       eager=False, shard=(0, 1), profile=False, hb=False) -> None:
        """shard=(index, count): report only races on location-key range `index`
        of `count` (address sharding; see include/gwcp_b200.h gw_opts)."""
        v = _View()
        v.cfg.blocks, v.cfg.warps, v.cfg.lanes = cfg
        v.n_events = n
        v.key, v.tidop, v.instr = key_ptr, tidop_ptr, instr_ptr
        flags = (OPT_EAGER if eager else 0) | (OPT_PROFILE if profile else 0) | (OPT_HB if hb else 0)
        o = _Opts(1 if inactive_opt else 0, flags, stream, shard[0], shard[1])
        _check(self._L.gw_ctx_analyze_device(self._c, C.byref(v), C.byref(o)))

    # ---- exchange mode (multi-GPU data plane; shard.analyze_exchange drives it) ----
    def xs_prep(self, cfg, n, key_ptr, tidop_ptr, instr_ptr, base, stream=None) -> XsStats:
        v = _View()
        v.cfg.blocks, v.cfg.warps, v.cfg.lanes = cfg
        v.n_events = n
        v.key, v.tidop, v.instr = key_ptr, tidop_ptr, instr_ptr
        out = XsStats()
        _check(self._L.gw_xs_prep(self._c, C.byref(v), base, stream, C.byref(out)))
        return out

    def xs_hard(self, ev_ptr, tidop_ptr, instr_ptr, key_ptr, stream=None) -> int:
        n = C.c_uint64(0)
        _check(self._L.gw_xs_hard(self._c, stream, ev_ptr, tidop_ptr, instr_ptr, key_ptr, C.byref(n)))
        return int(n.value)

    def xs_partition(self, glob: XsStats, shards, h_ptr, v_ptr, t_ptr, stream=None) -> list:
        counts = (C.c_uint64 * shards)()
        _check(self._L.gw_xs_partition(self._c, C.byref(glob), shards, stream, h_ptr, v_ptr, t_ptr, counts))
        return [int(x) for x in counts]

    def xs_check(self, glob: XsStats, shards, n_total, recv_ptrs, n_recv, hard_ptrs, n_hard, stream=None) -> int:
        n = C.c_uint64(0)
        _check(self._L.gw_xs_check(self._c, C.byref(glob), shards, n_total, stream, *recv_ptrs, n_recv, *hard_ptrs,
                                   n_hard, C.byref(n)))
        return int(n.value)

    def xs_fetch(self, n) -> dict:
        out = {"order_key": np.zeros(n, np.uint64), "loc": np.zeros(n, np.uint64), "prior": np.zeros(n, np.uint32),
               "current": np.zeros(n, np.uint32), "kind": np.zeros(n, np.uint32)}
        _check(self._L.gw_xs_fetch(self._c, *(out[k].ctypes.data for k in ("order_key", "loc", "prior", "current",
                                                                             "kind"))))
        return out

    def xs_lookup(self, ev) -> tuple:
        ev = np.ascontiguousarray(ev, np.uint32)
        to = np.zeros(len(ev), np.uint32)
        ins = np.zeros(len(ev), np.uint32)
        _check(self._L.gw_xs_lookup(self._c, ev.ctypes.data, len(ev), to.ctypes.data, ins.ctypes.data))
        return to, ins

    def fetch(self):
        r = _Result()
        _check(self._L.gw_ctx_fetch(self._c, C.byref(r)))
        return _take_result(self._L, r)

    def stats(self) -> Stats:
        s = Stats()
        _check(self._L.gw_ctx_stats(self._c, C.byref(s)))
        return s

    def launches(self) -> int:
        return int(self._L.gw_ctx_launches(self._c))

    def kernel_times(self) -> dict:
        """{kernel: (total ms, launches)} of the last analysis run with profile=True."""
        cap = 256
        names = (C.c_char * 64 * cap)()
        ms = (C.c_float * cap)()
        cnt = (C.c_uint32 * cap)()
        n = C.c_uint32(0)
        _check(self._L.gw_ctx_kernel_times(self._c, cap, names, ms, cnt, C.byref(n)))
        return {names[i].value.decode(): (float(ms[i]), int(cnt[i])) for i in range(n.value)}


def encode_delta(cfg, key, tidop, instr) -> dict:
    """The delta-varint form of a host SoA (gw_encode_delta, GWSOA v3):
    {"cfg", "n", "bytes": [key, tidop, instr byte streams], "offs": [...],
    "base": [...]} as numpy arrays (copied out of the library's buffers)."""
    L = lib()
    key = np.ascontiguousarray(key, np.uint64)
    tidop = np.ascontiguousarray(tidop, np.uint32)
    instr = np.ascontiguousarray(instr, np.uint32)
    v = _view(cfg, key, tidop, instr)
    d = _Delta()
    _check(L.gw_encode_delta(C.byref(v), C.byref(d)))
    try:
        k = int(d.n_chunks)

        def take(p, count, dt):
            if count == 0:
                return np.zeros(0, dt)
            return np.ctypeslib.as_array(C.cast(p, C.POINTER(np.ctypeslib.as_ctypes_type(dt))), shape=(count,)).copy()

        return {"cfg": tuple(cfg), "n": len(tidop),
                "bytes": [take(d.bytes[c], int(d.nbytes[c]), np.uint8) for c in range(3)],
                "offs": [take(d.offs[c], k + 1, np.uint64) for c in range(3)],
                "base": [take(d.base[c], k, np.uint64) for c in range(3)]}
    finally:
        L.gw_delta_free(C.byref(d))


def encode_bp(cfg, key, tidop, instr) -> dict:
    """The bit-packed form of a host SoA (gw_encode_bp, GWSOA v4): as
    encode_delta, plus "dbase" (each chunk's first difference before it)."""
    L = lib()
    key = np.ascontiguousarray(key, np.uint64)
    tidop = np.ascontiguousarray(tidop, np.uint32)
    instr = np.ascontiguousarray(instr, np.uint32)
    v = _view(cfg, key, tidop, instr)
    d = _BP()
    _check(L.gw_encode_bp(C.byref(v), C.byref(d)))
    try:
        k = int(d.n_chunks)

        def take(p, count, dt):
            if count == 0:
                return np.zeros(0, dt)
            return np.ctypeslib.as_array(C.cast(p, C.POINTER(np.ctypeslib.as_ctypes_type(dt))), shape=(count,)).copy()

        return {"cfg": tuple(cfg), "n": len(tidop),
                "bytes": [take(d.bytes[c], int(d.nbytes[c]), np.uint8) for c in range(3)],
                "offs": [take(d.offs[c], k + 1, np.uint64) for c in range(3)],
                "base": [take(d.base[c], k, np.uint64) for c in range(3)],
                "dbase": [take(d.dbase[c], k, np.uint64) for c in range(3)],
                "key_bits": int(d.key_bits)}
    finally:
        L.gw_bp_free(C.byref(d))


def decode_bp_host(enc: dict) -> tuple:
    """Host (Python) decoder of encode_bp's format -- test infrastructure,
    the format's executable spec (include/gwcp_b200.h); the product decodes
    on the device (k_bp_decode)."""
    n = enc["n"]
    cols = []
    for c, (T, w) in enumerate(((np.uint64, enc.get("key_bits", 64)), (np.uint32, 32), (np.uint32, 32))):
        M = (1 << w) - 1
        out = np.zeros(n, T)
        byts, offs = enc["bytes"][c], enc["offs"][c]
        for k in range(len(offs) - 1):
            lo = k * DELTA_CHUNK
            cnt = min(DELTA_CHUNK, n - lo)
            nb = (cnt + 31) // 32
            ch = byts[int(offs[k]):int(offs[k + 1])].tobytes()
            hdr = ch[:nb]
            nexc, xw, pos = [], [], nb
            for h in hdr:
                if h & 0x20:
                    nexc.append(ch[pos]); xw.append(ch[pos + 1]); pos += 2
                else:
                    nexc.append(0); xw.append(0)
            pos = (pos + 3) & ~3
            packed = []
            for h in hdr:
                b = h & 31
                packed.append(int.from_bytes(ch[pos:pos + 4 * b], "little")); pos += 4 * b
            E = sum(nexc)
            idx = ch[pos:pos + E]; pos += E
            x, d = int(enc["base"][c][k]), int(enc["dbase"][c][k])
            hist = [[0] * 32, [0] * 32]  # d of the blocks one and two back
            e = 0
            for kb, h in enumerate(hdr):
                b, mode = h & 31, h >> 6
                z = [(packed[kb] >> (l * b)) & ((1 << b) - 1) for l in range(32)]
                for _ in range(nexc[kb]):
                    z[idx[e]] = int.from_bytes(ch[pos:pos + xw[kb]], "little"); pos += xw[kb]; e += 1
                dcur = []
                for l in range(32):
                    r = (z[l] >> 1) ^ (-(z[l] & 1) & M)
                    pred = d if mode == 0 else hist[0][l] if mode == 1 else hist[1][l] if mode == 2 else 0
                    d = (pred + r) & M
                    dcur.append(d)
                    x = (x + d) & M
                    if 32 * kb + l < cnt:
                        out[lo + 32 * kb + l] = x
                hist = [dcur, hist[0]]
        cols.append(out)
    return tuple(cols)


def pack_columns(key, instr, tidop=None):
    """The narrowest packed widths holding every value (gw_trace_packed):
    key as uint32 when every non-barrier key < 2^32 (barrier keys are implied
    by their tidop and restored on the device; tidop=None: all keys count),
    instr as uint16 when < 2^16."""
    key = np.asarray(key, np.uint64)
    instr = np.asarray(instr, np.uint32)
    ks = key
    if tidop is not None and len(key):
        ks = key[((np.asarray(tidop, np.uint32) >> np.uint32(OP_SHIFT)) & np.uint32(7)) != K_BARRIER]
    k = key.astype(np.uint32) if len(ks) == 0 or int(ks.max()) < (1 << 32) else key
    i = instr.astype(np.uint16) if len(instr) == 0 or int(instr.max()) < (1 << 16) else instr
    return k, i


_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def analyze(cfg, key, tidop, instr, *, inactive_opt=True, hb=False):
    """Host SoA in -> report / diagnostic arrays out (GPU; no CPU path)."""
    ctx = default_context()
    ctx.analyze_host(cfg, key, tidop, instr, inactive_opt=inactive_opt, hb=hb)
    return ctx.fetch()


def gen_c2_device(key_ptr, tidop_ptr, instr_ptr, *, blocks, warps, lanes, phases, records, words_per_block, seed,
                  stream=None) -> int:
    """Write the C2/C5 recipe trace into device buffers; returns the event count."""
    _check(lib().gw_gen_c2_device(blocks, warps, lanes, phases, records, words_per_block, seed, key_ptr, tidop_ptr,
                                  instr_ptr, stream))
    return phases * (records * blocks * warps * lanes + blocks)


def c4_events(blocks, warps, iters) -> int:
    g = blocks * warps
    return iters * g * 32 + (iters // 4) * g + (iters // 64) * blocks


def gen_c4_device(key_ptr, tidop_ptr, instr_ptr, *, blocks, warps, iters, words_per_block, seed, stream=None) -> int:
    """Write the C4 recipe trace (workloads.c4_text, lanes=32) into device buffers."""
    _check(lib().gw_gen_c4_device(blocks, warps, iters, words_per_block, seed, key_ptr, tidop_ptr, instr_ptr, stream))
    return c4_events(blocks, warps, iters)


def gen_c3_device(key_ptr, tidop_ptr, instr_ptr, offsets_ptr, *, blocks, warps, lanes, iters, locks, region,
                  private, seed, stream=None) -> None:
    """Write the C3 recipe trace (workloads.c3_text) into device buffers, given
    the device copy of workloads.c3_group_offsets(...)[:-1]."""
    _check(lib().gw_gen_c3_device(blocks, warps, lanes, iters, locks, region, private, seed, offsets_ptr, key_ptr,
                                  tidop_ptr, instr_ptr, stream))
