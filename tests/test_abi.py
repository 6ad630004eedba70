"""CPU checks of the C-ABI library: it loads and exports every declared symbol."""

import ctypes
import os
import re

from paper_2111_12478_b200 import _native as N
from paper_2111_12478_b200 import workloads as WL

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(REPO, "include", "gwcp_b200.h")).read()
    return sorted(set(re.findall(r"\b(gw_[a-z0-9_]+)\s*\(", hdr)))


def test_header_declares_the_bound_symbols():
    assert set(declared_symbols()) == set(N.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(N.LIB_PATH)
    for sym in declared_symbols():
        assert hasattr(lib, sym), sym


def test_parse_and_validate_are_host_side():
    # text ingest and validate_trace need no GPU
    cfg, key, tidop, instr = N.parse_text("config blocks=1 warps=1 lanes=2\nwacc 0 0 0x3 wr g:0x10,g:0x10\n")
    assert cfg == (1, 1, 2) and len(tidop) == 2
    assert tidop[1] & N.F_CONT and not tidop[0] & N.F_CONT
    assert N.validate(cfg, key, tidop, instr) == []


def test_no_cpu_analysis_path_without_a_gpu():
    import torch

    if torch.cuda.is_available():
        return
    cfg, key, tidop, instr = N.parse_text("config blocks=1 warps=1 lanes=1\n0.0.0 wr g:0x10\n")
    try:
        N.analyze(cfg, key, tidop, instr)
    except N.EngineError as e:
        assert e.code in (N.GW_E_CUDA, N.GW_E_NOMEM)
    else:  # pragma: no cover
        raise AssertionError("analysis must fail loudly without a CUDA device")


def test_result_views_own_the_library_buffers():
    """fetch() returns zero-copy numpy views of a gw_result; the buffers are
    freed (gw_result_free) only after the last view is gone."""
    import gc
    import weakref

    import numpy as np

    libc = ctypes.CDLL(None)
    libc.malloc.restype = ctypes.c_void_p
    libc.malloc.argtypes = [ctypes.c_size_t]
    n, nd = 5, 2
    r = N._Result()
    r.n_reports, r.n_diags = n, nd

    def buf(ctype, vals):
        p = libc.malloc(ctypes.sizeof(ctype) * max(len(vals), 1))
        arr = ctypes.cast(p, ctypes.POINTER(ctype))
        for i, v in enumerate(vals):
            arr[i] = v
        return arr

    r.kind = buf(ctypes.c_uint8, [0, 1, 2, 1, 0])
    r.prior_event = buf(ctypes.c_uint32, [1, 2, 3, 4, 5])
    r.current_event = buf(ctypes.c_uint32, [6, 7, 8, 9, 10])
    r.order_key = buf(ctypes.c_uint64, [11, 12, 13, 14, 2**63 + 1])
    r.diag_event = buf(ctypes.c_uint32, [3, 4])
    r.diag_code = buf(ctypes.c_uint32, [1, 2])
    r.diag_lock = buf(ctypes.c_uint64, [2**40, 7])
    res = N._take_result(N.lib(), r)
    assert res["kind"].tolist() == [0, 1, 2, 1, 0]
    assert res["prior"].tolist() == [1, 2, 3, 4, 5] and res["current"].tolist() == [6, 7, 8, 9, 10]
    assert res["order_key"].tolist() == [11, 12, 13, 14, 2**63 + 1]
    assert res["diag_lock"].dtype == np.uint64 and res["diag_lock"].tolist() == [2**40, 7]
    owner = res["kind"].base._owner
    alive = weakref.ref(owner)
    del owner
    keep = res["order_key"]
    del res
    gc.collect()
    assert alive() is not None and keep.tolist()[-1] == 2**63 + 1  # a live view keeps the buffers
    del keep
    gc.collect()
    assert alive() is None  # the last view gone: gw_result_free ran


def test_pack_columns_widths():
    """gw_trace_packed widths: the narrowest holding every value."""
    import numpy as np

    k, i = N.pack_columns(np.array([1, 2**32 - 1], np.uint64), np.array([0, 2**16 - 1], np.uint32))
    assert k.dtype == np.uint32 and i.dtype == np.uint16
    assert k.tolist() == [1, 2**32 - 1] and i.tolist() == [0, 2**16 - 1]
    k, i = N.pack_columns(np.array([2**32], np.uint64), np.array([2**16], np.uint32))
    assert k.dtype == np.uint64 and i.dtype == np.uint32


def _delta_decode(b, offs, base, n, w):
    """Restatement of the delta-varint layout (gw_trace_delta): per chunk, from
    its base, zigzag LEB128 deltas."""
    import numpy as np

    out = np.zeros(n, np.uint64)
    mask = (1 << w) - 1
    for k in range(len(offs) - 1):
        p, x = int(offs[k]), int(base[k]) if k < len(base) else 0
        for i in range(k * N.DELTA_CHUNK, min(n, (k + 1) * N.DELTA_CHUNK)):
            z = sh = 0
            while True:
                by = int(b[p])
                p += 1
                z |= (by & 0x7F) << sh
                sh += 7
                if not by & 0x80:
                    break
            x = (x + ((z >> 1) ^ (-(z & 1) & mask))) & mask
            out[i] = x
    return out


def test_delta_encoding_roundtrip():
    """gw_encode_delta (host, chunk-parallel) against the layout's restatement,
    with extreme values (wrap-around deltas, 64-bit shared keys)."""
    import numpy as np

    rng = np.random.default_rng(1)
    n = 3 * N.DELTA_CHUNK + 77
    key = rng.integers(0, 2**63, n, dtype=np.uint64)
    key[::5] = np.uint64(2**64 - 1)
    key[1::7] = 0
    tidop = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    instr = np.arange(n, dtype=np.uint32) * np.uint32(3)
    enc = N.encode_delta((1, 1, 1), key, tidop, instr)
    assert len(enc["offs"][0]) == 4 + 1 and int(enc["offs"][1][-1]) == len(enc["bytes"][1])
    assert np.array_equal(_delta_decode(enc["bytes"][0], enc["offs"][0], enc["base"][0], n, 64), key)
    assert np.array_equal(_delta_decode(enc["bytes"][1], enc["offs"][1], enc["base"][1], n, 32), tidop)
    assert np.array_equal(_delta_decode(enc["bytes"][2], enc["offs"][2], enc["base"][2], n, 32), instr)


def test_bitpacked_encoding_roundtrip():
    """gw_encode_bp (host, chunk-parallel) against the format's executable
    spec (decode_bp_host): warp-structured traces (every predictor mode),
    random columns (exceptions of every width), partial chunks / blocks."""
    import numpy as np

    rng = np.random.default_rng(11)
    cases = []
    tr = WL.c2_soa_prefix(70_000, **{k: v for k, v in WL.CONFIGS["c5"].items() if k != "gen"})
    cases.append((tr.key, tr.tidop, tr.instr))
    n = 9_001  # two full chunks + a partial one, a partial last block
    cases.append((rng.integers(0, 2**64, n, dtype=np.uint64), rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32),
                  rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)))
    mixed = np.cumsum(rng.integers(0, 8, 5_000, dtype=np.uint64) * np.uint64(4)) + np.uint64(2**63)
    mixed[::97] = rng.integers(0, 2**64, len(mixed[::97]), dtype=np.uint64)  # rare wide jumps -> exceptions
    cases.append((mixed, (np.arange(5_000) % 4096).astype(np.uint32), np.zeros(5_000, np.uint32)))
    cases.append((np.zeros(1, np.uint64), np.ones(1, np.uint32), np.full(1, 2**32 - 1, np.uint32)))
    for key, tidop, instr in cases:
        enc = N.encode_bp((4, 8, 32), key, tidop, instr)
        assert all(len(b) % 4 == 0 for b in enc["bytes"]) and all(int(o[-1]) == len(b) for o, b in zip(enc["offs"], enc["bytes"]))
        k, t, i = N.decode_bp_host(enc)
        assert np.array_equal(k, key) and np.array_equal(t, tidop) and np.array_equal(i, instr)
    enc = N.encode_bp((4, 8, 32), *cases[0])
    assert sum(len(b) for b in enc["bytes"]) < 0.5 * len(cases[0][1])  # C5 recipe: < 0.5 B/event
