"""CPU checks of the C-ABI library: it loads and exports every declared symbol."""

import ctypes
import os
import re

from paper_2111_12478_b200 import _native as N

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
