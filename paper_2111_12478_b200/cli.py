"""``check`` front end with the reference's exit codes and output
(cli.py:20-84): 0 no races, 1 races found, 2 usage / parse error,
3 validation error.  NDJSON reports on stdout, diagnostics on stderr.
An engine failure (no CUDA device, library missing, CUDA or capacity error)
exits 4, never 1, so scripts gating on "races found" cannot misread it.
"""

from __future__ import annotations

import argparse
import sys
from typing import NoReturn

from . import _native as N
from .engine import diagnostics_of
from .report import ndjson_lines
from .trace import TraceParseError, UnsupportedTrace, infer_locks, load_trace, save_soa, validate_trace

EXIT_CLEAN = 0
EXIT_RACES = 1
EXIT_USAGE = 2
EXIT_INVALID = 3
EXIT_ENGINE = 4  # not in the reference (it has no engine that can fail): distinct from every code above


def _die(code: int, message: str) -> NoReturn:
    print(message, file=sys.stderr)
    raise SystemExit(code)


def _load(path: str, validate: bool = True, infer: bool = False):
    """Text trace or binary SoA file (by magic, trace.load_trace); lock
    inference and validate_trace run on the GPU (cli.py:26-43)."""
    try:
        tr = load_trace(path)
    except OSError as e:
        _die(EXIT_USAGE, f"cannot read {path}: {e}")
    except TraceParseError as e:
        _die(EXIT_USAGE, f"{path}: {e}")
    except UnsupportedTrace as e:
        _die(EXIT_USAGE, f"{path}: unsupported by the B200 engine: {e}")
    if not validate:
        return tr
    try:
        ctx = N.default_context()
        if infer:
            tr, idiags = infer_locks(tr, ctx=ctx)
            for d in idiags:
                print(f"{path}: lock inference: {d}", file=sys.stderr)
        diags = validate_trace(tr, ctx=ctx)
    except (N.NativeUnavailable, N.EngineError) as e:
        _die(EXIT_ENGINE, f"{path}: analysis engine failed: {e}")
    if diags:
        for d in diags:
            print(f"{path}: {d}", file=sys.stderr)
        _die(EXIT_INVALID, f"{path}: trace is not well formed")
    return tr


def _cmd_check(args) -> int:
    if args.detector not in ("gwcp", "hb"):
        _die(EXIT_USAGE, f"detector {args.detector!r} is not on the accelerated path (use gpurace)")
    if args.order_matrix:
        _die(EXIT_USAGE, "--order-matrix is not on the accelerated path (use gpurace)")
    tr = _load(args.trace, infer=args.infer_locks)
    try:
        res = N.analyze(tr.cfg_tuple, tr.key, tr.tidop, tr.instr, inactive_opt=not args.no_inactive_opt,
                        hb=args.detector == "hb")
    except (N.NativeUnavailable, N.EngineError) as e:
        _die(EXIT_ENGINE, f"{args.trace}: analysis engine failed: {e}")
    out = ndjson_lines(tr, res, args.detector)
    if out:
        sys.stdout.write("\n".join(out) + "\n")
    for d in diagnostics_of(tr, res):
        print(f"{args.trace}: {d}", file=sys.stderr)
    return EXIT_RACES if out else EXIT_CLEAN


def _cmd_convert(args) -> int:
    """Text trace -> binary SoA file (16 B/event; `check` reads either)."""
    tr = _load(args.trace, validate=False)
    try:
        save_soa(tr, args.out)
    except (OSError, N.EngineError) as e:
        _die(EXIT_USAGE, f"cannot write {args.out}: {e}")
    return EXIT_CLEAN


def _build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="gwcp-b200", description="B200 G-WCP trace race analysis.")
    sub = p.add_subparsers(dest="command", required=True)
    c = sub.add_parser("check", help="run the G-WCP detector over a trace")
    c.add_argument("trace")
    c.add_argument("--detector", choices=["gwcp", "hb", "lockset"], default="gwcp")
    c.add_argument("--no-compress", action="store_true", help="accepted; output is representation independent")
    c.add_argument("--no-inactive-opt", action="store_true")
    c.add_argument("--infer-locks", action="store_true")
    c.add_argument("--order-matrix", action="store_true")
    c.add_argument("--json", action="store_true", help="accepted for symmetry")
    c.set_defaults(func=_cmd_check)
    v = sub.add_parser("convert", help="write a trace as a binary SoA file")
    v.add_argument("trace")
    v.add_argument("out")
    v.set_defaults(func=_cmd_convert)
    return p


def main(argv: list[str] | None = None) -> int:
    parser = _build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as e:
        raise SystemExit(EXIT_USAGE if e.code not in (0,) else 0) from None
    try:
        return args.func(args)
    except SystemExit:
        raise
    except BrokenPipeError:
        return EXIT_CLEAN


if __name__ == "__main__":
    raise SystemExit(main())
