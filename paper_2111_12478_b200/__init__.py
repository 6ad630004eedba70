"""B200-native G-WCP predictive race analysis (arXiv 2111.12478), drop-in
for the ``gwcp`` path of the reference package ``gpurace``:

    from paper_2111_12478_b200 import parse_trace, run, GwcpDetector
    trace = parse_trace(text)
    for rep in run(trace, GwcpDetector(trace.config)).reports:
        print(rep.to_json())

The analysis runs as hand-written sm_100a CUDA kernels behind the C-ABI of
include/gwcp_b200.h (libgwcp_b200.so); there is no CPU path.
"""

from .engine import RunResult, run
from .gwcp import GwcpDetector
from .hb import HbDetector
from .report import Endpoint, RaceReport
from .trace import (
    Barrier,
    Diagnostic,
    Event,
    Location,
    Scope,
    ThreadId,
    Trace,
    TraceConfig,
    TraceParseError,
    UnsupportedTrace,
    encode,
    parse_trace,
    validate_trace,
)

__version__ = "0.1.0"

__all__ = [
    "Barrier",
    "Diagnostic",
    "Endpoint",
    "Event",
    "GwcpDetector",
    "HbDetector",
    "Location",
    "RaceReport",
    "RunResult",
    "Scope",
    "ThreadId",
    "Trace",
    "TraceConfig",
    "TraceParseError",
    "UnsupportedTrace",
    "encode",
    "parse_trace",
    "run",
    "validate_trace",
]
