"""``HbDetector`` for the batch engine (mirror of hb.py:30-49).

The scoped happens-before detector of the reference: the same sync pass and
access checks as G-WCP with the predictive parts removed — no lock queues,
no conflicting-section clocks, checks against the happens-before clock
(hb.py:95-121).  The engine runs it through the same kernels with the
GW_OPT_HB flag (include/gwcp_b200.h).  On lock-free traces its reports equal
G-WCP's; on lock traces it reports the races G-WCP's predictive edges hide
and vice versa (tests/golden/golden_hb.jsonl.gz).
"""

from __future__ import annotations

from .report import Reporter
from .trace import Diagnostic


class HbDetector:
    name = "hb"

    def __init__(self, config, *, compress: bool = True, forced_barriers: bool = False):
        if forced_barriers:
            raise NotImplementedError("forced_barriers is the stats-only mode of the reference detector")
        self.config = config
        self.compress = compress
        self.reporter = Reporter(self.name)
        self.diagnostics: list[Diagnostic] = []
