"""``GwcpDetector`` for the batch engine (mirror of gwcp.py:103-127).

The reference detector is driven event by event by ``engine.run``; here the
whole trace is analysed at once on the GPU, so the detector object carries
the configuration and options and, after :func:`engine.run`, the results in
the same attributes the reference exposes (``reporter.reports``,
``diagnostics``).  ``compress`` is accepted and ignored: report output does not
depend on the clock representation (acceptance 5,
pkg/tests/test_acceptance.py:152-172).  ``forced_barriers`` belongs to the
``stats`` subcommand and is not part of the analysed path.
"""

from __future__ import annotations

from .report import Reporter
from .trace import Diagnostic


class GwcpDetector:
    name = "gwcp"

    def __init__(self, config, *, compress: bool = True, inactive_opt: bool = True, forced_barriers: bool = False):
        if forced_barriers:
            raise NotImplementedError("forced_barriers is the stats-only mode of the reference detector")
        self.config = config
        self.compress = compress
        self.inactive_opt = inactive_opt
        self.reporter = Reporter(self.name)
        self.diagnostics: list[Diagnostic] = []
