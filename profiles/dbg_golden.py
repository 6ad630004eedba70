import sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from conftest import golden_records, golden_text
from paper_2111_12478_b200 import _native as N
from paper_2111_12478_b200.trace import parse_trace
from paper_2111_12478_b200.report import ndjson_lines
ctx = N.Context(0)
for r in golden_records():
    if r["name"] != "c2/small": continue
    tr = parse_trace(golden_text(r))
    ctx.analyze_host(tr.cfg_tuple, tr.key, tr.tidop, tr.instr)
    got = ndjson_lines(tr, ctx.fetch())
    want = r["reports"]
    print(len(got), len(want), tr.config)
    for i, (a, b) in enumerate(zip(got, want)):
        if a != b:
            print(i, "GOT ", a); print(i, "WANT", b)
            if i > 5: break
