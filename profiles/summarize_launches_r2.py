"""Per-kernel summary of an ncu launch list (--metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv): launches, device time and
DRAM bytes per kernel, sorted by time.  usage: summarize_launches_r2.py CSV [div]
(div = analyses in the list, e.g. 3 for run_one.py --repeat 1 under a bench-like warm-up)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hdr = None
agg = collections.OrderedDict()
SC = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    name = d["Kernel Name"].split("(")[0].replace("void ", "")[:60]
    a = agg.setdefault(name, {"us": 0.0, "n": 0, "bytes": 0.0})
    v = float(d["Metric Value"].replace(",", ""))
    u = SC.get(d.get("Metric Unit", ""), 1.0)
    if d["Metric Name"] == "gpu__time_duration.sum":
        a["us"] += v * u
        a["n"] += 1
    else:
        a["bytes"] += v * u
tot = sum(a["us"] for a in agg.values())
print(f"{'us/analysis':>12} {'launches':>8} {'GB/analysis':>11} {'GB/s':>7}  kernel")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["us"]):
    gbs = a["bytes"] / (a["us"] * 1e-6) / 1e9 if a["us"] else 0
    print(f"{a['us'] / div:12.1f} {a['n'] / div:8.1f} {a['bytes'] / div / 1e9:11.3f} {gbs:7.0f}  {k}")
print(f"total {tot / div:.1f} us/analysis (cold-cache, serialised ncu replay)")
