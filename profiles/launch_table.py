"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv) per launch: time, DRAM bytes, kernel."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data = {}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        e = data.setdefault(int(d["ID"]), {"name": d["Kernel Name"].split("(")[0][:64]})
        v = float(d["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}
        e[d["Metric Name"]] = v * scale.get(d["Metric Unit"], 1.0)
skip = set(sys.argv[2].split(",")) if len(sys.argv) > 2 else set()
tot = 0.0
print(f"{'id':>3} {'ms':>9} {'GB rd':>8} {'GB wr':>8} {'GB/s':>7}  kernel")
for k in sorted(data):
    v = data[k]
    if any(s and s in v["name"] for s in skip):
        continue
    ms = v.get("gpu__time_duration.sum", 0.0)
    rd, wr = v.get("dram__bytes_read.sum", 0.0), v.get("dram__bytes_write.sum", 0.0)
    tot += ms
    print(f"{k:>3} {ms:9.3f} {rd:8.2f} {wr:8.2f} {((rd + wr) / ms * 1e3 if ms else 0):7.0f}  {v['name']}")
print(f"total {tot:.3f} ms (serialised, cold-cache launches)")
