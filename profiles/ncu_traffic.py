"""Build profiles/ncu_traffic.json (per-launch DRAM bytes, mean over the
captured launches of each kernel) from ncu --set full reports:
    python profiles/ncu_traffic.py c5=gpurun_out/full_c5b.ncu-rep c5=gpurun_out/full_c5_access.ncu-rep c2=...
"""
import csv
import io
import json
import os
import subprocess
import sys

SC = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
out_path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ncu_traffic.json")
try:
    out = json.load(open(out_path))
except Exception:
    out = {}
acc = {}
for arg in sys.argv[1:]:
    wl, rep = arg.split("=", 1)
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = d["Kernel Name"].replace("void ", "").split("(")[0].split("<")[0].strip()
        b = sum(float(d[m].replace(",", "")) * SC[u[h.index(m)]] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        acc.setdefault(wl, {}).setdefault(name, []).append(b)
for wl, ks in acc.items():
    for k, v in ks.items():
        out.setdefault(wl, {})[k] = sum(v) / len(v)
json.dump(out, open(out_path, "w"), indent=1, sort_keys=True)
print(json.dumps(out, indent=1, sort_keys=True))
