"""Fold ncu DRAM-traffic captures (ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,
gpu__time_duration.sum --csv --log-file F) into profiles/ncu_traffic.json, the per-launch `traffic`
that bench.py reports.  usage: python tools/ncu_traffic_update.py KEY KERNEL_NAME CSV [KEY KERNEL CSV ...]"""
import csv
import json
import sys

P = "profiles/ncu_traffic.json"


def parse(path):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    h = rows[0]
    mi, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    out = {}
    for r in rows[1:]:
        if len(r) > vi:
            v = float(r[vi].replace(",", ""))
            u = r[ui]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0,
                     "usecond": 1e-3, "nsecond": 1e-6, "msecond": 1.0}.get(u, 1)
            out[r[mi]] = v * scale
    return out


d = json.load(open(P))
args = sys.argv[1:]
for k in range(0, len(args), 3):
    key, kernel, path = args[k:k + 3]
    m = parse(path)
    rd, wr = m["dram__bytes_read.sum"], m["dram__bytes_write.sum"]
    d[key] = {"kernel": kernel, "dram_bytes_per_launch": int(rd + wr), "dram_read": int(rd), "dram_write": int(wr),
              "duration_ms_ncu": round(m["gpu__time_duration.sum"], 6), "capture": path.split("/")[-1]}
    print(key, d[key])
json.dump(d, open(P, "w"), indent=1)
