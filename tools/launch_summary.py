"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per kernel, launches, total and
mean time, share of all our kernels' time (used for profiles/*_launches*.summary.txt)."""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0]
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        tot[name] += v
        cnt[name] += 1
    unit = rows[1][h.index("Metric Unit")] if "Metric Unit" in h else "?"
    ours = {k: v for k, v in tot.items() if "lbk::" in k}
    s = sum(ours.values()) or 1.0
    print(f"# {path}: per-kernel gpu__time_duration.sum ({unit}), our kernels only; share of their total")
    for k, v in sorted(ours.items(), key=lambda kv: -kv[1]):
        print(f"{v / s:7.2%}  n={cnt[k]:6d}  total={v:14.1f}  mean={v / cnt[k]:12.1f}  {k[:110]}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
