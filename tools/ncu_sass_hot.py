"""Top SASS instructions by stall samples / executed count from an ncu source page (csv)."""
import csv, subprocess, sys
path = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
ai, si, wi, ni = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
data = []
for idx, r in enumerate(rows[2:]):
    try:
        data.append((idx, float(r[wi] or 0), float(r[ni] or 0), r[si].strip()))
    except (ValueError, IndexError):
        pass
tw = sum(d[1] for d in data) or 1; tn = sum(d[2] for d in data) or 1
print(f"total stall samples {tw:.0f}, instructions {tn:.0f}")
mode = sys.argv[3] if len(sys.argv) > 3 else "stall"
if mode == "all":
    for idx, w, ni_, src in data:
        print(f"{idx:4d} {w/tw:6.1%} {ni_/tn:6.2%}  {src[:90]}")
else:
    for idx, w, ni_, src in sorted(data, key=lambda d: -d[1])[:n]:
        print(f"{idx:4d} {w/tw:6.1%} {ni_/tn:6.2%}  {src[:90]}")
