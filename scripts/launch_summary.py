"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into a
markdown table of kernels, launches, average time and share of kernel time.
usage: python scripts/launch_summary.py <launches.csv> <out.md> <title>"""
import csv
import sys
from collections import defaultdict

src, out, title = sys.argv[1], sys.argv[2], sys.argv[3]
rows = [r for r in csv.reader(l for l in open(src) if l.startswith('"'))]
hdr, rows = rows[0], rows[1:]
k, v = hdr.index("Kernel Name"), hdr.index("Metric Value")
t = defaultdict(list)
for r in rows:
    t[r[k]].append(float(r[v].replace(",", "")))
total = sum(sum(x) for x in t.values())
lines = [f"## {title}\n",
         "`LAQ_PROFILE_TIMED=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none` "
         "(cudaProfilerStart/Stop around the timed steps; serialised, cold-cache launches).\n",
         "| kernel | launches | avg us | share of kernel time |", "|---|---|---|---|"]
for name, xs in sorted(t.items(), key=lambda kv: -sum(kv[1])):
    lines.append(f"| `{name}` | {len(xs)} | {sum(xs) / len(xs) / 1e3:.1f} | {sum(xs) / total:.3f} |")
lines.append(f"\nTotal kernel time {total / 1e6:.3f} ms.")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
