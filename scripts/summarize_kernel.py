"""Summarise one ncu --set full report (any kernel) into profiles/<round>/<name>_ncu.{md,json}.
usage: python scripts/summarize_kernel.py <report.ncu-rep> <name> <title> [round]"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, name, title = sys.argv[1], sys.argv[2], sys.argv[3]
OUT = os.path.join(ROOT, "profiles", sys.argv[4] if len(sys.argv) > 4 else "round1")
os.makedirs(OUT, exist_ok=True)
METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor memory path active %"),
    ("sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active", "TMEM pipe %"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem->tensor wavefronts %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__block_size", "block"),
    ("launch__grid_size", "grid"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr, units = rows[0], rows[1]
res = []
for r in rows[2:]:
    d = {"kernel": r[hdr.index("Kernel Name")]}
    for m, _ in METRICS:
        hits = [i for i, h in enumerate(hdr) if h == m or h.endswith("." + m)]
        if hits:
            d[m] = f"{r[hits[0]]} {units[hits[0]]}".strip()
    res.append(d)
json.dump(res, open(os.path.join(OUT, f"{name}_ncu.json"), "w"), indent=1)
lines = [f"## {title}\n", f"source: `{os.path.basename(rep)}` (ncu --set full --clock-control none)\n"]
for d in res:
    lines.append(f"### {d['kernel'][:100]}\n")
    lines.append("| metric | value |\n|---|---|")
    for m, label in METRICS:
        if m in d:
            lines.append(f"| {label} (`{m}`) | {d[m]} |")
    lines.append("")
open(os.path.join(OUT, f"{name}_ncu.md"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
