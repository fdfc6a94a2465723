"""Turn gpurun_out/ ncu artefacts into the committed profiles/<round>/ summaries."""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", sys.argv[1] if len(sys.argv) > 1 else "round1")
G = os.path.join(ROOT, "gpurun_out")
os.makedirs(OUT, exist_ok=True)

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
           "launch__block_size", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                d[m] = f"{r[hdr.index(m)]} {units[hdr.index(m)]}".strip()
        out.append(d)
    return out


lines = []
for rep, title in (("scan_full.ncu-rep", "K4 scan (6 bench queries: Q1.1-Q1.3, Q2.1-Q2.3, SF=10)"),
                   ("shared_full.ncu-rep", "K4 shared scans (the bench's passes: Q1.1-Q1.3 and Q2.1-Q2.3, SF=10)"),
                   ("predict_full.ncu-rep", "K2+K3 fused predict (1e8 fact rows, cfg1 dims)")):
    p = os.path.join(G, rep)
    if not os.path.exists(p):
        continue
    rs = raw(p)
    json.dump(rs, open(os.path.join(OUT, rep.replace(".ncu-rep", "_metrics.json")), "w"), indent=1)
    lines.append(f"## {title}\n")
    lines.append("| kernel | time | DRAM read | DRAM write | DRAM % | issue % | warps % | regs | L1 hit | L2 hit |")
    lines.append("|---|---|---|---|---|---|---|---|---|---|")
    for d in rs:
        g = lambda k: d.get(k, "").replace(" ", "")
        lines.append(f"| {d['kernel'][:48]} | {g('gpu__time_duration.sum')} | {g('dram__bytes_read.sum')} | "
                     f"{g('dram__bytes_write.sum')} | {g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')} | "
                     f"{g('smsp__issue_active.avg.pct_of_peak_sustained_active')} | "
                     f"{g('sm__warps_active.avg.pct_of_peak_sustained_active')} | {g('launch__registers_per_thread')} | "
                     f"{g('l1tex__t_sector_hit_rate.pct')} | {g('lts__t_sector_hit_rate.pct')} |")
    lines.append("")

lc = os.path.join(G, "launches.csv")
if os.path.exists(lc):
    rows = list(csv.reader(open(lc)))
    hdr, agg = None, {}
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        agg.setdefault(d["Kernel Name"][:70], []).append(float(d["Metric Value"]))
    tot = sum(sum(v) for v in agg.values())
    lines.append("## Launch list of `bench.py --steps 2 --warmup 1` (ncu, cold-cache, serialised; includes setup + dial tuning)\n")
    lines.append("| share | launches | avg us | kernel |")
    lines.append("|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1]))[:15]:
        lines.append(f"| {sum(v) / tot * 100:.1f}% | {len(v)} | {sum(v) / len(v) / 1000:.1f} | {k} |")
    lines.append("")
    shutil.copy(lc, os.path.join(OUT, "launches.csv"))

bj = os.path.join(G, "bench.json")
if os.path.exists(bj):
    shutil.copy(bj, os.path.join(OUT, "bench.json"))
open(os.path.join(OUT, "ncu_summary.md"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
