"""Brief of an ncu --set full report: per kernel, duration / DRAM / issue / LSU
and the SASS opcode mix with per-source-line hot spots (needs -lineinfo builds
and the local cubin of the same build for line mapping: pass --cubin).

usage: python scripts/ncu_brief.py <report.ncu-rep> [--rows N] [--cubin file.cubin]
"""
import csv
import re
import subprocess
import sys
from collections import Counter, defaultdict

rep = sys.argv[1]
rows_n = float(sys.argv[sys.argv.index("--rows") + 1]) if "--rows" in sys.argv else None
cubin = sys.argv[sys.argv.index("--cubin") + 1] if "--cubin" in sys.argv else None
KEYS = ["gpu__time_duration.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "dram__bytes_read.sum", "launch__registers_per_thread"]
raw = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                     text=True).stdout.splitlines()))
hdr, units = raw[0], raw[1]
for r in raw[2:]:
    print(r[hdr.index("Kernel Name")])
    for k in KEYS:
        if k in hdr:
            print(f"   {k} = {r[hdr.index(k)]} {units[hdr.index(k)]}")
src = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                                     capture_output=True, text=True).stdout.splitlines()))
data, kern, shdr = {}, None, None
for r in src:
    if r and r[0] == "Kernel Name":
        kern = r[1]
        data[kern] = []
    elif r and r[0] == "Address":
        shdr = r
    elif kern and len(r) > 5:
        data[kern].append(r)
lines_of = {}
if cubin:
    txt = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.splitlines()
    fn, cur = None, None
    for l in txt:
        if l.startswith("//----") and ".text." in l:
            fn = l.split(".text.")[1].split()[0]
            lines_of[fn] = {}
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
        if m and fn and cur:
            lines_of[fn][int(m.group(1), 16)] = cur
for k, v in data.items():
    ie, st = shdr.index("Instructions Executed"), shdr.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(x[ie]) for x in v)
    samp = max(1, sum(int(x[st]) for x in v))
    per = f", {tot / rows_n:.2f} warp-instr/row" if rows_n else ""
    print(f"{k[:90]}: {tot} warp-instr{per}")
    c, s = Counter(), Counter()
    for x in v:
        t = x[1].split()
        op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        c[op] += int(x[ie])
        s[op] += int(x[st])
    print("   opcodes:", [(o, round(n / tot, 3)) for o, n in c.most_common(12)])
    print("   stalls :", [(o, round(n / samp, 3)) for o, n in s.most_common(8)])
    # source lines (mangled names differ between the report and the cubin: match by template args)
    cand = [fn for fn in lines_of if "scan_batch_kernel" in fn]
    args = re.findall(r"\(int\)(\d+)", k)
    fn = next((f for f in cand if "".join(f"ILi{a}E" if i == 0 else f"Li{a}E" for i, a in enumerate(args)) in f), None)
    if fn:
        base = int(v[0][0], 16)
        bl, bs = Counter(), Counter()
        for x in v:
            key = lines_of[fn].get(int(x[0], 16) - base)
            if key:
                bl[key] += int(x[ie])
                bs[key] += int(x[st])
        print("   hot lines:", [(f"{a}:{b}", round(n / tot, 3), round(bs[(a, b)] / samp, 3)) for (a, b), n in bl.most_common(10)])
