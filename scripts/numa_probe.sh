#!/bin/bash
# Host topology of the GPU box and pinned H2D bandwidth with the process bound
# to each NUMA node's CPUs (first-touch puts the pinned buffer on that node).
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
lscpu | grep -E "Model name|Socket|NUMA|^CPU\(s\)"
nvidia-smi topo -m 2>/dev/null | head -5
bus=$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | head -1 | tr 'A-F' 'a-f' | sed 's/^0000//;s/^/0000/' | cut -c1-12)
for f in /sys/bus/pci/devices/*; do :; done
python - <<'PY'
import glob, subprocess
bus = subprocess.check_output(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader"]).decode().split()[0].lower()
bus = bus[-12:]
for p in glob.glob("/sys/bus/pci/devices/*"):
    if p.endswith(bus):
        print("gpu", bus, "numa_node", open(p + "/numa_node").read().strip(), "local_cpulist", open(p + "/local_cpulist").read().strip())
for n in sorted(glob.glob("/sys/devices/system/node/node*/cpulist")):
    print(n.split("/")[-2], open(n).read().strip())
PY
for n in /sys/devices/system/node/node*; do
  cpus=$(cat $n/cpulist)
  echo "== bound to $(basename $n) cpus $cpus"
  timeout 300 taskset -c $cpus python scripts/h2d_probe.py 2>&1 | head -4
done
