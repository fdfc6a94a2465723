#!/bin/bash
# Box facts (host RAM, cores) + the GPU test suite.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
{ free -g; nproc; lscpu | grep -E "Model name|Socket|Thread|NUMA node\(s\)"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv; df -h /tmp | tail -1; } > gpurun_out/env.txt 2>&1
cat gpurun_out/env.txt
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
