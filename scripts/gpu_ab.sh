#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python scripts/scan_ab.py 2>&1 | tail -5
if [ "${LAQ_NCU:-0}" = "1" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_pipe -c 6 \
      -o gpurun_out/scan_full -f python scripts/profile_scan.py > gpurun_out/ncu_full.log 2>&1
  echo "ncu full rc=$?"; tail -2 gpurun_out/ncu_full.log
fi
