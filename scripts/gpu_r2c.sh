#!/bin/bash
# predict one-launch A/B + ncu full capture of the Q4 batch kernel.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python scripts/predict_ab.py > gpurun_out/r2c_predict_ab.json 2> gpurun_out/r2c_predict_ab.err; echo "ab rc=$?"
cat gpurun_out/r2c_predict_ab.json; tail -3 gpurun_out/r2c_predict_ab.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:scan_batch_kernel -s 2 -c 2 -o gpurun_out/r2c_batch \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-fused --no-cpu-baseline > gpurun_out/r2c_ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/r2c_ncu.log
