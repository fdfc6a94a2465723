#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python scripts/predict_ab.py > gpurun_out/r2o_predict_ab.json 2>&1; head -24 gpurun_out/r2o_predict_ab.json
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tree.py tests/test_gpu_tc.py -m gpu -q -x 2>&1 | tail -3
