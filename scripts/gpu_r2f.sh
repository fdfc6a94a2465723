#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python scripts/predict_ab.py > gpurun_out/r2f_predict_ab.json 2>&1; head -40 gpurun_out/r2f_predict_ab.json
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/r2f_pytest.log
cat gpurun_out/r2f_pytest.log
