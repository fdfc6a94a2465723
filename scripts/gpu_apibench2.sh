#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "dense_matmul" 2>&1 | tail -2
timeout 900 integration/_build/dropin_bench --pipeline 2000 5 > gpurun_out/api_pipeline_sf2000.json 2>&1; echo "rc=$?"; cat gpurun_out/api_pipeline_sf2000.json
