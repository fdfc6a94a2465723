#!/bin/bash
# batched scan v2: parity tests + bench + ncu of the batch kernels.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_batch.py tests/test_gpu_parity.py tests/test_gpu_queries.py -m gpu -x -q 2>&1 | tail -5 > gpurun_out/r2e_pytest.log
cat gpurun_out/r2e_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err
echo "bench rc=$?"; tail -3 gpurun_out/r2e_bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r2e_bench.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["details"]["per_query_scan_ms"], d["fused_join_predict"]["n1000000"])
PY
timeout 600 python scripts/predict_ab.py > gpurun_out/r2e_predict_ab.json 2>&1; head -20 gpurun_out/r2e_predict_ab.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:scan_batch_kernel -s 2 -c 2 -o gpurun_out/r2e_batch \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-fused --no-cpu-baseline > gpurun_out/r2e_ncu.log 2>&1; echo "ncu rc=$?"
