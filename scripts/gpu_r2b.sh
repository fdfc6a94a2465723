#!/bin/bash
# Batched scan: parity tests, drop-in extra checks, bench, ncu of the batch kernel.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_batch.py tests/test_reference_suites.py -m gpu -x -q 2>&1 | tail -25 > gpurun_out/r2b_pytest.log
cat gpurun_out/r2b_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
echo "bench rc=$?"; tail -3 gpurun_out/r2b_bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r2b_bench.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["details"])
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:scan_batch -c 4 --csv python bench.py --steps 1 --warmup 1 --no-e2e --no-fused --no-cpu-baseline > gpurun_out/r2b_ncu_launches.csv 2>/dev/null
tail -6 gpurun_out/r2b_ncu_launches.csv
