#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python bench.py --workload q1q2 --steps 20 --warmup 5 --no-e2e > gpurun_out/r2k_q1q2.json 2> gpurun_out/r2k_q1q2.err; echo "q1q2 rc=$?"; tail -2 gpurun_out/r2k_q1q2.err
python -c "import json; d=json.loads(open('gpurun_out/r2k_q1q2.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['details']['per_query_scan_ms'], d['details']['batched_scan'], d['parity']); print(d['fused_join_predict'].get('e2e_reference_api'))"
timeout 1200 python -m pytest tests/test_gpu_large.py tests/test_reference_suites.py -m gpu -q 2>&1 | tail -3
