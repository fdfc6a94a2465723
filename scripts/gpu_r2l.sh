#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_batch.py -m gpu -q -x 2>&1 | tail -3
timeout 900 python scripts/batch_ab.py > gpurun_out/r2l_batch_ab.json 2>&1; echo "batch_ab rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r2l_batch_ab.json')); print({k:(v['ms'],v['same_result']) for k,v in d.items() if k!='sf'})"
timeout 900 python bench.py --workload q1q2 --steps 20 --warmup 5 --no-e2e --no-fused > gpurun_out/r2l_q1q2.json 2> gpurun_out/r2l_q1q2.err; echo "q1q2 rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r2l_q1q2.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['details']['per_query_scan_ms'], d['parity']['whole_table_vs_golden'])"
timeout 1200 python bench.py --steps 10 --warmup 3 --no-e2e --no-fused > gpurun_out/r2l_bench.json 2> gpurun_out/r2l_bench.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r2l_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['details']['per_query_scan_ms'], d['parity'])"
