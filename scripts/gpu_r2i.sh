#!/bin/bash
# pipelined Q4 batch: parity + A/B + bench + step launch list.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_batch.py -m gpu -q -x 2>&1 | tail -4
timeout 900 python scripts/batch_ab.py > gpurun_out/r2i_batch_ab.json 2>&1; echo "batch_ab rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r2i_batch_ab.json')); print({k:v['ms'] for k,v in d.items() if k!='sf'})"
LAQ_BATCH_NO_PIPE=1 timeout 900 python scripts/batch_ab.py > gpurun_out/r2i_batch_ab_nopipe.json 2>&1
python -c "import json; d=json.load(open('gpurun_out/r2i_batch_ab_nopipe.json')); print('nopipe', {k:v['ms'] for k,v in d.items() if k!='sf'})"
timeout 600 python scripts/predict_ab.py > gpurun_out/r2i_predict_ab.json 2>&1; head -12 gpurun_out/r2i_predict_ab.json
timeout 1200 python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r2i_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['details']['per_query_scan_ms'], d['parity'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"scan_batch|dict_|codes_kernel" -c 60 --csv --log-file gpurun_out/r2i_step_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-fused > gpurun_out/r2i_launches.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:scan_batch_pipe -c 1 -o gpurun_out/r2i_pipe \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-fused --no-cpu-baseline > gpurun_out/r2i_ncu.log 2>&1; echo "ncu rc=$?"
