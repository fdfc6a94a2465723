#!/bin/bash
# Full evidence session: tests, bench JSON, ncu launch list of bench, ncu full captures.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m pytest tests -m gpu -q 2>&1 | tail -3
python __graft_entry__.py smoke 2>&1 | tail -2
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-secondary > gpurun_out/bench_ncu.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_direct -c 6 \
    -o gpurun_out/scan_full -f python scripts/profile_scan.py > gpurun_out/ncu_scan.log 2>&1; echo "ncu scan rc=$?"
LAQ_PROFILE_SHARED=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_shared -c 2 \
    -o gpurun_out/shared_full -f python scripts/profile_scan.py > gpurun_out/ncu_shared.log 2>&1; echo "ncu shared rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chunks_kernel -s 6 -c 2 \
    -o gpurun_out/predict_full -f python scripts/profile_predict.py > gpurun_out/ncu_pred.log 2>&1; echo "ncu predict rc=$?"
timeout 900 python bench.py --workload q3q4 --steps 10 --warmup 3 > gpurun_out/bench_q3q4.json 2> gpurun_out/bench_q3q4.err; echo "q3q4 rc=$?"
