#!/bin/bash
# Round-2 evidence run: tests, bench (both arms), launch list, ncu captures, racecheck of the TMA pipe.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_batch.py tests/test_gpu_dist.py tests/test_reference_suites.py tests/test_gpu_parity.py -m gpu -q 2>&1 | tail -4
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err; echo "bench rc=$?"; tail -2 gpurun_out/r2h_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2h_ref.json 2> gpurun_out/r2h_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2h_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r2h_launches.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:scan_batch_kernel -s 2 -c 2 -o gpurun_out/r2h_batch \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-fused --no-cpu-baseline > gpurun_out/r2h_ncu_batch.log 2>&1; echo "ncu batch rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:direct_chunks_kernel -s 3 -c 1 -o gpurun_out/r2h_predict \
  python scripts/predict_ab.py > gpurun_out/r2h_ncu_predict.log 2>&1; echo "ncu predict rc=$?"
timeout 900 python scripts/batch_ab.py > gpurun_out/r2h_batch_ab.json 2>&1; echo "batch_ab rc=$?"
timeout 600 python scripts/sortpath_bench.py > gpurun_out/r2h_sortpath.json 2>&1; echo "sortpath rc=$?"
timeout 1500 compute-sanitizer --tool racecheck --target-processes all --print-limit 20 --error-exitcode 9 \
  python -m pytest tests/test_gpu_scan_stress.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2h_racecheck_pipe.log 2>&1; echo "racecheck rc=$?"
grep -E "RACECHECK SUMMARY|ERROR SUMMARY|passed" gpurun_out/r2h_racecheck_pipe.log
