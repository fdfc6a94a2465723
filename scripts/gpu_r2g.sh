#!/bin/bash
# batch layout A/B (SF=100) + FFN L2-hint A/B + ncu of the FFN.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python scripts/batch_ab.py > gpurun_out/r2g_batch_ab.json 2> gpurun_out/r2g_batch_ab.err; echo "ab rc=$?"
cat gpurun_out/r2g_batch_ab.json; tail -2 gpurun_out/r2g_batch_ab.err
timeout 600 python scripts/ffn_perf.py > gpurun_out/r2g_ffn_hint.json 2>&1; tail -1 gpurun_out/r2g_ffn_hint.json
LAQ_FFN_NO_L2_HINT=1 timeout 600 python scripts/ffn_perf.py > gpurun_out/r2g_ffn_nohint.json 2>&1; tail -1 gpurun_out/r2g_ffn_nohint.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ffn_kernel -c 1 -o gpurun_out/r2g_ffn \
  python scripts/ffn_perf.py 10 --profile > gpurun_out/r2g_ffn_ncu.log 2>&1; echo "ncu rc=$?"
timeout 600 python scripts/sortpath_bench.py > gpurun_out/r2g_sortpath.json 2>&1; cat gpurun_out/r2g_sortpath.json | tail -30
timeout 1800 python scripts/complexity_sweep.py gpurun_out/r2g_holdout.json --holdout > gpurun_out/r2g_holdout.log 2>&1; echo "holdout rc=$?"; tail -1 gpurun_out/r2g_holdout.log
