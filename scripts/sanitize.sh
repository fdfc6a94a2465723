#!/bin/bash
# compute-sanitizer passes (memcheck / racecheck / synccheck) over small GPU
# tests that exercise every kernel family: shared-memory-atomic scans (direct,
# batched, shared), mbarrier/TMA pipelines (scan_pipe), tcgen05/TMEM GEMMs and
# the FFN, fused predict (one- and three-launch), tree, key domain, group-by,
# sparse ops.  Summaries -> gpurun_out/sanitize_*.log
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
SEL="tests/test_gpu_parity.py tests/test_gpu_batch.py::test_ssb_sf1_groups_fused_match_goldens tests/test_gpu_batch.py::test_empty_interval_and_tail_rows tests/test_gpu_queries.py::test_queries_s2_golden tests/test_gpu_tc.py tests/test_gpu_ffn.py tests/test_gpu_tree.py tests/test_gpu_sparse.py tests/test_gpu_scan_stress.py"
for tool in memcheck racecheck synccheck; do
  timeout ${T:-1500} compute-sanitizer --tool $tool --target-processes all --print-limit 20 --error-exitcode 9 \
     python -m pytest $SEL -m gpu -q -x -p no:cacheprovider > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"
  grep -E "ERROR SUMMARY|passed|failed|Invalid|Race|Barrier" gpurun_out/sanitize_$tool.log | tail -6
done
