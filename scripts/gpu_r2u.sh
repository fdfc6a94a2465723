#!/bin/bash
# sanitizers over the batched-scan and fused-predict tests after the round-2 kernel changes
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
SEL="tests/test_gpu_batch.py tests/test_gpu_parity.py"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 20 --error-exitcode 9 \
     python -m pytest $SEL -m gpu -q -p no:cacheprovider -k "not slow" > gpurun_out/sanitize2_$tool.log 2>&1
  echo "$tool rc=$?"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/sanitize2_$tool.log | tail -3
done
