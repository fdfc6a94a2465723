#!/bin/bash
# GPU test pass: every -m gpu test (slow ones included), summary to gpurun_out/.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout ${T:-2400} python -m pytest tests -m gpu -q ${ARGS} 2>&1 | tail -${TAIL:-40} > gpurun_out/pytest_gpu.log
cat gpurun_out/pytest_gpu.log
