#!/bin/bash
# Round 2: GPU tests (incl. the new distributed + large tests), then the new bench (both arms).
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2a_pytest.log
cat gpurun_out/r2a_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
echo "bench rc=$?"; tail -5 gpurun_out/r2a_bench.err
head -c 3000 gpurun_out/r2a_bench.json
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/r2a_ref.json 2> gpurun_out/r2a_ref.err
echo "ref rc=$?"; tail -5 gpurun_out/r2a_ref.err
head -c 1500 gpurun_out/r2a_ref.json
