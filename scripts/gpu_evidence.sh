#!/bin/bash
# Full evidence run: all GPU tests, smoke, bench (both arms), timed-step launch list, ncu of the batch passes.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/ev_pytest.log; cat gpurun_out/ev_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err; echo "bench rc=$?"; tail -2 gpurun_out/ev_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev_ref.json 2> gpurun_out/ev_ref.err; echo "ref rc=$?"
LAQ_PROFILE_TIMED=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_step_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-fused > gpurun_out/ev_launches.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:scan_batch_kernel -s 2 -c 2 -o gpurun_out/ev_batch \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-fused --no-cpu-baseline > gpurun_out/ev_ncu_batch.log 2>&1; echo "ncu batch rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/ev_bench.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["details"]["per_query_scan_ms"], d["e2e"]["value"], d["parity"])
r = json.loads(open("gpurun_out/ev_ref.json").read().strip().splitlines()[-1]); print("ref", r["value"])
PY
