#!/bin/bash
# Tests + A/B scan timings + bench (no ncu).
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python scripts/scan_ab.py 2>&1 | tail -4
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; tail -3 gpurun_out/bench.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
print("value %.3e  ms/step %.3f  frac %.3f  e2e %.3e" % (d["value"], d["ms_per_step"], d["roofline"]["frac"], d["e2e"]["value"]))
print("per-launch scan ms", d["config"]["per_launch_scan_ms"], d["config"]["shared_scan"])
print("secondary", json.dumps(d["secondary"])[:600])
PY
