#!/bin/bash
# CTA-pair (cta_group::2) FFN: parity under a hard timeout, then timing A/B.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
LAQ_FFN_2CTA=1 timeout 600 python -m pytest tests/test_gpu_ffn.py -m gpu -q -x 2>&1 | tail -5
echo "tests rc=${PIPESTATUS[0]}"
for v in 0 1; do LAQ_FFN_2CTA=$v timeout 300 python scripts/ffn_perf.py 2>&1 | tail -1; done
for d in 1 2 3; do LAQ_FFN_2CTA=1 LAQ_FFN_DIAG=$d timeout 300 python scripts/ffn_perf.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('diag', $d, round(d['ms_join_ffn_probe'],3))"; done
