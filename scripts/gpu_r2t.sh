#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_batch.py -m gpu -q -x 2>&1 | tail -3
timeout 900 python scripts/batch_ab.py > gpurun_out/r2t_batch_ab.json 2>&1; echo "batch_ab rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r2t_batch_ab.json')); print({k:(v['ms'],v['same_result']) for k,v in d.items() if k!='sf'})"
