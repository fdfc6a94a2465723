#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python scripts/batch_ab.py > gpurun_out/r2m_batch_ab.json 2>&1; echo "batch_ab rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r2m_batch_ab.json')); print({k:(v['ms'],v['same_result']) for k,v in d.items() if k!='sf'})"
