#!/bin/bash
# N=2 bench path on one GPU (gloo hook): the strong row-sharded code path incl. parity, e2e.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
LAQ_BENCH_SHARE_GPU=1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/r2n_n2.json 2> gpurun_out/r2n_n2.err; echo "n2 rc=$?"; tail -3 gpurun_out/r2n_n2.err
python -c "import json; d=json.loads(open('gpurun_out/r2n_n2.json').read().strip().splitlines()[-1]); print(d['n_gpus'], d['value'], d['ms_per_step'], d['parity'], d['details']['parallelism'], d['e2e']['value'])"
LAQ_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 \
  bench.py --gpus 2 --impl reference --steps 1 --warmup 1 > gpurun_out/r2n_n2_ref.json 2> gpurun_out/r2n_n2_ref.err; echo "n2 ref rc=$?"; head -c 300 gpurun_out/r2n_n2_ref.json
