"""GPU, world size 2: the row-sharded multi-GPU path with the DEVICE kernels.

Two processes share cuda:0 over gloo (the one-GPU stand-in for two GPUs over
NCCL; NCCL refuses two ranks on one device).  Each rank generates its
contiguous shard of the canonical lineorder (gen row_range), uploads it, and
attaches the gloo group to its C-ABI context (dist.attach -> host all-reduce
hook), so laq_run_query / laq_measure_selectivity / laq_allreduce_acc merge the
per-rank (count, sum) accumulators inside the library.  Every rank's result
must equal the whole-table oracle (oracle/fast_query, pinned to the
reference's goldens); fused predictions of the shards concatenated in rank
order must equal the whole-table prediction bit-for-bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_file):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from oracle import fast_query as F
    from oracle import laq_oracle as O
    from paper_2306_08367_b200 import dist as D, fusion, gen, query as Q, star
    from paper_2306_08367_b200.device import context
    errors = []
    ctx = context(0)
    D.attach(ctx)
    assert ctx.comm == (world, rank)
    full = gen.gen_star("Ssb", 1, 42, narrow=True)
    n = len(full.fact["lo_part"])
    rr = D.shard_range(n, rank, world)
    g = gen.gen_star("Ssb", 1, 42, narrow=True, row_range=rr)
    ds = star.upload_gen_star(g, ctx=ctx)
    for grp, qi, dial in ((1, 0, 222), (2, 1, 60), (3, 0, 105), (3, 2, 43), (4, 0, 249), (4, 2, 284)):
        q = Q.spec_with_dial(Q.group_defs(grp)[qi], grp, dial)
        want = F.run_query(full.tables, q)
        if not np.array_equal(ds.run_query(q), want):  # laq_run_query all-reduces inside
            errors.append(f"run_query {grp}.{qi}")
        p = ds.prepare(q)
        acc = ctx.allreduce_acc(p.execute())
        if not np.array_equal(p.emit(acc.cpu().numpy()), want):
            errors.append(f"plan {grp}.{qi}")
        if ds.measure_selectivity(q) != O.measure_selectivity(full.tables, q):
            errors.append(f"selectivity {grp}.{qi}")
    # batched scans (the bench's path): each rank scans its shard for a whole
    # query group in one pass; the per-query accumulators are all-reduced
    for grp, dials in ((3, (105, 79, 43)), (4, (249, 199, 284))):
        qs = [Q.spec_with_dial(d, grp, x) for d, x in zip(Q.group_defs(grp), dials)]
        b = star.Batch([ds.prepare(q) for q in qs])
        if not b.fused:
            errors.append(f"batch {grp} not fused: {b.why}")
        b.build()
        for q, p, acc in zip(qs, b.plans, b.scan()):
            if not np.array_equal(p.emit(ctx.allreduce_acc(acc).cpu().numpy()), F.run_query(full.tables, q)):
                errors.append(f"batch {grp} {q.id}")
    # fused join + predict: no collective; the rank-ordered concatenation is the answer
    fk, pk, feats, W = gen.cfg1_inputs(200_003, 1_000, 16, 1)
    fk[::997] = 5_000  # dangling keys: survivors differ per shard
    f = fusion.prefuse_linear([feats], [np.arange(16)], W)
    b, e = D.shard_range(len(fk), rank, world)
    y, surv = fusion.fused_star_predict([fk[b:e]], [pk], f.partials)
    off, total = D.gather_offsets(len(y))
    glob = torch.zeros(total, dtype=torch.float64)
    glob[off: off + len(y)] = torch.from_numpy(np.asarray(y)[:, 0])
    dist.all_reduce(glob)
    ws, wr = O.multiway_star_join([fk], [pk])
    if not np.array_equal(glob.numpy(), O.apply_fused_linear(wr, O.prefuse_linear([feats], [np.arange(16)], W))[:, 0]):
        errors.append("fused predict")
    flag = torch.tensor([0 if errors else 1])
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        with open(result_file, "w") as fh:
            fh.write(str(int(flag.item())) + " " + ";".join(errors))
    ctx.set_allreduce_host(1, 0, None)
    dist.destroy_process_group()


def test_row_sharded_device_path_two_ranks(tmp_path):
    out = tmp_path / "ok"
    mp.spawn(_worker, args=(2, _free_port(), str(out)), nprocs=2, join=True)
    assert out.read_text().startswith("1"), out.read_text()
