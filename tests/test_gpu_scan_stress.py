"""GPU: the stream (default) and TMA-pipelined scans equal the plain-load
fallback scan's accumulators, repeatedly, at full SF=10 size (guards the
mbarrier stage protocol against ordering races)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DIALS = {(1, 0): 222, (1, 1): 200, (1, 2): 133, (2, 0): 500, (2, 1): 199, (2, 2): 516, (3, 0): 90, (4, 0): 50}


def test_pipe_equals_ldg_repeatedly(gpu_ctx, monkeypatch):
    import torch
    from paper_2306_08367_b200 import gen, query as Q, star
    g = gen.gen_star("Ssb", 10, 42, narrow=True)
    ds = star.upload_gen_star(g)
    for (gr, qi), d in DIALS.items():
        q = Q.spec_with_dial(Q.group_defs(gr)[qi], gr, d)
        monkeypatch.setenv("LAQ_SCAN", "ldg")
        ref_plan = ds.prepare(q)
        want = ref_plan.execute().cpu().numpy().copy()
        for variant in ("stream", "pipe"):
            monkeypatch.setenv("LAQ_SCAN", variant)
            p = ds.prepare(q)
            p.build_codes()
            accs = [torch.zeros_like(p.acc) for _ in range(6)]
            for a in accs:
                p.scan(a)
            torch.cuda.synchronize()
            for a in accs:
                assert np.array_equal(a.cpu().numpy(), want), f"{variant} Q{gr}.{qi + 1}"
