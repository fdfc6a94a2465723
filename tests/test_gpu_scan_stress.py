"""GPU: the direct-probe (default), generic stream and TMA-pipelined scans equal the plain-load
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
        for variant in ("direct", "stream", "pipe"):
            monkeypatch.setenv("LAQ_SCAN", variant)
            p = ds.prepare(q)
            p.build_codes()
            accs = [torch.zeros_like(p.acc) for _ in range(6)]
            for a in accs:
                p.scan(a)
            torch.cuda.synchronize()
            for a in accs:
                assert np.array_equal(a.cpu().numpy(), want), f"{variant} Q{gr}.{qi + 1}"


def test_direct_ragged_ranges_equal_ldg(gpu_ctx, monkeypatch):
    """The direct kernel runs full grid steps without row bounds and one bounded
    tail step: ragged ranges (tail inside a 4-row group, ranges shorter than one
    grid step, empty) must match the plain-load scan exactly."""
    import torch
    from paper_2306_08367_b200 import gen, query as Q, star
    g = gen.gen_star("Ssb", 1, 42, narrow=True)
    ds = star.upload_gen_star(g)
    n = len(g.fact["lo_part"])
    for (gr, qi), d in {(1, 0): 222, (2, 0): 500, (4, 0): 50}.items():
        q = Q.spec_with_dial(Q.group_defs(gr)[qi], gr, d)
        for row0, rows in ((0, n), (4, n - 4), (0, 1), (8, 3), (0, 606_209), (1_000_000, 1_234_567), (n - 8, 8), (n - 12, 7), (12, 0)):
            monkeypatch.setenv("LAQ_SCAN", "ldg")
            ref = ds.prepare(q)
            ref.build_codes()
            want = ref.scan_range(row0, rows).cpu().numpy().copy()
            monkeypatch.delenv("LAQ_SCAN")
            p = ds.prepare(q)
            p.build_codes()
            got = p.scan_range(row0, rows).cpu().numpy()
            torch.cuda.synchronize()
            assert np.array_equal(got, want), (gr, qi, row0, rows)
