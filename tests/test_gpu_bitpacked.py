"""GPU: the bit-packed transfer format (laq_star_add_table_device_bitpacked,
scan_direct_kernel<..., 2>) gives the same accumulators as the int32 star for
every SSB query group, over full scans and ragged 32-aligned ranges."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DIALS = {(1, 0): 222, (1, 2): 133, (2, 0): 500, (2, 2): 516, (3, 0): 90, (3, 2): 40, (4, 0): 50, (4, 2): 20}


@pytest.fixture(scope="module")
def stars(gpu_ctx):
    import torch
    from paper_2306_08367_b200 import gen, star
    g = gen.gen_star("Ssb", 1, 42, narrow=True)
    plain = star.upload_gen_star(g)
    bp = star.DeviceStar(gpu_ctx)
    n = len(g.fact["lo_part"])
    packed = star.bitpack_columns(g.fact)
    dev = {c: (torch.from_numpy(w.view(np.int32)).cuda(), b, off) for c, (w, b, off) in packed.items()}
    bp.add_table_device_bitpacked("lineorder", dev, g.kinds["lineorder"], n, is_fact=True)
    for t, cols in g.tables.items():
        if t != "lineorder":
            bp.add_table(t, cols, g.kinds[t])
    for l in g.links():
        bp.add_link(*l)
    return g, plain, bp, n


def test_bitpacked_queries_equal_int32(stars):
    from paper_2306_08367_b200 import query as Q
    g, plain, bp, n = stars
    for (gr, qi), d in DIALS.items():
        q = Q.spec_with_dial(Q.group_defs(gr)[qi], gr, d)
        want = plain.prepare(q).execute().cpu().numpy()
        got = bp.prepare(q).execute().cpu().numpy()
        assert np.array_equal(got, want), (gr, qi)


def test_bitpacked_ragged_ranges(stars):
    from paper_2306_08367_b200 import query as Q
    g, plain, bp, n = stars
    for (gr, qi), d in ((1, 0), 222), ((2, 0), 500), ((4, 0), 50):
        q = Q.spec_with_dial(Q.group_defs(gr)[qi], gr, d)
        pa, pb = plain.prepare(q), bp.prepare(q)
        pa.build_codes()
        pb.build_codes()
        for row0, rows in ((0, n), (32, n - 32), (0, 1), (64, 33), (0, 606_209), (1_000_000 - 1_000_000 % 32, 1_234_567),
                           (n - n % 32, n % 32), (96, 0)):
            want = pa.scan_range(row0, rows).cpu().numpy().copy()
            got = pb.scan_range(row0, rows).cpu().numpy()
            assert np.array_equal(got, want), (gr, qi, row0, rows)


def test_bitpacked_rejects_unaligned_range(stars):
    from paper_2306_08367_b200 import errors, query as Q
    g, plain, bp, n = stars
    p = bp.prepare(Q.spec_with_dial(Q.group_defs(1)[0], 1, 222))
    p.build_codes()
    with pytest.raises(errors.ShapeError):
        p.scan_range(4, 100)
