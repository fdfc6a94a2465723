"""The general (sort-based) device paths that use CUB primitives, timed at
scale against the HBM roofline: rows a1 (build_key_domain on wide int64 keys:
radix sort + unique), a4 (key_matrix DomainByRows: stable sort of positions),
a19 (groupby_sum_multi: tuple sort + run-length + row-ordered segmented sums),
with the same work done by the dense (bitmap / direct-id) paths beside them.
alg_GBs counts one read of the inputs and one write of the outputs; a radix
sort moves several times that, which is what the gap to the HBM peak shows.

  python scripts/sortpath_bench.py [n=60000000]
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2306_08367_b200 import ops  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 60_000_000


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    out = {"n": n}
    wide = torch.randint(0, 1 << 40, (n,), dtype=torch.int64, device="cuda", generator=g)
    dense = torch.randint(0, 1 << 20, (n,), dtype=torch.int64, device="cuda", generator=g)
    s = torch.arange(1 << 10, dtype=torch.int64, device="cuda")
    for name, keys in (("a1 build_key_domain wide int64 (CUB radix sort + unique)", wide),
                       ("a1 build_key_domain dense (bitmap kernels)", dense)):
        ms = timed(lambda: ops.build_key_domain(keys, s))
        out[name] = {"ms": ms, "alg_GBs": 8 * n / ms / 1e6}
    # a4 on the device buffers (the C-ABI calls under ops.key_matrix, without
    # the Python mirror's host copies of the CSR)
    import ctypes as C
    from paper_2306_08367_b200.device import context
    ctx = context()
    d = ops.build_key_domain(dense, s).sorted_keys
    d = d if isinstance(d, torch.Tensor) else torch.from_numpy(d).cuda()
    nd = d.numel()
    pos = torch.empty(n, dtype=torch.int64, device="cuda")
    ms = timed(lambda: ctx.check(ctx.lib.laq_key_positions(ctx.h, dense.data_ptr(), n, d.data_ptr(), nd,
                                                             pos.data_ptr())))
    out["a4 key_matrix RowsByDomain, contiguous domain (laq_key_positions: key - base)"] = {
        "ms": ms, "alg_GBs": 16 * n / ms / 1e6}
    even = dense * 2  # every other key: a domain with gaps -> probe-table gathers
    de = ops.build_key_domain(even, s).sorted_keys
    de = de if isinstance(de, torch.Tensor) else torch.from_numpy(de).cuda()
    ms = timed(lambda: ctx.check(ctx.lib.laq_key_positions(ctx.h, even.data_ptr(), n, de.data_ptr(), de.numel(),
                                                             pos.data_ptr())))
    out["a4 key_matrix RowsByDomain, domain with gaps (laq_key_positions: probe gather)"] = {
        "ms": ms, "alg_GBs": 16 * n / ms / 1e6}
    row_ptr = torch.empty(nd + 1, dtype=torch.int64, device="cuda")
    col = torch.empty(n, dtype=torch.int64, device="cuda")
    ov = torch.empty(n, dtype=torch.float64, device="cuda")
    nnz = C.c_int64()
    ms = timed(lambda: ctx.check(ctx.lib.laq_key_matrix_dbr(ctx.h, dense.data_ptr(), n, d.data_ptr(), nd, None,
                                                              row_ptr.data_ptr(), col.data_ptr(), ov.data_ptr(),
                                                              C.byref(nnz))))
    out["a4 key_matrix DomainByRows (CUB stable radix sort of positions)"] = {"ms": ms,
                                                                           "alg_GBs": (8 + 16) * n / ms / 1e6}
    cols = [torch.randint(0, 7, (n,), dtype=torch.int64, device="cuda", generator=g),
            torch.randint(0, 25, (n,), dtype=torch.int64, device="cuda", generator=g),
            torch.randint(0, 40, (n,), dtype=torch.int64, device="cuda", generator=g)]
    vals = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
    ms = timed(lambda: ops.groupby_sum_multi(cols, vals))
    out["a19 groupby_sum_multi 3 cols, 7000 groups (CUB sort + RLE + segsum)"] = {"ms": ms,
                                                                                 "alg_GBs": 32 * n / ms / 1e6}
    # a7 mm_join on the device buffers: 60M R keys x 1M S keys over a 1M domain (~60M pairs)
    sk = torch.randint(0, 1 << 20, (1 << 20,), dtype=torch.int64, device="cuda", generator=g)
    orr = torch.empty(2 * n, dtype=torch.int64, device="cuda")
    oss = torch.empty(2 * n, dtype=torch.int64, device="cuda")
    nnz = C.c_int64()
    ms = timed(lambda: ctx.check(ctx.lib.laq_mm_join(ctx.h, dense.data_ptr(), n, sk.data_ptr(), sk.numel(),
                                                       orr.data_ptr(), oss.data_ptr(), 2 * n, C.byref(nnz))))
    out["a7 mm_join 60M x 1M keys (bucket sort of S + probe + pair writes)"] = {
        "ms": ms, "pairs": int(nnz.value), "alg_GBs": (8 * n + 8 * sk.numel() + 16 * nnz.value) / ms / 1e6}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
