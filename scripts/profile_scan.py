"""Profiling driver: the six bench queries (SSB SF=10 Q1.1-Q2.3, the dials the
device tuner picks for seed 42) each scanned once, for ncu capture:

  ncu --set full --clock-control none --import-source on -k regex:scan_pipe -c 6 \
      -o gpurun_out/scan python scripts/profile_scan.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2306_08367_b200 import gen, query as Q, star  # noqa: E402

DIALS = {(1, 0): 222, (1, 1): 200, (1, 2): 133, (2, 0): 500, (2, 1): 199, (2, 2): 516}


def main():
    sf = int(os.environ.get("LAQ_SF", "10"))
    g = gen.gen_star("Ssb", sf, 42, narrow=True)
    ds = star.upload_gen_star(g)
    plans = [ds.prepare(Q.spec_with_dial(Q.group_defs(gr)[qi], gr, d)) for (gr, qi), d in DIALS.items()]
    for p in plans:
        p.build_codes()
    torch.cuda.synchronize()
    if os.environ.get("LAQ_PROFILE_SHARED") == "1":  # the bench's shared passes (one per query group)
        star.scan_shared(plans[:3], [p.acc for p in plans[:3]])
        star.scan_shared(plans[3:], [p.acc for p in plans[3:]])
    else:
        for p in plans:
            p.scan()
    torch.cuda.synchronize()
    for p in plans:
        print(p.q.id, "pipe" if p.bytes_per_row else "", p.emit(p.acc.cpu().numpy())[:2].tolist())


if __name__ == "__main__":
    main()
