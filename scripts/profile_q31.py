"""ncu driver: one SF=100 Q3.1 scan (the direct kernel with the uint8 supplier table)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2306_08367_b200 import gen, star  # noqa: E402

g = gen.gen_star("Ssb", int(os.environ.get("LAQ_SF", "100")), 42, narrow=True, max_bytes=64 << 30)
ds = star.upload_gen_star(g)
q = ds.gen_queries(3)[0]
p = ds.prepare(q)
p.build_codes()
p.scan()
torch.cuda.synchronize()
print(q.id, p.bytes_per_row, p.scanned_links)
