"""Break the bench's e2e step (host int64 columns -> laq_star_add_table ->
laq_run_query x6) into its parts on the GPU box."""
import os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2306_08367_b200 import gen, query as Q, star  # noqa: E402
from paper_2306_08367_b200.device import context  # noqa: E402

ctx = context(0)
g = gen.gen_star("Ssb", 100, 42, narrow=True, max_bytes=64 << 30)
if os.environ.get("E2E_PROBE_MAIN_DS") == "1":  # hold the bench's resident device star as well
    main_ds = star.upload_gen_star(g, ctx=ctx)
    torch.cuda.synchronize()
dials = {3: (105, 79, 43), 4: (249, 199, 284)}
qs = [Q.spec_with_dial(d, grp, x) for grp in (3, 4) for d, x in zip(Q.group_defs(grp), dials[grp])]
used = sorted({c for q in qs for c in ({l.fact_fk for l in q.joins} | {q.measure})})
dims = {l.dim_name for q in qs for l in q.joins}
host, cud = {}, torch.cuda.cudart()
for t, cols in g.tables.items():
    if t != "lineorder" and t not in dims:
        continue
    keep = used if t == "lineorder" else [c for c in cols if cols[c].dtype != np.float64]
    host[t] = {}
    for c in keep:
        a = np.ascontiguousarray(cols[c], np.int64)
        cud.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
        host[t][c] = a
kinds = {t: {c: g.kinds[t][c] for c in host[t]} for t in host}
links = [l for l in g.links() if l[0] in host["lineorder"] and l[1] in host]
nbytes = sum(a.nbytes for cols in host.values() for a in cols.values())
for it in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    ds = star.DeviceStar.from_tables(host, kinds, links, ctx=ctx)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    out = [ds.run_query(q) for q in qs]
    torch.cuda.synchronize(); t2 = time.perf_counter()
    ds.close()
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"upload {1e3*(t1-t0):.1f} ms ({nbytes/(t1-t0)/1e9:.1f} GB/s)  queries {1e3*(t2-t1):.1f} ms  close {1e3*(t3-t2):.1f} ms", flush=True)
