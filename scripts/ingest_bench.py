"""Ingest throughput: the reference writes an SSB dataset
(write_dataset, cli.cpp:430-481); lineorder.csv is parsed on the device
(csv.cu: line index + parse) and by the reference's load_csv (1 host thread).
Prints one JSON line; bytes are the CSV text bytes."""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import ref as R  # noqa: E402
from paper_2306_08367_b200 import ingest  # noqa: E402
from paper_2306_08367_b200.device import context  # noqa: E402

sf = int(os.environ.get("SF", "1"))
d = tempfile.mkdtemp(prefix="laq_ingest_")
t0 = time.time()
R.write_dataset(d, "Ssb", sf, 42)
gen_s = time.time() - t0
man = json.load(open(os.path.join(d, "manifest.json")))
tj = [t for t in man["tables"] if t["name"] == "lineorder"][0]
schema = ingest.schema_from_json(tj["schema"])
path = os.path.join(d, tj["file"])
data = open(path, "rb").read()
nbytes = len(data)
ctx = context(0)
dev = torch.zeros(nbytes + 16, dtype=torch.uint8, device="cuda")
dev[:nbytes] = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()
rows = C.c_int64()
cols = {n: torch.empty(tj["rows"], dtype=torch.float64 if k == 2 else torch.int64, device="cuda") for n, k in schema}
kinds = (C.c_int32 * len(schema))(*[k for _, k in schema])
ptrs = (C.c_void_p * len(schema))(*[cols[n].data_ptr() for n, _ in schema])


def device_parse():
    h = C.c_void_p()
    ctx.check(ctx.lib.laq_csv_open(ctx.h, dev.data_ptr(), nbytes, C.byref(h), C.byref(rows)))
    ctx.check(ctx.lib.laq_csv_parse(ctx.h, h, len(schema), kinds, ptrs))
    ctx.lib.laq_csv_close(h)


for _ in range(2):
    device_parse()
torch.cuda.synchronize()
reps = 5
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    device_parse()
e1.record()
torch.cuda.synchronize()
dev_ms = e0.elapsed_time(e1) / reps
# e2e: host file bytes -> device -> parsed columns (ingest.load_csv, no cache)
t0 = time.time()
got = ingest.load_csv(path, schema)
torch.cuda.synchronize()
e2e_s = time.time() - t0
# reference load_csv on a bounded sample (first ~1M lines), 1 thread
sample = b"".join(data.splitlines(keepends=True)[:1_000_000])
sp = os.path.join(d, "sample.csv")
open(sp, "wb").write(sample)
t0 = time.time()
ref_cols, ref_rows = R.load_csv(sp, [k for _, k in schema], cap=1_000_001)
ref_s = time.time() - t0
ok = all(np.array_equal(got[n].cpu().numpy()[:ref_rows], ref_cols[i]) for i, (n, _) in enumerate(schema))
print(json.dumps({
    "workload": f"SSB SF={sf} lineorder.csv ({tj['rows']} rows, {len(schema)} int columns, {nbytes} bytes)",
    "device_parse_ms": round(dev_ms, 3), "device_gbs": round(nbytes / dev_ms / 1e6, 1),
    "device_rows_per_s": tj["rows"] / (dev_ms / 1e3),
    "e2e_load_csv_s": round(e2e_s, 3), "e2e_gbs": round(nbytes / e2e_s / 1e9, 2),
    "reference_load_csv_1thread": {"sample_bytes": len(sample), "s": round(ref_s, 3),
                                   "gbs": round(len(sample) / ref_s / 1e9, 3), "rows_per_s": ref_rows / ref_s},
    "parity_sample_rows": ref_rows, "parity_ok": bool(ok), "gen_write_s": round(gen_s, 1)}))
