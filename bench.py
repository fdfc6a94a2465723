"""Benchmark: SSB SF=100 Q3.1-Q4.3 as join-MM + group-by aggregation, lineorder
row-sharded over the GPUs (BASELINE.json configs[3], the metric's "SSB SF=100
query ms at 1/2/4/8"), plus the fused join+predict line (configs[0], the
metric's "fused join+predict fact-rows/sec").

  python bench.py [--gpus N --steps K --warmup W] [--impl laq|reference]
                  [--workload q3q4|q1q2]

One JSON line on rank 0 (contract in the task brief).

A "step" = the six queries over the WHOLE 600M-row lineorder: per query the
code tables are rebuilt from the dimension filters, one fused scan of the
rank's contiguous row shard (gen row_range: every rank draws the canonical
stream and keeps rows [r*n/N, (r+1)*n/N)), one int64 all-reduce of the
per-group (count, sum) accumulators through the C-ABI's own NCCL communicator
(laq_ctx_attach_nccl / laq_allreduce_acc), D2H, host emission of the result
rows.  Strong scaling: the total work is fixed, N GPUs split it.

Timing: CUDA events on the launch stream, barrier + synchronize on both sides,
max over ranks.  Every query streams >= 7.2 GB / N of fact columns, far above
the 126 MB L2, so no flush is needed.

Parity, inside the run (any mismatch fails the run):
  * every rank's emitted rows == the whole-table CPU check: oracle/fast_query
    (C restatement of run_query_oracle, pinned to the reference's goldens)
    over each rank's shard, the per-group partials all-reduced -- and == the
    committed whole-table goldens tests/golden/ssb_sf100.json;
  * N=1: the reference's own run_query_laq (oracle/_ref) on the first
    SAMPLE_ROWS rows of the SAME arrays == the device scan of those rows; the
    same reference run is the cpu_baseline.

--impl reference: the reference's own CPU path (oracle/_ref, compiled from
/root/reference/proj): data from the reference generator (bench::gen_star),
each step = the six queries' stock single-threaded run_query_laq, run
concurrently (one host thread per query), on lineorder rows [0, SAMPLE_ROWS)
-- the sample the GPU arm checks against.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "q3q4": {"queries": [(3, 0), (3, 1), (3, 2), (4, 0), (4, 1), (4, 2)], "sf": 100, "cfg": 3,
             "golden": "ssb_sf100.json"},
    "q1q2": {"queries": [(1, 0), (1, 1), (1, 2), (2, 0), (2, 1), (2, 2)], "sf": 10, "cfg": 1,
             "golden": "ssb_sf10.json"},
}
SEED = 42
SAMPLE_ROWS = 3_000_000  # the reference arm's per-step sample (= golden "sample")
UNIT = "fact-rows/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="laq", choices=["laq", "reference"])
    ap.add_argument("--workload", default="q3q4", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fused", action="store_true", help="skip the cfg1 fused join+predict line")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--secondary", action="store_true", help="q1q2 only: cfg3 FFN line")
    return ap.parse_args()


class Workload:
    def __init__(self, name):
        w = WORKLOADS[name]
        self.name = name
        self.pairs = w["queries"]
        self.sf = w["sf"]
        self.rows = self.sf * 6_000_000  # benchgen.cpp:182 (Ssb lineorder)
        self.qnames = [f"Q{g}.{i + 1}" for g, i in self.pairs]
        self.cfg_index = w["cfg"]
        path = os.path.join(ROOT, "tests", "golden", w["golden"])
        self.golden = json.load(open(path)) if os.path.exists(path) else None
        self.dials = [q["dial"] for q in self.golden["queries"]] if self.golden else None
        self.metric = (f"SSB SF={self.sf} {self.qnames[0]}-{self.qnames[-1]} fact-rows/sec "
                       "(join-MM + group-by aggregation)")

    def specs(self, dials=None):
        from paper_2306_08367_b200 import query as Q
        dials = dials or self.dials
        return [Q.spec_with_dial(Q.group_defs(g)[i], g, int(d)) for (g, i), d in zip(self.pairs, dials)]

    def config(self):
        """Identical in both arms (the driver compares them)."""
        return {"workload": f"SSB SF={self.sf} {self.qnames[0]}-{self.qnames[-1]} (BASELINE configs"
                            f"[{self.cfg_index}]), {self.rows} lineorder rows, seed {SEED}",
                "queries": self.qnames, "dials": self.dials,
                "l2": "every query streams >= 0.96 GB of fact columns per GPU > 126 MB L2: no flush needed"}


def dist_env():
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), \
        int(os.environ.get("LOCAL_RANK", "0"))


class Clocks:
    """SM clock + throttle-reason sampling (NVML, the library nvidia-smi reads)
    every 10 ms; the report uses the samples inside the timed region
    (B200_PROFILING.md recipe)."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self.marks = []
        self._stop = threading.Event()
        self.ok = False

    def start(self):
        try:
            import pynvml as N
            N.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.gpu]) if vis and vis.split(",")[self.gpu].isdigit() else self.gpu
            self.N, self.h = N, N.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            return
        self.t = threading.Thread(target=self._loop, daemon=True)
        self.t.start()

    def _loop(self):
        N = self.N
        while not self._stop.is_set():
            try:
                self.samples.append((time.perf_counter(), N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM),
                                     N.nvmlDeviceGetCurrentClocksEventReasons(self.h)))
            except Exception:
                pass
            time.sleep(0.01)

    def mark(self):
        self.marks.append(time.perf_counter())

    def stop(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        self._stop.set()
        self.t.join(timeout=2)
        N = self.N
        t0, t1 = (self.marks[0], self.marks[-1]) if len(self.marks) >= 2 else (0, 1e30)
        inside = [s for s in self.samples if t0 <= s[0] <= t1]
        use = inside if inside else self.samples
        names = {N.nvmlClocksEventReasonHwSlowdown: "hw_slowdown",
                 N.nvmlClocksEventReasonHwThermalSlowdown: "hw_thermal_slowdown",
                 N.nvmlClocksEventReasonSwThermalSlowdown: "sw_thermal_slowdown",
                 N.nvmlClocksEventReasonSwPowerCap: "sw_power_cap"}
        reasons = sorted({v for _, _, m in use for k, v in names.items() if m & k})
        return {"sm_mhz": float(np.median([s[1] for s in use])) if use else None, "sm_max_mhz": float(self.max_mhz),
                "reasons": reasons, "samples": len(use),
                "window": "timed region" if inside else "warm-up + timed region (timed region < 10 ms)"}


def parallel(fns):
    """Run callables on host threads (ctypes calls into oracle/_ref release the GIL)."""
    out = [None] * len(fns)

    def run(i):
        out[i] = fns[i]()
    th = [threading.Thread(target=run, args=(i,)) for i in range(len(fns))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return out


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "MEASURED_PEAKS.json"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 2250.0}, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------

def run_reference(args, W: Workload, world, rank):
    if rank != 0:
        return
    from oracle import ref
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/liblaq_ref.so was not built"}))
        return
    t0 = time.perf_counter()
    full = ref.gen_star("Ssb", W.sf, SEED, max_bytes=64 << 30)  # the reference generator (benchgen.cpp:103-161)
    gen_s = time.perf_counter() - t0
    m = min(SAMPLE_ROWS, W.rows)
    tables = [("lineorder", {c: a[:m] for c, a in full.fact.items()})]
    tables += [(t, dict(cols)) for t, cols in full.tables.items() if t != "lineorder"]
    links = [("lo_part", "part", "p_key"), ("lo_supplier", "supplier", "s_key"), ("lo_orderdate", "date", "d_key"),
             ("lo_commitdate", "date", "d_key"), ("lo_customer", "customer", "c_key")]
    rs = ref.star_from_tables(tables, links)
    del full, tables
    queries = W.specs()
    step_s, results = [], None
    for it in range(args.warmup + args.steps):
        t = time.perf_counter()
        results = parallel([lambda q=q: ref.run_query(rs, q) for q in queries])
        if it >= args.warmup:
            step_s.append(time.perf_counter() - t)
    ms = 1e3 * float(np.mean(step_s))
    value = len(queries) * m / (ms / 1e3)
    parity = None
    if W.golden and "sample" in W.golden:
        want = [np.array([float.fromhex(h) for h in s["result"]]).reshape(s["rows"], s["cols"])
                for s in W.golden["sample"]]
        parity = all(np.array_equal(r[0], w) for r, w in zip(results, want))
    cores = len(queries)
    line = {"metric": W.metric, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int64", "impl": "reference",
            "data": "synthetic: the reference's own generator (bench::gen_star, seed 42) through oracle/_ref",
            "config": W.config(),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                             "sample": f"lineorder rows [0, {m}) of the SF={W.sf} table (full dimension tables); "
                                       f"each step runs the {len(queries)} queries' stock single-threaded "
                                       f"run_query_laq (cli.cpp:73-138) concurrently, one host thread per query"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "details": {"per_query_s": [round(float(r[1]), 4) for r in results], "gen_s": round(gen_s, 1),
                        "sample_matches_golden": parity, "host_cores": os.cpu_count()}}
    if not args.no_fused:
        fk, pk, feats, Wm = ref.cfg1_inputs(1_000_000, 10_000, 16, 1)  # the reference's Rng / gen_linear
        best = None
        for _ in range(3):
            y, secs = ref.fused_pipeline([fk], [pk], [feats], Wm)
            best = secs if best is None or sum(secs) < sum(best) else best
        line["fused_join_predict"] = {
            "metric": "fused join+predict fact-rows/sec (BASELINE configs[0]: 1M-row fact x 10K dim, k=16, l=1)",
            "value": 1e6 / float(sum(best)), "unit": UNIT, "cores": 1,
            "stages_s": {"multiway_star_join": best[0], "csr_from_coo": best[1], "prefuse_linear": best[2],
                         "apply_fused_linear": best[3]},
            "apply_only_rows_per_s": 1e6 / float(best[3])}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def main():
    args = parse()
    W = Workload(args.workload)
    world, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, W, world, rank)
        return

    import torch
    # LAQ_BENCH_SHARE_GPU=1 (test hook): every rank on cuda:0 over gloo (the
    # C-ABI context then all-reduces through a host hook); the real run is one
    # rank per GPU with the context's own NCCL communicator.
    share = os.environ.get("LAQ_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))

    from paper_2306_08367_b200 import dist as D, gen, query as Q, star
    from paper_2306_08367_b200.device import context

    ctx = context(local)
    if dist is not None:
        D.attach(ctx)  # NCCL communicator inside liblaq_b200.so (gloo hook when sharing a GPU)
    stream = torch.cuda.current_stream()
    ctx.bind_stream(stream)

    def reduce_max(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def reduce_min_flag(ok):
        if dist is None:
            return bool(ok)
        t = torch.tensor([1 if ok else 0], dtype=torch.int64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return bool(t.item())

    rr = D.shard_range(W.rows, rank, world)
    t0 = time.perf_counter()
    g = gen.gen_star("Ssb", W.sf, SEED, narrow=True, max_bytes=64 << 30, row_range=rr)
    gen_s = time.perf_counter() - t0
    n_local = rr[1] - rr[0]
    ds = star.upload_gen_star(g, ctx=ctx)

    # Dials: gen_queries' constants for this table (pinned in the golden file);
    # the device tuner re-derives them here (measure_selectivity is all-reduced
    # inside the C-ABI, so every rank tunes on the whole table).
    t0 = time.perf_counter()
    tuned = []
    for grp in sorted({gr for gr, _ in W.pairs}):
        tuned += [int(q.filters[-1].pred.lo) for q in Q.gen_queries(ds.measure_selectivity, grp)]
    tune_s = time.perf_counter() - t0
    if W.dials is None:
        W.dials = tuned
    dials_match = tuned == W.dials
    queries = W.specs()
    plans = [ds.prepare(q) for q in queries]
    sizes = [2 * p.n_groups for p in plans]
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    # Batched scans: each query group (the same fact columns, different dials)
    # is ONE pass with one dictionary-encoded probe per dimension link for the
    # whole group (laq_batch_*, csrc/ssb_batch.cuh); a group the fused pass
    # cannot take is scanned query by query with the same results.
    groups = []
    for qi, q in enumerate(queries):
        if groups and queries[groups[-1][0]].group == q.group and len(groups[-1]) < 4:
            groups[-1].append(qi)
        else:
            groups.append([qi])
    batches = [star.Batch([plans[qi] for qi in grp]) for grp in groups]
    shared_flags = [b.fused for b in batches]
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in groups]
          for _ in range(args.steps)]
    accs = [torch.zeros(int(offs[-1]), dtype=torch.int64, device="cuda") for _ in range(2)]
    acc_hosts = [torch.zeros(int(offs[-1]), dtype=torch.int64, pin_memory=True) for _ in range(2)]
    done = [torch.cuda.Event(), torch.cuda.Event()]

    # Serving loop: step k+1 is enqueued before step k's rows are emitted on the
    # host (double-buffered accumulators), so host emission overlaps device work.
    def launch(k, i=None):
        b = k & 1
        accs[b].zero_()
        for gi, grp in enumerate(groups):
            batches[gi].build()  # the group's code tables (dimension filters) + link dictionaries
            if i is not None:
                ev[i][gi][0].record(stream)
            batches[gi].scan([accs[b][offs[qi]: offs[qi + 1]] for qi in grp], accumulate=True)
            if i is not None:
                ev[i][gi][1].record(stream)
        ctx.allreduce_acc(accs[b])  # C-ABI: ncclAllReduce on the context stream (no-op at N=1)
        acc_hosts[b].copy_(accs[b], non_blocking=True)
        done[b].record(stream)

    def collect(k):
        b = k & 1
        done[b].synchronize()
        a = acc_hosts[b].numpy()
        return [p.emit(a[offs[qi]: offs[qi + 1]]) for qi, p in enumerate(plans)]

    def run(n, timed):
        out = None
        for k in range(n):
            launch(k, k if timed else None)
            if k:
                out = collect(k - 1)
        return collect(n - 1) if n else out

    clocks = Clocks(local)
    clocks.start()
    run(args.warmup, False)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.launches
    clocks.mark()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    prof = os.environ.get("LAQ_PROFILE_TIMED") == "1"  # ncu --profile-from-start off: the timed steps only
    if prof:
        torch.cuda.cudart().cudaProfilerStart()
    t_start.record(stream)
    results = run(args.steps, True)
    t_end.record(stream)
    torch.cuda.synchronize()
    if prof:
        torch.cuda.cudart().cudaProfilerStop()
    clocks.mark()
    clk = clocks.stop()
    launches = ctx.launches - launches0
    ms_step = reduce_max(t_start.elapsed_time(t_end)) / args.steps
    value = len(plans) * W.rows / (ms_step / 1e3)  # whole-job fact rows per second

    # ---- roofline of the scan kernel (the dominant kernel), rank 0's shard ----
    scan_ms = np.array([[ev[i][gi][0].elapsed_time(ev[i][gi][1]) for gi in range(len(groups))]
                        for i in range(args.steps)]).mean(axis=0)
    bytes_per_launch = np.array([batches[gi].bytes_per_row * n_local for gi in range(len(groups))], dtype=np.float64)
    achieved = float(bytes_per_launch.sum() / (scan_ms.sum() / 1e3) / 1e9)
    pk, pk_src = peaks()
    peak = float(pk["hbm_gbs"])
    traffic, traffic_src = ncu_traffic(W.name)

    # ---- parity 1: whole table, every rank, vs the C checker + goldens ----
    from oracle import fast_query as F
    t0 = time.perf_counter()
    threads = max(1, (os.cpu_count() or 1) // world)
    full_ok, want_rows = True, []
    for q, got in zip(queries, results):
        p = F.Prepared(g.tables, q)
        cnt, s = p.partial(0, n_local, threads)
        if dist is not None:
            t = torch.from_numpy(np.concatenate([cnt, s])).cuda()
            dist.all_reduce(t)
            cs = t.cpu().numpy()
            cnt, s = cs[: len(cnt)], cs[len(cnt):]
        want = p.emit(cnt, s)
        want_rows.append(want)
        full_ok = full_ok and got.shape == want.shape and np.array_equal(got, want)
    full_ok = reduce_min_flag(full_ok)
    check_s = time.perf_counter() - t0
    golden_ok = None
    if W.golden and W.golden.get("lineorder_rows") == W.rows:
        gq = W.golden["queries"]
        golden_ok = all(np.array_equal(r.ravel(), np.array([float.fromhex(h) for h in x["result"]]))
                        and r.shape == (x["rows"], x["cols"]) for r, x in zip(results, gq))
    if not (full_ok and golden_ok is not False):
        raise SystemExit(f"PARITY FAILURE: whole-table check {full_ok}, golden {golden_ok}")

    # ---- parity 2 (N=1): the reference itself on the same arrays, sample rows ----
    cpu = None
    sample = None
    if world == 1 and not args.no_cpu_baseline:
        cpu, sample = reference_sample(g, queries, plans, ctx)
        if sample is not None and not sample["match"]:
            raise SystemExit("PARITY FAILURE: device != reference run_query_laq on the sample rows")

    # ---- e2e: the reference-facing C-ABI call with HOST buffers ----
    e2e = None
    if not args.no_e2e:
        e2e = e2e_bench(args, g, queries, results, ctx, dist, reduce_max, len(plans) * W.rows)

    fused = None
    if rank == 0 and world == 1 and not args.no_fused:
        fused = fused_predict_bench(ctx)
    secondary = None
    if rank == 0 and world == 1 and args.secondary and W.name == "q1q2":
        secondary = {"cfg3": ffn_bench(ctx, W, g)}

    if rank == 0:
        per_launch = [round(float(x), 4) for x in scan_ms]
        out = {
            "metric": W.metric, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int32",
            "data": "synthetic: the reference generator (benchgen.cpp, seed 42) restated bit-exactly; every rank "
                    "draws the canonical lineorder stream and keeps its contiguous row shard",
            "config": W.config(),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": None if traffic is None else float(sum(traffic) / len(traffic)),
                         "traffic_per_launch": traffic, "traffic_source": traffic_src,
                         "kernel": "scan_batch_kernel (K4 batched: one pass per query group, csrc/ssb_batch.cu)",
                         "algorithmic_bytes_per_launch": [int(b) for b in bytes_per_launch],
                         "unit_bytes": "the union of the group's touched fact columns x 4 B per row, read once per group (Q3.x: "
                                       "lo_supplier, lo_orderdate, lo_revenue = 12 B; Q4.x: + lo_part, lo_commitdate "
                                       "= 20 B; SURVEY §8d)",
                         "peak_source": pk_src + " hbm_gbs (copy bandwidth, burst)",
                         "frac_vs_nominal_7700": achieved / 7700.0},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
            "parity": {"whole_table_vs_cpu_checker": full_ok, "whole_table_vs_golden": golden_ok,
                       "sample_vs_reference": None if sample is None else sample["match"],
                       "sample_rows": None if sample is None else sample["rows"],
                       "dials_retuned_on_device_match": dials_match, "check_s": round(check_s, 2)},
            "details": {"per_query_scan_ms": dict(zip(["+".join(W.qnames[qi] for qi in grp) for grp in groups],
                                                      per_launch)),
                        "batched_scan": [bool(f) for f in shared_flags],
                        "batch_not_fused_why": [b.why for b in batches if not b.fused],
                        "result_rows": [int(r.shape[0]) for r in results],
                        "lineorder_rows_per_gpu": n_local,
                        "parallelism": f"row-sharded x{world}, int64 accumulators all-reduced through the "
                                       f"C-ABI: {ctx.transport}" if world > 1 else "1 GPU",
                        "gen_s": round(gen_s, 1), "device_tuning_s": round(tune_s, 2)},
            "fused_join_predict": fused,
        }
        if secondary:
            out["secondary"] = secondary
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.barrier()
        ctx.set_allreduce_host(1, 0, None)
        dist.destroy_process_group()


def reference_sample(g, queries, plans, ctx):
    """The reference's run_query_laq (oracle/_ref, 1 thread per query, the six
    concurrently) on lineorder rows [0, SAMPLE_ROWS) of the same arrays the GPU
    holds, against the device scan of exactly those rows."""
    import torch
    from oracle import ref
    if not ref.available():
        return None, None
    m = min(SAMPLE_ROWS, len(g.fact["lo_part"]))
    tables = [("lineorder", {c: np.asarray(a[:m], np.int64) for c, a in g.fact.items()})]
    tables += [(t, {c: np.asarray(a, np.int64) if a.dtype != np.float64 else a for c, a in cols.items()})
               for t, cols in g.tables.items() if t != "lineorder"]
    rs = ref.star_from_tables(tables, g.links())
    parallel([lambda q=q: ref.run_query(rs, q) for q in queries])  # warm-up
    t0 = time.perf_counter()
    res = parallel([lambda q=q: ref.run_query(rs, q) for q in queries])
    wall = time.perf_counter() - t0
    match = True
    for p, (want, _) in zip(plans, res):
        acc = torch.zeros(2 * p.n_groups, dtype=torch.int64, device="cuda")
        p.scan_range(0, m, acc)
        match = match and np.array_equal(p.emit(acc.cpu().numpy()), want)
    cpu = {"value": len(queries) * m / wall, "unit": UNIT, "cores": len(queries), "kind": "reference",
           "sample": f"the reference's run_query_laq (oracle/_ref) on lineorder rows [0, {m}) of the same arrays, "
                     f"full dimension tables; the {len(queries)} queries concurrently, one host thread each "
                     f"({wall:.2f} s); per-query s {[round(r[1], 2) for r in res]}"}
    return cpu, {"match": bool(match), "rows": m}


def e2e_bench(args, g, queries, results, ctx, dist, reduce_max, total_rows):
    """Per step, through the C-ABI with HOST buffers (what the drop-in
    run_query_laq does for a StarSchema it has not cached): the rank's int64
    columns -- the reference's IntColumn layout -- go H2D from pinned memory
    (laq_star_add_table, narrowed to int32 on the device), then laq_run_query
    per query (prepare + scan + all-reduce + D2H of the accumulators + emit)."""
    import torch
    from paper_2306_08367_b200 import star
    used = sorted({c for q in queries for c in _fact_cols(q)})
    dims = {l.dim_name for q in queries for l in q.joins}
    # The int64 columns live in page-locked buffers from cudaHostAlloc (torch
    # pin_memory), filled once outside the timed region.  (With numpy arrays
    # registered through cudaHostRegister -- return code unchecked -- the step
    # measured 0.52-1.46 s on different boxes, i.e. 16-46 GB/s for 24 GB.)
    host, pinned = {}, []
    for t, cols in g.tables.items():
        if t != "lineorder" and t not in dims:
            continue
        keep = used if t == "lineorder" else [c for c in cols if cols[c].dtype != np.float64]
        host[t] = {}
        for c in keep:
            buf = torch.empty(len(cols[c]), dtype=torch.int64, pin_memory=True)
            a = buf.numpy()
            a[:] = cols[c]
            pinned.append(buf)
            host[t][c] = a
    kinds = {t: {c: g.kinds[t][c] for c in host[t]} for t in host}
    h2d = sum(a.nbytes for cols in host.values() for a in cols.values())
    links = [l for l in g.links() if l[0] in host["lineorder"] and l[1] in host]

    def step():
        ds = star.DeviceStar.from_tables(host, kinds, links, ctx=ctx)
        out = [ds.run_query(q) for q in queries]
        ds.close()
        return out

    for _ in range(max(1, min(args.warmup, 2))):
        res = step()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        res = step()
    e1.record()
    torch.cuda.synchronize()
    ms = reduce_max(e0.elapsed_time(e1)) / args.steps
    del pinned
    if not all(np.array_equal(a, b) for a, b in zip(res, results)):
        raise SystemExit("PARITY FAILURE: e2e results differ from the device run")
    d2h = sum(2 * 8 * max(1, r.shape[0]) for r in results)
    return {"value": total_rows / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": ms,
            "path": "per step: laq_star_add_table (int64 host columns, pinned -> HBM, device narrowing) + "
                    "laq_run_query x6 (C-ABI; NCCL all-reduce inside when N > 1); results == the device run",
            "d2h_note": "laq_run_query copies each query's (count, sum) accumulator D2H; counted as 16 B per "
                        "emitted row (lower bound)"}


def _fact_cols(q):
    cols = {l.fact_fk for l in q.joins} | {q.measure}
    cols |= {f.column for f in q.filters if f.target == -1}
    cols |= {g.column for g in q.group_by if g.target == -1}
    return cols


def ncu_traffic(workload):
    """DRAM bytes (read + write) per batched-pass launch from the committed ncu
    --set full capture of this workload's passes (profiles/<round>/
    batch_scan_ncu.json; one entry per query group).  Returns (per-launch
    list, source) or (None, None) when no capture of this workload exists."""
    import glob
    if workload != "q3q4":
        return None, None
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "batch_scan_ncu.json")))
    if not files:
        return None, None
    rows = json.load(open(files[-1]))
    unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = []
    for r in rows:
        b = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            v, u = r[k].split()
            b += float(v) * unit[u]
        tot.append(b)
    return tot, os.path.relpath(files[-1], ROOT)


def fused_predict_bench(ctx):
    """configs[0]: 1M-row fact x 10K-row dim, 16 features, l=1 fused join +
    linear predict (probe + gather-sum, fp64, bit-exact vs the reference's
    fused_pipeline on the same arrays); 1e8 rows for the roofline (1M rows is
    launch-bound); e2e with host buffers."""
    import torch
    from paper_2306_08367_b200 import fusion, gen
    fk, pk, feats, W = gen.cfg1_inputs(1_000_000, 10_000, 16, 1)
    f = fusion.prefuse_linear([feats], [np.arange(16)], W)
    pred = fusion.FusedStarPredictor([pk], f.partials)
    s = torch.cuda.current_stream()
    out = {"metric": "fused join+predict fact-rows/sec (BASELINE configs[0]: 1M-row fact x 10K dim, k=16, l=1)",
           "unit": UNIT, "dtype": "f64"}
    for n in (1_000_000, 100_000_000):
        if n == 1_000_000:
            fkd = torch.from_numpy(fk.astype(np.int32)).cuda()
        else:
            fkd = torch.randint(0, 10_000, (n,), dtype=torch.int32, device="cuda")
        y = torch.empty((n, 1), dtype=torch.float64, device="cuda")
        for _ in range(3):
            pred([fkd], out=y, sync=False)
        # CUDA graph of 20 back-to-back calls removes host launch overhead
        graph = torch.cuda.CUDAGraph()
        reps = 20
        with torch.cuda.graph(graph):
            for _ in range(reps):
                pred([fkd], out=y, sync=False)
        pred.ctx.bind_stream(s)
        graph.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        iters = 5
        e0.record()
        for _ in range(iters):
            graph.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / (iters * reps)
        out[f"n{n}"] = {"ms": ms, "rows_per_s": n / (ms / 1e3), "bytes_per_row": 12,
                        "achieved_gbs": 12 * n / (ms / 1e3) / 1e9}
        if n == 1_000_000:
            y1 = y.cpu().numpy()
    # the floor at 1M rows: the same HBM traffic (4 MB of int32 read, 8 MB of fp64
    # written) as one torch elementwise copy, CUDA-graph replayed the same way
    fkd = torch.from_numpy(fk.astype(np.int32)).cuda()
    yc = torch.empty(1_000_000, dtype=torch.float64, device="cuda")
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        for _ in range(20):
            yc.copy_(fkd)
    graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        graph.replay()
    e1.record()
    torch.cuda.synchronize()
    out["n1000000"]["same_traffic_torch_copy_ms"] = e0.elapsed_time(e1) / 100
    pk_, _ = peaks()
    out["value"] = out["n1000000"]["rows_per_s"]
    big = out["n100000000"]
    out["roofline"] = {"bound": "hbm", "achieved": big["achieved_gbs"], "peak": float(pk_["hbm_gbs"]), "unit": "GB/s",
                       "frac": big["achieved_gbs"] / float(pk_["hbm_gbs"]),
                       "note": "12 B/row (4 B key + 8 B fp64 prediction), measured at 1e8 rows; at 1M rows one call "
                               "is a single launch (n1000000.ms) against a same-traffic torch copy "
                               "(n1000000.same_traffic_torch_copy_ms)"}
    # e2e through the API with host buffers: FusedStarPredictor.predict_host
    # (laq_probe_fused_predict_host): pinned keys in, pinned predictions out,
    # H2D / probe / D2H pipelined in chunks over two copy streams
    fk_pin = torch.from_numpy(fk.astype(np.int32)).pin_memory()
    y_pin = torch.empty((1_000_000, 1), dtype=torch.float64).pin_memory()
    for it in range(13):
        if it == 3:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
        yh, nnz = pred.predict_host([fk_pin], out=y_pin)
    e2e_ms = (time.perf_counter() - t0) * 1e3 / 10
    if nnz != 1_000_000 or not np.array_equal(yh.numpy(), y1):
        raise SystemExit("PARITY FAILURE: host-buffer fused predict differs from the device path")
    out["e2e"] = {"value": 1e6 / (e2e_ms / 1e3), "unit": UNIT, "ms": e2e_ms, "h2d_bytes_per_step": 4_000_000,
                  "d2h_bytes_per_step": 8_000_000,
                  "path": "FusedStarPredictor.predict_host -> laq_probe_fused_predict_host (C-ABI): pinned host keys "
                          "in, pinned host predictions out, one call (host clock)"}
    # the same call at 1e8 rows, where it pipelines 8 pieces over two copy streams
    big = torch.randint(0, 10_000, (100_000_000,), dtype=torch.int32).pin_memory()
    ybig = torch.empty((100_000_000, 1), dtype=torch.float64).pin_memory()
    pred.predict_host([big], out=ybig)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        _, nb = pred.predict_host([big], out=ybig)
    big_ms = (time.perf_counter() - t0) * 1e3 / 3
    out["e2e_n100000000"] = {"value": 1e8 / (big_ms / 1e3), "unit": UNIT, "ms": big_ms,
                             "h2d_bytes_per_step": 400_000_000, "d2h_bytes_per_step": 800_000_000,
                             "pcie_gbs": 1.2e9 / (big_ms / 1e3) / 1e9, "nnz": nb,
                             "path": "predict_host: 8 pieces, keys H2D / probe / predictions D2H overlapped"}
    del big, ybig
    # e2e through the reference's UNCHANGED C++ API with host std::vectors
    # (integration/dropin_bench.cpp over the drop-in: multiway_star_join ->
    # csr_from_coo -> prefuse_linear -> apply_fused_linear, each call H2D + D2H)
    exe = os.path.join(ROOT, "integration", "_build", "dropin_bench")
    if os.path.exists(exe):
        import subprocess
        import tempfile
        with tempfile.TemporaryDirectory() as d:
            np.ascontiguousarray(fk, np.int64).tofile(os.path.join(d, "fk.bin"))
            np.ascontiguousarray(pk, np.int64).tofile(os.path.join(d, "pk.bin"))
            np.ascontiguousarray(feats, np.float64).tofile(os.path.join(d, "feats.bin"))
            np.ascontiguousarray(W, np.float64).tofile(os.path.join(d, "W.bin"))
            with open(os.path.join(d, "meta.txt"), "w") as fh:
                fh.write(f"{len(fk)} {len(pk)} {feats.shape[1]} {W.shape[1]}\n")
            r = subprocess.run([exe, d, "10"], capture_output=True, text=True, timeout=600)
            if r.returncode == 0:
                res = json.loads(r.stdout.strip().splitlines()[-1])
                yb = np.fromfile(os.path.join(d, "y.bin"), np.float64).reshape(-1, W.shape[1])
                res["bit_exact_vs_device_path"] = bool(np.array_equal(yb, y1))
                if not res["bit_exact_vs_device_path"]:
                    raise SystemExit("PARITY FAILURE: drop-in C++ API predictions differ from the device path")
                res["path"] = ("integration/dropin_bench.cpp: the reference's C++ operator API (drop-in, liblaq_b200 "
                               "underneath) with host std::vector inputs/outputs; rows_per_s over join + csr + apply "
                               "(prefuse_linear is the one-time model preparation)")
                out["e2e_reference_api"] = res
            else:
                out["e2e_reference_api"] = {"error": (r.stderr or r.stdout)[-300:]}
    try:
        from oracle import ref
        if ref.available():
            y_ref, secs = ref.fused_pipeline([fk], [pk], [feats], W)
            out["parity_vs_reference_fused_pipeline"] = bool(np.array_equal(y_ref, y1))
            if not out["parity_vs_reference_fused_pipeline"]:
                raise SystemExit("PARITY FAILURE: cfg1 fused predictions differ from the reference")
            out["reference_cpu_1thread"] = {"join_csr_prefuse_apply_s": [float(x) for x in secs],
                                            "rows_per_s_end_to_end": 1e6 / float(sum(secs))}
    except ImportError:
        pass
    return out


def ffn_bench(ctx, W, g):
    """configs[2] (only with --workload q1q2 --secondary): SSB SF=10
    lineorder x customer x part + 2-layer FFN (h=256, l=1), the planner's
    non-fused plan on the tensor cores (csrc/ffn.cu)."""
    import torch
    from oracle import laq_oracle as O
    from paper_2306_08367_b200 import ffn, fusion
    fks, pks, dims, pl, W1, W2 = ffn.cfg3_inputs(g)
    n = len(fks[0])
    plan = fusion.plan_linear(n, 64, 256, [len(p) for p in pks])
    m = ffn.StarFFN(dims, pl, W1, W2, dim_pks=pks)
    fd = [torch.from_numpy(np.ascontiguousarray(f)).cuda() for f in fks]
    y = torch.empty((n, 1), dtype=torch.float32, device="cuda")
    for _ in range(3):
        m(fd, out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        m(fd, out=y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    pk_, _ = peaks()
    peak = float(pk_.get("bf16_tflops", 2250.0))
    tensor_tf = 3 * n * 2 * 64 * 256 / (ms / 1e3) / 1e12
    cut = 100_000
    ws, wrows = O.multiway_star_join([f[:cut] for f in fks], pks)
    ref_y, bound = O.ffn_predict(wrows, dims, pl, 64, W1, W2)
    got = y[:cut].double().cpu().numpy()
    m.close()
    return {"workload": f"cfg3: SSB SF={W.sf} lineorder x customer x part ({n} rows), FFN 64-256-1, plan={plan}",
            "ms": ms, "rows_per_s": n / (ms / 1e3), "alg_tflops": n * (2 * 64 * 256 + 2 * 256) / (ms / 1e3) / 1e12,
            "roofline": {"bound": "tensor", "achieved": tensor_tf, "peak": peak, "unit": "TFLOP/s",
                         "frac": tensor_tf / peak},
            "parity_ok_cond_1e-5": bool(np.all(np.abs(got - ref_y) <= 1e-5 * bound))}


if __name__ == "__main__":
    main()
