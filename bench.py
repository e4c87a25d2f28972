#!/usr/bin/env python
"""Benchmark of the LiNR pre-filtered exhaustive top-K scan on B200 (one JSON line on rank 0).

Workload (BASELINE.json configs[1], the config its metric is quoted on): 10M items per GPU,
d=128 bf16, one u64 attribute bitmask word per item, HIGH clause preset (geo Match 3/24 +
company Reverse 1/16 = 11.7% pass, the paper's high-pass dataset analog),
query batch B=1, K=1000. A step = one linr_search (fused filter+score+CTA top-K scan, then the
merge kernel); for N>1 each rank holds its own 10M-row shard of a 10M*N-row index (weak scaling)
and a step adds the all-gather of K packed keys (torch.distributed/NCCL) and the merge kernel.

value = aggregate items scanned per second (B * index rows / step time, max over ranks);
qps is reported next to it. e2e = the same metric through the host-buffer path
(linr_search_host: query H2D + search + ids/scores/pass D2H + sync every step).

--impl reference times the CPU oracle (oracle/, the reference arm of this tier) on a bounded
sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "filtered top-K QPS and items-scanned/s at 1/2/4/8 B200; % HBM roofline"
N_ITEMS = 10_000_000
DIM = 128
K = 1000
B = 1
PRESET = "HIGH"


def parse():
    global DIM, DT, ESZ
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=13000,
                    help="timed searches (default: >= 1 s of device time at the default workload, SURVEY §8(d))")
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="linr", choices=["linr", "reference"])
    ap.add_argument("--batch", type=int, default=B)
    ap.add_argument("--preset", default=PRESET)
    ap.add_argument("--items", type=int, default=N_ITEMS)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--pass-counts", action="store_true", help="batched path: also compute per-query pass counts")
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "f16", "i8", "f32"],
                    help="index dtype (c2: bf16; c3/c4 shards: i8)")
    ap.add_argument("--dim", type=int, default=DIM)
    ap.add_argument("--pipeline", type=int, default=2,
                    help="searches in flight on separate streams in the throughput region (1 = serial)")
    ap.add_argument("--path", default="scan", choices=["scan", "codes", "v3"],
                    help="scan: the exact filtered scan (default); codes: Sign-OPORP matched-bit search with "
                         "any K (PAPER.md P:4665 top-50M of 1B); v3: quantised pre-ranking + full-precision rerank")
    ap.add_argument("--code-bits", type=int, default=64)
    ap.add_argument("--topk", type=int, default=None, help="K (default 1000; --path codes: 5%% of the index)")
    ap.add_argument("--keep", type=float, default=0.01, help="--path v3 keep fraction (P:4595: 1%%)")
    ap.add_argument("--vectors", type=int, default=1,
                    help="query vectors per user V (c5 multi-embedding: 8; scores max-merged in the kernel)")
    ap.add_argument("--update-rate", type=float, default=0.0,
                    help="live row updates per second of device time, interleaved on the search stream in "
                         "64-row linr_index_update_rows calls (Table 5 rates 300/600 rows/s, P:4650-4655); "
                         "forces --pipeline 1")
    a = ap.parse_args()
    DIM = a.dim
    DT = {"bf16": 2, "f16": 1, "i8": 3, "f32": 0}[a.dtype]   # datagen / linr_dtype codes
    ESZ = {"bf16": 2, "f16": 2, "i8": 1, "f32": 4}[a.dtype]
    return a


DT = 2     # LINR_BF16 (set from --dtype)
ESZ = 2


def workload_name(args, n_items):
    tag = "c2" if (args.dtype, DIM) == ("bf16", 128) else "shard"
    if args.vectors > 1:
        tag = "c5"
    vv = f", V={args.vectors}" if args.vectors > 1 else ""
    up = f", updates {args.update_rate:g} rows/s" if args.update_rate > 0 else ""
    return (f"{tag}: {n_items // 1_000_000}M items/GPU d={DIM} {args.dtype}, 64-bit attribute bitmask pre-filter "
            f"({args.preset}), B={args.batch}{vv}, K={K}{up}")


# ------------------------------------------------------------------ clocks
class Clocks:
    def __init__(self, gpu_index: int):
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.close()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


def ncu_traffic(workload):
    """dram bytes per scan launch from the committed ncu --set full summary of the same workload
    (profiles/scan_traffic.json: {workload name: {...}}), else None."""
    p = os.path.join(ROOT, "profiles", "scan_traffic.json")
    if os.path.exists(p):
        try:
            e = json.load(open(p)).get(workload)
            return e.get("dram_bytes_per_launch") if e else None
        except Exception:
            return None
    return None


# ------------------------------------------------------------------ CPU oracle (reference arm / cpu_baseline)
def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_all_cores(oracle, np, vals, attrs, live, Q, cls, nthreads, pool):
    """The oracle as it stands, on `nthreads` host cores: one unmodified oracle.search per
    contiguous row partition (ctypes releases the GIL), then oracle.merge (exact, reading R13)."""
    n = vals.shape[0]
    bounds = [n * t // nthreads for t in range(nthreads + 1)]
    parts = list(pool.map(lambda t: oracle.search(DT, vals[bounds[t]:bounds[t + 1]], attrs[bounds[t]:bounds[t + 1]],
                                                  live[bounds[t]:bounds[t + 1]], Q, cls, K, row0=bounds[t]),
                          range(nthreads)))
    return oracle.merge(np.stack([r[0] for r in parts]), np.stack([r[1] for r in parts]),
                        np.stack([r[2] for r in parts]), K)


def oracle_sample(args, seconds_target=12.0, max_rows=2_000_000):
    """Time the CPU oracle as it stands (single thread) on a bounded slice of the same workload."""
    import numpy as np
    import datagen as dg
    import oracle
    rows = min(max_rows, args.items)
    vals, attrs = dg.gen_items(dg.DATA_SEED, 0, rows, DIM, DT, dg.MODE_DENSE)
    live = np.ones(rows, np.uint8)
    Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, args.items, args.batch, 1, DIM, DT)
    cls = dg.gen_clauses(dg.QUERY_SEED, args.batch, args.preset)
    oracle.lib()
    from concurrent.futures import ThreadPoolExecutor
    nth = host_cores()
    done_items, t_total, calls = 0, 0.0, 0
    with ThreadPoolExecutor(nth) as pool:
        oracle_all_cores(oracle, np, vals, attrs, live, Q, cls, nth, pool)   # warm-up
        while t_total < seconds_target or calls == 0:
            t0 = time.perf_counter()
            oracle_all_cores(oracle, np, vals, attrs, live, Q, cls, nth, pool)
            t_total += time.perf_counter() - t0
            done_items += rows * args.batch
            calls += 1
            if calls >= 20000:
                break
    ips = done_items / t_total
    return {"items_per_s": ips, "qps_equiv": ips / args.items, "rows": rows, "calls": calls, "seconds": t_total,
            "cores": nth}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    import datagen as dg
    import oracle
    rows = min(1_000_000, args.items)
    vals, attrs = dg.gen_items(dg.DATA_SEED, 0, rows, DIM, DT, dg.MODE_DENSE)
    live = np.ones(rows, np.uint8)
    Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, args.items, args.batch, 1, DIM, DT)
    cls = dg.gen_clauses(dg.QUERY_SEED, args.batch, args.preset)
    oracle.lib()
    from concurrent.futures import ThreadPoolExecutor
    nth = host_cores()
    with ThreadPoolExecutor(nth) as pool:
        for _ in range(args.warmup):
            oracle_all_cores(oracle, np, vals, attrs, live, Q, cls, nth, pool)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            oracle_all_cores(oracle, np, vals, attrs, live, Q, cls, nth, pool)
        dt = time.perf_counter() - t0
    ips = rows * args.batch * args.steps / dt
    sample = (f"first {rows} rows of the {args.items}-row workload per step, B={args.batch}, "
              f"{nth} threads (unmodified oracle per row partition + oracle.merge)")
    line = {
        "impl": "reference", "metric": METRIC, "value": ips, "unit": "items/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "qps": ips / args.items,
        "config": {"workload": workload_name(args, args.items), "n_items_per_gpu": args.items, "batch": args.batch,
                   "K": K, "preset": args.preset, "parallelism": f"host cores (oracle, {nth} threads)"},
        "cpu_baseline": {"value": ips, "unit": "items/s", "cores": nth, "kind": "oracle", "sample": sample},
        "e2e": {"value": ips, "unit": "items/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
def run_gpu(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import datagen as dg
    from paper_2407_13218_b200 import Index, ShardedIndex
    from paper_2407_13218_b200.linr import Clauses

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n_local = args.items
    n_total = n_local * world

    t_build = time.perf_counter()
    if world > 1:
        sidx = ShardedIndex(n_total, DIM, DT, 1, device=dev)
        sidx.generate(dg.DATA_SEED, dg.MODE_DENSE)
        ix = sidx.local
    else:
        sidx = None
        ix = Index(n_local, DIM, DT, 1, device=dev)
        ix.generate(dg.DATA_SEED, dg.MODE_DENSE, 0, n_local)
    Vq = args.vectors
    Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n_total, args.batch, Vq, DIM, DT)
    if DT in (dg.BF16, dg.F16):
        qh = torch.from_numpy(Q.view(np.int16)).view(torch.bfloat16 if DT == dg.BF16 else torch.float16).contiguous()
    else:
        qh = torch.from_numpy(Q).contiguous()
    qd = qh.to(dev)
    qpin = qh.pin_memory()
    cls_list = dg.gen_clauses(dg.QUERY_SEED, args.batch, args.preset)
    cls = Clauses(cls_list)
    upd = None
    if args.update_rate > 0:
        # live updates (Table 5): a pool of 64-row calls -- global row ids drawn
        # with the update seed, new rows from the datagen recipe (device generator, update seed)
        from paper_2407_13218_b200.linr import generate_rows
        if sidx is not None:
            raise SystemExit("--update-rate is a single-GPU measurement (updates route to one shard)")
        ncall = 256
        g = torch.Generator().manual_seed(dg.UPDATE_SEED)
        rows_pool = torch.randint(0, n_local, (ncall, 64), generator=g).to(dev)
        emb_pool, attr_pool = generate_rows(DT, DIM, 1, dg.UPDATE_SEED, dg.MODE_DENSE, 0, ncall * 64, device=dev)
        upd = {"rows": rows_pool, "emb": emb_pool.view(ncall, 64, DIM), "attrs": attr_pool.view(ncall, 64, 1), "next": 0}
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t_build

    ids = torch.empty((args.batch, K), dtype=torch.int64, device=dev)
    sc = torch.empty((args.batch, K), dtype=torch.float32, device=dev)
    ps = torch.empty(args.batch, dtype=torch.int64, device=dev)

    # pass counts are not part of the paper's result (reading R24): requested only where they are
    # free (one user: the fused scan counts its passers) or asked for
    want_pass = args.batch == 1 or args.pass_counts
    # the dense tcgen05 roofline applies where that path always runs; 3 <= B <= 16 (V = 1) without
    # pass counts take the union path, whose device-side gate picks the dense pass or the union
    # scans -- their algorithmic bytes are the attribute stream plus the union of passing rows
    union_route = args.vectors == 1 and 3 <= args.batch <= 16 and not want_pass
    tc_route = (args.batch * args.vectors >= 9 and not union_route) or (
        args.batch * args.vectors >= 7 and not want_pass and os.environ.get("LINR_TC_NOPASS") == "1")

    def step():
        if sidx is not None:
            return sidx.search(qd, cls, K)
        return ix.search(qd, cls, K, out=(ids, sc, ps), want_pass=want_pass)

    def update_call():
        j = upd["next"] % upd["rows"].shape[0]
        upd["next"] += 1
        ix.update_rows(upd["rows"][j], upd["emb"][j], upd["attrs"][j])

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    r0 = ix.search(qd, cls, K)   # with pass counts (for the roofline's algorithmic bytes)
    torch.cuda.synchronize()
    pass_count = int(r0[2][0].item())

    stream = torch.cuda.current_stream(dev)

    def timed(steps, pipe):
        """Device time of `steps` searches: pipe = 1 serial on one stream; pipe > 1 round-robin over
        pipe streams, each with its own workspace and outputs (pipelined serving: a search's merge
        tail overlaps the next search's scan). Returns ms."""
        streams = [stream] + [torch.cuda.Stream(dev) for _ in range(pipe - 1)]
        wss = [ix.workspace(args.batch, Vq, K)] + [ix.new_workspace(args.batch, Vq, K) for _ in range(pipe - 1)]
        outs = [(ids, sc, ps)] + [(torch.empty_like(ids), torch.empty_like(sc), torch.empty_like(ps))
                                  for _ in range(pipe - 1)]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for s_ in streams[1:]:
            s_.wait_event(e0)
        for k in range(steps):
            if sidx is not None:
                step()
                continue
            j = k % pipe
            with torch.cuda.stream(streams[j]):
                ix.search(qd, cls, K, out=outs[j], want_pass=want_pass, ws=wss[j])
        for s_ in streams[1:]:
            ej = torch.cuda.Event()
            ej.record(s_)
            stream.wait_event(ej)
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        return e0.elapsed_time(e1)

    def serial_with_events(steps, calls_per_step=0.0):
        """Serial searches on one stream, each bracketed by its own events. With live updates,
        update calls are spread evenly over the steps (calls_per_step on average) and a search's
        latency runs from before the update calls issued ahead of it to the end of the search (a
        query arriving just as an update starts waits for it). Returns (total ms, latencies ms)."""
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        credit, ncalls = 0.0, 0
        for k in range(steps):
            ev[k][0].record(stream)
            credit += calls_per_step
            while credit >= 1.0:
                update_call()
                credit -= 1.0
                ncalls += 1
            step()
            ev[k][1].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        lats = [a.elapsed_time(b) for a, b in ev]
        return ev[0][0].elapsed_time(ev[-1][1]), lats, ncalls

    # ---------------- serial latency (kernel timed alone: the roofline's launch durations)
    ix.profile(True)
    lat_ms = timed(args.steps, 1) / args.steps
    prof = ix.profile_read()
    ix.profile(False)
    upd_info = None
    calls_per_step = 0.0
    if upd is not None:
        # cost of one 64-row update call, timed alone on the search stream
        for _ in range(3):
            update_call()
        u0, u1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        u0.record(stream)
        for _ in range(50):
            update_call()
        u1.record(stream)
        torch.cuda.synchronize()
        upd_ms = u0.elapsed_time(u1) / 50
        calls_per_step = args.update_rate * (lat_ms / 1e3) / 64.0
    lsteps = args.steps if upd is not None else min(args.steps, 1000)
    _, lats, ncalls_lat = serial_with_events(lsteps, calls_per_step)
    lats.sort()
    lat_pct = {"mean": statistics.mean(lats), "p50": lats[len(lats) // 2],
               "p95": lats[min(len(lats) - 1, int(0.95 * len(lats)))],
               "p99": lats[min(len(lats) - 1, int(0.99 * len(lats)))], "samples": len(lats)}
    # ---------------- device-timed throughput region
    pipe = args.pipeline if sidx is None else 1
    if upd is not None:
        pipe = 1   # updates and searches stay stream-ordered (linr.h concurrency contract)
    for _ in range(3):
        timed(2 * pipe, pipe)   # warm the extra streams / workspaces
    clocks = Clocks(local)
    time.sleep(0.3)
    if upd is not None:
        ms, _, ncalls = serial_with_events(args.steps, calls_per_step)
        upd_info = {"rate_rows_per_s": args.update_rate, "rows_per_call": 64, "calls_in_timed_region": ncalls,
                    "rows_in_timed_region": 64 * ncalls, "achieved_rows_per_s": 64 * ncalls / (ms / 1e3),
                    "update_call_ms": upd_ms, "calls_in_latency_region": ncalls_lat,
                    "schedule": "calls spread evenly over the searches of the timed region at the requested "
                                "rate of device time (serial, one stream)"}
    else:
        ms = timed(args.steps, pipe)
    clk = clocks.stop()
    if world > 1:
        t = torch.tensor([ms, lat_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, lat_ms = float(t[0].item()), float(t[1].item())
    ms_step = ms / args.steps

    # ---------------- e2e through the host-buffer public API
    if sidx is None:
        # pipelined like the device-timed region: `pipe` streams, each with its own workspace and
        # pinned result buffers; every step = query H2D + search + ids/scores/pass D2H, and a
        # stream is synchronised (its results read back) before its buffers are reused
        epipe = max(1, args.pipeline)
        estreams = [torch.cuda.Stream(dev) for _ in range(epipe)]
        ews = [ix.new_workspace(args.batch, Vq, K, host_extra=True) for _ in range(epipe)]
        # pass counts as in the device-timed region (want_pass): the batched path computes them only
        # on request (a clause evaluation per (row, user))
        eouts = [(torch.empty((args.batch, K), dtype=torch.int64, pin_memory=True),
                  torch.empty((args.batch, K), dtype=torch.float32, pin_memory=True),
                  torch.empty(args.batch, dtype=torch.int64, pin_memory=True) if want_pass else None)
                 for _ in range(epipe)]

        def e2e_steps(n):
            for k in range(n):
                j = k % epipe
                estreams[j].synchronize()
                with torch.cuda.stream(estreams[j]):
                    ix.search_host(qpin, cls, K, out=eouts[j], ws=ews[j], sync=False)
            for s_ in estreams:
                s_.synchronize()

        e2e_steps(3 * epipe)
        t0 = time.perf_counter()
        e2e_steps(args.steps)
        e2e_s = time.perf_counter() - t0
    else:
        for _ in range(3):
            r = sidx.search(qpin.to(dev, non_blocking=True), cls, K)
            r[0].cpu(), r[1].cpu(), r[2].cpu()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            r = sidx.search(qpin.to(dev, non_blocking=True), cls, K)
            r[0].cpu(), r[1].cpu(), r[2].cpu()
        e2e_s = time.perf_counter() - t0
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    h2d = args.batch * Vq * DIM * ESZ
    d2h = args.batch * K * (8 + 4) + (args.batch * 8 if want_pass else 0)

    items_per_step = args.batch * Vq * n_total   # items-scanned/s = B*V*N / t
    value = items_per_step / (ms_step / 1e3)
    e2e_value = items_per_step * args.steps / e2e_s

    # roofline of the dominant kernel (the fused scan): algorithmic bytes per launch
    # = per item 8 B attribute word + 1/8 B liveness bit, + per passing item the row (256 B)
    rowbytes = DIM * ESZ
    alg_bytes = n_local * (8 + 1 / 8) + pass_count * rowbytes if args.batch == 1 else None
    scan_ms = prof["scan_ms"] / max(1, prof["searches"])
    peak, peak_src = measured_peaks()
    roof = None
    if 1 < args.batch <= 16 and not tc_route:
        # GEMV path with several users: the algorithmic bytes of the step are one read of the
        # attribute words + liveness bits and the rows that pass for at least one user (union)
        a = ix.attr_storage.view(torch.int64)[:n_local]
        union = torch.zeros(n_local, dtype=torch.bool, device=dev)
        for cl_b in cls_list:
            p = torch.ones(n_local, dtype=torch.bool, device=dev)
            for (m, w, r) in cl_b:
                mm = int(np.array([m], dtype=np.uint64).view(np.int64)[0])
                p &= ((a & mm) != 0) ^ bool(r)
            union |= p
        union_pass = int(union.sum().item())
        del a, union
        alg_bytes = n_local * (8 + 1 / 8) + union_pass * DIM * ESZ
    if alg_bytes is not None and scan_ms > 0:
        ach = alg_bytes / (scan_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s", "frac": round(ach / peak, 4),
                "traffic": ncu_traffic(workload_name(args, n_local)), "kernel": f"scan_ws_kernel<{args.dtype},{DIM},1> (warp-specialised ring scan; merge is a separate kernel)",
                "scan_ms_per_launch": round(scan_ms, 5), "merge_ms_per_launch": round(prof["merge_ms"] / max(1, prof["searches"]), 5),
                "alg_bytes_per_launch": int(alg_bytes), "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src})"}
        if args.batch > 1:
            roof["kernel"] = f"scan kernels of one B={args.batch} search (scan_ms = their summed durations)"
            roof["alg_bytes_note"] = ("one read of the attribute words + liveness bits, plus the rows passing for "
                                      f"at least one user ({union_pass} rows)")

    if tc_route and scan_ms > 0:   # the batched tcgen05 path (LINR_TC_MIN default 9; 7 without pass counts)
        # batched path: dense stream of every row (all of them pass for some query) + the GEMM
        import json as _json
        pk = _json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
            os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
        tflops_peak = pk.get("bf16_tflops_sustained", 1400.0)
        peak_note = "MEASURED_PEAKS.json bf16_tflops_sustained (measured)"
        if args.dtype == "i8":
            # kind::i8 contraction: the measured bf16 peak x the nominal dense ratio (4.5 / 2.25 POPS)
            tflops_peak *= 2.0
            peak_note = "MEASURED_PEAKS.json bf16_tflops_sustained x 2 (nominal dense int8 / bf16 ratio)"
        elif args.dtype == "f32":
            peak_note += " (f32 runs on the GEMV path; not a tensor-core contraction)"
        hbm_bytes = n_local * (rowbytes + 8 + 1 / 8)
        flops = 2.0 * args.batch * Vq * n_local * DIM
        hbm_ach = hbm_bytes / (scan_ms / 1e3) / 1e9
        tc_ach = flops / (scan_ms / 1e3) / 1e12
        hf, tf = hbm_ach / peak, tc_ach / tflops_peak
        common = {"kernel": f"tc_scan_kernel<{args.dtype},{DIM},NP> (sample + thresholds + main pass)",
                  "scan_ms_per_launch": round(scan_ms, 5),
                  "merge_ms_per_launch": round(prof["merge_ms"] / max(1, prof["searches"]), 5),
                  "hbm_frac": round(hf, 4), "tensor_frac": round(tf, 4),
                  "alg_bytes_per_launch": int(hbm_bytes), "alg_flops_per_launch": int(flops)}
        if tf >= hf:
            roof = {"bound": "tensor", "achieved": round(tc_ach, 1), "peak": tflops_peak, "unit": "TFLOP/s",
                    "frac": round(tf, 4), "traffic": ncu_traffic(workload_name(args, n_local)),
                    "peak_source": peak_note, **common}
        else:
            roof = {"bound": "hbm", "achieved": round(hbm_ach, 1), "peak": peak, "unit": "GB/s", "frac": round(hf, 4),
                    "traffic": ncu_traffic(workload_name(args, n_local)), "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src})", **common}
    launches_per_step = prof["launches"] / max(1, prof["searches"])
    if world > 1:
        launches_per_step += 1   # merge kernel after the all-gather

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            o = oracle_sample(args)
            cpu = {"value": o["items_per_s"], "unit": "items/s", "cores": o["cores"], "kind": "oracle",
                   "sample": f"oracle (fp64, unmodified, {o['cores']} threads over row partitions + oracle.merge) "
                             f"over the first {o['rows']} rows of the same workload, "
                             f"B={args.batch}, {o['calls']} calls in {o['seconds']:.1f}s; qps_equiv="
                             f"{o['qps_equiv']:.4g} for the {args.items}-row index"}
        line = {
            "metric": METRIC, "value": value, "unit": "items/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (datagen recipe, generated on device)",
            "qps": args.batch / (ms_step / 1e3),
            "latency_ms": lat_ms, "latency_pct_ms": lat_pct, "pipeline": pipe,
            "config": {"workload": workload_name(args, n_local), "n_items_per_gpu": n_local, "n_items_total": n_total,
                       "batch": args.batch, "vectors": Vq, "K": K, "dim": DIM, "preset": args.preset, "pass_count": pass_count,
                       "parallelism": f"row-shard x{world}" if world > 1 else "single GPU",
                       "l2": f"inputs larger than L2 (index {n_local * DIM * ESZ / 1e9:.3g} GB/GPU > 126 MB L2; no flush needed)"},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "items/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e_s / args.steps * 1e3},
            "gpu_launches": int(round(launches_per_step * args.steps)) + (upd_info["calls_in_timed_region"] if upd_info else 0),
            "clocks": clk,
            "build_s": round(t_build, 2),
        }
        if upd_info:
            line["updates"] = upd_info
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_codes(args):
    """Quantised path (§3.2): --path codes = linr_code_search (matched bits, any K; the
    notification case P:4665: top-50M of 1B members, 64-bit codes, one query); --path v3 =
    linr_search_v3 (512-bit codes, keep 1%, full-precision rerank). One GPU."""
    import numpy as np
    import torch

    import datagen as dg
    from paper_2407_13218_b200 import Index
    from paper_2407_13218_b200.linr import Clauses

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    n = args.items
    v3 = args.path == "v3"
    Kq = args.topk if args.topk else (1000 if v3 else max(1, n // 20))
    t_build = time.perf_counter()
    ix = Index(n, DIM, DT, 1, device=dev)
    ix.generate(dg.DATA_SEED, dg.MODE_DENSE, 0, n)
    src, sign = dg.oporp_params(dg.OPORP_SEED, DIM, args.code_bits)
    ix.attach_codes(args.code_bits, src, sign)
    Q = dg.gen_queries(dg.QUERY_SEED, dg.DATA_SEED, n, args.batch, 1, DIM, DT)
    if DT in (dg.BF16, dg.F16):
        qh = torch.from_numpy(Q.view(np.int16)).view(torch.bfloat16 if DT == dg.BF16 else torch.float16).contiguous()
    else:
        qh = torch.from_numpy(Q).contiguous()
    qd = qh.to(dev)
    cls = Clauses(dg.gen_clauses(dg.QUERY_SEED, args.batch, args.preset))
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t_build

    def step():
        return ix.search_v3(qd, cls, Kq, args.keep) if v3 else ix.code_search(qd, cls, Kq)

    for _ in range(args.warmup):
        r = step()
    torch.cuda.synchronize()
    pass_count = int(r[2][0].item())
    kept = int(r[3][0].item()) if v3 else min(Kq, pass_count)
    recall = None
    if v3:   # recall@K of the two-stage result against the exact search on the same index
        ex = ix.search(qd, cls, Kq)
        torch.cuda.synchronize()
        recall = float(np.mean([len(set(r[0][b].tolist()) & set(ex[0][b].tolist())) / max(1, min(Kq, pass_count))
                                for b in range(args.batch)]))
    stream = torch.cuda.current_stream(dev)
    ix.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lat = []
    for _ in range(min(args.steps, 50)):
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        step()
        a1.record(stream)
        a1.synchronize()
        lat.append(a0.elapsed_time(a1))
    prof = ix.profile_read()
    clocks = Clocks(0)
    time.sleep(0.3)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms_step = e0.elapsed_time(e1) / args.steps
    # e2e through the public API: query H2D + search + D2H of ids/matched (or scores) per step
    qpin = qh.pin_memory()
    oh = (torch.empty((args.batch, Kq), dtype=torch.int64, pin_memory=True),
          torch.empty((args.batch, Kq), dtype=torch.int32 if not v3 else torch.float32, pin_memory=True))
    t0 = time.perf_counter()
    esteps = max(3, min(args.steps, 50))
    for _ in range(esteps):
        qd.copy_(qpin, non_blocking=True)
        rr = step()
        oh[0].copy_(rr[0], non_blocking=True)
        oh[1].copy_(rr[1], non_blocking=True)
        torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / esteps
    words = args.code_bits // 64
    hist_ms = prof["scan_ms"] / max(1, prof["searches"])
    # algorithmic bytes of pass 1 (the dominant kernel): attribute word + liveness bit per item, the
    # code of every passing item (8 B per 64 bits); it also writes the 1-2 B matched-bit array
    msz = 1 if args.code_bits <= 192 else 2
    alg = n * (8 + 1 / 8) + pass_count * 8 * words
    peak, peak_src = measured_peaks()
    ach = alg / (hist_ms / 1e3) / 1e9 if hist_ms > 0 else None
    roof = {"bound": "hbm", "achieved": round(ach, 1) if ach else None, "peak": peak, "unit": "GB/s",
            "frac": round(ach / peak, 4) if ach else None, "traffic": None,
            "kernel": f"code_hist_kernel<{words}> (pass 1: filter + matched bits + histograms)",
            "pass1_ms_per_launch": round(hist_ms, 5),
            "rest_ms_per_launch": round(prof["merge_ms"] / max(1, prof["searches"]), 5),
            "alg_bytes_per_launch": int(alg), "matched_array_bytes_per_launch": int(n * msz),
            "step_alg_bytes": int(alg + n * msz * 2 + kept * (12 if not v3 else 4 + DIM * ESZ)),
            "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src})"}
    lat_sorted = sorted(lat)
    name = (f"{'V3 two-stage' if v3 else 'quantised code search'}: {n / 1e6:g}M items d={DIM} {args.dtype}, "
            f"{args.code_bits}-bit Sign-OPORP codes, ({args.preset}), B={args.batch}, K={Kq}"
            + (f", keep={args.keep}" if v3 else ""))
    line = {
        "metric": METRIC, "value": args.batch * n / (ms_step / 1e3), "unit": "items/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": f"{args.code_bits}-bit codes" + (f" + {args.dtype}" if v3 else ""),
        "data": "synthetic (datagen recipe, generated on device)", "qps": args.batch / (ms_step / 1e3),
        "latency_ms": {"mean": statistics.mean(lat), "p50": lat_sorted[len(lat) // 2],
                       "p95": lat_sorted[min(len(lat) - 1, int(0.95 * len(lat)))]},
        "config": {"workload": name, "n_items_per_gpu": n, "batch": args.batch, "K": Kq, "dim": DIM,
                   "preset": args.preset, "pass_count": pass_count, "kept": kept, "code_bits": args.code_bits,
                   "parallelism": "single GPU", "l2": "inputs larger than L2"},
        "recall_at_K_vs_exact": recall,
        "roofline": roof,
        "e2e": {"value": args.batch * n / e2e_s, "unit": "items/s", "h2d_bytes_per_step": args.batch * DIM * ESZ,
                "d2h_bytes_per_step": args.batch * Kq * 12, "ms_per_step": e2e_s * 1e3},
        "gpu_launches": int(round(prof["launches"] / max(1, prof["searches"]) * args.steps)),
        "clocks": clk, "build_s": round(t_build, 2),
        "paper": ("A100, top-50M of 1B members, 64-bit codes, one query: 97.6 ms p95 (P:4665)" if not v3 else
                  "V3 at 1% keep: ~10% lower latency than V2 with near-parity recall (P:4595)"),
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.path != "scan":
        run_codes(args)
        return
    run_gpu(args)


if __name__ == "__main__":
    main()
