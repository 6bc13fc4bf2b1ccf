#!/usr/bin/env python
"""Benchmark of the north-star path: exhaustive fused CNF term match +
embedding KNN + top-K on B200.

Default workload = BASELINE.json's metric config c3: 10M jobs, d=128 fp32,
8-clause CNF (~5% selectivity), batch B=64 queries, K=100, quant
pre-selection off (the exhaustive path).  A "step" is one execute_batch of
the B queries over the whole index.

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

Our arm prints one JSON line with the device-timed whole-job QPS (`value`,
index + queries resident in HBM), the end-to-end QPS through the C-ABI with
host buffers (`e2e`), p50 call latency, the roofline of the dominant kernel
and the reference CPU baseline.  `--impl reference` times the reference's
own CPU implementation (oracle/_ref, the unmodified reference sources) on a
bounded sample of the same workload.

Multi-GPU (torchrun, one rank per GPU): the 10M rows are sharded by
contiguous row ranges (strong scaling); each rank scores its shard, the
per-shard top-K lists are all-gathered over NCCL and merged exactly on
device (K4) -- the one collective of the path.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops_sustained"]), "measured"
    except Exception:
        return 6650.0, 1400.0, "fallback"


# ---------------------------------------------------------------------------
# clocks sampler (B200_PROFILING.md: sample nvidia-smi DURING the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    """Polls NVML every ~2 ms in a thread while the timed region runs: SM
    clock, max SM clock and the clock-event (throttle) reasons."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown"}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.N = None
        return self

    def _run(self):
        N = self.N
        get_reasons = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            N.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self._stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                r = get_reasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __exit__(self, *a):
        self._stop.set()
        if self.N:
            self.t.join(timeout=1)

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "NVML, 2 ms polling"}


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------
def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


def shard_range(n, rank, world):
    return rank * n // world, (rank + 1) * n // world


# ---------------------------------------------------------------------------
# reference (CPU) arm
# ---------------------------------------------------------------------------
FULL_REF_MAX_ROWS = 10_000_000  # larger corpora: the reference on a row prefix, scaled (stated)


def reference_index(w, so, ids, emb, threads):
    """The unmodified reference (oracle/_ref) over the corpus rows given,
    built as concurrent FrozenIndex shards by its own IndexBuilder/freeze
    (oracle/ref.py ShardedRef, SURVEY §8(d) sharded oracle)."""
    from oracle import ref as R
    t0 = time.perf_counter()
    sref = R.ShardedRef(so, ids, emb, w.num_clauses, w.max_num_attr, w.num_bits, w.seed, threads=threads)
    return sref, time.perf_counter() - t0


def ref_queries(w, batch, k):
    from oracle import ref as R
    from paper_2402_13435_b200 import workloads as W
    raws, qemb = W.queries(w, batch, high_pass=not LOW_PASS[0])
    return [(R.normalize_query(raw, w.num_clauses) if raw else [], qemb[i] if qemb is not None else None, k,
             False, 0, 100) for i, raw in enumerate(raws)]


def ref_rows(w):
    return min(w.n, FULL_REF_MAX_ROWS)


def ref_sample_text(w, rows, nq, threads, build_s, shards):
    scope = (f"the full {w.n}-row index" if rows == w.n else
             f"a {rows}-row prefix of the {w.n}-row index, QPS scaled by rows ({w.n}/{rows})")
    return (f"{nq} queries of the {w.name} batch per step on {scope}: reference Executor::execute (quant off) over "
            f"{threads} threads, the index built as {shards} reference FrozenIndex shards, each (query, shard) pair "
            f"one reference call, shard top-K lists merged by "
            f"(score desc, row asc); reference IndexBuilder+freeze {build_s:.1f}s")


def run_reference(args, w):
    """--impl reference: the reference's own CPU path (oracle/_ref, unmodified
    proj/src sources) timed on the host cores; rank 0 only.  Each step is a
    bounded sample of the workload: `threads` queries of the batch (cycling
    through it) over the whole index -- nothing of this repository's product
    library is loaded in this process."""
    from paper_2402_13435_b200 import workloads as W
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    rows = ref_rows(w)
    so, ids, emb = W.docs(w, 0, rows)
    sref, build_s = reference_index(w, so, ids, emb, threads)
    del so, ids, emb
    qs = ref_queries(w, args.batch, args.k)
    per = max(1, min(len(qs), args.ref_queries or threads))
    cursor = [0]

    def step():
        sample = [qs[(cursor[0] + i) % len(qs)] for i in range(per)]
        cursor[0] += per
        secs, _ = sref.execute(sample, threads)
        return secs

    for _ in range(args.warmup):
        step()
    per_step = [step() for _ in range(args.steps)]
    scale = w.n / rows
    total = sum(per_step) * scale
    qps = per * args.steps / total
    line = {
        "impl": "reference", "metric": "queries_per_sec", "value": qps, "unit": "queries/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.mean(per_step) * scale * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (SURVEY §8(d) generator, std::mt19937_64)",
        "config": workload_config(w, args),
        "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": threads, "kind": "reference",
                         "sample": ref_sample_text(w, rows, per, threads, build_s, sref.g)},
        "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


LOW_PASS = [False]  # --low-pass (c5 query shape), set once from the arguments


def workload_config(w, args):
    """Identical in both arms (the driver compares them)."""
    return {"workload": f"{w.name}: {w.n} jobs x d{w.dim} {w.dtype}, "
                        + ("match-all" if w.kind == "match_all" else f"{w.num_clauses}-clause CNF"),
            "jobs": w.n, "dim": w.dim, "emb_dtype": w.dtype, "clauses": w.num_clauses, "batch": args.batch,
            "k": args.k, "quant": False, "parallelism": f"rows-sharded x{dist_env()[1]}",
            "l2": "inputs larger than L2 (index >> 126 MB), no flush",
            **({"query_pass": "low (8 tail ids)" if LOW_PASS[0] else "high (32 head ids)"} if w.kind == "zipf" else {})}


def parity_check(sref, qs, got):
    """Our hits (rows, scores per query) against the reference's on the same
    index: rows identical except ties at the K-th score, scores within
    max(1e-3 |s|, 2e-5) of the reference's exact_scores of the same row
    (SURVEY §8(d) gates 2-3); term-only lists identical."""
    secs, want = sref.execute(qs)
    mism, max_err, detail = 0, 0.0, []
    for i, (q, (gr, gs), (st, rr, rs)) in enumerate(zip(qs, got, want)):
        ok = st == 0 and len(gr) == len(rr)
        if ok and q[1] is None:
            ok = bool(np.array_equal(gr, rr))
        elif ok and len(rr):
            o = sref.exact_scores(q[1], gr).astype(np.float64)
            err = np.abs(gs.astype(np.float64) - o)
            max_err = max(max_err, float(err.max()))
            tol = np.maximum(1e-3 * np.abs(o), 2e-5)
            tau = float(rs[-1])
            et = max(1e-3 * abs(tau), 2e-5)
            must = rr[rs > tau + et]
            extra = ~np.isin(gr, rr)
            ok = bool((err <= tol).all() and np.isin(must, gr).all() and (o[extra] >= tau - 2 * et).all())
        if not ok:
            mism += 1
            detail.append(i)
    return {"queries": len(qs), "mismatches": mism, "max_abs_err": max_err, "failed": detail[:8],
            "reference": "oracle/_ref (unmodified reference sources), same index and queries"}, secs


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, w):
    import torch

    import paper_2402_13435_b200 as hy
    from paper_2402_13435_b200 import _lib as L
    from paper_2402_13435_b200 import workloads as W

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = L.lib()
    t_setup = time.perf_counter()
    rb, re_ = shard_range(w.n, rank, world)
    so, ids, emb = W.docs(w, rb, re_)
    frozen = W.freeze_docs(w, so, ids, emb, rb)
    t_frozen = time.perf_counter() - t_setup
    # The reference over the same rows (N = 1): the parity check of our
    # results and the timed CPU baseline (full index up to 10M rows, else a
    # stated prefix).
    sref = ref_build_s = None
    ref_threads = os.cpu_count() or 1
    want_ref = world == 1 and not args.no_cpu_baseline
    if want_ref:
        try:
            if w.n <= FULL_REF_MAX_ROWS:
                sref, ref_build_s = reference_index(w, so, ids, emb, ref_threads)
            else:
                del so, ids, emb
                so, ids, emb = W.docs(w, 0, ref_rows(w))
                sref, ref_build_s = reference_index(w, so, ids, emb, ref_threads)
        except Exception as e:  # reported, never fatal
            sref, ref_build_s = None, str(e)[:200]
    del so, ids, emb
    dev = hy.DeviceIndex(frozen, device=local, dtype=w.dtype, tensor_path=True, row_offset=rb)
    stats = dev.stats()
    raws, qemb = W.queries(w, args.batch, high_pass=not LOW_PASS[0])
    hq = []
    for i, raw in enumerate(raws):
        hq.append(hy.HybridQuery(hy.normalize_query(raw, w.num_clauses), None if qemb is None else qemb[i],
                                 args.k, hy.ExecOptions(quant_enabled=False)))
    ex = hy.Executor(dev, max_batch=args.batch)
    h = ex._h
    pack = hy.QueryPack(hq)
    B = args.batch

    def check(rc):
        hy.hyre._check(rc)

    check(lib.hyre_batch_prepare(h, pack.arr, B))
    stream = torch.cuda.ExternalStream(lib.hyre_executor_stream(h), device=torch.device("cuda", local))

    gather = None
    if world > 1:
        import torch.distributed as dist
        hits_p, n_hits, off_p, cnt_p = C.c_void_p(), C.c_uint64(), C.c_void_p(), C.c_void_p()
        check(lib.hyre_batch_device_results(h, C.byref(hits_p), C.byref(n_hits), C.byref(off_p), C.byref(cnt_p)))

        class Dev:
            def __init__(self, ptr, shape, typestr):
                self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr, "data": (ptr, False),
                                                 "version": 3, "stream": None}

        n_words = int(n_hits.value) * 2  # hyre_hit = 2 x u32
        t_hits = torch.as_tensor(Dev(hits_p.value, (n_words,), "<i4"), device=f"cuda:{local}")
        t_off = torch.as_tensor(Dev(off_p.value, (B,), "<i8"), device=f"cuda:{local}")
        t_cnt = torch.as_tensor(Dev(cnt_p.value, (B,), "<i4"), device=f"cuda:{local}")
        # identical shapes on every rank: one packed record per rank (hits
        # padded to the max hit buffer, then the B u64 offsets, then the B u32
        # counts) -> ONE all-gather, merged exactly on device
        n_max = torch.tensor([n_words], device=f"cuda:{local}")
        dist.all_reduce(n_max, op=dist.ReduceOp.MAX)
        n_max = int(n_max.item())
        rec_words = n_max + 3 * B + (3 * B) % 2
        rec = torch.zeros(rec_words, dtype=torch.int32, device=f"cuda:{local}")
        g_rec = torch.zeros(world, rec_words, dtype=torch.int32, device=f"cuda:{local}")

        def gather():
            with torch.cuda.stream(stream):
                rec[:n_words].copy_(t_hits)
                rec[n_max:n_max + 2 * B].copy_(t_off.view(torch.int32))
                rec[n_max + 2 * B:n_max + 3 * B].copy_(t_cnt)
                dist.all_gather_into_tensor(g_rec.view(-1), rec)
            check(lib.hyre_batch_merge_packed(h, g_rec.data_ptr(), world, rec_words, n_max))

    # Two batches in flight (N = 1): a second executor with its own stream
    # runs every other step, so one batch's small kernels (sample, thresholds,
    # select) overlap the other's main pass -- the serving model of the
    # reference's ExecutorPool.  Every step is still one full pass over the
    # index for one batch; the timed region spans all K steps on both streams.
    # The headline `value` keeps one batch in flight (p50 = single-batch
    # latency); `inflight2` below repeats the timed region with two.
    ex_b = None
    alt = [False]
    if world == 1 and args.inflight > 1:
        ex_b = hy.Executor(dev, max_batch=args.batch)
        check(lib.hyre_batch_prepare(ex_b._h, pack.arr, B))
        stream_b = torch.cuda.ExternalStream(lib.hyre_executor_stream(ex_b._h), device=torch.device("cuda", local))
    n_step = [0]

    def step():
        hx = h if (not alt[0] or n_step[0] % 2 == 0) else ex_b._h
        n_step[0] += 1
        check(lib.hyre_batch_run(hx))
        if gather:
            gather()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    # ---- warm-up -----------------------------------------------------------
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # The timed steps enqueue hyre_batch_run only; threshold recovery rounds
    # and exhaustive queries would run later, at settle.  The batch is the
    # same every step, so its recovery need is too: measure it once and, if
    # any, settle inside every timed step so no work falls outside the clock.
    check(lib.hyre_batch_settle(h))
    rec = np.zeros(2, np.uint32)
    check(lib.hyre_batch_recovery(h, rec.ctypes.data_as(L.u32p)))
    reruns = {"recovery_rounds": int(rec[0]), "exhaustive_queries": int(rec[1]),
              "settled_in_timed_steps": bool(rec.any())}
    if rec.any():
        run_step = step

        def step():  # noqa: F811
            run_step()
            check(lib.hyre_batch_settle(h if not alt[0] or n_step[0] % 2 == 1 else ex_b._h))
    s6 = (C.c_float * 6)()

    # ---- timed region: exactly K back-to-back steps, device time ----------
    # Inner stage events are off here (a stream event between two kernels
    # ends their programmatic-dependent-launch overlap); each run still
    # records its start/end events, which give the per-batch latencies.
    check(lib.hyre_batch_set_stage_events(h, 0))
    if ex_b is not None:
        check(lib.hyre_batch_set_stage_events(ex_b._h, 0))
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    total_ms = e0.elapsed_time(e1)
    t = torch.tensor([total_ms], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    kernels_per_step = int(lib.hyre_batch_kernel_count(h)) + (1 if gather else 0)

    # ---- per-call latency + per-kernel times of the timed steps ------------
    # (CUDA events the executor records around each stage on its own stream;
    # it keeps the last 64 runs, read back after the timed region)
    lat = []
    for back in range(min(args.steps, 64)):
        check(lib.hyre_batch_stage_ms_hist(h, back, s6))
        lat.append(s6[5])
    # per-stage times (the dominant kernel's launch time for the roofline):
    # the same K steps again with the stage events on, right after the timed ones
    check(lib.hyre_batch_set_stage_events(h, 1))
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    stage_rows = []
    for back in range(min(args.steps, 64)):
        check(lib.hyre_batch_stage_ms_hist(h, back, s6))
        stage_rows.append(list(s6))
    inflight2 = None
    if ex_b is not None and not os.environ.get("HYRE_TC_DEBUG"):
        check(lib.hyre_batch_set_stage_events(h, 0))
        alt[0] = True
        for _ in range(2):
            step()
        torch.cuda.synchronize()
        f0, f1, fb = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
                      torch.cuda.Event())
        f0.record(stream)
        stream_b.wait_event(f0)
        n_step[0] = 0
        for _ in range(args.steps):
            step()
        fb.record(stream_b)
        stream.wait_event(fb)
        f1.record(stream)
        torch.cuda.synchronize()
        alt[0] = False
        ms2 = f0.elapsed_time(f1)
        inflight2 = {"value": B * args.steps / (ms2 * 1e-3), "unit": "queries/s", "ms_per_step": ms2 / args.steps,
                     "note": "the same K steps with two batches in flight on two executors/streams (device-timed); "
                             "p50 latency then includes queueing behind the other batch"}
    main_ms = [r[3] for r in stage_rows]
    p50 = statistics.median(lat)
    lat_sorted = sorted(lat)

    def pct(p):  # nearest-rank percentile (bench.cpp:113-123 reports p50/p95/p99)
        return lat_sorted[min(len(lat_sorted) - 1, max(0, int(np.ceil(p / 100 * len(lat_sorted))) - 1))]
    main_avg = statistics.mean(main_ms)

    # ---- end-to-end through the C-ABI with host buffers ---------------------
    # (throughput callers switch the inner stage events off, like the timed steps)
    check(lib.hyre_batch_set_stage_events(h, 0))
    caps = [min(args.k, re_ - rb)] * B
    offs = np.concatenate([[0], np.cumsum(caps)[:-1]]).astype(np.uint64)
    host_hits = (L.hyre_hit * sum(caps))()
    counts = np.zeros(B, np.uint32)
    sts = np.zeros(B, np.int32)
    tim = L.hyre_timings()
    e2e_steps = max(3, args.steps // 2)

    def e2e_call():
        if world == 1:
            check(lib.hyre_execute_batch(h, pack.arr, B, host_hits, offs.ctypes.data_as(L.u64p),
                                         counts.ctypes.data_as(L.u32p), sts.ctypes.data_as(L.i32p), C.byref(tim)))
        else:
            # host queries -> device; shard results (settled) -> all ranks (NCCL) -> exact device merge -> host
            check(lib.hyre_batch_prepare(h, pack.arr, B))
            check(lib.hyre_batch_run(h))
            check(lib.hyre_batch_settle(h))
            gather()
            check(lib.hyre_batch_fetch(h, host_hits, offs.ctypes.data_as(L.u64p), counts.ctypes.data_as(L.u32p),
                                       sts.ctypes.data_as(L.i32p), None))

    if os.environ.get("HYRE_TC_DEBUG"):  # diagnostics runs: results are invalid, device timings only
        e2e_call = lambda: check(lib.hyre_batch_run(h))  # noqa: E731
    e2e_call()
    # host-side cost of one prepare (validation, program build, packed H2D enqueue)
    t0 = time.perf_counter()
    for _ in range(5):
        check(lib.hyre_batch_prepare(h, pack.arr, B))
    torch.cuda.synchronize()
    prep_ms = (time.perf_counter() - t0) / 5 * 1e3
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_call()
    barrier()
    e2e_s = time.perf_counter() - t0
    e2e_t = torch.tensor([e2e_s], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_s = float(e2e_t.item())
    h2d, d2h = C.c_uint64(), C.c_uint64()
    check(lib.hyre_batch_io_bytes(h, C.byref(h2d), C.byref(d2h)))
    if not os.environ.get("HYRE_TC_DEBUG"):
        assert all(sts == 0) and (qemb is None or int(counts.min()) > 0), "empty results in the e2e run"
    single_e2e = B * e2e_steps / e2e_s
    # our final answers (the last public-API call) for the parity check
    hit_arr = np.frombuffer(host_hits, dtype=np.uint32).reshape(-1, 2)
    ours = [(hit_arr[int(offs[i]):int(offs[i]) + int(counts[i]), 0].astype(np.int64),
             hit_arr[int(offs[i]):int(offs[i]) + int(counts[i]), 1].view(np.float32).copy()) for i in range(B)]

    # ---- the same calls from three host threads, one executor each --------
    # (the reference's ExecutorPool model, service.cpp:99-141: one thread's
    # host work -- validation, program build, copies -- overlaps the other
    # executor's kernels; every call still copies its queries in and its
    # hits out).  N = 1 only: the multi-GPU e2e keeps one caller per rank.
    pooled = None
    n_callers = 3
    if world == 1 and not os.environ.get("HYRE_TC_DEBUG"):
        extra = [(hy.Executor(dev, max_batch=args.batch), hy.QueryPack(hq)) for _ in range(n_callers - 1)]
        for ex_x, _ in extra:
            check(lib.hyre_batch_set_stage_events(ex_x._h, 0))

        def worker(hx, pk, n, out):
            hh = (L.hyre_hit * sum(caps))()
            cn = np.zeros(B, np.uint32)
            st_ = np.zeros(B, np.int32)
            for _ in range(n):
                rc = lib.hyre_execute_batch(hx, pk.arr, B, hh, offs.ctypes.data_as(L.u64p), cn.ctypes.data_as(L.u32p),
                                            st_.ctypes.data_as(L.i32p), None)
                if rc != 0 or not all(st_ == 0):
                    out.append(False)
                    return
            out.append(True)

        n_each = max(3, e2e_steps)
        for ex_i, pk_i in extra:
            worker(ex_i._h, pk_i, 1, [])  # warm the other executors
        oks = []
        pairs = [(h, pack)] + [(ex_i._h, pk_i) for ex_i, pk_i in extra]
        threads = [threading.Thread(target=worker, args=(hx, pk, n_each, oks)) for hx, pk in pairs]
        t0 = time.perf_counter()
        for th in threads:
            th.start()
        for th in threads:
            th.join()
        pooled_s = time.perf_counter() - t0
        assert all(oks) and len(oks) == n_callers, "pooled e2e calls failed"
        pooled = n_callers * B * n_each / pooled_s

    if rank != 0:
        return
    hbm, _, peak_kind = peaks()
    n_local = re_ - rb
    elem = 2 if w.dtype == "bf16" else 4
    # algorithmic bytes of the dominant kernel's launch:
    #  K3 (batched): per query group, every row of the shard once -- the
    #     bf16 hi plane (prefilter; exact rescoring of the admitted rows is a
    #     separate small kernel) or hi + lo -- + its eligibility input (the
    #     compact CNF rows when the CNF is fused into K3, else the mask words
    #     K1 wrote), as the executor reports it (hyre_batch_scan_bytes);
    #  K2 (B <= 8): only eligible rows are loaded: U = the largest per-query
    #     eligible count (a lower bound on the union it streams) + the masks;
    #  K1 (term-only batches): distinct term bitmaps + CSR postings + mask writes.
    words = (n_local + 31) // 32
    path = int(lib.hyre_batch_path(h))
    fused = bool(path & 2)
    kernel = main_kernel_name(B, path)
    if qemb is None:
        kernel = "mask_tm_kernel (K1: term-major CNF over bitmaps/CSR)"
        bytes_main = int(lib.hyre_batch_term_bytes(h)) + B * words * 4
        main_avg = statistics.median(r[0] for r in stage_rows)
    elif path & 1:
        bytes_main = int(lib.hyre_batch_scan_bytes(h))
    else:
        elig = np.zeros(B, np.uint32)
        check(lib.hyre_batch_eligible(h, elig.ctypes.data_as(L.u32p)))
        elem_k2 = 1 if path & 32 else elem  # int8 prefilter rows
        bytes_main = int(min(n_local, elig.max())) * w.dim * elem_k2 + B * words * 4
    achieved = bytes_main / (main_avg * 1e-3) / 1e9
    traffic = load_traffic(w.name)
    step_ms = total_ms / args.steps
    qps = B * args.steps / (total_ms * 1e-3)
    line = {
        "metric": "queries_per_sec", "value": qps, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "p50_ms": p50, "jobs_scored_per_sec": qps * w.n,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        # returned scores are computed in f32 (bf16 rows for a bf16 index); the
        # scan itself runs on the int8 prefilter plane when path & 32
        "dtype": (f"{w.dtype} (scan: int8 prefilter)" if path & 32 else w.dtype),
        "data": "synthetic (SURVEY §8(d) generator, std::mt19937_64; index built by the product IndexBuilder)",
        "config": workload_config(w, args),
        "p95_ms": pct(95), "p99_ms": pct(99), "latency_samples": len(lat),
        "reruns": reruns,
        "inflight2": inflight2,
        "stages_ms_note": "per-stage CUDA events from K more steps right after the timed ones (the timed steps record "
                          "only each run's start/end: an event between kernels ends their PDL overlap)",
        "stages_ms": dict(zip(["mask", "quant", "sample", "main_scorer", "select_firstk", "run"],
                              [statistics.median(r[i] for r in stage_rows) for i in range(6)])),
        "roofline": {"bound": "hbm", "kernel": kernel, "achieved": achieved, "peak": hbm,
                     "peak_kind": f"{peak_kind} hbm_gbs (burst copy)", "unit": "GB/s", "frac": achieved / hbm,
                     "bytes_per_launch": bytes_main, "launch_ms": main_avg, "traffic": traffic,
                     "eligibility": ("none (match-all batch)" if path & 16 else
                                     "fused CNF over compact CNF rows" if fused else "K1 mask bitmaps"),
                     "path_flags": path},
        "e2e": {"value": pooled if pooled else single_e2e, "unit": "queries/s", "h2d_bytes_per_step": int(h2d.value),
                "d2h_bytes_per_step": int(d2h.value),
                "api": (f"hyre_execute_batch (C-ABI, host buffers) from {n_callers} host threads, one executor each "
                        "(ExecutorPool model)" if pooled else "hyre_execute_batch (C-ABI, host buffers)"),
                "single_caller_value": single_e2e, "host_prepare_ms": prep_ms},
        "gpu_launches": kernels_per_step * args.steps,
        "clocks": clocks.summary(),
        "index": {"build_s": t_frozen, **{k: stats[k] for k in ("num_terms", "bitmap_terms", "csr_terms")}},
    }
    if want_ref:
        if sref is None:
            line["cpu_baseline"] = {"value": None, "error": ref_build_s}
            line["parity"] = None
        else:
            qs = ref_queries(w, B, args.k)
            rows = ref_rows(w)
            if rows == w.n:
                par, secs = parity_check(sref, qs, ours)
                line["parity"] = par
            else:
                secs, _ = sref.execute(qs)
                line["parity"] = {"queries": 0, "note": f"reference built on a {rows}-row prefix only"}
            cqps = B / (secs * w.n / rows)
            line["cpu_baseline"] = {"value": cqps, "unit": "queries/s", "cores": ref_threads, "kind": "reference",
                                    "sample": ref_sample_text(w, rows, B, ref_threads, ref_build_s, sref.g)}
    print(json.dumps(line), flush=True)


def main_kernel_name(B, path=0):
    if B <= 8 and path & 32:
        return "score_kernel<int8> (K2: int8 prefilter rows, dp4a, exact rescoring in K4p)"
    if B > 8 and path & 32:
        return ("tc_score_kernel (K3: bulk-copy ring -> tcgen05.mma kind::i8, s32 accumulation in TMEM; int8 "
                "prefilter + fused CNF, admitted rows pruned + rescored exactly in fp32 by select_prefilter_kernel)")
    if B > 8:
        return ("tc_score_kernel (K3: bulk-copy ring -> tcgen05.mma kind::f16, fp32 accumulation in TMEM; bf16 "
                "prefilter or hi/lo split + fused CNF)")
    return "score_kernel (K2, CUDA-core streaming scorer)"


def load_traffic(name):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(name)
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--rows", type=int, default=None, help="override the workload's row count")
    ap.add_argument("--ref-queries", type=int, default=None,
                    help="reference arm: queries per step (default: one per host thread)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--low-pass", action="store_true", help="c5: low-selectivity queries (8 tail ids)")
    ap.add_argument("--inflight", type=int, default=2, help="batches in flight on separate executors (N = 1)")
    args = ap.parse_args()
    LOW_PASS[0] = args.low_pass
    from paper_2402_13435_b200.workloads import WORKLOADS
    import dataclasses
    w = WORKLOADS[args.workload]
    if args.rows:
        w = dataclasses.replace(w, n=args.rows)
    args.batch = args.batch or w.batch
    args.k = args.k or w.k
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        run_reference(args, w)
    else:
        run_ours(args, w)


if __name__ == "__main__":
    main()
