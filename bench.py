#!/usr/bin/env python
"""Benchmark of the PC-sample attribution path (BASELINE.json metric: PC samples
attributed/sec and % of HBM roofline, vs the CPU oracle).

One step = one pass of the whole hot path over one batch (DESIGN.md §1 rows a-1..a-10):
zero H||U, attribute this rank's shard of the record stream (K_attr); at N = 1 roll up +
derive metrics for INST/LINE/LOOP/INLINE/FUNC, reconstruct the CCT and derive its EXCL/INCL
metrics; at N > 1 reduce-scatter H||U over NCCL at function-aligned bounds, every rank derives
the rows of its own functions, and rank 0 reconstructs the CCT from the summed S_f||w.  Inputs are generated on the device
(untimed) and are 64 GB at C5, far larger than the 126 MB L2, so no L2 flush is needed.

    python bench.py [--gpus N --steps K --warmup W --config C5]        (N > 1: starts N ranks itself,
                                                                       or runs under torchrun)
    python bench.py --impl reference ...                              (the CPU oracle arm)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PC samples attributed/sec"
UNIT = "samples/s"
SCOPES = ["INST", "LINE", "LOOP", "INLINE", "FUNC"]


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        # wait for the first sample: nvidia-smi's start-up (NVML init) can stall the GPU briefly, so
        # it must not fall inside the timed region (measured: one 16-32 ms step out of ten)
        t_end = time.time() + 5.0
        while self.proc and time.time() < t_end:
            try:
                if open(self.path).read().strip():
                    break
            except Exception:
                pass
            time.sleep(0.05)
        time.sleep(0.15)
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        try:
            rows = [l.split(", ") for l in open(self.path).read().strip().splitlines() if l.strip()]
        except Exception:
            rows = []
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = max(float(r[2]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in rows for j in range(4) if len(r) > 5 + j and "Active" in r[5 + j]
                          and "Not" not in r[5 + j]})
        loaded = [x for x in sm if x >= 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": smax, "reasons": reasons,
                "samples": len(rows)}


def _dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ---------------------------------------------------------------------------------------
# CPU oracle legs (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------------------
def oracle_pass(w, n_sample: int, k0: int, threads: int, chunk: int = 1 << 27):
    """Time the oracle on records [k0, k0+n_sample): D1 attribution on `threads` cores
    (thread-private histograms, serial merge), chunk by chunk (host generation of each chunk
    is untimed), then D2 roll-up + D3-D6 CCT + D7 metrics once on the summed histogram
    (single-threaded: the oracle as it stands)."""
    import numpy as np
    import oracle
    st = w.structure
    H = np.zeros((w.meta["n_inst"], 16), np.uint64)
    U = np.zeros(16, np.uint64)
    buf = np.empty(min(chunk, n_sample), w.records_host(0, 1).dtype)
    ta = 0.0
    for c0 in range(0, n_sample, chunk):
        m = min(chunk, n_sample - c0)
        rec = w.records_host(k0 + c0, m, threads=threads, out=buf[:m])
        t0 = time.perf_counter()
        h, u, _ = oracle.attribute(st, rec, threads=threads)
        H += h
        U += u
        ta += time.perf_counter() - t0
    t1 = time.perf_counter()
    for sc in SCOPES:
        h, m = oracle.scope_hist(st, H, sc)
        oracle.derive_u64(h, m)
    R = oracle.cct(st, H)
    oracle.derive_f64(R["excl"])
    oracle.derive_f64(R["incl"])
    tr = time.perf_counter() - t1
    return ta + tr, ta, tr, int(H.sum() + U.sum())


def cpu_baseline(w, target_s: float = 12.0):
    """The oracle on the GPU box's host cores over a bounded prefix of the same workload,
    sized (after a calibration pass) for about target_s seconds of timed CPU work."""
    cores = len(os.sched_getaffinity(0))
    n = 1 << 26
    t, ta, tr, _ = oracle_pass(w, n, 0, cores)
    per_rec = ta / n
    n = int(min(w.cfg.records, max(n, (target_s - tr) / max(per_rec, 1e-12))))
    t, ta, tr, _ = oracle_pass(w, n, 0, cores)
    return {"value": n / t, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"first {n} records of {w.cfg.name} ({w.cfg.records} total); whole path: D1 attribution "
                      f"({cores} threads, {ta:.2f} s) + roll-up/derive/CCT ({tr:.2f} s, 1 thread)",
            "seconds": t, "attr_seconds": ta, "rest_seconds": tr}


def run_reference(args):
    rank, world, _ = _dist_env()
    if rank != 0:
        return
    import gen
    w = gen.workload(args.config)
    cores = len(os.sched_getaffinity(0))
    n = args.ref_sample
    times = []
    for i in range(args.warmup + args.steps):
        k0 = (i * n) % max(1, w.cfg.records - n)
        t, ta, tr, _ = oracle_pass(w, n, k0, cores)
        if i >= args.warmup:
            times.append(t)
    t = sum(times) / len(times)
    val = n / t
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64/f64", "data": "synthetic",
            "config": {"workload": w.cfg.name, "records": w.cfg.records, "sample_per_step": n,
                       "n_inst": w.meta["n_inst"], "n_func": w.meta["n_func"]},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{n} records per step of {w.cfg.name}, whole path"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------------------
def run_gpa(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import gen
    from paper_2109_06931_b200 import gpa
    from paper_2109_06931_b200.parallel import reduce_histogram, reduce_scatter_histogram, shard_range

    rank, world, local = _dist_env()
    local = local % max(1, torch.cuda.device_count())  # (a host-logic check may run 2 ranks on 1 GPU)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(args.dist_backend)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    w = gen.workload(args.config, records=args.records)
    n_all = w.cfg.records
    a, b = shard_range(n_all, rank, world)
    n = b - a
    s = gpa.load_structure(w.structure, local)
    ni = s.info["n_inst"]
    # the attribution and the latency-bound CCT chain run on a high-priority stream: when the
    # attribution ends, the CCT's single-CTA kernels are scheduled ahead of the side stream's
    # roll-up CTAs (which only have to finish by the end of the step)
    lo_pri, hi_pri = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
    stream = torch.cuda.Stream(dev, priority=min(lo_pri, hi_pri)) if not args.no_priority else torch.cuda.current_stream(dev)
    torch.cuda.set_stream(stream)

    CH = 1 << 28

    def make_shard(a, n):
        r = torch.empty((max(n, 1), 2), dtype=torch.int64, device=dev)
        for k in range(0, n, CH):
            w.records_device(r[k:k + CH], a + k, min(CH, n - k))
        torch.cuda.synchronize()
        return r

    rec = make_shard(a, n)
    rows = {sc: max(1, gpa.scope_row_count(s, sc)) for sc in SCOPES}
    met = {sc: torch.empty((rows[sc], gpa.NUM_DERIVED), dtype=torch.float64, device=dev) for sc in SCOPES}
    # N > 1: the reduced histogram is scattered at function-aligned
    # instruction bounds and every rank derives the rows of its own functions; the CCT's Step-1
    # inputs (S_f, w: 0.7 MB at C5) are summed to rank 0, which reconstructs the tree
    scatter = world > 1 and args.combine == "scatter"
    if scatter:
        bounds = [int(x) for x in gpa.partition_structure(w.structure, world)]
        lo, hi = bounds[rank], bounds[rank + 1]
        nf, nc = s.info["n_func"], s.info["n_call"]
    # Two batch buffers.  Default: one batch at a time (attribution, then the CCT on the
    # high-priority stream B with the scope roll-ups on a side stream).  --pipeline enqueues batch
    # i + 1's attribution (stream A) before batch i's analysis; with the asynchronous CCT the host
    # never waits inside a step, so the analysis kernels fill SMs the attribution leaves idle: C5
    # 12.56 -> 12.35 ms per step, but the attribution itself then measures 12.26 instead of 12.02 ms
    # (0.797 instead of 0.813 of peak: the analysis competes with it), so the default keeps the
    # kernel's own time clean.
    pipeline = args.pipeline
    class Buf:
        pass

    bufs = []
    for _ in range(2):
        x = Buf()
        x.HU = torch.zeros(ni * 16 + 16, dtype=torch.int64, device=dev)   # H_inst || U, one buffer
        x.H, x.U = x.HU[:ni * 16].view(ni, 16), x.HU[ni * 16:]
        if scatter:
            x.SW = torch.zeros(nf * 16 + nc, dtype=torch.int64, device=dev)   # S_f || w
            x.SF, x.CW = x.SW[:nf * 16].view(nf, 16), x.SW[nf * 16:]
        x.attr_done = torch.cuda.Event()
        x.freed = torch.cuda.Event()
        x.freed.record(stream)
        bufs.append(x)
    B = stream                                       # combine + CCT (high priority)
    A = torch.cuda.Stream(dev) if pipeline else B        # attribution
    side = torch.cuda.Stream(dev)                    # scope roll-ups
    ev_a0, ev_a1, ev_b0, ev_b1, ev_c1 = [], [], [], [], []

    def enqueue_attr(i: int, timed: bool, host=None):
        x = bufs[i % 2]
        A.wait_event(x.freed)
        with torch.cuda.stream(A):
            x.HU.zero_()
        if timed:
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record(A)
        if host is None:
            gpa.attribute_samples(s, rec, x.H, x.U, n=n, stream=A)
        else:
            gpa.attribute_samples_host(s, host, x.H, x.U, stream=A)
        if timed:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record(A)
            ev_a0.append(e0)
            ev_a1.append(e1)
        x.attr_done.record(A)

    def analyse(i: int, timed: bool, results=None):
        """Batch i after its attribution: combine (N > 1), the five scopes' roll-ups + metrics on the
        side stream concurrently with the CCT + its metrics on B; returns the context count."""
        x = bufs[i % 2]
        B.wait_event(x.attr_done)
        with torch.cuda.stream(B):
            if world > 1:
                if scatter:
                    reduce_scatter_histogram(x.HU, bounds, ni)
                else:
                    reduce_histogram(x.HU, dst=0)
            ready = torch.cuda.Event(enable_timing=timed)
            ready.record(B)
            if timed:
                ev_b0.append(ready)
            do_scopes = scatter or rank == 0
            if do_scopes:
                side.wait_event(ready)
                if scatter:
                    gpa.derive_scopes(s, x.H, {sc: {"metrics": met[sc]} for sc in SCOPES}, lo, hi, stream=side)
                else:
                    gpa.derive_scopes(s, x.H, {sc: {"metrics": met[sc]} for sc in SCOPES}, stream=side)
                if timed:
                    sd = torch.cuda.Event(enable_timing=True)
                    sd.record(side)
                    ev_b1.append(sd)
            nctx, cct = 0, None
            if scatter:
                x.SW.zero_()
                gpa.cct_inputs(s, x.H, lo, hi, x.SF, x.CW, stream=B)
                dist.reduce(x.SW, dst=0)
                if rank == 0:
                    cct = gpa.reconstruct_cct_inputs(s, x.SF, x.CW, stream=B)
            elif rank == 0 and async_cct:
                cct = gpa.reconstruct_cct_async(s, x.H, stream=B)   # no host synchronization
            elif rank == 0:
                cct = gpa.reconstruct_cct(s, x.H, stream=B)
            if cct is not None:
                if cct.pending:  # metrics rows = the capacity; the kernels read the size on the device
                    if cm_async[0] is None or cm_async[0].shape[0] < cct.capacity:
                        cm_async[0] = torch.empty((cct.capacity, gpa.NUM_DERIVED), dtype=torch.float64, device=dev)
                    cm = cm_async[0]
                else:
                    cm = torch.empty((max(cct.n, 1), gpa.NUM_DERIVED), dtype=torch.float64, device=dev)
                gpa.derive_metrics(s, "CCT_EXCL", cct=cct, metrics=cm, stream=B)
                gpa.derive_metrics(s, "CCT_INCL", cct=cct, metrics=cm, stream=B)
                if timed:
                    ce = torch.cuda.Event(enable_timing=True)
                    ce.record(B)
                    ev_c1.append(ce)
                nctx = cct if cct.pending else cct.n
            if do_scopes:
                B.wait_stream(side)
            if results is not None:      # e2e: read the batch's results back to the host
                for dst, src in results(x):
                    dst.copy_(src, non_blocking=True)
            x.freed.record(B)
            if cct is not None and not cct.pending:
                cct.free()               # stream-ordered on B
        return nctx

    # CCT without a host round trip inside the step (gpa_reconstruct_cct_async) when batches are
    # pipelined.  One batch at a time keeps the synchronous call: there the asynchronous tree's
    # settle() overlaps the next batch's attribution, and in 2 of 4 C5 runs that batch's
    # attribution then took 15-40 ms instead of 12 (never with the synchronous call: 12.43-12.45
    # ms per step over 4 runs)
    async_cct = world == 1 and (pipeline or args.async_cct) and not args.sync_cct
    cm_async = [None]

    def run_steps(k: int, timed: bool, host=None, results=None):
        """k batches; pipelined: attribution of i + 1 is enqueued before the analysis of i.
        An asynchronous tree is finished when the next batch's attribution is already queued (the
        host waits for the tree while the GPU attributes; a tree the one-launch build could not
        hold is rebuilt there and its metrics derived again, on B, inside the timed region)."""
        nctx, last = 0, None

        def settle():
            nonlocal last
            n = 0
            if last is not None:
                c, last = last, None
                if c.finish():
                    for sc in ("CCT_EXCL", "CCT_INCL"):
                        m = torch.empty((max(c.n, 1), gpa.NUM_DERIVED), dtype=torch.float64, device=dev)
                        gpa.derive_metrics(s, sc, cct=c, metrics=m, stream=B)
                n = c.n
                c.free()
            return n

        def keep(r):
            nonlocal last
            if isinstance(r, gpa.Cct):
                last = r
                return 0
            return r

        dbg = timed and os.environ.get("GPA_BENCH_HOSTTIME")
        for i in range(k):
            h0 = time.perf_counter()
            enqueue_attr(i, timed, host)
            h1 = time.perf_counter()
            nctx = settle() or nctx
            h2 = time.perf_counter()
            if not pipeline:
                nctx = keep(analyse(i, timed, results))
            elif i > 0:
                nctx = keep(analyse(i - 1, timed, results))
            if dbg:
                print(f"step {i}: enqueue {1e3 * (h1 - h0):.3f} ms, settle {1e3 * (h2 - h1):.3f} ms, analyse "
                      f"{1e3 * (time.perf_counter() - h2):.3f} ms", file=sys.stderr)
        if pipeline and k > 0:
            nctx = settle() or nctx
            nctx = keep(analyse(k - 1, timed, results))
        return settle() or nctx

    nctx = run_steps(args.warmup, False)
    torch.cuda.synchronize()
    root_less = 0
    if world > 1 and not args.no_balance:
        # Load balance (untimed): rank 0 also runs the CCT (and, with --combine reduce, every
        # roll-up) after the combine, so it takes D fewer records, D = (its combine + analysis
        # time - the slowest other rank's) / its attribution time per record (measured here);
        # the shards are regenerated and re-warmed before the timed region.
        cal = []
        for _ in range(2):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            ev[0].record(A)
            enqueue_attr(0, False)
            ev[1].record(A)
            ev[2].record(A)
            analyse(0, False)
            ev[3].record(B)
            torch.cuda.synchronize()
            cal.append((ev[0].elapsed_time(ev[1]), ev[2].elapsed_time(ev[3])))
        t_at, t_an = cal[-1]
        tt = torch.tensor([t_an if rank else 0.0], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)          # the other ranks' combine + analysis
        d = int(max(0.0, t_an - tt.item()) / max(t_at, 1e-6) * n) if rank == 0 else 0
        t = torch.tensor([max(0, d)], dtype=torch.int64, device=dev)
        dist.broadcast(t, 0)
        root_less = int(t.item())
        a2, b2 = shard_range(n_all, rank, world, root_less)
        if (a2, b2) != (a, b):
            del rec
            torch.cuda.empty_cache()
            a, b, n = a2, b2, b2 - a2
            rec = make_shard(a, n)
        nctx = run_steps(args.warmup, False)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    l0 = gpa.kernel_launches()
    import gc
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        gc.collect()
        gc.disable()  # no collector pause between a step's event and its kernels' launch
        t0.record(A)
        nctx = run_steps(args.steps, True)
        B.wait_stream(A)
        t1.record(B)
        torch.cuda.synchronize()
        gc.enable()
        if world > 1:
            dist.barrier()
    launches = gpa.kernel_launches() - l0
    ms = t0.elapsed_time(t1) / args.steps
    attr_ms = sum(x.elapsed_time(y) for x, y in zip(ev_a0, ev_a1)) / len(ev_a0)
    algo_bytes = 16 * n                              # this rank's K_attr launch
    if world > 1:
        t = torch.tensor([ms, attr_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, attr_ms = t.tolist()
        nb = torch.tensor([algo_bytes], dtype=torch.int64, device=dev)
        dist.all_reduce(nb)
        algo_bytes = int(nb.item())                  # all ranks; divided by N below
        lt = torch.tensor([launches], dtype=torch.int64, device=dev)
        dist.all_reduce(lt)
        launches = int(lt.item())
    clocks = clk.summary()

    # e2e: the same steps through the C ABI with HOST records (pinned), H2D inside the timed
    # region (gpa_attribute_samples_host pipelines the copies), D2H of each batch's results.
    e2e = None
    if not args.no_e2e:
        host = torch.empty((n, 2), dtype=torch.int64, pin_memory=True)
        w.records_host(a, n, out=host.numpy().view(gen.RECORD_DTYPE).reshape(-1))
        res_h = torch.empty(ni * 16 + 16, dtype=torch.int64, pin_memory=True)
        fm_h = torch.empty(met["FUNC"].shape, dtype=torch.float64, pin_memory=True)

        def results(x):
            return [(res_h, x.HU), (fm_h, met["FUNC"])] if rank == 0 else []

        e_w = min(args.warmup, 1) if args.e2e_steps else args.warmup
        e_k = args.e2e_steps or args.steps
        run_steps(e_w, False, host, results)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        q0 = torch.cuda.Event(enable_timing=True)
        q1 = torch.cuda.Event(enable_timing=True)
        q0.record(A)
        run_steps(e_k, False, host, results)
        B.wait_stream(A)
        q1.record(B)
        torch.cuda.synchronize()
        ems = q0.elapsed_time(q1) / e_k
        if world > 1:
            t = torch.tensor([ems], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = t.item()
        e2e = {"value": n_all / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": 16 * n_all,
               "d2h_bytes_per_step": (res_h.numel() * 8 + fm_h.numel() * 8) if rank == 0 else 0,
               "ms_per_step": ems, "steps": e_k}
        # the link's pinned H2D ceiling, for context: copy (up to) 4 GiB of this rank's host
        # records over their identical device copy
        m = min(n, 1 << 28)
        if m > 0:
            src, dst = host[:m], rec[:m]
            dst.copy_(src, non_blocking=True)
            torch.cuda.synchronize()
            h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            h0.record(torch.cuda.current_stream())
            dst.copy_(src, non_blocking=True)
            h1.record(torch.cuda.current_stream())
            torch.cuda.synchronize()
            link = 16 * m / (h0.elapsed_time(h1) / 1e3) / 1e9
            e2e["h2d_link_gbs"] = link
            e2e["h2d_link_frac"] = 16 * n / (ems / 1e3) / 1e9 / link
        del host

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    peak, peak_src = _peaks()
    achieved = algo_bytes / world / (attr_ms / 1e3) / 1e9   # per GPU: mean bytes / slowest launch
    # DRAM traffic of the timed kernel from the committed ncu capture (tools/capture_traffic.py),
    # used only while the kernel sources are the ones it was captured from; scaled to this launch
    traffic, traffic_src = None, "no capture"
    tp = os.path.join(ROOT, "profiles", f"k_attr_traffic_{w.cfg.name}.json")
    if os.path.exists(tp):
        try:
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            from capture_traffic import source_hash
            cap = json.load(open(tp))
            if cap.get("source_sha1") == source_hash():
                traffic = cap["dram_bytes_per_launch"] * (algo_bytes / world) / cap["algorithmic_bytes"]
                traffic_src = f"ncu capture {cap.get('when')} ({cap['records']} records, {cap['kernel']})"
            else:
                traffic_src = "stale capture (kernel sources changed): not used"
        except Exception as ex:
            traffic, traffic_src = None, f"capture unreadable: {ex}"
    # phase times on rank 0 and the secondary sum-of-counts rate
    phases = {"attr_ms": attr_ms,
              "scopes_ms_side_stream": sum(x.elapsed_time(y) for x, y in zip(ev_b0, ev_b1)) / max(1, len(ev_b1)),
              "cct_and_cct_metrics_ms": sum(x.elapsed_time(y) for x, y in zip(ev_b0, ev_c1)) / max(1, len(ev_c1)),
              "attr_ms_per_step": [round(x.elapsed_time(y), 4) for x, y in zip(ev_a0, ev_a1)]}
    observations = int(bufs[(args.steps - 1) % 2].HU.sum().item())  # sum of counts of the last batch (u64 as int64)
    line = {"metric": METRIC, "value": n_all / (ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64/f64", "data": "synthetic",
            "config": {"workload": w.cfg.name, "records": n_all, "records_per_gpu": n, "n_inst": ni,
                       "root_shard_less": root_less,
                       "n_func": s.info["n_func"], "n_call": s.info["n_call"], "cct_contexts": int(nctx),
                       "parallelism": (f"record shards x{world}, " + (
                           f"{args.dist_backend} reduce-scatter of H||U at function-aligned bounds, rows derived "
                           f"per rank, S_f||w reduced to rank 0 for the CCT" if scatter else
                           f"{args.dist_backend} reduce of H||U to rank 0") if world > 1 else "single GPU"),
                       "l2": "inputs (16 B x records) far exceed the 126 MB L2; no flush needed",
                       "schedule": "pipelined batches (attribution of i+1 queued before the analysis of i)"
                       if pipeline else "one batch at a time"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": gpa.ATTR_KERNEL_NAMES.get(gpa.attr_kernel_choice(s, n), "?"),
                         "kernel_ms": attr_ms, "algorithmic_bytes": algo_bytes, "peak_source": peak_src,
                         "traffic_source": traffic_src},
            "gpu_launches": int(launches), "clocks": clocks, "e2e": e2e, "phases_ms": phases,
            "observations_per_s": observations / (ms / 1e3)}
    if not args.no_cpu_baseline:   # rank 0 at every N (the other ranks have finished their GPU work)
        line["cpu_baseline"] = cpu_baseline(w, args.cpu_seconds)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _self_launch(args) -> int:
    """--gpus N > 1 without a torchrun environment: start N ranks of this same command with
    torch.distributed.run on this node (rendezvous on 127.0.0.1); rank 0 prints the line."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--records", type=int, default=None, help="override the config's record count")
    ap.add_argument("--impl", default="gpa", choices=["gpa", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-priority", action="store_true", help="attribution + CCT on the default-priority stream")
    ap.add_argument("--dist-backend", default="nccl", help="N > 1 process group (gloo: a host-logic check only)")
    ap.add_argument("--combine", default="scatter", choices=["scatter", "reduce"],
                    help="N > 1: reduce-scatter + per-rank roll-ups (default) or reduce to rank 0")
    ap.add_argument("--no-balance", action="store_true", help="N > 1: equal shards (rank 0 not lightened)")
    ap.add_argument("--sync-cct", action="store_true", help="synchronous gpa_reconstruct_cct (A/B of the async tree)")
    ap.add_argument("--async-cct", action="store_true", help="asynchronous tree also with one batch at a time")
    ap.add_argument("--pipeline", action="store_true",
                    help="enqueue batch i+1's attribution before batch i's analysis (C5: +1.7 %% throughput, "
                         "the attribution kernel slowed by the concurrent analysis; DESIGN.md §11)")
    ap.add_argument("--e2e-steps", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-sample", type=int, default=1 << 28)
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_self_launch(args))
    rank, world, _ = _dist_env()
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "gpa" and world > 1 and args.dist_backend == "nccl":
        import torch
        if torch.cuda.device_count() < world:
            print(f"bench.py: {world} NCCL ranks need {world} GPUs, this node has {torch.cuda.device_count()}",
                  file=sys.stderr)
            sys.exit(2)
    if args.warmup < 3 and args.impl == "gpa":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpa(args)


if __name__ == "__main__":
    main()
