#!/usr/bin/env python
"""Benchmark of MapSQ's join path on B200 (contract: one JSON line on rank 0).

A "step" is one pass of the whole hot path over the resident synthetic input: for LUBM configs
one ``mapsq_query`` (fused pattern scan -> chained Map/Sort/ReduceDuplicate joins ->
projection); for C4 one ``mapsq_join`` of the two Zipf tables.  The metric is BASELINE.json's:
join input+output tuples per second (sum over the query's joins of n1 + n2 + |RS|), plus the
modelled HBM GB/s.  ``--impl reference`` times the CPU oracle on a bounded sample instead.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl mapsq|reference]
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

import numpy as np  # noqa: E402

CONFIGS = {
    # name: (kind, universities, query, description)
    "C1": ("lubm", 1, "C1", "LUBM(1) chain join ?x worksFor ?d . ?d subOrganizationOf ?u"),
    "C2": ("lubm", 100, "C2", "LUBM(100) Q2-core triangle (memberOf, subOrganizationOf, undergraduateDegreeFrom)"),
    "C3": ("lubm", 1000, "C3", "LUBM(1000) 4-pattern star on department ?x"),
    "C4": ("zipf", 500_000_000, None, "2 x 5e8-row (key, value) tables, Zipf(1.1) keys over 2^29"),
    "C5": ("lubm", 10000, "C5", "LUBM(10000) Q9-core triangle (advisor, teacherOf, takesCourse)"),
}
METRIC = "join input+output tuples/s and HBM GB/s (% peak) at 1/2/4/8 B200"
NVLINK_PEER_GBS = 770.0  # measured peer copy per direction per GPU (B200_PROFILING.md)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md, no MEASURED_PEAKS.json)"


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML polled every ~2 ms from
    a thread (short regions such as C4's ~50 ms still get samples); nvidia-smi as a fallback."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.sm, self.mx, self.reasons = [], [], set()
        self.stop = None
        self.thread = None
        self.err = None

    def __enter__(self):
        import threading
        try:
            import pynvml as nv
            nv.nvmlInit()
            # NVML numbers devices ignoring CUDA_VISIBLE_DEVICES: find this rank's GPU by UUID
            h = None
            try:
                import torch
                uuid = str(torch.cuda.get_device_properties(self.gpu).uuid)
                uuid = uuid if uuid.startswith("GPU-") else "GPU-" + uuid
                h = nv.nvmlDeviceGetHandleByUUID(uuid.encode())
                self.sampled = uuid
            except Exception:  # noqa: BLE001 (older torch / NVML: index order)
                h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
                self.sampled = f"nvml index {self.gpu}"
            bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
        except Exception as e:  # no NVML: nvidia-smi below
            self.err = str(e)
            return self._smi_enter()
        self.stop = threading.Event()

        def poll():
            while not self.stop.is_set():
                try:
                    self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                    self.mx.append(mx)
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.reasons.update(n for n, bit in bits.items() if r & bit)
                except Exception as e:
                    self.err = str(e)
                    return
                time.sleep(0.002)

        self.thread = threading.Thread(target=poll, daemon=True)
        self.thread.start()
        return self

    def __exit__(self, *exc):
        if self.thread is not None:
            self.stop.set()
            self.thread.join(timeout=5)
        elif getattr(self, "proc", None) is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def _smi_enter(self):
        self.path = os.path.join("/tmp", f"mapsq_clocks_{os.getpid()}.csv")
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (FileNotFoundError, OSError):
            self.proc = None
        time.sleep(0.25)
        return self

    def summary(self):
        if self.thread is None:
            if getattr(self, "proc", None) is None or not os.path.exists(self.path):
                return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 6:
                    continue
                try:
                    self.sm.append(float(f[0]))
                    self.mx.append(float(f[1]))
                except ValueError:
                    continue
                self.reasons.update(n for n, v in zip(self.NAMES, f[2:6])
                                    if v.lower().startswith("active"))
            os.unlink(self.path)
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_max_mhz": max(self.mx) if self.mx else None,
                "reasons": sorted(self.reasons), "samples": len(self.sm),
                "source": "nvml" if self.thread is not None else "nvidia-smi",
                "gpu": getattr(self, "sampled", f"index {self.gpu}")}


# ----------------------------------------------------------------------------- workloads
def lubm_host(nuniv: int, u_lo: int, u_hi: int, pinned: bool):
    import torch

    import datagen
    st = datagen.lubm_count(nuniv, u_lo, u_hi)
    n = st["n_triples"]
    if pinned:
        bufs = [torch.empty(n, dtype=torch.int32).pin_memory() for _ in range(3)]
        arrs = [b.numpy().view(np.uint32) for b in bufs]
    else:
        bufs, arrs = None, [np.empty(n, np.uint32) for _ in range(3)]
    s, p, o, st = datagen.lubm(nuniv, u_lo, u_hi, out=arrs)
    return (s, p, o), st, bufs


def query_patterns(name):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from fixtures import config_query
    return config_query(name)


# ----------------------------------------------------------------------------- reference arm
def oracle_sample(cfg: str, budget_s: float = 20.0):
    """Time the CPU oracle (as it stands, 1 thread) on a bounded sample of the workload.
    Returns (tuples/s, sample description, join tuples, seconds)."""
    import datagen
    import oracle
    kind, nu, qname, _ = CONFIGS[cfg]
    if kind == "zipf":
        n = 4_000_000
        k1, v1 = datagen.zipf(n, 0)
        k2, v2 = datagen.zipf(n, 1)
        A, B = oracle.Table([0, 1], np.stack([k1, v1], 1)), oracle.Table([0, 2], np.stack([k2, v2], 1))
        t0 = time.perf_counter()
        r = oracle.join(A, B)
        dt = time.perf_counter() - t0
        tuples = 2 * n + r.nrows
        return tuples / dt, f"rows [0,{n}) of both C4 sides (Zipf(1.1), same generator/seed)", tuples, dt
    pats = query_patterns(qname)
    # universities [0, k) of the same dataset: identical triples to the full workload's prefix.
    # Like the GPU step (whose partial matches are zero-copy views of the resident predicate
    # index), the timed work is the query's joins: the oracle's linear-filter scans run first,
    # untimed (their time is reported in the sample description).
    k = {"C1": 1, "C2": 100, "C3": 300, "C5": 2500}[cfg]
    k = min(k, nu)
    (s, p, o), st, _ = lubm_host(nu, 0, k, pinned=False)
    t0 = time.perf_counter()
    tabs = [oracle.scan(s, p, o, pat) for pat in pats]
    t_scan = time.perf_counter() - t0
    t0 = time.perf_counter()
    acc = tabs[0]
    tuples = 0
    for t in tabs[1:]:
        r = oracle.join(acc, t)
        tuples += acc.nrows + t.nrows + r.nrows
        acc = r
    dt = time.perf_counter() - t0
    return tuples / dt, (f"universities [0,{k}) of LUBM({nu}) ({len(s)} triples, {k / nu:.4g} of "
                         f"the workload): the query's joins (sort-merge tier); its pattern scans "
                         f"took {t_scan:.2f} s more, untimed"), tuples, dt


def host_info() -> dict:
    """The host the oracle ran on (single-threaded): core count and CPU model."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"host_cores": os.cpu_count(), "cpu_model": model, "threads_used": 1}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = args.config
    vals = []
    tuples = 0
    for _ in range(args.warmup):
        oracle_sample(cfg)
    for _ in range(args.steps):
        v, sample, tuples, dt = oracle_sample(cfg)
        vals.append(v)
    value = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tuples/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": tuples / value * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": cfg, "description": CONFIGS[cfg][3], "sample": sample},
            "cpu_baseline": {"value": value, "unit": "tuples/s", "cores": 1, "kind": "oracle",
                             "sample": sample, **host_info()},
            "e2e": {"value": value, "unit": "tuples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
# random bitmap probes/s one B200 sustains from a 2^29-bit (L2-resident) bitmap through the
# read-only path, 5e8 probes (tools/bitmap_bench.cu, `probe ilp4 nc 2^29 bits`)
FILTER_PROBE_PEAK = 418e9


def filter_rate(st, steps, step_ms_total):
    """The semi-join filter kernels are bound by random L1/L2 bitmap accesses, not by HBM: their
    access rate against the measured probe rate (the HBM roofline understates them)."""
    names = ("filter_build", "filter_probe", "filter_set")
    ms = sum(st["kernels"][k]["ms"] for k in names if k in st["kernels"])
    acc = st.get("filter_accesses", 0)
    if not ms or not acc:
        return None
    rate = acc / (ms / 1e3)
    return {"accesses_per_step": acc / steps, "rate": rate, "peak": FILTER_PROBE_PEAK,
            "unit": "accesses/s", "frac": rate / FILTER_PROBE_PEAK,
            "share_of_step": ms / step_ms_total, "kernels": [k for k in names if k in st["kernels"]],
            "peak_source": "tools/bitmap_bench.cu probe ilp4 nc 2^29 bits (B200, measured)"}


def run_gpu(args):
    import torch
    import paper_1702_03484_b200 as mq

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or args.force_dist:
        return run_gpu_dist(args, world, rank, local)
    torch.cuda.set_device(local)
    cfg = args.config
    kind, nu, qname, desc = CONFIGS[cfg]
    if args.univ:
        nu = args.univ
    ctx = mq.Context(local)
    ctx.set_option(mq.OPT_SEMIJOIN, {"auto": mq.SEMIJOIN_AUTO, "on": mq.SEMIJOIN_ON,
                                     "off": mq.SEMIJOIN_OFF}[args.semijoin])
    index_build_ms = None
    stream = torch.cuda.current_stream()
    t_gen = time.perf_counter()
    if kind == "zipf":
        import datagen
        n = args.rows or nu
        k1, v1 = datagen.zipf(n, 0)
        k2, v2 = datagen.zipf(n, 1)
        cols = [torch.from_numpy(a.view(np.int32)).cuda() for a in (k1, v1, k2, v2)]
        del k1, v1, k2, v2
        A = mq.DeviceTable.from_torch([0, 1], cols[:2])
        B = mq.DeviceTable.from_torch([0, 2], cols[2:])
        ctx.table_bounds(A)
        ctx.table_bounds(B)
        in_bytes = 16 * n
        host = None

        def step():
            r = ctx.join(A, B)
            m = r.nrows
            r.release()
            return m
        workload = f"C4 Zipf(1.1) 2x{n} rows"
    else:
        # pinned raw triples only for the scan store's e2e (the index store's e2e reads the
        # index's pinned host mirror)
        (s, p, o), st, pinned = lubm_host(nu, 0, nu,
                                          pinned=not args.no_e2e and args.store == "scan")
        trip = tuple(torch.from_numpy(a.view(np.int32)).cuda() for a in (s, p, o))
        pats = query_patterns(qname)
        in_bytes = 12 * len(s)
        host = (s, p, o, pats)
        source = trip
        if args.store == "index":
            # the store's predicate-range index, built once at load time
            torch.cuda.synchronize()
            t_idx = time.perf_counter()
            source = ctx.index_build(trip)
            torch.cuda.synchronize()
            index_build_ms = (time.perf_counter() - t_idx) * 1e3
            del trip  # the index holds its own (predicate-partitioned) copy
            torch.cuda.empty_cache()
            if not args.no_e2e:  # the store's host-resident copy, mirrored once at load time
                host = (ctx.index_to_host(source), None, None, pats)

        prepared = ctx.prepare(source, pats)  # (the arguments marshalled once per run)

        def step():
            r = prepared()
            m = r.nrows
            r.release()
            return m
        workload = f"{cfg} LUBM({nu}) {len(s)} triples"
    torch.cuda.synchronize()
    log(f"[bench] {workload}: generated + resident in {time.perf_counter() - t_gen:.1f}s")

    l2 = torch.cuda.get_device_properties(local).L2_cache_size
    flush = None
    if in_bytes < 4 * l2:
        flush = torch.empty(4 * l2 // 4, dtype=torch.int32, device="cuda")

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    def timed(profile: bool):
        ctx.stats_reset()
        ctx.set_profiling(profile)
        evs = []
        with ClockSampler(local) as clk:
            time.sleep(0.01)  # (let the sampler thread start polling before the first timed step)
            for _ in range(args.steps):
                if flush is not None:
                    flush.fill_(1)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                m = step()
                e1.record(stream)
                evs.append((e0, e1))
            torch.cuda.synchronize()
        ctx.set_profiling(False)
        return [a.elapsed_time(b) for a, b in evs], ctx.stats(), clk.summary(), m

    # region 1 (the reported value): no per-kernel events; region 2: per-kernel CUDA events on
    # the library's stream for the roofline and the kernel shares
    step_ms, st_plain, clocks, m_final = timed(False)
    if os.environ.get("MAPSQ_BENCH_STEPLOG"):  # (diagnostics: every timed step's ms)
        with open(os.environ["MAPSQ_BENCH_STEPLOG"], "w") as f:
            f.write("\n".join(f"{x:.5f}" for x in step_ms) + "\n")
    prof_ms, st_k, _, _ = timed(True)
    total_s = sum(step_ms) / 1e3
    tuples = st_plain["join_in_rows"] + st_plain["join_out_rows"]
    value = tuples / total_s
    algo_bytes = sum(k["bytes"] for k in st_k["kernels"].values())
    peak, peak_src = measured_peaks()
    hbm_gbs = algo_bytes / total_s / 1e9
    # dominant kernel by time (profiled region)
    name, kd = max(st_k["kernels"].items(), key=lambda kv: kv[1]["ms"])
    avg_ms = kd["ms"] / kd["launches"]
    achieved = (kd["bytes"] / kd["launches"]) / (avg_ms / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"ncu_traffic_{cfg}.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(name)

    line = {"metric": METRIC, "value": value, "unit": "tuples/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": sum(step_ms) / len(step_ms), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": cfg, "description": desc, "detail": workload,
                       "l2": "inputs larger than L2" if flush is None else "L2 flushed between steps",
                       "store": ("pos-index (mapsq_query_indexed; built once at load in "
                                 f"{index_build_ms:.0f} ms)" if kind != "zipf" and args.store == "index"
                                 else "triple table scan (mapsq_query)") if kind != "zipf" else None,
                       "semijoin_filter": args.semijoin,
                       "join_tuples_per_step": tuples // args.steps,
                       "result_rows": m_final},
            "hbm": {"algo_bytes_per_step": algo_bytes // args.steps, "gbs": hbm_gbs,
                    "frac_of_peak": hbm_gbs / peak, "peak_gbs": peak},
            "roofline": {"kernel": name, "bound": "hbm", "achieved": achieved, "peak": peak,
                         "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "share_of_step": kd["ms"] / sum(prof_ms),
                         "timing": "per-kernel CUDA events on the library stream, second timed region"},
            "kernels": {k: {"launches": v["launches"], "avg_ms": v["ms"] / v["launches"],
                            "share": v["ms"] / sum(prof_ms)} for k, v in st_k["kernels"].items()},
            "filter": filter_rate(st_k, args.steps, sum(prof_ms)),
            "clocks": clocks, "gpu_launches": st_plain["launches"]}

    # e2e through the public API from pinned host buffers (H2D + query + D2H inside the region)
    if host is not None and not args.no_e2e:
        s, p, o, pats = host
        indexed = isinstance(s, mq.HostIndex)
        e2e_ms = []
        out_bytes = in_h2d = 0
        for i in range(max(1, min(args.steps, 5)) + 1):  # (median of up to 5 after a warm run)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if indexed:
                vars_, rows = ctx.query_host(s, pats)
            else:
                vars_, rows = ctx.query_host(s, p, o, pats)
            dt = time.perf_counter() - t0
            out_bytes = rows.nbytes
            in_h2d = s.last_h2d_bytes if indexed else 12 * len(s)
            if i:
                e2e_ms.append(dt * 1e3)
        e2e_s = statistics.median(e2e_ms) / 1e3
        line["e2e"] = {"value": (tuples / args.steps) / e2e_s, "unit": "tuples/s",
                       "h2d_bytes_per_step": in_h2d, "d2h_bytes_per_step": out_bytes,
                       "path": ("mapsq_query_host_indexed: the pinned host store's predicate ranges "
                                "the query touches H2D, joins, result D2H, every step" if indexed
                                else "mapsq_query_host: pinned triples H2D, full-table scan, joins, "
                                     "result D2H, every step"),
                       "ms_per_step": e2e_s * 1e3}
    elif kind == "zipf":
        line["e2e"] = None
    if not args.no_cpu_baseline:
        v, sample, _, dt = oracle_sample(cfg)
        line["cpu_baseline"] = {"value": v, "unit": "tuples/s", "cores": 1, "kind": "oracle",
                                "sample": sample, "seconds": dt, **host_info()}
    print(json.dumps(line), flush=True)


def run_gpu_dist(args, world, rank, local):
    """N > 1: one process per GPU over NCCL.  Each rank generates its own contiguous university
    range of the same dataset (identical triples for any N), runs the distributed query
    (mapsq_query_dist[_indexed]: local scan, hash exchange per join key, local joins); time = max over ranks of the device
    time; value = join tuples summed over ranks / that time (strong scaling: fixed dataset)."""
    import torch
    import torch.distributed as tdist

    import paper_1702_03484_b200 as mq
    from paper_1702_03484_b200 import dist as mqd
    # MAPSQ_BENCH_HOSTCOLL=1 (testing only: exercises this code path with several ranks on ONE
    # GPU): every rank uses cuda:0, torch.distributed runs on gloo and the library's control plane
    # on host collectives (mapsq_dist_init_host) — the numbers of such a run are not measurements
    hostcoll = os.environ.get("MAPSQ_BENCH_HOSTCOLL") == "1"
    if hostcoll:
        local = 0
    torch.cuda.set_device(local)
    if hostcoll:
        tdist.init_process_group("gloo")
    else:
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cdev = "cpu" if hostcoll else "cuda"  # device of the bench's own collective tensors
    cfg = args.config
    kind, nu, qname, desc = CONFIGS[cfg]
    if args.univ:
        nu = args.univ
    ctx = mq.Context(local)
    ctx.set_option(mq.OPT_SEMIJOIN, {"auto": mq.SEMIJOIN_AUTO, "on": mq.SEMIJOIN_ON,
                                     "off": mq.SEMIJOIN_OFF}[args.semijoin])
    if hostcoll:
        ctx.dist_init_host()
    else:
        mqd.ensure_dist(ctx)
    if kind == "zipf":
        # C4: each rank generates its contiguous row range of both sides (identical tables for any
        # N), step = mapsq_join_dist (both sides exchanged on the key, local join)
        import datagen
        n = args.rows or nu
        lo, hi = n * rank // world, n * (rank + 1) // world
        k1, v1 = datagen.zipf(hi - lo, 0, i_lo=lo)
        k2, v2 = datagen.zipf(hi - lo, 1, i_lo=lo)
        cols = [torch.from_numpy(a.view(np.int32)).cuda() for a in (k1, v1, k2, v2)]
        A = mq.DeviceTable.from_torch([0, 1], cols[:2])
        B = mq.DeviceTable.from_torch([0, 2], cols[2:])
        ctx.table_bounds(A)
        ctx.table_bounds(B)
        pinned_bufs = None
        args.no_e2e = True  # e2e is the LUBM query's host-buffer path

        def step():
            r, _ = mqd.join_dist(ctx, A, B)
            m = r.nrows
            r.release()
            return m
    else:
        lo, hi = nu * rank // world, nu * (rank + 1) // world
        (s, p, o), st, pinned_bufs = lubm_host(
            nu, lo, hi, pinned=not args.no_e2e and args.store == "scan")
        trip = tuple(torch.from_numpy(a.view(np.int32)).cuda() for a in (s, p, o))
        pats = query_patterns(qname)
        source = trip
        hidx = None
        if args.store == "index":  # each rank indexes its own shard once, at load time
            source = ctx.index_build(trip)
            del trip
            torch.cuda.empty_cache()
            if not args.no_e2e:  # and mirrors it into pinned host memory (the e2e store)
                hidx = ctx.index_to_host(source)

        def step():
            r = mqd.query_dist(ctx, source, pats)
            return r.nrows

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    tdist.barrier()

    def timed(profile: bool):
        ctx.stats_reset()
        ctx.set_profiling(profile)
        x0 = dict(mqd.EXCHANGE)  # (the torch all_to_all fallback counts here, not in the stats)
        ms = []
        with ClockSampler(local) as clk:
            time.sleep(0.01)  # (let the sampler thread start polling before the first timed step)
            for _ in range(args.steps):
                tdist.barrier()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                step()
                e1.record()
                torch.cuda.synchronize()
                ms.append(e0.elapsed_time(e1))
        ctx.set_profiling(False)
        st_ = ctx.stats()
        return ms, st_, clk.summary(), (st_["exchange_bytes"] + mqd.EXCHANGE["bytes_sent"]
                                        - x0["bytes_sent"])

    # region 1 (the value): no per-kernel events; region 2: per-kernel events for the roofline
    ms, st_plain, clocks, sent = timed(False)
    _, st_k, _, _ = timed(True)
    # e2e at N GPUs: every step each rank copies from pinned host memory what its shard's query
    # needs (index store: the touched predicate ranges of its host-resident store; scan store:
    # its whole shard), runs the distributed query and reads its result shard back; the step
    # time is the max over ranks
    e2e = None
    # every rank takes the same branch: the fused-exchange fallback flag is agreed on first
    fb = torch.tensor([1 if getattr(ctx, "ipc_unavailable", None) else 0], device=cdev)
    tdist.all_reduce(fb, op=tdist.ReduceOp.MAX)
    if not args.no_e2e and not (hidx is not None and int(fb.item())):
        if hidx is None:
            dev_bufs = [torch.empty(len(s), dtype=torch.int32, device="cuda") for _ in range(3)]
        e2e_ms, h2d, d2h = [], 12 * len(s), 0
        for i in range(max(1, min(args.steps, 5)) + 1):  # (median of up to 5 after a warm run)
            tdist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if hidx is not None:
                got = mqd._fused_call(ctx, lambda: ctx.query_dist_host(hidx, pats))
                if got is None:
                    raise RuntimeError(f"fused exchange unavailable: {ctx.ipc_unavailable}")
                _, rows = got
                h2d, d2h = hidx.last_h2d_bytes, rows.nbytes
            else:
                for d, h in zip(dev_bufs, pinned_bufs):
                    d.copy_(h, non_blocking=True)
                r = mqd.query_dist(ctx, tuple(dev_bufs), pats)
                host = [c.cpu() for c in r.columns]
                d2h = sum(x.numel() * 4 for x in host)
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t0) * 1e3
            if i:
                e2e_ms.append(dt)
        tm = torch.tensor([statistics.median(e2e_ms)], dtype=torch.float64, device=cdev)
        tdist.all_reduce(tm, op=tdist.ReduceOp.MAX)
        io = torch.tensor([h2d, d2h], dtype=torch.float64, device=cdev)
        tdist.all_reduce(io, op=tdist.ReduceOp.SUM)
        e2e = (float(tm.item()), float(io[0].item()), float(io[1].item()))
    t = torch.tensor([sum(ms)], dtype=torch.float64, device=cdev)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    agg = torch.tensor([st_plain["join_in_rows"] + st_plain["join_out_rows"], st_plain["launches"],
                        sent], dtype=torch.float64, device=cdev)
    tdist.all_reduce(agg, op=tdist.ReduceOp.SUM)
    # the fused scatter (partition + NVLink stores into the peers' arenas): bytes this rank sent
    # to peers over its scatter kernels' event-timed duration (profiled region), max over ranks
    sc = st_k["kernels"].get("partition_scatter", {"ms": 0.0, "launches": 0})
    xr = torch.tensor([st_k["exchange_bytes"] / max(sc["ms"], 1e-9) / 1e6 if sc["ms"] else 0.0,
                       sc["ms"] / args.steps], dtype=torch.float64, device=cdev)
    xmin = xr.clone()
    tdist.all_reduce(xr, op=tdist.ReduceOp.MAX)
    tdist.all_reduce(xmin, op=tdist.ReduceOp.MIN)
    total_s = float(t.item()) / 1e3
    if rank == 0:
        tup, launches, sent_all = (float(x) for x in agg.tolist())
        peak, peak_src = measured_peaks()
        name, kd = max(st_k["kernels"].items(), key=lambda kv: kv[1]["ms"])
        avg_ms = kd["ms"] / kd["launches"]
        achieved = (kd["bytes"] / kd["launches"]) / (avg_ms / 1e3) / 1e9
        line = {"metric": METRIC, "value": tup / total_s, "unit": "tuples/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": total_s * 1e3 / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
                "config": {"workload": cfg, "description": desc,
                           "parallelism": f"hash-partitioned x{world}",
                           "store": args.store if kind == "lubm" else None,
                           "semijoin_filter": args.semijoin, "l2": "inputs larger than L2",
                           "exchange_path": ("torch all_to_all (CUDA IPC unavailable: "
                                             f"{ctx.ipc_unavailable})"
                                             if getattr(ctx, "ipc_unavailable", None) else
                                             "fused K8 scatter into CUDA-IPC peer arenas "
                                             "(mapsq_*_dist)")},
                "exchange": {"bytes_per_step": sent_all / args.steps,
                             "gbs_over_step_time": sent_all / total_s / 1e9,
                             "scatter_ms_per_step_max_rank": float(xr[1].item()),
                             "per_rank_send_gbs": {"min": float(xmin[0].item()),
                                                   "max": float(xr[0].item())},
                             "nvlink_peak_gbs": NVLINK_PEER_GBS,
                             "nvlink_frac_min_rank": float(xmin[0].item()) / NVLINK_PEER_GBS,
                             "note": "bytes all ranks sent to peers per step (fused partition + "
                                     "NVLink exchange); per-rank send rate = bytes stored into "
                                     "peers' arenas / that rank's partition_scatter kernel time, "
                                     "against the measured 770 GB/s per-direction peer copy "
                                     "(B200_PROFILING.md; 900 nominal)"},
                "roofline": {"kernel": name, "bound": "hbm", "achieved": achieved, "peak": peak,
                             "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak,
                             "traffic": None, "rank": 0},
                "e2e": None if e2e is None else {
                    "value": (tup / args.steps) / (e2e[0] / 1e3), "unit": "tuples/s",
                    "h2d_bytes_per_step": e2e[1], "d2h_bytes_per_step": e2e[2],
                    "ms_per_step": e2e[0],
                    "path": ("per rank: mapsq_query_dist_host_indexed (touched predicate ranges "
                             "of the rank's host store H2D, distributed joins, result shard D2H)"
                             if args.store == "index" else
                             "per rank: pinned shard H2D, full-table scan, distributed joins, "
                             "result shard D2H") + "; max over ranks"},
                "clocks": clocks, "gpu_launches": int(launches),
                "kernels": {k: {"launches": v["launches"], "avg_ms": v["ms"] / v["launches"],
                                "rank": 0} for k, v in st_k["kernels"].items()}}
        print(json.dumps(line), flush=True)
    tdist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="mapsq", choices=["mapsq", "reference"])
    ap.add_argument("--univ", type=int, default=0, help="override the LUBM scale (testing)")
    ap.add_argument("--rows", type=int, default=0, help="override C4 rows per side (testing)")
    ap.add_argument("--store", default="index", choices=["index", "scan"],
                    help="LUBM configs: answer patterns from the predicate-range index (default) "
                         "or scan the whole triple table every step")
    ap.add_argument("--semijoin", default="auto", choices=["auto", "on", "off"],
                    help="semi-join key-presence filter in front of the Map (auto: joins of "
                         ">= 2^22 rows)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--force-dist", action="store_true",
                    help="testing: run the multi-GPU path (exchange per join) even at world size 1")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl != "reference":
        relaunch_under_torchrun(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


def relaunch_under_torchrun(args):
    """`bench.py --gpus N` started directly: re-exec under torch.distributed.run with N ranks on
    this node (the driver's launch, 127.0.0.1 rendezvous).  Fails loudly when fewer than N GPUs
    are visible instead of printing a 1-GPU line."""
    import socket

    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        log(f"bench.py --gpus {args.gpus}: only {have} GPU(s) visible")
        sys.exit(2)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(port), os.path.abspath(__file__), *sys.argv[1:]]
    log("relaunching:", " ".join(cmd))
    os.execv(sys.executable, cmd)


if __name__ == "__main__":
    main()
