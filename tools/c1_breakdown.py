"""Where C1's step time goes (TOOL, run on a B200): host wall time of the query call, the device
time between events around it (bench.py's step), and the small-join kernel alone."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import datagen  # noqa: E402
import paper_1702_03484_b200 as mq  # noqa: E402

ctx = mq.Context(0)
s, p, o, st = datagen.lubm(1, 0, 1)
trip = tuple(torch.from_numpy(a.view(np.int32)).cuda() for a in (s, p, o))
idx = ctx.index_build(trip)
pats = bench.query_patterns("C1")
stream = torch.cuda.current_stream()
N = 500
for _ in range(50):
    ctx.query(idx, pats).release()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(N):
    r = ctx.query(idx, pats)
    m = r.nrows
    r.release()
wall = (time.perf_counter() - t0) / N * 1e6
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(N):
    r = ctx.query(idx, pats)
    r.release()
e1.record(stream)
torch.cuda.synchronize()
ev = e0.elapsed_time(e1) / N * 1e3
# the C call alone (patterns marshalled once)
import ctypes  # noqa: E402
k = len(pats)
P = (mq._Pattern * k)(*[mq.pattern_struct(q) for q in pats])
pr = (ctypes.c_int32 * 1)()
out = mq._Table()
lib = mq.lib()
t0 = time.perf_counter()
for _ in range(N):
    lib.mapsq_query_indexed(ctx.handle, idx.handle, P, k, pr, 0, ctypes.byref(out), None)
    lib.mapsq_table_release(ctx.handle, ctypes.byref(out), None)
ccall = (time.perf_counter() - t0) / N * 1e6
q = ctx.prepare(idx, pats)
t0 = time.perf_counter()
for _ in range(N):
    r = q()
    m = r.nrows
    r.release()
prep = (time.perf_counter() - t0) / N * 1e6
ctx.set_profiling(True)
ctx.stats_reset()
for _ in range(N):
    ctx.query(idx, pats).release()
torch.cuda.synchronize()
ks = ctx.stats()["kernels"]
ctx.set_profiling(False)
print({"python_wall_us": round(wall, 1), "prepared_wall_us": round(prep, 1), "event_us": round(ev, 1), "c_call_wall_us": round(ccall, 1),
       "kernels_us": {kk: round(v["ms"] / v["launches"] * 1e3, 1) for kk, v in ks.items()},
       "rows": m})
# bench.py's loop: L2 flush, events around the step, with and without the flush
l2 = torch.cuda.get_device_properties(0).L2_cache_size
flush = torch.empty(4 * l2 // 4, dtype=torch.int32, device="cuda")
for fl in (True, False):
    evs = []
    for _ in range(200):
        if fl:
            flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        r = q()
        m = r.nrows
        r.release()
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    ts = sorted(x.elapsed_time(y) * 1e3 for x, y in evs)
    print({"flush": fl, "mean_us": round(sum(ts) / len(ts), 1), "median_us": round(ts[len(ts) // 2], 1),
           "min_us": round(ts[0], 1), "p90_us": round(ts[int(len(ts) * 0.9)], 1)})
# the same loop while bench.py's NVML sampler thread polls every `period` seconds
import threading  # noqa: E402

import pynvml as nv  # noqa: E402
nv.nvmlInit()
hdl = nv.nvmlDeviceGetHandleByIndex(0)
for period in (0.002, 0.02, None):
    stop = threading.Event()

    def poll():
        while not stop.is_set():
            t = time.perf_counter()
            nv.nvmlDeviceGetClockInfo(hdl, nv.NVML_CLOCK_SM)
            nv.nvmlDeviceGetCurrentClocksEventReasons(hdl)
            poll.cost.append(time.perf_counter() - t)
            time.sleep(period)
    poll.cost = []
    th = threading.Thread(target=poll, daemon=True) if period else None
    if th:
        th.start()
    evs = []
    for _ in range(2000):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        r = q()
        m = r.nrows
        r.release()
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    stop.set()
    if th:
        th.join()
    ts = sorted(x.elapsed_time(y) * 1e3 for x, y in evs)
    print({"sampler_period_s": period, "mean_us": round(sum(ts) / len(ts), 1),
           "median_us": round(ts[len(ts) // 2], 1), "p90_us": round(ts[int(len(ts) * 0.9)], 1),
           "nvml_call_us": round(1e6 * sum(poll.cost) / max(1, len(poll.cost)), 1)})
