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
ctx.set_profiling(True)
ctx.stats_reset()
for _ in range(N):
    ctx.query(idx, pats).release()
torch.cuda.synchronize()
ks = ctx.stats()["kernels"]
ctx.set_profiling(False)
print({"python_wall_us": round(wall, 1), "event_us": round(ev, 1), "c_call_wall_us": round(ccall, 1),
       "kernels_us": {kk: round(v["ms"] / v["launches"] * 1e3, 1) for kk, v in ks.items()},
       "rows": m})
