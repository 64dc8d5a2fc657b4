"""Diagnostic: host wall time vs device kernel time of one C4-style join, profiling on/off."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import datagen, paper_1702_03484_b200 as mq

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
ctx = mq.Context(0)
k1, v1 = datagen.zipf(n, 0); k2, v2 = datagen.zipf(n, 1)
cols = [torch.from_numpy(a.view(np.int32)).cuda() for a in (k1, v1, k2, v2)]
A = mq.DeviceTable.from_torch([0, 1], cols[:2]); B = mq.DeviceTable.from_torch([0, 2], cols[2:])
ctx.table_bounds(A); ctx.table_bounds(B)
for prof in (False, True, False):
    ctx.set_profiling(prof); ctx.stats_reset()
    for rep in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = ctx.join(A, B)
        e1.record(); torch.cuda.synchronize()
        t1 = time.perf_counter()
        m = r.nrows; r.release(); torch.cuda.synchronize(); t2 = time.perf_counter()
        print(f"prof={prof} rep={rep} host_join={1e3*(t1-t0):.2f}ms dev_join={e0.elapsed_time(e1):.2f}ms release={1e3*(t2-t1):.2f}ms m={m}")
    if prof:
        st = ctx.stats()
        print({k: round(v['ms'] / v['launches'], 4) for k, v in st['kernels'].items()})
# phase entry points
words = torch.empty(2 * n, dtype=torch.int64, device='cuda')
pl = mq.plan_join([0, 1], A.bounds, n, [0, 2], B.bounds, n)
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    ctx.map_words(A, B, pl, words); torch.cuda.synchronize(); t1 = time.perf_counter()
    ctx.sort_words(words, pl.ib, pl.ib + pl.kb); torch.cuda.synchronize(); t2 = time.perf_counter()
    g = ctx.reduce_groups(words, n, n, pl.ib); torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"map {1e3*(t1-t0):.2f} sort {1e3*(t2-t1):.2f} reduce {1e3*(t3-t2):.2f} ms")
# reference point only (never on the product path): CUB radix sort via torch.sort, 64-bit keys
x = torch.randint(0, 1 << 62, (2 * n,), device='cuda')
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    y = torch.sort(x).values; torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"torch.sort int64 2n={2*n}: {1e3*(t1-t0):.2f} ms (8 passes)")
x32 = torch.randint(0, 1 << 30, (2 * n,), device='cuda', dtype=torch.int32)
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    y = torch.sort(x32).values; torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"torch.sort int32 2n={2*n}: {1e3*(t1-t0):.2f} ms (4 passes)")
