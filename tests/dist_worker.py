"""One rank of the multi-process distributed tests (tests/test_gpu_dist2.py launches `world` of
these on ONE GPU).  The library's distributed path runs end to end — K8 partition plan, count
all-gather, CUDA-IPC receive arenas opened by every peer, the fused scatter kernel storing rows
into the peers' arenas, local Algorithm-1 joins — with its control plane carried by
torch.distributed's gloo backend (mapsq_dist_init_host; NCCL refuses two ranks on one device).
No kernel waits on another rank: every cross-rank dependency is a host collective.

Writes <out>/rank<r>.npz with every case's result shard and the exchange counters."""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def join_case_tables(case: int):
    """Deterministic random join inputs of a case (all ranks and the test build the same)."""
    rng = np.random.default_rng(1000 + case)
    if case == 0:    # single key, skewed: a hot key on both sides
        n1, n2 = 30000, 20000
        k1 = np.where(rng.random(n1) < 0.2, 7, rng.integers(0, 3000, n1))
        k2 = np.where(rng.random(n2) < 0.1, 7, rng.integers(0, 3000, n2))
        A = np.stack([k1, rng.integers(0, 1 << 32, n1, dtype=np.uint64)], 1)
        B = np.stack([rng.integers(0, 1 << 32, n2, dtype=np.uint64), k2], 1)
        return [0, 1], A.astype(np.uint32), [2, 0], B.astype(np.uint32)
    if case == 1:    # composite key (x, z), wide columns: HASH path after the exchange
        n1, n2 = 25000, 40000
        x1 = rng.integers(0, 2000, n1); z1 = rng.integers(0, 5, n1)
        x2 = rng.integers(0, 2000, n2); z2 = rng.integers(0, 5, n2)
        x1[0] = 0xFFFFFFFF; z2[0] = 0xFFFFFFFF
        A = np.stack([x1, rng.integers(0, 100, n1), z1], 1)
        B = np.stack([z2, x2, rng.integers(0, 100, n2)], 1)
        return [0, 1, 2], A.astype(np.uint32), [2, 0, 3], B.astype(np.uint32)
    if case == 3:    # skew: two heavy single keys (7: mostly tp1, 11: mostly tp2) + a cold tail
        n1, n2 = 40000, 30000
        u1, u2 = rng.random(n1), rng.random(n2)
        k1 = np.where(u1 < 0.4, 7, np.where(u1 < 0.43, 11, rng.integers(0, 5000, n1)))
        k2 = np.where(u2 < 0.05, 7, np.where(u2 < 0.35, 11, rng.integers(0, 5000, n2)))
        A = np.stack([k1, rng.integers(0, 1 << 32, n1, dtype=np.uint64)], 1)
        B = np.stack([rng.integers(0, 1 << 32, n2, dtype=np.uint64), k2], 1)
        return [0, 1], A.astype(np.uint32), [2, 0], B.astype(np.uint32)
    if case == 4:    # skew on a composite key (x, z) = (3, 4), wide columns: HASH path locally
        n1, n2 = 30000, 30000
        hot1, hot2 = rng.random(n1) < 0.3, rng.random(n2) < 0.2
        x1 = np.where(hot1, 3, rng.integers(0, 1 << 32, n1, dtype=np.uint64))
        z1 = np.where(hot1, 4, rng.integers(0, 9, n1))
        x2 = np.where(hot2, 3, rng.integers(0, 1 << 32, n2, dtype=np.uint64))
        z2 = np.where(hot2, 4, rng.integers(0, 9, n2))
        A = np.stack([x1, z1, np.arange(n1)], 1)
        B = np.stack([z2, x2], 1)
        return [0, 1, 2], A.astype(np.uint32), [1, 0], B.astype(np.uint32)
    # case 2: one side empty on some ranks (rows only in the first half)
    n1, n2 = 500, 6000
    A = np.stack([rng.integers(0, 50, n1), rng.integers(0, 9, n1)], 1)
    B = np.stack([rng.integers(0, 50, n2), rng.integers(0, 9, n2)], 1)
    return [0, 1], A.astype(np.uint32), [0, 2], B.astype(np.uint32)


NCASES = 5


def shard_rows(nrows: int, rank: int, world: int, case: int):
    if case == 2:  # uneven: all rows on rank 0
        return np.arange(nrows) if rank == 0 else np.arange(0)
    return np.arange(rank, nrows, world)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rank", type=int, required=True)
    ap.add_argument("--world", type=int, required=True)
    ap.add_argument("--port", type=int, required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--nu", type=int, default=2)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    import datagen
    import paper_1702_03484_b200 as mq
    from fixtures import config_query

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{args.port}", rank=args.rank,
                            world_size=args.world)
    torch.cuda.set_device(0)
    ctx = mq.Context(0)
    ctx.dist_init_host()
    res = {}

    def dev(a):
        return torch.from_numpy(np.ascontiguousarray(a, np.uint32).view(np.int32)).cuda()

    def put(name, t):
        res[name + ":vars"] = np.array(t.vars, np.int32)
        res[name] = t.to_numpy()

    # LUBM configs: each rank holds a contiguous university range of LUBM(nu)
    per = args.nu // args.world
    lo, hi = args.rank * per, (args.rank + 1) * per if args.rank + 1 < args.world else args.nu
    s, p, o, _ = datagen.lubm(args.nu, lo, hi)
    trip = (dev(s), dev(p), dev(o))
    idx = ctx.index_build(trip)
    for cfg in ("C1", "C2", "C3", "C5"):
        for mode in ("auto", "on"):
            ctx.set_option(mq.OPT_SEMIJOIN, mq.SEMIJOIN_ON if mode == "on" else mq.SEMIJOIN_AUTO)
            put(f"q_{cfg}_{mode}", ctx.query_dist(idx, config_query(cfg)))
        put(f"qscan_{cfg}", ctx.query_dist(trip, config_query(cfg)))
    ctx.set_option(mq.OPT_SEMIJOIN, mq.SEMIJOIN_AUTO)
    # random joins: rank r holds rows r::world of both inputs
    for case in range(NCASES):
        va, A, vb, B = join_case_tables(case)
        ra, rb = shard_rows(len(A), args.rank, args.world, case), shard_rows(len(B), args.rank, args.world, 0)
        ta = mq.DeviceTable.from_torch(va, [dev(A[ra, c]) for c in range(len(va))])
        tb = mq.DeviceTable.from_torch(vb, [dev(B[rb, c]) for c in range(len(vb))])
        for mode in ("auto", "on"):  # "on": the cross-rank pre-filter runs (masked exchange)
            ctx.set_option(mq.OPT_SEMIJOIN, mq.SEMIJOIN_ON if mode == "on" else mq.SEMIJOIN_AUTO)
            put(f"j{case}_{mode}", ctx.join_dist(ta, tb))
    ctx.set_option(mq.OPT_SEMIJOIN, mq.SEMIJOIN_AUTO)
    # the skew cases again with heavy-key handling off: same union, no split keys
    ctx.set_option(mq.OPT_SKEW, 0)
    for case in (3, 4):
        va, A, vb, B = join_case_tables(case)
        ra, rb = shard_rows(len(A), args.rank, args.world, case), shard_rows(len(B), args.rank, args.world, 0)
        ta = mq.DeviceTable.from_torch(va, [dev(A[ra, c]) for c in range(len(va))])
        tb = mq.DeviceTable.from_torch(vb, [dev(B[rb, c]) for c in range(len(vb))])
        sk0 = ctx.stats()["skew_keys"]
        put(f"j{case}_noskew", ctx.join_dist(ta, tb))
        assert ctx.stats()["skew_keys"] == sk0
    ctx.set_option(mq.OPT_SKEW, 1)
    st = ctx.stats()
    for k in ("exchanges", "exchange_rows", "exchange_bytes", "exchange_recv_rows",
              "exchange_recv_bytes", "skew_keys"):
        res["stat_" + k] = np.array(st[k], np.int64)
    torch.cuda.synchronize()
    dist.barrier()
    np.savez(os.path.join(args.out, f"rank{args.rank}.npz"), **res)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
