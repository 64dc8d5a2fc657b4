"""World-size-2 gloo tests of the multi-GPU join orchestration (paper_1702_03484_b200.dist) on CPU.

The hash partition and the local join are injected (numpy re-derivation of the K8 hash and the CPU
oracle) because this box has no GPU; what is exercised is the host-side exchange logic: count
all-to-all, row all-to-all with uneven splits, key-change detection and skipped re-partitioning.
Property checked: the union over ranks of the result shards equals the single-process join."""
from __future__ import annotations

import os
import socket
from collections import Counter

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle


class HostTable:
    def __init__(self, vars_, cols):
        self.vars = list(vars_)
        self.columns = [torch.as_tensor(np.asarray(c, np.uint32).view(np.int32)) for c in cols]
        self.nrows = int(self.columns[0].numel()) if self.columns else 0

    def column(self, v):
        return self.columns[self.vars.index(v)]

    def rows(self):
        if not self.columns:
            return np.zeros((0, 0), np.uint32)
        return np.stack([c.numpy().view(np.uint32) for c in self.columns], 1)


def fmix32(h):
    h = h ^ (h >> np.uint64(16)); h = (h * np.uint64(0x85EBCA6B)) & np.uint64(0xFFFFFFFF)
    h = h ^ (h >> np.uint64(13)); h = (h * np.uint64(0xC2B2AE35)) & np.uint64(0xFFFFFFFF)
    return h ^ (h >> np.uint64(16))


def np_partition(table, key_vars, world):
    """The K8 contract: dest = (fmix32(FNV-style fold of the key) * world) >> 32, stable within dest."""
    rows = table.rows()
    h = np.full(len(rows), 0x811C9DC5, np.uint64)
    for v in key_vars:
        h = ((h ^ rows[:, table.vars.index(v)].astype(np.uint64)) * np.uint64(0x01000193)) & np.uint64(0xFFFFFFFF)
    dest = ((fmix32(h) * np.uint64(world)) >> np.uint64(32)).astype(np.int64)
    order = np.argsort(dest, kind="stable")
    counts = np.bincount(dest, minlength=world).tolist()
    part = rows[order]
    cols = [torch.as_tensor(np.ascontiguousarray(part[:, c]).view(np.int32)) for c in range(part.shape[1])]
    return table.vars, cols, counts


def oracle_join(a, b):
    r = oracle.join(oracle.Table(a.vars, a.rows()), oracle.Table(b.vars, b.rows()))
    return HostTable(r.vars, [r.rows[:, c] for c in range(len(r.vars))])


def wrap(vars_, cols):
    return HostTable(vars_, [c.numpy().view(np.uint32) for c in cols])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1702_03484_b200 import dist as mqd
        rng = np.random.default_rng(100 + rank)   # each rank holds its own shard of the inputs
        A = HostTable([0, 1], [rng.integers(0, 50, 700 + 50 * rank), rng.integers(0, 9, 700 + 50 * rank)])
        B = HostTable([2, 0], [rng.integers(0, 9, 400), rng.integers(0, 60, 400)])
        C = HostTable([0, 3], [rng.integers(0, 50, 300 + 7 * rank), rng.integers(0, 5, 300 + 7 * rank)])
        D = HostTable([1, 3], [rng.integers(0, 9, 200), rng.integers(0, 5, 200)])
        kw = dict(partition_fn=np_partition, join_fn=oracle_join, wrap_fn=wrap)
        x0 = dict(mqd.EXCHANGE)
        _, _, ca = np_partition(A, [0], world)
        _, _, cb = np_partition(B, [0], world)
        r1, key1 = mqd.join_dist(None, A, B, **kw)
        # exchange accounting: bytes of the rows this rank sent to the OTHER rank
        other = 1 - rank
        assert mqd.EXCHANGE["exchanges"] - x0["exchanges"] == 2
        assert mqd.EXCHANGE["rows_sent"] - x0["rows_sent"] == ca[other] + cb[other]
        assert mqd.EXCHANGE["bytes_sent"] - x0["bytes_sent"] == 8 * (ca[other] + cb[other])
        # same key (?0): acc is not re-partitioned
        r2, key2 = mqd.join_dist(None, r1, C, tp1_partitioned_on=key1, **kw)
        # key change (?1, ?3): both sides exchanged on the composite key
        r3, key3 = mqd.join_dist(None, r2, D, tp1_partitioned_on=key2, **kw)
        q.put((rank, [A.rows(), B.rows(), C.rows(), D.rows()],
               [(r.vars, r.rows()) for r in (r1, r2, r3)], [key1, key2, key3]))
    finally:
        dist.destroy_process_group()


def test_join_dist_gloo_world2():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda t: t[0])
    inputs = [np.concatenate([r[1][i] for r in res]) for i in range(4)]
    A, B, C, D = (oracle.Table(v, x) for v, x in zip([[0, 1], [2, 0], [0, 3], [1, 3]], inputs))
    full1 = oracle.join(A, B)
    full2 = oracle.join(full1, C)
    full3 = oracle.join(full2, D)
    assert res[0][3] == [[0], [0], [1, 3]]
    for step, full in enumerate([full1, full2, full3]):
        vars_ = res[0][2][step][0]
        assert vars_ == full.vars
        union = Counter()
        for r in res:
            assert r[2][step][0] == vars_
            union.update(tuple(x) for x in r[2][step][1].tolist())
        assert union == Counter(tuple(x) for x in full.rows.tolist()), step
        # every key lives on exactly one rank
        keys = [set(tuple(x) for x in r[2][step][1][:, :len(res[0][3][step])].tolist()) for r in res]
        assert not (keys[0] & keys[1])


def test_exchange_layout_matches_all_to_all_order():
    """The fused exchange writes rank s's rows for d at rows sum_{s'<s} C[s'][d] of d's arena:
    exactly the source-rank-grouped order all_to_all_single produces."""
    from paper_1702_03484_b200.dist import exchange_layout
    C = [[3, 0, 5], [1, 2, 0], [4, 4, 4]]
    rows = [exchange_layout(C, r, 2)[0] for r in range(3)]
    _, recv, need = exchange_layout(C, 0, 2)
    assert recv == [8, 6, 9] and need == [64, 64, 96]  # columns padded to 4 rows (16 B)
    assert [rows[r][0] for r in range(3)] == [0, 3, 4]
    assert [rows[r][1] for r in range(3)] == [0, 0, 2]
    assert [rows[r][2] for r in range(3)] == [0, 5, 5]
    # blocks tile every destination arena exactly
    for d in range(3):
        spans = sorted((rows[r][d], rows[r][d] + C[r][d]) for r in range(3))
        assert spans[0][0] == 0 and spans[-1][1] == recv[d]
        assert all(spans[i][1] == spans[i + 1][0] for i in range(2))


def test_exchange_layout_c_abi_definition():
    """mapsq_exchange_layout against its definition, written out as brute force over the matrix."""
    import paper_1702_03484_b200 as mq
    rng = np.random.default_rng(7)
    for world in (1, 2, 3, 8, 64):
        C = rng.integers(0, 1000, (world, world)).tolist()
        for rank in {0, world - 1, world // 2}:
            for ncols in (1, 3, 16):
                dest_row, recv, need = mq.exchange_layout(C, rank, ncols)
                for d in range(world):
                    assert recv[d] == sum(C[s][d] for s in range(world))
                    assert dest_row[d] == sum(C[s][d] for s in range(rank))
                    stride = -(-recv[d] // 4) * 4            # 16 B aligned columns
                    assert need[d] == 4 * ncols * stride and need[d] % 16 == 0
    for bad in ((2, 1), (0, 17), (0, 0)):                     # (rank, ncols) out of range
        with pytest.raises(mq.MapsqError):
            mq.exchange_layout([[1, 2], [3, 4]], *bad)
    with pytest.raises(mq.MapsqError):
        mq.exchange_layout([[0] * 65] * 65, 0, 1)             # more ranks than partitions


def test_fused_call_falls_back_only_on_ipc_errors():
    """dist._fused_call: a CUDA IPC failure (same on every rank) switches the context to the
    torch all_to_all exchange; any other library error propagates."""
    import warnings

    import paper_1702_03484_b200 as mq
    from paper_1702_03484_b200 import dist as mqd

    class Ctx:
        pass

    ctx = Ctx()
    assert mqd._fused_call(ctx, lambda: 42) == 42 and not hasattr(ctx, "ipc_unavailable")

    def ipc_fail():
        raise mq.MapsqError(4, "CUDA IPC: cudaIpcOpenMemHandle(...): invalid device context")

    with warnings.catch_warnings(record=True):
        warnings.simplefilter("always")
        assert mqd._fused_call(ctx, ipc_fail) is None
    assert "cudaIpcOpenMemHandle" in ctx.ipc_unavailable

    def other_fail():
        raise mq.MapsqError(3, "device allocation failed")

    with pytest.raises(mq.MapsqError):
        mqd._fused_call(Ctx(), other_fail)
