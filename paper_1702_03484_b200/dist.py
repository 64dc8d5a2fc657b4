"""Multi-GPU MapSQ join (SURVEY §8 row e): hash partition on the join key, exchange, local join.

An equi-join decomposes over disjoint key sets, so each join needs exactly one exchange: every rank
hash-partitions both inputs on the shared variables (dest = fmix32(fold(key)) mod world) and runs
the local Algorithm-1 join (``mapsq_join``) on the rows it receives.  Results stay sharded: the union
over ranks is RS.  A chained join whose key equals the key the accumulated result is already
partitioned on skips re-partitioning that side (C3's star joins on ?x three times: one exchange).

Exchange on GPUs (``fused=True``, the default with NCCL): the partition and the all-to-all are ONE
kernel.  Every rank owns two receive arenas (one per join side) exported once with CUDA IPC and
opened by all peers; per exchange the ranks run the K8 plan (destination counts), all-gather the
world x world count matrix (the only collective), and ``mapsq_partition_scatter`` stores each row
straight into its destination rank's arena over NVLink/NVSwitch.  ``fused=False`` (and the CPU
gloo tests) use ``mapsq_partition`` + ``torch.distributed.all_to_all_single`` instead.

This module only orchestrates (argument marshalling + collectives); partition, exchange stores and
join run in libmapsq's CUDA kernels.  ``partition_fn`` / ``join_fn`` are injectable so the
host-side logic can be exercised on CPU with gloo (tests/test_dist_gloo.py).
"""
from __future__ import annotations

from typing import Callable, List, Sequence

import torch
import torch.distributed as dist


# bytes and rows this process sent to OTHER ranks (both exchange paths), for reporting the
# exchange volume against NVLink bandwidth (bench.py)
EXCHANGE = {"bytes_sent": 0, "rows_sent": 0, "exchanges": 0}


def _account(counts: Sequence[int], rank: int, ncols: int):
    rows = sum(int(c) for d, c in enumerate(counts) if d != rank)
    EXCHANGE["rows_sent"] += rows
    EXCHANGE["bytes_sent"] += 4 * ncols * rows
    EXCHANGE["exchanges"] += 1


def exchange_counts(counts: Sequence[int], group=None) -> List[int]:
    """all-to-all of per-destination row counts: returns the per-source counts received."""
    world = dist.get_world_size(group)
    dev = _comm_device(group)
    send = torch.tensor(list(counts), dtype=torch.int64, device=dev)
    recv = torch.empty(world, dtype=torch.int64, device=dev)
    dist.all_to_all_single(recv, send, group=group)
    return [int(x) for x in recv.cpu().tolist()]


def exchange_columns(columns: Sequence[torch.Tensor], send_counts: Sequence[int],
                     recv_counts: Sequence[int], group=None) -> List[torch.Tensor]:
    """Send rows grouped by destination (rows of destination d contiguous, in rank order) and
    receive the rows destined to this rank, grouped by source rank.  4-byte columns."""
    out = []
    total = int(sum(recv_counts))
    for col in columns:
        c = col.view(torch.int32)
        r = torch.empty(total, dtype=torch.int32, device=c.device)
        dist.all_to_all_single(r, c, output_split_sizes=list(recv_counts),
                               input_split_sizes=list(send_counts), group=group)
        out.append(r)
    return out


def _comm_device(group=None):
    backend = dist.get_backend(group)
    return torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")


def shared_vars(vars1, vars2) -> List[int]:
    return sorted(set(vars1) & set(vars2))


def exchange_layout(count_matrix, rank: int, ncols: int):
    """From C[s][d] (rows rank s sends to rank d): this rank's first row in every destination's
    arena block (rows of sources s < rank come first, so the received table is grouped by source
    rank exactly like all_to_all's output), every rank's received row count, and the arena bytes
    every rank needs (columns of length recv[d], back to back)."""
    world = len(count_matrix)
    recv = [sum(count_matrix[s][d] for s in range(world)) for d in range(world)]
    dest_row = [sum(count_matrix[s][d] for s in range(rank)) for d in range(world)]
    need = [4 * ncols * recv[d] for d in range(world)]
    return dest_row, recv, need


class PeerArenas:
    """Receive arenas of every rank, mapped into this process (own arena: local pointer; peers':
    CUDA IPC).  ``ensure`` is collective: every rank calls it with the same per-rank byte needs
    and grows exactly the arenas that are too small, re-exchanging their handles."""

    def __init__(self, ctx, group=None, nslots: int = 2):
        self.ctx, self.group = ctx, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.nslots = nslots
        self.own = [0] * nslots                        # this rank's arena per slot
        self.cap = [[0] * self.world for _ in range(nslots)]
        self.ptr = [[0] * self.world for _ in range(nslots)]   # mapped arenas, per slot and rank

    def ensure(self, slot: int, need: Sequence[int]):
        cap = self.cap[slot]
        grow = [need[r] > cap[r] for r in range(self.world)]
        if not any(grow):
            return
        if grow[self.rank]:
            if self.own[slot]:
                self.ctx.ipc_free(self.own[slot])
            nbytes = max(1 << 20, int(need[self.rank] * 1.25) + 4096)
            self.own[slot] = self.ctx.ipc_alloc(nbytes)
            handle = self.ctx.ipc_export(self.own[slot])
        else:
            nbytes, handle = cap[self.rank], None
        info = [None] * self.world
        dist.all_gather_object(info, (grow[self.rank], nbytes, handle), group=self.group)
        for r, (grew, nb, h) in enumerate(info):
            if not grew:
                continue
            if r == self.rank:
                self.ptr[slot][r] = self.own[slot]
            else:
                if self.ptr[slot][r]:
                    self.ctx.ipc_close(self.ptr[slot][r])
                self.ptr[slot][r] = self.ctx.ipc_open(h)
            cap[r] = nb

    def close(self):
        for slot in range(self.nslots):
            for r in range(self.world):
                if r != self.rank and self.ptr[slot][r]:
                    self.ctx.ipc_close(self.ptr[slot][r])
            if self.own[slot]:
                self.ctx.ipc_free(self.own[slot])


_ARENAS = {}


def _arenas(ctx, group):
    key = (id(ctx), id(group))
    if key not in _ARENAS:
        _ARENAS[key] = PeerArenas(ctx, group)
    return _ARENAS[key]


def redistribute_fused(ctx, table, key_vars, slot: int, group=None):
    """Fused partition + exchange: returns (vars, received columns) — views of this rank's arena,
    grouped by source rank — valid until the next exchange into the same slot."""
    import paper_1702_03484_b200 as mq
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    state, counts = ctx.partition_plan(table, list(key_vars), world)
    _account(counts, rank, len(table.vars))
    dev = torch.device("cuda", torch.cuda.current_device())
    mine = torch.tensor(counts, dtype=torch.int64, device=dev)
    allc = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(allc, mine, group=group)
    matrix = [[int(x) for x in t.cpu().tolist()] for t in allc]
    ncols = len(table.vars)
    dest_row, recv, need = exchange_layout(matrix, rank, ncols)
    ar = _arenas(ctx, group)
    ar.ensure(slot, need)
    dest_cols = [ar.ptr[slot][d] + 4 * c * recv[d] for d in range(world) for c in range(ncols)]
    torch.cuda.synchronize()
    dist.barrier(group=group)       # no rank still reads the arenas it is about to receive into
    ctx.partition_scatter(state, dest_row, dest_cols)
    dist.barrier(group=group)       # every peer's stores into this rank's arena have completed
    cols = mq.device_columns(ar.own[slot], recv[rank], ncols, recv[rank], owner=ar)
    return list(table.vars), cols


def redistribute(ctx, table, key_vars, group=None, partition_fn: Callable = None):
    """Hash-partition `table` on `key_vars` across the group; returns (vars, received columns)."""
    world = dist.get_world_size(group)
    if partition_fn is None:
        part, counts = ctx.partition(table, list(key_vars), world)
        cols, vars_ = part.columns, part.vars
    else:
        vars_, cols, counts = partition_fn(table, list(key_vars), world)
    _account(counts, dist.get_rank(group), len(vars_))
    recv = exchange_counts(counts, group)
    return vars_, exchange_columns(cols, counts, recv, group), recv


def join_dist(ctx, tp1, tp2, group=None, tp1_partitioned_on=None, partition_fn: Callable = None,
              join_fn: Callable = None, wrap_fn: Callable = None, fused: bool = None):
    """Distributed ``mapsq_join``: returns (local RS shard, the key variables it is partitioned on).

    ``tp1_partitioned_on``: key variables tp1 is already hash-partitioned on (skip its exchange
    when they equal this join's key).  ``fused`` (default: on with NCCL and no injected
    partition_fn) selects the one-kernel partition + NVLink exchange."""
    import paper_1702_03484_b200 as mq
    key = shared_vars(tp1.vars, tp2.vars)
    if not key:
        raise mq.MapsqError(2, "join inputs share no variable")
    if fused is None:
        fused = partition_fn is None and dist.get_backend(group) == "nccl"
    wrap = wrap_fn or (lambda vars_, cols: mq.DeviceTable.from_torch(vars_, cols))

    def move(t, slot):
        if fused:
            return redistribute_fused(ctx, t, key, slot, group)
        v, c, _ = redistribute(ctx, t, key, group, partition_fn)
        return v, c

    if tp1_partitioned_on is not None and list(tp1_partitioned_on) == key:
        a = tp1
    else:
        a = wrap(*move(tp1, 0))
    b = wrap(*move(tp2, 1))
    rs = (join_fn or ctx.join)(a, b)
    return rs, key


def query_dist(ctx, triples_shard, patterns, proj=None, group=None, fused: bool = None):
    """Distributed ``mapsq_query`` over a university-range shard of the triple table: local fused
    scan (no exchange: every pattern is matched on the shard the triple lives on), then the
    left-deep fold with one hash exchange per join key change, then zero-copy projection."""
    import paper_1702_03484_b200 as mq
    tabs = ctx.scan_patterns(triples_shard, patterns)
    acc, part_key = tabs[0], None
    for t in tabs[1:]:
        acc, part_key = join_dist(ctx, acc, t, group, tp1_partitioned_on=part_key, fused=fused)
    order = list(dict.fromkeys(x for pat in patterns for kind, x in pat if kind == "v"))
    want = list(proj) if proj else order
    # zero-copy projection: the column tensors keep the shard's allocation alive
    return mq.DeviceTable.from_torch(want, [acc.column(v) for v in want])
