"""Multi-GPU MapSQ join (SURVEY §8 rows b and e): hash partition on the join key, exchange, local join.

An equi-join decomposes over disjoint key sets, so each join needs exactly one exchange: every rank
hash-partitions both inputs on the shared variables (dest = (fmix32(fold(key)) * world) >> 32) and runs
the local Algorithm-1 join on the rows it receives.  Results stay sharded: the union over ranks is
RS.  A chained join whose key equals the key the accumulated result is already partitioned on skips
re-partitioning that side (C3's star joins on ?x three times: one exchange).

On GPUs with NCCL (``fused=True``, the default) the whole distributed join / query runs inside
libmapsq: ``mapsq_join_dist`` / ``mapsq_query_dist[_indexed]`` (csrc/dist.cu) partition with the K8
plan, all-gather the count matrix with NCCL, and ONE kernel stores every row straight into its
destination rank's CUDA-IPC receive arena over NVLink/NVSwitch.  This module only bootstraps the
library's communicator (``Context.dist_init``: the unique id travels over torch.distributed).

``fused=False`` (and the CPU gloo tests) run the same algorithm orchestrated here with
``mapsq_partition`` + ``torch.distributed.all_to_all_single``; ``partition_fn`` / ``join_fn`` are
injectable so that host-side logic is exercised on CPU (tests/test_dist_gloo.py).
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
    """The fused exchange's layout (``mapsq_exchange_layout``, host-only C): from C[s][d] (rows
    rank s sends to rank d), this rank's first row in every destination's receive block (rows of
    sources s < rank come first, so the received table is grouped by source rank exactly like
    all_to_all's output), every rank's received row count, and every rank's receive-block bytes."""
    import paper_1702_03484_b200 as mq
    return mq.exchange_layout(count_matrix, rank, ncols)


def ensure_dist(ctx, group=None):
    """Bootstrap the library's NCCL communicator for ``ctx`` once (collective)."""
    if getattr(ctx, "dist_world", None) is None:
        ctx.dist_init(group)


def _fused_call(ctx, fn):
    """Run a library distributed call; if CUDA IPC between the rank processes is unavailable (the
    error is the same on every rank: it happens while opening the peers' arenas), remember it and
    return None so the caller falls back to the torch all_to_all exchange."""
    import warnings

    import paper_1702_03484_b200 as mq
    try:
        return fn()
    except mq.MapsqError as e:
        if "CUDA IPC" not in str(e):
            raise
        ctx.ipc_unavailable = str(e)
        warnings.warn(f"fused NVLink exchange unavailable ({e}); using torch all_to_all")
        return None


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
    if fused is None:  # the library path: NCCL, or a context joined with host collectives
        fused = partition_fn is None and (dist.get_backend(group) == "nccl" or
                                          getattr(ctx, "dist_world", None) is not None)
    if fused and not getattr(ctx, "ipc_unavailable", None):
        ensure_dist(ctx, group)
        rs = _fused_call(ctx, lambda: ctx.join_dist(tp1, tp2))
        if rs is not None:
            return rs, key
    wrap = wrap_fn or (lambda vars_, cols: mq.DeviceTable.from_torch(vars_, cols))

    def move(t, slot):
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
    """Distributed ``mapsq_query`` over this rank's shard of the triple table ((s, p, o) tensors
    or an Index): local scan (no exchange: every pattern is matched on the shard the triple lives
    on), then the left-deep fold with one hash exchange per join key change, then zero-copy
    projection.  Returns this rank's shard of the result."""
    import paper_1702_03484_b200 as mq
    if fused is None:  # the library path: NCCL, or a context joined with host collectives
        fused = (dist.get_backend(group) == "nccl" or
                 getattr(ctx, "dist_world", None) is not None)
    if fused and not getattr(ctx, "ipc_unavailable", None):
        ensure_dist(ctx, group)
        rs = _fused_call(ctx, lambda: ctx.query_dist(triples_shard, patterns, proj))
        if rs is not None:
            return rs
    tabs = ctx.scan_patterns(triples_shard, patterns)
    acc, part_key = tabs[0], None
    for t in tabs[1:]:
        acc, part_key = join_dist(ctx, acc, t, group, tp1_partitioned_on=part_key, fused=False)
    order = list(dict.fromkeys(x for pat in patterns for kind, x in pat if kind == "v"))
    want = list(proj) if proj else order
    # zero-copy projection: the column tensors keep the shard's allocation alive
    return mq.DeviceTable.from_torch(want, [acc.column(v) for v in want])
