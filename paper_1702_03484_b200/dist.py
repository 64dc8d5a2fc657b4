"""Multi-GPU MapSQ join (SURVEY §8 row e): hash partition on the join key, all-to-all, local join.

An equi-join decomposes over disjoint key sets, so each join needs exactly one exchange: every rank
hash-partitions both inputs on the shared variables with the K8 kernel (``mapsq_partition``:
dest = fmix32(fold(key)) mod world), exchanges per-destination row counts and then the rows with
``torch.distributed.all_to_all_single`` (NCCL over NVLink/NVSwitch on GPUs, gloo in CPU tests), and
runs the local Algorithm-1 join (``mapsq_join``) on what it received.  Results stay sharded: the
union over ranks is RS.  A chained join whose key equals the key the accumulated result is already
partitioned on skips re-partitioning that side (C3's star joins on ?x three times: one exchange).

This module only orchestrates (argument marshalling + collectives); the partition and the join run
in libmapsq's CUDA kernels.  ``partition_fn`` / ``join_fn`` are injectable so the host-side logic
can be exercised on CPU with gloo (tests/test_dist_gloo.py).
"""
from __future__ import annotations

from typing import Callable, List, Sequence

import torch
import torch.distributed as dist


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


def redistribute(ctx, table, key_vars, group=None, partition_fn: Callable = None):
    """Hash-partition `table` on `key_vars` across the group; returns (vars, received columns)."""
    world = dist.get_world_size(group)
    if partition_fn is None:
        part, counts = ctx.partition(table, list(key_vars), world)
        cols, vars_ = part.columns, part.vars
    else:
        vars_, cols, counts = partition_fn(table, list(key_vars), world)
    recv = exchange_counts(counts, group)
    return vars_, exchange_columns(cols, counts, recv, group), recv


def join_dist(ctx, tp1, tp2, group=None, tp1_partitioned_on=None, partition_fn: Callable = None,
              join_fn: Callable = None, wrap_fn: Callable = None):
    """Distributed ``mapsq_join``: returns (local RS shard, the key variables it is partitioned on).

    ``tp1_partitioned_on``: key variables tp1 is already hash-partitioned on (skip its exchange
    when they equal this join's key)."""
    import paper_1702_03484_b200 as mq
    key = shared_vars(tp1.vars, tp2.vars)
    if not key:
        raise mq.MapsqError(2, "join inputs share no variable")
    wrap = wrap_fn or (lambda vars_, cols: mq.DeviceTable.from_torch(vars_, cols))
    if tp1_partitioned_on is not None and list(tp1_partitioned_on) == key:
        a = tp1
    else:
        va, ca, _ = redistribute(ctx, tp1, key, group, partition_fn)
        a = wrap(va, ca)
    vb, cb, _ = redistribute(ctx, tp2, key, group, partition_fn)
    b = wrap(vb, cb)
    rs = (join_fn or ctx.join)(a, b)
    return rs, key


def query_dist(ctx, triples_shard, patterns, proj=None, group=None):
    """Distributed ``mapsq_query`` over a university-range shard of the triple table: local fused
    scan (no exchange: every pattern is matched on the shard the triple lives on), then the
    left-deep fold with one hash exchange per join key change, then zero-copy projection."""
    import paper_1702_03484_b200 as mq
    tabs = ctx.scan_patterns(triples_shard, patterns)
    acc, part_key = tabs[0], None
    for t in tabs[1:]:
        acc, part_key = join_dist(ctx, acc, t, group, tp1_partitioned_on=part_key)
    order = list(dict.fromkeys(x for pat in patterns for kind, x in pat if kind == "v"))
    want = list(proj) if proj else order
    # zero-copy projection: the column tensors keep the shard's allocation alive
    return mq.DeviceTable.from_torch(want, [acc.column(v) for v in want])
