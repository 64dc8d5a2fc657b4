"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck, one tool per run):
every kernel family of the join path on small inputs — fused scan, index build + views, the
semi-join filter (exact single column, hashed composite key, word rounds), the one-sweep radix
passes and their decoupled look-back, find_groups, the u32/u64 scans, expand, the HASH/RESIDUAL
verify-emit, the K8 partition — each result checked against the CPU oracle.

  compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import datagen  # noqa: E402
import oracle  # noqa: E402
import paper_1702_03484_b200 as mq  # noqa: E402
from fixtures import config_query  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.uint32).view(np.int32)).cuda()


def check(got, ref, ordered=False):
    rows = got.to_numpy()
    assert got.vars == ref.vars
    if ordered:
        assert np.array_equal(rows, ref.rows)
    else:
        assert np.array_equal(oracle.canonical_rows(rows), oracle.canonical(ref).rows)


def main():
    ctx = mq.Context(0)
    s, p, o, _ = datagen.lubm(2)
    trip = (dev(s), dev(p), dev(o))
    idx = ctx.index_build(trip)
    for mode in (mq.SEMIJOIN_ON, mq.SEMIJOIN_OFF):
        ctx.set_option(mq.OPT_SEMIJOIN, mode)
        for cfg in ("C1", "C2", "C3", "C5"):
            ref = oracle.query(s, p, o, config_query(cfg))
            check(ctx.query(idx, config_query(cfg)), ref)
            check(ctx.query(trip, config_query(cfg)), ref)
    rng = np.random.default_rng(5)
    # single key, Zipf-like skew, filter on (exact bitmap) -> sort -> groups -> expand
    k1, v1 = datagen.zipf(200_000, 0, kbits=16)
    k2, v2 = datagen.zipf(200_000, 1, kbits=16)
    A = np.stack([k1, v1], 1)
    B = np.stack([k2, v2], 1)
    ref = oracle.join(oracle.Table([0, 1], A), oracle.Table([0, 2], B))
    got = ctx.join(mq.DeviceTable.from_torch([0, 1], [dev(k1), dev(v1)]),
                   mq.DeviceTable.from_torch([0, 2], [dev(k2), dev(v2)]))
    check(got, ref, ordered=True)
    # composite wide keys: HASH (filter rounds + verify-emit) and RESIDUAL (count-first)
    for wide in (mq.WIDE_KEY_HASH, mq.WIDE_KEY_RESIDUAL):
        ctx.set_option(mq.OPT_WIDE_KEY, wide)
        n1, n2 = 60_000, 90_000
        x1 = rng.integers(0, 3000, n1); z1 = rng.integers(0, 4, n1)
        x2 = rng.integers(0, 3000, n2); z2 = rng.integers(0, 4, n2)
        x1[:800] = 9; x2[:700] = 9
        x1[-1] = z1[-1] = 0xFFFFFFFF; x2[-1] = z2[-1] = 0
        A = np.stack([x1, z1, rng.integers(0, 99, n1)], 1).astype(np.uint32)
        B = np.stack([z2, x2], 1).astype(np.uint32)
        ref = oracle.join(oracle.Table([0, 1, 2], A), oracle.Table([1, 0], B))
        got = ctx.join(mq.DeviceTable.from_torch([0, 1, 2], [dev(A[:, c]) for c in range(3)]),
                       mq.DeviceTable.from_torch([1, 0], [dev(B[:, c]) for c in range(2)]))
        check(got, ref)
    ctx.set_option(mq.OPT_WIDE_KEY, mq.WIDE_KEY_HASH)
    # phase entry points: sort words, reduce groups; K8 partition
    w = rng.integers(0, 1 << 62, 300_001, dtype=np.uint64)
    t = torch.from_numpy(w.view(np.int64)).cuda()
    ctx.sort_words(t, 0, 62)
    assert np.array_equal(t.cpu().numpy().view(np.uint64), np.sort(w))
    tab = mq.DeviceTable.from_torch([0, 1], [dev(A[:, 0]), dev(A[:, 2])])
    part, counts = ctx.partition(tab, [0], 5)
    assert sum(counts) == len(A)
    torch.cuda.synchronize()
    print("sanitize_run ok")


if __name__ == "__main__":
    main()
