"""GPU parity of the semi-join filter in front of the Map (MAPSQ_OPT_SEMIJOIN).

Dropping rows whose key is absent from the other side must not change RS or its row order: every
case is compared IN ORDER against the oracle's sort-merge tier (same (key, tp1 row, tp2 row)
order as the unfiltered GPU join), with the filter forced on for all sizes, and the number of
dropped rows is checked against a brute-force count (exact bitmaps) or bounded (hashed).  Every
case runs with the filter's carried columns forced on, off and on auto."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import datagen  # noqa: E402
import oracle  # noqa: E402
import paper_1702_03484_b200 as mq  # noqa: E402
from fixtures import config_expected_counts, config_query  # noqa: E402


@pytest.fixture(params=["0", "1", "2"], autouse=True)
def carry(request, monkeypatch):
    """MAPSQ_SJ_CARRY: the column round carries ReduceDuplicate's columns through the filter
    (1), never (0), or when the sampled probe keeps at most half of the larger side (2, the
    default) — RS and its order must not depend on it."""
    monkeypatch.setenv("MAPSQ_SJ_CARRY", request.param)
    return request.param


@pytest.fixture(scope="module")
def ctx():
    c = mq.Context(0)
    yield c
    c.set_option(mq.OPT_SEMIJOIN, mq.SEMIJOIN_AUTO)


def dev(a):
    a = np.ascontiguousarray(a, dtype=np.uint32)
    return torch.from_numpy(a.view(np.int32)).cuda()


def dtable(vars_, rows):
    rows = np.asarray(rows, np.uint32).reshape(-1, len(vars_))
    return mq.DeviceTable.from_torch(vars_, [dev(rows[:, c]) for c in range(len(vars_))])


def unmatched_rows(A, B, ka, kb):
    """Rows of A and B whose key tuple does not occur on the other side."""
    sa = {tuple(r) for r in A[:, ka]}
    sb = {tuple(r) for r in B[:, kb]}
    return (sum(tuple(r) not in sb for r in A[:, ka]) + sum(tuple(r) not in sa for r in B[:, kb]))


@pytest.mark.parametrize("domain", [1, 7, 3000, 1 << 20, 1 << 31])
def test_filtered_join_equals_oracle(ctx, domain):
    rng = np.random.default_rng(domain % 65521)
    for n1, n2 in [(1, 1), (3, 4097), (4095, 4097), (20000, 7000), (70000, 90000)]:
        if n1 * n2 // domain > 20_000_000:  # keep |RS| (oracle memory) bounded
            continue
        A = np.stack([rng.integers(0, domain, n1, dtype=np.uint64),
                      rng.integers(0, 1 << 32, n1, dtype=np.uint64)], 1).astype(np.uint32)
        B = np.stack([rng.integers(0, 1 << 32, n2, dtype=np.uint64),
                      rng.integers(0, domain, n2, dtype=np.uint64)], 1).astype(np.uint32)
        ref = oracle.join(oracle.Table([0, 1], A), oracle.Table([2, 0], B))
        for mode in (mq.SEMIJOIN_ON, mq.SEMIJOIN_OFF):
            ctx.set_option(mq.OPT_SEMIJOIN, mode)
            got = ctx.join(dtable([0, 1], A), dtable([2, 0], B))
            assert got.vars == ref.vars
            assert np.array_equal(got.to_numpy(), ref.rows), (domain, n1, n2, mode)
            st = ctx.stats()
            if mode == mq.SEMIJOIN_OFF:
                assert st["last_filtered"] == 0
            elif max(A[:, 0].min(), B[:, 1].min()) > min(A[:, 0].max(), B[:, 1].max()):
                assert got.nrows == 0  # disjoint key bounds: the join returns before the Map
            elif st["last_kb"] <= 29:  # exact bitmaps: exactly the unmatched rows are dropped
                assert st["last_filtered"] == unmatched_rows(A, B, [0], [1])
            else:                      # hashed: never more than the unmatched rows
                assert st["last_filtered"] <= unmatched_rows(A, B, [0], [1])


def test_filtered_join_all_rows_dropped(ctx):
    ctx.set_option(mq.OPT_SEMIJOIN, mq.SEMIJOIN_ON)
    A = np.stack([np.arange(0, 5000, 2), np.arange(2500)], 1).astype(np.uint32)
    B = np.stack([np.arange(1, 5000, 2), np.arange(2500)], 1).astype(np.uint32)  # interleaved keys
    got = ctx.join(dtable([0, 1], A), dtable([0, 2], B))
    assert got.nrows == 0 and got.vars == [0, 1, 2]
    assert ctx.stats()["last_filtered"] == 5000


def test_filtered_composite_and_residual(ctx):
    ctx.set_option(mq.OPT_SEMIJOIN, mq.SEMIJOIN_ON)
    rng = np.random.default_rng(5)
    for dom in ([5, 9], [1 << 31, 3], [1 << 31, 1 << 31]):  # P64, P64 wide, RESIDUAL
        n1, n2 = 30000, 50000
        A = np.stack([rng.integers(0, dom[0], n1, dtype=np.uint64) % 300 * (dom[0] // 300 or 1),
                      rng.integers(0, dom[1], n1, dtype=np.uint64) % 40,
                      rng.integers(0, 1 << 32, n1, dtype=np.uint64)], 1).astype(np.uint32)
        B = np.stack([rng.integers(0, dom[0], n2, dtype=np.uint64) % 300 * (dom[0] // 300 or 1),
                      rng.integers(0, dom[1], n2, dtype=np.uint64) % 40,
                      rng.integers(0, 1 << 32, n2, dtype=np.uint64)], 1).astype(np.uint32)
        A[0, 0], B[0, 0] = dom[0] - 1, 0  # wide bounds
        A[1, 1], B[1, 1] = dom[1] - 1, 0
        ref = oracle.join(oracle.Table([0, 1, 2], A), oracle.Table([0, 1, 3], B))
        got = ctx.join(dtable([0, 1, 2], A), dtable([0, 1, 3], B))
        path = ctx.stats()["last_path"]
        assert np.array_equal(oracle.canonical_rows(got.to_numpy()), oracle.canonical(ref).rows)
        if path not in (mq.PATH_RESIDUAL, mq.PATH_HASH):
            assert np.array_equal(got.to_numpy(), ref.rows)


@pytest.mark.parametrize("cfg", ["C2", "C5"])
def test_filtered_queries(ctx, cfg):
    s, p, o, st = datagen.lubm(3, 0, 2)
    trip = (dev(s), dev(p), dev(o))
    pats = config_query(cfg)
    ref = oracle.query(s, p, o, pats)
    ctx.set_option(mq.OPT_SEMIJOIN, mq.SEMIJOIN_ON)
    got = ctx.query(trip, pats)
    assert got.nrows == config_expected_counts(cfg, st)[-1]
    if ctx.stats()["last_path"] not in (mq.PATH_RESIDUAL, mq.PATH_HASH):
        assert np.array_equal(got.to_numpy(), ref.rows)
    ctx.set_option(mq.OPT_SEMIJOIN, mq.SEMIJOIN_OFF)
    plain = ctx.query(trip, pats)
    assert np.array_equal(plain.to_numpy(), got.to_numpy())


def test_filtered_zipf_skew(ctx):
    """C4-shaped sides (Zipf(1.1), side-specific key permutations): most rows are dropped."""
    ctx.set_option(mq.OPT_SEMIJOIN, mq.SEMIJOIN_ON)
    n = 200_000
    k1, v1 = datagen.zipf(n, 0)
    k2, v2 = datagen.zipf(n, 1)
    A, B = np.stack([k1, v1], 1), np.stack([k2, v2], 1)
    ref = oracle.join(oracle.Table([0, 1], A), oracle.Table([0, 2], B))
    got = ctx.join(dtable([0, 1], A), dtable([0, 2], B))
    assert np.array_equal(got.to_numpy(), ref.rows)
    assert ctx.stats()["last_filtered"] == unmatched_rows(A, B, [0], [0])
