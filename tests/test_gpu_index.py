"""GPU parity of the predicate-range index against the CPU oracle.

The index is the triple table stably partitioned by predicate, so every constant-predicate
pattern's partial matches come out of it in the same row order as the full scan: the oracle's
scan (triple order) is compared IN ORDER; variable-predicate patterns (index order) are compared
canonically."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import datagen  # noqa: E402
import oracle  # noqa: E402
import paper_1702_03484_b200 as mq  # noqa: E402
from fixtures import config_expected_counts, config_query, load_table1  # noqa: E402

V, C = "v", "c"


@pytest.fixture(scope="module")
def ctx():
    return mq.Context(0)


def dev(a):
    a = np.ascontiguousarray(a, dtype=np.uint32)
    return torch.from_numpy(a.view(np.int32)).cuda()


def host(t):
    return t.view(torch.int32).cpu().numpy().view(np.uint32)


def assert_same(gpu, ref, ordered=True, exact_bounds=True):
    """exact_bounds: scan outputs carry exact column bounds; join outputs carry valid (inherited,
    possibly wider) bounds."""
    assert gpu.vars == ref.vars
    got = gpu.to_numpy()
    assert got.shape == ref.rows.shape
    if ordered:
        assert np.array_equal(got, ref.rows)
    else:
        assert np.array_equal(oracle.canonical_rows(got), oracle.canonical(ref).rows)
    if ref.nrows:
        tight = [(int(ref.rows[:, c].min()), int(ref.rows[:, c].max()))
                 for c in range(len(ref.vars))]
        if exact_bounds:
            assert gpu.bounds == tight
        else:
            assert all(lo <= a and b <= hi for (lo, hi), (a, b) in zip(gpu.bounds, tight))


@pytest.mark.parametrize("n,pdom", [(1, 3), (5, 1), (8191, 6), (8193, 6), (70_000, 40),
                                    (200_000, 300)])
def test_index_is_stable_partition_by_predicate(ctx, n, pdom):
    rng = np.random.default_rng(n + pdom)
    T = rng.integers(0, 1 << 32, (n, 3), dtype=np.uint64).astype(np.uint32)
    T[:, 1] = (rng.integers(0, pdom, n) * 7919 + 12345).astype(np.uint32)  # sparse predicate IDs
    idx = ctx.index_build(tuple(dev(T[:, j]) for j in range(3)))
    perm = np.argsort(T[:, 1], kind="stable")
    s2, p2, o2 = (host(x) for x in idx.triples())
    assert np.array_equal(s2, T[perm, 0])
    assert np.array_equal(p2, T[perm, 1])
    assert np.array_equal(o2, T[perm, 2])
    preds, counts = np.unique(T[:, 1], return_counts=True)
    assert idx.npreds == len(preds)
    starts = np.concatenate([[0], np.cumsum(counts)])
    for i, p in enumerate(preds):
        assert idx.range(int(p)) == (int(starts[i]), int(starts[i + 1]))
    assert idx.range(int(preds.max()) + 1) == (0, 0)


def test_indexed_scan_matches_oracle(ctx):
    rng = np.random.default_rng(11)
    for n in [1, 33, 8193, 60_000]:
        T = rng.integers(0, 6, (n, 3)).astype(np.uint32)
        idx = ctx.index_build(tuple(dev(T[:, j]) for j in range(3)))
        pats = [((V, 0), (C, 3), (V, 1)),   # view
                ((V, 1), (C, 2), (V, 0)),   # view, variables out of id order
                ((V, 0), (C, 3), (C, 5)),   # range scan: constant object
                ((C, 2), (C, 4), (V, 1)),   # range scan: constant subject
                ((V, 0), (C, 1), (V, 0)),   # range scan: repeated variable
                ((V, 0), (C, 99), (V, 1)),  # absent predicate: empty
                ((V, 0), (V, 1), (V, 2)),   # variable predicate: whole index
                ((V, 2), (V, 2), (V, 2)),
                ((C, 2), (V, 4), (V, 1))]
        got = ctx.scan_patterns(idx, pats)
        for g, p in zip(got, pats):
            ref = oracle.scan(*T.T, p)
            assert_same(g, ref, ordered=p[1][0] == C)


def test_indexed_views_are_zero_copy(ctx):
    s, p, o, _ = datagen.lubm(1)
    idx = ctx.index_build((dev(s), dev(p), dev(o)))
    tp, = ctx.scan_patterns(idx, [config_query("C1")[0]])
    b, e = idx.range(datagen.LUBM_PRED["worksFor"])
    s2, _, o2 = idx.triples()
    assert tp.nrows == e - b
    assert tp.columns[0].data_ptr() == s2.data_ptr() + 4 * b
    assert tp.columns[1].data_ptr() == o2.data_ptr() + 4 * b
    before = ctx.stats()["launches"]
    ctx.scan_patterns(idx, [config_query("C1")[0]])
    assert ctx.stats()["launches"] == before  # no kernel for a view


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C5"])
def test_indexed_query_configs(ctx, cfg):
    s, p, o, st = datagen.lubm(3, 0, 2)
    idx = ctx.index_build((dev(s), dev(p), dev(o)))
    pats = config_query(cfg)
    ref = oracle.query(s, p, o, pats)
    got = ctx.query(idx, pats)
    assert got.nrows == config_expected_counts(cfg, st)[-1]
    assert_same(got, ref, ordered=ctx.stats()["last_path"] not in (mq.PATH_RESIDUAL, mq.PATH_HASH),
                exact_bounds=False)
    plain = ctx.query((dev(s), dev(p), dev(o)), pats)
    assert np.array_equal(plain.to_numpy(), got.to_numpy())  # same rows, same order


def test_indexed_table1_and_projection(ctx):
    ids, T, sec = load_table1()
    idx = ctx.index_build(tuple(dev(T[:, j]) for j in range(3)))
    P1 = ((V, 0), (C, ids["hasJob"]), (V, 1))
    P2 = ((V, 1), (C, ids["workAt"]), (C, ids['"Hospital"']))
    q = ctx.query(idx, [P1, P2], [0])
    assert sorted(q.to_numpy()[:, 0].tolist()) == sorted(ids[r[0]] for r in sec["select_person"])
    one = ctx.query(idx, [P1])  # single-pattern query: a view of the index
    assert_same(one, oracle.scan(*T.T, P1))


@pytest.mark.parametrize("cfg", ["C1", "C5"])
def test_prepared_query_equals_query(ctx, cfg):
    """Context.prepare marshals a query's C arguments once; every call is the same library call
    (index store and plain triple table, with and without a projection)."""
    s, p, o, _ = datagen.lubm(2)
    trip = (dev(s), dev(p), dev(o))
    idx = ctx.index_build(trip)
    pats = config_query(cfg)
    for src in (idx, trip):
        for proj in (None, [0]):
            want = ctx.query(src, pats, proj).to_numpy()
            q = ctx.prepare(src, pats, proj)
            for _ in range(3):
                r = q()
                assert np.array_equal(r.to_numpy(), want)
                r.release()


def test_index_empty_table(ctx):
    z = torch.empty(0, dtype=torch.int32, device="cuda")
    idx = ctx.index_build((z, z, z))
    assert idx.n == 0 and idx.npreds == 0
    got = ctx.scan_patterns(idx, [((V, 0), (C, 1), (V, 1)), ((V, 0), (V, 1), (V, 2))])
    assert [g.nrows for g in got] == [0, 0]
    assert got[1].vars == [0, 1, 2]


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C5"])
def test_query_host_indexed_matches_device_index_and_oracle(ctx, cfg):
    """mapsq_query_host_indexed (pinned host mirror of the index; only the touched predicate
    ranges go host -> device) returns exactly mapsq_query_indexed's rows, which match the oracle,
    and copies exactly the bytes its contract states."""
    s, p, o, _ = datagen.lubm(2)
    idx = ctx.index_build((dev(s), dev(p), dev(o)))
    pats = config_query(cfg)
    want = ctx.query(idx, pats).to_numpy()
    ref = oracle.query(s, p, o, pats)
    # bytes of the plain mirror: 8 per row of every touched predicate (s, o), +4 where a pattern
    # scans the range; the compressed mirror (default) copies fewer and expands them losslessly
    need = {}
    for pat in pats:
        (ks, _), (kp, pid), (ko, _) = pat
        if kp == C:
            view = ks == V and ko == V and pat[0][1] != pat[2][1]
            need[pid] = max(need.get(pid, 0), 8 if view else 12)
    expect = sum(b * (idx.range(pid)[1] - idx.range(pid)[0]) for pid, b in need.items())
    for compress in (0, 1):
        ctx.set_option(mq.OPT_HOST_COMPRESS, compress)
        hidx = ctx.index_to_host(idx)
        vars_, rows = ctx.query_host(hidx, pats, copy=True)
        assert np.array_equal(rows, want), compress
        assert vars_ == ref.vars
        assert np.array_equal(oracle.canonical_rows(rows), oracle.canonical(ref).rows)
        if compress:
            assert 0 < hidx.last_h2d_bytes < expect
        else:
            assert hidx.last_h2d_bytes == expect
        hidx.release()
    ctx.set_option(mq.OPT_HOST_COMPRESS, 1)


def test_query_host_indexed_late_large_range(ctx):
    """C5's last pattern (takesCourse) owns the largest predicate range: its H2D copy is still
    streaming while the first join runs, and the second join must wait for exactly that range
    (the join waits on the ranges its input columns live in)."""
    s, p, o, _ = datagen.lubm(40)
    idx = ctx.index_build((dev(s), dev(p), dev(o)))
    hidx = ctx.index_to_host(idx)
    for cfg in ("C5", "C3"):
        pats = config_query(cfg)
        want = ctx.query(idx, pats).to_numpy()
        for _ in range(3):
            vars_, rows = ctx.query_host(hidx, pats, copy=True)
            assert np.array_equal(rows, want), cfg
    hidx.release()


@pytest.mark.parametrize("compress", [1, 0])
def test_query_host_indexed_streamed_chunks(ctx, monkeypatch, compress):
    """The predicate ranges stream in chunk by chunk and a join whose Tp2 is one range starts on
    the chunks that have landed (the filter's probe of the larger side waits per chunk).  With
    MAPSQ_DEBUG_COPY_DELAY every chunk's rows hold a poison value while the copy stream sleeps
    before copying it, so any read that does not wait for its chunk changes the result."""
    monkeypatch.setenv("MAPSQ_STREAM_CHUNK", "65536")
    monkeypatch.setenv("MAPSQ_DEBUG_COPY_DELAY", "300")
    s, p, o, _ = datagen.lubm(60)
    idx = ctx.index_build((dev(s), dev(p), dev(o)))
    ctx.set_option(mq.OPT_HOST_COMPRESS, compress)
    hidx = ctx.index_to_host(idx)
    for mode in (mq.SEMIJOIN_ON, mq.SEMIJOIN_AUTO, mq.SEMIJOIN_OFF):
        ctx.set_option(mq.OPT_SEMIJOIN, mode)
        for cfg in ("C5", "C3", "C2", "C1"):
            pats = config_query(cfg)
            want = ctx.query(idx, pats).to_numpy()
            vars_, rows = ctx.query_host(hidx, pats, copy=True)
            assert np.array_equal(rows, want), (cfg, mode)
    ctx.set_option(mq.OPT_SEMIJOIN, mq.SEMIJOIN_AUTO)
    ctx.set_option(mq.OPT_HOST_COMPRESS, 1)
    hidx.release()


def test_compressed_host_mirror_codec_edges(ctx):
    """The compressed mirror is lossless at every block width: full 32-bit ranges (bits = 32), a
    constant column (bits = 0), ranges of 1 and 1025 rows, a block boundary inside a range."""
    rng = np.random.default_rng(17)
    parts = [
        np.stack([rng.integers(0, 1 << 32, 5000, dtype=np.uint64), np.full(5000, 0),
                  rng.integers(0, 1 << 32, 5000, dtype=np.uint64)], 1),            # 32-bit
        np.stack([np.full(1025, 7), np.full(1025, 1), np.arange(1025) * 3 + 1], 1),  # bits 0 / 12
        np.array([[5, 2, 9]]),                                                       # one row
        np.stack([np.arange(3000) // 3, np.full(3000, 3), rng.integers(0, 77, 3000)], 1),
    ]
    T = np.unique(np.concatenate(parts).astype(np.uint32), axis=0)
    s, p, o = (np.ascontiguousarray(T[:, j]) for j in range(3))
    idx = ctx.index_build((dev(s), dev(p), dev(o)))
    ctx.set_option(mq.OPT_HOST_COMPRESS, 1)
    hidx = ctx.index_to_host(idx)
    for pid in range(4):
        pats = [((V, 0), (C, pid), (V, 1))]
        want = ctx.query(idx, pats).to_numpy()
        _, rows = ctx.query_host(hidx, pats, copy=True)
        assert np.array_equal(rows, want), pid
    _, rows = ctx.query_host(hidx, [((V, 0), (V, 1), (V, 2))], copy=True)   # every range, p too
    assert np.array_equal(oracle.canonical_rows(rows), oracle.canonical_rows(T))
    hidx.release()


def test_query_host_indexed_edge_cases(ctx):
    rng = np.random.default_rng(3)
    n = 50_000
    T = np.stack([rng.integers(0, 500, n), rng.integers(0, 7, n), rng.integers(0, 500, n)], 1)
    T = np.unique(T.astype(np.uint32), axis=0)
    s, p, o = (np.ascontiguousarray(T[:, j]) for j in range(3))
    idx = ctx.index_build((dev(s), dev(p), dev(o)))
    ctx.set_option(mq.OPT_HOST_COMPRESS, 0)  # (the byte count below is the plain mirror's)
    hidx = ctx.index_to_host(idx)
    ctx.set_option(mq.OPT_HOST_COMPRESS, 1)
    hidx_c = ctx.index_to_host(idx)
    cases = [
        [((V, 0), (C, 3), (V, 1))],                                  # one view: result is a view
        [((V, 0), (V, 1), (V, 2))],                                  # variable predicate: all rows
        [((V, 0), (C, 99), (V, 1)), ((V, 1), (C, 2), (V, 2))],      # absent predicate: empty
        [((V, 0), (C, 1), (V, 0))],                                  # repeated variable: a scan
        [((V, 0), (C, 2), (C, 17)), ((V, 0), (C, 5), (V, 1)), ((V, 1), (C, 5), (V, 2))],
    ]
    for pats in cases:
        ref = oracle.query(s, p, o, pats)
        for hx in (hidx, hidx_c):
            vars_, rows = ctx.query_host(hx, pats, copy=True)
            assert vars_ == ref.vars
            assert np.array_equal(oracle.canonical_rows(rows), oracle.canonical(ref).rows), pats
    ctx.query_host(hidx, [((V, 0), (V, 1), (V, 2))])
    assert hidx.last_h2d_bytes == 12 * len(s)
    hidx.release()
    hidx_c.release()
