"""GPU parity: the CUDA path through the C ABI against the CPU oracle, element by element.

Integer path, so the bar is bit-exact.  Because the GPU join emits rows in (key', tp1 row,
tp2 row) order and the oracle's sort-merge tier emits (key tuple, A row, B row), single-GPU
results are compared IN ORDER (stronger than the canonical-sort comparison), and canonically
where only the multiset is defined."""
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


def dtable(vars_, rows):
    rows = np.asarray(rows, np.uint32).reshape(-1, len(vars_))
    return mq.DeviceTable.from_torch(vars_, [dev(rows[:, c]) for c in range(len(vars_))])


def assert_same(gpu: mq.DeviceTable, ref: oracle.Table, ordered=True):
    assert gpu.vars == ref.vars
    got = gpu.to_numpy()
    assert got.shape == ref.rows.shape
    if ordered:
        assert np.array_equal(got, ref.rows)
    else:
        assert np.array_equal(oracle.canonical_rows(got), oracle.canonical(ref).rows)


# ------------------------------------------------------------------------- Table 1
def test_table1_scan_join_query(ctx):
    ids, T, sec = load_table1()
    trip = tuple(dev(T[:, j]) for j in range(3))
    P1 = ((V, 0), (C, ids["hasJob"]), (V, 1))
    P2 = ((V, 1), (C, ids["workAt"]), (C, ids['"Hospital"']))
    tp1, tp2 = ctx.scan_patterns(trip, [P1, P2])
    assert_same(tp1, oracle.scan(*T.T, P1))
    assert_same(tp2, oracle.scan(*T.T, P2))
    rs = ctx.join(tp1, tp2)
    assert_same(rs, oracle.join(oracle.scan(*T.T, P1), oracle.scan(*T.T, P2)))
    assert sorted(rs.to_numpy().tolist()) == sorted(
        [[ids[k], ids[v]] for k, v, _ in sec["rs"]])
    q = ctx.query(trip, [P1, P2], [0])
    assert sorted(q.to_numpy()[:, 0].tolist()) == sorted(ids[r[0]] for r in sec["select_person"])
    vars_, rows = ctx.query_host(*[np.ascontiguousarray(T[:, j]) for j in range(3)], [P1, P2], [0])
    assert vars_ == [0] and sorted(rows[:, 0].tolist()) == sorted(q.to_numpy()[:, 0].tolist())


# ------------------------------------------------------------------------- random joins
@pytest.mark.parametrize("domain", [1, 5, 50, 1000, 1 << 20, 1 << 32])
def test_join_random_single_key(ctx, domain):
    rng = np.random.default_rng(domain % 1000003)
    sizes = [(0, 5), (5, 0), (1, 1), (7, 3), (300, 200), (4095, 4097), (5000, 9000)]
    for n1, n2 in sizes:
        A = np.stack([rng.integers(0, domain, n1, dtype=np.uint64),
                      rng.integers(0, 1 << 32, n1, dtype=np.uint64)], 1).astype(np.uint32)
        B = np.stack([rng.integers(0, 1 << 32, n2, dtype=np.uint64),
                      rng.integers(0, domain, n2, dtype=np.uint64)], 1).astype(np.uint32)
        ka, ca = np.unique(A[:, 0], return_counts=True)
        kb, cb = np.unique(B[:, 1], return_counts=True)
        _, ia, ib_ = np.intersect1d(ka, kb, return_indices=True)
        if int((ca[ia].astype(np.int64) * cb[ib_]).sum()) > 3_000_000:
            continue
        ref = oracle.join(oracle.Table([3, 1], A), oracle.Table([2, 3], B))
        got = ctx.join(dtable([3, 1], A), dtable([2, 3], B))
        assert_same(got, ref)


def test_join_many_random_cases(ctx):
    rng = np.random.default_rng(1234)
    for case in range(200):
        n1, n2 = (int(x) for x in rng.integers(0, 400, 2))
        dom = int(rng.choice([1, 3, 17, 400]))
        w1, w2 = int(rng.integers(1, 4)), int(rng.integers(1, 4))
        A = rng.integers(0, dom, (n1, w1)).astype(np.uint32)
        B = rng.integers(0, dom, (n2, w2)).astype(np.uint32)
        # variable ids: column 0 of each side shares var 0; random extra sharing of var 1
        va = [0] + [10 + c for c in range(1, w1)]
        vb = [20 + c for c in range(1, w2)] + [0]
        if w1 > 1 and w2 > 1 and case % 3 == 0:
            va[1], vb[0] = 1, 1
        ta, tb = oracle.Table(va, A), oracle.Table(vb, B)
        ref = oracle.join(ta, tb)
        got = ctx.join(dtable(va, A), dtable(vb, B))
        assert_same(got, ref)


def test_join_composite_keys_and_kv_path(ctx):
    rng = np.random.default_rng(7)
    # two shared variables in different column orders (reading R5)
    A = rng.integers(0, 6, (3000, 3)).astype(np.uint32)
    B = rng.integers(0, 6, (2000, 2)).astype(np.uint32)
    ref = oracle.join(oracle.Table([0, 2, 1], A), oracle.Table([2, 0], B))
    assert_same(ctx.join(dtable([0, 2, 1], A), dtable([2, 0], B)), ref)
    # full-range 32-bit composite keys: kb = 64 > 64 - ib -> KV path
    base = rng.integers(0, 1 << 32, (500, 2), dtype=np.uint64).astype(np.uint32)
    A = np.concatenate([base[rng.integers(0, 500, 4000)], rng.integers(0, 9, (4000, 1)).astype(np.uint32)], 1)
    B = np.concatenate([base[rng.integers(0, 500, 3000)][:, ::-1], rng.integers(0, 9, (3000, 1)).astype(np.uint32)], 1)
    B[:2, :2] = [[0, 0], [0xFFFFFFFF, 0xFFFFFFFF]]
    ta, tb = oracle.Table([4, 5, 6], A), oracle.Table([5, 4, 7], np.ascontiguousarray(B))
    ref = oracle.join(ta, tb)
    # default: HASH path (32-bit hash of (x, z), every pair verified); rows grouped by hash
    got = ctx.join(dtable([4, 5, 6], A), dtable([5, 4, 7], np.ascontiguousarray(B)))
    assert ctx.stats()["last_path"] == mq.PATH_HASH
    assert_same(got, ref, ordered=False)
    # RESIDUAL path (x packed, z verified per group); rows ordered by (x', l, r)
    # KV path: (u64 key', u32 rowid) pairs over all 64 key bits, lexicographic order
    for mode, path, ordered in ((mq.WIDE_KEY_RESIDUAL, mq.PATH_RESIDUAL, False),
                                (mq.WIDE_KEY_KV, mq.PATH_KV, True)):
        ctx.set_option(mq.OPT_WIDE_KEY, mode)
        try:
            got = ctx.join(dtable([4, 5, 6], A), dtable([5, 4, 7], np.ascontiguousarray(B)))
            assert ctx.stats()["last_path"] == path
            assert_same(got, ref, ordered=ordered)
        finally:
            ctx.set_option(mq.OPT_WIDE_KEY, mq.WIDE_KEY_HASH)
    # three shared variables
    A = rng.integers(0, 3, (2000, 4)).astype(np.uint32)
    B = rng.integers(0, 3, (1500, 3)).astype(np.uint32)
    ref = oracle.join(oracle.Table([0, 1, 2, 9], A), oracle.Table([2, 1, 0], B))
    assert_same(ctx.join(dtable([0, 1, 2, 9], A), dtable([2, 1, 0], B)), ref)


@pytest.mark.parametrize("mode,path", [("RESIDUAL", "RESIDUAL"), ("HASH", "HASH")])
def test_join_residual_path_collisions_and_skew(ctx, mode, path):
    # RESIDUAL: packed column x with few values and a residual column z: many packed-key groups
    # mix several z values, so the per-group exact residual check decides every pair.
    # HASH: key' = 32-bit hash of (x, z); every pair's columns are verified
    ctx.set_option(mq.OPT_WIDE_KEY, getattr(mq, "WIDE_KEY_" + mode))
    rng = np.random.default_rng(13)
    for n1, n2, dx, dz in [(3000, 2000, 50, 7), (500, 40000, 3, 1 << 32), (20000, 20000, 5000, 3)]:
        x1 = rng.integers(0, dx, n1); z1 = rng.integers(0, dz, n1, dtype=np.uint64)
        x2 = rng.integers(0, dx, n2); z2 = rng.integers(0, dz, n2, dtype=np.uint64)
        # force both key columns to span 32 bits so the plan cannot pack both
        x1[0] = 0xFFFFFFFF; z1[0] = 0xFFFFFFFF; x2[0] = 0; z2[0] = 0
        A = np.stack([x1, z1, rng.integers(0, 100, n1)], 1).astype(np.uint32)
        B = np.stack([z2, rng.integers(0, 100, n2), x2], 1).astype(np.uint32)
        ref = oracle.join(oracle.Table([0, 1, 2], A), oracle.Table([1, 3, 0], B))
        got = ctx.join(dtable([0, 1, 2], A), dtable([1, 3, 0], B))
        assert ctx.stats()["last_path"] == getattr(mq, "PATH_" + path)
        assert_same(got, ref, ordered=False)
    ctx.set_option(mq.OPT_WIDE_KEY, mq.WIDE_KEY_HASH)


@pytest.mark.parametrize("mode", ["RESIDUAL", "HASH"])
def test_join_hot_composite_key(ctx, mode):
    # One hot composite key: x = 7 on 1500 LEFT and 1400 RIGHT rows with z in {5, 6}.  RESIDUAL
    # packs x and checks z: the hot x-group holds 2.1e6 candidate pairs, about half of them true
    # (more candidates than 2 (n1 + n2) + 2^20, so the matches are counted before the output is
    # sized); HASH groups by a hash of (x, z): two hot groups of ~5e5 true pairs.  Both spread a
    # group's pairs over many CTAs (candidate-parallel verification).
    ctx.set_option(mq.OPT_WIDE_KEY, getattr(mq, "WIDE_KEY_" + mode))
    rng = np.random.default_rng(29)
    nh1, nh2, nc = 1500, 1400, 3000
    x1 = np.concatenate([np.full(nh1, 7), rng.integers(0, 1 << 32, nc, dtype=np.uint64)])
    z1 = np.concatenate([rng.integers(5, 7, nh1), rng.integers(0, 1 << 32, nc, dtype=np.uint64)])
    x2 = np.concatenate([np.full(nh2, 7), rng.integers(0, 1 << 32, nc, dtype=np.uint64)])
    z2 = np.concatenate([rng.integers(5, 7, nh2), rng.integers(0, 1 << 32, nc, dtype=np.uint64)])
    x1[-1] = z1[-1] = 0xFFFFFFFF  # both key columns span 32 bits: the plan cannot pack both
    x2[-1] = z2[-1] = 0
    p1, p2 = rng.permutation(len(x1)), rng.permutation(len(x2))
    A = np.stack([x1, z1, np.arange(len(x1))], 1).astype(np.uint32)[p1]
    B = np.stack([z2, np.arange(len(x2)) + 10 ** 6, x2], 1).astype(np.uint32)[p2]
    ref = oracle.join(oracle.Table([0, 1, 2], A), oracle.Table([1, 3, 0], B))
    got = ctx.join(dtable([0, 1, 2], A), dtable([1, 3, 0], B))
    assert ctx.stats()["last_path"] == getattr(mq, "PATH_" + mode)
    hot = [(int((A[:, 1][A[:, 0] == 7] == z).sum()), int((B[:, 0][B[:, 2] == 7] == z).sum()))
           for z in (5, 6)]
    assert got.nrows == ref.nrows >= sum(a * b for a, b in hot) > 900_000
    assert_same(got, ref, ordered=False)
    ctx.set_option(mq.OPT_WIDE_KEY, mq.WIDE_KEY_HASH)


def test_small_join_one_launch_equals_multikernel_path(ctx):
    # joins of <= 4096 rows run Algorithm 1 in one CTA (small.cu): same rows, same order as the
    # multi-kernel path and the oracle; |RS| above the 2^16-row allocation falls back
    rng = np.random.default_rng(77)
    cases = [(1, 1, 3), (17, 5, 4), (700, 320, 300), (2048, 2048, 50), (4000, 96, 7), (300, 300, 1),
             (2500, 1596, 2000)]
    for n1, n2, dom in cases:
        A = np.stack([rng.integers(0, dom, n1), rng.integers(0, 1 << 32, n1, dtype=np.uint64)], 1).astype(np.uint32)
        B = np.stack([rng.integers(0, 1 << 32, n2, dtype=np.uint64), rng.integers(0, dom, n2)], 1).astype(np.uint32)
        ref = oracle.join(oracle.Table([0, 1], A), oracle.Table([2, 0], B))
        outs = []
        bA = [(int(A[:, c].min()), int(A[:, c].max())) for c in range(2)]
        bB = [(int(B[:, c].min()), int(B[:, c].max())) for c in range(2)]
        for small in (1, 0):
            ctx.set_option(mq.OPT_SMALL_JOIN, small)
            ctx.stats_reset()
            ta = mq.DeviceTable.from_torch([0, 1], [dev(A[:, c]) for c in range(2)], bA)
            tb = mq.DeviceTable.from_torch([2, 0], [dev(B[:, c]) for c in range(2)], bB)
            got = ctx.join(ta, tb)
            assert_same(got, ref)  # in order
            outs.append(got.to_numpy())
            launches = ctx.stats()["launches"]
            if small and n1 + n2 <= 4096 and ref.nrows <= (1 << 16):
                assert launches <= 1, (n1, n2, launches)  # (0: disjoint key ranges)
        assert np.array_equal(outs[0], outs[1])
    ctx.set_option(mq.OPT_SMALL_JOIN, 1)


@pytest.mark.parametrize("pv", ["1", "0"])
def test_value_carrying_words(ctx, monkeypatch, pv):
    # Filtered P64 joins with at most one non-key column per side sort words that carry (label,
    # value) instead of the row id (kPvIb; MAPSQ_PV=0: row-id words).  Same rows, same order:
    # 0 or 1 non-key columns on each side, full 32-bit values, a hot key, semi-join filter on / off
    # (its column round writes the value words in the gather), ragged sizes over many tiles.
    monkeypatch.setenv("MAPSQ_PV", pv)
    rng = np.random.default_rng(606)
    shapes = [([0, 1], [0, 2]), ([0], [0, 2]), ([0, 1], [0]), ([0], [0]), ([1, 0], [2, 0])]
    for n1, n2, dom in [(5000, 7000, 3000), (70001, 40003, 1 << 20), (30000, 9000, 60)]:
        for va, vb in shapes:
            A = rng.integers(0, 1 << 32, (n1, len(va)), dtype=np.uint64).astype(np.uint32)
            B = rng.integers(0, 1 << 32, (n2, len(vb)), dtype=np.uint64).astype(np.uint32)
            A[:, va.index(0)] = rng.integers(0, dom, n1)
            B[:, vb.index(0)] = rng.integers(0, dom, n2)
            A[: n1 // 10, va.index(0)] = 3  # hot key
            ref = oracle.join(oracle.Table(va, A), oracle.Table(vb, B))
            for mode in (mq.SEMIJOIN_ON, mq.SEMIJOIN_OFF):
                ctx.set_option(mq.OPT_SEMIJOIN, mode)
                ctx.set_option(mq.OPT_SMALL_JOIN, 0)
                got = ctx.join(dtable(va, A), dtable(vb, B))
                assert_same(got, ref)  # in order
                # (value words come from the filter's column round)
                assert ctx.stats()["last_ib"] == (33 if pv == "1" and mode == mq.SEMIJOIN_ON
                                                  else int(np.ceil(np.log2(n1 + n2))))
    ctx.set_option(mq.OPT_SEMIJOIN, mq.SEMIJOIN_AUTO)
    ctx.set_option(mq.OPT_SMALL_JOIN, 1)


def test_join_skewed_hot_key_large_groups(ctx):
    rng = np.random.default_rng(11)
    # one hot key: 6000 x 700 = 4.2e6 output rows, plus a cold tail
    A = np.stack([np.where(rng.random(20000) < 0.3, 77, rng.integers(0, 5000, 20000)),
                  rng.integers(0, 1 << 30, 20000)], 1).astype(np.uint32)
    B = np.stack([np.where(rng.random(15000) < 0.05, 77, rng.integers(0, 5000, 15000)),
                  rng.integers(0, 1 << 30, 15000)], 1).astype(np.uint32)
    ref = oracle.join(oracle.Table([0, 1], A), oracle.Table([0, 2], B))
    got = ctx.join(dtable([0, 1], A), dtable([0, 2], B))
    assert_same(got, ref)
    L = np.bincount(A[:, 0], minlength=5001)
    R = np.bincount(B[:, 0], minlength=5001)
    assert got.nrows == int((L.astype(np.int64) * R).sum())


def test_join_empty_and_disjoint(ctx):
    A = np.array([[1, 2], [3, 4]], np.uint32)
    B = np.array([[10, 5]], np.uint32)
    got = ctx.join(dtable([0, 1], A), dtable([0, 2], B))
    assert got.nrows == 0 and got.vars == [0, 1, 2]
    got = ctx.join(dtable([0, 1], np.zeros((0, 2), np.uint32)), dtable([0, 2], B))
    assert got.nrows == 0 and got.vars == [0, 1, 2]
    with pytest.raises(mq.MapsqError) as e:
        ctx.join(dtable([0], A[:, :1]), dtable([5], B[:, :1]))
    assert e.value.status == "E_NO_SHARED"


# ------------------------------------------------------------------------- phases
def test_sort_words_equals_library_sort(ctx):
    rng = np.random.default_rng(3)
    for n in [1, 2, 100, 4095, 4096, 4097, 100_000, 1_000_003]:
        # low bits ascending in input order (as the Map step builds them), random high bits
        w = np.arange(n, dtype=np.uint64) | (rng.integers(0, 1 << 40, n, dtype=np.uint64) << np.uint64(22))
        t = torch.from_numpy(w.view(np.int64)).cuda()
        ctx.sort_words(t, 22, 62)
        got = t.cpu().numpy().view(np.uint64)
        assert np.array_equal(got, np.sort(w)), n   # words are unique -> the sorted array is unique


def test_sort_pairs_stable(ctx):
    rng = np.random.default_rng(4)
    n = 300_001
    k = rng.integers(0, 1 << 44, n, dtype=np.uint64)
    k[rng.random(n) < 0.5] = 12345  # many equal keys: stability decides their order
    v = np.arange(n, dtype=np.uint32)
    tk, tv = torch.from_numpy(k.view(np.int64)).cuda(), torch.from_numpy(v.view(np.int32)).cuda()
    ctx.sort_pairs(tk, tv, 0, 44)
    order = np.argsort(k, kind="stable")
    assert np.array_equal(tk.cpu().numpy().view(np.uint64), k[order])
    assert np.array_equal(tv.cpu().numpy().view(np.uint32), v[order])


def test_map_words_layout(ctx):
    rng = np.random.default_rng(5)
    A = rng.integers(100, 200, (1000, 2)).astype(np.uint32)
    B = rng.integers(150, 260, (700, 1)).astype(np.uint32)
    ta, tb = dtable([0, 1], A), dtable([0], B)
    ctx.table_bounds(ta)
    ctx.table_bounds(tb)
    pl = mq.plan_join([0, 1], ta.bounds, 1000, [0], tb.bounds, 700)
    words = torch.empty(1700, dtype=torch.int64, device="cuda")
    ctx.map_words(ta, tb, pl, words)
    got = words.cpu().numpy().view(np.uint64)
    lo = min(A[:, 0].min(), B[:, 0].min())
    keys = np.concatenate([A[:, 0], B[:, 0]]).astype(np.uint64) - np.uint64(lo)
    want = (keys << np.uint64(pl.ib)) | np.arange(1700, dtype=np.uint64)  # LEFT rows 0..n1-1
    assert np.array_equal(got, want)
    assert pl.ib == 11 and (got[1000:] & np.uint64(2047) >= 1000).all()  # RIGHT label


def test_reduce_groups_counts(ctx):
    rng = np.random.default_rng(6)
    n1, n2, ib = 30000, 20000, 16
    kl, kr = rng.integers(0, 3000, n1), rng.integers(1000, 6000, n2)
    keys = np.concatenate([kl, kr]).astype(np.uint64)
    words = np.sort((keys << np.uint64(ib)) | np.arange(n1 + n2, dtype=np.uint64))
    t = torch.from_numpy(words.view(np.int64)).cuda()
    gs, gp, ge, go, total = ctx.reduce_groups(t, n1, n2, ib)
    uk, Lc = np.unique(kl, return_counts=True)
    Rc = np.bincount(kr, minlength=6000)[uk]
    both = Rc > 0
    assert total == int((Lc[both] * Rc[both]).sum())
    assert len(gs) == int(both.sum())
    cnt = (gp.cpu().numpy() - gs.cpu().numpy()).astype(np.int64) * (ge.cpu().numpy() - gp.cpu().numpy())
    assert np.array_equal(cnt, (Lc[both] * Rc[both]))
    assert np.array_equal(go.cpu().numpy(), np.concatenate([[0], np.cumsum(cnt)[:-1]]))
    wk = words >> np.uint64(ib)
    assert np.array_equal(wk[gs.cpu().numpy().astype(np.int64)], uk[both])


# ------------------------------------------------------------------------- scan + query
def test_scan_random_patterns(ctx):
    rng = np.random.default_rng(8)
    for n in [1, 31, 33, 8191, 8193, 50_000]:
        T = rng.integers(0, 6, (n, 3)).astype(np.uint32)
        trip = tuple(dev(T[:, j]) for j in range(3))
        pats = [((V, 0), (C, 3), (V, 1)), ((V, 0), (C, 3), (C, 5)), ((C, 2), (V, 4), (V, 1)),
                ((V, 0), (V, 1), (V, 2)), ((V, 0), (C, 1), (V, 0)), ((V, 2), (V, 2), (V, 2)),
                ((V, 0), (C, 99), (V, 1))]
        got = ctx.scan_patterns(trip, pats)
        for g, p in zip(got, pats):
            ref = oracle.scan(*T.T, p)
            assert_same(g, ref)
            if ref.nrows:
                assert g.bounds == [(int(ref.rows[:, c].min()), int(ref.rows[:, c].max()))
                                    for c in range(len(ref.vars))]


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C5"])
def test_query_configs_small_scale(ctx, cfg):
    s, p, o, st = datagen.lubm(3, 0, 2)
    trip = (dev(s), dev(p), dev(o))
    pats = config_query(cfg)
    ref = oracle.query(s, p, o, pats)
    got = ctx.query(trip, pats)
    assert got.nrows == config_expected_counts(cfg, st)[-1]
    # wide-key joins (RESIDUAL path) emit (packed key, l, r) order: compare canonically there
    assert_same(got, ref, ordered=ctx.stats()["last_path"] not in (mq.PATH_RESIDUAL, mq.PATH_HASH))
    # chained joins one by one agree with the generator's bookkeeping
    tabs = ctx.scan_patterns(trip, pats)
    acc = tabs[0]
    for i, t in enumerate(tabs[1:]):
        acc = ctx.join(acc, t)
        assert acc.nrows == config_expected_counts(cfg, st)[i]


def test_query_projection_and_errors(ctx):
    s, p, o, _ = datagen.lubm(1)
    trip = (dev(s), dev(p), dev(o))
    pats = config_query("C5")
    got = ctx.query(trip, pats, [2, 0])
    ref = oracle.query(s, p, o, pats, [2, 0])
    assert_same(got, ref, ordered=False)  # (?x, ?z) join key: HASH path
    with pytest.raises(mq.MapsqError) as e:
        ctx.query(trip, [((V, 0), (C, 5), (V, 1)), ((V, 2), (C, 5), (V, 3))])
    assert e.value.status == "E_NO_SHARED"


def test_partition_hash_and_stability(ctx):
    rng = np.random.default_rng(9)
    A = rng.integers(0, 1 << 20, (50_000, 3)).astype(np.uint32)
    for G in (1, 2, 3, 8, 37, 64):
        part, counts = ctx.partition(dtable([0, 1, 2], A), [0, 2], G)
        got = part.to_numpy()

        def fmix32(h):
            h = h ^ (h >> np.uint64(16)); h = (h * np.uint64(0x85EBCA6B)) & np.uint64(0xFFFFFFFF)
            h = h ^ (h >> np.uint64(13)); h = (h * np.uint64(0xC2B2AE35)) & np.uint64(0xFFFFFFFF)
            return h ^ (h >> np.uint64(16))
        h = np.full(len(A), 0x811C9DC5, np.uint64)
        for c in (0, 2):
            h = ((h ^ A[:, c].astype(np.uint64)) * np.uint64(0x01000193)) & np.uint64(0xFFFFFFFF)
        dest = (fmix32(h) * np.uint64(G)) >> np.uint64(32)
        assert counts == np.bincount(dest.astype(np.int64), minlength=G).tolist()
        want = A[np.argsort(dest, kind="stable")]
        assert np.array_equal(got, want)


def test_stats_and_launch_count(ctx):
    ctx.stats_reset()
    ctx.set_profiling(True)
    A = np.stack([np.arange(10000) % 97, np.arange(10000)], 1).astype(np.uint32)
    ctx.join(dtable([0, 1], A), dtable([0, 2], A))
    st = ctx.stats()
    ctx.set_profiling(False)
    assert st["launches"] >= 6 and st["joins"] == 1
    passes = [k for k in st["kernels"] if k.startswith("radix_pass")]
    assert passes and all(st["kernels"][k]["ms"] > 0 for k in passes)


def test_query_dist_world1_nccl(ctx, tmp_path):
    """The distributed path on one GPU: mapsq_query_dist[_indexed] / mapsq_join_dist (NCCL
    communicator, fused partition + exchange kernel into the IPC-exported arena, all-reduced
    bounds, local join) and the torch-orchestrated K8 partition + NCCL all-to-all (fused=False)."""
    import torch.distributed as tdist
    from paper_1702_03484_b200 import dist as mqd
    if not tdist.is_initialized():
        tdist.init_process_group("nccl", init_method=f"file://{tmp_path}/pg", rank=0, world_size=1,
                                 device_id=torch.device("cuda", 0))
    c2 = mq.Context(0)
    with pytest.raises(mq.MapsqError) as e:      # collective entry points need mapsq_dist_init
        c2.join_dist(dtable([0, 1], np.zeros((3, 2), np.uint32)), dtable([0, 2], np.zeros((3, 2), np.uint32)))
    assert e.value.code == 1
    s, p, o, st = datagen.lubm(2)
    trip = (dev(s), dev(p), dev(o))
    store = c2.index_build(trip)
    for fused in (True, False):
        for source in (trip, store):
            for cfg in ("C3", "C5", "C2", "C1"):
                pats = config_query(cfg)
                c2.stats_reset()
                got = mqd.query_dist(c2, source, pats, fused=fused)
                ref = oracle.query(s, p, o, pats)
                assert got.vars == ref.vars
                assert np.array_equal(oracle.canonical_rows(got.to_numpy()), oracle.canonical(ref).rows)
                if fused:
                    x = c2.stats()
                    # one exchange per side per join, minus tp1 when the key is unchanged (C3's
                    # star on ?x exchanges the accumulated result once); world 1 sends nothing
                    assert x["exchange_rows"] == 0 and x["exchange_bytes"] == 0
                    assert len(pats) <= x["exchanges"] <= 2 * (len(pats) - 1)
    # direct join_dist: caller-built inputs without bounds (min/max pass after the exchange),
    # ragged sizes, an empty side, a composite key
    rng = np.random.default_rng(5)
    A = rng.integers(0, 300, (12_345, 3)).astype(np.uint32)
    B = rng.integers(0, 300, (777, 2)).astype(np.uint32)
    for ta, tb in (([0, 1, 2], [2, 0]), ([0, 1, 2], [1, 3])):
        a = mq.DeviceTable.from_torch(ta, [torch.from_numpy(A[:, c].view(np.int32)).cuda() for c in range(3)])
        b = mq.DeviceTable.from_torch(tb, [torch.from_numpy(B[:, c].view(np.int32)).cuda() for c in range(2)])
        got = c2.join_dist(a, b)
        ref = oracle.join(oracle.Table(ta, A), oracle.Table(tb, B))
        assert got.vars == ref.vars
        assert np.array_equal(oracle.canonical_rows(got.to_numpy()), oracle.canonical(ref).rows)
    empty = dtable([0, 7], np.zeros((0, 2), np.uint32))
    assert c2.join_dist(a, empty).nrows == 0
    with pytest.raises(mq.MapsqError) as e:
        c2.join_dist(a, dtable([8, 9], B))
    assert e.value.code == 2
    with pytest.raises(mq.MapsqError) as e:
        c2.dist_init()                           # once per context
    assert e.value.code == 1
    hidx = c2.index_to_host(store)               # end to end over the host-resident store
    for cfg in ("C5", "C2"):
        pats = config_query(cfg)
        vars_, rows = c2.query_dist_host(hidx, pats, copy=True)
        ref = oracle.query(s, p, o, pats)
        assert vars_ == ref.vars
        assert np.array_equal(oracle.canonical_rows(rows), oracle.canonical(ref).rows)
        assert 0 < hidx.last_h2d_bytes < 12 * len(s)
    tdist.destroy_process_group()


def test_partition_scatter_into_external_columns(ctx):
    """mapsq_partition_scatter writes destination d's rows at dest_row[d] of arbitrary column
    pointers (the peer-store contract), stable within each destination."""
    rng = np.random.default_rng(21)
    A = rng.integers(0, 1 << 16, (30_000, 2)).astype(np.uint32)
    t = dtable([0, 1], A)
    G = 3
    state, counts = ctx.partition_plan(t, [0], G)
    ref, ref_counts = ctx.partition(t, [0], G)
    assert counts == ref_counts
    # three separate "arenas", each with a 7-row gap before this rank's block
    arenas = [torch.zeros((2, counts[d] + 7), dtype=torch.int32, device="cuda") for d in range(G)]
    cols = [arenas[d][c].data_ptr() for d in range(G) for c in range(2)]
    ctx.partition_scatter(state, [7] * G, cols)
    got = np.concatenate([arenas[d][:, 7:].cpu().numpy().view(np.uint32).T for d in range(G)])
    assert np.array_equal(got, ref.to_numpy())
    assert all(int(arenas[d][:, :7].abs().sum()) == 0 for d in range(G))


@pytest.mark.parametrize("G", [2, 3, 8])
def test_virtual_ranks_partition_invariance(ctx, G):
    """SURVEY T4's virtual-rank mode on one GPU: hash-partition both inputs into G parts (K8),
    join part g with part g for every g, and the union of the G local joins is the full join —
    the property the distributed join rests on (keys disjoint across parts)."""
    rng = np.random.default_rng(40 + G)
    A = np.stack([datagen_keys(rng, 20_011), rng.integers(0, 1 << 20, 20_011)], 1).astype(np.uint32)
    B = np.stack([rng.integers(0, 1 << 20, 9_001), datagen_keys(rng, 9_001)], 1).astype(np.uint32)
    ref = oracle.canonical(oracle.join(oracle.Table([0, 1], A), oracle.Table([2, 0], B))).rows
    pa, ca = ctx.partition(dtable([0, 1], A), [0], G)
    pb, cb = ctx.partition(dtable([2, 0], B), [0], G)
    parts, keysets, oa, ob = [], [], 0, 0
    for g in range(G):
        ta = mq.DeviceTable.from_torch([0, 1], [c[oa:oa + ca[g]] for c in pa.columns])
        tb = mq.DeviceTable.from_torch([2, 0], [c[ob:ob + cb[g]] for c in pb.columns])
        oa, ob = oa + ca[g], ob + cb[g]
        keysets.append(set(ta.to_numpy()[:, 0].tolist()) | set(tb.to_numpy()[:, 1].tolist()))
        if ca[g] and cb[g]:
            parts.append(ctx.join(ta, tb).to_numpy())
    assert sum(len(k) for k in keysets) == len(set().union(*keysets))  # keys disjoint across parts
    assert sum(1 for k in keysets if k) == G                           # every part is used
    got = oracle.canonical_rows(np.concatenate(parts)) if parts else np.zeros((0, 3), np.uint32)
    assert np.array_equal(got, ref)


def datagen_keys(rng, n):
    """Skewed keys (a few hot ones) over a small domain, so every part gets several groups."""
    hot = rng.integers(0, 50, n)
    cold = rng.integers(0, 3000, n)
    return np.where(rng.random(n) < 0.3, hot, cold)
