"""Pins for the CPU oracle (no GPU).  Each test ties the oracle to something other than itself:
the paper's worked example (Table 1), brute force from the SPARQL bag-join definition,
closed forms (the cardinality law via np.bincount), a library filter (numpy masks), and the
generator's own bookkeeping."""
from __future__ import annotations

import itertools

import numpy as np
import pytest

import datagen
import oracle
from fixtures import (brute_join_multiset, brute_query_multiset, config_expected_counts,
                      config_query, load_table1, rows_multiset)

V, C = "v", "c"


# --------------------------------------------------------------------------- Table 1
def test_table1_golden_scan_join_query():
    ids, T, sec = load_table1()
    s, p, o = T[:, 0], T[:, 1], T[:, 2]
    person, job = 0, 1
    P1 = ((V, person), (C, ids["hasJob"]), (V, job))            # P_1(?person, hasJob, ?job)
    P2 = ((V, job), (C, ids["workAt"]), (C, ids['"Hospital"']))  # P_2(?job, workAt, "Hospital")
    tp1 = oracle.scan(s, p, o, P1)
    tp2 = oracle.scan(s, p, o, P2)
    # Table 1(a): key ?job, value ?person
    assert tp1.vars == [person, job]
    assert rows_multiset(tp1.reorder([job, person]).rows) == rows_multiset(
        [[ids[k], ids[v]] for k, v in sec["tp1"]])
    # Table 1(b): keys Doctor, Nurse (reading R4(a): the constant is not a binding)
    assert tp2.vars == [job]
    assert sorted(tp2.rows[:, 0].tolist()) == sorted(ids[k] for k, _ in sec["tp2"])
    for tier in ("nested", "sortmerge"):
        rs = oracle.join(tp1, tp2, tier)
        assert rs.vars == [job, person]                          # Key | Value
        assert rows_multiset(rs.rows) == rows_multiset([[ids[k], ids[v]] for k, v, _ in sec["rs"]])
        # Proffesor (LEFT only) emits nothing (Alg. 1 l.8)
        assert ids["Proffesor"] not in rs.rows[:, 0]
    # Reading R4(b): Tp2 carrying the printed "Hospital" value column reproduces Table 1(c) exactly
    hosp = 2
    tp2b = oracle.Table([job, hosp], np.array([[ids[k], ids[v]] for k, v in sec["tp2"]], np.uint32))
    rsb = oracle.join(tp1, tp2b)
    assert rsb.vars == [job, person, hosp]
    assert rows_multiset(rsb.rows) == rows_multiset([[ids[x] for x in r] for r in sec["rs"]])
    # Query Q projected on ?person -> {Jim, Susan}
    q = oracle.query(s, p, o, [P1, P2], [person])
    assert rows_multiset(q.rows) == rows_multiset([[ids[r[0]]] for r in sec["select_person"]])


# ------------------------------------------------------------- brute force, exhaustive + random
def _tables(schema_len, alphabet, max_rows):
    rows = list(itertools.product(alphabet, repeat=schema_len))
    for k in range(max_rows + 1):
        for combo in itertools.combinations_with_replacement(rows, k):
            yield np.array(combo, np.uint32).reshape(k, schema_len)


def _check_join(a_vars, A, b_vars, B):
    ta, tb = oracle.Table(list(a_vars), A), oracle.Table(list(b_vars), B)
    for tier in ("nested", "sortmerge"):
        rs = oracle.join(ta, tb, tier)
        want = brute_join_multiset(a_vars, A, b_vars, B, rs.vars)
        assert rows_multiset(rs.rows) == want, (tier, A.tolist(), B.tolist())
    return rs


def test_exhaustive_tiny_single_key():
    # schema A = (k, a), B = (k, b); all multisets of <=3 rows over keys {0,1,2} x values {0,1}
    tabs = [t for t in _tables(2, (0, 1, 2), 2)]
    n = 0
    for A in tabs:
        for B in tabs:
            A2 = A.copy(); B2 = B.copy()
            A2[:, 1] %= 2; B2[:, 1] %= 2
            _check_join((0, 1), A2, (0, 2), B2)
            n += 1
    assert n == len(tabs) ** 2


def test_exhaustive_tiny_three_rows():
    tabs = list(_tables(2, (0, 1), 3))
    for A in tabs:
        for B in tabs:
            _check_join((5, 1), A, (2, 5), B)   # key var 5 sits at different positions


def test_exhaustive_tiny_composite_key():
    # A = (x, z, a), B = (z, x): composite key (x, z) in different column orders (reading R5)
    tabs_a = list(_tables(3, (0, 1), 2))
    tabs_b = list(_tables(2, (0, 1), 2))
    for A in tabs_a:
        for B in tabs_b:
            _check_join((0, 2, 1), A, (2, 0), B)


@pytest.mark.parametrize("domain", [1, 5, 50])
def test_random_skewed_tier0_equals_tier1_and_cardinality_law(domain):
    rng = np.random.default_rng(domain)
    for case in range(60):
        n1, n2 = rng.integers(0, 200, 2)
        A = np.stack([rng.integers(0, domain, n1), rng.integers(0, 1000, n1)], 1).astype(np.uint32)
        B = np.stack([rng.integers(0, domain, n2), rng.integers(0, 1000, n2)], 1).astype(np.uint32)
        ta, tb = oracle.Table([0, 1], A), oracle.Table([0, 2], B)
        r0, r1 = oracle.join(ta, tb, "nested"), oracle.join(ta, tb, "sortmerge")
        assert r0.vars == r1.vars == [0, 1, 2]
        assert np.array_equal(oracle.canonical(r0).rows, oracle.canonical(r1).rows)
        # cardinality law |RS| = sum_k L_k R_k, closed form via bincount
        L = np.bincount(A[:, 0], minlength=domain)
        R = np.bincount(B[:, 0], minlength=domain)
        assert r1.nrows == int((L * R).sum())
        # every output row pairs a real A row with a real B row on the same key
        if r1.nrows:
            a_set = {tuple(r) for r in A.tolist()}
            b_set = {tuple(r) for r in B.tolist()}
            for k, va, vb in r1.rows.tolist()[:50]:
                assert (k, va) in a_set and (k, vb) in b_set


def test_commutativity_up_to_column_order():
    rng = np.random.default_rng(3)
    for _ in range(40):
        A = rng.integers(0, 6, (rng.integers(0, 60), 3)).astype(np.uint32)
        B = rng.integers(0, 6, (rng.integers(0, 60), 2)).astype(np.uint32)
        ta, tb = oracle.Table([3, 1, 0], A), oracle.Table([0, 3], B)
        ab, ba = oracle.join(ta, tb), oracle.join(tb, ta)
        assert ab.vars == [0, 3, 1] and ba.vars == [0, 3, 1]
        assert np.array_equal(oracle.canonical(ab).rows, oracle.canonical(ba.reorder(ab.vars)).rows)


def test_empty_sides_and_errors():
    A = np.zeros((0, 2), np.uint32)
    B = np.array([[1, 2]], np.uint32)
    rs = oracle.join(oracle.Table([0, 1], A), oracle.Table([0, 2], B))
    assert rs.nrows == 0 and rs.vars == [0, 1, 2]
    rs = oracle.join(oracle.Table([0, 2], B), oracle.Table([0, 1], A))
    assert rs.nrows == 0 and rs.vars == [0, 2, 1]
    with pytest.raises(oracle.OracleError) as e:
        oracle.join(oracle.Table([0], B[:, :1]), oracle.Table([1], B[:, :1]))
    assert e.value.code == oracle.E_NO_SHARED


def test_group_2L_3R_gives_6_rows():
    A = np.array([[7, 1], [7, 2]], np.uint32)
    B = np.array([[7, 10], [7, 11], [7, 12], [8, 13]], np.uint32)
    rs = oracle.join(oracle.Table([0, 1], A), oracle.Table([0, 2], B))
    assert rs.nrows == 6
    # tier-1 emission order is (A row, B row) within the key
    assert rs.rows.tolist() == [[7, 1, 10], [7, 1, 11], [7, 1, 12], [7, 2, 10], [7, 2, 11], [7, 2, 12]]


# ------------------------------------------------------------------------------------ scan
def test_scan_equals_numpy_filter_and_repeated_vars():
    rng = np.random.default_rng(11)
    T = rng.integers(0, 8, (5000, 3)).astype(np.uint32)
    s, p, o = T.T
    pats = [((V, 0), (C, 3), (V, 1)), ((V, 0), (C, 3), (C, 5)), ((C, 2), (V, 4), (V, 1)),
            ((V, 0), (V, 1), (V, 2)), ((V, 0), (C, 1), (V, 0)), ((V, 2), (V, 2), (V, 2)),
            ((V, 0), (C, 99), (V, 1)), ((C, 1), (C, 2), (V, 3))]
    for pat in pats:
        got = oracle.scan(s, p, o, pat)
        mask = np.ones(len(T), bool)
        first = {}
        for j, (kind, x) in enumerate(pat):
            if kind == C:
                mask &= T[:, j] == x
            elif x in first:
                mask &= T[:, j] == T[:, first[x]]
            else:
                first[x] = j
        want = T[mask][:, list(first.values())]
        assert got.vars == list(first.keys())
        assert np.array_equal(got.rows, want)  # triple order preserved


def test_scan_zero_vars_is_invalid():
    with pytest.raises(oracle.OracleError):
        oracle.scan([1], [2], [3], ((C, 1), (C, 2), (C, 3)))


# ------------------------------------------------------------------------------- query
def test_query_equals_bruteforce_enumeration():
    rng = np.random.default_rng(5)
    for case in range(25):
        nt = int(rng.integers(5, 40))
        T = np.unique(rng.integers(0, 5, (nt, 3)), axis=0).astype(np.uint32)
        s, p, o = T.T
        # random connected BGP of 2-3 patterns over variables 0..3
        pats = [((V, 0), (C, int(rng.integers(0, 5))), (V, 1))]
        if case % 2:
            pats.append(((V, 1), (C, int(rng.integers(0, 5))), (V, 2)))
        else:
            pats.append(((V, 2), (V, 1), (V, 0)))
        if case % 3 == 0:
            pats.append(((V, 2), (C, int(rng.integers(0, 5))), (V, 0)))
        proj = [] if case % 4 else [1]
        try:
            got = oracle.query(s, p, o, pats, proj)
        except oracle.OracleError:
            raise
        assert rows_multiset(got.rows) == brute_query_multiset(T, pats, proj)


def test_query_plan_invariance():
    rng = np.random.default_rng(9)
    T = np.unique(rng.integers(0, 6, (120, 3)), axis=0).astype(np.uint32)
    s, p, o = T.T
    pats = [((V, 0), (C, 1), (V, 1)), ((V, 1), (C, 2), (V, 2)), ((V, 2), (C, 3), (V, 0))]
    a = oracle.query(s, p, o, pats, [0, 1, 2])
    b = oracle.query(s, p, o, [pats[1], pats[2], pats[0]], [0, 1, 2])
    assert np.array_equal(oracle.canonical(a).rows, oracle.canonical(b).rows)


def test_query_disconnected_is_error():
    with pytest.raises(oracle.OracleError) as e:
        oracle.query([1], [2], [3], [((V, 0), (C, 2), (V, 1)), ((V, 2), (C, 2), (V, 3))])
    assert e.value.code == oracle.E_NO_SHARED


# ------------------------------------------------- generator bookkeeping (independent counts)
@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C5"])
def test_oracle_matches_generator_bookkeeping(cfg):
    s, p, o, st = datagen.lubm(3, u_lo=0, u_hi=2)   # two universities of LUBM(3)
    pats = config_query(cfg)
    want = config_expected_counts(cfg, st)
    acc = oracle.scan(s, p, o, pats[0])
    for i, pat in enumerate(pats[1:]):
        acc = oracle.join(acc, oracle.scan(s, p, o, pat))
        assert acc.nrows == want[i], (cfg, i)
    q = oracle.query(s, p, o, pats)
    assert q.nrows == want[-1]


# -------------------------------------- composite keys of 3, 4 and 5 shared variables (R5)
# sortmerge_fixed<3> and sortmerge_generic (>= 4 key columns) pinned to brute force and to the
# cardinality law of the equivalent single-key join (the key tuple encoded as one integer).
def test_exhaustive_tiny_three_shared_vars():
    # A = (x, y, z), B = (z, b, x, y): key (x, y, z) at different positions on each side
    tabs_a = list(_tables(3, (0, 1), 2))
    tabs_b = list(_tables(4, (0, 1), 2))
    for A in tabs_a:
        for B in tabs_b:
            rs = _check_join((0, 1, 2), A, (2, 7, 0, 1), B)
            assert rs.vars == [0, 1, 2, 7]


def test_exhaustive_tiny_four_shared_vars():
    # A = (w, x, y, z, a) with a fixed per row, B = (z, y, x, w): the generic (>= 4) tier
    tabs_a = list(_tables(4, (0, 1), 2))
    tabs_b = list(_tables(4, (0, 1), 2))
    for i, A in enumerate(tabs_a):
        A5 = np.concatenate([A, (np.arange(len(A), dtype=np.uint32) % 2)[:, None]], 1)
        for B in tabs_b[i % 3::3]:
            rs = _check_join((3, 4, 5, 6, 9), A5, (6, 5, 4, 3), B)
            assert rs.vars == [3, 4, 5, 6, 9]


@pytest.mark.parametrize("nkey", [3, 4, 5])
def test_random_wide_keys_bruteforce_and_encoded_single_key(nkey):
    rng = np.random.default_rng(100 + nkey)
    D = 2
    for case in range(40):
        n1, n2 = (int(x) for x in rng.integers(0, 14, 2))
        # A: key columns in order 0..nkey-1 plus one rest column; B: keys reversed plus one rest
        A = rng.integers(0, D, (n1, nkey + 1)).astype(np.uint32)
        B = rng.integers(0, D, (n2, nkey + 1)).astype(np.uint32)
        a_vars = list(range(nkey)) + [20]
        b_vars = [21] + list(range(nkey))[::-1]
        rs = _check_join(a_vars, A, b_vars, B)
        assert rs.vars == list(range(nkey)) + [20, 21]
        # cardinality law on the encoded key: code = sum_i key_i * D^i
        wa = D ** np.arange(nkey)
        ca = (A[:, :nkey].astype(np.int64) * wa).sum(1)
        cb = (B[:, 1:][:, ::-1].astype(np.int64) * wa).sum(1)
        L = np.bincount(ca, minlength=D ** nkey)
        R = np.bincount(cb, minlength=D ** nkey)
        assert rs.nrows == int((L * R).sum())


@pytest.mark.parametrize("nkey", [3, 4, 5])
def test_wide_key_equals_single_key_join_on_encoded_key(nkey):
    # The natural join on nkey shared columns equals the single-key join (pinned above) on the
    # key tuple encoded as one integer, with the tuple decoded back: a transposed or dropped key
    # column in either tier would break the equality.
    rng = np.random.default_rng(7 * nkey)
    D = 3
    for case in range(15):
        n1, n2 = (int(x) for x in rng.integers(0, 300, 2))
        KA = rng.integers(0, D, (n1, nkey)).astype(np.uint32)
        KB = rng.integers(0, D, (n2, nkey)).astype(np.uint32)
        va = rng.integers(0, 1 << 31, n1).astype(np.uint32)
        vb = rng.integers(0, 1 << 31, n2).astype(np.uint32)
        perm = rng.permutation(nkey)            # B stores its key columns in a shuffled order
        A = np.concatenate([KA, va[:, None]], 1)
        B = np.concatenate([vb[:, None], KB[:, perm]], 1)
        wide = oracle.join(oracle.Table(list(range(nkey)) + [40], A),
                           oracle.Table([41] + [int(v) for v in perm], B))
        w = D ** np.arange(nkey)[::-1]
        code_a = (KA.astype(np.int64) * w).sum(1).astype(np.uint32)
        code_b = (KB.astype(np.int64) * w).sum(1).astype(np.uint32)
        single = oracle.join(oracle.Table([50, 40], np.stack([code_a, va], 1)),
                             oracle.Table([41, 50], np.stack([vb, code_b], 1)), "nested")
        code = single.rows[:, 0].astype(np.int64)
        dec = np.stack([(code // D ** (nkey - 1 - i)) % D for i in range(nkey)], 1)
        want = np.concatenate([dec.astype(np.uint32), single.rows[:, 1:]], 1)
        assert wide.vars == list(range(nkey)) + [40, 41]
        assert np.array_equal(oracle.canonical(wide).rows, oracle.canonical_rows(want))


# ----------------------------------------------- whole-output fingerprint
def test_fingerprint_row_hash_is_splitmix64():
    # One row (0): h = splitmix64 output from state 0 = 0xE220A8397B1DCDAF (the generator's
    # published first output for seed 0).
    t = oracle.Table([0], np.zeros((1, 1), np.uint32))
    assert oracle.fingerprint(t) == (1, 0xE220A8397B1DCDAF, 0xE220A8397B1DCDAF)
    assert oracle.fingerprint(oracle.Table([0], np.zeros((0, 1), np.uint32))) == (0, 0, 0)


def test_fingerprint_is_a_multiset_function():
    rng = np.random.default_rng(1)
    rows = rng.integers(0, 1 << 32, (5000, 4), dtype=np.uint64).astype(np.uint32)
    base = oracle.fingerprint(oracle.Table([0, 1, 2, 3], rows))
    # order-independent, chunkable, and the SoA entry point agrees with the row-major one
    assert oracle.fingerprint(oracle.Table([0, 1, 2, 3], rows[rng.permutation(5000)])) == base
    f = oracle.Fingerprint()
    for lo in range(0, 5000, 1234):
        f.add_cols([rows[lo:lo + 1234, c] for c in range(4)])
    assert f.value == base
    # sensitive to a duplicated row, a changed value and swapped columns
    assert oracle.fingerprint(oracle.Table([0, 1, 2, 3], np.concatenate([rows, rows[:1]]))) != base
    r2 = rows.copy(); r2[17, 2] ^= 1
    assert oracle.fingerprint(oracle.Table([0, 1, 2, 3], r2)) != base
    assert oracle.fingerprint(oracle.Table([0, 1, 2, 3], rows[:, [1, 0, 2, 3]])) != base
