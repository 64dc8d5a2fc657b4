"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (one
mapsq_query / mapsq_join on the resident inputs).  The oracle cannot run the full sizes, so:

* LUBM configs: every C1/C2/C3/C5 answer relates entities of ONE university (departments,
  their members and courses live in the university's ID block; C2's ?Y is the home university),
  so the full-size GPU result restricted to a sampled university's ID block must equal — row for
  row, canonically — the oracle's answer on that university alone; plus |RS| must equal the
  generator's independent bookkeeping count of the full dataset.
* C4: |RS| must equal the cardinality law sum_k L_k R_k from np.bincount of both key columns,
  the per-key output counts must equal L_k R_k for sampled keys, and sampled output rows must be
  (key, v1, v2) with (key, v1) in Tp1 and (key, v2) in Tp2.
"""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")

import datagen  # noqa: E402
import oracle  # noqa: E402
import paper_1702_03484_b200 as mq  # noqa: E402
from fixtures import config_expected_counts, config_query  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.uint32).view(np.int32)).cuda()


@pytest.fixture(scope="module")
def ctx():
    return mq.Context(0)


_DATA = {}


def lubm_full(nu):
    if nu not in _DATA:
        _DATA.clear()
        _DATA[nu] = datagen.lubm(nu)
    return _DATA[nu]


# (config, its BASELINE.json scale)
@pytest.mark.parametrize("cfg,nu", [("C5", 10000), ("C3", 1000), ("C2", 100), ("C1", 1)])
def test_lubm_full_size_sampled_universities(ctx, cfg, nu):
    s, p, o, st = lubm_full(nu)
    trip = (dev(s), dev(p), dev(o))
    pats = config_query(cfg)
    got = ctx.query(trip, pats)
    assert got.nrows == config_expected_counts(cfg, st)[-1]
    rows = got.to_numpy()
    del trip
    # the variable whose value identifies the university block: a person (C1/C2/C5 ?x, ?X) or a
    # department (C3 ?x) — always variable 0
    col0 = rows[:, got.vars.index(0)].astype(np.int64)
    rng = np.random.default_rng(5)
    picks = sorted(set(rng.choice(nu, min(nu, 4), replace=False).tolist()) | {nu - 1})
    for u in picks:
        lo, hi = datagen.lubm_univ_base(nu, u), datagen.lubm_univ_base(nu, u + 1)
        mine = rows[(col0 >= lo) & (col0 < hi)]
        su, pu, ou, _ = datagen.lubm(nu, u, u + 1)
        ref = oracle.query(su, pu, ou, pats)
        assert ref.vars == got.vars
        assert np.array_equal(oracle.canonical_rows(mine), oracle.canonical(ref).rows), (cfg, u)


def test_c4_full_size(ctx):
    n = 500_000_000
    k1, v1 = datagen.zipf(n, 0)
    k2, v2 = datagen.zipf(n, 1)
    A = mq.DeviceTable.from_torch([0, 1], [dev(k1), dev(v1)])
    B = mq.DeviceTable.from_torch([0, 2], [dev(k2), dev(v2)])
    got = ctx.join(A, B)
    L = np.bincount(k1, minlength=1 << 29)
    R = np.bincount(k2, minlength=1 << 29)
    assert got.nrows == int((L * R).sum())
    assert got.vars == [0, 1, 2]
    key = got.columns[0].view(torch.int32).cpu().numpy().view(np.uint32)
    # output is grouped by key in ascending order: per-key counts must be L_k * R_k
    assert np.all(key[1:] >= key[:-1])
    uk, cnt = np.unique(key, return_counts=True)
    assert np.array_equal(cnt, L[uk] * R[uk])
    rng = np.random.default_rng(3)
    idx = rng.choice(got.nrows, 20000, replace=False)
    tk = torch.as_tensor(idx, device="cuda")
    sample = np.stack([c.view(torch.int32)[tk].cpu().numpy().view(np.uint32) for c in got.columns], 1)
    want = np.zeros(1 << 29, bool)
    want[sample[:, 0]] = True
    selA, selB = want[k1], want[k2]
    setA = set(zip(k1[selA].tolist(), v1[selA].tolist()))
    setB = set(zip(k2[selB].tolist(), v2[selB].tolist()))
    for kk, a, b in sample.tolist():
        assert (kk, a) in setA and (kk, b) in setB
