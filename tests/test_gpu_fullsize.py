"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (one
mapsq_query over the resident store, one mapsq_join on the resident C4 tables).

The oracle cannot run on the GPU box at these sizes, so it ran once on a big host:
tools/oracle_fingerprint.py (oracle/ + datagen/ only) stored the whole-output multiset
fingerprint of every config in tests/golden/fingerprints.json — row count, sum mod 2^64 and xor
of a per-row splitmix64 hash (oracle.h oracle_fingerprint).  Here the FULL
GPU output is copied to the host in chunks and hashed by the same oracle routine, so every row
of every config is compared (a missing, duplicated, mis-paired or altered row changes the
fingerprint), for every store and semi-join filter mode the bench can run.
"""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")

import datagen  # noqa: E402
import oracle  # noqa: E402
import paper_1702_03484_b200 as mq  # noqa: E402
from fixtures import GOLDEN, config_query  # noqa: E402

GOLD = json.load(open(os.path.join(GOLDEN, "fingerprints.json")))
MODES = {"auto": mq.SEMIJOIN_AUTO, "off": mq.SEMIJOIN_OFF, "on": mq.SEMIJOIN_ON}


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.uint32).view(np.int32)).cuda()


@pytest.fixture(scope="module")
def ctx():
    c = mq.Context(0)
    yield c
    c.set_option(mq.OPT_SEMIJOIN, mq.SEMIJOIN_AUTO)


def device_fingerprint(t) -> tuple:
    """oracle.Fingerprint of a device table, copied to the host 2^25 rows at a time."""
    f = oracle.Fingerprint()
    step = 1 << 25
    for lo in range(0, t.nrows, step):
        f.add_cols([c[lo:lo + step].view(torch.int32).cpu().numpy().view(np.uint32)
                    for c in t.columns])
    return f.value


def check(cfg, got, what):
    g = GOLD[cfg]
    assert got.vars == g["vars"], (cfg, what)
    want = (g["nrows"], int(g["sum"], 16), int(g["xor"], 16))
    assert got.nrows == want[0], (cfg, what, got.nrows, want[0])
    assert device_fingerprint(got) == want, (cfg, what)


# (config, its BASELINE.json scale)
@pytest.mark.parametrize("cfg,nu", [("C5", 10000), ("C3", 1000), ("C2", 100), ("C1", 1)])
def test_lubm_full_size_fingerprint(ctx, cfg, nu):
    s, p, o, st = datagen.lubm(nu)
    trip = (dev(s), dev(p), dev(o))
    del s, p, o
    idx = ctx.index_build(trip)
    pats = config_query(cfg)
    runs = [("index", m) for m in ("auto", "off", "on")] + [("scan", "auto")]
    for store, mode in runs:
        ctx.set_option(mq.OPT_SEMIJOIN, MODES[mode])
        got = ctx.query(idx if store == "index" else trip, pats)
        check(cfg, got, (store, mode))
        got.release()
    ctx.set_option(mq.OPT_SEMIJOIN, mq.SEMIJOIN_AUTO)
    idx.release()


def test_c4_full_size_fingerprint(ctx):
    n = 500_000_000
    k1, v1 = datagen.zipf(n, 0)
    k2, v2 = datagen.zipf(n, 1)
    A = mq.DeviceTable.from_torch([0, 1], [dev(k1), dev(v1)])
    B = mq.DeviceTable.from_torch([0, 2], [dev(k2), dev(v2)])
    del k1, v1, k2, v2
    for mode in ("auto", "off"):
        ctx.set_option(mq.OPT_SEMIJOIN, MODES[mode])
        got = ctx.join(A, B)
        check("C4", got, mode)
        if mode == "auto":
            # one GPU: rows come out in (key, Tp1 row, Tp2 row) order — keys ascend
            key = got.columns[0]
            assert bool((key[1:].view(torch.int32).long() & 0xffffffff
                         >= (key[:-1].view(torch.int32).long() & 0xffffffff)).all())
        got.release()
    ctx.set_option(mq.OPT_SEMIJOIN, mq.SEMIJOIN_AUTO)
