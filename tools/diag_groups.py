"""Developer diagnostic: HASH-path groups of C5's second join vs the true matching (x, z) keys.

  python tools/diag_groups.py 50
Runs J1 on the GPU, Maps J2's words with the HASH plan, sorts them, finds the groups through the
phase entry points and checks every group's key columns on the host."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import datagen  # noqa: E402
import paper_1702_03484_b200 as mq  # noqa: E402
from fixtures import config_query  # noqa: E402


def host(t):
    return t.view(torch.int32).cpu().numpy().view(np.uint32)


def main():
    nu = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    s, p, o, _ = datagen.lubm(nu)
    trip = tuple(torch.from_numpy(a.view(np.int32)).cuda() for a in (s, p, o))
    ctx = mq.Context(0)
    tabs = ctx.scan_patterns(trip, config_query("C5"))
    j1 = ctx.join(tabs[0], tabs[1])
    t2 = tabs[2]
    plan = mq.plan_join(j1.vars, j1.bounds, j1.nrows, t2.vars, t2.bounds, t2.nrows)
    print("plan path", plan.path, "kb", plan.kb, "ib", plan.ib, "n1", j1.nrows, "n2", t2.nrows)
    n = j1.nrows + t2.nrows
    words = torch.empty(n, dtype=torch.int64, device="cuda")
    ctx.map_words(j1, t2, plan, words)
    w0 = words.cpu().numpy().view(np.uint64).copy()
    ctx.sort_words(words, plan.ib, plan.ib + plan.kb)
    w = words.cpu().numpy().view(np.uint64)
    assert np.array_equal(np.sort(w0 >> np.uint64(plan.ib), kind="stable"), w >> np.uint64(plan.ib))
    gs, gp, ge, go, tot = ctx.reduce_groups(words, j1.nrows, t2.nrows, plan.ib)
    ng = gs.numel()
    print("groups", ng, "sum nL*nR", tot)
    A = np.stack([host(j1.column(0)), host(j1.column(2))], 1)
    B = np.stack([host(t2.column(0)), host(t2.column(2))], 1)
    ka = A[:, 0].astype(np.uint64) << np.uint64(32) | A[:, 1]
    kb = B[:, 0].astype(np.uint64) << np.uint64(32) | B[:, 1]
    print("true common keys", len(np.intersect1d(ka, kb)))
    mask = np.uint64((1 << plan.ib) - 1)
    rid = (w & mask).astype(np.int64)
    keyv = np.where(rid < j1.nrows, ka[np.minimum(rid, j1.nrows - 1)], kb[np.maximum(rid - j1.nrows, 0)])
    gs, gp, ge = (x.cpu().numpy().astype(np.int64) for x in (gs, gp, ge))
    bad = 0
    for g in range(min(ng, 200000)):
        if not np.isin(keyv[gs[g]:gp[g]], keyv[gp[g]:ge[g]]).any():
            bad += 1
    print("groups (first 200000) without a true match:", bad)
    hs = w >> np.uint64(plan.ib)
    print("distinct hashes", len(np.unique(hs)), "distinct keys", len(np.unique(keyv)))


if __name__ == "__main__":
    main()
