"""Developer diagnostic: per-join shapes and per-kernel event times of a LUBM config query.

  python tools/diag_query.py C5 10000 [scan]
Answers the query's patterns from the predicate index (or the full scan), then runs each join
alone with profiling on and prints n1, n2, key bits, path, groups, |RS| and kernel times with
the GB/s of each kernel's algorithmic bytes."""
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


def main():
    cfg, nu = sys.argv[1], int(sys.argv[2])
    use_scan = len(sys.argv) > 3 and sys.argv[3] == "scan"
    s, p, o, _ = datagen.lubm(nu)
    trip = tuple(torch.from_numpy(a.view(np.int32)).cuda() for a in (s, p, o))
    ctx = mq.Context(0)
    src = trip if use_scan else ctx.index_build(trip)
    pats = config_query(cfg)
    for rep in range(2):
        tabs = ctx.scan_patterns(src, pats)
        acc = tabs[0]
        for j, t in enumerate(tabs[1:]):
            torch.cuda.synchronize()
            ctx.stats_reset()
            ctx.set_profiling(True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = ctx.join(acc, t)
            e1.record()
            torch.cuda.synchronize()
            st = ctx.stats()
            ctx.set_profiling(False)
            if rep:
                print(f"J{j + 1}: n1={acc.nrows} n2={t.nrows} kb={st['last_kb']} ib={st['last_ib']} "
                      f"passes={st['last_passes']} path={st['last_path']} groups={st['last_groups']} "
                      f"|RS|={r.nrows} join {e0.elapsed_time(e1):.3f} ms")
                for k, v in st["kernels"].items():
                    print(f"    {k:16s} x{v['launches']:<3d} {v['ms']:8.3f} ms  "
                          f"{v['bytes'] / 1e9:7.2f} GB  {v['bytes'] / v['ms'] / 1e6 if v['ms'] else 0:7.0f} GB/s")
            acc = r


if __name__ == "__main__":
    main()
