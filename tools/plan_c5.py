"""Join plans of C5's two joins at full scale (TOOL, run on a B200): key bits, passes, paths."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1702_03484_b200 as mq  # noqa: E402

nu = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
(s, p, o), st, _ = bench.lubm_host(nu, 0, nu, pinned=False)
ctx = mq.Context(0)
idx = ctx.index_build(tuple(torch.from_numpy(a.view(np.int32)).cuda() for a in (s, p, o)))
pats = bench.query_patterns("C5")
t = ctx.scan_patterns(idx, pats)
for i, x in enumerate(t):
    print("pattern", i, x.vars, x.nrows, x.bounds)
ctx.stats_reset()
j1 = ctx.join(t[0], t[1])
st1 = ctx.stats()
print("J1", {k: st1[k] for k in ("last_kb", "last_ib", "last_passes", "last_path", "last_filtered")}, j1.nrows, j1.bounds)
ctx.stats_reset()
j2 = ctx.join(j1, t[2])
st2 = ctx.stats()
print("J2", {k: st2[k] for k in ("last_kb", "last_ib", "last_passes", "last_path", "last_filtered")}, j2.nrows)
