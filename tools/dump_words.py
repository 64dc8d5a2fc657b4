"""Developer tool: dump the Map words of a config's joins (raw u64) for tools/radix_ablate.

  python tools/dump_words.py C5 2000 /tmp/words   -> /tmp/words_J1.u64, /tmp/words_J2.u64 + meta
Prints one line per join: path, n, ib, kb (the arguments of `radix_ablate file`)."""
import json
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
    cfg, nu, prefix = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    s, p, o, _ = datagen.lubm(nu)
    trip = tuple(torch.from_numpy(a.view(np.int32)).cuda() for a in (s, p, o))
    ctx = mq.Context(0)
    tabs = ctx.scan_patterns(trip, config_query(cfg))
    acc = tabs[0]
    meta = []
    for j, t in enumerate(tabs[1:]):
        plan = mq.plan_join(acc.vars, acc.bounds, acc.nrows, t.vars, t.bounds, t.nrows)
        n = acc.nrows + t.nrows
        words = torch.empty(n, dtype=torch.int64, device="cuda")
        ctx.map_words(acc, t, plan, words)
        path = f"{prefix}_J{j + 1}.u64"
        words.cpu().numpy().tofile(path)
        meta.append(dict(join=j + 1, path=path, n=n, ib=plan.ib, kb=plan.kb, plan_path=plan.path))
        print(f"J{j + 1} {path} {plan.ib} {plan.kb}  n={n} path={plan.path}", flush=True)
        acc = ctx.join(acc, t)
    json.dump(meta, open(prefix + "_meta.json", "w"))


if __name__ == "__main__":
    main()
