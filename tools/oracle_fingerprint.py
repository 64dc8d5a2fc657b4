"""Write tests/golden/fingerprints.json: the CPU oracle's whole-output fingerprint of every
BASELINE.json config at its full size.

Calls only ``oracle/`` (scan, sort-merge join, query fold, fingerprint) and ``datagen/`` (the
seeded inputs); nothing here touches the CUDA path.  The GPU full-size tests
(tests/test_gpu_fullsize.py) hash the device result with the same ``oracle.Fingerprint`` and
must match these numbers exactly.

    python tools/oracle_fingerprint.py C1 C2 C3 C5 C4     # ~62 GB host RAM for C4 / C5

Each config runs in its own process (the inputs of C4 / C5 are 8-15 GB).
"""
from __future__ import annotations

import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
OUT = os.path.join(ROOT, "tests", "golden", "fingerprints.json")

LUBM_SCALE = {"C1": 1, "C2": 100, "C3": 1000, "C5": 10000}
C4_ROWS = 500_000_000


def one(cfg: str) -> dict:
    import numpy as np

    import datagen
    import oracle
    from fixtures import config_query

    t0 = time.time()
    if cfg == "C4":
        k1, v1 = datagen.zipf(C4_ROWS, 0)
        k2, v2 = datagen.zipf(C4_ROWS, 1)
        a = oracle.Table([0, 1], np.stack([k1, v1], 1))
        del k1, v1
        b = oracle.Table([0, 2], np.stack([k2, v2], 1))
        del k2, v2
        t1 = time.time()
        rs = oracle.join(a, b)
        desc = {"input": "datagen.zipf(5e8, side 0 / 1), seed 1702, s=1.1, kbits=29 (reading R15)",
                "call": "oracle.join(Table([0,1], key|val side 0), Table([0,2], key|val side 1))"}
    else:
        nu = LUBM_SCALE[cfg]
        s, p, o, st = datagen.lubm(nu)
        t1 = time.time()
        rs = oracle.query(s, p, o, config_query(cfg))
        desc = {"input": f"datagen.lubm({nu}), seed 42, {len(s)} triples",
                "call": f"oracle.query(triples, fixtures.config_query('{cfg}'))"}
    t2 = time.time()
    fp = oracle.fingerprint(rs)
    return {"vars": rs.vars, "nrows": fp[0], "sum": f"{fp[1]:#018x}", "xor": f"{fp[2]:#018x}",
            **desc, "oracle_s": round(t2 - t1, 1), "gen_s": round(t1 - t0, 1)}


def main(cfgs: list[str]) -> None:
    if len(cfgs) == 1 and os.environ.get("FP_CHILD"):
        print(json.dumps(one(cfgs[0])))
        return
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    data.setdefault("_doc", "Whole-output multiset fingerprints written by tools/oracle_fingerprint.py "
                    "from oracle/ only: nrows, sum mod 2^64 and xor of the per-row splitmix64 hash "
                    "(oracle.h oracle_fingerprint), row values in the listed variable order.")
    for cfg in cfgs:
        r = subprocess.run([sys.executable, __file__, cfg], env={**os.environ, "FP_CHILD": "1"},
                           capture_output=True, text=True)
        if r.returncode:
            sys.exit(f"{cfg}: {r.stderr[-2000:]}")
        data[cfg] = json.loads(r.stdout.strip().splitlines()[-1])
        print(cfg, data[cfg], flush=True)
        with open(OUT, "w") as f:
            json.dump(data, f, indent=1, sort_keys=True)
            f.write("\n")


if __name__ == "__main__":
    main(sys.argv[1:] or ["C1", "C2", "C3", "C5", "C4"])
