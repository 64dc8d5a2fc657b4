"""Row e at world size 2 (and 3) on ONE GPU: the library's distributed join / query end to end.

tests/dist_worker.py runs as `world` processes sharing cuda:0, gloo for the control plane
(mapsq_dist_init_host).  Every exchange runs the product path — K8 plan, count all-gather,
CUDA-IPC receive arenas mapped by the peers, the fused scatter kernel storing rows into the
OTHER process's arena, local Algorithm-1 join — and the union of the rank shards must equal the
CPU oracle's result on the union of the inputs (an equi-join decomposes over disjoint key sets:
Alg. 1 joins each key group on its own).  The exchange counters must show rows
crossing between the processes."""
from __future__ import annotations

import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import datagen  # noqa: E402
import oracle  # noqa: E402
from dist_worker import NCASES, join_case_tables  # noqa: E402
from fixtures import config_query  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def run_world(world: int, tmp_path, nu: int):
    port = free_port()
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "dist_worker.py"), "--rank",
                               str(r), "--world", str(world), "--port", str(port), "--out",
                               str(tmp_path), "--nu", str(nu)],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
             for r in range(world)]
    logs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=600)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        logs.append(out.decode(errors="replace"))
    for r, (p, log) in enumerate(zip(procs, logs)):
        assert p.returncode == 0, f"rank {r} failed:\n{log[-4000:]}"
    return [dict(np.load(os.path.join(tmp_path, f"rank{r}.npz"))) for r in range(world)]


def union(shards, name):
    vars_ = [list(s[name + ":vars"]) for s in shards]
    assert all(v == vars_[0] for v in vars_)
    rows = np.concatenate([s[name].reshape(-1, len(vars_[0])) for s in shards])
    return vars_[0], rows


@pytest.mark.parametrize("world,nu", [(2, 2), (3, 3)])
def test_dist_multiprocess_one_gpu(tmp_path, world, nu):
    shards = run_world(world, tmp_path, nu)
    # LUBM configs: the union of the rank shards is the oracle's answer on the whole dataset
    s, p, o, _ = datagen.lubm(nu)
    for cfg in ("C1", "C2", "C3", "C5"):
        ref = oracle.query(s, p, o, config_query(cfg))
        for name in (f"q_{cfg}_auto", f"q_{cfg}_on", f"qscan_{cfg}"):
            vars_, rows = union(shards, name)
            assert vars_ == ref.vars, name
            assert np.array_equal(oracle.canonical_rows(rows), oracle.canonical(ref).rows), name
    # random joins (skewed single key, composite wide key, everything on one rank, two heavy
    # single keys, a heavy composite key), with and without the pre-filter and the skew handling
    for case in range(NCASES):
        va, A, vb, B = join_case_tables(case)
        ref = oracle.join(oracle.Table(va, A), oracle.Table(vb, B))
        names = [f"j{case}_auto", f"j{case}_on"] + ([f"j{case}_noskew"] if case in (3, 4) else [])
        for name in names:
            vars_, rows = union(shards, name)
            assert vars_ == ref.vars
            assert np.array_equal(oracle.canonical_rows(rows), oracle.canonical(ref).rows), name
    # the heavy keys of cases 3 and 4 were detected (split / broadcast) on every rank
    assert all(int(sh["stat_skew_keys"]) >= 2 * 2 + 2 for sh in shards)
    # rows really crossed between the processes, and what one rank sent the others received
    sent = sum(int(sh["stat_exchange_rows"]) for sh in shards)
    recv = sum(int(sh["stat_exchange_recv_rows"]) for sh in shards)
    assert sent > 0 and sent == recv
    assert all(int(sh["stat_exchange_rows"]) > 0 for sh in shards)
    assert sum(int(sh["stat_exchange_bytes"]) for sh in shards) == \
        sum(int(sh["stat_exchange_recv_bytes"]) for sh in shards)
