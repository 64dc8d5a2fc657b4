"""SPARQL text through the GPU path: parse, match, join (greedy or textual
order), project and decode, against the paper's Table 1 answer and the CPU oracle."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import datagen  # noqa: E402
import oracle  # noqa: E402
import paper_1702_03484_b200 as mq  # noqa: E402
from paper_1702_03484_b200 import sparql as sq  # noqa: E402
from test_sparql import Q, table1_lines  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    return mq.Context(0)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).cuda()


@pytest.mark.parametrize("plan", ["greedy", "textual"])
def test_table1_query_text(ctx, plan):
    d, s, p, o = sq.load_ntriples(table1_lines())
    trip = (dev(s), dev(p), dev(o))
    for store in (trip, ctx.index_build(trip)):
        rs = sq.execute(ctx, store, d, Q, plan=plan)
        assert rs.schema == ["person"]
        assert sorted(str(t) for t in rs.rows[:, 0]) == ["Jim", "Susan"]
    rs = sq.execute(ctx, trip, d, "SELECT * WHERE { ?s ?p ?o . }", plan=plan)
    assert rs.schema == ["s", "p", "o"] and rs.rows.shape == (5, 3)
    rs = sq.execute(ctx, trip, d, "SELECT ?x WHERE { ?x hasJob ?y . ?y nosuch ?z }", plan=plan)
    assert rs.rows.shape == (0, 1)  # unknown constant matches nothing


def lubm_dictionary(nu: int) -> sq.Dictionary:
    d = sq.Dictionary()
    names = {v: k for k, v in datagen.LUBM_PRED.items()}
    names.update({v: k for k, v in datagen.LUBM_CLASS.items()})
    for i in range(datagen.lubm_id_end(nu)):
        d.intern(sq.Term("iri", names.get(i, f"e{i}")))
    return d


@pytest.mark.parametrize("cfg,text", [
    ("C1", "SELECT ?x ?d ?u WHERE { ?x worksFor ?d . ?d subOrganizationOf ?u }"),
    ("C5", "SELECT * WHERE { ?x advisor ?y . ?y teacherOf ?z . ?x takesCourse ?z . }"),
    ("C2", "SELECT ?X ?Y WHERE { ?X memberOf ?Z . ?Z subOrganizationOf ?Y . "
           "?X undergraduateDegreeFrom ?Y }"),
])
def test_lubm_query_text_matches_oracle(ctx, cfg, text):
    from fixtures import config_query
    s, p, o, _ = datagen.lubm(2)
    d = lubm_dictionary(2)
    trip = (dev(s), dev(p), dev(o))
    q = sq.parse_query(text)
    pats, proj, names = sq.encode(q, d)
    assert pats == config_query(cfg)  # the text encodes to the config's descriptors
    ref = oracle.query(s, p, o, pats, proj)
    want = sorted(tuple(str(t) for t in row) for row in d.decode(ref.rows.reshape(-1)).reshape(ref.rows.shape))
    for plan in ("greedy", "textual"):
        rs = sq.execute(ctx, ctx.index_build(trip), d, text, plan=plan)
        assert rs.schema == [names[v] for v in proj]
        assert sorted(tuple(str(t) for t in row) for row in rs.rows) == want
