"""SPARQL front-end, dictionary and greedy planner — host logic, no GPU.

Pinned to the paper's query Q and Table 1 fixture, to the
SPEC's first-seen dictionary IDs and its planner example."""
from __future__ import annotations

import os

import numpy as np
import pytest

from paper_1702_03484_b200 import sparql as sq

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "table1.txt")
Q = 'SELECT ?person WHERE {?person hasJob ?job. ?job workAt "Hospital".}'


def table1_lines():
    lines, on = [], False
    for line in open(GOLDEN):
        line = line.strip()
        if line.startswith("["):
            on = line == "[triples]"
            continue
        if on and line and not line.startswith("#"):
            lines.append(line + " .")
    return lines


def test_parse_paper_query_q():
    q = sq.parse_query(Q)
    assert q.projection == ["person"]
    assert q.patterns == [(sq.Var("person"), sq.Term("iri", "hasJob"), sq.Var("job")),
                          (sq.Var("job"), sq.Term("iri", "workAt"), sq.Term("lit", "Hospital"))]
    assert q.variables() == ["person", "job"]


def test_parse_star_iris_literals_and_round_trip():
    q = sq.parse_query('select * where { ?s ?p ?o . }')
    assert q.projection is None and q.patterns == [(sq.Var("s"), sq.Var("p"), sq.Var("o"))]
    text = 'SELECT ?a ?b WHERE {\n ?a <http://x.org/p#1> ?b .\n ?b q "a \\"quoted\\" lit" }'
    q = sq.parse_query(text)
    assert q.patterns[0][1] == sq.Term("iri", "http://x.org/p#1")
    assert q.patterns[1][2] == sq.Term("lit", 'a "quoted" lit')
    assert sq.parse_query(str(q)) == q  # printer round trip
    assert sq.parse_query(str(sq.parse_query(Q))) == sq.parse_query(Q)


@pytest.mark.parametrize("text,where", [
    ("SELECT ?x WHERE { ?y p q . }", "projected variable ?x"),
    ("SELECT ?x WHERE { ?x p }", "line 1, column 24"),
    ("SELECT ?x\nWHERE { ?x p q . ] }", "line 2, column 18"),
    ("SELECT WHERE { ?x p q }", "line 1, column 8"),
    ("SELECT ?x WHERE { }", "empty"),
    ("SELECT ?x WHERE { ?x p q } extra", "trailing"),
])
def test_parse_errors_have_positions(text, where):
    with pytest.raises(sq.SparqlError) as e:
        sq.parse_query(text)
    assert where in str(e.value)


def test_dictionary_first_seen_ids_and_set_semantics():
    d, s, p, o = sq.load_ntriples(table1_lines() + ["Jim hasJob Doctor ."])  # duplicate dropped
    names = ["Anny", "hasJob", "Proffesor", "Jim", "Doctor", "Susan", "Nurse", "workAt"]
    assert [d.lookup(sq.Term("iri", x)) for x in names] == list(range(8))
    assert d.lookup(sq.Term("lit", "Hospital")) == 8
    assert len(s) == 5
    assert np.array_equal(np.stack([s, p, o], 1),
                          [[0, 1, 2], [3, 1, 4], [5, 1, 6], [4, 7, 8], [6, 7, 8]])
    assert d.resolve(d.intern(sq.Term("iri", "Jim"))) == sq.Term("iri", "Jim")
    assert [str(t) for t in d.decode(np.array([3, 8]))] == ["Jim", '"Hospital"']


def test_encode_and_greedy_plan():
    d, *_ = sq.load_ntriples(table1_lines())
    q = sq.parse_query(Q)
    pats, proj, names = sq.encode(q, d)
    assert pats == [(("v", 0), ("c", 1), ("v", 1)), (("v", 1), ("c", 7), ("c", 8))]
    assert proj == [0] and names == ["person", "job"]
    # on the fixture pattern 2 (2 rows) comes before pattern 1 (3 rows)
    assert sq.greedy_order([3, 2], [[0, 1], [1]]) == [1, 0]
    assert sq.greedy_order([5, 5, 1], [[0, 1], [1, 2], [2, 3]]) == [2, 1, 0]  # connected growth
    with pytest.raises(sq.SparqlError):
        sq.greedy_order([1, 1], [[0], [1]])
    pats, _, _ = sq.encode(sq.parse_query("SELECT ?x WHERE { ?x nosuch ?y }"), d)
    assert pats[0][1] == ("c", sq.ABSENT)  # unknown constant: matches nothing
