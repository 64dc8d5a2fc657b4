"""Shared test helpers: the Table 1 golden fixture, brute-force definitions, query configs.

Nothing here computes a join the way the method or the oracle does: the brute-force helpers
enumerate candidate solution mappings from first principles (SPARQL algebra multiplicities).
"""
from __future__ import annotations

import itertools
import os
from collections import Counter

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_table1():
    """Parse tests/golden/table1.txt -> (ids, triples, sections) with first-seen IDs."""
    sections: dict = {}
    cur = None
    for line in open(os.path.join(GOLDEN, "table1.txt")):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        if line.startswith("["):
            cur = line.strip("[]")
            sections[cur] = []
            continue
        sections[cur].append(line.split())
    ids: dict = {}
    for t in sections["triples"]:
        for term in t:
            ids.setdefault(term, len(ids))
    triples = np.array([[ids[x] for x in t] for t in sections["triples"]], np.uint32)
    return ids, triples, sections


def brute_join_multiset(a_vars, a_rows, b_vars, b_rows, out_vars):
    """Join multiset from the definition of SPARQL Join over bags: every solution mapping mu over
    vars(A) ∪ vars(B) has multiplicity card_A(mu|A) * card_B(mu|B).  Enumerates all mappings
    over the values that occur, so it never pairs rows directly."""
    all_vars = list(dict.fromkeys(list(a_vars) + list(b_vars)))
    card_a = Counter(tuple(int(x) for x in r) for r in a_rows)
    card_b = Counter(tuple(int(x) for x in r) for r in b_rows)
    values = sorted({int(x) for r in list(a_rows) + list(b_rows) for x in r})
    out = Counter()
    if not values:
        return out
    for assign in itertools.product(values, repeat=len(all_vars)):
        mu = dict(zip(all_vars, assign))
        m = card_a[tuple(mu[v] for v in a_vars)] * card_b[tuple(mu[v] for v in b_vars)]
        if m:
            out[tuple(mu[v] for v in out_vars)] += m
    return out


def brute_query_multiset(triples, patterns, proj):
    """Query answer by enumerating assignments of the query variables to dictionary terms and
    checking each instantiated pattern against the triple set, then projecting
    with bag semantics."""
    tset = {tuple(int(x) for x in t) for t in triples}
    terms = sorted({int(x) for t in triples for x in t})
    qvars = list(dict.fromkeys(x for pat in patterns for kind, x in pat if kind == "v"))
    proj = list(proj) if proj else qvars
    out = Counter()
    for assign in itertools.product(terms, repeat=len(qvars)):
        mu = dict(zip(qvars, assign))
        ok = all(tuple(mu[x] if kind == "v" else x for kind, x in pat) in tset for pat in patterns)
        if ok:
            out[tuple(mu[v] for v in proj)] += 1
    return out


def rows_multiset(rows) -> Counter:
    return Counter(tuple(int(x) for x in r) for r in rows)


# ---- BASELINE.json config queries over the LUBM-shaped vocabulary ----
def _v(i):
    return ("v", i)


def _c(i):
    return ("c", i)


def config_query(name: str):
    """Patterns (textual left-deep order) of configs C1, C2, C3, C5; variables numbered in
    first-appearance order."""
    from datagen import LUBM_PRED as P
    if name == "C1":   # ?x worksFor ?d . ?d subOrganizationOf ?u
        return [(_v(0), _c(P["worksFor"]), _v(1)), (_v(1), _c(P["subOrganizationOf"]), _v(2))]
    if name == "C2":   # ?X memberOf ?Z . ?Z subOrganizationOf ?Y . ?X undergraduateDegreeFrom ?Y
        return [(_v(0), _c(P["memberOf"]), _v(1)), (_v(1), _c(P["subOrganizationOf"]), _v(2)),
                (_v(0), _c(P["undergraduateDegreeFrom"]), _v(2))]
    if name == "C3":   # ?x subOrganizationOf ?u . ?h headOf ?x . ?f worksFor ?x . ?s memberOf ?x
        return [(_v(0), _c(P["subOrganizationOf"]), _v(1)), (_v(2), _c(P["headOf"]), _v(0)),
                (_v(3), _c(P["worksFor"]), _v(0)), (_v(4), _c(P["memberOf"]), _v(0))]
    if name == "C5":   # ?x advisor ?y . ?y teacherOf ?z . ?x takesCourse ?z
        return [(_v(0), _c(P["advisor"]), _v(1)), (_v(1), _c(P["teacherOf"]), _v(2)),
                (_v(0), _c(P["takesCourse"]), _v(2))]
    raise KeyError(name)


def config_expected_counts(name: str, stats: dict) -> list:
    """Per-join |RS| from the generator's bookkeeping (independent of oracle and GPU)."""
    return {"C1": [stats["c1_rs"]], "C2": [stats["c2_j1"], stats["c2_j2"]],
            "C3": [stats["c3_j1"], stats["c3_j2"], stats["c3_j3"]],
            "C5": [stats["c5_j1"], stats["c5_j2"]]}[name]
