"""CLUTRR-style kinship workload of BASELINE configs[3]: the relation alphabet, a 20 x 20
composition rule table and the two symbol functions of the closure (pure Python, no
imports from the package, so the reference CPU arm can load this file on its own and
run the SAME black-box functions through the reference API)."""

from __future__ import annotations

from collections import namedtuple

__all__ = ["Fact", "KINSHIP_RELATIONS", "compose_with", "chain_link"]

Fact = namedtuple("Fact", ["x", "y", "rel"])

KINSHIP_RELATIONS = (
    "father", "mother", "son", "daughter", "brother", "sister", "husband", "wife",
    "grandfather", "grandmother", "grandson", "granddaughter", "uncle", "aunt",
    "nephew", "niece", "father-in-law", "mother-in-law", "son-in-law", "daughter-in-law",
)

_GENDER = {
    "father": "m", "mother": "f", "son": "m", "daughter": "f", "brother": "m", "sister": "f",
    "husband": "m", "wife": "f", "grandfather": "m", "grandmother": "f", "grandson": "m",
    "granddaughter": "f", "uncle": "m", "aunt": "f", "nephew": "m", "niece": "f",
    "father-in-law": "m", "mother-in-law": "f", "son-in-law": "m", "daughter-in-law": "f",
}


def _by_gender(rel, male, female):
    return male if _GENDER[rel] == "m" else female


def _kinship_table():
    """(r1, r2) -> r for "x r1 y, y r2 z => x r z" (z's relation to... read as: y is x's r1,
    z is y's r2, so z is x's r).  A deterministic 20x20 rule table in the spirit of the
    CLUTRR composition rules; combinations with no rule are UNDEFINED."""
    t = {}
    parent = ("father", "mother")
    child = ("son", "daughter")
    sibling = ("brother", "sister")
    spouse = ("husband", "wife")
    grandparent = ("grandfather", "grandmother")
    grandchild = ("grandson", "granddaughter")
    uncle_aunt = ("uncle", "aunt")
    child_in_law = ("son-in-law", "daughter-in-law")
    parent_in_law = ("father-in-law", "mother-in-law")
    rules = [
        (parent, parent, lambda r2: _by_gender(r2, "grandfather", "grandmother")),
        (parent, sibling, lambda r2: _by_gender(r2, "uncle", "aunt")),
        (parent, spouse, lambda r2: _by_gender(r2, "father", "mother")),
        (child, child, lambda r2: _by_gender(r2, "grandson", "granddaughter")),
        (child, sibling, lambda r2: _by_gender(r2, "son", "daughter")),
        (child, spouse, lambda r2: _by_gender(r2, "son-in-law", "daughter-in-law")),
        (sibling, child, lambda r2: _by_gender(r2, "nephew", "niece")),
        (sibling, parent, lambda r2: r2),
        (sibling, sibling, lambda r2: r2),
        (spouse, child, lambda r2: r2),
        (spouse, parent, lambda r2: _by_gender(r2, "father-in-law", "mother-in-law")),
        (uncle_aunt, spouse, lambda r2: _by_gender(r2, "uncle", "aunt")),
        (grandparent, spouse, lambda r2: _by_gender(r2, "grandfather", "grandmother")),
        (grandchild, sibling, lambda r2: _by_gender(r2, "grandson", "granddaughter")),
        (child_in_law, child, lambda r2: _by_gender(r2, "grandson", "granddaughter")),
        (parent_in_law, spouse, lambda r2: _by_gender(r2, "father-in-law", "mother-in-law")),
    ]
    for left, right, rule in rules:
        for r1 in left:
            for r2 in right:
                t[(r1, r2)] = rule(r2)
    return t


_KINSHIP = _kinship_table()


def compose_with(undefined):
    """Compose two facts sharing the middle entity; ``undefined`` when no rule applies."""

    def compose(f1, f2):
        rel = _KINSHIP.get((f1.rel, f2.rel))
        return undefined if rel is None else Fact(f1.x, f2.y, rel)

    return compose


def chain_link(f1, f2):
    """cond of the closure: f1's object is f2's subject, and no self-relation results."""
    return f1.y == f2.x and f1.x != f2.y


def story_facts(n_entities, rels=KINSHIP_RELATIONS):
    """Every relation candidate on the chain of entities 0 - 1 - ... - (n-1)."""
    return [Fact(i, i + 1, r) for i in range(n_entities - 1) for r in rels]
