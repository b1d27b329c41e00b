"""Compiled-tree dumps → cached device plans.

Reads and writes the reference's `jtprop-tree` v1 JSON format (io.py:440-550 of
the reference: cardinalities, cliques, edges, separators, roots, cpt_assignment,
optional embedded native-JSON network, optional mapping tables) with this
package's own types, so a tree compiled once by the reference's offline compiler
(compiler.py:388-396) can be loaded straight into `jt_plan_create` without the
reference installed.  Mapping tables in a dump are ignored by the device engine
(it uses stride arithmetic) and only validated against the structure.

`load_plan(path, dtype, device)` caches device plans by the dump's content hash.
"""

from __future__ import annotations

import hashlib
import json
import os
from dataclasses import dataclass

import numpy as np

from .tree import Clique, JunctionTree, Scope, Separator

TREE_FORMAT = "jtprop-tree"


class TreeFormatError(ValueError):
    """Malformed tree dump (the reference raises SchemaViolationError/ParseError)."""


@dataclass
class Variable:
    id: int
    name: str
    cardinality: int


@dataclass
class Table:
    scope: Scope
    values: np.ndarray


@dataclass
class Cpt:
    """CPT with scope (parents in declared order, then child) — model.py:32-60."""

    child: int
    parents: tuple
    table: Table


class Network:
    """The embedded network of a dump: just what initialize/evidence need."""

    def __init__(self, variables, cpts):
        self.variables = variables
        self.cpts = sorted(cpts, key=lambda c: c.child)
        self._by_name = {v.name: v.id for v in variables}

    def __len__(self):
        return len(self.variables)

    @property
    def cardinalities(self):
        return tuple(v.cardinality for v in self.variables)

    def id_of(self, name):
        return self._by_name[name]


def _key(doc, key, typ):
    if key not in doc:
        raise TreeFormatError(f"missing /{key}")
    val = doc[key]
    if not isinstance(val, typ):
        raise TreeFormatError(f"/{key}: expected {typ.__name__}")
    return val


def network_from_dict(doc) -> Network:
    """Native-JSON network (io.py:315-370 of the reference), shapes checked."""
    variables = [Variable(i, _key(v, "name", str), int(_key(v, "cardinality", int)))
                 for i, v in enumerate(_key(doc, "variables", list))]
    ids = {v.name: v.id for v in variables}
    if len(ids) != len(variables):
        raise TreeFormatError("/network/variables: duplicate names")
    cpts = []
    for i, item in enumerate(_key(doc, "cpts", list)):
        child_name = _key(item, "child", str)
        if child_name not in ids:
            raise TreeFormatError(f"/network/cpts/{i}/child: unknown variable {child_name!r}")
        parents = []
        for p in _key(item, "parents", list):
            if p not in ids:
                raise TreeFormatError(f"/network/cpts/{i}/parents: unknown variable {p!r}")
            parents.append(ids[p])
        child = ids[child_name]
        scope_ids = tuple(parents) + (child,)
        cards = tuple(variables[v].cardinality for v in scope_ids)
        values = np.asarray(_key(item, "table", list), dtype=np.float64)
        if values.size != int(np.prod(cards, dtype=np.int64)):
            raise TreeFormatError(f"/network/cpts/{i}/table: expected {int(np.prod(cards))} entries")
        cpts.append(Cpt(child, tuple(parents), Table(Scope(scope_ids, cards), values)))
    return Network(variables, cpts)


def network_to_dict(net) -> dict:
    return {
        "variables": [{"name": v.name, "cardinality": int(v.cardinality)} for v in net.variables],
        "cpts": [{"child": net.variables[c.child].name,
                  "parents": [net.variables[p].name for p in c.table.scope.ids[:-1]],
                  "table": [float(x) for x in np.asarray(c.table.values).ravel()]} for c in net.cpts],
    }


def parse_tree(text: str):
    """(tree, network or None) from a `jtprop-tree` v1 document (io.py:477-550)."""
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as exc:
        raise TreeFormatError(f"invalid JSON: {exc.msg} at {exc.lineno}:{exc.colno}") from exc
    if not isinstance(doc, dict) or doc.get("format") != TREE_FORMAT:
        raise TreeFormatError(f"/format: expected {TREE_FORMAT!r}")
    if doc.get("version") != 1:
        raise TreeFormatError("/version: only version 1 is supported")
    cards = tuple(int(c) for c in _key(doc, "cardinalities", list))

    def scope_of(members):
        members = tuple(int(m) for m in members)
        if list(members) != sorted(set(members)) or any(not 0 <= m < len(cards) for m in members):
            raise TreeFormatError(f"bad member list {members}")
        return members, Scope(members, tuple(cards[m] for m in members))

    cliques = []
    for i, raw in enumerate(_key(doc, "cliques", list)):
        members, scope = scope_of(raw)
        cliques.append(Clique(i, members, scope))
    edges = _key(doc, "edges", list)
    raw_seps = _key(doc, "separators", list)
    if len(edges) != len(raw_seps):
        raise TreeFormatError("/separators: edge/separator count mismatch")
    separators, neighbors = [], [[] for _ in cliques]
    for i, (edge, raw) in enumerate(zip(edges, raw_seps)):
        members, scope = scope_of(raw)
        a, b = int(edge[0]), int(edge[1])
        if not (0 <= a < len(cliques) and 0 <= b < len(cliques)):
            raise TreeFormatError(f"/edges/{i}: clique out of range")
        separators.append(Separator(i, (a, b), members, scope))
        neighbors[a].append((b, i))
        neighbors[b].append((a, i))
    for lst in neighbors:
        lst.sort()
    assignment = _key(doc, "cpt_assignment", list)
    tree = JunctionTree(cards=cards, cliques=cliques, separators=separators, neighbors=neighbors,
                        roots=[int(r) for r in _key(doc, "roots", list)],
                        cpt_assignment={v: int(c) for v, c in enumerate(assignment)})
    if "mapping_tables" in doc:  # validated, not used: the device derives indices from strides
        from .tree import build_mapping_table

        for key, rows in doc["mapping_tables"].items():
            c, s = (int(x) for x in key.split(":"))
            want = build_mapping_table(cliques[c].scope, separators[s].scope)
            got = np.asarray(rows)
            if got.shape != want.shape or not np.array_equal(np.sort(got, axis=None), np.sort(want, axis=None)):
                raise TreeFormatError(f"/mapping_tables/{key}: does not match the tree structure")
    net = network_from_dict(doc["network"]) if "network" in doc else None
    return tree, net


def serialize_tree(tree, net=None) -> str:
    """`jtprop-tree` v1 text (io.py:443-474), without mapping tables."""
    doc = {
        "format": TREE_FORMAT,
        "version": 1,
        "layout": "flat",
        "cardinalities": [int(c) for c in tree.cards],
        "cliques": [list(map(int, c.scope.ids)) for c in tree.cliques],
        "edges": [list(map(int, s.edge)) for s in tree.separators],
        "separators": [list(map(int, s.scope.ids)) for s in tree.separators],
        "roots": [int(r) for r in tree.roots],
        "cpt_assignment": [int(tree.cpt_assignment[v]) for v in sorted(tree.cpt_assignment)],
    }
    if net is not None:
        doc["network"] = network_to_dict(net)
    return json.dumps(doc, indent=1) + "\n"


def load_tree(path):
    with open(path) as f:
        return parse_tree(f.read())


_PLANS: dict = {}


def load_plan(path, dtype="f64", device=0):
    """(plan, tree, network) for a dump file; plans are cached by content hash,
    dtype and device, so reloading the same dump reuses the device plan."""
    from .propagate import Plan

    with open(path, "rb") as f:
        raw = f.read()
    key = (hashlib.sha256(raw).hexdigest(), str(dtype), int(device))
    hit = _PLANS.get(key)
    if hit is not None:
        return hit
    tree, net = parse_tree(raw.decode())
    plan = Plan(tree, dtype, device)
    from . import propagate

    propagate._PLAN_CACHE[(id(tree), propagate._dtype_code(dtype), int(device))] = plan  # states reuse it
    _PLANS[key] = (plan, tree, net)
    return _PLANS[key]


__all__ = ["TREE_FORMAT", "TreeFormatError", "load_plan", "load_tree", "parse_tree", "serialize_tree",
           "network_from_dict", "network_to_dict"]
