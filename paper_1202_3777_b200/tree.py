"""Junction-tree input types, duck-compatible with the reference's.

The engine consumes a compiled junction tree; it does not rebuild the
reference's compiler (moralize/triangulate/cliques, compiler.py:89-184 is out
of scope).  These types mirror the reference's data model field for field so
that either the reference's own `JunctionTree` (compiler.py:40-80) or one built
here can be handed to the engine:

* `Scope`            potential.py:24-66   (ids, cards, size, strides, position)
* `Clique`           compiler.py:25-29
* `Separator`        compiler.py:32-37
* `JunctionTree`     compiler.py:40-80
* `build_tree`       compiler.py:187-246  (Kruskal max-spanning tree; the
                     synthetic configs are assembled with it, exactly as the
                     survey's Appendix A recipe does with the reference)
* `build_mapping_table(s)` compiler.py:270-339 (host μ tables, used only by the
                     engine-protocol plugin path and for inspection; the device
                     engine uses stride arithmetic instead)
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import ScopeNotContainedError

FLAT = "flat"
INTERLEAVED = "interleaved"


@dataclass(frozen=True)
class Scope:
    """Ordered variable ids with cardinalities; last variable varies fastest."""

    ids: tuple
    cards: tuple

    def __post_init__(self):
        if len(self.ids) != len(self.cards):
            raise ValueError("ids and cards must have equal length")
        if len(set(self.ids)) != len(self.ids):
            raise ValueError(f"duplicate variable ids in scope {self.ids}")
        object.__setattr__(self, "ids", tuple(int(i) for i in self.ids))
        object.__setattr__(self, "cards", tuple(int(c) for c in self.cards))

    def __len__(self):
        return len(self.ids)

    @property
    def size(self) -> int:
        n = 1
        for c in self.cards:
            n *= c
        return n

    def strides(self) -> tuple:
        out = [1] * len(self.cards)
        for i in range(len(self.cards) - 2, -1, -1):
            out[i] = out[i + 1] * self.cards[i + 1]
        return tuple(out)

    def position(self, var_id: int) -> int:
        try:
            return self.ids.index(var_id)
        except ValueError:
            raise ScopeNotContainedError(
                f"variable {var_id} not in scope {self.ids}") from None

    def contains(self, other) -> bool:
        return set(other.ids) <= set(self.ids)


@dataclass(frozen=True)
class Clique:
    id: int
    members: tuple
    scope: Scope


@dataclass(frozen=True)
class Separator:
    id: int
    edge: tuple
    members: tuple
    scope: Scope


@dataclass
class JunctionTree:
    cards: tuple
    cliques: list
    separators: list
    neighbors: list
    roots: list
    cpt_assignment: dict = field(default_factory=dict)

    def __len__(self):
        return len(self.cliques)

    def clique_sizes(self):
        return [c.scope.size for c in self.cliques]

    def separator_sizes(self):
        return [s.scope.size for s in self.separators]

    def components(self):
        return tree_components(self)


def tree_components(tree) -> list:
    """Clique ids per connected component, one sorted list per root
    (compiler.py:65-80)."""
    seen = set()
    out = []
    for root in tree.roots:
        comp = []
        stack = [root]
        while stack:
            c = stack.pop()
            if c in seen:
                continue
            seen.add(c)
            comp.append(c)
            stack.extend(n for n, _ in tree.neighbors[c])
        out.append(sorted(comp))
    return out


def _scope_of(members, cards) -> Scope:
    return Scope(tuple(members), tuple(cards[m] for m in members))


def build_tree(clique_members, cards, cpt_assignment=None) -> JunctionTree:
    """Maximum-weight spanning forest over |shared variables| (Kruskal, ties to
    the lower (i, k) pair); root per component = largest table, ties to the
    lowest id.  Same contract as compiler.py:187-246."""
    members = [tuple(sorted(int(v) for v in m)) for m in clique_members]
    cliques = [Clique(i, m, _scope_of(m, cards)) for i, m in enumerate(members)]
    n = len(cliques)
    sets = [set(m) for m in members]
    # candidate edges sorted by (-|shared|, i, k); bucketed by variable so that
    # large sparse trees (c4M: 870 cliques) do not pay an O(n^2) set scan
    holders: dict = {}
    for i, m in enumerate(members):
        for v in m:
            holders.setdefault(v, []).append(i)
    pairs = set()
    for hs in holders.values():
        for a in range(len(hs)):
            for b in range(a + 1, len(hs)):
                pairs.add((hs[a], hs[b]))
    candidates = []
    for i, k in pairs:
        shared = tuple(sorted(sets[i] & sets[k]))
        candidates.append((-len(shared), i, k, shared))
    candidates.sort()

    parent = list(range(n))

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    separators = []
    neighbors = [[] for _ in range(n)]
    for _, i, k, shared in candidates:
        ri, rk = find(i), find(k)
        if ri == rk:
            continue
        parent[ri] = rk
        sep = Separator(len(separators), (i, k), shared, _scope_of(shared, cards))
        separators.append(sep)
        neighbors[i].append((k, sep.id))
        neighbors[k].append((i, sep.id))
    for lst in neighbors:
        lst.sort()

    by_component: dict = {}
    for c in range(n):
        by_component.setdefault(find(c), []).append(c)
    roots = sorted(max(comp, key=lambda c: (cliques[c].scope.size, -c))
                   for comp in by_component.values())
    return JunctionTree(tuple(int(c) for c in cards), cliques, separators,
                        neighbors, roots, dict(cpt_assignment or {}))


# --- host mapping tables (compiler.py:270-350) -------------------------------

def _index_offsets(scope, positions) -> np.ndarray:
    strides = scope.strides()
    offsets = np.zeros(1, dtype=np.int64)
    for pos in positions:
        step = np.arange(scope.cards[pos], dtype=np.int64) * strides[pos]
        offsets = (offsets[:, None] + step[None, :]).ravel()
    return offsets


def build_mapping_table(clique_scope, sep_scope, dtype=None) -> np.ndarray:
    """μ[j][p] = row_base[j] + rest[p] (compiler.py:285-304)."""
    sep_pos = [clique_scope.position(v) for v in sep_scope.ids]
    rest_pos = [p for p in range(len(clique_scope)) if p not in sep_pos]
    table = _index_offsets(clique_scope, sep_pos)[:, None] + \
        _index_offsets(clique_scope, rest_pos)[None, :]
    if dtype is None:
        dtype = np.int32 if clique_scope.size <= np.iinfo(np.int32).max else np.int64
    return np.ascontiguousarray(table, dtype=dtype)


@dataclass
class MappingTableSet:
    layout: str
    tables: dict = field(default_factory=dict)

    def mu(self, clique_id, sep_id):
        return self.tables[(clique_id, sep_id)]

    def physical(self, clique_id, sep_id):
        order = "F" if self.layout == INTERLEAVED else "C"
        return self.tables[(clique_id, sep_id)].ravel(order=order)


def build_mapping_tables(tree, layout=FLAT) -> MappingTableSet:
    if layout not in (FLAT, INTERLEAVED):
        raise ValueError(f"unknown layout {layout!r}")
    out = MappingTableSet(layout=layout)
    for sep in tree.separators:
        for cid in sep.edge:
            t = build_mapping_table(tree.cliques[cid].scope, sep.scope)
            out.tables[(cid, sep.id)] = np.asfortranarray(t) if layout == INTERLEAVED else t
    return out


def relayout_mapping_tables(mapping, layout) -> MappingTableSet:
    if layout not in (FLAT, INTERLEAVED):
        raise ValueError(f"unknown layout {layout!r}")
    conv = np.asfortranarray if layout == INTERLEAVED else np.ascontiguousarray
    return MappingTableSet(layout, {k: conv(t) for k, t in mapping.tables.items()})


def directed_messages(tree):
    """Every (separator id, source clique id) pair (perfmodel.py:60-64)."""
    for sep in tree.separators:
        yield sep.id, sep.edge[0]
        yield sep.id, sep.edge[1]


def algorithmic_elements(tree) -> int:
    """Σ over the 2(n−1) directed messages of |φ_src| + 2|φ_tgt| + 2|φ_sep|:
    the elements Alg. 1 must touch per propagation (B_alg1/b)."""
    total = 0
    for sid, src in directed_messages(tree):
        sep = tree.separators[sid]
        tgt = sep.edge[1] if src == sep.edge[0] else sep.edge[0]
        total += tree.cliques[src].scope.size + 2 * tree.cliques[tgt].scope.size \
            + 2 * sep.scope.size
    return total
