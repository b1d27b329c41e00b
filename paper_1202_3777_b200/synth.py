"""Synthetic inputs for the BASELINE.json configs.

Trees are grown so the running-intersection property holds by construction
(clique c = a random earlier clique minus d variables plus f fresh ones) and
then assembled with `build_tree` (the reference's Kruskal contract,
compiler.py:187-246).  Potentials are uniform(0.1, 1) per clique in id order
(the reference generator's draw, synth.py:105-107) rescaled so each clique sums
to the size of its parent separator (root: 1), which keeps fp32 in range
(SURVEY.md Appendix B).  Evidence cases follow §8d: k ~ U{1..8} distinct
variables, states uniform, owning clique = smallest holder (ties → lowest id).

These are input generators only; nothing here computes on the hot path.
"""

from __future__ import annotations

from collections import deque

import numpy as np

from .tree import build_tree

CONFIGS = ("c1", "c2", "c3", "c4B", "c4M", "c5")


def grow_jt(n, seed, w0, wmin, wmax, card_fn, d_fn, f_fn, max_table):
    rng = np.random.default_rng(seed)
    cards, members = [], []

    def new(k):
        return [int(card_fn(rng)) for _ in range(k)]

    c0 = new(w0)
    while np.prod(c0, dtype=np.int64) > max_table:
        c0 = new(w0)
    cards += c0
    members.append(list(range(w0)))
    for c in range(1, n):
        for _ in range(1000):
            p = int(rng.integers(0, c))
            P = members[p]
            d = int(min(max(1, d_fn(rng)), len(P) - 1)) if len(P) > 1 else 0
            f = int(max(1, f_fn(rng)))
            w = len(P) - d + f
            if w > wmax:
                d = min(len(P) - 1, d + (w - wmax))
                w = len(P) - d + f
            if w < wmin:
                f += wmin - w
                w = wmin
            S = sorted(rng.choice(P, size=len(P) - d, replace=False).tolist()) \
                if len(P) - d > 0 else []
            fc = new(f)
            if np.prod([cards[v] for v in S] + fc, dtype=np.int64) <= max_table:
                break
        base = len(cards)
        cards += fc
        members.append(sorted(S + list(range(base, base + f))))
    return [tuple(m) for m in members], tuple(cards)


def _choice(vals, probs):
    vals = np.asarray(vals)
    p = np.asarray(probs, dtype=float)
    p = p / p.sum()
    return lambda r: r.choice(vals, p=p)


def config_members(name):
    """(clique member tuples, cardinalities) for one BASELINE config."""
    if name == "c1":
        return grow_jt(12, 1, 5, 3, 6, lambda r: 3, lambda r: r.integers(1, 3),
                       lambda r: r.integers(1, 3), 3 ** 6)
    if name == "c2":
        return grow_jt(368, 2, 6, 3, 11, lambda r: 3,
                       lambda r: 1 if r.uniform() < .85 else 2,
                       lambda r: 1 if r.uniform() < .82 else 2, 3 ** 11)
    if name == "c4B":
        return grow_jt(36, 4, 5, 3, 6, _choice([2, 3, 4, 5, 8, 16, 32, 64], [.15] * 4 + [.1] * 4),
                       lambda r: 1, lambda r: 1, 7_257_600)
    if name == "c4M":
        return grow_jt(870, 5, 4, 2, 5, _choice([2, 3, 4, 5, 8, 16, 32, 64], [.15] * 4 + [.1] * 4),
                       lambda r: 1 if r.uniform() < .85 else 2, lambda r: 1, 784_000)
    if name == "c5":
        return grow_jt(28, 6, 5, 3, 6,
                       _choice([2, 3, 4, 5, 7, 10, 20, 50, 100], [.12] * 5 + [.1] * 4),
                       lambda r: 1, lambda r: 1, 4_372_480)
    if name == "c3":
        return ([tuple(range(0, 12)), tuple(range(6, 18)),
                 (13, 15, 17) + tuple(range(18, 27)),
                 tuple(range(0, 6)) + tuple(range(27, 33))], (4,) * 33)
    raise ValueError(f"unknown config {name!r}; use one of {CONFIGS}")


def smallest_holder(tree, var):
    best = None
    for c in tree.cliques:
        if var in c.members:
            key = (c.scope.size, c.id)
            if best is None or key < best[0]:
                best = (key, c.id)
    return None if best is None else best[1]


def bfs_parents(tree):
    """Parent clique per clique (−1 for roots), BFS from every root."""
    parent = [-1] * len(tree.cliques)
    seen = set(tree.roots)
    q = deque(tree.roots)
    while q:
        c = q.popleft()
        for nbr, sid in tree.neighbors[c]:
            if nbr not in seen:
                seen.add(nbr)
                parent[nbr] = (c, sid)
                q.append(nbr)
    return parent


def scaled_potentials(tree, seed=0):
    """uniform(0.1,1) per clique in id order, scaled so clique c sums to the size
    of the separator to its BFS parent (roots sum to 1)."""
    rng = np.random.default_rng(seed)
    parent = bfs_parents(tree)
    tables = []
    for c in tree.cliques:
        t = rng.uniform(0.1, 1.0, size=c.scope.size)
        target = 1.0 if parent[c.id] == -1 else float(tree.separators[parent[c.id][1]].scope.size)
        t *= target / t.sum()
        tables.append(t)
    return tables


def make_config(name, seed=0):
    """(tree, clique tables) for config `name`; cpt_assignment[v] = smallest
    holder so evidence can be entered on every variable."""
    members, cards = config_members(name)
    tree = build_tree(members, cards)
    tree.cpt_assignment = {v: smallest_holder(tree, v) for v in range(len(cards))
                           if smallest_holder(tree, v) is not None}
    return tree, scaled_potentials(tree, seed)


def evidence_cases(tree, n_cases, seed=1234, kmax=8, first=0):
    """Case i: k ~ U{1..kmax} distinct variables with uniform states.  Cases are
    drawn from one stream so a shard [first, first+n) is reproducible without
    generating the others' evidence (each case uses its own child stream)."""
    n_vars = len(tree.cards)
    out = []
    for i in range(first, first + n_cases):
        rng = np.random.default_rng([seed, i])
        k = int(rng.integers(1, kmax + 1))
        vars_ = rng.choice(n_vars, size=min(k, n_vars), replace=False)
        out.append({int(v): int(rng.integers(0, tree.cards[v])) for v in sorted(vars_)})
    return out
