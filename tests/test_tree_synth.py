"""Host-side inputs: tree assembly and config generators match the reference's."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, have_reference, load_golden
from paper_1202_3777_b200 import synth
from paper_1202_3777_b200.tree import algorithmic_elements, build_mapping_table, build_tree, Scope

# Σ|φ| and B_alg1 element counts from SURVEY.md §8d
SURVEY = {"c1": (6642, 42498), "c2": (538380, 3541662), "c3": (67108864, 302022912),
          "c4B": (30522496, 144336000), "c4M": (3629893, 22483447), "c5": (8026240, 45620160)}


@pytest.mark.parametrize("name", sorted(SURVEY))
def test_config_tree_matches_reference_golden(name):
    members, cards = synth.config_members(name)
    tree = build_tree(members, cards)
    with open(os.path.join(GOLDEN, f"{name}_tree.json")) as f:
        doc = json.load(f)
    assert [list(c.members) for c in tree.cliques] == doc["cliques"]
    assert [[list(s.edge), list(s.members)] for s in tree.separators] == doc["separators"]
    assert tree.roots == doc["roots"]
    assert sum(tree.clique_sizes()) == SURVEY[name][0]
    assert algorithmic_elements(tree) == SURVEY[name][1]


@pytest.mark.parametrize("name", ["c1", "c2", "c5"])
def test_scaled_potentials_reproducible(name):
    tree, data = load_golden(name)
    tables = synth.scaled_potentials(tree, seed=0)
    want = data["tables_checksum"]
    got = np.array([float(np.sum(t)) for t in tables] + [float(np.sum(t * np.arange(t.size) % 7)) for t in tables])
    assert np.array_equal(got, want)


def test_evidence_cases_shardable():
    tree, _ = load_golden("c5")
    full = synth.evidence_cases(tree, 16)
    assert synth.evidence_cases(tree, 6, first=10) == full[10:]
    for ev in full:
        assert 1 <= len(ev) <= 8
        for v, x in ev.items():
            assert 0 <= x < tree.cards[v]


def test_host_mapping_table_matches_golden():
    data = np.load(os.path.join(GOLDEN, "mapping_tables.npz"))
    for i in range(80):
        ids, cards = tuple(data[f"case{i}_ids"]), tuple(data[f"case{i}_cards"])
        sep = tuple(data[f"case{i}_sep"])
        sc = Scope(sep, tuple(cards[list(ids).index(v)] for v in sep))
        assert np.array_equal(build_mapping_table(Scope(ids, cards), sc), data[f"case{i}_mu"])


@pytest.mark.skipif(not have_reference(), reason="reference not mounted")
def test_build_tree_matches_reference_on_random_members():
    import sys
    sys.path.insert(0, "/root/reference/pkg/src")
    from jtprop.compiler import build_tree as rbuild

    rng = np.random.default_rng(5)
    for k in range(20):
        n = int(rng.integers(2, 30))
        members = [tuple(sorted(rng.choice(12, size=int(rng.integers(1, 5)), replace=False).tolist()))
                   for _ in range(n)]
        cards = tuple(int(c) for c in rng.integers(2, 4, size=12))
        a, b = build_tree(members, cards), rbuild(members, cards)
        assert [(s.edge, s.members) for s in a.separators] == [(s.edge, s.members) for s in b.separators]
        assert a.roots == b.roots and a.neighbors == b.neighbors
