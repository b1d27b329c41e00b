"""`jtprop-tree` v1 dumps (reference io.py:440-550) parsed without the reference:
the fixtures were written by the reference's serialize_tree (make_golden.py)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_corpus_networks
from paper_1202_3777_b200 import io


def corpus_tree_doc(k):
    with open(os.path.join(GOLDEN, "corpus.json")) as f:
        return json.load(f)[k]["tree"]


@pytest.mark.parametrize("k", [3, 5])
def test_reference_dump_parses_to_the_same_tree(k):
    tree, net = io.load_tree(os.path.join(GOLDEN, f"tree_dump{k}.jt.json"))
    want = corpus_tree_doc(k)
    assert list(tree.cards) == want["cards"]
    assert [list(c.scope.ids) for c in tree.cliques] == want["cliques"]
    assert [[list(s.edge), list(s.scope.ids)] for s in tree.separators] == want["separators"]
    assert tree.roots == want["roots"]
    assert {str(a): b for a, b in tree.cpt_assignment.items()} == want["cpt_assignment"]
    # embedded network: same CPT values as the reference's network
    _, _, gnet, _, _, _ = load_corpus_networks()[k]
    assert len(net) == len(gnet)
    for a, b in zip(net.cpts, gnet.cpts):
        assert a.child == b.child and tuple(a.table.scope.ids) == tuple(b.table.scope.ids)
        assert np.array_equal(a.table.values, b.table.values)


def test_roundtrip():
    tree, net = io.load_tree(os.path.join(GOLDEN, "tree_dump3.jt.json"))
    tree2, net2 = io.parse_tree(io.serialize_tree(tree, net))
    assert [c.scope for c in tree2.cliques] == [c.scope for c in tree.cliques]
    assert [s.edge for s in tree2.separators] == [s.edge for s in tree.separators]
    assert tree2.cpt_assignment == tree.cpt_assignment
    assert all(np.array_equal(a.table.values, b.table.values) for a, b in zip(net.cpts, net2.cpts))


@pytest.mark.parametrize("bad", [
    "not json", '{"format": "other"}', '{"format": "jtprop-tree", "version": 2}',
    '{"format": "jtprop-tree", "version": 1, "cardinalities": [2], "cliques": [[0]], "edges": [[0, 1]], '
    '"separators": [], "roots": [0], "cpt_assignment": [0]}',
])
def test_malformed_dumps_raise(bad):
    with pytest.raises(io.TreeFormatError):
        io.parse_tree(bad)


def test_mapping_tables_validated():
    text = open(os.path.join(GOLDEN, "tree_dump5.jt.json")).read()
    doc = json.loads(text)
    key = next(iter(doc["mapping_tables"]))
    doc["mapping_tables"][key][0][0] += 1  # corrupt one index
    with pytest.raises(io.TreeFormatError):
        io.parse_tree(json.dumps(doc))
