"""Pin the CPU oracle (oracle/jtref.py) to the reference before trusting it.

* Known-answer tests restated from the reference's own suite
  (test_propagate.py:53-89, test_compiler.py:201-218, 260-264).
* Golden vectors produced by running the reference (tests/golden/make_golden.py):
  μ tables on random scope pairs (bit-exact), full BP posteriors on the config
  trees with and without evidence, corpus networks with CPT-initialized tables.
* When /root/reference is present, a live cross-check on fresh random inputs.
"""

import numpy as np
import pytest

from conftest import golden_cases, have_reference, load_corpus, load_golden
from oracle import jtref
from paper_1202_3777_b200 import synth
from paper_1202_3777_b200.tree import build_tree


def demo(src=None):
    tree = build_tree([(0, 1, 3), (1, 2)], (2, 2, 2, 2))
    tables = [np.arange(8.0) if src is None else np.asarray(src, float), np.ones(4)]
    return tree, jtref.from_potentials(tree, tables)


class TestKnownAnswers:
    def test_worked_example(self):  # test_propagate.py:54-59
        tree, st = demo()
        jtref.message_passing(st, 0, 1, 0)
        assert st.sep_values[0].tolist() == [10.0, 18.0]
        assert st.clique_values[1].tolist() == [10.0, 10.0, 18.0, 18.0]
        assert st.clique_values[0].tolist() == list(range(8))

    def test_zero_over_zero(self):  # test_propagate.py:61-68
        tree, st = demo([0, 0, 1, 2, 0, 0, 3, 4])
        st.sep_values[0][:] = [0.0, 1.0]
        st.clique_values[1][:] = [5.0, 6.0, 7.0, 8.0]
        jtref.message_passing(st, 0, 1, 0)
        assert st.clique_values[1].tolist() == [0.0, 0.0, 70.0, 80.0]
        assert st.sep_values[0].tolist() == [0.0, 10.0]

    def test_nonzero_over_zero(self):  # test_propagate.py:70-74
        tree, st = demo()
        st.sep_values[0][:] = [0.0, 1.0]
        with pytest.raises(jtref.InconsistentDivision):
            jtref.message_passing(st, 0, 1, 0)

    def test_fixed_point(self):  # test_propagate.py:76-81
        tree, st = demo(np.ones(8))
        st.sep_values[0][:] = [4.0, 4.0]
        before = st.clique_values[1].copy()
        jtref.message_passing(st, 0, 1, 0)
        assert np.array_equal(st.clique_values[1], before)

    def test_figure2_mapping_tables(self):  # test_compiler.py:201-209
        assert jtref.build_mapping_table((0, 1, 3), (2, 2, 2), (1,)).tolist() == [[0, 1, 4, 5], [2, 3, 6, 7]]
        assert jtref.build_mapping_table((1, 2), (2, 2), (1,)).tolist() == [[0, 1], [2, 3]]
        mu = jtref.build_mapping_table((0, 1, 3), (2, 2, 2), (1,))
        assert np.asfortranarray(mu).ravel(order="F").tolist() == [0, 2, 1, 3, 4, 6, 5, 7]

    def test_identity_when_separator_is_clique(self):  # test_compiler.py:211-218
        assert jtref.build_mapping_table((0, 1), (2, 2), (0, 1)).tolist() == [[0], [1], [2], [3]]

    def test_int32_dtype(self):  # test_compiler.py:351-354
        assert jtref.build_mapping_table((0, 1), (2, 3), (1,)).dtype == np.int32


def test_mapping_tables_bit_exact_vs_reference_golden():
    data = np.load(__import__("os").path.join(__import__("conftest").GOLDEN, "mapping_tables.npz"))
    i = 0
    while f"case{i}_mu" in data:
        mu = jtref.build_mapping_table(data[f"case{i}_ids"], data[f"case{i}_cards"], data[f"case{i}_sep"])
        assert mu.dtype == data[f"case{i}_mu"].dtype
        assert np.array_equal(mu, data[f"case{i}_mu"]), i
        i += 1
    assert i == 80


@pytest.mark.parametrize("name", ["c1", "c2", "c5", "c4M"])
def test_oracle_posteriors_match_reference_golden(name):
    tree, data = load_golden(name)
    tables = synth.scaled_potentials(tree, seed=0)
    template = jtref.from_potentials(tree, tables)
    for ev, want in golden_cases(data):
        got = jtref.case_posteriors(template, ev, range(len(tree.cards)))
        # same numpy operations in the same order as the reference: bit-identical
        assert np.array_equal(got, want), (name, ev)


def test_oracle_final_tables_match_reference_c1():
    tree, data = load_golden("c1")
    st = jtref.from_potentials(tree, synth.scaled_potentials(tree, seed=0))
    jtref.belief_propagation(st)
    assert np.array_equal(np.concatenate(st.clique_values), data["cliques0"])
    assert np.array_equal(np.concatenate(st.sep_values), data["sep0"])


def test_oracle_corpus_matches_reference_golden():
    for name, tree, tables, post, cliques, seps in load_corpus():
        st = jtref.from_potentials(tree, tables)
        jtref.apply_evidence(st, {0: 0})
        jtref.belief_propagation(st)
        got = jtref.posteriors(st, range(len(tree.cards)))
        assert np.array_equal(got, post), name
        assert np.array_equal(np.concatenate(st.clique_values), cliques), name


def test_parallel_engine_bit_identical():  # test_acceptance.py C3 restated on the oracle
    tree, data = load_golden("c2")
    tables = synth.scaled_potentials(tree, seed=0)
    a = jtref.from_potentials(tree, tables)
    b = jtref.from_potentials(tree, tables, engine=jtref.ParallelEngine(4, small_message_threshold=0))
    jtref.belief_propagation(a)
    jtref.belief_propagation(b)
    b.engine.close()
    for x, y in zip(a.clique_values, b.clique_values):
        assert np.array_equal(x, y)


@pytest.mark.skipif(not have_reference(), reason="reference not mounted")
def test_oracle_live_vs_reference_random_trees():
    import sys

    sys.path.insert(0, "/root/reference/pkg/src")
    from jtprop.compiler import build_tree as rbuild
    from jtprop.propagate import apply_evidence, belief_propagation, from_potentials, query_marginal

    rng = np.random.default_rng(77)
    for seed in range(6):
        members, cards = synth.grow_jt(int(rng.integers(3, 14)), 100 + seed, 4, 2, 5,
                                       lambda r: int(r.integers(2, 5)), lambda r: 1, lambda r: 1, 4000)
        rt = rbuild(members, cards)
        mt = build_tree(members, cards)
        tables = [rng.uniform(0.1, 1.0, size=c.scope.size) for c in mt.cliques]
        owner = {v: synth.smallest_holder(mt, v) for v in range(len(cards))}
        rt.cpt_assignment = dict(owner)
        ev = {int(v): int(rng.integers(0, cards[v])) for v in rng.choice(len(cards), 2, replace=False)}
        rs = from_potentials(rt, tables)
        apply_evidence(rs, ev)
        belief_propagation(rs)
        want = np.concatenate([query_marginal(rs, v).values for v in range(len(cards))])
        os_ = jtref.from_potentials(mt, tables)
        got = jtref.case_posteriors(os_, ev, range(len(cards)), owner)
        assert np.array_equal(got, want)
