"""Randomised shapes against the oracle: many small random junction trees with
mixed cardinalities (2..7, some 20-64 state variables) through the single-tree
path (fp64 and fp32) and the batch path (shared and materialized), so every
planner choice — row, thread-owned, general (2/4 vectors), contraction,
row-per-i, K-split — is exercised on shapes no config pins down."""
import numpy as np
import pytest

from oracle import jtref
from paper_1202_3777_b200 import synth
from paper_1202_3777_b200.tree import build_tree

pytestmark = pytest.mark.gpu

TOL = {"f64": 1e-10, "f32": 1e-5}


def rel_err(got, want):
    got, want = np.asarray(got, float), np.asarray(want, float)
    return float(np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-300)))


def random_tree(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 14))
    vals = np.array([2, 3, 4, 5, 7, 20, 64])
    probs = np.array([.22, .22, .18, .14, .12, .07, .05])
    members, cards = synth.grow_jt(
        n, seed, int(rng.integers(2, 5)), 1, 6, lambda r: r.choice(vals, p=probs / probs.sum()),
        lambda r: r.integers(1, 3), lambda r: r.integers(1, 3), 60000)
    tree = build_tree(members, cards)
    tree.cpt_assignment = {v: synth.smallest_holder(tree, v) for v in range(len(cards))}
    return tree, synth.scaled_potentials(tree, seed)


@pytest.mark.parametrize("seed", range(40))
def test_random_single_trees(seed):
    from paper_1202_3777_b200 import propagate as P

    tree, tables = random_tree(seed)
    template = jtref.from_potentials(tree, tables)
    for ev in [{}] + synth.evidence_cases(tree, 2, seed=seed):
        want = jtref.case_posteriors(template, ev, range(len(tree.cards)))
        for dtype in ("f64", "f32"):
            st = P.from_potentials(tree, tables, engine=P.CudaEngine(dtype=dtype))
            if ev:
                P.apply_evidence(st, ev)
            P.belief_propagation(st)
            got = np.concatenate([P.query_marginal(st, v).values for v in range(len(tree.cards))])
            assert rel_err(got, want) < TOL[dtype], (seed, dtype, ev)


@pytest.mark.parametrize("seed", range(16))
def test_random_batches(seed):
    from paper_1202_3777_b200.batch import BatchPropagator, shared_supported

    tree, tables = random_tree(100 + seed)
    cases = synth.evidence_cases(tree, 300, seed=seed)
    template = jtref.from_potentials(tree, tables)
    check = [0, 1, 150, 299]
    want = {i: jtref.case_posteriors(template, cases[i], range(len(tree.cards))) for i in check}
    modes = ("shared", "materialized") if shared_supported(tree) else ("materialized",)
    for mode in modes:
        for dtype, batch in (("f32", 256), ("f64", 128), ("f32", 6)):
            bp = BatchPropagator(tree, tables, batch=batch, dtype=dtype, mode=mode)
            out = bp.run(cases).cpu().numpy()
            bp.sync()
            for i in check:
                assert rel_err(out[i], want[i]) < TOL[dtype], (seed, mode, dtype, i)


@pytest.mark.parametrize("seed", range(16))
def test_random_batches_virtual_separators(seed, monkeypatch):
    """Every leaf message a program can gather instead of storing becomes a
    virtual separator (JT_VSEP_MIN_MB=0): unobserved, observed and
    never-observed leaf variables, fp64 and fp32, against the oracle."""
    from paper_1202_3777_b200.batch import BatchPropagator, shared_supported

    monkeypatch.setenv("JT_VSEP_MIN_MB", "0")
    tree, tables = random_tree(100 + seed)
    if not shared_supported(tree):
        pytest.skip("materialized-only tree")
    cases = synth.evidence_cases(tree, 300, seed=seed)
    template = jtref.from_potentials(tree, tables)
    check = [0, 1, 150, 299]
    want = {i: jtref.case_posteriors(template, cases[i], range(len(tree.cards))) for i in check}
    for dtype, batch in (("f64", 128), ("f32", 256)):
        bp = BatchPropagator(tree, tables, batch=batch, dtype=dtype, mode="shared")
        out = bp.run(cases, to_host=True)
        for i in check:
            assert rel_err(out[i], want[i]) < TOL[dtype], (seed, dtype, i)
