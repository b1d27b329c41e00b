"""Generate golden vectors by running the REFERENCE implementation (jtprop).

Run in a container where /root/reference exists:
    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_golden.py
Outputs small fixtures next to this script; they travel to the GPU box, the
reference does not.  Every fixture records the reference call that produced it.
"""

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
sys.path.insert(0, "/root/reference/pkg/tests")

from jtprop.compiler import build_mapping_table, build_tree, compile_network  # noqa: E402
from jtprop.potential import Scope  # noqa: E402
from jtprop.propagate import (  # noqa: E402
    apply_evidence,
    belief_propagation,
    from_potentials,
    initialize,
    query_marginal,
)

from paper_1202_3777_b200 import synth  # noqa: E402  (input generator only)

HERE = os.path.dirname(os.path.abspath(__file__))


def tree_json(tree):
    return {
        "cards": list(tree.cards),
        "cliques": [list(c.members) for c in tree.cliques],
        "separators": [[list(s.edge), list(s.members)] for s in tree.separators],
        "roots": list(tree.roots),
        "cpt_assignment": {str(k): v for k, v in tree.cpt_assignment.items()},
    }


def mapping_tables():
    """compiler.py:285-304 on seeded random scope pairs (the hypothesis property
    test_compiler.py:233-256 draws from the same space: 1-5 vars, cards 2-4)."""
    rng = np.random.default_rng(20240601)
    out = {}
    for i in range(80):
        n = int(rng.integers(1, 7))
        ids = tuple(sorted(rng.choice(40, size=n, replace=False).tolist()))
        cards = tuple(int(c) for c in rng.integers(2, 6, size=n))
        k = int(rng.integers(1, n + 1))
        pick = sorted(rng.choice(n, size=k, replace=False).tolist())
        clique = Scope(ids, cards)
        sep = Scope(tuple(ids[p] for p in pick), tuple(cards[p] for p in pick))
        mu = build_mapping_table(clique, sep)
        out[f"case{i}_ids"] = np.array(ids)
        out[f"case{i}_cards"] = np.array(cards)
        out[f"case{i}_sep"] = np.array(sep.ids)
        out[f"case{i}_mu"] = mu
    np.savez_compressed(os.path.join(HERE, "mapping_tables.npz"), **out)


def config_golden(name, n_cases, evidence_seed=1234):
    """Reference SequentialEngine BP on the Appendix-A config: posteriors of every
    variable with no evidence and with `n_cases` evidence cases, final separator
    tables, and per-clique sums of the final clique tables."""
    members, cards = synth.config_members(name)
    tree = build_tree(members, cards)
    tree.cpt_assignment = {v: synth.smallest_holder(tree, v) for v in range(len(cards))}
    tables = synth.scaled_potentials(tree, seed=0)
    out = {"tables_checksum": np.array([float(np.sum(t)) for t in tables] +
                                       [float(np.sum(t * np.arange(t.size) % 7)) for t in tables])}
    n_vars = len(cards)
    cases = [dict()] + synth.evidence_cases(tree, n_cases, seed=evidence_seed)
    for i, ev in enumerate(cases):
        st = from_potentials(tree, tables)
        if ev:
            apply_evidence(st, ev)
        belief_propagation(st)
        post = np.concatenate([query_marginal(st, v).values for v in range(n_vars)])
        raw = np.array([query_marginal(st, v, normalize_result=False).total() for v in range(min(n_vars, 4))])
        out[f"post{i}"] = post
        out[f"raw{i}"] = raw
        out[f"ev{i}"] = np.array(sorted(ev.items()), dtype=np.int64).reshape(-1, 2)
        if i == 0:
            seps = np.concatenate([s for s in st.sep_values])
            out["sep_sums0"] = np.array([s.sum() for s in st.sep_values])
            if seps.size <= 50000:
                out["sep0"] = seps
            else:  # keep fixtures small: a fixed stride sample of the final separators
                stride = seps.size // 20000 + 1
                out["sep_sample_stride"] = np.array([stride])
                out["sep_sample0"] = seps[::stride]
            out["clique_sums0"] = np.array([c.sum() for c in st.clique_values])
            if sum(t.size for t in tables) <= 20000:
                out["cliques0"] = np.concatenate(st.clique_values)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    with open(os.path.join(HERE, f"{name}_tree.json"), "w") as f:
        json.dump(tree_json(tree), f)


def corpus():
    """conftest.corpus_networks() compiled by the reference; CPT-initialized
    clique tables (initialize, propagate.py:204-222) and posteriors after BP with
    evidence {0: 0} (test_acceptance.py C3/C5 use the same evidence)."""
    from conftest import corpus_networks

    doc = []
    arrays = {}
    for k, (name, net) in enumerate(corpus_networks()):
        compiled = compile_network(net)
        st = initialize(compiled.tree, net, compiled.mappings)
        init = np.concatenate(st.clique_values)
        apply_evidence(st, {0: 0})
        belief_propagation(st)
        post = np.concatenate([query_marginal(st, v).values for v in range(len(net))])
        doc.append({"name": name, "tree": tree_json(compiled.tree),
                    "network": {"variables": [[v.name, v.cardinality] for v in net.variables],
                                "cpts": [[c.child, list(c.table.scope.ids)] for c in net.cpts]}})
        for c in net.cpts:
            arrays[f"cpt{k}_{c.child}"] = np.asarray(c.table.values, dtype=np.float64)
        # reference estimator (estimator.py:118-134), target = last variable, per-row loop
        from jtprop.estimator import JunctionTreeEngine

        rows = [{}, {0: 0}] + ([{len(net) - 2: 1}] if len(net) > 2 and net.variables[len(net) - 2].cardinality > 1 else [])
        est = JunctionTreeEngine(target=net.variables[-1].name).fit(net)
        arrays[f"est{k}"] = est.predict_proba(rows)
        arrays[f"estX{k}"] = np.array([[a, b] for r in rows for a, b in r.items()] or [[-1, -1]])
        arrays[f"estXrow{k}"] = np.array([i for i, r in enumerate(rows) for _ in r.items()] or [-1])
        arrays[f"init{k}"] = init
        arrays[f"post{k}"] = post
        arrays[f"cliques{k}"] = np.concatenate(st.clique_values)
        arrays[f"seps{k}"] = np.concatenate(st.sep_values) if st.sep_values else np.zeros(0)
    # reference tree dumps (io.py:443-474) of two corpus networks: with the
    # network embedded, and with mapping tables in the interleaved layout
    from jtprop.io import serialize_tree

    nets = corpus_networks()
    for k, kw in ((3, {"net": True}), (5, {"net": True, "include_mappings": True, "layout": "interleaved"})):
        name, net = nets[k]
        compiled = compile_network(net, layout=kw.get("layout", "flat"))
        text = serialize_tree(compiled.tree, compiled.mappings, net if kw.get("net") else None,
                              include_mappings=kw.get("include_mappings", False))
        with open(os.path.join(HERE, f"tree_dump{k}.jt.json"), "w") as f:
            f.write(text)
    np.savez_compressed(os.path.join(HERE, "corpus.npz"), **arrays)
    with open(os.path.join(HERE, "corpus.json"), "w") as f:
        json.dump(doc, f)


def unscaled_golden(name="c2", n_cases=3, evidence_seed=77):
    """The reference generator's own potentials, NOT rescaled: uniform(0.1, 1)
    per clique in id order (synth.py:105-107, default_rng(0)).  On the
    Pigs-shaped c2 tree these reach ~1e107 after propagation:
    far outside fp32.  Reference posteriors and unnormalized masses P(e)
    (query_marginal(..., normalize_result=False).total(), propagate.py:363-377)."""
    members, cards = synth.config_members(name)
    tree = build_tree(members, cards)
    tree.cpt_assignment = {v: synth.smallest_holder(tree, v) for v in range(len(cards))}
    rng = np.random.default_rng(0)
    tables = [rng.uniform(0.1, 1.0, size=c.scope.size) for c in tree.cliques]
    out = {}
    cases = [dict()] + synth.evidence_cases(tree, n_cases, seed=evidence_seed)
    for i, ev in enumerate(cases):
        st = from_potentials(tree, tables)
        if ev:
            apply_evidence(st, ev)
        belief_propagation(st)
        out[f"post{i}"] = np.concatenate([query_marginal(st, v).values for v in range(len(cards))])
        out[f"mass{i}"] = np.array([query_marginal(st, v, normalize_result=False).total() for v in (0, 5, 17)])
        out[f"ev{i}"] = np.array(sorted(ev.items()), dtype=np.int64).reshape(-1, 2)
        out[f"maxabs{i}"] = np.array([max(float(c.max()) for c in st.clique_values)])
    np.savez_compressed(os.path.join(HERE, f"{name}_unscaled.npz"), **out)


BENCH_IDX = list(range(0, 24)) + list(range(4072, 4120)) + list(range(8168, 8192))


def bench_golden(name="c5", n_total=8192, evidence_seed=1234):
    """The bench workload itself (bench.py: c5, seed-1234 evidence, 8192 cases per
    GPU in two 4096-case micro-batches): reference SequentialEngine posteriors of
    every variable for a sample of case indices that covers the start and end of
    BOTH micro-batches (0..23, 4072..4119 across the boundary, 8168..8191)."""
    members, cards = synth.config_members(name)
    tree = build_tree(members, cards)
    tree.cpt_assignment = {v: synth.smallest_holder(tree, v) for v in range(len(cards))}
    tables = synth.scaled_potentials(tree, seed=0)
    posts = []
    for i in BENCH_IDX:
        ev = synth.evidence_cases(tree, 1, seed=evidence_seed, first=i)[0]
        st = from_potentials(tree, tables)
        apply_evidence(st, ev)
        belief_propagation(st)
        posts.append(np.concatenate([query_marginal(st, v).values for v in range(len(cards))]))
    np.savez_compressed(os.path.join(HERE, f"{name}_bench.npz"), idx=np.array(BENCH_IDX),
                        n_total=np.array([n_total]), seed=np.array([evidence_seed]), post=np.stack(posts))


if __name__ == "__main__":
    if sys.argv[1:] == ["corpus"]:
        corpus()
        sys.exit(0)
    if sys.argv[1:] == ["bench"]:
        bench_golden()
        sys.exit(0)
    if sys.argv[1:] == ["unscaled"]:
        unscaled_golden()
        sys.exit(0)
    mapping_tables()
    corpus()
    for name, n in (("c1", 8), ("c2", 4), ("c4M", 2), ("c5", 8), ("c4B", 1), ("c3", 1)):
        config_golden(name, n)
        print("golden", name)
    bench_golden()
    unscaled_golden()
