"""Small workload for compute-sanitizer: single-tree c1 (fp32, fp64) with
evidence, the per-message path, and a 16-case shared-base batch on c1 and a
128-case one on c5 (contraction passes).  Checks results against the oracle so
a sanitizer run also proves the instrumented kernels computed the right thing."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import jtref  # noqa: E402
from paper_1202_3777_b200 import propagate as P  # noqa: E402
from paper_1202_3777_b200 import synth  # noqa: E402
from paper_1202_3777_b200.batch import BatchPropagator  # noqa: E402


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


tree, tables = synth.make_config("c1")
ev = {3: 1, 17: 2}
want = jtref.case_posteriors(jtref.from_potentials(tree, tables), ev, range(len(tree.cards)))
for dt, tol in (("f64", 1e-10), ("f32", 1e-5)):
    st = P.from_potentials(tree, tables, engine=P.CudaEngine(dtype=dt))
    P.apply_evidence(st, ev)
    P.belief_propagation(st)
    got = np.concatenate([P.query_marginal(st, v).values for v in range(len(tree.cards))])
    assert rel(got, want) < tol, dt
    st2 = P.from_potentials(tree, tables)
    P.apply_evidence(st2, ev)
    for r in tree.roots:
        P.collect_evidence(st2, r)
        P.distribute_evidence(st2, r)
    got2 = np.concatenate([P.query_marginal(st2, v).values for v in range(len(tree.cards))])
    assert rel(got2, want) < 1e-10
for name, B in (("c1", 16), ("c5", 128)):
    tr, tb = synth.make_config(name)
    cases = synth.evidence_cases(tr, B, seed=5)
    bp = BatchPropagator(tr, tb, batch=B, dtype="f32", mode="shared")
    out = bp.run(cases).cpu().numpy()
    bp.sync()
    tmpl = jtref.from_potentials(tr, tb)
    for i in (0, B - 1):
        assert rel(out[i], jtref.case_posteriors(tmpl, cases[i], range(len(tr.cards)))) < 1e-5, (name, i)
print("sanitize workload ok")
