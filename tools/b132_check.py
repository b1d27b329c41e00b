"""Partial-chunk batch check (debug): which cases / variables of a shared-base
micro-batch differ from the oracle."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1202_3777_b200 import synth
from paper_1202_3777_b200.batch import BatchPropagator
from oracle import jtref
tree, tables = synth.make_config("c5")
cases = synth.evidence_cases(tree, 264, seed=3)
tp = jtref.from_potentials(tree, tables)
offs = np.cumsum([0] + list(tree.cards))
for dt, B in (("f64", 132), ("f64", 136), ("f32", 132), ("f32", 260)):
    bp = BatchPropagator(tree, tables, batch=B, dtype=dt, mode="shared")
    out = bp.run(cases[:B])
    try:
        bp.sync()
    except Exception as e:
        print(dt, B, "ERR", type(e).__name__)
    out = out.cpu().numpy()
    bad = []
    for i in range(B):
        w = jtref.case_posteriors(tp, cases[i], range(len(tree.cards)))
        e = np.abs(out[i] - w) / np.maximum(np.abs(w), 1e-300)
        if not np.all(e < (1e-10 if dt == "f64" else 1e-5)):
            vs = [v for v in range(len(tree.cards)) if not np.all(e[offs[v]:offs[v + 1]] < 1e-8)]
            bad.append((i, vs[:6]))
    print(dt, B, "bad cases", len(bad), bad[:12])
