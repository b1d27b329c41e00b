"""Batch posteriors of a config vs the oracle on a few cases (debug driver).
usage: python tools/batch_check.py c4M f64 2048 [mode] [n_cases]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import jtref  # noqa: E402  (checker only)
from paper_1202_3777_b200 import synth  # noqa: E402
from paper_1202_3777_b200.batch import BatchPropagator  # noqa: E402

name, dt, B = sys.argv[1], sys.argv[2], int(sys.argv[3])
mode = sys.argv[4] if len(sys.argv) > 4 else "auto"
tree, tables = synth.make_config(name)
n = int(sys.argv[5]) if len(sys.argv) > 5 else B
cases = synth.evidence_cases(tree, n, seed=1234)
bp = BatchPropagator(tree, tables, batch=B, dtype=dt, mode=mode)
out = bp.run(cases, to_host=True)
template = jtref.from_potentials(tree, tables)
idx = sorted({0, 1, B // 2, B - 1, min(B, n - 1), n - 1})
errs = []
for i in idx:
    want = jtref.case_posteriors(template, cases[i], range(len(tree.cards)))
    errs.append(float(np.max(np.abs(out[i] - want) / np.maximum(np.abs(want), 1e-300))))
print(name, dt, B, bp.mode, "max rel err per case", ["%.2e" % e for e in errs], flush=True)
