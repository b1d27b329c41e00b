"""One shared-base batch step of a config (debug driver for compute-sanitizer)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1202_3777_b200 import synth
from paper_1202_3777_b200.batch import BatchPropagator
name, dt, B = sys.argv[1], sys.argv[2], int(sys.argv[3])
tree, tables = synth.make_config(name)
cases = synth.evidence_cases(tree, B, seed=1234)
bp = BatchPropagator(tree, tables, batch=B, dtype=dt, mode="auto")
print(name, dt, B, bp.mode, flush=True)
out = bp.run(cases, to_host=True)
print("ok", out.shape, flush=True)
