"""Profiling driver: warm up one workload, then run it `--reps` more times so
ncu (-s/-c) can capture steady-state launches.  Never a bench number."""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--dtype", default="f32")
ap.add_argument("--batch", type=int, default=4096)
ap.add_argument("--mode", default="auto")
ap.add_argument("--single", action="store_true", help="single-tree jt_propagate instead of batch")
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()

import torch  # noqa: E402

from paper_1202_3777_b200 import _lib, synth  # noqa: E402

tree, tables = synth.make_config(a.config)
L = _lib.lib()
if a.single:
    from paper_1202_3777_b200 import propagate as P
    st = P.from_potentials(tree, tables, engine=P.CudaEngine(dtype=a.dtype))
    s = torch.cuda.Stream()
    h = C.c_void_p(s.cuda_stream)
    for _ in range(3 + a.reps):
        L.jt_state_reset(st.handle, h)
        _lib.check(L.jt_propagate(st.handle, None, h))
    s.synchronize()
    st.sync()
else:
    from paper_1202_3777_b200.batch import BatchPropagator
    bp = BatchPropagator(tree, tables, batch=a.batch, dtype=a.dtype, mode=a.mode)
    cases = synth.evidence_cases(tree, a.batch)
    obs = torch.from_numpy(bp.encode_obs(cases)).cuda()
    out = torch.empty((a.batch, bp.cols), dtype=torch.float64, device="cuda")
    for _ in range(3 + a.reps):
        bp.step_device(obs, out)
    bp.stream.synchronize()
    bp.sync()
print("done", bp.mode if not a.single else "single")
