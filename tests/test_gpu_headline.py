"""The bench workload itself, pinned against the reference (VERDICT r1 "next" #1).

bench.py's headline: c5 (Mildew-shaped), shared-base mode, micro-batches of
4096 cases, 8192 cases per step (two micro-batches), fp64 (the reference's own
arithmetic) and fp32.  96 cases spread over the start and end of BOTH
micro-batches (0..23, 4072..4119 across the boundary, 8168..8191) are compared
with posteriors the reference jtprop computed for the same cases
(tests/golden/c5_bench.npz, tests/golden/make_golden.py bench).  Micro-batch 1
is where state reused across micro-batches (K-split partials, arrival counters,
evidence masks, swapped separator roles) would show a reset bug.

Tolerances (north_star): 1e-10 relative in fp64, 1e-5 in fp32.
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden
from paper_1202_3777_b200 import synth

pytestmark = pytest.mark.gpu

TOL = {"f64": 1e-10, "f32": 1e-5}
N_CASES, BATCH = 8192, 4096


def rel_err(got, want):
    return float(np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-300)))


@pytest.fixture(scope="module")
def workload():
    tree, _ = load_golden("c5")
    tables = synth.scaled_potentials(tree, 0)
    cases = synth.evidence_cases(tree, N_CASES, seed=1234)
    g = np.load(os.path.join(GOLDEN, "c5_bench.npz"))
    assert int(g["seed"][0]) == 1234 and int(g["n_total"][0]) == N_CASES
    return tree, tables, cases, g["idx"], g["post"]


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_bench_workload_both_micro_batches(workload, dtype):
    from paper_1202_3777_b200.batch import BatchPropagator

    tree, tables, cases, idx, want = workload
    bp = BatchPropagator(tree, tables, batch=BATCH, dtype=dtype, mode="shared")
    assert bp.mode == "shared"
    # device path of the bench's `value` (run twice: programs are graph-replayed
    # from the second step on, and state left by step 1 must not leak into step 2)
    for _ in range(2):
        out = bp.run(cases).cpu().numpy()
        bp.sync()
        assert out.shape == (N_CASES, bp.cols)
        assert {int(i) // BATCH for i in idx} == {0, 1}
        assert rel_err(out[idx], want) < TOL[dtype], dtype
        # every case is a distribution
        assert np.all(np.isfinite(out))
    # the e2e path: Python dicts in, host numpy out
    host = bp.run(cases, to_host=True)
    assert isinstance(host, np.ndarray)
    assert np.array_equal(host, out)
    bp.close()



@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_odd_micro_batch_pads_case_lanes(workload, dtype):
    """A micro-batch that is not a whole number of thread-owned blocks (4000
    cases) is padded to whole blocks inside the state (it
    used to fall to the general kernels at half the speed, or fail to plan in
    fp64).  The padded lanes never reach the caller: 8000 cases in two
    micro-batches of 4000 match the reference on every golden case below 8000,
    across the micro-batch boundary (cases 3999/4000)."""
    from paper_1202_3777_b200.batch import BatchPropagator

    tree, tables, cases, idx, want = workload
    keep = idx < 8000
    bp = BatchPropagator(tree, tables, batch=4000, dtype=dtype, mode="shared")
    out = bp.run(cases[:8000], to_host=True)
    assert out.shape == (8000, bp.cols)
    assert rel_err(out[idx[keep]], want[keep]) < TOL[dtype], dtype
    assert {int(i) // 4000 for i in idx[keep]} == {0, 1}
    bp.close()
