"""bench-style rows: the τ fit (perfmodel.py:115-150 restated) and the columns."""
import numpy as np
import pytest

from paper_1202_3777_b200 import benchcsv


def test_tau_fit_recovers_parameters():
    rng = np.random.default_rng(0)
    work = rng.uniform(1e3, 1e6, 200)
    time = 3e-6 + work / 5e9
    tau, theta = benchcsv.estimate_tau(list(zip(work, time)))
    assert tau == pytest.approx(3e-6, rel=1e-6) and theta == pytest.approx(5e9, rel=1e-6)


def test_tau_fit_overhead_dominated():
    tau, theta = benchcsv.estimate_tau([(1.0, 5.0), (2.0, 4.0), (3.0, 3.0)])
    assert theta == np.inf and tau == pytest.approx(4.0)


def test_columns_match_reference():  # cli.py:46-49
    assert benchcsv.BENCH_COLUMNS == ("tree", "n_cliques", "avg_spt", "seq_ms", "par_ms", "speedup",
                                      "pred_speedup", "tau_est", "overhead_frac")


def test_message_order_is_collect_then_distribute():
    from paper_1202_3777_b200 import synth

    tree, _ = synth.make_config("c1")
    msgs = benchcsv._messages(tree)
    n = len(tree.cliques) - len(tree.roots)
    assert len(msgs) == 2 * n
    # the first n are child→parent (collect), the last n parent→child (distribute)
    assert {(c, p) for c, p, _ in msgs[:n]} == {(c, p) for p, c, _ in msgs[n:]}
