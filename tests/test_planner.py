"""Host planner (no device): every BASELINE config compiles into a propagation
program in every mode the engine supports, and the program has the structure
DESIGN.md §3 describes (waves by height/depth, row passes on the row kernel)."""
import os
import sys

import pytest

from conftest import ROOT

sys.path.insert(0, os.path.join(ROOT, "tools"))

CONFIGS = ["c1", "c2", "c3", "c4B", "c4M", "c5"]


def report(*a, **k):
    import plan_report

    return plan_report.report(*a, **k)


@pytest.mark.parametrize("name", CONFIGS)
@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("kind", [0, 1])
def test_single_tree_program_compiles(name, dtype, kind):
    text = report(name, batch=1, mode="materialized", kind=kind, dtype=dtype)
    assert "compulsory total MB" in text and "\nwave 0" in text
    # small waves of single trees run as tiny passes (jt_tiny.cu), the rest as general passes
    assert "pass clique" in text or text.startswith("tiny passes")


@pytest.mark.parametrize("name", ["c1", "c5", "c4B"])
@pytest.mark.parametrize("batch", [8, 16, 1024])
def test_batch_programs_compile(name, batch):
    for mode in ("shared", "materialized"):
        if mode == "materialized" and batch > 16 and name != "c1":
            continue  # a c5 materialized micro-batch of 1024 cases would need 33 GB of clique tables
        report(name, batch=batch, mode=mode, kind=1, dtype="f32")


def test_shared_mode_hub_cliques_keep_per_case_tables():
    # c2 (Pigs-shaped) has cliques with > 8 neighbour ratios + evidence masks: in
    # shared-base mode those hubs get per-case tables (initialised from base x
    # evidence, children absorbed eagerly) instead of a materialized fallback
    from paper_1202_3777_b200 import synth
    from paper_1202_3777_b200.batch import shared_supported

    tree, _ = synth.make_config("c2")
    assert shared_supported(tree)
    text = report("c2", batch=8, mode="shared", kind=1)
    assert "compulsory total MB" in text
    # wave 0 initialises the hubs: write passes from the base replica (src 1)
    first = [l for l in text.split("\nwave 1 ")[0].splitlines() if l.startswith("  pass")]
    assert first and all(" src 1 " in l and " wr 1 " in l for l in first)


def test_large_cliques_use_row_kernel():
    text = report("c3", batch=1, mode="materialized", kind=0, dtype="f32")
    rows = [l for l in text.splitlines() if l.startswith("  pass") and " row 1 " in l]
    assert len(rows) >= 5, text


def test_batch_program_uses_contraction_passes():
    text = report("c5", batch=2048, mode="shared", kind=1, dtype="f32")
    assert "contract clique" in text
    total = float(next(l for l in text.splitlines() if l.startswith("compulsory total MB")).split()[-1])
    assert 20000 < total < 60000  # ~29 GB per 2048-case micro-batch (46.6 before X / virtual separators)


@pytest.mark.parametrize("batch", [128, 4096])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_ksplit_contraction_is_compiled(batch, dtype):
    """The K-split contraction path (long sums over few units, partials combined
    in chunk order by the last warp) must really be in the programs the GPU
    parity tests run: B = 128 (test_gpu_parity) and the bench's B = 4096
    (test_gpu_headline).  Guards against the planner heuristics silently
    dropping the coverage."""
    text = report("c5", batch=batch, mode="shared", kind=1, dtype=dtype)
    ks = [int(line.split(" ks ")[1].split()[0]) for line in text.splitlines() if " ks " in line]
    assert ks and max(ks) > 1, (batch, dtype)


def test_small_single_trees_use_tiny_passes():
    """Single trees: waves touching at most 2^18 elements run as tiny passes
    (one launch per wave, PDL-chained); c1 entirely, c3 (16.8M-entry cliques) never."""
    c1 = report("c1", batch=1, mode="materialized", kind=0, dtype="f32")
    assert c1.startswith("tiny passes (mode 2): 7 of 7 waves")
    c3 = report("c3", batch=1, mode="materialized", kind=0, dtype="f32")
    assert not c3.startswith("tiny passes")


def test_batch_program_pairs_siblings_and_shares_the_hub_product(monkeypatch):
    """c5's hub clique 2 sends distribute messages to two children over the same
    140000-entry separator: the planner pairs them into ONE row-per-i pass with
    two epilogues; that pass also writes the clique product X and the
    hub's two other distribute passes read it (one sub-wave later), which the
    compulsory-bytes accounting reflects."""
    monkeypatch.setenv("JT_VSEP", "0")  # (virtual separators: the next test)
    f64 = report("c5", batch=4096, mode="shared", kind=1, dtype="f64")
    paired = [l for l in f64.splitlines() if l.startswith("  contract clique 2 out 4 nI 140000")]
    assert len(paired) == 1, paired  # two DFRESH passes -> one paired pass
    total = lambda t: float(next(l for l in t.splitlines() if l.startswith("compulsory total MB")).split()[-1])
    monkeypatch.setenv("JT_HUBX", "0")
    f64_nox = report("c5", batch=4096, mode="shared", kind=1, dtype="f64")
    assert total(f64) < total(f64_nox) - 5000  # ~9 GB fewer per 4096-case micro-batch (13.8 before ratio-only outputs)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_batch_program_gathers_virtual_separators(dtype, monkeypatch):
    """c5's leaves 3 and 12 send 140000-entry collect messages that only hub
    clique 2 reads: the planner drops their producer passes and the hub's
    row-per-i passes (its collect pass and the paired distribute pass) gather the
    messages from the leaves' summed tables by each case's evidence code, which
    removes 4.59 GB (fp64) of writes plus their re-reads per message from the
    compulsory bytes."""
    monkeypatch.setenv("JT_DEBUG_SPECS", "1")
    total = lambda t: float(next(l for l in t.splitlines() if l.startswith("compulsory total MB")).split()[-1])
    on = report("c5", batch=4096, mode="shared", kind=1, dtype=dtype)
    readers = [l for l in on.splitlines() if l.startswith("  spec") and not l.endswith("vsep 0")]
    hub = [l for l in readers if " clique 2 " in l]
    assert len(hub) == 3, readers  # the collect pass and the two (paired) distribute passes
    assert all(l.endswith("vsep 2") for l in hub)
    assert len(readers) == 3, readers  # (leaf 14's message is a K-sum factor of clique 13: stored)
    monkeypatch.setenv("JT_VSEP_MIN_MB", "0")
    assert total(report("c5", batch=4096, mode="shared", kind=1, dtype=dtype)) <= total(on)
    monkeypatch.setenv("JT_VSEP", "0")
    off = report("c5", batch=4096, mode="shared", kind=1, dtype=dtype)
    assert "vsep 2" not in off
    saved = total(off) - total(on)
    assert saved > (20000 if dtype == "f64" else 10000), saved
