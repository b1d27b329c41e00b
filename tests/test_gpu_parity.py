"""Parity of the CUDA path against the oracle / reference golden vectors.

Tolerances (BASELINE.json north_star): posteriors within 1e-10 relative in the
fp64 mode and 1e-5 relative in fp32.  Integer index maps are bit-exact.
"""

import numpy as np
import pytest

from conftest import golden_cases, load_corpus, load_golden
from oracle import jtref
from paper_1202_3777_b200 import synth
from paper_1202_3777_b200.tree import build_tree

pytestmark = pytest.mark.gpu

TOL = {"f64": 1e-10, "f32": 1e-5}


def P():
    from paper_1202_3777_b200 import propagate

    return propagate


def rel_err(got, want):
    got, want = np.asarray(got, float), np.asarray(want, float)
    return float(np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-300))) if want.size else 0.0


def all_posteriors(st, n):
    return np.concatenate([P().query_marginal(st, v).values for v in range(n)])


def demo(src=None, dtype="f64"):
    tree = build_tree([(0, 1, 3), (1, 2)], (2, 2, 2, 2))
    tables = [np.arange(8.0) if src is None else np.asarray(src, float), np.ones(4)]
    return tree, P().from_potentials(tree, tables, engine=P().CudaEngine(dtype=dtype))


class TestMessageKnownAnswers:  # test_propagate.py:53-89 through the device path
    @pytest.mark.parametrize("dtype", ["f64", "f32"])
    def test_worked_example(self, dtype):
        tree, st = demo(dtype=dtype)
        P().message_passing(st, P().Message(0, 1, 0))
        assert st.sep_values[0].tolist() == [10.0, 18.0]
        assert st.clique_values[1].tolist() == [10.0, 10.0, 18.0, 18.0]
        assert st.clique_values[0].tolist() == list(range(8))

    def test_zero_over_zero(self):
        tree, st = demo([0, 0, 1, 2, 0, 0, 3, 4])
        st.sep_values[0][:] = [0.0, 1.0]
        st.clique_values[1][:] = [5.0, 6.0, 7.0, 8.0]
        P().message_passing(st, P().Message(0, 1, 0))
        assert st.clique_values[1].tolist() == [0.0, 0.0, 70.0, 80.0]
        assert st.sep_values[0].tolist() == [0.0, 10.0]

    def test_nonzero_over_zero_raises(self):
        from paper_1202_3777_b200.errors import InconsistentDivisionError

        tree, st = demo()
        st.sep_values[0][:] = [0.0, 1.0]
        with pytest.raises(InconsistentDivisionError):
            P().message_passing(st, P().Message(0, 1, 0))

    def test_fixed_point(self):
        tree, st = demo(np.ones(8))
        st.sep_values[0][:] = [4.0, 4.0]
        before = st.clique_values[1].copy()
        P().message_passing(st, P().Message(0, 1, 0))
        assert np.array_equal(st.clique_values[1], before)

    def test_mass_conservation(self):
        rng = np.random.default_rng(0)
        tree, st = demo(rng.uniform(size=8))
        P().message_passing(st, P().Message(0, 1, 0))
        assert st.sep_values[0].sum() == pytest.approx(st.clique_values[0].sum(), rel=1e-12)


def test_device_mapping_tables_bit_exact():
    for name in ("c1", "c3", "c5"):
        tree, _ = load_golden(name)
        plan = P().plan_for(tree, "f64")
        for sep in tree.separators:
            for cid in sep.edge:
                c = tree.cliques[cid]
                want = jtref.build_mapping_table(c.scope.ids, c.scope.cards, sep.scope.ids)
                got = plan.mapping_table(cid, sep.id)
                assert got.dtype == want.dtype and np.array_equal(got, want), (name, cid, sep.id)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("name", ["c1", "c2", "c4M", "c5", "c4B", "c3"])
def test_config_posteriors_vs_reference(name, dtype):
    tree, data = load_golden(name)
    tables = synth.scaled_potentials(tree, seed=0)
    cases = golden_cases(data)
    for ev, want in cases[:3]:
        st = P().from_potentials(tree, tables, engine=P().CudaEngine(dtype=dtype))
        if ev:
            P().apply_evidence(st, ev)
        P().belief_propagation(st)
        got = all_posteriors(st, len(tree.cards))
        assert rel_err(got, want) < TOL[dtype], (name, dtype, ev, rel_err(got, want))


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_final_tables_c1(dtype):
    tree, data = load_golden("c1")
    st = P().from_potentials(tree, synth.scaled_potentials(tree, 0), engine=P().CudaEngine(dtype=dtype))
    P().belief_propagation(st)
    assert rel_err(np.concatenate(st.clique_values), data["cliques0"]) < TOL[dtype] * 10
    assert rel_err(np.concatenate(st.sep_values), data["sep0"]) < TOL[dtype] * 10


def test_separator_tables_c5_vs_reference():
    tree, data = load_golden("c5")
    st = P().from_potentials(tree, synth.scaled_potentials(tree, 0))
    P().belief_propagation(st)
    seps = st.sep_values
    assert rel_err([s.sum() for s in seps], data["sep_sums0"]) < 1e-10
    assert rel_err([c.sum() for c in st.clique_values], data["clique_sums0"]) < 1e-10


def test_corpus_initialized_networks():
    for name, tree, tables, post, cliques, seps in load_corpus():
        st = P().from_potentials(tree, tables)
        P().apply_evidence(st, {0: 0})
        P().belief_propagation(st)
        got = all_posteriors(st, len(tree.cards))
        assert rel_err(got, post) < 1e-10, name
        assert rel_err(np.concatenate(st.clique_values), cliques) < 1e-9, name


def test_per_message_traversal_matches_fused():
    tree, data = load_golden("c2")
    tables = synth.scaled_potentials(tree, 0)
    a = P().from_potentials(tree, tables)
    for r in tree.roots:
        P().collect_evidence(a, r)
        P().distribute_evidence(a, r)
    b = P().from_potentials(tree, tables)
    P().belief_propagation(b)
    assert rel_err(np.concatenate(a.clique_values), np.concatenate(b.clique_values)) < 1e-10
    assert rel_err(all_posteriors(a, len(tree.cards)), data["post0"]) < 1e-10


def test_traversal_spy_sees_reference_order(monkeypatch):  # test_propagate.py:168-200
    from paper_1202_3777_b200 import propagate as prop

    log = []
    orig = prop.message_passing

    def spy(state, msg):
        log.append((msg.source, msg.target))
        return orig(state, msg)

    monkeypatch.setattr(prop, "message_passing", spy)
    tree = build_tree([(0, 1), (1, 2, 3), (3, 4)], (2,) * 5)
    st = prop.from_potentials(tree, [np.ones(4), np.ones(8), np.ones(4)])
    prop.collect_evidence(st, 1)
    assert log == [(0, 1), (2, 1)]
    del log[:]
    prop.distribute_evidence(st, 1)
    assert log == [(1, 0), (1, 2)]


def test_root_choice_and_second_run():
    tree, data = load_golden("c1")
    tables = synth.scaled_potentials(tree, 0)
    ref = None
    for root in range(len(tree.cliques)):
        st = P().from_potentials(tree, tables)
        P().apply_evidence(st, {5: 1})
        P().belief_propagation(st, root=root)
        got = all_posteriors(st, len(tree.cards))
        ref = got if ref is None else ref
        assert rel_err(got, ref) < 1e-12
        P().belief_propagation(st)
        assert rel_err(all_posteriors(st, len(tree.cards)), ref) < 1e-12


def test_incremental_evidence():  # test_propagate.py:289-300
    tree, _ = load_golden("c1")
    tables = synth.scaled_potentials(tree, 0)
    st = P().from_potentials(tree, tables)
    P().apply_evidence(st, {3: 1})
    P().belief_propagation(st)
    P().apply_evidence(st, {9: 0})
    P().belief_propagation(st)
    want = jtref.case_posteriors(jtref.from_potentials(tree, tables), {3: 1, 9: 0}, range(len(tree.cards)))
    assert rel_err(all_posteriors(st, len(tree.cards)), want) < 1e-10


def test_unnormalized_mass_and_zero_mass():
    from paper_1202_3777_b200.errors import ZeroMassError

    tree, data = load_golden("c1")
    tables = synth.scaled_potentials(tree, 0)
    st = P().from_potentials(tree, tables)
    P().apply_evidence(st, {2: 1})
    P().belief_propagation(st)
    o = jtref.from_potentials(tree, tables)
    jtref.apply_evidence(o, {2: 1})
    jtref.belief_propagation(o)
    raw = P().query_marginal(st, 0, normalize_result=False).total()
    assert raw == pytest.approx(jtref.query_marginal(o, 0, False).sum(), rel=1e-12)
    # impossible evidence: two observations of one variable that disagree
    st2 = P().from_potentials(tree, tables)
    P().apply_evidence(st2, {2: 1})
    P().apply_evidence(st2, {2: 0})
    P().belief_propagation(st2)
    with pytest.raises(ZeroMassError):
        P().query_marginal(st2, 0)


def test_unknown_engine_and_variable():
    from paper_1202_3777_b200.errors import UnknownVariableError

    with pytest.raises(ValueError):
        P().make_engine("gpu")
    tree, _ = load_golden("c1")
    st = P().from_potentials(tree, synth.scaled_potentials(tree, 0))
    with pytest.raises(UnknownVariableError):
        P().apply_evidence(st, {999: 0})
    with pytest.raises(UnknownVariableError):
        P().belief_propagation(st, root=99)


def test_engine_protocol_on_host_arrays():
    """CudaEngine.run_message speaks the reference engine protocol (propagate.py:84)."""
    rng = np.random.default_rng(3)
    eng = P().CudaEngine()
    for ids, cards, sep in [((0, 1, 3), (2, 2, 2), (1,)), ((0, 1, 2, 3), (3, 4, 2, 5), (0, 2)),
                            ((4, 7, 9), (5, 3, 4), (7,))]:
        sc = tuple(cards[ids.index(v)] for v in sep)
        mu_s = jtref.build_mapping_table(ids, cards, sep)
        tgt_ids = tuple(sorted(set(sep) | {50}))
        tgt_cards = tuple(sc[list(sep).index(v)] if v in sep else 3 for v in tgt_ids)
        mu_t = jtref.build_mapping_table(tgt_ids, tgt_cards, sep)
        src = rng.uniform(size=mu_s.size)
        tgt = rng.uniform(size=mu_t.size)
        sp = rng.uniform(0.5, 1.5, size=mu_s.shape[0])
        a_t, a_s = tgt.copy(), sp.copy()
        jtref.pass_block(src, a_t, a_s, mu_s, mu_t, 0, len(a_s))
        b_t, b_s = tgt.copy(), sp.copy()
        eng.run_message(src, b_t, b_s, mu_s, mu_t)
        assert rel_err(b_t, a_t) < 1e-13 and rel_err(b_s, a_s) < 1e-13


@pytest.mark.parametrize("mode", ["shared", "materialized"])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_batch_engine_vs_reference(mode, dtype):
    from paper_1202_3777_b200.batch import BatchPropagator

    for name in ("c1", "c5"):
        tree, data = load_golden(name)
        tables = synth.scaled_potentials(tree, 0)
        cases = golden_cases(data)
        bp = BatchPropagator(tree, tables, batch=8, dtype=dtype, mode=mode)
        out = bp.run([ev for ev, _ in cases]).cpu().numpy()
        bp.sync()
        for i, (ev, want) in enumerate(cases):
            assert rel_err(out[i], want) < TOL[dtype], (name, mode, dtype, i)


def test_batch_engine_vs_oracle_many_cases():
    from paper_1202_3777_b200.batch import BatchPropagator

    tree, _ = load_golden("c2")
    tables = synth.scaled_potentials(tree, 0)
    cases = synth.evidence_cases(tree, 40, seed=99)
    template = jtref.from_potentials(tree, tables)
    want = np.stack([jtref.case_posteriors(template, ev, range(len(tree.cards))) for ev in cases[:6]])
    for mode in ("auto", "materialized"):
        bp = BatchPropagator(tree, tables, batch=16, dtype="f64", mode=mode)
        out = bp.run(cases).cpu().numpy()
        bp.sync()
        assert rel_err(out[:6], want) < 1e-10, mode


def test_calibration_full_size_c3():
    """Size-independent property at full size: every separator equals the
    marginal of both adjacent cliques after BP (check_global_consistency)."""
    tree, data = load_golden("c3")
    st = P().from_potentials(tree, synth.scaled_potentials(tree, 0), engine=P().CudaEngine(dtype="f64"))
    P().belief_propagation(st)
    P().check_global_consistency(st, rtol=1e-9)
    got = all_posteriors(st, len(tree.cards))
    assert rel_err(got, data["post0"]) < 1e-10


def test_device_initialize_matches_reference():  # initialize, propagate.py:204-222
    from conftest import load_corpus_networks

    for name, tree, net, init, _, _ in load_corpus_networks():
        for dtype, tol in (("f64", 1e-14), ("f32", 1e-6)):
            st = P().initialize(tree, net, engine=P().CudaEngine(dtype=dtype))
            got = np.concatenate(st.clique_values)
            assert rel_err(got, init) < tol, (name, dtype)
            assert all(np.all(s == 1.0) for s in st.sep_values), name


def test_estimator_matches_reference_predict_proba():  # estimator.py:118-134
    from conftest import load_corpus_networks
    from paper_1202_3777_b200.estimator import JunctionTreeEngine

    for name, tree, net, _, rows, want in load_corpus_networks():
        est = JunctionTreeEngine(target=net.variables[-1].name, batch=4).fit_compiled(tree, net)
        got = est.predict_proba(rows)
        assert got.shape == want.shape
        assert rel_err(got, want) < 1e-10, name
        assert np.array_equal(est.predict(rows), want.argmax(axis=1))
        q = est.query(evidence=rows[-1])
        assert rel_err(q[net.variables[-1].name], want[-1]) < 1e-10, name


def test_tree_dump_to_device_plan():  # §8f row 4: .jt.json → cached device plan
    import os

    from conftest import GOLDEN, load_corpus
    from paper_1202_3777_b200 import io

    corpus = load_corpus()
    for k in (3, 5):
        path = os.path.join(GOLDEN, f"tree_dump{k}.jt.json")
        plan, tree, net = io.load_plan(path, "f64")
        assert io.load_plan(path, "f64")[0] is plan  # cached
        st = P().initialize(tree, net)
        assert st.plan is plan
        P().apply_evidence(st, {0: 0})
        P().belief_propagation(st)
        got = all_posteriors(st, len(tree.cards))
        assert rel_err(got, corpus[k][3]) < 1e-10, k


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("batch", [128, 132])
def test_batch_contraction_path_large_batch(dtype, batch):
    """Shared-base micro-batches large enough for the contraction passes
    (DESIGN.md §3b): every case matches the reference goldens / the oracle.
    128 cases run the K-split contraction passes (test_planner asserts the
    planner compiles them); 132 cases leave a partial last case chunk, which
    routes the long sums to the general kernels (K-split needs whole chunks)."""
    from paper_1202_3777_b200.batch import BatchPropagator

    tree, data = load_golden("c5")
    tables = synth.scaled_potentials(tree, 0)
    golden = golden_cases(data)
    extra = synth.evidence_cases(tree, 6, seed=7)
    template = jtref.from_potentials(tree, tables)
    want_extra = [jtref.case_posteriors(template, ev, range(len(tree.cards))) for ev in extra]
    cases = [golden[i % len(golden)][0] for i in range(250)] + extra
    bp = BatchPropagator(tree, tables, batch=batch, dtype=dtype, mode="shared")
    out = bp.run(cases).cpu().numpy()
    bp.sync()
    for i in range(250):
        assert rel_err(out[i], golden[i % len(golden)][1]) < TOL[dtype], (dtype, i)
    for i, want in enumerate(want_extra):
        assert rel_err(out[250 + i], want) < TOL[dtype], (dtype, "extra", i)


def test_bench_rows_on_device():  # §8f row 3: bench-style CSV under the device engine
    from paper_1202_3777_b200 import benchcsv

    tree, tables = synth.make_config("c1")
    row = benchcsv.bench_tree("c1", tree, tables, repeats=2)
    assert set(row) == set(benchcsv.BENCH_COLUMNS)
    assert row["seq_ms"] > 0 and row["par_ms"] > 0 and 0 <= row["overhead_frac"] <= 1


@pytest.mark.parametrize("batch", [1, 7, 33])
def test_batch_odd_sizes_and_partial_micro_batches(batch):
    """Micro-batches that are not a multiple of the vector width, and a final
    partial micro-batch (40 cases in steps of `batch`)."""
    from paper_1202_3777_b200.batch import BatchPropagator

    tree, data = load_golden("c1")
    tables = synth.scaled_potentials(tree, 0)
    golden = golden_cases(data)
    cases = [golden[i % len(golden)][0] for i in range(40)]
    for mode in ("shared", "materialized"):
        bp = BatchPropagator(tree, tables, batch=batch, dtype="f64", mode=mode)
        out = bp.run(cases).cpu().numpy()
        bp.sync()
        assert out.shape[0] == 40
        for i in range(40):
            assert rel_err(out[i], golden[i % len(golden)][1]) < 1e-10, (mode, batch, i)


def test_batch_from_networks_with_components():
    """Device-initialized batches on the reference corpus (including a network
    whose tree has two components) against the reference estimator."""
    from conftest import load_corpus_networks
    from paper_1202_3777_b200.batch import BatchPropagator

    for name, tree, net, _, rows, want in load_corpus_networks():
        target = len(net.variables) - 1
        for mode in ("shared", "materialized"):
            bp = BatchPropagator(tree, None, batch=4, dtype="f64", mode=mode, query_vars=[target], net=net)
            got = bp.run(rows).cpu().numpy()
            bp.sync()
            assert rel_err(got, want) < 1e-10, (name, mode)


def test_tiny_wave_launch_modes_match_reference(monkeypatch):
    """Small single trees run their small waves as tiny-pass launches (JT_TINY=2,
    default), or the whole program as one cooperative launch with grid barriers
    (JT_TINY=1), or the general kernels only (JT_TINY=0): the same posteriors as
    the reference in every mode, fp32 and fp64, on c1, c2 and c4M."""
    for mode in ("1", "2", "0"):
        monkeypatch.setenv("JT_TINY", mode)
        for name in ("c1", "c2", "c4M"):
            tree, data = load_golden(name)
            tables = synth.scaled_potentials(tree, 0)
            for dtype in ("f32", "f64"):
                for ev, want in golden_cases(data)[:2]:
                    st = P().from_potentials(tree, tables, engine=P().CudaEngine(dtype=dtype))
                    if ev:
                        P().apply_evidence(st, ev)
                    P().belief_propagation(st)
                    got = all_posteriors(st, len(tree.cards))
                    assert rel_err(got, want) < TOL[dtype], (mode, name, dtype, ev)


def test_device_mapping_tables_random_scope_pairs():
    """K0 on the 80 reference-generated random (clique, separator) scope pairs
    (the property test_compiler.py:233-256 draws from): bit-exact, int32."""
    from conftest import GOLDEN
    import os

    d = np.load(os.path.join(GOLDEN, "mapping_tables.npz"))
    n = len([k for k in d.files if k.endswith("_ids")])
    assert n == 80
    for i in range(n):
        ids = [int(x) for x in d[f"case{i}_ids"]]
        cards = [int(x) for x in d[f"case{i}_cards"]]
        sep = [int(x) for x in d[f"case{i}_sep"]]
        all_cards = [2] * (max(ids) + 1)
        for v, c in zip(ids, cards):
            all_cards[v] = c
        # a two-clique tree: the clique, and the separator scope as its neighbour
        tree = build_tree([tuple(ids), tuple(sep)], tuple(all_cards))
        plan = P().Plan(tree, "f64")
        cid = next(c.id for c in tree.cliques if list(c.scope.ids) == ids)
        mu = plan.mapping_table(cid, 0)
        want = d[f"case{i}_mu"]
        assert mu.dtype == want.dtype and np.array_equal(mu, want), i


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_shared_state_repropagation_and_incremental_evidence(dtype):
    """a shared-base state propagated twice without a reset, and
    again after incremental evidence, must give the reference's posteriors
    (test_propagate.py:278-300 semantics), through the C ABI."""
    import ctypes as C

    from paper_1202_3777_b200 import _lib
    from paper_1202_3777_b200.batch import BatchPropagator
    from paper_1202_3777_b200._lib import i32, ptr

    tree, tables = synth.make_config("c5")
    B = 8
    cases = synth.evidence_cases(tree, B, seed=5)
    more = synth.evidence_cases(tree, B, seed=6)
    bp = BatchPropagator(tree, tables, batch=B, dtype=dtype, mode="shared")
    L = _lib.lib()
    import torch

    out = torch.empty((B, bp.cols), dtype=torch.float64, device="cuda")

    def enter(evs):
        cidx, vs, cs, xs = bp.encode(evs)
        _lib.check(L.jt_apply_evidence(bp.handle, len(vs), ptr(cidx, C.c_int32), ptr(vs, C.c_int32),
                                       ptr(cs, C.c_int32), ptr(xs, C.c_int32), None))

    def prop():
        _lib.check(L.jt_propagate_query(bp.handle, len(bp._qv), ptr(bp._qv, C.c_int32), 1,
                                        C.c_void_p(out.data_ptr()), None))
        bp.sync()
        return out.cpu().numpy()

    template = jtref.from_potentials(tree, tables)
    n = len(tree.cards)
    _lib.check(L.jt_state_reset(bp.handle, None))
    enter(cases)
    first = prop()
    want = np.stack([jtref.case_posteriors(template, ev, range(n)) for ev in cases])
    assert rel_err(first, want) < TOL[dtype]
    second = prop()  # no reset: a no-op on normalized marginals
    assert rel_err(second, want) < TOL[dtype]
    # incremental evidence on the propagated state: accumulates with the first
    extra = [{v: x for v, x in m.items() if v not in c} for c, m in zip(cases, more)]
    enter(extra)
    third = prop()
    want3 = np.stack([jtref.case_posteriors(template, {**c, **e}, range(n)) for c, e in zip(cases, extra)])
    assert rel_err(third, want3) < TOL[dtype]
    # queries on a reset state that was never propagated: base × evidence only
    _lib.check(L.jt_state_reset(bp.handle, None))
    v = i32([0])
    got = np.empty((B, tree.cards[0]))
    _lib.check(L.jt_query(bp.handle, 1, ptr(v, C.c_int32), None, 1, ptr(got, C.c_double), None))
    holder = min((c for c in tree.cliques if 0 in c.scope.ids), key=lambda c: (c.scope.size, c.id))
    t = np.asarray(tables[holder.id]).reshape(holder.scope.cards)
    marg = t.sum(axis=tuple(range(1, t.ndim)))
    assert rel_err(got, np.broadcast_to(marg / marg.sum(), got.shape)) < TOL[dtype]
    bp.close()


def test_batch_zero_mass_names_the_case():
    """Impossible evidence in one case of a micro-batch: ZeroMassError names
    that case (the reference raises per case, potential.py:181-186 via
    estimator.py:130-133); the other cases' posteriors are unaffected."""
    from paper_1202_3777_b200.batch import BatchPropagator
    from paper_1202_3777_b200.errors import ZeroMassError

    tree, tables = synth.make_config("c1")
    v = 3
    cid = tree.cpt_assignment[v]
    scope = tree.cliques[cid].scope
    pos = list(scope.ids).index(v)
    t = np.asarray(tables[cid], dtype=np.float64).reshape(scope.cards).copy()
    idx = [slice(None)] * t.ndim
    idx[pos] = 0
    t[tuple(idx)] = 0.0  # state 0 of variable 3 is impossible
    tables = list(tables)
    tables[cid] = t.ravel()
    cases = [{1: 0}] * 5 + [{v: 0}] + [{2: 1}] * 2
    for mode in ("shared", "materialized"):
        bp = BatchPropagator(tree, tables, batch=4, dtype="f64", mode=mode)
        with pytest.raises(ZeroMassError) as ei:
            bp.run(cases, to_host=True)
        assert ei.value.case == 5 and "case 5" in str(ei.value), mode
        ok = bp.run(cases[:5], to_host=True)
        template = jtref.from_potentials(tree, tables)
        want = jtref.case_posteriors(template, cases[0], range(len(tree.cards)))
        assert rel_err(ok[0], want) < 1e-10, mode


def test_state_copy_is_device_side_and_independent():
    """PropagationState.copy() (propagate.py:193-201) through jt_state_clone:
    the copy has the same tables, and evolving it leaves the original alone."""
    tree, data = load_golden("c1")
    tables = synth.scaled_potentials(tree, 0)
    st = P().from_potentials(tree, tables, engine=P().CudaEngine(dtype="f64"))
    P().apply_evidence(st, {3: 1})
    base_c = [c.copy() for c in st.clique_values]
    cp = st.copy()
    assert all(np.array_equal(a, b) for a, b in zip(cp.clique_values, base_c))
    P().apply_evidence(cp, {17: 2})
    P().belief_propagation(cp)
    assert all(np.array_equal(a, b) for a, b in zip(st.clique_values, base_c))
    P().belief_propagation(st)
    template = jtref.from_potentials(tree, tables)
    n = len(tree.cards)
    assert rel_err(all_posteriors(st, n), jtref.case_posteriors(template, {3: 1}, range(n))) < 1e-10
    assert rel_err(all_posteriors(cp, n), jtref.case_posteriors(template, {3: 1, 17: 2}, range(n))) < 1e-10
    assert st._mappings is None  # μ tables are built only when asked for
    assert st.mappings is not None


def test_estimator_rejects_bad_evidence_like_reference():
    """predict_proba raises the reference's error types
    (model.py:130-137) for unknown variables and out-of-range states."""
    from conftest import load_corpus_networks
    from paper_1202_3777_b200.errors import StateOutOfRangeError, UnknownVariableError
    from paper_1202_3777_b200.estimator import JunctionTreeEngine

    name, tree, net, _, rows, want = load_corpus_networks()[0]
    est = JunctionTreeEngine(target=net.variables[-1].name, batch=4).fit_compiled(tree, net)
    with pytest.raises(UnknownVariableError):
        est.predict_proba([{len(net.variables) + 3: 0}])
    with pytest.raises(UnknownVariableError):
        est.predict_proba([{"no-such-variable": 0}])
    with pytest.raises(StateOutOfRangeError):
        est.predict_proba([{0: net.variables[0].cardinality}])


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_unscaled_generator_potentials_and_evidence_probability(dtype):
    """Row f2: the reference generator's own potentials, not
    rescaled (uniform(0.1, 1), synth.py:105-107), on the Pigs-shaped c2 tree
    reach ~1e107 -- beyond fp32.  The power-of-two prescaling
    (jt_state: exact, tracked per table) keeps the fp32 state in range, and
    unnormalized queries restore P(e) (propagate.py:363-377,
    test_propagate.py:318-326).  Posteriors and P(e) vs the reference at
    1e-5 (fp32) / 1e-10 (fp64); host views are the exact (unscaled) tables."""
    import os

    from conftest import GOLDEN

    tree, _ = load_golden("c2")
    rng = np.random.default_rng(0)
    tables = [rng.uniform(0.1, 1.0, size=c.scope.size) for c in tree.cliques]
    g = np.load(os.path.join(GOLDEN, "c2_unscaled.npz"))
    n = len(tree.cards)
    for i in range(4):
        ev = {int(v): int(x) for v, x in g[f"ev{i}"]}
        st = P().from_potentials(tree, tables, engine=P().CudaEngine(dtype=dtype))
        if ev:
            P().apply_evidence(st, ev)
        P().belief_propagation(st)
        assert rel_err(all_posteriors(st, n), g[f"post{i}"]) < TOL[dtype], (dtype, i)
        mass = np.array([P().query_marginal(st, v, normalize_result=False).total() for v in (0, 5, 17)])
        assert rel_err(mass, g[f"mass{i}"]) < TOL[dtype], (dtype, i, mass, g[f"mass{i}"])
        top = max(float(np.max(c)) for c in st.clique_values)
        assert rel_err(top, g[f"maxabs{i}"][0]) < TOL[dtype], (dtype, i)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_unscaled_munin_shaped_tree_stays_finite(dtype):
    """On the Munin-shaped c4M tree the reference's own fp64 path overflows to
    inf/NaN with unscaled generator potentials.  Posteriors are
    invariant under per-clique rescaling, so the oracle on the same tables
    rescaled per Appendix A is the reference answer; the device gets the raw
    tables in both precisions."""
    tree, _ = load_golden("c4M")
    rng = np.random.default_rng(3)
    raw = [rng.uniform(0.1, 1.0, size=c.scope.size) for c in tree.cliques]
    parent = synth.bfs_parents(tree)
    scaled = []
    for c, t in zip(tree.cliques, raw):
        target = 1.0 if parent[c.id] == -1 else float(tree.separators[parent[c.id][1]].scope.size)
        scaled.append(t * (target / t.sum()))
    n = len(tree.cards)
    ev = synth.evidence_cases(tree, 1, seed=11)[0]
    want = jtref.case_posteriors(jtref.from_potentials(tree, scaled), ev, range(n))
    st = P().from_potentials(tree, raw, engine=P().CudaEngine(dtype=dtype))
    P().apply_evidence(st, ev)
    P().belief_propagation(st)
    got = all_posteriors(st, n)
    assert np.all(np.isfinite(got))
    assert rel_err(got, want) < TOL[dtype]


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("batch", [16, 128])
def test_shared_base_batches_with_hub_cliques(dtype, batch):
    """the Pigs-shaped c2 tree has cliques with more neighbour
    ratios + owned evidence masks than one pass carries (MAXF).  In shared-base
    mode those hubs keep per-case tables (base x evidence, children absorbed
    eagerly) while every other clique stays shared: batches run in shared mode
    (no materialized fallback) and match the reference goldens / the oracle
    (estimator.py:118-134)."""
    from paper_1202_3777_b200.batch import BatchPropagator, shared_supported

    tree, data = load_golden("c2")
    assert shared_supported(tree)
    tables = synth.scaled_potentials(tree, 0)
    golden = golden_cases(data)
    extra = synth.evidence_cases(tree, 4, seed=21)
    template = jtref.from_potentials(tree, tables)
    want_extra = [jtref.case_posteriors(template, ev, range(len(tree.cards))) for ev in extra]
    n = batch + 8
    cases = [golden[i % len(golden)][0] for i in range(n - len(extra))] + extra
    bp = BatchPropagator(tree, tables, batch=batch, dtype=dtype, mode="auto")
    assert bp.mode == "shared"
    out = bp.run(cases, to_host=True)
    for i in range(n - len(extra)):
        assert rel_err(out[i], golden[i % len(golden)][1]) < TOL[dtype], (dtype, batch, i)
    for k, want in enumerate(want_extra):
        assert rel_err(out[n - len(extra) + k], want) < TOL[dtype], (dtype, batch, "extra", k)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_virtual_separators_c5(dtype, monkeypatch):
    """c5's two 140000-entry leaf messages are gathered by their readers instead
    of stored (virtual separators): the batch program at a
    contraction-path batch size matches the reference goldens and the oracle,
    with the threshold at 0 (every qualifying leaf) and with them off."""
    from paper_1202_3777_b200.batch import BatchPropagator

    tree, data = load_golden("c5")
    tables = synth.scaled_potentials(tree, 0)
    golden = golden_cases(data)
    extra = synth.evidence_cases(tree, 4, seed=31)
    template = jtref.from_potentials(tree, tables)
    want_extra = [jtref.case_posteriors(template, ev, range(len(tree.cards))) for ev in extra]
    cases = [golden[i % len(golden)][0] for i in range(124)] + extra
    outs = []
    for on in ("1", "0"):
        monkeypatch.setenv("JT_VSEP_MIN_MB", "0")
        monkeypatch.setenv("JT_VSEP", on)
        bp = BatchPropagator(tree, tables, batch=128, dtype=dtype, mode="shared")
        out = bp.run(cases, to_host=True)
        for i in range(124):
            assert rel_err(out[i], golden[i % len(golden)][1]) < TOL[dtype], (dtype, on, i)
        for k, want in enumerate(want_extra):
            assert rel_err(out[124 + k], want) < TOL[dtype], (dtype, on, "extra", k)
        outs.append(out)
    assert rel_err(outs[0], outs[1]) < (1e-12 if dtype == "f64" else 1e-5)


def test_virtual_separators_materialised_for_later_queries(monkeypatch):
    """After a fused propagation that gathered leaf messages instead of storing
    them, a later query on the hub clique (which reads its children's collect
    messages) first materialises them: its marginals equal the fused ones."""
    import ctypes as C

    from paper_1202_3777_b200 import _lib
    from paper_1202_3777_b200._lib import i32, ptr
    from paper_1202_3777_b200.batch import BatchPropagator

    monkeypatch.setenv("JT_VSEP_MIN_MB", "0")
    tree, data = load_golden("c5")
    tables = synth.scaled_potentials(tree, 0)
    cases = [ev for ev, _ in golden_cases(data)]
    cases = [cases[i % len(cases)] for i in range(128)]
    bp = BatchPropagator(tree, tables, batch=128, dtype="f64", mode="shared")
    fused = bp.run(cases, to_host=True)
    cols = np.cumsum([0] + [int(tree.cards[v]) for v in bp.query_vars])
    hub = 2
    for v in tree.cliques[hub].scope.ids:
        k = list(bp.query_vars).index(v)
        got = np.zeros((128, int(tree.cards[v])))
        _lib.check(_lib.lib().jt_query(bp.handle, 1, ptr(i32([v]), C.c_int32), ptr(i32([hub]), C.c_int32), 1,
                                       got.ctypes.data_as(C.POINTER(C.c_double)), None), "jt_query")
        assert rel_err(got, fused[:, cols[k]:cols[k + 1]]) < 1e-10, v


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_lazy_final_separator_tables(dtype, monkeypatch):
    """A fused batch propagation does not store the final separator tables its
    queries do not read (collect message x distribute ratio); reading them back
    afterwards rebuilds them: equal to a program that stores them, for a case
    with evidence and one without (c5's 140000-entry hub separators included,
    virtual separators on)."""
    import ctypes as C

    from paper_1202_3777_b200 import _lib
    from paper_1202_3777_b200.batch import BatchPropagator

    monkeypatch.setenv("JT_VSEP_MIN_MB", "0")
    tree, data = load_golden("c5")
    tables = synth.scaled_potentials(tree, 0)
    cases = [ev for ev, _ in golden_cases(data)]
    cases = [cases[i % len(cases)] for i in range(127)] + [{}]
    seps = {}
    for lazy in ("1", "0"):
        monkeypatch.setenv("JT_LAZY_FINAL", lazy)
        bp = BatchPropagator(tree, tables, batch=128, dtype=dtype, mode="shared")
        bp.run(cases, to_host=True)
        n = sum(int(np.prod([tree.cards[v] for v in s.scope.ids])) for s in tree.separators)
        got = []
        for case in (0, 127):
            buf = np.zeros(n)
            _lib.check(_lib.lib().jt_state_store(bp.handle, case, None, buf.ctypes.data_as(C.POINTER(C.c_double))),
                       "jt_state_store")
            got.append(buf)
        seps[lazy] = np.stack(got)
        bp.close()
    assert np.all(np.isfinite(seps["1"])) and seps["1"].max() > 0
    assert rel_err(seps["1"], seps["0"]) < (1e-13 if dtype == "f64" else 1e-6)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_zero_entries_under_ratio_only_and_virtual_separators(dtype, monkeypatch):
    """Tables with exact zeros make separator entries 0: ratio-only distribute
    outputs then store Σ where the reference's ratio is 0/0 = 0, and gathered
    leaf messages are 0 there. Posteriors must still match the oracle (and the
    programs with those features off), with a hub variable's state 0 impossible."""
    from paper_1202_3777_b200.batch import BatchPropagator

    monkeypatch.setenv("JT_VSEP_MIN_MB", "0")
    tree, data = load_golden("c5")
    tables = list(synth.scaled_potentials(tree, 0))
    hub = 2
    scope = tree.cliques[hub].scope
    v = int(scope.ids[0])
    t = np.asarray(tables[hub], dtype=np.float64).reshape(scope.cards).copy()
    idx = [slice(None)] * t.ndim
    idx[0] = 0
    t[tuple(idx)] = 0.0
    tables[hub] = t.ravel()
    cases = [{k: s for k, s in ev.items() if k != v} for ev, _ in golden_cases(data)]
    cases = [cases[i % len(cases)] for i in range(124)] + synth.evidence_cases(tree, 4, seed=5)
    cases = [{k: s for k, s in ev.items() if k != v} for ev in cases]
    template = jtref.from_potentials(tree, tables)
    check = [0, 1, 2, 60, 124, 125, 126, 127]
    want = {i: jtref.case_posteriors(template, cases[i], range(len(tree.cards))) for i in check}
    outs = []
    for env in ({}, {"JT_DRATIO": "0", "JT_VSEP": "0", "JT_LAZY_FINAL": "0"}):
        for k in ("JT_DRATIO", "JT_VSEP", "JT_LAZY_FINAL"):
            monkeypatch.delenv(k, raising=False)
        for k, x in env.items():
            monkeypatch.setenv(k, x)
        bp = BatchPropagator(tree, tables, batch=128, dtype=dtype, mode="shared")
        out = bp.run(cases, to_host=True)
        for i in check:
            assert rel_err(out[i], want[i]) < TOL[dtype], (dtype, env, i)
        outs.append(out)
        bp.close()
    assert np.all(np.isfinite(outs[0]))
    assert rel_err(outs[0], outs[1]) < (1e-12 if dtype == "f64" else 1e-5)
