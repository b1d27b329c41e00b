"""`jtprop bench`-style rows for the device engine (cli.py:46-49, 289-347 of the
reference).

Same columns as the reference's BENCH_COLUMNS, measured on the GPU:

* seq_ms   — the paper's schedule: one Alg. 1 message per launch (2(n-1)
             `jt_message` calls in the reference's DFS order, propagate.py:296-334);
* par_ms   — the level-batched program (`jt_propagate`, one CUDA graph);
* speedup  — seq_ms / par_ms;
* tau_est  — per-message launch overhead fitted on per-message CUDA-event
             timings with the reference's least-squares model (perfmodel.py:115-150:
             time = tau + work / throughput, work = source + target size);
* pred_speedup — that model's prediction of the batching gain:
             Σ(tau + w/θ) / (launches_of_program · tau + Σ w/θ);
* overhead_frac — n_messages · tau / seq time: the share of per-message execution
             spent on launch overhead (the paper's analysis).

usage: python -m paper_1202_3777_b200.benchcsv c1 c2 tree.jt.json ... [--format csv|json] [--repeats 5]
"""

from __future__ import annotations

import argparse
import csv
import ctypes as C
import json
import statistics
import sys

import numpy as np

BENCH_COLUMNS = ("tree", "n_cliques", "avg_spt", "seq_ms", "par_ms", "speedup", "pred_speedup", "tau_est",
                 "overhead_frac")


def estimate_tau(samples):
    """(tau, throughput) by least squares of time = tau + work / throughput
    (perfmodel.py:115-150): non-positive slope → overhead dominated (tau = mean
    time, throughput inf); negative intercept clamped to 0."""
    work = np.asarray([s[0] for s in samples], dtype=np.float64)
    time = np.asarray([s[1] for s in samples], dtype=np.float64)
    if len(work) < 2 or np.ptp(work) == 0.0:
        return float(max(time.mean(), 0.0)) if len(time) else 0.0, np.inf
    wbar, tbar = work.mean(), time.mean()
    slope = float(((work - wbar) * (time - tbar)).sum() / ((work - wbar) ** 2).sum())
    if slope <= 0.0:
        return float(max(tbar, 0.0)), np.inf
    return float(max(tbar - slope * wbar, 0.0)), 1.0 / slope


def _messages(tree):
    from .propagate import _children_first_order

    out = []
    for r in tree.roots:
        out += [(c, p, s) for c, p, s in _children_first_order(tree, r)]
        stack = [(r, -1, -1)]
        while stack:
            node, parent, sep_id = stack.pop()
            if parent >= 0:
                out.append((parent, node, sep_id))
            for nbr, s in reversed(tree.neighbors[node]):
                if nbr != parent:
                    stack.append((nbr, node, s))
    return out


def bench_tree(name, tree, tables, repeats=5, dtype="f32"):
    import torch

    from . import _lib
    from . import propagate as P

    L = _lib.lib()
    st = P.from_potentials(tree, tables, engine=P.CudaEngine(dtype=dtype))
    s = torch.cuda.Stream()
    h = C.c_void_p(s.cuda_stream)
    msgs = _messages(tree)
    sizes = [c.scope.size for c in tree.cliques]

    def ev():
        return torch.cuda.Event(enable_timing=True)

    # warm-up: builds and caches every per-message program and the batched one
    L.jt_state_reset(st.handle, h)
    for m in msgs:
        _lib.check(L.jt_message(st.handle, m[0], m[1], m[2], h))
    L.jt_state_reset(st.handle, h)
    _lib.check(L.jt_propagate(st.handle, None, h))
    L.jt_state_reset(st.handle, h)
    _lib.check(L.jt_propagate(st.handle, None, h))
    s.synchronize()
    seq, par, per_msg = [], [], [[] for _ in msgs]
    for _ in range(repeats):
        L.jt_state_reset(st.handle, h)
        e = [ev() for _ in range(len(msgs) + 1)]
        e[0].record(s)
        for i, m in enumerate(msgs):
            L.jt_message(st.handle, m[0], m[1], m[2], h)
            e[i + 1].record(s)
        L.jt_state_reset(st.handle, h)
        p0, p1 = ev(), ev()
        launches0 = L.jt_state_launch_count(st.handle)
        p0.record(s)
        _lib.check(L.jt_propagate(st.handle, None, h))
        p1.record(s)
        n_par_launches = L.jt_state_launch_count(st.handle) - launches0
        s.synchronize()
        seq.append(e[0].elapsed_time(e[-1]) * 1e-3)
        par.append(p0.elapsed_time(p1) * 1e-3)
        for i in range(len(msgs)):
            per_msg[i].append(e[i].elapsed_time(e[i + 1]) * 1e-3)
    st.sync()
    work = [sizes[m[0]] + sizes[m[1]] for m in msgs]  # MessageCost.sequential_ops, perfmodel.py:37-39
    tau, theta = estimate_tau([(w, statistics.median(t)) for w, t in zip(work, per_msg)])
    seq_s, par_s = statistics.median(seq), statistics.median(par)
    compute = sum(work) / theta if np.isfinite(theta) else 0.0
    pred = (len(msgs) * tau + compute) / (n_par_launches * tau + compute) if (tau or compute) else 1.0
    seps = [sp.scope.size for sp in tree.separators]
    return {"tree": name, "n_cliques": len(tree.cliques), "avg_spt": float(np.mean(seps)) if seps else 0.0,
            "seq_ms": seq_s * 1e3, "par_ms": par_s * 1e3, "speedup": seq_s / par_s if par_s > 0 else float("inf"),
            "pred_speedup": pred, "tau_est": tau,
            "overhead_frac": min(len(msgs) * tau / seq_s, 1.0) if seq_s > 0 else 0.0}


def _load(spec):
    from . import synth

    if spec.endswith(".json"):
        from . import io
        from .propagate import initialize

        tree, net = io.load_tree(spec)
        if net is None:
            raise ValueError(f"{spec}: tree dump carries no network")
        st = initialize(tree, net)
        return tree, [np.array(v) for v in st.clique_values]
    return synth.make_config(spec)


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("inputs", nargs="+", help="config names (c1..c5) or jtprop-tree .json dumps")
    ap.add_argument("--format", choices=("csv", "json"), default="csv")
    ap.add_argument("--repeats", type=int, default=5)
    ap.add_argument("--dtype", default="f32")
    a = ap.parse_args(argv)
    rows = []
    for spec in a.inputs:
        tree, tables = _load(spec)
        rows.append(bench_tree(spec, tree, tables, a.repeats, a.dtype))
    if a.format == "json":
        print(json.dumps(rows, indent=1))
    else:
        w = csv.writer(sys.stdout)
        w.writerow(BENCH_COLUMNS)
        for r in rows:
            w.writerow([r["tree"], r["n_cliques"], f"{r['avg_spt']:.1f}", f"{r['seq_ms']:.3f}", f"{r['par_ms']:.3f}",
                        f"{r['speedup']:.3f}", f"{r['pred_speedup']:.3f}", f"{r['tau_est']:.6g}",
                        f"{r['overhead_frac']:.4f}"])
    return 0


if __name__ == "__main__":
    sys.exit(main())
