"""Benchmark: junction-tree propagations/s on B200 (BASELINE.json metric).

Workload (config 5): batches of evidence cases on the Mildew-shaped synthetic
junction tree (28 cliques, Σ|φ| = 8.03M entries, fp32),
one full propagation (reset → evidence → collect+distribute → posteriors of
all 32 variables) per case.  One "step" = CASES_PER_GPU cases on every GPU
(weak scaling: the cases shard across GPUs with no data-path collective; the
posteriors are gathered to rank 0 with one NCCL gather per step).

  value  : cases/s over all ranks, evidence already resident in HBM.
  e2e    : same metric through the public API (BatchPropagator) with the
           evidence in pinned host memory and posteriors copied back to host
           inside the timed region.
  roofline: the propagation program (wave kernels) of one micro-batch;
           algorithmic bytes = B_alg1 × cases in the micro-batch.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
For N>1 the driver launches it with torch.distributed.run (one rank per GPU,
NCCL); run directly with --gpus N > 1 it re-launches itself that way (and, on a
box with fewer GPUs than N, as an N-rank gloo smoke sharing GPU 0).

The headline (`value`, `e2e`, `roofline`) is fp64, the reference's own
arithmetic (propagate.py:214-240); the fp32 mode is reported beside it under
the key "f32" with its own roofline.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def baseline_metric():
    """Both arms print BASELINE.json's metric string verbatim (the driver pairs
    the arms by metric, unit and direction)."""
    try:
        with open(os.path.join(ROOT, "BASELINE.json")) as f:
            return json.load(f)["metric"]
    except Exception:
        return "JT propagations/sec (collect+distribute); achieved HBM GB/s vs B200 peak"


METRIC = baseline_metric()
UNIT = "cases/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c5")
    ap.add_argument("--cases", type=int, default=8192, help="evidence cases per GPU per step")
    ap.add_argument("--batch", type=int, default=4096, help="cases per device micro-batch")
    ap.add_argument("--dtype", default="f64", choices=["f32", "f64"])
    ap.add_argument("--mode", default="auto", choices=["auto", "shared", "materialized"])
    ap.add_argument("--cpu-sample", type=int, default=24, help="cases in the CPU baseline sample")
    ap.add_argument("--ref-sample", type=int, default=4, help="cases per step of the reference arm")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the single-tree per-config table")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def measured_traffic(config, dtype, batch):
    """DRAM bytes (read + write) of one micro-batch program, summed from the ncu
    launch list committed under profiles/ (tools/traffic_from_ncu.py), or None."""
    p = os.path.join(ROOT, "profiles", f"traffic_{config}_{dtype}_b{batch}.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return None


def compulsory_bytes(tree, batch, dtype, mode):
    """The planner's compulsory HBM traffic of one micro-batch program (every
    factor tensor read once, outputs written once)."""
    try:
        import ctypes as C

        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import plan_report
        from paper_1202_3777_b200 import _lib

        h, _keep = plan_report.plan_handle(tree, dtype)
        buf = C.create_string_buffer(1 << 22)
        _lib.check(_lib.lib().jt_debug_plan(h, batch, 1 if mode == "shared" else 0, 1, 148, 2, buf, len(buf)))
        _lib.lib().jt_plan_destroy(h)
        for line in buf.value.decode().splitlines():
            if line.startswith("compulsory total MB"):
                return float(line.split()[-1]) * 1e6
    except Exception:
        return None
    return None


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return dict(PEAKS_FALLBACK), "fallback"


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------- CPU legs ----
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _reference_module():
    """The unmodified reference package (`jtprop`), installed by
    `pip install --no-deps --target baseline/_ref`; None if absent."""
    if not os.path.isdir(os.path.join(REF_DIR, "jtprop")):
        return None
    if REF_DIR not in sys.path:
        sys.path.append(REF_DIR)
    try:
        import jtprop.compiler
        import jtprop.propagate
        return jtprop
    except Exception:
        return None


def cpu_case_rate(config, tree, tables, cases, variables, workers):
    """The reference's per-case loop (estimator.py:89-96): copy → apply_evidence
    → belief_propagation → every query_marginal, with the reference's
    ParallelEngine (propagate.py:97-161) over `workers` threads.  Runs the real
    `jtprop` when it is installed under baseline/_ref (kind "reference"), else
    the oracle port (kind "port").  Returns (cases/s, seconds, kind)."""
    ref = _reference_module()
    if ref is not None:
        from paper_1202_3777_b200 import synth

        members, cards = synth.config_members(config)
        rtree = ref.compiler.build_tree(members, cards)
        rtree.cpt_assignment = dict(tree.cpt_assignment)
        P = ref.propagate
        eng = P.make_engine("parallel" if workers > 1 else "sequential", workers=workers)
        template = P.from_potentials(rtree, tables, engine=eng)
        t0 = time.perf_counter()
        for ev in cases:
            st = template.copy()
            if ev:
                P.apply_evidence(st, ev)
            P.belief_propagation(st)
            for v in variables:
                P.query_marginal(st, v)
        dt = time.perf_counter() - t0
        eng.close()
        return len(cases) / dt, dt, "reference"
    from oracle import jtref

    eng = jtref.ParallelEngine(workers) if workers > 1 else jtref.SequentialEngine()
    template = jtref.from_potentials(tree, tables, engine=eng)
    t0 = time.perf_counter()
    for ev in cases:
        jtref.case_posteriors(template, ev, variables)
    dt = time.perf_counter() - t0
    eng.close()
    return len(cases) / dt, dt, "port"


# -------------------------------------------------------------- GPU leg ----
def single_tree_table(dtype_list=("f32", "f64"), configs=("c1", "c2", "c3", "c4B", "c4M", "c5")):
    """Per-config single-tree propagations/s (jt_propagate, state reset outside
    the timer, median of CUDA-event timings) and B_alg1 roofline fraction."""
    import ctypes as C

    import torch

    from paper_1202_3777_b200 import _lib
    from paper_1202_3777_b200 import propagate as P
    from paper_1202_3777_b200 import synth
    from paper_1202_3777_b200.tree import algorithmic_elements

    pk, _ = peaks()
    out = {}
    L = _lib.lib()
    for name in configs:
        tree, tables = synth.make_config(name)
        alg = algorithmic_elements(tree)
        for dt in dtype_list:
            st = P.from_potentials(tree, tables, engine=P.CudaEngine(dtype=dt))
            s = torch.cuda.Stream()
            h = C.c_void_p(s.cuda_stream)
            times = []
            for i in range(25):
                L.jt_state_reset(st.handle, h)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                _lib.check(L.jt_propagate(st.handle, None, h))
                e1.record(s)
                s.synchronize()
                if i >= 5:
                    times.append(e0.elapsed_time(e1) * 1e-3)
            st.sync()
            t = statistics.median(times)
            b = 4 if dt == "f32" else 8
            gbs = alg * b / t / 1e9
            out[f"{name}_{dt}"] = {"props_per_s": round(1.0 / t, 2), "ms": round(t * 1e3, 4),
                                   "alg_GBps": round(gbs, 1), "frac_hbm": round(gbs / pk["hbm_gbs"], 3)}
            del st
    return out


def relaunch(args):
    """`python bench.py --gpus N` outside torchrun: start N ranks through
    torch.distributed.run (127.0.0.1 rendezvous).  With fewer visible GPUs than
    N every rank shares GPU 0 over gloo (a functional smoke of the multi-rank
    path; the line says so in config.parallelism)."""
    import socket

    import torch

    env = dict(os.environ)
    if torch.cuda.device_count() < args.gpus:
        env["BENCH_DEVICE_OVERRIDE"] = "0"
        env["BENCH_DIST_BACKEND"] = "gloo"
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd, env=env))


def golden_sample(config, n_cases, seed=1234):
    """Reference posteriors of a sample of this workload's cases covering both
    micro-batches (tests/golden/c5_bench.npz, made by running the reference:
    tests/golden/make_golden.py bench); None when the workload differs."""
    p = os.path.join(ROOT, "tests", "golden", f"{config}_bench.npz")
    if not os.path.exists(p):
        return None
    d = np.load(p)
    if int(d["seed"][0]) != seed:
        return None
    keep = d["idx"] < n_cases
    return d["idx"][keep], d["post"][keep]


def rel_err(got, want):
    return float(np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-300)))


def measure(args, dtype, tree, tables, cases, world, rank, local, dist, primary):
    """Time K steps of one dtype: device-resident evidence (value), then the
    public API from Python evidence dicts to host posteriors (e2e)."""
    import ctypes as C

    import torch

    from paper_1202_3777_b200 import _lib
    from paper_1202_3777_b200.batch import BatchPropagator

    dev = torch.device("cuda", local)
    n_vars = len(tree.cards)
    n_cases = len(cases)
    B = min(args.batch, n_cases)
    steps_mb = (n_cases + B - 1) // B
    bp = BatchPropagator(tree, tables, batch=B, dtype=dtype, mode=args.mode, device=local)
    stream = bp.stream
    sh = C.c_void_p(stream.cuda_stream)
    L = _lib.lib()

    def barrier():
        if world > 1:
            dist.barrier()

    obs_host = [bp.encode_obs(cases[m * B:(m + 1) * B]) for m in range(steps_mb)]
    obs_dev = [torch.from_numpy(o).to(dev) for o in obs_host]
    post = torch.empty((steps_mb * B, bp.cols), dtype=torch.float64, device=dev)
    gathered = torch.empty((world * steps_mb * B, bp.cols), dtype=torch.float64, device=dev) \
        if (world > 1 and rank == 0) else None
    prog_events = []

    def gather(src):
        if world > 1:
            with torch.cuda.stream(stream):
                dist.gather(src, [gathered[r * steps_mb * B:(r + 1) * steps_mb * B] for r in range(world)]
                            if rank == 0 else None, dst=0)

    def one_step(record=False):
        for m in range(steps_mb):
            if record:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            bp.step_device(obs_dev[m], post[m * B:(m + 1) * B], sh)
            if record:
                e1.record(stream)
                prog_events.append((e0, e1))
        gather(post)

    # warm-up (also builds and graph-captures the programs)
    for _ in range(max(args.warmup, 3)):
        one_step()
    stream.synchronize()
    bp.sync()

    clocks = ClockSampler(local) if primary else None
    barrier()
    torch.cuda.synchronize()
    if clocks:
        clocks.start()
    launches0 = bp.launches()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        one_step(record=True)
    t1.record(stream)
    t1.synchronize()
    barrier()
    torch.cuda.synchronize()
    clock_info = clocks.stop() if clocks else None
    launches = bp.launches() - launches0
    ms = t0.elapsed_time(t1) / args.steps
    if world > 1:
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    bp.sync()
    value = world * n_cases / (ms * 1e-3)
    # the program launches interleave with reset/evidence kernels on the same
    # stream: per-micro-batch program time (events bracket jt_propagate_query
    # plus the reset/evidence launches of its step)
    prog_ms = statistics.mean(a.elapsed_time(b) for a, b in prog_events) if prog_events else None

    # e2e: the public API (BatchPropagator.run) from Python evidence dicts to host
    # posteriors -- encode, pinned H2D of the observations, device step, D2H of the
    # posteriors -- every step; multi-rank: gather to rank 0 and read it back there
    e2e = None
    host_post = None
    if not args.no_e2e:
        def e2e_step():
            if world == 1:
                return bp.run(cases, to_host=True)
            out = bp.run(cases, out=post)
            stream.wait_stream(torch.cuda.current_stream(dev))
            gather(post)
            bp.sync()
            return gathered.cpu().numpy() if rank == 0 else None

        for _ in range(2):
            e2e_step()
        barrier()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        for _ in range(args.steps):
            host_post = e2e_step()
        barrier()
        torch.cuda.synchronize()
        e_ms = (time.perf_counter() - w0) * 1e3 / args.steps
        if world > 1:
            tt = torch.tensor([e_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e_ms = float(tt.item())
        h2d = sum(int(o.size) * 4 for o in obs_host)
        e2e = {"value": round(world * n_cases / (e_ms * 1e-3), 2), "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": int(n_cases * bp.cols * 8 * (world if world > 1 else 1)),
               "ms_per_step": round(e_ms, 3),
               "path": "BatchPropagator.run(list of evidence dicts, to_host=True): encode + pinned H2D of "
                       "int32 observations + device step + D2H of float64 posteriors"}

    # correctness of this run: reference goldens over both micro-batches (rank 0)
    spot = None
    if rank == 0:
        gs = golden_sample(args.config, n_cases)
        got = post.cpu().numpy()
        if gs is not None and len(gs[0]):
            idx, want = gs
            spot = {"cases": int(len(idx)), "micro_batches": sorted({int(i) // B for i in idx}),
                    "max_rel_err": rel_err(got[idx], want),
                    "against": f"reference jtprop posteriors (tests/golden/{args.config}_bench.npz)"}
            if host_post is not None:
                spot["e2e_max_rel_err"] = rel_err(host_post[idx], want)
        else:
            from oracle import jtref

            idx = sorted({0, B - 1, min(B, n_cases - 1), n_cases - 1})
            template = jtref.from_potentials(tree, tables)
            want = np.stack([jtref.case_posteriors(template, cases[i], range(n_vars)) for i in idx])
            spot = {"cases": len(idx), "max_rel_err": rel_err(got[idx], want), "against": "oracle/jtref.py"}
    res = {"value": value, "ms": ms, "prog_ms": prog_ms, "launches": int(launches), "clocks": clock_info,
           "e2e": e2e, "spot": spot, "mode": bp.mode, "B": B}
    bp.close()
    del post, gathered, obs_dev
    torch.cuda.empty_cache()
    return res


def roofline_block(args, tree, dtype, r, alg_elems):
    pk, pk_kind = peaks()
    esz = 4 if dtype == "f32" else 8
    B = r["B"]
    prog_ms = r["prog_ms"]
    alg_bytes_launch = alg_elems * esz * B
    achieved = alg_bytes_launch / (prog_ms * 1e-3) / 1e9
    comp = compulsory_bytes(tree, B, dtype, r["mode"])
    traffic = measured_traffic(args.config, dtype, B)
    # achieved/frac use the compulsory bytes of the algorithm that runs (every factor
    # tensor read once, every output written once): the shared-base
    # batch path never moves per-case clique tables, so B_alg1 (materialized-
    # equivalent bytes) is reported beside it, not as the denominator
    return {"bound": "hbm",
            "achieved": round(comp / (prog_ms * 1e-3) / 1e9, 1) if comp else round(achieved, 1),
            "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": round(comp / (prog_ms * 1e-3) / 1e9 / pk["hbm_gbs"], 3) if comp
            else round(achieved / pk["hbm_gbs"], 3),
            "traffic": traffic["bytes_per_launch"] if traffic else None,
            "kernel": "propagation program of one micro-batch (reset + evidence masks + jt_propagate_query: "
                      "contraction, thread-owned and general wave kernels)",
            "alg_bytes_per_launch": comp if comp else alg_bytes_launch,
            "alg_bytes_def": "compulsory bytes of the shared-base program: factor tensors read once, "
                             "outputs written once, separator updates read old + write ratio (+ final table "
                             "unless rebuilt on demand); virtual separators (gathered leaf messages) move no "
                             "bytes (planner, DESIGN.md 3b/5)" if comp else "B_alg1 x cases",
            "b_alg1_bytes_per_launch": alg_bytes_launch,
            "frac_b_alg1": round(achieved / pk["hbm_gbs"], 3),
            "physical_frac": round(traffic["bytes_per_launch"] / (prog_ms * 1e-3) / 1e9 / pk["hbm_gbs"], 3)
            if traffic else None,
            "traffic_source": traffic.get("source") if traffic else None,
            "launch_ms": round(prog_ms, 4), "peak_kind": pk_kind}


def batch_table(configs=("c2", "c4M"), dtypes=("f64", "f32"), n_cases=4096, batch=2048, steps=5):
    """Evidence batches on the other config shapes (shared-base mode; hub cliques
    keep per-case tables): cases/s with evidence resident on the device, and the
    oracle spot check of two cases from different micro-batches."""
    import ctypes as C

    import torch

    from oracle import jtref
    from paper_1202_3777_b200 import synth
    from paper_1202_3777_b200.batch import BatchPropagator

    out = {}
    for name in configs:
        tree, tables = synth.make_config(name)
        cases = synth.evidence_cases(tree, n_cases, seed=1234)
        template = jtref.from_potentials(tree, tables)
        check = (1, n_cases - 1)
        want = np.stack([jtref.case_posteriors(template, cases[i], range(len(tree.cards))) for i in check])
        for dt in dtypes:
            bp = BatchPropagator(tree, tables, batch=batch, dtype=dt, mode="auto")
            sh = C.c_void_p(bp.stream.cuda_stream)
            obs = [torch.from_numpy(bp.encode_obs(cases[m:m + batch])).cuda() for m in range(0, n_cases, batch)]
            post = torch.empty((n_cases, bp.cols), dtype=torch.float64, device="cuda")

            def step():
                for k, o in enumerate(obs):
                    bp.step_device(o, post[k * batch:(k + 1) * batch], sh)

            for _ in range(3):
                step()
            bp.stream.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(bp.stream)
            for _ in range(steps):
                step()
            e1.record(bp.stream)
            e1.synchronize()
            bp.sync()
            ms = e0.elapsed_time(e1) / steps
            got = post[list(check)].cpu().numpy()
            out[f"{name}_{dt}"] = {"cases_per_s": round(n_cases / (ms * 1e-3), 1), "ms_per_step": round(ms, 3),
                                  "micro_batch": batch, "mode": bp.mode,
                                  "spot_max_rel_err": rel_err(got, want)}
            bp.close()
            del post, obs
            torch.cuda.empty_cache()
    return out


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl != "reference":
        relaunch(args)

    from paper_1202_3777_b200 import synth
    from paper_1202_3777_b200.tree import algorithmic_elements

    tree, tables = synth.make_config(args.config)
    n_vars = len(tree.cards)
    alg_elems = algorithmic_elements(tree)

    # ------------------------------------------------------ reference arm --
    if args.impl == "reference":
        if rank != 0:
            return
        workers = os.cpu_count() or 1
        cases_all = synth.evidence_cases(tree, args.ref_sample * (args.steps + args.warmup), seed=1234)
        rates = []
        for s in range(args.warmup + args.steps):
            chunk = cases_all[s * args.ref_sample:(s + 1) * args.ref_sample]
            r, _, kind = cpu_case_rate(args.config, tree, tables, chunk, range(n_vars), workers)
            if s >= args.warmup:
                rates.append(r)
        v = statistics.median(rates)
        line = {"impl": "reference", "metric": METRIC,
                "value": round(v, 4), "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(args.ref_sample / v * 1e3, 2),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": f"{args.config}: Mildew-shaped synthetic JT (SURVEY Appendix A), per-case "
                                       "copy→evidence→BP→posteriors of all variables (estimator.py:89-134)",
                           "cases_per_step": args.ref_sample},
                "cpu_baseline": {"value": round(v, 4), "unit": UNIT, "cores": workers, "kind": kind,
                                 "sample": f"{args.ref_sample} cases/step × {args.steps} steps, "
                                           + ("unmodified jtprop from baseline/_ref" if kind == "reference"
                                              else "oracle/jtref.py (numpy restatement of jtprop)")
                                           + f", ParallelEngine({workers} threads), per-case "
                                             "copy→evidence→BP→all posteriors"},
                "e2e": {"value": round(v, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist

    # BENCH_DEVICE_OVERRIDE / BENCH_DIST_BACKEND: the multi-rank path on a box with
    # fewer GPUs than ranks (every rank on one device, gloo); production runs use
    # NCCL, one GPU per rank
    shared_dev = os.environ.get("BENCH_DEVICE_OVERRIDE") is not None
    if shared_dev:
        local = int(os.environ["BENCH_DEVICE_OVERRIDE"])
        # every rank's state on one device: shrink the micro-batch to fit
        args.batch = max(256, args.batch // world)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    n_cases = args.cases
    cases = synth.evidence_cases(tree, n_cases, seed=1234, first=rank * n_cases)
    r = measure(args, args.dtype, tree, tables, cases, world, rank, local, dist, primary=True)
    extra = None
    if not args.no_extra and world == 1:
        other = "f32" if args.dtype == "f64" else "f64"
        extra = measure(args, other, tree, tables, cases, world, rank, local, dist, primary=False)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    B = r["B"]
    line = {
        "metric": METRIC,
        "value": round(r["value"], 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": round(r["ms"], 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": {"workload": f"{args.config}: Mildew-shaped synthetic JT (28 cliques, Σ|φ|=8.03M), "
                               f"{n_cases} evidence cases per GPU per step, full collect+distribute + "
                               f"posteriors of all {n_vars} variables per case",
                   "cases_per_gpu": n_cases, "micro_batch": B, "mode": r["mode"],
                   "l2": "per-micro-batch separator/ratio working set > L2 (126 MB); base replica "
                         "L2-resident by design",
                   "parallelism": f"dp{world} (evidence shards, NCCL gather of posteriors)"
                   if not shared_dev else f"dp{world} smoke: {world} gloo ranks sharing GPU {local}"},
        "roofline": roofline_block(args, tree, args.dtype, r, alg_elems),
        "e2e": r["e2e"],
        "gpu_launches": r["launches"],
        "clocks": r["clocks"],
        "spot_check": r["spot"],
    }
    if extra is not None:
        line[("f32" if args.dtype == "f64" else "f64")] = {
            "value": round(extra["value"], 2), "unit": UNIT, "ms_per_step": round(extra["ms"], 3),
            "micro_batch": extra["B"], "mode": extra["mode"],
            "roofline": roofline_block(args, tree, "f32" if args.dtype == "f64" else "f64", extra, alg_elems),
            "e2e": extra["e2e"], "gpu_launches": extra["launches"], "spot_check": extra["spot"]}
    if not args.no_cpu_baseline and world == 1:
        workers = os.cpu_count() or 1
        sample = synth.evidence_cases(tree, args.cpu_sample, seed=1234)
        rr, dt, kind = cpu_case_rate(args.config, tree, tables, sample, range(n_vars), workers)
        line["cpu_baseline"] = {"value": round(rr, 4), "unit": UNIT, "cores": workers, "kind": kind,
                                "sample": f"{args.cpu_sample} cases of the same workload, per-case "
                                          f"copy→evidence→BP→posteriors, "
                                          + ("unmodified jtprop (baseline/_ref)" if kind == "reference"
                                             else "oracle/jtref.py") + f" ParallelEngine ({dt:.1f}s)"}
    if not args.no_extra and world == 1:
        try:
            line["single_tree"] = single_tree_table()
        except Exception as exc:  # report, never hide
            line["single_tree"] = {"error": repr(exc)}
        try:
            line["batch_other"] = batch_table()
        except Exception as exc:
            line["batch_other"] = {"error": repr(exc)}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
