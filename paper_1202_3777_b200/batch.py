"""Batched evidence cases on one device: the config-5 path.

The reference answers a list of evidence cases one propagation at a time
(`JunctionTreeEngine.predict_proba`, estimator.py:118-134: initialize →
apply_evidence → belief_propagation → query_marginal per case).  Here a batch
of cases is one device state whose tables carry the case as the innermost
(stride-1) index, so every kernel access is coalesced across cases:

* mode "shared"  (JT_SHARED_BASE): the clique tables live once (the base
  replica); each case's evidence masks and every separator ratio enter the
  passes as factors, and clique tables are never written — the per-case HBM
  traffic is separator-sized.  Posteriors are reduced inside the distribute
  waves.
* mode "materialized" (JT_MATERIALIZED): every case owns a copy of every
  clique table (reset on device from the base replica), i.e. exactly the
  reference's state semantics, micro-batched to fit HBM.

Multi-GPU: one process per GPU; rank r takes a contiguous shard of the cases
and generates / receives only its own evidence (no scatter).  Posteriors are
gathered with one NCCL all-gather (`gather_posteriors`).
"""

from __future__ import annotations

import ctypes as C
from itertools import chain
from operator import methodcaller

import numpy as np

from . import _lib
from ._lib import JT_MATERIALIZED, JT_SHARED_BASE, check, f64, i32, ptr
from .errors import StateOutOfRangeError, UnknownVariableError, ZeroMassError
from .propagate import _scope_size, plan_for

_values = methodcaller("values")

MODES = {"shared": JT_SHARED_BASE, "materialized": JT_MATERIALIZED}
MAX_FACTORS = 8  # jt::MAXF


def _owners(tree):
    owner = dict(getattr(tree, "cpt_assignment", {}) or {})
    for v in range(len(tree.cards)):
        if v not in owner:
            holders = [c for c in tree.cliques if v in c.scope.ids]
            if holders:
                owner[v] = min(holders, key=lambda c: (_scope_size(c.scope), c.id)).id
    return owner


def _smallest_holder_counts(tree):
    counts = {}
    for v in range(len(tree.cards)):
        holders = [c for c in tree.cliques if v in c.scope.ids]
        if holders:
            c = min(holders, key=lambda c: (_scope_size(c.scope), c.id)).id
            counts[c] = counts.get(c, 0) + 1
    return counts


def shared_supported(tree) -> bool:
    """Shared-base passes carry every factor of a clique at once (neighbours'
    ratios plus one evidence mask per variable the clique owns, <= MAX_FACTORS).
    Hub cliques beyond that keep per-case tables (the library allocates them for
    cliques over the limit under smallest-holder ownership, jt_state::hub), so
    the mode is supported unless the tree's own evidence assignment puts more
    factors on a clique that is not such a hub."""
    hub_owned = _smallest_holder_counts(tree)
    hub = {c for c in range(len(tree.cliques)) if len(tree.neighbors[c]) + hub_owned.get(c, 0) > MAX_FACTORS}
    owned = {}
    for v, c in _owners(tree).items():
        owned[c] = owned.get(c, 0) + 1
    return all(len(tree.neighbors[c]) + owned.get(c, 0) <= MAX_FACTORS or c in hub
               for c in range(len(tree.cliques)))


class BatchPropagator:
    """`batch` evidence cases per device step over one tree.

    run(cases) → posteriors [len(cases), Σ_v card(v)] of `query_vars`
    (normalized), computed `batch` cases per step.
    """

    def __init__(self, tree, clique_tables, batch, dtype="f32", mode="auto", device=0,
                 query_vars=None, net=None):
        _lib.require_device()
        import torch

        self.tree = tree
        self.batch = int(batch)
        if mode == "auto":
            mode = "shared" if shared_supported(tree) else "materialized"
        elif mode == "shared" and not shared_supported(tree):
            raise ValueError(f"shared-base mode needs <= {MAX_FACTORS} factors per clique "
                             "(children + parent + observed variables); use mode='materialized'")
        self.mode = mode
        self.device = int(device)
        self.plan = plan_for(tree, dtype, device)
        h = C.c_void_p()
        check(_lib.lib().jt_state_create(self.plan.handle, self.batch, MODES[mode], C.byref(h)),
              "jt_state_create")
        self.handle = h
        import weakref

        self._fin = weakref.finalize(self, _lib.lib().jt_state_destroy, h)
        if clique_tables is None:
            # base tables = CPT products, formed on the device (initialize, propagate.py:204-222)
            if net is None:
                raise ValueError("need clique_tables or a network (net=) to initialize from")
            from .propagate import cpt_arrays

            cl, off, vs, vals, n = cpt_arrays(tree, net)
            check(_lib.lib().jt_state_initialize(self.handle, n, ptr(cl, C.c_int32), ptr(off, C.c_int32),
                                                 ptr(vs, C.c_int32), ptr(vals, C.c_double)), "initialize")
        else:
            cat = f64(np.concatenate([np.asarray(t, dtype=np.float64).ravel() for t in clique_tables]))
            if cat.size != sum(self.plan.clique_sizes):
                raise ValueError("clique tables do not match the tree")
            check(_lib.lib().jt_state_load(self.handle, -1, ptr(cat, C.c_double), None), "jt_state_load")
        self.query_vars = list(range(len(tree.cards))) if query_vars is None else list(query_vars)
        self.cards = [int(tree.cards[v]) for v in self.query_vars]
        self.cols = int(sum(self.cards))
        self._qv = i32(self.query_vars)
        self.owner = _owners(tree)
        self.torch_device = torch.device("cuda", self.device)
        # all device work of this propagator is ordered on one non-default torch
        # stream (graph-capturable); callers' streams join it in run()
        self.stream = torch.cuda.Stream(device=self.torch_device)

    @property
    def device_bytes(self) -> int:
        return int(_lib.lib().jt_state_device_bytes(self.handle))

    def launches(self) -> int:
        return int(_lib.lib().jt_state_launch_count(self.handle))

    def encode(self, cases):
        """(case, var, clique, value) int32 arrays for jt_apply_evidence."""
        obs = self.encode_obs(cases)
        own = self._owner_arr[obs[:, 1]] if len(obs) else np.zeros(0, np.int32)
        return i32(obs[:, 0]), i32(obs[:, 1]), i32(own), i32(obs[:, 2])

    def step(self, encoded, out, stream=None):
        """One device step over ≤ batch cases: reset, evidence, propagate and
        posteriors into `out` (a CUDA double tensor [batch, cols]), enqueued on
        `stream` (default: this propagator's stream)."""
        cidx, vs, cs, xs = encoded
        L = _lib.lib()
        stream = self._raw_stream(stream)
        check(L.jt_state_reset(self.handle, stream), "reset")
        if len(vs):
            check(L.jt_apply_evidence(self.handle, len(vs), ptr(cidx, C.c_int32), ptr(vs, C.c_int32),
                                      ptr(cs, C.c_int32), ptr(xs, C.c_int32), stream), "evidence")
        check(L.jt_propagate_query(self.handle, len(self._qv), ptr(self._qv, C.c_int32), 1,
                                   C.c_void_p(out.data_ptr()), stream), "propagate")

    @property
    def _owner_arr(self):
        if not hasattr(self, "_own_np"):
            a = np.full(len(self.tree.cards), -1, dtype=np.int32)
            for v, c in self.owner.items():
                a[v] = c
            self._own_np = a
            self._card_np = np.asarray(self.tree.cards, dtype=np.int64)
        return self._own_np

    def encode_obs(self, cases):
        """Compact device-evidence encoding: int32 [n_obs, 3] (case, var, state),
        validated like the reference's Evidence.check (model.py:130-137):
        unknown variables raise UnknownVariableError, states outside [0, card)
        raise StateOutOfRangeError."""
        evs = [ev.assignments if hasattr(ev, "assignments") else ev for ev in cases]
        counts = list(map(len, evs))
        n = sum(counts)
        if not n:
            return np.zeros((0, 3), np.int32)
        obs = np.empty((n, 3), dtype=np.int64)
        obs[:, 0] = np.repeat(np.arange(len(evs), dtype=np.int64), counts)
        # (C-level iteration: the e2e path encodes every micro-batch's dicts here)
        obs[:, 1] = np.fromiter(chain.from_iterable(evs), dtype=np.int64, count=n)
        obs[:, 2] = np.fromiter(chain.from_iterable(map(_values, evs)), dtype=np.int64, count=n)
        own = self._owner_arr
        v, x = obs[:, 1], obs[:, 2]
        bad_v = (v < 0) | (v >= len(own))
        if bad_v.any() or (own[np.where(bad_v, 0, v)] < 0).any():
            i = int(np.flatnonzero(bad_v | (own[np.where(bad_v, 0, v)] < 0))[0])
            raise UnknownVariableError(int(v[i]))
        card = self._card_np[v]
        bad_x = (x < 0) | (x >= card)
        if bad_x.any():
            i = int(np.flatnonzero(bad_x)[0])
            raise StateOutOfRangeError(int(v[i]), int(x[i]), int(card[i]))
        return np.ascontiguousarray(obs, dtype=np.int32)

    def active_vars(self):
        """Every variable of the tree listed as active with its owning clique, so
        the propagation program is the same for every micro-batch."""
        if not hasattr(self, "_act"):
            vs = sorted(self.owner)
            self._act = (i32(vs), i32([self.owner[v] for v in vs]))
        return self._act

    def _raw_stream(self, stream):
        if stream is None:
            return C.c_void_p(self.stream.cuda_stream)
        if hasattr(stream, "cuda_stream"):
            return C.c_void_p(stream.cuda_stream)
        return stream if isinstance(stream, C.c_void_p) else C.c_void_p(stream)

    def step_device(self, obs_dev, out, stream=None):
        """One step with observations already on the device (int32 [n, 3] CUDA
        tensor): reset → masks built on device → propagate → posteriors."""
        L = _lib.lib()
        stream = self._raw_stream(stream)
        av, ac = self.active_vars()
        check(L.jt_state_reset(self.handle, stream), "reset")
        n = int(obs_dev.shape[0])
        if n:
            check(L.jt_apply_evidence_device(self.handle, n, C.c_void_p(obs_dev.data_ptr()), len(av),
                                             ptr(av, C.c_int32), ptr(ac, C.c_int32), stream), "evidence")
        check(L.jt_propagate_query(self.handle, len(self._qv), ptr(self._qv, C.c_int32), 1,
                                   C.c_void_p(out.data_ptr()), stream), "propagate")

    def run(self, cases, out=None, stream=None, to_host=False):
        """Posteriors of every case (list of {var: state} dicts or Evidence),
        `batch` cases per device step — the batched form of the reference's
        per-case loop (estimator.py:118-134).

        Pipelined: while micro-batch m runs on the device, the host encodes and
        pins micro-batch m+1; observations cross PCIe as int32 triples and the
        evidence masks are built on the device.  `stream` (a torch.cuda.Stream)
        orders the work after the caller's queued work and the caller after it;
        default: the current stream.  Returns a CUDA tensor [n, cols], or with
        `to_host=True` a host numpy array (copied back inside this call).
        A case whose evidence has zero probability raises ZeroMassError naming
        the case index (the reference raises per case, potential.py:181-186)."""
        import torch

        n = len(cases)
        steps = (n + self.batch - 1) // self.batch
        caller = stream if stream is not None else torch.cuda.current_stream(self.torch_device)
        if out is None:
            out = torch.empty((steps * self.batch, self.cols), dtype=torch.float64, device=self.torch_device)
        elif out.shape[0] < steps * self.batch or out.shape[1] != self.cols:
            raise ValueError(f"out must be at least [{steps * self.batch}, {self.cols}]")
        host = torch.empty((n, self.cols), dtype=torch.float64, pin_memory=True) if to_host else None
        self.stream.wait_stream(caller)
        raw = C.c_void_p(self.stream.cuda_stream)
        with torch.cuda.stream(self.stream):
            for s in range(steps):
                lo, hi = s * self.batch, min(n, (s + 1) * self.batch)
                obs = self.encode_obs(cases[lo:hi])
                d_obs = torch.from_numpy(obs).pin_memory().to(self.torch_device, non_blocking=True)
                self.step_device(d_obs, out[s * self.batch:(s + 1) * self.batch], raw)
                if to_host:  # this micro-batch's posteriors cross PCIe while the next one runs
                    host[lo:hi].copy_(out[lo:hi], non_blocking=True)
        caller.wait_stream(self.stream)
        if to_host:
            self.stream.synchronize()
            self._check(out, n)
            return host.numpy()
        return out[:n]

    def _check(self, out, n):
        try:
            self.sync()
        except ZeroMassError as exc:
            import torch

            bad = torch.isnan(out[:n]).any(dim=1).nonzero()
            case = int(bad[0, 0]) if bad.numel() else -1
            err = ZeroMassError(f"evidence of case {case} has zero probability ({exc})")
            err.case = case
            raise err from None

    def close(self):
        """Free the device state now (also happens when the propagator is collected)."""
        self._fin()

    def sync(self):
        check(_lib.lib().jt_sync_error(self.handle))


def shard_bounds(n_cases, world, rank):
    """Contiguous shard [lo, hi) of rank `rank`."""
    lo = (n_cases * rank) // world
    hi = (n_cases * (rank + 1)) // world
    return lo, hi


def gather_posteriors(local, n_cases, group=None):
    """All-gather every rank's [shard, cols] posterior block over NCCL (the only
    collective on the path).  Shards may differ by one row: pad to the max."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    per = max(shard_bounds(n_cases, world, r)[1] - shard_bounds(n_cases, world, r)[0] for r in range(world))
    padded = torch.zeros((per, local.shape[1]), dtype=local.dtype, device=local.device)
    padded[: local.shape[0]] = local
    full = torch.empty((world * per, local.shape[1]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(full, padded, group=group)
    parts = []
    for r in range(world):
        lo, hi = shard_bounds(n_cases, world, r)
        parts.append(full[r * per: r * per + (hi - lo)])
    return torch.cat(parts, 0)
