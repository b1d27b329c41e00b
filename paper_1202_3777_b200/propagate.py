"""Hugin belief propagation on B200: the reference's functional API, device-backed.

Same names, argument meaning and error behaviour as the reference module
`jtprop.propagate` (propagate.py:49-402), so a caller switches engines by
switching imports.  What changes underneath:

* `PropagationState` keeps every clique and separator table in HBM (one arena,
  mixed-radix offsets).  `clique_values` / `sep_values` are host views
  materialised on access; edits made through them are written back before the
  next device operation.
* `belief_propagation` runs the whole collect+distribute as a handful of
  level-batched wave launches (replayed as a CUDA graph) instead of 2(n−1)
  per-message calls (propagate.py:337-360).
* `collect_evidence` / `distribute_evidence` keep the reference's DFS order and
  route every message through the module-global `message_passing`
  (propagate.py:313-334), so traversal spies keep working; each message is one
  device Alg. 1 call (`jt_message`).
* `CudaEngine` also speaks the reference's engine protocol
  (`run_message(phi_src, phi_tgt, phi_sep, mu_src, mu_tgt)`,
  propagate.py:79-161), so it can be installed on the *reference's* own
  PropagationState: each message then runs the μ-table-driven kernel of the
  paper (one warp per separator entry) on the device.

There is no CPU fallback: without the CUDA library or a device every call
raises DeviceError.
"""

from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import JT_F32, JT_F64, JT_MATERIALIZED, check, f64, i32, ptr
from .errors import (
    NoCoveringCliqueError,
    StateOutOfRangeError,
    UnknownVariableError,
    ZeroMassError,
)
from .tree import FLAT, Scope, build_mapping_tables, tree_components

DEFAULT_SMALL_MESSAGE_THRESHOLD = 64
ENGINE_NAMES = ("cuda", "b200")


@dataclass(frozen=True)
class Message:
    source: int
    target: int
    separator: int


class PotentialTable:
    """Flat float64 table over a scope (potential.py:125-157)."""

    def __init__(self, scope, values):
        self.scope = scope
        self.values = np.asarray(values, dtype=np.float64)
        if self.values.ndim != 1 or self.values.shape[0] != _scope_size(scope):
            raise ValueError(f"table over scope {scope.ids} needs {_scope_size(scope)} values")

    def total(self) -> float:
        return float(self.values.sum())

    def copy(self):
        return PotentialTable(self.scope, self.values.copy())


def _scope_size(scope) -> int:
    n = 1
    for c in scope.cards:
        n *= int(c)
    return n


# --------------------------------------------------------------------- plans --

def _dtype_code(dtype) -> int:
    if dtype in ("f32", "float32", np.float32, JT_F32):
        return JT_F32
    if dtype in ("f64", "float64", np.float64, JT_F64):
        return JT_F64
    raise ValueError(f"unknown dtype {dtype!r}; use 'f32' or 'f64'")


class Plan:
    """Device plan of one junction tree (jt_plan): structure only, no data.
    Holds only a weak reference to its tree, so the plan cache never pins a
    tree (or its device plan) beyond the tree's own lifetime."""

    def __init__(self, tree, dtype="f64", device=0):
        _lib.require_device()
        self._tree_ref = weakref.ref(tree)
        self.dtype = _dtype_code(dtype)
        self.device = int(device)
        cards = i32(tree.cards)
        c_off, c_vars = [0], []
        for c in tree.cliques:
            ids = list(c.scope.ids)
            if ids != sorted(ids):
                raise ValueError("clique scopes must list variables in ascending order")
            c_vars += ids
            c_off.append(len(c_vars))
        s_edge, s_off, s_vars = [], [0], []
        for s in tree.separators:
            s_edge += [int(s.edge[0]), int(s.edge[1])]
            s_vars += list(s.scope.ids)
            s_off.append(len(s_vars))
        self._arrays = [i32(x) for x in (c_off, c_vars, s_edge or [0], s_off, s_vars or [0], tree.roots)]
        a = self._arrays
        h = C.c_void_p()
        check(_lib.lib().jt_plan_create(len(cards), ptr(cards, C.c_int32), len(tree.cliques),
                                        ptr(a[0], C.c_int32), ptr(a[1], C.c_int32), len(tree.separators),
                                        ptr(a[2], C.c_int32), ptr(a[3], C.c_int32), ptr(a[4], C.c_int32),
                                        len(tree.roots), ptr(a[5], C.c_int32), self.dtype, self.device,
                                        C.byref(h)), "jt_plan_create")
        self.handle = h
        self.clique_sizes = [_scope_size(c.scope) for c in tree.cliques]
        self.sep_sizes = [_scope_size(s.scope) for s in tree.separators]
        self._fin = weakref.finalize(self, _lib.lib().jt_plan_destroy, h)

    @property
    def tree(self):
        return self._tree_ref()

    def mapping_table(self, clique_id: int, sep_id: int) -> np.ndarray:
        """μ[clique, sep] built on the device (K0), as the reference's int array."""
        n_sep = self.sep_sizes[sep_id]
        out = np.empty((n_sep, self.clique_sizes[clique_id] // max(n_sep, 1)), dtype=np.int64)
        check(_lib.lib().jt_plan_mapping_table(self.handle, int(clique_id), int(sep_id),
                                               ptr(out, C.c_int64)), "jt_plan_mapping_table")
        dt = np.int32 if self.clique_sizes[clique_id] <= np.iinfo(np.int32).max else np.int64
        return out.astype(dt)


_PLAN_CACHE: dict = {}


def plan_for(tree, dtype="f64", device=0) -> Plan:
    key = (id(tree), _dtype_code(dtype), int(device))
    hit = _PLAN_CACHE.get(key)
    if hit is not None and hit.tree is tree:
        return hit
    plan = Plan(tree, dtype, device)
    _PLAN_CACHE[key] = plan
    try:
        weakref.finalize(tree, _PLAN_CACHE.pop, key, None)
    except TypeError:  # pragma: no cover - non-weakrefable tree type
        pass
    return plan


# ------------------------------------------------------------------- engine --

class CudaEngine:
    """B200 message engine.

    * Installed on this package's PropagationState, it selects the device
      dtype ('f64' default, reference parity 1e-10; 'f32' for throughput).
    * Installed on the reference's PropagationState, `run_message` receives the
      reference's host arrays and μ tables (propagate.py:84-85) and runs the
      message on the device, writing φ_tgt and φ_sep in place.
    """

    name = "cuda"

    def __init__(self, dtype="f64", device=0, workers=None,
                 small_message_threshold=DEFAULT_SMALL_MESSAGE_THRESHOLD):
        _lib.require_device()
        self.dtype = _dtype_code(dtype)
        self.device = int(device)
        if small_message_threshold < 0:
            raise ValueError("threshold must be >= 0")
        self.small_message_threshold = small_message_threshold
        self.workers = workers

    def run_message(self, phi_src, phi_tgt, phi_sep, mu_src, mu_tgt):
        """Alg. 1 on host arrays: φ_sep ← Σ_row φ_src[μ_src]; φ_tgt[μ_tgt] *= new/old."""
        for a, nm in ((phi_tgt, "phi_tgt"), (phi_sep, "phi_sep")):
            if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous):
                raise TypeError(f"{nm} must be a C-contiguous float64 array (updated in place)")
        src = f64(phi_src)
        ms = np.ascontiguousarray(mu_src)
        mt = np.ascontiguousarray(mu_tgt)
        is64 = ms.dtype == np.int64 or mt.dtype == np.int64
        idt = np.int64 if is64 else np.int32
        ms = np.ascontiguousarray(ms, dtype=idt)
        mt = np.ascontiguousarray(mt, dtype=idt)
        n_sep = len(phi_sep)
        if ms.shape[0] != n_sep or mt.shape[0] != n_sep:
            raise ValueError("mapping tables must have one row per separator entry")
        rs = ms.shape[1] if ms.ndim == 2 else 0
        rt = mt.shape[1] if mt.ndim == 2 else 0
        check(_lib.lib().jt_run_message_mu(
            ptr(src, C.c_double), src.size, ptr(phi_tgt, C.c_double), phi_tgt.size,
            ptr(phi_sep, C.c_double), n_sep, ms.ctypes.data_as(C.c_void_p), rs,
            mt.ctypes.data_as(C.c_void_p), rt, int(is64), self.device), "run_message")

    def close(self):
        pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def make_engine(name="cuda", workers=None, small_message_threshold=DEFAULT_SMALL_MESSAGE_THRESHOLD,
                dtype="f64", device=0):
    """Engine factory (propagate.py:164-169).  Only the device engine exists
    here; any other name (including the reference's 'gpu' placeholder) is a
    ValueError."""
    if name in ENGINE_NAMES:
        return CudaEngine(dtype=dtype, device=device, workers=workers,
                          small_message_threshold=small_message_threshold)
    raise ValueError(f"unknown engine {name!r}; this package provides {ENGINE_NAMES}")


# -------------------------------------------------------------------- state --

class PropagationState:
    """Clique and separator tables of one propagation run, resident in HBM
    (propagate.py:172-201)."""

    def __init__(self, tree, mappings, engine=None, _plan=None, _handle=None):
        self.tree = tree
        self._mappings = mappings
        self.engine = engine if engine is not None else CudaEngine()
        self.evidence_applied = False
        self.plan = _plan if _plan is not None else plan_for(tree, _engine_dtype(self.engine),
                                                              _engine_device(self.engine))
        if _handle is None:
            h = C.c_void_p()
            check(_lib.lib().jt_state_create(self.plan.handle, 1, JT_MATERIALIZED, C.byref(h)),
                  "jt_state_create")
        else:
            h = _handle
        self.handle = h
        self._fin = weakref.finalize(self, _lib.lib().jt_state_destroy, h)
        self._c_off = np.concatenate([[0], np.cumsum(self.plan.clique_sizes)]).astype(np.int64)
        self._s_off = np.concatenate([[0], np.cumsum(self.plan.sep_sizes)]).astype(np.int64)
        self._hc = None  # host concat buffers when materialised
        self._hs = None
        self._exposed = False

    @property
    def mappings(self):
        """μ tables (compiler.py:330-339), built on first access only: the device
        never reads them (stride arithmetic), so states do not pay for them."""
        if self._mappings is None:
            self._mappings = build_mapping_tables(self.tree, layout=FLAT)
        return self._mappings

    @mappings.setter
    def mappings(self, value):
        self._mappings = value

    # -- host views ---------------------------------------------------------
    def _pull(self):
        if self._hc is None:
            self._hc = np.empty(int(self._c_off[-1]), dtype=np.float64)
            self._hs = np.empty(max(int(self._s_off[-1]), 1), dtype=np.float64)
            check(_lib.lib().jt_state_store(self.handle, 0, ptr(self._hc, C.c_double),
                                            ptr(self._hs, C.c_double)), "jt_state_store")

    def _push(self):
        """Write host-side edits back before any device operation."""
        if self._exposed and self._hc is not None:
            check(_lib.lib().jt_state_load(self.handle, 0, ptr(self._hc, C.c_double),
                                           ptr(self._hs, C.c_double)), "jt_state_load")
        self._exposed = False
        self._hc = self._hs = None

    def _views(self, buf, off):
        return [buf[off[i]:off[i + 1]] for i in range(len(off) - 1)]

    @property
    def clique_values(self):
        self._pull()
        self._exposed = True
        return self._views(self._hc, self._c_off)

    @property
    def sep_values(self):
        self._pull()
        self._exposed = True
        return self._views(self._hs, self._s_off)

    def copy(self) -> "PropagationState":
        """Deep copy (propagate.py:193-201), device to device (jt_state_clone)."""
        self._push()
        h = C.c_void_p()
        check(_lib.lib().jt_state_clone(self.handle, C.byref(h)), "copy")
        other = PropagationState(self.tree, self._mappings, self.engine, _plan=self.plan, _handle=h)
        other.evidence_applied = self.evidence_applied
        return other

    def clique_table(self, clique_id: int) -> PotentialTable:
        return PotentialTable(self.tree.cliques[clique_id].scope, self.clique_values[clique_id].copy())

    def sep_table(self, sep_id: int) -> PotentialTable:
        return PotentialTable(self.tree.separators[sep_id].scope, self.sep_values[sep_id].copy())

    def sync(self):
        """Wait for queued device work; map the device error word to exceptions."""
        check(_lib.lib().jt_sync_error(self.handle))


def _engine_dtype(engine):
    return getattr(engine, "dtype", JT_F64)


def _engine_device(engine):
    return getattr(engine, "device", 0)


def _as_engine(engine):
    if engine is None:
        return CudaEngine()
    if not isinstance(engine, CudaEngine):
        raise ValueError(f"engine {getattr(engine, 'name', engine)!r} is not a device engine")
    return engine


def _load(state, tables):
    cat = np.ascontiguousarray(np.concatenate([np.asarray(t, dtype=np.float64).ravel() for t in tables])
                               if tables else np.zeros(0))
    check(_lib.lib().jt_state_load(state.handle, -1, ptr(cat, C.c_double), None), "jt_state_load")


def cpt_arrays(tree, net):
    """The network's CPTs as jt_state_initialize arguments: owning clique
    (tree.cpt_assignment, propagate.py:212-217), variables in the table's own
    axis order, values concatenated."""
    cl, off, vs, vals = [], [0], [], []
    for cpt in net.cpts:
        cid = tree.cpt_assignment.get(cpt.child)
        if cid is None:
            raise NoCoveringCliqueError(f"no clique assigned for the CPT of variable {cpt.child}")
        scope = cpt.table.scope
        members = set(tree.cliques[cid].scope.ids)
        if not set(scope.ids) <= members:
            raise NoCoveringCliqueError(f"clique {cid} does not cover the CPT of variable {cpt.child}")
        cl.append(cid)
        vs.extend(int(v) for v in scope.ids)
        off.append(len(vs))
        vals.append(np.ascontiguousarray(cpt.table.values, dtype=np.float64).ravel())
    values = np.concatenate(vals) if vals else np.zeros(1)
    return i32(cl or [0]), i32(off), i32(vs or [0]), f64(values), len(cl)


def initialize(tree, net, mappings=None, engine=None) -> PropagationState:
    """All-ones cliques, each CPT multiplied into its assigned clique
    (propagate.py:204-222).  The products are formed on the device
    (jt_state_initialize): only the CPTs cross PCIe."""
    cl, off, vs, vals, n = cpt_arrays(tree, net)
    state = PropagationState(tree, mappings, _as_engine(engine))
    check(_lib.lib().jt_state_initialize(state.handle, n, ptr(cl, C.c_int32), ptr(off, C.c_int32),
                                         ptr(vs, C.c_int32), ptr(vals, C.c_double)), "initialize")
    return state


def from_potentials(tree, clique_tables, mappings=None, engine=None) -> PropagationState:
    """State over externally supplied clique tables (propagate.py:225-240)."""
    tables = []
    for clique, values in zip(tree.cliques, clique_tables):
        values = np.ascontiguousarray(values, dtype=np.float64)
        if values.shape != (_scope_size(clique.scope),):
            raise ValueError(f"clique {clique.id} table has wrong size")
        tables.append(values)
    if len(tables) != len(tree.cliques):
        raise ValueError("need one table per clique")
    state = PropagationState(tree, mappings, _as_engine(engine))
    _load(state, tables)
    return state


def apply_evidence(state, evidence):
    """Zero every entry that disagrees with an observation, in the clique owning
    the variable's CPT (propagate.py:243-260)."""
    assignments = evidence.assignments if hasattr(evidence, "assignments") else dict(evidence)
    vs, cs, xs = [], [], []
    for var, observed in sorted(assignments.items()):
        if var not in state.tree.cpt_assignment:
            raise UnknownVariableError(var)
        cid = state.tree.cpt_assignment[var]
        scope = state.tree.cliques[cid].scope
        card = scope.cards[list(scope.ids).index(var)]
        if not 0 <= observed < card:
            raise StateOutOfRangeError(var, observed, card)
        vs.append(var)
        cs.append(cid)
        xs.append(observed)
    state._push()
    if vs:
        v, c, x = i32(vs), i32(cs), i32(xs)
        check(_lib.lib().jt_apply_evidence(state.handle, len(vs), None, ptr(v, C.c_int32),
                                           ptr(c, C.c_int32), ptr(x, C.c_int32), None),
              "apply_evidence")
    state.evidence_applied = True
    return state


def message_passing(state, msg: Message):
    """One directed message: marginalize onto the separator, then scatter
    (propagate.py:263-274)."""
    state._push()
    check(_lib.lib().jt_message(state.handle, int(msg.source), int(msg.target), int(msg.separator), None),
          "message_passing")
    state.sync()
    return state


def _children_first_order(tree, root):
    """(child, parent, separator) edges in post-order, children ascending
    (propagate.py:296-310)."""
    out = []
    stack = [(root, -1, -1, False)]
    while stack:
        node, parent, sep_id, expanded = stack.pop()
        if expanded:
            if parent >= 0:
                out.append((node, parent, sep_id))
            continue
        stack.append((node, parent, sep_id, True))
        for nbr, s in reversed(tree.neighbors[node]):
            if nbr != parent:
                stack.append((nbr, node, s, False))
    return out


def collect_evidence(state, root):
    """Child → parent messages, leaves first (propagate.py:313-317)."""
    for child, parent, sep_id in _children_first_order(state.tree, root):
        message_passing(state, Message(child, parent, sep_id))
    return state


def distribute_evidence(state, root):
    """Parent → child messages in pre-order (propagate.py:320-334)."""
    stack = [(root, -1, -1)]
    while stack:
        node, parent, sep_id = stack.pop()
        if parent >= 0:
            message_passing(state, Message(parent, node, sep_id))
        for nbr, s in reversed(state.tree.neighbors[node]):
            if nbr != parent:
                stack.append((nbr, node, s))
    return state


def _roots_for(tree, root):
    if root is None:
        return list(tree.roots)
    comps = tree_components(tree)
    comp = next((i for i, c in enumerate(comps) if root in c), None)
    if comp is None:
        raise UnknownVariableError(f"clique {root}")
    return [root if i == comp else r for i, r in enumerate(tree.roots)]


def belief_propagation(state, root=None, stream=None):
    """Collect then distribute for every component (propagate.py:337-360), as
    one device program of level-batched waves.  `root` redirects only its own
    component.  Posteriors do not depend on message order inside a wave."""
    roots = _roots_for(state.tree, root)
    state._push()
    r = i32(roots)
    check(_lib.lib().jt_propagate(state.handle, ptr(r, C.c_int32), stream), "belief_propagation")
    state.sync()
    return state


def _best_holder(tree, variable):
    holders = [c for c in tree.cliques if variable in c.scope.ids]
    if not holders:
        raise UnknownVariableError(variable)
    return min(holders, key=lambda c: (_scope_size(c.scope), c.id))


def query_marginal(state, variable, normalize_result=True) -> PotentialTable:
    """Marginal of one variable from the smallest clique holding it
    (propagate.py:363-377); ZeroMassError on zero total when normalizing."""
    best = _best_holder(state.tree, variable)
    card = best.scope.cards[list(best.scope.ids).index(variable)]
    state._push()
    out = np.empty(card, dtype=np.float64)
    v, c = i32([variable]), i32([best.id])
    check(_lib.lib().jt_query(state.handle, 1, ptr(v, C.c_int32), ptr(c, C.c_int32),
                              1 if normalize_result else 0, ptr(out, C.c_double), None), "query_marginal")
    state.sync()
    return PotentialTable(Scope((variable,), (card,)), out)


def posterior_marginals(compiled, net, evidence=None, engine=None) -> dict:
    """initialize → evidence → propagate → query every variable
    (propagate.py:380-390), the queries batched into one device call."""
    state = initialize(compiled.tree, net, compiled.mappings, engine=engine)
    if evidence:
        apply_evidence(state, evidence)
    belief_propagation(state)
    n = len(net)
    cards = [net.variables[v].cardinality for v in range(n)]
    out = np.empty(sum(cards), dtype=np.float64)
    vs = i32(range(n))
    cs = i32([_best_holder(state.tree, v).id for v in range(n)])
    check(_lib.lib().jt_query(state.handle, n, ptr(vs, C.c_int32), ptr(cs, C.c_int32), 1,
                              ptr(out, C.c_double), None), "posterior_marginals")
    state.sync()
    res, o = {}, 0
    for v in range(n):
        res[v] = out[o:o + cards[v]].copy()
        o += cards[v]
    return res


def check_global_consistency(state, rtol=1e-9):
    """After propagation each separator equals both adjacent marginals
    (propagate.py:393-402); host-side debug helper."""
    seps = state.sep_values
    cliques = state.clique_values
    for sep in state.tree.separators:
        target = seps[sep.id]
        for cid in sep.edge:
            got = _marginal(state.tree.cliques[cid].scope, cliques[cid], sep.scope)
            if not np.allclose(got, target, rtol=rtol, atol=0.0):
                raise AssertionError(f"clique {cid} disagrees with separator {sep.id}")


def _marginal(outer, values, inner):
    size = _scope_size(outer)
    idx = np.arange(size, dtype=np.int64)
    strides = Scope(outer.ids, outer.cards).strides()
    istr = Scope(inner.ids, inner.cards).strides()
    proj = np.zeros(size, dtype=np.int64)
    for pos, var in enumerate(inner.ids):
        p = list(outer.ids).index(var)
        proj += ((idx // strides[p]) % outer.cards[p]) * istr[pos]
    return np.bincount(proj, weights=values, minlength=_scope_size(inner))


__all__ = [
    "CudaEngine", "Message", "Plan", "PotentialTable", "PropagationState", "apply_evidence",
    "belief_propagation", "check_global_consistency", "collect_evidence", "distribute_evidence",
    "from_potentials", "initialize", "make_engine", "message_passing", "plan_for",
    "posterior_marginals", "query_marginal", "ZeroMassError",
]
