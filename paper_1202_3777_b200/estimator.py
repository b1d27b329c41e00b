"""Scikit-learn style facade over the device pipeline (estimator.py:29-138 of
the reference), with one change of substance: `predict_proba` answers all of
its evidence rows in batched device steps (BatchPropagator) instead of one
initialize → evidence → propagate → query loop per row (estimator.py:118-134).

Compilation (moralize → triangulate → tree → CPT assignment) is the reference's
offline CPU step and is consumed as-is: `fit` calls `jtprop.compile_network`
(the compiler is out of scope to rebuild); `fit_compiled` takes an
already compiled tree.
"""

from __future__ import annotations

import numpy as np

try:  # sklearn is only the parameter protocol (get_params/set_params/clone)
    from sklearn.base import BaseEstimator
except Exception:  # pragma: no cover
    BaseEstimator = object

from .errors import StateOutOfRangeError, UnknownVariableError
from .propagate import ENGINE_NAMES, CudaEngine, apply_evidence, belief_propagation, initialize
from .tree import FLAT, INTERLEAVED


class JunctionTreeEngine(BaseEstimator):
    """Exact posterior marginals for discrete Bayesian networks on a B200.

    Parameters mirror the reference's (engine, layout, target) plus the device
    knobs: `dtype` ('f64': 1e-10 parity, 'f32': 1e-5), `device`, and `batch`
    (evidence rows per device step in `predict_proba`).
    """

    def __init__(self, engine="cuda", dtype="f64", device=0, batch=1024, layout=FLAT, target=None):
        self.engine = engine
        self.dtype = dtype
        self.device = device
        self.batch = batch
        self.layout = layout
        self.target = target

    # -- fitting ---------------------------------------------------------------
    def _check_params(self):
        if self.engine not in ENGINE_NAMES:
            raise ValueError(f"unknown engine {self.engine!r}; use one of {ENGINE_NAMES}")
        if self.layout not in (FLAT, INTERLEAVED):
            raise ValueError(f"unknown layout {self.layout!r}")
        if int(self.batch) < 1:
            raise ValueError("batch must be >= 1")

    def fit(self, network, y=None):
        """Validate and compile a network (or a network file) with the reference
        front end, then keep the compiled tree for device queries."""
        self._check_params()
        try:
            from jtprop.compiler import compile_network
            from jtprop.io import load_network
            from jtprop.model import validate_network
        except ImportError as exc:  # the compiler is the reference's (out of scope here)
            raise ImportError("fit() compiles with the reference package `jtprop`; install it or use "
                              "fit_compiled(tree, network)") from exc
        if isinstance(network, (str, bytes)) or hasattr(network, "__fspath__"):
            network = load_network(network).network
        validate_network(network)
        compiled = compile_network(network, layout=self.layout)
        return self.fit_compiled(compiled.tree, network, compiled.mappings)

    def fit_compiled(self, tree, network, mappings=None):
        """Use an already compiled junction tree (tree.cpt_assignment set)."""
        self._check_params()
        self.network_ = network
        self.tree_ = tree
        self.mappings_ = mappings
        self.n_cliques_ = len(tree.cliques)
        self._batch_prop = None
        return self

    def _fitted(self):
        if not hasattr(self, "tree_"):
            raise ValueError("this JunctionTreeEngine is not fitted yet; call fit()")

    def _var_id(self, key):
        if isinstance(key, (int, np.integer)):
            return key
        try:
            return self.network_.id_of(key)
        except (KeyError, ValueError, LookupError) as exc:
            raise UnknownVariableError(key) from exc

    def _evidence(self, evidence):
        if evidence is None:
            return {}
        if hasattr(evidence, "assignments"):
            evidence = evidence.assignments
        out = {}
        n_vars = len(self.network_.variables)
        for k, v in dict(evidence).items():
            var = int(self._var_id(k))
            if not 0 <= var < n_vars:  # model.py:130-137: Evidence.check
                raise UnknownVariableError(k)
            card = int(self.network_.variables[var].cardinality)
            if not 0 <= int(v) < card:
                raise StateOutOfRangeError(k, int(v), card)
            out[var] = int(v)
        return out

    def _name(self, v):
        return self.network_.variables[v].name

    # -- queries -----------------------------------------------------------------
    def query(self, variables=None, evidence=None) -> dict:
        """Posterior marginals {variable name: probability vector} for one evidence set."""
        self._fitted()
        targets = list(range(len(self.network_.variables))) if variables is None else \
            [int(self._var_id(v)) for v in variables]
        state = initialize(self.tree_, self.network_, self.mappings_,
                           engine=CudaEngine(dtype=self.dtype, device=self.device))
        ev = self._evidence(evidence)
        if ev:
            apply_evidence(state, ev)
        belief_propagation(state)
        from .propagate import query_marginal

        return {self._name(v): query_marginal(state, v).values for v in targets}

    def _propagator(self, target_id):
        bp = getattr(self, "_batch_prop", None)
        if bp is None or bp.query_vars != [target_id]:
            from .batch import BatchPropagator

            bp = BatchPropagator(self.tree_, None, batch=int(self.batch), dtype=self.dtype,
                                 device=int(self.device), query_vars=[target_id], net=self.network_)
            self._batch_prop = bp
        return bp

    def predict_proba(self, X) -> np.ndarray:
        """Posterior of `target` for every evidence mapping in X, shape
        (n_samples, card(target)); all rows in batched device steps."""
        self._fitted()
        if self.target is None:
            raise ValueError("set target=<variable name> to use predict_proba")
        target_id = int(self._var_id(self.target))
        if isinstance(X, dict) or X is None:
            X = [X]
        rows = [self._evidence(x) for x in X]
        bp = self._propagator(target_id)
        return bp.run(rows, to_host=True)

    def predict(self, X) -> np.ndarray:
        """Most probable state of `target` per sample."""
        return self.predict_proba(X).argmax(axis=1)
