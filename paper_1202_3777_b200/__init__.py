"""paper_1202_3777_b200 — B200-native junction-tree belief propagation.

Drop-in for the propagation path of the reference package `jtprop`
(arXiv:1202.3777, Zheng, Mengshoel & Chong): same functional API
(`from_potentials`, `initialize`, `apply_evidence`, `message_passing`,
`collect_evidence`, `distribute_evidence`, `belief_propagation`,
`query_marginal`, `posterior_marginals`) and engine protocol, executed by
hand-written sm_100a kernels in libjtb200.so (C ABI: include/jt_b200.h).
The batch API (`BatchPropagator`) answers many evidence cases per device step
and shards across GPUs.  See DESIGN.md.
"""

from .errors import (
    DeviceError,
    InconsistentDivisionError,
    JtpropError,
    NoCoveringCliqueError,
    StateOutOfRangeError,
    UnknownVariableError,
    ZeroMassError,
)
from .tree import (
    FLAT,
    INTERLEAVED,
    Clique,
    JunctionTree,
    MappingTableSet,
    Scope,
    Separator,
    algorithmic_elements,
    build_mapping_table,
    build_mapping_tables,
    build_tree,
    directed_messages,
    relayout_mapping_tables,
)

_API = (
    "CudaEngine", "Message", "Plan", "PotentialTable", "PropagationState", "apply_evidence",
    "belief_propagation", "check_global_consistency", "collect_evidence", "distribute_evidence",
    "from_potentials", "initialize", "make_engine", "message_passing", "plan_for",
    "posterior_marginals", "query_marginal",
)


def __getattr__(name):
    # the device API is imported lazily so that tree/synth utilities stay usable
    # (and importable by the CPU test-suite) on hosts without the CUDA library
    if name in _API:
        from . import propagate

        return getattr(propagate, name)
    if name == "JunctionTreeEngine":
        from .estimator import JunctionTreeEngine

        return JunctionTreeEngine
    if name in ("BatchPropagator", "gather_posteriors", "shard_bounds"):
        from . import batch

        return getattr(batch, name)
    raise AttributeError(name)


__version__ = "0.1.0"
__all__ = list(_API) + [
    "BatchPropagator", "Clique", "DeviceError", "FLAT", "INTERLEAVED", "InconsistentDivisionError",
    "JtpropError", "JunctionTree", "JunctionTreeEngine", "MappingTableSet", "NoCoveringCliqueError", "Scope", "Separator",
    "StateOutOfRangeError", "UnknownVariableError", "ZeroMassError", "algorithmic_elements",
    "build_mapping_table", "build_mapping_tables", "build_tree", "directed_messages",
    "gather_posteriors", "relayout_mapping_tables", "shard_bounds",
]
