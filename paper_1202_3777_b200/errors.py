"""Exception hierarchy mirroring the reference's (errors.py:8-131).

Only the classes the propagation path raises are mirrored.  When the reference
package `jtprop` is importable, each class here also derives from the
reference class of the same name, so `except jtprop.errors.ZeroMassError`
keeps working for code switching engines.
"""

from __future__ import annotations

try:  # optional: make our exceptions catchable as the reference's
    from jtprop import errors as _ref  # type: ignore
except Exception:  # pragma: no cover - reference absent (GPU box)
    _ref = None


def _bases(name, *own):
    ref = getattr(_ref, name, None) if _ref is not None else None
    return ((ref,) if ref is not None else ()) + own


class JtpropError(*_bases("JtpropError", Exception)):
    """Base class (errors.py:8)."""


class InputError(*_bases("InputError", JtpropError)):
    """User-supplied data problem (errors.py:12)."""


class UnknownVariableError(*_bases("UnknownVariableError", InputError)):
    def __init__(self, name):
        self.name = name
        Exception.__init__(self, f"unknown variable {name!r}")


class StateOutOfRangeError(*_bases("StateOutOfRangeError", InputError)):
    def __init__(self, variable, state, cardinality):
        self.variable = variable
        Exception.__init__(
            self, f"state {state} out of range for variable {variable!r} "
                  f"(cardinality {cardinality})")


class ScopeNotContainedError(*_bases("ScopeNotContainedError", InputError)):
    pass


class ZeroMassError(*_bases("ZeroMassError", JtpropError)):
    """Total mass is zero (errors.py:98)."""


class NoCoveringCliqueError(*_bases("NoCoveringCliqueError", JtpropError)):
    """No clique covers a CPT scope (errors.py:108)."""


class InconsistentDivisionError(*_bases("InconsistentDivisionError", JtpropError)):
    """A separator entry is zero while its fresh marginal is not (errors.py:114)."""


class DeviceError(JtpropError):
    """CUDA runtime failure or missing native library (no reference analogue)."""
