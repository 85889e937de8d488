"""Exception classes of the drop-in boundary.

Same names and meaning as the reference's ``stabsim/errors.py:4-13`` so that
callers (and the parity tests) can catch them unchanged.  ``NativeError`` is
the one addition: the CUDA library is missing or a CUDA call failed -- the
product path never falls back to the CPU, it raises this instead.
"""


class ResourceLimitError(RuntimeError):
    """A size cap or term budget would be exceeded (reference errors.py:4)."""


class NumericalCollapseError(RuntimeError):
    """Every term of a generator was dropped by the merge (reference errors.py:8)."""


class ConsistencyError(RuntimeError):
    """An internal invariant failed, e.g. a non-real density coefficient (reference errors.py:12)."""


class NativeError(RuntimeError):
    """libqimax_b200.so is missing, no CUDA device is usable, or a CUDA call failed."""
