"""Exception types, one per failure class of the reference's hot path.

Names and the subclass tree follow ``trainsim.errors`` (reference
``pkg/src/trainsim/errors.py:4-55``) so callers catching the reference's
exceptions keep working.  The C-ABI reports each class as an ``int`` status
code (``include/flint_b200.h``: ``FL_ERR_*``); ``raise_for_status`` maps them
back.
"""

from __future__ import annotations


class TrainsimError(Exception):
    """Base class (errors.py:4)."""


class FormatError(TrainsimError):
    """A file or spec string does not conform to its format (errors.py:8)."""


class UnresolvedReferenceError(FormatError):
    pass


class MissingShapeError(FormatError):
    pass


class UnknownOperatorError(TrainsimError):
    pass


class CyclicGraphError(TrainsimError):
    pass


class InvalidGraphError(TrainsimError):
    def __init__(self, violations):
        self.violations = list(violations)
        super().__init__(f"{len(self.violations)} violation(s)")


class UnsupportedComboError(TrainsimError):
    """Model/parallelism combination the graph families cannot realise."""


class UnsupportedAlgoTopologyError(TrainsimError):
    """Collective algorithm undefined on the topology (errors.py:42)."""


class InconsistentGroupsError(TrainsimError):
    """Collective instances disagree across ranks (errors.py:46)."""


class DeadlockError(TrainsimError):
    """Simulation stalled with work remaining (errors.py:50)."""


class RankMismatchError(TrainsimError):
    pass


class EngineError(RuntimeError):
    """The CUDA engine itself failed (launch error, capacity limit, no GPU)."""


# status codes shared with include/flint_b200.h
FL_OK = 0
FL_ERR_INVALID = 1          # bad argument / malformed descriptor
FL_ERR_CUDA = 2             # CUDA runtime failure
FL_ERR_DEADLOCK = 3         # DeadlockError
FL_ERR_UNSUPPORTED_ALGO = 4  # UnsupportedAlgoTopologyError
FL_ERR_INCONSISTENT = 5     # InconsistentGroupsError
FL_ERR_CAPACITY = 6         # engine limit exceeded (graph too large for a build)
FL_ERR_NOT_RUN = 7          # row not computed (slice owned by another GPU)

_STATUS_EXC = {
    FL_ERR_DEADLOCK: DeadlockError,
    FL_ERR_UNSUPPORTED_ALGO: UnsupportedAlgoTopologyError,
    FL_ERR_INCONSISTENT: InconsistentGroupsError,
}


REFERENCE_NAMES = ("TrainsimError", "FormatError", "UnresolvedReferenceError", "MissingShapeError",
                   "UnknownOperatorError", "CyclicGraphError", "InvalidGraphError", "UnsupportedComboError",
                   "UnsupportedAlgoTopologyError", "InconsistentGroupsError", "DeadlockError", "RankMismatchError")


def _adopt_reference_classes() -> bool:
    """A caller switching from the reference catches ``trainsim.errors`` classes
    (errors.py:4-55).  When that package is importable, this module re-exports
    the reference's own classes, so every exception raised here *is* the
    reference's type.  ``FLINT_OWN_ERRORS=1`` keeps the local tree."""
    import os
    if os.environ.get("FLINT_OWN_ERRORS") == "1":
        return False
    try:
        from trainsim import errors as ref
    except Exception:       # not installed: keep the identical local tree above
        return False
    if not all(hasattr(ref, n) for n in REFERENCE_NAMES):
        return False
    g = globals()
    for n in REFERENCE_NAMES:
        g[n] = getattr(ref, n)
    _STATUS_EXC.update({FL_ERR_DEADLOCK: ref.DeadlockError, FL_ERR_UNSUPPORTED_ALGO: ref.UnsupportedAlgoTopologyError,
                        FL_ERR_INCONSISTENT: ref.InconsistentGroupsError})
    return True


USING_REFERENCE_CLASSES = _adopt_reference_classes()


def raise_for_status(code: int, what: str = "") -> None:
    if code == FL_OK:
        return
    exc = _STATUS_EXC.get(code)
    if exc is not None:
        raise exc(what or f"engine status {code}")
    raise EngineError(what or f"engine status {code}")
