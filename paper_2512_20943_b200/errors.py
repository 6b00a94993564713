"""Error classes of the drop-in.

Names, base class and ``code`` strings are the reference's public contract
(``ss/errors.py:8-67``) so that ``except StructuralError`` in existing callers
catches failures raised here; the C-ABI returns negative statuses that
``_lib.Engine.call`` turns into these classes.
"""

_TABLE = (
    # class name            code                status in include/airgs_b200.h
    ("StructuralError", "STRUCTURAL"),        # AIRGS_E_STRUCTURAL (-1)
    ("ValidationError", "VALIDATION"),        # AIRGS_E_VALIDATION (-2)
    ("CapacityError", "CAPACITY"),            # AIRGS_E_CAPACITY   (-3)
    ("DecodeError", "DECODE"),                # AIRGS_E_DECODE     (-5)
    ("ProtocolError", "PROTOCOL"),
    ("TraceExhaustedError", "TRACE"),
    ("MissingArtifactError", "MISSING_ARTIFACT"),
    ("InfeasibleError", "INFEASIBLE"),
)


class SplatStreamError(Exception):
    """Root of every error this package raises on purpose."""

    code = "ERR"


for _name, _code in _TABLE:
    globals()[_name] = type(_name, (SplatStreamError,), {"code": _code, "__module__": __name__})


class TrainingError(SplatStreamError):
    """A fit diverged (ss/errors.py; raised by train.py)."""

    code = "TRAINING"

    def __init__(self, message, iteration=None):
        super().__init__(message)
        self.iteration = iteration


StructuralError = globals()["StructuralError"]
ValidationError = globals()["ValidationError"]
CapacityError = globals()["CapacityError"]
DecodeError = globals()["DecodeError"]
ProtocolError = globals()["ProtocolError"]
TraceExhaustedError = globals()["TraceExhaustedError"]
MissingArtifactError = globals()["MissingArtifactError"]
InfeasibleError = globals()["InfeasibleError"]

__all__ = ["SplatStreamError", "TrainingError"] + [n for n, _ in _TABLE]
