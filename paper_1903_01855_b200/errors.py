"""Exception taxonomy of the runtime.

The class names (and their grouping under one root) are part of the
drop-in surface: user code written against the reference catches these
exact types (reference: stageflow/errors.py:8-159).  One type is new here:
``DeviceUnavailable``, raised when a computation needs the GPU backend but
no CUDA device (or no built ``libsfb200.so``) is present — the backend never
falls back to host arithmetic.
"""


class StageflowError(Exception):
    """Root of every error this runtime raises on purpose."""


def _family(*names, base=StageflowError, doc=None):
    made = []
    for n in names:
        made.append(type(n, (base,), {"__doc__": doc, "__module__": __name__}))
    return made


# tensors and host interchange
LengthMismatch, NarrowingOverflow, SymbolicTensor, BroadcastIncompatible = _family(
    "LengthMismatch", "NarrowingOverflow", "SymbolicTensor", "BroadcastIncompatible"
)
# op registry and dispatch
DuplicateOp, UnknownOp, ArityMismatch, AttrMismatch, KernelError = _family(
    "DuplicateOp", "UnknownOp", "ArityMismatch", "AttrMismatch", "KernelError"
)
# gradient tapes
NonNestedEnd, InactiveTape, NonScalarTarget, UnwatchedSource, ConsumedTape = _family(
    "NonNestedEnd", "InactiveTape", "NonScalarTarget", "UnwatchedSource", "ConsumedTape"
)
# staging
(SignatureMismatch, StagingError, VariableCreationError, UnencodableArgument,
 MissingConcreteFunction) = _family(
    "SignatureMismatch", "StagingError", "VariableCreationError", "UnencodableArgument",
    "MissingConcreteFunction",
)
# graph functions
NotSerializable, FormatVersionMismatch, CorruptGraph, InputMismatch, MissingFunction = _family(
    "NotSerializable", "FormatVersionMismatch", "CorruptGraph", "InputMismatch",
    "MissingFunction",
)
# state and checkpoints
ShapeMismatch, DeadVariable, StorageError, DTypeOrShapeConflict = _family(
    "ShapeMismatch", "DeadVariable", "StorageError", "DTypeOrShapeConflict"
)
# devices, callbacks, benchmarks
(UnknownDevice,) = _family("UnknownDevice")
CallbackError, SignatureViolation = _family("CallbackError", "SignatureViolation")
ConfigError, NumericalDivergence = _family("ConfigError", "NumericalDivergence")


class DeviceUnavailable(KernelError):
    """The GPU backend is required but absent (no device or no native library)."""


__all__ = [n for n, v in dict(globals()).items()
           if isinstance(v, type) and issubclass(v, StageflowError)]
