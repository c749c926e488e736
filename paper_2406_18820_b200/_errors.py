"""Exception taxonomy of the drop-in, and the C-ABI status-code mapping.

The class names and the inheritance tree are the reference's
(``ucp/errors.py:8-69``) so ``except ucp.ReplicateMismatchError`` keeps working
after swapping the import. Each data-dependent class also owns a negative
status code that ``libucp_b200.so`` reports through ``ucp_status``
(``include/ucp_b200.h``); :func:`from_status` maps it back.
"""

from __future__ import annotations


class UcpError(Exception):
    """Root of every error this package raises."""


def _mk(name: str, base: type, doc: str) -> type:
    return type(name, (base,), {"__doc__": doc, "__module__": __name__})


# (name, parent, doc) in the reference's order; parents precede children
_TABLE = (
    ("TensorFileError", "UcpError", "Tensor container problem other than a bare OS error."),
    ("CorruptHeaderError", "TensorFileError", "Bad magic/version/dtype/dims in a UCPT header."),
    ("TruncatedPayloadError", "TensorFileError", "UCPT payload shorter than its header says."),
    ("TensorIOError", "TensorFileError", "OS-level failure reading or writing a UCPT file."),
    ("UnsupportedCastError", "UcpError", "Cast outside {f32<->bf16, f32<->f16}."),
    ("ShapeError", "UcpError", "Shape or bounds violation."),
    ("ModelConfigError", "UcpError", "Invalid model family/scale/description."),
    ("IncompatibleConfigError", "UcpError", "ParallelConfig invalid alone or for a model."),
    ("PatternCoverageError", "UcpError", "No TP rule covers (param kind, tp)."),
    ("CheckpointLayoutError", "UcpError", "Checkpoint directory not in the expected state."),
    ("ManifestError", "UcpError", "Rank manifest missing, malformed or inconsistent."),
    ("MissingFragmentError", "UcpError", "Fragments do not cover the tensor."),
    ("OverlappingRangeError", "UcpError", "Fragments claim the same elements."),
    ("ReplicateMismatchError", "UcpError", "Replicas that must be bit-identical differ."),
    ("PaddingError", "UcpError", "ZeRO pad tail nonzero or pad bookkeeping wrong."),
)

_CLASSES: dict[str, type] = {"UcpError": UcpError}
for _name, _parent, _doc in _TABLE:
    _CLASSES[_name] = _mk(_name, _CLASSES[_parent], _doc)

TensorFileError = _CLASSES["TensorFileError"]
CorruptHeaderError = _CLASSES["CorruptHeaderError"]
TruncatedPayloadError = _CLASSES["TruncatedPayloadError"]
TensorIOError = _CLASSES["TensorIOError"]
UnsupportedCastError = _CLASSES["UnsupportedCastError"]
ShapeError = _CLASSES["ShapeError"]
ModelConfigError = _CLASSES["ModelConfigError"]
IncompatibleConfigError = _CLASSES["IncompatibleConfigError"]
PatternCoverageError = _CLASSES["PatternCoverageError"]
CheckpointLayoutError = _CLASSES["CheckpointLayoutError"]
ManifestError = _CLASSES["ManifestError"]
MissingFragmentError = _CLASSES["MissingFragmentError"]
OverlappingRangeError = _CLASSES["OverlappingRangeError"]
ReplicateMismatchError = _CLASSES["ReplicateMismatchError"]
PaddingError = _CLASSES["PaddingError"]


class NativeUnavailableError(UcpError, RuntimeError):
    """libucp_b200.so or a CUDA device is missing. There is no CPU path."""


# status codes shared with include/ucp_b200.h (UCP_E*)
STATUS_OK = 0
STATUS_REPLICA = -1   # UCP_EREPLICA: replicas differ
STATUS_PAD = -2       # UCP_EPAD: nonzero pad tail
STATUS_INVAL = -10    # UCP_EINVAL: bad descriptor / argument
STATUS_CUDA = -11     # UCP_ECUDA: launch / runtime failure

_BY_CODE = {STATUS_REPLICA: ReplicateMismatchError, STATUS_PAD: PaddingError,
            STATUS_INVAL: ShapeError}


def from_status(code: int, msg: str) -> UcpError:
    """Exception instance for a nonzero C-ABI status code."""
    cls = _BY_CODE.get(code)
    if cls is None:
        return NativeUnavailableError(f"native call failed ({code}): {msg}")
    return cls(msg)


def by_name(name: str) -> type:
    return _CLASSES[name]
