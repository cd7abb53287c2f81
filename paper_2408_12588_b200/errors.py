"""Error kinds of the PAB hot path.

Mirrors the reference's stable machine-readable ``kind`` strings
(pkg/src/pab_engine/errors.py:4-40) so callers that switch on ``err.kind``
keep working.  The C ABI returns integer status codes; ``raise_for_status``
maps them back onto these classes (include/pab_b200.h lists the codes).
"""

from __future__ import annotations


class EngineError(Exception):
    kind = "engine-error"

    def __init__(self, message, kind=None):
        super().__init__(message)
        if kind is not None:
            self.kind = kind


class ShapeError(EngineError):
    kind = "shape-mismatch"


class ValidationError(EngineError):
    kind = "invalid-config"


class PolicyError(EngineError):
    kind = "policy-error"


class MetricError(EngineError):
    kind = "undefined-metric"


class ArtifactError(EngineError):
    kind = "missing-artifact"


class DeviceError(EngineError):
    """A CUDA / NCCL / driver call failed inside the native library."""

    kind = "device-error"


# status codes returned by every pab_* C entry point (include/pab_b200.h)
PAB_OK = 0
PAB_ERR_SHAPE = 1
PAB_ERR_INVALID = 2
PAB_ERR_POLICY = 3
PAB_ERR_CUDA = 4
PAB_ERR_UNSUPPORTED = 5

_STATUS_CLASS = {
    PAB_ERR_SHAPE: ShapeError,
    PAB_ERR_INVALID: ValidationError,
    PAB_ERR_POLICY: PolicyError,
    PAB_ERR_CUDA: DeviceError,
    PAB_ERR_UNSUPPORTED: ValidationError,
}


def raise_for_status(status: int, what: str, detail: str = "") -> None:
    if status == PAB_OK:
        return
    cls = _STATUS_CLASS.get(status, EngineError)
    msg = f"{what} failed with status {status}"
    if detail:
        msg += f": {detail}"
    raise cls(msg)
