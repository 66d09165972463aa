"""Error types mirroring the reference (errors.hpp:11-37).

Each exception carries the reference's stable ``code`` string, and the C ABI
status maps 1:1 onto them (include/mgrg.h)."""
from __future__ import annotations


class Error(RuntimeError):
    """mgr::Error: ``code`` is stable and machine-parsable (errors.hpp:11-21)."""

    code = "Error"

    def __init__(self, what: str = ""):
        super().__init__(what)


def _make(name: str):
    return type(name, (Error,), {"code": name})


InvalidGrid = _make("InvalidGrid")
InvalidLevel = _make("InvalidLevel")
ShapeError = _make("ShapeError")
InvalidFusion = _make("InvalidFusion")
SingularSystem = _make("SingularSystem")
TooManyWorkers = _make("TooManyWorkers")
WorkerFailure = _make("WorkerFailure")
CorruptFile = _make("CorruptFile")
MissingClass = _make("MissingClass")
InvalidBound = _make("InvalidBound")
IoError = _make("IoError")
# device-side failures have no reference counterpart
CudaError = _make("CudaError")
NcclError = _make("NcclError")
Unsupported = _make("Unsupported")
InvalidArgument = _make("InvalidArgument")
OutOfMemory = _make("OutOfMemory")

_BY_STATUS = {
    1: InvalidGrid, 2: InvalidLevel, 3: ShapeError, 4: InvalidFusion,
    5: SingularSystem, 6: TooManyWorkers, 7: WorkerFailure, 8: CorruptFile,
    9: MissingClass, 10: InvalidBound, 11: IoError, 12: CudaError, 13: NcclError,
    14: Unsupported, 15: InvalidArgument, 16: OutOfMemory,
}


def from_status(status: int, what: str) -> Error:
    return _BY_STATUS.get(status, Error)(what)
