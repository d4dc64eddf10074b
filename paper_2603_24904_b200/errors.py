"""Exception types mirroring the reference's (SURVEY.md §8b "Errors").

Each C-ABI status (include/dimg.h) maps back to the type the reference throws,
so callers and tests can assert the same contract as proj/tests/*.cpp.
"""


class DimError(Exception):
    code = -1


class InvalidArgument(DimError, ValueError):       # std::invalid_argument
    code = 1


class OutOfRange(DimError, IndexError):            # std::out_of_range
    code = 2


class LogicError(DimError, RuntimeError):          # std::logic_error
    code = 3


class ContextOverflow(DimError, RuntimeError):     # dim::ContextOverflow
    code = 4


class LengthError(DimError, RuntimeError):         # std::length_error
    code = 5


class DomainError(DimError, ValueError):           # std::domain_error
    code = 6


class ParseError(DimError):                        # dim::ParseError
    code = 7
    KINDS = ("bad_magic", "bad_version", "truncated", "invariant")

    def __init__(self, msg, kind=None):
        super().__init__(msg)
        self.kind = kind


class CudaError(DimError, RuntimeError):
    code = 8


class NcclError(DimError, RuntimeError):
    code = 9


class DeviceOutOfMemory(DimError, MemoryError):
    code = 10


class IOFailure(DimError, OSError):
    code = 11


_BY_CODE = {c.code: c for c in (InvalidArgument, OutOfRange, LogicError, ContextOverflow,
                                LengthError, DomainError, ParseError, CudaError, NcclError,
                                DeviceOutOfMemory, IOFailure)}


def from_status(code: int, msg: str, parse_kind: int = -1) -> DimError:
    cls = _BY_CODE.get(code, DimError)
    if cls is ParseError:
        kind = ParseError.KINDS[parse_kind] if 0 <= parse_kind < 4 else None
        return ParseError(msg, kind)
    e = cls(msg)
    e.code = code
    return e
