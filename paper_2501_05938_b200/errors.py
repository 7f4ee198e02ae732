"""Python mirror of the streamtune error taxonomy.

/root/reference/proj/include/streamtune/errors.hpp:9-118: two roots,
ValidationError (exit / status 1) and ComputationError (exit / status 2),
with the same subclass names.  CudaRuntimeError is status 3 of the C ABI.
"""


class StreamtuneError(Exception):
    status = 0


class ValidationError(StreamtuneError, ValueError):
    status = 1


class ComputationError(StreamtuneError, ArithmeticError):
    status = 2


class MalformedRowError(ValidationError):
    pass


class NegativeDurationError(ValidationError):
    pass


class DuplicateSizeError(ValidationError):
    pass


class InvalidStreamCountError(ValidationError):
    pass


class MissingStageTimingsError(ValidationError):
    pass


class TooFewObservationsError(ComputationError):
    pass


class RankDeficiencyError(ComputationError):
    pass


class ZeroVarianceError(ComputationError):
    pass


class NonpositiveTauError(ComputationError):
    pass


class SingularPivotError(ComputationError):
    pass


class CudaRuntimeError(RuntimeError):
    status = 3


_BY_NAME = {c.__name__: c for c in (
    ValidationError, ComputationError, MalformedRowError, NegativeDurationError, DuplicateSizeError,
    InvalidStreamCountError, MissingStageTimingsError, TooFewObservationsError, RankDeficiencyError,
    ZeroVarianceError, NonpositiveTauError, SingularPivotError)}


def raise_for(status: int, message: str):
    """Raises the exception for a C-ABI status / "<Class>: msg" string."""
    name, _, rest = message.partition(": ")
    cls = _BY_NAME.get(name)
    if cls is not None:
        raise cls(rest)
    if status == 1:
        if "stream count" in message:
            raise InvalidStreamCountError(message)
        raise ValidationError(message)
    if status == 2:
        raise SingularPivotError(message)
    raise CudaRuntimeError(message)
