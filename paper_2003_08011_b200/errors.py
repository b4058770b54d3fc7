"""Exception taxonomy mirroring /root/reference/proj/include/containerstress/errors.hpp:9-74.

The C-ABI returns a cs_status 1:1 with these classes; messages reproduce the
reference texts so sweep exclusion reasons (sweep.cpp:229-236) read the same.
"""


class Error(RuntimeError):
    """Base class for all errors raised by this library (errors.hpp:9-12)."""


class MomentInfeasible(Error):
    pass


class BadCorrelation(Error):
    pass


class TooFewSamples(Error):
    pass


class ConstraintViolated(Error):
    pass


class InsufficientTraining(Error):
    pass


class DegenerateModel(Error):
    pass


class EigFailure(Error):
    pass


class ShapeError(Error):
    pass


class EmptyGrid(Error):
    pass


class UnknownBackend(Error):
    pass


class BadSlice(Error):
    pass


class ConfigError(Error):
    pass


class IoError(Error):
    pass


_BY_STATUS = {
    1: Error, 2: ConstraintViolated, 3: InsufficientTraining, 4: DegenerateModel,
    5: EigFailure, 6: ShapeError, 7: ConfigError, 8: IoError, 9: MomentInfeasible,
    10: BadCorrelation, 11: TooFewSamples, 12: EmptyGrid,
}


def from_status(code: int, msg: str) -> Error:
    return _BY_STATUS.get(code, Error)(msg)
