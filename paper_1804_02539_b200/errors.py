"""Exception classes of the reference (include/patchmg/errors.hpp:9-56), one per
C ABI status code (include/pmg_types.h)."""


class Error(RuntimeError):
    """Base class for all solver errors."""


class ConfigError(Error):
    pass


class DomainError(Error):
    pass


class NonMatchingError(Error):
    pass


class SingularGeometryError(Error):
    pass


class DecompositionError(Error):
    pass


class DefinitenessError(Error):
    pass


class DivergenceError(Error):
    pass


class TransportError(Error):
    pass


class CudaError(Error):
    """Device failure; no reference analogue."""


_BY_CODE = {
    1: Error, 2: ConfigError, 3: DivergenceError, 4: TransportError, 5: DomainError,
    6: DefinitenessError, 7: DecompositionError, 8: SingularGeometryError, 9: NonMatchingError, 10: CudaError,
}

# exit codes of the reference CLI (harness.cpp:573-581)
EXIT_CODES = {ConfigError: 2, DivergenceError: 3, TransportError: 4}


def raise_for(code: int, message: str):
    if code != 0:
        raise _BY_CODE.get(code, Error)(message)
