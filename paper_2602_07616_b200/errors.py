"""Exception hierarchy of the reference `sere` package, restated.

Mirrors `/root/reference/pkg/src/sere/errors.py:9-34` class for class so that
code written against the reference (``except ConfigError`` ...) keeps working
when it is pointed at this package. The C-ABI returns integer status codes
(`include/sere_b200.h`, ``SERE_ERR_*``); :func:`raise_for_status` maps them
1:1 onto these classes.
"""

from __future__ import annotations


class SereError(Exception):
    """Base class for all errors raised by this package (errors.py:9)."""


class DimensionError(SereError):
    """Array shapes do not line up (errors.py:13)."""


class DomainError(SereError):
    """Numerically invalid input: NaN/inf ... (errors.py:17)."""


class RoutingError(SereError):
    """A routing assignment refers to an expert that does not exist (errors.py:21)."""


class ConfigError(SereError):
    """A configuration value violates its contract (errors.py:25)."""


class InputError(SereError):
    """Input data is structurally valid but semantically unusable (errors.py:29)."""


class DegenerateInputWarning(UserWarning):
    """Emitted when a computation falls back to a documented degenerate value (errors.py:33)."""


class DeviceError(SereError):
    """The CUDA runtime or the device rejected a launch (no reference analogue)."""


# status codes of include/sere_b200.h
SERE_OK = 0
SERE_ERR_CONFIG = 1
SERE_ERR_DIMENSION = 2
SERE_ERR_INPUT = 3
SERE_ERR_ROUTING = 4
SERE_ERR_DOMAIN = 5
SERE_ERR_CUDA = 6
SERE_ERR_UNSUPPORTED = 7
SERE_ERR_WORKSPACE = 8

_STATUS_TO_EXC = {
    SERE_ERR_CONFIG: ConfigError,
    SERE_ERR_DIMENSION: DimensionError,
    SERE_ERR_INPUT: InputError,
    SERE_ERR_ROUTING: RoutingError,
    SERE_ERR_DOMAIN: DomainError,
    SERE_ERR_CUDA: DeviceError,
    SERE_ERR_UNSUPPORTED: DeviceError,
    SERE_ERR_WORKSPACE: DimensionError,
}


def exception_for_status(code: int, what: str = "") -> SereError | None:
    """Exception instance for a non-zero C-ABI status, or None for SERE_OK."""
    if code == SERE_OK:
        return None
    cls = _STATUS_TO_EXC.get(int(code), SereError)
    return cls(f"{what}: status {int(code)}" if what else f"status {int(code)}")


def raise_for_status(code: int, what: str = "") -> None:
    exc = exception_for_status(code, what)
    if exc is not None:
        raise exc
