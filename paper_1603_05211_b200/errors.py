"""Exception hierarchy of the reference (errors.hpp:10-77), raised from af_status."""
from __future__ import annotations


class Error(RuntimeError):
    """adaptflow::Error"""


class NonPhysicalState(Error):
    """adaptflow::NonPhysicalState (errors.hpp:18-21)"""


class RegisterMismatch(Error):
    """adaptflow::RegisterMismatch (errors.hpp:69-72)"""


class ConfigError(Error):
    """adaptflow::ConfigError (errors.hpp:33-36)"""


class LevelMismatch(Error):
    """adaptflow::LevelMismatch (errors.hpp:23-26)"""


class DeviceError(Error):
    """CUDA / NCCL failure (no reference equivalent)."""


class UnsupportedOption(ConfigError):
    """Option outside the device path (e.g. MUSCL-Hancock in the MR solver)."""


class IoError(Error):
    """adaptflow::IoError (errors.hpp:38-41)"""


class DivisionDomain(Error):
    """adaptflow::DivisionDomain (errors.hpp:49-52)."""


_BY_STATUS = {1: NonPhysicalState, 2: RegisterMismatch, 3: ConfigError, 4: LevelMismatch,
              5: DeviceError, 6: DeviceError, 7: ValueError, 8: UnsupportedOption,
              9: DeviceError, 10: IoError, 11: DivisionDomain}


def raise_status(status: int, message: str) -> None:
    if status == 0:
        return
    raise _BY_STATUS.get(status, Error)(message)
