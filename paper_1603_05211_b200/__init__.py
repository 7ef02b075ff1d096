"""adaptflow-b200: B200-native (sm_100a) MR/FV compressible-Euler hot path.

The compute path is libafgpu.so (hand-written CUDA behind the C ABI of
include/af_gpu.h); importing the solver API loads it and fails loudly if it
is missing — there is no CPU fallback.
"""
from .errors import (ConfigError, DeviceError, Error, LevelMismatch, NonPhysicalState,
                     RegisterMismatch, UnsupportedOption)

__all__ = ["Error", "NonPhysicalState", "RegisterMismatch", "ConfigError", "LevelMismatch",
           "DeviceError", "UnsupportedOption", "load_library"]


def load_library():
    from . import _abi
    return _abi.load()
