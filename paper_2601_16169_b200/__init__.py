"""B200-native Davidson sigma build (H*C) for detci (arxiv 2601.16169).

The hot path lives in libdetci_gpu.so (csrc/, C-ABI in include/detci_gpu.h);
this package is the host-side mirror of the reference API used by the tests
and bench.py.
"""
from .errors import (CapacityError, ConfigError, CudaError, Error, FormatError, InputError,  # noqa: F401
                     UnsupportedError)

__all__ = ["Error", "InputError", "FormatError", "ConfigError", "CapacityError", "UnsupportedError",
           "CudaError"]
