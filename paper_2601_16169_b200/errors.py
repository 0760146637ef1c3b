"""Exception hierarchy mirroring detci::Error (error.hpp:12-48).

Status codes returned by the C-ABI map 1:1 onto these classes.
"""


class Error(RuntimeError):
    """Base class (detci::Error); also CUDA/NCCL runtime failures."""


class InputError(Error):
    """Invalid value passed by the caller (detci::InputError)."""


class FormatError(Error):
    """Malformed input file (detci::FormatError)."""


class ConfigError(Error):
    """Invalid configuration (detci::ConfigError)."""


class CapacityError(Error):
    """Allocation exceeds the memory budget (detci::CapacityError)."""


class UnsupportedError(Error):
    """Accepted by the interface, not supported by this build (detci::UnsupportedError)."""


class CudaError(Error):
    """CUDA or NCCL runtime failure (status DETCI_GPU_E_CUDA)."""


_BY_CODE = {
    1: Error,
    2: InputError,
    3: FormatError,
    4: ConfigError,
    5: CapacityError,
    6: UnsupportedError,
    7: CudaError,
}


def raise_for(code: int, message: str) -> None:
    if code != 0:
        raise _BY_CODE.get(code, Error)(message)
