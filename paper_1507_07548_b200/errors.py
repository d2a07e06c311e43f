"""Exception hierarchy mirroring include/tmd/error.hpp:8-30, mapped from the
C-ABI status codes of include/b200md.h."""
from __future__ import annotations

from . import _abi


class Error(RuntimeError):
    """tmd::Error"""


class ModelError(Error):
    """tmd::ModelError — invalid molecular model definition"""


class ConfigError(Error):
    """tmd::ConfigError — invalid or inconsistent configuration"""


class IoError(Error):
    """tmd::IoError"""


class NumericalError(Error):
    """tmd::NumericalError — non-finite state, diverged integration"""


class CudaError(Error):
    """device / driver failure (no reference analogue)"""


_BY_CODE = {
    _abi.MODEL_ERROR: ModelError,
    _abi.CONFIG_ERROR: ConfigError,
    _abi.IO_ERROR: IoError,
    _abi.NUMERICAL_ERROR: NumericalError,
    _abi.CUDA_ERROR: CudaError,
    _abi.INVALID_ARGUMENT: ValueError,
}


def check(rc: int) -> None:
    if rc == _abi.OK:
        return
    msg = _abi.lib().b2md_last_error().decode(errors="replace")
    raise _BY_CODE.get(rc, Error)(msg)
