"""Exception types mirroring proj/core/include/vqkv/errors.hpp:12-49."""


class Error(RuntimeError):
    """vqkv::Error"""


class InvalidInput(Error):
    """Malformed arguments: dimension mismatch, out-of-range request, bad config."""


class InvalidState(Error):
    """Operation not legal in the current object state."""


class InvalidCode(Error):
    """A code index exceeds its stage's codebook size."""


class FormatError(Error):
    """Malformed binary file; carries the byte offset of the first bad field."""

    def __init__(self, msg: str, offset: int):
        super().__init__(f"{msg} (byte offset {offset})")
        self.byte_offset = offset


class IoError(Error):
    pass


class CudaError(Error):
    """Device-side failure (no reference counterpart)."""


class Unsupported(Error):
    """Shape the device path does not implement (no reference counterpart)."""


_BY_STATUS = {1: InvalidInput, 2: InvalidState, 3: InvalidCode, 5: IoError, 6: CudaError, 7: Unsupported}


def raise_for_status(status: int, msg: str):
    if status == 4:
        raise FormatError(msg, 0)
    raise _BY_STATUS.get(status, Error)(msg)
