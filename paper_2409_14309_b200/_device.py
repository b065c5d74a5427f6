"""Device plumbing: torch is used only for device memory, streams and
``torch.distributed``; all arithmetic on the hot path runs in the native
library's kernels."""

from __future__ import annotations

import warnings

import numpy as np

try:  # torch is plumbing; importing the package must not require a GPU
    import torch
except Exception:  # pragma: no cover - torch is present in this image
    torch = None

from .errors import DeviceError


_CUDA_OK = False


def require_cuda() -> None:
    # a device, once seen, stays (the check sat on every call of the solve
    # path: torch.cuda.is_available() costs microseconds of host time)
    global _CUDA_OK
    if _CUDA_OK:
        return
    if torch is None or not torch.cuda.is_available():
        raise DeviceError(
            "the sketch engine needs a CUDA device (sm_100a); there is no CPU fallback")
    _CUDA_OK = True


try:  # the raw cudaStream_t of the current stream without building a Stream object
    _raw_stream = torch._C._cuda_getCurrentRawStream
    _cur_dev = torch._C._cuda_getDevice
except Exception:  # pragma: no cover - older torch
    _raw_stream = None


def current_stream() -> int:
    """cudaStream_t (as an int) of torch's current stream on the current
    device.  Every native call takes it; torch.cuda.current_stream() builds a
    Python Stream object (~10 us of host time), the raw accessor does not."""
    if _raw_stream is not None:
        return _raw_stream(_cur_dev())
    return torch.cuda.current_stream().cuda_stream


def device_f64(shape, fortran: bool = False, ld: int | None = None):
    """Uninitialised CUDA float64 tensor; column-major if ``fortran``.
    ``ld`` pads the leading dimension of a column-major matrix."""
    require_cuda()
    if fortran and len(shape) == 2:
        rows, cols = shape
        ld = ld or rows
        base = torch.empty((cols, ld), dtype=torch.float64, device="cuda")
        return base.t()[:rows, :]
    return torch.empty(shape, dtype=torch.float64, device="cuda")


def to_device(a: np.ndarray):
    """Copy a host numpy array (any strides) to the current CUDA device,
    keeping its layout."""
    require_cuda()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)  # read-only numpy buffers
        t = torch.from_numpy(a)
    return t.to("cuda", non_blocking=False)


def pinned_empty_f64(shape, fortran: bool = False) -> np.ndarray:
    """Page-locked host float64 array (numpy view of a pinned torch buffer)."""
    if fortran and len(shape) == 2:
        rows, cols = shape
        t = torch.empty((cols, rows), dtype=torch.float64, pin_memory=True)
        return t.numpy().T
    t = torch.empty(shape, dtype=torch.float64, pin_memory=True)
    return t.numpy()
