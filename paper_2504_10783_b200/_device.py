"""Device plumbing: the CUDA device and stream the native calls run on.

PyTorch provides device memory, streams and the current-device notion; the
native library receives raw pointers only.  There is no CPU path: asking for
a device on a machine without CUDA raises :class:`NativeError`.
"""

from __future__ import annotations

import os

from .errors import NativeError


def torch_mod():
    import torch

    return torch


def require_cuda() -> None:
    torch = torch_mod()
    if not torch.cuda.is_available():
        raise NativeError("no CUDA device: the B200 path has no CPU fallback")


def device_index() -> int:
    """Device of the calling rank: LOCAL_RANK under torchrun, else the current device."""
    require_cuda()
    torch = torch_mod()
    lr = os.environ.get("LOCAL_RANK")
    if lr is not None and torch.cuda.device_count() > int(lr):
        return int(lr)
    return torch.cuda.current_device()


def torch_device():
    return torch_mod().device("cuda", device_index())


def stream_handle() -> int:
    torch = torch_mod()
    return torch.cuda.current_stream(torch_device()).cuda_stream
