"""Device plumbing: torch owns device memory and streams, the C ABI does the math."""

from __future__ import annotations

import warnings

import numpy as np
import torch

from . import _lib

_checked = False

_NP2T = {
    np.dtype(np.uint16): torch.uint16,
    np.dtype(np.float32): torch.float32,
    np.dtype(np.float64): torch.float64,
    np.dtype(np.int32): torch.int32,
    np.dtype(np.uint8): torch.uint8,
    np.dtype(np.uint32): torch.uint32,
    np.dtype(np.bool_): torch.bool,
}


def require_cuda() -> torch.device:
    """The hot path runs only on a sm_100 GPU; there is no CPU fallback."""
    global _checked
    if not torch.cuda.is_available():
        raise _lib.SkyrxCudaError(
            "no CUDA device visible: paper_2602_13509_b200 runs only on B200 (sm_100a)")
    if not _checked:
        _lib.load()
        _lib.call("skyrx_device_check")
        _checked = True
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def is_device(x) -> bool:
    return isinstance(x, torch.Tensor) and x.is_cuda


def to_device(x, dtype=None) -> torch.Tensor:
    """numpy / host tensor -> contiguous device tensor (no copy if already there)."""
    dev = require_cuda()
    if isinstance(x, torch.Tensor):
        t = x
        if dtype is not None and t.dtype != dtype:
            t = t.to(dtype)
        if not t.is_cuda:
            t = t.to(dev, non_blocking=t.is_pinned())
        return t.contiguous()
    a = np.asarray(x)
    if dtype is not None:
        want = {v: k for k, v in _NP2T.items()}[dtype]
        if a.dtype != want:
            a = a.astype(want)
    a = np.ascontiguousarray(a)
    if not a.flags.writeable:  # e.g. np.frombuffer(bytes): only read by the copy below
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", UserWarning)
            return torch.from_numpy(a).to(dev)
    return torch.from_numpy(a).to(dev)


def to_host(t: torch.Tensor) -> np.ndarray:
    """Device tensor -> numpy.  Large results land in pinned memory (torch's
    caching host allocator): a pageable D2H runs at ~2 GB/s on the B200 host,
    a pinned one at the PCIe rate (~55 GB/s, tools/h2d_probe.py)."""
    t = t.detach()
    if not t.is_cuda or t.numel() * t.element_size() < (1 << 20):
        return t.cpu().numpy()
    out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    out.copy_(t, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return out.numpy()


def empty(shape, dtype) -> torch.Tensor:
    return torch.empty(shape, dtype=dtype, device=require_cuda())


def zeros(shape, dtype) -> torch.Tensor:
    return torch.zeros(shape, dtype=dtype, device=require_cuda())


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def like_input(x, t: torch.Tensor):
    """Return device tensors for device inputs, numpy for host inputs."""
    return t if is_device(x) else to_host(t)
