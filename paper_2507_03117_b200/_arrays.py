"""Array plumbing shared by the API modules.

The API mirrors the reference package (numpy in, numpy out) and adds the
device-resident form (torch CUDA tensors in, CUDA tensors out). Whatever the
caller passes, compute happens on the GPU through libblast_b200.so; numpy
inputs are copied to the device and results copied back, which is what a
drop-in replacement of the reference functions has to do.
"""
from __future__ import annotations

import numpy as np
import torch

DEVICE = "cuda"


def is_host(x) -> bool:
    return isinstance(x, np.ndarray) or (not isinstance(x, torch.Tensor))


def to_device(x, dtype: torch.dtype | None = None) -> torch.Tensor:
    """numpy / python sequence / tensor -> contiguous CUDA tensor."""
    if isinstance(x, torch.Tensor):
        t = x
        if not t.is_cuda:
            t = t.to(DEVICE)
    else:
        arr = np.asarray(x)
        if arr.dtype == np.float64 and dtype is None:
            dtype = torch.float64
        t = torch.from_numpy(np.ascontiguousarray(arr)).to(DEVICE)
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    return t.contiguous()


def to_host(t: torch.Tensor) -> np.ndarray:
    if t.dtype == torch.bfloat16:
        t = t.float()
    return t.detach().cpu().numpy()


def like_input(t: torch.Tensor, host: bool):
    return to_host(t) if host else t


def float_dtype(x) -> torch.dtype:
    """Compute dtype for an input: bf16 tensors stay bf16, everything else is float32."""
    if isinstance(x, torch.Tensor) and x.dtype == torch.bfloat16:
        return torch.bfloat16
    return torch.float32


def ndim(x) -> int:
    return x.dim() if isinstance(x, torch.Tensor) else np.asarray(x).ndim


def shape(x) -> tuple:
    return tuple(x.shape) if isinstance(x, torch.Tensor) else np.asarray(x).shape
