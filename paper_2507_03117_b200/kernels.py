"""Block-sparse products and activations (mirrors blocksparse/kernels.py).

``bspmm`` / ``bspmm_fused`` / ``bspmm_rt`` run the tcgen05 tile engine
(csrc/spmm_tc.cuh) for b in {16, 32, 64, 128} and the CUDA-core engine
(csrc/spmm_simt.cuh) for other block sizes. Accumulation order per output
partition is fixed (ascending block index), so results are bitwise
reproducible call to call (kernels.py:117-121 contract). float32 matrices
compute in 3xTF32 (fp32-class accuracy), bfloat16 matrices in bf16 with fp32
accumulation.
"""
from __future__ import annotations

import ctypes as C
import math

import torch

from . import _arrays as A
from . import _lib as L
from .bcsc import BlockSparseMatrix

NONLINEARITIES = ("none", "relu", "gelu", "silu")
_GELU_C = float(torch.tensor(math.sqrt(2.0 / math.pi), dtype=torch.float32))
_GELU_A = float(torch.tensor(0.044715, dtype=torch.float32))


# ------------------------------------------------------------------ activations
# Scalar utilities (kernels.py:17-62). They evaluate on the GPU in the input's
# precision (float64 allowed); the fused epilogues use csrc/activations.cuh.
def _elementwise(fn):
    def wrapper(x):
        host = A.is_host(x)
        t = A.to_device(x)
        if not t.is_floating_point():
            t = t.to(torch.float64)
        return A.like_input(fn(t), host)
    wrapper.__name__ = fn.__name__
    wrapper.__doc__ = fn.__doc__
    return wrapper


@_elementwise
def sigmoid(x):
    """Split-form logistic: never evaluates exp on a large positive argument."""
    pos = x >= 0
    e = torch.exp(torch.where(pos, -x, x))
    return torch.where(pos, 1.0 / (1.0 + e), e / (1.0 + e))


def _sig(x):
    pos = x >= 0
    e = torch.exp(torch.where(pos, -x, x))
    return torch.where(pos, 1.0 / (1.0 + e), e / (1.0 + e))


@_elementwise
def silu(x):
    return x * _sig(x)


@_elementwise
def silu_grad(x):
    s = _sig(x)
    return s * (1.0 + x * (1.0 - s))


@_elementwise
def gelu(x):
    return 0.5 * x * (1.0 + torch.tanh(_GELU_C * (x + _GELU_A * x * x * x)))


@_elementwise
def relu(x):
    return torch.where((x > 0) | torch.isnan(x), x, torch.zeros_like(x))


def _act_code(f: str) -> int:
    if f not in L.ACT:
        raise ValueError(f"unknown nonlinearity {f!r}, expected one of {NONLINEARITIES}")
    return L.ACT[f]


def apply_nonlinearity(x, f: str):
    """Elementwise f on the GPU with the same device function the fused epilogue
    uses, so bspmm_fused(x, w, f) == apply_nonlinearity(bspmm(x, w), f) bit for bit."""
    code = _act_code(f)
    host = A.is_host(x)
    t = A.to_device(x, A.float_dtype(x))
    if code == 0:
        return A.like_input(t, host)
    out = torch.empty_like(t)
    L.check(L.load().blast_activation(t.data_ptr(), out.data_ptr(), t.numel(),
                                      L.dtype_code(t.dtype), code, L.stream()), "activation")
    return A.like_input(out, host)


# ------------------------------------------------------------------ products
def _check_lhs(x, w: BlockSparseMatrix, expected_cols: int) -> torch.Tensor:
    if A.ndim(x) != 2:
        raise ValueError(f"X must be 2-D, got ndim={A.ndim(x)}")
    if A.shape(x)[1] != expected_cols:
        raise ValueError(
            f"dimension mismatch: X has {A.shape(x)[1]} columns, W expects {expected_cols}")
    return A.to_device(x, w.values.dtype)


def _product(x, w: BlockSparseMatrix, act: int, transposed: bool, bias=None):
    host = A.is_host(x) or (w.host_api and not isinstance(x, torch.Tensor))
    xt = _check_lhs(x, w, w.cols if transposed else w.rows)
    m = xt.shape[0]
    out_cols = w.rows if transposed else w.cols
    y = torch.empty(m, out_cols, dtype=w.values.dtype, device=A.DEVICE)
    bias_t = None
    if bias is not None:
        bias_t = A.to_device(bias, torch.float32).reshape(-1)
        if bias_t.numel() != out_cols:
            raise ValueError(f"bias has {bias_t.numel()} entries, expected {out_cols}")
    if m:
        d = w.desc()
        lib = L.load()
        if transposed:
            rc = lib.blast_bspmm_rt(xt.data_ptr(), m, C.byref(d), y.data_ptr(), L.stream())
        else:
            rc = lib.blast_bspmm_ex(xt.data_ptr(), m, C.byref(d), L.ptr(bias_t), act,
                                    y.data_ptr(), None, L.stream())
        L.check(rc, "bspmm_rt" if transposed else "bspmm")
    return A.like_input(y, host)


def column_sums(x: torch.Tensor) -> torch.Tensor:
    """fp32 sums over the rows of a [m, n] CUDA tensor (bias gradients), deterministic."""
    if x.dim() != 2 or not x.is_cuda or x.dtype not in (torch.bfloat16, torch.float32):
        raise ValueError("column_sums expects a 2-D bf16/fp32 CUDA tensor")
    x = x.contiguous()
    out = torch.empty(x.shape[1], dtype=torch.float32, device=x.device)
    L.check(L.load().blast_column_sums(x.data_ptr(), L.dtype_code(x.dtype), x.shape[0],
                                       x.shape[1], out.data_ptr(), L.stream()), "column_sums")
    return out


def bspmm_act_save(x: torch.Tensor, w: BlockSparseMatrix, f: str, bias=None):
    """(f(X @ W + bias), X @ W + bias) in one launch: the activation and the
    pre-activation the backward needs (device tensors)."""
    code = _act_code(f)
    xt = _check_lhs(x, w, w.rows)
    m = xt.shape[0]
    y = torch.empty(m, w.cols, dtype=w.values.dtype, device=A.DEVICE)
    pre = torch.empty_like(y)
    bias_t = None if bias is None else A.to_device(bias, torch.float32).reshape(-1)
    if m:
        L.check(L.load().blast_bspmm_ex(xt.data_ptr(), m, C.byref(w.desc()), L.ptr(bias_t), code,
                                        y.data_ptr(), pre.data_ptr(), L.stream()), "bspmm_ex")
    return y, pre


def bspmm_rt_act_grad(dy: torch.Tensor, w: BlockSparseMatrix, f: str, pre: torch.Tensor):
    """(dY @ W^T) * f'(pre): the gradient through W and the activation that produced
    its input, fused in one launch (device tensors)."""
    code = _act_code(f)
    dyt = _check_lhs(dy, w, w.cols)
    m = dyt.shape[0]
    out = torch.empty(m, w.rows, dtype=w.values.dtype, device=A.DEVICE)
    if m:
        pre_t = pre.to(w.values.dtype).contiguous()
        L.check(L.load().blast_bspmm_rt_act(dyt.data_ptr(), m, C.byref(w.desc()), code,
                                            pre_t.data_ptr(), out.data_ptr(), L.stream()),
                "bspmm_rt_act")
    return out


def bspmm(x, w: BlockSparseMatrix, blk_m: int | None = None):
    """Y = X @ W for dense X (M x K) and block-sparse W (K x N) (kernels.py:86-124).

    ``blk_m`` is accepted for API compatibility; the device kernel always tiles
    rows by 128 and its result does not depend on the host-side row tiling.
    """
    if blk_m is not None and blk_m < 1:
        m = A.shape(x)[0] if A.ndim(x) >= 1 else 0
        if blk_m < m:
            raise ValueError(f"blk_m must be >= 1, got {blk_m}")
    return _product(x, w, 0, False)


def bspmm_fused(x, w: BlockSparseMatrix, f: str = "none", blk_m: int | None = None,
                bias=None):
    """f(X @ W [+ bias]) with bias and f applied in the kernel epilogue
    (kernels.py:127-140; the optional bias serves biased model layers such as
    GPT-2's Conv1D)."""
    code = _act_code(f)
    if blk_m is not None and blk_m < 1:
        raise ValueError(f"blk_m must be >= 1, got {blk_m}")
    return _product(x, w, code, False, bias)


def bspmm_rt(x, w: BlockSparseMatrix):
    """Y = X @ W.T for dense X (M x N) and block-sparse W (K x N) (kernels.py:143-170)."""
    return _product(x, w, 0, True)


def flops(m: int, n: int, k: int, nnzb: int, b: int) -> tuple[int, int]:
    """(dense, sparse) FLOP counts of an M x K by K x N product (kernels.py:173-179)."""
    return 2 * m * n * k, 2 * m * nnzb * b * b
