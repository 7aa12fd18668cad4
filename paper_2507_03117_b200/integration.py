"""Model integration: block-sparse MLPs inside transformers models.

* ``SparseGatedMLP`` replaces ``LlamaMLP`` (transformers
  models/llama/modeling_llama.py: ``down_proj(act_fn(gate_proj(x)) * up_proj(x))``,
  Eq. 1 of the paper with W = ``weight.T``; the BCSC of W is the BSR of the
  ``nn.Linear`` weight). Forward: the fused gate+up kernel plus the down
  projection. Backward: this package's dX kernels, with the weight gradients
  restricted to the stored blocks (``grad_mode="active"``). The trainable
  parameters are the BCSC ``values`` tensors.
* ``SparseGeluMLP`` replaces ``GPT2MLP`` (Conv1D weight is [in, out], the
  reference orientation; ``gelu_new`` is the tanh GELU of kernels.py:17-19,
  :42-43). It runs bias + GELU fused in the first product's epilogue.
* ``sparsify_llama`` / ``sparsify_gpt2`` swap every MLP of a model for its
  block-sparse version. The masks come from ``prune_s`` on the block norms of
  each weight (magnitude pruning, ties by (column, row)).
"""
from __future__ import annotations

import torch
from torch import nn

from . import bcsc, ops
from .bcsc import BlockMask, BlockSparseMatrix
from .kernels import bspmm_act_save, bspmm_fused, bspmm_rt, bspmm_rt_act_grad, column_sums
from .mlp import SparseMlp, _wgrad, mlp_backward, mlp_forward
from .pruner import block_norms, prune_s


def magnitude_mask(w: torch.Tensor, b: int, sparsity: float) -> BlockMask:
    """Keep the round((1-s)*blocks) largest-norm blocks (pruner.py:88-125)."""
    keep = prune_s(block_norms(w, b), sparsity)
    return BlockMask(kept=keep, regrown=torch.zeros_like(keep))


def _bcsc_param(w: BlockSparseMatrix) -> nn.Parameter:
    p = nn.Parameter(w.values, requires_grad=True)
    # The kernels read the parameter storage in place. detach() (unlike .data) shares the
    # parameter's version counter, so in-place optimizer steps / load_state_dict are visible
    # to derived caches (the float32 3xTF32 images, BlockSparseMatrix._tf32).
    w.values = p.detach()
    return p


class _GatedFn(torch.autograd.Function):
    # through the dispatcher-visible ops (ops.py): traceable by torch.compile / export
    @staticmethod
    def forward(ctx, x2d, handle: int, vg, vu, vd):
        y, a, b, g = torch.ops.blast.mlp_forward_train(x2d, handle)
        ctx.save_for_backward(x2d, a, b, g)
        ctx.handle = handle
        ctx.dtypes = (vg.dtype, vu.dtype, vd.dtype)
        return y

    @staticmethod
    def backward(ctx, dy):
        x2d, a, b, g = ctx.saved_tensors
        dx, dwg, dwu, dwd = torch.ops.blast.mlp_backward(dy.contiguous(), x2d, a, b, g, ctx.handle)
        tg, tu, td = ctx.dtypes
        return dx, None, dwg.to(tg), dwu.to(tu), dwd.to(td)


class SparseGatedMLP(nn.Module):
    """Drop-in for transformers' LlamaMLP with block-sparse gate/up/down."""

    def __init__(self, gate: BlockSparseMatrix, up: BlockSparseMatrix, down: BlockSparseMatrix):
        super().__init__()
        self.net = SparseMlp.from_caches(gate, up, down)
        self.handle = ops.register(self.net)
        self.gate_values = _bcsc_param(gate)
        self.up_values = _bcsc_param(up)
        self.down_values = _bcsc_param(down)

    @classmethod
    def from_llama(cls, mlp: nn.Module, block: int, sparsity: float,
                   dtype: torch.dtype = torch.bfloat16) -> "SparseGatedMLP":
        mats = []
        for lin in (mlp.gate_proj, mlp.up_proj, mlp.down_proj):
            w = lin.weight.detach().t().contiguous().float().cuda()  # [in, out] = reference W
            mats.append(bcsc.from_dense(w, block, magnitude_mask(w, block, sparsity), dtype=dtype))
        return cls(*mats)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        shape = x.shape
        x2d = x.reshape(-1, shape[-1]).to(self.gate_values.dtype).contiguous()
        if torch.is_grad_enabled() and (x.requires_grad or self.gate_values.requires_grad):
            y = _GatedFn.apply(x2d, self.handle, self.gate_values, self.up_values, self.down_values)
        else:
            y = torch.ops.blast.mlp_forward(x2d, self.handle)
        return y.reshape(*shape[:-1], y.shape[-1]).to(x.dtype)


class _GeluFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x2d, w1: BlockSparseMatrix, b1, w2: BlockSparseMatrix, b2, v1, v2):
        hid, pre = bspmm_act_save(x2d, w1, "gelu", bias=b1)   # bias + GELU in the epilogue
        y = bspmm_fused(hid, w2, "none", bias=b2)
        ctx.save_for_backward(x2d, pre, hid)
        ctx.w = (w1, w2)
        return y

    @staticmethod
    def backward(ctx, dy):
        x2d, pre, hid = ctx.saved_tensors
        w1, w2 = ctx.w
        dy = dy.contiguous().to(hid.dtype)
        dpre = bspmm_rt_act_grad(dy, w2, "gelu", pre)          # (dY W2^T) * gelu'(pre), fused
        dx = bspmm_rt(dpre, w1)
        dv2 = _wgrad(hid, dy, w2.rows, w2.cols, w2, full=False)
        dv1 = _wgrad(x2d, dpre, w1.rows, w1.cols, w1, full=False)
        # bias gradients: column sums accumulated in fp32 straight from the bf16 tensors
        return (dx, None, column_sums(dpre), None, column_sums(dy),
                dv1.to(w1.values.dtype), dv2.to(w2.values.dtype))


_C = 0.7978845608028654


def _gelu_tanh(x):
    return 0.5 * x * (1.0 + torch.tanh(_C * (x + 0.044715 * x * x * x)))


def _gelu_tanh_grad(x):
    u = _C * (x + 0.044715 * x ** 3)
    t = torch.tanh(u)
    return 0.5 * (1.0 + t) + 0.5 * x * (1.0 - t * t) * _C * (1.0 + 3 * 0.044715 * x * x)


class SparseGeluMLP(nn.Module):
    """Drop-in for transformers' GPT2MLP: gelu(x W1 + b1) W2 + b2 with block-sparse W."""

    def __init__(self, w1: BlockSparseMatrix, b1: torch.Tensor, w2: BlockSparseMatrix,
                 b2: torch.Tensor, dropout: float = 0.0):
        super().__init__()
        self.w1, self.w2 = w1, w2
        self.v1 = _bcsc_param(w1)
        self.v2 = _bcsc_param(w2)
        self.b1 = nn.Parameter(b1.detach().float().cuda().contiguous())
        self.b2 = nn.Parameter(b2.detach().float().cuda().contiguous())
        self.dropout = nn.Dropout(dropout)

    @classmethod
    def from_gpt2(cls, mlp: nn.Module, block: int, sparsity: float,
                  dtype: torch.dtype = torch.bfloat16) -> "SparseGeluMLP":
        mats = []
        for conv in (mlp.c_fc, mlp.c_proj):
            w = conv.weight.detach().float().cuda().contiguous()  # Conv1D: [in, out]
            mats.append(bcsc.from_dense(w, block, magnitude_mask(w, block, sparsity), dtype=dtype))
        return cls(mats[0], mlp.c_fc.bias, mats[1], mlp.c_proj.bias, mlp.dropout.p)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        shape = x.shape
        x2d = x.reshape(-1, shape[-1]).to(self.v1.dtype).contiguous()
        if torch.is_grad_enabled() and (x.requires_grad or self.v1.requires_grad):
            y = _GeluFn.apply(x2d, self.w1, self.b1, self.w2, self.b2, self.v1, self.v2)
        else:
            hid = bspmm_fused(x2d, self.w1, "gelu", bias=self.b1)
            y = bspmm_fused(hid, self.w2, "none", bias=self.b2)
        y = y.reshape(*shape[:-1], y.shape[-1]).to(x.dtype)
        return self.dropout(y) if self.dropout.p > 0 else y


def sparsify_llama(model: nn.Module, block: int = 64, sparsity: float = 0.95,
                   dtype: torch.dtype = torch.bfloat16) -> nn.Module:
    """Replace every LlamaMLP of a (Llama)ForCausalLM with SparseGatedMLP, in place."""
    layers = model.model.layers if hasattr(model, "model") else model.layers
    for layer in layers:
        layer.mlp = SparseGatedMLP.from_llama(layer.mlp, block, sparsity, dtype)
    return model


def sparsify_gpt2(model: nn.Module, block: int = 64, sparsity: float = 0.9,
                  dtype: torch.dtype = torch.bfloat16) -> nn.Module:
    """Replace every GPT2MLP of a GPT2 model with SparseGeluMLP, in place."""
    blocks = model.transformer.h if hasattr(model, "transformer") else model.h
    for blk in blocks:
        blk.mlp = SparseGeluMLP.from_gpt2(blk.mlp, block, sparsity, dtype)
    return model
