"""Dispatcher-visible operators: the thin torch layer over the C ABI (north star: "calls the
CUDA kernels through a thin C-ABI torch extension").

``torch.ops.blast.*`` are ``torch.library`` custom operators whose implementations are the
package's C-ABI calls (``libblast_b200.so`` through ``_lib``). They carry fake (meta)
implementations, so ``torch.compile`` / ``torch.export`` trace them as single opaque nodes
instead of breaking the graph, and they dispatch like any ATen op. A block-sparse matrix or
a ``SparseMlp`` is passed by an integer handle (``register``): its index arrays, execution
plans and 3xTF32 images stay cached on the object, which the caller keeps alive.

    h = ops.register(net)                       # SparseMlp
    y = torch.ops.blast.mlp_forward(x, h)       # inference forward (mlp.py:102-115)
    y, a, b, g = torch.ops.blast.mlp_forward_train(x, h)
    dx, dwg, dwu, dwd = torch.ops.blast.mlp_backward(dy, x, a, b, g, h)   # stored blocks
    y = torch.ops.blast.bspmm(x, ops.register(w), act)                  # kernels.py:86-140
"""
from __future__ import annotations

import itertools
import weakref

import torch

from .bcsc import BlockSparseMatrix
from .kernels import bspmm_fused
from .mlp import MlpActivations, SparseMlp, mlp_backward, mlp_forward

_ACTS = ("none", "relu", "silu", "gelu")
_REG: dict[int, weakref.ref] = {}
_IDS = itertools.count(1)


def register(obj) -> int:
    """Integer handle of a ``BlockSparseMatrix`` or ``SparseMlp`` for the ``blast`` ops (weakly
    held: the handle is valid while the caller keeps the object alive)."""
    if not isinstance(obj, (BlockSparseMatrix, SparseMlp)):
        raise TypeError(f"blast ops take BlockSparseMatrix or SparseMlp handles, got {type(obj)}")
    h = next(_IDS)
    _REG[h] = weakref.ref(obj)
    return h


def _get(handle: int, kind):
    ref = _REG.get(handle)
    obj = ref() if ref is not None else None
    if obj is None or not isinstance(obj, kind):
        raise ValueError(f"blast op: handle {handle} is not a live {kind.__name__}")
    return obj


@torch.library.custom_op("blast::bspmm", mutates_args=())
def bspmm(x: torch.Tensor, handle: int, act: int) -> torch.Tensor:
    """f(X @ W) with f in (none, relu, silu, gelu) fused in the epilogue (kernels.py:86-140)."""
    if not 0 <= act < len(_ACTS):
        raise ValueError(f"unknown nonlinearity code {act}")
    return bspmm_fused(x, _get(handle, BlockSparseMatrix), _ACTS[act])


@bspmm.register_fake
def _bspmm_fake(x, handle, act):
    w = _get(handle, BlockSparseMatrix)
    return x.new_empty(x.shape[0], w.cols, dtype=w.values.dtype)


@torch.library.custom_op("blast::mlp_forward", mutates_args=())
def mlp_forward_op(x: torch.Tensor, handle: int) -> torch.Tensor:
    """Inference forward of the gated MLP (mlp.py:102-115); G never leaves the library."""
    y, _ = mlp_forward(x, _get(handle, SparseMlp), save_activations=False)
    return y


@mlp_forward_op.register_fake
def _mlp_forward_fake(x, handle):
    net = _get(handle, SparseMlp)
    return x.new_empty(x.shape[0], net.embed_dim, dtype=net.dtype)


@torch.library.custom_op("blast::mlp_forward_train", mutates_args=())
def mlp_forward_train(x: torch.Tensor, handle: int) -> tuple[torch.Tensor, torch.Tensor,
                                                               torch.Tensor, torch.Tensor]:
    """Training forward: Y and the saved activations (gate_pre, up_out, G) (mlp.py:102-115)."""
    y, acts = mlp_forward(x, _get(handle, SparseMlp), save_activations=True)
    return y, acts.gate_pre, acts.up_out, acts.gated


@mlp_forward_train.register_fake
def _mlp_forward_train_fake(x, handle):
    net = _get(handle, SparseMlp)
    m, dt = x.shape[0], net.dtype
    return (x.new_empty(m, net.embed_dim, dtype=dt),
            *(x.new_empty(m, net.hidden_dim, dtype=dt) for _ in range(3)))


@torch.library.custom_op("blast::mlp_backward", mutates_args=())
def mlp_backward_op(dy: torch.Tensor, x: torch.Tensor, a: torch.Tensor, b: torch.Tensor,
                    g: torch.Tensor, handle: int) -> tuple[torch.Tensor, torch.Tensor,
                                                           torch.Tensor, torch.Tensor]:
    """dX and the stored-block weight gradients [nnzb, b, b] (mlp.py:118-143, grad_mode
    "active")."""
    net = _get(handle, SparseMlp)
    return mlp_backward(dy, MlpActivations(x=x, gate_pre=a, up_out=b, gated=g), net,
                        grad_mode="active")


@mlp_backward_op.register_fake
def _mlp_backward_fake(dy, x, a, b, g, handle):
    net = _get(handle, SparseMlp)
    blk = net.block
    return (dy.new_empty(x.shape[0], net.embed_dim, dtype=net.dtype),
            *(dy.new_empty(mat.cache.nnzb, blk, blk, dtype=torch.float32)
              for mat in net.matrices()))
