"""Gated block-sparse MLP: Y = (SiLU(X Wg) * (X Wu)) Wd (mirrors blocksparse/mlp.py).

Forward (mlp.py:102-115): one fused kernel computes both gate and up products
of a block column from a single load of each activation panel and applies
SiLU*mul in the epilogue; a second launch of the same engine applies the down
projection. Backward (mlp.py:118-143): dG = dY Wd^T with the gating derivative
fused into its epilogue (-> dA, dB), dX = dA Wg^T + dB Wu^T in one pass, and
weight gradients either on the full grid (the reference's dense gradients,
``grad_mode="full"``) or only on the stored blocks (``grad_mode="active"``).
"""
from __future__ import annotations


import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _arrays as A
from . import _lib as L
from . import bcsc
from .bcsc import BlockMask, BlockSparseMatrix


@dataclass(eq=False)
class MaskedMatrix:
    """Dense float32 master + block mask + BCSC cache (mlp.py:21-46), all in HBM."""
    dense: torch.Tensor
    mask: BlockMask
    cache: BlockSparseMatrix

    @classmethod
    def dense_init(cls, dense, b: int, dtype: torch.dtype = torch.float32) -> "MaskedMatrix":
        d = A.to_device(dense, torch.float32)
        gr, gc = -(-d.shape[0] // b), -(-d.shape[1] // b)
        mask = BlockMask.all_active(gr, gc, device=True)
        return cls(dense=d, mask=mask, cache=bcsc.from_dense(d, b, mask, dtype=dtype))

    @property
    def block(self) -> int:
        return self.cache.block

    def rebuild_cache(self) -> None:
        self.cache = bcsc.from_dense(self.dense, self.block, self.mask, dtype=self.cache.dtype)

    def achieved_sparsity(self) -> float:
        return self.mask.block_sparsity()


@dataclass(eq=False)
class SparseMlp:
    """gate: e x h, up: e x h, down: h x e, one block size (mlp.py:49-89)."""
    gate: MaskedMatrix
    up: MaskedMatrix
    down: MaskedMatrix
    _plan_cache: dict = field(default_factory=dict, repr=False)

    @classmethod
    def create(cls, e: int, h: int, b: int, rng: np.random.Generator,
               dtype: torch.dtype = torch.float32) -> "SparseMlp":
        """Same initialisation stream as mlp.py:61-68 (N(0, gain^2/rows), down at half gain),
        so a given numpy seed yields the reference's weights bit for bit."""
        def init(rows, cols, gain):
            w = (rng.standard_normal((rows, cols)) * (gain * np.sqrt(1.0 / rows))).astype(np.float32)
            return MaskedMatrix.dense_init(w, b, dtype)
        return cls(gate=init(e, h, 1.0), up=init(e, h, 1.0), down=init(h, e, 0.5))

    @property
    def embed_dim(self) -> int:
        return self.gate.cache.rows

    @property
    def hidden_dim(self) -> int:
        return self.gate.cache.cols

    @classmethod
    def from_caches(cls, gate: BlockSparseMatrix, up: BlockSparseMatrix,
                    down: BlockSparseMatrix) -> "SparseMlp":
        """Inference-only network from BCSC matrices (no dense masters kept in HBM)."""
        def mm(w):
            km = w._kmap()
            return MaskedMatrix(dense=None, mask=BlockMask(kept=km >= 0, regrown=torch.zeros_like(km, dtype=torch.bool)), cache=w)
        return cls(mm(gate), mm(up), mm(down))

    @property
    def block(self) -> int:
        return self.gate.block

    @property
    def dtype(self) -> torch.dtype:
        return self.gate.cache.dtype

    def matrices(self) -> tuple[MaskedMatrix, MaskedMatrix, MaskedMatrix]:
        return self.gate, self.up, self.down

    def achieved_sparsity(self) -> float:
        active = sum(m.mask.n_active for m in self.matrices())
        total = sum(m.mask.grid_rows * m.mask.grid_cols for m in self.matrices())
        return 1.0 - active / total

    def workspace(self, m: int) -> torch.Tensor:
        """Intermediate-activation buffer reused across inference calls (grow-only), so a
        forward never pays an allocation."""
        ws = self._plan_cache.get("ws")
        if ws is None or ws.dtype != self.dtype or ws.numel() < m * self.hidden_dim:
            ws = torch.empty(max(m, 1) * self.hidden_dim, dtype=self.dtype, device=A.DEVICE)
            self._plan_cache["ws"] = ws
        return ws[: m * self.hidden_dim].view(m, self.hidden_dim)

    def plan(self) -> L.MlpPlanDesc:
        """Merged gate/up step lists (csrc/plan.cu), rebuilt when a cache is replaced."""
        g, u = self.gate.cache, self.up.cache
        # keyed on the index maps: caches re-gathered for an unchanged mask share them
        key = (id(g._kmap()), id(u._kmap()))
        if self._plan_cache.get("key") != key:
            gr, gc = g.grid_rows, g.grid_cols
            gu = bcsc.build_plan(g._kmap(), u._kmap(), gr, gc, 0)
            dx = bcsc.build_plan(g._kmap(), u._kmap(), gr, gc, 1)
            desc = L.MlpPlanDesc(*(t.data_ptr() for t in gu), *(t.data_ptr() for t in dx))
            ws = self._plan_cache.get("ws")
            self._plan_cache = {"key": key, "tensors": (gu, dx, g, u), "desc": desc}
            if ws is not None:
                self._plan_cache["ws"] = ws
        return self._plan_cache["desc"]


@dataclass
class MlpActivations:
    """Saved by the forward pass for the backward (mlp.py:92-99)."""
    x: object          # M x e
    gate_pre: object   # X Wg
    up_out: object     # X Wu
    gated: object      # SiLU(gate_pre) * up_out


def _to_host_acts(acts: MlpActivations) -> MlpActivations:
    return MlpActivations(*(A.to_host(t) for t in (acts.x, acts.gate_pre, acts.up_out,
                                                    acts.gated)))


def _host_tensor(x, dt: torch.dtype) -> torch.Tensor:
    """Contiguous CPU tensor of X in the network dtype (no copy when it already is one)."""
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
    if t.dtype != dt:
        t = t.to(dt)
    return t.contiguous()


def _forward_host(x, mlp: SparseMlp, out: torch.Tensor | None, chunk_tokens: int):
    """Inference on host buffers: chunked copy-in / MLP / copy-out pipeline in the library
    (blast_mlp_forward_host). Returns once the host result is complete."""
    dt = mlp.dtype
    xt = _host_tensor(x, dt)
    m, e = xt.shape
    if out is None:
        y = torch.empty(m, e, dtype=dt, pin_memory=xt.is_pinned())
    else:
        if out.is_cuda or out.dtype != dt or tuple(out.shape) != (m, e) or not out.is_contiguous():
            raise ValueError(f"out must be a contiguous host {dt} tensor of shape {(m, e)}")
        y = out
    if m:
        dg, du, dd = (mat.cache.desc() for mat in mlp.matrices())
        plan = mlp.plan()
        L.check(L.load().blast_mlp_forward_host(xt.data_ptr(), m, C.byref(dg), C.byref(du),
                                                C.byref(dd), C.byref(plan), y.data_ptr(),
                                                chunk_tokens, L.stream()), "mlp_forward")
        torch.cuda.current_stream().synchronize()
    if isinstance(x, torch.Tensor):
        return y
    return A.to_host(y)


def mlp_forward(x, mlp: SparseMlp, save_activations: bool = True, out=None,
                chunk_tokens: int = 0):
    """Run the gated MLP; returns (y, MlpActivations) (mlp.py:102-115).

    With ``save_activations=False`` (inference) the intermediate never leaves
    the library and the second element is None. Host inputs (numpy, or a CPU
    tensor — page-locked for full overlap) then go through the library's
    chunked transfer pipeline and the result is returned on the host (``out``:
    optional preallocated host tensor; ``chunk_tokens``: 0 = automatic).
    """
    if A.ndim(x) != 2:
        raise ValueError(f"X must be 2-D (flatten batch/sequence first), got ndim={A.ndim(x)}")
    if A.shape(x)[1] != mlp.embed_dim:
        raise ValueError(f"X feature dim {A.shape(x)[1]} != embedding dim {mlp.embed_dim}")
    on_host = not (isinstance(x, torch.Tensor) and x.is_cuda)
    if not save_activations and on_host:
        return _forward_host(x, mlp, out, chunk_tokens), None
    if out is not None:
        raise ValueError("out= is only supported for host inputs with save_activations=False")
    host = A.is_host(x)
    dt = mlp.dtype
    xt = A.to_device(x, dt)
    m, e, h = xt.shape[0], mlp.embed_dim, mlp.hidden_dim
    y = torch.empty(m, e, dtype=dt, device=A.DEVICE)
    a = b = None
    if save_activations:
        a, b, g = (torch.empty(m, h, dtype=dt, device=A.DEVICE) for _ in range(3))
    elif dt == torch.float32:
        g = None  # fp32: the library keeps G as its tf32 hi / lo split in pooled scratch
    else:
        g = mlp.workspace(m)
    if m:
        dg, du, dd = (mat.cache.desc() for mat in mlp.matrices())
        plan = mlp.plan()
        L.check(L.load().blast_mlp_forward(xt.data_ptr(), m, C.byref(dg), C.byref(du), C.byref(dd),
                                           C.byref(plan), y.data_ptr(), L.ptr(a), L.ptr(b),
                                           L.ptr(g), L.stream()), "mlp_forward")
    if not save_activations:
        return A.like_input(y, host), None
    acts = MlpActivations(x=xt, gate_pre=a, up_out=b, gated=g)
    if host:
        return A.to_host(y), _to_host_acts(acts)
    return y, acts


def _wgrad(a: torch.Tensor, d: torch.Tensor, rows: int, cols: int, w: BlockSparseMatrix,
           full: bool) -> torch.Tensor:
    m = a.shape[0]
    lib = L.load()
    b = w.block
    if full:
        out = torch.empty(rows, cols, dtype=torch.float32, device=A.DEVICE)
        L.check(lib.blast_block_wgrad(a.data_ptr(), d.data_ptr(), m, rows, cols, b,
                                      L.dtype_code(a.dtype), None, None, 0, None, out.data_ptr(),
                                      L.stream()), "wgrad")
        return out
    out = torch.empty(w.nnzb, b, b, dtype=torch.float32, device=A.DEVICE)
    if w.nnzb:
        plan = w.wgrad_plan() if a.dtype == torch.bfloat16 else None
        if plan is not None:  # work list cached with the structure
            L.check(lib.blast_block_wgrad_planned(
                a.data_ptr(), d.data_ptr(), m, rows, cols, b, L.dtype_code(a.dtype),
                w.col_ptr.data_ptr(), w.block_row_idx.data_ptr(), w.nnzb, plan[0].data_ptr(),
                plan[1].data_ptr(), out.data_ptr(), L.stream()), "wgrad")
        else:
            L.check(lib.blast_block_wgrad(a.data_ptr(), d.data_ptr(), m, rows, cols, b,
                                          L.dtype_code(a.dtype), w.col_ptr.data_ptr(),
                                          w.block_row_idx.data_ptr(), w.nnzb, out.data_ptr(), None,
                                          L.stream()), "wgrad")
    return out


def mlp_backward(dy, acts: MlpActivations, mlp: SparseMlp, grad_mode: str = "full",
                 grad_ready=None):
    """Exact gradients at the saved activations (mlp.py:118-143).

    Returns (dX, dWgate, dWup, dWdown). ``grad_mode="full"`` gives the
    reference's dense float32 weight gradients over the whole grid (needed for
    regrowth and the global-norm clip); ``grad_mode="active"`` gives float32
    [nnzb, b, b] gradients of the stored blocks only, in each cache's BCSC order.

    ``grad_ready(i, grad)`` (optional, device path) is called as soon as weight gradient i
    (1 gate, 2 up, 3 down: its index in the returned tuple) has been enqueued on the current
    stream, so a data-parallel all-reduce can overlap the rest of the backward
    (parallel.OverlappedGradAllReduce). dWdown needs only G and dY and is computed first.
    """
    if acts is None:
        raise ValueError("missing saved activations: run mlp_forward first")
    if grad_mode not in ("full", "active"):
        raise ValueError(f"grad_mode must be 'full' or 'active', got {grad_mode!r}")
    m = A.shape(acts.x)[0]
    if A.shape(dy) != (m, mlp.embed_dim):
        raise ValueError(f"dY shape {A.shape(dy)} does not match forward output")
    host = A.is_host(dy)
    dt = mlp.dtype
    dyt = A.to_device(dy, dt)
    x, a, b, g = (A.to_device(t, dt) for t in (acts.x, acts.gate_pre, acts.up_out, acts.gated))
    e, h = mlp.embed_dim, mlp.hidden_dim
    dx = torch.empty(m, e, dtype=dt, device=A.DEVICE)
    da = torch.empty(m, h, dtype=dt, device=A.DEVICE)
    db = torch.empty(m, h, dtype=dt, device=A.DEVICE)
    full = grad_mode == "full"
    ready = grad_ready if grad_ready is not None else (lambda i, t: None)
    d_down = _wgrad(g, dyt, h, e, mlp.down.cache, full)
    ready(3, d_down)
    if m:
        dg, du, dd = (mat.cache.desc() for mat in mlp.matrices())
        plan = mlp.plan()
        L.check(L.load().blast_mlp_backward_dgrad(
            dyt.data_ptr(), m, a.data_ptr(), b.data_ptr(), C.byref(dg), C.byref(du), C.byref(dd),
            C.byref(plan), dx.data_ptr(), da.data_ptr(), db.data_ptr(), L.stream()), "mlp_backward")
    d_gate = _wgrad(x, da, e, h, mlp.gate.cache, full)
    ready(1, d_gate)
    d_up = _wgrad(x, db, e, h, mlp.up.cache, full)
    ready(2, d_up)
    if host:
        return tuple(A.to_host(t) for t in (dx, d_gate, d_up, d_down))
    return dx, d_gate, d_up, d_down


class GraphedMlpForward:
    """Inference forward captured once in a CUDA graph for a fixed token count (serving /
    decode): every kernel of mlp_forward(save_activations=False) replays without host launch
    work. Results are bitwise those of the eager call. The structure of ``mlp`` must not
    change after capture (a mask refresh needs a new instance); weight values may.

    Measured on one B200 (tools/graph_probe.py, Llama-3-8B MLP at 95 %): 128 tokens 36 -> 18.5
    us per forward, 8192 tokens 218 -> 216 us."""

    def __init__(self, mlp: SparseMlp, tokens: int):
        if tokens <= 0:
            raise ValueError("tokens must be positive")
        self.mlp = mlp
        self.x = torch.zeros(tokens, mlp.embed_dim, dtype=mlp.dtype, device=A.DEVICE)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # build plans, configure kernels, warm the pools
            for _ in range(2):
                mlp_forward(self.x, mlp, save_activations=False)
        torch.cuda.current_stream().wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.y, _ = mlp_forward(self.x, mlp, save_activations=False)

    def __call__(self, x: torch.Tensor) -> torch.Tensor:
        """y = mlp(x) for x of shape [tokens, embed_dim]; returns the graph's output buffer
        (overwritten by the next call)."""
        if tuple(x.shape) != tuple(self.x.shape):
            raise ValueError(f"graphed forward was captured for {tuple(self.x.shape)}, "
                             f"got {tuple(x.shape)}")
        self.x.copy_(x)
        self.graph.replay()
        return self.y

