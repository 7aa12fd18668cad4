"""Blocked prune-and-grow on the GPU (mirrors blocksparse/pruner.py).

``block_norms`` (fp64 Frobenius norms, pruner.py:88-98), ``prune_s`` (exact
top-k with ties broken toward ascending (block column, block row),
pruner.py:101-125), ``generate_masks`` (prune by weight norm, regrow by
gradient norm, pruner.py:128-157) and ``apply_mask`` (zero + BCSC repack,
pruner.py:160-186) run as CUDA kernels (csrc/prune.cu). The sparsity schedule
is host arithmetic (pruner.py:21-67).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _arrays as A
from . import _lib as L
from . import bcsc
from .bcsc import BlockMask, BlockSparseMatrix

REPORT_CSV_HEADER = "iter,s_target,kept,regrown,regrown_ratio,s_achieved"


@dataclass(frozen=True)
class SparsitySchedule:
    """Cubic ramp from initial_sparsity to max_sparsity (paper Eq. 2, pruner.py:21-50).

    The ramp ends ``decay_iters`` before ``total_iters``; ``step_size`` is the
    number of iterations between mask regenerations.
    """
    initial_sparsity: float = 0.0
    max_sparsity: float = 0.0
    total_iters: int = 1
    decay_iters: int = 0
    step_size: int = 1

    def __post_init__(self):
        if not 0.0 <= self.initial_sparsity < 1.0:
            raise ValueError(f"initial_sparsity must be in [0, 1), got {self.initial_sparsity}")
        if not 0.0 <= self.max_sparsity <= 1.0:
            raise ValueError(f"max_sparsity must be in [0, 1], got {self.max_sparsity}")
        if self.initial_sparsity > self.max_sparsity:
            raise ValueError("initial_sparsity must not exceed max_sparsity")
        if not 0 <= self.decay_iters < self.total_iters:
            raise ValueError("decay_iters must satisfy 0 <= decay_iters < total_iters")
        if self.step_size < 1:
            raise ValueError(f"step_size must be >= 1, got {self.step_size}")

    def target(self, i: int) -> float:
        return target_sparsity(i, self)


def target_sparsity(i: int, sched: SparsitySchedule) -> float:
    """s_i = s_init * f^3 + s_max * (1 - f^3), f = 1 - i / ramp; s_max once i >= ramp
    (pruner.py:53-67; this form hits both endpoints exactly)."""
    if i < 0 or i > sched.total_iters:
        raise ValueError(f"iteration {i} outside [0, {sched.total_iters}]")
    ramp = sched.total_iters - sched.decay_iters
    if i >= ramp:
        return sched.max_sparsity
    f3 = (1.0 - i / ramp) ** 3
    return sched.initial_sparsity * f3 + sched.max_sparsity * (1.0 - f3)


@dataclass(frozen=True)
class PruneReport:
    """One mask generation on one matrix (pruner.py:70-85)."""
    iteration: int
    s_target: float
    kept: int
    regrown: int
    regrown_ratio: float
    s_achieved: float

    def csv_row(self) -> str:
        return (f"{self.iteration},{self.s_target:.10g},{self.kept},{self.regrown},"
                f"{self.regrown_ratio:.10g},{self.s_achieved:.10g}")


def _check_block_input(dense, b):
    if A.ndim(dense) != 2:
        raise ValueError(f"expected a 2-D matrix, got ndim={A.ndim(dense)}")
    if b < 1:
        raise ValueError(f"block size must be >= 1, got {b}")


def _norms_device(w: torch.Tensor, g: torch.Tensor | None, b: int):
    rows, cols = w.shape
    gr, gc = -(-rows // b), -(-cols // b)
    nw = torch.empty(gr, gc, dtype=torch.float64, device=A.DEVICE)
    ng = torch.empty(gr, gc, dtype=torch.float64, device=A.DEVICE) if g is not None else None
    L.check(L.load().blast_block_norms(w.data_ptr(), L.ptr(g), rows, cols, b, _norm_code(w),
                                       nw.data_ptr(), L.ptr(ng), L.stream()), "block_norms")
    return nw, ng


def block_norms(dense, b: int):
    """Frobenius norm of each b x b block in float64 (boundary blocks zero-padded)
    (pruner.py:88-98). float32, bfloat16 and float64 inputs are read in their own precision."""
    _check_block_input(dense, b)
    host = A.is_host(dense)
    nw, _ = _norms_device(_norm_input(dense), None, b)
    return A.like_input(nw, host)


def _k_of(s: float, total: int) -> int:
    return int(math.floor((1.0 - s) * total + 0.5))  # pruner.py:111, half-up rounding


def _topk_device(norms: torch.Tensor, k: int) -> torch.Tensor:
    gr, gc = norms.shape
    keep = torch.empty(gr, gc, dtype=torch.uint8, device=A.DEVICE)
    L.check(L.load().blast_topk_mask(norms.data_ptr(), gr, gc, k, keep.data_ptr(), L.stream()),
            "topk")
    return keep


def prune_s(norms, s: float):
    """Keep round((1-s) * total) blocks with the largest norms (pruner.py:101-125).

    Ties go to ascending (block column, block row); NaN norms rank last.
    """
    if not 0.0 <= s <= 1.0:
        raise ValueError(f"sparsity must be in [0, 1], got {s}")
    host = A.is_host(norms)
    n = A.to_device(norms, torch.float64)
    gr, gc = n.shape
    keep = _topk_device(n.contiguous(), _k_of(s, gr * gc)).bool()
    return A.like_input(keep, host)


def _norm_input(x) -> torch.Tensor:
    """Device tensor of a dense matrix for the norm kernels, in its own precision: float32,
    bfloat16 and float64 are read as given (every element squared in fp64, pruner.py:95);
    other dtypes are widened to float32."""
    t = A.to_device(x)
    if t.dtype not in (torch.float32, torch.bfloat16, torch.float64):
        t = t.to(torch.float32)
    return t.contiguous()


def _norm_code(t: torch.Tensor) -> int:
    return L.F64 if t.dtype == torch.float64 else L.dtype_code(t.dtype)


_COUNTS_HOST = {}


def _pinned_counts() -> torch.Tensor:
    dev = torch.cuda.current_device()
    buf = _COUNTS_HOST.get(dev)
    if buf is None:
        buf = torch.zeros(2, dtype=torch.int64).pin_memory()
        _COUNTS_HOST[dev] = buf
    return buf


_MASK_SCRATCH = {}


def _mask_scratch(gr: int, gc: int):
    """Per (device, grid) fp64 norm grids [2, gr, gc] and device counts of generate_masks
    (stream-ordered reuse: the refresh synchronises before returning)."""
    key = (torch.cuda.current_device(), gr, gc)
    buf = _MASK_SCRATCH.get(key)
    if buf is None:
        buf = (torch.empty(2, gr, gc, dtype=torch.float64, device=A.DEVICE),
               torch.empty(2, dtype=torch.int64, device=A.DEVICE))
        _MASK_SCRATCH[key] = buf
    return buf


def generate_masks(w_dense, g_dense, b: int, s: float, iteration: int = 0):
    """kept = top-k(|W| block norms), regrown = top-k(|G| block norms) minus kept
    (pruner.py:128-157). One library call (blast_generate_masks): a fused norm pass over W
    and G, each in its own dtype, both top-k selections and the set difference; the report
    counts come back in the one host synchronisation of a refresh."""
    if A.shape(w_dense) != A.shape(g_dense):
        raise ValueError(f"weight shape {A.shape(w_dense)} != gradient shape {A.shape(g_dense)}")
    _check_block_input(w_dense, b)
    if not 0.0 <= s <= 1.0:
        raise ValueError(f"sparsity must be in [0, 1], got {s}")
    host = A.is_host(w_dense)
    w, g = _norm_input(w_dense), _norm_input(g_dense)
    rows, cols = w.shape
    gr, gc = -(-rows // b), -(-cols // b)
    total = gr * gc
    k = _k_of(s, total)
    # norm grids and device counts are scratch, reused across refreshes of this grid shape;
    # kept / regrown are returned, so they come from one fresh allocation
    nrm, counts = _mask_scratch(gr, gc)
    grids = torch.empty(2, gr, gc, dtype=torch.uint8, device=A.DEVICE)
    kept, regrown = grids[0], grids[1]
    counts_h = _pinned_counts()
    L.check(L.load().blast_generate_masks(w.data_ptr(), _norm_code(w), g.data_ptr(), _norm_code(g),
                                          rows, cols, b, k, nrm[0].data_ptr(), nrm[1].data_ptr(),
                                          kept.data_ptr(), regrown.data_ptr(), counts.data_ptr(),
                                          counts_h.data_ptr(), L.stream()), "generate_masks")
    n_kept, n_regrown = int(counts_h[0]), int(counts_h[1])
    kept_b, regrown_b = kept.view(torch.bool), regrown.view(torch.bool)
    if host:
        mask = BlockMask(kept=A.to_host(kept_b), regrown=A.to_host(regrown_b))
    else:  # disjoint by construction; the counts ride along for apply_mask (no nnzb sync)
        mask = BlockMask.trusted(kept_b, regrown_b, n_kept, n_regrown)
    report = PruneReport(iteration=iteration, s_target=s, kept=n_kept, regrown=n_regrown,
                         regrown_ratio=n_regrown / total,
                         s_achieved=1.0 - (n_kept + n_regrown) / total)
    return mask, report


def apply_mask(w_dense, mask: BlockMask, b: int, zero_regrown: bool = True,
               dtype: torch.dtype | None = None, structure: BlockSparseMatrix | None = None):
    """masked = W * expand(survivors); BCSC of the masked matrix over the active blocks
    (pruner.py:160-186). survivors = kept (zero_regrown, a fresh mask: regrown blocks
    enter as explicit zero blocks) or kept | regrown (re-application between refreshes).
    ``dtype`` is the stored value type of the returned matrix (default float32).

    ``structure``: a matrix already built for this very mask (the trainer's cache between
    refreshes). Its index arrays and execution plans are reused, so a re-application is
    a single gather launch with no host synchronisation."""
    host = A.is_host(w_dense)
    w = A.to_device(w_dense, torch.float32)
    rows, cols = w.shape
    gr, gc = -(-rows // b), -(-cols // b)
    if (mask.grid_rows, mask.grid_cols) != (gr, gc):
        raise ValueError(f"mask grid {mask.grid_rows}x{mask.grid_cols} does not match "
                         f"matrix grid {gr}x{gc} for block size {b}")
    kept, regrown = mask.device_u8()
    vdt = dtype or torch.float32
    if structure is not None and (structure.rows, structure.cols, structure.block) == (rows, cols, b):
        col_ptr, row_idx, kmap = structure.col_ptr, structure.block_row_idx, structure._kmap()
        alloc = torch.zeros if (rows % b or cols % b) else torch.empty
        values = alloc((structure.nnzb, b, b), dtype=vdt, device=A.DEVICE)
        plans = {k: v for k, v in structure._cache.items() if k[0] == "plan"}
    else:
        col_ptr, row_idx, kmap, values = bcsc._repack(w, b, kept, regrown, vdt,
                                                      nnzb=mask.known_active)
        plans = {}
    masked = torch.empty_like(w)
    L.check(L.load().blast_apply_mask_gather(w.data_ptr(), rows, cols, b, L.F32, kept.data_ptr(),
                                             regrown.data_ptr(), 1 if zero_regrown else 0,
                                             kmap.data_ptr(), masked.data_ptr(),
                                             values.data_ptr() if values.numel() else None,
                                             L.dtype_code(vdt), L.stream()), "apply_mask")
    cache = BlockSparseMatrix(rows, cols, b, col_ptr, row_idx, values, kmap, host)
    cache._cache.update(plans)
    return A.like_input(masked, host), cache
