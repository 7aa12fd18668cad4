"""Multi-GPU sharding of the block-sparse gated MLP.

The reference has no distribution. This module adds the two
layouts the north star names, one process per GPU over ``torch.distributed``
(NCCL on B200 / NVLink; gloo works for the CPU protocol tests):

* **Tensor parallel (Llama-3-70B MLP, cfg4).** Rank k owns hidden block
  columns [k*h/n, (k+1)*h/n) of gate and up (column-parallel) and the same
  block rows of down (row-parallel). Forward: the local fused gate+up gives
  G_k; the local down projection gives a partial Y_k; an all-reduce sums the
  partials. Backward mirrors it: dG_k from the replicated dY, local dW, and an
  all-reduce of the partial dX. h must split into whole blocks per rank.
* **Prune-and-grow under TP** stays bit-exact with the single-GPU masks. Each
  rank computes the fp64 block norms of its shard, the norm grids are
  all-gathered, and every rank runs the same global top-k (ties by global
  (column, row)) and keeps its slice. A per-shard top-k would change the
  semantics of pruner.py:101-125.
* **Data parallel (pretraining, cfg2).** Replicated weights, token-sharded
  batches, weight gradients averaged with one all-reduce per step. Masks stay
  identical on all ranks because they derive from identical weights and the
  all-reduced gradients.

The compute hooks (``ops``) default to this package (CUDA kernels). Tests may
inject the CPU oracle to check the communication protocol on gloo.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist


def shard_range(total_blocks: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block range of `rank`; total must divide evenly (block-aligned TP)."""
    if total_blocks % world:
        raise ValueError(f"{total_blocks} block lines do not split over {world} ranks")
    per = total_blocks // world
    return rank * per, (rank + 1) * per


def column_shard(dense, b: int, rank: int, world: int):
    """Columns [c0*b, c1*b) of a dense [rows, cols] matrix (gate/up of a TP rank)."""
    gc = -(-dense.shape[1] // b)
    c0, c1 = shard_range(gc, rank, world)
    return dense[:, c0 * b: min(c1 * b, dense.shape[1])]


def row_shard(dense, b: int, rank: int, world: int):
    """Rows [r0*b, r1*b) of a dense matrix (down projection of a TP rank)."""
    gr = -(-dense.shape[0] // b)
    r0, r1 = shard_range(gr, rank, world)
    return dense[r0 * b: min(r1 * b, dense.shape[0]), :]


def _host_staged(group) -> bool:
    """gloo (CPU protocol tests, or ranks sharing one GPU) reduces host tensors."""
    return dist.get_backend(group) == "gloo"


def _all_reduce_sum_(t: torch.Tensor, group=None) -> torch.Tensor:
    """In-place sum over ranks. NCCL reduces CUDA bf16/fp32 tensors directly over
    NVLink; on gloo the tensor is staged through host memory in fp32."""
    if _host_staged(group) and (t.is_cuda or t.dtype == torch.bfloat16):
        h = t.detach().float().cpu()
        dist.all_reduce(h, group=group)
        t.copy_(h.to(t.device, t.dtype))
    else:
        dist.all_reduce(t, group=group)
    return t


def _all_gather_cat(t: torch.Tensor, dim: int, group=None) -> torch.Tensor:
    world = dist.get_world_size(group)
    src = t.detach().cpu() if (_host_staged(group) and t.is_cuda) else t.contiguous()
    parts = [torch.empty_like(src) for _ in range(world)]
    dist.all_gather(parts, src.contiguous(), group=group)
    return torch.cat(parts, dim=dim).to(t.device)


def global_keep(local_norms: torch.Tensor, s: float, shard_dim: int, ops, group=None) -> torch.Tensor:
    """Global top-k mask restricted to this rank's shard of the block grid.

    local_norms: float64 [gr_k, gc_k] of this rank's shard; shard_dim = 1 for column
    shards (gate/up), 0 for row shards (down). Every rank evaluates prune_s on the
    same full grid, so the kept set equals the single-GPU one bit for bit.
    """
    full = _all_gather_cat(local_norms, shard_dim, group)
    keep = ops.prune_s(full, s)
    keep = keep if isinstance(keep, torch.Tensor) else torch.from_numpy(np.asarray(keep))
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    n = local_norms.shape[shard_dim]
    sl = slice(rank * n, (rank + 1) * n)
    return keep[:, sl] if shard_dim == 1 else keep[sl, :]


def generate_masks_tp(w_shard, g_shard, b: int, s: float, shard_dim: int, ops, group=None,
                      iteration: int = 0):
    """pruner.py:128-157 over a TP-sharded matrix: returns (kept, regrown, counts) of
    this rank's shard; counts are the GLOBAL (kept, regrown) totals."""
    nw = ops.block_norms(w_shard, b)
    ng = ops.block_norms(g_shard, b)
    nw = nw if isinstance(nw, torch.Tensor) else torch.from_numpy(np.asarray(nw))
    ng = ng if isinstance(ng, torch.Tensor) else torch.from_numpy(np.asarray(ng))
    kept = global_keep(nw, s, shard_dim, ops, group)
    gsel = global_keep(ng, s, shard_dim, ops, group)
    kept = kept.to(torch.bool)
    regrown = gsel.to(torch.bool) & ~kept
    counts = torch.tensor([int(kept.sum()), int(regrown.sum())], dtype=torch.int64,
                          device=nw.device)
    _all_reduce_sum_(counts, group)
    return kept, regrown, (int(counts[0]), int(counts[1]))


def allreduce_mean_(tensors, group=None) -> None:
    """Data-parallel gradient averaging (in place)."""
    world = dist.get_world_size(group)
    for t in tensors:
        _all_reduce_sum_(t, group)
        t.div_(world)


@dataclass
class TPShardedMlp:
    """One rank's shard of a gated sparse MLP: gate/up column shards, down row shard.

    ``net`` is a SparseMlp built from the shards (this package's CUDA path by
    default). forward/backward return full (replicated) activations / gradients
    after the all-reduces; weight gradients stay sharded.
    """
    net: object
    rank: int
    world: int
    ops: object
    group: object = None

    @classmethod
    def from_dense(cls, wg, wu, wd, b: int, rank: int, world: int, ops=None, group=None,
                   dtype=torch.bfloat16):
        if ops is None:
            import paper_2507_03117_b200 as ops  # noqa: PLW0127 (the CUDA path)
        mats = []
        for dense in (column_shard(wg, b, rank, world), column_shard(wu, b, rank, world),
                      row_shard(wd, b, rank, world)):
            mats.append(ops.MaskedMatrix.dense_init(dense, b, dtype))
        return cls(ops.SparseMlp(*mats), rank, world, ops, group)

    def forward(self, x, save_activations: bool = True):
        """Column/row-parallel forward + all-reduce of the partial Y. Inference
        (save_activations=False) keeps the intermediate inside the library and returns
        (y, None)."""
        y_part, acts = self.ops.mlp_forward(x, self.net, save_activations=save_activations)
        y = _all_reduce_sum_(torch.as_tensor(y_part), self.group)
        return y, acts

    def backward(self, dy, acts, grad_mode: str = "full"):
        dx_part, dwg, dwu, dwd = self.ops.mlp_backward(dy, acts, self.net, grad_mode=grad_mode)
        dx = _all_reduce_sum_(torch.as_tensor(dx_part), self.group)
        return dx, dwg, dwu, dwd


def comm_bytes_per_token(d: int, world: int, elt: int = 2) -> float:
    """Ring all-reduce bytes each rank sends per token for the partial Y."""
    return 2.0 * (world - 1) / world * d * elt


def tp_roofline_ns_per_token(d: int, h: int, b: int, nnzb_total: int, world: int,
                             tflops: float, link_gbs: float = 770.0) -> dict:
    """Per-rank compute vs NVLink time per token for the TP forward."""
    flop = 2.0 * nnzb_total * b * b / world
    t_c = flop / (tflops * 1e12) * 1e9
    t_n = comm_bytes_per_token(d, world) / (link_gbs * 1e9) * 1e9
    return {"compute_ns": t_c, "comm_ns": t_n, "bound": "comm" if t_n > t_c else "compute"}
