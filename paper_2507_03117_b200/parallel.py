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
* **Fused TP all-reduce.** ``FusedTPGroup`` runs the row-parallel
  down projection with the reduction inside its epilogue (``blast_tp_mlp_forward``): each
  finished fp32 partial tile is stored straight into its owner rank's receive buffer over
  peer memory, a system-scope counter on the owner counts the ranks' tiles, and the rank whose
  tile completes the set sums the partials in rank order and writes the result into every
  rank's output. The exchange overlaps the remaining tiles; no NCCL call sits on the path.
  Buffers come from torch symmetric memory (one process per GPU) or, for single-device tests,
  from plain allocations shared by "virtual" ranks.
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


class OverlappedGradAllReduce:
    """Data-parallel gradient averaging overlapped with the backward:
    pass as ``mlp_backward(..., grad_ready=reducer)``. Each weight gradient's all-reduce is
    enqueued on a side stream as soon as the gradient is ready (dWdown first, while the data
    gradient and the other weight gradients still run); ``wait()`` makes the current stream
    wait for all of them and divides by the world size. CPU tensors (gloo) reduce
    synchronously, with the same result."""

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.pending = []
        self.stream = None

    def __call__(self, index: int, grad: torch.Tensor) -> None:
        if self.world == 1:
            return
        if not grad.is_cuda or _host_staged(self.group):
            _all_reduce_sum_(grad, self.group)
            self.pending.append((None, grad))
            return
        if self.stream is None:
            self.stream = torch.cuda.Stream()
        ready = torch.cuda.Event()
        ready.record()
        with torch.cuda.stream(self.stream):
            self.stream.wait_event(ready)
            grad.record_stream(self.stream)
            work = dist.all_reduce(grad, group=self.group, async_op=True)
        self.pending.append((work, grad))

    def wait(self) -> None:
        for work, grad in self.pending:
            if work is not None:
                work.wait()  # the current stream waits for the collective
            grad.div_(self.world)
        self.pending.clear()


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


# ---------------------------------------------------------------- fused TP all-reduce
class FusedTPGroup:
    """Buffers and launch state of the fused down-projection + all-reduce (blast_tp_t in
    include/blast.h) for token count ``m``, output width ``d`` and block size ``b``.

    ``FusedTPGroup.symmetric(group, ...)`` allocates one rank's buffers with torch symmetric
    memory and exchanges the peer pointers (one process per GPU, NVLink peer access).
    ``FusedTPGroup.local(n, ...)`` puts all n ranks' buffers on the current device: n "virtual"
    ranks then run their shards one after another in one process (the protocol is identical,
    used by the single-GPU tests)."""

    def __init__(self, n: int, m: int, d: int, b: int, dtype: torch.dtype, ptrs, keep):
        self.n, self.m, self.d, self.b, self.dtype = n, m, d, b, dtype
        self.tiles = -(-m // 128)
        self.lines = -(-d // b)
        self.owned = -(-self.lines // n)
        self.ptrs = ptrs          # {"recv": [..n], "flags": [..], "y": [..], "done": [..]}
        self._keep = keep         # tensors / handles that own the memory
        self.epoch = 0

    @staticmethod
    def _sizes(n, m, d, b, dtype):
        tiles, lines = -(-m // 128), -(-d // b)
        owned = -(-lines // n)
        recv = 2 * n * tiles * owned * 128 * b * 4
        flags = tiles * owned * 4
        y = m * d * torch.tensor([], dtype=dtype).element_size()
        return recv, flags, y, 64

    @classmethod
    def local(cls, n: int, m: int, d: int, b: int, dtype=torch.bfloat16):
        if not 1 <= n <= 8:
            raise ValueError("TP group size must be 1..8")
        recv_b, flags_b, y_b, done_b = cls._sizes(n, m, d, b, dtype)
        keep, ptrs = [], {"recv": [], "flags": [], "y": [], "done": []}
        for _ in range(n):
            recv = torch.empty(recv_b // 4, dtype=torch.float32, device="cuda")
            flags = torch.zeros(flags_b // 4, dtype=torch.int32, device="cuda")
            y = torch.empty(m, d, dtype=dtype, device="cuda")
            done = torch.zeros(done_b // 4, dtype=torch.int32, device="cuda")
            keep += [recv, flags, y, done]
            for k, t in zip(("recv", "flags", "y", "done"), (recv, flags, y, done)):
                ptrs[k].append(t.data_ptr())
        g = cls(n, m, d, b, dtype, ptrs, keep)
        g._y = keep[2::4]
        return g

    @classmethod
    def symmetric(cls, group, m: int, d: int, b: int, dtype=torch.bfloat16):
        """Collective over ``group`` (one rank per GPU): symmetric-memory buffers and the peer
        pointer table of every rank."""
        import torch.distributed._symmetric_memory as symm_mem
        n = dist.get_world_size(group)
        recv_b, flags_b, y_b, done_b = cls._sizes(n, m, d, b, dtype)
        keep, ptrs = [], {}
        dev = torch.device("cuda", torch.cuda.current_device())
        for key, nbytes in (("recv", recv_b), ("flags", flags_b), ("y", y_b), ("done", done_b)):
            t = symm_mem.empty(nbytes, dtype=torch.uint8, device=dev)
            if key in ("flags", "done"):
                t.zero_()
            hdl = symm_mem.rendezvous(t, group)
            keep += [t, hdl]
            ptrs[key] = list(hdl.buffer_ptrs)
        torch.cuda.synchronize()
        dist.barrier(group)
        g = cls(n, m, d, b, dtype, ptrs, keep)
        rank = dist.get_rank(group)
        g._y = [None] * n
        g._y[rank] = keep[2 * 2].view(dtype).view(m, d)
        return g

    def desc(self, rank: int):
        from . import _lib as L
        dsc = L.TpDesc()
        dsc.n, dsc.rank, dsc.epoch = self.n, rank, self.epoch & 0xFFFFFFFF
        for r in range(self.n):
            dsc.recv[r] = self.ptrs["recv"][r]
            dsc.flags[r] = self.ptrs["flags"][r]
            dsc.y[r] = self.ptrs["y"][r]
            dsc.done[r] = self.ptrs["done"][r]
        return dsc

    def y(self, rank: int) -> torch.Tensor:
        return self._y[rank]

    def forward(self, x: torch.Tensor, net, rank: int) -> None:
        """Launch rank ``rank``'s fused forward for the current epoch (asynchronous)."""
        import ctypes as C
        from . import _lib as L
        if x.shape != (self.m, net.embed_dim) or net.embed_dim != self.d:
            raise ValueError(f"x shape {tuple(x.shape)} does not match the group ({self.m}, {self.d})")
        dg, du, dd = (mat.cache.desc() for mat in net.matrices())
        plan = net.plan()
        dsc = self.desc(rank)
        L.check(L.load().blast_tp_mlp_forward(x.data_ptr(), self.m, C.byref(dg), C.byref(du),
                                              C.byref(dd), C.byref(plan), C.byref(dsc),
                                              L.stream()), "tp_mlp_forward")

    def wait(self, rank: int) -> torch.Tensor:
        """Stream-ordered wait until rank's output holds the current epoch's sum; returns it
        and advances the epoch."""
        from . import _lib as L
        target = ((self.epoch + 1) * self.tiles * self.lines) & 0xFFFFFFFF
        L.check(L.load().blast_tp_wait(self.ptrs["done"][rank], target, L.stream()), "tp_wait")
        return self.y(rank)

    def step(self) -> None:
        self.epoch += 1

