"""cfg4 (Llama-3-70B MLP, d=8192, h=28672, b=64, 90 % block sparsity, bf16) tensor-parallel
forward: column-parallel gate/up, row-parallel down, NCCL all-reduce of the
partial Y.

    python tools/tp_bench.py                 # one GPU: every TP degree's rank-0 shard, timed
    python tools/tp_bench.py --fused         # one GPU: fused down + all-reduce, virtual ranks
    torchrun --nproc-per-node N tools/tp_bench.py --tp [--fused]  # N GPUs: real TP

On one GPU the script times the shard a rank of an n-way TP group computes (h/n hidden
columns, exact-k uniform masks per shard) for n = 1, 2, 4, 8, reports per-rank tokens/s and
the all-reduce bytes each rank would move, and the §8(e) per-token compute vs NVLink
estimate. Under torchrun it runs the actual sharded forward (parallel.TPShardedMlp layout)
and times compute and the NCCL all-reduce separately (max over ranks). One JSON line each.
"""
import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2507_03117_b200 as bs  # noqa: E402
from paper_2507_03117_b200 import parallel  # noqa: E402

D, H, B, S = 8192, 28672, 64, 0.9


def shard_net(rank, world, seed=0):
    h = H // world
    rng = np.random.default_rng([seed, rank, world])
    ws = (bench.synth_bcsc(D, h, B, S, rng, D ** -0.5), bench.synth_bcsc(D, h, B, S, rng, D ** -0.5),
          bench.synth_bcsc(h, D, B, S, rng, 0.5 * H ** -0.5))
    return bs.SparseMlp.from_caches(*[bs.from_host(w, torch.bfloat16) for w in ws])


def timed(fn, iters=20, warmup=3):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def single_gpu(tokens):
    tf_peak = bench.load_peaks()[1]
    x = torch.randn(tokens, D, device="cuda").bfloat16()
    for world in (1, 2, 4, 8):
        net = shard_net(0, world)
        ms = timed(lambda: bs.mlp_forward(x, net, save_activations=False))
        nnzb = sum(m.cache.nnzb for m in net.matrices())
        flops = 2 * tokens * nnzb * B * B
        est = parallel.tp_roofline_ns_per_token(D, H, B, nnzb * world, world, tf_peak)
        print(json.dumps({
            "config": "cfg4 TP shard (rank 0) on one B200", "tp": world, "tokens": tokens,
            "shard_hidden": H // world, "ms": ms, "tokens_per_s_per_rank": tokens / ms * 1e3,
            "tflops": flops / (ms * 1e-3) / 1e12,
            "allreduce_bytes_per_rank": parallel.comm_bytes_per_token(D, world) * tokens,
            "estimate_ns_per_token": est}), flush=True)
        del net


def single_gpu_fused(tokens):
    """All ranks of an n-way group on one device (FusedTPGroup.local): the fused forward of
    every rank back to back vs the same shards' plain forwards; the difference is the cost of
    the fused epilogue (fp32 partial tiles to the owner, arrival counters, the last arriver's
    rank-order sum written to every rank's output), exchange bandwidth being local HBM here."""
    x = torch.randn(tokens, D, device="cuda").bfloat16()
    for world in (2, 4, 8):
        nets = [shard_net(r, world) for r in range(world)]
        group = parallel.FusedTPGroup.local(world, tokens, D, B)

        def plain():
            for n in nets:
                bs.mlp_forward(x, n, save_activations=False)

        def fused():
            for r, n in enumerate(nets):
                group.forward(x, n, r)
            for r in range(world):
                group.wait(r)
            group.step()

        t_plain, t_fused = timed(plain), timed(fused)
        print(json.dumps({
            "config": "cfg4 TP, fused down + all-reduce, all ranks on one B200", "tp": world,
            "tokens": tokens, "ms_all_ranks_plain": t_plain, "ms_all_ranks_fused": t_fused,
            "fused_overhead_per_rank_ms": (t_fused - t_plain) / world,
            "partial_bytes_per_rank": tokens * D * 4}), flush=True)
        del nets, group
        torch.cuda.empty_cache()


def multi_gpu(tokens, fused=False):
    import torch.distributed as dist
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    net = shard_net(rank, world)
    gen = torch.Generator(device="cuda").manual_seed(1234)  # same tokens on every rank
    x = torch.randn(tokens, D, device="cuda", generator=gen).bfloat16()
    y_part, _ = bs.mlp_forward(x, net, save_activations=False)

    def compute():
        return bs.mlp_forward(x, net, save_activations=False)[0]

    def reduce():
        dist.all_reduce(y_part)

    def both():
        dist.all_reduce(compute())

    res = {}
    cases = [("compute_ms", compute), ("allreduce_ms", reduce), ("forward_ms", both)]
    if fused:
        group = parallel.FusedTPGroup.symmetric(dist.group.WORLD, tokens, D, B)

        def fused_fwd():
            group.forward(x, net, rank)
            group.wait(rank)
            group.step()

        cases.append(("fused_forward_ms", fused_fwd))
    for name, fn in cases:
        dist.barrier()
        t = torch.tensor([timed(fn)], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res[name] = float(t.item())
    if rank == 0:
        nbytes = parallel.comm_bytes_per_token(D, world) * tokens
        print(json.dumps({"config": "cfg4 TP forward", "tp": world, "tokens": tokens, **res,
                          "tokens_per_s": tokens / res["forward_ms"] * 1e3,
                          "allreduce_bus_GBps": nbytes / (res["allreduce_ms"] * 1e-3) / 1e9}),
              flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--tp", action="store_true", help="real TP under torchrun")
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--fused", action="store_true", help="fused down + all-reduce")
    a = ap.parse_args()
    if a.tp:
        multi_gpu(a.tokens, a.fused)
    elif a.fused:
        single_gpu_fused(a.tokens)
    else:
        single_gpu(a.tokens)
