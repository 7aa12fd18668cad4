"""Multi-process (world_size 2, gloo, CPU) tests of the sharding protocol in
paper_2507_03117_b200/parallel.py. The compute hooks are the CPU oracle (test
infrastructure); on the GPU box the same code runs the CUDA kernels over NCCL.

Checks: TP forward/backward equals the unsharded reference; TP prune-and-grow
(all-gathered norms, global top-k) gives exactly the single-process masks;
DP gradient averaging."""
import os
import socket
from types import SimpleNamespace

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2507_03117_b200 import parallel


class OracleOps:
    """The package API surface parallel.py needs, backed by the numpy oracle."""

    class MaskedMatrix:
        @staticmethod
        def dense_init(dense, b, dtype=None):
            d = np.ascontiguousarray(np.asarray(dense, dtype=np.float32))
            return SimpleNamespace(dense=d, cache=oracle.from_dense(
                d, b, oracle.Mask(np.ones((-(-d.shape[0] // b), -(-d.shape[1] // b)), bool),
                                  np.zeros((-(-d.shape[0] // b), -(-d.shape[1] // b)), bool))))

    class SparseMlp:
        def __init__(self, gate, up, down):
            self.mats = (gate.cache, up.cache, down.cache)

    @staticmethod
    def mlp_forward(x, net, save_activations=True):
        y, acts = oracle.mlp_forward(np.asarray(x), *net.mats)
        return torch.from_numpy(y), (acts if save_activations else None)

    @staticmethod
    def mlp_backward(dy, acts, net, grad_mode="full"):
        dx, dg, du, dd = oracle.mlp_backward(np.asarray(dy), acts, *net.mats)
        return torch.from_numpy(dx), dg, du, dd

    @staticmethod
    def prune_s(norms, s):
        return torch.from_numpy(oracle.prune_s(np.asarray(norms), s))

    @staticmethod
    def block_norms(w, b):
        return torch.from_numpy(oracle.block_norms(np.asarray(w), b))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    finally:
        dist.destroy_process_group()


def run_world(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return [out[r] for r in range(world)]


E, H, B, M = 32, 64, 8, 12


def _weights():
    rng = np.random.default_rng(0)
    return oracle.mlp_init(E, H, rng), rng.standard_normal((M, E)).astype(np.float32), \
        rng.standard_normal((M, E)).astype(np.float32)


def _tp_fwd_bwd(rank, world):
    (wg, wu, wd), x, dy = _weights()
    shard = parallel.TPShardedMlp.from_dense(wg, wu, wd, B, rank, world, ops=OracleOps)
    y, acts = shard.forward(torch.from_numpy(x))
    dx, dwg, dwu, dwd = shard.backward(torch.from_numpy(dy), acts)
    y_inf, none = shard.forward(torch.from_numpy(x), save_activations=False)
    assert none is None and np.array_equal(y_inf.numpy(), y.numpy())
    return y.numpy(), dx.numpy(), dwg, dwu, dwd


def test_tp_forward_backward_matches_unsharded():
    res = run_world(_tp_fwd_bwd)
    (wg, wu, wd), x, dy = _weights()
    full = [oracle.from_dense(w, B) for w in (wg, wu, wd)]
    y_ref, acts = oracle.mlp_forward(x, *full)
    dx_ref, dwg_ref, dwu_ref, dwd_ref = oracle.mlp_backward(dy, acts, *full)
    for rank, (y, dx, dwg, dwu, dwd) in enumerate(res):
        assert oracle.rel_err(y, y_ref) <= 1e-5
        assert oracle.rel_err(dx, dx_ref) <= 1e-5
        c0, c1 = parallel.shard_range(H // B, rank, 2)
        assert oracle.rel_err(dwg, dwg_ref[:, c0 * B:c1 * B]) <= 1e-5
        assert oracle.rel_err(dwu, dwu_ref[:, c0 * B:c1 * B]) <= 1e-5
        assert oracle.rel_err(dwd, dwd_ref[c0 * B:c1 * B, :]) <= 1e-5


def _tp_masks(rank, world):
    rng = np.random.default_rng(5)
    w = rng.standard_normal((E, H)).astype(np.float32)
    g = rng.standard_normal((E, H)).astype(np.float32)
    w[:, :16] = 1.0  # exact ties across the shard boundary
    out = {}
    for dim, shard_fn in ((1, parallel.column_shard), (0, parallel.row_shard)):
        src_w = w if dim == 1 else w.T.copy()
        src_g = g if dim == 1 else g.T.copy()
        kept, regrown, counts = parallel.generate_masks_tp(
            shard_fn(src_w, B, rank, world), shard_fn(src_g, B, rank, world), B, 0.8, dim,
            OracleOps)
        out[dim] = (kept.numpy(), regrown.numpy(), counts)
    return out


def test_tp_global_masks_bit_exact():
    res = run_world(_tp_masks)
    rng = np.random.default_rng(5)
    w = rng.standard_normal((E, H)).astype(np.float32)
    g = rng.standard_normal((E, H)).astype(np.float32)
    w[:, :16] = 1.0
    for dim in (1, 0):
        src_w = w if dim == 1 else w.T.copy()
        src_g = g if dim == 1 else g.T.copy()
        ref, rep = oracle.generate_masks(src_w, src_g, B, 0.8)
        kept = np.concatenate([r[dim][0] for r in res], axis=dim)
        regrown = np.concatenate([r[dim][1] for r in res], axis=dim)
        np.testing.assert_array_equal(kept, ref.kept)
        np.testing.assert_array_equal(regrown, ref.regrown)
        for r in res:
            assert r[dim][2] == rep[:2]


def _dp_mean(rank, world):
    t = [torch.full((3, 4), float(rank + 1)), torch.arange(5, dtype=torch.float32) * (rank + 1)]
    parallel.allreduce_mean_(t)
    return [x.numpy() for x in t]


def test_dp_gradient_average():
    for out in run_world(_dp_mean):
        np.testing.assert_array_equal(out[0], np.full((3, 4), 1.5))
        np.testing.assert_allclose(out[1], np.arange(5) * 1.5)


def _dp_overlapped(rank, world):
    # the backward's hook order (dWdown first), then wait(): same averages as allreduce_mean_
    red = parallel.OverlappedGradAllReduce()
    t = [torch.full((3, 4), float(rank + 1)), torch.arange(5, dtype=torch.float32) * (rank + 1),
         torch.full((2, 2), 10.0 * (rank + 1))]
    for i in (2, 0, 1):
        red(i + 1, t[i])
    red.wait()
    return [x.numpy() for x in t]


def test_dp_overlapped_gradient_average():
    for out in run_world(_dp_overlapped):
        np.testing.assert_array_equal(out[0], np.full((3, 4), 1.5))
        np.testing.assert_allclose(out[1], np.arange(5) * 1.5)
        np.testing.assert_array_equal(out[2], np.full((2, 2), 15.0))


def test_shard_ranges_and_roofline_helpers():
    assert parallel.shard_range(448, 3, 8) == (168, 224)
    with pytest.raises(ValueError):
        parallel.shard_range(10, 0, 3)
    r = parallel.tp_roofline_ns_per_token(8192, 28672, 64, 3 * 5734, 8, 1636.8)
    assert r["bound"] == "comm"
    assert parallel.comm_bytes_per_token(8192, 2) == 16384.0
