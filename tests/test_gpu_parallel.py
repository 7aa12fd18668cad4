"""Tensor-parallel MLP and TP prune-and-grow through the CUDA kernels: two ranks
share the one GPU of the test box and talk over gloo (NCCL needs one GPU per
rank; the protocol is identical). Results must equal the unsharded CUDA path."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist

pytestmark = pytest.mark.gpu

from test_parallel_gloo import _free_port  # noqa: E402


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_2507_03117_b200 as bs
        from paper_2507_03117_b200 import parallel
        e, h, b, m = 256, 1024, 64, 300
        rng = np.random.default_rng(0)
        wg, wu, wd = oracle.mlp_init(e, h, rng)
        x = torch.from_numpy(rng.standard_normal((m, e)).astype(np.float32)).cuda().bfloat16()
        dy = torch.from_numpy(rng.standard_normal((m, e)).astype(np.float32)).cuda().bfloat16()
        shard = parallel.TPShardedMlp.from_dense(wg, wu, wd, b, rank, world)
        y, acts = shard.forward(x)
        dx, dwg, dwu, dwd = shard.backward(dy, acts)
        g = rng.standard_normal((e, h)).astype(np.float32)
        kept, regrown, counts = parallel.generate_masks_tp(
            torch.from_numpy(parallel.column_shard(wg, b, rank, world)).cuda(),
            torch.from_numpy(parallel.column_shard(g, b, rank, world)).cuda(), b, 0.9, 1, bs)
        q.put((rank, (y.float().cpu().numpy(), dx.float().cpu().numpy(), dwg.cpu().numpy(),
                      kept.cpu().numpy(), regrown.cpu().numpy(), counts)))
    finally:
        dist.destroy_process_group()


def test_tp_two_ranks_on_one_gpu():
    import torch.multiprocessing as mp
    import oracle
    import paper_2507_03117_b200 as bs
    from paper_2507_03117_b200 import parallel
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    e, h, b, m = 256, 1024, 64, 300
    rng = np.random.default_rng(0)
    wg, wu, wd = oracle.mlp_init(e, h, rng)
    x = torch.from_numpy(rng.standard_normal((m, e)).astype(np.float32)).cuda().bfloat16()
    dy = torch.from_numpy(rng.standard_normal((m, e)).astype(np.float32)).cuda().bfloat16()
    net = bs.SparseMlp(*(bs.MaskedMatrix.dense_init(w, b, torch.bfloat16) for w in (wg, wu, wd)))
    y, acts = bs.mlp_forward(x, net)
    dx, dwg, _, _ = bs.mlp_backward(dy, acts, net)
    for r in (0, 1):
        y_r, dx_r, dwg_r, _, _, _ = res[r]
        assert oracle.max_norm_rel(y_r, y.float().cpu().numpy()) <= 2e-2
        assert oracle.max_norm_rel(dx_r, dx.float().cpu().numpy()) <= 2e-2
        c0, c1 = parallel.shard_range(h // b, r, 2)
        assert oracle.max_norm_rel(dwg_r, dwg[:, c0 * b:c1 * b].cpu().numpy()) <= 2e-2
    g = rng.standard_normal((e, h)).astype(np.float32)
    ref, rep = oracle.generate_masks(wg, g, b, 0.9)
    np.testing.assert_array_equal(np.concatenate([res[0][3], res[1][3]], 1), ref.kept)
    np.testing.assert_array_equal(np.concatenate([res[0][4], res[1][4]], 1), ref.regrown)
    assert res[0][5] == rep[:2]


def _shard_nets(wg, wu, wd, b, world, dtype):
    import paper_2507_03117_b200 as bs
    from paper_2507_03117_b200 import parallel
    return [bs.SparseMlp(*(bs.MaskedMatrix.dense_init(m, b, dtype) for m in (
        parallel.column_shard(wg, b, r, world), parallel.column_shard(wu, b, r, world),
        parallel.row_shard(wd, b, r, world)))) for r in range(world)]


@pytest.mark.parametrize("world,m,dtype", [(2, 300, torch.bfloat16), (4, 1024, torch.bfloat16),
                                           (2, 256, torch.float32), (8, 128, torch.bfloat16)])
def test_fused_tp_allreduce_virtual_ranks(world, m, dtype):
    """The fused down-projection + all-reduce (blast_tp_mlp_forward)
    with `world` virtual ranks on one device: every rank's output is the same bits, equal to
    the sum of the ranks' partial outputs in rank order, and matches the unsharded forward;
    a second epoch (the other half of the double-buffered receive area) gives the same."""
    import oracle
    import paper_2507_03117_b200 as bs
    from paper_2507_03117_b200 import parallel
    e, h, b = 512, 2048, 64
    rng = np.random.default_rng(world * 100 + m)
    wg, wu, wd = oracle.mlp_init(e, h, rng)
    for w in (wg, wu, wd):  # 85 % block sparsity so lines hold few blocks
        keep = rng.random((w.shape[0] // b, w.shape[1] // b)) < 0.15
        w *= np.kron(keep, np.ones((b, b), np.float32))
    x = torch.from_numpy(rng.standard_normal((m, e)).astype(np.float32)).cuda().to(dtype)
    nets = _shard_nets(wg, wu, wd, b, world, dtype)
    group = parallel.FusedTPGroup.local(world, m, e, b, dtype)
    # reference: each rank's partial y (its shards alone, unfused), summed in rank order in fp32
    parts = [bs.mlp_forward(x, n, save_activations=False)[0].float() for n in nets]
    ref = parts[0]
    for p in parts[1:]:
        ref = ref + p
    full = bs.SparseMlp(*(bs.MaskedMatrix.dense_init(w, b, dtype) for w in (wg, wu, wd)))
    y_full, _ = bs.mlp_forward(x, full, save_activations=False)
    for epoch in range(2):
        for r in range(world):
            group.forward(x, nets[r], r)
        ys = [group.wait(r).clone() for r in range(world)]
        torch.cuda.synchronize()
        for r in range(1, world):
            assert torch.equal(ys[r], ys[0])
        tol = 1e-4 if dtype == torch.float32 else 2e-2
        assert oracle.max_norm_rel(ys[0].float().cpu().numpy(), ref.cpu().numpy()) <= tol
        assert oracle.max_norm_rel(ys[0].float().cpu().numpy(),
                                   y_full.float().cpu().numpy()) <= tol
        group.step()
