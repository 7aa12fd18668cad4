"""GPU parity of the gated sparse MLP forward/backward (ports of tests/test_mlp.py)."""
import numpy as np
import pytest
import torch

import oracle
from conftest import golden, golden_bcsc

pytestmark = pytest.mark.gpu
bs = pytest.importorskip("paper_2507_03117_b200")

SILU_1 = 0.7310585786300049


def mlp_from_golden(d, i, dtype=torch.float32):
    mats = []
    for n in ("gate", "up", "down"):
        w = golden_bcsc(d, f"c{i}_{n}")
        mask = bs.BlockMask(kept=d[f"c{i}_{n}_kept"], regrown=d[f"c{i}_{n}_regrown"])
        dense = torch.from_numpy(d[f"c{i}_{n}_dense"]).cuda()
        mats.append(bs.MaskedMatrix(dense=dense, mask=mask, cache=bs.from_host(w, dtype)))
    return bs.SparseMlp(*mats), [golden_bcsc(d, f"c{i}_{n}") for n in ("gate", "up", "down")]


def round_bf16(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).bfloat16().float().numpy()


class TestGolden:
    d = golden("mlp")

    @pytest.mark.parametrize("i", range(5))
    def test_fp32_forward_backward(self, i):
        d = self.d
        net, _ = mlp_from_golden(d, i)
        y, acts = bs.mlp_forward(d[f"c{i}_x"], net)
        for got, key in ((y, "y"), (acts.gate_pre, "a"), (acts.up_out, "b"), (acts.gated, "g")):
            assert oracle.rel_err(got, d[f"c{i}_{key}"]) <= 1e-5, key
            assert oracle.max_norm_rel(got, d[f"c{i}_{key}"]) <= 1e-4, key
        grads = bs.mlp_backward(d[f"c{i}_dy"], acts, net)
        for got, key in zip(grads, ("dx", "dwg", "dwu", "dwd")):
            assert oracle.rel_err(got, d[f"c{i}_{key}"]) <= 1e-4, key
            assert oracle.max_norm_rel(got, d[f"c{i}_{key}"]) <= 1e-4, key

    @pytest.mark.parametrize("i", range(5))
    def test_bf16_forward_backward(self, i):
        d = self.d
        net, mats = mlp_from_golden(d, i, torch.bfloat16)
        mats = [m._replace(values=round_bf16(m.values)) for m in mats]
        x, dy = round_bf16(d[f"c{i}_x"]), round_bf16(d[f"c{i}_dy"])
        y_ref, acts_ref = oracle.mlp_forward(x, *mats)
        grads_ref = oracle.mlp_backward(dy, acts_ref, *mats)
        xt = torch.from_numpy(x).cuda().bfloat16()
        y, acts = bs.mlp_forward(xt, net)
        assert oracle.max_norm_rel(y.float().cpu().numpy(), y_ref) <= 2e-2
        grads = bs.mlp_backward(torch.from_numpy(dy).cuda().bfloat16(), acts, net)
        for got, ref, key in zip(grads, grads_ref, ("dx", "dwg", "dwu", "dwd")):
            assert oracle.max_norm_rel(got.float().cpu().numpy(), ref) <= 2e-2, key

    @pytest.mark.parametrize("i", [1, 2, 4])
    @pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
    def test_active_grads_are_full_grads_on_stored_blocks(self, i, dtype):
        d = self.d
        net, _ = mlp_from_golden(d, i, dtype)
        x = torch.from_numpy(d[f"c{i}_x"]).cuda().to(dtype)
        dy = torch.from_numpy(d[f"c{i}_dy"]).cuda().to(dtype)
        _, acts = bs.mlp_forward(x, net)
        full = bs.mlp_backward(dy, acts, net, grad_mode="full")
        act = bs.mlp_backward(dy, acts, net, grad_mode="active")
        assert torch.equal(full[0], act[0])
        for mat, g_full, g_act in zip(net.matrices(), full[1:], act[1:]):
            w = mat.cache
            blocks = bs.from_dense(g_full, w.block, bs.BlockMask(kept=mat.mask.kept,
                                                                  regrown=mat.mask.regrown))
            tol = 1e-5 if dtype == torch.float32 else 1e-3
            assert torch.allclose(blocks.values, g_act, rtol=tol, atol=tol)


def build_mlp(rng, e, h, b, sparsity=0.0, dtype=torch.float32):
    net = bs.SparseMlp.create(e, h, b, rng, dtype)
    if sparsity > 0:
        for mat in net.matrices():
            g = rng.standard_normal(tuple(mat.dense.shape)).astype(np.float32)
            mask, _ = bs.generate_masks(mat.dense, torch.from_numpy(g).cuda(), b, sparsity)
            mat.mask = mask
            mat.dense, mat.cache = bs.apply_mask(mat.dense, mask, b, dtype=dtype)
    return net


def dense_f64(net):
    return [m.dense.double().cpu().numpy() for m in net.matrices()]


def gated_mlp_f64(x, wg, wu, wd):
    a = x @ wg
    b = x @ wu
    return ((a / (1.0 + np.exp(-a))) * b) @ wd


class TestForward:
    def test_zero_weights_zero_output(self):
        z = np.zeros((8, 8), dtype=np.float32)
        net = bs.SparseMlp(*(bs.MaskedMatrix.dense_init(z, 4) for _ in range(3)))
        x = np.random.default_rng(0).standard_normal((5, 8)).astype(np.float32)
        y, _ = bs.mlp_forward(x, net)
        np.testing.assert_array_equal(y, np.zeros((5, 8)))

    def test_identity_weights_hand_value(self):
        eye = np.eye(8, dtype=np.float32)
        net = bs.SparseMlp(*(bs.MaskedMatrix.dense_init(eye, 4) for _ in range(3)))
        y, _ = bs.mlp_forward(eye, net)
        assert oracle.rel_err(y, np.diag(np.full(8, SILU_1))) <= 1e-6

    @pytest.mark.parametrize("seed", range(6))
    def test_random_sweep(self, seed):
        rng = np.random.default_rng(100 + seed)
        e, h = int(rng.integers(2, 33)), int(rng.integers(2, 33))
        b = int(rng.integers(1, 9))
        net = build_mlp(rng, e, h, b, float(rng.choice([0.0, 0.3, 0.6])))
        x = rng.standard_normal((int(rng.integers(1, 12)), e)).astype(np.float32)
        y, _ = bs.mlp_forward(x, net)
        assert oracle.rel_err(y, gated_mlp_f64(x.astype(np.float64), *dense_f64(net))) <= 1e-5

    @pytest.mark.parametrize("b,s", [(16, 0.5), (64, 0.9), (32, 0.75)])
    def test_tensor_core_shapes_match_dense_composition(self, b, s):
        rng = np.random.default_rng(b)
        net = build_mlp(rng, 4 * b, 8 * b, b, s)
        x = rng.standard_normal((300, 4 * b)).astype(np.float32)
        y, _ = bs.mlp_forward(x, net)
        ref = gated_mlp_f64(x.astype(np.float64), *dense_f64(net))
        assert oracle.rel_err(y, ref) <= 1e-5

    def test_shape_mismatch(self):
        net = build_mlp(np.random.default_rng(2), 8, 8, 4)
        with pytest.raises(ValueError, match="feature dim"):
            bs.mlp_forward(np.ones((3, 9), dtype=np.float32), net)

    def test_inference_mode_matches_training_mode(self):
        rng = np.random.default_rng(12)
        net = build_mlp(rng, 256, 512, 64, 0.9, torch.bfloat16)
        x = torch.randn(333, 256, device="cuda").bfloat16()
        y1, acts = bs.mlp_forward(x, net)
        y2, none = bs.mlp_forward(x, net, save_activations=False)
        assert none is None and torch.equal(y1, y2)

    @pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
    @pytest.mark.parametrize("chunk", [0, 128, 300, 5000])
    def test_host_pipeline_matches_device(self, dtype, chunk):
        """Host buffers through the chunked copy/compute pipeline: bit-identical to the
        device-resident forward (rows are independent, so chunking changes nothing)."""
        rng = np.random.default_rng(13)
        net = build_mlp(rng, 256, 512, 64, 0.8, dtype)
        x = torch.randn(2100, 256, device="cuda").to(dtype)  # auto: half/full/ragged chunks
        y_dev, _ = bs.mlp_forward(x, net, save_activations=False)
        xh = x.cpu().pin_memory()
        y_pin, none = bs.mlp_forward(xh, net, save_activations=False, chunk_tokens=chunk)
        assert none is None and not y_pin.is_cuda and y_pin.is_pinned()
        assert torch.equal(y_pin, y_dev.cpu())
        out = torch.full((2100, 256), float("nan"), dtype=dtype)  # pageable preallocated out
        y_out, _ = bs.mlp_forward(x.cpu(), net, save_activations=False, out=out,
                                  chunk_tokens=chunk)
        assert y_out is out and torch.equal(out, y_dev.cpu())
        if dtype == torch.float32:
            y_np, _ = bs.mlp_forward(x.cpu().numpy(), net, save_activations=False)
            assert isinstance(y_np, np.ndarray)
            np.testing.assert_array_equal(y_np, y_dev.cpu().numpy())

    def test_host_pipeline_errors(self):
        net = build_mlp(np.random.default_rng(2), 8, 8, 4)
        with pytest.raises(ValueError, match="out"):
            bs.mlp_forward(np.ones((3, 8), np.float32), net, save_activations=False,
                           out=torch.empty(3, 7))
        y, _ = bs.mlp_forward(np.ones((0, 8), np.float32), net, save_activations=False)
        assert y.shape == (0, 8)


class TestBackward:
    def test_zero_upstream_zero_grads(self):
        rng = np.random.default_rng(4)
        net = build_mlp(rng, 8, 8, 4, 0.5)
        x = rng.standard_normal((5, 8)).astype(np.float32)
        _, acts = bs.mlp_forward(x, net)
        for g in bs.mlp_backward(np.zeros((5, 8), np.float32), acts, net):
            np.testing.assert_array_equal(g, np.zeros_like(g))

    def test_scalar_network_hand_chain_rule(self):
        x, w1, w2, w3 = 0.7, 0.9, -1.1, 1.3
        mk = lambda v: bs.MaskedMatrix.dense_init(np.array([[v]], np.float32), 1)  # noqa: E731
        net = bs.SparseMlp(mk(w1), mk(w2), mk(w3))
        _, acts = bs.mlp_forward(np.array([[x]], np.float32), net)
        dx, dg, du, dd = bs.mlp_backward(np.array([[1.0]], np.float32), acts, net)
        a = x * w1
        sig = 1.0 / (1.0 + np.exp(-a))
        s = a * sig
        bb = x * w2
        da = w3 * bb * sig * (1.0 + a * (1.0 - sig))
        assert dd[0, 0] == pytest.approx(s * bb, rel=1e-6)
        assert dg[0, 0] == pytest.approx(x * da, rel=1e-6)
        assert du[0, 0] == pytest.approx(x * w3 * s, rel=1e-6)
        assert dx[0, 0] == pytest.approx(da * w1 + w3 * s * w2, rel=1e-6)

    @pytest.mark.parametrize("seed,sparsity", [(0, 0.0), (1, 0.5), (2, 0.75)])
    def test_grads_match_finite_differences(self, seed, sparsity):
        rng = np.random.default_rng(200 + seed)
        e, h, b = int(rng.integers(2, 17)), int(rng.integers(2, 17)), int(rng.integers(1, 5))
        net = build_mlp(rng, e, h, b, sparsity)
        x = rng.standard_normal((4, e)).astype(np.float32)
        y, acts = bs.mlp_forward(x, net)
        grads = bs.mlp_backward(y, acts, net)
        wg, wu, wd = dense_f64(net)
        point = {"x": x.astype(np.float64), "wg": wg, "wu": wu, "wd": wd}

        def loss(name, arr):
            args = dict(point, **{name: arr})
            out = gated_mlp_f64(args["x"], args["wg"], args["wu"], args["wd"])
            return 0.5 * float(np.sum(out * out))

        for got, name in zip(grads, ("x", "wg", "wu", "wd")):
            base = point[name].copy()
            fd = np.zeros_like(base)
            for idx in np.ndindex(base.shape):
                hp, hm = base.copy(), base.copy()
                hp[idx] += 1e-3
                hm[idx] -= 1e-3
                fd[idx] = (loss(name, hp) - loss(name, hm)) / 2e-3
            assert oracle.rel_err(got, fd) <= 1e-3, name

    def test_weight_grads_dense_over_pruned_blocks(self):
        rng = np.random.default_rng(5)
        net = build_mlp(rng, 16, 16, 4, 0.5)
        x = rng.standard_normal((6, 16)).astype(np.float32)
        y, acts = bs.mlp_forward(x, net)
        _, dg, _, _ = bs.mlp_backward(y, acts, net)
        inactive = ~net.gate.mask.active.cpu().numpy()
        assert inactive.any()
        assert np.any(dg[bs.expand_mask(inactive, 4, 16, 16)] != 0.0)

    def test_missing_activations(self):
        net = build_mlp(np.random.default_rng(6), 8, 8, 4)
        with pytest.raises(ValueError, match="saved activations"):
            bs.mlp_backward(np.ones((2, 8), np.float32), None, net)

    def test_bad_upstream_shape(self):
        rng = np.random.default_rng(7)
        net = build_mlp(rng, 8, 8, 4)
        _, acts = bs.mlp_forward(rng.standard_normal((3, 8)).astype(np.float32), net)
        with pytest.raises(ValueError, match="dY shape"):
            bs.mlp_backward(np.ones((4, 8), np.float32), acts, net)

    @pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
    def test_backward_deterministic(self, dtype):
        rng = np.random.default_rng(8)
        net = build_mlp(rng, 256, 512, 64, 0.8, dtype)
        x = torch.randn(300, 256, device="cuda").to(dtype)
        dy = torch.randn(300, 256, device="cuda").to(dtype)
        _, acts = bs.mlp_forward(x, net)
        g1 = bs.mlp_backward(dy, acts, net)
        g2 = bs.mlp_backward(dy, acts, net)
        for a, b in zip(g1, g2):
            assert torch.equal(a, b)


@pytest.mark.parametrize("m", [128, 300, 1024])
def test_graphed_forward_equals_eager(m):
    """CUDA-graph capture of the inference forward: bitwise the eager result, reusable."""
    rng = np.random.default_rng(m)
    mats = []
    for rows, cols in ((512, 1536), (512, 1536), (1536, 512)):
        w = oracle.random_bcsc(rows, cols, 64, 0.9, rng)
        w = w._replace(values=(w.values / np.sqrt(rows)).astype(np.float32))
        mats.append(bs.from_host(w, torch.bfloat16))
    net = bs.SparseMlp.from_caches(*mats)
    fwd = bs.GraphedMlpForward(net, m)
    for seed in (1, 2):
        x = torch.from_numpy(np.random.default_rng(seed).standard_normal((m, 512))
                             .astype(np.float32)).cuda().bfloat16()
        y_eager, _ = bs.mlp_forward(x, net, save_activations=False)
        y_graph = fwd(x)
        torch.cuda.synchronize()
        assert torch.equal(y_graph, y_eager)
    with pytest.raises(ValueError, match="captured for"):
        fwd(torch.zeros(m + 1, 512, device="cuda", dtype=torch.bfloat16))


def test_backward_grad_ready_hook_order_and_bits():
    """mlp_backward(grad_ready=...) reports dWdown first (it needs only G and dY), then dWgate
    and dWup, and the gradients are bitwise those of the call without a hook (the hook only
    lets a data-parallel all-reduce overlap the rest of the backward)."""
    import bench
    ws = bench.make_weights(512, 1024, 64, 0.75, 3)
    net = bs.SparseMlp.from_caches(*[bs.from_host(w, torch.bfloat16) for w in ws])
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(384, 512, device="cuda", generator=g).bfloat16()
    dy = torch.randn(384, 512, device="cuda", generator=g).bfloat16()
    _, acts = bs.mlp_forward(x, net)
    ref = bs.mlp_backward(dy, acts, net, grad_mode="active")
    seen = []
    got = bs.mlp_backward(dy, acts, net, grad_mode="active",
                          grad_ready=lambda i, t: seen.append((i, t.data_ptr())))
    torch.cuda.synchronize()
    assert [i for i, _ in seen] == [3, 1, 2]
    assert [p for _, p in seen] == [got[3].data_ptr(), got[1].data_ptr(), got[2].data_ptr()]
    for r, o in zip(ref, got):
        assert torch.equal(r, o)


@pytest.mark.parametrize("which", [0, 1, 2])
def test_stored_block_wgrad_item_layouts(which):
    """Stored-block weight gradients at the cfg3 mask structures (csrc/wgrad.cu): 4-block items
    per column, the up mask's 446 items (3 waves of 148 + 2, the last two split along the
    tokens into fp32 partials) and the down mask's long columns; every stored block against
    x^T d in fp32 (mlp.py:137-141) and bitwise reproducible."""
    import bench
    from paper_2507_03117_b200 import mlp as M
    rows, cols = (4096, 14336) if which < 2 else (14336, 4096)
    w = bs.from_host(bench.make_weights(4096, 14336, 64, 0.9, 0)[which], torch.bfloat16)
    g = torch.Generator(device="cuda").manual_seed(7 + which)
    m = 256
    a = torch.randn(m, rows, device="cuda", generator=g).bfloat16()
    d = torch.randn(m, cols, device="cuda", generator=g).bfloat16()
    got = M._wgrad(a, d, rows, cols, w, False)
    assert torch.equal(got, M._wgrad(a, d, rows, cols, w, False))
    full = a.float().t() @ d.float()
    cp = w.col_ptr.cpu().numpy()
    ri = w.block_row_idx.cpu().numpy()
    ref = torch.empty_like(got)
    for c in range(len(cp) - 1):
        for s in range(cp[c], cp[c + 1]):
            r = int(ri[s])
            ref[s] = full[r * 64:(r + 1) * 64, c * 64:(c + 1) * 64]
    err = ((got - ref).abs().max() / ref.abs().max()).item()
    assert err <= 1e-5, err
