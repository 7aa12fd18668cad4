"""Oracle parity at the BASELINE.json configuration shapes.

* cfg3 (Llama-3-8B MLP, d=4096 h=14336, b=64, 90 %, bf16): the full 8192-token inference
  forward (the benchmarked call, mlp_forward(save_activations=False)) with a stride-8 row
  sample checked against the oracle; the training forward + backward at 1024 tokens checked
  in full (dX, and the dense weight gradients of mlp.py:133-142).
* cfg0 (d=2048 h=8192, b=64, 90 %, 2048 tokens, fp32 — the reference's own precision):
  forward and backward at 1e-4 under both the reference rel_err and max-norm-relative error.
* cfg2 (GPT-2 small MLP shape d=768 h=3072, b=64, 90 %): bf16 forward + backward.
* cfg1 (Llama-3.2-1B MLP d=2048 h=8192, b=64, 95 %, bf16): forward, row sample of 16384 tokens.

Weights follow SparseMlp.create (mlp.py:61-68: N(0,1/e) gate/up, N(0,0.25/h) down) on exact-k
uniform block placement (bench.py:50-72). bf16 comparisons feed the oracle the same
bf16-rounded inputs and weights (the 2e-2 max-norm-relative bar of the north star).
"""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu
bs = pytest.importorskip("paper_2507_03117_b200")


def make_mats(e, h, b, s, seed, bf16):
    rng = np.random.default_rng(seed)
    mats = []
    for rows, cols, gain in ((e, h, 1.0), (e, h, 1.0), (h, e, 0.5)):
        w = oracle.random_bcsc(rows, cols, b, s, rng)
        vals = (w.values * np.float32(gain / np.sqrt(rows))).astype(np.float32)
        if bf16:
            vals = torch.from_numpy(vals).bfloat16().float().numpy()
        mats.append(w._replace(values=vals))
    dt = torch.bfloat16 if bf16 else torch.float32
    net = bs.SparseMlp.from_caches(*(bs.from_host(w, dt) for w in mats))
    return net, mats


def tokens(m, e, seed, bf16):
    x = np.random.default_rng(seed).standard_normal((m, e)).astype(np.float32)
    if bf16:
        x = torch.from_numpy(x).bfloat16().float().numpy()
    return x


def to_dev(a, bf16):
    t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    return t.bfloat16() if bf16 else t


def host(t):
    return t.float().cpu().numpy()


def check(got, ref, tol, name, fp32):
    mnr = oracle.max_norm_rel(got, ref)
    assert mnr <= tol, f"{name}: max-norm-relative {mnr:.3e} > {tol}"
    if fp32:
        re = oracle.rel_err(got, ref)
        assert re <= tol, f"{name}: rel_err {re:.3e} > {tol}"


def test_cfg3_inference_forward_8192_tokens_row_sample():
    e, h, b, s, m = 4096, 14336, 64, 0.9, 8192
    net, mats = make_mats(e, h, b, s, seed=0, bf16=True)
    assert [w.nnzb for w in mats] == [1434, 1434, 1434]
    x = tokens(m, e, 1, True)
    y, none = bs.mlp_forward(to_dev(x, True), net, save_activations=False)
    assert none is None
    rows = np.arange(3, m, 8)  # every 8th token: covers all 64 token tiles and both halves
    y_ref, _ = oracle.mlp_forward(x[rows], *mats)
    check(host(y)[rows], y_ref, 2e-2, "y", fp32=False)
    # the training-mode forward computes the same y bitwise
    y2, _ = bs.mlp_forward(to_dev(x, True), net)
    assert torch.equal(y, y2)


def test_cfg3_training_forward_backward_1024_tokens():
    e, h, b, s, m = 4096, 14336, 64, 0.9, 1024
    net, mats = make_mats(e, h, b, s, seed=1, bf16=True)
    x, dy = tokens(m, e, 2, True), tokens(m, e, 3, True)
    y, acts = bs.mlp_forward(to_dev(x, True), net)
    y_ref, acts_ref = oracle.mlp_forward(x, *mats)
    check(host(y), y_ref, 2e-2, "y", fp32=False)
    for got, ref, name in zip((acts.gate_pre, acts.up_out, acts.gated), acts_ref[1:],
                              ("a", "b", "g")):
        check(host(got), ref, 2e-2, name, fp32=False)
    grads = bs.mlp_backward(to_dev(dy, True), acts, net)
    grads_ref = oracle.mlp_backward(dy, acts_ref, *mats)
    for got, ref, name in zip(grads, grads_ref, ("dx", "dWg", "dWu", "dWd")):
        check(host(got), ref, 2e-2, name, fp32=False)


def test_cfg0_fp32_forward_backward():
    e, h, b, s, m = 2048, 8192, 64, 0.9, 2048
    net, mats = make_mats(e, h, b, s, seed=2, bf16=False)
    assert [w.nnzb for w in mats] == [410, 410, 410]
    x, dy = tokens(m, e, 4, False), tokens(m, e, 5, False)
    y, acts = bs.mlp_forward(to_dev(x, False), net)
    y_ref, acts_ref = oracle.mlp_forward(x, *mats)
    check(host(y), y_ref, 1e-4, "y", fp32=True)
    for got, ref, name in zip((acts.gate_pre, acts.up_out, acts.gated), acts_ref[1:],
                              ("a", "b", "g")):
        check(host(got), ref, 1e-4, name, fp32=True)
    y_inf, _ = bs.mlp_forward(to_dev(x, False), net, save_activations=False)
    check(host(y_inf), y_ref, 1e-4, "y (inference)", fp32=True)
    grads = bs.mlp_backward(to_dev(dy, False), acts, net)
    grads_ref = oracle.mlp_backward(dy, acts_ref, *mats)
    for got, ref, name in zip(grads, grads_ref, ("dx", "dWg", "dWu", "dWd")):
        # dW entries of inactive blocks are O(1e-3) sums of cancelling terms: the reference's
        # rel_err (denominator 1 + |ref|) and max-norm-relative both bound them at 1e-4
        check(host(got), ref, 1e-4, name, fp32=True)


def test_cfg2_gpt2_shape_bf16_forward_backward():
    e, h, b, s, m = 768, 3072, 64, 0.9, 2048
    net, mats = make_mats(e, h, b, s, seed=3, bf16=True)
    assert [w.nnzb for w in mats] == [58, 58, 58]
    x, dy = tokens(m, e, 6, True), tokens(m, e, 7, True)
    y, acts = bs.mlp_forward(to_dev(x, True), net)
    y_ref, acts_ref = oracle.mlp_forward(x, *mats)
    check(host(y), y_ref, 2e-2, "y", fp32=False)
    for mode in ("full", "active"):
        grads = bs.mlp_backward(to_dev(dy, True), acts, net, grad_mode=mode)
        grads_ref = oracle.mlp_backward(dy, acts_ref, *mats)
        check(host(grads[0]), grads_ref[0], 2e-2, "dx", fp32=False)
        for got, ref, w, name in zip(grads[1:], grads_ref[1:], mats, ("dWg", "dWu", "dWd")):
            if mode == "active":  # stored-block gradients = the dense gradient's blocks
                grid = _stored_grid(w)
                ref = oracle.from_dense(ref, b, oracle.Mask(grid, np.zeros_like(grid))).values
            check(host(got), ref, 2e-2, f"{name} ({mode})", fp32=False)


def _stored_grid(w):
    g = np.zeros((oracle.grid_dim(w.rows, w.block), oracle.grid_dim(w.cols, w.block)), bool)
    for c in range(g.shape[1]):
        g[w.block_row_idx[w.col_ptr[c]:w.col_ptr[c + 1]], c] = True
    return g


def test_cfg1_llama32_1b_shape_forward_row_sample():
    e, h, b, s, m = 2048, 8192, 64, 0.95, 16384
    net, mats = make_mats(e, h, b, s, seed=4, bf16=True)
    assert [w.nnzb for w in mats] == [205, 205, 205]
    x = tokens(m, e, 8, True)
    y, _ = bs.mlp_forward(to_dev(x, True), net, save_activations=False)
    rows = np.arange(5, m, 16)
    y_ref, _ = oracle.mlp_forward(x[rows], *mats)
    check(host(y)[rows], y_ref, 2e-2, "y", fp32=False)
