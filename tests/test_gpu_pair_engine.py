"""The CTA-pair engine (cta_group::2, resident weights) against the single-CTA
engine (bitwise: same per-output accumulation order) and the oracle (bf16 bar),
over every product of the MLP, including lines with more stored blocks than the
resident region holds (streamed overflow) and token counts that are not a
multiple of 256."""
import ctypes

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu
bs = pytest.importorskip("paper_2507_03117_b200")
from paper_2507_03117_b200 import _lib  # noqa: E402


class engine:
    def __init__(self, pair: bool):
        self.pair = pair

    def __enter__(self):
        self.prev = _lib.load().blast_set_pair_engine(1 if self.pair else 0)

    def __exit__(self, *a):
        _lib.load().blast_set_pair_engine(self.prev)


def rand_w(rows, cols, b, s, seed):
    rng = np.random.default_rng(seed)
    w = oracle.random_bcsc(rows, cols, b, s, rng)
    w = w._replace(values=(w.values / np.sqrt(rows)).astype(np.float32))
    wb = w._replace(values=torch.from_numpy(w.values).bfloat16().float().numpy())
    return wb, bs.from_host(wb, torch.bfloat16)


def run_both(fn):
    with engine(False):
        ref = fn()
    with engine(True):
        got = fn()
    torch.cuda.synchronize()
    return got, ref


@pytest.mark.parametrize("b", [32, 64])
@pytest.mark.parametrize("m", [256, 300, 1000, 2048])
@pytest.mark.parametrize("s", [0.0, 0.5, 0.9])
def test_bspmm_and_rt(b, m, s):
    k, n = 8 * b, 6 * b
    w_np, w = rand_w(k, n, b, s, seed=b + m)
    x = torch.randn(m, k, device="cuda").bfloat16()
    xt = torch.randn(m, n, device="cuda").bfloat16()
    got, ref = run_both(lambda: bs.bspmm(x, w))
    assert torch.equal(got, ref)
    assert oracle.max_norm_rel(got.float().cpu().numpy(),
                               oracle.bspmm(x.float().cpu().numpy(), w_np)) <= 2e-2
    got, ref = run_both(lambda: bs.bspmm_rt(xt, w))
    assert torch.equal(got, ref)
    assert oracle.max_norm_rel(got.float().cpu().numpy(),
                               oracle.bspmm_rt(xt.float().cpu().numpy(), w_np)) <= 2e-2


@pytest.mark.parametrize("rows", [64 * 40, 64 * 80])
def test_long_lines_stream_overflow(rows):
    # 0% sparsity, 40 / 80 blocks per column: more than the resident capacity
    b = 64
    w_np, w = rand_w(rows, 4 * b, b, 0.0, seed=rows)
    x = torch.randn(512, rows, device="cuda").bfloat16()
    got, ref = run_both(lambda: bs.bspmm(x, w))
    assert torch.equal(got, ref)
    assert oracle.max_norm_rel(got.float().cpu().numpy(),
                               oracle.bspmm(x.float().cpu().numpy(), w_np)) <= 2e-2


@pytest.mark.parametrize("b,s,m", [(64, 0.9, 2048), (64, 0.5, 512), (32, 0.75, 700)])
def test_mlp_forward_backward(b, s, m):
    e, h = 8 * b, 24 * b
    rng = np.random.default_rng(b)
    net = bs.SparseMlp.create(e, h, b, rng, torch.bfloat16)
    for mat in net.matrices():
        g = torch.randn(*mat.dense.shape, device="cuda")
        mask, _ = bs.generate_masks(mat.dense, g, b, s)
        mat.mask = mask
        mat.dense, mat.cache = bs.apply_mask(mat.dense, mask, b, dtype=torch.bfloat16)
    x = torch.randn(m, e, device="cuda").bfloat16()
    dy = torch.randn(m, e, device="cuda").bfloat16()

    def fwd_bwd():
        y, acts = bs.mlp_forward(x, net)
        return (y,) + tuple(bs.mlp_backward(dy, acts, net, grad_mode="active"))

    got, ref = run_both(fwd_bwd)
    for a, r in zip(got, ref):
        assert torch.equal(a, r)
