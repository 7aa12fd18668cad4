"""The fused gate+up -> down forward (one persistent kernel, G in an L2 ring; csrc/mlp_fused.cuh)
against the two-launch path (bitwise: same per-output accumulation order and epilogue math)
and against the oracle (bf16 bar), including token counts that are not a multiple of 256,
more tiles than ring slots (ring reuse), empty lines and dense matrices."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu
bs = pytest.importorskip("paper_2507_03117_b200")
from paper_2507_03117_b200 import _lib as L  # noqa: E402


def make_net(e, h, s, seed):
    rng = np.random.default_rng(seed)
    mats, ref = [], []
    for rows, cols in ((e, h), (e, h), (h, e)):
        w = oracle.random_bcsc(rows, cols, 64, s, rng)
        w = w._replace(values=(w.values / np.sqrt(rows)).astype(np.float32))
        wb = w._replace(values=torch.from_numpy(w.values).bfloat16().float().numpy())
        ref.append(wb)
        mats.append(bs.from_host(wb, torch.bfloat16))
    return bs.SparseMlp.from_caches(*mats), ref


def two_launch(x, net, m):
    lib = L.load()
    g = torch.empty(m, net.hidden_dim, dtype=torch.bfloat16, device="cuda")
    y = torch.empty(m, net.embed_dim, dtype=torch.bfloat16, device="cuda")
    dg, du, dd = (mat.cache.desc() for mat in net.matrices())
    plan = net.plan()
    L.check(lib.blast_mlp_gate_up(x.data_ptr(), m, C.byref(dg), C.byref(du), C.byref(plan),
                                  g.data_ptr(), None, None, L.stream()))
    L.check(lib.blast_bspmm(g.data_ptr(), m, C.byref(dd), 0, y.data_ptr(), L.stream()))
    return y


def fused(x, net, m):
    lib = L.load()
    y = torch.empty(m, net.embed_dim, dtype=torch.bfloat16, device="cuda")
    dg, du, dd = (mat.cache.desc() for mat in net.matrices())
    plan = net.plan()
    rc = lib.blast_mlp_forward_fused(x.data_ptr(), m, C.byref(dg), C.byref(du), C.byref(dd),
                                     C.byref(plan), y.data_ptr(), L.stream())
    L.check(rc)
    return y


@pytest.mark.parametrize("e,h", [(256, 512), (512, 1536), (1024, 4096)])
@pytest.mark.parametrize("m", [256, 300, 1000, 2048, 4096])
@pytest.mark.parametrize("s", [0.0, 0.5, 0.9, 0.97])
def test_fused_equals_two_launch(e, h, m, s):
    net, _ = make_net(e, h, s, seed=e + h + m)
    torch.manual_seed(m)
    x = torch.randn(m, e, device="cuda").bfloat16()
    y2 = two_launch(x, net, m)
    yf = fused(x, net, m)
    torch.cuda.synchronize()
    assert torch.equal(yf, y2)


@pytest.mark.parametrize("m", [512, 2304])
def test_fused_vs_oracle_and_public_api(m):
    e, h = 512, 2048
    net, ref = make_net(e, h, 0.9, seed=7)
    rng = np.random.default_rng(3)
    x = torch.from_numpy(rng.standard_normal((m, e)).astype(np.float32)).cuda().bfloat16()
    y_api, _ = bs.mlp_forward(x, net, save_activations=False)  # two-launch path (default)
    yf = fused(x, net, m)
    torch.cuda.synchronize()
    assert torch.equal(y_api, yf)
    y_ref, _ = oracle.mlp_forward(x.float().cpu().numpy(), *ref)
    assert oracle.max_norm_rel(yf.float().cpu().numpy(), y_ref) <= 2e-2


def test_fused_is_deterministic():
    net, _ = make_net(1024, 4096, 0.9, seed=11)
    x = torch.randn(8192, 1024, device="cuda").bfloat16()
    a = fused(x, net, 8192)
    b = fused(x, net, 8192)
    torch.cuda.synchronize()
    assert torch.equal(a, b)


def test_fused_unsupported_shapes_launch_nothing():
    lib = L.load()
    net, _ = make_net(256, 512, 0.9, seed=1)
    x = torch.randn(128, 256, device="cuda").bfloat16()  # m < 256: two-launch path only
    y = torch.empty(128, 256, dtype=torch.bfloat16, device="cuda")
    dg, du, dd = (mat.cache.desc() for mat in net.matrices())
    plan = net.plan()
    rc = lib.blast_mlp_forward_fused(x.data_ptr(), 128, C.byref(dg), C.byref(du), C.byref(dd),
                                     C.byref(plan), y.data_ptr(), L.stream())
    assert rc == 6  # BLAST_EUNSUPPORTED
