"""Dispatcher-visible operators (paper_2507_03117_b200/ops.py): torch.ops.blast.* give the same
bits as the package functions, pass torch.library.opcheck (schema, fake tensors, dispatch), and
trace into a single torch.compile graph without breaks."""
import pytest
import torch

pytestmark = pytest.mark.gpu
bs = pytest.importorskip("paper_2507_03117_b200")


def _net(dtype=torch.bfloat16):
    import bench
    ws = bench.make_weights(512, 1024, 64, 0.75, 11)
    return bs.SparseMlp.from_caches(*[bs.from_host(w, dtype) for w in ws]), ws


def test_ops_match_package_functions_bitwise():
    net, ws = _net()
    h = bs.ops.register(net)
    g = torch.Generator(device="cuda").manual_seed(2)
    x = torch.randn(300, 512, device="cuda", generator=g).bfloat16()
    dy = torch.randn(300, 512, device="cuda", generator=g).bfloat16()
    y_ref, acts = bs.mlp_forward(x, net)
    assert torch.equal(torch.ops.blast.mlp_forward(x, h), y_ref)
    y, a, b, gg = torch.ops.blast.mlp_forward_train(x, h)
    assert torch.equal(y, y_ref) and torch.equal(gg, acts.gated)
    ref = bs.mlp_backward(dy, acts, net, grad_mode="active")
    for r, o in zip(ref, torch.ops.blast.mlp_backward(dy, x, a, b, gg, h)):
        assert torch.equal(r, o)
    w = net.gate.cache
    hw = bs.ops.register(w)
    assert torch.equal(torch.ops.blast.bspmm(x, hw, 2), bs.bspmm_fused(x, w, "silu"))


def test_opcheck():
    net, _ = _net()
    h = bs.ops.register(net)
    x = torch.randn(256, 512, device="cuda").bfloat16()
    torch.library.opcheck(torch.ops.blast.mlp_forward.default, (x, h))
    torch.library.opcheck(torch.ops.blast.mlp_forward_train.default, (x, h))
    torch.library.opcheck(torch.ops.blast.bspmm.default, (x, bs.ops.register(net.gate.cache), 0))


def test_compile_fullgraph():
    net, _ = _net()
    h = bs.ops.register(net)
    x = torch.randn(256, 512, device="cuda").bfloat16()

    def f(t):
        return torch.ops.blast.mlp_forward(t * 2, h) + 1

    got = torch.compile(f, backend="eager", fullgraph=True)(x)
    assert torch.equal(got, f(x))


def test_dead_handle_raises():
    net, _ = _net()
    h = bs.ops.register(net)
    del net
    import gc
    gc.collect()
    with pytest.raises(ValueError, match="handle"):
        torch.ops.blast.mlp_forward(torch.zeros(128, 512, device="cuda").bfloat16(), h)
