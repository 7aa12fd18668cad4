"""Block-sparse MLPs inside transformers models (LlamaMLP / GPT2MLP swaps):
forward and autograd backward against torch on the same masked dense weights."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
bs = pytest.importorskip("paper_2507_03117_b200")
transformers = pytest.importorskip("transformers")
from paper_2507_03117_b200 import integration  # noqa: E402


def masked_dense(w: bs.BlockSparseMatrix) -> torch.Tensor:
    return bs.to_dense(w).float()


def mnr(got, ref):
    return float((got.float() - ref.float()).abs().max() / ref.float().abs().max().clamp_min(1e-30))


def llama_cfg(**kw):
    from transformers import LlamaConfig
    base = dict(hidden_size=256, intermediate_size=1024, num_hidden_layers=2,
                num_attention_heads=4, num_key_value_heads=4, vocab_size=512,
                max_position_embeddings=512)
    base.update(kw)
    return LlamaConfig(**base)


def test_llama_mlp_forward_backward():
    from transformers.models.llama.modeling_llama import LlamaMLP
    torch.manual_seed(0)
    mlp = LlamaMLP(llama_cfg()).cuda().float()
    sp = integration.SparseGatedMLP.from_llama(mlp, 64, 0.75)
    wg, wu, wd = (masked_dense(w) for w in (sp.net.gate.cache, sp.net.up.cache, sp.net.down.cache))
    x = torch.randn(3, 100, 256, device="cuda", requires_grad=True)
    y = sp(x)
    xr = x.detach().clone().requires_grad_(True)
    wgr, wur, wdr = (w.clone().requires_grad_(True) for w in (wg, wu, wd))
    xb = xr.bfloat16().float()
    yr = (torch.nn.functional.silu(xb @ wgr) * (xb @ wur)) @ wdr
    assert mnr(y, yr) <= 2e-2
    dy = torch.randn_like(y)
    y.backward(dy)
    yr.backward(dy)
    assert mnr(x.grad, xr.grad) <= 2e-2
    # parameter grads = dense grads gathered at the stored blocks
    for w, ref, par in ((sp.net.gate.cache, wgr.grad, sp.gate_values),
                        (sp.net.down.cache, wdr.grad, sp.down_values)):
        blocks = bs.from_dense(ref, 64, bs.BlockMask(kept=w._kmap() >= 0,
                                                     regrown=torch.zeros_like(w._kmap(),
                                                                              dtype=torch.bool)))
        assert mnr(par.grad.float(), blocks.values.float()) <= 2e-2


def test_gpt2_mlp_forward_backward():
    from transformers import GPT2Config
    from transformers.models.gpt2.modeling_gpt2 import GPT2MLP
    torch.manual_seed(1)
    cfg = GPT2Config(n_embd=256, n_inner=1024, resid_pdrop=0.0)
    mlp = GPT2MLP(1024, cfg).cuda().float()
    with torch.no_grad():
        mlp.c_fc.bias.normal_()
        mlp.c_proj.bias.normal_()
    sp = integration.SparseGeluMLP.from_gpt2(mlp, 64, 0.5)
    w1, w2 = masked_dense(sp.w1), masked_dense(sp.w2)
    x = torch.randn(2, 70, 256, device="cuda", requires_grad=True)
    y = sp(x)
    xr = x.detach().clone().requires_grad_(True)
    b1r = mlp.c_fc.bias.detach().clone().requires_grad_(True)
    yr = integration._gelu_tanh(xr.bfloat16().float() @ w1 + b1r) @ w2 + mlp.c_proj.bias
    assert mnr(y, yr) <= 2e-2
    with torch.no_grad():
        assert mnr(sp(x), yr) <= 2e-2  # inference path (fused bias + gelu epilogue)
    dy = torch.randn_like(y)
    y.backward(dy)
    yr.backward(dy)
    assert mnr(x.grad, xr.grad) <= 3e-2
    assert mnr(sp.b1.grad, b1r.grad) <= 3e-2


def test_sparsify_llama_model_runs_and_matches_masked_dense():
    from transformers import LlamaForCausalLM
    torch.manual_seed(2)
    model = LlamaForCausalLM(llama_cfg()).cuda().to(torch.bfloat16).eval()
    ids = torch.randint(0, 512, (2, 128), device="cuda")
    integration.sparsify_llama(model, 64, 0.9)
    with torch.no_grad():
        logits = model(ids).logits
    assert torch.isfinite(logits).all()
    assert sum(isinstance(l.mlp, integration.SparseGatedMLP) for l in model.model.layers) == 2


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("m,n", [(1, 1), (7, 3), (300, 769), (8192, 3072), (4096, 768)])
def test_column_sums(dtype, m, n):
    """Bias-gradient column sums: fp32 accumulation, deterministic, against an fp64 reference."""
    from paper_2507_03117_b200.kernels import column_sums
    torch.manual_seed(m * 31 + n)
    x = torch.randn(m, n, device="cuda").to(dtype)
    got = column_sums(x)
    ref = x.double().sum(0)
    scale = x.double().abs().sum(0).clamp_min(1e-30)
    assert ((got.double() - ref).abs() / scale).max().item() <= 1e-5
    assert torch.equal(got, column_sums(x))  # run-to-run bitwise


@pytest.mark.parametrize("block", [64, 128])
def test_float32_forward_sees_optimizer_step(block):
    """float32 weights: the 3xTF32 tensor-core images are refreshed after an in-place
    optimizer step / load_state_dict, so the next forward uses the updated values
    (cached hi/lo copies went stale)."""
    from transformers.models.llama.modeling_llama import LlamaMLP
    torch.manual_seed(3)
    mlp = LlamaMLP(llama_cfg()).cuda().float()
    sp = integration.SparseGatedMLP.from_llama(mlp, block, 0.5, dtype=torch.float32)
    x = torch.randn(130, 256, device="cuda")

    def ref_out():
        wg, wu, wd = (masked_dense(w) for w in (sp.net.gate.cache, sp.net.up.cache,
                                                sp.net.down.cache))
        return (torch.nn.functional.silu(x @ wg) * (x @ wu)) @ wd

    with torch.no_grad():
        assert mnr(sp(x), ref_out()) <= 1e-4
    opt = torch.optim.SGD(sp.parameters(), lr=0.5)
    y = sp(x.requires_grad_(True))
    y.square().sum().backward()
    opt.step()
    with torch.no_grad():
        assert mnr(sp(x), ref_out()) <= 1e-4
        state = {k: v.clone() * 0.5 for k, v in sp.state_dict().items()}
        sp.load_state_dict(state)
        assert mnr(sp(x), ref_out()) <= 1e-4
