"""One GPT-2-small MLP-stack training step (fwd + bwd) on the sparse path, after warm-up,
for launch-list captures: ncu --metrics gpu__time_duration.sum ... python tools/cfg2_once.py"""
import sys
sys.path.insert(0, ".")
import torch
from transformers import GPT2Config
from transformers.models.gpt2.modeling_gpt2 import GPT2MLP
from paper_2507_03117_b200 import integration

d, h, layers, m = 768, 3072, 12, 8192
cfg = GPT2Config(n_embd=d, n_inner=h, resid_pdrop=0.0)
torch.manual_seed(0)
dense = [GPT2MLP(h, cfg).cuda() for _ in range(layers)]
sparse = [integration.SparseGeluMLP.from_gpt2(mlp, 64, 0.9) for mlp in dense]
x = torch.randn(m, d, device="cuda", dtype=torch.bfloat16, requires_grad=True)


def run():
    h_ = x
    for mlp in sparse:
        h_ = mlp(h_)
    h_.float().sum().backward()


for _ in range(3):
    run()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("step")
run()
torch.cuda.synchronize()
