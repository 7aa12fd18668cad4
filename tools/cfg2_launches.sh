#!/bin/bash
# launch list of the cfg2 GPT-2 MLP fwd+bwd (sparse only)
python - <<'PY'
import sys; sys.path.insert(0,'.')
import torch
import tools.config_sweep as cs
from transformers import GPT2Config
from transformers.models.gpt2.modeling_gpt2 import GPT2MLP
from paper_2507_03117_b200 import integration
d,h,m=768,3072,8192
cfg=GPT2Config(n_embd=d,n_inner=h,resid_pdrop=0.0)
mlps=[integration.SparseGeluMLP.from_gpt2(GPT2MLP(h,cfg).cuda().float(),64,0.9) for _ in range(2)]
x=torch.randn(m,d,device='cuda',dtype=torch.bfloat16,requires_grad=True)
for it in range(3):
    y=x
    for mlp in mlps: y=mlp(y)
    y.float().sum().backward()
torch.cuda.synchronize()
PY
