"""cfg2 (GPT-2 small MLP stack, 12 layers, 90 %, 8192 tokens) fwd+bwd: eager vs one CUDA graph
replay of the whole step (gradients accumulate into .grad buffers captured once)."""
import sys, time
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
params = [p for mlp in sparse for p in mlp.parameters()]
x = torch.randn(m, d, device="cuda", dtype=torch.bfloat16, requires_grad=True)

def step():
    h_ = x
    for mlp in sparse:
        h_ = mlp(h_)
    h_.float().sum().backward()

def timed(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n

eager = timed(step)
# capture: warm up on a side stream, then one graph of forward + backward
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(3):
        for p in params + [x]:
            p.grad = None
        step()
torch.cuda.current_stream().wait_stream(s)
for p in params + [x]:
    p.grad = None
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
ref = [p.grad.clone() for p in params]
g.replay()
torch.cuda.synchronize()
same = all(torch.equal(r, p.grad) for r, p in zip(ref, params))
graphed = timed(g.replay)
print(f"cfg2 fwd+bwd eager {eager:.3f} ms, CUDA graph replay {graphed:.3f} ms, grads equal {same}")
