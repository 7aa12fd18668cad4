"""cfg0 (fp32, d=2048 h=8192 b=64 s=0.9, 2048 tokens) forward, repeated, for ncu launch lists."""
import sys
sys.path.insert(0, ".")
import torch, bench
import paper_2507_03117_b200 as bs
ws = bench.make_weights(2048, 8192, 64, 0.9, 0)
net = bs.SparseMlp.from_caches(*[bs.from_host(w, torch.float32) for w in ws])
x = torch.randn(2048, 2048, device="cuda")
for _ in range(4):
    bs.mlp_forward(x, net, save_activations=False)
torch.cuda.synchronize()
