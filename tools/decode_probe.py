"""One decode-sized (m tokens) MLP forward repeated, for ncu launch lists."""
import sys
sys.path.insert(0, ".")
import torch, bench
import paper_2507_03117_b200 as bs
m = int(sys.argv[1]) if len(sys.argv) > 1 else 128
sp = float(sys.argv[2]) if len(sys.argv) > 2 else 0.95
ws = bench.make_weights(4096, 14336, 64, sp, 0)
net = bs.SparseMlp.from_caches(*[bs.from_host(w, torch.bfloat16) for w in ws])
x = torch.randn(m, 4096, device="cuda").bfloat16()
for _ in range(5):
    bs.mlp_forward(x, net, save_activations=False)
torch.cuda.synchronize()
