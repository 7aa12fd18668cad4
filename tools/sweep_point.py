"""One cfg3-shape forward (bf16, 8192 tokens) at block b / sparsity s, repeated (ncu / counters)."""
import sys
sys.path.insert(0, ".")
import torch, bench
import paper_2507_03117_b200 as bs
b = int(sys.argv[1]) if len(sys.argv) > 1 else 32
s = float(sys.argv[2]) if len(sys.argv) > 2 else 0.9
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
ws = bench.make_weights(4096, 14336, b, s, 0)
net = bs.SparseMlp.from_caches(*[bs.from_host(w, torch.bfloat16) for w in ws])
x = torch.randn(8192, 4096, device="cuda").bfloat16()
for _ in range(reps):
    bs.mlp_forward(x, net, save_activations=False)
torch.cuda.synchronize()
