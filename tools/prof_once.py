"""One cfg3 MLP forward (after warm-up) for ncu captures:
ncu --set full --import-source on -k regex:spmm_tc -s 2 -c 2 python tools/prof_once.py"""
import sys
sys.path.insert(0, ".")
import bench, torch
import paper_2507_03117_b200 as bs
ws = bench.make_weights(4096, 14336, 64, 0.9, 0)
net = bs.SparseMlp.from_caches(*[bs.from_host(w, torch.bfloat16) for w in ws])
x = torch.randn(8192, 4096, device="cuda").bfloat16()
for _ in range(2):
    bs.mlp_forward(x, net, save_activations=False)
torch.cuda.synchronize()
