"""One cfg3 MLP forward per engine with per-role wait counters (BLAST_DEBUG_COUNTERS=1)."""
import sys
sys.path.insert(0, ".")
import bench, torch
import paper_2507_03117_b200 as bs
from paper_2507_03117_b200 import _lib
ws = bench.make_weights(4096, 14336, 64, 0.9, 0)
net = bs.SparseMlp.from_caches(*[bs.from_host(w, torch.bfloat16) for w in ws])
x = torch.randn(8192, 4096, device="cuda").bfloat16()
for pair in (0, 1):
    _lib.load().blast_set_pair_engine(pair)
    for _ in range(2):
        bs.mlp_forward(x, net, save_activations=False)
    torch.cuda.synchronize()
    print("---- pair", pair, file=sys.stderr, flush=True)
    bs.mlp_forward(x, net, save_activations=False)
    torch.cuda.synchronize()
