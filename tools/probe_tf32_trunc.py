"""Does kind::tf32 truncate fp32 operands? One fp32 product and forward saved for a bitwise
comparison between builds (tools: BLAST_LIB=... python tools/probe_tf32_trunc.py out.npy)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch, bench
import paper_2507_03117_b200 as bs
ws = bench.make_weights(1024, 2048, 64, 0.8, 0)
mt = bs.from_host(ws[0], torch.float32)
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.randn(512, 1024, device="cuda", generator=g)
y = bs.bspmm(x, mt)
net = bs.SparseMlp.from_caches(*[bs.from_host(w, torch.float32) for w in ws])
y2, _ = bs.mlp_forward(x, net, save_activations=False)
ref = x.double() @ torch.as_tensor(bs.to_dense(mt)).cuda().double()
print("max rel err vs fp64:", ((y.double() - ref).abs().max() / ref.abs().max()).item())
np.save(sys.argv[1], np.concatenate([y.cpu().numpy().ravel(), y2.cpu().numpy().ravel()]))
