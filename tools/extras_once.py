"""One call of each bench extra after warm-up, for ncu launch lists:
ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/extras_once.py"""
import sys
sys.path.insert(0, ".")
import torch
import bench
import paper_2507_03117_b200 as bs

what = sys.argv[1] if len(sys.argv) > 1 else "train"
if what == "train":
    ws = bench.make_weights(4096, 14336, 64, 0.9, 0)
    net = bs.SparseMlp.from_caches(*[bs.from_host(w, torch.bfloat16) for w in ws])
    x = torch.randn(8192, 4096, device="cuda").bfloat16()
    dy = (torch.randn(8192, 4096, device="cuda") * 0.1).bfloat16()
    for _ in range(3):
        _, acts = bs.mlp_forward(x, net)
        bs.mlp_backward(dy, acts, net, grad_mode="active")
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("timed")
    _, acts = bs.mlp_forward(x, net)
    bs.mlp_backward(dy, acts, net, grad_mode="active")
elif what == "cfg0":
    ws = bench.make_weights(2048, 8192, 64, 0.9, 0)
    net = bs.SparseMlp.from_caches(*[bs.from_host(w, torch.float32) for w in ws])
    x = torch.randn(2048, 2048, device="cuda")
    for _ in range(4):
        bs.mlp_forward(x, net, save_activations=False)
elif what == "decode":
    ws = bench.make_weights(4096, 14336, 64, 0.95, 0)
    net = bs.SparseMlp.from_caches(*[bs.from_host(w, torch.bfloat16) for w in ws])
    x = torch.randn(128, 4096, device="cuda").bfloat16()
    for _ in range(4):
        bs.mlp_forward(x, net, save_activations=False)
torch.cuda.synchronize()
