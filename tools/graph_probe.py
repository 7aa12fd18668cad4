import sys, time
sys.path.insert(0, ".")
import torch, bench
import paper_2507_03117_b200 as bs
ws = bench.make_weights(4096, 14336, 64, 0.95, 0)
net = bs.SparseMlp.from_caches(*[bs.from_host(w, torch.bfloat16) for w in ws])
for m in (128, 1024, 8192):
    x = torch.randn(m, 4096, device="cuda").bfloat16()
    for _ in range(3):
        y, _ = bs.mlp_forward(x, net, save_activations=False)
    torch.cuda.synchronize()
    def timed(fn, n=50):
        fn(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n): fn()
        b.record(); torch.cuda.synchronize()
        return a.elapsed_time(b) / n * 1e3
    eager = timed(lambda: bs.mlp_forward(x, net, save_activations=False))
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):
            bs.mlp_forward(x, net, save_activations=False)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        yg, _ = bs.mlp_forward(x, net, save_activations=False)
    graph = timed(lambda: g.replay())
    yref, _ = bs.mlp_forward(x, net, save_activations=False)
    g.replay(); torch.cuda.synchronize()
    print(f"m={m} eager {eager:.1f} us  graph {graph:.1f} us  equal={torch.equal(yg, yref)}")
