"""Forward timing for A/B builds of the interleaved gate+up (decode graph replay at 95 %, and
8192-token forwards at 50 % / 70 % where the interleaved layout is used): python tools/gu_variant_time.py"""
import sys
sys.path.insert(0, ".")
import torch, bench
import paper_2507_03117_b200 as bs


def timed(fn, n=50):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


out = []
for s, m in ((0.95, 128), (0.5, 8192), (0.7, 8192)):
    ws = bench.make_weights(4096, 14336, 64, s, 0)
    net = bs.SparseMlp.from_caches(*[bs.from_host(w, torch.bfloat16) for w in ws])
    x = torch.randn(m, 4096, device="cuda").bfloat16()
    for _ in range(3):
        bs.mlp_forward(x, net, save_activations=False)
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        for _ in range(2):
            bs.mlp_forward(x, net, save_activations=False)
    torch.cuda.current_stream().wait_stream(st)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        bs.mlp_forward(x, net, save_activations=False)
    out.append(f"s={s} m={m}: {timed(lambda: g.replay()):.1f} us")
print("  ".join(out))
