"""Per-matrix stored-block weight-gradient timing (cfg3 shapes): each mask with its own
gradient and with the other matrix's gradient, to separate mask effects from data effects."""
import sys
sys.path.insert(0, ".")
import torch, bench
import paper_2507_03117_b200 as bs
from paper_2507_03117_b200 import mlp as M
ws = bench.make_weights(4096, 14336, 64, 0.9, 0)
net = bs.SparseMlp.from_caches(*[bs.from_host(w, torch.bfloat16) for w in ws])
x = torch.randn(8192, 4096, device="cuda").bfloat16()
da = (torch.randn(8192, 14336, device="cuda") * 0.1).bfloat16()
db = (torch.randn(8192, 14336, device="cuda") * 0.1).bfloat16()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
def t(fn, n=10):
    fn(); torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for a, b in ev:
        flush.zero_(); a.record(); fn(); b.record()
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in ev)[n // 2] * 1e3
g, u = net.gate.cache, net.up.cache
for name, w, d in (("gate mask, dA", g, da), ("up mask, dB", u, db), ("gate mask, dB", g, db), ("up mask, dA", u, da)):
    print(f"{name}: {t(lambda: M._wgrad(x, d, 4096, 14336, w, False)):.1f} us  nnzb={w.nnzb}", flush=True)
