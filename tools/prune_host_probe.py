"""Host overhead of generate_masks: API time vs the bare C call (CUDA events, L2 warm)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2507_03117_b200 as bs
from paper_2507_03117_b200 import _lib as L
rows, cols, b, s = 4096, 14336, 64, 0.9
g0 = torch.Generator(device="cuda").manual_seed(3)
w = torch.randn(rows, cols, device="cuda", generator=g0)
g = torch.randn(rows, cols, device="cuda", generator=g0)
def ev(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    e.record(); torch.cuda.synchronize()
    return a.elapsed_time(e) / n * 1e3
gr, gc = rows // b, cols // b
k = gr * gc - int(round(0.9 * gr * gc))
nw = torch.empty(gr, gc, dtype=torch.float64, device="cuda"); ng = torch.empty_like(nw)
kept = torch.empty(gr, gc, dtype=torch.uint8, device="cuda"); reg = torch.empty_like(kept)
cnt = torch.empty(2, dtype=torch.int64, device="cuda"); cnth = torch.zeros(2, dtype=torch.int64).pin_memory()
def bare():
    L.check(L.load().blast_generate_masks(w.data_ptr(), L.F32, g.data_ptr(), L.F32, rows, cols, b, k,
            nw.data_ptr(), ng.data_ptr(), kept.data_ptr(), reg.data_ptr(), cnt.data_ptr(),
            cnth.data_ptr(), L.stream()), "gm")
print(f"generate_masks API {ev(lambda: bs.generate_masks(w, g, b, s)):.1f} us, bare C call {ev(bare):.1f} us")
