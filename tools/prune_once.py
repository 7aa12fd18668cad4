"""cfg3-gate prune-and-grow refresh (generate_masks + apply_mask), repeated, for ncu launch lists."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2507_03117_b200 as bs
rows, cols, b, s = 4096, 14336, 64, 0.9
gen = torch.Generator(device="cuda").manual_seed(3)
w = torch.randn(rows, cols, device="cuda", generator=gen) * rows ** -0.5
g = torch.randn(rows, cols, device="cuda", generator=gen)
for _ in range(3):
    mask, rep = bs.generate_masks(w, g, b, s)
    bs.apply_mask(w, mask, b, dtype=torch.bfloat16)
torch.cuda.synchronize()
