"""Time the LPT item schedule (blast_balanced_schedule) at the cfg0 / cfg3 plan shapes."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2507_03117_b200 import _lib as L, bcsc

for name, gr, gc, n_tiles, seq in (("cfg0 gate+up", 32, 128, 16, 1), ("cfg0 down", 128, 32, 16, 0),
                                   ("cfg3 gate+up", 64, 224, 32, 1), ("cfg3 down", 224, 64, 32, 0),
                                   ("decode gate+up", 64, 224, 1, 1)):
    rng = np.random.default_rng(0)
    def km():
        k = -np.ones((gr, gc), np.int32)
        sel = rng.random((gr, gc)) < 0.1
        k[sel] = np.arange(sel.sum())
        return torch.from_numpy(k).cuda()
    sp, st, fl = bcsc.build_plan(km(), km() if seq else None, gr, gc, 0)
    grid = 148
    rows = -(-n_tiles * gc // grid)
    out = torch.empty(rows * grid, dtype=torch.int32, device="cuda")
    run = lambda: L.check(L.load().blast_balanced_schedule(sp.data_ptr(), fl.data_ptr(), gc, n_tiles, grid,
                                                           seq, out.data_ptr(), L.stream()), "schedule")
    run(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        run()
    b.record(); torch.cuda.synchronize()
    print(f"{name:16s} items {n_tiles * gc:6d} rows {rows:4d}  {a.elapsed_time(b) / 10 * 1e3:8.1f} us")
