"""Prune-and-grow kernels at full size: per-kernel time and achieved GB/s.

Shapes: Llama-3-8B gate (4096 x 14336) and Llama-3-70B gate (8192 x 28672), b = 64,
s = 0.9, float32 masters (the trainer's dense masters) and the gradient G.
Algorithmic bytes per kernel (HBM):
  block_norms (W and G, one launch)  : 2 * R * C * 4 read + 2 * grid * 8 write
  top-k (one grid)                   : grid * 8 read (norms) + grid write (mask)
  repack index (count/scan/kmap)     : 2 * grid read (masks) + grid * 4 + (gc+1) * 8 write
  apply_mask gather                  : R * C * 4 read + R * C * 4 (masked) + nnzb*b*b*elt write
Prints one JSON line per shape with microseconds and GB/s per kernel.
"""
import ctypes as C
import json
import math
import sys

import torch

sys.path.insert(0, ".")
import paper_2507_03117_b200 as bs  # noqa: E402
from paper_2507_03117_b200 import _lib as L  # noqa: E402


def ev_time(fn, iters=20, warmup=3):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters * 1e3  # us


def run(rows, cols, b=64, s=0.9, vdt=torch.bfloat16):
    lib = L.load()
    st = L.stream()
    gen = torch.Generator(device="cuda").manual_seed(0)
    w = torch.randn(rows, cols, device="cuda", generator=gen)
    g = torch.randn(rows, cols, device="cuda", generator=gen)
    gr, gc = rows // b, cols // b
    grid = gr * gc
    nw = torch.empty(gr, gc, dtype=torch.float64, device="cuda")
    ng = torch.empty_like(nw)
    k = int(math.floor((1.0 - s) * grid + 0.5))
    keep = torch.empty(gr, gc, dtype=torch.uint8, device="cuda")
    gsel = torch.empty_like(keep)
    regrown = torch.empty_like(keep)
    counts = torch.empty(2, dtype=torch.int64, device="cuda")
    col_ptr = torch.empty(gc + 1, dtype=torch.int64, device="cuda")
    kmap = torch.empty(gr, gc, dtype=torch.int32, device="cuda")
    masked = torch.empty_like(w)

    t_norm = ev_time(lambda: lib.blast_block_norms(w.data_ptr(), g.data_ptr(), rows, cols, b, L.F32,
                                                   nw.data_ptr(), ng.data_ptr(), st))
    t_topk = ev_time(lambda: lib.blast_topk_mask(nw.data_ptr(), gr, gc, k, keep.data_ptr(), st))
    lib.blast_topk_mask(ng.data_ptr(), gr, gc, k, gsel.data_ptr(), st)
    t_diff = ev_time(lambda: lib.blast_mask_difference(keep.data_ptr(), gsel.data_ptr(), grid,
                                                       regrown.data_ptr(), counts.data_ptr(), st))
    t_index = ev_time(lambda: lib.blast_repack_index(keep.data_ptr(), regrown.data_ptr(), None, rows,
                                                     cols, b, L.F32, col_ptr.data_ptr(),
                                                     kmap.data_ptr(), st))
    nnzb = int(col_ptr[-1])
    row_idx = torch.empty(nnzb, dtype=torch.int32, device="cuda")
    values = torch.empty(nnzb, b, b, dtype=vdt, device="cuda")
    t_rows = ev_time(lambda: lib.blast_repack_rows(kmap.data_ptr(), col_ptr.data_ptr(), gr, gc,
                                                   row_idx.data_ptr(), st))
    t_gather = ev_time(lambda: lib.blast_apply_mask_gather(
        w.data_ptr(), rows, cols, b, L.F32, keep.data_ptr(), regrown.data_ptr(), 1,
        kmap.data_ptr(), masked.data_ptr(), values.data_ptr(), L.dtype_code(vdt), st))
    # whole API calls (includes the two small device->host reads)
    t_gen = ev_time(lambda: bs.generate_masks(w, g, b, s), iters=10)
    mask, _ = bs.generate_masks(w, g, b, s)
    t_apply = ev_time(lambda: bs.apply_mask(w, mask, b, dtype=vdt), iters=10)

    elt = torch.finfo(vdt).bits // 8
    bytes_norm = 2 * rows * cols * 4 + 2 * grid * 8
    bytes_topk = grid * 8 * 1 + grid
    bytes_gather = rows * cols * 8 + nnzb * b * b * elt
    gbs = lambda by, us: by / (us * 1e-6) / 1e9  # noqa: E731
    print(json.dumps({
        "shape": [rows, cols], "block": b, "sparsity": s, "grid_cells": grid, "nnzb": nnzb,
        "block_norms_us": t_norm, "block_norms_GBps": gbs(bytes_norm, t_norm),
        "topk_us": t_topk, "topk_GBps_norm_bytes": gbs(bytes_topk, t_topk),
        "mask_difference_us": t_diff, "repack_index_us": t_index, "repack_rows_us": t_rows,
        "apply_mask_gather_us": t_gather, "apply_mask_gather_GBps": gbs(bytes_gather, t_gather),
        "generate_masks_api_us": t_gen, "apply_mask_api_us": t_apply,
    }), flush=True)


if __name__ == "__main__":
    run(4096, 14336)
    run(8192, 28672)
    run(768, 3072)
