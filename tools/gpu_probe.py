"""First on-device check of the native engine against torch references.

Builds random block-sparse matrices directly as device arrays, calls the C ABI
through ctypes and compares with dense torch fp32/fp64 products. Prints one line
per case; exits non-zero on a mismatch. Used for the very first GPU bring-up.
"""
import ctypes as C
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2507_03117_b200 import _lib as L  # noqa: E402

lib = L.load()
dev = "cuda"
torch.manual_seed(0)
fails = 0


def rand_bcsc(rows, cols, b, dens, dtype, gen):
    gr, gc = -(-rows // b), -(-cols // b)
    mask = torch.rand(gr, gc, generator=gen) < dens
    dense = torch.randn(rows, cols, generator=gen) / (rows ** 0.5)
    pad = torch.zeros(gr * b, gc * b)
    pad[:rows, :cols] = dense
    blocks = pad.view(gr, b, gc, b).permute(0, 2, 1, 3)  # gr,gc,b,b
    cols_idx, rows_idx = torch.nonzero(mask.t(), as_tuple=True)  # column-major
    values = blocks[rows_idx, cols_idx].contiguous()
    col_ptr = torch.zeros(gc + 1, dtype=torch.int64)
    col_ptr[1:] = torch.cumsum(mask.sum(0), 0)
    wd = torch.zeros(gr * b, gc * b)
    for k in range(values.shape[0]):
        r, c = rows_idx[k].item(), cols_idx[k].item()
        wd[r * b:(r + 1) * b, c * b:(c + 1) * b] = values[k]
    wd = wd[:rows, :cols]
    v = values.to(dtype).to(dev)
    if dtype == torch.bfloat16:
        wd = wd.to(torch.bfloat16).float()
    return dict(rows=rows, cols=cols, b=b, gr=gr, gc=gc, col_ptr=col_ptr.to(dev),
                row_idx=rows_idx.to(torch.int32).to(dev), values=v, dense=wd.to(dev),
                nnzb=values.shape[0])


def desc(w, dtype):
    s = torch.cuda.current_stream().cuda_stream
    gr, gc = w["gr"], w["gc"]
    kmap = torch.empty(gr, gc, dtype=torch.int32, device=dev)
    L.check(lib.blast_kmap_from_bcsc(w["col_ptr"].data_ptr(), w["row_idx"].data_ptr(), gr, gc,
                                     kmap.data_ptr(), s))
    plans = {}
    for name, by_rows in (("fwd", 0), ("rt", 1)):
        lines = gr if by_rows else gc
        sp = torch.empty(lines + 1, dtype=torch.int32, device=dev)
        st = torch.empty(gr * gc * 4 + 4, dtype=torch.int32, device=dev)
        fl = torch.empty(lines, dtype=torch.int32, device=dev)
        L.check(lib.blast_build_plan(kmap.data_ptr(), None, gr, gc, by_rows, sp.data_ptr(),
                                     st.data_ptr(), fl.data_ptr(), s))
        plans[name] = (sp, st, fl)
    lo = None
    vals = w["values"]
    if dtype == torch.float32:
        hi = torch.empty_like(vals)
        lo = torch.empty_like(vals)
        L.check(lib.blast_split_tf32(vals.data_ptr(), hi.data_ptr(), lo.data_ptr(), vals.numel(), s))
        vals = hi
    d = L.BcscDesc(w["rows"], w["cols"], w["b"], L.dtype_code(dtype), w["nnzb"],
                   w["col_ptr"].data_ptr(), w["row_idx"].data_ptr(), vals.data_ptr(),
                   lo.data_ptr() if lo is not None else None, kmap.data_ptr(),
                   plans["fwd"][0].data_ptr(), plans["fwd"][1].data_ptr(), plans["fwd"][2].data_ptr(),
                   plans["rt"][0].data_ptr(), plans["rt"][1].data_ptr(), plans["rt"][2].data_ptr())
    keep = (kmap, plans, vals, lo)
    return d, keep


def maxrel(got, ref):
    return ((got.double() - ref.double()).abs().max() / ref.double().abs().max().clamp_min(1e-30)).item()


def case(m, rows, cols, b, dens, dtype, tol):
    global fails
    gen = torch.Generator().manual_seed(m * 7 + rows + b)
    w = rand_bcsc(rows, cols, b, dens, dtype, gen)
    d, keep = desc(w, dtype)
    x = torch.randn(m, rows, generator=gen).to(dtype).to(dev)
    y = torch.empty(m, cols, dtype=dtype, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    L.check(lib.blast_bspmm(x.data_ptr(), m, C.byref(d), 0, y.data_ptr(), s), "bspmm")
    torch.cuda.synchronize()
    ref = x.double() @ w["dense"].double()
    e1 = maxrel(y, ref)
    # transposed
    xt = torch.randn(m, cols, generator=gen).to(dtype).to(dev)
    yt = torch.empty(m, rows, dtype=dtype, device=dev)
    L.check(lib.blast_bspmm_rt(xt.data_ptr(), m, C.byref(d), yt.data_ptr(), s), "bspmm_rt")
    torch.cuda.synchronize()
    e2 = maxrel(yt, xt.double() @ w["dense"].double().t())
    ok = e1 <= tol and e2 <= tol
    fails += not ok
    print(f"{'OK ' if ok else 'BAD'} bspmm m={m} {rows}x{cols} b={b} dens={dens} {dtype}: fwd {e1:.2e} rt {e2:.2e}", flush=True)


t0 = time.time()
for dtype, tol in ((torch.bfloat16, 2e-2), (torch.float32, 1e-5)):
    for b in (16, 32, 64, 128):
        if dtype == torch.float32 and b == 128:
            continue
        case(256, 512, 768, b, 0.3, dtype, tol)
        case(100, 256, 384, b, 0.5, dtype, tol)
case(37, 13, 11, 4, 0.6, torch.float32, 1e-5)
case(5, 24, 40, 8, 0.5, torch.bfloat16, 2e-2)
print("elapsed", time.time() - t0)
sys.exit(1 if fails else 0)
