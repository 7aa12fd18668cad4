"""3xTF32 precision probe: GPU float32 products vs float64 and vs the oracle."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_2507_03117_b200 as bs  # noqa: E402

rng = np.random.default_rng(0)
for (m, k, n, b, scale) in ((128, 256, 64, 64, 1.0), (128, 256, 64, 64, 1 / 16), (70, 100, 72, 16, 1.0),
                            (128, 256, 64, 8, 1.0), (128, 64, 64, 64, 1.0), (128, 64, 64, 16, 1.0)):
    x = rng.standard_normal((m, k)).astype(np.float32)
    dense = (rng.standard_normal((k, n)) * scale).astype(np.float32)
    w = bs.from_dense(dense, b)
    ref64 = x.astype(np.float64) @ dense.astype(np.float64)
    got = bs.bspmm(x, w)
    orc = oracle.bspmm(x, oracle.from_dense(dense, b))
    gt = bs.bspmm_rt(np.ascontiguousarray(x[:, :n]) if k >= n else x, w) if False else None
    print(f"m={m} k={k} n={n} b={b} scale={scale}: gpu-vs-f64 rel_err {oracle.rel_err(got, ref64):.2e} "
          f"maxnorm {oracle.max_norm_rel(got, ref64):.2e} | oracle-vs-f64 rel_err {oracle.rel_err(orc, ref64):.2e} "
          f"maxnorm {oracle.max_norm_rel(orc, ref64):.2e}")
    # transposed product
    xt = rng.standard_normal((m, n)).astype(np.float32)
    r64 = xt.astype(np.float64) @ dense.astype(np.float64).T
    gt = bs.bspmm_rt(xt, w)
    print(f"      rt: gpu-vs-f64 rel_err {oracle.rel_err(gt, r64):.2e} maxnorm {oracle.max_norm_rel(gt, r64):.2e}")
