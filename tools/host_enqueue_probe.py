"""Host time to enqueue one host-buffer forward (no sync) vs its GPU time: is the chunked
copy-in / compute / copy-out pipeline bound by the host's API calls?"""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2507_03117_b200 as bs  # noqa: E402

m = 8192
ws = bench.make_weights(bench.D, bench.H, bench.BLOCK, bench.SPARSITY, 0)
net = bs.SparseMlp.from_caches(*[bs.from_host(w, torch.bfloat16) for w in ws])
xh = torch.randn(m, bench.D).bfloat16().pin_memory()
yh = torch.empty_like(xh).pin_memory()
xd = xh.cuda()
import ctypes as C  # noqa: E402
from paper_2507_03117_b200 import _lib as L  # noqa: E402
dg, du, dd = (mat.cache.desc() for mat in net.matrices())
plan = net.plan()


def call(chunk):  # the C entry point alone: returns once the pipeline is enqueued
    L.check(L.load().blast_mlp_forward_host(xh.data_ptr(), m, C.byref(dg), C.byref(du),
                                            C.byref(dd), C.byref(plan), yh.data_ptr(),
                                            chunk, L.stream()), "mlp_forward_host")


for chunk in (0, 1536):
    for _ in range(3):
        call(chunk)
    torch.cuda.synchronize()
    enq = []
    for _ in range(10):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        call(chunk)
        enq.append((time.perf_counter() - t0) * 1e3)
    torch.cuda.synchronize()
    enq.sort()
    print(f"chunk {chunk}: host enqueue {enq[5]:.3f} ms (median of 10)")
for _ in range(3):
    bs.mlp_forward(xd, net, save_activations=False)
torch.cuda.synchronize()
t0 = time.perf_counter()
bs.mlp_forward(xd, net, save_activations=False)
print(f"device-buffer forward enqueue {(time.perf_counter() - t0) * 1e3:.3f} ms")
