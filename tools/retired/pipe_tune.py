"""Host-buffer forward (cfg3, 8192 tokens): automatic chunk schedule under BLAST_PIPE_MID /
BLAST_PIPE_EDGE (read per call by the library), median of 10 event-timed calls."""
import os
import sys
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


def timed(reps=10):
    fn = lambda: bs.mlp_forward(xh, net, save_activations=False, out=yh)  # noqa: E731
    fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[reps // 2]


for mid, edge in ((0, 0), (1024, 256), (1024, 384), (1536, 512), (1536, 256), (1792, 512),
                  (1792, 256), (2048, 512), (2048, 256), (1280, 256), (0, 0)):
    for k, v in (("BLAST_PIPE_MID", mid), ("BLAST_PIPE_EDGE", edge)):
        if v:
            os.environ[k] = str(v)
        else:
            os.environ.pop(k, None)
    print(f"mid {mid} edge {edge}: {timed():.3f} ms", flush=True)
