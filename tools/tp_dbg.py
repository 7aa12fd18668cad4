import sys; sys.path.insert(0, ".")
import numpy as np, torch
sys.argv = ["x"]
sys.path.insert(0, "tests"); import test_gpu_parallel as T
import oracle
import paper_2507_03117_b200 as bs
from paper_2507_03117_b200 import parallel
world, m, dtype = 2, 300, torch.bfloat16
e, h, b = 512, 2048, 64
rng = np.random.default_rng(world * 100 + m)
wg, wu, wd = oracle.mlp_init(e, h, rng)
for w in (wg, wu, wd):
    keep = rng.random((w.shape[0] // b, w.shape[1] // b)) < 0.15
    w *= np.kron(keep, np.ones((b, b), np.float32))
x = torch.from_numpy(rng.standard_normal((m, e)).astype(np.float32)).cuda().to(dtype)
nets = T._shard_nets(wg, wu, wd, b, world, dtype)
group = parallel.FusedTPGroup.local(world, m, e, b, dtype)
for epoch in range(2):
    for r in range(world):
        group.forward(x, nets[r], r)
    ys = [group.wait(r).clone() for r in range(world)]
    torch.cuda.synchronize()
    d = (ys[1].float() - ys[0].float()).abs()
    bad = (d > 0).nonzero()
    print("epoch", epoch, "ndiff", bad.shape[0], "rows", bad[:, 0].unique()[:20].tolist(), "cols", bad[:, 1].unique()[:20].tolist(), "max", d.max().item())
    print(ys[0][bad[:3,0], bad[:3,1]] if bad.shape[0] else "", ys[1][bad[:3,0], bad[:3,1]] if bad.shape[0] else "")
    group.step()
