#!/bin/bash
# cluster-pair split of decode-size single-matrix products: parity first, then decode A/B
timeout 120 python - <<'PY'
import sys; sys.path.insert(0, ".")
import torch, bench
import paper_2507_03117_b200 as bs
torch.manual_seed(0)
for m, k, n, sp in ((128, 14336, 4096, 0.95), (100, 512, 256, 0.5), (128, 256, 128, 0.0)):
    dense = torch.randn(k, n) * (torch.rand(k // 64, n // 64).repeat_interleave(64, 0).repeat_interleave(64, 1) > sp)
    mat = bs.from_dense(dense.cuda().bfloat16(), 64)
    x = torch.randn(m, k, device="cuda").bfloat16()
    y = bs.bspmm(x, mat)
    y2 = bs.bspmm(x, mat)
    assert torch.equal(y, y2), "not reproducible"
    ref = x.float() @ dense.cuda().bfloat16().float()
    err = ((y.float() - ref).abs().max() / ref.abs().max()).item()
    print("parity", m, k, n, sp, "rel max err", err, flush=True)
PY
echo "rc=$?"
for r in 1 2; do for v in 1 0; do echo -n "CLUSTER_SPLIT=$v "; BLAST_CLUSTER_SPLIT=$v timeout 120 python tools/extras_quick.py decode | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['us'],2), 'us flushed')"; done; done
for v in 1 0; do echo -n "CLUSTER_SPLIT=$v warm: "; BLAST_CLUSTER_SPLIT=$v timeout 120 python tools/graph_probe.py 2>&1 | head -1; done
