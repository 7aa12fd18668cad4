"""Single invocations (after warm-up) of the SURVEY §8(d) ncu cases, for
`ncu --set full -k regex:spmm_tc -s 4 -c 2 python tools/prof_cases.py A` (one case per run):
  A  cfg3 MLP forward at 50 % sparsity, 8192 tokens   (tensor-pipe utilisation, compute regime)
  B  cfg3 MLP forward at 95 % sparsity, 128 tokens    (HBM regime: nonzero weights dominate)
  C  prune-and-grow refresh of the cfg3 gate matrix   (block norms, top-k, apply-mask gather)
Each case is preceded by an NVTX range push so the report can be split by case."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2507_03117_b200 as bs  # noqa: E402


def mlp_case(s, m):
    ws = bench.make_weights(bench.D, bench.H, bench.BLOCK, s, 0)
    net = bs.SparseMlp.from_caches(*[bs.from_host(w, torch.bfloat16) for w in ws])
    x = torch.randn(m, bench.D, device="cuda").bfloat16()
    for _ in range(2):
        bs.mlp_forward(x, net, save_activations=False)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push(f"mlp s={s} m={m}")
    bs.mlp_forward(x, net, save_activations=False)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()


def prune_case():
    w = torch.randn(bench.D, bench.H, device="cuda") * bench.D ** -0.5
    g = torch.randn_like(w)
    for _ in range(2):
        mask, _ = bs.generate_masks(w, g, 64, 0.9)
        bs.apply_mask(w, mask, 64, dtype=torch.bfloat16)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("prune refresh 4096x14336")
    mask, _ = bs.generate_masks(w, g, 64, 0.9)
    bs.apply_mask(w, mask, 64, dtype=torch.bfloat16)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()


if __name__ == "__main__":
    case = sys.argv[1] if len(sys.argv) > 1 else "all"
    if case in ("A", "all"):
        mlp_case(0.5, 8192)
    if case in ("B", "all"):
        mlp_case(0.95, 128)
    if case in ("C", "all"):
        prune_case()
