"""Quick timing of bench extras without the full bench: python tools/extras_quick.py cfg0 decode ..."""
import sys, json
sys.path.insert(0, ".")
import torch, bench
import paper_2507_03117_b200 as bs
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
hbm, tf, _ = bench.load_peaks()
for what in sys.argv[1:] or ["cfg0", "decode"]:
    if what == "cfg0":
        print(json.dumps(bench.extra_cfg0_fp32(bs, flush, tf, 20, 0)))
    elif what == "prune":
        import paper_2507_03117_b200._lib as L
        print(json.dumps(bench.extra_prune_refresh(bs, L, flush, hbm, 20)))
    elif what == "train":
        ws = bench.make_weights(bench.D, bench.H, bench.BLOCK, bench.SPARSITY, 0)
        net = bs.SparseMlp.from_caches(*[bs.from_host(w, torch.bfloat16) for w in ws])
        x = torch.randn(8192, bench.D, device="cuda").bfloat16()
        print(json.dumps(bench.extra_train_step(bs, net, x, 1, flush, tf, 10)))
    elif what == "decode":
        print(json.dumps(bench.extra_decode(bs, flush, hbm, 50, 0)))
