"""Measurements for the non-headline BASELINE.json configs (one B200):

  cfg3 sweep: Llama-3-8B MLP shape, sparsity {0.5,0.7,0.8,0.9,0.95} x block {16,32,64,128},
              M = 8192 tokens, bf16, sparse fused MLP vs dense cuBLAS MLP (same protocol as
              bench.py: CUDA events, L2 flushed between steps).
  cfg1 e2e:   Llama-3.2-1B (16 layers, d=2048, h=8192) forward over batch 16 x seq 2048,
              95% block-sparse MLPs (b=64) vs the dense model, bf16, random weights.
  cfg2 step:  GPT-2 small (12 layers, d=768, h=3072) MLP stack training step at 90%
              (fwd + bwd + weight update, masks refreshed every step_size steps) vs dense.

Prints one JSON line per measurement. Usage: python tools/config_sweep.py [cfg3|cfg1|cfg2|all]
"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2507_03117_b200 as bs  # noqa: E402

F = torch.nn.functional
FLUSH = None


def timed(fn, iters=10, warmup=3):
    global FLUSH
    if FLUSH is None:
        FLUSH = torch.empty(64 * 1024 * 1024, device="cuda")
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        FLUSH.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def cfg3_sweep():
    """argv: cfg3 [blocks] [token counts] [sparsities], comma lists."""
    d, h = 4096, 14336
    peak = bench.load_peaks()[1]
    hbm = bench.load_peaks()[0]
    blocks = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else (16, 32, 64, 128)
    ms_list = [int(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 else (8192,)
    sps = [float(v) for v in sys.argv[4].split(",")] if len(sys.argv) > 4 else (0.5, 0.7, 0.8, 0.9, 0.95)
    for m in ms_list:
        x = torch.randn(m, d, device="cuda").bfloat16()
        wg = torch.randn(h, d, device="cuda", dtype=torch.bfloat16) * d ** -0.5
        wu = torch.randn(h, d, device="cuda", dtype=torch.bfloat16) * d ** -0.5
        wd = torch.randn(d, h, device="cuda", dtype=torch.bfloat16) * h ** -0.5
        dense_ms = timed(lambda: F.linear(F.silu(F.linear(x, wg)) * F.linear(x, wu), wd))
        del wg, wu, wd
        for b in blocks:
            for s in sps:
                ws = bench.make_weights(d, h, b, s, 0)
                net = bs.SparseMlp.from_caches(*[bs.from_host(w, torch.bfloat16) for w in ws])
                ms = timed(lambda: bs.mlp_forward(x, net, save_activations=False))
                nnzb = sum(w.cache.nnzb for w in net.matrices())
                fl = 2 * m * b * b * nnzb
                # roofline of the north star: the slower of nnz-block FLOPs at tensor peak and
                # nonzero-weight + activation (X in, Y out) bytes at HBM bandwidth
                byts = nnzb * b * b * 2 + 2 * m * d * 2
                t_fl, t_by = fl / (peak * 1e12) * 1e3, byts / (hbm * 1e9) * 1e3
                print(json.dumps({"config": "cfg3", "block": b, "sparsity": s, "tokens": m,
                                  "sparse_ms": ms, "dense_cublas_ms": dense_ms,
                                  "speedup_vs_dense": dense_ms / ms,
                                  "tokens_per_s": m / (ms * 1e-3),
                                  "tflops": fl / (ms * 1e-3) / 1e12,
                                  "frac_of_peak": fl / (ms * 1e-3) / 1e12 / peak,
                                  "bound": "tensor" if t_fl >= t_by else "hbm",
                                  "roofline_ms": max(t_fl, t_by),
                                  "frac_roofline": max(t_fl, t_by) / ms,
                                  "hbm_gbs": byts / (ms * 1e-3) / 1e9}), flush=True)
                del net
        del x


def cfg1_e2e():
    from transformers import LlamaConfig, LlamaForCausalLM
    from paper_2507_03117_b200 import integration
    cfg = LlamaConfig(hidden_size=2048, intermediate_size=8192, num_hidden_layers=16,
                      num_attention_heads=32, num_key_value_heads=8, vocab_size=128256,
                      max_position_embeddings=4096, tie_word_embeddings=True)
    torch.manual_seed(0)
    model = LlamaForCausalLM(cfg).cuda().to(torch.bfloat16).eval()
    ids = torch.randint(0, cfg.vocab_size, (16, 2048), device="cuda")

    def run():
        with torch.no_grad():
            return model.model(ids).last_hidden_state   # decoder stack (LM head excluded)

    dense_ms = timed(run, iters=5, warmup=2)
    integration.sparsify_llama(model, 64, 0.95)
    sparse_ms = timed(run, iters=5, warmup=2)
    tok = 16 * 2048
    print(json.dumps({"config": "cfg1", "model": "Llama-3.2-1B decoder (random init)",
                      "batch": 16, "seq": 2048, "mlp_sparsity": 0.95, "block": 64,
                      "dense_ms": dense_ms, "sparse_ms": sparse_ms,
                      "dense_tokens_per_s": tok / (dense_ms * 1e-3),
                      "sparse_tokens_per_s": tok / (sparse_ms * 1e-3),
                      "e2e_speedup": dense_ms / sparse_ms}), flush=True)


def cfg2_step():
    """GPT-2 small MLP stack (12 x GPT2MLP, GELU, bias) at 90% block sparsity, b=64:
    forward + backward through SparseGeluMLP (autograd) vs the dense torch MLP, plus the
    cost of one prune-and-grow refresh of all 24 matrices (amortised over step_size=10)."""
    from transformers import GPT2Config
    from transformers.models.gpt2.modeling_gpt2 import GPT2MLP
    from paper_2507_03117_b200 import integration
    d, h, layers, m = 768, 3072, 12, 8192
    cfg = GPT2Config(n_embd=d, n_inner=h, resid_pdrop=0.0)
    torch.manual_seed(0)
    dense = [GPT2MLP(h, cfg).cuda().to(torch.bfloat16) for _ in range(layers)]
    sparse = [integration.SparseGeluMLP.from_gpt2(mlp.float(), 64, 0.9) for mlp in dense]
    for mlp in dense:
        mlp.to(torch.bfloat16)
    x = torch.randn(m, d, device="cuda", dtype=torch.bfloat16, requires_grad=True)

    def run(stack):
        h_ = x
        for mlp in stack:
            h_ = mlp(h_)
        h_.float().sum().backward()

    dense_ms = timed(lambda: run(dense), iters=5, warmup=2)
    sparse_ms = timed(lambda: run(sparse), iters=5, warmup=2)
    masters = [(torch.randn(d, h, device="cuda"), torch.randn(h, d, device="cuda"))
               for _ in range(layers)]

    def refresh():
        for w1, w2 in masters:
            for w in (w1, w2):
                mask, _ = bs.generate_masks(w, torch.randn_like(w), 64, 0.9)
                bs.apply_mask(w, mask, 64, dtype=torch.bfloat16)

    refresh_ms = timed(refresh, iters=3, warmup=1)
    print(json.dumps({"config": "cfg2", "model": "GPT-2 small MLP stack (12 x GPT2MLP)",
                      "tokens": m, "sparsity": 0.9, "block": 64,
                      "sparse_fwd_bwd_ms": sparse_ms, "dense_fwd_bwd_ms": dense_ms,
                      "refresh_all_24_matrices_ms": refresh_ms,
                      "step_ms_refresh_every_10": sparse_ms + refresh_ms / 10,
                      "speedup_vs_dense": dense_ms / (sparse_ms + refresh_ms / 10)}), flush=True)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("cfg3", "all"):
        cfg3_sweep()
    if which in ("cfg1", "all"):
        cfg1_e2e()
    if which in ("cfg2", "all"):
        cfg2_step()
