"""Per-chunk timeline of the host-buffer forward (BLAST_PIPE_TRACE=1): cfg3 shape, 8192 tokens."""
import sys, time
sys.path.insert(0, ".")
import torch, bench
import paper_2507_03117_b200 as bs
chunk = int(sys.argv[1]) if len(sys.argv) > 1 else 0
ws = bench.make_weights(4096, 14336, 64, 0.9, 0)
net = bs.SparseMlp.from_caches(*[bs.from_host(w, torch.bfloat16) for w in ws])
x = torch.randn(8192, 4096).bfloat16().pin_memory()
y = torch.empty(8192, 4096, dtype=torch.bfloat16).pin_memory()
for _ in range(3):
    bs.mlp_forward(x, net, save_activations=False, out=y, chunk_tokens=chunk)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    bs.mlp_forward(x, net, save_activations=False, out=y, chunk_tokens=chunk)
torch.cuda.synchronize()
print(f"chunk {chunk}: {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms per forward", flush=True)
