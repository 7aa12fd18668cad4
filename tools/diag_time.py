"""cfg3 MLP forward timed with CUDA events (warm, back to back); used with the diagnosis
switches (BLAST_SKIP_EPILOGUE=1/2/3) to split a kernel's time between its stages."""
import sys
sys.path.insert(0, ".")
import bench, torch
import paper_2507_03117_b200 as bs
sp = float(sys.argv[1]) if len(sys.argv) > 1 else 0.9
ws = bench.make_weights(4096, 14336, 64, sp, 0)
net = bs.SparseMlp.from_caches(*[bs.from_host(w, torch.bfloat16) for w in ws])
x = torch.randn(8192, 4096, device="cuda").bfloat16()
for _ in range(3):
    bs.mlp_forward(x, net, save_activations=False)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    bs.mlp_forward(x, net, save_activations=False)
b.record()
torch.cuda.synchronize()
print(f"forward {a.elapsed_time(b) / 20 * 1e3:.1f} us")
