"""Quick forward check of the gated MLP (bf16 and fp32) against torch on masked weights."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2507_03117_b200 as bs
import bench

def run(e, h, b, s, m, dt):
    ws = bench.make_weights(e, h, b, s, 0)
    mats = [bs.from_host(w, dt) for w in ws]
    net = bs.SparseMlp.from_caches(*mats)
    x = torch.randn(m, e, device="cuda").to(dt)
    dense = [torch.as_tensor(bs.to_dense(mt)).cuda().float() for mt in mats]
    xf = x.float()
    a = xf @ dense[0]; u = xf @ dense[1]
    g = torch.nn.functional.silu(a) * u
    yref = g @ dense[2]
    for save in (False, True):
        y, acts = bs.mlp_forward(x, net, save_activations=save)
        torch.cuda.synchronize()
        err = ((y.float() - yref).abs().max() / yref.abs().max()).item()
        gerr = ((acts.gated.float() - g).abs().max() / g.abs().max()).item() if acts else -1
        print(f"e={e} h={h} b={b} m={m} {dt} save={save}: y {err:.2e} g {gerr:.2e}", flush=True)

for dt in (torch.bfloat16, torch.float32):
    for (e, h, b, s, m) in [(256, 512, 64, 0.5, 200), (512, 1024, 64, 0.75, 512), (256, 512, 32, 0.5, 256),
                            (1024, 2048, 16, 0.9, 512), (1024, 2048, 32, 0.9, 300), (1024, 2048, 16, 0.8, 1000)]:
        run(e, h, b, s, m, dt)

print("single products:")
for dt in (torch.bfloat16, torch.float32):
    for (e, h, b, s, m) in [(256, 512, 64, 0.5, 200), (512, 1024, 64, 0.75, 512)]:
        ws = bench.make_weights(e, h, b, s, 0)
        mt = bs.from_host(ws[0], dt)
        x = torch.randn(m, e, device="cuda").to(dt)
        ref = x.float() @ torch.as_tensor(bs.to_dense(mt)).cuda().float()
        y = bs.bspmm(x, mt)
        torch.cuda.synchronize()
        print(dt, e, h, b, m, "bspmm", ((y.float() - ref).abs().max() / ref.abs().max()).item(), flush=True)
