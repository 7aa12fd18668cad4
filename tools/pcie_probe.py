"""PCIe copy rates with 1 / 2 / 4 streams per direction, H2D alone and H2D + D2H together."""
import torch, time
n = 8192 * 4096
xh = torch.empty(n, dtype=torch.bfloat16).pin_memory()
yh = torch.empty(n, dtype=torch.bfloat16).pin_memory()
xd = torch.empty(n, dtype=torch.bfloat16, device="cuda")
yd = torch.empty(n, dtype=torch.bfloat16, device="cuda")
def run(k, both):
    ins = [torch.cuda.Stream() for _ in range(k)]
    outs = [torch.cuda.Stream() for _ in range(k)]
    step = n // k
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for rep in range(5):
        for i in range(k):
            with torch.cuda.stream(ins[i]):
                xd[i * step:(i + 1) * step].copy_(xh[i * step:(i + 1) * step], non_blocking=True)
            if both:
                with torch.cuda.stream(outs[i]):
                    yh[i * step:(i + 1) * step].copy_(yd[i * step:(i + 1) * step], non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    gb = n * 2 / 1e9
    print(f"streams {k} {'h2d+d2h' if both else 'h2d    '}: {dt*1e3:.3f} ms  {gb/dt:.1f} GB/s per direction", flush=True)
for both in (False, True):
    for k in (1, 2, 4):
        run(k, both)
