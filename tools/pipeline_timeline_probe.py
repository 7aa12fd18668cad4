"""Per-chunk event timeline of a Python replica of the host-buffer pipeline
(csrc/pipeline.cu): copy-in on one stream, the MLP on the current stream, copy-out on a
third, `slots` device buffers. Prints start/end (us from the first copy) per chunk and
stage, and the totals for 3 and 4 slots."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2507_03117_b200 as bs  # noqa: E402

m, D = 8192, bench.D
ws = bench.make_weights(bench.D, bench.H, bench.BLOCK, bench.SPARSITY, 0)
net = bs.SparseMlp.from_caches(*[bs.from_host(w, torch.bfloat16) for w in ws])
xh = torch.randn(m, D).bfloat16().pin_memory()
yh = torch.empty_like(xh).pin_memory()
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()


def run(chunk, slots, verbose):
    bounds = list(range(0, m, chunk)) + [m]
    xs = [torch.empty(chunk, D, dtype=torch.bfloat16, device="cuda") for _ in range(slots)]
    ys = [torch.empty(chunk, D, dtype=torch.bfloat16, device="cuda") for _ in range(slots)]
    cur = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    t0 = ev()
    t0.record(cur)
    s_in.wait_stream(cur)
    s_out.wait_stream(cur)
    rec = []
    comp_done, out_done = [], []
    for c in range(len(bounds) - 1):
        r0, r1 = bounds[c], bounds[c + 1]
        n, k = r1 - r0, c % slots
        a, b = ev(), ev()
        if c >= slots:
            s_in.wait_event(comp_done[c - slots])
        with torch.cuda.stream(s_in):
            a.record(s_in)
            xs[k][:n].copy_(xh[r0:r1], non_blocking=True)
            b.record(s_in)
        cur.wait_event(b)
        if c >= slots:
            cur.wait_event(out_done[c - slots])
        ca, cb = ev(), ev()
        ca.record(cur)
        y, _ = bs.mlp_forward(xs[k][:n], net, save_activations=False)
        ys[k][:n].copy_(y)  # device copy (~10 us) so the copy-out reads a slot like the library
        cb.record(cur)
        comp_done.append(cb)
        oa, ob = ev(), ev()
        s_out.wait_event(cb)
        with torch.cuda.stream(s_out):
            oa.record(s_out)
            yh[r0:r1].copy_(ys[k][:n], non_blocking=True)
            ob.record(s_out)
        out_done.append(ob)
        rec.append((a, b, ca, cb, oa, ob))
    cur.wait_stream(s_out)
    torch.cuda.synchronize()
    if verbose:
        for c, evs in enumerate(rec):
            t = [t0.elapsed_time(e) * 1e3 for e in evs]
            print(f"  chunk {c}: in {t[0]:7.1f}-{t[1]:7.1f}  mlp {t[2]:7.1f}-{t[3]:7.1f}  "
                  f"out {t[4]:7.1f}-{t[5]:7.1f} us")
    return t0.elapsed_time(rec[-1][5])


for chunk in (1024, 1536):
    for slots in (3, 4):
        for _ in range(2):
            run(chunk, slots, False)
        total = run(chunk, slots, chunk == 1024 and slots == 3)
        print(f"chunk {chunk} slots {slots}: {total:.3f} ms")
