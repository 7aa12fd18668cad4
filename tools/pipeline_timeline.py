"""Per-stage timeline of the chunked host-buffer forward, re-enacted with torch streams
and timing events (same schedule as csrc/pipeline.cu) to see which stage stretches."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2507_03117_b200 as bs  # noqa: E402


def main(chunk=1024, slots=3, compute=True):
    m = 8192
    weights = bench.make_weights(bench.D, bench.H, bench.BLOCK, bench.SPARSITY, 0)
    net = bs.SparseMlp.from_caches(*[bs.from_host(w, torch.bfloat16) for w in weights])
    xh = torch.randn(m, bench.D).bfloat16().pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    xd = [torch.empty(chunk, bench.D, dtype=torch.bfloat16, device="cuda") for _ in range(slots)]
    yd = [torch.empty_like(xd[0]) for _ in range(slots)]
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    st = torch.cuda.current_stream()
    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    for rep in range(3):
        n = m // chunk
        t0 = E()
        t0.record(st)
        s_in.wait_stream(st)
        s_out.wait_stream(st)
        ev = []
        comp_done, out_done = [], []
        for c in range(n):
            k = c % slots
            e_in0, e_in1, e_c0, e_c1, e_o0, e_o1 = (E() for _ in range(6))
            if c >= slots:
                s_in.wait_event(comp_done[c - slots])
            e_in0.record(s_in)
            with torch.cuda.stream(s_in):
                xd[k].copy_(xh[c * chunk:(c + 1) * chunk], non_blocking=True)
            e_in1.record(s_in)
            st.wait_event(e_in1)
            if c >= slots:
                st.wait_event(out_done[c - slots])
            e_c0.record(st)
            if compute:
                y, _ = bs.mlp_forward(xd[k], net, save_activations=False)
                yd[k].copy_(y)
            e_c1.record(st)
            comp_done.append(e_c1)
            s_out.wait_event(e_c1)
            e_o0.record(s_out)
            with torch.cuda.stream(s_out):
                yh[c * chunk:(c + 1) * chunk].copy_(yd[k], non_blocking=True)
            e_o1.record(s_out)
            out_done.append(e_o1)
            ev.append((e_in0, e_in1, e_c0, e_c1, e_o0, e_o1))
        st.wait_event(out_done[-1])
        torch.cuda.synchronize()
        if rep == 2:
            rows = [[round(t0.elapsed_time(e), 3) for e in evs] for evs in ev]
            print(json.dumps({"chunk": chunk, "slots": slots, "compute": compute,
                              "total_ms": rows[-1][-1], "stages_ms": rows}))


if __name__ == "__main__":
    for compute in (True, False):
        main(compute=compute)
