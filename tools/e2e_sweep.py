"""Host-buffer forward at cfg3: chunk-size sweep of blast_mlp_forward_host against the
bare PCIe copy times (H2D alone, D2H alone, both directions concurrently).
Prints one JSON line per measurement."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2507_03117_b200 as bs  # noqa: E402


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(reps)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in ev)[reps // 2]


def main():
    m = 8192
    weights = bench.make_weights(bench.D, bench.H, bench.BLOCK, bench.SPARSITY, 0)
    net = bs.SparseMlp.from_caches(*[bs.from_host(w, torch.bfloat16) for w in weights])
    xh = torch.randn(m, bench.D).bfloat16().pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    xd = xh.cuda()
    yd = torch.empty_like(xd)
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()

    def both():
        cur = torch.cuda.current_stream()
        s_in.wait_stream(cur)
        s_out.wait_stream(cur)
        with torch.cuda.stream(s_in):
            xd.copy_(xh, non_blocking=True)
        with torch.cuda.stream(s_out):
            yh.copy_(yd, non_blocking=True)
        cur.wait_stream(s_in)
        cur.wait_stream(s_out)

    nbytes = xh.numel() * 2
    try:
        from cuda.bindings import runtime as rt
        for name, t in (("x_host", xh), ("y_host", yh)):
            err, attr = rt.cudaPointerGetAttributes(t.data_ptr())
            print(json.dumps({"what": "pointer", "name": name, "err": str(err),
                              "type": str(getattr(attr, "type", None))}))
    except Exception as exc:  # diagnostic only
        print(json.dumps({"what": "pointer", "error": repr(exc)}))
    for name, fn in (("h2d", lambda: xd.copy_(xh, non_blocking=True)),
                     ("d2h", lambda: yh.copy_(yd, non_blocking=True)), ("both", both),
                     ("device_fwd", lambda: bs.mlp_forward(xd, net, save_activations=False))):
        ms = timed(fn)
        print(json.dumps({"what": name, "ms": ms, "GBps_per_direction": nbytes / ms / 1e6}))
    import time
    for chunk in (0, 256, 512, 768, 1024, 1536, 2048, 4096):
        fn = lambda: bs.mlp_forward(xh, net, save_activations=False, out=yh,  # noqa: E731
                                    chunk_tokens=chunk)
        ms = timed(fn)
        t0 = time.perf_counter()
        for _ in range(5):
            fn()
        wall = (time.perf_counter() - t0) / 5 * 1e3
        print(json.dumps({"what": "forward_host", "chunk_tokens": chunk, "ms": ms,
                          "wall_ms": wall, "tokens_per_s": m / ms * 1e3}))


if __name__ == "__main__":
    main()
