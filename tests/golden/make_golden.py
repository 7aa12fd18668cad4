"""Generate golden vectors by running the REAL reference package.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
It imports ``blocksparse`` from /root/reference/pkg/src, evaluates the hot-path
functions on seeded inputs and writes compressed .npz fixtures next to this
file. The fixtures are committed; nothing on the GPU box reads /root/reference.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF_SRC))

from blocksparse import bcsc, kernels, mlp, pruner  # noqa: E402
from blocksparse.bench import random_bcsc  # noqa: E402


def pack_bcsc(prefix: str, w, d: dict) -> None:
    d[f"{prefix}_meta"] = np.array([w.rows, w.cols, w.block], dtype=np.int64)
    d[f"{prefix}_col_ptr"] = w.col_ptr
    d[f"{prefix}_row_idx"] = w.block_row_idx
    d[f"{prefix}_values"] = w.values


def gen_products() -> None:
    cases = [
        # m, k, n, b, sparsity, seed
        (6, 8, 12, 4, 0.5, 1), (16, 8, 12, 4, 0.5, 2), (9, 13, 11, 4, 0.0, 3),
        (33, 40, 24, 8, 0.5, 4), (17, 7, 9, 1, 0.3, 5), (20, 30, 18, 2, 0.6, 6),
        (40, 64, 48, 16, 0.5, 7), (64, 64, 64, 16, 1.0, 8), (50, 96, 80, 16, 0.9, 9),
        (130, 128, 192, 32, 0.5, 10), (200, 256, 384, 64, 0.5, 11), (129, 192, 128, 64, 0.9, 12),
        (64, 256, 256, 128, 0.5, 13), (70, 100, 72, 16, 0.4, 14), (12, 24, 16, 8, 0.0, 15),
    ]
    d = {"cases": np.array(cases, dtype=np.float64)}
    for i, (m, k, n, b, s, seed) in enumerate(cases):
        rng = np.random.default_rng(seed)
        w = random_bcsc(int(k), int(n), int(b), float(s), rng)
        # tame the scale like SparseMlp.create so fp32 values stay O(1)
        w.values[...] *= np.float32(1.0 / np.sqrt(k))
        x = rng.standard_normal((int(m), int(k))).astype(np.float32)
        xt = rng.standard_normal((int(m), int(n))).astype(np.float32)
        pack_bcsc(f"c{i}_w", w, d)
        d[f"c{i}_x"] = x
        d[f"c{i}_xt"] = xt
        d[f"c{i}_y"] = kernels.bspmm(x, w)
        d[f"c{i}_yt"] = kernels.bspmm_rt(xt, w)
        for f in ("relu", "gelu", "silu"):
            d[f"c{i}_y_{f}"] = kernels.bspmm_fused(x, w, f)
        d[f"c{i}_dense"] = w.to_dense()
    np.savez_compressed(OUT / "products.npz", **d)


def gen_mlp() -> None:
    cases = [
        # e, h, b, sparsity, m, seed
        (12, 20, 4, 0.3, 7, 21), (64, 128, 16, 0.5, 40, 22), (128, 256, 64, 0.75, 130, 23),
        (128, 192, 32, 0.0, 64, 24), (256, 512, 64, 0.9, 256, 25),
    ]
    d = {"cases": np.array(cases, dtype=np.float64)}
    for i, (e, h, b, s, m, seed) in enumerate(cases):
        e, h, b, m = int(e), int(h), int(b), int(m)
        rng = np.random.default_rng(seed)
        net = mlp.SparseMlp.create(e, h, b, rng)
        if s > 0:
            for name, mat in zip(("gate", "up", "down"), net.matrices()):
                g = rng.standard_normal(mat.dense.shape).astype(np.float32)
                mask, _ = pruner.generate_masks(mat.dense, g, b, float(s))
                mat.mask = mask
                mat.dense, mat.cache = pruner.apply_mask(mat.dense, mask, b)
        x = rng.standard_normal((m, e)).astype(np.float32)
        y, acts = mlp.mlp_forward(x, net)
        dy = rng.standard_normal((m, e)).astype(np.float32)
        dx, dwg, dwu, dwd = mlp.mlp_backward(dy, acts, net)
        for name, mat in zip(("gate", "up", "down"), net.matrices()):
            d[f"c{i}_{name}_dense"] = mat.dense
            d[f"c{i}_{name}_kept"] = mat.mask.kept
            d[f"c{i}_{name}_regrown"] = mat.mask.regrown
            pack_bcsc(f"c{i}_{name}", mat.cache, d)
        d[f"c{i}_x"] = x
        d[f"c{i}_dy"] = dy
        d[f"c{i}_y"] = y
        d[f"c{i}_a"] = acts.gate_pre
        d[f"c{i}_b"] = acts.up_out
        d[f"c{i}_g"] = acts.gated
        d[f"c{i}_dx"] = dx
        d[f"c{i}_dwg"] = dwg
        d[f"c{i}_dwu"] = dwu
        d[f"c{i}_dwd"] = dwd
    np.savez_compressed(OUT / "mlp.npz", **d)


def block_fill(grid_vals, b):
    g = np.asarray(grid_vals, dtype=np.float32)
    return np.repeat(np.repeat(g, b, axis=0), b, axis=1)


def gen_prune() -> None:
    cases = []
    rng = np.random.default_rng(31)
    # random dense pairs, several shapes / block sizes / sparsities (incl. padding)
    all_s = (0.0, 0.3, 0.5, 0.9, 0.95, 1.0)
    for (rows, cols, b, ss) in ((16, 16, 4, all_s), (12, 12, 3, all_s), (13, 11, 4, all_s),
                                (64, 96, 16, all_s), (100, 60, 8, all_s), (256, 128, 32, (0.5, 0.9)),
                                (128, 448, 64, (0.9,))):
        for s in ss:
            w = rng.standard_normal((rows, cols)).astype(np.float32)
            g = rng.standard_normal((rows, cols)).astype(np.float32)
            cases.append((w, g, b, s))
    # hand-worked grids and ties (tests/test_pruner.py:166-175, :128-134)
    cases.append((block_fill([[4.0, 1.0], [2.0, 3.0]], 2), block_fill([[4.0, 3.0], [1.0, 2.0]], 2), 2, 0.5))
    cases.append((np.ones((4, 6), np.float32), np.ones((4, 6), np.float32), 2, 0.5))
    ties = rng.integers(0, 3, size=(8, 12)).astype(np.float32)
    cases.append((block_fill(ties, 4), block_fill(ties[::-1].copy(), 4), 4, 0.6))
    # NaN / -0.0 / inf blocks
    w = rng.standard_normal((32, 32)).astype(np.float32)
    w[0:8, 8:16] = np.nan
    w[8:16, 0:8] = -0.0
    w[16:24, 16:24] = np.inf
    cases.append((w, rng.standard_normal((32, 32)).astype(np.float32), 8, 0.5))
    d = {"n": np.array(len(cases))}
    for i, (w, g, b, s) in enumerate(cases):
        d[f"c{i}_w"] = w
        d[f"c{i}_g"] = g
        d[f"c{i}_bs"] = np.array([b, s], dtype=np.float64)
        nw = pruner.block_norms(w, b)
        ng = pruner.block_norms(g, b)
        d[f"c{i}_nw"] = nw
        d[f"c{i}_ng"] = ng
        d[f"c{i}_keep"] = pruner.prune_s(nw, s)
        mask, rep = pruner.generate_masks(w, g, b, s)
        d[f"c{i}_kept"] = mask.kept
        d[f"c{i}_regrown"] = mask.regrown
        d[f"c{i}_report"] = np.array([rep.kept, rep.regrown, rep.regrown_ratio, rep.s_achieved])
        for zr in (True, False):
            masked, cache = pruner.apply_mask(w, mask, b, zero_regrown=zr)
            tag = "z" if zr else "nz"
            d[f"c{i}_{tag}_masked"] = masked
            pack_bcsc(f"c{i}_{tag}", cache, d)
    # prune_s on raw norm grids with heavy ties / NaN (test_pruner.py:136-144)
    r2 = np.random.default_rng(32)
    for j in range(30):
        gr, gc = int(r2.integers(1, 13)), int(r2.integers(1, 13))
        norms = r2.integers(0, 4, size=(gr, gc)).astype(np.float64)
        if j % 5 == 0:
            norms[r2.random((gr, gc)) < 0.2] = np.nan
        s = float(r2.random())
        d[f"p{j}_norms"] = norms
        d[f"p{j}_s"] = np.array(s)
        d[f"p{j}_keep"] = pruner.prune_s(norms, s)
    d["n_prune_s"] = np.array(30)
    np.savez_compressed(OUT / "prune.npz", **d)


def gen_format() -> None:
    rng = np.random.default_rng(41)
    d = {}
    cases = []
    for (rows, cols, b) in ((8, 8, 4), (13, 11, 4), (64, 96, 16), (130, 70, 32), (3, 3, 2)):
        dense = rng.standard_normal((rows, cols)).astype(np.float32)
        gr, gc = -(-rows // b), -(-cols // b)
        zero = rng.random((gr, gc)) < 0.4
        for r in range(gr):
            for c in range(gc):
                if zero[r, c]:
                    dense[r * b:(r + 1) * b, c * b:(c + 1) * b] = 0.0
        dense[0, 0] = -0.0
        cases.append((dense, b))
    for i, (dense, b) in enumerate(cases):
        d[f"c{i}_dense"] = dense
        d[f"c{i}_b"] = np.array(b)
        pack_bcsc(f"c{i}_auto", bcsc.from_dense(dense, b), d)
        gr, gc = -(-dense.shape[0] // b), -(-dense.shape[1] // b)
        kept = rng.random((gr, gc)) < 0.5
        regrown = (rng.random((gr, gc)) < 0.3) & ~kept
        m = bcsc.BlockMask(kept=kept, regrown=regrown)
        d[f"c{i}_kept"] = kept
        d[f"c{i}_regrown"] = regrown
        pack_bcsc(f"c{i}_mask", bcsc.from_dense(dense, b, m), d)
        d[f"c{i}_bytes"] = np.frombuffer(bcsc.serialize(bcsc.from_dense(dense, b, m)), dtype=np.uint8)
    d["n"] = np.array(len(cases))
    # schedule values (pruner.py:53-67)
    sched_rows = []
    r3 = np.random.default_rng(42)
    for _ in range(50):
        s_max = float(r3.uniform(0.05, 1.0))
        s_init = float(r3.uniform(0.0, s_max))
        mt = int(r3.integers(2, 100000))
        dc = int(r3.integers(0, mt))
        i = int(r3.integers(0, mt + 1))
        sch = pruner.SparsitySchedule(s_init, s_max, mt, dc, 1)
        sched_rows.append([s_init, s_max, mt, dc, i, pruner.target_sparsity(i, sch)])
    d["schedule"] = np.array(sched_rows, dtype=np.float64)
    np.savez_compressed(OUT / "format.npz", **d)


TRAIN_CASES = {
    # name: TrainConfig fields (schedule as a dict); fp32, toy sizes, 3+ refreshes each
    "reg": dict(layers=2, embed_dim=32, hidden_dim=32, block_size=8, lr=0.1, batch_size=32,
                seed=0, schedule=dict(initial_sparsity=0.0, max_sparsity=0.8, total_iters=24,
                                      decay_iters=0, step_size=8)),
    "reg_dense": dict(layers=3, embed_dim=32, hidden_dim=64, block_size=8, lr=0.05,
                      batch_size=16, seed=3, dense_layers=1, lr_final_frac=0.5,
                      teacher_in_dims=20, teacher_out_dims=12, distractor_scale=0.3,
                      schedule=dict(initial_sparsity=0.2, max_sparsity=0.7, total_iters=20,
                                    decay_iters=4, step_size=5)),
    "cls": dict(layers=2, embed_dim=32, hidden_dim=32, block_size=8, lr=0.2, batch_size=32,
                seed=1, task="classification", alpha=0.5, beta=0.5, teacher_hidden=16,
                schedule=dict(initial_sparsity=0.0, max_sparsity=0.75, total_iters=18,
                              decay_iters=0, step_size=6)),
}


def gen_trainer() -> None:
    """Run the real train() (trainer.py:318-408) and record per-iteration losses, FLOPs
    and refresh flags, every generate_masks call's kept/regrown grids and report counts,
    and the final dense masters."""
    from blocksparse import trainer
    d = {}
    orig = trainer.generate_masks
    for name, raw in TRAIN_CASES.items():
        calls = []

        def rec(w, g, b, s, iteration=0, _calls=calls):
            mask, rep = orig(w, g, b, s, iteration=iteration)
            _calls.append((mask, rep, s))
            return mask, rep

        trainer.generate_masks = rec
        try:
            log, stack = trainer.train(trainer.TrainConfig.from_dict(raw))
        finally:
            trainer.generate_masks = orig
        d[f"{name}_config"] = np.frombuffer(json.dumps(raw).encode(), dtype=np.uint8)
        task = trainer.make_task(trainer.TrainConfig.from_dict(raw))  # data stream, 2 batches
        for k in range(2):
            for j, arr in enumerate(task.next_batch(raw["batch_size"])):
                d[f"{name}_batch{k}_{j}"] = arr
        d[f"{name}_loss"] = np.array([r.loss for r in log.records], dtype=np.float64)
        d[f"{name}_flops"] = np.array([r.flops_cum for r in log.records], dtype=np.int64)
        d[f"{name}_refresh"] = np.array([r.refresh for r in log.records], dtype=bool)
        d[f"{name}_sparsity"] = np.array([r.layer_sparsity for r in log.records])
        d[f"{name}_n_calls"] = np.array(len(calls))
        for k, (mask, rep, s) in enumerate(calls):
            d[f"{name}_call{k}_kept"] = mask.kept
            d[f"{name}_call{k}_regrown"] = mask.regrown
            d[f"{name}_call{k}_counts"] = np.array([rep.kept, rep.regrown, rep.iteration])
            d[f"{name}_call{k}_s"] = np.array(s)
        for li, blk in enumerate(stack.blocks):
            for tag, mat in zip(("gate", "up", "down"), blk.matrices()):
                d[f"{name}_final_l{li}_{tag}"] = mat.dense
    np.savez_compressed(OUT / "trainer.npz", **d)


def main() -> None:
    gen_products()
    gen_mlp()
    gen_prune()
    gen_format()
    gen_trainer()
    meta = {"reference": str(REF_SRC), "numpy": np.__version__,
            "files": sorted(p.name for p in OUT.glob("*.npz"))}
    (OUT / "MANIFEST.json").write_text(json.dumps(meta, indent=1) + "\n")
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    main()
