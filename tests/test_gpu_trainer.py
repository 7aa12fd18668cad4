"""GPU training loop with prune-and-grow: ports of the reference's tests/test_trainer.py:100-210,
and a step-for-step comparison with the REAL reference ``train()`` (trainer.py:318-408) on three
toy fp32 configurations recorded in tests/golden/trainer.npz (per-iteration losses, FLOPs and
refresh flags; every generate_masks call's kept/regrown grids and counts; final masters)."""
import json

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
bs = pytest.importorskip("paper_2507_03117_b200")
from paper_2507_03117_b200 import trainer  # noqa: E402
from paper_2507_03117_b200.pruner import SparsitySchedule  # noqa: E402


def config(**kw):
    base = dict(layers=2, embed_dim=16, hidden_dim=16, block_size=4, lr=0.1, batch_size=16)
    base.update(kw)
    return trainer.TrainConfig(**base)


def test_sgd_matches_reference_rounding():
    w = torch.full((3, 3), 1.0, device="cuda")
    trainer.sgd_step(w, torch.full((3, 3), 1.0, device="cuda"), 0.1)
    assert float(w[0, 0]) == float(np.float32(1.0) - np.float32(0.1) * np.float32(1.0))
    w0 = torch.ones(3, 3, device="cuda")
    trainer.sgd_step(w0, torch.full((3, 3), 7.0, device="cuda"), 0.0)
    assert torch.equal(w0, torch.ones(3, 3, device="cuda"))


def test_clip_gradients_global_norm():
    g = [torch.full((2, 2), 3.0, device="cuda"), torch.full((1, 4), 4.0, device="cuda")]
    out = trainer.clip_gradients(g, 1.0)
    norm = np.sqrt(4 * 9 + 4 * 16)
    assert torch.allclose(out[0], torch.full((2, 2), 3.0 * float(np.float32(1.0 / norm)),
                                             device="cuda"))
    assert trainer.clip_gradients(g, 100.0) is g


def test_dense_anchor_bitwise():
    sched = SparsitySchedule(0.0, 0.0, 30, 0, 5)
    log_m, _ = trainer.train(config(schedule=sched, sparsify=True))
    log_f, _ = trainer.train(config(schedule=sched, sparsify=False))
    assert [r.loss for r in log_m.records] == [r.loss for r in log_f.records]


def test_refresh_iterations_flagged():
    log, _ = trainer.train(config(schedule=SparsitySchedule(0.0, 0.5, 22, 0, 7)))
    assert [r.iteration for r in log.records if r.refresh] == [0, 7, 14, 21]


def test_masked_blocks_zero_after_step_and_apply():
    cfg = config(schedule=SparsitySchedule(0.5, 0.5, 12, 0, 3))
    _, stack = trainer.train(cfg)
    b = cfg.block_size
    for blk, ok in zip(stack.blocks, stack.sparsifiable):
        for mat in blk.matrices():
            inactive = ~mat.mask.active
            if bool(inactive.any()):
                sel = bs.expand_mask(inactive, b, *mat.dense.shape)
                assert bool((mat.dense[sel] == 0).all())


def test_dense_layer_exemption_and_reports():
    cfg = config(layers=3, dense_layers=1, schedule=SparsitySchedule(0.3, 0.6, 30, 0, 5))
    log, stack = trainer.train(cfg)
    assert stack.sparsifiable == [True, True, False]
    final = log.records[-1].layer_sparsity
    assert final[2] == 0.0 and final[0] > 0.0 and final[1] > 0.0
    for mat in stack.blocks[2].matrices():
        assert mat.cache.nnzb == mat.mask.kept.numel()
    assert log.prune_reports
    for rep in log.prune_reports:
        assert 0.0 <= rep.regrown_ratio <= 1.0 and 0.0 <= rep.s_achieved <= 1.0


def test_flops_step_down_across_refresh():
    log, _ = trainer.train(config(schedule=SparsitySchedule(0.0, 0.8, 60, 0, 15)))
    per_iter = [log.records[0].flops_cum] + [b.flops_cum - a.flops_cum
                                             for a, b in zip(log.records, log.records[1:])]
    assert all(b <= a for a, b in zip(per_iter, per_iter[1:])) and per_iter[-1] < per_iter[0]


def test_divergence_raises():
    with pytest.raises(trainer.DivergenceError, match="diverged"):
        trainer.train(config(lr=1e4, schedule=SparsitySchedule(0.0, 0.0, 200, 0, 10)))


def test_loss_decreases_regression_and_bf16():
    for dt in ("float32", "bfloat16"):
        cfg = config(schedule=SparsitySchedule(0.0, 0.5, 200, 50, 20), dtype=dt, batch_size=64,
                     embed_dim=32, hidden_dim=64, block_size=16)
        log, _ = trainer.train(cfg)
        first = np.mean([r.loss for r in log.records[:20]])
        last = np.mean([r.loss for r in log.records[-20:]])
        assert np.isfinite(last) and last < first


def test_save_model_bytes(tmp_path):
    _, stack = trainer.train(config(schedule=SparsitySchedule(0.0, 0.5, 6, 0, 3)))
    names = trainer.save_model(stack, tmp_path)
    assert len(names) == 6
    w = bs.load(tmp_path / names[0])
    h = stack.blocks[0].gate.cache.to_host()
    np.testing.assert_array_equal(w.to_host().values, h.values)


@pytest.mark.parametrize("name", ["reg", "reg_dense", "cls"])
def test_train_matches_reference_train(name, monkeypatch):
    from conftest import golden
    d = golden("trainer")
    raw = json.loads(bytes(d[f"{name}_config"]).decode())
    calls = []
    orig = trainer.generate_masks

    def rec(w, g, b, s, iteration=0):
        mask, rep = orig(w, g, b, s, iteration=iteration)
        calls.append((mask, rep, s))
        return mask, rep

    monkeypatch.setattr(trainer, "generate_masks", rec)
    log, stack = trainer.train(trainer.TrainConfig.from_dict(raw))
    assert [r.refresh for r in log.records] == d[f"{name}_refresh"].tolist()
    assert [r.flops_cum for r in log.records] == d[f"{name}_flops"].tolist()
    loss = np.array([r.loss for r in log.records])
    np.testing.assert_allclose(loss, d[f"{name}_loss"], rtol=1e-4, atol=0)
    np.testing.assert_allclose(np.array([r.layer_sparsity for r in log.records]),
                               d[f"{name}_sparsity"], rtol=0, atol=1e-12)
    assert len(calls) == int(d[f"{name}_n_calls"])
    for k, (mask, rep, s) in enumerate(calls):
        kept = mask.kept.cpu().numpy() if hasattr(mask.kept, "cpu") else np.asarray(mask.kept)
        reg = mask.regrown.cpu().numpy() if hasattr(mask.regrown, "cpu") else np.asarray(mask.regrown)
        np.testing.assert_array_equal(kept, d[f"{name}_call{k}_kept"], err_msg=f"call {k} kept")
        np.testing.assert_array_equal(reg, d[f"{name}_call{k}_regrown"], err_msg=f"call {k} regrown")
        assert [rep.kept, rep.regrown, rep.iteration] == d[f"{name}_call{k}_counts"].tolist()
        assert s == float(d[f"{name}_call{k}_s"])
    for li, blk in enumerate(stack.blocks):
        for tag, mat in zip(("gate", "up", "down"), blk.matrices()):
            ref = d[f"{name}_final_l{li}_{tag}"]
            got = mat.dense.cpu().numpy()
            assert np.array_equal(got == 0, ref == 0), f"layer {li} {tag}: zero pattern"
            err = np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30)
            assert err <= 1e-4, f"layer {li} {tag}: master max-norm-relative {err:.2e}"
