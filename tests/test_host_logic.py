"""Host-side logic of the package (no GPU): the schedule and FLOP accounting against the
reference's golden values, the trainer's config parsing, and its toy-task data streams
against batches recorded from the real reference (tests/golden/make_golden.py)."""
import json

import numpy as np
import pytest

from conftest import golden

bs = pytest.importorskip("paper_2507_03117_b200")
from paper_2507_03117_b200 import kernels, pruner, trainer  # noqa: E402


def test_target_sparsity_matches_reference_golden():
    # pruner.py:53-67 evaluated by the reference on 50 (schedule, iteration) points
    for s_init, s_max, total, decay, i, val in golden("format")["schedule"]:
        sched = pruner.SparsitySchedule(float(s_init), float(s_max), int(total), int(decay), 1)
        assert pruner.target_sparsity(int(i), sched) == val
        assert sched.target(int(i)) == val


def test_schedule_known_answer_and_errors():
    # tests/test_pruner.py:25-27 and the validation of pruner.py:37-47
    assert abs(pruner.target_sparsity(5000, pruner.SparsitySchedule(0.0, 0.8, 10000, 0, 1))
               - 0.7) < 1e-12
    for bad in [dict(initial_sparsity=1.0), dict(max_sparsity=1.5),
                dict(initial_sparsity=0.5, max_sparsity=0.4), dict(decay_iters=5, total_iters=5),
                dict(step_size=0)]:
        with pytest.raises(ValueError):
            pruner.SparsitySchedule(**bad)


def test_flops_known_answer():
    # tests/test_kernels.py:197-200 worked value; kernels.py:173-179
    dense, sparse = kernels.flops(1024, 4096, 1024, 16, 128)
    assert sparse == 536_870_912 and dense == 2 * 1024 * 4096 * 1024
    assert kernels.flops(3, 5, 7, 0, 4) == (210, 0)


@pytest.mark.parametrize("name", ["reg", "reg_dense", "cls"])
def test_train_config_and_task_stream(name):
    d = golden("trainer")
    raw = json.loads(bytes(d[f"{name}_config"]).decode())
    cfg = trainer.TrainConfig.from_dict(raw)
    assert cfg.schedule.step_size == raw["schedule"]["step_size"]
    task = trainer.make_task(cfg)
    for k in range(2):
        got = task.next_batch(cfg.batch_size)
        for j, arr in enumerate(got):
            np.testing.assert_array_equal(arr, d[f"{name}_batch{k}_{j}"])


def test_train_config_rejects_unknown_fields():
    with pytest.raises(ValueError, match="bad config field"):
        trainer.TrainConfig.from_dict({"no_such_field": 1})
    with pytest.raises(ValueError, match="bad schedule field"):
        trainer.TrainConfig.from_dict({"schedule": {"bogus": 2}})
    with pytest.raises(ValueError, match="schedule"):
        trainer.TrainConfig.from_dict({"schedule": 3})


GOLDEN_DIR = __import__("pathlib").Path(__file__).resolve().parent / "golden"


def test_dense_file_bytes_match_reference(tmp_path):
    # bcsc.py:292-314: c1.dnse was written by the reference's write_dense_file
    d = golden("format")
    ref = (GOLDEN_DIR / "c1.dnse").read_bytes()
    from paper_2507_03117_b200 import bcsc
    out = tmp_path / "c1.dnse"
    bcsc.write_dense_file(d["c1_dense"], out)
    assert out.read_bytes() == ref
    np.testing.assert_array_equal(bcsc.read_dense_file(GOLDEN_DIR / "c1.dnse"), d["c1_dense"])


def test_dense_file_errors(tmp_path):
    from paper_2507_03117_b200 import bcsc
    with pytest.raises(ValueError, match="2-D"):
        bcsc.write_dense_file(np.zeros(3, np.float32), tmp_path / "x")
    good = (GOLDEN_DIR / "c1.dnse").read_bytes()
    for name, data, msg in [("short", good[:8], "incomplete dense header"),
                            ("magic", b"XXXX" + good[4:], "bad magic"),
                            ("size", good + b"\0", "size mismatch")]:
        f = tmp_path / name
        f.write_bytes(data)
        with pytest.raises(bcsc.FormatError, match=msg):
            bcsc.read_dense_file(f)
    f = tmp_path / "other"
    f.write_bytes(b"ABCD" + good[4:])
    with pytest.raises(bcsc.FormatError, match="unrecognized magic"):
        bcsc.convert(f, tmp_path / "out", 4)
