"""Engine modes (read once per process from the environment) give bitwise the same MLP
forward as the default engine: the interleaved gate+up layout (default: sequential), round-robin
items instead of the cost-balanced schedule, and the narrow-tile / direct-store fallbacks. Each
mode runs in a subprocess."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent

SCRIPT = r"""
import sys
sys.path.insert(0, {root!r})
import numpy as np, torch
import oracle
import paper_2507_03117_b200 as bs
rng = np.random.default_rng(5)
mats = []
for rows, cols in ((1024, 3072), (1024, 3072), (3072, 1024)):
    w = oracle.random_bcsc(rows, cols, 64, 0.85, rng)
    w = w._replace(values=(w.values / np.sqrt(rows)).astype(np.float32))
    mats.append(bs.from_host(w, torch.bfloat16))
net = bs.SparseMlp.from_caches(*mats)
x = torch.from_numpy(rng.standard_normal(({m}, 1024)).astype(np.float32)).cuda().bfloat16()
y, _ = bs.mlp_forward(x, net, save_activations=False)
y2, acts = bs.mlp_forward(x, net, save_activations=True)
torch.cuda.synchronize()
np.save({out!r}, torch.stack([y.float(), y2.float()]).cpu().numpy())
"""

MODES = {
    "default": {},
    "interleaved": {"BLAST_SPLIT_STAGES": "0"},
    "round_robin": {"BLAST_SCHEDULE": "0"},
    "narrow": {"BLAST_WIDE_TILES": "0"},
    "direct": {"BLAST_DIRECT_STORES": "1"},
}


def run_mode(env_extra, m, tmp_path, name):
    out = str(tmp_path / f"{name}_{m}.npy")
    env = dict(os.environ, **env_extra)
    code = SCRIPT.format(root=str(ROOT), m=m, out=out)
    res = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    return np.load(out)


@pytest.mark.parametrize("m", [1000, 4096])
def test_modes_bitwise_equal(m, tmp_path):
    ref = run_mode(MODES["default"], m, tmp_path, "default")
    for name, env in MODES.items():
        if name == "default":
            continue
        got = run_mode(env, m, tmp_path, name)
        assert np.array_equal(got, ref), name


SCRIPT_B = r"""
import sys
sys.path.insert(0, {root!r})
import numpy as np, torch
import oracle
import paper_2507_03117_b200 as bs
rng = np.random.default_rng(7)
mats = []
for rows, cols in ((1024, 2048), (1024, 2048), (2048, 1024)):
    w = oracle.random_bcsc(rows, cols, {b}, {sp}, rng)
    w = w._replace(values=(w.values / np.sqrt(rows)).astype(np.float32))
    mats.append(bs.from_host(w, torch.bfloat16))
net = bs.SparseMlp.from_caches(*mats)
x = torch.from_numpy(rng.standard_normal((777, 1024)).astype(np.float32)).cuda().bfloat16()
y, _ = bs.mlp_forward(x, net, save_activations=False)
torch.cuda.synchronize()
np.save({out!r}, y.float().cpu().numpy())
"""


@pytest.mark.parametrize("b,sp", [(128, 0.9), (64, 0.5), (64, 0.7), (32, 0.9)])
def test_gate_up_layouts_bitwise_equal(b, sp, tmp_path):
    """The default picks the sequential or interleaved gate+up layout by block size and
    density (csrc/spmm.cu seq_gate_up_pays); both give the same bits."""
    outs = []
    for name, env in (("default", {}), ("interleaved", {"BLAST_SPLIT_STAGES": "0"}),
                      ("sequential", {"BLAST_SPLIT_STAGES": "2"})):
        out = str(tmp_path / f"{name}.npy")
        res = subprocess.run([sys.executable, "-c", SCRIPT_B.format(root=str(ROOT), b=b, sp=sp, out=out)],
                             env=dict(os.environ, **env), capture_output=True, text=True, timeout=600)
        assert res.returncode == 0, res.stderr[-2000:]
        outs.append(np.load(out))
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


SCRIPT_BWD = r"""
import sys
sys.path.insert(0, {root!r})
import numpy as np, torch
import oracle
import paper_2507_03117_b200 as bs
rng = np.random.default_rng(11)
mats = []
for rows, cols in ((1024, 4096), (1024, 4096), (4096, 1024)):
    w = oracle.random_bcsc(rows, cols, 64, 0.6, rng)
    w = w._replace(values=(w.values / np.sqrt(rows)).astype(np.float32))
    mats.append(bs.from_host(w, torch.bfloat16))
net = bs.SparseMlp.from_caches(*mats)
x = torch.from_numpy(rng.standard_normal(({m}, 1024)).astype(np.float32)).cuda().bfloat16()
dy = torch.from_numpy(rng.standard_normal(({m}, 1024)).astype(np.float32)).cuda().bfloat16()
y, acts = bs.mlp_forward(x, net, save_activations=True)
g = bs.mlp_backward(dy, acts, net, grad_mode="active")
torch.cuda.synchronize()
np.savez({out!r}, y=y.float().cpu().numpy(), a=acts.gate_pre.float().cpu().numpy(),
         dx=g[0].float().cpu().numpy(), dwg=g[1].cpu().numpy(), dwu=g[2].cpu().numpy(),
         dwd=g[3].cpu().numpy())
"""

MODES_BWD = {
    "default": {},
    "narrow_gating_backward": {"BLAST_WIDE_BWD2": "0"},
    "round_robin_training_forward": {"BLAST_LPT_SAVE": "0"},
    "wgrad_unit_by_unit": {"BLAST_WG_SWEEP": "0"},
    "no_pdl": {"BLAST_PDL": "0"},
}


@pytest.mark.parametrize("m", [640, 3000])
def test_training_modes_bitwise_equal(m, tmp_path):
    """Training forward + backward (mlp.py:102-143): the 256-token gating backward, the LPT
    schedule of the G/a/b-writing gate+up, the weight-gradient sweep mode and programmatic
    dependent launch change no bit of Y, the saved activations, dX or the stored-block dW."""
    def run(env_extra, name):
        out = str(tmp_path / f"bwd_{name}_{m}.npz")
        env = dict(os.environ, **env_extra)
        res = subprocess.run([sys.executable, "-c", SCRIPT_BWD.format(root=str(ROOT), m=m, out=out)],
                             env=env, capture_output=True, text=True, timeout=600)
        assert res.returncode == 0, res.stderr[-2000:]
        return np.load(out)
    ref = run(MODES_BWD["default"], "default")
    for name, env in MODES_BWD.items():
        if name == "default":
            continue
        got = run(env, name)
        for k in ref.files:
            assert np.array_equal(got[k], ref[k]), (name, k)
