"""bench.py's multi-GPU launcher on CPU: `--gpus N` without WORLD_SIZE re-launches itself with
N ranks (torch.distributed.run, gloo in --dry-run), and rank 0's line reports n_gpus = N;
N = 1 stays a single process."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def run(*args):
    env = {k: v for k, v in __import__("os").environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True,
                         text=True, timeout=300, env=env, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("n", [1, 2])
def test_gpus_flag_spawns_ranks(n):
    line = run("--gpus", str(n), "--dry-run", "--steps", "3", "--warmup", "3")
    assert line["n_gpus"] == n
    assert line["dry_run"] is True


def test_world_size_must_match_gpus():
    env_ok = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run"],
                            capture_output=True, text=True, timeout=120, cwd=ROOT,
                            env={**__import__("os").environ, "WORLD_SIZE": "1", "RANK": "0"})
    assert env_ok.returncode != 0 and "WORLD_SIZE" in (env_ok.stderr + env_ok.stdout)


def test_l2_feed_roof_counts_panel_and_block_bytes():
    """The bench line's L2-feed roof: every stored block reads its 256-token activation panel
    and the block itself (cfg3: 5.64 GB per 8192-token step, the ncu xbar2l1tex bytes)."""
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    import bench
    ws = bench.make_weights(4096, 14336, 64, 0.9, 0)
    r = bench.l2_feed_roof(ws, 8192, 0.34)
    nnzb = sum(len(w.block_row_idx) for w in ws)
    assert nnzb == 3 * 1434
    assert r["bytes_per_step"] == nnzb * 32 * (256 * 64 * 2 + 64 * 64 * 2) == 5638717440
    assert abs(r["ms_at_peak"] - 5638717440 / 17.96e12 * 1e3) < 1e-9
    assert abs(r["frac"] - r["ms_at_peak"] / 0.34) < 1e-12
