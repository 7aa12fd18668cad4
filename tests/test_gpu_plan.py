"""Engine work plans (csrc/plan.cu) against a numpy restatement: per line, the steps are the
inner indices holding a block of either matrix, in order, as {inner, k0, k1, bits}; bits
0/1 = block of matrix 0/1 present, bits 2/3 = first block of matrix 0/1 in the line. The
per-line flags carry presence (bits 0/1) and the block count of each matrix (bits 2..16,
17..31), which the sequential gate+up mode uses as its MMA recipe."""
import numpy as np
import pytest
import torch

from paper_2507_03117_b200 import bcsc

pytestmark = pytest.mark.gpu


def expected(k0, k1, by_rows):
    gr, gc = k0.shape
    lines, inner = (gr, gc) if by_rows else (gc, gr)
    ptr, steps, flags = [0], [], []
    for line in range(lines):
        seen0 = seen1 = False
        n0 = n1 = 0
        for i in range(inner):
            a = k0[line, i] if by_rows else k0[i, line]
            b = (k1[line, i] if by_rows else k1[i, line]) if k1 is not None else -1
            if a < 0 and b < 0:
                continue
            w = (int(a >= 0) | (int(b >= 0) << 1) | (int(a >= 0 and not seen0) << 2) |
                 (int(b >= 0 and not seen1) << 3))
            steps.append((i, int(a), int(b), w))
            seen0 |= a >= 0
            seen1 |= b >= 0
            n0 += a >= 0
            n1 += b >= 0
        ptr.append(len(steps))
        flags.append(int(seen0) | (int(seen1) << 1) | (n0 << 2) | (n1 << 17))
    return np.array(ptr), np.array(steps, dtype=np.int64).reshape(-1, 4), np.array(flags)


def kmap(rng, gr, gc, density):
    m = rng.random((gr, gc)) < density
    k = np.full((gr, gc), -1, np.int32)
    k[m] = rng.permutation(int(m.sum())).astype(np.int32)
    return k


@pytest.mark.parametrize("by_rows", [0, 1])
@pytest.mark.parametrize("gr,gc,density,two", [(100, 7, 0.3, True), (5, 90, 0.2, True),
                                                (64, 64, 0.1, False), (33, 3, 0.0, True),
                                                (40, 40, 1.0, True)])
def test_plan_matches_numpy(gr, gc, density, two, by_rows):
    rng = np.random.default_rng(gr * 1000 + gc)
    k0 = kmap(rng, gr, gc, density)
    k1 = kmap(rng, gr, gc, density * 0.7) if two else None
    ptr, steps, flags = bcsc.build_plan(torch.from_numpy(k0).cuda(),
                                        torch.from_numpy(k1).cuda() if two else None,
                                        gr, gc, by_rows)
    torch.cuda.synchronize()
    eptr, esteps, eflags = expected(k0, k1, by_rows)
    got_ptr = ptr.cpu().numpy()
    assert np.array_equal(got_ptr, eptr)
    n = int(eptr[-1])
    got = steps.cpu().numpy()[: 4 * n].reshape(-1, 4).astype(np.int64)
    assert np.array_equal(got, esteps)
    assert np.array_equal(flags.cpu().numpy().astype(np.int64), eflags)


def lpt_reference(costs, n_tiles, grid):
    """numpy restatement of csrc/schedule.cu: t-major sequence with each tile's lines in
    descending cost (ties by index); batches of `grid` items, the k-th largest item of a batch
    (ties by sequence position) to the k-th least loaded CTA (ties by CTA index)."""
    L = len(costs)
    order = sorted(range(L), key=lambda j: (-costs[j], j))
    total = n_tiles * L
    rows = -(-total // grid)
    out = -np.ones((rows, grid), np.int64)
    load = np.zeros(grid, np.int64)
    for r in range(rows):
        pos = list(range(r * grid, min(total, (r + 1) * grid)))
        items = sorted(pos, key=lambda p: (-costs[order[p % L]], p - r * grid))
        ctas = sorted(range(grid), key=lambda c: (load[c], c))
        for k, p in enumerate(items):
            j = order[p % L]
            out[r, ctas[k]] = (p // L) * L + j
            load[ctas[k]] += costs[j]
    return out


@pytest.mark.parametrize("gr,gc,density,n_tiles,grid,seq",
                         [(64, 64, 0.1, 32, 148, 0), (64, 224, 0.1, 32, 148, 1),
                          (12, 48, 0.3, 5, 148, 0), (8, 8, 0.5, 3, 7, 1),
                          (4, 5, 0.5, 50, 37, 0), (64, 1000, 0.1, 3, 148, 1)])
def test_balanced_schedule(gr, gc, density, n_tiles, grid, seq):
    from paper_2507_03117_b200 import _lib as L
    rng = np.random.default_rng(gr * gc + n_tiles)
    k0, k1 = kmap(rng, gr, gc, density), kmap(rng, gr, gc, density)
    step_ptr, steps, flags = bcsc.build_plan(torch.from_numpy(k0).cuda(),
                                            torch.from_numpy(k1).cuda() if seq else None,
                                            gr, gc, 0)
    rows = -(-n_tiles * gc // grid)
    out = torch.full((rows * grid,), -7, dtype=torch.int32, device="cuda")
    L.check(L.load().blast_balanced_schedule(step_ptr.data_ptr(), flags.data_ptr(), gc, n_tiles,
                                             grid, seq, out.data_ptr(), L.stream()), "schedule")
    got = out.cpu().numpy().reshape(rows, grid)
    sp, fl = step_ptr.cpu().numpy(), flags.cpu().numpy()
    stages = ((fl >> 2) & 0x7fff) + ((fl >> 17) & 0x7fff) if seq else np.diff(sp)
    costs = [int(4 * s + 3) for s in stages[:gc]]
    # every item exactly once: the schedule is a permutation (results are order-independent)
    items = got[got >= 0]
    assert np.array_equal(np.sort(items), np.arange(n_tiles * gc))
    assert np.array_equal(got, lpt_reference(costs, n_tiles, grid))
    # balance: no CTA above the mean by more than one item
    load = np.zeros(grid)
    for c in range(grid):
        load[c] = sum(costs[i % gc] for i in got[:, c] if i >= 0)
    assert load.max() - load.mean() <= max(costs) + 1e-9
