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
