"""Pin the CPU oracle (oracle/ref_numpy.py) to outputs of the real reference
package (tests/golden/*.npz, produced by tests/golden/make_golden.py).

Integer / index / mask outputs must match exactly; floating outputs to within
a few float32 ulps (the fixtures may come from a different BLAS build)."""
import numpy as np
import pytest

import oracle
from conftest import golden, golden_bcsc


def assert_bcsc_equal(got: oracle.Bcsc, ref: oracle.Bcsc, exact_values=True):
    assert (got.rows, got.cols, got.block) == (ref.rows, ref.cols, ref.block)
    np.testing.assert_array_equal(got.col_ptr, ref.col_ptr)
    assert got.col_ptr.dtype == np.int64
    np.testing.assert_array_equal(got.block_row_idx, ref.block_row_idx)
    assert got.block_row_idx.dtype == np.uint32
    if exact_values:
        np.testing.assert_array_equal(got.values.view(np.uint32), ref.values.view(np.uint32))


class TestProducts:
    d = golden("products")

    @pytest.mark.parametrize("i", range(15))
    def test_bspmm_case(self, i):
        d = self.d
        w = golden_bcsc(d, f"c{i}_w")
        x, xt = d[f"c{i}_x"], d[f"c{i}_xt"]
        np.testing.assert_allclose(oracle.bspmm(x, w), d[f"c{i}_y"], rtol=2e-6, atol=2e-6)
        np.testing.assert_allclose(oracle.bspmm_rt(xt, w), d[f"c{i}_yt"], rtol=2e-6, atol=2e-6)
        for f in ("relu", "gelu", "silu"):
            np.testing.assert_allclose(oracle.bspmm_fused(x, w, f), d[f"c{i}_y_{f}"],
                                       rtol=2e-6, atol=2e-6)
        np.testing.assert_array_equal(oracle.dense_of(w), d[f"c{i}_dense"])

    def test_random_bcsc_stream(self):
        # same generator stream as bench.random_bcsc (bench.py:50-72)
        cases = self.d["cases"]
        for i, (m, k, n, b, s, seed) in enumerate(cases):
            rng = np.random.default_rng(int(seed))
            w = oracle.random_bcsc(int(k), int(n), int(b), float(s), rng)
            ref = golden_bcsc(self.d, f"c{i}_w")
            np.testing.assert_array_equal(w.col_ptr, ref.col_ptr)
            np.testing.assert_array_equal(w.block_row_idx, ref.block_row_idx)
            scaled = w.values * np.float32(1.0 / np.sqrt(k))
            np.testing.assert_array_equal(scaled, ref.values)


class TestMlp:
    d = golden("mlp")

    @pytest.mark.parametrize("i", range(5))
    def test_forward_backward(self, i):
        d = self.d
        mats = [golden_bcsc(d, f"c{i}_{n}") for n in ("gate", "up", "down")]
        y, acts = oracle.mlp_forward(d[f"c{i}_x"], *mats)
        np.testing.assert_allclose(y, d[f"c{i}_y"], rtol=1e-5, atol=1e-6)
        for got, key in zip(acts[1:], ("a", "b", "g")):
            np.testing.assert_allclose(got, d[f"c{i}_{key}"], rtol=1e-5, atol=1e-6)
        dx, dwg, dwu, dwd = oracle.mlp_backward(d[f"c{i}_dy"], acts, *mats)
        for got, key in ((dx, "dx"), (dwg, "dwg"), (dwu, "dwu"), (dwd, "dwd")):
            assert oracle.rel_err(got, d[f"c{i}_{key}"]) <= 1e-5, key

    @pytest.mark.parametrize("i", range(5))
    def test_masks_and_caches(self, i):
        d = self.d
        for n in ("gate", "up", "down"):
            mask = oracle.Mask(d[f"c{i}_{n}_kept"], d[f"c{i}_{n}_regrown"])
            w = oracle.from_dense(d[f"c{i}_{n}_dense"], golden_bcsc(d, f"c{i}_{n}").block, mask)
            assert_bcsc_equal(w, golden_bcsc(d, f"c{i}_{n}"))

    def test_init_stream(self):
        # SparseMlp.create draws gate, up, down in order (mlp.py:61-68)
        d = self.d
        e, h, b, s, m, seed = d["cases"][3]
        wg, wu, wd = oracle.mlp_init(int(e), int(h), np.random.default_rng(int(seed)))
        np.testing.assert_array_equal(wg, d["c3_gate_dense"])
        np.testing.assert_array_equal(wu, d["c3_up_dense"])
        np.testing.assert_array_equal(wd, d["c3_down_dense"])


class TestPrune:
    d = golden("prune")

    def test_cases(self):
        d = self.d
        for i in range(int(d["n"])):
            w, g = d[f"c{i}_w"], d[f"c{i}_g"]
            b, s = int(d[f"c{i}_bs"][0]), float(d[f"c{i}_bs"][1])
            nw = oracle.block_norms(w, b)
            np.testing.assert_allclose(nw, d[f"c{i}_nw"], rtol=1e-14, equal_nan=True)
            np.testing.assert_array_equal(oracle.prune_s(d[f"c{i}_nw"], s), d[f"c{i}_keep"])
            mask, rep = oracle.generate_masks(w, g, b, s)
            np.testing.assert_array_equal(mask.kept, d[f"c{i}_kept"])
            np.testing.assert_array_equal(mask.regrown, d[f"c{i}_regrown"])
            np.testing.assert_array_equal(np.array(rep), d[f"c{i}_report"])
            for zr, tag in ((True, "z"), (False, "nz")):
                masked, cache = oracle.apply_mask(w, mask, b, zero_regrown=zr)
                np.testing.assert_array_equal(masked.view(np.uint32),
                                              d[f"c{i}_{tag}_masked"].view(np.uint32))
                assert_bcsc_equal(cache, golden_bcsc(d, f"c{i}_{tag}"))

    def test_prune_s_ties_nan(self):
        d = self.d
        for j in range(int(d["n_prune_s"])):
            np.testing.assert_array_equal(oracle.prune_s(d[f"p{j}_norms"], float(d[f"p{j}_s"])),
                                          d[f"p{j}_keep"])


class TestFormat:
    d = golden("format")

    def test_from_dense(self):
        d = self.d
        for i in range(int(d["n"])):
            dense, b = d[f"c{i}_dense"], int(d[f"c{i}_b"])
            assert_bcsc_equal(oracle.from_dense(dense, b), golden_bcsc(d, f"c{i}_auto"))
            m = oracle.Mask(d[f"c{i}_kept"], d[f"c{i}_regrown"])
            assert_bcsc_equal(oracle.from_dense(dense, b, m), golden_bcsc(d, f"c{i}_mask"))

    def test_schedule(self):
        for s_init, s_max, mt, dc, i, val in self.d["schedule"]:
            assert oracle.target_sparsity(int(i), s_init, s_max, int(mt), int(dc)) == val


def test_known_answers():
    # tests/test_kernels.py:160-161, :177-181, :197-200; tests/test_pruner.py:25-27
    assert abs(oracle.silu(np.array([1.0]))[0] - 0.7310585786300049) < 1e-12
    assert abs(oracle.gelu(np.array([1.0]))[0] - 0.841192) < 1e-5
    assert oracle.flops(1024, 4096, 1024, 16, 128)[1] == 536_870_912
    assert abs(oracle.target_sparsity(5000, 0.0, 0.8, 10000, 0) - 0.7) < 1e-12
    keep = oracle.prune_s(np.ones((2, 3)), 0.5)
    np.testing.assert_array_equal(keep, [[True, True, False], [True, False, False]])
