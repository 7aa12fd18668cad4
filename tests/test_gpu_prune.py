"""GPU prune-and-grow: masks, BSR/BCSC indices and values bit-exact vs the
reference (golden vectors) and the oracle; ports of tests/test_pruner.py and
tests/test_bcsc.py, plus full-size (Llama-3-8B / 70B MLP grid) properties."""
import numpy as np
import pytest
import torch

import oracle
from conftest import golden, golden_bcsc

pytestmark = pytest.mark.gpu
bs = pytest.importorskip("paper_2507_03117_b200")


def assert_bits_equal(got, ref):
    """Bitwise float32 equality (so -0.0 != +0.0) with NaN == NaN: the NaN bit
    pattern of w * 0 is platform-defined (x86 returns 0xffc00000, the GPU 0x7fffffff)."""
    got, ref = np.asarray(got, np.float32), np.asarray(ref, np.float32)
    np.testing.assert_array_equal(np.isnan(got), np.isnan(ref))
    ok = ~np.isnan(ref)
    np.testing.assert_array_equal(got[ok].view(np.uint32), ref[ok].view(np.uint32))


def assert_cache_equal(cache, ref: oracle.Bcsc):
    h = cache.to_host()
    assert (h.rows, h.cols, h.block) == (ref.rows, ref.cols, ref.block)
    np.testing.assert_array_equal(h.col_ptr, ref.col_ptr)
    np.testing.assert_array_equal(h.block_row_idx, ref.block_row_idx)
    assert_bits_equal(h.values, ref.values)


class TestGoldenPrune:
    d = golden("prune")

    def test_all_cases(self):
        d = self.d
        for i in range(int(d["n"])):
            w, g = d[f"c{i}_w"], d[f"c{i}_g"]
            b, s = int(d[f"c{i}_bs"][0]), float(d[f"c{i}_bs"][1])
            nw = bs.block_norms(w, b)
            np.testing.assert_allclose(nw, d[f"c{i}_nw"], rtol=1e-14, atol=0, equal_nan=True)
            np.testing.assert_array_equal(bs.prune_s(d[f"c{i}_nw"], s), d[f"c{i}_keep"])
            mask, rep = bs.generate_masks(w, g, b, s)
            np.testing.assert_array_equal(mask.kept, d[f"c{i}_kept"])
            np.testing.assert_array_equal(mask.regrown, d[f"c{i}_regrown"])
            assert [rep.kept, rep.regrown, rep.regrown_ratio, rep.s_achieved] == \
                list(d[f"c{i}_report"])
            for zr, tag in ((True, "z"), (False, "nz")):
                masked, cache = bs.apply_mask(w, mask, b, zero_regrown=zr)
                assert_bits_equal(masked, d[f"c{i}_{tag}_masked"])
                assert_cache_equal(cache, golden_bcsc(d, f"c{i}_{tag}"))

    def test_prune_s_ties_and_nan(self):
        d = self.d
        for j in range(int(d["n_prune_s"])):
            np.testing.assert_array_equal(bs.prune_s(d[f"p{j}_norms"], float(d[f"p{j}_s"])),
                                          d[f"p{j}_keep"])


class TestGoldenFormat:
    d = golden("format")

    def test_from_dense_and_serialize(self):
        d = self.d
        for i in range(int(d["n"])):
            dense, b = d[f"c{i}_dense"], int(d[f"c{i}_b"])
            assert_cache_equal(bs.from_dense(dense, b), golden_bcsc(d, f"c{i}_auto"))
            m = bs.BlockMask(kept=d[f"c{i}_kept"], regrown=d[f"c{i}_regrown"])
            w = bs.from_dense(dense, b, m)
            assert_cache_equal(w, golden_bcsc(d, f"c{i}_mask"))
            assert bs.serialize(w) == d[f"c{i}_bytes"].tobytes()
            w2 = bs.deserialize(d[f"c{i}_bytes"].tobytes())
            assert_cache_equal(w2, golden_bcsc(d, f"c{i}_mask"))

    def test_convert_matches_reference_files(self, tmp_path):
        # cli.py:231-247 (convert): DNSE -> BCSC bytes identical to the file the reference
        # wrote for the same input (tests/golden/make_dense_files.py), and back to DNSE
        from pathlib import Path
        gdir = Path(__file__).resolve().parent / "golden"
        d = self.d
        w = bs.convert(gdir / "c1.dnse", tmp_path / "c1.bcsc", int(d["c1_b"]))
        assert (tmp_path / "c1.bcsc").read_bytes() == (gdir / "c1.bcsc").read_bytes()
        assert_cache_equal(w, golden_bcsc(d, "c1_auto"))
        bs.convert(tmp_path / "c1.bcsc", tmp_path / "back.dnse")
        assert (tmp_path / "back.dnse").read_bytes() == (gdir / "c1_back.dnse").read_bytes()


class TestPruneS:
    def test_count_exactness(self):
        rng = np.random.default_rng(1)
        for _ in range(100):
            gr, gc = int(rng.integers(1, 17)), int(rng.integers(1, 17))
            s = float(rng.random())
            keep = bs.prune_s(rng.random((gr, gc)), s)
            assert keep.sum() == int(np.floor((1.0 - s) * gr * gc + 0.5))

    def test_matches_sort_oracle_duplicates(self):
        rng = np.random.default_rng(3)
        for _ in range(100):
            gr, gc = int(rng.integers(1, 13)), int(rng.integers(1, 13))
            norms = rng.integers(0, 4, size=(gr, gc)).astype(np.float64)
            s = float(rng.random())
            np.testing.assert_array_equal(bs.prune_s(norms, s), oracle.prune_s(norms, s))

    def test_scale_invariance(self):
        rng = np.random.default_rng(2)
        norms = rng.random((6, 6))
        base = bs.prune_s(norms, 0.4)
        for alpha in (1e-6, 0.5, 3.0, 1e6):
            np.testing.assert_array_equal(bs.prune_s(alpha * norms, 0.4), base)

    def test_special_values(self):
        norms = np.array([[np.inf, 0.0, -0.0, np.nan], [1.0, np.nan, 2.0, 0.0]])
        for s in np.linspace(0, 1, 9):
            np.testing.assert_array_equal(bs.prune_s(norms, s), oracle.prune_s(norms, s))

    def test_invalid_sparsity(self):
        with pytest.raises(ValueError, match="sparsity"):
            bs.prune_s(np.ones((2, 2)), 1.5)

    @pytest.mark.parametrize("gr,gc", [(64, 224), (224, 64), (128, 448), (512, 1792)])
    @pytest.mark.parametrize("s", [0.5, 0.9, 0.95])
    def test_large_grids_match_oracle(self, gr, gc, s):
        rng = np.random.default_rng(gr + gc)
        norms = rng.random((gr, gc))
        norms[rng.random((gr, gc)) < 0.05] = 0.5  # exact ties
        np.testing.assert_array_equal(bs.prune_s(norms, s), oracle.prune_s(norms, s))


class TestFullSizeMasks:
    """Llama-3-8B and Llama-3-70B MLP gate grids at b = 64: masks bit-exact vs the
    oracle run on the same inputs (and counts exact)."""

    @pytest.mark.parametrize("rows,cols,s", [(4096, 14336, 0.9), (8192, 28672, 0.9),
                                             (14336, 4096, 0.95)])
    def test_generate_and_apply(self, rows, cols, s):
        b = 64
        gen = torch.Generator(device="cuda").manual_seed(rows)
        w = torch.randn(rows, cols, device="cuda", generator=gen) * (rows ** -0.5)
        g = torch.randn(rows, cols, device="cuda", generator=gen)
        mask, rep = bs.generate_masks(w, g, b, s)
        w_np, g_np = w.cpu().numpy(), g.cpu().numpy()
        nw = bs.block_norms(w, b).cpu().numpy()
        np.testing.assert_allclose(nw, oracle.block_norms(w_np, b), rtol=1e-13)
        ref_mask, ref_rep = oracle.generate_masks(w_np, g_np, b, s)
        np.testing.assert_array_equal(mask.kept.cpu().numpy(), ref_mask.kept)
        np.testing.assert_array_equal(mask.regrown.cpu().numpy(), ref_mask.regrown)
        assert (rep.kept, rep.regrown) == ref_rep[:2]
        masked, cache = bs.apply_mask(w, mask, b)
        ref_masked, ref_cache = oracle.apply_mask(w_np, ref_mask, b)
        h = cache.to_host()
        np.testing.assert_array_equal(h.col_ptr, ref_cache.col_ptr)
        np.testing.assert_array_equal(h.block_row_idx, ref_cache.block_row_idx)
        assert_bits_equal(h.values, ref_cache.values)
        assert torch.equal(masked.cpu(), torch.from_numpy(ref_masked))


class TestGenerateMasks:
    def test_equal_inputs_no_regrowth(self):
        w = np.random.default_rng(4).standard_normal((16, 16)).astype(np.float32)
        mask, rep = bs.generate_masks(w, w.copy(), 4, 0.5)
        assert rep.regrown == 0 and not mask.regrown.any() and mask.kept.sum() == rep.kept == 8

    def test_shape_mismatch(self):
        with pytest.raises(ValueError, match="shape"):
            bs.generate_masks(np.ones((4, 4)), np.ones((4, 2)), 2, 0.5)

    def test_regrow_disjoint_always(self):
        rng = np.random.default_rng(7)
        for _ in range(20):
            w = rng.standard_normal((12, 12)).astype(np.float32)
            g = rng.standard_normal((12, 12)).astype(np.float32)
            mask, _ = bs.generate_masks(w, g, 3, float(rng.random()))
            assert not (mask.kept & mask.regrown).any()

    def test_bf16_device_inputs(self):
        rng = np.random.default_rng(9)
        w = rng.standard_normal((256, 512)).astype(np.float32)
        g = rng.standard_normal((256, 512)).astype(np.float32)
        wb = torch.from_numpy(w).cuda().bfloat16()
        gb = torch.from_numpy(g).cuda().bfloat16()
        mask, _ = bs.generate_masks(wb, gb, 32, 0.8)
        ref, _ = oracle.generate_masks(wb.float().cpu().numpy(), gb.float().cpu().numpy(), 32, 0.8)
        np.testing.assert_array_equal(mask.kept.cpu().numpy(), ref.kept)
        np.testing.assert_array_equal(mask.regrown.cpu().numpy(), ref.regrown)


class TestApplyMask:
    def test_grid_mismatch(self):
        with pytest.raises(ValueError, match="grid"):
            bs.apply_mask(np.ones((8, 8), np.float32), bs.BlockMask.all_active(3, 3), 4)

    def test_idempotent(self):
        rng = np.random.default_rng(10)
        w = rng.standard_normal((12, 12)).astype(np.float32)
        g = rng.standard_normal((12, 12)).astype(np.float32)
        mask, _ = bs.generate_masks(w, g, 3, 0.6)
        once, c1 = bs.apply_mask(w, mask, 3)
        twice, c2 = bs.apply_mask(once, mask, 3)
        np.testing.assert_array_equal(once, twice)
        assert torch.equal(c1.values, c2.values) and torch.equal(c1.block_row_idx, c2.block_row_idx)

    @pytest.mark.parametrize("rows,cols,b", [(12, 12, 3), (130, 70, 16), (512, 768, 64)])
    def test_structure_reuse_matches_repack(self, rows, cols, b):
        """Re-application between refreshes with the previous cache's structure gives
        the same masked matrix and BCSC bits as a full repack, and shares its plans."""
        rng = np.random.default_rng(rows + cols)
        w = torch.from_numpy(rng.standard_normal((rows, cols)).astype(np.float32)).cuda()
        g = torch.from_numpy(rng.standard_normal((rows, cols)).astype(np.float32)).cuda()
        mask, _ = bs.generate_masks(w, g, b, 0.7)
        _, fresh = bs.apply_mask(w, mask, b, zero_regrown=True)
        fresh.desc()
        w2 = w + 0.25 * g
        for dt in (torch.float32, torch.bfloat16):
            ref_m, ref_c = bs.apply_mask(w2, mask, b, zero_regrown=False, dtype=dt)
            got_m, got_c = bs.apply_mask(w2, mask, b, zero_regrown=False, dtype=dt,
                                         structure=fresh)
            assert torch.equal(got_m, ref_m)
            assert torch.equal(got_c.col_ptr, ref_c.col_ptr)
            assert torch.equal(got_c.block_row_idx, ref_c.block_row_idx)
            assert torch.equal(got_c.values.view(torch.int16 if dt == torch.bfloat16 else torch.int32),
                               ref_c.values.view(torch.int16 if dt == torch.bfloat16 else torch.int32))
            assert got_c._cache[("plan", 0)] is fresh._cache[("plan", 0)]

    def test_bf16_cache_values(self):
        rng = np.random.default_rng(11)
        w = rng.standard_normal((128, 192)).astype(np.float32)
        mask, _ = bs.generate_masks(w, rng.standard_normal((128, 192)).astype(np.float32), 64, 0.5)
        _, c32 = bs.apply_mask(w, mask, 64)
        _, c16 = bs.apply_mask(w, mask, 64, dtype=torch.bfloat16)
        assert torch.equal(c32.values.bfloat16(), c16.values)


@pytest.mark.parametrize("wdt,gdt", [(torch.float64, torch.float64), (torch.bfloat16, torch.float32),
                                     (torch.float32, torch.bfloat16), (torch.float64, torch.float32)])
def test_generate_masks_input_precisions(wdt, gdt):
    """Norms are taken of each matrix in its own precision (pruner.py:95 squares the values
    as given in float64): W and G of different dtypes, and float64 masters, give the oracle's
    masks and counts on the same values."""
    rng = np.random.default_rng(11)
    rows, cols, b, s = 320, 448, 32, 0.8
    w = torch.from_numpy(rng.standard_normal((rows, cols))).to(wdt).cuda()
    g = torch.from_numpy(rng.standard_normal((rows, cols))).to(gdt).cuda()
    mask, rep = bs.generate_masks(w, g, b, s)
    wn, gn = (t.double().cpu().numpy() for t in (w, g))
    np.testing.assert_allclose(bs.block_norms(w, b).cpu().numpy(), oracle.block_norms(wn, b),
                               rtol=1e-13, atol=0)
    ref_mask, ref_rep = oracle.generate_masks(wn, gn, b, s)
    np.testing.assert_array_equal(mask.kept.cpu().numpy(), ref_mask.kept)
    np.testing.assert_array_equal(mask.regrown.cpu().numpy(), ref_mask.regrown)
    assert (rep.kept, rep.regrown) == (int(ref_mask.kept.sum()), int(ref_mask.regrown.sum()))


def test_device_refresh_without_host_round_trips():
    """Device masks carry their counts from generate_masks, so apply_mask sizes the repack
    without reading nnzb back; the result equals the host-input path bit for bit."""
    rng = np.random.default_rng(12)
    rows, cols, b, s = 512, 768, 64, 0.75
    w = rng.standard_normal((rows, cols)).astype(np.float32)
    g = rng.standard_normal((rows, cols)).astype(np.float32)
    mask_d, rep_d = bs.generate_masks(torch.from_numpy(w).cuda(), torch.from_numpy(g).cuda(), b, s)
    assert mask_d.counts == (rep_d.kept, rep_d.regrown)
    assert mask_d.n_active == rep_d.kept + rep_d.regrown
    masked_d, cache_d = bs.apply_mask(torch.from_numpy(w).cuda(), mask_d, b)
    mask_h, rep_h = bs.generate_masks(w, g, b, s)
    masked_h, cache_h = bs.apply_mask(w, mask_h, b)
    assert (rep_d.kept, rep_d.regrown) == (rep_h.kept, rep_h.regrown)
    assert_bits_equal(masked_d.cpu().numpy(), masked_h)
    hd, hh = cache_d.to_host(), cache_h.to_host()
    np.testing.assert_array_equal(hd.col_ptr, hh.col_ptr)
    np.testing.assert_array_equal(hd.block_row_idx, hh.block_row_idx)
    assert_bits_equal(hd.values, hh.values)
    ref = oracle.apply_mask(w, oracle.generate_masks(w, g, b, s)[0], b)
    assert_cache_equal(cache_d, ref[1])


def _fixed_order_norms(x: np.ndarray, b: int, vw: int) -> np.ndarray:
    """The kernels' summation order in numpy: lane l of a block's warp adds the squares of the
    16-byte vectors e = l, l + 32, ... (row-major, vw elements each, in order) in float64, then
    the lanes combine by the xor-shuffle tree 16, 8, 4, 2, 1. A float32 / bfloat16 square is
    exact in float64, so fma(x, x, acc) == acc + x * x here."""
    rows, cols = x.shape
    gr, gc = rows // b, cols // b
    per_row = b // vw
    out = np.empty((gr, gc))
    for r in range(gr):
        for c in range(gc):
            blk = x[r * b:(r + 1) * b, c * b:(c + 1) * b].astype(np.float64).reshape(b * per_row, vw)
            lanes = np.zeros(32)
            for lane in range(32):
                acc = 0.0
                for v in blk[lane::32]:
                    for e in v:
                        acc = acc + e * e
                lanes[lane] = acc
            for o in (16, 8, 4, 2, 1):
                lanes = lanes + lanes[np.arange(32) ^ o]
            out[r, c] = np.sqrt(lanes[0])
    return out


@pytest.mark.parametrize("dtype,b,shape", [(torch.float32, 64, (128, 320)),
                                           (torch.float32, 32, (64, 288)),
                                           (torch.float32, 128, (256, 384)),
                                           (torch.bfloat16, 64, (192, 448)),
                                           (torch.bfloat16, 32, (96, 256))])
def test_block_norms_fixed_order_bitwise(dtype, b, shape):
    # the TMA-staged norms kernel (tiles of up to 256 columns, partial last tile) and the
    # per-warp kernel share one summation order; check it bit for bit
    rng = np.random.default_rng(b + shape[1])
    x = torch.from_numpy(rng.standard_normal(shape).astype(np.float32) * 3).cuda().to(dtype)
    g = (x * 0.5).contiguous()
    from paper_2507_03117_b200 import _lib as L
    gr, gc = shape[0] // b, shape[1] // b
    nw = torch.empty(gr, gc, dtype=torch.float64, device="cuda")
    ng = torch.empty_like(nw)
    L.check(L.load().blast_block_norms(x.data_ptr(), g.data_ptr(), shape[0], shape[1], b,
                                       L.dtype_code(dtype), nw.data_ptr(), ng.data_ptr(),
                                       L.stream()), "norms")
    vw = 4 if dtype == torch.float32 else 8
    for t, n in ((x, nw), (g, ng)):
        ref = _fixed_order_norms(t.float().cpu().numpy(), b, vw)
        assert np.array_equal(n.cpu().numpy().view(np.uint64), ref.view(np.uint64))
