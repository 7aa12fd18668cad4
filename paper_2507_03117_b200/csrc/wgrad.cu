// Weight gradients of the block-sparse MLP (mlp.py:137-141):
//     dW = A^T @ D      A: [m, rows] activations, D: [m, cols] upstream gradient
// evaluated only on a set of b x b blocks (the active blocks of the BCSC
// structure -> [nnzb, b, b] in BCSC order), or on the full grid (the
// reference's dense gradient, needed at mask refresh for regrowth norms and by
// the global-norm clip, trainer.py:365-384) -> dense [rows, cols].
//
// Tensor-core path (bf16, b in {64, 128}): one item = up to NACC x 128 output rows of one
// block column c: up to 2 * NACC consecutive stored blocks of that column for b = 64 (all
// share the D panel, loaded once per stage), one block for b = 128. Both operands are
// MN-major (A^T and D are read straight from the row-major activations), K = tokens.
#include "host.hpp"
#include "scan.cuh"
#include "spmm_tc.cuh"

namespace blast {

struct WgradParams {
  int32_t m;
  int64_t rows, cols;
  int32_t n_items;              // upper bound (grid sizing)
  const int64_t* n_items_dev;   // exact count, on device
  const int4* items;   // {c, s0, n, 0}: block column, first slot, n consecutive slots
  const int32_t* row_of;  // slot -> block row (row_idx); nullptr in dense mode (slot = row)
  float* out_blocks;   // [nnzb, b, b] (selected mode)
  float* dense_out;    // [rows, cols]  (dense mode)
  // split-K over tokens when there are too few blocks to fill the GPU: work item
  // (item, split) covers token stages [split*kps, (split+1)*kps) and writes an fp32
  // partial block; wgrad_reduce_kernel sums the partials in split order.
  int32_t n_split;
  int32_t kps;
  float* partial;      // [n_split][n_slots][b][b]
  int64_t n_slots;     // selected blocks, or gr*gc in dense mode (slot = c*gr + r)
  int64_t gr;
  // tail split (selected mode, n_split = 1): when the last wave would hold few items
  // (r = items mod grid <= grid / 4), those r items are split along the tokens into
  // tail_splits(r) parts written as fp32 partials [kWgTailSplit][tail_cap][b][b] and summed in
  // split order by wgrad_tail_reduce_kernel; nullptr disables.
  float* tail_partial;
  int64_t tail_cap;    // partial slots per split (>= grid / 4 * items' blocks)
  // sweep mode (when every CTA has at most WgCfg::MAX_SWEEP units): a CTA keeps all its
  // units' accumulators in TMEM and walks the tokens once, stage by stage over its units, so
  // all CTAs sweep the activations together and each panel is read from HBM about once (one
  // unit after another, the CTAs restart the sweep per wave and re-read the panels that L2
  // did not keep: dWdown read 731 MB of DRAM for 300 MB of operands)
  int32_t sweep_ok;
};

constexpr int kWgTailSplit = 8;
// number of parts of each tail item (1: no tail split) for n_items items on a grid of g CTAs
__host__ __device__ __forceinline__ int wgrad_tail_splits(int n_items, int g) {
  const int r = n_items % g;
  if (r == 0 || 4 * r > g) return 1;
  return g / r < kWgTailSplit ? g / r : kWgTailSplit;
}

// Accumulators (128 output rows each) per b = 64 item: 2 -> four blocks of one column share
// each D panel load (L2 -> smem bytes per block and 128 tokens: 20 KB instead of 24 KB for
// block pairs). b = 128: one block (one accumulator) per item.
#ifndef BLAST_WG_NACC
#define BLAST_WG_NACC 2
#endif
constexpr int kWgNacc64 = BLAST_WG_NACC;

template <int B>
struct WgCfg {
  static constexpr int NACC = B == 64 ? kWgNacc64 : 1;
  // tokens per pipeline stage (the K of one handshake): 8 MMAs per stage
  static constexpr int TK = 128 / NACC >= 64 ? 128 / NACC : 64;
  static constexpr int PER_ITEM = B == 64 ? 2 * NACC : 1;  // stored blocks per item
  static constexpr int ATOM = TK * 128;         // one [TK x 64 bf16] swizzle-128 atom
  static constexpr int A_TILE = 2 * NACC * ATOM;  // NACC x 128 output rows
  static constexpr int NB_ATOM = B / 64;
  static constexpr int B_TILE = NB_ATOM * ATOM;
  static constexpr int STAGE = A_TILE + B_TILE;
  static constexpr int STAGES = (200 * 1024) / STAGE > 8 ? 8 : (200 * 1024) / STAGE;
  static constexpr int ACC_COLS = NACC * B;     // TMEM columns per accumulator stage
  // all 512 columns: the sweep mode keeps up to 512 / ACC_COLS units' accumulators live
  static constexpr int TMEM_COLS = 512;
  static constexpr int MAX_SWEEP = 512 / ACC_COLS;
  static constexpr uint32_t IDESC = make_idesc(128, B, 1u, 1u, 1u);
  static constexpr int SMEM_BYTES = STAGES * STAGE + 256 + 1024;
  static_assert(STAGES >= 3 && 2 * ACC_COLS <= 512, "wgrad stage / accumulator budget");
};
static bool wgrad_pdl() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BLAST_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}
// BLAST_WG_SWEEP=0 disables the sweep mode (WgradParams::sweep_ok)
static bool wgrad_sweep_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BLAST_WG_SWEEP");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}
static int wgrad_per_item(int block) { return block == 64 ? WgCfg<64>::PER_ITEM : WgCfg<128>::PER_ITEM; }
static int wgrad_tk(int block) { return block == 64 ? WgCfg<64>::TK : WgCfg<128>::TK; }

constexpr uint32_t kWgBarAcc = 2;    // + accumulator stage (2 ids)
constexpr uint32_t kWgBarStage = 4;  // + ring stage (<= 8 ids)

template <int B>
__global__ void __launch_bounds__(256, 1)
wgrad_tc_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapD,
                const WgradParams p) {
  using C = WgCfg<B>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tmem_full = empty + C::STAGES;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
  const uint32_t warp = warp_id(), lane = lane_id();
  const int ksteps = (p.m + C::TK - 1) / C::TK;
  const int n_items = static_cast<int>(*p.n_items_dev);
  const int t_s = (p.tail_partial && p.n_split == 1) ? wgrad_tail_splits(n_items, gridDim.x) : 1;
  const int t_base = t_s > 1 ? n_items - n_items % static_cast<int>(gridDim.x) : n_items;
  const int n_work = t_s > 1 ? t_base + (n_items - t_base) * t_s : n_items * p.n_split;
  // work unit -> item (tail units: t_s per item)
  auto item_of = [&](int w) -> int {
    return (t_s > 1 && w >= t_base) ? t_base + (w - t_base) / t_s : w / p.n_split;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapA);
    tma_prefetch(&mapD);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tmem_full[s], 1);
      mbar_init(&tmem_empty[s], 4);
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, C::TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // the setup above may overlap the previous kernel's tail (programmatic dependent launch)
  griddep_wait();

  auto block_row = [&](int slot) -> int { return p.row_of ? p.row_of[slot] : slot; };
  // k-th work unit of this CTA: round robin over the column-ordered list (-1: past the end)
  const int G = static_cast<int>(gridDim.x), bx = static_cast<int>(blockIdx.x);
  auto unit = [&](int k) -> int {
    const int w = k * G + bx;
    return w < n_work ? w : -1;
  };

  // token-stage range of a work item (split-K)
  auto krange = [&](int w, int& k0, int& k1) {
    int sp, kps;
    if (t_s > 1 && w >= t_base) {
      sp = (w - t_base) % t_s;
      kps = (ksteps + t_s - 1) / t_s;
    } else {
      sp = w % p.n_split;
      kps = p.kps;
    }
    k0 = sp * kps;
    k1 = min(ksteps, k0 + kps);
  };

  // sweep mode: this CTA's units are unit(0..n_mine-1), all resident in TMEM
  const bool sweep = p.sweep_ok && n_work <= C::MAX_SWEEP * G;
  const int n_mine = sweep ? (n_work - bx + G - 1) / G : 0;
  int sk0 = 0, sk1 = 0;  // token-stage span of the sweep
  if (sweep) {
    sk0 = ksteps;
    for (int j = 0; j < n_mine; ++j) {
      int a0, a1;
      krange(unit(j), a0, a1);
      sk0 = min(sk0, a0);
      sk1 = max(sk1, a1);
    }
  }

  // the item's block rows: lane i reads the i-th, then every lane holds all (warp-uniform)
  auto item_rows = [&](const int4& it, int (&rows)[C::PER_ITEM]) {
    const int my_r = static_cast<int>(lane) < it.z ? block_row(it.y + static_cast<int>(lane)) : 0;
#pragma unroll
    for (int i = 0; i < C::PER_ITEM; ++i) rows[i] = __shfl_sync(0xffffffffu, my_r, i);
  };
  // one stage of item `it` at token stage ks (elected lane)
  auto load_stage = [&](uint32_t stage, const int4& it, const int (&rows)[C::PER_ITEM], int ks) {
    const int n = it.z;
    // A atoms: one per block (b = 64), both halves of the block (b = 128)
    const int n_atoms = B == 64 ? n : 2;
    mbar_expect_tx(&full[stage], (n_atoms + C::NB_ATOM) * C::ATOM);
    uint8_t* sa = smem + stage * C::STAGE;
    uint8_t* sb = sa + C::A_TILE;
    const int tok = ks * C::TK;
    if (B == 64) {
#pragma unroll
      for (int i = 0; i < C::PER_ITEM; ++i)
        if (i < n) tma_load_2d(sa + i * C::ATOM, &mapA, &full[stage], rows[i] * B, tok);
    } else {
      tma_load_2d(sa, &mapA, &full[stage], rows[0] * B, tok);
      tma_load_2d(sa + C::ATOM, &mapA, &full[stage], rows[0] * B + 64, tok);
    }
#pragma unroll
    for (int a = 0; a < C::NB_ATOM; ++a)
      tma_load_2d(sb + a * C::ATOM, &mapD, &full[stage], it.x * B + a * 64, tok);
  };
  // MMAs of one stage into the accumulators at TMEM column d (elected lane)
  auto mma_stage = [&](uint32_t stage, uint32_t d, int na, bool first, uint64_t a_desc0,
                       uint64_t b_desc0) {
    const uint32_t soff = (stage * C::STAGE) >> 4;
#pragma unroll
    for (int a = 0; a < C::NACC; ++a) {
      if (a >= na) break;
#pragma unroll
      for (int kk = 0; kk < C::TK / 16; ++kk)
        mma_f16(d + a * B, a_desc0 + soff + ((a * 2 * C::ATOM + kk * 16 * 128) >> 4),
                b_desc0 + soff + ((kk * 16 * 128) >> 4), C::IDESC, (!first || kk > 0) ? 1u : 0u);
    }
    mma_commit(&empty[stage]);
  };
  // accumulators in use: one per two blocks (b = 64); an odd last block leaves rows 64..127 of
  // its accumulator computed from a stale atom and never stored
  auto n_acc = [](int n) { return B == 64 ? (n + 1) / 2 : 1; };

  if (warp == 0) {
    // whole warp walks the work list; one elected lane issues the copies
    uint32_t stage = 0, phase = 0;
    if (sweep) {
      int4 its[C::MAX_SWEEP];
      int rows[C::MAX_SWEEP][C::PER_ITEM], k0s[C::MAX_SWEEP], k1s[C::MAX_SWEEP];
#pragma unroll
      for (int j = 0; j < C::MAX_SWEEP; ++j) {
        if (j < n_mine) {
          const int w = unit(j);
          its[j] = __ldg(&p.items[item_of(w)]);
          item_rows(its[j], rows[j]);
          krange(w, k0s[j], k1s[j]);
        } else {
          its[j] = make_int4(0, 0, 0, 0);
          k0s[j] = k1s[j] = 0;
        }
      }
      for (int ks = sk0; ks < sk1; ++ks) {
#pragma unroll
        for (int j = 0; j < C::MAX_SWEEP; ++j) {
          if (j >= n_mine || ks < k0s[j] || ks >= k1s[j]) continue;
          mbar_wait(&empty[stage], phase ^ 1);
          if (elect_one()) load_stage(stage, its[j], rows[j], ks);
          __syncwarp();
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    } else {
      for (int k = 0; k * G < n_work; ++k) {
        const int w = unit(k);
        if (w < 0) continue;
        const int4 it = __ldg(&p.items[item_of(w)]);
        int rows[C::PER_ITEM];
        item_rows(it, rows);
        int k0, k1;
        krange(w, k0, k1);
        for (int ks = k0; ks < k1; ++ks) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (elect_one()) load_stage(stage, it, rows, ks);
          __syncwarp();
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // MN-major operands: K slice kk = 16 token rows (2 KB); LBO = 64-wide atom stride.
    // The MMA warp waits on named barriers released by the waiter warp (3): an mbarrier wait
    // or shared-memory read in this warp queues behind its own in-flight MMAs (DESIGN.md
    // section 3, tools/mma_probe.cu P8).
    const uint64_t a_desc0 = make_sdesc(smem_u32(smem), C::ATOM, 1024, 2);
    const uint64_t b_desc0 = make_sdesc(smem_u32(smem) + C::A_TILE, C::ATOM, 1024, 2);
    uint32_t stage = 0, it = 0;
    if (sweep) {
      int nas[C::MAX_SWEEP], k0s[C::MAX_SWEEP], k1s[C::MAX_SWEEP];
#pragma unroll
      for (int j = 0; j < C::MAX_SWEEP; ++j) {
        nas[j] = 0;
        k0s[j] = k1s[j] = 0;
        if (j < n_mine) {
          const int w = unit(j);
          nas[j] = n_acc(__ldg(&p.items[item_of(w)]).z);
          krange(w, k0s[j], k1s[j]);
        }
      }
      tc_fence_after();
      for (int ks = sk0; ks < sk1; ++ks) {
#pragma unroll
        for (int j = 0; j < C::MAX_SWEEP; ++j) {
          if (j >= n_mine || ks < k0s[j] || ks >= k1s[j]) continue;
          named_bar_sync(kWgBarStage + stage, 64);  // warp 3 saw full[stage]
          tc_fence_after();
          if (elect_one())
            mma_stage(stage, tmem_base + j * C::ACC_COLS, nas[j], ks == k0s[j], a_desc0, b_desc0);
          __syncwarp();
          if (++stage == C::STAGES) stage = 0;
        }
      }
      if (elect_one()) mma_commit(&tmem_full[0]);
      __syncwarp();
    } else {
      for (int k = 0; k * G < n_work; ++k) {
        const int w = unit(k);
        if (w < 0) continue;
        const uint32_t as = it++ & 1;
        int k0, k1;
        krange(w, k0, k1);
        const int na = n_acc(__ldg(&p.items[item_of(w)]).z);
        named_bar_sync(kWgBarAcc + as, 64);  // warp 3 saw tmem_empty[as]
        tc_fence_after();
        const uint32_t d = tmem_base + as * C::ACC_COLS;
        for (int ks = k0; ks < k1; ++ks) {
          named_bar_sync(kWgBarStage + stage, 64);  // warp 3 saw full[stage]
          tc_fence_after();
          if (elect_one()) mma_stage(stage, d, na, ks == k0, a_desc0, b_desc0);
          __syncwarp();
          if (++stage == C::STAGES) stage = 0;
        }
        if (elect_one()) mma_commit(&tmem_full[as]);
        __syncwarp();
      }
    }
  } else if (warp == 3) {
    // barrier waiter: mirrors the MMA warp's sequence
    uint32_t stage = 0, phase = 0, it = 0;
    if (sweep) {
      int k0s[C::MAX_SWEEP], k1s[C::MAX_SWEEP];
#pragma unroll
      for (int j = 0; j < C::MAX_SWEEP; ++j) {
        k0s[j] = k1s[j] = 0;
        if (j < n_mine) krange(unit(j), k0s[j], k1s[j]);
      }
      for (int ks = sk0; ks < sk1; ++ks) {
#pragma unroll
        for (int j = 0; j < C::MAX_SWEEP; ++j) {
          if (j >= n_mine || ks < k0s[j] || ks >= k1s[j]) continue;
          mbar_wait(&full[stage], phase);
          named_bar_arrive(kWgBarStage + stage, 64);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    } else {
      for (int k = 0; k * G < n_work; ++k) {
        const int w = unit(k);
        if (w < 0) continue;
        const uint32_t as = it & 1, use = it >> 1;
        ++it;
        int k0, k1;
        krange(w, k0, k1);
        mbar_wait(&tmem_empty[as], (use & 1) ^ 1);
        named_bar_arrive(kWgBarAcc + as, 64);
        for (int ks = k0; ks < k1; ++ks) {
          mbar_wait(&full[stage], phase);
          named_bar_arrive(kWgBarStage + stage, 64);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp >= 4) {
    const uint32_t q = warp - 4;
    const int lrow = static_cast<int>(q * 32 + lane);  // 0..127
    // TMEM -> global for work unit w whose accumulators start at TMEM column `col`
    auto store_unit = [&](int w, uint32_t col) {
      const int4 itm = __ldg(&p.items[item_of(w)]);
      const bool tail = t_s > 1 && w >= t_base;
      const int sp = tail ? (w - t_base) % t_s : w % p.n_split;
      // tail units: partial slot index relative to the first tail item's first block
      const int64_t tslot0 = tail ? __ldg(&p.items[t_base]).y : 0;
      int k0, k1;
      krange(w, k0, k1);
      const int n = itm.z;
      const int na = n_acc(n);
#pragma unroll 1
      for (int acc = 0; acc < na; ++acc) {
        // accumulator acc holds blocks 2 acc (rows 0..63) and 2 acc + 1 (rows 64..127), b = 64
        const int bi = B == 64 ? 2 * acc + (lrow >> 6) : 0;
        const int slot = bi < n ? itm.y + bi : -1;
        const int li = B == 64 ? (lrow & 63) : lrow;
        const int r = slot >= 0 ? block_row(slot) : -1;
        const uint32_t tbase = tmem_base + ((q * 32u) << 16) + col + acc * B;
#pragma unroll 1
        for (int ch = 0; ch < B / 16; ++ch) {
          float v[16];
          tmem_ld16(tbase + ch * 16, v);
          if (k1 <= k0) {
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = 0.0f;
          }
          if (slot < 0) continue;
          if (tail) {  // fp32 partial of a tail item, reduced in split order afterwards
            float* dst = p.tail_partial + ((sp * p.tail_cap + (slot - tslot0)) * B + li) * B + ch * 16;
            store_chunk16<float>(dst, v, 16, true);
          } else if (p.n_split > 1) {  // fp32 partial, reduced in split order afterwards
            const int64_t flat = p.dense_out ? static_cast<int64_t>(itm.x) * p.gr + r : slot;
            float* dst = p.partial + ((sp * p.n_slots + flat) * B + li) * B + ch * 16;
            store_chunk16<float>(dst, v, 16, true);
          } else if (p.dense_out) {
            const int64_t row = static_cast<int64_t>(r) * B + li;
            const int64_t col = static_cast<int64_t>(itm.x) * B + ch * 16;
            if (row < p.rows) {
              const int valid = static_cast<int>(p.cols - col);
              store_chunk16<float>(p.dense_out + row * p.cols + col, v, valid, (p.cols % 4) == 0);
            }
          } else {
            float* dst = p.out_blocks + (static_cast<int64_t>(slot) * B + li) * B + ch * 16;
            store_chunk16<float>(dst, v, 16, true);
          }
        }
      }
    };
    if (sweep) {
      if (n_mine > 0) {
        mbar_wait(&tmem_full[0], 0);
        tc_fence_after();
        for (int j = 0; j < n_mine; ++j) store_unit(unit(j), j * C::ACC_COLS);
      }
    } else {
      uint32_t it = 0;
      for (int k = 0; k * G < n_work; ++k) {
        const int w = unit(k);
        if (w < 0) continue;
        const uint32_t as = it & 1, use = it >> 1;
        ++it;
        mbar_wait(&tmem_full[as], use & 1);
        tc_fence_after();
        store_unit(w, as * C::ACC_COLS);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tmem_empty[as]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

// CUDA-core fallback: 64x64 output tile per CTA, 16-token smem stages, 4x4 per thread.
template <typename T>
__global__ void __launch_bounds__(256) wgrad_simt_kernel(const T* __restrict__ A,
                                                         const T* __restrict__ D, int b,
                                                         const int4* items, const WgradParams p) {
  constexpr int TT = 16;
  __shared__ float sa[TT][64];
  __shared__ float sd[TT][64];
  const int4 it = items[blockIdx.x];  // {c, slot, -, tile}: tile = (ti, tj) sub-tile of a block
  const int c = it.x, slot = it.y;
  const int r = p.row_of ? p.row_of[slot] : slot;
  const int ti = it.w >> 16, tj = it.w & 0xFFFF;
  const int i0 = ti * 64, j0 = tj * 64;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[4][4] = {};
  for (int t0 = 0; t0 < p.m; t0 += TT) {
    for (int e = threadIdx.x; e < TT * 64; e += 256) {
      const int tt = e >> 6, cc = e & 63;
      const int tok = t0 + tt;
      const int64_t ar = static_cast<int64_t>(r) * b + i0 + cc;
      const int64_t dc = static_cast<int64_t>(c) * b + j0 + cc;
      sa[tt][cc] = (tok < p.m && i0 + cc < b && ar < p.rows) ? to_f32<T>(A[(int64_t)tok * p.rows + ar]) : 0.0f;
      sd[tt][cc] = (tok < p.m && j0 + cc < b && dc < p.cols) ? to_f32<T>(D[(int64_t)tok * p.cols + dc]) : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int tt = 0; tt < TT; ++tt) {
      float av[4], dv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        av[u] = sa[tt][ty * 4 + u];
        dv[u] = sd[tt][tx * 4 + u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fmaf(av[u], dv[v], acc[u][v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int li = i0 + ty * 4 + u, lj = j0 + tx * 4 + v;
      if (li >= b || lj >= b) continue;
      if (p.dense_out) {
        const int64_t row = static_cast<int64_t>(r) * b + li, col = static_cast<int64_t>(c) * b + lj;
        if (row < p.rows && col < p.cols) p.dense_out[row * p.cols + col] = acc[u][v];
      } else {
        p.out_blocks[(static_cast<int64_t>(slot) * b + li) * b + lj] = acc[u][v];
      }
    }
}

// items for the tensor-core kernel: per block column, runs of up to per_item consecutive
// stored blocks (WgCfg::PER_ITEM), in column order, so the items of one column (sharing its
// D panels) run side by side in the same wave. Dense mode: every block of the grid.
// (A size-sorted list dealt in snake order balances the CTAs better but puts a column's items
// in different waves: its D panels are then read from HBM once per item, which costs more;
// profiles/r02/train_step/wgrad_items.txt.)
__global__ void wgrad_items_kernel(const int64_t* col_ptr, int64_t gr, int64_t gc, int per_item,
                                   const int64_t* item_ptr, int4* items) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= gc) return;
  const int64_t lo = col_ptr ? col_ptr[c] : c * gr;  // dense mode: slot = row
  const int64_t hi = col_ptr ? col_ptr[c + 1] : c * gr + gr;
  int64_t out = item_ptr[c];
  for (int64_t s = lo; s < hi; s += per_item) {
    const int s0 = static_cast<int>(col_ptr ? s : s - c * gr);
    const int n = static_cast<int>(hi - s < per_item ? hi - s : per_item);
    items[out++] = make_int4(static_cast<int>(c), s0, n, 0);
  }
}
__global__ void wgrad_item_count_kernel(const int64_t* col_ptr, int64_t gr, int64_t gc,
                                        int per_item, int64_t* item_ptr) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c == 0) item_ptr[0] = 0;
  if (c >= gc) return;
  const int64_t n = col_ptr ? col_ptr[c + 1] - col_ptr[c] : gr;
  item_ptr[c + 1] = (n + per_item - 1) / per_item;
}
// split-K reduction: out = sum_{sp=0..n_split-1} partial[sp] (fixed order -> deterministic)
__global__ void wgrad_reduce_kernel(const WgradParams p, int b) {
  const int64_t bb = static_cast<int64_t>(b) * b;
  const int64_t total = p.n_slots * bb;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    float acc = p.partial[i];
    for (int sp = 1; sp < p.n_split; ++sp) acc = __fadd_rn(acc, p.partial[sp * total + i]);
    const int64_t slot = i / bb, e = i - slot * bb;
    if (p.dense_out) {
      const int64_t c = slot / p.gr, r = slot - c * p.gr;
      const int64_t row = r * b + e / b, col = c * b + e % b;
      if (row < p.rows && col < p.cols) p.dense_out[row * p.cols + col] = acc;
    } else {
      p.out_blocks[i] = acc;
    }
  }
}
// tail-split reduction: blocks of the last r items = sum of their t_s partials in split order
__global__ void wgrad_tail_reduce_kernel(const WgradParams p, int b, int grid) {
  const int n_items = static_cast<int>(*p.n_items_dev);
  const int t_s = wgrad_tail_splits(n_items, grid);
  if (t_s <= 1) return;
  const int t_base = n_items - n_items % grid;
  const int64_t s0 = p.items[t_base].y;
  const int64_t bb = static_cast<int64_t>(b) * b;
  const int64_t total = (p.n_slots - s0) * bb;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    float acc = p.tail_partial[i];
    for (int sp = 1; sp < t_s; ++sp) acc = __fadd_rn(acc, p.tail_partial[sp * p.tail_cap * bb + i]);
    p.out_blocks[s0 * bb + i] = acc;
  }
}
// simt items: one per (slot, 64x64 sub-tile)
__global__ void wgrad_simt_items_kernel(const int64_t* col_ptr, int64_t gr, int64_t gc, int tiles,
                                        int4* items) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= gc) return;
  const int64_t lo = col_ptr ? col_ptr[c] : 0, hi = col_ptr ? col_ptr[c + 1] : gr;
  const int64_t base = col_ptr ? col_ptr[c] : c * gr;
  for (int64_t s = lo; s < hi; ++s)
    for (int t = 0; t < tiles * tiles; ++t) {
      const int ti = t / tiles, tj = t % tiles;
      items[(base + (s - lo)) * tiles * tiles + t] =
          make_int4(static_cast<int>(c), static_cast<int>(col_ptr ? s : s - lo + 0), 0,
                    (ti << 16) | tj);
    }
}

template <int B>
static int launch_wgrad_tc(const void* a, const void* d, const WgradParams& p, cudaStream_t st) {
  using C = WgCfg<B>;
  auto kern = wgrad_tc_kernel<B>;
  static bool configured[64] = {};
  if (int rc = configure_smem(kern, C::SMEM_BYTES, configured, "wgrad smem attribute")) return rc;
  CUtensorMap ma, md;
  if (!encode_map_2d(&ma, a, BLAST_BF16, p.rows, p.m, p.rows * 2, 64, C::TK, 128)) return BLAST_EINVAL;
  if (!encode_map_2d(&md, d, BLAST_BF16, p.cols, p.m, p.cols * 2, 64, C::TK, 128)) return BLAST_EINVAL;
  if (p.n_items <= 0) return BLAST_OK;
  const int64_t work = static_cast<int64_t>(p.n_items) * p.n_split;
  const int grid = static_cast<int>(work < num_sms() ? work : num_sms());
  // programmatic dependent launch: barrier init / TMEM allocation on SMs freed by the previous
  // kernel's tail (the kernel waits for its completion before reading); BLAST_PDL=0 disables
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = C::SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = wgrad_pdl() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, ma, md, p);
  int rc = check_launch("wgrad_tc");
  if (rc == BLAST_OK && p.tail_partial) {  // no-op on the device when no tail split happened
    const int64_t total = std::min<int64_t>(p.n_slots, p.tail_cap) * B * B;
    const int rg = static_cast<int>(std::min<int64_t>(cdiv(total, 256), (int64_t)num_sms() * 4));
    wgrad_tail_reduce_kernel<<<rg, 256, 0, st>>>(p, B, grid);
    rc = check_launch("wgrad_tail_reduce");
  }
  if (rc == BLAST_OK && p.n_split > 1) {
    const int64_t total = p.n_slots * B * B;
    const int rg = static_cast<int>(std::min<int64_t>(cdiv(total, 256), (int64_t)num_sms() * 8));
    wgrad_reduce_kernel<<<rg, 256, 0, st>>>(p, B);
    rc = check_launch("wgrad_reduce");
  }
  return rc;
}

}  // namespace blast

using namespace blast;

static int block_wgrad_impl(const void* a, const void* d, int64_t m, int64_t rows, int64_t cols,
                            int32_t block, int dtype, const int64_t* col_ptr,
                            const int32_t* row_idx, int64_t nnzb, float* out_blocks,
                            float* dense_out, const int32_t* plan_items,
                            const int64_t* plan_counts, void* stream);

extern "C" int blast_block_wgrad(const void* a, const void* d, int64_t m, int64_t rows,
                                 int64_t cols, int32_t block, int dtype, const int64_t* col_ptr,
                                 const int32_t* row_idx, int64_t nnzb, float* out_blocks,
                                 float* dense_out, void* stream) {
  return block_wgrad_impl(a, d, m, rows, cols, block, dtype, col_ptr, row_idx, nnzb, out_blocks,
                          dense_out, nullptr, nullptr, stream);
}

extern "C" int blast_wgrad_plan(const int64_t* col_ptr, int64_t grid_rows, int64_t grid_cols,
                                int32_t block, int32_t* items, int64_t* counts, void* stream) {
  if (!col_ptr || !items || !counts || grid_cols < 1 || (block != 64 && block != 128)) {
    set_error("wgrad_plan: col_ptr, items, counts required; block 64 or 128");
    return BLAST_EINVAL;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int per_item = wgrad_per_item(block);
  const int thr = 256, blk = static_cast<int>(cdiv(grid_cols, thr));
  wgrad_item_count_kernel<<<blk, thr, 0, st>>>(col_ptr, grid_rows, grid_cols, per_item, counts);
  offsets_scan_kernel<int64_t><<<1, 1024, 0, st>>>(counts, grid_cols);
  wgrad_items_kernel<<<blk, thr, 0, st>>>(col_ptr, grid_rows, grid_cols, per_item, counts,
                                          reinterpret_cast<int4*>(items));
  return check_launch("wgrad_plan");
}

extern "C" int blast_block_wgrad_planned(const void* a, const void* d, int64_t m, int64_t rows,
                                         int64_t cols, int32_t block, int dtype,
                                         const int64_t* col_ptr, const int32_t* row_idx,
                                         int64_t nnzb, const int32_t* items,
                                         const int64_t* counts, float* out_blocks,
                                         void* stream) {
  return block_wgrad_impl(a, d, m, rows, cols, block, dtype, col_ptr, row_idx, nnzb, out_blocks,
                          nullptr, items, counts, stream);
}

static int block_wgrad_impl(const void* a, const void* d, int64_t m, int64_t rows, int64_t cols,
                            int32_t block, int dtype, const int64_t* col_ptr,
                            const int32_t* row_idx, int64_t nnzb, float* out_blocks,
                            float* dense_out, const int32_t* plan_items,
                            const int64_t* plan_counts, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (rows < 1 || cols < 1 || block < 1 || m < 0) {
    set_error("block_wgrad: invalid shape");
    return BLAST_EINVAL;
  }
  const bool dense = dense_out != nullptr;
  if (!dense && (!col_ptr || !row_idx || !out_blocks)) {
    set_error("block_wgrad: selection (col_ptr,row_idx,out_blocks) or dense_out required");
    return BLAST_EINVAL;
  }
  const int64_t gr = cdiv(rows, block), gc = cdiv(cols, block);
  const int64_t nsel = dense ? gr * gc : nnzb;
  if (m == 0) {
    if (dense) cudaMemsetAsync(dense_out, 0, sizeof(float) * rows * cols, st);
    else if (nnzb) cudaMemsetAsync(out_blocks, 0, sizeof(float) * nnzb * block * block, st);
    return check_launch("wgrad zero");
  }
  if (nsel == 0) return BLAST_OK;
  WgradParams p{};
  p.sweep_ok = wgrad_sweep_enabled() ? 1 : 0;
  p.m = static_cast<int32_t>(m);
  p.rows = rows;
  p.cols = cols;
  p.row_of = dense ? nullptr : row_idx;
  p.out_blocks = out_blocks;
  p.dense_out = dense_out;
  const int elt = bytes_of(dtype);
  const bool tc = dtype == BLAST_BF16 && (block == 64 || block == 128) &&
                  (rows * elt) % 16 == 0 && (cols * elt) % 16 == 0 && aligned16(a) &&
                  aligned16(d) && m <= INT32_MAX;
  const int64_t* cp = dense ? nullptr : col_ptr;
  if (tc) {
    const int per_item = wgrad_per_item(block);
    Scratch sp, si;
    if (plan_items && plan_counts && !dense) {  // item list cached with the matrix structure
      p.n_items_dev = plan_counts + gc;
      p.items = reinterpret_cast<const int4*>(plan_items);
    } else {
      if (!sp.alloc(sizeof(int64_t) * (gc + 1), st)) return cuda_status(cudaGetLastError(), "wgrad");
      if (!si.alloc(sizeof(int4) * nsel, st)) return cuda_status(cudaGetLastError(), "wgrad");
      const int thr = 256, blk = static_cast<int>(cdiv(gc, thr));
      wgrad_item_count_kernel<<<blk, thr, 0, st>>>(cp, gr, gc, per_item, sp.as<int64_t>());
      offsets_scan_kernel<int64_t><<<1, 1024, 0, st>>>(sp.as<int64_t>(), gc);
      wgrad_items_kernel<<<blk, thr, 0, st>>>(cp, gr, gc, per_item, sp.as<int64_t>(), si.as<int4>());
      p.n_items_dev = sp.as<int64_t>() + gc;
      p.items = si.as<int4>();
    }
    // upper bound of sum over columns of ceil(blocks / per_item) (grid sizing, split-K choice)
    p.n_items = static_cast<int32_t>(std::min<int64_t>(nsel, (nsel + gc * (per_item - 1)) / per_item));
    // split-K when the blocks cannot fill the GPU (e.g. GPT-2 small at 90%: ~60 blocks)
    const int ksteps = static_cast<int>(cdiv(m, wgrad_tk(block)));
    int n_split = 1;
    if (p.n_items < 2 * num_sms() && ksteps >= 8)
      n_split = std::min<int>({static_cast<int>(cdiv(2 * num_sms(), p.n_items)), ksteps / 4, 32});
    n_split = std::max(1, n_split);
    p.kps = static_cast<int32_t>(cdiv(ksteps, n_split));
    p.n_split = static_cast<int32_t>(cdiv(ksteps, p.kps));
    p.n_slots = nsel;
    p.gr = gr;
    Scratch spart, stail;
    if (p.n_split > 1) {
      if (!spart.alloc(sizeof(float) * p.n_split * nsel * block * block, st))
        return cuda_status(cudaGetLastError(), "wgrad partials");
      p.partial = spart.as<float>();
    } else if (!dense && p.n_items >= num_sms()) {
      // tail split: at most grid / 4 tail items of per_item blocks each
      p.tail_cap = std::min<int64_t>(nsel, static_cast<int64_t>(num_sms() / 4) * per_item);
      if (!stail.alloc(sizeof(float) * kWgTailSplit * p.tail_cap * block * block, st))
        return cuda_status(cudaGetLastError(), "wgrad tail partials");
      p.tail_partial = stail.as<float>();
    }
    return block == 64 ? launch_wgrad_tc<64>(a, d, p, st) : launch_wgrad_tc<128>(a, d, p, st);
  }
  const int tiles = static_cast<int>(cdiv(block, 64));
  const int64_t n_items = nsel * tiles * tiles;
  Scratch si;
  if (!si.alloc(sizeof(int4) * n_items, st)) return cuda_status(cudaGetLastError(), "wgrad");
  wgrad_simt_items_kernel<<<static_cast<int>(cdiv(gc, 256)), 256, 0, st>>>(cp, gr, gc, tiles,
                                                                          si.as<int4>());
  if (n_items > INT32_MAX) {
    set_error("block_wgrad: too many blocks");
    return BLAST_EINVAL;
  }
  if (dtype == BLAST_BF16)
    wgrad_simt_kernel<__nv_bfloat16><<<static_cast<unsigned>(n_items), 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(a), static_cast<const __nv_bfloat16*>(d), block,
        si.as<int4>(), p);
  else
    wgrad_simt_kernel<float><<<static_cast<unsigned>(n_items), 256, 0, st>>>(
        static_cast<const float*>(a), static_cast<const float*>(d), block, si.as<int4>(), p);
  return check_launch("wgrad_simt");
}
