// CTA-pair block-sparse engine (tcgen05 cta_group::2, M = 256 tokens per MMA)
// with weight blocks kept resident in shared memory across token tiles.
//
// Why: at 90% block sparsity the single-CTA engine (spmm_tc.cuh) streams one
// 128 x b activation panel plus one b x b weight block per 128 x b x b product
// and is bound by L2 -> SM bandwidth (profiles/r01_*). Here
//   * a CTA pair computes 256 tokens per MMA: each CTA loads its own 128 rows of
//     the activation panel (A is M-split) and HALF of every weight block (B is
//     N-split), halving weight traffic and MMA issue count;
//   * an item is (output line j, a range of R token tiles): the line's weight
//     halves are loaded into a resident shared-memory region once per item and
//     reused for all R tiles, so the weight stream almost disappears. Blocks
//     beyond the resident capacity are streamed with the activation panel.
// Same plans, step order (fixed accumulation order) and epilogues as
// spmm_tc.cuh, so results match the single-CTA engine's contract.
//
// Roles per CTA (384 threads): warp 0 TMA producer (both CTAs), warp 1 MMA
// issuer (leader CTA only), warp 2 TMEM allocator, warps 4..11 epilogue.
#pragma once

#include "spmm_tc.cuh"

namespace blast {

// TM = 2: a pair tile is 512 tokens; each CTA stages two 128-row halves per step (rows
// t*512 + h*256 + rank*128), and every half accumulates into its own TMEM columns: 8 pair
// MMAs per pipeline round trip instead of 4.
template <int B, int NMAT, bool SUMACC, bool B_KMAJOR, int OUT_ELT = 0, int TM = 1>
struct PairCfg {
  static constexpr int ELT = 2;
  static constexpr int BM = 128;                          // rows per CTA per half (M = 256 per pair)
  static constexpr int PT = 256 * TM;                     // tokens per pair tile
  static constexpr int ROWB = B * ELT;                    // bytes of an activation panel row
  static constexpr int SW = ROWB < 128 ? ROWB : 128;
  static constexpr int SWE = SW / ELT;
  static constexpr int NATOM = ROWB / SW;
  static constexpr int MMA_K = 16;
  static constexpr int KSL = B / MMA_K;
  static constexpr int NA = SUMACC ? NMAT : 1;
  static constexpr int A_HALF = (BM * ROWB + 1023) / 1024 * 1024;  // one 128-row half
  static constexpr int A_TILE = TM * A_HALF;
  // weight half: MN-major (forward) = [B k-rows x B/2 n-cols]; K-major (transposed
  // product) = [B/2 n-rows x B k-cols]. Either way B*B/2 elements.
  static constexpr int WH = B * (B / 2) * ELT;
  static constexpr int WH_ROWB = B_KMAJOR ? ROWB : (B / 2) * ELT;  // bytes per smem row
  static constexpr int WH_SW = WH_ROWB < 128 ? WH_ROWB : 128;
  static constexpr int WH_NATOM = WH_ROWB / WH_SW;
  static constexpr int WH_ROWS = B_KMAJOR ? B / 2 : B;
  static constexpr int MAX_STAGES = 12;
  static constexpr int STAGE = NA * A_TILE + NMAT * WH;
  // staged output tile (TMA store), double-buffered: see TcCfg
  static constexpr int OUT_ROWB = B * OUT_ELT;
  static constexpr int OUT_SW = OUT_ROWB < 128 ? OUT_ROWB : 128;
  static constexpr int OUT_NATOM = OUT_ELT ? OUT_ROWB / OUT_SW : 0;
  static constexpr int OUT_TILE = OUT_ELT ? (BM * OUT_ROWB + 1023) / 1024 * 1024 : 0;
#ifndef BLAST_PAIR_OUTBUFS
#define BLAST_PAIR_OUTBUFS (TM == 2 ? 1 : 2)
#endif
  // single-buffered output staging at TM = 2 buys a fifth panel stage (measured: 0.386 ->
  // 0.362 ms per cfg3 step with streamed weights)
  static constexpr int OUT_BUFS = BLAST_PAIR_OUTBUFS;
  static constexpr int STAGING = OUT_BUFS * OUT_TILE;
  // dynamic shared memory: [1 KiB barriers + meta][staging][n_stages x STAGE][res_cap x WH]
  static constexpr int SMEM_BYTES = 232448;
  static constexpr int DATA_BYTES = SMEM_BYTES - 2048 - STAGING;  // stages + resident weights
  static constexpr int NACC = SUMACC ? 1 : NMAT;
  static constexpr int HALF_ACC = NACC * B;
  static constexpr int ACC_STRIDE = TM * HALF_ACC;
  static constexpr int TMEM_COLS = 2 * ACC_STRIDE <= 32    ? 32
                                   : 2 * ACC_STRIDE <= 64  ? 64
                                   : 2 * ACC_STRIDE <= 128 ? 128
                                   : 2 * ACC_STRIDE <= 256 ? 256
                                                           : 512;
  static constexpr uint32_t IDESC = make_idesc(256, B, 1u, 0u, B_KMAJOR ? 0u : 1u);
  static_assert(B == 32 || B == 64, "pair engine block sizes");
  static_assert(2 * ACC_STRIDE <= 512, "accumulators exceed TMEM");
};

struct PairParams {
  SpmmParams p;
  int32_t n_pair_tiles;  // ceil(m / 256)
  int32_t tiles_per_item;
  int32_t n_chunks;      // ceil(n_pair_tiles / tiles_per_item)
  int32_t n_stages;      // pipeline depth (activation panels in flight per CTA)
  int32_t res_cap;       // resident weight halves per line (the rest is streamed)
};

// descriptor of a weight half for K slice ks (start-address units of 16 B added)
template <int B, bool B_KMAJOR>
__device__ __forceinline__ uint32_t wh_koff(int ks) {
  using C = PairCfg<B, 1, false, B_KMAJOR>;
  if (B_KMAJOR) {
    const uint32_t byte_k = static_cast<uint32_t>(ks) * 16 * 2;
    return ((byte_k / C::WH_SW) * C::WH_ROWS * C::WH_SW + (byte_k % C::WH_SW)) >> 4;
  }
  return (static_cast<uint32_t>(ks) * 16 * C::WH_SW) >> 4;
}

// Per-stage recipe written by the producer (see kMeta* in spmm_tc.cuh) plus, per matrix, the
// resident slot of its weight half (bits 8-15 / 16-23; 0xff = streamed with the panel).
constexpr uint32_t kPairStreamed = 0xffu;
constexpr uint32_t kBarW = 12;  // named barrier: resident weights of the item landed

template <int B, int NMAT, bool SUMACC, bool B_KMAJOR, int EPI, typename OutT, int OUT_ELT = 0,
          int TM = 1>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kTcThreads, 1)
spmm_pair_kernel(const __grid_constant__ CUtensorMap mapO,
                 const __grid_constant__ CUtensorMap mapA0, const __grid_constant__ CUtensorMap mapA1,
                 const __grid_constant__ CUtensorMap mapW0, const __grid_constant__ CUtensorMap mapW1,
                 const PairParams pp) {
  using C = PairCfg<B, NMAT, SUMACC, B_KMAJOR, OUT_ELT, TM>;
  static_assert(OUT_ELT == 0 || OUT_ELT == static_cast<int>(sizeof(OutT)), "staged output type");
  const SpmmParams& p = pp.p;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int NST = pp.n_stages;
  const int RCAP = pp.res_cap;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + C::MAX_STAGES;
  uint64_t* tmem_full = empty + C::MAX_STAGES;
  uint64_t* tmem_empty = tmem_full + 2;
  uint64_t* wfull = tmem_empty + 2;
  uint64_t* wempty = wfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wempty + 1);
  uint8_t* staging = smem + 1024;                // [2][OUT_TILE]
  uint8_t* stages = staging + C::STAGING;        // activation panels (+ streamed weights)
  uint8_t* res = stages + NST * C::STAGE;        // resident weight halves

  const uint32_t warp = __shfl_sync(0xffffffffu, warp_id(), 0);
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();  // 0 = leader (issues the MMAs)
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  const int n_items = pp.n_chunks * p.n_lines;

  if (warp == 0 && lane == 0) {
    if (OUT_ELT) tma_prefetch(&mapO);
    tma_prefetch(&mapA0);
    tma_prefetch(&mapW0);
    if (NMAT > 1) tma_prefetch(&mapW1);
    if (SUMACC) tma_prefetch(&mapA1);
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tmem_full[s], 1);
      mbar_init(&tmem_empty[s], 2 * kEpiWarps);
    }
    mbar_init(wfull, 1);
    mbar_init(wempty, 1);
    fence_mbar_init();
  }
  if (warp == 2) {
    tmem_alloc_pair(tmem_slot, C::TMEM_COLS);
    tmem_relinquish_pair();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  WaitClock wc;
#ifdef BLAST_WAIT_COUNTERS
  const bool dbg_on = p.dbg != nullptr;
#else
  constexpr bool dbg_on = false;
#endif

  if (warp == 0 || warp == 3) {
    // ------------------------------------------------------------ TMA producers (both CTAs)
    // Per item (line j, R pair tiles): warp 0 puts the line's weight halves into the resident
    // region once (as many as fit), then every tile streams its activation panels through
    // the ring; warps 0 and 3 issue the even / odd steps. The first 32 steps of the line stay
    // in registers across the tiles.
    const uint64_t pol_w = policy_evict_last();
    // activation panels are re-read by every line of the same token tile: keep them in L2
    const uint64_t pol_a = policy_evict_last();
    const uint32_t full0 = mapa_shared(&full[0], 0);
    const uint32_t wfull0 = mapa_shared(wfull, 0);
    const uint32_t mine_p = warp == 0 ? 0u : 1u;
    uint32_t stage = 0, phase = 0, it = 0, n = 0;
    for (int item = pair; item < n_items; item += n_pairs, ++it) {
      const int chunk = item / p.n_lines;
      const int j = item - chunk * p.n_lines;
      const int t0 = chunk * pp.tiles_per_item;
      const int t1 = min(t0 + pp.tiles_per_item, pp.n_pair_tiles);
      const int s0 = __ldg(&p.step_ptr[j]), s1 = __ldg(&p.step_ptr[j + 1]);
      StepCursor first;
      first.start(p.steps, s0, s1);
      const int4 first_mine = first.mine;
      if (warp == 0) {
        // resident weight halves of this line: its first RCAP blocks in step order
        wc.wait(1, wempty, (it & 1) ^ 1, dbg_on);
        int nres = 0;
        {
          StepCursor cur = first;
          for (int s = s0; s < s1 && nres < RCAP; ++s) {
            const int4 st = cur.get(s);
            nres += (st.y >= 0 ? 1 : 0);
            if (NMAT > 1 && nres < RCAP) nres += (st.z >= 0 ? 1 : 0);
          }
        }
        if (rank == 0 && elect_one()) mbar_expect_tx(wfull, 2u * nres * C::WH);
        __syncwarp();
        StepCursor cur;
        cur.steps = p.steps; cur.end = s1; cur.base = s0; cur.mine = first_mine;
        int r = 0;
        for (int s = s0; s < s1 && r < nres; ++s) {
          const int4 st = cur.get(s);
          const int kb[2] = {st.y, st.z};
#pragma unroll
          for (int mm = 0; mm < NMAT; ++mm) {
            if (kb[mm] < 0 || r >= nres) continue;
            if (elect_one()) {
              const CUtensorMap* mw = mm == 0 ? &mapW0 : &mapW1;
              uint8_t* dst = res + r * C::WH;
#pragma unroll
              for (int at = 0; at < C::WH_NATOM; ++at) {
                if (B_KMAJOR)
                  tma_load_2d_pair(dst + at * C::WH_ROWS * C::WH_SW, mw, wfull0,
                                   at * (C::WH_SW / 2),
                                   kb[mm] * B + static_cast<int>(rank) * (B / 2), pol_w);
                else
                  tma_load_2d_pair(dst, mw, wfull0, static_cast<int>(rank) * (B / 2), kb[mm] * B,
                                   pol_w);
              }
            }
            __syncwarp();
            ++r;
          }
        }
      }
      for (int t = t0; t < t1; ++t) {
        int rcount = 0;  // blocks of the line so far (resident while < RCAP)
        StepCursor cur;
        cur.steps = p.steps; cur.end = s1; cur.base = s0; cur.mine = first_mine;
        const int row0 = t * C::PT + static_cast<int>(rank) * C::BM;
        for (int s = s0; s < s1; ++s) {
          const int4 st = cur.get(s);
          const int kb[2] = {st.y, st.z};
          bool streamed[2] = {false, false};
          int nstream = 0;
#pragma unroll
          for (int mm = 0; mm < NMAT; ++mm) {
            if (kb[mm] < 0) continue;
            if (rcount >= RCAP) { streamed[mm] = true; ++nstream; }
            ++rcount;
          }
          if ((n++ & 1u) != mine_p) {
            if (++stage == static_cast<uint32_t>(NST)) { stage = 0; phase ^= 1; }
            continue;
          }
          wc.wait(0, &empty[stage], phase ^ 1, dbg_on);
          if (elect_one()) {
            uint32_t bytes = 0;
#pragma unroll
            for (int a2 = 0; a2 < C::NA; ++a2)
              if (!SUMACC || kb[a2] >= 0) bytes += TM * C::BM * C::ROWB;
            bytes += nstream * C::WH;
            if (rank == 0) mbar_expect_tx(&full[stage], 2u * bytes);
            const uint32_t fb = full0 + stage * 8;
            uint8_t* sbase = stages + stage * C::STAGE;
#pragma unroll
            for (int a2 = 0; a2 < C::NA; ++a2) {
              if (SUMACC && kb[a2] < 0) continue;
              const CUtensorMap* ma = a2 == 0 ? &mapA0 : &mapA1;
#pragma unroll
              for (int h = 0; h < TM; ++h)
#pragma unroll
                for (int at = 0; at < C::NATOM; ++at)
                  tma_load_2d_pair(sbase + a2 * C::A_TILE + h * C::A_HALF + at * C::BM * C::SW,
                                   ma, fb, st.x * B + at * C::SWE, row0 + h * 256, pol_a);
            }
#pragma unroll
            for (int mm = 0; mm < NMAT; ++mm) {
              if (!streamed[mm]) continue;
              const CUtensorMap* mw = mm == 0 ? &mapW0 : &mapW1;
              uint8_t* dst = sbase + C::NA * C::A_TILE + mm * C::WH;
#pragma unroll
              for (int at = 0; at < C::WH_NATOM; ++at) {
                if (B_KMAJOR)
                  tma_load_2d_pair(dst + at * C::WH_ROWS * C::WH_SW, mw, fb, at * (C::WH_SW / 2),
                                   kb[mm] * B + static_cast<int>(rank) * (B / 2), pol_w);
                else
                  tma_load_2d_pair(dst, mw, fb, static_cast<int>(rank) * (B / 2), kb[mm] * B,
                                   pol_w);
              }
            }
          }
          __syncwarp();
          if (++stage == static_cast<uint32_t>(NST)) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1 && rank == 0) {
    // ------------------------------------------------------------ MMA issuer (leader CTA)
    // Walks the line's step list itself (presence ballots, 32 steps per load) and is
    // released by warp 2 through named barriers, so nothing between its MMAs reads shared
    // memory or waits on an mbarrier (see kBarAcc in spmm_tc.cuh).
    const uint32_t smem0 = smem_u32(stages);
    const uint32_t res0 = smem_u32(res);
    const uint64_t a_desc0 = kmajor_desc<C::SW, C::MMA_K, 2>(smem0, C::BM, 0);
    const uint64_t wdesc_res0 =
        B_KMAJOR ? kmajor_desc<C::WH_SW, C::MMA_K, 2>(res0, C::WH_ROWS, 0)
                 : make_sdesc(res0, C::WH, 8u * C::WH_SW, swizzle_layout_code(C::WH_SW));
    const uint32_t wstream_off = C::NA * C::A_TILE;
    const uint64_t wdesc_str0 =
        B_KMAJOR ? kmajor_desc<C::WH_SW, C::MMA_K, 2>(smem0 + wstream_off, C::WH_ROWS, 0)
                 : make_sdesc(smem0 + wstream_off, C::WH, 8u * C::WH_SW,
                              swizzle_layout_code(C::WH_SW));
    auto a_koff = [](int ks) -> uint32_t {
      const uint32_t byte_k = static_cast<uint32_t>(ks) * 32;
      return ((byte_k / C::SW) * C::BM * C::SW + (byte_k % C::SW)) >> 4;
    };
    uint32_t stage = 0, tile_it = 0;
    for (int item = pair; item < n_items; item += n_pairs) {
      const int chunk = item / p.n_lines;
      const int j = item - chunk * p.n_lines;
      const int t0 = chunk * pp.tiles_per_item;
      const int t1 = min(t0 + pp.tiles_per_item, pp.n_pair_tiles);
      const int s0 = __ldg(&p.step_ptr[j]), s1 = __ldg(&p.step_ptr[j + 1]);
      const int idx0 = s0 + static_cast<int>(lane);
      const int4 first = idx0 < s1 ? __ldg(&p.steps[idx0]) : make_int4(0, -1, -1, 0);
      named_bar_sync(kBarW, 64);  // warp 2 saw wfull: this line's resident halves landed
      tc_fence_after();
      for (int t = t0; t < t1; ++t, ++tile_it) {
        const uint32_t as = tile_it & 1;
        named_bar_sync(kBarAcc + as, 64);  // warp 2 saw tmem_empty[as]
        tc_fence_after();
        const uint32_t d_base = tmem_base + as * C::ACC_STRIDE;
        int4 mine = first;
        uint32_t m0 = 0, m1 = 0, seen0 = 0, seen1 = 0;
        int base_blocks = 0;  // stored blocks of this line before the current 32-step chunk
        for (int s = s0; s < s1; ++s) {
          const int i = (s - s0) & 31;
          if (NMAT > 1 && i == 0) {  // single-matrix plans: every step is block s - s0
            if (s != s0) {
              base_blocks += __popc(m0) + __popc(m1);
              const int idx = s + static_cast<int>(lane);
              mine = idx < s1 ? __ldg(&p.steps[idx]) : make_int4(0, -1, -1, 0);
            }
            seen0 |= m0;
            seen1 |= m1;
            m0 = __ballot_sync(0xffffffffu, mine.y >= 0);
            m1 = __ballot_sync(0xffffffffu, NMAT > 1 && mine.z >= 0);
          }
          const uint32_t below = (1u << i) - 1u;
          const bool has0 = NMAT == 1 || ((m0 >> i) & 1u), has1 = NMAT > 1 && ((m1 >> i) & 1u);
          const bool init0 = NMAT == 1 ? s != s0
                             : SUMACC ? (((m0 | m1) & below) | seen0 | seen1) != 0
                                      : ((m0 & below) | seen0) != 0;
          const bool init1 = ((m1 & below) | seen1) != 0;
          // block order in the line: step order, matrix 0 before matrix 1 (the producer's)
          const int b0 = NMAT == 1 ? s - s0 : base_blocks + __popc(m0 & below) + __popc(m1 & below);
          const int bidx[2] = {b0, b0 + (has0 ? 1 : 0)};
          named_bar_sync(kBarStage + stage, 64);  // warp 2 saw full[stage]
          tc_fence_after();
          if (elect_one()) {
            const uint32_t soff = (stage * C::STAGE) >> 4;
#pragma unroll
            for (int hm = 0; hm < TM * NMAT; ++hm) {
              const int h = hm / NMAT, mm = hm % NMAT;  // half-major: one B operand per half
              if (!(mm == 0 ? has0 : has1)) continue;
              const int acc_i = SUMACC ? 0 : mm;
              const int a_i = SUMACC ? mm : 0;
              const uint32_t d = d_base + h * C::HALF_ACC + acc_i * B;
              const uint64_t ad = a_desc0 + soff + ((a_i * C::A_TILE + h * C::A_HALF) >> 4);
              const uint64_t wd = bidx[mm] < RCAP
                                      ? wdesc_res0 + ((static_cast<uint32_t>(bidx[mm]) * C::WH) >> 4)
                                      : wdesc_str0 + soff + ((mm * C::WH) >> 4);
              const uint32_t init = mm == 0 ? (init0 ? 1u : 0u)
                                            : (SUMACC ? ((init0 || has0) ? 1u : 0u) : (init1 ? 1u : 0u));
#pragma unroll
              for (int ks = 0; ks < C::KSL; ++ks)
                mma_f16_pair(d, ad + a_koff(ks), wd + wh_koff<B, B_KMAJOR>(ks), C::IDESC,
                             (init | ks) ? 1u : 0u);
            }
            mma_commit_pair(&empty[stage]);
          }
          __syncwarp();
          if (++stage == static_cast<uint32_t>(NST)) stage = 0;
        }
        if (elect_one()) mma_commit_pair(&tmem_full[as]);
        __syncwarp();
      }
      if (elect_one()) mma_commit_pair(wempty);
      __syncwarp();
    }
  } else if (warp == 2 && rank == 0) {
    // ------------------------------------------------------------ barrier waiter (leader)
    uint32_t stage = 0, phase = 0, it = 0, tile_it = 0;
    for (int item = pair; item < n_items; item += n_pairs, ++it) {
      const int chunk = item / p.n_lines;
      const int j = item - chunk * p.n_lines;
      const int t0 = chunk * pp.tiles_per_item;
      const int t1 = min(t0 + pp.tiles_per_item, pp.n_pair_tiles);
      const int n_steps = __ldg(&p.step_ptr[j + 1]) - __ldg(&p.step_ptr[j]);
      wc.wait(4, wfull, it & 1, dbg_on);
      named_bar_arrive(kBarW, 64);
      for (int t = t0; t < t1; ++t, ++tile_it) {
        const uint32_t as = tile_it & 1, use = tile_it >> 1;
        wc.wait(3, &tmem_empty[as], (use & 1) ^ 1, dbg_on);
        named_bar_arrive(kBarAcc + as, 64);
        for (int s = 0; s < n_steps; ++s) {
          wc.wait(2, &full[stage], phase, dbg_on);
          named_bar_arrive(kBarStage + stage, 64);
          if (++stage == static_cast<uint32_t>(NST)) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const uint32_t q = warp & 3;
    const int half = static_cast<int>(warp - 4) >> 2;
    const uint32_t etid = threadIdx.x - 128;
    const uint64_t pol_out = policy_evict_first();
    const bool vec_ok = (p.ld_out * static_cast<int64_t>(sizeof(OutT))) % 16 == 0;
    uint32_t tile_it = 0;
    for (int item = pair; item < n_items; item += n_pairs) {
      const int chunk = item / p.n_lines;
      const int j = item - chunk * p.n_lines;
      const int t0 = chunk * pp.tiles_per_item;
      const int t1 = min(t0 + pp.tiles_per_item, pp.n_pair_tiles);
      const int flags = __ldg(&p.line_flags[j]);
      for (int t = t0; t < t1; ++t, ++tile_it) {
        const uint32_t as = tile_it & 1, use = tile_it >> 1;
        wc.wait(5, &tmem_full[as], use & 1, dbg_on);
        tc_fence_after();
#pragma unroll
        for (int h = 0; h < TM; ++h) {
          const int row0 = t * C::PT + h * 256 + static_cast<int>(rank) * C::BM;
          uint8_t* stg = staging + ((tile_it * TM + h) % C::OUT_BUFS) * C::OUT_TILE;
          const uint32_t tacc =
              tmem_base + ((q * 32u) << 16) + as * C::ACC_STRIDE + h * C::HALF_ACC;
          epi_tile_compute<B, EPI, OutT, SUMACC, C::OUT_SW, C::OUT_BUFS>(
              p, tacc, row0, j * B, flags, stg, half, q, lane, etid, vec_ok);
          if (h == TM - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              if (rank == 0) mbar_arrive(&tmem_empty[as]);
              else mbar_arrive_cluster(&tmem_empty[as], 0);
            }
          }
          epi_tile_store<C::OUT_SW, C::OUT_NATOM, OUT_ELT>(&mapO, stg, row0, j * B, etid, pol_out);
        }
      }
    }
    if constexpr (OUT_ELT > 0) {
      if (etid == 0) bulk_wait_group<0>();
    }
  }

  if (warp == 0 || warp == 2 || warp == 4) wc.flush(p.dbg);
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, C::TMEM_COLS);
  }
}

}  // namespace blast
