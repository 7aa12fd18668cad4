// Fused block-sparse gated MLP forward: gate+up and down in ONE persistent kernel, with the
// intermediate G = silu(X Wg) * (X Wu) kept in a small L2-resident ring instead of a full
// [tokens x h] tensor in HBM (north star: "the intermediate activation never round-trips to
// HBM"; reference mlp_forward, blocksparse/mlp.py:102-115).
//
// Work items (256-token tile t, output line j) of two kinds run through one pipeline:
//   GU(t, j): G[t, j-block] = silu(X_t Wg[:, j]) * (X_t Wu[:, j])  -> ring slot t % RING
//   DN(t, j): Y[t, j-block] = G_t Wd[:, j]                          -> Y
// in a fixed global order of rounds r = 0, 1, ...: the GU items of tile r, then the DN items
// of tile r - LAG. CTAs take items k = blockIdx.x + i * gridDim.x. Every dependency points to
// an earlier item (DN(t) needs all GU(t); GU(t) reuses the ring slot of DN(t - RING)), each
// CTA processes its items in order and all CTAs are co-resident (one per SM), so the
// earliest unfinished item can always run: no deadlock.
//   * GU completion: the epilogue thread that issued a G tile's TMA stores waits for them
//     (cp.async.bulk.wait_group 0), fences, and adds 1 to gu_done[t] (release).
//   * DN start: the producer spins on gu_done[t] == n_gu_lines (acquire) and fences the async
//     proxy before its first TMA load of G.
//   * ring reuse: before storing G of tile t >= RING the GU epilogue waits for
//     dn_done[t - RING] == n_dn_lines; a DN item signals dn_done once its accumulator is
//     full (its MMAs, hence its reads of G, are complete).
// Per-item math, accumulation order and epilogues are those of spmm_tc.cuh (TM = 2, staged
// bf16 outputs), so results equal the two-launch path bit for bit.
#pragma once

#include "spmm_tc.cuh"

namespace blast {

constexpr int kFusedRing = 5;  // G ring slots (256-token tiles): 5 x 256 x h x 2 B
constexpr int kFusedLag = 2;   // DN(t) items follow the GU items of tile t + LAG

struct FusedParams {
  SpmmParams gu;  // gated gate+up product (out0 = G ring, n_valid = h, ld_out = h)
  SpmmParams dn;  // down product (out0 = Y, n_valid = d, ld_out = d)
  int32_t n_tiles;       // 256-token tiles
  int32_t n_gu_lines;    // h / 64
  int32_t n_dn_lines;    // d / 64
  int32_t* gu_done;      // [n_tiles]
  int32_t* dn_done;      // [n_tiles]
  int32_t dbg;           // diagnosis only (BLAST_FUSED_DBG): 1 signal GU before store completion
};

struct FusedItem {
  int kind;  // 0 GU, 1 DN, -1 none
  int tile;
  int line;
};

__device__ __forceinline__ FusedItem fused_item(const FusedParams& fp, int k) {
  const int rw = fp.n_gu_lines + fp.n_dn_lines;
  const int round = k / rw, off = k - round * rw;
  FusedItem it;
  if (off < fp.n_gu_lines) {
    it.kind = round < fp.n_tiles ? 0 : -1;
    it.tile = round;
    it.line = off;
  } else {
    it.tile = round - kFusedLag;
    it.kind = (it.tile >= 0 && it.tile < fp.n_tiles) ? 1 : -1;
    it.line = off - fp.n_gu_lines;
  }
  return it;
}

__device__ __forceinline__ int ld_acquire_gpu(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_gpu_add(int32_t* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void spin_until_at_least(const int32_t* p, int target) {
  if (ld_acquire_gpu(p) >= target) return;
  while (ld_acquire_gpu(p) < target) __nanosleep(64);
}

// Config shared by both item kinds: b = 64, bf16, 256-token items, stage = panel + 2 blocks.
using FusedCfg = TcCfg<64, 2, 1, 2, false, false, 2, 2>;

__global__ void __launch_bounds__(kTcThreads, 1)
mlp_fused_kernel(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapWg,
                 const __grid_constant__ CUtensorMap mapWu, const __grid_constant__ CUtensorMap mapGin,
                 const __grid_constant__ CUtensorMap mapGout, const __grid_constant__ CUtensorMap mapWd,
                 const __grid_constant__ CUtensorMap mapY, const FusedParams fp) {
  using C = FusedCfg;
  constexpr int B = 64;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* staging = smem + C::STAGES * C::STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE + C::STAGING);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tmem_full = empty + C::STAGES;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
  uint32_t* stage_meta = tmem_slot + 4;

  const uint32_t warp = __shfl_sync(0xffffffffu, warp_id(), 0);
  const uint32_t lane = lane_id();
  const int n_items = (fp.n_tiles + kFusedLag) * (fp.n_gu_lines + fp.n_dn_lines);

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapX);
    tma_prefetch(&mapWg);
    tma_prefetch(&mapWu);
    tma_prefetch(&mapGin);
    tma_prefetch(&mapGout);
    tma_prefetch(&mapWd);
    tma_prefetch(&mapY);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tmem_full[s], 1);
      mbar_init(&tmem_empty[s], kEpiWarps);
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

  if (warp == 0 || warp == 3) {
    // ------------------------------------------------------------ TMA producers
    const uint64_t pol_w = policy_evict_last();
    const uint32_t mine = warp == 0 ? 0u : 1u;
    uint32_t stage = 0, phase = 0, n = 0;
    for (int k = blockIdx.x; k < n_items; k += gridDim.x) {
      const FusedItem fi = fused_item(fp, k);
      if (fi.kind < 0) continue;
      const bool gu = fi.kind == 0;
      const SpmmParams& p = gu ? fp.gu : fp.dn;
      const int s0 = __ldg(&p.step_ptr[fi.line]), s1 = __ldg(&p.step_ptr[fi.line + 1]);
      if (!gu && s1 > s0 && !(fp.dbg & 2)) {
        // G of this tile must be complete (all GU items of the tile signalled)
        spin_until_at_least(&fp.gu_done[fi.tile], fp.n_gu_lines);
        fence_proxy_async_global();
      }
      const CUtensorMap* ma = gu ? &mapX : &mapGin;
      const CUtensorMap* mw0 = gu ? &mapWg : &mapWd;
      const int arow = gu ? fi.tile * C::TROWS : (fi.tile % kFusedRing) * C::TROWS;
      StepCursor cur;
      cur.start(p.steps, s0, s1);
      uint32_t init0 = 0, init1 = 0;
      for (int s = s0; s < s1; ++s) {
        const int4 st = cur.get(s);
        const int kb[2] = {st.y, gu ? st.z : -1};
        const int4 stv = make_int4(st.x, kb[0], kb[1], 0);
        const uint32_t meta = step_recipe<2, false, true>(stv, init0, init1);
        if ((n++ & 1u) != mine) {
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
          continue;
        }
        mbar_wait(&empty[stage], phase ^ 1);
        if (elect_one()) {
          uint32_t bytes = C::TROWS * C::ROWB;
          if (kb[0] >= 0) bytes += B * C::ROWB;
          if (kb[1] >= 0) bytes += B * C::ROWB;
          stage_meta[stage] = meta;
          mbar_expect_tx(&full[stage], bytes);
          uint8_t* sbase = smem + stage * C::STAGE;
          tma_load_2d(sbase, ma, &full[stage], st.x * B, arow);
          if (kb[0] >= 0)
            tma_load_2d_hint(sbase + C::A_TILE, mw0, &full[stage], 0, kb[0] * B, pol_w);
          if (kb[1] >= 0)
            tma_load_2d_hint(sbase + C::A_TILE + C::B_TILE, &mapWu, &full[stage], 0, kb[1] * B,
                             pol_w);
        }
        __syncwarp();
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t smem0 = smem_u32(smem);
    const uint64_t a_desc0 = kmajor_desc<C::SW, C::MMA_K, 2>(smem0, C::TROWS, 0);
    const uint32_t b_off = C::A_TILE;
    const uint64_t b_desc0 = mnmajor_desc<C::SW, C::MMA_K, B>(smem0 + b_off, 0);
    const uint64_t b_desc0_merged = make_sdesc(smem0 + b_off, C::B_TILE, 8u * C::SW, swizzle_layout_code(C::SW));
    constexpr uint32_t kIdescMerged = make_idesc(C::BM, 2 * B, 1u, 0u, 1u);
    auto a_koff = [](int ks) -> uint32_t { return (static_cast<uint32_t>(ks) * 32) >> 4; };
    auto b_koff = [](int ks) -> uint32_t { return (static_cast<uint32_t>(ks) * C::MMA_K * C::SW) >> 4; };
    uint32_t stage = 0, phase = 0, it = 0;
    for (int k = blockIdx.x; k < n_items; k += gridDim.x) {
      const FusedItem fi = fused_item(fp, k);
      if (fi.kind < 0) continue;
      const SpmmParams& p = fi.kind == 0 ? fp.gu : fp.dn;
      const int n_steps = __ldg(&p.step_ptr[fi.line + 1]) - __ldg(&p.step_ptr[fi.line]);
      const uint32_t as = it & 1, use = it >> 1;
      ++it;
      mbar_wait(&tmem_empty[as], (use & 1) ^ 1);
      tc_fence_after();
      const uint32_t d_base = tmem_base + as * C::ACC_STRIDE;
      for (int s = 0; s < n_steps; ++s) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t meta = ld_shared_u32(&stage_meta[stage]);
        if (elect_one()) {
          const uint32_t soff = (stage * C::STAGE) >> 4;
          const uint64_t bd = b_desc0 + soff;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint64_t ad = a_desc0 + soff + ((h * C::BM * C::SW) >> 4);
            const uint32_t dh = d_base + h * C::HALF_ACC;
            if (meta & kMetaMerged) {
              const uint32_t acc = (meta & kMetaAccFirst) ? 1u : 0u;
#pragma unroll
              for (int ks = 0; ks < C::KSL; ++ks)
                mma_f16(dh, ad + a_koff(ks), b_desc0_merged + soff + b_koff(ks), kIdescMerged,
                        (acc | ks) ? 1u : 0u);
            } else {
#pragma unroll
              for (int mm = 0; mm < 2; ++mm) {
                if (!(meta & (mm == 0 ? kMetaHas0 : kMetaHas1))) continue;
                const uint32_t init = (meta & (mm == 0 ? kMetaAccFirst : kMetaAccSecond)) ? 1u : 0u;
                const uint64_t b_mat = bd + ((mm * C::B_TILE) >> 4);
#pragma unroll
                for (int ks = 0; ks < C::KSL; ++ks)
                  mma_f16(dh + mm * B, ad + a_koff(ks), b_mat + b_koff(ks), C::IDESC,
                          (init | ks) ? 1u : 0u);
              }
            }
          }
          mma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
      if (elect_one()) mma_commit(&tmem_full[as]);
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const uint32_t q = warp & 3;
    const int half = static_cast<int>(warp - 4) >> 2;
    const uint32_t etid = threadIdx.x - 128;
    const uint64_t pol_out = policy_evict_first();
    // G stays in L2 for the down product: keep its lines (evict_last) rather than stream them
    const uint64_t pol_g = policy_evict_last();
    uint32_t it = 0, tile_ctr = 0;
    for (int k = blockIdx.x; k < n_items; k += gridDim.x) {
      const FusedItem fi = fused_item(fp, k);
      if (fi.kind < 0) continue;
      const bool gu = fi.kind == 0;
      const SpmmParams& p = gu ? fp.gu : fp.dn;
      const uint32_t as = it & 1, use = it >> 1;
      ++it;
      const int flags = __ldg(&p.line_flags[fi.line]);
      mbar_wait(&tmem_full[as], use & 1);
      tc_fence_after();
      if (!gu && etid == 0) red_release_gpu_add(&fp.dn_done[fi.tile], 1);  // its G reads are done
      if (gu && fi.tile >= kFusedRing && etid == 0 && !(fp.dbg & 4))  // ring slot consumed
        spin_until_at_least(&fp.dn_done[fi.tile - kFusedRing], fp.n_dn_lines);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint8_t* stg = staging + (tile_ctr++ & 1) * C::OUT_TILE;
        const uint32_t tacc = tmem_base + ((q * 32u) << 16) + as * C::ACC_STRIDE + h * C::HALF_ACC;
        if (gu) {
          const int row0 = (fi.tile % kFusedRing) * C::TROWS + h * C::BM;
          epi_tile_compute<B, EPI_GATED_FWD, __nv_bfloat16, false, C::OUT_SW>(
              p, tacc, row0, fi.line * B, flags, stg, half, q, lane, etid, true);
        } else {
          const int row0 = fi.tile * C::TROWS + h * C::BM;
          epi_tile_compute<B, EPI_STORE, __nv_bfloat16, false, C::OUT_SW>(
              p, tacc, row0, fi.line * B, flags, stg, half, q, lane, etid, true);
        }
        if (h == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tmem_empty[as]);
        }
        if (gu)
          epi_tile_store<C::OUT_SW, C::OUT_NATOM, 2>(&mapGout, stg,
                                                    (fi.tile % kFusedRing) * C::TROWS + h * C::BM,
                                                    fi.line * B, etid, pol_g);
        else
          epi_tile_store<C::OUT_SW, C::OUT_NATOM, 2>(&mapY, stg, fi.tile * C::TROWS + h * C::BM,
                                                    fi.line * B, etid, pol_out);
      }
      if (gu && etid == 0) {
        // G tile written: make it visible, then count this item for the tile
        if (!(fp.dbg & 1)) bulk_wait_group<0>();
        fence_proxy_async_global();
        __threadfence();
        red_release_gpu_add(&fp.gu_done[fi.tile], 1);
      }
    }
    if (etid == 0) bulk_wait_group<0>();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

}  // namespace blast
