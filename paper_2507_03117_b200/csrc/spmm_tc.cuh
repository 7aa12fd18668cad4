// Block-sparse tile engine on 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// One engine serves every sparse product of the gated MLP:
//   forward   Y = X * W           (reference bspmm,      blocksparse/kernels.py:86-124)
//   fused     Y = f(X * W)        (bspmm_fused,           kernels.py:127-140)
//   gated     G = silu(X Wg) * (X Wu)   (mlp_forward,     mlp.py:111-113)
//   transpose Y = X * W^T         (bspmm_rt,              kernels.py:143-170)
//   gated bwd dA, dB from dG = dY Wd^T  (mlp_backward,    mlp.py:133-139)
//   dX        dX = dA Wg^T + dB Wu^T    (mlp_backward,    mlp.py:142)
//
// Work item = (token tile t of 128 rows, output block line j). The plan
// (built on device from the block index maps, see plan.cu) lists the steps of
// line j in ascending block order, which fixes the accumulation order and
// makes every output bitwise reproducible run to run (kernels.py:117-121).
// Each step names the A panel (a b-wide column panel of the activations) and
// the stored block(s) it multiplies; absent blocks never reach the tensor core.
//
// Warp roles (256 threads, persistent over items, 1 CTA per SM):
//   warp 0      TMA producer: A panel + W block(s) -> smem ring (mbarrier full/empty)
//   warp 1      MMA issuer:   tcgen05.mma 128 x b x K into a double-buffered TMEM accumulator
//   warp 2      TMEM allocator
//   warps 4..7  epilogue: tcgen05.ld -> activation / gating -> global stores
#pragma once

#include "activations.cuh"
#include "ptx.cuh"
#include "../../include/blast.h"

namespace blast {

// EPI_GATED_BWD2: the two-input gating backward (dA, dB from dG, a, b) with both inputs and
// both outputs staged through shared memory by TMA (the engine-level form of EPI_GATED_BWD
// with in1 set; see in_staged)
// EPI_GATED_FWD_SAVE: the training gated forward (G plus the saved a, b), all three outputs
// staged through shared memory and written by TMA stores.
enum Epi : int {
  EPI_STORE = 0,
  EPI_GATED_FWD = 1,
  EPI_GATED_BWD = 2,
  EPI_GATED_BWD2 = 3,
  EPI_GATED_FWD_SAVE = 4
};
// staged output tiles per 128-row output tile
template <int EPI>
constexpr int staged_outputs() {
  return EPI == EPI_GATED_BWD2 ? 2 : EPI == EPI_GATED_FWD_SAVE ? 3 : 1;
}

struct SpmmParams {
  int32_t m;            // activation rows (tokens)
  int32_t n_lines;      // output block lines (block columns of Y)
  int32_t n_valid;      // logical output width; columns >= n_valid are not stored
  int32_t n_tok_tiles;  // ceil(m / 128)
  const int32_t* step_ptr;  // [n_lines + 1]
  const int4* steps;        // {a_blk, k0, k1, 0}
  const int32_t* line_flags;  // bit i: accumulator i received at least one MMA; bits 2..16 /
                              // 17..31: blocks of matrix 0 / 1 in the line
  int32_t act;
  int32_t accumulate;  // EPI_STORE: out0 += result (second half of a split dX sum)
  void* out0;  // Y | G | dA
  void* out1;  // saved gate_pre (fwd) | dB (bwd)
  void* out2;  // saved up_out (fwd)
  void* out3;  // fp32 gated fwd: G for the down projection's hi operand when out0 is null
  void* out4;  // fp32 gated fwd: G's 3xTF32 lo part (G - tf32(G)), the down's lo operand
  const void* in0;  // bwd: gate_pre
  const void* in1;  // bwd: up_out
  int64_t ld_out;   // row stride (elements) of every out*/in* array
  unsigned long long* dbg;  // optional per-role wait-cycle counters (BLAST_DEBUG_COUNTERS)
  const float* bias;        // EPI_STORE: optional per-output-column bias, added before act
  int32_t skip_epilogue;    // diagnosis only (BLAST_SKIP_EPILOGUE): 1 release accumulators unread,
                            // 2 mark stages full without loading operands
  int32_t reverse_tiles;    // process token tiles last-to-first (reads the most recently
                            // written rows of the activations first, while they are in L2)
  const int32_t* sched;     // optional cost-balanced item lists: sched[k * gridDim.x + cta] is
                            // the k-th item of CTA `cta`, -1 past its end (csrc/schedule.cu);
                            // nullptr: static round robin (item = cta + k * gridDim.x)
  int32_t sched_rows;       // rows of `sched`
  int32_t early_trigger;    // 1: release the next PDL launch once every CTA is resident
                            // (decode-size products, fewer than two items per CTA)
  blast_tp_t tp;            // tp.n > 0: fused down-projection + all-reduce epilogue (epi_tp_tile)
};

// BLAST_SKIP_EPILOGUE (diagnosis: skip epilogues / operand loads) is compiled in only on request
#ifndef BLAST_DIAG_SWITCHES
#define BLAST_DIAG_SWITCHES 0  // 0.3472 vs 0.3485 ms per cfg3 step with it in (same box)
#endif
constexpr bool kDiagSwitches = BLAST_DIAG_SWITCHES != 0;

// token tile of a work item (items are t-major: item = t * n_lines + j)
__device__ __forceinline__ int item_tile(const SpmmParams& p, int item) {
  const int t = item / p.n_lines;
  return p.reverse_tiles ? p.n_tok_tiles - 1 - t : t;
}

// k-th work item of this CTA (n_items once its list is exhausted). Every role warp walks the
// same sequence, so all of them agree on the item order without communicating.
__device__ __forceinline__ int item_at(const SpmmParams& p, int k, int n_items) {
  if (p.sched) {
    const int v = k < p.sched_rows ? __ldg(&p.sched[k * static_cast<int>(gridDim.x) +
                                                     static_cast<int>(blockIdx.x)])
                                   : -1;
    return v < 0 ? n_items : v;
  }
  const int it = static_cast<int>(blockIdx.x) + k * static_cast<int>(gridDim.x);
  return it < n_items ? it : n_items;
}

// v[i] += bias[col + i] for the valid columns of a 16-column chunk
__device__ __forceinline__ void add_bias16(float (&v)[16], const float* bias, int col, int valid) {
  if (!bias) return;
#pragma unroll
  for (int i = 0; i < 16; ++i)
    if (i < valid) v[i] = __fadd_rn(v[i], __ldg(&bias[col + i]));
}

// Role-level wait accounting for pipeline diagnosis (only when p.dbg is set):
// 0 producer waits on empty, 1 producer waits on resident-weight release,
// 2 MMA waits on full, 3 MMA waits on accumulator release, 4 MMA waits on
// resident weights, 5 epilogue waits on accumulator, 6 epilogue busy, 7 MMA steps.
// diagnosis counters (BLAST_WAIT_COUNTERS builds): kDbgSlots summed role counters, then the
// per-CTA start / end globaltimer pairs
constexpr int kDbgSlots = 10;
struct WaitClock {
  unsigned long long acc[kDbgSlots] = {};
  __device__ __forceinline__ void wait(int slot, uint64_t* bar, uint32_t parity, bool on) {
    if (!on) {
      mbar_wait(bar, parity);
      return;
    }
    const long long t0 = clock64();
    mbar_wait(bar, parity);
    acc[slot] += static_cast<unsigned long long>(clock64() - t0);
  }
  __device__ __forceinline__ void flush(unsigned long long* dbg) {
    if (!dbg || lane_id() != 0) return;
    for (int i = 0; i < kDbgSlots; ++i)
      if (acc[i]) atomicAdd(&dbg[i], acc[i]);
  }
};

// Warp-cooperative reader of a line's step list: one coalesced load fetches 32
// steps (one per lane) and each step is then broadcast with shuffles, so the
// producer / MMA loops never wait on a dependent global load per step. Must be
// used by a full, converged warp.
struct StepCursor {
  const int4* steps;
  int end;
  int base;
  int4 mine;
  __device__ __forceinline__ void fetch() {
    const int idx = base + static_cast<int>(lane_id());
    mine = idx < end ? __ldg(&steps[idx]) : make_int4(0, -1, -1, 0);
  }
  __device__ __forceinline__ void start(const int4* s, int s0, int s1) {
    steps = s;
    end = s1;
    base = s0;
    fetch();
  }
  __device__ __forceinline__ int4 get(int s) {
    if (s - base >= 32) {
      base += 32;
      fetch();
    }
    const int i = s - base;
    return make_int4(__shfl_sync(0xffffffffu, mine.x, i), __shfl_sync(0xffffffffu, mine.y, i),
                     __shfl_sync(0xffffffffu, mine.z, i), 0);
  }
};

// OUT_ELT > 0: out0 is staged in shared memory (double-buffered, swizzled) and
// written by TMA stores (whole 128-byte lines) instead of per-thread row-strided stores.
// TM = 2: an item covers 2 x 128 tokens; every stage carries a 256-row activation panel,
// its weight block(s) are loaded once for both halves, and each half accumulates into its
// own TMEM columns (twice the MMAs per pipeline round trip, half the weight traffic).
// IN_ST = 1 (staged single-input activation-derivative epilogue): the epilogue also stages the
// items' `in0` tiles (TM x 128 rows x B) in shared memory with one TMA load per tile, one item
// ahead (double-buffered), instead of row-strided per-thread loads.
// IN_ST = 2 (EPI_GATED_BWD2): both inputs (a, b) staged that way, and both outputs (dA, dB)
// leave through staged tiles and TMA stores.
// SPLIT = 1 (gate+up): a stage carries ONE weight block; a step with both a gate and an up
// block becomes two stages (the panel is loaded twice, ~5 % of steps at 90 % sparsity), and
// the output is staged single-buffered. The 16 + 16 KB saved buy a fifth pipeline stage,
// which the TMA latency under load needs.
// SPLIT = 2 (gate+up, sequential): same stage layout; an item runs all of its line's gate
// blocks, then all of its up blocks (the plan walked twice), so the MMA issuer's recipe is
// the stage index against the line's gate-block count (plan flags) and a waiter warp
// handles the mbarriers, as for single-matrix products.
template <int B, int ELT, int NPASS, int NMAT, bool SUMACC, bool B_KMAJOR, int OUT_ELT = 0,
          int TM = 1, int IN_ST = 0, int SPLIT = 0, int NOUT_ = 1>
struct TcCfg {
  static constexpr int BM = 128;                          // rows per MMA / per output tile
  static constexpr int TROWS = BM * TM;                   // token rows per item
  static constexpr int ROWB = B * ELT;                    // bytes of one block row
  static constexpr int SW = ROWB < 128 ? ROWB : 128;      // swizzle span
  static constexpr int SWE = SW / ELT;                    // elements per swizzle row
  static constexpr int NATOM = ROWB / SW;                 // swizzle atoms along a row
  static constexpr int MMA_K = 32 / ELT;                  // 16 (bf16) / 8 (tf32)
  static constexpr int KSL = B / MMA_K;                   // MMAs per block along K
  static constexpr int NCOPY = NPASS == 3 ? 2 : 1;        // hi / lo operand copies
  // 3xTF32 (fp32): a stage carries ONE swizzle atom of K (32 fp32) of the hi and lo copies of
  // the panel and of the block, so a 64-wide block is NATOM stages of 48 KB instead of one
  // 96 KB stage (four in flight instead of two). Per K slice one N = 2B MMA multiplies A_hi
  // by [W_hi; W_lo] (adjacent in smem) into an accumulator pair and one N = B MMA adds
  // A_lo * W_hi to the pair's second half; the epilogue sums the pair (hi*hi and the cross
  // terms accumulate separately).
  static constexpr bool SK = NPASS == 3;
  static constexpr int KPS = SK ? 1 : NATOM;              // K atoms per stage
  static constexpr int SPS = SK ? NATOM : 1;              // stages per step (stored block)
  static constexpr int KSL_ST = KSL / SPS;                // MMA K slices per stage
  static constexpr int ACC_W = SK ? 2 * B : B;            // TMEM columns per accumulator
  static constexpr int NA = (SUMACC && !SPLIT) ? NMAT : 1;  // distinct A panels per stage
  static constexpr int round1k(int x) { return (x + 1023) / 1024 * 1024; }
  static constexpr int A_BYTES = TROWS * SW * KPS;        // one copy of a stage's panel
  static constexpr int B_BYTES = B * SW * KPS;            // one copy of a stage's block
  static constexpr int A_TILE = round1k(A_BYTES);
  static constexpr int B_TILE = round1k(B_BYTES);
  static constexpr int WSLOTS = SPLIT ? 1 : NMAT;           // weight blocks per stage
  static constexpr int STAGE = NA * NCOPY * A_TILE + WSLOTS * NCOPY * B_TILE;
#ifndef BLAST_ONE_OUTBUF_1MAT
#define BLAST_ONE_OUTBUF_1MAT 1  // down: 0.3467 vs 0.3487 ms per cfg3 step (same box)
#endif
  // single-buffered output staging buys a fifth 40 KB stage (gate+up SPLIT layouts; with
  // BLAST_ONE_OUTBUF_1MAT also the 256-token single-matrix products)
#ifndef BLAST_ONE_OUTBUF_BWD2
#define BLAST_ONE_OUTBUF_BWD2 1
#endif
  static constexpr int OUT_BUFS =
      (SPLIT || (BLAST_ONE_OUTBUF_1MAT && NMAT == 1 && TM == 2 && IN_ST == 0 && B >= 64) ||
       (BLAST_ONE_OUTBUF_BWD2 && IN_ST == 2))
          ? 1
          : 2;
  static constexpr int OUT_ROWB = B * OUT_ELT;                          // bytes of an output tile row
  static constexpr int OUT_SW = OUT_ROWB < 128 ? OUT_ROWB : 128;
  static constexpr int OUT_NATOM = OUT_ELT ? OUT_ROWB / OUT_SW : 0;
  static constexpr int OUT_TILE = OUT_ELT ? round1k(BM * OUT_ROWB) : 0;
  static constexpr int NOUT = NOUT_;                                // staged outputs per tile
  // staged inputs per 128-row half, double-buffered across halves: [2 bufs][IN_ST] tiles
  static constexpr int IN_STAGING = IN_ST * 2 * OUT_TILE;
  static constexpr int STAGING = OUT_BUFS * NOUT * OUT_TILE + IN_STAGING;
  // 227 KB opt-in maximum minus barriers, alignment slack and the output staging
  static constexpr int SMEM_BUDGET = OUT_ELT ? 232448 - 1024 - 512 - STAGING : 200 * 1024;
  static constexpr int STAGES_RAW = SMEM_BUDGET / STAGE;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int NACC = SUMACC ? 1 : NMAT;
  static constexpr int HALF_ACC = NACC * ACC_W;           // TMEM columns per 128-row half
  static constexpr int ACC_STRIDE = TM * HALF_ACC;        // TMEM columns per accumulator stage
  static constexpr int TMEM_COLS_RAW = 2 * ACC_STRIDE;
  static constexpr int TMEM_COLS = TMEM_COLS_RAW <= 32    ? 32
                                   : TMEM_COLS_RAW <= 64  ? 64
                                   : TMEM_COLS_RAW <= 128 ? 128
                                   : TMEM_COLS_RAW <= 256 ? 256
                                                          : 512;
  static constexpr uint32_t IDESC =
      make_idesc(BM, B, ELT == 2 ? 1u : 2u, 0u, B_KMAJOR ? 0u : 1u);
  static constexpr uint32_t IDESC_PAIR = make_idesc(BM, 2 * B, 2u, 0u, 0u);  // SK: N = 2B
  static_assert(!SK || (ELT == 4 && B_KMAJOR && 2 * B <= 256 && SW == ROWB / NATOM),
                "split-K stages: fp32, K-major blocks");
  // barriers + tmem slot live after the stages
  static constexpr int BAR_BYTES = 512;
  static constexpr int SMEM_BYTES = STAGES * STAGE + STAGING + BAR_BYTES + 1024;  // +1024 alignment slack
  static_assert(STAGES >= 2, "stage does not fit twice in shared memory");
  static_assert(B % 16 == 0 && B >= 16 && B <= 256, "tensor-core block size");
  static_assert(TMEM_COLS_RAW <= 512, "accumulators exceed TMEM");
  static_assert(ROWB % SW == 0, "row must be whole swizzle atoms");
  static_assert(OUT_ELT == 0 || (OUT_ROWB >= 32 && OUT_ROWB % (OUT_SW ? OUT_SW : 1) == 0), "staged output rows");
  static_assert(TM == 1 || TM == 2, "token multiplier");
};

// Write 16 consecutive output values of tile row `row` starting at tile column `col`
// into a staged output tile laid out as OUT_NATOM swizzle atoms of [128 rows x SW bytes]
// (the layout a SWIZZLE_<SW> TMA store reads): 16-byte unit u of a row lands at
// u ^ ((row * SW / 128) mod (SW / 16)).
// Inverse of stage_chunk16: 16 consecutive values of a staged (TMA-loaded, swizzled) tile.
template <typename OutT, int SW>
__device__ __forceinline__ void unstage_chunk16(const uint8_t* tile, int row, int col,
                                                float (&v)[16]) {
  constexpr int E = sizeof(OutT);
  constexpr int UNITS = 16 * E / 16;
  const int byte0 = col * E;
  const uint8_t* atom = tile + (byte0 / SW) * (128 * SW) + row * SW;
  const int u0 = (byte0 % SW) / 16;
  const int x = ((row * SW) >> 7) & (SW / 16 - 1);
#pragma unroll
  for (int k = 0; k < UNITS; ++k) {
    const uint4 w = *reinterpret_cast<const uint4*>(atom + (((u0 + k) ^ x) * 16));
    if constexpr (E == 4) {
      v[4 * k] = __uint_as_float(w.x); v[4 * k + 1] = __uint_as_float(w.y);
      v[4 * k + 2] = __uint_as_float(w.z); v[4 * k + 3] = __uint_as_float(w.w);
    } else {
      const uint32_t h[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&h[i]));
        v[8 * k + 2 * i] = f.x;
        v[8 * k + 2 * i + 1] = f.y;
      }
    }
  }
}
template <typename OutT, int SW>
__device__ __forceinline__ void stage_chunk16(uint8_t* tile, int row, int col, const float (&v)[16]) {
  constexpr int E = sizeof(OutT);
  constexpr int UNITS = 16 * E / 16;  // 16-byte units of this chunk
  const int byte0 = col * E;
  uint8_t* atom = tile + (byte0 / SW) * (128 * SW) + row * SW;
  const int u0 = (byte0 % SW) / 16;
  const int x = ((row * SW) >> 7) & (SW / 16 - 1);
#pragma unroll
  for (int k = 0; k < UNITS; ++k) {
    uint4 w;
    if constexpr (E == 4) {
      w = make_uint4(__float_as_uint(v[4 * k]), __float_as_uint(v[4 * k + 1]),
                     __float_as_uint(v[4 * k + 2]), __float_as_uint(v[4 * k + 3]));
    } else {
      uint32_t h[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        __nv_bfloat162 pr = __floats2bfloat162_rn(v[8 * k + 2 * i], v[8 * k + 2 * i + 1]);
        h[i] = *reinterpret_cast<uint32_t*>(&pr);
      }
      w = make_uint4(h[0], h[1], h[2], h[3]);
    }
    *reinterpret_cast<uint4*>(atom + (((u0 + k) ^ x) * 16)) = w;
  }
}

// K-major operand (rows x B elements, stored as NATOM swizzle atoms of `rows` x SW bytes):
// descriptor for K slice `ks`.
template <int SW, int MMA_K, int ELT>
__device__ __forceinline__ uint64_t kmajor_desc(uint32_t base, int rows, int ks) {
  const uint32_t byte_k = static_cast<uint32_t>(ks) * MMA_K * ELT;  // 32 B per K slice
  const uint32_t atom = byte_k / SW;
  const uint32_t within = byte_k % SW;
  return make_sdesc(base + atom * static_cast<uint32_t>(rows) * SW + within, 16u, 8u * SW,
                    swizzle_layout_code(SW));
}
// MN-major B operand (B rows of K, each row B elements of N in NATOM atoms).
template <int SW, int MMA_K, int B>
__device__ __forceinline__ uint64_t mnmajor_desc(uint32_t base, int ks) {
  return make_sdesc(base + static_cast<uint32_t>(ks) * MMA_K * SW, static_cast<uint32_t>(B) * SW,
                    8u * SW, swizzle_layout_code(SW));
}

#ifndef BLAST_V8
#define BLAST_V8 1
#endif
// V8: 256-bit stores when 32-byte aligned. Not used in the out-of-line TP epilogue
// (epi_tp_tile): there the 256-bit store of a pointer loaded from the local copy of the
// parameters wrote wrong data (tests/test_gpu_parallel.py virtual ranks), the 128-bit path
// is correct.
template <typename OutT, bool V8 = true>
__device__ __forceinline__ void store_chunk16(OutT* dst, const float (&v)[16], int valid,
                                              bool vec_ok) {
  if (V8 && BLAST_V8 && vec_ok && valid >= 16 && (reinterpret_cast<uintptr_t>(dst) & 31u) == 0) {
    // whole 32-byte sectors per thread and instruction (row-strided tiles: one row per lane)
    if constexpr (sizeof(OutT) == 4) {
#pragma unroll
      for (int i = 0; i < 2; ++i)
        st_global_v8(dst + 8 * i, __float_as_uint(v[8 * i]), __float_as_uint(v[8 * i + 1]),
                     __float_as_uint(v[8 * i + 2]), __float_as_uint(v[8 * i + 3]),
                     __float_as_uint(v[8 * i + 4]), __float_as_uint(v[8 * i + 5]),
                     __float_as_uint(v[8 * i + 6]), __float_as_uint(v[8 * i + 7]));
    } else {
      uint32_t w[8];
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        __nv_bfloat162 pr = __floats2bfloat162_rn(v[2 * h], v[2 * h + 1]);
        w[h] = *reinterpret_cast<uint32_t*>(&pr);
      }
      st_global_v8(dst, w[0], w[1], w[2], w[3], w[4], w[5], w[6], w[7]);
    }
  } else if (vec_ok && valid >= 16) {
    if constexpr (sizeof(OutT) == 4) {
      float4* d = reinterpret_cast<float4*>(dst);
#pragma unroll
      for (int i = 0; i < 4; ++i) d[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    } else {
      uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        uint32_t w[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          __nv_bfloat162 pr = __floats2bfloat162_rn(v[8 * i + 2 * h], v[8 * i + 2 * h + 1]);
          w[h] = *reinterpret_cast<uint32_t*>(&pr);
        }
        d[i] = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (i < valid) dst[i] = from_f32<OutT>(v[i]);
  }
}
template <typename T>
__device__ __forceinline__ void load_chunk16(const T* src, float (&v)[16], int valid, bool vec_ok) {
  if (BLAST_V8 && vec_ok && valid >= 16 && (reinterpret_cast<uintptr_t>(src) & 31u) == 0) {
    uint32_t w[sizeof(T) == 4 ? 2 : 1][8];
#pragma unroll
    for (int i = 0; i < (sizeof(T) == 4 ? 2 : 1); ++i) ld_global_v8(src + 8 * i * (sizeof(T) == 4 ? 1 : 2), w[i]);
    if constexpr (sizeof(T) == 4) {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(w[i / 8][i % 8]);
    } else {
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[0][h]));
        v[2 * h] = f.x;
        v[2 * h + 1] = f.y;
      }
    }
  } else if (vec_ok && valid >= 16) {
    if constexpr (sizeof(T) == 4) {
      const float4* s = reinterpret_cast<const float4*>(src);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float4 q = s[i];
        v[4 * i] = q.x; v[4 * i + 1] = q.y; v[4 * i + 2] = q.z; v[4 * i + 3] = q.w;
      }
    } else {
      const uint4* s = reinterpret_cast<const uint4*>(src);
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        uint4 q = s[i];
        uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          __nv_bfloat162 pr = *reinterpret_cast<__nv_bfloat162*>(&w[h]);
          float2 f = __bfloat1622float2(pr);
          v[8 * i + 2 * h] = f.x; v[8 * i + 2 * h + 1] = f.y;
        }
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = (i < valid) ? to_f32<T>(src[i]) : 0.0f;
  }
}
// One 16-column chunk of an output tile, shared by the single-CTA and CTA-pair
// engines. v0 holds the first accumulator (already zeroed if it received no
// MMA); acc1_addr is the TMEM address of the second accumulator's chunk (gated
// forward). Must be called by the whole warp (tcgen05.ld is warp-collective).
//   EPI_STORE      out0 = act(v0 + bias) [+= out0]; out1 (optional) = v0 + bias
//   EPI_GATED_FWD  out0 = silu(a) * b; out1 = a, out2 = b (optional)   (mlp.py:111-113)
//   EPI_GATED_BWD  in1 set: out0 = dA, out1 = dB from dG = v0          (mlp.py:133-139)
//                  in1 NULL: out0 = v0 * act'(in0)  (backward of a fused activation)
// STG_SW > 0: out0 goes to the staged tile `stg` (tile row `trow`, tile column `tcol`)
// instead of global memory; rows / columns outside the tensor are clipped by the TMA store.
template <int EPI, typename OutT, int STG_SW = 0>
__device__ __forceinline__ void epilogue_chunk(const SpmmParams& p, float (&v0)[16],
                                               float (&v1)[16], int flags, bool row_ok,
                                               int col, int valid, int64_t off, bool vec_ok,
                                               uint8_t* stg = nullptr, int trow = 0,
                                               int tcol = 0, const uint8_t* in_stg = nullptr,
                                               int out1_off = 0, int in1_off = 0) {
  const bool live = row_ok && valid > 0;
  if constexpr (EPI == EPI_STORE) {
    add_bias16(v0, p.bias, col, valid);
    if (p.out1 && live)
      store_chunk16<OutT>(reinterpret_cast<OutT*>(p.out1) + off, v0, valid, vec_ok);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if constexpr (sizeof(OutT) == 2)
        v0[i] = apply_act_fast(v0[i], p.act);
      else
        v0[i] = apply_act(v0[i], p.act);
    }
    if constexpr (STG_SW > 0) {
      stage_chunk16<OutT, STG_SW>(stg, trow, tcol, v0);
    } else if (live) {
      if (p.accumulate) {
        float prev[16];
        load_chunk16<OutT>(reinterpret_cast<const OutT*>(p.out0) + off, prev, valid, vec_ok);
#pragma unroll
        for (int i = 0; i < 16; ++i) v0[i] = __fadd_rn(prev[i], v0[i]);
      }
      store_chunk16<OutT>(reinterpret_cast<OutT*>(p.out0) + off, v0, valid, vec_ok);
    }
  } else if constexpr (EPI == EPI_GATED_FWD) {
    if (!(flags & 2)) {
#pragma unroll
      for (int i = 0; i < 16; ++i) v1[i] = 0.0f;
    }
    if (live) {
      if (p.out1) store_chunk16<OutT>(reinterpret_cast<OutT*>(p.out1) + off, v0, valid, vec_ok);
      if (p.out2) store_chunk16<OutT>(reinterpret_cast<OutT*>(p.out2) + off, v1, valid, vec_ok);
    }
    if (live || STG_SW > 0) {
      float g[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if constexpr (sizeof(OutT) == 2)
          g[i] = gated_fwd_fast(v0[i], v1[i]);
        else
          g[i] = gated_fwd(v0[i], v1[i]);
      }
      if constexpr (STG_SW > 0) {
        stage_chunk16<OutT, STG_SW>(stg, trow, tcol, g);
      } else {
        if (p.out0) store_chunk16<OutT>(reinterpret_cast<OutT*>(p.out0) + off, g, valid, vec_ok);
        if constexpr (sizeof(OutT) == 4) {
          // fp32: G also leaves as its 3xTF32 hi / lo split, the down projection's operands
          if (p.out4) {  // lo part only: G itself (out0 / out3) is the hi operand
            float lo[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float v = g[i];
              lo[i] = isfinite(v) ? __fsub_rn(v, __uint_as_float(__float_as_uint(v) & 0xFFFFE000u)) : 0.0f;
            }
            if (p.out3 && p.out3 != p.out0)
              store_chunk16<OutT>(reinterpret_cast<OutT*>(p.out3) + off, g, valid, vec_ok);
            store_chunk16<OutT>(reinterpret_cast<OutT*>(p.out4) + off, lo, valid, vec_ok);
          }
        }
      }
    }
  } else if constexpr (EPI == EPI_GATED_FWD_SAVE) {
    // G, a, b into three staged tiles (rows / columns outside the tensor clipped by TMA)
    static_assert(STG_SW > 0, "EPI_GATED_FWD_SAVE is the staged form");
    if (!(flags & 2)) {
#pragma unroll
      for (int i = 0; i < 16; ++i) v1[i] = 0.0f;
    }
    float g[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if constexpr (sizeof(OutT) == 2)
        g[i] = gated_fwd_fast(v0[i], v1[i]);
      else
        g[i] = gated_fwd(v0[i], v1[i]);
    }
    stage_chunk16<OutT, STG_SW>(stg, trow, tcol, g);
    stage_chunk16<OutT, STG_SW>(stg + out1_off, trow, tcol, v0);
    stage_chunk16<OutT, STG_SW>(stg + 2 * out1_off, trow, tcol, v1);
  } else if constexpr (EPI == EPI_GATED_BWD2) {
    // staged a, b tiles in; staged dA, dB tiles out (rows past the end are clipped by TMA)
    static_assert(STG_SW > 0, "EPI_GATED_BWD2 is the staged form");
    float a[16], b[16], da[16], db[16];
    unstage_chunk16<OutT, STG_SW>(in_stg, trow, tcol, a);
    unstage_chunk16<OutT, STG_SW>(in_stg + in1_off, trow, tcol, b);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if constexpr (sizeof(OutT) == 2)
        gated_bwd_fast(v0[i], a[i], b[i], da[i], db[i]);
      else
        gated_bwd(v0[i], a[i], b[i], da[i], db[i]);
    }
    stage_chunk16<OutT, STG_SW>(stg, trow, tcol, da);
    stage_chunk16<OutT, STG_SW>(stg + out1_off, trow, tcol, db);
  } else {
    if (!live) return;
    if (p.in1) {
      float a[16], b[16], da[16], db[16];
      load_chunk16<OutT>(reinterpret_cast<const OutT*>(p.in0) + off, a, valid, vec_ok);
      load_chunk16<OutT>(reinterpret_cast<const OutT*>(p.in1) + off, b, valid, vec_ok);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if constexpr (sizeof(OutT) == 2)
          gated_bwd_fast(v0[i], a[i], b[i], da[i], db[i]);
        else
          gated_bwd(v0[i], a[i], b[i], da[i], db[i]);
      }
      store_chunk16<OutT>(reinterpret_cast<OutT*>(p.out0) + off, da, valid, vec_ok);
      store_chunk16<OutT>(reinterpret_cast<OutT*>(p.out1) + off, db, valid, vec_ok);
    } else {
      float pre[16];
      if constexpr (STG_SW > 0) {
        if (in_stg) unstage_chunk16<OutT, STG_SW>(in_stg, trow, tcol, pre);
        else load_chunk16<OutT>(reinterpret_cast<const OutT*>(p.in0) + off, pre, valid, vec_ok);
      } else {
        load_chunk16<OutT>(reinterpret_cast<const OutT*>(p.in0) + off, pre, valid, vec_ok);
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if constexpr (sizeof(OutT) == 2)
          v0[i] = __fmul_rn(v0[i], apply_act_grad_fast(pre[i], p.act));
        else
          v0[i] = __fmul_rn(v0[i], apply_act_grad(pre[i], p.act));
      }
      if constexpr (STG_SW > 0)
        stage_chunk16<OutT, STG_SW>(stg, trow, tcol, v0);
      else
        store_chunk16<OutT>(reinterpret_cast<OutT*>(p.out0) + off, v0, valid, vec_ok);
    }
  }
}

constexpr int kEpiWarpsT = 8;  // epilogue warps of both engines (named barrier 1)

// ---------------------------------------------------------------- epilogue tile
// One 128-row output tile of one CTA, shared by the single-CTA and CTA-pair engines.
// Called by the kEpiWarps epilogue warps after the accumulator's tmem_full wait:
//   epi_tile_compute  TMEM -> registers -> activation / gating -> out1/out2 stores and
//                     out0 (staged tile when OUT_SW > 0, else direct stores)
//   (caller: tcgen05.fence::before_thread_sync + arrive on the accumulator's empty barrier)
//   epi_tile_store    staged tile -> TMA store (one elected thread)
// `tacc` is the TMEM address of accumulator 0 for this warp's lane quarter; row0 / col0 are
// the tile's first output row / column. Staging buffers alternate per tile (`stg`); the TMA
// store issued from a buffer two tiles ago must have finished reading it.
struct EpiNoOp {
  __device__ __forceinline__ void operator()() const {}
};
// Gating backward with the reordered tile (epi_tile_compute): every staged-input read of the
// tile precedes its staging barrier, after which `after_inputs` may refill the input buffer.
template <int B, int EPI, int ACC_W>
constexpr bool early_inputs() { return EPI == EPI_GATED_BWD2 && B / 16 <= 4 && ACC_W == B; }

template <int B, int EPI, typename OutT, bool SUMACC, int OUT_SW, int NBUF = 2, int ACC_W = B,
          typename AfterInputs = EpiNoOp>
__device__ __forceinline__ void epi_tile_compute(const SpmmParams& p, uint32_t tacc, int row0,
                                                 int col0, int flags, uint8_t* stg, int half,
                                                 uint32_t q, uint32_t lane, uint32_t etid,
                                                 bool vec_ok, const uint8_t* in_stg = nullptr,
                                                 int out1_off = 0, int in1_off = 0,
                                                 AfterInputs after_inputs = AfterInputs{}) {
  const int trow = static_cast<int>(q * 32 + lane);
  const int row = row0 + trow;
  const bool row_ok = row < p.m;
  constexpr int NCH = B / 16;
  if constexpr (early_inputs<B, EPI, ACC_W>()) {
    // Gating backward: accumulator, staged inputs and the math for all of this thread's
    // chunks (c = half, half + 2) first, so they overlap the previous tile's TMA store still
    // reading the (single) output staging buffer; only the staging writes wait for it.
    const bool acc0_init = (flags & 1) != 0;
    uint32_t r[2][16];
    float da[2][16], db[2][16];
#pragma unroll
    for (int k = 0; k < 2; ++k)
      if (half + 2 * k < NCH) tmem_ld16_nowait(tacc + (half + 2 * k) * 16, r[k]);
    tmem_wait_ld();
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int c = half + 2 * k;
      if (c >= NCH) break;
      float a[16], b[16];
      unstage_chunk16<OutT, OUT_SW>(in_stg, trow, c * 16, a);
      unstage_chunk16<OutT, OUT_SW>(in_stg + in1_off, trow, c * 16, b);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float g = acc0_init ? __uint_as_float(r[k][i]) : 0.0f;
        if constexpr (sizeof(OutT) == 2)
          gated_bwd_fast(g, a[i], b[i], da[k][i], db[k][i]);
        else
          gated_bwd(g, a[i], b[i], da[k][i], db[k][i]);
      }
    }
    if (etid == 0) bulk_wait_group_read<NBUF - 1>();
    named_bar_sync(1, kEpiWarpsT * 32);
    if (etid == 0) after_inputs();  // every thread has read this tile's staged inputs
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int c = half + 2 * k;
      if (c >= NCH) break;
      stage_chunk16<OutT, OUT_SW>(stg, trow, c * 16, da[k]);
      stage_chunk16<OutT, OUT_SW>(stg + out1_off, trow, c * 16, db[k]);
    }
    return;
  }
  if constexpr ((EPI == EPI_GATED_FWD || EPI == EPI_GATED_FWD_SAVE) && OUT_SW > 0 && NCH <= 4 &&
                ACC_W == B) {
    // Staged gated forward: both accumulators and the SiLU-mul of this thread's chunks
    // (c = half, half + 2) before the output-staging wait, so they overlap the previous tile's
    // TMA store still reading the staging buffer (as the gating backward above). Same
    // arithmetic as epilogue_chunk. The inference form with a / b requested as direct outputs
    // takes the general path; the training form stages a and b next to G.
    constexpr bool kSave = EPI == EPI_GATED_FWD_SAVE;
    if (kSave || (!p.out1 && !p.out2)) {
      uint32_t r0[2][16], r1[2][16];
#pragma unroll
      for (int k = 0; k < 2; ++k)
        if (half + 2 * k < NCH) {
          tmem_ld16_nowait(tacc + (half + 2 * k) * 16, r0[k]);
          tmem_ld16_nowait(tacc + ACC_W + (half + 2 * k) * 16, r1[k]);
        }
      tmem_wait_ld();
      const bool a_init = (flags & 1) != 0, b_init = (flags & 2) != 0;
      float g[2][16];
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float a = a_init ? __uint_as_float(r0[k][i]) : 0.0f;
          const float b = b_init ? __uint_as_float(r1[k][i]) : 0.0f;
          if constexpr (sizeof(OutT) == 2)
            g[k][i] = gated_fwd_fast(a, b);
          else
            g[k][i] = gated_fwd(a, b);
        }
      if (etid == 0) bulk_wait_group_read<NBUF - 1>();
      named_bar_sync(1, kEpiWarpsT * 32);
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int c = half + 2 * k;
        if (c >= NCH) break;
        stage_chunk16<OutT, OUT_SW>(stg, trow, c * 16, g[k]);
        if constexpr (kSave) {
          float a[16], b[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            a[i] = a_init ? __uint_as_float(r0[k][i]) : 0.0f;
            b[i] = b_init ? __uint_as_float(r1[k][i]) : 0.0f;
          }
          stage_chunk16<OutT, OUT_SW>(stg + out1_off, trow, c * 16, a);
          stage_chunk16<OutT, OUT_SW>(stg + 2 * out1_off, trow, c * 16, b);
        }
      }
      return;
    }
  }
  if constexpr (OUT_SW > 0) {
    if (etid == 0) bulk_wait_group_read<NBUF - 1>();
    named_bar_sync(1, kEpiWarpsT * 32);
  }
  constexpr bool kTwoAcc = EPI == EPI_GATED_FWD || EPI == EPI_GATED_FWD_SAVE;
  // ACC_W = 2B: every accumulator is a pair (hi*hi in columns [0, B), the 3xTF32 cross terms
  // in [B, 2B)) summed here
  constexpr bool kPair = ACC_W == 2 * B;
  const bool acc0_init = SUMACC ? ((flags & 3) != 0) : ((flags & 1) != 0);
  // this warp's 16-column chunks are c = half, half + 2, ...; the TMEM loads of two chunks
  // (both accumulators when gated) are issued before one wait
#pragma unroll 1
  for (int c0 = half; c0 < NCH; c0 += 4) {
    uint32_t r0[2][16], r1[2][16];
    [[maybe_unused]] uint32_t p0[kPair ? 2 : 1][16], p1[kPair && kTwoAcc ? 2 : 1][16];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int c = c0 + 2 * k;
      if (c < NCH) {
        tmem_ld16_nowait(tacc + c * 16, r0[k]);
        if (kTwoAcc) tmem_ld16_nowait(tacc + ACC_W + c * 16, r1[k]);
        if constexpr (kPair) {
          tmem_ld16_nowait(tacc + B + c * 16, p0[k]);
          if constexpr (kTwoAcc) tmem_ld16_nowait(tacc + ACC_W + B + c * 16, p1[k]);
        }
      }
    }
    tmem_wait_ld();
    if constexpr (kPair) {
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          r0[k][i] = __float_as_uint(__fadd_rn(__uint_as_float(r0[k][i]), __uint_as_float(p0[k][i])));
          if constexpr (kTwoAcc)
            r1[k][i] = __float_as_uint(__fadd_rn(__uint_as_float(r1[k][i]), __uint_as_float(p1[k][i])));
        }
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int c = c0 + 2 * k;
      if (c >= NCH) break;
      const int col = col0 + c * 16;
      const int valid = p.n_valid - col;
      const int64_t off = static_cast<int64_t>(row) * p.ld_out + col;
      float v0[16], v1[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        v0[i] = acc0_init ? __uint_as_float(r0[k][i]) : 0.0f;
        v1[i] = kTwoAcc ? __uint_as_float(r1[k][i]) : 0.0f;
      }
      epilogue_chunk<EPI, OutT, OUT_SW>(p, v0, v1, flags, row_ok, col, valid, off, vec_ok, stg,
                                        trow, c * 16, in_stg, out1_off, in1_off);
    }
  }
}
template <int OUT_SW, int OUT_NATOM, int OUT_ELT, int NOUT = 1>
__device__ __forceinline__ void epi_tile_store(const CUtensorMap* mapO, const CUtensorMap* mapO1,
                                               const CUtensorMap* mapO2, uint8_t* stg,
                                               int out1_off, int row0, int col0, uint32_t etid,
                                               uint64_t pol_out) {
  if constexpr (OUT_SW > 0) {
    fence_proxy_async_smem();
    named_bar_sync(1, kEpiWarpsT * 32);
    if (etid == 0) {
#pragma unroll
      for (int o = 0; o < NOUT; ++o)
#pragma unroll
        for (int a = 0; a < OUT_NATOM; ++a)
          tma_store_2d_hint(o == 0 ? mapO : o == 1 ? mapO1 : mapO2,
                            stg + o * out1_off + a * (128 * OUT_SW),
                            col0 + a * (OUT_SW / OUT_ELT), row0, pol_out);
      bulk_commit_group();
    }
  }
}

// ---------------------------------------------------------------- fused TP all-reduce
__device__ __forceinline__ uint32_t atomic_add_sys(uint32_t* addr, uint32_t v) {
  uint32_t old;
  asm volatile("atom.add.sys.u32 %0, [%1], %2;" : "=r"(old) : "l"(addr), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ float4 ld_volatile_f4(const float* p) {
  return __ldcv(reinterpret_cast<const float4*>(p));
}

// Fused tensor-parallel epilogue of one 128-row output tile of the row-parallel down
// projection (partial Y summed over the TP ranks):
//   1. the tile's fp32 partial goes straight into the recv buffer of the line's owner rank
//      (peer stores over NVLink; slot [epoch parity][this rank][tile][line]);
//   2. a system-scope arrival counter on the owner counts the ranks' partials;
//   3. the rank whose partial completes the tile (whichever arrives last) sums the n partials
//      in rank order (deterministic) and writes the rounded sum into every rank's y, then
//      bumps every rank's `done` counter.
// No CTA ever waits on another GPU inside the kernel, so ranks overlap the exchange with
// their own remaining tiles; consumers wait for done[rank] (blast_tp_wait) before reading y.
// The TMEM reads come first; `release` frees the accumulator stage right after them.
template <int B, typename OutT, int ACC_W = B>
__device__ __noinline__ void epi_tp_tile(const SpmmParams& p, uint32_t tacc, int t128, int j,
                                         int flags, int half, uint32_t q, uint32_t lane,
                                         uint32_t etid, bool release, uint64_t* acc_empty,
                                         volatile int* last_flag) {
  constexpr int NCH = B / 16;
  const blast_tp_t& tp = p.tp;
  const int n = tp.n;
  const int trow = static_cast<int>(q * 32 + lane);
  const int tiles = (p.m + 127) / 128;
  const int owned = (p.n_lines + n - 1) / n;
  const int o = j % n, lo = j / n;
  const int par = static_cast<int>(tp.epoch & 1u);
  float v[NCH / 2 + 1][16];
#pragma unroll
  for (int k = 0; k < (NCH + 1) / 2; ++k) {
    const int c = half + 2 * k;
    if (c < NCH) {
      tmem_ld16(tacc + c * 16, v[k]);
      if constexpr (ACC_W == 2 * B) {  // 3xTF32 accumulator pair
        float w[16];
        tmem_ld16(tacc + B + c * 16, w);
#pragma unroll
        for (int i = 0; i < 16; ++i) v[k][i] = __fadd_rn(v[k][i], w[i]);
      }
    }
  }
  if (release) {
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(acc_empty);
  }
  const int64_t tile_elems = 128 * B;
  const int64_t slot = (((static_cast<int64_t>(par) * n + tp.rank) * tiles + t128) * owned + lo);
  float* dst = tp.recv[o] + slot * tile_elems + static_cast<int64_t>(trow) * B;
#pragma unroll
  for (int k = 0; k < (NCH + 1) / 2; ++k) {
    const int c = half + 2 * k;
    if (c >= NCH) break;
    if (!(flags & 1)) {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[k][i] = 0.0f;
    }
    float4* d4 = reinterpret_cast<float4*>(dst + c * 16);
#pragma unroll
    for (int i = 0; i < 4; ++i)
      d4[i] = make_float4(v[k][4 * i], v[k][4 * i + 1], v[k][4 * i + 2], v[k][4 * i + 3]);
  }
  __threadfence_system();
  named_bar_sync(1, kEpiWarpsT * 32);
  if (etid == 0) {
    const uint32_t old = atomic_add_sys(tp.flags[o] + static_cast<int64_t>(t128) * owned + lo, 1u);
    *last_flag = old == static_cast<uint32_t>(n) * tp.epoch + static_cast<uint32_t>(n - 1);
  }
  named_bar_sync(1, kEpiWarpsT * 32);
  if (!*last_flag) return;
  __threadfence_system();
  const int row = t128 * 128 + trow;
  if (row < p.m) {
    const float* src0 = tp.recv[o] + ((static_cast<int64_t>(par) * n * tiles + t128) * owned + lo) *
                                         tile_elems + static_cast<int64_t>(trow) * B;
    const int64_t rank_stride = static_cast<int64_t>(tiles) * owned * tile_elems;
#pragma unroll 1
    for (int c = half; c < NCH; c += 2) {
      float s[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) s[i] = 0.0f;
      for (int r = 0; r < n; ++r) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float4 f = ld_volatile_f4(src0 + r * rank_stride + c * 16 + 4 * i);
          s[4 * i] = __fadd_rn(s[4 * i], f.x);
          s[4 * i + 1] = __fadd_rn(s[4 * i + 1], f.y);
          s[4 * i + 2] = __fadd_rn(s[4 * i + 2], f.z);
          s[4 * i + 3] = __fadd_rn(s[4 * i + 3], f.w);
        }
      }
      const int col = j * B + c * 16;
      const int valid = p.n_valid - col;
      const int64_t off = static_cast<int64_t>(row) * p.ld_out + col;
      for (int r = 0; r < n; ++r)
        store_chunk16<OutT, false>(reinterpret_cast<OutT*>(tp.y[r]) + off, s, valid,
                            (p.ld_out * static_cast<int64_t>(sizeof(OutT))) % 16 == 0);
    }
  }
  __threadfence_system();
  named_bar_sync(1, kEpiWarpsT * 32);
  if (etid == 0)
    for (int r = 0; r < n; ++r) atomic_add_sys(tp.done[r], 1u);
}

// per-stage MMA recipe bits (producer -> MMA warp through shared memory)
constexpr uint32_t kMetaHas0 = 1u;        // block of matrix 0 in this stage
constexpr uint32_t kMetaHas1 = 2u;        // block of matrix 1 in this stage
constexpr uint32_t kMetaMerged = 4u;      // one N = 2B MMA covers both (gate | up)
constexpr uint32_t kMetaAccFirst = 8u;    // first MMA group accumulates (else overwrites)
constexpr uint32_t kMetaAccSecond = 16u;  // second MMA group accumulates
constexpr uint32_t kMetaLast = 32u;       // SPLIT: last stage of the item

// MMA recipe of one step {a_blk, k0, k1}: presence, merge and accumulate flags. init0/init1
// track which accumulators already hold a partial sum of the current output line.
template <int NMAT, bool SUMACC, bool MERGE>
__device__ __forceinline__ uint32_t step_recipe(const int4& st, uint32_t& init0, uint32_t& init1) {
  const bool has0 = st.y >= 0, has1 = NMAT > 1 && st.z >= 0;
  uint32_t meta = (has0 ? kMetaHas0 : 0u) | (has1 ? kMetaHas1 : 0u);
  if (MERGE && has0 && has1 && init0 == init1) {
    meta |= kMetaMerged | (init0 ? kMetaAccFirst : 0u);
    init0 = init1 = 1;
  } else {
    if (has0) { meta |= init0 ? kMetaAccFirst : 0u; init0 = 1; }
    if (has1) {
      if (SUMACC) { meta |= init0 ? kMetaAccSecond : 0u; init0 = 1; }
      else { meta |= init1 ? kMetaAccSecond : 0u; init1 = 1; }
    }
  }
  return meta;
}

// Named barriers (ids; 0 = __syncthreads, 1 = epilogue warps). The MMA warp never waits on an
// mbarrier or reads shared memory itself: both stall its issue until its in-flight MMAs
// drain (tools/mma_probe.cu P8: 354 vs 205 cycles per 4 x N=64 step). Warp 2 waits on the
// mbarriers instead and releases the MMA warp through these hardware barriers.
constexpr uint32_t kBarAcc = 2;    // + accumulator stage (2 ids)
constexpr uint32_t kBarStage = 4;  // + ring stage (<= 8 ids)
// Measured on cfg3 (b = 64): the waiter handoff wins for single-matrix products (down
// projection 124 -> 118 us) but loses for the gate+up product, whose 48 KB stages leave only
// 4 in flight so the extra handoff latency is exposed (237 -> 247 us); there the MMA warp
// waits on the mbarriers itself.
#ifndef BLAST_WAITER_GU
#define BLAST_WAITER_GU 0
#endif
#ifndef BLAST_BALLOT_GU
#define BLAST_BALLOT_GU 0
#endif
// SPLIT = 2 (sequential gate+up) always uses the waiter: its recipe is the stage index.
template <int NMAT, int TM, int SPLIT = 0>
constexpr bool use_waiter() { return SPLIT == 2 || (SPLIT == 0 && (NMAT == 1 || BLAST_WAITER_GU)); }

// 12 warps: 0 TMA producer, 1 MMA issuer, 2 TMEM allocator, 3 idle, 4..11 epilogue
// (two warps per TMEM lane quarter, splitting the 16-column chunks).
constexpr int kTcThreads = 384;
constexpr int kEpiWarps = kEpiWarpsT;

template <int EPI, int OUT_ELT>
constexpr int in_staged() {
  return OUT_ELT == 0 ? 0 : EPI == EPI_GATED_BWD ? 1 : EPI == EPI_GATED_BWD2 ? 2 : 0;
}

template <int B, int ELT, int NPASS, int NMAT, bool SUMACC, bool B_KMAJOR, int EPI, typename OutT,
          int OUT_ELT = 0, int TM = 1, int SPLIT = 0>
__global__ void __launch_bounds__(kTcThreads, 1)
spmm_tc_kernel(const __grid_constant__ CUtensorMap mapO, const __grid_constant__ CUtensorMap mapI,
               const __grid_constant__ CUtensorMap mapO1, const __grid_constant__ CUtensorMap mapI1,
               const __grid_constant__ CUtensorMap mapO2,
               const __grid_constant__ CUtensorMap mapA0, const __grid_constant__ CUtensorMap mapA0lo,
               const __grid_constant__ CUtensorMap mapA1, const __grid_constant__ CUtensorMap mapA1lo,
               const __grid_constant__ CUtensorMap mapW0, const __grid_constant__ CUtensorMap mapW0lo,
               const __grid_constant__ CUtensorMap mapW1, const __grid_constant__ CUtensorMap mapW1lo,
               const SpmmParams p) {
  constexpr int IN_ST = in_staged<EPI, OUT_ELT>();
  using C = TcCfg<B, ELT, NPASS, NMAT, SUMACC, B_KMAJOR, OUT_ELT, TM, IN_ST, SPLIT,
                  staged_outputs<EPI>()>;
  static_assert(!SPLIT || (NMAT == 2 && (NPASS == 1 || SPLIT == 2) &&
                           (SPLIT == 2) == use_waiter<NMAT, TM, SPLIT>()),
                "split stages: gate+up products only");
  static_assert(!C::SK || NMAT == 1 || SPLIT == 2, "3xTF32 two-matrix products: sequential layout");
  static_assert(OUT_ELT == 0 || OUT_ELT == static_cast<int>(sizeof(OutT)), "staged output type");
#ifdef BLAST_WAIT_COUNTERS
  const long long t_kernel0 = clock64();
  if (p.dbg && threadIdx.x == 0) p.dbg[kDbgSlots + 2 * blockIdx.x] = globaltimer_ns();
#endif
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* staging = smem + C::STAGES * C::STAGE;  // [2][OUT_TILE] when OUT_ELT > 0
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE + C::STAGING);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tmem_full = empty + C::STAGES;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
  // per-stage MMA recipe (when the MMA warp waits on the mbarriers itself): written by the
  // producer before its expect_tx arrive (release), read after the full wait (acquire)
  uint32_t* stage_meta = tmem_slot + 4;
  uint64_t* in_full = reinterpret_cast<uint64_t*>(stage_meta + 8);  // [2] staged in0 landed
  uint8_t* in_staging = staging + C::OUT_BUFS * C::NOUT * C::OUT_TILE;  // [2][IN_ST][OUT_TILE]

  const uint32_t warp = __shfl_sync(0xffffffffu, warp_id(), 0);
  const uint32_t lane = lane_id();
  // items: (token tile, line); this CTA's sequence is item_at(p, 0), item_at(p, 1), ...
  const int n_items = p.n_tok_tiles * p.n_lines;
  auto tile_of = [&](int item) -> int { return item_tile(p, item); };

  if (warp == 0 && lane == 0) {
    if (OUT_ELT) tma_prefetch(&mapO);
    if (C::NOUT > 1) tma_prefetch(&mapO1);
    if (C::NOUT > 2) tma_prefetch(&mapO2);
    if (IN_ST == 2) tma_prefetch(&mapI1);
    tma_prefetch(&mapA0);
    tma_prefetch(&mapW0);
    if (NMAT > 1) tma_prefetch(&mapW1);
    if (SUMACC) tma_prefetch(&mapA1);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tmem_full[s], 1);
      mbar_init(&tmem_empty[s], kEpiWarps);
    }
    mbar_init(&in_full[0], 1);
    mbar_init(&in_full[1], 1);
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
  // Everything above (barriers, TMEM, descriptor prefetch) may overlap the previous kernel's
  // tail under programmatic dependent launch; nothing below runs before it has completed.
  griddep_wait();
  // every CTA of this persistent grid is resident: the next engine launch may now take SMs as
  // CTAs of this grid exit (it still waits for our completion). Decode-size products only:
  // cfg3 shape at 95 %, 128 tokens, graph replay 18.6 -> 17.0 us (24.6 -> 22.5 us with the L2
  // flushed); on the 8192-token training step the trigger cost 0.3 %
  // (profiles/r02/late/early_trigger_ab.txt)
  if (BLAST_EARLY_TRIGGER && p.early_trigger) griddep_launch_dependents();
  WaitClock wc;
#ifdef BLAST_WAIT_COUNTERS
  const bool dbg_on = p.dbg != nullptr;
#else
  constexpr bool dbg_on = false;  // keep the role loops free of diagnosis code
#endif

  if (warp == 0 || warp == 3) {
    // ------------------------------------------------------------ TMA producers
    // Two warps walk the same schedule (warp-uniform control flow keeps the loop
    // state in uniform registers); warp 0 issues the copies of even steps, warp 3
    // those of odd steps, so the per-step issue latency is overlapped. One elected
    // lane issues each copy.
    const uint64_t pol_w = policy_evict_last();
    // sequential gate+up / dX panels: L2 evict_last like the weights (X and W stay resident
    // against the streamed G stores; cfg3 0.3382-0.3390 vs 0.3396-0.3402 ms, tools/ab_lib.sh)
#ifndef BLAST_A_POLICY
#define BLAST_A_POLICY 2
#endif
    const uint64_t pol_a = BLAST_A_POLICY == 2 ? policy_evict_last() : policy_evict_normal();
    const uint32_t mine = warp == 0 ? 0u : 1u;
    uint32_t stage = 0, phase = 0, n = 0;
    constexpr bool kMergeP = (NMAT == 2) && !SUMACC && !B_KMAJOR && (2 * B <= 256) &&
                             (C::NATOM == 1 || C::B_TILE == C::NATOM * B * C::SW);
    // The next item's step range and first 32 steps are fetched one item ahead, so
    // the item boundary does not stall the ring on two dependent global loads.
    int nx_s0 = 0, nx_s1 = 0;
    int4 nx_first = make_int4(0, -1, -1, 0);
    auto prefetch = [&](int item) {
      if (item >= n_items) return;
      const int jn = item % p.n_lines;
      nx_s0 = __ldg(&p.step_ptr[jn]);
      nx_s1 = __ldg(&p.step_ptr[jn + 1]);
      const int idx = nx_s0 + static_cast<int>(lane);
      nx_first = idx < nx_s1 ? __ldg(&p.steps[idx]) : make_int4(0, -1, -1, 0);
    };
    prefetch(item_at(p, 0, n_items));
    if constexpr (SPLIT == 2) {
      // sequential gate+up: pass 0 loads the line's gate blocks, pass 1 its up blocks; one
      // panel + one weight block (slot 0) per stage
      for (int k = 0, item = item_at(p, 0, n_items); item < n_items;
           item = item_at(p, ++k, n_items)) {
        const int t = tile_of(item);
        const int s0 = nx_s0, s1 = nx_s1;
        const int4 first = nx_first;
        prefetch(item_at(p, k + 1, n_items));
#pragma unroll 1
        for (int pass = 0; pass < 2; ++pass) {
          StepCursor cur;
          cur.steps = p.steps;
          cur.end = s1;
          cur.base = s0;
          cur.mine = first;
          for (int s = s0; s < s1; ++s) {
            const int4 st = cur.get(s);
            const int kb = pass == 0 ? st.y : st.z;
            if (kb < 0) continue;
#pragma unroll 1
            for (int sa = 0; sa < C::SPS; ++sa) {  // SK: one stage per K atom of the block
              if ((n++ & 1u) != mine) {
                if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
                continue;
              }
              wc.wait(0, &empty[stage], phase ^ 1, dbg_on);
              if (elect_one()) {
                uint8_t* sbase = smem + stage * C::STAGE;
                if (kDiagSwitches && (p.skip_epilogue & 2)) {  // diagnosis: stale operands
                  mbar_arrive(&full[stage]);
                } else {
                  mbar_expect_tx(&full[stage], C::NCOPY * (C::A_BYTES + C::B_BYTES));
                  const bool a1 = SUMACC && pass == 1;
#pragma unroll
                  for (int c = 0; c < C::NCOPY; ++c)
#pragma unroll
                    for (int at = 0; at < C::KPS; ++at)
                      tma_load_2d_hint(sbase + c * C::A_TILE + at * C::TROWS * C::SW,
                                       c == 0 ? (a1 ? &mapA1 : &mapA0) : (a1 ? &mapA1lo : &mapA0lo),
                                       &full[stage], st.x * B + (C::SK ? sa : at) * C::SWE,
                                       t * C::TROWS, pol_a);
#pragma unroll
                  for (int c = 0; c < C::NCOPY; ++c)
#pragma unroll
                    for (int at = 0; at < C::KPS; ++at)
                      tma_load_2d_hint(sbase + C::NCOPY * C::A_TILE + c * C::B_TILE + at * B * C::SW,
                                       c == 0 ? (pass == 0 ? &mapW0 : &mapW1)
                                              : (pass == 0 ? &mapW0lo : &mapW1lo),
                                       &full[stage], (C::SK ? sa : at) * C::SWE, kb * B, pol_w);
                }
              }
              __syncwarp();
              if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
            }
          }
        }
      }
    } else
    for (int k = 0, item = item_at(p, 0, n_items); item < n_items;
         item = item_at(p, ++k, n_items)) {
      const int t = tile_of(item);
      const int s0 = nx_s0, s1 = nx_s1;
      StepCursor cur;
      cur.steps = p.steps;
      cur.end = s1;
      cur.base = s0;
      cur.mine = nx_first;
      prefetch(item_at(p, k + 1, n_items));
      uint32_t init0 = 0, init1 = 0;  // accumulator i already holds a partial sum
      for (int s = s0; s < s1; ++s) {
        const int4 st = cur.get(s);
        // SPLIT: a step holding both a gate and an up block becomes two stages
        const bool both = SPLIT && st.y >= 0 && st.z >= 0;
        const int nparts = both ? 2 : 1;
#pragma unroll 1
        for (int part = 0; part < nparts; ++part) {
        const int kb[2] = {(both && part == 1) ? -1 : st.y, (both && part == 0) ? -1 : st.z};
        uint32_t meta = step_recipe<NMAT, SUMACC, kMergeP && !SPLIT>(make_int4(st.x, kb[0], kb[1], 0),
                                                                     init0, init1);
        if (SPLIT && s + 1 == s1 && part + 1 == nparts) meta |= kMetaLast;
#pragma unroll 1
        for (int sa = 0; sa < C::SPS; ++sa) {  // SK: one stage per K atom of the block(s)
        if ((n++ & 1u) != mine) {
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
          continue;
        }
        wc.wait(0, &empty[stage], phase ^ 1, dbg_on);
        if (elect_one()) {
          uint32_t bytes = 0;
#pragma unroll
          for (int a = 0; a < C::NA; ++a)
            if (!SUMACC || kb[a] >= 0) bytes += C::NCOPY * C::A_BYTES;
#pragma unroll
          for (int mm = 0; mm < NMAT; ++mm)
            if (kb[mm] >= 0) bytes += C::NCOPY * C::B_BYTES;
          if (!use_waiter<NMAT, TM, SPLIT>()) stage_meta[stage] = meta;
          if (kDiagSwitches && (p.skip_epilogue & 2)) {  // diagnosis: stale operands
            mbar_arrive(&full[stage]);
            bytes = 0;
          } else {
            mbar_expect_tx(&full[stage], bytes);
          }
          uint8_t* sbase = smem + stage * C::STAGE;
#pragma unroll
          for (int a = 0; a < C::NA; ++a) {
            if (kDiagSwitches && bytes == 0) break;
            if (SUMACC && kb[a] < 0) continue;
            const CUtensorMap* mh = (a == 0) ? &mapA0 : &mapA1;
            const CUtensorMap* ml = (a == 0) ? &mapA0lo : &mapA1lo;
#pragma unroll
            for (int c = 0; c < C::NCOPY; ++c) {
              uint8_t* dst = sbase + (a * C::NCOPY + c) * C::A_TILE;
#pragma unroll
              for (int at = 0; at < C::KPS; ++at)
                tma_load_2d(dst + at * C::TROWS * C::SW, c == 0 ? mh : ml, &full[stage],
                            st.x * B + (C::SK ? sa : at) * C::SWE, t * C::TROWS);
            }
          }
#pragma unroll
          for (int mm = 0; mm < NMAT; ++mm) {
            if (kb[mm] < 0 || (kDiagSwitches && bytes == 0)) continue;
            const CUtensorMap* mh = (mm == 0) ? &mapW0 : &mapW1;
            const CUtensorMap* ml = (mm == 0) ? &mapW0lo : &mapW1lo;
            const int slot = SPLIT ? 0 : mm;
#pragma unroll
            for (int c = 0; c < C::NCOPY; ++c) {
              uint8_t* dst = sbase + C::NA * C::NCOPY * C::A_TILE + (slot * C::NCOPY + c) * C::B_TILE;
#pragma unroll
              for (int at = 0; at < C::KPS; ++at) {
                tma_load_2d_hint(dst + at * B * C::SW, c == 0 ? mh : ml, &full[stage],
                                 (C::SK ? sa : at) * C::SWE, kb[mm] * B, pol_w);
              }
            }
          }
        }
        __syncwarp();
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // Descriptors are built once for stage 0 and advanced by adding byte offsets
    // >> 4 to the start-address field (no carry: shared addresses < 2^18).
    const uint32_t smem0 = smem_u32(smem);
    const uint64_t a_desc0 = kmajor_desc<C::SW, C::MMA_K, ELT>(smem0, C::TROWS, 0);
    const uint32_t b_off = C::NA * C::NCOPY * C::A_TILE;
    const uint64_t b_desc0 = B_KMAJOR ? kmajor_desc<C::SW, C::MMA_K, ELT>(smem0 + b_off, B, 0)
                                      : mnmajor_desc<C::SW, C::MMA_K, B>(smem0 + b_off, 0);
    // merged gate+up: one N = 2B MMA over [W_gate | W_up] (adjacent MN-major atoms)
    constexpr bool kMerge = (NMAT == 2) && !SUMACC && !B_KMAJOR && (2 * B <= 256) &&
                            (C::NATOM == 1 || C::B_TILE == C::NATOM * B * C::SW);
    constexpr uint32_t kMergeLbo = C::NATOM == 1 ? C::B_TILE : B * C::SW;
    const uint64_t b_desc0_merged =
        make_sdesc(smem0 + b_off, kMergeLbo, 8u * C::SW, swizzle_layout_code(C::SW));
    constexpr uint32_t kIdescMerged = make_idesc(C::BM, kMerge ? 2 * B : B, ELT == 2 ? 1u : 2u, 0u,
                                                 B_KMAJOR ? 0u : 1u);
    // per-K-slice descriptor increments (in 16-byte units)
    auto a_koff = [](int ks) -> uint32_t {
      const uint32_t byte_k = static_cast<uint32_t>(ks) * C::MMA_K * ELT;
      return ((byte_k / C::SW) * C::TROWS * C::SW + (byte_k % C::SW)) >> 4;
    };
    auto b_koff = [](int ks) -> uint32_t {
      if (B_KMAJOR) {
        const uint32_t byte_k = static_cast<uint32_t>(ks) * C::MMA_K * ELT;
        return ((byte_k / C::SW) * B * C::SW + (byte_k % C::SW)) >> 4;
      }
      return (static_cast<uint32_t>(ks) * C::MMA_K * C::SW) >> 4;
    };
    // One stage's MMAs for one 128-row half into accumulator `d` (init: accumulate into it).
    // bf16 / tf32: KSL_ST K slices of N = B. SK (3xTF32): per K slice A_hi x [W_hi; W_lo]
    // (N = 2B) into the pair (d, d + B), then A_lo x W_hi into d + B.
    auto issue_stage = [&](uint32_t d, uint64_t ad, uint64_t bd, uint32_t init) {
#pragma unroll
      for (int ks = 0; ks < C::KSL_ST; ++ks) {
        const uint32_t acc_flag = (init | ks) ? 1u : 0u;
        if constexpr (C::SK) {
          mma_tf32(d, ad + a_koff(ks), bd + b_koff(ks), C::IDESC_PAIR, acc_flag);
          mma_tf32(d + B, ad + (C::A_TILE >> 4) + a_koff(ks), bd + b_koff(ks), C::IDESC, 1u);
        } else if constexpr (ELT == 4) {
          mma_tf32(d, ad + a_koff(ks), bd + b_koff(ks), C::IDESC, acc_flag);
        } else {
          mma_f16(d, ad + a_koff(ks), bd + b_koff(ks), C::IDESC, acc_flag);
        }
      }
    };
    constexpr bool kWaiter = use_waiter<NMAT, TM, SPLIT>();
    uint32_t stage = 0, phase = 0, it = 0;
    // kWaiter: the step list is walked here (next item's first 32 steps fetched one item
    // ahead; recipes from two presence ballots per 32 steps), so the per-step loop issues no
    // shared-memory reads or shuffles between MMAs. Otherwise only the step count is needed
    // and the recipe comes from the producer through shared memory.
    int nx_s0 = 0, nx_s1 = 0;
    int4 nx_first = make_int4(0, -1, -1, 0);
    // kBallot: the MMA warp derives each step's recipe from the step list itself (no
    // shared-memory read queued behind the in-flight MMAs' operand reads)
    // (single-matrix plans hold only present blocks: every step is one block of matrix 0)
    constexpr bool kBallot = NMAT > 1 && (kWaiter || (!SPLIT && BLAST_BALLOT_GU));
    auto prefetch = [&](int item) {
      if (item >= n_items) return;
      const int jn = item % p.n_lines;
      nx_s0 = __ldg(&p.step_ptr[jn]);
      nx_s1 = __ldg(&p.step_ptr[jn + 1]);
      if constexpr (kBallot) {
        const int idx = nx_s0 + static_cast<int>(lane);
        nx_first = idx < nx_s1 ? __ldg(&p.steps[idx]) : make_int4(0, -1, -1, 0);
      }
    };
    const long long t_loop = dbg_on ? clock64() : 0;
    if constexpr (SPLIT == 2) {
      // sequential gate+up: stage i of an item is gate block i (i < n0) or up block i - n0
      int nxt = item_at(p, 0, n_items);
      int nx_fl = nxt < n_items ? __ldg(&p.line_flags[nxt % p.n_lines]) : 0;
      for (int k = 0, item = nxt; item < n_items; item = nxt, ++k, ++it) {
        const uint32_t as = it & 1;
        const int fl = nx_fl;
        nxt = item_at(p, k + 1, n_items);
        if (nxt < n_items) nx_fl = __ldg(&p.line_flags[nxt % p.n_lines]);
        const int n0 = (fl >> 2) & 0x7fff, n = n0 + ((fl >> 17) & 0x7fff);
        named_bar_sync(kBarAcc + as, 64);  // warp 2 saw tmem_empty[as]
        tc_fence_after();
        const uint32_t d_base = tmem_base + as * C::ACC_STRIDE;
        for (int i = 0; i < n; ++i) {
          // SUMACC (dX = dA Wg^T + dB Wu^T): both passes accumulate into one accumulator
          const uint32_t sel = (!SUMACC && i >= n0) ? 1u : 0u;
          const uint32_t init = SUMACC ? (i != 0 ? 1u : 0u) : ((i != 0 && i != n0) ? 1u : 0u);
#pragma unroll 1
          for (int sa = 0; sa < C::SPS; ++sa) {  // SK: the block's K atoms, one stage each
            named_bar_sync(kBarStage + stage, 64);  // warp 2 saw full[stage]
            tc_fence_after();
            const long long ti0 = dbg_on ? clock64() : 0;
            if (elect_one()) {
              const uint32_t soff = (stage * C::STAGE) >> 4;
              const uint64_t bb = b_desc0 + soff;
#pragma unroll
              for (int h = 0; h < TM; ++h) {
                const uint64_t ad = a_desc0 + soff + ((h * C::BM * C::SW) >> 4);
                const uint32_t d = d_base + h * C::HALF_ACC + sel * C::ACC_W;
                issue_stage(d, ad, bb, (init | (sa != 0 ? 1u : 0u)));
              }
              mma_commit(&empty[stage]);
            }
            __syncwarp();
            if (dbg_on) {
              wc.acc[6] += static_cast<unsigned long long>(clock64() - ti0);
              wc.acc[7] += 1;
            }
            if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
          }
        }
        if (elect_one()) mma_commit(&tmem_full[as]);
        __syncwarp();
      }
    } else {
    prefetch(item_at(p, 0, n_items));
    for (int k = 0, item = item_at(p, 0, n_items); item < n_items;
         item = item_at(p, ++k, n_items), ++it) {
      const uint32_t as = it & 1;
      const int s0 = nx_s0, s1 = nx_s1;
      int4 mine = nx_first;
      prefetch(item_at(p, k + 1, n_items));
      if constexpr (kWaiter)
        named_bar_sync(kBarAcc + as, 64);  // warp 2 saw tmem_empty[as]
      else
        wc.wait(3, &tmem_empty[as], ((it >> 1) & 1) ^ 1, dbg_on);
      tc_fence_after();
      const uint32_t d_base = tmem_base + as * C::ACC_STRIDE;
      bool done = s0 >= s1;  // SPLIT: an item's stages end at the producer's kMetaLast
      for (int s = s0; SPLIT ? !done : s < s1; ++s) {
        uint32_t meta = 0;
        if constexpr (NMAT == 1) {
          meta = kMetaHas0 | (s != s0 ? kMetaAccFirst : 0u);
        } else if constexpr (kBallot) {
          // the plan's per-step bits (plan.cu): presence and first block of each matrix
          const int i = (s - s0) & 31;
          if (i == 0 && s != s0) {  // next 32 steps of a long line
            const int idx = s + static_cast<int>(lane);
            mine = idx < s1 ? __ldg(&p.steps[idx]) : make_int4(0, -1, -1, 0);
          }
          const uint32_t w = static_cast<uint32_t>(__shfl_sync(0xffffffffu, mine.w, i));
          const bool has0 = w & 1u, has1 = (w & 2u) != 0;
          // accumulator already holds a partial sum before this step
          const bool init0 = SUMACC ? s != s0 : !(w & 4u);
          const bool init1 = !(w & 8u);
          meta = (has0 ? kMetaHas0 : 0u) | (has1 ? kMetaHas1 : 0u);
          if (kMerge && has0 && has1 && init0 == init1) {
            meta |= kMetaMerged | (init0 ? kMetaAccFirst : 0u);
          } else {
            meta |= init0 ? kMetaAccFirst : 0u;
            if (SUMACC) meta |= (init0 || has0) ? kMetaAccSecond : 0u;
            else meta |= init1 ? kMetaAccSecond : 0u;
          }
        }
#pragma unroll 1
        for (int sa = 0; sa < C::SPS; ++sa) {  // SK (single-matrix): one stage per K atom
        if constexpr (NMAT == 1 || kBallot) {
          if constexpr (kWaiter) {
            const long long tw0 = dbg_on ? clock64() : 0;
            named_bar_sync(kBarStage + stage, 64);  // warp 2 saw full[stage]
            if (dbg_on) wc.acc[2] += static_cast<unsigned long long>(clock64() - tw0);
          } else {
            wc.wait(2, &full[stage], phase, dbg_on);
          }
          tc_fence_after();
        } else {
          wc.wait(2, &full[stage], phase, dbg_on);
          tc_fence_after();
          meta = ld_shared_u32(&stage_meta[stage]);  // the producer's recipe
          if (SPLIT) done = (meta & kMetaLast) != 0;
        }
        if (sa != 0) meta |= kMetaAccFirst | kMetaAccSecond;  // later K atoms accumulate
        const long long ti0 = dbg_on ? clock64() : 0;
        if (elect_one()) {
          const uint32_t soff = (stage * C::STAGE) >> 4;
          const uint64_t bd = b_desc0 + soff;
#pragma unroll
          for (int h = 0; h < TM; ++h) {
            // half h: rows [h*128, h*128+128) of the panel, its own accumulator columns
            const uint64_t ad = a_desc0 + soff + ((h * C::BM * C::SW) >> 4);
            const uint32_t dh = d_base + h * C::HALF_ACC;
            if (kMerge && (meta & kMetaMerged)) {
              const uint32_t acc = (meta & kMetaAccFirst) ? 1u : 0u;
#pragma unroll
              for (int ks = 0; ks < C::KSL; ++ks)
                mma_f16(dh, ad + a_koff(ks), b_desc0_merged + soff + b_koff(ks), kIdescMerged,
                        (acc | ks) ? 1u : 0u);
            } else {
#pragma unroll
              for (int mm = 0; mm < NMAT; ++mm) {
                if (!(meta & (mm == 0 ? kMetaHas0 : kMetaHas1))) continue;
                const int acc_i = SUMACC ? 0 : mm;
                const int a_i = SUMACC ? mm : 0;
                const uint32_t init =
                    (meta & (mm == 0 ? kMetaAccFirst : kMetaAccSecond)) ? 1u : 0u;
                issue_stage(dh + acc_i * C::ACC_W, ad + ((a_i * C::NCOPY * C::A_TILE) >> 4),
                            bd + (((SPLIT ? 0 : mm) * C::NCOPY * C::B_TILE) >> 4), init);
              }
            }
          }
          mma_commit(&empty[stage]);
        }
        __syncwarp();
        if (dbg_on) {
          wc.acc[6] += static_cast<unsigned long long>(clock64() - ti0);
          wc.acc[7] += 1;
        }
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
      if (elect_one()) mma_commit(&tmem_full[as]);
      __syncwarp();
    }
    }
    if (dbg_on) wc.acc[4] += static_cast<unsigned long long>(clock64() - t_loop);
  } else if (warp == 2 && use_waiter<NMAT, TM, SPLIT>()) {
    // ------------------------------------------------------------ barrier waiter
    // Mirrors the MMA warp's item / step sequence: waits on the accumulator-free and
    // stage-full mbarriers and releases the MMA warp through named barriers.
    uint32_t stage = 0, phase = 0, it = 0;
    for (int k = 0, item = item_at(p, 0, n_items); item < n_items;
         item = item_at(p, ++k, n_items), ++it) {
      const uint32_t as = it & 1, use = it >> 1;
      const int j = item % p.n_lines;
      int n_steps;
      if constexpr (SPLIT == 2) {
        const int fl = __ldg(&p.line_flags[j]);
        n_steps = ((fl >> 2) & 0x7fff) + ((fl >> 17) & 0x7fff);
      } else {
        n_steps = __ldg(&p.step_ptr[j + 1]) - __ldg(&p.step_ptr[j]);
      }
      n_steps *= C::SPS;  // SK: one stage per K atom of every block
      wc.wait(3, &tmem_empty[as], (use & 1) ^ 1, dbg_on);
      named_bar_arrive(kBarAcc + as, 64);
      for (int s = 0; s < n_steps; ++s) {
        wc.wait(2, &full[stage], phase, dbg_on);
        named_bar_arrive(kBarStage + stage, 64);
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const uint32_t q = warp & 3;                 // TMEM lane quarter
    const int half = static_cast<int>(warp - 4) >> 2;  // which 16-column chunks
    const uint32_t etid = threadIdx.x - 128;     // 0..255 over the epilogue warps
    // outputs stream through L2 (evict first) so they do not push out the re-read
    // activation panels and weight blocks
    const uint64_t pol_out = policy_evict_first();
    uint32_t it = 0;
    const bool vec_ok = (p.ld_out * static_cast<int64_t>(sizeof(OutT))) % 16 == 0;
    [[maybe_unused]] auto load_in = [&](int itm, int h, uint32_t buf) {
      const int tt = tile_of(itm), jj = itm % p.n_lines;
      mbar_expect_tx(&in_full[buf], IN_ST * C::BM * C::OUT_ROWB);
#pragma unroll
      for (int i = 0; i < IN_ST; ++i)
#pragma unroll
        for (int a = 0; a < C::OUT_NATOM; ++a)
          tma_load_2d(in_staging + (buf * IN_ST + i) * C::OUT_TILE + a * (C::BM * C::OUT_SW),
                      i == 0 ? &mapI : &mapI1, &in_full[buf], jj * B + a * (C::OUT_SW / OUT_ELT),
                      tt * C::TROWS + h * C::BM);
    };
    for (int k = 0, item = item_at(p, 0, n_items); item < n_items;
         item = item_at(p, ++k, n_items), ++it) {
      const int t = tile_of(item);
      const int j = item % p.n_lines;
      const uint32_t as = it & 1, use = it >> 1;
      const int flags = __ldg(&p.line_flags[j]);
      // in0 (and in1) tiles per 128-row half, two buffers indexed by the half's sequence
      // number: the first two halves are requested up front, half seq + 2 as soon as every
      // thread has read half seq's inputs (mid-tile for the reordered gating backward, after
      // the tile's store barrier otherwise).
      [[maybe_unused]] auto load_half = [&](uint32_t seq) {
        const int kk = static_cast<int>(seq / TM), hh = static_cast<int>(seq % TM);
        const int itm = item_at(p, kk, n_items);
        if (itm < n_items) load_in(itm, hh, seq & 1);
      };
      if constexpr (IN_ST) {
        if (etid == 0 && it == 0) {
          load_half(0);
          load_half(1);
        }
      }
      wc.wait(5, &tmem_full[as], use & 1, dbg_on);
      tc_fence_after();
      if (kDiagSwitches && (p.skip_epilogue & 1)) {  // diagnosis: release the accumulator unread
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tmem_empty[as]);
        continue;
      }
      if constexpr (NMAT == 1 && EPI == EPI_STORE) {
        if (p.tp.n > 0) {  // fused TP all-reduce of the row-parallel down projection
#pragma unroll 1
          for (int h = 0; h < TM; ++h)
            epi_tp_tile<B, OutT, C::ACC_W>(p, tmem_base + ((q * 32u) << 16) + as * C::ACC_STRIDE +
                                        h * C::HALF_ACC,
                                 t * TM + h, j, flags, half, q, lane, etid, h == TM - 1,
                                 &tmem_empty[as], reinterpret_cast<volatile int*>(in_full + 2));
          continue;
        }
      }
#pragma unroll
      for (int h = 0; h < TM; ++h) {
        const uint32_t seq = it * TM + h;  // half sequence number of this CTA
        if constexpr (IN_ST) wc.wait(8, &in_full[seq & 1], (seq >> 1) & 1, dbg_on);
        constexpr bool kEarly = IN_ST && early_inputs<B, EPI, C::ACC_W>();
        auto refill = [&]() {
          if constexpr (IN_ST) load_half(seq + 2);
        };
        uint8_t* stg = staging + ((it * TM + h) % C::OUT_BUFS) * C::NOUT * C::OUT_TILE;
        const uint32_t tacc =
            tmem_base + ((q * 32u) << 16) + as * C::ACC_STRIDE + h * C::HALF_ACC;
        const int row0 = t * C::TROWS + h * C::BM;
        const long long te0 = dbg_on ? clock64() : 0;
        epi_tile_compute<B, EPI, OutT, SUMACC, C::OUT_SW, C::OUT_BUFS, C::ACC_W>(
            p, tacc, row0, j * B, flags, stg, half, q, lane, etid, vec_ok,
            IN_ST ? in_staging + (seq & 1) * IN_ST * C::OUT_TILE : nullptr,
            C::OUT_TILE, C::OUT_TILE, [&]() {
              if constexpr (kEarly) refill();
            });
        if (h == TM - 1) {  // every TMEM read of this accumulator stage is done
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tmem_empty[as]);
        }
        epi_tile_store<C::OUT_SW, C::OUT_NATOM, OUT_ELT, C::NOUT>(&mapO, &mapO1, &mapO2, stg,
                                                                  C::OUT_TILE, row0, j * B, etid,
                                                                  pol_out);
        if (!kEarly && etid == 0) refill();  // the store barrier ordered every input read
        if (dbg_on) wc.acc[9] += static_cast<unsigned long long>(clock64() - te0);
      }
    }
    if constexpr (OUT_ELT > 0) {
      if (etid == 0) bulk_wait_group<0>();
    }
  }

#ifdef BLAST_WAIT_COUNTERS
  if (warp == 4 && dbg_on) {
    wc.acc[1] += static_cast<unsigned long long>(clock64() - t_kernel0);
    if (lane == 0) p.dbg[kDbgSlots + 2 * blockIdx.x + 1] = globaltimer_ns();
  }
#endif
  if (warp <= 2 || warp == 4) wc.flush(p.dbg);
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

}  // namespace blast
