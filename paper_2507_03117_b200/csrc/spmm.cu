// Host dispatch of the block-sparse engine and the C-ABI product entry points:
// blast_bspmm (kernels.py:86/127), blast_bspmm_rt (kernels.py:143),
// blast_mlp_forward (mlp.py:102), blast_mlp_backward_dgrad (mlp.py:118-142).
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "host.hpp"
#include "spmm_simt.cuh"
#include "spmm_tc.cuh"

namespace blast {

struct EngineCall {
  int dtype = BLAST_BF16;
  int block = 0;
  bool transposed = false;
  int nmat = 1;
  bool sumacc = false;
  int epi = EPI_STORE;
  int act = ACT_NONE;
  int accumulate = 0;
  int64_t m = 0;
  int64_t a_cols = 0;  // columns (and row pitch) of the A sources
  const void* a0 = nullptr;
  const void* a1 = nullptr;
  // F32: activations already split into tf32 hi (a0 / a1) and lo parts (e.g. G written split by
  // the gate+up epilogue); when null the engine splits a0 / a1 itself
  const void* a0_lo = nullptr;
  const void* a1_lo = nullptr;
  const void* w0 = nullptr;
  const void* w0_hi = nullptr;  // F32: 3xTF32 operands (K-major image of the blocks)
  const void* w0_lo = nullptr;
  int64_t nnzb0 = 0;
  const void* w1 = nullptr;
  const void* w1_hi = nullptr;
  const void* w1_lo = nullptr;
  int64_t nnzb1 = 0;
  int64_t n_lines = 0, n_valid = 0;
  const int32_t* step_ptr = nullptr;
  const int32_t* steps = nullptr;
  const int32_t* flags = nullptr;
  void* out0 = nullptr;
  void* out1 = nullptr;
  void* out2 = nullptr;
  void* out3 = nullptr;  // F32 gated fwd: G hi / lo split (SpmmParams::out3 / out4)
  void* out4 = nullptr;
  const void* in0 = nullptr;
  const void* in1 = nullptr;
  int64_t ld_out = 0;
  const float* bias = nullptr;
  bool reverse_tiles = false;  // last token tile first (see SpmmParams::reverse_tiles)
  const blast_tp_t* tp = nullptr;  // fused TP all-reduce epilogue (single-matrix products)
};

// BLAST_DEBUG_COUNTERS=1: per-role wait cycles of every tensor-core launch to stderr
// (synchronizes after each launch; diagnosis only).
static unsigned long long* dbg_buffer() {
  static unsigned long long* buf = nullptr;
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("BLAST_DEBUG_COUNTERS");
    on = (e && e[0] == '1') ? 1 : 0;
    // [0, kDbgSlots): summed role counters; then 2 * 1024 per-CTA start / end globaltimer
    if (on && cudaMalloc(&buf, (kDbgSlots + 2048) * sizeof(unsigned long long)) != cudaSuccess) on = 0;
  }
  return on ? buf : nullptr;
}
static void dbg_begin(cudaStream_t st) {
  if (auto* b = dbg_buffer()) cudaMemsetAsync(b, 0, (kDbgSlots + 2048) * sizeof(unsigned long long), st);
}
static void dbg_end(const char* name, cudaStream_t st, int ctas) {
  auto* b = dbg_buffer();
  if (!b) return;
  static unsigned long long h[kDbgSlots + 2048];
  cudaMemcpyAsync(h, b, sizeof(h), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  const double n = ctas > 0 ? ctas : 1;
  if (ctas > 0 && ctas <= 1024 && h[kDbgSlots] != 0) {  // per-CTA spans (globaltimer, ns)
    unsigned long long t0 = ~0ull, t1 = 0, e0 = ~0ull;
    double sum = 0, mx = 0;
    for (int i = 0; i < ctas; ++i) {
      const unsigned long long a = h[kDbgSlots + 2 * i], z = h[kDbgSlots + 2 * i + 1];
      t0 = std::min(t0, a);
      t1 = std::max(t1, z);
      e0 = std::min(e0, z);
      sum += double(z - a);
      mx = std::max(mx, double(z - a));
    }
    unsigned long long s1 = 0;
    for (int i = 0; i < ctas; ++i) s1 = std::max(s1, h[kDbgSlots + 2 * i]);
    fprintf(stderr,
            "[blast dbg] %s span %.1f us: CTA starts within %.1f us, ends within %.1f us, "
            "per-CTA avg %.1f max %.1f us\n",
            name, (t1 - t0) * 1e-3, (s1 - t0) * 1e-3, (t1 - e0) * 1e-3, sum / ctas * 1e-3, mx * 1e-3);
    if (getenv("BLAST_DEBUG_CTAS")) {
      fprintf(stderr, "[blast dbg] per-CTA end (us after first start):");
      for (int i = 0; i < ctas; ++i) fprintf(stderr, " %.1f", (h[kDbgSlots + 2 * i + 1] - t0) * 1e-3);
      fprintf(stderr, "\n");
    }
  }
  fprintf(stderr,
          "[blast dbg] %s ctas=%d per-CTA cycles: prod.wait_empty=%.0f cta.total=%.0f "
          "mma.wait_full=%.0f mma.wait_acc=%.0f mma.loop=%.0f epi.wait_acc=%.0f mma.issue=%.0f "
          "mma.steps=%.0f epi.wait_in=%.0f epi.tile=%.0f\n",
          name, ctas, h[0] / n, h[1] / n, h[2] / n, h[3] / n, h[4] / n, h[5] / n, h[6] / n, h[7] / n,
          h[8] / n, h[9] / n);
}

static SpmmParams make_params(const EngineCall& c) {
  SpmmParams p{};
  p.dbg = dbg_buffer();
  if constexpr (kDiagSwitches) {  // diagnosis builds only (-DBLAST_DIAG_SWITCHES=1)
    static int skip = -1;
    if (skip < 0) {
      const char* e = getenv("BLAST_SKIP_EPILOGUE");
      skip = e ? atoi(e) & 3 : 0;  // 1: skip epilogues, 2: skip operand loads (timing only)
    }
    p.skip_epilogue = skip;
  }
  p.m = static_cast<int32_t>(c.m);
  p.n_lines = static_cast<int32_t>(c.n_lines);
  p.n_valid = static_cast<int32_t>(c.n_valid);
  p.n_tok_tiles = static_cast<int32_t>(cdiv(c.m, 128));
  p.step_ptr = c.step_ptr;
  p.steps = reinterpret_cast<const int4*>(c.steps);
  p.line_flags = c.flags;
  p.act = c.act;
  p.accumulate = c.accumulate;
  p.out0 = c.out0;
  p.out1 = c.out1;
  p.out2 = c.out2;
  p.out3 = c.out3;
  p.out4 = c.out4;
  p.in0 = c.in0;
  p.in1 = c.in1;
  p.ld_out = c.ld_out;
  p.bias = c.bias;
  p.reverse_tiles = c.reverse_tiles ? 1 : 0;
  if (c.tp) p.tp = *c.tp;
  return p;
}

// Programmatic dependent launch for the tensor-core engine; BLAST_PDL=0 disables.
static bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BLAST_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

const int32_t* balanced_schedule(const int32_t* step_ptr, const int32_t* flags, int n_lines,
                                 int n_tiles, int grid, bool seq_gu, cudaStream_t st,
                                 int* rows_out);

// 0/1 switch read once per name from the environment (default `dflt`)
static bool env_flag(const char* name, int dflt) {
  static std::mutex mu;
  static std::vector<std::pair<std::string, int>> seen;
  std::lock_guard<std::mutex> lock(mu);
  for (auto& kv : seen)
    if (kv.first == name) return kv.second != 0;
  const char* e = getenv(name);
  const int v = e ? (e[0] == '1') : dflt;
  seen.emplace_back(name, v);
  return v != 0;
}

template <int B, int ELT, int NPASS, int NMAT, bool SUM, bool BK, int EPI, typename OutT,
          int OUT_ELT = 0, int TM = 1, int SPLIT = 0>
static int launch_tc(const EngineCall& c, const void* a0lo, const void* a1lo, cudaStream_t st) {
  constexpr int IN_ST = in_staged<EPI, OUT_ELT>();
  using Cfg = TcCfg<B, ELT, NPASS, NMAT, SUM, BK, OUT_ELT, TM, IN_ST, SPLIT, staged_outputs<EPI>()>;
  auto kern = spmm_tc_kernel<B, ELT, NPASS, NMAT, SUM, BK, EPI, OutT, OUT_ELT, TM, SPLIT>;
  static bool configured[64] = {};
  if (int rc = configure_smem(kern, Cfg::SMEM_BYTES, configured, "spmm_tc smem attribute"))
    return rc;
  const int dt = ELT == 2 ? BLAST_BF16 : BLAST_F32;
  CUtensorMap mA0, mA0lo, mA1, mA1lo, mW0, mW0lo, mW1, mW1lo;
  auto mkA = [&](CUtensorMap* mp, const void* ptr) {
    return encode_map_2d(mp, ptr, dt, static_cast<uint64_t>(c.a_cols), static_cast<uint64_t>(c.m),
                         static_cast<uint64_t>(c.a_cols) * ELT, Cfg::SWE, Cfg::TROWS, Cfg::SW);
  };
  auto mkW = [&](CUtensorMap* mp, const void* ptr, int64_t nnzb) {
    if (ptr == nullptr || nnzb <= 0) {
      ptr = c.a0;
      nnzb = 1;
    }
    return encode_map_2d(mp, ptr, dt, B, static_cast<uint64_t>(nnzb) * B,
                         static_cast<uint64_t>(B) * ELT, Cfg::SWE, B, Cfg::SW);
  };
  bool ok = mkA(&mA0, c.a0);
  mA0lo = mA0;
  if (ok && NPASS == 3) ok = mkA(&mA0lo, a0lo);
  mA1 = mA0;
  mA1lo = mA0lo;
  if (ok && SUM) {
    ok = mkA(&mA1, c.a1);
    mA1lo = mA1;
    if (ok && NPASS == 3) ok = mkA(&mA1lo, a1lo);
  }
  if (ok) ok = mkW(&mW0, NPASS == 3 ? c.w0_hi : c.w0, c.nnzb0);
  mW0lo = mW0;
  if (ok && NPASS == 3) ok = mkW(&mW0lo, c.w0_lo, c.nnzb0);
  mW1 = mW0;
  mW1lo = mW0lo;
  if (ok && NMAT > 1) {
    ok = mkW(&mW1, NPASS == 3 ? c.w1_hi : c.w1, c.nnzb1);
    mW1lo = mW1;
    if (ok && NPASS == 3) ok = mkW(&mW1lo, c.w1_lo, c.nnzb1);
  }
  // staged output: out0 [m x n_valid], row pitch ld_out, box = one swizzle atom x 128 rows
  CUtensorMap mO = mA0;
  if (ok && OUT_ELT > 0)
    ok = encode_map_2d(&mO, c.out0, OUT_ELT == 2 ? BLAST_BF16 : BLAST_F32,
                       static_cast<uint64_t>(c.n_valid), static_cast<uint64_t>(c.m),
                       static_cast<uint64_t>(c.ld_out) * OUT_ELT, Cfg::OUT_SW / (OUT_ELT ? OUT_ELT : 1),
                       Cfg::BM, Cfg::OUT_SW);
  // staged in0 (and in1) tiles (activation-derivative / gating-backward epilogues) and the
  // second staged output (dB): same geometry as the output
  CUtensorMap mI = mO, mI1 = mO, mO1 = mO, mO2 = mO;
  auto mkTile = [&](CUtensorMap* mp, const void* ptr) {
    return encode_map_2d(mp, ptr, BLAST_BF16, static_cast<uint64_t>(c.n_valid),
                         static_cast<uint64_t>(c.m), static_cast<uint64_t>(c.ld_out) * 2,
                         Cfg::OUT_SW / 2, Cfg::BM, Cfg::OUT_SW);
  };
  if (ok && IN_ST) ok = mkTile(&mI, c.in0);
  if (ok && IN_ST == 2) ok = mkTile(&mI1, c.in1) && mkTile(&mO1, c.out1);
  if (ok && EPI == EPI_GATED_FWD_SAVE) ok = mkTile(&mO1, c.out1) && mkTile(&mO2, c.out2);
  if (!ok) return BLAST_EINVAL;
  SpmmParams p = make_params(c);
  p.n_tok_tiles = static_cast<int32_t>(cdiv(c.m, Cfg::TROWS));
  const int64_t items = static_cast<int64_t>(p.n_tok_tiles) * p.n_lines;
  if (items <= 0) return BLAST_OK;
  const int grid = static_cast<int>(std::min<int64_t>(items, num_sms()));
  p.early_trigger = items < 2 * static_cast<int64_t>(num_sms()) ? 1 : 0;
  // Persistent CTAs of single-matrix products take cost-balanced item lists (csrc/schedule.cu).
  // Same box, cfg3 (profiles/r02/cta_spans.txt): down 111.3 -> 108.0 us (CTA ends within 8.6
  // instead of 18.0 us); the gate+up kernel got slower (238.7 -> 243.0 us) although its CTAs
  // also end together: its per-CTA work rose by the same amount, i.e. it is bound by the
  // chip-wide L2 -> SM feed, which an even split cannot raise, so it keeps round robin.
  // Decode-size products (fewer than two items per CTA) balance the gate+up product too:
  // cfg3 shape at 95 %, 128 tokens, graph replay 18.6 -> 16.7 us (profiles/r02/decode_ab.txt).
  // 3xTF32 gate+up (cfg0 fp32: per-CTA ends spread over 22.5 of 104.6 us with round robin) is
  // balanced as well: its 48 KB stages make it latency- rather than L2-feed-bound
  // The training gate+up (G, a and b written) is balanced too: its per-item HBM writes make the
  // round-robin tail long (CTA ends spread over 47.7 us); LPT 310 -> 294 us, training step
  // 1.331 -> 1.315 ms same box (tools/ab_lpt_save.sh; BLAST_LPT_SAVE=0 disables). The same
  // schedule for the inference gate+up stays neutral (tools/ab_lpt_gu.sh, round 2).
#ifndef BLAST_LPT_SUMACC
#define BLAST_LPT_SUMACC 1
#endif
  if (NMAT == 1 || NPASS == 3 || (BLAST_LPT_SUMACC && SUM) ||
      (EPI == EPI_GATED_FWD_SAVE && env_flag("BLAST_LPT_SAVE", 1)) ||
      items < 2 * static_cast<int64_t>(num_sms()))
    p.sched = balanced_schedule(c.step_ptr, c.flags, p.n_lines, p.n_tok_tiles, grid, SPLIT == 2,
                                st, &p.sched_rows);
  dbg_begin(st);
  // programmatic dependent launch: this grid's CTAs start their setup on SMs freed by the
  // previous kernel's tail and wait in-kernel (griddep_wait) for its completion
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(kTcThreads);
  cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, mO, mI, mO1, mI1, mO2, mA0, mA0lo, mA1, mA1lo, mW0, mW0lo, mW1,
                     mW1lo, p);
  const int rc = check_launch("spmm_tc");
  dbg_end("spmm_tc", st, grid);
  return rc;
}

// Compile-time guard: does this configuration have >= 2 pipeline stages?
// (NPASS = 3: split-K stages of one 128-byte K atom, accumulator pairs; two-matrix products
// only in the sequential layout, one panel + one block per stage)
template <int B, int ELT, int NPASS, int NMAT, bool SUM>
constexpr bool tc_fits() {
  constexpr bool sk = NPASS == 3;
  constexpr int rowb = B * ELT;
  constexpr int krow = sk ? (rowb < 128 ? rowb : 128) : rowb;  // bytes of K per stage row
  constexpr int a_tile = (128 * krow + 1023) / 1024 * 1024;
  constexpr int b_tile = (B * krow + 1023) / 1024 * 1024;
  constexpr int ncopy = sk ? 2 : 1;
  constexpr int na = (SUM && !sk) ? NMAT : 1;
  constexpr int nw = sk ? 1 : NMAT;
  constexpr int stage = na * ncopy * a_tile + nw * ncopy * b_tile;
  constexpr int nacc = SUM ? 1 : NMAT;
  constexpr int accw = sk ? 2 * B : B;
  return (200 * 1024) / stage >= 2 && 2 * nacc * accw <= 512 && (!sk || 2 * B <= 256);
}

// Staged (TMA-store) output for out0: bf16 outputs whose rows are 16-byte aligned, when
// the staging buffers still leave >= 3 pipeline stages. BLAST_DIRECT_STORES=1 disables it.
static bool staged_out_disabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BLAST_DIRECT_STORES");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}
// >= 3 pipeline stages next to the double-buffered bf16 output staging (TcCfg arithmetic),
// and (TM = 2) both token halves' accumulators double-buffered in TMEM
template <int B, int ELT, int NPASS, int NMAT, bool SUM, int TM = 1, int IN_ST = 0>
constexpr bool staged_fits() {
  if (ELT != 2 || NPASS != 1) return false;
  if (2 * TM * (SUM ? 1 : NMAT) * B > 512) return false;
  constexpr int rowb = B * ELT;
  constexpr int a_tile = (128 * TM * rowb + 1023) / 1024 * 1024;
  constexpr int b_tile = (B * rowb + 1023) / 1024 * 1024;
  constexpr int na = SUM ? NMAT : 1;
  constexpr int stage = na * a_tile + NMAT * b_tile;
  constexpr int nout = IN_ST == 2 ? 2 : 1;
  constexpr int staging = (2 * nout + 2 * IN_ST) * ((128 * B * 2 + 1023) / 1024 * 1024);
  return (232448 - 1024 - 512 - staging) / stage >= 3;
}
// gate+up stage layout (TcCfg SPLIT) for the 256-token staged product:
//   2 (default): sequential items (all gate blocks of the line, then all up blocks), one weight
//      block per stage, waiter warp; same box cfg3 0.3388 vs 0.3433 ms for the interleaved
//      layout (gate+up 227 vs 235 us; profiles/r01/mma_side/mode_ab.txt)
//   0: interleaved steps (a step holding both blocks loads the panel once), 48 KB stages
// BLAST_SPLIT_STAGES=0/2 selects.
// The sequential layout loads the panel once per block, so steps holding both a gate and an
// up block cost a second panel load: it pays at b >= 64 when such steps are rare (cfg3 sweep,
// profiles/r01/cfg3_sweep.jsonl: b = 64 at 70-95 % faster, at 50 % and b = 16 / 32 slower).
// Plan flags hold per-line block counts below 2^15.
template <int B>
static bool seq_gate_up_pays(const EngineCall& c) {
  if (B < 64 || c.a_cols / B >= 0x7fff) return false;
  const double cells = static_cast<double>(c.a_cols / B) * static_cast<double>(c.n_lines);
  const double d0 = c.nnzb0 / cells, d1 = c.nnzb1 / cells;
  const double both = d0 * d1, any = d0 + d1 - both;
  return any > 0.0 && both / any < 0.25;
}

static int split_stages() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BLAST_SPLIT_STAGES");
    v = (e && e[0] == '0') ? 0 : 2;
  }
  return v;
}
// 256-token items (TcCfg TM = 2) for the forward products; BLAST_WIDE_TILES=0 disables.
static bool wide_tiles() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BLAST_WIDE_TILES");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}
// 256-token items for the two-input gating backward (EPI_GATED_BWD2); BLAST_WIDE_BWD2=0 disables.
static bool wide_bwd2() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BLAST_WIDE_BWD2");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}
template <int B, int ELT, int NPASS, int NMAT, bool SUM>
static bool use_staged(const EngineCall& c) {
  if (!staged_fits<B, ELT, NPASS, NMAT, SUM>() || staged_out_disabled()) return false;
  if (c.accumulate || !aligned16(c.out0) || (c.ld_out * 2) % 16 != 0) return false;
  // EPI_GATED_BWD: the single-output form (y = (x W^T) * act'(pre)) and the two-input gating
  // backward (EPI_GATED_BWD2, needs its second input / output 16-byte aligned too)
  if (c.epi == EPI_GATED_BWD && c.in1)
    return aligned16(c.in0) && aligned16(c.in1) && c.out1 && aligned16(c.out1);
  return c.epi == EPI_STORE || c.epi == EPI_GATED_FWD || c.epi == EPI_GATED_BWD;
}

template <int B, int ELT, int NPASS, typename OutT>
static int dispatch_b(const EngineCall& c, const void* a0lo, const void* a1lo, cudaStream_t st) {
  constexpr int SO = (ELT == 2 && NPASS == 1) ? 2 : 0;  // staged-output element size
  if (!c.transposed) {
    if (c.nmat == 1 && c.epi == EPI_STORE) {
      if constexpr (tc_fits<B, ELT, NPASS, 1, false>()) {
        if constexpr (staged_fits<B, ELT, NPASS, 1, false, 2>())
          if (use_staged<B, ELT, NPASS, 1, false>(c) && c.m >= 256 && wide_tiles())
            return launch_tc<B, ELT, NPASS, 1, false, (ELT == 4), EPI_STORE, OutT, SO, 2>(c, a0lo, a1lo, st);
        if constexpr (staged_fits<B, ELT, NPASS, 1, false>())
          if (use_staged<B, ELT, NPASS, 1, false>(c))
            return launch_tc<B, ELT, NPASS, 1, false, (ELT == 4), EPI_STORE, OutT, SO>(c, a0lo, a1lo, st);
        return launch_tc<B, ELT, NPASS, 1, false, (ELT == 4), EPI_STORE, OutT>(c, a0lo, a1lo, st);
      }
    } else if (c.nmat == 2 && c.epi == EPI_GATED_FWD) {
      if constexpr (NPASS == 3) {
        // 3xTF32 gate+up: sequential layout (all gate blocks of the line, then all up blocks),
        // split-K stages, accumulator pairs (the plan flags carry per-line block counts)
        if constexpr (tc_fits<B, ELT, NPASS, 2, false>())
          if (c.a_cols / B < 0x7fff)
            return launch_tc<B, ELT, NPASS, 2, false, true, EPI_GATED_FWD, OutT, 0, 1, 2>(c, a0lo, a1lo, st);
      } else if constexpr (tc_fits<B, ELT, NPASS, 2, false>()) {
        if constexpr (staged_fits<B, ELT, NPASS, 2, false, 2>())
          if (use_staged<B, ELT, NPASS, 2, false>(c) && c.m >= 256 && wide_tiles())
            return (split_stages() == 2 && seq_gate_up_pays<B>(c))
                       ? ((c.out1 && c.out2 && aligned16(c.out1) && aligned16(c.out2))
                              // training forward: G, a and b all through staged TMA stores
                              ? launch_tc<B, ELT, NPASS, 2, false, (ELT == 4), EPI_GATED_FWD_SAVE, OutT, SO, 2, 2>(c, a0lo, a1lo, st)
                              : launch_tc<B, ELT, NPASS, 2, false, (ELT == 4), EPI_GATED_FWD, OutT, SO, 2, 2>(c, a0lo, a1lo, st))
                       : launch_tc<B, ELT, NPASS, 2, false, (ELT == 4), EPI_GATED_FWD, OutT, SO, 2>(c, a0lo, a1lo, st);
        if constexpr (staged_fits<B, ELT, NPASS, 2, false>())
          if (use_staged<B, ELT, NPASS, 2, false>(c))
            return launch_tc<B, ELT, NPASS, 2, false, (ELT == 4), EPI_GATED_FWD, OutT, SO>(c, a0lo, a1lo, st);
        return launch_tc<B, ELT, NPASS, 2, false, (ELT == 4), EPI_GATED_FWD, OutT>(c, a0lo, a1lo, st);
      }
    }
  } else {
    if (c.nmat == 1 && c.epi == EPI_STORE) {
      if constexpr (staged_fits<B, ELT, NPASS, 1, false, 2>())
        if (use_staged<B, ELT, NPASS, 1, false>(c) && c.m >= 256 && wide_tiles())
          return launch_tc<B, ELT, NPASS, 1, false, true, EPI_STORE, OutT, SO, 2>(c, a0lo, a1lo, st);
      if constexpr (staged_fits<B, ELT, NPASS, 1, false>())
        if (use_staged<B, ELT, NPASS, 1, false>(c))
          return launch_tc<B, ELT, NPASS, 1, false, true, EPI_STORE, OutT, SO>(c, a0lo, a1lo, st);
      if constexpr (tc_fits<B, ELT, NPASS, 1, false>())
        return launch_tc<B, ELT, NPASS, 1, false, true, EPI_STORE, OutT>(c, a0lo, a1lo, st);
    } else if (c.nmat == 1 && c.epi == EPI_GATED_BWD && c.in1) {
      // gating backward (dA, dB): a, b in and dA, dB out through staged TMA tiles; 256-token
      // items (the weight blocks read once per 256 tokens) with 3 x 40 KB stages
      if constexpr (B == 64 && ELT == 2 && NPASS == 1)
        if (use_staged<B, ELT, NPASS, 1, false>(c) && c.m >= 256 && wide_tiles() && wide_bwd2())
          return launch_tc<B, ELT, NPASS, 1, false, true, EPI_GATED_BWD2, OutT, SO, 2>(c, a0lo, a1lo, st);
      if constexpr (staged_fits<B, ELT, NPASS, 1, false, 1, 2>())
        if (use_staged<B, ELT, NPASS, 1, false>(c))
          return launch_tc<B, ELT, NPASS, 1, false, true, EPI_GATED_BWD2, OutT, SO>(c, a0lo, a1lo, st);
      if constexpr (tc_fits<B, ELT, NPASS, 1, false>())
        return launch_tc<B, ELT, NPASS, 1, false, true, EPI_GATED_BWD, OutT>(c, a0lo, a1lo, st);
    } else if (c.nmat == 1 && c.epi == EPI_GATED_BWD) {
      if constexpr (staged_fits<B, ELT, NPASS, 1, false, 2, 1>())
        if (use_staged<B, ELT, NPASS, 1, false>(c) && c.m >= 256 && wide_tiles() &&
            aligned16(c.in0))
          return launch_tc<B, ELT, NPASS, 1, false, true, EPI_GATED_BWD, OutT, SO, 2>(c, a0lo, a1lo, st);
      if constexpr (staged_fits<B, ELT, NPASS, 1, false, 1, 1>())
        if (use_staged<B, ELT, NPASS, 1, false>(c) && aligned16(c.in0))
          return launch_tc<B, ELT, NPASS, 1, false, true, EPI_GATED_BWD, OutT, SO>(c, a0lo, a1lo, st);
      if constexpr (tc_fits<B, ELT, NPASS, 1, false>())
        return launch_tc<B, ELT, NPASS, 1, false, true, EPI_GATED_BWD, OutT>(c, a0lo, a1lo, st);
    } else if (c.nmat == 2 && c.sumacc && c.epi == EPI_STORE && NPASS == 3) {
      // 3xTF32 dX = dA Wg^T + dB Wu^T: sequential layout into one accumulator pair
      if constexpr (NPASS == 3 && tc_fits<B, ELT, NPASS, 2, true>())
        if (c.a_cols / B < 0x7fff)
          return launch_tc<B, ELT, NPASS, 2, true, true, EPI_STORE, OutT, 0, 1, 2>(c, a0lo, a1lo, st);
    } else if (c.nmat == 2 && c.sumacc && c.epi == EPI_STORE) {
      // dX = dA Wg^T + dB Wu^T in one accumulator, staged (TMA-store) output. 256-token items
      // with the sequential layout (all dA blocks of the line, then all dB blocks; one panel +
      // one weight block per stage, as the gate+up forward) where steps holding both are rare
      if constexpr (ELT == 2 && NPASS == 1 && B >= 64)
        if (use_staged<B, ELT, NPASS, 2, true>(c) && c.m >= 256 && wide_tiles() &&
            split_stages() == 2 && seq_gate_up_pays<B>(c))
          return launch_tc<B, ELT, NPASS, 2, true, true, EPI_STORE, OutT, SO, 2, 2>(c, a0lo, a1lo, st);
      if constexpr (staged_fits<B, ELT, NPASS, 2, true>())
        if (use_staged<B, ELT, NPASS, 2, true>(c))
          return launch_tc<B, ELT, NPASS, 2, true, true, EPI_STORE, OutT, SO>(c, a0lo, a1lo, st);
      if constexpr (NPASS != 3 && tc_fits<B, ELT, NPASS, 2, true>())
        return launch_tc<B, ELT, NPASS, 2, true, true, EPI_STORE, OutT>(c, a0lo, a1lo, st);
    }
  }
  return -1;  // not available on the tensor-core path
}

// Which configurations the tensor-core engine takes (the rest run on CUDA cores).
static bool tc_shape_ok(const EngineCall& c) {
  const int elt = bytes_of(c.dtype);
  if (!(c.block == 16 || c.block == 32 || c.block == 64 || c.block == 128)) return false;
  if ((c.a_cols * elt) % 16 != 0) return false;
  if (!aligned16(c.a0) || (c.a1 && !aligned16(c.a1))) return false;
  if ((c.w0 && !aligned16(c.w0)) || (c.w1 && !aligned16(c.w1))) return false;
  if (c.m > INT32_MAX || c.n_valid > INT32_MAX) return false;
  return true;
}

template <typename OutT, int ELT, int NPASS>
static int dispatch_tc(const EngineCall& c, const void* a0lo, const void* a1lo, cudaStream_t st) {
  switch (c.block) {
    case 16: return dispatch_b<16, ELT, NPASS, OutT>(c, a0lo, a1lo, st);
    case 32: return dispatch_b<32, ELT, NPASS, OutT>(c, a0lo, a1lo, st);
    case 64: return dispatch_b<64, ELT, NPASS, OutT>(c, a0lo, a1lo, st);
    case 128: return dispatch_b<128, ELT, NPASS, OutT>(c, a0lo, a1lo, st);
    default: return -1;
  }
}

static int run_simt(const EngineCall& c, cudaStream_t st) {
  const SpmmParams p = make_params(c);
  SimtArgs s{};
  s.a0 = c.a0;
  s.a1 = c.a1;
  s.lda = c.a_cols;
  s.a_cols = c.a_cols;
  s.w0 = c.w0;
  s.w1 = c.w1;
  s.block = c.block;
  s.transposed = c.transposed ? 1 : 0;
  s.nmat = c.nmat;
  s.sumacc = c.sumacc ? 1 : 0;
  s.epi = c.epi;
  if (c.m <= 0 || c.n_lines <= 0) return BLAST_OK;
  dim3 grid(static_cast<unsigned>(c.n_lines), static_cast<unsigned>(cdiv(c.m, 32)));
  if (c.dtype == BLAST_BF16)
    spmm_simt_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(p, s);
  else
    spmm_simt_kernel<float><<<grid, 256, 0, st>>>(p, s);
  return check_launch("spmm_simt");
}

// Runs one engine call on the tensor cores when the shape allows it, else on CUDA cores.
int run_engine(const EngineCall& c_in, cudaStream_t st) {
  if (c_in.m <= 0 || c_in.n_lines <= 0) return BLAST_OK;
  if (!c_in.step_ptr || !c_in.steps || !c_in.flags) {
    set_error("execution plan missing (build it with blast_build_plan)");
    return BLAST_EINVAL;
  }
  if (c_in.tp && (c_in.nmat != 1 || c_in.epi != EPI_STORE || c_in.transposed || c_in.accumulate)) {
    set_error("fused TP all-reduce: single-matrix forward products only");
    return BLAST_EINVAL;
  }
  if (tc_shape_ok(c_in)) {
    if (c_in.dtype == BLAST_BF16) {
      int r = dispatch_tc<__nv_bfloat16, 2, 1>(c_in, nullptr, nullptr, st);
      if (r >= 0) return r;
    } else {
      // 3xTF32: split the activations into hi/lo (unless the caller passes them split);
      // weights carry their own split (kind::tf32 reads B K-major, so forward products use
      // transposed block copies)
      const bool w_split = c_in.w0_hi && c_in.w0_lo && (c_in.nmat == 1 || (c_in.w1_hi && c_in.w1_lo));
      if (w_split) {
        const int64_t n = c_in.m * c_in.a_cols;
        Scratch s0, s1;
        EngineCall c = c_in;
        const void* lo0 = c_in.a0_lo;
        const void* lo1 = c_in.a1_lo;
        // the raw activation is the hi operand: kind::tf32 reads fp32 truncated to tf32,
        // bitwise equal to a pre-split hi copy (tools/probe_tf32_trunc.py); only lo is built
        if (!lo0) {
          if (!s0.alloc(sizeof(float) * n, st)) return cuda_status(cudaGetLastError(), "scratch");
          blast_split_tf32(static_cast<const float*>(c_in.a0), nullptr, s0.as<float>(), n, st);
          lo0 = s0.ptr;
        }
        if (c_in.sumacc && !lo1) {
          if (!s1.alloc(sizeof(float) * n, st)) return cuda_status(cudaGetLastError(), "scratch");
          blast_split_tf32(static_cast<const float*>(c_in.a1), nullptr, s1.as<float>(), n, st);
          lo1 = s1.ptr;
        }
        int r = dispatch_tc<float, 4, 3>(c, lo0, lo1, st);
        if (r >= 0) return r;
        if (c_in.a0_lo || c_in.a1_lo) {
          set_error("pre-split fp32 activations need the tensor-core engine");
          return BLAST_EUNSUPPORTED;
        }
      }
    }
  }
  if (c_in.tp) {
    set_error("fused TP all-reduce needs the tensor-core engine (b in {16, 32, 64, 128})");
    return BLAST_EUNSUPPORTED;
  }
  return run_simt(c_in, st);
}

static bool check_w(const blast_bcsc_t* w) {
  if (!w || w->block < 1 || w->rows < 1 || w->cols < 1) {
    set_error("invalid block-sparse matrix descriptor");
    return false;
  }
  if (w->dtype != BLAST_F32 && w->dtype != BLAST_BF16) {
    set_error("unsupported dtype %d", w->dtype);
    return false;
  }
  return true;
}

}  // namespace blast

using namespace blast;

extern "C" int blast_bspmm(const void* x, int64_t m, const blast_bcsc_t* w, int act, void* y,
                           void* stream) {
  return blast_bspmm_ex(x, m, w, nullptr, act, y, nullptr, stream);
}

static int bspmm_impl(const void* x, int64_t m, const blast_bcsc_t* w, const float* bias, int act,
                      void* y, void* pre, bool reverse_tiles, void* stream);

extern "C" int blast_bspmm_ex(const void* x, int64_t m, const blast_bcsc_t* w, const float* bias,
                              int act, void* y, void* pre, void* stream) {
  return bspmm_impl(x, m, w, bias, act, y, pre, false, stream);
}

static int bspmm_impl(const void* x, int64_t m, const blast_bcsc_t* w, const float* bias, int act,
                      void* y, void* pre, bool reverse_tiles, void* stream) {
  if (!check_w(w)) return BLAST_EINVAL;
  if (act < 0 || act > 3) {
    set_error("unknown nonlinearity code %d", act);
    return BLAST_EINVAL;
  }
  EngineCall c;
  c.dtype = w->dtype;
  c.block = w->block;
  c.act = act;
  c.bias = bias;
  c.m = m;
  c.a_cols = w->rows;
  c.a0 = x;
  c.w0 = w->values;
  c.w0_hi = w->tf32_fwd_hi;
  c.w0_lo = w->tf32_fwd_lo;
  c.nnzb0 = w->nnzb;
  c.n_lines = cdiv(w->cols, w->block);
  c.n_valid = w->cols;
  c.step_ptr = w->fwd_step_ptr;
  c.steps = w->fwd_steps;
  c.flags = w->fwd_flags;
  c.out0 = y;
  c.out1 = pre;
  c.ld_out = w->cols;
  c.reverse_tiles = reverse_tiles;
  return run_engine(c, static_cast<cudaStream_t>(stream));
}

extern "C" int blast_bspmm_rt_act(const void* x, int64_t m, const blast_bcsc_t* w, int act,
                                  const void* pre, void* y, void* stream) {
  if (!check_w(w)) return BLAST_EINVAL;
  if (act < 0 || act > 3 || !pre) {
    set_error("bspmm_rt_act: activation code %d / pre-activation required", act);
    return BLAST_EINVAL;
  }
  EngineCall c;
  c.dtype = w->dtype;
  c.block = w->block;
  c.transposed = true;
  c.epi = EPI_GATED_BWD;  // single-input form: y = (x W^T) * act'(pre)
  c.act = act;
  c.m = m;
  c.a_cols = w->cols;
  c.a0 = x;
  c.w0 = w->values;
  c.w0_hi = w->tf32_rt_hi;
  c.w0_lo = w->tf32_rt_lo;
  c.nnzb0 = w->nnzb;
  c.n_lines = cdiv(w->rows, w->block);
  c.n_valid = w->rows;
  c.step_ptr = w->rt_step_ptr;
  c.steps = w->rt_steps;
  c.flags = w->rt_flags;
  c.out0 = y;
  c.in0 = pre;
  c.ld_out = w->rows;
  return run_engine(c, static_cast<cudaStream_t>(stream));
}

static int bspmm_rt_impl(const void* x, int64_t m, const blast_bcsc_t* w, void* y, int accumulate,
                         cudaStream_t st) {
  EngineCall c;
  c.dtype = w->dtype;
  c.block = w->block;
  c.transposed = true;
  c.accumulate = accumulate;
  c.m = m;
  c.a_cols = w->cols;
  c.a0 = x;
  c.w0 = w->values;
  c.w0_hi = w->tf32_rt_hi;
  c.w0_lo = w->tf32_rt_lo;
  c.nnzb0 = w->nnzb;
  c.n_lines = cdiv(w->rows, w->block);
  c.n_valid = w->rows;
  c.step_ptr = w->rt_step_ptr;
  c.steps = w->rt_steps;
  c.flags = w->rt_flags;
  c.out0 = y;
  c.ld_out = w->rows;
  return run_engine(c, st);
}

extern "C" int blast_bspmm_rt(const void* x, int64_t m, const blast_bcsc_t* w, void* y,
                              void* stream) {
  if (!check_w(w)) return BLAST_EINVAL;
  return bspmm_rt_impl(x, m, w, y, 0, static_cast<cudaStream_t>(stream));
}

namespace blast {
template <typename T>
__global__ void gated_fwd_kernel(const T* a, const T* b, T* g, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    g[i] = from_f32<T>(gated_fwd(to_f32<T>(a[i]), to_f32<T>(b[i])));
}
}  // namespace blast

namespace blast {
static bool f32_fused_ok(const void* x, int64_t e, const blast_bcsc_t* gate, const blast_bcsc_t* up);
static int gate_up_impl(const void* x, int64_t m, const blast_bcsc_t* gate, const blast_bcsc_t* up,
                        const blast_mlp_plan_t* plan, void* gated, void* gate_pre, void* up_out,
                        void* g_hi, void* g_lo, cudaStream_t st);
}  // namespace blast

extern "C" int blast_mlp_forward(const void* x, int64_t m, const blast_bcsc_t* gate,
                                 const blast_bcsc_t* up, const blast_bcsc_t* down,
                                 const blast_mlp_plan_t* plan, void* y, void* gate_pre,
                                 void* up_out, void* gated, void* stream) {
  if (!check_w(gate) || !check_w(up) || !check_w(down)) return BLAST_EINVAL;
  const int64_t e = gate->rows, h = gate->cols;
  const int b = gate->block;
  if (up->rows != e || up->cols != h || down->rows != h || down->cols != e || up->block != b ||
      down->block != b || up->dtype != gate->dtype || down->dtype != gate->dtype) {
    set_error("gated MLP shape mismatch");
    return BLAST_EMISMATCH;
  }
  if (m <= 0) return BLAST_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t elt = bytes_of(gate->dtype);
  if (plan && plan->gu_step_ptr && f32_fused_ok(x, e, gate, up) && down->tf32_fwd_hi &&
      down->tf32_fwd_lo) {
    // fp32: the gate+up epilogue writes G already split into tf32 hi / lo (the down
    // projection's 3xTF32 operands; G itself only when the caller asked for it)
    // G itself is the hi operand (kind::tf32 truncates); only its lo part is extra
    Scratch ss;
    if (!ss.alloc((gated ? 1 : 2) * sizeof(float) * m * h, st))
      return cuda_status(cudaGetLastError(), "scratch G");
    float* g_lo = ss.as<float>();
    float* g_hi = gated ? static_cast<float*>(gated) : g_lo + m * h;
    int r = gate_up_impl(x, m, gate, up, plan, gated, gate_pre, up_out, g_hi, g_lo, st);
    if (r) return r;
    EngineCall c;
    c.dtype = BLAST_F32;
    c.block = b;
    c.m = m;
    c.a_cols = h;
    c.a0 = g_hi;
    c.a0_lo = g_lo;
    c.w0 = down->values;
    c.w0_hi = down->tf32_fwd_hi;
    c.w0_lo = down->tf32_fwd_lo;
    c.nnzb0 = down->nnzb;
    c.n_lines = cdiv(down->cols, b);
    c.n_valid = down->cols;
    c.step_ptr = down->fwd_step_ptr;
    c.steps = down->fwd_steps;
    c.flags = down->fwd_flags;
    c.out0 = y;
    c.ld_out = down->cols;
    c.reverse_tiles = true;
    return run_engine(c, st);
  }
  Scratch sg;
  if (!gated) {
    if (!sg.alloc(elt * m * h, st)) return cuda_status(cudaGetLastError(), "scratch G");
    gated = sg.ptr;
  }
  int r = gate_up_impl(x, m, gate, up, plan, gated, gate_pre, up_out, nullptr, nullptr, st);
  if (r) return r;
  // gate+up wrote G tile by tile in order: read it back last tile first, while the most
  // recently written rows are still in L2
  return bspmm_impl(gated, m, down, nullptr, BLAST_ACT_NONE, y, nullptr, true, stream);
}

namespace blast {
static bool check_tp(const blast_tp_t* tp) {
  if (!tp || tp->n < 1 || tp->n > BLAST_TP_MAX || tp->rank < 0 || tp->rank >= tp->n) {
    set_error("invalid TP group descriptor");
    return false;
  }
  for (int r = 0; r < tp->n; ++r)
    if (!tp->recv[r] || !tp->flags[r] || !tp->y[r] || !tp->done[r]) {
      set_error("TP group descriptor: missing buffer of rank %d", r);
      return false;
    }
  return true;
}

// one thread polls the counter (system scope) until it reaches `target`; a bounded wait
// turns a missing peer into a reported launch error instead of a hung device
__global__ void tp_wait_kernel(const uint32_t* done, uint32_t target) {
  const unsigned long long t0 = globaltimer_ns();
  while (true) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(done) : "memory");
    if (static_cast<int32_t>(v - target) >= 0) break;
    if (globaltimer_ns() - t0 > 20ull * 1000 * 1000 * 1000) {
      printf("blast: tp_wait timed out (done %u < %u)\n", v, target);
      __trap();
    }
    __nanosleep(200);
  }
}
}  // namespace blast

extern "C" int blast_tp_down_allreduce(const void* g, int64_t m, const blast_bcsc_t* down_shard,
                                       const blast_tp_t* tp, void* stream) {
  if (!check_w(down_shard) || !check_tp(tp)) return BLAST_EINVAL;
  if (m <= 0) return BLAST_OK;
  EngineCall c;
  c.dtype = down_shard->dtype;
  c.block = down_shard->block;
  c.m = m;
  c.a_cols = down_shard->rows;
  c.a0 = g;
  c.w0 = down_shard->values;
  c.w0_hi = down_shard->tf32_fwd_hi;
  c.w0_lo = down_shard->tf32_fwd_lo;
  c.nnzb0 = down_shard->nnzb;
  c.n_lines = cdiv(down_shard->cols, down_shard->block);
  c.n_valid = down_shard->cols;
  c.step_ptr = down_shard->fwd_step_ptr;
  c.steps = down_shard->fwd_steps;
  c.flags = down_shard->fwd_flags;
  c.out0 = tp->y[tp->rank];
  c.ld_out = down_shard->cols;
  c.tp = tp;
  return run_engine(c, static_cast<cudaStream_t>(stream));
}

extern "C" int blast_tp_mlp_forward(const void* x, int64_t m, const blast_bcsc_t* gate_shard,
                                    const blast_bcsc_t* up_shard, const blast_bcsc_t* down_shard,
                                    const blast_mlp_plan_t* plan, const blast_tp_t* tp,
                                    void* stream) {
  if (!check_w(gate_shard) || !check_w(up_shard) || !check_w(down_shard) || !check_tp(tp))
    return BLAST_EINVAL;
  if (gate_shard->cols != down_shard->rows || up_shard->cols != gate_shard->cols ||
      down_shard->cols != gate_shard->rows) {
    set_error("TP shard shape mismatch");
    return BLAST_EMISMATCH;
  }
  if (m <= 0) return BLAST_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Scratch sg;
  if (!sg.alloc(bytes_of(gate_shard->dtype) * m * gate_shard->cols, st))
    return cuda_status(cudaGetLastError(), "scratch G");
  int r = blast_mlp_gate_up(x, m, gate_shard, up_shard, plan, sg.ptr, nullptr, nullptr, stream);
  if (r) return r;
  return blast_tp_down_allreduce(sg.ptr, m, down_shard, tp, stream);
}

extern "C" int blast_tp_wait(const uint32_t* done, uint32_t target, void* stream) {
  if (!done) return BLAST_EINVAL;
  tp_wait_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(done, target);
  return check_launch("tp_wait");
}

namespace blast {
// fp32 gate+up through the fused 3xTF32 engine (sequential layout, accumulator pairs):
// b in {16, 32, 64} (the two accumulator pairs fit TMEM twice), transposed tf32 block images
static bool f32_fused_ok(const void* x, int64_t e, const blast_bcsc_t* gate, const blast_bcsc_t* up) {
  const int b = gate->block;
  return gate->dtype == BLAST_F32 && (b == 16 || b == 32 || b == 64) && gate->tf32_fwd_hi &&
         gate->tf32_fwd_lo && up->tf32_fwd_hi && up->tf32_fwd_lo && aligned16(x) &&
         (e * 4) % 16 == 0 && e / b < 0x7fff;
}

// G = silu(X Wg) * (X Wu) (mlp.py:111-113). g_hi / g_lo (fp32, optional): G also written as
// its tf32 hi / lo split for a 3xTF32 down projection; `gated` may then be null.
static int gate_up_impl(const void* x, int64_t m, const blast_bcsc_t* gate, const blast_bcsc_t* up,
                        const blast_mlp_plan_t* plan, void* gated, void* gate_pre, void* up_out,
                        void* g_hi, void* g_lo, cudaStream_t st) {
  const int64_t e = gate->rows, h = gate->cols;
  const int b = gate->block;
  const int dt = gate->dtype;
  const size_t elt = bytes_of(dt);
  int r;
  const bool fused = plan && plan->gu_step_ptr &&
                     (dt == BLAST_BF16 || f32_fused_ok(x, e, gate, up));
  if (!fused && !gated) {
    set_error("gate_up: output buffer required");
    return BLAST_EINVAL;
  }
  if (fused) {
    EngineCall c;
    c.dtype = dt;
    c.block = b;
    c.nmat = 2;
    c.epi = EPI_GATED_FWD;
    c.m = m;
    c.a_cols = e;
    c.a0 = x;
    c.w0 = gate->values;
    c.w0_hi = gate->tf32_fwd_hi;
    c.w0_lo = gate->tf32_fwd_lo;
    c.nnzb0 = gate->nnzb;
    c.w1 = up->values;
    c.w1_hi = up->tf32_fwd_hi;
    c.w1_lo = up->tf32_fwd_lo;
    c.nnzb1 = up->nnzb;
    c.n_lines = cdiv(h, b);
    c.n_valid = h;
    c.step_ptr = plan->gu_step_ptr;
    c.steps = plan->gu_steps;
    c.flags = plan->gu_flags;
    c.out0 = gated;
    c.out1 = gate_pre;
    c.out2 = up_out;
    c.ld_out = h;
    if (dt == BLAST_F32) {
      c.out3 = g_hi;
      c.out4 = g_lo;
    }
    return run_engine(c, st);
  }
  Scratch sa, sb;
  if (!gate_pre) {
    if (!sa.alloc(elt * m * h, st)) return cuda_status(cudaGetLastError(), "scratch a");
    gate_pre = sa.ptr;
  }
  if (!up_out) {
    if (!sb.alloc(elt * m * h, st)) return cuda_status(cudaGetLastError(), "scratch b");
    up_out = sb.ptr;
  }
  if ((r = blast_bspmm(x, m, gate, BLAST_ACT_NONE, gate_pre, st))) return r;
  if ((r = blast_bspmm(x, m, up, BLAST_ACT_NONE, up_out, st))) return r;
  const int64_t n = m * h;
  const int grid = static_cast<int>(std::min<int64_t>(cdiv(n, 256), (int64_t)num_sms() * 16));
  if (dt == BLAST_BF16)
    gated_fwd_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(gate_pre), static_cast<const __nv_bfloat16*>(up_out),
        static_cast<__nv_bfloat16*>(gated), n);
  else
    gated_fwd_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(gate_pre),
                                                  static_cast<const float*>(up_out),
                                                  static_cast<float*>(gated), n);
  return check_launch("gated_fwd");
}
}  // namespace blast

extern "C" int blast_mlp_gate_up(const void* x, int64_t m, const blast_bcsc_t* gate,
                                 const blast_bcsc_t* up, const blast_mlp_plan_t* plan,
                                 void* gated, void* gate_pre, void* up_out, void* stream) {
  if (!check_w(gate) || !check_w(up)) return BLAST_EINVAL;
  const int64_t e = gate->rows, h = gate->cols;
  const int b = gate->block;
  if (up->rows != e || up->cols != h || up->block != b || up->dtype != gate->dtype) {
    set_error("gated MLP shape mismatch");
    return BLAST_EMISMATCH;
  }
  if (m <= 0) return BLAST_OK;
  if (!gated) {
    set_error("gate_up: output buffer required");
    return BLAST_EINVAL;
  }
  return gate_up_impl(x, m, gate, up, plan, gated, gate_pre, up_out, nullptr, nullptr,
                      static_cast<cudaStream_t>(stream));
}

extern "C" int blast_mlp_backward_dgrad(const void* dy, int64_t m, const void* gate_pre,
                                        const void* up_out, const blast_bcsc_t* gate,
                                        const blast_bcsc_t* up, const blast_bcsc_t* down,
                                        const blast_mlp_plan_t* plan, void* dx, void* da,
                                        void* db, void* stream) {
  if (!check_w(gate) || !check_w(up) || !check_w(down)) return BLAST_EINVAL;
  const int64_t e = gate->rows, h = gate->cols;
  const int b = gate->block;
  if (up->rows != e || up->cols != h || down->rows != h || down->cols != e || up->block != b ||
      down->block != b) {
    set_error("gated MLP shape mismatch");
    return BLAST_EMISMATCH;
  }
  if (m <= 0) return BLAST_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int dt = gate->dtype;
  // dG = dY Wd^T with the gating backward fused into the epilogue -> dA, dB
  EngineCall c;
  c.dtype = dt;
  c.block = b;
  c.transposed = true;
  c.epi = EPI_GATED_BWD;
  c.m = m;
  c.a_cols = e;
  c.a0 = dy;
  c.w0 = down->values;
  c.w0_hi = down->tf32_rt_hi;
  c.w0_lo = down->tf32_rt_lo;
  c.nnzb0 = down->nnzb;
  c.n_lines = cdiv(h, b);
  c.n_valid = h;
  c.step_ptr = down->rt_step_ptr;
  c.steps = down->rt_steps;
  c.flags = down->rt_flags;
  c.out0 = da;
  c.out1 = db;
  c.in0 = gate_pre;
  c.in1 = up_out;
  c.ld_out = h;
  int r = run_engine(c, st);
  if (r) return r;
  // dX = dA Wg^T + dB Wu^T
  const bool fused = dt == BLAST_BF16 && b <= 64 && plan && plan->dx_step_ptr;
  if (fused) {
    EngineCall d;
    d.dtype = dt;
    d.block = b;
    d.transposed = true;
    d.nmat = 2;
    d.sumacc = true;
    d.m = m;
    d.a_cols = h;
    d.a0 = da;
    d.a1 = db;
    d.w0 = gate->values;
    d.nnzb0 = gate->nnzb;
    d.w1 = up->values;
    d.nnzb1 = up->nnzb;
    d.n_lines = cdiv(e, b);
    d.n_valid = e;
    d.step_ptr = plan->dx_step_ptr;
    d.steps = plan->dx_steps;
    d.flags = plan->dx_flags;
    d.out0 = dx;
    d.ld_out = e;
    return run_engine(d, st);
  }
  if ((r = bspmm_rt_impl(da, m, gate, dx, 0, st))) return r;
  return bspmm_rt_impl(db, m, up, dx, 1, st);
}
