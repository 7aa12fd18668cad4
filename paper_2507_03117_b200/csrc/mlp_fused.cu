// Host side of the fused gated-MLP forward (csrc/mlp_fused.cuh): blast_mlp_forward_fused.
#include "host.hpp"
#include "mlp_fused.cuh"

namespace blast {

// Opt-in (BLAST_FUSED_MLP=1): measured on cfg3 it is slower than the two-launch path
// (0.435 vs 0.352 ms) and the ring does not keep G out of HBM (ncu: 220 MB of DRAM writes,
// about the size of G), see DESIGN.md section 5. blast_mlp_forward_fused itself always runs.
static bool fused_disabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BLAST_FUSED_MLP");
    v = (e && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
}

static bool fused_ok(const void* x, int64_t m, const blast_bcsc_t* g, const blast_bcsc_t* u,
                     const blast_bcsc_t* d, const blast_mlp_plan_t* plan, const void* y) {
  if (!plan || !plan->gu_step_ptr || !d->fwd_step_ptr) return false;
  if (g->dtype != BLAST_BF16 || g->block != 64 || m < 256 || m > INT32_MAX) return false;
  const int64_t e = g->rows, h = g->cols;
  if (e % 64 || h % 64 || u->rows != e || u->cols != h || d->rows != h || d->cols != e) return false;
  if (u->dtype != BLAST_BF16 || d->dtype != BLAST_BF16 || u->block != 64 || d->block != 64)
    return false;
  return aligned16(x) && aligned16(y) && aligned16(g->values) && aligned16(u->values) &&
         aligned16(d->values);
}

static SpmmParams fused_side(int64_t m, int64_t n_lines, int64_t n_valid, const int32_t* sp,
                             const int32_t* steps, const int32_t* flags, void* out) {
  SpmmParams p{};
  p.m = static_cast<int32_t>(m);
  p.n_lines = static_cast<int32_t>(n_lines);
  p.n_valid = static_cast<int32_t>(n_valid);
  p.n_tok_tiles = static_cast<int32_t>(cdiv(m, 256));
  p.step_ptr = sp;
  p.steps = reinterpret_cast<const int4*>(steps);
  p.line_flags = flags;
  p.out0 = out;
  p.ld_out = n_valid;
  return p;
}

}  // namespace blast

using namespace blast;

int blast_mlp_forward_fused_impl(const void* x, int64_t m, const blast_bcsc_t* gate,
                                 const blast_bcsc_t* up, const blast_bcsc_t* down,
                                 const blast_mlp_plan_t* plan, void* y, void* stream);

// y = (silu(x Wg) * (x Wu)) Wd in one persistent kernel; G lives in a 4-tile ring in L2.
// Returns BLAST_EUNSUPPORTED (nothing launched) when the shape or dtype is not covered.
extern "C" int blast_mlp_forward_fused(const void* x, int64_t m, const blast_bcsc_t* gate,
                                       const blast_bcsc_t* up, const blast_bcsc_t* down,
                                       const blast_mlp_plan_t* plan, void* y, void* stream) {
  return blast_mlp_forward_fused_impl(x, m, gate, up, down, plan, y, stream);
}

// blast_mlp_forward's inference path: fused only when enabled (BLAST_FUSED_MLP=1).
int blast_mlp_forward_fused_if_enabled(const void* x, int64_t m, const blast_bcsc_t* gate,
                                       const blast_bcsc_t* up, const blast_bcsc_t* down,
                                       const blast_mlp_plan_t* plan, void* y, void* stream) {
  if (fused_disabled()) return BLAST_EUNSUPPORTED;
  return blast_mlp_forward_fused_impl(x, m, gate, up, down, plan, y, stream);
}

int blast_mlp_forward_fused_impl(const void* x, int64_t m, const blast_bcsc_t* gate,
                                 const blast_bcsc_t* up, const blast_bcsc_t* down,
                                 const blast_mlp_plan_t* plan, void* y, void* stream) {
  if (!gate || !up || !down) return BLAST_EINVAL;
  if (!fused_ok(x, m, gate, up, down, plan, y)) return BLAST_EUNSUPPORTED;
  using C = FusedCfg;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(mlp_fused_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
    if (e != cudaSuccess) return cuda_status(e, "mlp_fused smem attribute");
    configured = true;
  }
  const int64_t e = gate->rows, h = gate->cols;
  const int64_t n_tiles = cdiv(m, 256);
  Scratch ring, ctr;
  if (!ring.alloc(sizeof(__nv_bfloat16) * kFusedRing * 256 * h, st))
    return cuda_status(cudaGetLastError(), "mlp_fused ring");
  if (!ctr.alloc(sizeof(int32_t) * 2 * n_tiles, st))
    return cuda_status(cudaGetLastError(), "mlp_fused counters");
  cudaMemsetAsync(ctr.ptr, 0, sizeof(int32_t) * 2 * n_tiles, st);
  CUtensorMap mX, mWg, mWu, mGin, mGout, mWd, mY;
  const uint64_t ring_rows = static_cast<uint64_t>(kFusedRing) * 256;
  bool ok = encode_map_2d(&mX, x, BLAST_BF16, e, m, e * 2, 64, 256, 128);
  ok = ok && encode_map_2d(&mWg, gate->values, BLAST_BF16, 64, std::max<int64_t>(gate->nnzb, 1) * 64, 128, 64, 64, 128);
  ok = ok && encode_map_2d(&mWu, up->values, BLAST_BF16, 64, std::max<int64_t>(up->nnzb, 1) * 64, 128, 64, 64, 128);
  ok = ok && encode_map_2d(&mWd, down->values, BLAST_BF16, 64, std::max<int64_t>(down->nnzb, 1) * 64, 128, 64, 64, 128);
  ok = ok && encode_map_2d(&mGin, ring.ptr, BLAST_BF16, h, ring_rows, h * 2, 64, 256, 128);
  ok = ok && encode_map_2d(&mGout, ring.ptr, BLAST_BF16, h, ring_rows, h * 2, 64, 128, 128);
  ok = ok && encode_map_2d(&mY, y, BLAST_BF16, e, m, e * 2, 64, 128, 128);
  if (!ok) return BLAST_EINVAL;
  FusedParams fp{};
  fp.gu = fused_side(m, h / 64, h, plan->gu_step_ptr, plan->gu_steps, plan->gu_flags, ring.ptr);
  fp.dn = fused_side(m, e / 64, e, down->fwd_step_ptr, down->fwd_steps, down->fwd_flags, y);
  fp.n_tiles = static_cast<int32_t>(n_tiles);
  fp.n_gu_lines = static_cast<int32_t>(h / 64);
  fp.n_dn_lines = static_cast<int32_t>(e / 64);
  fp.gu_done = ctr.as<int32_t>();
  fp.dn_done = ctr.as<int32_t>() + n_tiles;
  if (const char* dbg = getenv("BLAST_FUSED_DBG")) fp.dbg = atoi(dbg);
  const int64_t n_items = (n_tiles + kFusedLag) * (fp.n_gu_lines + fp.n_dn_lines);
  const int grid = static_cast<int>(std::min<int64_t>(n_items, num_sms()));
  mlp_fused_kernel<<<grid, kTcThreads, C::SMEM_BYTES, st>>>(mX, mWg, mWu, mGin, mGout, mWd, mY, fp);
  return check_launch("mlp_fused");
}
