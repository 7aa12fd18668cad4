// CUDA-core block-sparse product over the same plans and epilogues as the
// tensor-core engine. It serves the shapes tcgen05 cannot take: block sizes
// that are not a multiple of 16 (the reference tests sweep b = 1..16,
// tests/test_kernels.py:48-59) and activations whose row pitch is not 16-byte
// aligned (TMA requirement). fp32 accumulation; per block a fused-multiply-add
// chain, then the block partial is added to the running sum in ascending
// block order, like the reference's `a += t` (kernels.py:117-121).
#pragma once
#include "activations.cuh"
#include "spmm_tc.cuh"

namespace blast {

struct SimtArgs {
  const void* a0;  // A panel source for mat 0 (and mat 1 unless SUMACC)
  const void* a1;  // SUMACC: A source for mat 1
  int64_t lda;     // row pitch of a0/a1 (elements)
  int64_t a_cols;  // valid columns of A (panel columns beyond are zero)
  const void* w0;
  const void* w1;
  int32_t block;
  int32_t transposed;  // 0: Y = A W (W[k][n]);  1: Y = A W^T (W[n][k])
  int32_t nmat;
  int32_t sumacc;
  int32_t epi;
};

template <typename T>
__global__ void __launch_bounds__(256) spmm_simt_kernel(const SpmmParams p, const SimtArgs s) {
  constexpr int TM = 32;
  const int j = blockIdx.x;
  const int r0 = blockIdx.y * TM;
  const int B = s.block;
  const int s0 = p.step_ptr[j], s1 = p.step_ptr[j + 1];
  const int flags = p.line_flags[j];
  const T* A0 = static_cast<const T*>(s.a0);
  const T* A1 = static_cast<const T*>(s.a1 ? s.a1 : s.a0);
  const T* W0 = static_cast<const T*>(s.w0);
  const T* W1 = static_cast<const T*>(s.w1 ? s.w1 : s.w0);
  const int64_t bb = static_cast<int64_t>(B) * B;
  for (int idx = threadIdx.x; idx < TM * B; idx += blockDim.x) {
    const int rl = idx / B, c = idx - rl * B;
    const int row = r0 + rl;
    const int col = j * B + c;
    if (row >= p.m || col >= p.n_valid) continue;
    float acc[2] = {0.0f, 0.0f};
    bool init[2] = {false, false};
    for (int st = s0; st < s1; ++st) {
      const int4 step = p.steps[st];
      const int kb[2] = {step.y, step.z};
      for (int mm = 0; mm < s.nmat; ++mm) {
        if (kb[mm] < 0) continue;
        const T* A = (s.sumacc && mm == 1) ? A1 : A0;
        const T* W = (mm == 0 ? W0 : W1) + kb[mm] * bb;
        const int64_t acol0 = static_cast<int64_t>(step.x) * B;
        float t = 0.0f;
        for (int kk = 0; kk < B; ++kk) {
          const int64_t ac = acol0 + kk;
          if (ac >= s.a_cols) break;
          const float x = to_f32<T>(A[static_cast<int64_t>(row) * s.lda + ac]);
          const float w = to_f32<T>(s.transposed ? W[static_cast<int64_t>(c) * B + kk]
                                                 : W[static_cast<int64_t>(kk) * B + c]);
          t = fmaf(x, w, t);
        }
        const int ai = s.sumacc ? 0 : mm;
        acc[ai] = init[ai] ? __fadd_rn(acc[ai], t) : t;
        init[ai] = true;
      }
    }
    (void)flags;
    const int64_t off = static_cast<int64_t>(row) * p.ld_out + col;
    if (s.epi == EPI_STORE) {
      float v = acc[0];
      if (p.bias) v = __fadd_rn(v, p.bias[col]);
      if (p.out1) static_cast<T*>(p.out1)[off] = from_f32<T>(v);
      v = apply_act(v, p.act);
      if (p.accumulate) v = __fadd_rn(to_f32<T>(static_cast<T*>(p.out0)[off]), v);
      static_cast<T*>(p.out0)[off] = from_f32<T>(v);
    } else if (s.epi == EPI_GATED_FWD) {
      if (p.out1) static_cast<T*>(p.out1)[off] = from_f32<T>(acc[0]);
      if (p.out2) static_cast<T*>(p.out2)[off] = from_f32<T>(acc[1]);
      static_cast<T*>(p.out0)[off] = from_f32<T>(gated_fwd(acc[0], acc[1]));
    } else if (!p.in1) {
      const float pre = to_f32<T>(static_cast<const T*>(p.in0)[off]);
      static_cast<T*>(p.out0)[off] = from_f32<T>(__fmul_rn(acc[0], apply_act_grad(pre, p.act)));
    } else {
      const float a = to_f32<T>(static_cast<const T*>(p.in0)[off]);
      const float b = to_f32<T>(static_cast<const T*>(p.in1)[off]);
      float da, db;
      gated_bwd(acc[0], a, b, da, db);
      static_cast<T*>(p.out0)[off] = from_f32<T>(da);
      static_cast<T*>(p.out1)[off] = from_f32<T>(db);
    }
  }
}

}  // namespace blast
