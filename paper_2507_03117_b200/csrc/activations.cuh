// Elementwise functions of the sparse MLP, written op-for-op after the
// reference's float32 numpy expressions so that a fused epilogue and a
// post-applied elementwise kernel produce identical bits:
//   sigmoid (split form)  blocksparse/kernels.py:24-30
//   silu / silu_grad      blocksparse/kernels.py:33-39
//   gelu (tanh form)      blocksparse/kernels.py:17-19, 42-43
//   relu                  blocksparse/kernels.py:46-47 (np.maximum: -0.0 -> +0.0, NaN kept)
//   gated product         blocksparse/mlp.py:113   g = (a * sigmoid(a)) * b
//   gated backward        blocksparse/mlp.py:133-139
// The explicit __f*_rn intrinsics stop nvcc from contracting into FMAs,
// which would make results depend on the calling context.
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

namespace blast {

enum Act : int { ACT_NONE = 0, ACT_RELU = 1, ACT_GELU = 2, ACT_SILU = 3 };

// Split form with t = exp(-|x|) <= 1 (never overflows): x >= 0 -> 1/(1+t), x < 0 -> t/(1+t).
// exp via ex2.approx (__expf, ~2 ulp) and a correctly rounded reciprocal
// (__frcp_rn) instead of an IEEE division: a few ulp of float32, far inside the
// 1e-5 fp32 / 2e-2 bf16 bars, and cheap enough for the SiLU-gating epilogue to
// keep pace with the tensor cores.
__device__ __forceinline__ float act_sigmoid(float x) {
  const float t = __expf(-fabsf(x));
  const float r = __frcp_rn(__fadd_rn(1.0f, t));
  return x >= 0.0f ? r : __fmul_rn(t, r);
}
__device__ __forceinline__ float act_silu(float x) { return __fmul_rn(x, act_sigmoid(x)); }
__device__ __forceinline__ float act_relu(float x) {
  return (x > 0.0f || x != x) ? x : 0.0f;
}
__device__ __forceinline__ float act_gelu(float x) {
  const float c = 0.7978845834732056f;   // float32(sqrt(2/pi))
  const float a = 0.044714998453855515f; // float32(0.044715)
  const float cube = __fmul_rn(__fmul_rn(__fmul_rn(a, x), x), x);
  const float t = tanhf(__fmul_rn(c, __fadd_rn(x, cube)));
  return __fmul_rn(__fmul_rn(0.5f, x), __fadd_rn(1.0f, t));
}
__device__ __forceinline__ float apply_act(float x, int act) {
  switch (act) {
    case ACT_RELU: return act_relu(x);
    case ACT_GELU: return act_gelu(x);
    case ACT_SILU: return act_silu(x);
    default: return x;
  }
}
// d act / d x at x (backward of bspmm_fused for model layers): relu' = [x > 0],
// silu' = s (1 + x (1 - s)) (kernels.py:37-39), gelu' of the tanh form.
__device__ __forceinline__ float apply_act_grad(float x, int act) {
  switch (act) {
    case ACT_RELU: return x > 0.0f ? 1.0f : 0.0f;
    case ACT_SILU: {
      const float s = act_sigmoid(x);
      return __fmul_rn(s, __fadd_rn(1.0f, __fmul_rn(x, __fsub_rn(1.0f, s))));
    }
    case ACT_GELU: {
      const float c = 0.7978845834732056f, a = 0.044714998453855515f;
      const float x2 = __fmul_rn(x, x);
      const float t = tanhf(__fmul_rn(c, __fadd_rn(x, __fmul_rn(__fmul_rn(a, x2), x))));
      const float du = __fmul_rn(c, __fadd_rn(1.0f, __fmul_rn(3.0f * a, x2)));
      return __fadd_rn(__fmul_rn(0.5f, __fadd_rn(1.0f, t)),
                       __fmul_rn(__fmul_rn(__fmul_rn(0.5f, x), __fsub_rn(1.0f, __fmul_rn(t, t))),
                                 du));
    }
    default: return 1.0f;
  }
}
// bf16-output variants (far below bf16 rounding, the 2e-2 bf16 bar): tanh.approx.f32 and
// ex2.approx instead of the accurate libm forms; the fp32 paths keep the forms above.
__device__ __forceinline__ float tanh_approx_f32(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float apply_act_fast(float x, int act) {
  switch (act) {
    case ACT_RELU: return act_relu(x);
    case ACT_GELU: {
      const float u = 0.7978845834732056f * fmaf(0.044714998453855515f * x, x * x, x);
      const float h = 0.5f * x;
      return fmaf(h, tanh_approx_f32(u), h);
    }
    case ACT_SILU: {
      const float h = 0.5f * x;
      return fmaf(h, tanh_approx_f32(h), h);
    }
    default: return x;
  }
}
__device__ __forceinline__ float apply_act_grad_fast(float x, int act) {
  switch (act) {
    case ACT_RELU: return x > 0.0f ? 1.0f : 0.0f;
    case ACT_SILU: {
      const float s = fmaf(0.5f, tanh_approx_f32(0.5f * x), 0.5f);  // sigmoid(x)
      return s * fmaf(x, 1.0f - s, 1.0f);
    }
    case ACT_GELU: {
      const float c = 0.7978845834732056f, a = 0.044714998453855515f;
      const float x2 = x * x;
      const float t = tanh_approx_f32(c * fmaf(a * x, x2, x));
      const float du = c * fmaf(3.0f * a, x2, 1.0f);
      return fmaf(0.5f * x * fmaf(-t, t, 1.0f), du, fmaf(0.5f, t, 0.5f));
    }
    default: return 1.0f;
  }
}
// g = (a * sigmoid(a)) * b
__device__ __forceinline__ float gated_fwd(float a, float b) {
  return __fmul_rn(__fmul_rn(a, act_sigmoid(a)), b);
}
// bf16-output variant of gated_fwd (the fp32 path keeps the split form above). Its error
// is far below bf16 rounding and the 2e-2 bf16 bar; limits: a -> -inf gives h - h = NaN at
// -inf exactly (the reference gives -inf * 0 = NaN), a -> +inf gives +inf, NaN propagates.
__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// silu(a) = h + h * tanh(h), h = a / 2: one MUFU op per element (tanh.approx, ~2^-11
// relative), which keeps the gated epilogue off the SFU ceiling.
__device__ __forceinline__ float gated_fwd_fast(float a, float b) {
  const float h = 0.5f * a;
  return fmaf(h, tanh_approx(h), h) * b;
}
// db = dg * (a*sig); da = (dg * b) * (sig * (1 + a * (1 - sig)))
__device__ __forceinline__ void gated_bwd(float dg, float a, float b, float& da, float& db) {
  const float sig = act_sigmoid(a);
  const float s = __fmul_rn(a, sig);
  db = __fmul_rn(dg, s);
  const float dsil = __fmul_rn(sig, __fadd_rn(1.0f, __fmul_rn(a, __fsub_rn(1.0f, sig))));
  da = __fmul_rn(__fmul_rn(dg, b), dsil);
}

// bf16-output variant of gated_bwd (the fp32 path keeps the form above): sigmoid from one
// tanh.approx (~2^-11 relative, far below bf16 rounding and the 2e-2 bf16 bar) instead of
// ex2 + a correctly rounded reciprocal, which kept the gating-backward epilogue SFU / ALU bound.
__device__ __forceinline__ void gated_bwd_fast(float dg, float a, float b, float& da, float& db) {
  const float sig = fmaf(0.5f, tanh_approx(0.5f * a), 0.5f);
  db = dg * (a * sig);
  da = (dg * b) * (sig * fmaf(a, 1.0f - sig, 1.0f));
}

template <typename T> __device__ __forceinline__ float to_f32(T v);
template <> __device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) {
  return __bfloat162float(v);
}
template <typename T> __device__ __forceinline__ T from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

}  // namespace blast
