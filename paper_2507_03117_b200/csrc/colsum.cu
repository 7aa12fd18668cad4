// Column sums of a row-major [m, n] matrix into fp32 [n]: the bias gradients of a layer
// with bias (the GPT2MLP integration), sum over tokens. Deterministic: the
// rows are cut into a fixed number of splits, each CTA sums its split in a fixed order
// (8 row groups, combined in order through shared memory), and the split partials are added
// in split order by a second kernel. 16-byte loads: a thread owns 8 (bf16) / 4 (fp32)
// adjacent columns, a warp a 256 / 128-column run of one row.
#include <cuda_bf16.h>

#include "host.hpp"

namespace blast {

constexpr int kCsRowGroups = 8;  // warps per CTA, each walks every 8th row of the split

template <typename T>
__global__ void __launch_bounds__(256) colsum_partial_kernel(const T* __restrict__ x, int64_t m,
                                                             int64_t n, int64_t rows_per,
                                                             float* __restrict__ part) {
  constexpr int V = 16 / sizeof(T);          // columns per thread
  constexpr int COLS = 32 * V;               // columns per CTA
  __shared__ float red[kCsRowGroups][COLS];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t c0 = blockIdx.x * static_cast<int64_t>(COLS) + lane * V;
  const int64_t r0 = blockIdx.y * rows_per, r1 = min(m, r0 + rows_per);
  float acc[V];
#pragma unroll
  for (int i = 0; i < V; ++i) acc[i] = 0.0f;
  const bool vec = (c0 + V <= n) && (n % V == 0);
  // U rows' loads in flight per thread, added in row order (same sums as one row at a time)
  constexpr int U = 8;
  auto add = [&](const uint4& w) {
    if constexpr (sizeof(T) == 2) {
      const uint32_t h[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&h[i]));
        acc[2 * i] += f.x;
        acc[2 * i + 1] += f.y;
      }
    } else {
      acc[0] += __uint_as_float(w.x); acc[1] += __uint_as_float(w.y);
      acc[2] += __uint_as_float(w.z); acc[3] += __uint_as_float(w.w);
    }
  };
  if (vec) {
    for (int64_t rb = r0 + g; rb < r1; rb += static_cast<int64_t>(kCsRowGroups) * U) {
      uint4 w[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t r = rb + static_cast<int64_t>(u) * kCsRowGroups;
        if (r < r1) w[u] = __ldcs(reinterpret_cast<const uint4*>(x + r * n + c0));
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (rb + static_cast<int64_t>(u) * kCsRowGroups < r1) add(w[u]);
    }
  }
  for (int64_t r = r0 + g; !vec && r < r1; r += kCsRowGroups) {
    const T* row = x + r * n;
    {
#pragma unroll
      for (int i = 0; i < V; ++i)
        if (c0 + i < n) {
          if constexpr (sizeof(T) == 2)
            acc[i] += __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(row)[c0 + i]);
          else
            acc[i] += reinterpret_cast<const float*>(row)[c0 + i];
        }
    }
  }
#pragma unroll
  for (int i = 0; i < V; ++i) red[g][lane * V + i] = acc[i];
  __syncthreads();
  for (int col = threadIdx.x; col < COLS; col += blockDim.x) {
    float s = 0.0f;
#pragma unroll
    for (int k = 0; k < kCsRowGroups; ++k) s += red[k][col];  // fixed order
    const int64_t c = blockIdx.x * static_cast<int64_t>(COLS) + col;
    if (c < n) part[blockIdx.y * n + c] = s;
  }
}

__global__ void colsum_final_kernel(const float* __restrict__ part, int64_t splits, int64_t n,
                                    float* __restrict__ out) {
  const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (c >= n) return;
  float s = 0.0f;
  int64_t k = 0;
  for (; k + 8 <= splits; k += 8) {  // 8 loads in flight, added in split order
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = part[(k + u) * n + c];
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  for (; k < splits; ++k) s += part[k * n + c];  // split order
  out[c] = s;
}

}  // namespace blast

using namespace blast;

extern "C" int blast_column_sums(const void* x, int dtype, int64_t m, int64_t n, float* out,
                                 void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (m < 0 || n < 0 || (dtype != BLAST_BF16 && dtype != BLAST_F32)) {
    set_error("column_sums: invalid shape or dtype");
    return BLAST_EINVAL;
  }
  if (n == 0) return BLAST_OK;
  if (m == 0) return cuda_status(cudaMemsetAsync(out, 0, sizeof(float) * n, st), "column_sums");
  const int cols_per_cta = dtype == BLAST_BF16 ? 256 : 128;
  const int64_t col_blocks = cdiv(n, cols_per_cta);
  // enough CTAs for the whole GPU, each split at least 64 rows
  int64_t splits = std::max<int64_t>(1, std::min<int64_t>(cdiv(4 * num_sms(), col_blocks), cdiv(m, 64)));
  const int64_t rows_per = cdiv(m, splits);
  splits = cdiv(m, rows_per);
  Scratch part;
  if (!part.alloc(sizeof(float) * splits * n, st)) return cuda_status(cudaGetLastError(), "column_sums");
  const dim3 grid(static_cast<unsigned>(col_blocks), static_cast<unsigned>(splits));
  if (dtype == BLAST_BF16)
    colsum_partial_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(x), m, n, rows_per, part.as<float>());
  else
    colsum_partial_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(x), m, n,
                                                       rows_per, part.as<float>());
  colsum_final_kernel<<<static_cast<unsigned>(cdiv(n, 256)), 256, 0, st>>>(part.as<float>(), splits,
                                                                           n, out);
  return check_launch("column_sums");
}
