// Single-CTA inclusive-to-exclusive prefix sum used by the plan and repack
// builders: ptr[0] = 0, ptr[l+1] = sum(count[0..l]) where the counts were
// written to ptr[1..lines]. Launch with one CTA of up to 1024 threads.
#pragma once
#include <stdint.h>

namespace blast {

template <typename T>
__global__ void offsets_scan_kernel(T* ptr, int64_t lines) {
  __shared__ T warp_sums[32];
  __shared__ T carry;
  if (threadIdx.x == 0) {
    carry = 0;
    ptr[0] = 0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t base = 0; base < lines; base += blockDim.x) {
    const int64_t l = base + threadIdx.x;
    T v = l < lines ? ptr[l + 1] : T(0);
    for (int o = 1; o < 32; o <<= 1) {
      const T n = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += n;
    }
    if (lane == 31) warp_sums[wid] = v;
    __syncthreads();
    if (wid == 0) {
      T w = lane < static_cast<int>(blockDim.x >> 5) ? warp_sums[lane] : T(0);
      for (int o = 1; o < 32; o <<= 1) {
        const T n = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += n;
      }
      warp_sums[lane] = w;
    }
    __syncthreads();
    const T prefix = (wid > 0 ? warp_sums[wid - 1] : T(0)) + carry;
    if (l < lines) ptr[l + 1] = v + prefix;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = v + prefix;
    __syncthreads();
  }
}

}  // namespace blast
