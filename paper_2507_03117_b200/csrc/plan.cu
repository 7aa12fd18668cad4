// Block index maps and execution plans.
//
// kmap[r][c] = stored block index or -1 is the inverse of the BCSC arrays
// (bcsc.py:205-210). A plan is the per-output-line step list the tile engine
// walks: for column lines (Y = X W) the steps of block column j are its stored
// blocks in ascending block row (kernels.py:117-121); for row lines
// (Y = X W^T) the steps of block row i are in ascending block column, the
// order in which bspmm_rt accumulates into output block row i
// (kernels.py:159-167). Two maps of the same grid (gate/up) merge into one
// step list so a single A panel load feeds both products.
#include "activations.cuh"
#include "host.hpp"

namespace blast {

__global__ void kmap_fill_kernel(int32_t* kmap, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    kmap[i] = -1;
}

// one warp per block column
__global__ void kmap_scatter_kernel(const int64_t* col_ptr, const int32_t* row_idx, int64_t gc,
                                    int32_t* kmap) {
  const int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= gc) return;
  for (int64_t s = col_ptr[j] + lane; s < col_ptr[j + 1]; s += 32)
    kmap[(int64_t)row_idx[s] * gc + j] = static_cast<int32_t>(s);
}

__device__ __forceinline__ int64_t plan_index(int64_t line, int64_t i, int64_t gc, int by_rows) {
  return by_rows ? line * gc + i : i * gc + line;
}

// one warp per line: number of steps
__global__ void plan_count_kernel(const int32_t* kmap0, const int32_t* kmap1, int64_t gr,
                                  int64_t gc, int by_rows, int32_t* step_ptr) {
  const int64_t lines = by_rows ? gr : gc;
  const int64_t inner = by_rows ? gc : gr;
  const int64_t line = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (line >= lines) return;
  int count = 0;
  for (int64_t base = 0; base < inner; base += 32) {
    const int64_t i = base + lane;
    bool present = false;
    if (i < inner) {
      const int64_t idx = plan_index(line, i, gc, by_rows);
      present = kmap0[idx] >= 0 || (kmap1 && kmap1[idx] >= 0);
    }
    count += __popc(__ballot_sync(0xffffffffu, present));
  }
  if (lane == 0) step_ptr[line + 1] = count;
}

// single CTA exclusive scan: step_ptr[0] = 0, step_ptr[l+1] = sum(count[0..l])
__global__ void plan_scan_kernel(int32_t* step_ptr, int64_t lines) {
  __shared__ int32_t warp_sums[32];
  __shared__ int32_t carry;
  if (threadIdx.x == 0) {
    carry = 0;
    step_ptr[0] = 0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t base = 0; base < lines; base += blockDim.x) {
    const int64_t l = base + threadIdx.x;
    int v = l < lines ? step_ptr[l + 1] : 0;
    // inclusive warp scan
    for (int o = 1; o < 32; o <<= 1) {
      int n = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += n;
    }
    if (lane == 31) warp_sums[wid] = v;
    __syncthreads();
    if (wid == 0) {
      int w = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        int n = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += n;
      }
      warp_sums[lane] = w;
    }
    __syncthreads();
    const int prefix = (wid > 0 ? warp_sums[wid - 1] : 0) + carry;
    if (l < lines) step_ptr[l + 1] = v + prefix;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = v + prefix;
    __syncthreads();
  }
}

__global__ void plan_fill_kernel(const int32_t* kmap0, const int32_t* kmap1, int64_t gr,
                                 int64_t gc, int by_rows, const int32_t* step_ptr, int4* steps,
                                 int32_t* flags) {
  const int64_t lines = by_rows ? gr : gc;
  const int64_t inner = by_rows ? gc : gr;
  const int64_t line = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (line >= lines) return;
  int out = step_ptr[line];
  int f = 0, seen = 0;  // seen: warp-uniform, matrices with a block in earlier chunks
  int n0 = 0, n1 = 0;   // blocks of matrix 0 / 1 in the line (warp-uniform)
  for (int64_t base = 0; base < inner; base += 32) {
    const int64_t i = base + lane;
    int k0 = -1, k1 = -1;
    if (i < inner) {
      const int64_t idx = plan_index(line, i, gc, by_rows);
      k0 = kmap0[idx];
      k1 = kmap1 ? kmap1[idx] : -1;
    }
    const bool present = k0 >= 0 || k1 >= 0;
    const unsigned bal = __ballot_sync(0xffffffffu, present);
    // .w: presence and first-occurrence bits, so the MMA issuer reads a step's recipe
    // with one shuffle: bit 0/1 block of matrix 0/1, bit 2/3 its first block in the line
    const unsigned lt = (1u << lane) - 1u;
    const unsigned bal0 = __ballot_sync(0xffffffffu, k0 >= 0);
    const unsigned bal1 = __ballot_sync(0xffffffffu, k1 >= 0);
    const bool first0 = k0 >= 0 && !(seen & 1) && !(bal0 & lt);
    const bool first1 = k1 >= 0 && !(seen & 2) && !(bal1 & lt);
    seen |= (bal0 ? 1 : 0) | (bal1 ? 2 : 0);
    n0 += __popc(bal0);
    n1 += __popc(bal1);
    if (present) {
      const int pos = out + __popc(bal & lt);
      steps[pos] = make_int4(static_cast<int>(i), k0, k1,
                             (k0 >= 0 ? 1 : 0) | (k1 >= 0 ? 2 : 0) | (first0 ? 4 : 0) |
                                 (first1 ? 8 : 0));
    }
    f |= (k0 >= 0 ? 1 : 0) | (k1 >= 0 ? 2 : 0);
    out += __popc(bal);
  }
  for (int o = 16; o > 0; o >>= 1) f |= __shfl_xor_sync(0xffffffffu, f, o);
  // bits 0/1: matrix 0/1 present; bits 2..16 / 17..31: its block count (inner < 2^15)
  if (lane == 0) flags[line] = f | (min(n0, 0x7fff) << 2) | (min(n1, 0x7fff) << 17);
}

__device__ __forceinline__ void tf32_split1(float v, float& h, float& l) {
  h = v;
  l = 0.0f;
  if (isfinite(v)) {
    h = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
    l = __fsub_rn(v, h);
  }
}
// 16-byte vectors, 4 per thread in flight (scalar tail for n % 4 or unaligned buffers)
__global__ void split_tf32_kernel(const float* x, float* hi, float* lo, int64_t n) {
  // hi may be null (lo only: the raw x serves as the hi operand)
  const bool vec = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(hi) |
                     reinterpret_cast<uintptr_t>(lo)) & 15u) == 0;
  const int64_t n4 = vec ? n / 4 : 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n4; i0 += 4 * stride) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i0 + u * stride < n4) v[u] = __ldg(x4 + i0 + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = i0 + u * stride;
      if (i >= n4) break;
      float4 h, l;
      tf32_split1(v[u].x, h.x, l.x);
      tf32_split1(v[u].y, h.y, l.y);
      tf32_split1(v[u].z, h.z, l.z);
      tf32_split1(v[u].w, h.w, l.w);
      if (hi) reinterpret_cast<float4*>(hi)[i] = h;
      reinterpret_cast<float4*>(lo)[i] = l;
    }
  }
  for (int64_t i = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    float h, l;
    tf32_split1(x[i], h, l);
    if (hi) hi[i] = h;
    lo[i] = l;
  }
}

// hi/lo split of every block, once as stored (rt) and once transposed (fwd)
__global__ void tf32_prepare_kernel(const float* v, int64_t n, int b, float* fhi, float* flo,
                                    float* rhi, float* rlo) {
  const int64_t bb = static_cast<int64_t>(b) * b;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float x = v[i];
    float h = x, l = 0.0f;
    if (isfinite(x)) {
      h = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
      l = __fsub_rn(x, h);
    }
    rhi[i] = h;
    rlo[i] = l;
    const int64_t k = i / bb, e = i - k * bb;
    const int64_t r = e / b, c = e - r * b;
    const int64_t t = k * bb + c * b + r;
    fhi[t] = h;
    flo[t] = l;
  }
}

template <typename T>
__global__ void activation_kernel(const T* x, T* y, int64_t n, int act) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = from_f32<T>(apply_act(to_f32<T>(x[i]), act));
}

static int grid_for(int64_t n, int threads) {
  int64_t g = cdiv(n, threads);
  const int64_t cap = (int64_t)num_sms() * 16;
  if (g > cap) g = cap;
  return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace blast

using namespace blast;

extern "C" int blast_kmap_from_bcsc(const int64_t* col_ptr, const int32_t* row_idx,
                                    int64_t grid_rows, int64_t grid_cols, int32_t* kmap,
                                    void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t n = grid_rows * grid_cols;
  if (n <= 0) return BLAST_OK;
  kmap_fill_kernel<<<grid_for(n, 256), 256, 0, st>>>(kmap, n);
  kmap_scatter_kernel<<<static_cast<int>(cdiv(grid_cols * 32, 256)), 256, 0, st>>>(
      col_ptr, row_idx, grid_cols, kmap);
  return check_launch("kmap_from_bcsc");
}

extern "C" int blast_build_plan(const int32_t* kmap0, const int32_t* kmap1, int64_t grid_rows,
                                int64_t grid_cols, int by_rows, int32_t* step_ptr,
                                int32_t* steps, int32_t* flags, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t lines = by_rows ? grid_rows : grid_cols;
  if (lines <= 0) return BLAST_OK;
  const int blocks = static_cast<int>(cdiv(lines * 32, 256));
  plan_count_kernel<<<blocks, 256, 0, st>>>(kmap0, kmap1, grid_rows, grid_cols, by_rows,
                                            step_ptr);
  plan_scan_kernel<<<1, 1024, 0, st>>>(step_ptr, lines);
  plan_fill_kernel<<<blocks, 256, 0, st>>>(kmap0, kmap1, grid_rows, grid_cols, by_rows, step_ptr,
                                           reinterpret_cast<int4*>(steps), flags);
  return check_launch("build_plan");
}

extern "C" int blast_split_tf32(const float* x, float* hi, float* lo, int64_t n, void* stream) {
  if (n <= 0) return BLAST_OK;
  split_tf32_kernel<<<grid_for(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(x, hi, lo, n);
  return check_launch("split_tf32");
}

extern "C" int blast_tf32_prepare(const float* values, int64_t nnzb, int32_t block,
                                  float* fwd_hi, float* fwd_lo, float* rt_hi, float* rt_lo,
                                  void* stream) {
  const int64_t n = nnzb * block * block;
  if (n <= 0) return BLAST_OK;
  tf32_prepare_kernel<<<grid_for(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      values, n, block, fwd_hi, fwd_lo, rt_hi, rt_lo);
  return check_launch("tf32_prepare");
}

extern "C" int blast_activation(const void* x, void* y, int64_t n, int dtype, int act,
                                void* stream) {
  if (n <= 0) return BLAST_OK;
  if (act < 0 || act > 3) {
    set_error("unknown nonlinearity code %d", act);
    return BLAST_EINVAL;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == BLAST_BF16)
    activation_kernel<__nv_bfloat16><<<grid_for(n, 256), 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(x), static_cast<__nv_bfloat16*>(y), n, act);
  else
    activation_kernel<float><<<grid_for(n, 256), 256, 0, st>>>(static_cast<const float*>(x),
                                                               static_cast<float*>(y), n, act);
  return check_launch("activation");
}
