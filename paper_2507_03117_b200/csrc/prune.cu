// Blocked prune-and-grow on device (pruner.py:88-186, bcsc.py:175-214).
//
//   blast_block_norms       fp64 Frobenius norm per b x b block      pruner.py:88-98
//   blast_topk_mask         exact top-k with (col, row) tie-break    pruner.py:101-125
//   blast_mask_difference   regrown = grad_sel & ~kept + counts      pruner.py:142-156
//   blast_repack_index      store grid -> col_ptr + kmap             bcsc.py:200-206
//   blast_repack_rows       block_row_idx (column-major walk)        bcsc.py:207-209
//   blast_apply_mask_gather masked = w * mask; values <- blocks      pruner.py:183-186, bcsc.py:210
//
// All reductions use a fixed order (no floating-point atomics), so masks and
// norms are bitwise reproducible run to run.
#include "activations.cuh"
#include "host.hpp"
#include "ptx.cuh"

namespace blast {

// ------------------------------------------------------------------ block norms
// One warp per block; lanes walk the block row-major with 16-byte loads when the
// geometry allows it, accumulating x*x in float64 (each product of two fp32
// values is exact in fp64, as in pruner.py:95's astype(float64)). The warp
// reduction tree is fixed, so the result is deterministic.
__device__ __forceinline__ double to_f64(double v) { return v; }
__device__ __forceinline__ double to_f64(float v) { return static_cast<double>(v); }
__device__ __forceinline__ double to_f64(__nv_bfloat16 v) {
  return static_cast<double>(__bfloat162float(v));
}

template <typename T, bool VEC>
__global__ void __launch_bounds__(256) block_norms_kernel(const T* __restrict__ x,
                                                          const T* __restrict__ x2, int64_t rows,
                                                          int64_t cols, int b, int64_t gr,
                                                          int64_t gc, double* __restrict__ out,
                                                          double* __restrict__ out2) {
  const int64_t nblk = gr * gc;
  const int64_t wg = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const T* src = blockIdx.y == 0 ? x : x2;
  double* dst = blockIdx.y == 0 ? out : out2;
  for (int64_t blk = wg; blk < nblk; blk += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t r = blk / gc, c = blk - r * gc;
    const int64_t i0 = r * b, j0 = c * b;
    const int64_t ih = (i0 + b < rows ? i0 + b : rows) - i0;
    const int64_t jw = (j0 + b < cols ? j0 + b : cols) - j0;
    double acc = 0.0;
    if constexpr (VEC) {
      // b % VW == 0 and full blocks only (dispatch guarantees it)
      constexpr int VW = 16 / sizeof(T);
      const int per_row = b / VW;
      const int total = b * per_row;
      // U loads in flight per lane before their FMAs (the products are still accumulated in
      // ascending e, so the sum is bitwise the one-load-at-a-time loop's)
      constexpr int U = 8;
      for (int e0 = lane; e0 < total; e0 += 32 * U) {
        uint4 qs[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = e0 + 32 * u;
          if (e < total) {
            const int ii = e / per_row, jj = (e - ii * per_row) * VW;
            qs[u] = __ldg(reinterpret_cast<const uint4*>(src + (i0 + ii) * cols + j0 + jj));
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
        if (e0 + 32 * u >= total) break;
        const uint4 q = qs[u];
        if constexpr (sizeof(T) == 8) {
          const double d0 = __hiloint2double(static_cast<int>(q.y), static_cast<int>(q.x));
          const double d1 = __hiloint2double(static_cast<int>(q.w), static_cast<int>(q.z));
          acc = fma(d0, d0, acc);
          acc = fma(d1, d1, acc);
        } else if constexpr (sizeof(T) == 4) {
          const float f[4] = {__uint_as_float(q.x), __uint_as_float(q.y), __uint_as_float(q.z),
                              __uint_as_float(q.w)};
#pragma unroll
          for (int h = 0; h < 4; ++h) acc = fma((double)f[h], (double)f[h], acc);
        } else {
          const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[h]));
            acc = fma((double)f.x, (double)f.x, acc);
            acc = fma((double)f.y, (double)f.y, acc);
          }
        }
        }
      }
    } else {
      const int64_t total = ih * jw;
      for (int64_t e = lane; e < total; e += 32) {
        const int64_t ii = e / jw, jj = e - ii * jw;
        const double v = to_f64(src[(i0 + ii) * cols + j0 + jj]);
        acc = fma(v, v, acc);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) dst[blk] = sqrt(acc);
  }
}

// ------------------------------------------------------------------ top-k
// Sort key of pruner.py:118-124: lexsort((row, col, -norm)) == ascending
// (K1(-norm), lin) with lin = col * grid_rows + row (column-major block index).
// K1 is the order-preserving uint64 image of the float64 -norm: -0.0 is folded
// onto +0.0 (equal in numpy's comparison sort) and every NaN maps to the
// largest key (numpy sorts NaN last).
__device__ __forceinline__ uint64_t norm_key(double norm) {
  double v = -norm;
  if (v != v) return ~0ull;
  if (v == 0.0) v = 0.0;
  const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(v));
  return (bits >> 63) ? ~bits : (bits | 0x8000000000000000ull);
}

struct TopkState {
  unsigned int count;   // grid barrier arrivals
  unsigned int gen;     // grid barrier generation
  unsigned int pad[2];
  unsigned int hist[2][2048];
};

__device__ __forceinline__ void grid_barrier(TopkState* st, unsigned int nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* gen = &st->gen;
    const unsigned int g = *gen;
    __threadfence();
    if (atomicAdd(&st->count, 1u) == nblocks - 1) {
      st->count = 0;
      __threadfence();
      atomicAdd(&st->gen, 1u);
    } else {
      while (*gen == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// Radix select on the 96-bit composite (K1, lin) in 11-bit digits: 6 passes
// over K1 (64 bits), then 3 over lin restricted to K1 == threshold. Every CTA
// histograms its cells into a global histogram with integer atomics (order
// independent), then after a grid barrier each CTA scans it redundantly to
// pick the digit holding the k-th smallest key.
__global__ void __launch_bounds__(1024) topk_kernel(const double* __restrict__ norms, int64_t gr,
                                                    int64_t gc, int64_t k,
                                                    uint8_t* __restrict__ keep, TopkState* st) {
  __shared__ unsigned int sh[2048];
  __shared__ unsigned int wsum[32];
  __shared__ int sel_bucket;
  __shared__ unsigned int sel_below;
  const int64_t n = gr * gc;
  const unsigned int nblocks = gridDim.x;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;

  uint64_t pre1 = 0;       // selected K1 prefix (bits above the current digit)
  uint32_t pre2 = 0;       // selected lin prefix
  int64_t krem = k;        // rank still to place inside the current prefix
  int pass = 0;
  // digit table: (which key, shift, width)
  const int shifts[9] = {53, 42, 31, 20, 9, 0, 21, 10, 0};
  const int widths[9] = {11, 11, 11, 11, 11, 9, 11, 11, 10};
  for (pass = 0; pass < 9; ++pass) {
    const int sh_ = shifts[pass], w = widths[pass];
    const bool on_lin = pass >= 6;
    const int buf = pass & 1;
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    for (int64_t idx = tid; idx < n; idx += nthreads) {
      const uint64_t k1 = norm_key(norms[idx]);
      unsigned int digit;
      if (!on_lin) {
        const int top = sh_ + w;  // bits [top, 64) must match pre1
        if (top < 64 && (k1 >> top) != (pre1 >> top)) continue;
        digit = static_cast<unsigned int>((k1 >> sh_) & ((1ull << w) - 1));
      } else {
        if (k1 != pre1) continue;
        const int64_t r = idx / gc, c = idx - r * gc;
        const uint32_t lin = static_cast<uint32_t>(c * gr + r);
        const int top = sh_ + w;
        if (top < 32 && (lin >> top) != (pre2 >> top)) continue;
        digit = (lin >> sh_) & ((1u << w) - 1);
      }
      atomicAdd(&sh[digit], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 2048; i += blockDim.x)
      if (sh[i]) atomicAdd(&st->hist[buf][i], sh[i]);
    grid_barrier(st, nblocks);
    // scan the global histogram (2048 bins, 2 per thread)
    const unsigned int h0 = st->hist[buf][2 * threadIdx.x];
    const unsigned int h1 = st->hist[buf][2 * threadIdx.x + 1];
    unsigned int v = h0 + h1;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned int t = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += t;
    }
    if (lane == 31) wsum[wid] = v;
    __syncthreads();
    if (wid == 0) {
      unsigned int s = wsum[lane];
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned int t = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += t;
      }
      wsum[lane] = s;
    }
    __syncthreads();
    const unsigned int incl = v + (wid > 0 ? wsum[wid - 1] : 0u);  // inclusive through bin 2t+1
    const unsigned int excl = incl - h0 - h1;                       // before bin 2t
    const uint64_t kr = static_cast<uint64_t>(krem);
    if (excl < kr && kr <= excl + h0) {
      sel_bucket = 2 * threadIdx.x;
      sel_below = excl;
    } else if (excl + h0 < kr && kr <= incl) {
      sel_bucket = 2 * threadIdx.x + 1;
      sel_below = excl + h0;
    }
    // clear the other buffer for the next pass (nobody reads it in this pass)
    for (int i = threadIdx.x; i < 2048; i += blockDim.x)
      if (blockIdx.x == 0) st->hist[buf ^ 1][i] = 0;
    __syncthreads();
    krem -= sel_below;
    if (!on_lin) pre1 |= static_cast<uint64_t>(sel_bucket) << sh_;
    else pre2 |= static_cast<uint32_t>(sel_bucket) << sh_;
    grid_barrier(st, nblocks);
  }
  // keep = (K1 < T1) || (K1 == T1 && lin <= T2)
  for (int64_t idx = tid; idx < n; idx += nthreads) {
    const uint64_t k1 = norm_key(norms[idx]);
    bool kp = k1 < pre1;
    if (k1 == pre1) {
      const int64_t r = idx / gc, c = idx - r * gc;
      kp = static_cast<uint32_t>(c * gr + r) <= pre2;
    }
    keep[idx] = kp ? 1 : 0;
  }
}

// Single-CTA top-k for grids whose keys fit in shared memory (the common case:
// the Llama-3-8B grid is 14,336 cells, 70B 57,344 at b=64 goes to topk_kernel).
// Same composite key and selection as topk_kernel, radix passes of 8 bits over
// the 64-bit norm key, then over the column-major index among exact ties. No
// grid barriers and no scratch; blockIdx.x selects one of two independent grids
// (the weight and gradient selections of generate_masks run in one launch).
// one warp scans the 256 bins (8 per lane) and names the bucket holding the krem-th key:
// its index, the count of keys in lower buckets and its own count
__device__ __forceinline__ void topk_pick_bucket(const unsigned int* hist, unsigned int krem,
                                                 unsigned int* bucket, unsigned int* below_out,
                                                 unsigned int* count) {
  unsigned int local[8], sum = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    local[j] = hist[threadIdx.x * 8 + j];
    sum += local[j];
  }
  unsigned int incl = sum;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (threadIdx.x >= static_cast<unsigned int>(o)) incl += t;
  }
  unsigned int below = incl - sum;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (below < krem && krem <= below + local[j]) {
      *bucket = threadIdx.x * 8 + j;
      *below_out = below;
      *count = local[j];
    }
    below += local[j];
  }
}

constexpr int kTopkSmemMax = 24576;

// regrown / counts (optional, two grids): the fused set difference of pruner.py:142-156 —
// launched as a cluster of the two CTAs, CTA 1 (grad_sel) waits for CTA 0's kept grid at the
// cluster barrier and writes regrown = grad_sel & ~kept (regrown may alias keep1) and the
// (kept, regrown) counts.
__global__ void __launch_bounds__(1024) topk_smem_kernel(const double* __restrict__ norms0,
                                                         uint8_t* keep0,
                                                         const double* __restrict__ norms1,
                                                         uint8_t* keep1, int64_t gr,
                                                         int64_t gc, int64_t k, uint8_t* regrown,
                                                         unsigned long long* counts) {
  extern __shared__ uint64_t keys[];
  __shared__ unsigned int hist[256];
  __shared__ unsigned int sel_bucket, sel_below;
  const double* norms = blockIdx.x == 0 ? norms0 : norms1;
  uint8_t* keep = blockIdx.x == 0 ? keep0 : keep1;
  const int n = static_cast<int>(gr * gc);
  // 8 independent loads in flight per thread (the norms come from L2 / HBM)
  for (int i0 = threadIdx.x; i0 < n; i0 += 8 * blockDim.x) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * blockDim.x;
      v[u] = i < n ? __ldg(&norms[i]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < n) keys[i] = norm_key(v[u]);
    }
  }
  __shared__ unsigned int sel_count;
  __shared__ uint64_t red_and[32], red_or[32];
  // bits common to every key: the radix passes start below them (block norms of similar
  // magnitude share sign, exponent and the top mantissa bits)
  {
    uint64_t ka = ~0ull, ko = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      ka &= keys[i];
      ko |= keys[i];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ka &= __shfl_xor_sync(0xffffffffu, ka, o);
      ko |= __shfl_xor_sync(0xffffffffu, ko, o);
    }
    if ((threadIdx.x & 31) == 0) {
      red_and[threadIdx.x >> 5] = ka;
      red_or[threadIdx.x >> 5] = ko;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int nw = static_cast<int>(blockDim.x >> 5);
      ka = threadIdx.x < nw ? red_and[threadIdx.x] : ~0ull;
      ko = threadIdx.x < nw ? red_or[threadIdx.x] : 0ull;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        ka &= __shfl_xor_sync(0xffffffffu, ka, o);
        ko |= __shfl_xor_sync(0xffffffffu, ko, o);
      }
      if (threadIdx.x == 0) {
        red_and[0] = ka;
        red_or[0] = ko;
      }
    }
    __syncthreads();
  }
  const uint64_t kdiff = red_and[0] ^ red_or[0];
  int top = kdiff ? 64 - __clzll(static_cast<long long>(kdiff)) : 0;  // bits [top, 64) common
  uint64_t pre1 = top >= 64 ? 0ull : (top == 0 ? red_and[0] : (red_and[0] >> top) << top);
  uint32_t pre2 = 0;
  unsigned int krem = static_cast<unsigned int>(k);
  uint64_t thr_all = 0;  // early exit: every key <= thr_all is selected (no tie-break needed)
  bool early = false;
  // digits of <= 8 bits over K1 from the highest differing bit, then 2 passes over lin among
  // exact ties (n <= 24576 < 2^16); stops as soon as the bucket holding the k-th key is
  // selected whole (it holds exactly the keys still needed)
  while (top > 0 && !early) {
    const int sh = top > 8 ? top - 8 : 0;
    const int w = top - sh;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int idx = threadIdx.x; idx < n; idx += blockDim.x) {
      const uint64_t k1 = keys[idx];
      if (top < 64 && (k1 >> top) != (pre1 >> top)) continue;
      const unsigned int digit = static_cast<unsigned int>((k1 >> sh) & ((1ull << w) - 1));
      // warp-aggregated: keys of similar norms share digits
      const unsigned int peers = __match_any_sync(__activemask(), digit);
      if ((threadIdx.x & 31) == static_cast<unsigned int>(__ffs(peers) - 1))
        atomicAdd(&hist[digit], static_cast<unsigned int>(__popc(peers)));
    }
    __syncthreads();
    if (threadIdx.x < 32) topk_pick_bucket(hist, krem, &sel_bucket, &sel_below, &sel_count);
    __syncthreads();
    krem -= sel_below;
    pre1 |= static_cast<uint64_t>(sel_bucket) << sh;
    if (sel_count == krem) {  // the whole bucket is selected: done
      thr_all = sh ? (pre1 | ((uint64_t(1) << sh) - 1)) : pre1;
      early = true;
    }
    top = sh;
    __syncthreads();
  }
  // exact ties on K1 (pre1 is the k-th key): two 8-bit passes over the column-major index
  for (int lp = 0; lp < 2 && !early; ++lp) {
    const int sh = (1 - lp) * 8;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int idx = threadIdx.x; idx < n; idx += blockDim.x) {
      if (keys[idx] != pre1) continue;
      const int r = idx / static_cast<int>(gc), c = idx - r * static_cast<int>(gc);
      const uint32_t lin = static_cast<uint32_t>(c * gr + r);
      if (lp == 1 && (lin >> 8) != (pre2 >> 8)) continue;
      atomicAdd(&hist[(lin >> sh) & 0xFF], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) topk_pick_bucket(hist, krem, &sel_bucket, &sel_below, &sel_count);
    __syncthreads();
    krem -= sel_below;
    pre2 |= static_cast<uint32_t>(sel_bucket) << sh;
    __syncthreads();
  }
  for (int idx = threadIdx.x; idx < n; idx += blockDim.x) {
    const uint64_t k1 = keys[idx];
    bool kp = early ? k1 <= thr_all : k1 < pre1;
    if (!early && k1 == pre1) {
      const int r = idx / static_cast<int>(gc), c = idx - r * static_cast<int>(gc);
      kp = static_cast<uint32_t>(c * gr + r) <= pre2;
    }
    keep[idx] = kp ? 1 : 0;
  }
  if (counts != nullptr) {
    cluster_sync();  // release / acquire: CTA 0's kept grid is visible to CTA 1
    if (blockIdx.x == 1) {
      unsigned long long ck = 0, cr = 0;
      for (int idx = threadIdx.x; idx < n; idx += blockDim.x) {
        const bool kp = keep0[idx] != 0;
        const bool rg = keep1[idx] != 0 && !kp;
        regrown[idx] = rg ? 1 : 0;
        ck += kp;
        cr += rg;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        ck += __shfl_xor_sync(0xffffffffu, ck, o);
        cr += __shfl_xor_sync(0xffffffffu, cr, o);
      }
      if ((threadIdx.x & 31) == 0) {
        red_and[threadIdx.x >> 5] = ck;
        red_or[threadIdx.x >> 5] = cr;
      }
      __syncthreads();
      if (threadIdx.x < 32) {
        const int nw = static_cast<int>(blockDim.x >> 5);
        ck = threadIdx.x < nw ? red_and[threadIdx.x] : 0ull;
        cr = threadIdx.x < nw ? red_or[threadIdx.x] : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          ck += __shfl_xor_sync(0xffffffffu, ck, o);
          cr += __shfl_xor_sync(0xffffffffu, cr, o);
        }
        if (threadIdx.x == 0) {
          counts[0] = ck;
          counts[1] = cr;
        }
      }
    }
  }
}

__global__ void fill_u8_kernel(uint8_t* p, int64_t n, uint8_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void mask_difference_kernel(const uint8_t* kept, const uint8_t* gsel, int64_t n,
                                       uint8_t* regrown, unsigned long long* counts) {
  unsigned long long ck = 0, cr = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool kp = kept[i] != 0;
    const bool rg = gsel[i] != 0 && !kp;
    regrown[i] = rg ? 1 : 0;
    ck += kp;
    cr += rg;
  }
  for (int o = 16; o > 0; o >>= 1) {
    ck += __shfl_xor_sync(0xffffffffu, ck, o);
    cr += __shfl_xor_sync(0xffffffffu, cr, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&counts[0], ck);
    atomicAdd(&counts[1], cr);
  }
}

// ------------------------------------------------------------------ repack
// store grid from masks (kept | regrown) or from dense contents (any x != 0).
template <typename T>
__global__ void store_from_dense_kernel(const T* x, int64_t rows, int64_t cols, int b, int64_t gr,
                                        int64_t gc, uint8_t* store) {
  const int64_t nblk = gr * gc;
  const int64_t wg = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t blk = wg; blk < nblk; blk += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t r = blk / gc, c = blk - r * gc;
    const int64_t i0 = r * b, j0 = c * b;
    const int64_t ih = (i0 + b < rows ? i0 + b : rows) - i0;
    const int64_t jw = (j0 + b < cols ? j0 + b : cols) - j0;
    bool nz = false;
    for (int64_t e = lane; e < ih * jw && !nz; e += 32) {
      const int64_t ii = e / jw, jj = e - ii * jw;
      nz = to_f32<T>(x[(i0 + ii) * cols + j0 + jj]) != 0.0f;
    }
    nz = __any_sync(0xffffffffu, nz);
    if (lane == 0) store[blk] = nz ? 1 : 0;
  }
}

// one warp per block column: count stored blocks -> col_ptr[c + 1]
__global__ void col_count_kernel(const uint8_t* kept, const uint8_t* regrown, const uint8_t* store,
                                 int64_t gr, int64_t gc, int64_t* col_ptr) {
  const int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= gc) return;
  int64_t cnt = 0;
  for (int64_t base = 0; base < gr; base += 32) {
    const int64_t r = base + lane;
    bool s = false;
    if (r < gr) {
      const int64_t idx = r * gc + c;
      s = store ? store[idx] != 0 : ((kept && kept[idx]) || (regrown && regrown[idx]));
    }
    cnt += __popc(__ballot_sync(0xffffffffu, s));
  }
  if (lane == 0) col_ptr[c + 1] = cnt;
}

__global__ void scan_i64_kernel(int64_t* ptr, int64_t lines) {
  __shared__ int64_t warp_sums[32];
  __shared__ int64_t carry;
  if (threadIdx.x == 0) {
    carry = 0;
    ptr[0] = 0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t base = 0; base < lines; base += blockDim.x) {
    const int64_t l = base + threadIdx.x;
    int64_t v = l < lines ? ptr[l + 1] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t n = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += n;
    }
    if (lane == 31) warp_sums[wid] = v;
    __syncthreads();
    if (wid == 0) {
      int64_t w = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t n = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += n;
      }
      warp_sums[lane] = w;
    }
    __syncthreads();
    const int64_t prefix = (wid > 0 ? warp_sums[wid - 1] : 0) + carry;
    if (l < lines) ptr[l + 1] = v + prefix;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = v + prefix;
    __syncthreads();
  }
}

// one warp per block column: kmap[r][c] = col_ptr[c] + rank among stored rows (ascending r)
__global__ void kmap_assign_kernel(const uint8_t* kept, const uint8_t* regrown,
                                   const uint8_t* store, int64_t gr, int64_t gc,
                                   const int64_t* col_ptr, int32_t* kmap) {
  const int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= gc) return;
  int64_t out = col_ptr[c];
  for (int64_t base = 0; base < gr; base += 32) {
    const int64_t r = base + lane;
    bool s = false;
    int64_t idx = 0;
    if (r < gr) {
      idx = r * gc + c;
      s = store ? store[idx] != 0 : ((kept && kept[idx]) || (regrown && regrown[idx]));
    }
    const unsigned bal = __ballot_sync(0xffffffffu, s);
    if (r < gr) kmap[idx] = s ? static_cast<int32_t>(out + __popc(bal & ((1u << lane) - 1u))) : -1;
    out += __popc(bal);
  }
}

// count -> scan -> kmap in ONE single-CTA launch for grids of up to kRepackOneCtaCells cells and
// kRepackOneCta columns (three launches otherwise): the store flags are read once, coalesced,
// into shared memory; a warp per column counts them with ballots, warp 0 scans the counts, and
// the warps assign ranks exactly as kmap_assign_kernel does.
constexpr int kRepackOneCta = 4096;
constexpr int kRepackOneCtaCells = 98304;
__global__ void __launch_bounds__(1024) repack_index_one_cta_kernel(
    const uint8_t* kept, const uint8_t* regrown, const uint8_t* store, int64_t gr, int64_t gc,
    int64_t* col_ptr, int32_t* kmap) {
  __shared__ int64_t cnt[kRepackOneCta + 1];
  extern __shared__ __align__(16) uint8_t sflag[];  // [gr * gc] row-major store flags (nonzero)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int n = static_cast<int>(gr * gc);
  // nonzero = stored; 16 flags per load when the grids allow it (one round trip for cfg3)
  const bool vec = (n % 16) == 0 &&
                   ((reinterpret_cast<uintptr_t>(kept) | reinterpret_cast<uintptr_t>(regrown) |
                     reinterpret_cast<uintptr_t>(store)) & 15u) == 0;
  if (vec) {
    const uint4 z = make_uint4(0, 0, 0, 0);
    for (int i = threadIdx.x; i < n / 16; i += blockDim.x) {
      uint4 v;
      if (store) {
        v = reinterpret_cast<const uint4*>(store)[i];
      } else {
        const uint4 a = kept ? reinterpret_cast<const uint4*>(kept)[i] : z;
        const uint4 b = regrown ? reinterpret_cast<const uint4*>(regrown)[i] : z;
        v = make_uint4(a.x | b.x, a.y | b.y, a.z | b.z, a.w | b.w);
      }
      reinterpret_cast<uint4*>(sflag)[i] = v;
    }
  } else {
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      sflag[i] = store ? (store[i] != 0) : ((kept && kept[i]) || (regrown && regrown[i]));
  }
  __syncthreads();
  for (int64_t c = wid; c < gc; c += nw) {
    int64_t cn = 0;
    for (int64_t base = 0; base < gr; base += 32) {
      const int64_t r = base + lane;
      cn += __popc(__ballot_sync(0xffffffffu, r < gr && sflag[r * gc + c]));
    }
    if (lane == 0) cnt[c + 1] = cn;
  }
  if (threadIdx.x == 0) cnt[0] = 0;
  __syncthreads();
  if (wid == 0) {  // inclusive scan of cnt[1..gc]: 32 contiguous chunks, one per lane
    const int64_t per = (gc + 31) / 32;
    const int64_t lo = 1 + lane * per, hi = min(gc + 1, lo + per);
    int64_t sum = 0;
    for (int64_t i = lo; i < hi; ++i) sum += cnt[i];
    int64_t pre = sum;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t v = __shfl_up_sync(0xffffffffu, pre, o);
      if (lane >= o) pre += v;
    }
    int64_t run = pre - sum;
    for (int64_t i = lo; i < hi; ++i) {
      run += cnt[i];
      cnt[i] = run;
    }
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i <= gc; i += blockDim.x) col_ptr[i] = cnt[i];
  for (int64_t c = wid; c < gc; c += nw) {
    int64_t out = cnt[c];
    for (int64_t base = 0; base < gr; base += 32) {
      const int64_t r = base + lane;
      const bool sd = r < gr && sflag[r * gc + c];
      const unsigned bal = __ballot_sync(0xffffffffu, sd);
      if (r < gr)
        kmap[r * gc + c] = sd ? static_cast<int32_t>(out + __popc(bal & ((1u << lane) - 1u))) : -1;
      out += __popc(bal);
    }
  }
}

__global__ void repack_rows_kernel(const int32_t* kmap, int64_t gr, int64_t gc, int32_t* row_idx) {
  const int64_t n = gr * gc;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t k = kmap[i];
    if (k >= 0) row_idx[k] = static_cast<int32_t>(i / gc);
  }
}

// masked = w * float(survive) (pruner.py:185; multiply keeps -0.0 and NaN); stored blocks are
// copied into values[k] (bcsc.py:210). mode: 0 = copy verbatim (no mask), 1 = survive = kept,
// 2 = survive = kept | regrown.
template <typename T, typename V>
__global__ void apply_mask_gather_kernel(const T* __restrict__ x, int64_t rows, int64_t cols,
                                         int b, int64_t gc, const uint8_t* __restrict__ kept,
                                         const uint8_t* __restrict__ regrown, int mode,
                                         const int32_t* __restrict__ kmap, T* masked, V* values) {
  const int64_t n = rows * cols;
  const int64_t bb = static_cast<int64_t>(b) * b;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / cols, col = i - row * cols;
    const int64_t r = row / b, c = col / b;
    const int64_t cell = r * gc + c;
    const T v = x[i];
    float m = to_f32<T>(v);
    if (mode != 0) {
      const bool surv = kept[cell] != 0 || (mode == 2 && regrown[cell] != 0);
      m = __fmul_rn(m, surv ? 1.0f : 0.0f);
    }
    if (masked) masked[i] = mode != 0 ? from_f32<T>(m) : v;
    const int32_t k = kmap[cell];
    if (k >= 0) {
      const int64_t off = k * bb + (row - r * b) * b + (col - c * b);
      const float val = mode != 0 ? m : to_f32<T>(v);
      if constexpr (sizeof(T) == sizeof(V))
        values[off] = mode == 0 ? *reinterpret_cast<const V*>(&v) : from_f32<V>(val);
      else
        values[off] = from_f32<V>(val);
    }
  }
}

// Vectorised form for float32 masters with cols % 4 == 0 and b % 4 == 0: four
// consecutive columns share a block, so one mask / kmap lookup and one 16-byte
// load serve four elements. Same arithmetic as apply_mask_gather_kernel.
template <typename V>
__global__ void __launch_bounds__(256) apply_mask_gather_vec4_kernel(
    const float4* __restrict__ x, int64_t rows, int64_t cols4, int b, int64_t gc,
    const uint8_t* __restrict__ kept, const uint8_t* __restrict__ regrown, int mode,
    const int32_t* __restrict__ kmap, float4* masked, V* values) {
  const int64_t n4 = rows * cols4;
  const int64_t bb = static_cast<int64_t>(b) * b;
  // 4 independent 16-byte loads in flight per thread; 32-bit index arithmetic when it fits
  constexpr int U = 4;
  const bool small = n4 < (int64_t(1) << 31);
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x * U + threadIdx.x; i0 < n4;
       i0 += (int64_t)gridDim.x * blockDim.x * U) {
    float4 vs[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i0 + u * (int64_t)blockDim.x < n4) vs[u] = __ldg(&x[i0 + u * (int64_t)blockDim.x]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
    const int64_t i = i0 + u * (int64_t)blockDim.x;
    if (i >= n4) break;
    int64_t row, col;
    if (small) {
      const uint32_t q = static_cast<uint32_t>(i) / static_cast<uint32_t>(cols4);
      row = q;
      col = (static_cast<uint32_t>(i) - q * static_cast<uint32_t>(cols4)) * 4;
    } else {
      row = i / cols4;
      col = (i - row * cols4) * 4;
    }
    const int64_t r = static_cast<uint32_t>(row) / static_cast<uint32_t>(b);
    const int64_t c = static_cast<uint32_t>(col) / static_cast<uint32_t>(b);
    const int64_t cell = r * gc + c;
    const float4 v = vs[u];
    float4 m = v;
    if (mode != 0) {
      const bool surv = kept[cell] != 0 || (mode == 2 && regrown[cell] != 0);
      const float s = surv ? 1.0f : 0.0f;
      m = make_float4(__fmul_rn(v.x, s), __fmul_rn(v.y, s), __fmul_rn(v.z, s), __fmul_rn(v.w, s));
    }
    if (masked) masked[i] = m;
    const int32_t k = __ldg(&kmap[cell]);
    if (k >= 0) {
      const int64_t off = k * bb + (row - r * b) * b + (col - c * b);
      if constexpr (sizeof(V) == 4) {
        *reinterpret_cast<float4*>(values + off) = mode == 0 ? v : m;
      } else {
        const float4 s = mode == 0 ? v : m;
        __nv_bfloat162 lo = __floats2bfloat162_rn(s.x, s.y), hi = __floats2bfloat162_rn(s.z, s.w);
        uint2 pk;
        pk.x = *reinterpret_cast<uint32_t*>(&lo);
        pk.y = *reinterpret_cast<uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(values + off) = pk;
      }
    }
    }
  }
}

// ------------------------------------------------------------------ optimizer glue
__global__ void sgd_kernel(float* w, const float* g, int64_t n, float lr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    w[i] = __fsub_rn(w[i], __fmul_rn(lr, g[i]));
}

template <typename T>
__global__ void sumsq_partial_kernel(const T* x, int64_t n, double* partial) {
  __shared__ double ws[32];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = (double)to_f32<T>(x[i]);
    acc = fma(v, v, acc);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? ws[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) partial[blockIdx.x] = v;
  }
}
__global__ void sumsq_final_kernel(const double* partial, int n, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += partial[i];
    out[0] += s;
  }
}

static int topk_smem_launch(const double* n0, uint8_t* k0, const double* n1, uint8_t* k1,
                            int64_t gr, int64_t gc, int64_t k, cudaStream_t st,
                            uint8_t* regrown = nullptr, int64_t* counts = nullptr) {
  static bool configured[64] = {};
  const int smem = kTopkSmemMax * 8;
  if (int rc = configure_smem(topk_smem_kernel, smem, configured, "topk smem attribute")) return rc;
  const int n = static_cast<int>(gr * gc);
  if (!(n1 && counts)) {
    topk_smem_kernel<<<n1 ? 2 : 1, 1024, n * 8, st>>>(n0, k0, n1, k1, gr, gc, k, nullptr, nullptr);
    return check_launch("topk_smem");
  }
  // both grids + the set difference: one cluster of two CTAs
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2);
  cfg.blockDim = dim3(1024);
  cfg.dynamicSmemBytes = static_cast<size_t>(n) * 8;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, topk_smem_kernel, n0, k0, n1, k1, gr, gc, k, regrown,
                     reinterpret_cast<unsigned long long*>(counts));
  return check_launch("topk_smem (fused difference)");
}

static int grid_for(int64_t n, int threads, int per_sm = 16) {
  int64_t g = cdiv(n, threads);
  const int64_t cap = (int64_t)num_sms() * per_sm;
  if (g > cap) g = cap;
  return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace blast

using namespace blast;

namespace blast {
template <typename T>
static void norms_launch(const void* x, const void* x2, int64_t rows, int64_t cols, int block,
                         double* norms, double* norms2, cudaStream_t st) {
  const int64_t gr = cdiv(rows, block), gc = cdiv(cols, block);
  constexpr int vw = 16 / sizeof(T);
  const bool vec = block % vw == 0 && rows % block == 0 && cols % block == 0 && aligned16(x) &&
                   (!x2 || aligned16(x2)) && (cols * static_cast<int64_t>(sizeof(T))) % 16 == 0;
  dim3 grid(grid_for(gr * gc * 32, 256, 32), x2 ? 2 : 1);
  auto* a = static_cast<const T*>(x);
  auto* a2 = static_cast<const T*>(x2);
  if (vec)
    block_norms_kernel<T, true><<<grid, 256, 0, st>>>(a, a2, rows, cols, block, gr, gc, norms, norms2);
  else
    block_norms_kernel<T, false><<<grid, 256, 0, st>>>(a, a2, rows, cols, block, gr, gc, norms, norms2);
}

// norms of x (dtype) and, when given, of x2 (dtype2): one launch covers both when they share a
// dtype (blockIdx.y picks the matrix), else one launch each; every element is squared in fp64.
static int norms_any(const void* x, int dtype, const void* x2, int dtype2, int64_t rows,
                     int64_t cols, int block, double* norms, double* norms2, cudaStream_t st) {
  if (rows < 1 || cols < 1 || block < 1) {
    set_error("block_norms: invalid shape %lld x %lld block %d", (long long)rows, (long long)cols,
              block);
    return BLAST_EINVAL;
  }
  for (int d : {dtype, x2 ? dtype2 : dtype})
    if (d != BLAST_F32 && d != BLAST_BF16 && d != BLAST_F64) {
      set_error("block_norms: unsupported dtype %d", d);
      return BLAST_EINVAL;
    }
  auto one = [&](const void* a, const void* a2, int d, double* o, double* o2) {
    if (d == BLAST_BF16) norms_launch<__nv_bfloat16>(a, a2, rows, cols, block, o, o2, st);
    else if (d == BLAST_F64) norms_launch<double>(a, a2, rows, cols, block, o, o2, st);
    else norms_launch<float>(a, a2, rows, cols, block, o, o2, st);
  };
  if (!x2 || dtype2 == dtype) {
    one(x, x2, dtype, norms, norms2);
  } else {
    one(x, nullptr, dtype, norms, nullptr);
    one(x2, nullptr, dtype2, norms2, nullptr);
  }
  return check_launch("block_norms");
}
}  // namespace blast

extern "C" int blast_block_norms(const void* x, const void* x2, int64_t rows, int64_t cols,
                                 int32_t block, int dtype, double* norms, double* norms2,
                                 void* stream) {
  return norms_any(x, dtype, x2, dtype, rows, cols, block, norms, norms2,
                   static_cast<cudaStream_t>(stream));
}

extern "C" int blast_topk_mask(const double* norms, int64_t grid_rows, int64_t grid_cols,
                               int64_t k, uint8_t* keep, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t n = grid_rows * grid_cols;
  if (n <= 0) return BLAST_OK;
  if (n > (int64_t)UINT32_MAX) {
    set_error("topk: grid too large");
    return BLAST_EINVAL;
  }
  if (k <= 0 || k >= n) {
    fill_u8_kernel<<<grid_for(n, 256), 256, 0, st>>>(keep, n, k <= 0 ? 0 : 1);
    return check_launch("topk fill");
  }
  if (n <= kTopkSmemMax) return topk_smem_launch(norms, keep, nullptr, nullptr, grid_rows,
                                                 grid_cols, k, st);
  Scratch s;
  if (!s.alloc(sizeof(TopkState), st)) return cuda_status(cudaGetLastError(), "topk scratch");
  cudaMemsetAsync(s.ptr, 0, sizeof(TopkState), st);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, topk_kernel, 1024, 0);
  int64_t want = cdiv(n, 4096);
  int64_t cap = (int64_t)num_sms() * (per_sm > 0 ? per_sm : 1);
  int grid = static_cast<int>(want < 1 ? 1 : (want > cap ? cap : want));
  TopkState* state = s.as<TopkState>();
  void* args[] = {const_cast<double**>(&norms), &grid_rows, &grid_cols, &k, &keep, &state};
  cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(topk_kernel), dim3(grid),
                                              dim3(1024), args, 0, st);
  return cuda_status(e, "topk launch");
}

extern "C" int blast_topk_mask2(const double* norms_a, const double* norms_b, int64_t grid_rows,
                                int64_t grid_cols, int64_t k, uint8_t* keep_a, uint8_t* keep_b,
                                void* stream) {
  const int64_t n = grid_rows * grid_cols;
  if (n > 0 && k > 0 && k < n && n <= kTopkSmemMax)
    return topk_smem_launch(norms_a, keep_a, norms_b, keep_b, grid_rows, grid_cols, k,
                            static_cast<cudaStream_t>(stream));
  const int r = blast_topk_mask(norms_a, grid_rows, grid_cols, k, keep_a, stream);
  if (r) return r;
  return blast_topk_mask(norms_b, grid_rows, grid_cols, k, keep_b, stream);
}

extern "C" int blast_mask_difference(const uint8_t* kept, const uint8_t* grad_sel, int64_t n,
                                     uint8_t* regrown, int64_t* counts, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaMemsetAsync(counts, 0, 2 * sizeof(int64_t), st);
  if (n <= 0) return check_launch("mask_difference");
  mask_difference_kernel<<<grid_for(n, 256, 4), 256, 0, st>>>(
      kept, grad_sel, n, regrown, reinterpret_cast<unsigned long long*>(counts));
  return check_launch("mask_difference");
}

extern "C" int blast_generate_masks(const void* w, int dtype_w, const void* g, int dtype_g,
                                    int64_t rows, int64_t cols, int32_t block, int64_t k,
                                    double* norms_w, double* norms_g, uint8_t* kept,
                                    uint8_t* regrown, int64_t* counts, int64_t* counts_host,
                                    void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int r = norms_any(w, dtype_w, g, dtype_g, rows, cols, block, norms_w, norms_g, st);
  if (r) return r;
  const int64_t gr = cdiv(rows, block), gc = cdiv(cols, block);
  // grad_sel goes into `regrown` and is turned into grad_sel & ~kept in place; for grids that
  // fit one CTA's shared memory the difference and the counts run inside the top-k launch
  const int64_t n = gr * gc;
  if (n > 0 && k > 0 && k < n && n <= kTopkSmemMax) {
    r = topk_smem_launch(norms_w, kept, norms_g, regrown, gr, gc, k, st, regrown, counts);
  } else {
    r = blast_topk_mask2(norms_w, norms_g, gr, gc, k, kept, regrown, stream);
    if (!r) r = blast_mask_difference(kept, regrown, n, regrown, counts, stream);
  }
  if (r) return r;
  if (counts_host) {
    cudaError_t e = cudaMemcpyAsync(counts_host, counts, 2 * sizeof(int64_t),
                                    cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    return cuda_status(e, "generate_masks counts");
  }
  return BLAST_OK;
}


extern "C" int blast_repack_index(const uint8_t* kept, const uint8_t* regrown, const void* dense,
                                  int64_t rows, int64_t cols, int32_t block, int dtype,
                                  int64_t* col_ptr, int32_t* kmap, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (rows < 1 || cols < 1 || block < 1) {
    set_error("matrix dimensions must be positive");
    return BLAST_EINVAL;
  }
  const int64_t gr = cdiv(rows, block), gc = cdiv(cols, block);
  Scratch s;
  const uint8_t* store = nullptr;
  if (!kept && !regrown) {
    if (!s.alloc(gr * gc, st)) return cuda_status(cudaGetLastError(), "repack scratch");
    if (dtype == BLAST_BF16)
      store_from_dense_kernel<__nv_bfloat16><<<grid_for(gr * gc * 32, 256, 32), 256, 0, st>>>(
          static_cast<const __nv_bfloat16*>(dense), rows, cols, block, gr, gc, s.as<uint8_t>());
    else
      store_from_dense_kernel<float><<<grid_for(gr * gc * 32, 256, 32), 256, 0, st>>>(
          static_cast<const float*>(dense), rows, cols, block, gr, gc, s.as<uint8_t>());
    store = s.as<uint8_t>();
  }
  const int blocks = static_cast<int>(cdiv(gc * 32, 256));
  if (gc <= kRepackOneCta && gr * gc <= kRepackOneCtaCells) {
    static bool configured[64] = {};
    if (configure_smem(repack_index_one_cta_kernel, kRepackOneCtaCells, configured,
                       "repack smem attribute") == 0) {
      repack_index_one_cta_kernel<<<1, 1024, static_cast<size_t>(gr * gc), st>>>(
          kept, regrown, store, gr, gc, col_ptr, kmap);
      return check_launch("repack_index");
    }
    cudaGetLastError();
  }
  col_count_kernel<<<blocks, 256, 0, st>>>(kept, regrown, store, gr, gc, col_ptr);
  scan_i64_kernel<<<1, 1024, 0, st>>>(col_ptr, gc);
  kmap_assign_kernel<<<blocks, 256, 0, st>>>(kept, regrown, store, gr, gc, col_ptr, kmap);
  return check_launch("repack_index");
}

extern "C" int blast_repack_rows(const int32_t* kmap, const int64_t* col_ptr, int64_t grid_rows,
                                 int64_t grid_cols, int32_t* row_idx, void* stream) {
  (void)col_ptr;
  const int64_t n = grid_rows * grid_cols;
  if (n <= 0) return BLAST_OK;
  repack_rows_kernel<<<grid_for(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      kmap, grid_rows, grid_cols, row_idx);
  return check_launch("repack_rows");
}

extern "C" int blast_apply_mask_gather(const void* dense, int64_t rows, int64_t cols,
                                       int32_t block, int dtype, const uint8_t* kept,
                                       const uint8_t* regrown, int zero_regrown,
                                       const int32_t* kmap, void* masked_out, void* values,
                                       int values_dtype, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t n = rows * cols;
  if (n <= 0) return BLAST_OK;
  const int64_t gc = cdiv(cols, block);
  const int mode = !kept ? 0 : (zero_regrown ? 1 : 2);
  if (mode == 2 && !regrown) {
    set_error("apply_mask: regrown grid required");
    return BLAST_EINVAL;
  }
  const int grid = grid_for(n, 256, 32);
  const bool vec = dtype == BLAST_F32 && cols % 4 == 0 && block % 4 == 0 && aligned16(dense) &&
                   (!masked_out || aligned16(masked_out)) && aligned16(values);
  if (vec) {
    const int g4 = grid_for(cdiv(n / 4, 4), 256, 32);
    if (values_dtype == BLAST_F32)
      apply_mask_gather_vec4_kernel<float><<<g4, 256, 0, st>>>(
          static_cast<const float4*>(dense), rows, cols / 4, block, gc, kept, regrown, mode, kmap,
          static_cast<float4*>(masked_out), static_cast<float*>(values));
    else
      apply_mask_gather_vec4_kernel<__nv_bfloat16><<<g4, 256, 0, st>>>(
          static_cast<const float4*>(dense), rows, cols / 4, block, gc, kept, regrown, mode, kmap,
          static_cast<float4*>(masked_out), static_cast<__nv_bfloat16*>(values));
    return check_launch("apply_mask_gather_vec4");
  }
#define BLAST_GATHER(T, V)                                                                    \
  apply_mask_gather_kernel<T, V><<<grid, 256, 0, st>>>(                                       \
      static_cast<const T*>(dense), rows, cols, block, gc, kept, regrown, mode, kmap,         \
      static_cast<T*>(masked_out), static_cast<V*>(values))
  if (dtype == BLAST_F32 && values_dtype == BLAST_F32) BLAST_GATHER(float, float);
  else if (dtype == BLAST_F32 && values_dtype == BLAST_BF16) BLAST_GATHER(float, __nv_bfloat16);
  else if (dtype == BLAST_BF16 && values_dtype == BLAST_BF16)
    BLAST_GATHER(__nv_bfloat16, __nv_bfloat16);
  else BLAST_GATHER(__nv_bfloat16, float);
#undef BLAST_GATHER
  return check_launch("apply_mask_gather");
}

extern "C" int blast_sgd_step(float* w, const float* g, int64_t n, float lr, void* stream) {
  if (n <= 0) return BLAST_OK;
  sgd_kernel<<<grid_for(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(w, g, n, lr);
  return check_launch("sgd_step");
}

extern "C" int blast_sumsq_f64(const void* x, int64_t n, int dtype, double* out, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n <= 0) return BLAST_OK;
  const int grid = grid_for(n, 256, 4);
  Scratch s;
  if (!s.alloc(sizeof(double) * grid, st)) return cuda_status(cudaGetLastError(), "sumsq");
  if (dtype == BLAST_BF16)
    sumsq_partial_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(x), n, s.as<double>());
  else
    sumsq_partial_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(x), n,
                                                      s.as<double>());
  sumsq_final_kernel<<<1, 32, 0, st>>>(s.as<double>(), grid, out);
  return check_launch("sumsq_f64");
}
