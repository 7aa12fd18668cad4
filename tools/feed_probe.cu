// Producer-feed microbenchmark: how fast can one SM stream the engine's step
// pattern (one 128 x 64 bf16 activation panel + one 64 x 64 weight block per step)?
//   P producer warps (producer p owns steps n % P == p; stage = n % S),
//   consumer = release immediately (MMA=0) or 4 x tcgen05.mma M=128 N=64 K=16 SS (MMA=1)
//   committed to the stage's empty barrier (the engine's MMA loop without epilogue).
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a
//        -Ipaper_2507_03117_b200/csrc tools/feed_probe.cu -o tools/feed_probe -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include "ptx.cuh"

using namespace blast;

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

constexpr int M = 8192, D = 4096, LINES = 224, STEPS = 12, NBLK = LINES * STEPS;
constexpr int PANEL = 128 * 128, WBLK = 8192;

template <int P, int S, int MMA, int ASC = 0, int GU = 0, int BULK = 0, int HYB = 0>
__global__ void __launch_bounds__(256, 1) feed_kernel(const __grid_constant__ CUtensorMap mx,
                                                      const __grid_constant__ CUtensorMap mw, const __grid_constant__ CUtensorMap mw2, int n_items,
                                                      const uint8_t* xg, const uint8_t* wg) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[16], empty[16];
  __shared__ uint32_t tslot;
  constexpr int STAGE = PANEL + (GU ? 2 : 1) * WBLK;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) { mbar_init(&full[i], HYB ? 33 : 1); mbar_init(&empty[i], 1); }
    fence_mbar_init();
  }
  if (MMA && warp == 7) { tmem_alloc(&tslot, 128); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  constexpr int n_tiles = M / 128;
  if (warp < P) {
    uint32_t n = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int t = item / LINES, line = item - (item / LINES) * LINES;
      for (int s = 0; s < STEPS; ++s, ++n) {
        if ((n % P) != static_cast<uint32_t>(warp)) continue;
        const uint32_t stage = n % S, phase = (n / S) & 1;
        const int r = ASC == 3 ? ((line * 37 + s * 19) % 224)
                      : ASC ? (s * 5 + (line & 3)) : ((line * 7 + s * 5) & 63);
        const int k = line * STEPS + s;
        mbar_wait(&empty[stage], phase ^ 1);
        if (elect_one()) {
          mbar_expect_tx(&full[stage], HYB ? PANEL : PANEL + WBLK);
          uint8_t* dst = smem + stage * STAGE;
          if (HYB) {
            tma_load_2d(dst, &mx, &full[stage], r * 64, (t & (n_tiles - 1)) * 128);
          } else if (BULK) {
            // block-major activation layout: panel (t, r) is one contiguous 16 KB run
            bulk_g2s(dst, xg + (static_cast<size_t>(r) * n_tiles + (t & (n_tiles - 1))) * PANEL, PANEL, &full[stage]);
            // (ASC == 3: the same index formula over a 224 x 64-tile block-major matrix)
            bulk_g2s(dst + PANEL, wg + static_cast<size_t>(k) * WBLK, WBLK, &full[stage]);
          } else {
            tma_load_2d(dst, &mx, &full[stage], r * 64, (t & (n_tiles - 1)) * 128);
            tma_load_2d(dst + PANEL + (GU ? (s & 1) * WBLK : 0), (ASC == 2 && (s & 1)) ? &mw2 : &mw, &full[stage], 0, k * 64);
          }
        }
        __syncwarp();
      }
    }
  } else if (HYB && warp == 5) {
    // W block via cp.async (16 B per lane x 16 per step), swizzled like TMA SW128
    const int lane = threadIdx.x & 31;
    uint32_t n = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int line = item - (item / LINES) * LINES;
      for (int s = 0; s < STEPS; ++s, ++n) {
        const uint32_t stage = n % S, phase = (n / S) & 1;
        const int k = line * STEPS + s;
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* dst = smem + stage * (PANEL + WBLK) + PANEL;
        const uint8_t* src = wg + static_cast<size_t>(k) * WBLK;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int chunk = i * 32 + lane;          // 16-B chunk of the 8 KB block
          const int row = chunk >> 3, c = chunk & 7;
          const uint32_t d = smem_u32(dst + row * 128 + ((c ^ (row & 7)) * 16));
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + chunk * 16) : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[stage])) : "memory");
      }
    }
  } else if (warp == 4) {
    const uint32_t tbase = MMA ? tslot : 0;
    const uint32_t idesc = make_idesc(128, 64, 1u, 0u, 0u);
    const uint32_t s0 = smem_u32(smem);
    const uint64_t ad0 = make_sdesc(s0, 16, 1024, 2), bd0 = make_sdesc(s0 + PANEL, 16, 1024, 2);
    uint32_t stage = 0, phase = 0, n = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      for (int s = 0; s < STEPS; ++s, ++n) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          if (MMA) {
            const uint32_t off = (stage * STAGE) >> 4;
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
              mma_f16(tbase + (GU ? (s & 1) * 64 : (n & 1) * 64), ad0 + off + ks * 2,
                      bd0 + off + ks * 2 + (GU ? (s & 1) * (WBLK >> 4) : 0), idesc, (s | ks) ? 1u : 0u);
            mma_commit(&empty[stage]);
          } else {
            mbar_arrive(&empty[stage]);
          }
        }
        __syncwarp();
        if (++stage == S) { stage = 0; phase ^= 1; }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (MMA && warp == 7) { tc_fence_after(); tmem_dealloc(tslot, 128); }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

static CUtensorMap map2d(void* base, uint64_t inner, uint64_t outer, uint32_t box_in, uint32_t box_out) {
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {box_in, box_out};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); exit(1); }
  return m;
}

template <int P, int S, int MMA, int ASC = 0, int GU = 0, int BULK = 0, int HYB = 0>
void run(const CUtensorMap& mx, const CUtensorMap& mw, const CUtensorMap& mw2, cudaEvent_t e0, cudaEvent_t e1,
         const void* xg = nullptr, const void* wg = nullptr, int ctas = 148) {
  auto k = feed_kernel<P, S, MMA, ASC, GU, BULK, HYB>;
  constexpr int STAGE = PANEL + (GU ? 2 : 1) * WBLK;
  const int smem = S * STAGE + 2048;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int n_items = (M / 128) * LINES;
  k<<<ctas, 256, smem>>>(mx, mw, mw2, n_items, (const uint8_t*)xg, (const uint8_t*)wg);
  CK(cudaEventRecord(e0));
  k<<<ctas, 256, smem>>>(mx, mw, mw2, n_items, (const uint8_t*)xg, (const uint8_t*)wg);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  CK(cudaGetLastError());
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double bytes = double(n_items) * STEPS * (PANEL + WBLK);
  const double steps_per_sm = double(n_items) * STEPS / ctas;
  printf("hyb=%d ctas=%d bulk=%d gu=%d asc=%d producers=%d stages=%d consumer=%s: %.3f ms  %.0f GB/s  %.0f cyc/step/SM  (MMA-only floor 280)\n", HYB, ctas, BULK, GU, ASC, P, S,
         MMA ? "mma" : "release", ms, bytes / (ms * 1e6), ms * 1e-3 * 1.965e9 / steps_per_sm);
}

int main() {
  void *x, *w;
  CK(cudaMalloc(&x, size_t(M) * D * 2));
  CK(cudaMalloc(&w, size_t(NBLK) * 64 * 64 * 2));
  CK(cudaMemset(x, 0, size_t(M) * D * 2));
  CK(cudaMemset(w, 0, size_t(NBLK) * 64 * 64 * 2));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const CUtensorMap mx = map2d(x, D, M, 64, 128);
  const CUtensorMap mw = map2d(w, 64, size_t(NBLK) * 64, 64, 64);
  const CUtensorMap mw2 = map2d(w, 64, size_t(NBLK) * 64, 64, 64);
  run<1, 8, 0>(mx, mw, mw2, e0, e1);
  run<1, 8, 0, 0, 0, 0, 1>(mx, mw, mw2, e0, e1, x, w);
  run<1, 8, 1>(mx, mw, mw2, e0, e1);
  run<1, 8, 1, 0, 0, 0, 1>(mx, mw, mw2, e0, e1, x, w);
  return 0;
}
