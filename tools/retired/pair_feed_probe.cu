// Does the CTA-pair TMA form (cp.async.bulk.tensor ... .cta_group::2, completion counted on
// the leader CTA's mbarrier) feed a CTA pair as fast as per-CTA TMA with local barriers?
// Both variants stream one 128 x 64 bf16 panel per CTA per step through an 8-stage ring, a
// consumer releasing each stage at once (no MMA).
//   local: each CTA: its own full/empty barriers
//   pair : both CTAs' loads complete on the leader's full barrier (expect 2x bytes); the
//          leader's consumer releases the stage in both CTAs (remote arrive for the peer)
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a
//        -Ipaper_2507_03117_b200/csrc tools/pair_feed_probe.cu -o tools/pair_feed_probe -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include "ptx.cuh"

using namespace blast;

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

constexpr int M = 8192, D = 4096, PANEL = 128 * 128, S = 8;

template <int PAIR>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
pair_feed_kernel(const __grid_constant__ CUtensorMap mx, int steps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[S], empty[S];
  const int warp = threadIdx.x / 32;
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
  }
  cluster_sync();
  const int pair = blockIdx.x / 2;
  const long long t0 = clock64();
  if (warp == 0) {
    const uint32_t full0 = mapa_shared(&full[0], 0);
    for (int n = 0; n < steps; ++n) {
      const int stage = n % S;
      const uint32_t phase = (n / S) & 1;
      mbar_wait(&empty[stage], phase ^ 1);
      if (elect_one()) {
        const int r = (n * 5 + pair * 7) & 63, t = (n / 64 + pair) & 63;
        uint8_t* dst = smem + stage * PANEL;
        if (PAIR) {
          if (rank == 0) mbar_expect_tx(&full[stage], 2 * PANEL);
          tma_load_2d_pair(dst, &mx, full0 + stage * 8, r * 64, t * 128, 0ull);
        } else {
          mbar_expect_tx(&full[stage], PANEL);
          tma_load_2d(dst, &mx, &full[stage], r * 64, t * 128);
        }
      }
      __syncwarp();
    }
  } else if (warp == 1 && (!PAIR || rank == 0)) {
    for (int n = 0; n < steps; ++n) {
      const int stage = n % S;
      mbar_wait(&full[stage], (n / S) & 1);
      if (elect_one()) {
        mbar_arrive(&empty[stage]);
        if (PAIR) mbar_arrive_cluster(&empty[stage], 1);
      }
      __syncwarp();
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  cluster_sync();
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

template <int PAIR>
void run(const CUtensorMap& mx) {
  auto k = pair_feed_kernel<PAIR>;
  const int smem = S * PANEL + 2048;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  unsigned long long* d;
  CK(cudaMalloc(&d, 148 * 8));
  const int steps = 4000;
  k<<<148, 128, smem>>>(mx, steps, d);
  CK(cudaDeviceSynchronize());
  k<<<148, 128, smem>>>(mx, steps, d);
  CK(cudaDeviceSynchronize());
  unsigned long long h[148];
  CK(cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost));
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("%s: %.0f cycles per 16 KB step per CTA (%.1f B/cycle/SM)\n", PAIR ? "pair " : "local",
         avg / steps, PANEL / (avg / steps));
  CK(cudaFree(d));
}

int main() {
  void* x;
  CK(cudaMalloc(&x, size_t(M) * D * 2));
  CK(cudaMemset(x, 0, size_t(M) * D * 2));
  CUtensorMap m;
  cuuint64_t dims[2] = {D, M};
  cuuint64_t strides[1] = {D * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  if (enc()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  run<0>(m);
  run<1>(m);
  return 0;
}
