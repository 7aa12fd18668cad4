// Microbenchmark: issue rate of tcgen05.mma (SS, bf16) from resident shared memory,
// for M=128 (1 CTA) with N = 64/128/256, to measure the operand-read ceiling that
// bounds the block-sparse engine. Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -I../paper_2507_03117_b200/csrc tools/mma_rate.cu -o mma_rate
#include <cstdio>
#include "../paper_2507_03117_b200/csrc/ptx.cuh"

using namespace blast;

template <int N>
__global__ void __launch_bounds__(128, 1) mma_loop(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32;
  if (warp == 0) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  // A: 128 x 64 bf16 K-major SW128 (16 KB); B: 64 K x N MN-major SW128 (N/64 atoms of 8 KB)
  const uint32_t a0 = smem_u32(smem), b0 = a0 + 16384;
  const uint32_t idesc = make_idesc(128, N, 1u, 0u, 1u);
  if (warp == 1) {
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint64_t ad = make_sdesc(a0 + ks * 32, 16, 1024, 2);
          const uint64_t bd = make_sdesc(b0 + ks * 16 * 128, 64 * 128, 1024, 2);
          mma_f16(tbase, ad, bd, idesc, (i | ks) ? 1u : 0u);
        }
        if ((i & 63) == 63) {
          mma_commit(&bar);
        }
      }
      __syncwarp();
      if ((i & 63) == 63) mbar_wait(&bar, (i >> 6) & 1);
    }
    const long long t1 = clock64();
    if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tbase, 512); }
}

template <int N>
void run(int iters) {
  auto k = mma_loop<N>;
  const int smem = 16384 + N * 128 + 2048;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  k<<<148, 128, smem>>>(iters, d);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double per_mma = avg / (iters * 4.0);
  const double ideal = 128.0 * N / 256.0;
  printf("M=128 N=%3d K=16: %.1f cycles/MMA (ideal %.0f) -> %.0f%% of tensor peak, operand bytes/cycle %.0f\n",
         N, per_mma, ideal, 100.0 * ideal / per_mma, (4096.0 + N * 32.0) / per_mma);
  cudaFree(d);
}

int main() {
  run<64>(4000);
  run<128>(4000);
  run<256>(2000);
  const cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
