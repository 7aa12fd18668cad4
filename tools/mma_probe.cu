// Microbenchmarks that decide the engine-v3 design (round 1, session 2):
//   P1 SS-MMA M=128 issue rate vs N and vs the number of rotating accumulators
//   P2 TS-MMA (A operand in TMEM) issue rate
//   P3 TS-MMA correctness: A written to TMEM with tcgen05.st (row per lane, bf16 pairs per
//      32-bit column) must give the same D as the same A in shared memory (SS)
//   P4 SS-MMA N=64 rate while other warps write shared memory (bulk copies from L2)
//   P5 chip-wide L2->SM bandwidth with 1-D bulk copies (cp.async.bulk) into a smem ring
//   P6 chip-wide LDG -> tcgen05.st (registers -> TMEM) panel feed rate
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Ipaper_2507_03117_b200/csrc
//        tools/mma_probe.cu -o tools/mma_probe -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>
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

__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                       uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, "
      "%29, %30, %31, %32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ----------------------------------------------------------------------------- P1/P2/P4
// MODE 0: SS, MODE 1: TS. NACC accumulators rotate per 4-MMA block. STREAM: warps 4..7 keep
// bulk-copying 16 KB chunks from global into a separate smem ring (P4).
template <int N, int NACC, int MODE, bool STREAM, int M = 128, int BMN = 0>
__global__ void __launch_bounds__(256, 1) rate_kernel(int iters, const uint8_t* gsrc, size_t gbytes,
                                                      unsigned long long* out, unsigned long long* out2) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t sbar[4];
  __shared__ volatile int done;
  const int warp = threadIdx.x / 32;
  if (warp == 0) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    for (int i = 0; i < 4; ++i) mbar_init(&sbar[i], 1);
    done = 0;
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  const uint32_t a0 = smem_u32(smem), b0 = a0 + 16384;
  const uint32_t idesc = make_idesc(M, N, 1u, 0u, BMN ? 1u : 0u);  // A K-major, B K- or MN-major
  uint8_t* ring = smem + 16384 + 32768;
  if (warp == 1) {
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (elect_one()) {
        const uint32_t d = tbase + 256 * (MODE == 1) + (NACC > 1 ? (i % NACC) * N : 0);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint64_t bd = BMN ? make_sdesc(b0 + ks * 16 * 128, N * 128, 1024, 2)
                                  : make_sdesc(b0 + ks * 32, 16, 1024, 2);
          if (MODE == 0) {
            const uint64_t ad = make_sdesc(a0 + ks * 32, 16, 1024, 2);
            mma_f16(d, ad, bd, idesc, (i | ks) ? 1u : 0u);
          } else {
            mma_ts(d, tbase + ks * 8, bd, idesc, (i | ks) ? 1u : 0u);
          }
        }
        if ((i & 63) == 63) mma_commit(&bar);
      }
      __syncwarp();
      if ((i & 63) == 63) mbar_wait(&bar, (i >> 6) & 1);
    }
    const long long t1 = clock64();
    if (threadIdx.x == 32) { out[blockIdx.x] = t1 - t0; done = 1; }
  } else if (STREAM && warp == 4) {
    // bulk-copy 16 KB chunks round-robin into a 4-slot ring until the MMA loop finishes
    const size_t nchunks = gbytes / 16384;
    size_t c = blockIdx.x * 97;
    unsigned long long bytes = 0;
    uint32_t ph[4] = {0, 0, 0, 0};
    int k = 0;
    // prime
    for (int s = 0; s < 4; ++s) {
      if (elect_one()) {
        mbar_expect_tx(&sbar[s], 16384);
        bulk_g2s(ring + s * 16384, gsrc + (c++ % nchunks) * 16384, 16384, &sbar[s]);
      }
      __syncwarp();
    }
    const long long t0 = clock64();
    while (!done) {
      const int s = k & 3;
      mbar_wait(&sbar[s], ph[s]);
      ph[s] ^= 1;
      bytes += 16384;
      if (elect_one()) {
        mbar_expect_tx(&sbar[s], 16384);
        bulk_g2s(ring + s * 16384, gsrc + (c++ % nchunks) * 16384, 16384, &sbar[s]);
      }
      __syncwarp();
      ++k;
    }
    for (int s = 0; s < 4; ++s) { mbar_wait(&sbar[(k + s) & 3], ph[(k + s) & 3]); ph[(k + s) & 3] ^= 1; }
    const long long t1 = clock64();
    if (threadIdx.x == 128) out2[blockIdx.x] = (bytes * 1000ull) / (unsigned long long)(t1 - t0);  // mB/cyc
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tbase, 512); }
}

template <int N, int NACC, int MODE, bool STREAM, int M = 128, int BMN = 0>
void run_rate(const char* name, int iters, const uint8_t* gsrc, size_t gbytes) {
  auto k = rate_kernel<N, NACC, MODE, STREAM, M, BMN>;
  const int smem = 16384 + 32768 + 65536 + 2048;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  unsigned long long *d, *d2;
  CK(cudaMalloc(&d, 148 * 8));
  CK(cudaMalloc(&d2, 148 * 8));
  CK(cudaMemset(d2, 0, 148 * 8));
  k<<<148, 256, smem>>>(iters, gsrc, gbytes, d, d2);
  CK(cudaDeviceSynchronize());
  unsigned long long h[148], h2[148];
  CK(cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h2, d2, sizeof(h2), cudaMemcpyDeviceToHost));
  double avg = 0, avg2 = 0;
  for (int i = 0; i < 148; ++i) { avg += h[i]; avg2 += h2[i]; }
  avg /= 148;
  avg2 /= 148;
  const double per_mma = avg / (iters * 4.0);
  const double ideal = M * N / 256.0;
  printf("%-34s M=%3d N=%3d nacc=%d: %6.1f cyc/MMA (floor %3.0f) -> %5.1f%% of peak", name, M, N,
         NACC, per_mma, ideal, 100.0 * ideal / per_mma);
  if (STREAM) printf("   concurrent bulk-copy fill %.1f B/cyc/SM", avg2 / 1000.0);
  printf("\n");
  CK(cudaFree(d));
  CK(cudaFree(d2));
}

// ----------------------------------------------------------------------------- P3
// A: 128 x 64 bf16 (row-major in global), B: 64(N) x 64(K) bf16 row-major (B[n][k]).
// D_ss and D_ts: 128 x 64 fp32 each.
__global__ void __launch_bounds__(256, 1) ts_check_kernel(const uint16_t* A, const uint16_t* Bm,
                                                          float* dss, float* dts) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (warp == 0) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  // SW128 K-major staging: row r (128 B) at r*128, 16-B chunk c at position c ^ (r & 7)
  for (int idx = threadIdx.x; idx < 128 * 8; idx += blockDim.x) {
    const int r = idx / 8, c = idx % 8;
    const uint4 v = reinterpret_cast<const uint4*>(A + r * 64)[c];
    *reinterpret_cast<uint4*>(smem + r * 128 + ((c ^ (r & 7)) * 16)) = v;
  }
  for (int idx = threadIdx.x; idx < 64 * 8; idx += blockDim.x) {
    const int r = idx / 8, c = idx % 8;
    const uint4 v = reinterpret_cast<const uint4*>(Bm + r * 64)[c];
    *reinterpret_cast<uint4*>(smem + 16384 + r * 128 + ((c ^ (r & 7)) * 16)) = v;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  // A into TMEM columns [0, 32): lane = row, column j = bf16 pair (2j, 2j+1)
  if (warp < 4) {
    const int row = warp * 32 + lane;
    uint32_t r[32];
    const uint32_t* src = reinterpret_cast<const uint32_t*>(A + row * 64);
    for (int j = 0; j < 32; ++j) r[j] = src[j];
    tmem_st32(tbase + ((warp * 32) << 16), r);
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 4) {
    const uint32_t idesc = make_idesc(128, 64, 1u, 0u, 0u);
    const uint32_t a0 = smem_u32(smem), b0 = a0 + 16384;
    if (elect_one()) {
      for (int ks = 0; ks < 4; ++ks) {
        const uint64_t bd = make_sdesc(b0 + ks * 32, 16, 1024, 2);
        mma_f16(tbase + 64, make_sdesc(a0 + ks * 32, 16, 1024, 2), bd, idesc, ks ? 1u : 0u);
        mma_ts(tbase + 128, tbase + ks * 8, bd, idesc, ks ? 1u : 0u);
      }
      mma_commit(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (warp < 4) {
    const int row = warp * 32 + lane;
    for (int c = 0; c < 64; c += 16) {
      float v[16];
      tmem_ld16(tbase + ((warp * 32) << 16) + 64 + c, v);
      for (int i = 0; i < 16; ++i) dss[row * 64 + c + i] = v[i];
      tmem_ld16(tbase + ((warp * 32) << 16) + 128 + c, v);
      for (int i = 0; i < 16; ++i) dts[row * 64 + c + i] = v[i];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tbase, 512); }
}

static uint16_t f2bf(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return static_cast<uint16_t>(u >> 16);
}

void run_ts_check() {
  std::vector<uint16_t> A(128 * 64), Bm(64 * 64);
  std::vector<float> Af(128 * 64), Bf(64 * 64);
  srand(1);
  for (int i = 0; i < 128 * 64; ++i) { Af[i] = (rand() % 9) - 4; A[i] = f2bf(Af[i]); }
  for (int i = 0; i < 64 * 64; ++i) { Bf[i] = (rand() % 7) - 3; Bm[i] = f2bf(Bf[i]); }
  uint16_t *dA, *dB;
  float *dss, *dts;
  CK(cudaMalloc(&dA, A.size() * 2));
  CK(cudaMalloc(&dB, Bm.size() * 2));
  CK(cudaMalloc(&dss, 128 * 64 * 4));
  CK(cudaMalloc(&dts, 128 * 64 * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, Bm.data(), Bm.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(ts_check_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000));
  ts_check_kernel<<<1, 256, 40000>>>(dA, dB, dss, dts);
  CK(cudaDeviceSynchronize());
  std::vector<float> ss(128 * 64), ts(128 * 64);
  CK(cudaMemcpy(ss.data(), dss, ss.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(ts.data(), dts, ts.size() * 4, cudaMemcpyDeviceToHost));
  int bad_ss = 0, bad_ts = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 64; ++n) {
      float ref = 0;
      for (int k = 0; k < 64; ++k) ref += Af[m * 64 + k] * Bf[n * 64 + k];
      bad_ss += ss[m * 64 + n] != ref;
      bad_ts += ts[m * 64 + n] != ref;
    }
  printf("P3 TS layout check: SS mismatches %d / 8192, TS mismatches %d / 8192 (ts[0]=%g ref-ss[0]=%g)\n",
         bad_ss, bad_ts, ts[0], ss[0]);
}

// ----------------------------------------------------------------------------- P5
// every CTA streams `per_cta` bytes of 16 KB chunks from gsrc into a 6-slot smem ring
__global__ void __launch_bounds__(64, 1) l2bw_kernel(const uint8_t* gsrc, size_t gbytes, int chunks_per_cta,
                                                     int chunk, int S) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t sbar[16];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) mbar_init(&sbar[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const size_t nchunks = gbytes / chunk;
  size_t c = static_cast<size_t>(blockIdx.x) * 7919;
  uint32_t ph[16] = {0};
  for (int i = 0; i < chunks_per_cta + S; ++i) {
    const int s = i % S;
    if (i >= S) { mbar_wait(&sbar[s], ph[s]); ph[s] ^= 1; }
    if (i < chunks_per_cta) {
      if (elect_one()) {
        mbar_expect_tx(&sbar[s], chunk);
        bulk_g2s(smem_raw + s * chunk, gsrc + (c % nchunks) * chunk, chunk, &sbar[s]);
      }
      c += 131;
      __syncwarp();
    }
  }
}

// P5b: plain 16-B loads by many warps (LSU path), each warp sums its loads
__global__ void __launch_bounds__(1024, 1) ldg_bw_kernel(const uint4* gsrc, size_t n16, int iters, uint32_t* sink) {
  uint32_t acc = 0;
  size_t base = (static_cast<size_t>(blockIdx.x) * 1024 + threadIdx.x) * 4;
  const size_t stride = static_cast<size_t>(gridDim.x) * 1024 * 4;
  for (int i = 0; i < iters; ++i) {
    uint4 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = __ldcg(gsrc + ((base + j) % n16));
#pragma unroll
    for (int j = 0; j < 4; ++j) acc ^= v[j].x ^ v[j].y ^ v[j].z ^ v[j].w;
    base += stride;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

// ----------------------------------------------------------------------------- P6
// 4 warps per CTA: each thread loads its 128-B row of a 128x64 bf16 panel with 8 x 16-B loads
// and writes it to TMEM (32 columns), double-buffered across two column slots.
__global__ void __launch_bounds__(128, 1) ldg_sttm_kernel(const uint8_t* gsrc, size_t gbytes, int panels,
                                                           unsigned long long* out) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (warp == 0) { tmem_alloc(&tslot, 64); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  const size_t npan = gbytes / 16384;
  size_t c = static_cast<size_t>(blockIdx.x) * 7919;
  const long long t0 = clock64();
  uint4 buf[2][8];
  {
    const uint4* src = reinterpret_cast<const uint4*>(gsrc + (c % npan) * 16384 + (warp * 32 + lane) * 128);
#pragma unroll
    for (int j = 0; j < 8; ++j) buf[0][j] = __ldcs(src + j);
  }
  for (int p = 0; p < panels; ++p) {
    c += 131;
    const int cur = p & 1;
    if (p + 1 < panels) {
      const uint4* src = reinterpret_cast<const uint4*>(gsrc + (c % npan) * 16384 + (warp * 32 + lane) * 128);
#pragma unroll
      for (int j = 0; j < 8; ++j) buf[cur ^ 1][j] = __ldcs(src + j);
    }
    uint32_t r[32];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      r[4 * j] = buf[cur][j].x; r[4 * j + 1] = buf[cur][j].y; r[4 * j + 2] = buf[cur][j].z; r[4 * j + 3] = buf[cur][j].w;
    }
    tmem_st32(tbase + ((warp * 32) << 16) + cur * 32, r);
  }
  tmem_wait_st();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tbase, 64); }
}

// ----------------------------------------------------------------------------- P7
// cta_group::2 SS-MMA issue rate: M=256 (128 rows per CTA), N (B split N/2 per CTA)
template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) pair_rate_kernel(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32;
  const uint32_t rank = cluster_ctarank();
  if (warp == 0) { tmem_alloc_pair(&tslot, 512); tmem_relinquish_pair(); }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = tslot;
  const uint32_t a0 = smem_u32(smem), b0 = a0 + 16384;
  const uint32_t idesc = make_idesc(256, N, 1u, 0u, 0u);
  if (warp == 1 && rank == 0) {
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint64_t bd = make_sdesc(b0 + ks * 32, 16, 1024, 2);
          const uint64_t ad = make_sdesc(a0 + ks * 32, 16, 1024, 2);
          mma_f16_pair(tbase, ad, bd, idesc, (i | ks) ? 1u : 0u);
        }
        if ((i & 63) == 63) mma_commit_pair(&bar);
      }
      __syncwarp();
      if ((i & 63) == 63) mbar_wait(&bar, (i >> 6) & 1);
    }
    const long long t1 = clock64();
    if (threadIdx.x == 32) out[blockIdx.x / 2] = t1 - t0;
  } else if (warp == 1 && rank == 1) {
    for (int i = 63; i < iters; i += 64) mbar_wait(&bar, (i >> 6) & 1);
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 0) { tc_fence_after(); tmem_dealloc_pair(tbase, 512); }
}

template <int N>
void run_pair_rate(int iters) {
  auto k = pair_rate_kernel<N>;
  const int smem = 16384 + 32768 + 2048;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  unsigned long long* d;
  CK(cudaMalloc(&d, 74 * 8));
  k<<<148, 128, smem>>>(iters, d);
  CK(cudaDeviceSynchronize());
  unsigned long long h[74];
  CK(cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost));
  double avg = 0;
  for (int i = 0; i < 74; ++i) avg += h[i];
  avg /= 74;
  const double per_mma = avg / (iters * 4.0);
  printf("P7 pair SS M=256 N=%3d: %6.1f cyc/MMA -> per SM %.1f cyc per 128x%dx16 (single-CTA SS N=%d: see P1)\n", N,
         per_mma, per_mma, N, N);
  CK(cudaFree(d));
}


__device__ __forceinline__ bool mbar_test(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
               : "=r"(ok) : "r"(addr), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool mbar_try_hint(uint32_t addr, uint32_t parity, uint32_t ns) {
  uint32_t ok;
  asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\nselp.u32 %0, 1, 0, p;\n}\n"
               : "=r"(ok) : "r"(addr), "r"(parity), "r"(ns) : "memory");
  return ok != 0;
}
template <int W>
__device__ __forceinline__ void wait_v(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  if (W == 0) { while (!mbar_try_wait(a, parity)) {} }
  else if (W == 1) { while (!mbar_test(a, parity)) {} }
  else { while (!mbar_try_hint(a, parity, 20)) {} }
}
// ----------------------------------------------------------------------------- P8
// Per-step synchronisation overhead of the engine's MMA loop without TMA:
// MODE 0: 4 MMAs (N=64) + commit to a ring of 8 mbarriers per step;
// MODE 1: MODE 0 + wait on a "full" mbarrier that a helper warp arrives on 8 steps ahead,
//         and tcgen05.fence::after_thread_sync (the engine's loop shape)
// MODE 2: MODE 1 but two steps (8 MMAs, 2 commits) per wait
template <int MODE, int W = 0, int S = 8>
__global__ void __launch_bounds__(128, 1) sync_rate_kernel(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t emptyb[16], fullb[16];
  const int warp = threadIdx.x / 32;
  if (warp == 0) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) { mbar_init(&emptyb[i], 1); mbar_init(&fullb[i], 1); }
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  const uint32_t a0 = smem_u32(smem), b0 = a0 + 16384;
  const uint32_t idesc = make_idesc(128, 64, 1u, 0u, 0u);
  const uint64_t ad0 = make_sdesc(a0, 16, 1024, 2), bd0 = make_sdesc(b0, 16, 1024, 2);
  __shared__ volatile int ready_count;
  if (threadIdx.x == 0) ready_count = 0;
  __syncthreads();
  if (warp == 1 && MODE == 10) {
    // the MMA warp never touches shared memory: warp 3 waits on full[] and releases the
    // MMA warp through a named barrier (bar.sync / bar.arrive, ids 1..8 by stage)
    const long long t0 = clock64();
    uint32_t stage = 0;
    for (int i = 0; i < iters; ++i) {
      asm volatile("bar.sync %0, 64;" ::"r"(1 + stage));
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          mma_f16(tbase + (i & 1) * 64, ad0 + ks * 2, bd0 + ks * 2, idesc, ks ? 1u : 0u);
        mma_commit(&emptyb[stage]);
      }
      __syncwarp();
      if (++stage == S) stage = 0;
    }
    const long long t1 = clock64();
    if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
  } else if (warp == 3 && MODE == 10) {
    uint32_t stage = 0, phase = 0;
    for (int i = 0; i < iters; ++i) {
      wait_v<0>(&fullb[stage], phase);
      asm volatile("bar.arrive %0, 64;" ::"r"(1 + stage));
      if (++stage == S) { stage = 0; phase ^= 1; }
    }
  } else if (warp == 1 && MODE == 9) {
    // the MMA warp never waits on an mbarrier: warp 3 waits on full[] and publishes a
    // counter in shared memory that the MMA warp polls
    const long long t0 = clock64();
    uint32_t stage = 0;
    for (int i = 0; i < iters; ++i) {
      while (ready_count <= i) {
      }
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          mma_f16(tbase + (i & 1) * 64, ad0 + ks * 2, bd0 + ks * 2, idesc, ks ? 1u : 0u);
        mma_commit(&emptyb[stage]);
      }
      __syncwarp();
      if (++stage == S) stage = 0;
    }
    const long long t1 = clock64();
    if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
  } else if (warp == 3 && MODE == 9) {
    uint32_t stage = 0, phase = 0;
    for (int i = 0; i < iters; ++i) {
      wait_v<0>(&fullb[stage], phase);
      if (lane_id() == 0) ready_count = i + 1;
      __syncwarp();
      if (++stage == S) { stage = 0; phase ^= 1; }
    }
  } else if (warp == 1 && MODE == 8) {
    // warp-uniform; the wait for step k+1 sits before step k's last MMA
    const long long t0 = clock64();
    uint32_t stage = 0, phase = 0;
    wait_v<0>(&fullb[0], 0);
    tc_fence_after();
    for (int i = 0; i < iters; ++i) {
      const uint32_t ns = stage + 1 == S ? 0 : stage + 1;
      const uint32_t nph = stage + 1 == S ? phase ^ 1 : phase;
      if (elect_one()) {
        mma_f16(tbase + (i & 1) * 64, ad0, bd0, idesc, 0u);
        mma_f16(tbase + (i & 1) * 64, ad0 + 2, bd0 + 2, idesc, 1u);
        mma_f16(tbase + (i & 1) * 64, ad0 + 4, bd0 + 4, idesc, 1u);
      }
      __syncwarp();
      if (i + 1 < iters) wait_v<0>(&fullb[ns], nph);
      tc_fence_after();
      if (elect_one()) {
        mma_f16(tbase + (i & 1) * 64, ad0 + 6, bd0 + 6, idesc, 1u);
        mma_commit(&emptyb[stage]);
      }
      __syncwarp();
      stage = ns;
      phase = nph;
    }
    const long long t1 = clock64();
    if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
  } else if (warp == 1 && MODE == 7) {
    // single-lane loop; the wait for step k+1 sits between step k's 2nd and 3rd MMA
    const long long t0 = clock64();
    if (lane_id() == 0) {
      uint32_t stage = 0, phase = 0;
      wait_v<0>(&fullb[0], 0);
      for (int i = 0; i < iters; ++i) {
        const uint32_t ns = stage + 1 == S ? 0 : stage + 1;
        const uint32_t nph = stage + 1 == S ? phase ^ 1 : phase;
        tc_fence_after();
        mma_f16(tbase + (i & 1) * 64, ad0, bd0, idesc, 0u);
        mma_f16(tbase + (i & 1) * 64, ad0 + 2, bd0 + 2, idesc, 1u);
        if (i + 1 < iters) wait_v<0>(&fullb[ns], nph);
        mma_f16(tbase + (i & 1) * 64, ad0 + 4, bd0 + 4, idesc, 1u);
        mma_f16(tbase + (i & 1) * 64, ad0 + 6, bd0 + 6, idesc, 1u);
        mma_commit(&emptyb[stage]);
        stage = ns;
        phase = nph;
      }
    }
    __syncwarp();
    const long long t1 = clock64();
    if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
  } else if (warp == 1 && MODE == 5) {
    // look-ahead: test full[k+1] before issuing step k's MMAs, block only if it failed
    const long long t0 = clock64();
    uint32_t stage = 0, phase = 0;
    wait_v<0>(&fullb[0], 0);
    for (int i = 0; i < iters; ++i) {
      const uint32_t ns = stage + 1 == S ? 0 : stage + 1;
      const uint32_t nph = stage + 1 == S ? phase ^ 1 : phase;
      const bool ready = i + 1 >= iters || mbar_test(smem_u32(&fullb[ns]), nph);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          mma_f16(tbase + (i & 1) * 64, ad0 + ks * 2, bd0 + ks * 2, idesc, ks ? 1u : 0u);
        mma_commit(&emptyb[stage]);
      }
      __syncwarp();
      if (!ready) wait_v<0>(&fullb[ns], nph);
      stage = ns;
      phase = nph;
    }
    const long long t1 = clock64();
    if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
  } else if (warp == 1) {
    const long long t0 = clock64();
    uint32_t stage = 0, phase = 0;
    const int per = MODE == 2 ? 2 : 1;
    long long tw = 0, tm = 0;
    for (int i = 0; i < iters; i += per) {
      const long long a = clock64();
      if (MODE >= 1 && MODE != 4 && MODE != 6) {
        wait_v<W>(&fullb[stage], phase);
        if (MODE == 2) wait_v<W>(&fullb[stage + 1], phase);
      }
      if (MODE == 1 || MODE == 2 || MODE == 4) tc_fence_after();
      const long long b = clock64();
      if (elect_one()) {
        for (int k = 0; k < per; ++k) {
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            mma_f16(tbase + ((i + k) & 1) * 64, ad0 + ks * 2, bd0 + ks * 2, idesc, ks ? 1u : 0u);
          mma_commit(&emptyb[stage + k]);
        }
      }
      __syncwarp();
      const long long c = clock64();
      tw += b - a;
      tm += c - b;
      stage += per;
      if (stage == S) { stage = 0; phase ^= 1; }
    }
    const long long t1 = clock64();
    if (threadIdx.x == 32) {
      out[blockIdx.x] = t1 - t0;
      if (blockIdx.x == 0) printf("   mode %d: per step wait+fence %.1f, mma issue+commit %.1f cycles\n", MODE,
                                  double(tw) * per / iters, double(tm) * per / iters);
    }
  } else if (warp == 2 && MODE == 6) {
    // observer only: waits on every empty phase, arrives nowhere (MMA warp runs mode 0)
    uint32_t stage = 0, phase = 0;
    for (int i = 0; i < iters; ++i) {
      wait_v<0>(&emptyb[stage], phase);
      if (++stage == S) { stage = 0; phase ^= 1; }
    }
  } else if (warp == 2 && MODE >= 1 && MODE != 4) {
    // "producer": arrive full[s] once the MMAs that used stage s (8 steps ago) are done
    uint32_t stage = 0, phase = 0;
    for (int i = 0; i < iters; ++i) {
      if (i >= S) wait_v<W>(&emptyb[stage], phase ^ 1);
      if (elect_one()) mbar_arrive(&fullb[stage]);
      __syncwarp();
      if (++stage == S) { stage = 0; phase ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tbase, 512); }
}

template <int MODE, int W = 0, int S = 8>
void run_sync_rate(int iters) {
  auto k = sync_rate_kernel<MODE, W, S>;
  const int smem = 16384 + 32768 + 2048;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  unsigned long long* d;
  CK(cudaMalloc(&d, 148 * 8));
  k<<<148, 128, smem>>>(iters, d);
  CK(cudaDeviceSynchronize());
  unsigned long long h[148];
  CK(cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost));
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("P8 sync mode %d wait %d stages %d: %.1f cycles per step (4 x SS N=64 MMAs)\n", MODE, W, S, avg / iters);
  CK(cudaFree(d));
}

// ----------------------------------------------------------------------------- P11
// Accumulator dependency chains: 8 SS M=128 N=64 MMAs per iteration spread over NCH
// accumulators, either blocked (all of one accumulator's MMAs back to back, like the
// engine's TM = 2 step: h0 k0..k3, h1 k0..k3) or interleaved round-robin. All accumulate.
template <int NCH, bool INTERLEAVE>
__global__ void __launch_bounds__(128, 1) chain_kernel(int iters, unsigned long long* out) {
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
  const uint32_t a0 = smem_u32(smem), b0 = a0 + 32768;
  const uint32_t idesc = make_idesc(128, 64, 1u, 0u, 0u);
  if (warp == 1) {
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (elect_one()) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int per = 8 / NCH;
          const int acc = INTERLEAVE ? j % NCH : j / per;
          const int ks = (INTERLEAVE ? j / NCH : j % per) & 3;
          const uint64_t ad = make_sdesc(a0 + (acc & 1) * 16384 + ks * 32, 16, 1024, 2);
          const uint64_t bd = make_sdesc(b0 + ks * 32, 16, 1024, 2);
          mma_f16(tbase + acc * 64, ad, bd, idesc, 1u);
        }
        if ((i & 7) == 7) mma_commit(&bar);
      }
      __syncwarp();
      if ((i & 7) == 7) mbar_wait(&bar, (i >> 3) & 1);
    }
    const long long t1 = clock64();
    if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

template <int NCH, bool INTERLEAVE>
void run_chain(int iters) {
  auto k = chain_kernel<NCH, INTERLEAVE>;
  const int smem = 65536 + 2048;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  unsigned long long* d;
  CK(cudaMalloc(&d, 148 * 8));
  k<<<148, 128, smem>>>(iters, d);
  CK(cudaDeviceSynchronize());
  unsigned long long h[148];
  CK(cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost));
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("P11 %d accumulators %-11s: %6.1f cyc/MMA (8 MMAs per commit group of 1)\n", NCH,
         INTERLEAVE ? "interleaved" : "blocked", avg / (iters * 8.0));
  CK(cudaFree(d));
}

int main(int argc, char** argv) {
  int clk_khz = 0;
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  printf("SM clock attr %.0f MHz\n", clk_khz / 1000.0);
  const size_t gbytes = 48ull << 20;  // L2-resident source
  uint8_t* g;
  CK(cudaMalloc(&g, gbytes));
  CK(cudaMemset(g, 1, gbytes));
  if (argc > 1 && argv[1][0] == 'm') {  // P9: M = 64 vs M = 128 issue rate by N
    run_rate<64, 1, 0, false, 64>("P9 SS", 4000, g, gbytes);
    run_rate<128, 1, 0, false, 64>("P9 SS", 4000, g, gbytes);
    run_rate<256, 1, 0, false, 64>("P9 SS", 2000, g, gbytes);
    run_rate<64, 1, 0, false>("P9 SS", 4000, g, gbytes);
    run_rate<128, 1, 0, false>("P9 SS", 4000, g, gbytes);
    run_rate<256, 1, 0, false>("P9 SS", 2000, g, gbytes);
    run_rate<256, 2, 0, false>("P9 SS", 2000, g, gbytes);
    return 0;
  }
  if (argc > 1 && argv[1][0] == 'c') {
    run_chain<1, false>(2000);
    run_chain<2, false>(2000);
    run_chain<2, true>(2000);
    run_chain<4, false>(2000);
    run_chain<4, true>(2000);
    run_chain<8, true>(2000);
    return 0;
  }
  if (argc > 1 && argv[1][0] == 'b') {  // P10: B operand K-major vs MN-major (weights)
    run_rate<64, 1, 0, false>("P10 SS B K-major", 4000, g, gbytes);
    run_rate<64, 2, 0, false>("P10 SS B K-major", 4000, g, gbytes);
    run_rate<64, 1, 0, false, 128, 1>("P10 SS B MN-major", 4000, g, gbytes);
    run_rate<64, 2, 0, false, 128, 1>("P10 SS B MN-major", 4000, g, gbytes);
    run_rate<128, 1, 0, false, 128, 1>("P10 SS B MN-major", 4000, g, gbytes);
    run_rate<64, 1, 1, false, 128, 1>("P10 TS B MN-major", 4000, g, gbytes);
    return 0;
  }

  run_sync_rate<0>(4000);
  run_sync_rate<1>(4000);
  run_sync_rate<2>(4000);
  run_sync_rate<9, 0, 8>(4000);
  run_sync_rate<10, 0, 8>(4000);

  run_pair_rate<64>(4000);
  run_pair_rate<128>(4000);
  run_pair_rate<256>(2000);
  run_ts_check();
  run_rate<64, 1, 0, false>("P1 SS", 4000, g, gbytes);
  run_rate<64, 2, 0, false>("P1 SS", 4000, g, gbytes);
  run_rate<64, 4, 0, false>("P1 SS", 4000, g, gbytes);
  run_rate<128, 1, 0, false>("P1 SS", 4000, g, gbytes);
  run_rate<128, 2, 0, false>("P1 SS", 4000, g, gbytes);
  run_rate<256, 1, 0, false>("P1 SS", 2000, g, gbytes);
  run_rate<64, 1, 1, false>("P2 TS", 4000, g, gbytes);
  run_rate<64, 2, 1, false>("P2 TS", 4000, g, gbytes);
  run_rate<128, 1, 1, false>("P2 TS", 4000, g, gbytes);
  run_rate<64, 1, 0, true>("P4 SS + bulk-copy stream", 8000, g, gbytes);
  run_rate<64, 1, 1, true>("P4 TS + bulk-copy stream", 8000, g, gbytes);
  run_rate<128, 1, 0, true>("P4 SS + bulk-copy stream", 8000, g, gbytes);

  // P5 chip L2 -> SM bandwidth vs bytes in flight per SM
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const size_t src_bytes = 16ull << 20;
  for (int chunk : {16384, 32768}) {
    for (int S : {2, 4, 6, 8, 12}) {
      for (int per_sm : {1, 2}) {
        const int smem = S * chunk;
        if (smem * per_sm > 220 * 1024) continue;
        const int ctas = 148 * per_sm;
        const int per = (int)((1024ull << 20) / chunk / ctas);
        CK(cudaFuncSetAttribute(l2bw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        l2bw_kernel<<<ctas, 64, smem>>>(g, src_bytes, per, chunk, S);
        CK(cudaEventRecord(e0));
        l2bw_kernel<<<ctas, 64, smem>>>(g, src_bytes, per, chunk, S);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("P5 bulk L2->smem chunk %5d slots %2d ctas/SM %d (%3d KB in flight/SM): %.0f GB/s\n", chunk, S,
               per_sm, S * chunk * per_sm / 1024, (double)per * ctas * chunk / (ms * 1e6));
      }
    }
  }
  {
    uint32_t* sink;
    CK(cudaMalloc(&sink, 4));
    const size_t n16 = src_bytes / 16;
    for (int ctas : {148, 296}) {
      const int iters = 2000;
      ldg_bw_kernel<<<ctas, 1024>>>(reinterpret_cast<const uint4*>(g), n16, iters, sink);
      CK(cudaEventRecord(e0));
      ldg_bw_kernel<<<ctas, 1024>>>(reinterpret_cast<const uint4*>(g), n16, iters, sink);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      printf("P5b LDG.128 L2->SM ctas %d x 1024 thr: %.0f GB/s\n", ctas, (double)iters * ctas * 1024 * 64 / (ms * 1e6));
    }
  }
  // P6 LDG -> TMEM
  {
    unsigned long long* d;
    CK(cudaMalloc(&d, 296 * 8));
    for (int ctas : {148, 296}) {
      const int panels = 2000;
      ldg_sttm_kernel<<<ctas, 128>>>(g, gbytes, panels, d);
      CK(cudaEventRecord(e0));
      ldg_sttm_kernel<<<ctas, 128>>>(g, gbytes, panels, d);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      unsigned long long h[296];
      CK(cudaMemcpy(h, d, ctas * 8, cudaMemcpyDeviceToHost));
      double avg = 0;
      for (int i = 0; i < ctas; ++i) avg += h[i];
      avg /= ctas;
      printf("P6 LDG->TMEM ctas %d: %.0f GB/s chip, %.1f cyc per 16 KB panel per CTA\n", ctas,
             (double)panels * ctas * 16384 / (ms * 1e6), avg / panels);
    }
  }
  CK(cudaGetLastError());
  printf("done\n");
  return 0;
}
