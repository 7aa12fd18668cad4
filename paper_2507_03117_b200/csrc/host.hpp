// Host-side helpers shared by the C-ABI translation units: error state, device
// properties, TMA descriptor encoding, stream-ordered scratch.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <string>

#include "../../include/blast.h"

namespace blast {

void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* what);
int num_sms();
int bytes_of(int dtype);  // BLAST_F32 -> 4, BLAST_BF16 -> 2
void retain_pool_memory();  // keep freed cudaMallocAsync blocks cached in the default pool

inline int check_launch(const char* what) { return cuda_status(cudaGetLastError(), what); }

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per kernel and per device: `configured`
// is the calling kernel's own per-device flag array (a function-local static of the caller)
template <typename K>
inline int configure_smem(K kern, int bytes, bool (&configured)[64], const char* what) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cuda_status(cudaGetLastError(), what);
  if (dev >= 0 && dev < 64 && configured[dev]) return 0;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return cuda_status(e, what);
  if (dev >= 0 && dev < 64) configured[dev] = true;
  return 0;
}

// 2-D tiled tensor map over a row-major [outer, inner] array (inner contiguous).
// box = {box_inner, box_outer}; swizzle in bytes (0, 32, 64, 128).
bool encode_map_2d(CUtensorMap* map, const void* base, int dtype, uint64_t inner, uint64_t outer,
                   uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer,
                   int swizzle_bytes);

// Stream-ordered scratch (cudaMallocAsync pool); freed on the same stream.
struct Scratch {
  void* ptr = nullptr;
  cudaStream_t stream = nullptr;
  Scratch() = default;
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  ~Scratch() {
    if (ptr) cudaFreeAsync(ptr, stream);
  }
  bool alloc(size_t bytes, cudaStream_t s) {
    retain_pool_memory();
    stream = s;
    if (bytes == 0) bytes = 16;
    return cudaMallocAsync(&ptr, bytes, s) == cudaSuccess;
  }
  template <typename T> T* as() const { return reinterpret_cast<T*>(ptr); }
};

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace blast
