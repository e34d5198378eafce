// Shared host/device helpers of the kernel translation units (leaf.cu, preadd.cu,
// combine.cu, misc.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "kernels.hpp"
#include "ptx.cuh"

namespace adj {

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

// rows a pre-addition / split launch covers: [0, rows_pad), or the listed ranges (output-tile
// sharding: only the tile bands the rank's tiles read)
__host__ __device__ __forceinline__ int64_t range_rows(const RowRanges &R, int64_t rows_pad) {
  if (R.n == 0) return rows_pad;
  int64_t t = 0;
  for (int i = 0; i < R.n; ++i) t += R.hi[i] - R.lo[i];
  return t;
}
__device__ __forceinline__ int64_t range_row(const RowRanges &R, int64_t j) {
  if (R.n == 0) return j;
  for (int i = 0; i < R.n; ++i) {
    const int64_t len = R.hi[i] - R.lo[i];
    if (j < len) return R.lo[i] + j;
    j -= len;
  }
  return -1;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device): the attribute is
// per device, `done` is a per-kernel bitmask of device ordinals (thread-safe)
template <typename K>
inline cudaError_t ensure_smem(K kernel, int bytes, std::atomic<uint64_t> &done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

}  // namespace adj
