// Device copy of the counter-based input generator of inputs/gen.py (same formula,
// bit-identical output).  Holds none of the method's arithmetic; it exists so that
// multi-GiB synthetic inputs can be produced in HBM.
//
//   out[j] = mulhi64(splitmix64(splitmix64(seed) ^ (start + j)), p),  mulhi64(x,p) = (x*p) >> 64
#include <cstdint>
#include <cuda_runtime.h>

static __host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void adjgen_uniform_kernel(uint32_t* __restrict__ out, uint64_t n, uint64_t key,
                                      uint32_t p, uint64_t start) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
    uint64_t z = splitmix64((start + j) ^ key);
    out[j] = (uint32_t)__umul64hi(z, (uint64_t)p);
  }
}

extern "C" int adjgen_uniform(uint32_t* out, uint64_t n, uint64_t seed, uint32_t p,
                              uint64_t start, cudaStream_t stream) {
  if (n == 0) return 0;
  if (out == nullptr || p < 2) return 1;
  uint64_t key = splitmix64(seed);
  int threads = 256;
  uint64_t blocks = (n + threads - 1) / threads;
  if (blocks > 148ull * 64) blocks = 148ull * 64;
  adjgen_uniform_kernel<<<(unsigned)blocks, threads, 0, stream>>>(out, n, key, p, start);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
