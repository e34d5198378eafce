// Microbenchmark: sustained tcgen05 int8 MMA rate on this B200 (no TMA, operands resident in smem).
//   mode 0: cta_group::2, M=256 N=256 K=32 per instruction (the leaf kernel's shape)
//   mode 1: cta_group::1, M=128 N=256
//   mode 2: cta_group::1, M=128 N=128
// Reports int8 TOP/s (2 ops per MAC) over all SMs, timed with CUDA events.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "../paper_2101_01025_b200/csrc/ptx.cuh"

using namespace adj;

template <int MODE>
__global__ void __launch_bounds__(128, 1) mma_loop(int iters, int *sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr bool PAIR = MODE == 0;
  constexpr int M = MODE == 0 ? 256 : 128;
  constexpr int N = MODE == 2 ? 128 : 256;
  uint32_t rank = 0;
  if constexpr (PAIR) rank = ptx::cluster_ctarank();
  // fill operand smem (64 KB) with small values
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0x01010101u * (i & 3);
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    if constexpr (PAIR) ptx::tmem_alloc_2sm(&holder, 512);
    else ptx::tmem_alloc(&holder, 512);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tbase = holder;
  if (warp == 1 && lane == 0 && rank == 0) {
    const uint32_t sa = ptx::smem_u32(smem);
    const uint64_t adesc = ptx::smem_desc_sw128(sa);
    const uint64_t bdesc = ptx::smem_desc_sw128(sa + 32768);
    const uint32_t idesc = ptx::idesc_i8(M, N, true, true);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        if constexpr (PAIR) ptx::mma_i8_2sm(tbase + (it & 1) * 256, adesc + 2 * kk, bdesc + 2 * kk, idesc, it | kk);
        else ptx::mma_i8(tbase + (it & 1) * 256, adesc + 2 * kk, bdesc + 2 * kk, idesc, it | kk);
      }
    }
    if constexpr (PAIR) ptx::mma_commit_2sm(&bar, 0x3);
    else ptx::mma_commit(&bar);
  }
  if (!PAIR || true) {
    if (threadIdx.x == 64) ptx::mbar_wait(&bar, 0);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) ptx::cluster_sync();
  if (warp == 0) {
    ptx::tc_fence_after();
    if constexpr (PAIR) ptx::tmem_dealloc_2sm(tbase, 512);
    else ptx::tmem_dealloc(tbase, 512);
  }
  if (threadIdx.x == 0 && sink) sink[blockIdx.x] = (int)tbase;
}

template <int MODE>
double run(int sms, int iters) {
  auto k = mma_loop<MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024 + 1024);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 66 * 1024 + 1024;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = MODE == 0 ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int *sink;
  cudaMalloc(&sink, sms * sizeof(int));
  for (int w = 0; w < 2; ++w) cudaLaunchKernelEx(&cfg, k, iters, sink);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) cudaLaunchKernelEx(&cfg, k, iters, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
  const int M = MODE == 0 ? 256 : 128, N = MODE == 2 ? 128 : 256;
  const double units = MODE == 0 ? sms / 2 : sms;   // MMA issuers
  const double macs = units * (double)iters * 4 * M * N * 32 * reps;
  cudaFree(sink);
  return 2 * macs / (ms * 1e-3) / 1e12;
}

int main(int argc, char **argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = argc > 1 ? atoi(argv[1]) : 20000;
  printf("{\"sms\": %d, \"iters\": %d, \"pair_256x256_tops\": %.1f, \"single_128x256_tops\": %.1f, "
         "\"single_128x128_tops\": %.1f}\n",
         sms, iters, run<0>(sms, iters), run<1>(sms, iters), run<2>(sms, iters));
  return 0;
}
