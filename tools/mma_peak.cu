// Microbenchmark: sustained tcgen05 int8 MMA rate on this B200 (no TMA, operands resident in smem).
//   mode 0: cta_group::2, M=256 N=256 K=32 per instruction (the leaf kernel's shape)
//   mode 1: cta_group::1, M=128 N=256
//   mode 2: cta_group::1, M=128 N=128
// Reports int8 TOP/s (2 ops per MAC) over all SMs, timed with CUDA events.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>
#include <cuda_runtime.h>

#include "../paper_2101_01025_b200/csrc/ptx.cuh"

using namespace adj;

// VAR bits (pair mode only): 1 = tcgen05.commit after every 4 MMAs, 2 = try_wait on a completed
// mbarrier + tcgen05.fence::after_thread_sync before every 4 MMAs, 4 = 8 MMAs per group
template <int MODE, int VAR = 0>
__global__ void __launch_bounds__(128, 1) mma_loop(int iters, int *sink, int rnd = 0) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar, bar2, bar3;
  __shared__ uint64_t fullb[5], emptyb[5];
  __shared__ uint32_t holder;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr bool PAIR = MODE == 0;
  constexpr int M = MODE == 0 ? 256 : 128;
  constexpr int N = MODE == 2 ? 128 : 256;
  uint32_t rank = 0;
  if constexpr (PAIR) rank = ptx::cluster_ctarank();
  // fill operand smem (64 KB) with small values
  // rnd: uniformly random bytes (the leaf's limb planes of uniform residues toggle like this;
  // tensor-core power depends on the operand bits)
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 0x9E3779B9u + blockIdx.x * 0x85EBCA6Bu;
    h ^= h >> 15; h *= 0x2C1B3C6Du; h ^= h >> 12; h *= 0x297A2D39u; h ^= h >> 15;
    reinterpret_cast<uint32_t *>(smem)[i] = rnd ? h : 0x01010101u * (i & 3);
  }
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::mbar_init(&bar2, 1 << 20);
    ptx::mbar_init(&bar3, 1);
    ptx::fence_barrier_init();
    ptx::mbar_arrive(&bar3);   // phase 0 of bar3 complete
    for (int i = 0; i < 5; ++i) { ptx::mbar_init(&fullb[i], 1); ptx::mbar_init(&emptyb[i], 1); }
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
  if constexpr ((VAR & 8) != 0) {
    // 5-stage ring like the leaf kernel: producer (warp 2) waits empty -> arrives full; MMA waits
    // full -> 4 MMAs -> commit (multicast to both CTAs when VAR & 16) on empty.
    const int nst = iters;
    if (warp == 2 && lane == 0 && (rank == 0 || (VAR & 16))) {
      int st = 0; uint32_t ph = 0;
      for (int it = 0; it < nst; ++it) {
        ptx::mbar_wait(&emptyb[st], ph ^ 1);
        if (rank == 0) ptx::mbar_arrive(&fullb[st]);
        if (++st == 5) { st = 0; ph ^= 1; }
      }
    }
    if (warp == 1 && lane == 0 && rank == 0) {
      const uint32_t idesc = ptx::idesc_i8(M, N, true, true);
      int st = 0; uint32_t ph = 0;
      for (int it = 0; it < nst; ++it) {
        ptx::mbar_wait(&fullb[st], ph);
        ptx::tc_fence_after();
        const uint32_t sa = ptx::smem_u32(smem) + (st & 1) * 16384;   // A alternates within [0, 32K)
        const uint64_t adesc = ptx::smem_desc_sw128(sa);
        const uint64_t bdesc = ptx::smem_desc_sw128(ptx::smem_u32(smem) + 32768);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          if constexpr (PAIR) ptx::mma_i8_2sm(tbase + (it & 1) * 256, adesc + 2 * kk, bdesc + 2 * kk, idesc, it | kk);
          else ptx::mma_i8(tbase + (it & 1) * 256, adesc + 2 * kk, bdesc + 2 * kk, idesc, it | kk);
        }
        if constexpr (PAIR) ptx::mma_commit_2sm(&emptyb[st], (VAR & 16) ? 0x3 : 0x1);
        else ptx::mma_commit(&emptyb[st]);
        if (++st == 5) { st = 0; ph ^= 1; }
      }
      if constexpr (PAIR) ptx::mma_commit_2sm(&bar, 0x3);
      else ptx::mma_commit(&bar);
    }
  } else if (warp == 1 && lane == 0 && rank == 0) {
    const uint32_t sa = ptx::smem_u32(smem);
    const uint64_t adesc = ptx::smem_desc_sw128(sa);
    const uint64_t bdesc = ptx::smem_desc_sw128(sa + 32768);
    const uint32_t idesc = ptx::idesc_i8(M, N, true, true);
    constexpr int G = (VAR & 4) ? 8 : 4;
    for (int it = 0; it < iters * 4 / G; ++it) {
      if constexpr ((VAR & 2) != 0) {
        ptx::mbar_wait(&bar3, 0);
        ptx::tc_fence_after();
      }
#pragma unroll
      for (int kk = 0; kk < G; ++kk) {
        if constexpr (PAIR) ptx::mma_i8_2sm(tbase + (it & 1) * 256, adesc + 2 * (kk & 3), bdesc + 2 * (kk & 3), idesc, it | kk);
        else ptx::mma_i8(tbase + (it & 1) * 256, adesc + 2 * (kk & 3), bdesc + 2 * (kk & 3), idesc, it | kk);
      }
      if constexpr ((VAR & 1) != 0) {
        if constexpr (PAIR) ptx::mma_commit_2sm(&bar2, 0x1);
        else ptx::mma_commit(&bar2);
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

template <int MODE, int VAR = 0>
double run(int sms, int iters) {
  auto k = mma_loop<MODE, VAR>;
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
  for (int w = 0; w < 2; ++w) cudaLaunchKernelEx(&cfg, k, iters, sink, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) cudaLaunchKernelEx(&cfg, k, iters, sink, 0);
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

// back-to-back launches of the pair kernel (random operands) for `seconds`: TOP/s of every launch;
// prints the first launch and the median of the second half (the board at its steady state)
int sustain(int sms, int iters, double seconds) {
  auto k = mma_loop<0, 0>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024 + 1024);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 66 * 1024 + 1024;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int *sink;
  cudaMalloc(&sink, sms * sizeof(int));
  const double macs = (sms / 2) * (double)iters * 4 * 256 * 256 * 32;
  const int batch = 20;
  cudaEvent_t ev[batch + 1];
  for (int i = 0; i <= batch; ++i) cudaEventCreate(&ev[i]);
  std::vector<double> tops;
  double total = 0;
  while (total < seconds * 1e3) {
    cudaEventRecord(ev[0]);
    for (int i = 0; i < batch; ++i) {
      cudaLaunchKernelEx(&cfg, k, iters, sink, 1);
      cudaEventRecord(ev[i + 1]);
    }
    cudaEventSynchronize(ev[batch]);
    for (int i = 0; i < batch; ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
      total += ms;
      tops.push_back(2 * macs / (ms * 1e-3) / 1e12);
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<double> tail(tops.begin() + tops.size() / 2, tops.end());
  std::sort(tail.begin(), tail.end());
  printf("{\"mode\": \"sustain\", \"operands\": \"random bytes\", \"sms\": %d, \"launches\": %zu, \"seconds\": %.2f, "
         "\"first_launch_tops\": %.1f, \"steady_median_tops\": %.1f, \"steady_min_tops\": %.1f}\n",
         sms, tops.size(), total * 1e-3, tops[0], tail[tail.size() / 2], tail[0]);
  cudaFree(sink);
  return 0;
}

int main(int argc, char **argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  if (argc > 1 && std::string(argv[1]) == "sustain")
    return sustain(sms, argc > 2 ? atoi(argv[2]) : 20000, argc > 3 ? atof(argv[3]) : 8.0);
  const int iters = argc > 1 ? atoi(argv[1]) : 20000;
  printf("{\"sms\": %d, \"iters\": %d, \"pair_256x256_tops\": %.1f, \"single_128x256_tops\": %.1f, "
         "\"single_128x128_tops\": %.1f,\n", sms, iters, run<0>(sms, iters), run<1>(sms, iters), run<2>(sms, iters));
  printf(" \"pair_commit_every4\": %.1f, \"pair_wait_fence_every4\": %.1f, \"pair_both_every4\": %.1f, "
         "\"pair_both_every8\": %.1f, \"single128x256_both_every4\": %.1f}\n",
         run<0, 1>(sms, iters), run<0, 2>(sms, iters), run<0, 3>(sms, iters), run<0, 7>(sms, iters), run<1, 3>(sms, iters));
  printf(" {\"ring5_pair_commit_leader\": %.1f, \"ring5_pair_commit_multicast\": %.1f, \"ring5_single\": %.1f}\n",
         run<0, 8>(sms, iters), run<0, 24>(sms, iters), run<1, 8>(sms, iters));
  return 0;
}
