// sm_100a kernels of the hot path:
//   K1  preadd_kernel   : a2  S1=(A21-A11)Y, S2=A22-A21 Y, S3=S1-A22, S4=S3+A12 (mod p) fused with
//                         the centered int8 limb split of every leaf operand (Alg. alg:MIAHMM,
//                         PAPER.md:303-307)
//       split_kernel    : limb split of a plain operand (depth 0, gemm_modp, 2M's X / Y)
//   K2/K3 leaf_kernel   : a4/a5 grouped persistent tcgen05 int8 GEMM / lower-triangle SYRK with
//                         int32 TMEM accumulators and a mod-p limb-recombination epilogue
//                         (P1..P5 of PAPER.md:308-314)
//   K4  combine_kernel  : a6 U1=P1+P5 (+Up(U1)=Low(U1)^T), U2=U1+P4, U4=U2+P3, U5=Low(U2+P4^T),
//                         U3=P1+P2 -> [[U3],[U4,U5]]
//   K5  twom_kernel     : a7 Re = G - eps H - phi(H), Im = H^T - H (Alg. alg:2M)
//       mod_lower_kernel, fill_upper_kernel : split-K finalisation, optional Up(C) = phi(Low(C))
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.hpp"
#include "ptx.cuh"

namespace adj {

// ============================================================================ leaf kernel
template <int BN>
struct LeafCfg {
  static constexpr int STAGES = (BN == 256) ? 4 : 6;
  static constexpr int SLOTS = 512 / BN;            // TMEM accumulator slots of BN columns
  static constexpr int A_BYTES = kBM * kBK;         // 16 KiB
  static constexpr int B_BYTES = BN * kBK;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_BYTES = 8 * (2 * STAGES + 2 * SLOTS) + 16;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + BAR_BYTES;
};

__device__ __forceinline__ void decode_tile(uint32_t packed, int &q, int &I, int &J) {
  q = (int)(packed >> 24);
  I = (int)((packed >> 12) & 0xFFF);
  J = (int)(packed & 0xFFF);
}

// store 32 consecutive residues r[0..31] of output row `row`, columns col..col+31
__device__ __forceinline__ void store_chunk(const LeafProduct &pr, int64_t row, int64_t col,
                                            const uint32_t (&r)[32]) {
  if (row >= pr.out_rows || col >= pr.out_cols) return;
  if (pr.sym && col > row) return;
  const bool full = (col + 32 <= pr.out_cols) && (!pr.sym || col + 31 <= row) && pr.vec_ok;
  if (pr.out_u32) {
    uint32_t *o = reinterpret_cast<uint32_t *>(pr.out) + row * pr.ldo + col;
    if (full) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        reinterpret_cast<uint4 *>(o)[i] = make_uint4(r[4 * i], r[4 * i + 1], r[4 * i + 2], r[4 * i + 3]);
    } else {
#pragma unroll
      for (int e = 0; e < 32; ++e)
        if (col + e < pr.out_cols && (!pr.sym || col + e <= row)) o[e] = r[e];
    }
  } else {
    uint16_t *o = reinterpret_cast<uint16_t *>(pr.out) + row * pr.ldo + col;
    if (full) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint4 v;
        v.x = r[8 * i + 0] | (r[8 * i + 1] << 16);
        v.y = r[8 * i + 2] | (r[8 * i + 3] << 16);
        v.z = r[8 * i + 4] | (r[8 * i + 5] << 16);
        v.w = r[8 * i + 6] | (r[8 * i + 7] << 16);
        reinterpret_cast<uint4 *>(o)[i] = v;
      }
    } else {
#pragma unroll
      for (int e = 0; e < 32; ++e)
        if (col + e < pr.out_cols && (!pr.sym || col + e <= row)) o[e] = (uint16_t)r[e];
    }
  }
}

// Warp roles (256 threads): warp 0 = TMA producer, warp 1 = MMA issuer, warp 2 = TMEM
// allocator, warp 3 idle, warps 4..7 = epilogue (warp w reads TMEM lanes 32(w%4)..+31).
// Work stream per CTA: tiles blockIdx.x, +gridDim.x, ...; per tile NACC accumulators, each a
// full K loop into its own TMEM slot (slot = unit % SLOTS) so that the epilogue of one
// accumulator overlaps the MMAs of the next.
template <int BN, int NACC>
__global__ void __launch_bounds__(256, 1) leaf_kernel(const __grid_constant__ LeafParams P) {
  using Cfg = LeafCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *full_bar = reinterpret_cast<uint64_t *>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t *empty_bar = full_bar + Cfg::STAGES;
  uint64_t *slot_full = empty_bar + Cfg::STAGES;
  uint64_t *slot_empty = slot_full + Cfg::SLOTS;
  uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(slot_empty + Cfg::SLOTS);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < Cfg::SLOTS; ++s) {
      ptx::mbar_init(&slot_full[s], 1);
      ptx::mbar_init(&slot_empty[s], 4);
    }
    ptx::fence_barrier_init();
    for (int i = 0; i < kMaxMaps; ++i) ptx::prefetch_tmap(&P.maps[i]);
  }
  if (warp == 2) ptx::tmem_alloc(tmem_holder, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < P.n_tiles; t += gridDim.x) {
        int q, I, J;
        decode_tile(P.tiles[t], q, I, J);
        const LeafProduct &pr = P.prod[q];
        const CUtensorMap *map = &P.maps[pr.map];
        const int arow = pr.a_row0 + I * kBM;
        const int brow = pr.b_row0 + J * BN;
#pragma unroll 1
        for (int j = 0; j < NACC; ++j) {
#pragma unroll 1
          for (int kb = 0; kb < pr.kblocks; ++kb) {
#pragma unroll 1
            for (int tt = P.acc_begin[j]; tt < P.acc_begin[j + 1]; ++tt) {
              const LeafTerm term = P.terms[tt];
              ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
              ptx::mbar_expect_tx(&full_bar[stage], Cfg::STAGE_BYTES);
              uint8_t *sa = smem + stage * Cfg::STAGE_BYTES;
              uint8_t *sb = sa + Cfg::A_BYTES;
              ptx::tma_load_2d(sa, map, kb * kBK, arow + term.a_plane * pr.a_plane_rows, &full_bar[stage]);
#pragma unroll
              for (int h = 0; h < BN / 128; ++h)
                ptx::tma_load_2d(sb + h * 128 * kBK, map, kb * kBK,
                                 brow + term.b_plane * pr.b_plane_rows + h * 128, &full_bar[stage]);
              if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (one thread)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      uint32_t unit = 0;
      for (int t = blockIdx.x; t < P.n_tiles; t += gridDim.x) {
        int q, I, J;
        decode_tile(P.tiles[t], q, I, J);
        const LeafProduct &pr = P.prod[q];
#pragma unroll 1
        for (int j = 0; j < NACC; ++j, ++unit) {
          const uint32_t slot = unit % Cfg::SLOTS, use = unit / Cfg::SLOTS;
          ptx::mbar_wait(&slot_empty[slot], (use & 1) ^ 1);
          ptx::tc_fence_after();
          const uint32_t d_tmem = tmem_base + slot * BN;
          uint32_t accumulate = 0;
#pragma unroll 1
          for (int kb = 0; kb < pr.kblocks; ++kb) {
#pragma unroll 1
            for (int tt = P.acc_begin[j]; tt < P.acc_begin[j + 1]; ++tt) {
              const LeafTerm term = P.terms[tt];
              const uint32_t idesc = ptx::idesc_i8(kBM, BN, term.a_signed != 0, term.b_signed != 0);
              ptx::mbar_wait(&full_bar[stage], phase);
              ptx::tc_fence_after();
              const uint32_t sa = ptx::smem_u32(smem + stage * Cfg::STAGE_BYTES);
              const uint64_t adesc = ptx::smem_desc_sw128(sa);
              const uint64_t bdesc = ptx::smem_desc_sw128(sa + Cfg::A_BYTES);
#pragma unroll
              for (int kk = 0; kk < kBK / 32; ++kk) {   // UMMA_K = 32 bytes of int8
                ptx::mma_i8(d_tmem, adesc + 2 * kk, bdesc + 2 * kk, idesc, accumulate);
                accumulate = 1;
              }
              ptx::mma_commit(&empty_bar[stage]);     // frees the smem stage when MMAs finish
              if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
            }
          }
          ptx::mma_commit(&slot_full[slot]);          // accumulator ready for the epilogue
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 4;
    const uint32_t lane_off = (uint32_t)(ew * 32) << 16;
    const ModP mod = P.mod;
    uint32_t unit = 0;
    for (int t = blockIdx.x; t < P.n_tiles; t += gridDim.x) {
      int q, I, J;
      decode_tile(P.tiles[t], q, I, J);
      const LeafProduct &pr = P.prod[q];
      const int64_t row = (int64_t)I * kBM + ew * 32 + lane;
      const int64_t col0 = (int64_t)J * BN;
      uint32_t part[NACC > 1 ? BN / 2 : 1];
#pragma unroll
      for (int j = 0; j < NACC; ++j, ++unit) {
        const uint32_t slot = unit % Cfg::SLOTS, use = unit / Cfg::SLOTS;
        ptx::mbar_wait(&slot_full[slot], use & 1);
        ptx::tc_fence_after();
        const uint32_t w = P.weight[j];
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t v[32];
          ptx::tmem_ld32(tmem_base + lane_off + slot * BN + c * 32, v);
          ptx::tmem_wait_ld();
          uint32_t r[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) r[e] = mod_s32((int32_t)v[e], mod);
          if constexpr (NACC == 1) {
            if (w != 1) {
#pragma unroll
              for (int e = 0; e < 32; ++e) r[e] = mulmod(r[e], w, mod);
            }
            store_chunk(pr, row, col0 + c * 32, r);
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e) r[e] = mulmod(r[e], w, mod);
            if (j == 0) {
#pragma unroll
              for (int e = 0; e < 16; ++e) part[c * 16 + e] = r[2 * e] | (r[2 * e + 1] << 16);
            } else {
#pragma unroll
              for (int e = 0; e < 16; ++e) {
                r[2 * e] = addmod(r[2 * e], part[c * 16 + e] & 0xFFFF, mod);
                r[2 * e + 1] = addmod(r[2 * e + 1], part[c * 16 + e] >> 16, mod);
              }
              if (j == NACC - 1) {
                store_chunk(pr, row, col0 + c * 32, r);
              } else {
#pragma unroll
                for (int e = 0; e < 16; ++e) part[c * 16 + e] = r[2 * e] | (r[2 * e + 1] << 16);
              }
            }
          }
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&slot_empty[slot]);
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, 512);
  }
}

template <int BN, int NACC>
static cudaError_t launch_leaf_t(const LeafParams &p, int grid, cudaStream_t s) {
  using Cfg = LeafCfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(leaf_kernel<BN, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  leaf_kernel<BN, NACC><<<grid, 256, Cfg::SMEM, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_leaf(const LeafParams &p, int bn, int nacc, int grid, cudaStream_t s) {
  if (p.n_tiles == 0) return cudaSuccess;
  if (bn == 256 && nacc == 1) return launch_leaf_t<256, 1>(p, grid, s);
  if (bn == 128 && nacc == 3) return launch_leaf_t<128, 3>(p, grid, s);
  if (bn == 128 && nacc == 1) return launch_leaf_t<128, 1>(p, grid, s);
  return cudaErrorInvalidValue;
}

// ============================================================================ leaf kernel, CTA pair
// cta_group::2 version: a cluster of 2 CTAs (one TPC) computes a 256 x 256 tile with
// tcgen05.mma.cta_group::2 M=256 N=256 K=32 (int8).  CTA r holds rows r*128.. of the A tile and
// rows r*128.. of the B tile in its shared memory, and accumulator rows r*128.. in its TMEM.
// Per SM this halves shared-memory traffic versus the 1-CTA M=128 N=128 tile (TMA writes 64 B/clk
// + MMA operand reads 64 B/clk at full tensor rate).  TMEM holds 2 slots of 256 columns; the NACC
// limb accumulators of a tile run one after the other (acc-major), the epilogue folds each into
// a weighted mod-p partial sum kept in registers (8 warps x 128 columns).
struct Leaf2Cfg {
  static constexpr int STAGES = 6;
  static constexpr int TILE = 256;
  static constexpr int A_BYTES = 128 * kBK;
  static constexpr int B_BYTES = 128 * kBK;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SLOTS = 2;
  static constexpr int BAR_BYTES = 8 * (2 * STAGES + 2 * SLOTS) + 16;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + BAR_BYTES;
  static constexpr int THREADS = 384;
};

template <int NACC>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    leaf2_kernel(const __grid_constant__ LeafParams P) {
  using Cfg = Leaf2Cfg;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *full_bar = reinterpret_cast<uint64_t *>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t *empty_bar = full_bar + Cfg::STAGES;
  uint64_t *slot_full = empty_bar + Cfg::STAGES;
  uint64_t *slot_empty = slot_full + Cfg::SLOTS;
  uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(slot_empty + Cfg::SLOTS);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  const int cid = (int)ptx::cluster_id_x();
  const int ncl = (int)ptx::num_clusters_x();

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < Cfg::SLOTS; ++s) {
      ptx::mbar_init(&slot_full[s], 1);
      ptx::mbar_init(&slot_empty[s], 16);   // 8 epilogue warps x 2 CTAs (used in the leader)
    }
    ptx::fence_barrier_init();
    for (int i = 0; i < kMaxMaps; ++i) ptx::prefetch_tmap(&P.maps[i]);
  }
  if (warp == 2) ptx::tmem_alloc_2sm(tmem_holder, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cid; t < P.n_tiles; t += ncl) {
        int q, I, J;
        decode_tile(P.tiles[t], q, I, J);
        const LeafProduct &pr = P.prod[q];
        const CUtensorMap *map = &P.maps[pr.map];
        const int arow = pr.a_row0 + I * Cfg::TILE + (int)rank * 128;
        const int brow = pr.b_row0 + J * Cfg::TILE + (int)rank * 128;
#pragma unroll 1
        for (int j = 0; j < NACC; ++j) {
#pragma unroll 1
          for (int kb = 0; kb < pr.kblocks; ++kb) {
#pragma unroll 1
            for (int tt = P.acc_begin[j]; tt < P.acc_begin[j + 1]; ++tt) {
              const LeafTerm term = P.terms[tt];
              ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
              if (leader) ptx::mbar_expect_tx(&full_bar[stage], 2 * Cfg::STAGE_BYTES);
              uint8_t *sa = smem + stage * Cfg::STAGE_BYTES;
              ptx::tma_load_2d_2sm(sa, map, kb * kBK, arow + term.a_plane * pr.a_plane_rows, &full_bar[stage]);
              ptx::tma_load_2d_2sm(sa + Cfg::A_BYTES, map, kb * kBK, brow + term.b_plane * pr.b_plane_rows,
                                   &full_bar[stage]);
              if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader CTA, one thread)
    if (leader && lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      uint32_t unit = 0;
      for (int t = cid; t < P.n_tiles; t += ncl) {
        int q, I, J;
        decode_tile(P.tiles[t], q, I, J);
        const LeafProduct &pr = P.prod[q];
#pragma unroll 1
        for (int j = 0; j < NACC; ++j, ++unit) {
          const uint32_t slot = unit & 1, use = unit >> 1;
          ptx::mbar_wait_cluster(&slot_empty[slot], (use & 1) ^ 1);
          ptx::tc_fence_after();
          const uint32_t d_tmem = tmem_base + slot * Cfg::TILE;
          uint32_t accumulate = 0;
#pragma unroll 1
          for (int kb = 0; kb < pr.kblocks; ++kb) {
#pragma unroll 1
            for (int tt = P.acc_begin[j]; tt < P.acc_begin[j + 1]; ++tt) {
              const LeafTerm term = P.terms[tt];
              const uint32_t idesc = ptx::idesc_i8(256, 256, term.a_signed != 0, term.b_signed != 0);
              ptx::mbar_wait(&full_bar[stage], phase);
              ptx::tc_fence_after();
              const uint32_t sa = ptx::smem_u32(smem + stage * Cfg::STAGE_BYTES);
              const uint64_t adesc = ptx::smem_desc_sw128(sa);
              const uint64_t bdesc = ptx::smem_desc_sw128(sa + Cfg::A_BYTES);
#pragma unroll
              for (int kk = 0; kk < kBK / 32; ++kk) {
                ptx::mma_i8_2sm(d_tmem, adesc + 2 * kk, bdesc + 2 * kk, idesc, accumulate);
                accumulate = 1;
              }
              ptx::mma_commit_2sm(&empty_bar[stage], 0x3);
              if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
            }
          }
          ptx::mma_commit_2sm(&slot_full[slot], 0x3);
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue (8 warps per CTA)
    const int q4 = warp & 3;               // TMEM lane quadrant this warp may access
    const int h = (warp - 4) >> 2;          // column half of the 256-wide tile
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const ModP mod = P.mod;
    uint32_t unit = 0;
    for (int t = cid; t < P.n_tiles; t += ncl) {
      int q, I, J;
      decode_tile(P.tiles[t], q, I, J);
      const LeafProduct &pr = P.prod[q];
      const int64_t row = (int64_t)I * Cfg::TILE + rank * 128 + q4 * 32 + lane;
      const int64_t col0 = (int64_t)J * Cfg::TILE + h * 128;
      uint32_t part[NACC > 1 ? 64 : 1];
#pragma unroll
      for (int j = 0; j < NACC; ++j, ++unit) {
        const uint32_t slot = unit & 1, use = unit >> 1;
        ptx::mbar_wait(&slot_full[slot], use & 1);
        ptx::tc_fence_after();
        const uint32_t w = P.weight[j];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t v[32];
          ptx::tmem_ld32(tmem_base + lane_off + slot * Cfg::TILE + h * 128 + c * 32, v);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = mod_s32((int32_t)v[e], mod);
          if constexpr (NACC == 1) {
            if (w != 1) {
#pragma unroll
              for (int e = 0; e < 32; ++e) v[e] = mulmod(v[e], w, mod);
            }
            store_chunk(pr, row, col0 + c * 32, v);
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = mulmod(v[e], w, mod);
            if (j == 0) {
#pragma unroll
              for (int e = 0; e < 16; ++e) part[c * 16 + e] = v[2 * e] | (v[2 * e + 1] << 16);
            } else {
#pragma unroll
              for (int e = 0; e < 16; ++e) {
                v[2 * e] = addmod(v[2 * e], part[c * 16 + e] & 0xFFFF, mod);
                v[2 * e + 1] = addmod(v[2 * e + 1], part[c * 16 + e] >> 16, mod);
              }
              if (j == NACC - 1) {
                store_chunk(pr, row, col0 + c * 32, v);
              } else {
#pragma unroll
                for (int e = 0; e < 16; ++e) part[c * 16 + e] = v[2 * e] | (v[2 * e + 1] << 16);
              }
            }
          }
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&slot_empty[slot]), 0));
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_2sm(tmem_base, 512);
  }
}

template <int NACC>
static cudaError_t launch_leaf2_t(const LeafParams &p, int grid, cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(leaf2_kernel<NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Leaf2Cfg::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  leaf2_kernel<NACC><<<grid, Leaf2Cfg::THREADS, Leaf2Cfg::SMEM, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_leaf2(const LeafParams &p, int nacc, int grid, cudaStream_t s) {
  if (p.n_tiles == 0) return cudaSuccess;
  if (grid % 2) return cudaErrorInvalidValue;
  if (nacc == 1) return launch_leaf2_t<1>(p, grid, s);
  if (nacc == 3) return launch_leaf2_t<3>(p, grid, s);
  return cudaErrorInvalidValue;
}

// ============================================================================ input loads
// 4 consecutive logical elements (R, C..C+3) of a view; zero outside the valid region.
__device__ __forceinline__ void load4(const InView &v, int64_t R, int64_t C, const ModP &m,
                                      uint32_t (&x)[4]) {
#pragma unroll
  for (int e = 0; e < 4; ++e) x[e] = 0;
  if (R >= v.rows_valid || C >= v.cols_valid) return;
  const bool all = (C + 3 < v.cols_valid) && v.vec_ok;
  if (v.type == IN_U32) {
    const uint32_t *p = static_cast<const uint32_t *>(v.ptr) + R * v.ld + C;
    if (all) {
      uint4 q = __ldg(reinterpret_cast<const uint4 *>(p));
      x[0] = q.x; x[1] = q.y; x[2] = q.z; x[3] = q.w;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) if (C + e < v.cols_valid) x[e] = __ldg(p + e);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) x[e] = mod_u32(x[e], m);
  } else if (v.type == IN_U16) {
    const uint16_t *p = static_cast<const uint16_t *>(v.ptr) + R * v.ld + C;
    if (all) {
      uint2 q = __ldg(reinterpret_cast<const uint2 *>(p));
      x[0] = q.x & 0xFFFF; x[1] = q.x >> 16; x[2] = q.y & 0xFFFF; x[3] = q.y >> 16;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) if (C + e < v.cols_valid) x[e] = __ldg(p + e);
    }
  } else {
    const uint32_t *p = static_cast<const uint32_t *>(v.ptr) + 2 * (R * v.ld + C);
    uint32_t re[4] = {0, 0, 0, 0}, im[4] = {0, 0, 0, 0};
    if (all) {
      uint4 a = __ldg(reinterpret_cast<const uint4 *>(p));
      uint4 b = __ldg(reinterpret_cast<const uint4 *>(p) + 1);
      re[0] = a.x; im[0] = a.y; re[1] = a.z; im[1] = a.w;
      re[2] = b.x; im[2] = b.y; re[3] = b.z; im[3] = b.w;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (C + e < v.cols_valid) { re[e] = __ldg(p + 2 * e); im[e] = __ldg(p + 2 * e + 1); }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      uint32_t a = mod_u32(re[e], m), b = mod_u32(im[e], m);
      x[e] = v.type == IN_PAIR_SUM ? addmod(a, b, m) : (v.type == IN_PAIR_RE ? a : b);
    }
  }
}

// write the int8 limb planes of 4 residues at (arena row `row` of plane 0, byte column col)
__device__ __forceinline__ void store_limbs4(int8_t *arena, int64_t kpad, int64_t rows_pad,
                                             int64_t row, int64_t col, const uint32_t (&x)[4],
                                             int scheme, int planes, const ModP &m) {
  uint32_t l[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) l[e] = limb_split(x[e], scheme, m);
#pragma unroll
  for (int pl = 0; pl < 3; ++pl) {
    if (pl >= planes) break;
    const int sh = 8 * pl;
    uint32_t w = ((l[0] >> sh) & 0xFF) | (((l[1] >> sh) & 0xFF) << 8) | (((l[2] >> sh) & 0xFF) << 16) |
                 (((l[3] >> sh) & 0xFF) << 24);
    *reinterpret_cast<uint32_t *>(arena + (row + pl * rows_pad) * kpad + col) = w;
  }
}

__device__ __forceinline__ void zero_limbs4(int8_t *arena, int64_t kpad, int64_t rows_pad, int64_t row,
                                            int64_t col, int planes) {
  for (int pl = 0; pl < planes; ++pl)
    *reinterpret_cast<uint32_t *>(arena + (row + pl * rows_pad) * kpad + col) = 0u;
}

// ============================================================================ K1 pre-addition
__device__ __forceinline__ void apply_Y(uint32_t a, uint32_t b, uint32_t &oa, uint32_t &ob,
                                        const PreParams &P) {
  // X Y on the column pair (c, c + kh/2): Y = i I -> (i a, i b);
  // Y = [[ya, yb], [-yb, ya]] (x) I -> [X1 X2] Y = [ya X1 - yb X2, yb X1 + ya X2]
  if (P.ykind == 0) {
    oa = mulmod(P.ya, a, P.mod);
    ob = mulmod(P.ya, b, P.mod);
  } else {
    oa = submod(mulmod(P.ya, a, P.mod), mulmod(P.yb, b, P.mod), P.mod);
    ob = addmod(mulmod(P.yb, a, P.mod), mulmod(P.ya, b, P.mod), P.mod);
  }
}

__global__ void __launch_bounds__(256) preadd_kernel(const __grid_constant__ PreParams P) {
  const PreNode &N = P.nodes[blockIdx.z];
  const int64_t h2 = P.kh / 2;
  const int64_t g_main = h2 / 4;                 // 4-column groups of the first half
  const int64_t g_pad = (P.kpad - P.kh) / 4;     // zero padding columns [kh, kpad)
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= g_main + g_pad) return;
  const ModP &m = P.mod;
  for (int64_t r = blockIdx.y; r < P.rows_pad; r += gridDim.y) {
    if (g >= g_main) {
      const int64_t col = P.kh + (g - g_main) * 4;
      for (int o = 0; o < OUT_N; ++o)
        if (N.op_row[o] >= 0) zero_limbs4(P.arena, P.kpad, P.rows_pad, N.op_row[o] + r, col, P.planes);
      continue;
    }
    const int64_t c = g * 4;
    uint32_t x11a[4], x11b[4], x12a[4], x12b[4], x21a[4], x21b[4], x22a[4], x22b[4];
    InView v = N.in;
    if (r >= P.mh) v.rows_valid = 0;             // rows of the zero padding up to rows_pad
    load4(v, r, c, m, x11a);
    load4(v, r, c + h2, m, x11b);
    load4(v, r, P.kh + c, m, x12a);
    load4(v, r, P.kh + c + h2, m, x12b);
    load4(v, P.mh + r, c, m, x21a);
    load4(v, P.mh + r, c + h2, m, x21b);
    load4(v, P.mh + r, P.kh + c, m, x22a);
    load4(v, P.mh + r, P.kh + c + h2, m, x22b);
    uint32_t s1a[4], s1b[4], s2a[4], s2b[4], s3a[4], s3b[4], s4a[4], s4b[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      uint32_t ta, tb;
      apply_Y(submod(x21a[e], x11a[e], m), submod(x21b[e], x11b[e], m), s1a[e], s1b[e], P);  // S1
      apply_Y(x21a[e], x21b[e], ta, tb, P);                                                 // A21 Y
      s2a[e] = submod(x22a[e], ta, m); s2b[e] = submod(x22b[e], tb, m);                      // S2
      s3a[e] = submod(s1a[e], x22a[e], m); s3b[e] = submod(s1b[e], x22b[e], m);              // S3
      s4a[e] = addmod(s3a[e], x12a[e], m); s4b[e] = addmod(s3b[e], x12b[e], m);              // S4
    }
    const uint32_t(*outs_a[OUT_N])[4] = {&s1a, &s2a, &s4a, &x22a, &x11a, &x12a, &s3a};
    const uint32_t(*outs_b[OUT_N])[4] = {&s1b, &s2b, &s4b, &x22b, &x11b, &x12b, &s3b};
#pragma unroll
    for (int o = 0; o < OUT_N; ++o) {
      if (N.op_row[o] < 0) continue;
      store_limbs4(P.arena, P.kpad, P.rows_pad, N.op_row[o] + r, c, *outs_a[o], P.scheme, P.planes, m);
      store_limbs4(P.arena, P.kpad, P.rows_pad, N.op_row[o] + r, c + h2, *outs_b[o], P.scheme, P.planes, m);
    }
    if (N.s3 != nullptr && r < P.mh) {
      uint16_t *d = N.s3 + r * N.s3_ld;
      uint2 va, vb;
      va.x = s3a[0] | (s3a[1] << 16); va.y = s3a[2] | (s3a[3] << 16);
      vb.x = s3b[0] | (s3b[1] << 16); vb.y = s3b[2] | (s3b[3] << 16);
      *reinterpret_cast<uint2 *>(d + c) = va;
      *reinterpret_cast<uint2 *>(d + c + h2) = vb;
    }
  }
}

cudaError_t launch_preadd(const PreParams &p, cudaStream_t s) {
  if (p.n_nodes == 0) return cudaSuccess;
  const int64_t groups = p.kh / 8 + (p.kpad - p.kh) / 4;
  dim3 block(256);
  dim3 grid((unsigned)((groups + 255) / 256), (unsigned)(p.rows_pad < 65535 ? p.rows_pad : 65535),
            (unsigned)p.n_nodes);
  preadd_kernel<<<grid, block, 0, s>>>(p);
  return cudaGetLastError();
}

// ============================================================================ plain split
__global__ void __launch_bounds__(256) split_kernel(const __grid_constant__ SplitParams P) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= P.kpad / 4) return;
  const int64_t c = g * 4;
  for (int64_t r = blockIdx.y; r < P.rows_pad; r += gridDim.y) {
    uint32_t x[4];
    InView v = P.in;
    if (r >= P.rows) v.rows_valid = 0;
    if (c >= P.cols) v.cols_valid = 0;
    load4(v, r, c, P.mod, x);
    store_limbs4(P.arena, P.kpad, P.rows_pad, P.op_row + r, c, x, P.scheme, P.planes, P.mod);
  }
}

cudaError_t launch_split(const SplitParams &p, cudaStream_t s) {
  dim3 grid((unsigned)((p.kpad / 4 + 255) / 256), (unsigned)(p.rows_pad < 65535 ? p.rows_pad : 65535));
  split_kernel<<<grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

// ============================================================================ K4 recombination
template <typename OutT>
__global__ void __launch_bounds__(256) combine_kernel(const __grid_constant__ CombParams P) {
  const CombNode &N = P.nodes[blockIdx.z];
  const int ti = blockIdx.y, tj = blockIdx.x;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t mh = P.mh, ldp = P.ldp;
  const int64_t i0 = (int64_t)ti * 32, j0 = (int64_t)tj * 32;
  const ModP &m = P.mod;
  const uint16_t *P1 = N.P[0], *P2 = N.P[1], *P3 = N.P[2], *P4 = N.P[3], *P5 = N.P[4];
  __shared__ uint32_t sU[32][33];   // U1 on the mirrored tile (tj, ti)
  __shared__ uint32_t sQ[32][33];   // P4 on the mirrored tile (tj, ti)
  const bool lowtile = ti >= tj, uptile = ti <= tj;
  for (int y = ty; y < 32; y += 8) {
    const int64_t gi = j0 + y, gj = i0 + tx;
    if (gi < mh && gj < mh) {
      if (uptile && gi >= gj) sU[y][tx] = addmod(P1[gi * ldp + gj], P5[gi * ldp + gj], m);
      if (lowtile) sQ[y][tx] = P4[gi * ldp + gj];
    }
  }
  __syncthreads();
  OutT *O = static_cast<OutT *>(N.out);
  const int64_t ov = N.out_valid;
  for (int y = ty; y < 32; y += 8) {
    const int64_t i = i0 + y, j = j0 + tx;
    if (i >= mh || j >= mh) continue;
    const uint32_t p4 = P4[i * ldp + j];
    uint32_t u1;
    if (i >= j) u1 = addmod(P1[i * ldp + j], P5[i * ldp + j], m);   // Low(U1) = Low(P1) + Low(P5)
    else u1 = sU[tx][y];                                             // Up(U1) = Low(U1)^T
    const uint32_t u2 = addmod(u1, p4, m);                           // U2 = U1 + P4
    const uint32_t u4 = addmod(u2, P3[i * ldp + j], m);              // U4 = U2 + P3
    if (mh + i < ov && j < ov) O[(mh + i) * N.ldo + j] = (OutT)u4;   // C21
    if (i >= j) {
      const uint32_t u5 = addmod(u2, sQ[tx][y], m);                  // U5 = Low(U2) + Low(P4^T)
      if (mh + i < ov) O[(mh + i) * N.ldo + mh + j] = (OutT)u5;      // C22
      const uint32_t u3 = addmod(P1[i * ldp + j], P2[i * ldp + j], m);  // U3 = P1 + P2
      if (i < ov) O[i * N.ldo + j] = (OutT)u3;                       // C11
    }
  }
}

cudaError_t launch_combine(const CombParams &p, cudaStream_t s) {
  if (p.n_nodes == 0) return cudaSuccess;
  const unsigned nt = (unsigned)((p.mh + 31) / 32);
  dim3 grid(nt, nt, (unsigned)p.n_nodes), block(32, 8);
  if (p.out_u32) combine_kernel<uint32_t><<<grid, block, 0, s>>>(p);
  else combine_kernel<uint16_t><<<grid, block, 0, s>>>(p);
  return cudaGetLastError();
}

// ============================================================================ K5 2M combine
// Re = G - eps H - phi(H) with eps = i phi(i) = 1, Im: H phi(i) + i phi(H) = i (H^T - H);
// G lower (u16, ldg), H full (u16, ldh); C interleaved (re, im) uint32 pairs, Low only.
__global__ void __launch_bounds__(256) twom_kernel(int64_t m, const uint16_t *G, int64_t ldg,
                                                   const uint16_t *H, int64_t ldh, uint32_t *C,
                                                   int64_t ldc, ModP mod) {
  const int ti = blockIdx.y, tj = blockIdx.x;
  if (ti < tj) return;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t i0 = (int64_t)ti * 32, j0 = (int64_t)tj * 32;
  __shared__ uint32_t sH[32][33];   // H on the mirrored tile
  for (int y = ty; y < 32; y += 8) {
    const int64_t gi = j0 + y, gj = i0 + tx;
    if (gi < m && gj < m) sH[y][tx] = H[gi * ldh + gj];
  }
  __syncthreads();
  for (int y = ty; y < 32; y += 8) {
    const int64_t i = i0 + y, j = j0 + tx;
    if (i >= m || j > i) continue;
    const uint32_t h = H[i * ldh + j], ht = sH[tx][y];   // H(i,j), H(j,i)
    const uint32_t re = submod(submod(G[i * ldg + j], h, mod), ht, mod);
    const uint32_t im = submod(ht, h, mod);
    C[2 * (i * ldc + j)] = re;
    C[2 * (i * ldc + j) + 1] = im;
  }
}

cudaError_t launch_twom(int64_t m, const uint16_t *G, int64_t ldg, const uint16_t *H, int64_t ldh,
                        uint32_t *C, int64_t ldc, const ModP &mod, cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  const unsigned nt = (unsigned)((m + 31) / 32);
  twom_kernel<<<dim3(nt, nt), dim3(32, 8), 0, s>>>(m, G, ldg, H, ldh, C, ldc, mod);
  return cudaGetLastError();
}

// ============================================================================ helpers
// dst[i][j] = src[i][j] mod p on the lower triangle (w = 1: uint32, w = 2: (re, im) pairs)
__global__ void mod_lower_kernel(int64_t row0, int w, const uint32_t *src, int64_t lds, uint32_t *dst,
                                 int64_t ldd, ModP mod) {
  const int64_t i = row0 + blockIdx.y;
  const uint32_t *a = src + i * lds * w;
  uint32_t *b = dst + i * ldd * w;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < (i + 1) * w;
       j += (int64_t)gridDim.x * blockDim.x)
    b[j] = mod_u32(a[j], mod);
}

cudaError_t launch_mod_lower(int64_t m, int w, const uint32_t *src, int64_t lds, uint32_t *dst, int64_t ldd,
                             const ModP &mod, cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  const int64_t per_row = (m * w + 255) / 256;
  for (int64_t r0 = 0; r0 < m; r0 += 65535) {
    const int64_t rows = (m - r0) < 65535 ? (m - r0) : 65535;
    mod_lower_kernel<<<dim3((unsigned)(per_row < 64 ? per_row : 64), (unsigned)rows), 256, 0, s>>>(
        r0, w, src, lds, dst, ldd, mod);
  }
  return cudaGetLastError();
}

// Up(C) = phi(Low(C)) (Lemma lem:uplow): C[j][i] = C[i][j] (conjugated for phi = H), i > j
__global__ void __launch_bounds__(256) fill_upper_kernel(int64_t m, int w, uint32_t *C, int64_t ldc, ModP mod) {
  const int ti = blockIdx.y, tj = blockIdx.x;
  if (ti < tj) return;
  const int tx = threadIdx.x, ty = threadIdx.y;
  __shared__ uint32_t s[32][33][2];
  const int64_t i0 = (int64_t)ti * 32, j0 = (int64_t)tj * 32;
  for (int y = ty; y < 32; y += 8) {
    const int64_t i = i0 + y, j = j0 + tx;
    if (i < m && j < m && j < i) {
      s[y][tx][0] = C[(i * ldc + j) * w];
      s[y][tx][1] = w == 2 ? C[(i * ldc + j) * w + 1] : 0;
    }
  }
  __syncthreads();
  for (int y = ty; y < 32; y += 8) {
    const int64_t r = j0 + y, c = i0 + tx;   // upper element (r, c) = phi(C[c][r])
    if (r < m && c < m && r < c) {
      C[(r * ldc + c) * w] = s[tx][y][0];
      if (w == 2) C[(r * ldc + c) * w + 1] = submod(0, s[tx][y][1], mod);
    }
  }
}

cudaError_t launch_fill_upper(int64_t m, int w, uint32_t *C, int64_t ldc, const ModP &mod, cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  const unsigned nt = (unsigned)((m + 31) / 32);
  fill_upper_kernel<<<dim3(nt, nt), dim3(32, 8), 0, s>>>(m, w, C, ldc, mod);
  return cudaGetLastError();
}

}  // namespace adj
