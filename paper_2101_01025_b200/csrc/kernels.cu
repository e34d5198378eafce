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

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>

#include "kernels.hpp"
#include "ptx.cuh"

namespace adj {

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device): the attribute is
// per device, `done` is a per-kernel bitmask of device ordinals (thread-safe)
template <typename K>
static cudaError_t ensure_smem(K kernel, int bytes, std::atomic<uint64_t> &done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

// ============================================================================ leaf kernel
__device__ __forceinline__ void decode_tile(uint32_t packed, int &q, int &I, int &J) {
  q = (int)(packed >> 24);
  I = (int)((packed >> 12) & 0xFFF);
  J = (int)(packed & 0xFFF);
}

// k-block range, fixup piece and column half of a job (whole tile: [0, kblocks), piece 0,
// nhalf 0; nhalf 1 / 2: columns 0..127 / 128..255 of the tile with an N = 128 MMA)
__device__ __forceinline__ void decode_range(uint32_t y, int kblocks, int &kb0, int &kb1, int &piece, int &nhalf) {
  nhalf = 0;
  if (y == 0 || (y & 0xFFFFFFu) == 0xFFFFFFu) {   // whole tile, or column half (empty range sentinel)
    kb0 = 0; kb1 = kblocks; piece = 0;
    if (y != 0) nhalf = 1 + (int)(y >> 24);
    return;
  }
  kb0 = (int)(y & 0xFFF);
  kb1 = (int)((y >> 12) & 0xFFF);
  piece = (int)(y >> 24);
}

// store 32 consecutive residues r[0..31] of output row `row`, columns col..col+31
__device__ __forceinline__ void store_chunk(const LeafProduct &pr, int64_t row, int64_t col,
                                            const uint32_t (&r)[32], const ModP &m) {
  if (row >= pr.out_rows || col >= pr.out_cols) return;
  if (pr.sym && col > row) return;
  const bool full = (col + 32 <= pr.out_cols) && (!pr.sym || col + 31 <= row) && pr.vec_ok;
  if (pr.out_u32) {
    uint32_t *o = reinterpret_cast<uint32_t *>(pr.out) + row * pr.ldo + col;
    if (pr.axpby) {   // SYRK form: out <- alpha v + beta out_old (scalar path, final output only)
#pragma unroll
      for (int e = 0; e < 32; ++e)
        if (col + e < pr.out_cols && (!pr.sym || col + e <= row))
          o[e] = addmod(mulmod_any(pr.alpha, r[e], m), mulmod_any(pr.beta, mod_u32(o[e], m), m), m);
      return;
    }
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

// ============================================================================ leaf kernel, CTA pair
// cta_group::2 version: a cluster of 2 CTAs (one TPC) computes a 256 x 256 tile with
// tcgen05.mma.cta_group::2 M=256 N=256 K=32 (int8).  CTA r holds rows r*128.. of the A tile and
// rows r*128.. of the B tile in its shared memory, and accumulator rows r*128.. in its TMEM.
// Per SM this halves shared-memory traffic versus the 1-CTA M=128 N=128 tile (TMA writes 64 B/clk
// + MMA operand reads 64 B/clk at full tensor rate).  TMEM holds 2 slots of 256 columns; the NACC
// limb accumulators of a tile run one after the other (acc-major), the epilogue folds each into
// a weighted mod-p partial sum kept in registers (8 warps x 128 columns).
#ifndef ADJ_EPI_WARPS
#define ADJ_EPI_WARPS 8
#endif
template <int NACC, bool PART, bool WIDE = false>
struct Leaf2Cfg {
  static constexpr int STAGES = PART ? (WIDE ? 4 : 5) : 6;
  static constexpr int TILE = 256;
  static constexpr int A_BYTES = 128 * kBK;
  static constexpr int B_BYTES = 128 * kBK;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SLOTS = 2;
  // weighted mod-p partial sums of the limb accumulators: 128 rows x 128 words (u16 pairs)
  // WIDE (p > 2^16): residues < 2^18 packed 24-bit (4 values in 3 words): 192 words + 1 pad per row
  // (non-WIDE: stride 130 words = 65 8-byte granules, so 64-bit accesses of the 32 rows a warp
  //  touches are conflict-free)
  static constexpr int PART_STRIDE = WIDE ? 193 : 130;
  static constexpr int PART_BYTES = PART ? 128 * PART_STRIDE * 4 : 0;
  static constexpr int JQ = 4;   // dynamic job queue depth (job index ring + full / empty barriers)
  static constexpr int BAR_BYTES = 8 * (2 * STAGES + 2 * SLOTS + 2 * JQ) + 16 + 8 * JQ;
  static constexpr int SMEM = STAGES * STAGE_BYTES + PART_BYTES + 1024 + BAR_BYTES;
  static constexpr int EPI_WARPS = ADJ_EPI_WARPS;       // 4, 8 or 16: 1, 2 or 4 warps per TMEM lane quadrant
  static constexpr int THREADS = 32 * (EPI_WARPS + 3);   // + TMEM allocator, MMA issuer, TMA producer
};

// NACC limb accumulators per tile; each may be split into K segments of at most pr.kseg k-blocks
// (int32 bound).  A (accumulator, segment) pair is one TMEM unit; PART = the
// epilogue folds units into the shared-memory partial sum (needed when a tile has > 1 unit).
template <int NACC, bool PART, bool WIDE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(32 * (ADJ_EPI_WARPS + 3), 1)
    leaf2_kernel(const __grid_constant__ LeafParams P) {
  using Cfg = Leaf2Cfg<NACC, PART, WIDE>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment (128B swizzle atoms) by pointer arithmetic on the __shared__ array, so
  // that the compiler keeps the shared state space (LDS/STS, not generic LD/ST)
  uint8_t *smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint32_t *part_s = reinterpret_cast<uint32_t *>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t *full_bar = reinterpret_cast<uint64_t *>(smem + Cfg::STAGES * Cfg::STAGE_BYTES + Cfg::PART_BYTES);
  uint64_t *empty_bar = full_bar + Cfg::STAGES;
  uint64_t *slot_full = empty_bar + Cfg::STAGES;
  uint64_t *slot_empty = slot_full + Cfg::SLOTS;
  uint64_t *jq_full = slot_empty + Cfg::SLOTS;
  uint64_t *jq_empty = jq_full + Cfg::JQ;
  uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(jq_empty + Cfg::JQ);
  uint2 *jq = reinterpret_cast<uint2 *>(tmem_holder + 4);   // job descriptors (P.tiles entries)

  uint64_t g_enter = 0;
  long long c_enter = clock64();
  if (P.debug & (128 | 16384)) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_enter));
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  const int cid = (int)ptx::cluster_id_x();
  const int ncl = (int)ptx::num_clusters_x();

  // warp roles: 0..7 epilogue, 8 TMEM allocator, 9 MMA issuer, 10 TMA producer.  The issue
  // arbiter favours the highest warp id, so the two latency-critical single-thread loops win
  // their sub-partition against the ALU-heavy epilogue warps.
  constexpr int EW = Cfg::EPI_WARPS;
  constexpr int W_ALLOC = EW, W_MMA = EW + 1, W_TMA = EW + 2;
  if (warp == W_TMA && lane == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < Cfg::SLOTS; ++s) {
      ptx::mbar_init(&slot_full[s], 1);
      ptx::mbar_init(&slot_empty[s], 2 * EW);   // epilogue warps x 2 CTAs (used in the leader)
    }
    for (int s = 0; s < Cfg::JQ; ++s) {
      ptx::mbar_init(&jq_full[s], 1);
      // consumers of a job index: leader MMA thread, peer producer, epilogue warps of both CTAs
      ptx::mbar_init(&jq_empty[s], 2 + 2 * EW);
    }
    ptx::fence_barrier_init();
    for (int i = 0; i < kMaxMaps; ++i) {
      ptx::prefetch_tmap(&P.maps[i]);
      ptx::prefetch_tmap(&P.maps_half[i]);
    }
  }
  if (warp == W_ALLOC) ptx::tmem_alloc_2sm(tmem_holder, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  // Job sequence of this cluster.  Static: cid, cid + ncl, ...  Dynamic (P.job_counter): the
  // leader's producer claims job indices with an atomic (two jobs ahead, so neither the atomic
  // nor the descriptor load stalls it), publishes each job descriptor in the job ring of both
  // CTAs (jq, jq_full); every other role reads the same sequence and releases the ring slot in
  // the leader (jq_empty).  Descriptor .x = ~0u ends the sequence.  In-order claiming keeps the
  // 74 concurrent tiles a contiguous window of the rasterised list even when clusters run at
  // different speeds (L2 reuse: measured -14% time at c3 / c4).
  const bool dyn = P.job_counter != nullptr;
  constexpr uint32_t kEnd = 0xFFFFFFFFu;
  auto job_consume = [&](int i, bool remote_release) -> uint2 {   // all roles but the leader producer
    const int s = i & (Cfg::JQ - 1);
    ptx::mbar_wait_cluster(&jq_full[s], (uint32_t)(i / Cfg::JQ) & 1);
    const volatile uint32_t *src = reinterpret_cast<volatile uint32_t *>(&jq[s]);
    const uint2 d = make_uint2(src[0], src[1]);
    const uint32_t e = ptx::smem_u32(&jq_empty[s]);
    if (remote_release) ptx::mbar_arrive_cluster_release(ptx::mapa(e, 0));
    else ptx::mbar_arrive(&jq_empty[s]);
    return d;
  };

  if (warp == W_TMA) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const bool skip_tma = (P.debug & 1) != 0;
      const bool prof = (P.debug & 128) != 0;
      long long t_empty = 0, t_tma = 0, t_begin = clock64();
      uint2 next = (!dyn && cid < P.n_tiles) ? __ldg(&P.tiles[cid]) : make_uint2(0u, 0u);
      int idx2 = 0;
      uint2 d1 = make_uint2(kEnd, 0u);
      if (dyn && leader) {
        const int idx1 = atomicAdd(P.job_counter, 1);
        idx2 = atomicAdd(P.job_counter, 1);
        if (idx1 < P.n_tiles) d1 = __ldg(&P.tiles[idx1]);
      }
      for (int i = 0;; ++i) {
        int t = 0;
        if (!dyn) {
          t = cid + i * ncl;
          if (t >= P.n_tiles) break;
        } else if (leader) {
          const int s = i & (Cfg::JQ - 1);
          ptx::mbar_wait_cluster(&jq_empty[s], ((uint32_t)(i / Cfg::JQ) & 1) ^ 1);
          next = d1;
          jq[s] = next;
          const uint32_t peer = ptx::mapa(ptx::smem_u32(&jq[s]), 1);
          ptx::st_shared_cluster_u32(peer, next.x);
          ptx::st_shared_cluster_u32(peer + 4, next.y);
          ptx::mbar_arrive(&jq_full[s]);
          ptx::mbar_arrive_cluster_release(ptx::mapa(ptx::smem_u32(&jq_full[s]), 1));
          if (next.x == kEnd) break;
          d1 = idx2 < P.n_tiles ? __ldg(&P.tiles[idx2]) : make_uint2(kEnd, 0u);   // used next iteration
          idx2 = atomicAdd(P.job_counter, 1);                                     // claimed for i + 2
        } else {
          next = job_consume(i, true);
          if (next.x == kEnd) break;
        }
        int q, I, J, jb0, jb1, piece, nh;
        decode_tile(next.x, q, I, J);
        const uint32_t range = next.y;
        if (!dyn && t + ncl < P.n_tiles) next = __ldg(&P.tiles[t + ncl]);   // prefetch the next job
        const LeafProduct &pr = P.prod[q];
        const CUtensorMap *map = &P.maps[pr.map];
        const int kseg = pr.kseg;
        decode_range(range, pr.kblocks, jb0, jb1, piece, nh);
        const CUtensorMap *bmap = nh ? &P.maps_half[pr.map] : map;
        const int a_pr = pr.a_plane_rows, b_pr = pr.b_plane_rows;
        const int arow = pr.a_row0 + I * Cfg::TILE + (int)rank * 128;
        // N = 128 half jobs: this CTA's 64 rows of the B column half
        const int brow = nh ? pr.b_row0 + J * Cfg::TILE + (nh - 1) * 128 + (int)rank * 64
                            : pr.b_row0 + J * Cfg::TILE + (int)rank * 128;
        const uint32_t stage_tx = nh ? 2 * (Cfg::A_BYTES + Cfg::B_BYTES / 2) : 2 * Cfg::STAGE_BYTES;
        const int nseg = (jb1 - jb0 + kseg - 1) / kseg;
#pragma unroll 1
        for (int u = 0; u < NACC * nseg; ++u) {
          const int j = u / nseg, kb0 = jb0 + (u % nseg) * kseg;
          const int kb1 = min(jb1, kb0 + kseg);
          // the (at most 2) operand-plane pairs accumulated into accumulator j, hoisted out of the K loop
          const int t0 = P.acc_begin[j], nt = P.acc_begin[j + 1] - t0;
          const int ar0 = arow + P.terms[t0].a_plane * a_pr, br0 = brow + P.terms[t0].b_plane * b_pr;
          const int ar1 = nt > 1 ? arow + P.terms[t0 + 1].a_plane * a_pr : ar0;
          const int br1 = nt > 1 ? brow + P.terms[t0 + 1].b_plane * b_pr : br0;
#pragma unroll 1
          for (int kb = kb0; kb < kb1; ++kb) {
#pragma unroll 1
            for (int tt = 0; tt < nt; ++tt) {
              long long c0 = prof ? clock64() : 0;
              ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
              long long c1 = prof ? clock64() : 0;
              if (prof) t_empty += c1 - c0;
              if (skip_tma) {
                if (leader) ptx::mbar_arrive(&full_bar[stage]);
              } else {
                const bool skip_b = (P.debug & 256) != 0;   // diagnostics: A operand only (L2-bound test)
                if (leader) ptx::mbar_expect_tx(&full_bar[stage], skip_b ? 2 * Cfg::A_BYTES : stage_tx);
                uint8_t *sa = smem + stage * Cfg::STAGE_BYTES;
                ptx::tma_load_2d_2sm(sa, map, kb * kBK, tt ? ar1 : ar0, &full_bar[stage]);
                if (!skip_b) ptx::tma_load_2d_2sm(sa + Cfg::A_BYTES, bmap, kb * kBK, tt ? br1 : br0, &full_bar[stage]);
              }
              if (prof) t_tma += clock64() - c1;
              if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
            }
          }
        }
      }
      if (prof && (cid == 0 || cid == ncl / 2))
        printf("[leaf prof] cluster %d rank %u producer: total %lld cyc, empty-wait %lld, tma-issue %lld\n", cid,
               rank, clock64() - t_begin, t_empty, t_tma);
    }
  } else if (warp == W_MMA) {
    // ------------------------------------------------------------ MMA issuer (leader CTA, one thread)
    if (leader && lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      uint32_t unit = 0;
      const uint32_t smem_base = ptx::smem_u32(smem);
      const bool prof = (P.debug & 128) != 0;
      long long t_full = 0, t_slot = 0, t_issue = 0, t_begin = clock64();
      uint2 next = (!dyn && cid < P.n_tiles) ? __ldg(&P.tiles[cid]) : make_uint2(0u, 0u);
      for (int i = 0;; ++i) {
        int t;
        if (!dyn) {
          t = cid + i * ncl;
          if (t >= P.n_tiles) break;
        } else {
          next = job_consume(i, false);
          if (next.x == kEnd) break;
        }
        int q, I, J, jb0, jb1, piece, nh;
        decode_tile(next.x, q, I, J);
        const uint32_t range = next.y;
        if (!dyn && t + ncl < P.n_tiles) next = __ldg(&P.tiles[t + ncl]);
        const LeafProduct &pr = P.prod[q];
        const int kseg = pr.kseg;
        decode_range(range, pr.kblocks, jb0, jb1, piece, nh);
        const int nseg = (jb1 - jb0 + kseg - 1) / kseg;
        const int mma_n = nh ? 128 : 256;
#pragma unroll 1
        for (int u = 0; u < NACC * nseg; ++u, ++unit) {
          const int j = u / nseg, kb0 = jb0 + (u % nseg) * kseg;
          const int kb1 = min(jb1, kb0 + kseg);
          const int t0 = P.acc_begin[j], nt = P.acc_begin[j + 1] - t0;
          const uint32_t id0 = ptx::idesc_i8(256, mma_n, P.terms[t0].a_signed != 0, P.terms[t0].b_signed != 0);
          const uint32_t id1 = nt > 1 ? ptx::idesc_i8(256, mma_n, P.terms[t0 + 1].a_signed != 0,
                                                      P.terms[t0 + 1].b_signed != 0) : id0;
          const uint32_t slot = unit & 1, use = unit >> 1;
          long long c0 = prof ? clock64() : 0;
          if (!(P.debug & 64)) ptx::mbar_wait_cluster(&slot_empty[slot], (use & 1) ^ 1);   // 64: timing only
          if (prof) t_slot += clock64() - c0;
          ptx::tc_fence_after();
          const uint32_t d_tmem = tmem_base + slot * Cfg::TILE;
          uint32_t accumulate = 0;
#pragma unroll 1
          for (int kb = kb0; kb < kb1; ++kb) {
#pragma unroll 1
            for (int tt = 0; tt < nt; ++tt) {
              long long c1 = prof ? clock64() : 0;
              ptx::mbar_wait(&full_bar[stage], phase);
              long long c2 = prof ? clock64() : 0;
              if (prof) t_full += c2 - c1;
              ptx::tc_fence_after();
              const uint32_t sa = smem_base + stage * Cfg::STAGE_BYTES;
              const uint64_t adesc = ptx::smem_desc_sw128(sa);
              const uint64_t bdesc = ptx::smem_desc_sw128(sa + Cfg::A_BYTES);
              const uint32_t idesc = tt ? id1 : id0;
#pragma unroll
              for (int kk = 0; kk < kBK / 32; ++kk) {
                ptx::mma_i8_2sm(d_tmem, adesc + 2 * kk, bdesc + 2 * kk, idesc, accumulate);
                accumulate = 1;
              }
              ptx::mma_commit_2sm(&empty_bar[stage], 0x3);
              if (prof) t_issue += clock64() - c2;
              if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
            }
          }
          ptx::mma_commit_2sm(&slot_full[slot], 0x3);
        }
      }
      if (prof && (cid == 0 || cid == ncl / 2))
        printf("[leaf prof] cluster %d MMA thread: total %lld cyc, full-wait %lld, slot-wait %lld, issue %lld\n", cid,
               clock64() - t_begin, t_full, t_slot, t_issue);
    }
  } else if (warp < EW) {
    // ------------------------------------------------------------ epilogue (8 warps per CTA)
    const int q4 = warp & 3;               // TMEM lane quadrant this warp may access
    constexpr int CPW = 1024 / EW;             // tile columns per warp (EW / 4 warps per TMEM lane quadrant)
    const int h0 = warp >> 2;                  // which CPW-column part of the 256-wide tile
    constexpr int NCH = CPW / 32;              // 32-column chunks per warp and unit
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const int lrow = q4 * 32 + lane;
    uint32_t *prow0 = part_s + lrow * Cfg::PART_STRIDE;
    const ModP mod = P.mod;
    const int nchunks = (P.debug & 2) ? 0 : NCH;
    const bool dbg_noldtm = (P.debug & 16) != 0, dbg_nomath = (P.debug & 8) != 0, dbg_nostore = (P.debug & 32) != 0;
    const uint32_t empty_remote0 = ptx::mapa(ptx::smem_u32(&slot_empty[0]), 0);
    const uint32_t empty_remote1 = ptx::mapa(ptx::smem_u32(&slot_empty[1]), 0);
    uint32_t unit = 0;
    for (int i = 0;; ++i) {
      uint2 job = make_uint2(0u, 0u);
      if (!dyn) {
        const int t = cid + i * ncl;
        if (t >= P.n_tiles) break;
        job = P.tiles[t];
      } else {
        if (lane == 0) job = job_consume(i, !leader);
        job.x = __shfl_sync(0xFFFFFFFFu, job.x, 0);
        job.y = __shfl_sync(0xFFFFFFFFu, job.y, 0);
        if (job.x == kEnd) break;
      }
      int q, I, J, jb0, jb1, piece, nh;
      decode_tile(job.x, q, I, J);
      const LeafProduct &pr = P.prod[q];
      decode_range(job.y, pr.kblocks, jb0, jb1, piece, nh);
      const int64_t row = (int64_t)I * Cfg::TILE + rank * 128 + lrow;
      // N = 128 half jobs: TMEM columns 0..127 hold output columns (nh-1)*128..; only h0 = 0 warps work
      const int64_t col0 = (int64_t)J * Cfg::TILE + (nh ? (nh - 1) * 128 : 0) + h0 * CPW;
      const int nch = (nh && h0 * CPW >= 128) ? 0 : nchunks;
      // tail piece: residue partial of this CTA's 128 x 256 half-tile into the fixup slot
      const size_t fxo = (size_t)(piece - 1) * 65536 + (rank * 128 + lrow) * 256 + h0 * CPW;
      uint16_t *fx = (piece && !P.fixup32) ? static_cast<uint16_t *>(P.fixup) + fxo : nullptr;
      uint32_t *fx32 = (piece && P.fixup32) ? static_cast<uint32_t *>(P.fixup) + fxo : nullptr;
      const int nseg = (jb1 - jb0 + pr.kseg - 1) / pr.kseg;
      const int nunits = NACC * nseg;
#pragma unroll 1
      for (int u = 0; u < nunits; ++u, ++unit) {
        const int j = u / nseg;
        const uint32_t slot = unit & 1, use = unit >> 1;
        ptx::mbar_wait(&slot_full[slot], use & 1);
        ptx::tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < nch; ++c) {
          uint32_t v[32];
          if (dbg_noldtm) {
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = (uint32_t)(e * 977 + c + u) ^ (uint32_t)lrow;
          } else {
            ptx::tmem_ld32(tmem_base + lane_off + slot * Cfg::TILE + h0 * CPW + c * 32, v);
            ptx::tmem_wait_ld();
          }
          if (dbg_nomath) {
            if (v[0] == 0xFFFFFFFFu && v[31] == 0x12345u) prow0[0] = v[1];   // keep the loads alive
            continue;
          }
          // (partial + acc_j * weight_j) mod p per element, Shoup-fused (modp.cuh: acc_mulred)
          const int32_t wc = P.wshoup[j].wc, wq = P.wshoup[j].wq;
          const uint32_t pm = mod.p;
          if constexpr (PART && !WIDE) {
            uint2 *pc = reinterpret_cast<uint2 *>(prow0 + h0 * (CPW / 2) + c * 16);
            if (u > 0) {
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const uint2 wd = pc[e];
                v[4 * e] = acc_mulred((int32_t)v[4 * e], wc, wq, wd.x & 0xFFFF, pm);
                v[4 * e + 1] = acc_mulred((int32_t)v[4 * e + 1], wc, wq, wd.x >> 16, pm);
                v[4 * e + 2] = acc_mulred((int32_t)v[4 * e + 2], wc, wq, wd.y & 0xFFFF, pm);
                v[4 * e + 3] = acc_mulred((int32_t)v[4 * e + 3], wc, wq, wd.y >> 16, pm);
              }
            } else {
#pragma unroll
              for (int e = 0; e < 32; ++e) v[e] = acc_mulred((int32_t)v[e], wc, wq, 0u, pm);
            }
            if (u < nunits - 1) {
#pragma unroll
              for (int e = 0; e < 8; ++e)
                pc[e] = make_uint2(v[4 * e] | (v[4 * e + 1] << 16), v[4 * e + 2] | (v[4 * e + 3] << 16));
              continue;
            }
          } else if constexpr (PART && WIDE) {
            uint32_t *pc = prow0 + h0 * (CPW * 3 / 4) + c * 24;     // 32 residues of 24 bits = 24 words
            if (u > 0) {
#pragma unroll
              for (int g = 0; g < 8; ++g) {
                const uint32_t w0 = pc[3 * g], w1 = pc[3 * g + 1], w2 = pc[3 * g + 2];
                v[4 * g] = acc_mulred((int32_t)v[4 * g], wc, wq, w0 & 0xFFFFFF, pm);
                v[4 * g + 1] = acc_mulred((int32_t)v[4 * g + 1], wc, wq, (w0 >> 24) | ((w1 & 0xFFFF) << 8), pm);
                v[4 * g + 2] = acc_mulred((int32_t)v[4 * g + 2], wc, wq, (w1 >> 16) | ((w2 & 0xFF) << 16), pm);
                v[4 * g + 3] = acc_mulred((int32_t)v[4 * g + 3], wc, wq, w2 >> 8, pm);
              }
            } else {
#pragma unroll
              for (int e = 0; e < 32; ++e) v[e] = acc_mulred((int32_t)v[e], wc, wq, 0u, pm);
            }
            if (u < nunits - 1) {
#pragma unroll
              for (int g = 0; g < 8; ++g) {
                pc[3 * g] = v[4 * g] | (v[4 * g + 1] << 24);
                pc[3 * g + 1] = (v[4 * g + 1] >> 8) | (v[4 * g + 2] << 16);
                pc[3 * g + 2] = (v[4 * g + 2] >> 16) | (v[4 * g + 3] << 8);
              }
              continue;
            }
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = acc_mulred((int32_t)v[e], wc, wq, 0u, pm);
          }
          if (fx32) {
            uint4 *d = reinterpret_cast<uint4 *>(fx32 + c * 32);
#pragma unroll
            for (int i4 = 0; i4 < 8; ++i4) d[i4] = make_uint4(v[4 * i4], v[4 * i4 + 1], v[4 * i4 + 2], v[4 * i4 + 3]);
          } else if (fx) {
            uint4 *d = reinterpret_cast<uint4 *>(fx + c * 32);
#pragma unroll
            for (int i4 = 0; i4 < 4; ++i4)
              d[i4] = make_uint4(v[8 * i4] | (v[8 * i4 + 1] << 16), v[8 * i4 + 2] | (v[8 * i4 + 3] << 16),
                                 v[8 * i4 + 4] | (v[8 * i4 + 5] << 16), v[8 * i4 + 6] | (v[8 * i4 + 7] << 16));
          } else if (!dbg_nostore) {
            store_chunk(pr, row, col0 + c * 32, v, mod);
          } else if (v[0] == 0xFFFFFFFFu && v[31] == 0x12345u) {
            prow0[0] = v[1];
          }
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(slot ? empty_remote1 : empty_remote0);
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();
  if (warp == W_ALLOC) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_2sm(tmem_base, 512);
  }
  if ((P.debug & (128 | 16384)) && threadIdx.x == 0 && rank == 0) {   // 16384: exit times only
    uint64_t g_exit;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_exit));
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    const long long c_exit = clock64();
    printf("[leaf time] cluster %d sm %u enter %llu exit %llu cycles %lld eff_mhz %.1f\n", cid, smid,
           (unsigned long long)g_enter, (unsigned long long)g_exit, c_exit - c_enter,
           1e3 * (double)(c_exit - c_enter) / (double)(g_exit - g_enter));
  }
}

template <int NACC, bool PART, bool WIDE>
static cudaError_t launch_leaf2_t(const LeafParams &p, int grid, cudaStream_t s) {
  using Cfg = Leaf2Cfg<NACC, PART, WIDE>;
  static std::atomic<uint64_t> done{0};
  cudaError_t e = ensure_smem(leaf2_kernel<NACC, PART, WIDE>, Cfg::SMEM, done);
  if (e != cudaSuccess) return e;
  leaf2_kernel<NACC, PART, WIDE><<<grid, Cfg::THREADS, Cfg::SMEM, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_leaf2(const LeafParams &p, int nacc, bool segmented, int grid, cudaStream_t s) {
  if (p.n_tiles == 0) return cudaSuccess;
  if (grid % 2) return cudaErrorInvalidValue;
  if (nacc == 1)
    return segmented ? launch_leaf2_t<1, true, false>(p, grid, s) : launch_leaf2_t<1, false, false>(p, grid, s);
  if (nacc == 3) return launch_leaf2_t<3, true, false>(p, grid, s);
  if (nacc == 6) return launch_leaf2_t<6, true, true>(p, grid, s);
  return cudaErrorInvalidValue;
}

// ============================================================================ tail fixup
// out(tile) = sum over its K pieces of the residue partials, mod p; same masking as the leaf
// epilogue (store_chunk).  One thread per (row, 32-column chunk) of a 256 x 256 tile.
__global__ void __launch_bounds__(256) fixup_kernel(const __grid_constant__ LeafParams P, const FixupTile *tiles) {
  const FixupTile ft = tiles[blockIdx.y];
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;   // 0 .. 256*8-1
  const int lr = idx >> 3, c = idx & 7;
  const LeafProduct &pr = P.prod[ft.q];
  uint32_t acc[32];
#pragma unroll
  for (int e = 0; e < 32; ++e) acc[e] = 0;
  for (int pc = 0; pc < ft.npieces; ++pc) {
    const size_t off = (size_t)(ft.slot0 + pc) * 65536 + lr * 256 + c * 32;
    if (P.fixup32) {
      const uint4 *src = reinterpret_cast<const uint4 *>(static_cast<const uint32_t *>(P.fixup) + off);
#pragma unroll
      for (int i4 = 0; i4 < 8; ++i4) {
        const uint4 w = src[i4];
        acc[4 * i4] += w.x; acc[4 * i4 + 1] += w.y; acc[4 * i4 + 2] += w.z; acc[4 * i4 + 3] += w.w;
      }
      continue;
    }
    const uint4 *src = reinterpret_cast<const uint4 *>(static_cast<const uint16_t *>(P.fixup) + off);
#pragma unroll
    for (int i4 = 0; i4 < 4; ++i4) {
      const uint4 w = src[i4];
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        acc[8 * i4 + 2 * e] += ws[e] & 0xFFFF;
        acc[8 * i4 + 2 * e + 1] += ws[e] >> 16;
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 32; ++e) acc[e] = mod_u32(acc[e], P.mod);   // < npieces * p < 2^32
  store_chunk(pr, (int64_t)ft.I * 256 + lr, (int64_t)ft.J * 256 + c * 32, acc, P.mod);
}

cudaError_t launch_fixup(const LeafParams &p, const FixupTile *tiles, int n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  fixup_kernel<<<dim3(8, n), 256, 0, s>>>(p, tiles);
  return cudaGetLastError();
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
  } else if (v.type == IN_QUAD_SUM) {
    const uint32_t *p = static_cast<const uint32_t *>(v.ptr) + 4 * (R * v.ld + C);
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (C + e < v.cols_valid) {
        uint4 q = all ? __ldg(reinterpret_cast<const uint4 *>(p) + e)
                      : make_uint4(__ldg(p + 4 * e), __ldg(p + 4 * e + 1), __ldg(p + 4 * e + 2), __ldg(p + 4 * e + 3));
        x[e] = addmod(addmod(mod_u32(q.x, m), mod_u32(q.y, m), m), addmod(mod_u32(q.z, m), mod_u32(q.w, m), m), m);
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

// ============================================================================ K1 pre-addition
// Scheme-specialised limb split of 4 residues into packed int8 plane words (one u32 per plane).
template <int SCHEME>
__device__ __forceinline__ void limbs4(const uint32_t (&x)[4], const ModP &m, uint32_t (&w)[3]) {
  int32_t c[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) c[e] = centered(x[e], m);
  if constexpr (SCHEME == 0) {
    w[0] = __byte_perm(__byte_perm(c[0], c[1], 0x40), __byte_perm(c[2], c[3], 0x40), 0x5410);
  } else if constexpr (SCHEME == 1) {
    int32_t hi[4], lo[4], mid[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      hi[e] = (c[e] + 64) >> 7;
      lo[e] = c[e] - (hi[e] << 7);
      mid[e] = hi[e] + lo[e];
    }
    w[0] = __byte_perm(__byte_perm(hi[0], hi[1], 0x40), __byte_perm(hi[2], hi[3], 0x40), 0x5410);
    w[1] = __byte_perm(__byte_perm(lo[0], lo[1], 0x40), __byte_perm(lo[2], lo[3], 0x40), 0x5410);
    w[2] = __byte_perm(__byte_perm(mid[0], mid[1], 0x40), __byte_perm(mid[2], mid[3], 0x40), 0x5410);
  } else {
    int32_t hi[4], lo[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      hi[e] = c[e] >> 8;
      lo[e] = c[e] - (hi[e] << 8);
    }
    w[0] = __byte_perm(__byte_perm(hi[0], hi[1], 0x40), __byte_perm(hi[2], hi[3], 0x40), 0x5410);
    w[1] = __byte_perm(__byte_perm(lo[0], lo[1], 0x40), __byte_perm(lo[2], lo[3], 0x40), 0x5410);
  }
}

// K7 limbs of 4 already-centered values c in [-(p-1)/2, (p-1)/2]
__device__ __forceinline__ void put_limbs4_k7c(int8_t *base, int64_t plane_stride, const int32_t (&c)[4]) {
  int32_t hi[4], lo[4], mid[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    hi[e] = (c[e] + 64) >> 7;
    lo[e] = c[e] - (hi[e] << 7);
    mid[e] = hi[e] + lo[e];
  }
  *reinterpret_cast<uint32_t *>(base) =
      __byte_perm(__byte_perm(hi[0], hi[1], 0x40), __byte_perm(hi[2], hi[3], 0x40), 0x5410);
  *reinterpret_cast<uint32_t *>(base + plane_stride) =
      __byte_perm(__byte_perm(lo[0], lo[1], 0x40), __byte_perm(lo[2], lo[3], 0x40), 0x5410);
  *reinterpret_cast<uint32_t *>(base + 2 * plane_stride) =
      __byte_perm(__byte_perm(mid[0], mid[1], 0x40), __byte_perm(mid[2], mid[3], 0x40), 0x5410);
}

// centered residue of a signed v with |v| < 2^30, 257 <= p <= 16763: float quotient estimate
// (error < 0.2) then one fix in each direction
__device__ __forceinline__ int32_t center_lazy(int32_t v, float invp, int32_t p, int32_t h) {
  const int32_t q = __float2int_rn(__int2float_rn(v) * invp);
  int32_t r = v - q * p;
  r = r > h ? r - p : r;
  r = r < -h ? r + p : r;
  return r;
}

// wide scheme: three balanced base-64 digits d2, d1, d0 in [-32, 32] of the centered residue
// and the pair sums d2+d1, d1+d0, d2+d0 (6 s8 planes, 3-way Karatsuba)
__device__ __forceinline__ void put_limbs4_t6(int8_t *base, int64_t plane_stride, const uint32_t (&x)[4],
                                              const ModP &m) {
  int32_t d[6][4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int32_t c = centered(x[e], m);
    const int32_t d0 = ((c + 32) & 63) - 32;
    const int32_t c1 = (c - d0) >> 6;
    const int32_t d1 = ((c1 + 32) & 63) - 32;
    const int32_t d2 = (c1 - d1) >> 6;
    d[0][e] = d2; d[1][e] = d1; d[2][e] = d0;
    d[3][e] = d2 + d1; d[4][e] = d1 + d0; d[5][e] = d2 + d0;
  }
#pragma unroll
  for (int pl = 0; pl < 6; ++pl)
    *reinterpret_cast<uint32_t *>(base + pl * plane_stride) =
        __byte_perm(__byte_perm(d[pl][0], d[pl][1], 0x40), __byte_perm(d[pl][2], d[pl][3], 0x40), 0x5410);
}

template <int SCHEME>
__device__ __forceinline__ void put_limbs4(int8_t *base, int64_t plane_stride, const uint32_t (&x)[4],
                                           const ModP &m) {
  if constexpr (SCHEME == 3) {
    put_limbs4_t6(base, plane_stride, x, m);
    return;
  }
  constexpr int NP = SCHEME == 0 ? 1 : (SCHEME == 1 ? 3 : 2);
  uint32_t w[3];
  limbs4<SCHEME>(x, m, w);
#pragma unroll
  for (int pl = 0; pl < NP; ++pl) *reinterpret_cast<uint32_t *>(base + pl * plane_stride) = w[pl];
}

// limb planes of 8 consecutive residues (two 4-groups), one 8-byte store per plane
template <int SCHEME>
__device__ __forceinline__ void put_limbs8(int8_t *base, int64_t plane_stride, const uint32_t (&x0)[4],
                                           const uint32_t (&x1)[4], const ModP &m) {
  if constexpr (SCHEME == 3) {
    put_limbs4_t6(base, plane_stride, x0, m);
    put_limbs4_t6(base + 4, plane_stride, x1, m);
    return;
  }
  constexpr int NP = SCHEME == 0 ? 1 : (SCHEME == 1 ? 3 : 2);
  uint32_t w0[3], w1[3];
  limbs4<SCHEME>(x0, m, w0);
  limbs4<SCHEME>(x1, m, w1);
#pragma unroll
  for (int pl = 0; pl < NP; ++pl) *reinterpret_cast<uint2 *>(base + pl * plane_stride) = make_uint2(w0[pl], w1[pl]);
}

// limb planes of 16 consecutive residues (four 4-groups), one 16-byte store per plane
template <int SCHEME>
__device__ __forceinline__ void put_limbs16(int8_t *base, int64_t plane_stride, const uint32_t (&x)[4][4],
                                            const ModP &m) {
  if constexpr (SCHEME == 3) {
#pragma unroll
    for (int g = 0; g < 4; ++g) put_limbs4_t6(base + 4 * g, plane_stride, x[g], m);
    return;
  }
  constexpr int NP = SCHEME == 0 ? 1 : (SCHEME == 1 ? 3 : 2);
  uint32_t w[4][3];
#pragma unroll
  for (int g = 0; g < 4; ++g) limbs4<SCHEME>(x[g], m, w[g]);
#pragma unroll
  for (int pl = 0; pl < NP; ++pl)
    *reinterpret_cast<uint4 *>(base + pl * plane_stride) = make_uint4(w[0][pl], w[1][pl], w[2][pl], w[3][pl]);
}

template <int YK, bool WIDE = false>
__device__ __forceinline__ void apply_Y4(const uint32_t (&a)[4], const uint32_t (&b)[4], uint32_t (&oa)[4],
                                         uint32_t (&ob)[4], uint32_t ya, uint32_t yb, const ModP &m) {
  if constexpr (WIDE) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if constexpr (YK == 0) {
        oa[e] = mulmod_w(ya, a[e], m);
        ob[e] = mulmod_w(ya, b[e], m);
      } else {
        oa[e] = submod(mulmod_w(ya, a[e], m), mulmod_w(yb, b[e], m), m);
        ob[e] = addmod(mulmod_w(yb, a[e], m), mulmod_w(ya, b[e], m), m);
      }
    }
    return;
  }
  // X Y on the column pair (c, c + kh/2): Y = i I -> (i a, i b);
  // Y = [[ya, yb], [-yb, ya]] (x) I -> [X1 X2] Y = [ya X1 - yb X2, yb X1 + ya X2]
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    if constexpr (YK == 0) {
      oa[e] = mulmod(ya, a[e], m);
      ob[e] = mulmod(ya, b[e], m);
    } else {
      oa[e] = submod(mulmod(ya, a[e], m), mulmod(yb, b[e], m), m);
      ob[e] = addmod(mulmod(yb, a[e], m), mulmod(ya, b[e], m), m);
    }
  }
}

// fast 4-element load of a fully valid, vector-aligned position (type known by the caller)
template <int T>
__device__ __forceinline__ void load4_fast(const void *ptr, int64_t off, const ModP &m, uint32_t (&x)[4]) {
  if constexpr (T == IN_U32) {
    uint4 q = __ldg(reinterpret_cast<const uint4 *>(static_cast<const uint32_t *>(ptr) + off));
    x[0] = mod_u32(q.x, m); x[1] = mod_u32(q.y, m); x[2] = mod_u32(q.z, m); x[3] = mod_u32(q.w, m);
  } else if constexpr (T == IN_U16) {
    uint2 q = __ldg(reinterpret_cast<const uint2 *>(static_cast<const uint16_t *>(ptr) + off));
    x[0] = q.x & 0xFFFF; x[1] = q.x >> 16; x[2] = q.y & 0xFFFF; x[3] = q.y >> 16;
  } else if constexpr (T == IN_QUAD_SUM) {
    const uint4 *p = reinterpret_cast<const uint4 *>(static_cast<const uint32_t *>(ptr) + 4 * off);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint4 q = __ldg(p + e);
      x[e] = addmod(addmod(mod_u32(q.x, m), mod_u32(q.y, m), m), addmod(mod_u32(q.z, m), mod_u32(q.w, m), m), m);
    }
  } else {
    const uint4 *p = reinterpret_cast<const uint4 *>(static_cast<const uint32_t *>(ptr) + 2 * off);
    uint4 a = __ldg(p), b = __ldg(p + 1);
    x[0] = addmod(mod_u32(a.x, m), mod_u32(a.y, m), m);
    x[1] = addmod(mod_u32(a.z, m), mod_u32(a.w, m), m);
    x[2] = addmod(mod_u32(b.x, m), mod_u32(b.y, m), m);
    x[3] = addmod(mod_u32(b.z, m), mod_u32(b.w, m), m);
  }
}

// re / im of 4 consecutive GF(p^2) elements (interleaved pairs), reduced mod p
__device__ __forceinline__ void load4_pair(const InView &v, int64_t R, int64_t C, bool fast, const ModP &m,
                                           uint32_t (&re)[4], uint32_t (&im)[4]) {
  if (fast) {
    const uint4 *p = reinterpret_cast<const uint4 *>(static_cast<const uint32_t *>(v.ptr) + 2 * (R * v.ld + C));
    uint4 a = __ldg(p), b = __ldg(p + 1);
    re[0] = mod_u32(a.x, m); im[0] = mod_u32(a.y, m); re[1] = mod_u32(a.z, m); im[1] = mod_u32(a.w, m);
    re[2] = mod_u32(b.x, m); im[2] = mod_u32(b.y, m); re[3] = mod_u32(b.z, m); im[3] = mod_u32(b.w, m);
  } else {
    InView vr = v, vi = v;
    vr.type = IN_PAIR_RE;
    vi.type = IN_PAIR_IM;
    load4(vr, R, C, m, re);
    load4(vi, R, C, m, im);
  }
}

template <int SCHEME>
__device__ __forceinline__ void put_side(const PreNode &N, int64_t R, int64_t C, const uint32_t (&re)[4],
                                         const uint32_t (&im)[4], const ModP &m) {
  const int64_t ps = N.side_rows_pad * N.side_kpad;
  put_limbs4<SCHEME>(N.side + (N.side_x_row + R) * N.side_kpad + C, ps, re, m);
  put_limbs4<SCHEME>(N.side + (N.side_y_row + R) * N.side_kpad + C, ps, im, m);
}

template <int SCHEME, int YK, int T>
__device__ __forceinline__ void preadd_row(const PreParams &P, const PreNode &N, int64_t r, int64_t c) {
  const ModP &m = P.mod;
  const int64_t h2 = P.kh / 2;
  const InView &v = N.in;
  uint32_t x11a[4], x11b[4], x12a[4], x12b[4], x21a[4], x21b[4], x22a[4], x22b[4];
  const bool top_ok = r < P.mh && r < v.rows_valid;
  const bool bot_ok = r < P.mh && P.mh + r < v.rows_valid;
  const bool fast = v.vec_ok && top_ok && bot_ok && P.kh + c + h2 + 3 < v.cols_valid;
  if (T == IN_PAIR_SUM && N.side != nullptr) {
    // 2M root: T = Re(A) + Im(A) for the pre-addition, and the limb planes of Re(A), Im(A) for H
    InView vv = v;
    if (r >= P.mh) vv.rows_valid = 0;
    const int64_t R[2] = {r, P.mh + r};
    const int64_t Cc[4] = {c, c + h2, P.kh + c, P.kh + c + h2};
    uint32_t(*dst[2][4])[4] = {{&x11a, &x11b, &x12a, &x12b}, {&x21a, &x21b, &x22a, &x22b}};
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        uint32_t re[4], im[4];
        load4_pair(vv, R[a], Cc[b], fast, m, re, im);
        if (r < P.mh) put_side<SCHEME>(N, R[a], Cc[b], re, im, m);
#pragma unroll
        for (int e = 0; e < 4; ++e) (*dst[a][b])[e] = addmod(re[e], im[e], m);
      }
  } else if (fast && T == IN_U32) {
    // all 32 loads first; one check that they are canonical (the usual case) skips the 32
    // Barrett reductions, non-canonical input takes the reducing path (inputs are read mod p)
    const uint32_t *src = static_cast<const uint32_t *>(v.ptr);
    const int64_t o1 = r * v.ld, o2 = (P.mh + r) * v.ld;
    const int64_t offs[8] = {o1 + c, o1 + c + h2, o1 + P.kh + c, o1 + P.kh + c + h2,
                             o2 + c, o2 + c + h2, o2 + P.kh + c, o2 + P.kh + c + h2};
    uint32_t(*dst[8])[4] = {&x11a, &x11b, &x12a, &x12b, &x21a, &x21b, &x22a, &x22b};
    uint4 q[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) q[i] = __ldg(reinterpret_cast<const uint4 *>(src + offs[i]));
    uint32_t mx = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) mx = max(mx, max(max(q[i].x, q[i].y), max(q[i].z, q[i].w)));
    if (mx < m.p) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        (*dst[i])[0] = q[i].x; (*dst[i])[1] = q[i].y; (*dst[i])[2] = q[i].z; (*dst[i])[3] = q[i].w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        (*dst[i])[0] = mod_u32(q[i].x, m); (*dst[i])[1] = mod_u32(q[i].y, m);
        (*dst[i])[2] = mod_u32(q[i].z, m); (*dst[i])[3] = mod_u32(q[i].w, m);
      }
    }
  } else if (fast) {
    const int64_t o1 = r * v.ld, o2 = (P.mh + r) * v.ld;
    load4_fast<T>(v.ptr, o1 + c, m, x11a);
    load4_fast<T>(v.ptr, o1 + c + h2, m, x11b);
    load4_fast<T>(v.ptr, o1 + P.kh + c, m, x12a);
    load4_fast<T>(v.ptr, o1 + P.kh + c + h2, m, x12b);
    load4_fast<T>(v.ptr, o2 + c, m, x21a);
    load4_fast<T>(v.ptr, o2 + c + h2, m, x21b);
    load4_fast<T>(v.ptr, o2 + P.kh + c, m, x22a);
    load4_fast<T>(v.ptr, o2 + P.kh + c + h2, m, x22b);
  } else {
    InView vv = v;
    if (r >= P.mh) vv.rows_valid = 0;             // rows of the zero padding up to rows_pad
    load4(vv, r, c, m, x11a);
    load4(vv, r, c + h2, m, x11b);
    load4(vv, r, P.kh + c, m, x12a);
    load4(vv, r, P.kh + c + h2, m, x12b);
    load4(vv, P.mh + r, c, m, x21a);
    load4(vv, P.mh + r, c + h2, m, x21b);
    load4(vv, P.mh + r, P.kh + c, m, x22a);
    load4(vv, P.mh + r, P.kh + c + h2, m, x22b);
  }
  if constexpr (SCHEME == 1) {
    // Lazy reduction (p <= 16763 so 2 p^2 < 2^31): Y products in raw int32, one centered
    // reduction per S output; X outputs and S3/S4 need one conditional correction each.
    const int32_t p = (int32_t)m.p, h = (int32_t)m.half;
    const float invp = 1.0f / (float)m.p;
    const int32_t ya = (int32_t)P.ya, yb = (int32_t)P.yb;
    int32_t c1a[4], c1b[4], c2a[4], c2b[4], c3a[4], c3b[4], c4a[4], c4b[4];
    int32_t c11a[4], c11b[4], c12a[4], c12b[4], c22a[4], c22b[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int32_t d1 = (int32_t)x21a[e] - (int32_t)x11a[e], d2 = (int32_t)x21b[e] - (int32_t)x11b[e];
      int32_t s1r_a, s1r_b, tr_a, tr_b;
      if constexpr (YK == 0) {
        s1r_a = ya * d1; s1r_b = ya * d2;
        tr_a = ya * (int32_t)x21a[e]; tr_b = ya * (int32_t)x21b[e];
      } else {
        s1r_a = ya * d1 - yb * d2; s1r_b = yb * d1 + ya * d2;                         // (A21 - A11) Y
        tr_a = ya * (int32_t)x21a[e] - yb * (int32_t)x21b[e];                          // A21 Y
        tr_b = yb * (int32_t)x21a[e] + ya * (int32_t)x21b[e];
      }
      c1a[e] = center_lazy(s1r_a, invp, p, h); c1b[e] = center_lazy(s1r_b, invp, p, h);               // S1
      c2a[e] = center_lazy((int32_t)x22a[e] - tr_a, invp, p, h);                                        // S2
      c2b[e] = center_lazy((int32_t)x22b[e] - tr_b, invp, p, h);
      c3a[e] = c1a[e] - (int32_t)x22a[e]; c3a[e] = c3a[e] < -h ? c3a[e] + p : c3a[e];                 // S3
      c3b[e] = c1b[e] - (int32_t)x22b[e]; c3b[e] = c3b[e] < -h ? c3b[e] + p : c3b[e];
      c4a[e] = c3a[e] + (int32_t)x12a[e]; c4a[e] = c4a[e] > h ? c4a[e] - p : c4a[e];                  // S4
      c4b[e] = c3b[e] + (int32_t)x12b[e]; c4b[e] = c4b[e] > h ? c4b[e] - p : c4b[e];
      c11a[e] = (int32_t)x11a[e] > h ? (int32_t)x11a[e] - p : (int32_t)x11a[e];
      c11b[e] = (int32_t)x11b[e] > h ? (int32_t)x11b[e] - p : (int32_t)x11b[e];
      c12a[e] = (int32_t)x12a[e] > h ? (int32_t)x12a[e] - p : (int32_t)x12a[e];
      c12b[e] = (int32_t)x12b[e] > h ? (int32_t)x12b[e] - p : (int32_t)x12b[e];
      c22a[e] = (int32_t)x22a[e] > h ? (int32_t)x22a[e] - p : (int32_t)x22a[e];
      c22b[e] = (int32_t)x22b[e] > h ? (int32_t)x22b[e] - p : (int32_t)x22b[e];
    }
    const int64_t ps = P.rows_pad * P.kpad;
#define PUTC(o, A, B)                                                                  \
  if (N.op_row[o] >= 0) {                                                              \
    int8_t *b = P.arena + (N.op_row[o] + r) * P.kpad;                                  \
    put_limbs4_k7c(b + c, ps, A);                                                      \
    put_limbs4_k7c(b + c + h2, ps, B);                                                 \
  }
    PUTC(OUT_S1, c1a, c1b)
    PUTC(OUT_S2, c2a, c2b)
    PUTC(OUT_S4, c4a, c4b)
    PUTC(OUT_X22, c22a, c22b)
    PUTC(OUT_X11, c11a, c11b)
    PUTC(OUT_X12, c12a, c12b)
    PUTC(OUT_S3, c3a, c3b)
#undef PUTC
    if (N.s3 != nullptr && r < P.mh) {
      uint16_t *d = static_cast<uint16_t *>(N.s3) + r * N.s3_ld;
      uint32_t u[8];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        u[e] = (uint32_t)(c3a[e] < 0 ? c3a[e] + p : c3a[e]);
        u[4 + e] = (uint32_t)(c3b[e] < 0 ? c3b[e] + p : c3b[e]);
      }
      *reinterpret_cast<uint2 *>(d + c) = make_uint2(u[0] | (u[1] << 16), u[2] | (u[3] << 16));
      *reinterpret_cast<uint2 *>(d + c + h2) = make_uint2(u[4] | (u[5] << 16), u[6] | (u[7] << 16));
    }
    return;
  }
  uint32_t da[4], db[4], s1a[4], s1b[4], ta[4], tb[4], s2a[4], s2b[4], s3a[4], s3b[4], s4a[4], s4b[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) { da[e] = submod(x21a[e], x11a[e], m); db[e] = submod(x21b[e], x11b[e], m); }
  apply_Y4<YK, SCHEME == 3>(da, db, s1a, s1b, P.ya, P.yb, m);   // S1 = (A21 - A11) Y
  apply_Y4<YK, SCHEME == 3>(x21a, x21b, ta, tb, P.ya, P.yb, m); // A21 Y
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    s2a[e] = submod(x22a[e], ta[e], m); s2b[e] = submod(x22b[e], tb[e], m);   // S2 = A22 - A21 Y
    s3a[e] = submod(s1a[e], x22a[e], m); s3b[e] = submod(s1b[e], x22b[e], m); // S3 = S1 - A22
    s4a[e] = addmod(s3a[e], x12a[e], m); s4b[e] = addmod(s3b[e], x12b[e], m); // S4 = S3 + A12
  }
  const int64_t ps = P.rows_pad * P.kpad;
#define PUT(o, A, B)                                                                   \
  if (N.op_row[o] >= 0) {                                                              \
    int8_t *b = P.arena + (N.op_row[o] + r) * P.kpad;                                  \
    put_limbs4<SCHEME>(b + c, ps, A, m);                                               \
    put_limbs4<SCHEME>(b + c + h2, ps, B, m);                                          \
  }
  PUT(OUT_S1, s1a, s1b)
  PUT(OUT_S2, s2a, s2b)
  PUT(OUT_S4, s4a, s4b)
  PUT(OUT_X22, x22a, x22b)
  PUT(OUT_X11, x11a, x11b)
  PUT(OUT_X12, x12a, x12b)
  PUT(OUT_S3, s3a, s3b)
#undef PUT
  if (N.s3 != nullptr && r < P.mh && P.res32) {
    uint32_t *d = static_cast<uint32_t *>(N.s3) + r * N.s3_ld;
    *reinterpret_cast<uint4 *>(d + c) = make_uint4(s3a[0], s3a[1], s3a[2], s3a[3]);
    *reinterpret_cast<uint4 *>(d + c + h2) = make_uint4(s3b[0], s3b[1], s3b[2], s3b[3]);
  } else if (N.s3 != nullptr && r < P.mh) {
    uint16_t *d = static_cast<uint16_t *>(N.s3) + r * N.s3_ld;
    uint2 va, vb;
    va.x = s3a[0] | (s3a[1] << 16); va.y = s3a[2] | (s3a[3] << 16);
    vb.x = s3b[0] | (s3b[1] << 16); vb.y = s3b[2] | (s3b[3] << 16);
    *reinterpret_cast<uint2 *>(d + c) = va;
    *reinterpret_cast<uint2 *>(d + c + h2) = vb;
  }
}

template <int SCHEME, int YK>
__global__ void __launch_bounds__(256) preadd_kernel(const __grid_constant__ PreParams P) {
  constexpr int NP = SCHEME == 0 ? 1 : (SCHEME == 1 ? 3 : (SCHEME == 2 ? 2 : 6));
  const PreNode &N = P.nodes[blockIdx.z];
  const int64_t g_main = P.kh / 8;               // 4-column groups of the first half
  const int64_t g_pad = (P.kpad - P.kh) / 4;     // zero padding columns [kh, kpad)
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= g_main + g_pad) return;
  const int type = N.in.type;
  for (int64_t r = blockIdx.y; r < P.rows_pad; r += gridDim.y) {
    if (g >= g_main) {
      const int64_t col = P.kh + (g - g_main) * 4;
#pragma unroll
      for (int o = 0; o < OUT_N; ++o)
        if (N.op_row[o] >= 0)
#pragma unroll
          for (int pl = 0; pl < NP; ++pl)
            *reinterpret_cast<uint32_t *>(P.arena + (N.op_row[o] + r + pl * P.rows_pad) * P.kpad + col) = 0u;
      continue;
    }
    const int64_t c = g * 4;
    if (type == IN_U32) preadd_row<SCHEME, YK, IN_U32>(P, N, r, c);
    else if (type == IN_U16) preadd_row<SCHEME, YK, IN_U16>(P, N, r, c);
    else if (type == IN_QUAD_SUM) preadd_row<SCHEME, YK, IN_QUAD_SUM>(P, N, r, c);
    else preadd_row<SCHEME, YK, IN_PAIR_SUM>(P, N, r, c);
  }
}

cudaError_t launch_preadd(const PreParams &p, cudaStream_t s) {
  if (p.n_nodes == 0) return cudaSuccess;
  const int64_t groups = p.kh / 8 + (p.kpad - p.kh) / 4;
  dim3 block(256);
  dim3 grid((unsigned)((groups + 255) / 256), (unsigned)(p.rows_pad < 65535 ? p.rows_pad : 65535),
            (unsigned)p.n_nodes);
#define PRE(S, Y) preadd_kernel<S, Y><<<grid, block, 0, s>>>(p)
  if (p.scheme == 0) { if (p.ykind == 0) PRE(0, 0); else PRE(0, 1); }
  else if (p.scheme == 1) { if (p.ykind == 0) PRE(1, 0); else PRE(1, 1); }
  else if (p.scheme == 2) { if (p.ykind == 0) PRE(2, 0); else PRE(2, 1); }
  else { if (p.ykind == 0) PRE(3, 0); else PRE(3, 1); }
#undef PRE
  return cudaGetLastError();
}

// ============================================================================ plain split
// One thread per (row, 8 columns): both 4-column groups are loaded before any limb store so
// that each thread keeps 32-64 bytes of loads in flight.
template <int SCHEME>
__global__ void __launch_bounds__(256) split_kernel(const __grid_constant__ SplitParams P) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= P.kpad / 8) return;
  const int64_t c0 = g * 8;
  const int64_t ps = P.rows_pad * P.kpad;
  const InView &v = P.in;
  for (int64_t r = blockIdx.y; r < P.rows_pad; r += gridDim.y) {
    InView vv = v;
    if (r >= P.rows) vv.rows_valid = 0;
    const bool fast = vv.vec_ok && r < vv.rows_valid && c0 + 7 < vv.cols_valid && c0 + 7 < P.cols;
    if (P.mode == 2) {
      // quaternion M = A + B i + C j + D k: the operands of Alg. alg:2M3M
      // A, B, C, D, U1 = A + B, U2 = C + D and (depth 0) W = U1 + U2, from one read of M
      uint32_t q[2][4][4];   // [half][component][element]
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t c = c0 + 4 * h;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          uint4 w4 = make_uint4(0u, 0u, 0u, 0u);
          if (r < vv.rows_valid && c + e < vv.cols_valid && c + e < P.cols) {
            const uint32_t *src = static_cast<const uint32_t *>(v.ptr) + 4 * (r * v.ld + c + e);
            w4 = vv.vec_ok ? __ldg(reinterpret_cast<const uint4 *>(src))
                           : make_uint4(__ldg(src), __ldg(src + 1), __ldg(src + 2), __ldg(src + 3));
          }
          q[h][0][e] = mod_u32(w4.x, P.mod); q[h][1][e] = mod_u32(w4.y, P.mod);
          q[h][2][e] = mod_u32(w4.z, P.mod); q[h][3][e] = mod_u32(w4.w, P.mod);
        }
      }
#pragma unroll
      for (int o = 0; o < 4; ++o)
        put_limbs8<SCHEME>(P.arena + (P.qrow[o] + r) * P.kpad + c0, ps, q[0][o], q[1][o], P.mod);
      uint32_t u1[2][4], u2[2][4];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          u1[h][e] = addmod(q[h][0][e], q[h][1][e], P.mod);
          u2[h][e] = addmod(q[h][2][e], q[h][3][e], P.mod);
        }
      put_limbs8<SCHEME>(P.arena + (P.qrow[4] + r) * P.kpad + c0, ps, u1[0], u1[1], P.mod);
      put_limbs8<SCHEME>(P.arena + (P.qrow[5] + r) * P.kpad + c0, ps, u2[0], u2[1], P.mod);
      if (P.qrow[6] >= 0) {
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int e = 0; e < 4; ++e) u1[h][e] = addmod(u1[h][e], u2[h][e], P.mod);
        put_limbs8<SCHEME>(P.arena + (P.qrow[6] + r) * P.kpad + c0, ps, u1[0], u1[1], P.mod);
      }
      continue;
    }
    if (P.mode == 1) {
      // 2M at depth 0: one read of the interleaved A gives X = Re, Y = Im and T = X + Y
      uint32_t re[2][4], im[2][4];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        InView vh = vv;
        if (c0 + 4 * h >= P.cols) vh.cols_valid = 0;
        load4_pair(vh, r, c0 + 4 * h, fast, P.mod, re[h], im[h]);
      }
      uint32_t x[2][4];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int e = 0; e < 4; ++e) x[h][e] = addmod(re[h][e], im[h][e], P.mod);
      put_limbs8<SCHEME>(P.arena + (P.op_row + r) * P.kpad + c0, ps, re[0], re[1], P.mod);
      put_limbs8<SCHEME>(P.arena + (P.op_row2 + r) * P.kpad + c0, ps, im[0], im[1], P.mod);
      put_limbs8<SCHEME>(P.arena + (P.op_row3 + r) * P.kpad + c0, ps, x[0], x[1], P.mod);
      continue;
    }
    uint32_t x[2][4];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t c = c0 + 4 * h;
      if (fast && v.type == IN_U32) {
        load4_fast<IN_U32>(v.ptr, r * v.ld + c, P.mod, x[h]);
      } else {
        InView vh = vv;
        if (c >= P.cols) vh.cols_valid = 0;
        load4(vh, r, c, P.mod, x[h]);
      }
    }
    put_limbs8<SCHEME>(P.arena + (P.op_row + r) * P.kpad + c0, ps, x[0], x[1], P.mod);
  }
}

// Plain split (mode 0): one thread per (row, 16 columns), four 16-byte loads in flight before
// the 16-byte limb-plane stores.
template <int SCHEME>
__global__ void __launch_bounds__(256) split_plain_kernel(const __grid_constant__ SplitParams P) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= P.kpad / 16) return;
  const int64_t c0 = g * 16;
  const int64_t ps = P.rows_pad * P.kpad;
  const InView &v = P.in;
  for (int64_t r = blockIdx.y; r < P.rows_pad; r += gridDim.y) {
    InView vv = v;
    if (r >= P.rows) vv.rows_valid = 0;
    const bool fast = vv.vec_ok && vv.type == IN_U32 && r < vv.rows_valid && c0 + 15 < vv.cols_valid && c0 + 15 < P.cols;
    uint32_t x[4][4];
    if (fast) {
      uint4 q[4];
#pragma unroll
      for (int h = 0; h < 4; ++h)
        q[h] = __ldg(reinterpret_cast<const uint4 *>(static_cast<const uint32_t *>(v.ptr) + r * v.ld + c0 + 4 * h));
      uint32_t mx = 0;
#pragma unroll
      for (int h = 0; h < 4; ++h) mx = max(mx, max(max(q[h].x, q[h].y), max(q[h].z, q[h].w)));
      if (mx < P.mod.p) {   // canonical input (the usual case) needs no reduction
#pragma unroll
        for (int h = 0; h < 4; ++h) { x[h][0] = q[h].x; x[h][1] = q[h].y; x[h][2] = q[h].z; x[h][3] = q[h].w; }
      } else {
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          x[h][0] = mod_u32(q[h].x, P.mod); x[h][1] = mod_u32(q[h].y, P.mod);
          x[h][2] = mod_u32(q[h].z, P.mod); x[h][3] = mod_u32(q[h].w, P.mod);
        }
      }
    } else {
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        InView vh = vv;
        if (c0 + 4 * h >= P.cols) vh.cols_valid = 0;
        load4(vh, r, c0 + 4 * h, P.mod, x[h]);
      }
    }
    put_limbs16<SCHEME>(P.arena + (P.op_row + r) * P.kpad + c0, ps, x, P.mod);
  }
}

cudaError_t launch_split(const SplitParams &p, cudaStream_t s) {
  if (p.mode == 0) {
    dim3 g16((unsigned)((p.kpad / 16 + 255) / 256), (unsigned)(p.rows_pad < 65535 ? p.rows_pad : 65535));
    if (p.scheme == 0) split_plain_kernel<0><<<g16, 256, 0, s>>>(p);
    else if (p.scheme == 1) split_plain_kernel<1><<<g16, 256, 0, s>>>(p);
    else if (p.scheme == 2) split_plain_kernel<2><<<g16, 256, 0, s>>>(p);
    else split_plain_kernel<3><<<g16, 256, 0, s>>>(p);
    return cudaGetLastError();
  }
  dim3 grid((unsigned)((p.kpad / 8 + 255) / 256), (unsigned)(p.rows_pad < 65535 ? p.rows_pad : 65535));
  if (p.scheme == 0) split_kernel<0><<<grid, 256, 0, s>>>(p);
  else if (p.scheme == 1) split_kernel<1><<<grid, 256, 0, s>>>(p);
  else if (p.scheme == 2) split_kernel<2><<<grid, 256, 0, s>>>(p);
  else split_kernel<3><<<grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

// ============================================================================ K4 recombination
// One block per lower pair {L = (ti, tj), U = (tj, ti)}, ti >= tj, of 64 x 64 tiles of the
// (mh x mh) product grid, so that every product tile is read once:
//   L: U1 = P1 + P5, C21 = U1 + P4 + P3, C22 = Low(U1 + P4 + P4^T), C11 = Low(P1 + P2)
//   U (ti > tj): C21 = Up(U1) + P4 + P3 with Up(U1) = Low(U1)^T
// P4(U) and U1(L) are staged in shared memory for the two transposed uses.  Thread (tx, ty) of
// 8 x 32 owns 8 consecutive columns (16-byte u16 loads) of rows ty and ty + 32.
// SYRK form on the final output: v <- alpha v + beta old (mod p)
__device__ __forceinline__ void axpby_n(const uint32_t *o, int64_t ncols_ok, uint32_t *v, int n, uint32_t alpha,
                                        uint32_t beta, const ModP &m) {
  for (int e = 0; e < n; ++e)
    if (e < ncols_ok) v[e] = addmod(mulmod_any(alpha, v[e], m), mulmod_any(beta, mod_u32(o[e], m), m), m);
}

template <typename OutT>
__device__ __forceinline__ void store8(OutT *o, int64_t ncols_ok, const uint32_t (&v)[8]) {
  if (ncols_ok >= 8 && (reinterpret_cast<uintptr_t>(o) % (8 * sizeof(OutT)) == 0)) {
    if constexpr (sizeof(OutT) == 4) {   // final C: streaming stores (not re-read by this call)
      __stcs(reinterpret_cast<uint4 *>(o), make_uint4(v[0], v[1], v[2], v[3]));
      __stcs(reinterpret_cast<uint4 *>(o) + 1, make_uint4(v[4], v[5], v[6], v[7]));
    } else {
      *reinterpret_cast<uint4 *>(o) = make_uint4(v[0] | (v[1] << 16), v[2] | (v[3] << 16), v[4] | (v[5] << 16),
                                                 v[6] | (v[7] << 16));
    }
  } else {
#pragma unroll
    for (int e = 0; e < 8; ++e) if (e < ncols_ok) o[e] = (OutT)v[e];
  }
}

// 8 residues of a product buffer, kept packed until used (u16: one uint4; u32: two)
template <typename InT> struct Pk8;
template <> struct Pk8<uint16_t> {
  uint4 q;
  __device__ __forceinline__ void load(const uint16_t *p) { q = *reinterpret_cast<const uint4 *>(p); }
  __device__ __forceinline__ void get(uint32_t (&v)[8]) const {
    v[0] = q.x & 0xFFFF; v[1] = q.x >> 16; v[2] = q.y & 0xFFFF; v[3] = q.y >> 16;
    v[4] = q.z & 0xFFFF; v[5] = q.z >> 16; v[6] = q.w & 0xFFFF; v[7] = q.w >> 16;
  }
};
template <> struct Pk8<uint32_t> {
  uint4 q0, q1;
  __device__ __forceinline__ void load(const uint32_t *p) {
    q0 = reinterpret_cast<const uint4 *>(p)[0];
    q1 = reinterpret_cast<const uint4 *>(p)[1];
  }
  __device__ __forceinline__ void get(uint32_t (&v)[8]) const {
    v[0] = q0.x; v[1] = q0.y; v[2] = q0.z; v[3] = q0.w; v[4] = q1.x; v[5] = q1.y; v[6] = q1.z; v[7] = q1.w;
  }
};

template <typename InT, typename OutT>
__global__ void __launch_bounds__(256) combine_kernel(const __grid_constant__ CombParams P) {
  const CombNode &N = P.nodes[blockIdx.y];
  // lower pair index -> (ti, tj), ti >= tj (or the sharded pair list)
  const int x = (int)blockIdx.x;
  int ti, tj;
  if (P.pairs != nullptr) {
    ti = (int)(P.pairs[x] >> 16);
    tj = (int)(P.pairs[x] & 0xFFFF);
  } else {
    ti = (int)((sqrtf(8.0f * (float)x + 1.0f) - 1.0f) * 0.5f);
    while ((ti + 1) * (ti + 2) / 2 <= x) ++ti;
    while (ti * (ti + 1) / 2 > x) --ti;
    tj = x - ti * (ti + 1) / 2;
  }
  const bool diag = ti == tj;
  const int tx = threadIdx.x & 7, ty = threadIdx.x >> 3;   // 8 x 32
  const int64_t mh = P.mh, ldp = P.ldp;                     // ldp multiple of 128 -> aligned 16-byte loads
  const int64_t i0 = (int64_t)ti * 64, j0 = (int64_t)tj * 64;
  const ModP &m = P.mod;
  const InT *P1 = static_cast<const InT *>(N.P[0]), *P2 = static_cast<const InT *>(N.P[1]);
  const InT *P3 = static_cast<const InT *>(N.P[2]), *P4 = static_cast<const InT *>(N.P[3]);
  const InT *P5 = static_cast<const InT *>(N.P[4]);
  __shared__ uint32_t sU[64][65];   // U1 on L (Low part; on a diagonal tile the full tile is filled)
  __shared__ uint32_t sQ[64][65];   // P4 on U (rows j0.., cols i0..)
  const int cx = tx * 8;
  // every load of the block up front (buffers are rows_pad x rows_pad: always in range)
  Pk8<InT> l1[2], l5[2], l2[2], l3[2], l4[2], u4[2], u3[2];
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const int y = ty + 32 * rr;
    const int64_t oL = (i0 + y) * ldp + j0 + cx, oU = (j0 + y) * ldp + i0 + cx;
    l1[rr].load(P1 + oL);
    l5[rr].load(P5 + oL);
    u4[rr].load(P4 + oU);
    l4[rr].load(P4 + oL);
    l3[rr].load(P3 + oL);
    l2[rr].load(P2 + oL);
    if (!diag) u3[rr].load(P3 + oU);
  }
  uint32_t u1[2][8];
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const int y = ty + 32 * rr;
    uint32_t a[8], b[8], q[8];
    l1[rr].get(a);
    l5[rr].get(b);
    u4[rr].get(q);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      u1[rr][e] = addmod(a[e], b[e], m);
      sU[y][cx + e] = u1[rr][e];
      sQ[y][cx + e] = q[e];
    }
  }
  __syncthreads();
  OutT *O = static_cast<OutT *>(N.out);
  const int64_t ov = N.out_valid;
  const bool ax = sizeof(OutT) == 4 && P.axpby;
  // ---- tile L (and, on the diagonal, its upper part of C21)
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const int y = ty + 32 * rr;
    const int64_t i = i0 + y, j = j0 + cx;
    if (i >= mh || j >= mh) continue;
    uint32_t p4[8], p3[8], c21[8], u[8];
    l4[rr].get(p4);
    l3[rr].get(p3);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      u[e] = (j + e <= i) ? u1[rr][e] : sU[cx + e][y];       // Up(U1) = Low(U1)^T (diagonal tile)
      c21[e] = addmod(addmod(u[e], p4[e], m), p3[e], m);      // U4 = U1 + P4 + P3
    }
    const int64_t n21 = min64(8, min64(mh - j, ov - j));
    if (mh + i < ov) {
      if (ax) axpby_n(reinterpret_cast<const uint32_t *>(O + (mh + i) * N.ldo + j), n21, c21, 8, P.alpha, P.beta, m);
      store8<OutT>(O + (mh + i) * N.ldo + j, n21, c21);                                      // C21
    }
    if (j <= i) {
      uint32_t p1[8], p2[8], c22[8], c11[8];
      l1[rr].get(p1);
      l2[rr].get(p2);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        c22[e] = addmod(addmod(u[e], p4[e], m), sQ[cx + e][y], m);   // U5 = U2 + P4^T
        c11[e] = addmod(p1[e], p2[e], m);                            // U3 = P1 + P2
      }
      const int64_t nlow = min64(8, i - j + 1);           // columns j..i only
      if (mh + i < ov) {
        const int64_t n = min64(nlow, ov - mh - j);
        if (ax) axpby_n(reinterpret_cast<const uint32_t *>(O + (mh + i) * N.ldo + mh + j), n, c22, 8, P.alpha, P.beta, m);
        store8<OutT>(O + (mh + i) * N.ldo + mh + j, n, c22);                                // C22
      }
      if (i < ov) {
        const int64_t n = min64(nlow, ov - j);
        if (ax) axpby_n(reinterpret_cast<const uint32_t *>(O + i * N.ldo + j), n, c11, 8, P.alpha, P.beta, m);
        store8<OutT>(O + i * N.ldo + j, n, c11);                                            // C11
      }
    }
  }
  if (diag) return;
  // ---- tile U = (tj, ti): C21 = Up(U1) + P4 + P3 (rows j0.., cols i0..)
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const int y = ty + 32 * rr;
    const int64_t r = j0 + y, c = i0 + cx;
    if (r >= mh || c >= mh) continue;
    uint32_t p3[8], q4[8], c21[8];
    u3[rr].get(p3);
    u4[rr].get(q4);
#pragma unroll
    for (int e = 0; e < 8; ++e) c21[e] = addmod(addmod(sU[cx + e][y], q4[e], m), p3[e], m);
    const int64_t n21 = min64(8, min64(mh - c, ov - c));
    if (mh + r < ov) {
      if (ax) axpby_n(reinterpret_cast<const uint32_t *>(O + (mh + r) * N.ldo + c), n21, c21, 8, P.alpha, P.beta, m);
      store8<OutT>(O + (mh + r) * N.ldo + c, n21, c21);
    }
  }
}

cudaError_t launch_combine(const CombParams &p, cudaStream_t s) {
  if (p.n_nodes == 0) return cudaSuccess;
  const unsigned nt = (unsigned)((p.mh + 63) / 64);
  dim3 grid(p.pairs ? (unsigned)p.n_pairs : nt * (nt + 1) / 2, (unsigned)p.n_nodes), block(256);
  if (grid.x == 0) return cudaSuccess;
  if (p.in32) combine_kernel<uint32_t, uint32_t><<<grid, block, 0, s>>>(p);
  else if (p.out_u32) combine_kernel<uint16_t, uint32_t><<<grid, block, 0, s>>>(p);
  else combine_kernel<uint16_t, uint16_t><<<grid, block, 0, s>>>(p);
  return cudaGetLastError();
}

// ============================================================================ GF(p^2) Alg. 1 (PLAN_HERK1)
// K1 over GF(p^2) with the scalar skew-unitary Y = y I, y = ya + i yb, y conj(y) = -1
// (PAPER.md:750-758): S1 = y (A21 - A11), S2 = A22 - y A21, S3 = S1 - A22, S4 = S3 + A12
// (Alg. alg:MIAHMM), then the 21 real limb operands of the leaves:
//   2M for P1, P2, P5 (T = re + im, X = re, Y = im of A11, A12, S3),
//   3M for P3 = A22 S4^H and P4 = S1 S2^H (re, im and re + im of the left factor, re, im and
//   re - im of the right factor).
// One thread per (row, 4 consecutive columns) of the (mh x kh) quadrants.
template <int SCHEME>
__global__ void __launch_bounds__(256) herk_preadd_kernel(const __grid_constant__ HerkPreParams P) {
  constexpr int NP = SCHEME == 0 ? 1 : (SCHEME == 1 ? 3 : (SCHEME == 2 ? 2 : 6));
  constexpr bool WIDE = SCHEME == 3;
  const int64_t g_main = P.kh / 4;
  const int64_t g_pad = (P.kpad - P.kh) / 4;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= g_main + g_pad) return;
  const ModP &m = P.mod;
  const int64_t ps = P.rows_pad * P.kpad;
  auto out = [&](int o, int64_t r, int64_t c) { return P.arena + ((int64_t)o * P.planes * P.rows_pad + r) * P.kpad + c; };
  for (int64_t r = blockIdx.y; r < P.rows_pad; r += gridDim.y) {
    if (g >= g_main) {
      const int64_t col = P.kh + (g - g_main) * 4;
#pragma unroll 1
      for (int o = 0; o < HO_N; ++o)
#pragma unroll
        for (int pl = 0; pl < NP; ++pl) *reinterpret_cast<uint32_t *>(out(o, r, col) + pl * ps) = 0u;
      continue;
    }
    const int64_t c = g * 4;
    InView v = P.in;
    if (r >= P.mh) v.rows_valid = 0;    // zero padding rows [mh, rows_pad)
    const bool fast = v.vec_ok && r < P.mh && P.mh + r < v.rows_valid && P.kh + c + 3 < v.cols_valid;
    uint32_t a11r[4], a11i[4], a12r[4], a12i[4], a21r[4], a21i[4], a22r[4], a22i[4];
    load4_pair(v, r, c, fast, m, a11r, a11i);
    load4_pair(v, r, P.kh + c, fast, m, a12r, a12i);
    load4_pair(v, P.mh + r, c, fast, m, a21r, a21i);
    load4_pair(v, P.mh + r, P.kh + c, fast, m, a22r, a22i);
    uint32_t dr[4], di[4], s1r[4], s1i[4], tr[4], ti[4], s2r[4], s2i[4], s3r[4], s3i[4], s4r[4], s4i[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) { dr[e] = submod(a21r[e], a11r[e], m); di[e] = submod(a21i[e], a11i[e], m); }
    apply_Y4<1, WIDE>(dr, di, s1r, s1i, P.ya, P.yb, m);        // S1 = y (A21 - A11)
    apply_Y4<1, WIDE>(a21r, a21i, tr, ti, P.ya, P.yb, m);      // y A21
    uint32_t w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      s2r[e] = submod(a22r[e], tr[e], m); s2i[e] = submod(a22i[e], ti[e], m);     // S2 = A22 - y A21
      s3r[e] = submod(s1r[e], a22r[e], m); s3i[e] = submod(s1i[e], a22i[e], m);   // S3 = S1 - A22
      s4r[e] = addmod(s3r[e], a12r[e], m); s4i[e] = addmod(s3i[e], a12i[e], m);   // S4 = S3 + A12
    }
#define HPUT(o, X) put_limbs4<SCHEME>(out(o, r, c), ps, X, m)
#define HSUM(X, Y) for (int e = 0; e < 4; ++e) w[e] = addmod(X[e], Y[e], m)
#define HDIF(X, Y) for (int e = 0; e < 4; ++e) w[e] = submod(X[e], Y[e], m)
    HSUM(a11r, a11i); HPUT(HO_T11, w); HPUT(HO_X11, a11r); HPUT(HO_Y11, a11i);
    HSUM(a12r, a12i); HPUT(HO_T12, w); HPUT(HO_X12, a12r); HPUT(HO_Y12, a12i);
    HSUM(s3r, s3i);   HPUT(HO_T3, w);  HPUT(HO_X3, s3r);   HPUT(HO_Y3, s3i);
    HSUM(a22r, a22i); HPUT(HO_Z22, w); HPUT(HO_X22, a22r); HPUT(HO_Y22, a22i);
    HDIF(s4r, s4i);   HPUT(HO_W4, w);  HPUT(HO_X4, s4r);   HPUT(HO_Y4, s4i);
    HSUM(s1r, s1i);   HPUT(HO_Z1, w);  HPUT(HO_X1, s1r);   HPUT(HO_Y1, s1i);
    HDIF(s2r, s2i);   HPUT(HO_W2, w);  HPUT(HO_X2, s2r);   HPUT(HO_Y2, s2i);
#undef HPUT
#undef HSUM
#undef HDIF
  }
}

cudaError_t launch_herk_preadd(const HerkPreParams &p, cudaStream_t s) {
  const int64_t groups = p.kh / 4 + (p.kpad - p.kh) / 4;
  dim3 grid((unsigned)((groups + 255) / 256), (unsigned)(p.rows_pad < 65535 ? p.rows_pad : 65535));
  if (p.scheme == 0) herk_preadd_kernel<0><<<grid, 256, 0, s>>>(p);
  else if (p.scheme == 1) herk_preadd_kernel<1><<<grid, 256, 0, s>>>(p);
  else if (p.scheme == 2) herk_preadd_kernel<2><<<grid, 256, 0, s>>>(p);
  else herk_preadd_kernel<3><<<grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

// 8 consecutive complex results (re, im) of C row `o` (interleaved pairs), n <= 8 valid
__device__ __forceinline__ void store_c8(uint32_t *o, int64_t n, uint32_t (&re)[8], uint32_t (&im)[8],
                                         const HerkCombParams &P) {
  if (n <= 0) return;
  if (P.axpby) {
    for (int e = 0; e < n; ++e) {
      re[e] = addmod(mulmod_any(P.alpha, re[e], P.mod), mulmod_any(P.beta, mod_u32(o[2 * e], P.mod), P.mod), P.mod);
      im[e] = addmod(mulmod_any(P.alpha, im[e], P.mod), mulmod_any(P.beta, mod_u32(o[2 * e + 1], P.mod), P.mod), P.mod);
    }
  }
  if (n == 8 && (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
#pragma unroll
    for (int e = 0; e < 4; ++e)
      reinterpret_cast<uint4 *>(o)[e] = make_uint4(re[2 * e], im[2 * e], re[2 * e + 1], im[2 * e + 1]);
  } else {
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (e < n) { o[2 * e] = re[e]; o[2 * e + 1] = im[e]; }
  }
}

// K4 over GF(p^2) (PAPER.md:315-323 with phi = conjugate transpose), fused with the leaf
// combinations: P1, P2, P5 = (G - H - H^T) + i (H^T - H) (2M) and
// P3, P4 = (t1 + t2) + i (t3 - t1 + t2) (3M).  One block per lower pair {L = (ti, tj),
// U = (tj, ti)} of 64 x 64 tiles:
//   phase 1: U1 = P1 + P5 and U3 = P1 + P2 on L (only the sums H1 + H5, H1 + H2 are needed
//            transposed), C11 = Low(U3);
//   phase 2: P3, P4 on L and U; C21 = U1 + P4 + P3 on L and U (Up(U1) = conj(Low(U1))^T),
//            C22 = Low(U1 + P4 + conj(P4)^T).
// Dynamic shared memory: 4 tiles of 64 x 65 words.
template <typename InT>
__global__ void __launch_bounds__(256, 2) herk_combine_kernel(const __grid_constant__ HerkCombParams P) {
  extern __shared__ uint32_t hsm[];
  uint32_t(*S0)[65] = reinterpret_cast<uint32_t(*)[65]>(hsm);
  uint32_t(*S1)[65] = reinterpret_cast<uint32_t(*)[65]>(hsm + 64 * 65);
  uint32_t(*S2)[65] = reinterpret_cast<uint32_t(*)[65]>(hsm + 2 * 64 * 65);
  uint32_t(*S3)[65] = reinterpret_cast<uint32_t(*)[65]>(hsm + 3 * 64 * 65);
  const int x = (int)blockIdx.x;
  int ti = (int)((sqrtf(8.0f * (float)x + 1.0f) - 1.0f) * 0.5f);
  while ((ti + 1) * (ti + 2) / 2 <= x) ++ti;
  while (ti * (ti + 1) / 2 > x) --ti;
  const int tj = x - ti * (ti + 1) / 2;
  const bool diag = ti == tj;
  const int tx = threadIdx.x & 7, ty = threadIdx.x >> 3;
  const int64_t mh = P.mh, ldp = P.ldp, ov = P.out_valid;
  const int64_t i0 = (int64_t)ti * 64, j0 = (int64_t)tj * 64;
  const int cx = tx * 8;
  const ModP &m = P.mod;
  auto buf = [&](int b) { return static_cast<const InT *>(P.B[b]); };
  // ---------------- phase 1: U1, U3 on L (U1 kept in S0 / S1 for the rest of the block)
  {
    Pk8<InT> g1[2], g5[2], g2[2], h1[2], h5[2], h2[2], h1u[2], h5u[2], h2u[2];
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int y = ty + 32 * rr;
      const int64_t oL = (i0 + y) * ldp + j0 + cx, oU = (j0 + y) * ldp + i0 + cx;
      h1u[rr].load(buf(HB_H1) + oU); h5u[rr].load(buf(HB_H5) + oU); h2u[rr].load(buf(HB_H2) + oU);
      g1[rr].load(buf(HB_G1) + oL); g5[rr].load(buf(HB_G5) + oL); g2[rr].load(buf(HB_G2) + oL);
      h1[rr].load(buf(HB_H1) + oL); h5[rr].load(buf(HB_H5) + oL); h2[rr].load(buf(HB_H2) + oL);
    }
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int y = ty + 32 * rr;
      uint32_t a[8], b[8], c[8];
      h1u[rr].get(a); h5u[rr].get(b); h2u[rr].get(c);
#pragma unroll
      for (int e = 0; e < 8; ++e) { S0[y][cx + e] = addmod(a[e], b[e], m); S1[y][cx + e] = addmod(a[e], c[e], m); }
    }
    __syncthreads();
    uint32_t u1r[2][8], u1i[2][8];
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int y = ty + 32 * rr;
      const int64_t i = i0 + y, j = j0 + cx;
      uint32_t G1[8], G5[8], G2[8], H1[8], H5[8], H2[8], c11r[8], c11i[8];
      g1[rr].get(G1); g5[rr].get(G5); g2[rr].get(G2); h1[rr].get(H1); h5[rr].get(H5); h2[rr].get(H2);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const uint32_t t15 = S0[cx + e][y], t12 = S1[cx + e][y];     // (H1 + H5)(j, i), (H1 + H2)(j, i)
        const uint32_t h15 = addmod(H1[e], H5[e], m), h12 = addmod(H1[e], H2[e], m);
        u1r[rr][e] = submod(submod(addmod(G1[e], G5[e], m), h15, m), t15, m);   // Re U1 = G1 + G5 - H15 - H15^T
        u1i[rr][e] = submod(t15, h15, m);                                         // Im U1 = H15^T - H15
        c11r[e] = submod(submod(addmod(G1[e], G2[e], m), h12, m), t12, m);      // U3 = P1 + P2
        c11i[e] = submod(t12, h12, m);
      }
      if (i < mh && j <= i && i < ov) store_c8(P.C + 2 * (i * P.ldc + j), min64(8, min64(i - j + 1, ov - j)), c11r, c11i, P);
    }
    __syncthreads();
#pragma unroll
    for (int rr = 0; rr < 2; ++rr)
#pragma unroll
      for (int e = 0; e < 8; ++e) { S0[ty + 32 * rr][cx + e] = u1r[rr][e]; S1[ty + 32 * rr][cx + e] = u1i[rr][e]; }
  }
  // ---------------- phase 2a: P4 on U -> S2 / S3
  {
    Pk8<InT> b1u[2], b2u[2], b3u[2];
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int64_t oU = (j0 + ty + 32 * rr) * ldp + i0 + cx;
      b1u[rr].load(buf(HB_B1) + oU); b2u[rr].load(buf(HB_B2) + oU); b3u[rr].load(buf(HB_B3) + oU);
    }
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int y = ty + 32 * rr;
      uint32_t t1[8], t2[8], t3[8];
      b1u[rr].get(t1); b2u[rr].get(t2); b3u[rr].get(t3);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        S2[y][cx + e] = addmod(t1[e], t2[e], m);                             // Re P4 = t1 + t2
        S3[y][cx + e] = addmod(submod(t3[e], t1[e], m), t2[e], m);           // Im P4 = t3 - t1 + t2
      }
    }
  }
  __syncthreads();
  // ---------------- phase 2b: tile L
  {
    Pk8<InT> a1[2], a2[2], a3[2], b1[2], b2[2], b3[2];
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int64_t oL = (i0 + ty + 32 * rr) * ldp + j0 + cx;
      b1[rr].load(buf(HB_B1) + oL); b2[rr].load(buf(HB_B2) + oL); b3[rr].load(buf(HB_B3) + oL);
      a1[rr].load(buf(HB_A1) + oL); a2[rr].load(buf(HB_A2) + oL); a3[rr].load(buf(HB_A3) + oL);
    }
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int y = ty + 32 * rr;
      const int64_t i = i0 + y, j = j0 + cx;
      if (i >= mh || j >= mh || mh + i >= ov) continue;
      uint32_t t1[8], t2[8], t3[8], q1[8], q2[8], q3[8], cr[8], ci[8], dr[8], di[8];
      b1[rr].get(t1); b2[rr].get(t2); b3[rr].get(t3);
      a1[rr].get(q1); a2[rr].get(q2); a3[rr].get(q3);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const bool low = j + e <= i;
        const uint32_t ur = low ? S0[y][cx + e] : S0[cx + e][y];                    // Up(U1) = conj(Low(U1))^T
        const uint32_t ui = low ? S1[y][cx + e] : submod(0u, S1[cx + e][y], m);
        const uint32_t p4r = addmod(t1[e], t2[e], m), p4i = addmod(submod(t3[e], t1[e], m), t2[e], m);
        const uint32_t p3r = addmod(q1[e], q2[e], m), p3i = addmod(submod(q3[e], q1[e], m), q2[e], m);
        const uint32_t u2r = addmod(ur, p4r, m), u2i = addmod(ui, p4i, m);           // U2 = U1 + P4
        cr[e] = addmod(u2r, p3r, m); ci[e] = addmod(u2i, p3i, m);                     // U4 = U2 + P3
        dr[e] = addmod(u2r, S2[cx + e][y], m);                                       // U5 = U2 + conj(P4)^T
        di[e] = submod(u2i, S3[cx + e][y], m);
      }
      store_c8(P.C + 2 * ((mh + i) * P.ldc + j), min64(8, mh - j), cr, ci, P);                          // C21
      if (j <= i) store_c8(P.C + 2 * ((mh + i) * P.ldc + mh + j), min64(8, min64(i - j + 1, ov - mh - j)), dr, di, P);  // C22
    }
  }
  if (diag) return;
  // ---------------- phase 2c: tile U = (tj, ti): rows j0.., cols i0..
  {
    Pk8<InT> a1u[2], a2u[2], a3u[2];
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int64_t oU = (j0 + ty + 32 * rr) * ldp + i0 + cx;
      a1u[rr].load(buf(HB_A1) + oU); a2u[rr].load(buf(HB_A2) + oU); a3u[rr].load(buf(HB_A3) + oU);
    }
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int y = ty + 32 * rr;
      const int64_t r = j0 + y, c = i0 + cx;
      if (r >= mh || c >= mh || mh + r >= ov) continue;
      uint32_t q1[8], q2[8], q3[8], cr[8], ci[8];
      a1u[rr].get(q1); a2u[rr].get(q2); a3u[rr].get(q3);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const uint32_t ur = S0[cx + e][y], ui = submod(0u, S1[cx + e][y], m);       // conj(U1(c, r))
        const uint32_t p3r = addmod(q1[e], q2[e], m), p3i = addmod(submod(q3[e], q1[e], m), q2[e], m);
        cr[e] = addmod(addmod(ur, S2[y][cx + e], m), p3r, m);
        ci[e] = addmod(addmod(ui, S3[y][cx + e], m), p3i, m);
      }
      store_c8(P.C + 2 * ((mh + r) * P.ldc + c), min64(8, mh - c), cr, ci, P);
    }
  }
}

cudaError_t launch_herk_combine(const HerkCombParams &p, cudaStream_t s) {
  if (p.mh == 0) return cudaSuccess;
  const unsigned nt = (unsigned)((p.mh + 63) / 64);
  const dim3 grid(nt * (nt + 1) / 2);
  const int smem = 4 * 64 * 65 * 4;
  if (p.in32) {
    static std::atomic<uint64_t> set32{0};
    cudaError_t e = ensure_smem(herk_combine_kernel<uint32_t>, smem, set32);
    if (e != cudaSuccess) return e;
    herk_combine_kernel<uint32_t><<<grid, 256, smem, s>>>(p);
  } else {
    static std::atomic<uint64_t> set16{0};
    cudaError_t e = ensure_smem(herk_combine_kernel<uint16_t>, smem, set16);
    if (e != cudaSuccess) return e;
    herk_combine_kernel<uint16_t><<<grid, 256, smem, s>>>(p);
  }
  return cudaGetLastError();
}

// ============================================================================ quaternion 6M combine
// Alg. alg:2M3M: T1 = Q1 - Q2, T2 = Q4 + Q5, T3 = (Q1 + Q2) - Q3,
//   Low(H1) = Low(Q6 - (Q3^T + Q3) - (T2^T + T2)), Low(H2) = Low(T2^T - T2),
//   Low(H3) = Low(T1 - T1^T), Low(H4) = Low(T3^T - T3);  C = H1 + H2 i + H3 j + H4 k.
// One block per lower 64 x 64 tile L = (ti, tj); Q3, T1, T2, T3 of the mirrored tile U = (tj, ti)
// are staged in shared memory (4 tiles of 64 x 65 words, dynamic) for the transposed terms.
__device__ __forceinline__ void store_q8(uint32_t *o, int64_t n, uint32_t (&h)[4][8], const QuatCombParams &P) {
  if (n <= 0) return;
  if (P.axpby) {
    for (int e = 0; e < n; ++e)
#pragma unroll
      for (int c = 0; c < 4; ++c)
        h[c][e] = addmod(mulmod_any(P.alpha, h[c][e], P.mod), mulmod_any(P.beta, mod_u32(o[4 * e + c], P.mod), P.mod), P.mod);
  }
  if (n == 8 && (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
#pragma unroll
    for (int e = 0; e < 8; ++e) reinterpret_cast<uint4 *>(o)[e] = make_uint4(h[0][e], h[1][e], h[2][e], h[3][e]);
  } else {
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (e < n)
#pragma unroll
        for (int c = 0; c < 4; ++c) o[4 * e + c] = h[c][e];
  }
}

template <typename InT>
__global__ void __launch_bounds__(256) quat_combine_kernel(const __grid_constant__ QuatCombParams P) {
  extern __shared__ uint32_t qsm[];
  uint32_t(*S3q)[65] = reinterpret_cast<uint32_t(*)[65]>(qsm);                 // Q3 on U
  uint32_t(*S1t)[65] = reinterpret_cast<uint32_t(*)[65]>(qsm + 64 * 65);       // T1 on U
  uint32_t(*S2t)[65] = reinterpret_cast<uint32_t(*)[65]>(qsm + 2 * 64 * 65);   // T2 on U
  uint32_t(*S3t)[65] = reinterpret_cast<uint32_t(*)[65]>(qsm + 3 * 64 * 65);   // T3 on U
  const int x = (int)blockIdx.x;
  int ti = (int)((sqrtf(8.0f * (float)x + 1.0f) - 1.0f) * 0.5f);
  while ((ti + 1) * (ti + 2) / 2 <= x) ++ti;
  while (ti * (ti + 1) / 2 > x) --ti;
  const int tj = x - ti * (ti + 1) / 2;
  const int tx = threadIdx.x & 7, ty = threadIdx.x >> 3;
  const int64_t m = P.m, ldq = P.ldq;
  const int64_t i0 = (int64_t)ti * 64, j0 = (int64_t)tj * 64;
  const int cx = tx * 8;
  const ModP &md = P.mod;
  auto buf = [&](int b) { return static_cast<const InT *>(P.Q[b]); };
  {
    Pk8<InT> q1[2], q2[2], q3[2], q4[2], q5[2];
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int64_t oU = (j0 + ty + 32 * rr) * ldq + i0 + cx;
      q1[rr].load(buf(0) + oU); q2[rr].load(buf(1) + oU); q3[rr].load(buf(2) + oU);
      q4[rr].load(buf(3) + oU); q5[rr].load(buf(4) + oU);
    }
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int y = ty + 32 * rr;
      uint32_t a1[8], a2[8], a3[8], a4[8], a5[8];
      q1[rr].get(a1); q2[rr].get(a2); q3[rr].get(a3); q4[rr].get(a4); q5[rr].get(a5);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        S3q[y][cx + e] = a3[e];
        S1t[y][cx + e] = submod(a1[e], a2[e], md);                       // T1 = Q1 - Q2
        S2t[y][cx + e] = addmod(a4[e], a5[e], md);                       // T2 = Q4 + Q5
        S3t[y][cx + e] = submod(addmod(a1[e], a2[e], md), a3[e], md);    // T3 = Q1 + Q2 - Q3
      }
    }
  }
  Pk8<InT> q1[2], q2[2], q3[2], q4[2], q5[2], q6[2];
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const int64_t oL = (i0 + ty + 32 * rr) * ldq + j0 + cx;
    q1[rr].load(buf(0) + oL); q2[rr].load(buf(1) + oL); q3[rr].load(buf(2) + oL);
    q4[rr].load(buf(3) + oL); q5[rr].load(buf(4) + oL); q6[rr].load(buf(5) + oL);
  }
  __syncthreads();
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const int y = ty + 32 * rr;
    const int64_t i = i0 + y, j = j0 + cx;
    if (i >= m || j > i) continue;
    uint32_t a1[8], a2[8], a3[8], a4[8], a5[8], a6[8], h[4][8];
    q1[rr].get(a1); q2[rr].get(a2); q3[rr].get(a3); q4[rr].get(a4); q5[rr].get(a5); q6[rr].get(a6);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const uint32_t t1 = submod(a1[e], a2[e], md), t2 = addmod(a4[e], a5[e], md);
      const uint32_t t3 = submod(addmod(a1[e], a2[e], md), a3[e], md);
      const uint32_t q3t = S3q[cx + e][y], t1t = S1t[cx + e][y], t2t = S2t[cx + e][y], t3t = S3t[cx + e][y];
      h[0][e] = submod(submod(a6[e], addmod(q3t, a3[e], md), md), addmod(t2t, t2, md), md);  // H1
      h[1][e] = submod(t2t, t2, md);                                                       // H2
      h[2][e] = submod(t1, t1t, md);                                                       // H3
      h[3][e] = submod(t3t, t3, md);                                                       // H4
    }
    store_q8(P.C + 4 * (i * P.ldc + j), min64(8, min64(i - j + 1, m - j)), h, P);
  }
}

cudaError_t launch_quat_combine(const QuatCombParams &p, cudaStream_t s) {
  if (p.m == 0) return cudaSuccess;
  const unsigned nt = (unsigned)((p.m + 63) / 64);
  const dim3 grid(nt * (nt + 1) / 2);
  const int smem = 4 * 64 * 65 * 4;
  if (p.in32) {
    static std::atomic<uint64_t> set32{0};
    cudaError_t e = ensure_smem(quat_combine_kernel<uint32_t>, smem, set32);
    if (e != cudaSuccess) return e;
    quat_combine_kernel<uint32_t><<<grid, 256, smem, s>>>(p);
  } else {
    static std::atomic<uint64_t> set16{0};
    cudaError_t e = ensure_smem(quat_combine_kernel<uint16_t>, smem, set16);
    if (e != cudaSuccess) return e;
    quat_combine_kernel<uint16_t><<<grid, 256, smem, s>>>(p);
  }
  return cudaGetLastError();
}

// ============================================================================ K5 2M combine
// Re = G - eps H - phi(H) with eps = i phi(i) = 1, Im: H phi(i) + i phi(H) = i (H^T - H);
// G lower (u16, ldg), H full (u16, ldh); C interleaved (re, im) uint32 pairs, Low only.
// One block per lower 64 x 64 tile (grid over lower tile pairs as K4); G, H are rows_pad x
// rows_pad (multiple of 128, ld a multiple of 8) so every 16-byte tile load is in range.  The
// mirrored H tile is staged in shared memory; C pairs are stored as 16-byte (re, im, re, im).
template <typename InT>
__global__ void __launch_bounds__(256) twom_kernel(int64_t m, const InT *G, int64_t ldg,
                                                   const InT *H, int64_t ldh, uint32_t *C,
                                                   int64_t ldc, ModP mod, uint32_t alpha, uint32_t beta,
                                                   int axpby) {
  const int x = (int)blockIdx.x;
  int ti = (int)((sqrtf(8.0f * (float)x + 1.0f) - 1.0f) * 0.5f);
  while ((ti + 1) * (ti + 2) / 2 <= x) ++ti;
  while (ti * (ti + 1) / 2 > x) --ti;
  const int tj = x - ti * (ti + 1) / 2;
  const int tx = threadIdx.x & 7, ty = threadIdx.x >> 3;   // 8 x 32
  const int64_t i0 = (int64_t)ti * 64, j0 = (int64_t)tj * 64;
  const int cx = tx * 8;
  __shared__ uint32_t sH[64][65];   // H on the mirrored tile (rows j0.., cols i0..)
  Pk8<InT> g[2], h[2], hu[2];
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const int y = ty + 32 * rr;
    g[rr].load(G + (i0 + y) * ldg + j0 + cx);
    h[rr].load(H + (i0 + y) * ldh + j0 + cx);
    hu[rr].load(H + (j0 + y) * ldh + i0 + cx);
  }
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    uint32_t q[8];
    hu[rr].get(q);
#pragma unroll
    for (int e = 0; e < 8; ++e) sH[ty + 32 * rr][cx + e] = q[e];
  }
  __syncthreads();
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const int y = ty + 32 * rr;
    const int64_t i = i0 + y, j = j0 + cx;
    if (i >= m || j > i) continue;
    uint32_t gv[8], hv[8], re[8], im[8];
    g[rr].get(gv);
    h[rr].get(hv);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const uint32_t ht = sH[cx + e][y];                                  // H(j, i)
      re[e] = submod(submod(gv[e], hv[e], mod), ht, mod);                 // G - H - H^T
      im[e] = submod(ht, hv[e], mod);                                     // H^T - H
    }
    const int64_t n = min64(8, min64(i - j + 1, m - j));
    uint32_t *o = C + 2 * (i * ldc + j);
    if (axpby) {
      for (int e = 0; e < n; ++e) {
        re[e] = addmod(mulmod_any(alpha, re[e], mod), mulmod_any(beta, mod_u32(o[2 * e], mod), mod), mod);
        im[e] = addmod(mulmod_any(alpha, im[e], mod), mulmod_any(beta, mod_u32(o[2 * e + 1], mod), mod), mod);
      }
    }
    if (n == 8 && (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        __stcs(reinterpret_cast<uint4 *>(o) + e, make_uint4(re[2 * e], im[2 * e], re[2 * e + 1], im[2 * e + 1]));
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (e < n) { o[2 * e] = re[e]; o[2 * e + 1] = im[e]; }
    }
  }
}

cudaError_t launch_twom(int64_t m, const void *G, int64_t ldg, const void *H, int64_t ldh, int in32,
                        uint32_t *C, int64_t ldc, const ModP &mod, uint32_t alpha, uint32_t beta, int axpby,
                        cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  const unsigned nt = (unsigned)((m + 63) / 64);
  const dim3 grid(nt * (nt + 1) / 2);
  if (in32)
    twom_kernel<uint32_t><<<grid, 256, 0, s>>>(m, static_cast<const uint32_t *>(G), ldg,
                                               static_cast<const uint32_t *>(H), ldh, C, ldc, mod, alpha, beta, axpby);
  else
    twom_kernel<uint16_t><<<grid, 256, 0, s>>>(m, static_cast<const uint16_t *>(G), ldg,
                                               static_cast<const uint16_t *>(H), ldh, C, ldc, mod, alpha, beta, axpby);
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

// Low(X) <- beta Low(X) (SYRK form with k = 0)
__global__ void scale_lower_kernel(int64_t row0, int w, uint32_t *X, int64_t ldx, uint32_t beta, ModP mod) {
  const int64_t i = row0 + blockIdx.y;
  uint32_t *row = X + i * ldx * w;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < (i + 1) * w;
       j += (int64_t)gridDim.x * blockDim.x)
    row[j] = mulmod_any(beta, mod_u32(row[j], mod), mod);
}

cudaError_t launch_scale_lower(int64_t m, int w, uint32_t *X, int64_t ldx, uint32_t beta, const ModP &mod,
                               cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  const int64_t per_row = (m * w + 255) / 256;
  for (int64_t r0 = 0; r0 < m; r0 += 65535) {
    const int64_t rows = (m - r0) < 65535 ? (m - r0) : 65535;
    scale_lower_kernel<<<dim3((unsigned)(per_row < 64 ? per_row : 64), (unsigned)rows), 256, 0, s>>>(
        r0, w, X, ldx, beta, mod);
  }
  return cudaGetLastError();
}

// Up(C) = phi(Low(C)) (Lemma lem:uplow): C[j][i] = C[i][j] (conjugated for phi = H), i > j
// one block per (region row, region); threads over the columns.  The packed buffer holds
// uint16 residues when p < 2^16 (half the bytes on the wire), uint32 otherwise.
template <typename BT>
__global__ void __launch_bounds__(256) rect_copy_kernel(const RectDev *rects, uint32_t *C, int64_t ldc, BT *buf,
                                                        int to_buf) {
  const RectDev R = rects[blockIdx.y];
  const int64_t i = blockIdx.x;
  if (i >= R.rows) return;
  uint32_t *c = C + (R.r0 + i) * ldc + R.c0;
  BT *b = buf + R.off + i * R.cols;
  const int64_t ncol = R.lower ? min64(R.cols, R.r0 + i - R.c0 + 1) : R.cols;
  for (int64_t j = threadIdx.x; j < ncol; j += blockDim.x) {
    if (to_buf) b[j] = (BT)c[j];
    else c[j] = b[j];
  }
}

cudaError_t launch_rect_copy(const RectDev *rects, int n, int max_rows, uint32_t *C, int64_t ldc, void *buf,
                             int esize, int to_buf, cudaStream_t s) {
  if (n == 0 || max_rows == 0) return cudaSuccess;
  const dim3 grid((unsigned)max_rows, (unsigned)n);
  if (esize == 2) rect_copy_kernel<uint16_t><<<grid, 256, 0, s>>>(rects, C, ldc, static_cast<uint16_t *>(buf), to_buf);
  else rect_copy_kernel<uint32_t><<<grid, 256, 0, s>>>(rects, C, ldc, static_cast<uint32_t *>(buf), to_buf);
  return cudaGetLastError();
}

// exact residue sum of n partials (each < p, n (p - 1) < 2^32) then mod p, on Low; one block per row
template <typename T>
__global__ void __launch_bounds__(256) sum_partials_kernel(int64_t m, const T *R, int64_t ldr, int64_t stride, int n,
                                                           uint32_t *C, int64_t ldc, ModP mod) {
  const int64_t i = blockIdx.x;
  if (i >= m) return;
  for (int64_t j = threadIdx.x; j <= i; j += blockDim.x) {
    uint32_t acc = 0;
    for (int r = 0; r < n; ++r) acc += (uint32_t)R[(int64_t)r * stride + i * ldr + j];
    C[i * ldc + j] = mod_u32(acc, mod);
  }
}

cudaError_t launch_sum_partials(int64_t m, const void *R, int64_t ldr, int64_t stride, int n, int esize, uint32_t *C,
                                int64_t ldc, const ModP &mod, cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  if (esize == 2)
    sum_partials_kernel<uint16_t><<<(unsigned)m, 256, 0, s>>>(m, static_cast<const uint16_t *>(R), ldr, stride, n, C,
                                                               ldc, mod);
  else
    sum_partials_kernel<uint32_t><<<(unsigned)m, 256, 0, s>>>(m, static_cast<const uint32_t *>(R), ldr, stride, n, C,
                                                               ldc, mod);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(256) fill_upper_kernel(int64_t m, int w, uint32_t *C, int64_t ldc, ModP mod) {
  const int ti = blockIdx.y, tj = blockIdx.x;
  if (ti < tj) return;
  const int tx = threadIdx.x, ty = threadIdx.y;
  __shared__ uint32_t s[32][33][4];
  const int64_t i0 = (int64_t)ti * 32, j0 = (int64_t)tj * 32;
  for (int y = ty; y < 32; y += 8) {
    const int64_t i = i0 + y, j = j0 + tx;
    if (i < m && j < m && j < i)
      for (int c = 0; c < w; ++c) s[y][tx][c] = C[(i * ldc + j) * w + c];
  }
  __syncthreads();
  for (int y = ty; y < 32; y += 8) {
    const int64_t r = j0 + y, c = i0 + tx;   // upper element (r, c) = phi(C[c][r]): conjugate, transposed
    if (r < m && c < m && r < c) {
      C[(r * ldc + c) * w] = s[tx][y][0];
      for (int q = 1; q < w; ++q) C[(r * ldc + c) * w + q] = submod(0, s[tx][y][q], mod);
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
