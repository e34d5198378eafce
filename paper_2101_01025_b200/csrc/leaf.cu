// K2/K3 leaf kernel: grouped persistent tcgen05 int8 GEMM /
// lower-triangle SYRK on CTA pairs, int32 TMEM accumulators, mod-p limb-recombination epilogue
// (P1..P5 of Alg. alg:MIAHMM), and the tail fixup kernel.
#include <algorithm>
#include <cstdio>

#include "kernel_util.cuh"

namespace adj {

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

// Claim-wave gate wait: until `need` jobs have issued their loads.  The gate only
// orders job starts (results never depend on it) and cannot deadlock when every CTA of the launch
// is resident; should CTAs ever be time-sliced (another context, MPS), it gives up after 50 ms
// instead of waiting on a CTA that is not running.
__device__ __forceinline__ void gate_wait(const int32_t *counter, int need) {
  const volatile int32_t *done = counter;
  if (*done >= need) return;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (*done < need) {
    __nanosleep(64);
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 50000000ull) return;
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
      int idx2 = 0, idx_d1 = 0;
      uint2 d1 = make_uint2(kEnd, 0u);
      // claim-wave gate (as in leafw_kernel; api.cpp launch_leaf_all)
      const bool claim1 = P.gate < 0 || P.gate > 100;
      const int gate = claim1 ? (P.gate < 0 ? 0 : P.gate - 1000) : P.gate;
      if (dyn && leader && !claim1) {
        const int idx1 = atomicAdd(P.job_counter, 1);
        idx2 = atomicAdd(P.job_counter, 1);
        idx_d1 = idx1;
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
          if (claim1) {
            idx_d1 = atomicAdd(P.job_counter, 1);
            d1 = idx_d1 < P.n_tiles ? __ldg(&P.tiles[idx_d1]) : make_uint2(kEnd, 0u);
          }
          if (gate > 0 && d1.x != kEnd && idx_d1 >= ncl) {
            const int w = idx_d1 / ncl;
            const int need = min(P.n_tiles, (w - 1) * ncl + (gate * ncl + 99) / 100);
            gate_wait(P.job_counter + 1, need);
          }
          next = d1;
          jq[s] = next;
          const uint32_t peer = ptx::mapa(ptx::smem_u32(&jq[s]), 1);
          ptx::st_shared_cluster_u32(peer, next.x);
          ptx::st_shared_cluster_u32(peer + 4, next.y);
          ptx::mbar_arrive(&jq_full[s]);
          ptx::mbar_arrive_cluster_release(ptx::mapa(ptx::smem_u32(&jq_full[s]), 1));
          if (next.x == kEnd) break;
          if (!claim1) {
            d1 = idx2 < P.n_tiles ? __ldg(&P.tiles[idx2]) : make_uint2(kEnd, 0u);   // used next iteration
            idx_d1 = idx2;
            idx2 = atomicAdd(P.job_counter, 1);                                     // claimed for i + 2
          }
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
          const bool rev = P.kalt && (u & 1);   // odd units walk K backwards (as in leafw_kernel)
#pragma unroll 1
          for (int x = 0; x < kb1 - kb0; ++x) {
            const int kb = rev ? kb1 - 1 - x : kb0 + x;
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
        if (dyn && leader && P.gate != 0) atomicAdd(P.job_counter + 1, 1);   // this job's loads are issued
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

// ============================================================================ wide-N leaf (256 x 512)
// The same CTA-pair tcgen05 kind::i8 leaf with 256 x 512 output tiles: each k-block stage holds the
// A tile (128 rows per CTA) and two B tiles (the two N = 256 halves), and the MMA thread issues
// both halves against the one A tile, so A is staged once per 2 x 256 x 256 MACs: 25% fewer
// operand bytes per MAC through L2, the crossbar and shared memory than 256 x 256 tiles.  Under
// the board's power cap the operand stream is about a third of the leaf's energy per MAC (DESIGN
// §5), so the bytes buy clock.  The accumulator takes all 512 TMEM columns (two 256-column halves),
// so the limb accumulators of a tile cannot alternate between slots; instead the recombination
// runs Horner-style in TMEM: after unit u (accumulator j, K segment) the epilogue replaces each
// value t by t * h_u mod p (h_u = w_j / w_{j+1}, or 1 between K segments of one accumulator) and
// stores it back (tcgen05.st), the next unit accumulates on top of it, and the last unit's drain
// multiplies by w_last and writes the residue:  sum_u w_u a_u = w_last (a_last + h (a_prev + ...)).
// No shared-memory partial sums.  The MMA thread hides the drain behind the halves: the first
// H stages of a unit run half 0 only (half 1 is still being drained), the last T stages run
// half 0 first and commit it, so half 0's drain overlaps half 1's last MMAs.
template <int NACC, int EW_ = 8>
struct LeafWCfg {
  static constexpr int STAGES = 4;
  static constexpr int A_BYTES = 128 * kBK;
  static constexpr int B_BYTES = 128 * kBK;          // one N = 256 half: 128 rows per CTA
  static constexpr int STAGE_BYTES = A_BYTES + 2 * B_BYTES;
  static constexpr int JQ = 4;
  static constexpr int BAR_BYTES = 8 * (2 * STAGES + 4 + 2 * JQ) + 16 + 8 * JQ;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + BAR_BYTES;
  static constexpr int EPI_WARPS = EW_;              // 4 TMEM lane quadrants x 2 column halves x EW_ / 8 column parts
  static constexpr int THREADS = 32 * (EPI_WARPS + 3);
  static constexpr int EDGE = STAGES - 1;            // H = T: stages run half-0-first at a unit's edges
};

template <int NACC, bool WIDE, int EWN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(32 * (EWN + 3), 1)
    leafw_kernel(const __grid_constant__ LeafParams P) {
  using Cfg = LeafWCfg<NACC, EWN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t *full_bar = reinterpret_cast<uint64_t *>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t *empty_bar = full_bar + Cfg::STAGES;
  uint64_t *acc_full = empty_bar + Cfg::STAGES;     // [2]: MMA -> epilogue, one per N half
  uint64_t *acc_empty = acc_full + 2;               // [2]: epilogue -> MMA (leader CTA)
  uint64_t *jq_full = acc_empty + 2;
  uint64_t *jq_empty = jq_full + Cfg::JQ;
  uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(jq_empty + Cfg::JQ);
  uint2 *jq = reinterpret_cast<uint2 *>(tmem_holder + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  const int cid = (int)ptx::cluster_id_x();
  const int ncl = (int)ptx::num_clusters_x();
  constexpr int EW = Cfg::EPI_WARPS;
  constexpr int W_ALLOC = EW, W_MMA = EW + 1, W_TMA = EW + 2;
  if (warp == W_TMA && lane == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int h = 0; h < 2; ++h) {
      ptx::mbar_init(&acc_full[h], 1);
      ptx::mbar_init(&acc_empty[h], 2 * (EW / 2));   // the EW / 2 warps of half h in both CTAs
    }
    for (int s = 0; s < Cfg::JQ; ++s) {
      ptx::mbar_init(&jq_full[s], 1);
      ptx::mbar_init(&jq_empty[s], 2 + 2 * EW);
    }
    ptx::fence_barrier_init();
    for (int i = 0; i < kMaxMaps; ++i) ptx::prefetch_tmap(&P.maps[i]);
  }
  if (warp == W_ALLOC) ptx::tmem_alloc_2sm(tmem_holder, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  const bool dyn = P.job_counter != nullptr;
  constexpr uint32_t kEnd = 0xFFFFFFFFu;
  auto job_consume = [&](int i, bool remote_release) -> uint2 {
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
      uint2 next = (!dyn && cid < P.n_tiles) ? __ldg(&P.tiles[cid]) : make_uint2(0u, 0u);
      int idx2 = 0, idx_d1 = 0;
      int gate_need = 0;   // soft gate: the wait of the current job, after its first P.gate_pre stages
      uint2 d1 = make_uint2(kEnd, 0u);
      // claim1: a job is claimed when its loads are about to start (claim order = start order);
      // otherwise two ahead (claim latency hidden, claim order = start order of the previous job)
      const bool claim1 = P.gate < 0 || P.gate > 100;
      const int gate = claim1 ? (P.gate < 0 ? 0 : P.gate - 1000) : P.gate;
      if (dyn && leader && !claim1) {
        const int idx1 = atomicAdd(P.job_counter, 1);
        idx2 = atomicAdd(P.job_counter, 1);
        idx_d1 = idx1;
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
          if (claim1) {
            idx_d1 = atomicAdd(P.job_counter, 1);
            d1 = idx_d1 < P.n_tiles ? __ldg(&P.tiles[idx_d1]) : make_uint2(kEnd, 0u);
          }
          gate_need = 0;
          if (gate > 0 && d1.x != kEnd && idx_d1 >= ncl) {
            // claim-wave gate: every dependency is a job of a lower claim index, whose producer
            // never waits on a higher one, so the wait always ends
            const int w = idx_d1 / ncl;
            const int need = min(P.n_tiles, (w - 1) * ncl + (gate * ncl + 99) / 100);
            if (P.gate_pre > 0) {
              gate_need = need;   // waited for inside the load loop below
            } else {
              gate_wait(P.job_counter + 1, need);
            }
          }
          next = d1;
          jq[s] = next;
          const uint32_t peer = ptx::mapa(ptx::smem_u32(&jq[s]), 1);
          ptx::st_shared_cluster_u32(peer, next.x);
          ptx::st_shared_cluster_u32(peer + 4, next.y);
          ptx::mbar_arrive(&jq_full[s]);
          ptx::mbar_arrive_cluster_release(ptx::mapa(ptx::smem_u32(&jq_full[s]), 1));
          if (next.x == kEnd) break;
          if (!claim1) {
            d1 = idx2 < P.n_tiles ? __ldg(&P.tiles[idx2]) : make_uint2(kEnd, 0u);
            idx_d1 = idx2;
            idx2 = atomicAdd(P.job_counter, 1);
          }
        } else {
          next = job_consume(i, true);
          if (next.x == kEnd) break;
        }
        int q, I, J;
        decode_tile(next.x, q, I, J);
        if (!dyn && t + ncl < P.n_tiles) next = __ldg(&P.tiles[t + ncl]);
        const LeafProduct &pr = P.prod[q];
        const CUtensorMap *map = &P.maps[pr.map];
        const int kseg = pr.kseg, kblocks = pr.kblocks;
        const int a_pr = pr.a_plane_rows, b_pr = pr.b_plane_rows;
        const int arow = pr.a_row0 + I * 256 + (int)rank * 128;
        const int brow = pr.b_row0 + J * 512 + (int)rank * 128;   // half h: + h * 256
        // diagonal SYRK tile whose column half 1 lies wholly above its rows: half 0 only.  Dynamic
        // (gated) launches only: there the early finish waits at the gate and saves energy; in a
        // static short launch (c2, L2-bound at full clock) the early finishers run ahead into the
        // next wave and the step got 1.8% slower (profiles/r02/skip_half_ab.txt)
        const bool skip1 = dyn && pr.sym && J * 512 + 256 > I * 256 + 255;
        const int nseg = (kblocks + kseg - 1) / kseg;
        int issued = 0;   // stages of this job issued so far (soft gate)
#pragma unroll 1
        for (int u = 0; u < NACC * nseg; ++u) {
          const int j = u / nseg, kb0 = (u % nseg) * kseg;
          const int kb1 = min(kblocks, kb0 + kseg);
          const int t0 = P.acc_begin[j], nt = P.acc_begin[j + 1] - t0;
          const int ar0 = arow + P.terms[t0].a_plane * a_pr, br0 = brow + P.terms[t0].b_plane * b_pr;
          const int ar1 = nt > 1 ? arow + P.terms[t0 + 1].a_plane * a_pr : ar0;
          const int br1 = nt > 1 ? brow + P.terms[t0 + 1].b_plane * b_pr : br0;
          // odd units walk K backwards: a unit starts on the k-blocks the previous one loaded last
          const bool rev = P.kalt && (u & 1);
#pragma unroll 1
          for (int x = 0; x < kb1 - kb0; ++x) {
            const int kb = rev ? kb1 - 1 - x : kb0 + x;
#pragma unroll 1
            for (int tt = 0; tt < nt; ++tt) {
              if (gate_need > 0 && issued++ == P.gate_pre) {   // leader only (gate_need stays 0 elsewhere)
                gate_wait(P.job_counter + 1, gate_need);
                gate_need = 0;
              }
              ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
              if (leader)
                ptx::mbar_expect_tx(&full_bar[stage], skip1 ? 2 * (Cfg::A_BYTES + Cfg::B_BYTES) : 2 * Cfg::STAGE_BYTES);
              uint8_t *sa = smem + stage * Cfg::STAGE_BYTES;
              const int br = tt ? br1 : br0;
              ptx::tma_load_2d_2sm(sa, map, kb * kBK, tt ? ar1 : ar0, &full_bar[stage]);
              ptx::tma_load_2d_2sm(sa + Cfg::A_BYTES, map, kb * kBK, br, &full_bar[stage]);
              if (!skip1)
                ptx::tma_load_2d_2sm(sa + Cfg::A_BYTES + Cfg::B_BYTES, map, kb * kBK, br + 256, &full_bar[stage]);
              if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
            }
          }
        }
        if (dyn && leader && P.gate != 0) atomicAdd(P.job_counter + 1, 1);   // this job's loads are issued
      }
    }
  } else if (warp == W_MMA) {
    // ------------------------------------------------------------ MMA issuer (leader CTA, one thread)
    if (leader && lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      uint32_t unit = 0;   // units issued so far (acc_empty / acc_full phases: both halves per unit)
      const uint32_t smem_base = ptx::smem_u32(smem);
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
        int q, I, J;
        decode_tile(next.x, q, I, J);
        if (!dyn && t + ncl < P.n_tiles) next = __ldg(&P.tiles[t + ncl]);
        const LeafProduct &pr = P.prod[q];
        const int kseg = pr.kseg, kblocks = pr.kblocks;
        const int nseg = (kblocks + kseg - 1) / kseg;
        const bool skip1 = dyn && pr.sym && J * 512 + 256 > I * 256 + 255;   // half 0 only (as the producer)
#pragma unroll 1
        for (int u = 0; u < NACC * nseg; ++u, ++unit) {
          const int j = u / nseg, kb0 = (u % nseg) * kseg;
          const int kb1 = min(kblocks, kb0 + kseg);
          const int t0 = P.acc_begin[j], nt = P.acc_begin[j + 1] - t0;
          const uint32_t id0 = ptx::idesc_i8(256, 256, P.terms[t0].a_signed != 0, P.terms[t0].b_signed != 0);
          const uint32_t id1 = nt > 1 ? ptx::idesc_i8(256, 256, P.terms[t0 + 1].a_signed != 0,
                                                      P.terms[t0 + 1].b_signed != 0) : id0;
          const int nst = (kb1 - kb0) * nt;                      // stages of this unit
          const int edge = min(Cfg::EDGE, nst / 2);              // H = T
          // the first unit of a job starts from zero; later ones accumulate onto the Horner value
          uint32_t acc0 = u > 0 ? 1u : 0u, acc1 = acc0;
          auto issue = [&](int h, uint32_t sa, uint32_t idesc, uint32_t &acc) {
            if (h == 1 && skip1) return;
            const uint64_t adesc = ptx::smem_desc_sw128(sa);
            const uint64_t bdesc = ptx::smem_desc_sw128(sa + Cfg::A_BYTES + h * Cfg::B_BYTES);
#pragma unroll
            for (int kk = 0; kk < kBK / 32; ++kk) {
              ptx::mma_i8_2sm(tmem_base + h * 256, adesc + 2 * kk, bdesc + 2 * kk, idesc, acc);
              acc = 1;
            }
          };
          // head: half 0 on the first `edge` stages while half 1 of the previous unit drains
          ptx::mbar_wait_cluster(&acc_empty[0], (unit & 1) ^ 1);
          ptx::tc_fence_after();
          int st = stage;
          uint32_t ph = phase;
          for (int x = 0; x < edge; ++x) {
            ptx::mbar_wait(&full_bar[st], ph);
            ptx::tc_fence_after();
            issue(0, smem_base + st * Cfg::STAGE_BYTES, (x % nt) ? id1 : id0, acc0);
            if (++st == Cfg::STAGES) { st = 0; ph ^= 1; }
          }
          ptx::mbar_wait_cluster(&acc_empty[1], (unit & 1) ^ 1);
          ptx::tc_fence_after();
          for (int x = 0; x < edge; ++x) {
            issue(1, smem_base + stage * Cfg::STAGE_BYTES, (x % nt) ? id1 : id0, acc1);
            ptx::mma_commit_2sm(&empty_bar[stage], 0x3);
            if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
          }
          // body: both halves per stage
          for (int x = edge; x < nst - edge; ++x) {
            ptx::mbar_wait(&full_bar[stage], phase);
            ptx::tc_fence_after();
            const uint32_t sa = smem_base + stage * Cfg::STAGE_BYTES;
            const uint32_t idesc = (x % nt) ? id1 : id0;
            issue(0, sa, idesc, acc0);
            issue(1, sa, idesc, acc1);
            ptx::mma_commit_2sm(&empty_bar[stage], 0x3);
            if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
          }
          // tail: half 0 on the last `edge` stages and its commit, then half 1
          st = stage;
          ph = phase;
          for (int x = nst - edge; x < nst; ++x) {
            ptx::mbar_wait(&full_bar[st], ph);
            ptx::tc_fence_after();
            issue(0, smem_base + st * Cfg::STAGE_BYTES, (x % nt) ? id1 : id0, acc0);
            if (++st == Cfg::STAGES) { st = 0; ph ^= 1; }
          }
          ptx::mma_commit_2sm(&acc_full[0], 0x3);
          for (int x = nst - edge; x < nst; ++x) {
            issue(1, smem_base + stage * Cfg::STAGE_BYTES, (x % nt) ? id1 : id0, acc1);
            ptx::mma_commit_2sm(&empty_bar[stage], 0x3);
            if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
          }
          ptx::mma_commit_2sm(&acc_full[1], 0x3);
        }
      }
    }
  } else if (warp < EW) {
    // ------------------------------------------------------------ epilogue (8 warps per CTA)
    constexpr int NPART = EW / 8;     // column parts per half
    constexpr int NCH = 8 / NPART;    // 32-column chunks per warp and unit
    const int q4 = warp & 3;          // TMEM lane quadrant
    const int h = (warp >> 2) & 1;    // N half: TMEM columns h * 256 .. + 255
    const int part = warp >> 3;       // columns part * NCH * 32 .. of the half
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const int lrow = q4 * 32 + lane;
    const ModP mod = P.mod;
    const uint32_t pm = mod.p;
    const uint32_t empty_remote = ptx::mapa(ptx::smem_u32(&acc_empty[h]), 0);
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
      int q, I, J;
      decode_tile(job.x, q, I, J);
      const LeafProduct &pr = P.prod[q];
      const int64_t row = (int64_t)I * 256 + rank * 128 + lrow;
      const int64_t col0 = (int64_t)J * 512 + h * 256 + part * NCH * 32;
      const int nseg = (pr.kblocks + pr.kseg - 1) / pr.kseg;
      const int nunits = NACC * nseg;
#pragma unroll 1
      for (int u = 0; u < nunits; ++u, ++unit) {
        const int j = u / nseg;
        const bool last = u == nunits - 1;
        // Horner step: the last unit's weight, 1 between K segments, w_j / w_{j+1} between accumulators
        const ShoupW w = last ? P.wshoup[j] : ((u + 1) % nseg ? P.one : P.hshoup[j]);
        ptx::mbar_wait(&acc_full[h], unit & 1);
        ptx::tc_fence_after();
        // a diagonal SYRK tile whose column half 1 lies wholly above its rows ran no half-1 MMAs:
        // nothing to drain there, but its TMEM is still released below
        const bool skip = h == 1 && dyn && pr.sym && J * 512 + 256 > I * 256 + 255;
#pragma unroll 1
        for (int c = 0; c < (skip ? 0 : NCH); ++c) {
          uint32_t v[32];
          const uint32_t taddr = tmem_base + lane_off + h * 256 + (part * NCH + c) * 32;
          ptx::tmem_ld32(taddr, v);
          ptx::tmem_wait_ld();
          if (last) {
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = acc_mulred((int32_t)v[e], w.wc, w.wq, 0u, pm);
            store_chunk(pr, row, col0 + c * 32, v, mod);
          } else {   // intermediate Horner step: a value < 3p stays in TMEM (modp.cuh mulred_lazy3)
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = mulred_lazy3((int32_t)v[e], w.wc, w.wq, pm);
            ptx::tmem_st32(taddr, v);
          }
        }
        if (!last && !skip) ptx::tmem_wait_st();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(empty_remote);
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
}

template <int NACC, bool WIDE, int EWN>
static cudaError_t launch_leafw_t(const LeafParams &p, int grid, cudaStream_t s) {
  using Cfg = LeafWCfg<NACC, EWN>;
  static std::atomic<uint64_t> done{0};
  cudaError_t e = ensure_smem(leafw_kernel<NACC, WIDE, EWN>, Cfg::SMEM, done);
  if (e != cudaSuccess) return e;
  leafw_kernel<NACC, WIDE, EWN><<<grid, Cfg::THREADS, Cfg::SMEM, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_leafw(const LeafParams &p, int nacc, int grid, cudaStream_t s) {
  if (p.n_tiles == 0) return cudaSuccess;
  if (grid % 2) return cudaErrorInvalidValue;
  // 8 epilogue warps (16 measured the same at c3 / c4: the drain is not the limit); ADJ_LEAFW_EPI=16 (A/B)
  static const int ew = getenv("ADJ_LEAFW_EPI") ? atoi(getenv("ADJ_LEAFW_EPI")) : 8;
  if (ew == 8) {
    if (nacc == 1) return launch_leafw_t<1, false, 8>(p, grid, s);
    if (nacc == 3) return launch_leafw_t<3, false, 8>(p, grid, s);
    if (nacc == 6) return launch_leafw_t<6, true, 8>(p, grid, s);
    return cudaErrorInvalidValue;
  }
  if (nacc == 1) return launch_leafw_t<1, false, 16>(p, grid, s);
  if (nacc == 3) return launch_leafw_t<3, false, 16>(p, grid, s);
  if (nacc == 6) return launch_leafw_t<6, true, 16>(p, grid, s);
  return cudaErrorInvalidValue;
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

}  // namespace adj
