// K4 recombination: U1=P1+P5 (+Up(U1)=Low(U1)^T), U2=U1+P4, U4=U2+P3,
// U5=Low(U2+P4^T), U3=P1+P2 -> [[U3],[U4,U5]]; K5 2M combine Re = G - eps H -
// phi(H), Im = H^T - H (Alg. alg:2M); the GF(p^2) and quaternion (6M,
// PAPER.md:2016-2037) recombinations.
#include <algorithm>
#include <type_traits>
#include <cstdio>

#include "kernel_util.cuh"

namespace adj {

// ============================================================================ K4 recombination
// One block per lower pair {L = (ti, tj), U = (tj, ti)}, ti >= tj, of T x T tiles (T = 32; 64
// for a sharded pair list) of the (mh x mh) product grid, so that every product tile is read once:
//   L: U1 = P1 + P5, C21 = U1 + P4 + P3, C22 = Low(U1 + P4 + P4^T), C11 = Low(P1 + P2)
//   U (ti > tj): C21 = Up(U1) + P4 + P3 with Up(U1) = Low(U1)^T
// P4(U) and U1(L) are staged in shared memory for the two transposed uses.  Thread (tx, ty) of
// T/8 x T/2 owns 8 consecutive columns (16-byte u16 loads) of rows ty and ty + T/2.
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

// store8 of 8 in-range residues at a 16-byte aligned position (the FULL instance)
template <typename OutT>
__device__ __forceinline__ void store8_full(OutT *o, const uint32_t (&v)[8]) {
  if constexpr (sizeof(OutT) == 4) {
    __stcs(reinterpret_cast<uint4 *>(o), make_uint4(v[0], v[1], v[2], v[3]));
    __stcs(reinterpret_cast<uint4 *>(o) + 1, make_uint4(v[4], v[5], v[6], v[7]));
  } else {
    *reinterpret_cast<uint4 *>(o) =
        make_uint4(v[0] | (v[1] << 16), v[2] | (v[3] << 16), v[4] | (v[5] << 16), v[6] | (v[7] << 16));
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

// INPL (low-memory schedule): P1, P3 and P5 are read from C's own C11, C21 and C22
// blocks (OutT, leading dimension ldo), where the children and the root leaf wrote them.  Each
// thread writes only positions it has itself read above (C11 / C21 / C22 on L over its P1 / P3 /
// P5 loads, C21 on U over its P3 load), so the in-place update needs no extra ordering.
// FULL (host-checked in launch_combine): mh a multiple of T, every node's output covers its
// 2 mh x 2 mh positions with 16-byte aligned rows, no SYRK form: off-diagonal pairs then need no
// bounds, masks or diagonal selects (the generic path below still runs the diagonal pairs).
template <typename InT, typename OutT, int T, bool INPL = false, bool FULL = false>
__global__ void __launch_bounds__(T * T / 16) combine_kernel(const __grid_constant__ CombParams P) {
  constexpr int TX = T / 8, H = T / 2;   // TX threads of 8 columns per row; rows ty and ty + H
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
  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  const int64_t mh = P.mh, ldp = P.ldp;                     // ldp multiple of 128 -> aligned 16-byte loads
  const int64_t i0 = (int64_t)ti * T, j0 = (int64_t)tj * T;
  const ModP &m = P.mod;
  using T1 = typename std::conditional<INPL, OutT, InT>::type;   // type of P1, P3, P5
  const int64_t ld1 = INPL ? N.ldo : ldp;
  const T1 *P1 = INPL ? static_cast<const T1 *>(N.out) : static_cast<const T1 *>(N.P[0]);
  const T1 *P3 = INPL ? static_cast<const T1 *>(N.out) + mh * ld1 : static_cast<const T1 *>(N.P[2]);
  const T1 *P5 = INPL ? static_cast<const T1 *>(N.out) + mh * ld1 + mh : static_cast<const T1 *>(N.P[4]);
  const InT *P2 = static_cast<const InT *>(N.P[1]), *P4 = static_cast<const InT *>(N.P[3]);
  __shared__ uint32_t sU[T][T + 1];   // U1 on L (Low part; on a diagonal tile the full tile is filled)
  __shared__ uint32_t sQ[T][T + 1];   // P4 on U (rows j0.., cols i0..)
  const int cx = tx * 8;
  // every load of the block up front (buffers are rows_pad x rows_pad: always in range)
  Pk8<T1> l1[2], l5[2], l3[2], u3[2];
  Pk8<InT> l2[2], l4[2], u4[2];
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const int y = ty + H * rr;
    const int64_t oL = (i0 + y) * ldp + j0 + cx, oU = (j0 + y) * ldp + i0 + cx;
    const int64_t oL1 = (i0 + y) * ld1 + j0 + cx, oU1 = (j0 + y) * ld1 + i0 + cx;
    l1[rr].load(P1 + oL1);
    l5[rr].load(P5 + oL1);
    u4[rr].load(P4 + oU);
    l4[rr].load(P4 + oL);
    l3[rr].load(P3 + oL1);
    l2[rr].load(P2 + oL);
    if (!diag) u3[rr].load(P3 + oU1);
  }
  uint32_t u1[2][8];
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const int y = ty + H * rr;
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
  if constexpr (FULL) {
    if (!diag) {
      const int64_t ldo = N.ldo;
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {   // tile L: C21 = U1 + P4 + P3, C22 = U1 + P4 + P4^T, C11 = P1 + P2
        const int y = ty + H * rr;
        const int64_t i = i0 + y, j = j0 + cx;
        uint32_t p4[8], p3[8], p1[8], p2[8], c21[8], c22[8], c11[8];
        l4[rr].get(p4);
        l3[rr].get(p3);
        l1[rr].get(p1);
        l2[rr].get(p2);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const uint32_t u2 = addmod(u1[rr][e], p4[e], m);
          c21[e] = addmod(u2, p3[e], m);
          c22[e] = addmod(u2, sQ[cx + e][y], m);
          c11[e] = addmod(p1[e], p2[e], m);
        }
        store8_full<OutT>(O + (mh + i) * ldo + j, c21);
        store8_full<OutT>(O + (mh + i) * ldo + mh + j, c22);
        store8_full<OutT>(O + i * ldo + j, c11);
      }
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {   // tile U: C21 = Up(U1) + P4 + P3
        const int y = ty + H * rr;
        const int64_t r = j0 + y, c = i0 + cx;
        uint32_t p3[8], q4[8], c21[8];
        u3[rr].get(p3);
        u4[rr].get(q4);
#pragma unroll
        for (int e = 0; e < 8; ++e) c21[e] = addmod(addmod(sU[cx + e][y], q4[e], m), p3[e], m);
        store8_full<OutT>(O + (mh + r) * ldo + c, c21);
      }
      return;
    }
  }
  const bool ax = sizeof(OutT) == 4 && P.axpby;
  // ---- tile L (and, on the diagonal, its upper part of C21)
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const int y = ty + H * rr;
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
    const int y = ty + H * rr;
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
  // 32 x 32 tile pairs of 64 threads: ~4x as many blocks as 64 x 64 ones (the 64-tile grid of an
  // 8192^2 depth-1 call is 7.03 waves of 296 blocks, a near-empty last wave); the sharded pair
  // list (P.pairs) is in 64-tile units
  const int T = p.pairs ? 64 : 32;
  const unsigned nt = (unsigned)((p.mh + T - 1) / T);
  dim3 grid(p.pairs ? (unsigned)p.n_pairs : nt * (nt + 1) / 2, (unsigned)p.n_nodes), block(T * T / 16);
  if (grid.x == 0) return cudaSuccess;
  // FULL instance: no bounds on the off-diagonal pairs (see combine_kernel)
  const int osz = p.out_u32 ? 4 : 2;
  bool full = !p.inplace && !p.axpby && p.pairs == nullptr && p.mh % 32 == 0;
  for (int n = 0; n < p.n_nodes && full; ++n) {
    const CombNode &N = p.nodes[n];
    full = N.out_valid >= 2 * p.mh && (N.ldo * osz) % 16 == 0 && (reinterpret_cast<uintptr_t>(N.out) & 15) == 0;
  }
#define COMB(I, O)                                                              \
  if (p.inplace) combine_kernel<I, O, 32, true><<<grid, block, 0, s>>>(p);       \
  else if (T == 64) combine_kernel<I, O, 64><<<grid, block, 0, s>>>(p);        \
  else if (full) combine_kernel<I, O, 32, false, true><<<grid, block, 0, s>>>(p); \
  else combine_kernel<I, O, 32><<<grid, block, 0, s>>>(p)
  if (p.in32) COMB(uint32_t, uint32_t);
  else if (p.out_u32) COMB(uint16_t, uint32_t);
  else COMB(uint16_t, uint16_t);
#undef COMB
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
    for (int e = 0; e < 8; ++e) __stcs(reinterpret_cast<uint4 *>(o) + e, make_uint4(h[0][e], h[1][e], h[2][e], h[3][e]));
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
    const int64_t nq = min64(8, min64(i - j + 1, m - j));
    if (P.out16) {   // ADJ_OUT_U16: 4 uint16 components per quaternion (plain form only)
      uint16_t *o = reinterpret_cast<uint16_t *>(P.C) + 4 * (i * P.ldc + j);
      if (nq == 8 && (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          __stcs(reinterpret_cast<uint4 *>(o) + e,
                 make_uint4(h[0][2 * e] | (h[1][2 * e] << 16), h[2][2 * e] | (h[3][2 * e] << 16),
                            h[0][2 * e + 1] | (h[1][2 * e + 1] << 16), h[2][2 * e + 1] | (h[3][2 * e + 1] << 16)));
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (e < nq)
#pragma unroll
            for (int c = 0; c < 4; ++c) o[4 * e + c] = (uint16_t)h[c][e];
      }
      continue;
    }
    store_q8(P.C + 4 * (i * P.ldc + j), nq, h, P);
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
template <typename InT, bool O16>
__global__ void __launch_bounds__(256) twom_kernel(int64_t m, const InT *G, int64_t ldg,
                                                   const InT *H, int64_t ldh, void *Cv,
                                                   int64_t ldc, ModP mod, uint32_t alpha, uint32_t beta,
                                                   int axpby) {
  uint32_t *C = static_cast<uint32_t *>(Cv);   // (re, im) uint32 pairs, or uint16 pairs when O16
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
    if constexpr (O16) {   // ADJ_OUT_U16: one 32-bit word (re | im << 16) per element
      uint32_t *o = C + (i * ldc + j);
      if (n == 8 && (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
        __stcs(reinterpret_cast<uint4 *>(o), make_uint4(re[0] | (im[0] << 16), re[1] | (im[1] << 16),
                                                        re[2] | (im[2] << 16), re[3] | (im[3] << 16)));
        __stcs(reinterpret_cast<uint4 *>(o) + 1, make_uint4(re[4] | (im[4] << 16), re[5] | (im[5] << 16),
                                                            re[6] | (im[6] << 16), re[7] | (im[7] << 16)));
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (e < n) o[e] = re[e] | (im[e] << 16);
      }
      continue;
    }
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
                        void *C, int64_t ldc, const ModP &mod, uint32_t alpha, uint32_t beta, int axpby,
                        int out16, cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  const unsigned nt = (unsigned)((m + 63) / 64);
  const dim3 grid(nt * (nt + 1) / 2);
  if (in32)
    twom_kernel<uint32_t, false><<<grid, 256, 0, s>>>(m, static_cast<const uint32_t *>(G), ldg,
                                                      static_cast<const uint32_t *>(H), ldh, C, ldc, mod, alpha,
                                                      beta, axpby);
  else if (out16)
    twom_kernel<uint16_t, true><<<grid, 256, 0, s>>>(m, static_cast<const uint16_t *>(G), ldg,
                                                     static_cast<const uint16_t *>(H), ldh, C, ldc, mod, alpha,
                                                     beta, axpby);
  else
    twom_kernel<uint16_t, false><<<grid, 256, 0, s>>>(m, static_cast<const uint16_t *>(G), ldg,
                                                      static_cast<const uint16_t *>(H), ldh, C, ldc, mod, alpha,
                                                      beta, axpby);
  return cudaGetLastError();
}

}  // namespace adj
