// K1: pre-addition S1=(A21-A11)Y, S2=A22-A21 Y, S3=S1-A22, S4=S3+A12 (mod p)
// fused with the centered int8 limb split of every leaf operand (Alg. alg:MIAHMM,
// PAPER.md:303-307); the plain / 2M / quaternion limb splits (depth 0, gemm_modp, 2M's X / Y,
// 6M's A..W); the GF(p^2) pre-addition of ADJ_HERK_ALG1.
#include <algorithm>
#include <cstdio>

#include "kernel_util.cuh"

namespace adj {

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
  } else if (v.type == IN_U16 || v.type == IN_U16R) {
    const uint16_t *p = static_cast<const uint16_t *>(v.ptr) + R * v.ld + C;
    if (all) {
      uint2 q = __ldg(reinterpret_cast<const uint2 *>(p));
      x[0] = q.x & 0xFFFF; x[1] = q.x >> 16; x[2] = q.y & 0xFFFF; x[3] = q.y >> 16;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) if (C + e < v.cols_valid) x[e] = __ldg(p + e);
    }
    if (v.type == IN_U16R) {
#pragma unroll
      for (int e = 0; e < 4; ++e) x[e] = mod_u32(x[e], m);
    }
  } else if (v.type == IN_QUAD_SUM && v.e16) {   // 4 uint16 components per quaternion (ADJ_IN_U16)
    const uint16_t *p = static_cast<const uint16_t *>(v.ptr) + 4 * (R * v.ld + C);
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (C + e < v.cols_valid) {
        uint2 q = all ? __ldg(reinterpret_cast<const uint2 *>(p) + e)
                      : make_uint2((uint32_t)__ldg(p + 4 * e) | ((uint32_t)__ldg(p + 4 * e + 1) << 16),
                                   (uint32_t)__ldg(p + 4 * e + 2) | ((uint32_t)__ldg(p + 4 * e + 3) << 16));
        x[e] = addmod(addmod(mod_u32(q.x & 0xFFFF, m), mod_u32(q.x >> 16, m), m),
                      addmod(mod_u32(q.y & 0xFFFF, m), mod_u32(q.y >> 16, m), m), m);
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
    uint32_t re[4] = {0, 0, 0, 0}, im[4] = {0, 0, 0, 0};
    if (v.e16) {   // (re, im) uint16 pairs (ADJ_IN_U16)
      const uint16_t *p = static_cast<const uint16_t *>(v.ptr) + 2 * (R * v.ld + C);
      if (all) {
        const uint4 q = __ldg(reinterpret_cast<const uint4 *>(p));
        re[0] = q.x & 0xFFFF; im[0] = q.x >> 16; re[1] = q.y & 0xFFFF; im[1] = q.y >> 16;
        re[2] = q.z & 0xFFFF; im[2] = q.z >> 16; re[3] = q.w & 0xFFFF; im[3] = q.w >> 16;
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (C + e < v.cols_valid) { re[e] = __ldg(p + 2 * e); im[e] = __ldg(p + 2 * e + 1); }
      }
    } else {
      const uint32_t *p = static_cast<const uint32_t *>(v.ptr) + 2 * (R * v.ld + C);
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
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      uint32_t a = mod_u32(re[e], m), b = mod_u32(im[e], m);
      x[e] = v.type == IN_PAIR_SUM ? addmod(a, b, m) : (v.type == IN_PAIR_RE ? a : b);
    }
  }
}

// K7 limbs of 4 already-centered values c in [-(p-1)/2, (p-1)/2] (p <= 16763: |c| <= 8381):
// hi = floor((c + 64) / 128), lo = c - 128 hi, mid = hi + lo.  Two values per register in
// 16-bit lanes: v = c + 64 + 128 * 66 lies in [131, 16893], so hi = (v >> 7) - 66 and
// lo = (v & 127) - 64 per lane; the int8 bytes are the low bytes of the lanes after adding
// 256 - 66 and 256 - 64 (all lane values stay below 2^16, no carries between lanes).
// a[] are the lane values v - off of the K7 words above: v = a + off (off = 64 + 128 * 66 for
// centered c, or 64 + 128 * 66 - (p - 1) / 2 for the offset residues c + (p - 1) / 2 of K1)
__device__ __forceinline__ void k7_words(const uint32_t (&a)[4], uint32_t off, uint32_t (&w)[3]) {
  constexpr uint32_t kHi = 190u * 0x10001u, kLo = 192u * 0x10001u;
  const uint32_t off2 = off * 0x10001u;
  const uint32_t v01 = a[0] + (a[1] << 16) + off2;
  const uint32_t v23 = a[2] + (a[3] << 16) + off2;
  const uint32_t h01 = ((v01 >> 7) & 0x01FF01FFu) + kHi, h23 = ((v23 >> 7) & 0x01FF01FFu) + kHi;
  const uint32_t l01 = (v01 & 0x007F007Fu) + kLo, l23 = (v23 & 0x007F007Fu) + kLo;
  w[0] = __byte_perm(h01, h23, 0x6420);
  w[1] = __byte_perm(l01, l23, 0x6420);
  w[2] = __byte_perm(h01 + l01, h23 + l23, 0x6420);
}

__device__ __forceinline__ void k7c_words(const int32_t (&c)[4], uint32_t (&w)[3]) {
  const uint32_t a[4] = {(uint32_t)c[0], (uint32_t)c[1], (uint32_t)c[2], (uint32_t)c[3]};
  k7_words(a, 64u + 128u * 66u, w);
}

// K7 limb planes of 4 offset residues u = c + (p - 1) / 2 (off = 64 + 128 * 66 - (p - 1) / 2)
__device__ __forceinline__ void put_limbs4_k7u(int8_t *base, int64_t plane_stride, const uint32_t (&u)[4],
                                               uint32_t off) {
  uint32_t w[3];
  k7_words(u, off, w);
  *reinterpret_cast<uint32_t *>(base) = w[0];
  *reinterpret_cast<uint32_t *>(base + plane_stride) = w[1];
  *reinterpret_cast<uint32_t *>(base + 2 * plane_stride) = w[2];
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
    // hi = floor((c + 64) / 128), lo = c - 128 hi, mid = hi + lo (SWAR, k7c_words above)
    k7c_words(c, w);
  } else {
    // s8 hi = c >> 8 and u8 lo = c & 255 are bytes 1 and 0 of the two's-complement c
    w[0] = __byte_perm(__byte_perm(c[0], c[1], 0x51), __byte_perm(c[2], c[3], 0x51), 0x5410);
    w[1] = __byte_perm(__byte_perm(c[0], c[1], 0x40), __byte_perm(c[2], c[3], 0x40), 0x5410);
  }
}

// wide scheme: three balanced base-64 digits d2, d1, d0 of the centered residue c (|c| <= 131069;
// d1, d0 in [-32, 31], d2 in [-32, 32]) and the pair sums d2+d1, d1+d0, d2+d0 (6 s8 planes,
// 3-way Karatsuba).  v = c + 32 (1 + 64 + 4096) = (d0 + 32) + 64 (d1 + 32) + 4096 (d2 + 32) is
// non-negative, so the digits are its bit fields e0, e1, e2 minus 32.  The fields are packed as
// bytes; d = e - 32 is the byte (e + 96) ^ 128 and d + d' = e + e' - 64 the byte
// (e + e' + 64) ^ 128 (no byte exceeds 255, so the packed adds carry nothing between bytes).
__device__ __forceinline__ void t6_words_v(const uint32_t (&vv)[4], uint32_t (&w)[6]) {
  uint32_t e0[4], e1[4], e2[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const uint32_t v = vv[e];
    e0[e] = v & 63u;
    e1[e] = (v >> 6) & 63u;
    e2[e] = v >> 12;
  }
  const uint32_t E0 = __byte_perm(__byte_perm(e0[0], e0[1], 0x40), __byte_perm(e0[2], e0[3], 0x40), 0x5410);
  const uint32_t E1 = __byte_perm(__byte_perm(e1[0], e1[1], 0x40), __byte_perm(e1[2], e1[3], 0x40), 0x5410);
  const uint32_t E2 = __byte_perm(__byte_perm(e2[0], e2[1], 0x40), __byte_perm(e2[2], e2[3], 0x40), 0x5410);
  w[0] = (E2 + 0x60606060u) ^ 0x80808080u;        // d2
  w[1] = (E1 + 0x60606060u) ^ 0x80808080u;        // d1
  w[2] = (E0 + 0x60606060u) ^ 0x80808080u;        // d0
  w[3] = (E2 + E1 + 0x40404040u) ^ 0x80808080u;   // d2 + d1
  w[4] = (E1 + E0 + 0x40404040u) ^ 0x80808080u;   // d1 + d0
  w[5] = (E2 + E0 + 0x40404040u) ^ 0x80808080u;   // d2 + d0
}

__device__ __forceinline__ void t6_words(const uint32_t (&x)[4], const ModP &m, uint32_t (&w)[6]) {
  const uint32_t v[4] = {(uint32_t)(centered(x[0], m) + 133152), (uint32_t)(centered(x[1], m) + 133152),
                         (uint32_t)(centered(x[2], m) + 133152), (uint32_t)(centered(x[3], m) + 133152)};
  t6_words_v(v, w);
}

// the single s8 plane of 4 offset residues u = c + (p - 1) / 2 (p <= 255: byte 0 of c = u - h)
__device__ __forceinline__ void put_limbs4_s8u(int8_t *base, const uint32_t (&u)[4], uint32_t h) {
  *reinterpret_cast<uint32_t *>(base) =
      __byte_perm(__byte_perm(u[0] - h, u[1] - h, 0x40), __byte_perm(u[2] - h, u[3] - h, 0x40), 0x5410);
}

// s8 hi / u8 lo planes of 4 offset residues u = c + (p - 1) / 2 (bytes 1 and 0 of c = u - h)
__device__ __forceinline__ void put_limbs4_s8u8u(int8_t *base, int64_t plane_stride, const uint32_t (&u)[4],
                                                 uint32_t h) {
  const uint32_t c0 = u[0] - h, c1 = u[1] - h, c2 = u[2] - h, c3 = u[3] - h;
  *reinterpret_cast<uint32_t *>(base) = __byte_perm(__byte_perm(c0, c1, 0x51), __byte_perm(c2, c3, 0x51), 0x5410);
  *reinterpret_cast<uint32_t *>(base + plane_stride) =
      __byte_perm(__byte_perm(c0, c1, 0x40), __byte_perm(c2, c3, 0x40), 0x5410);
}

// 8-byte global store of (v0, v1) at base + off for a 32-bit off (8-byte aligned)
__device__ __forceinline__ void st2_off32(const int8_t *base, uint32_t off, uint32_t v0, uint32_t v1) {
  asm volatile("{\n\t.reg .u64 a;\n\tmad.wide.u32 a, %1, 1, %0;\n\tst.global.v2.u32 [a], {%2, %3};\n\t}" ::"l"(base),
               "r"(off), "r"(v0), "r"(v1));
}

// packed plane words of 4 offset residues u = c + (p - 1) / 2 (koff as for put_limbs4_*):
//   scheme 0: byte 0 of c = u - h;  scheme 1: as k7_words;
//   scheme 2: v = u - h + 2^15 = c + 2^15 lies in [0, 2^16), so two of them packed in one word add
//   without carries between the 16-bit lanes; byte 0 of v is the u8 lo of c, byte 1 is its s8 hi
//   + 128 (flipped back by the xor)
template <int SCHEME>
__device__ __forceinline__ void limb_words_u(const uint32_t (&u)[4], uint32_t koff, uint32_t (&w)[3]) {
  if constexpr (SCHEME == 0) {
    w[0] = __byte_perm(__byte_perm(u[0] - koff, u[1] - koff, 0x40), __byte_perm(u[2] - koff, u[3] - koff, 0x40),
                       0x5410);
  } else if constexpr (SCHEME == 1) {
    // k7_words with v = c + 64 + 2^15 (koff + 2^15 - 128 * 66): v >> 7 = hi + 256 and v & 127 =
    // lo + 64, so the hi bytes need no constant and hi + lo stays inside its 16-bit lane
    const uint32_t K = (koff + 32768u - 128u * 66u) * 0x10001u;
    const uint32_t v01 = (u[0] + (u[1] << 16)) + K, v23 = (u[2] + (u[3] << 16)) + K;
    const uint32_t h01 = (v01 >> 7) & 0x00FF00FFu, h23 = (v23 >> 7) & 0x00FF00FFu;
    const uint32_t l01 = (v01 & 0x007F007Fu) + 0x00C000C0u, l23 = (v23 & 0x007F007Fu) + 0x00C000C0u;
    w[0] = __byte_perm(h01, h23, 0x6420);
    w[1] = __byte_perm(l01, l23, 0x6420);
    w[2] = __byte_perm(h01 + l01, h23 + l23, 0x6420);
  } else {
    const uint32_t K = (0x8000u - koff) * 0x10001u;
    const uint32_t v01 = (u[0] + (u[1] << 16)) + K, v23 = (u[2] + (u[3] << 16)) + K;
    w[0] = __byte_perm(v01, v23, 0x7531) ^ 0x80808080u;
    w[1] = __byte_perm(v01, v23, 0x6420);
  }
}

// the six planes of 4 offset residues u = c + (p - 1) / 2: v = u + off, off = 133152 - (p - 1) / 2
__device__ __forceinline__ void put_limbs4_t6u(int8_t *base, int64_t plane_stride, const uint32_t (&u)[4],
                                               uint32_t off) {
  const uint32_t v[4] = {u[0] + off, u[1] + off, u[2] + off, u[3] + off};
  uint32_t w[6];
  t6_words_v(v, w);
#pragma unroll
  for (int pl = 0; pl < 6; ++pl) *reinterpret_cast<uint32_t *>(base + pl * plane_stride) = w[pl];
}

__device__ __forceinline__ void put_limbs4_t6(int8_t *base, int64_t plane_stride, const uint32_t (&x)[4],
                                              const ModP &m) {
  uint32_t w[6];
  t6_words(x, m, w);
#pragma unroll
  for (int pl = 0; pl < 6; ++pl) *reinterpret_cast<uint32_t *>(base + pl * plane_stride) = w[pl];
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
    uint32_t w0[6], w1[6];
    t6_words(x0, m, w0);
    t6_words(x1, m, w1);
#pragma unroll
    for (int pl = 0; pl < 6; ++pl) *reinterpret_cast<uint2 *>(base + pl * plane_stride) = make_uint2(w0[pl], w1[pl]);
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
    uint32_t w[4][6];
#pragma unroll
    for (int g = 0; g < 4; ++g) t6_words(x[g], m, w[g]);
#pragma unroll
    for (int pl = 0; pl < 6; ++pl)
      *reinterpret_cast<uint4 *>(base + pl * plane_stride) = make_uint4(w[0][pl], w[1][pl], w[2][pl], w[3][pl]);
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
  } else if constexpr (T == IN_U16 || T == IN_U16R) {
    uint2 q = __ldg(reinterpret_cast<const uint2 *>(static_cast<const uint16_t *>(ptr) + off));
    x[0] = q.x & 0xFFFF; x[1] = q.x >> 16; x[2] = q.y & 0xFFFF; x[3] = q.y >> 16;
    if constexpr (T == IN_U16R) {
      x[0] = mod_u32(x[0], m); x[1] = mod_u32(x[1], m); x[2] = mod_u32(x[2], m); x[3] = mod_u32(x[3], m);
    }
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
  if (fast && v.e16) {
    const uint4 q = __ldg(reinterpret_cast<const uint4 *>(static_cast<const uint16_t *>(v.ptr) + 2 * (R * v.ld + C)));
    re[0] = mod_u32(q.x & 0xFFFF, m); im[0] = mod_u32(q.x >> 16, m); re[1] = mod_u32(q.y & 0xFFFF, m);
    im[1] = mod_u32(q.y >> 16, m); re[2] = mod_u32(q.z & 0xFFFF, m); im[2] = mod_u32(q.z >> 16, m);
    re[3] = mod_u32(q.w & 0xFFFF, m); im[3] = mod_u32(q.w >> 16, m);
  } else if (fast) {
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

// O32: every plane byte offset of the launch (rows_pad * kpad * planes) fits 32 bits, so each
// store address is one uniform operand base plus a 32-bit thread offset (the fused K1)
// NOPS > 0: the node writes exactly operands 0 .. NOPS-1 and no S3 buffer (known at compile time:
// the fused K1 at depth 2, where level 1 writes S1, S2, S4, X22 and level 2 all seven)
template <int SCHEME, int YK, bool O32 = false, int NOPS = 0>
__device__ __forceinline__ void k1_core(const PreParams &P, const PreNode &N, int64_t r, int64_t c,
                                        const uint32_t (&x11a)[4], const uint32_t (&x11b)[4],
                                        const uint32_t (&x12a)[4], const uint32_t (&x12b)[4],
                                        const uint32_t (&x21a)[4], const uint32_t (&x21b)[4],
                                        const uint32_t (&x22a)[4], const uint32_t (&x22b)[4],
                                        uint32_t *s3a = nullptr, uint32_t *s3b = nullptr);

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
  } else if (fast && T == IN_U16R) {
    // the same for uint16 input (ADJ_IN_U16): 8 x 8-byte loads first, one canonical check
    const uint16_t *src = static_cast<const uint16_t *>(v.ptr);
    const int64_t o1 = r * v.ld, o2 = (P.mh + r) * v.ld;
    const int64_t offs[8] = {o1 + c, o1 + c + h2, o1 + P.kh + c, o1 + P.kh + c + h2,
                             o2 + c, o2 + c + h2, o2 + P.kh + c, o2 + P.kh + c + h2};
    uint32_t(*dst[8])[4] = {&x11a, &x11b, &x12a, &x12b, &x21a, &x21b, &x22a, &x22b};
    uint2 q[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) q[i] = __ldg(reinterpret_cast<const uint2 *>(src + offs[i]));
    uint32_t mx = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      (*dst[i])[0] = q[i].x & 0xFFFF; (*dst[i])[1] = q[i].x >> 16;
      (*dst[i])[2] = q[i].y & 0xFFFF; (*dst[i])[3] = q[i].y >> 16;
      mx = max(mx, max(max((*dst[i])[0], (*dst[i])[1]), max((*dst[i])[2], (*dst[i])[3])));
    }
    if (mx >= m.p) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) (*dst[i])[e] = mod_u32((*dst[i])[e], m);
    }
  } else if (fast && !v.e16) {
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
  k1_core<SCHEME, YK>(P, N, r, c, x11a, x11b, x12a, x12b, x21a, x21b, x22a, x22b);
}

// The arithmetic and stores of K1 at one position (row r, columns c..c+3 and c+h2..c+h2+3 of the
// quadrants) from the canonical residues of the 8 quadrant quads.  Writes the node's limb
// operands and, when N.s3 is set, its canonical S3; s3a / s3b (if given) receive the canonical
// S3 residues (the fused two-level K1 keeps them in registers for the next level).
template <int SCHEME, int YK, bool O32, int NOPS>
__device__ __forceinline__ void k1_core(const PreParams &P, const PreNode &N, int64_t r, int64_t c,
                                        const uint32_t (&x11a)[4], const uint32_t (&x11b)[4],
                                        const uint32_t (&x12a)[4], const uint32_t (&x12b)[4],
                                        const uint32_t (&x21a)[4], const uint32_t (&x21b)[4],
                                        const uint32_t (&x22a)[4], const uint32_t (&x22b)[4],
                                        uint32_t *s3a, uint32_t *s3b) {
  const ModP &m = P.mod;
  const int64_t h2 = P.kh / 2;
  {
    // One reduction per S output (modp.cuh k1_s1_s2).  Residues are carried as offset values
    // u = c + h in [0, p) of the centered c (h = (p - 1) / 2), so every correction is an unsigned
    // min of u, u - p, u + p.
    const int32_t h = (int32_t)m.half;
    const uint32_t up = m.p;
    auto wrap_lo = [&](uint32_t u) { return umin32(u, u + up); };   // u in (-p, p)
    auto wrap_hi = [&](uint32_t u) { return umin32(u, u - up); };   // u in [0, 2p)
    uint32_t u1a[4], u1b[4], u2a[4], u2b[4], u3a[4], u3b[4], u4a[4], u4b[4];
    uint32_t u11a[4], u11b[4], u12a[4], u12b[4], u22a[4], u22b[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      // S1, S2 by the host-checked helper (modp.cuh: k1_s1_s2)
      k1_s1_s2<(SCHEME >= 2), YK>(x11a[e], x11b[e], x21a[e], x21b[e], x22a[e], x22b[e], P.kc, u1a[e], u1b[e], u2a[e],
                                  u2b[e]);
      u3a[e] = wrap_lo(u1a[e] - x22a[e]); u3b[e] = wrap_lo(u1b[e] - x22b[e]);                       // S3
      u4a[e] = wrap_hi(u3a[e] + x12a[e]); u4b[e] = wrap_hi(u3b[e] + x12b[e]);                       // S4
      u11a[e] = wrap_hi(x11a[e] + h); u11b[e] = wrap_hi(x11b[e] + h);
      u12a[e] = wrap_hi(x12a[e] + h); u12b[e] = wrap_hi(x12b[e] + h);
      u22a[e] = wrap_hi(x22a[e] + h); u22b[e] = wrap_hi(x22b[e] + h);
    }
    const int64_t ps = P.plane_bytes;
    const uint32_t koff = SCHEME == 1 ? 64u + 128u * 66u - (uint32_t)h
                          : (SCHEME == 3 ? 133152u - (uint32_t)h : (uint32_t)h);   // (0, 2: h)
    // one row address per call; each operand adds its host-computed byte offset
    int8_t *const rc = P.arena + r * P.kpad + c;
    // O32 (the fused K1): the (a, b) column halves c.. and c + kh/2.. of a thread are stored side by
    // side, one 8-byte word per plane at byte 2c of the row: every limb operand of the level is
    // written with the same permutation of its K columns (4-column groups of the two halves
    // interleaved), and the leaf's sums over K do not depend on K order
    const uint32_t t0 = O32 ? (uint32_t)(r * P.kpad + 2 * c) : 0u;
    const uint32_t pst = (uint32_t)ps;
#define PUTC(o, A, B)                                                                  \
  if (O32 && SCHEME <= 2 && (NOPS > 0 ? (o) < NOPS : N.op_row[o] >= 0)) {              \
    int8_t *const ob = P.arena + N.op_off[o];                                          \
    uint32_t wa[3], wb[3];                                                             \
    limb_words_u<SCHEME>(A, koff, wa);                                                 \
    limb_words_u<SCHEME>(B, koff, wb);                                                 \
    _Pragma("unroll") for (int pl = 0; pl < (SCHEME == 0 ? 1 : (SCHEME == 1 ? 3 : 2)); ++pl) \
      st2_off32(ob, t0 + pl * pst, wa[pl], wb[pl]);                                    \
  } else if (!(O32 && SCHEME <= 2) && N.op_row[o] >= 0) {                              \
    int8_t *b = rc + N.op_off[o];                                                      \
    if constexpr (SCHEME == 0) {                                                       \
      put_limbs4_s8u(b, A, koff);                                                      \
      put_limbs4_s8u(b + h2, B, koff);                                                 \
    } else if constexpr (SCHEME == 1) {                                                \
      put_limbs4_k7u(b, ps, A, koff);                                                  \
      put_limbs4_k7u(b + h2, ps, B, koff);                                             \
    } else if constexpr (SCHEME == 2) {                                                \
      put_limbs4_s8u8u(b, ps, A, koff);                                                \
      put_limbs4_s8u8u(b + h2, ps, B, koff);                                           \
    } else {                                                                           \
      put_limbs4_t6u(b, ps, A, koff);                                                  \
      put_limbs4_t6u(b + h2, ps, B, koff);                                             \
    }                                                                                  \
  }
    PUTC(OUT_S1, u1a, u1b)
    PUTC(OUT_S2, u2a, u2b)
    PUTC(OUT_S4, u4a, u4b)
    PUTC(OUT_X22, u22a, u22b)
    PUTC(OUT_X11, u11a, u11b)
    PUTC(OUT_X12, u12a, u12b)
    PUTC(OUT_S3, u3a, u3b)
#undef PUTC
    if (NOPS > 0) {
      // no S3 buffer
    } else if (SCHEME == 3 && N.s3 != nullptr && r < P.mh) {   // canonical uint32 S3 for the next level
      uint32_t *d = static_cast<uint32_t *>(N.s3) + r * N.s3_ld;
      *reinterpret_cast<uint4 *>(d + c) = make_uint4(wrap_lo(u3a[0] - (uint32_t)h), wrap_lo(u3a[1] - (uint32_t)h),
                                                     wrap_lo(u3a[2] - (uint32_t)h), wrap_lo(u3a[3] - (uint32_t)h));
      *reinterpret_cast<uint4 *>(d + c + h2) = make_uint4(wrap_lo(u3b[0] - (uint32_t)h), wrap_lo(u3b[1] - (uint32_t)h),
                                                          wrap_lo(u3b[2] - (uint32_t)h), wrap_lo(u3b[3] - (uint32_t)h));
    } else if (N.s3 != nullptr && r < P.mh) {   // canonical S3 = (u3 - h) mod p for the next level
      uint16_t *d = static_cast<uint16_t *>(N.s3) + r * N.s3_ld;
      uint32_t v[8];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        v[e] = wrap_lo(u3a[e] - (uint32_t)h);
        v[4 + e] = wrap_lo(u3b[e] - (uint32_t)h);
      }
      *reinterpret_cast<uint2 *>(d + c) = make_uint2(v[0] | (v[1] << 16), v[2] | (v[3] << 16));
      *reinterpret_cast<uint2 *>(d + c + h2) = make_uint2(v[4] | (v[5] << 16), v[6] | (v[7] << 16));
    }
    if (s3a != nullptr) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        s3a[e] = wrap_lo(u3a[e] - (uint32_t)h);
        s3b[e] = wrap_lo(u3b[e] - (uint32_t)h);
      }
    }
  }
}

// TSEL: 0 = any input type (runtime switch per node), 1 = every node reads uint16 (caller
// ADJ_IN_U16 or workspace residues), 2 = every node reads uint32 -- the specialised instances
// carry only their own load path (less register pressure in the hot loop)
template <int SCHEME, int YK, int TSEL>
__global__ void __launch_bounds__(256, 4) preadd_kernel(const __grid_constant__ PreParams P) {
  constexpr int NP = SCHEME == 0 ? 1 : (SCHEME == 1 ? 3 : (SCHEME == 2 ? 2 : 6));
  const PreNode &N = P.nodes[blockIdx.z];
  const int64_t g_main = P.kh / 8;               // 4-column groups of the first half
  const int64_t g_pad = (P.kpad - P.kh) / 4;     // zero padding columns [kh, kpad)
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= g_main + g_pad) return;
  const int type = N.in.type;
  const int64_t nrows = range_rows(P.rows, P.rows_pad);
  for (int64_t j = blockIdx.y; j < nrows; j += gridDim.y) {
    const int64_t r = range_row(P.rows, j);
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
    if constexpr (TSEL == 1) {
      preadd_row<SCHEME, YK, IN_U16R>(P, N, r, c);   // canonical workspace residues pass its check
    } else if constexpr (TSEL == 2) {
      preadd_row<SCHEME, YK, IN_U32>(P, N, r, c);
    } else {
      if (type == IN_U32) preadd_row<SCHEME, YK, IN_U32>(P, N, r, c);
      else if (type == IN_U16) preadd_row<SCHEME, YK, IN_U16>(P, N, r, c);
      else if (type == IN_U16R) preadd_row<SCHEME, YK, IN_U16R>(P, N, r, c);
      else if (type == IN_QUAD_SUM) preadd_row<SCHEME, YK, IN_QUAD_SUM>(P, N, r, c);
      else preadd_row<SCHEME, YK, IN_PAIR_SUM>(P, N, r, c);
    }
  }
}

cudaError_t launch_preadd(const PreParams &p, cudaStream_t s) {
  if (p.n_nodes == 0) return cudaSuccess;
  const int64_t groups = p.kh / 8 + (p.kpad - p.kh) / 4;
  dim3 block(256);
  const int64_t nrows = range_rows(p.rows, p.rows_pad);
  dim3 grid((unsigned)((groups + 255) / 256), (unsigned)(nrows < 65535 ? nrows : 65535), (unsigned)p.n_nodes);
  // the specialised instance when every node of the launch reads the same storage
  bool all16 = true, all32 = true;
  for (int n = 0; n < p.n_nodes; ++n) {
    const InView &v = p.nodes[n].in;
    all16 = all16 && (v.type == IN_U16 || v.type == IN_U16R) && p.nodes[n].side == nullptr;
    all32 = all32 && v.type == IN_U32 && p.nodes[n].side == nullptr;
  }
  const int tsel = all16 ? 1 : (all32 ? 2 : 0);
#define PRE(S, Y)                                                   \
  do {                                                              \
    if (tsel == 1) preadd_kernel<S, Y, 1><<<grid, block, 0, s>>>(p); \
    else if (tsel == 2) preadd_kernel<S, Y, 2><<<grid, block, 0, s>>>(p); \
    else preadd_kernel<S, Y, 0><<<grid, block, 0, s>>>(p);          \
  } while (0)
  if (p.scheme == 0) { if (p.ykind == 0) PRE(0, 0); else PRE(0, 1); }
  else if (p.scheme == 1) { if (p.ykind == 0) PRE(1, 0); else PRE(1, 1); }
  else if (p.scheme == 2) { if (p.ykind == 0) PRE(2, 0); else PRE(2, 1); }
  else { if (p.ykind == 0) PRE(3, 0); else PRE(3, 1); }
#undef PRE
  return cudaGetLastError();
}

// ============================================================================ fused K1, levels 1 + 2
// Depth >= 2, phi = T, uint16 input (ADJ_IN_U16), p < 2^16 and exact halving without padding
// (m, k multiples of 512; api.cpp k1_fused_ok).  The quads a level-2 position (r2, c2) of the
// three level-2 nodes reads -- X11 = A11, X12 = A12 and S3 of level 1, rows {r2, r2 + mh2},
// columns {c2, c2 + kh2/2, c2 + kh2, c2 + 3 kh2/2} -- are exactly the level-1 quadrant positions
// of rows {r2, r2 + mh1/2} and columns {c2 + j kh1/4} (kh2 = kh1/2, mh2 = mh1/2).  One thread
// loads those 32 quads of A once, runs the level-1 pre-addition at its 4 positions (writing the
// level-1 limb operands), keeps the 8 S3 quads in registers and runs the level-2 pre-addition of
// the three nodes from registers: A is read once and, at depth 2, the level-1 S3 never goes
// through HBM (at depth >= 3 it is still written: level 3 reads views of it) (Alg. alg:MIAHMM
// applied twice; level 2 reads only what level 1 produced).
struct Pre2Params {
  PreParams l1, l2;
};

__device__ __forceinline__ void unpack4(uint2 q, uint32_t (&x)[4]) {
  x[0] = q.x & 0xFFFF; x[1] = q.x >> 16; x[2] = q.y & 0xFFFF; x[3] = q.y >> 16;
}
__device__ __forceinline__ uint2 pack4(const uint32_t (&x)[4]) {
  return make_uint2(x[0] | (x[1] << 16), x[2] | (x[3] << 16));
}

// D2: depth 2 (level 1 writes S1, S2, S4, X22, level 2 every operand, no S3 buffers)
template <int SCHEME, int YK, bool D2>
__global__ void __launch_bounds__(256, 2) preadd2_kernel(const __grid_constant__ Pre2Params P) {
  const PreParams &L1 = P.l1, &L2 = P.l2;
  const PreNode &N1 = L1.nodes[0];
  const int64_t kq = L1.kh / 4;               // = kh2 / 2
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (4 * g >= kq) return;
  const int64_t c2 = 4 * g;
  const uint16_t *src = static_cast<const uint16_t *>(N1.in.ptr);
  const int64_t ld = N1.in.ld;
  const ModP &m = L1.mod;
  for (int64_t r2 = blockIdx.y; r2 < L2.mh; r2 += gridDim.y) {
    uint2 q[4][2][4];   // quadrant (A11, A12, A21, A22) x row (r2, r2 + mh2) x column c2 + j kq
#pragma unroll
    for (int qd = 0; qd < 4; ++qd)
#pragma unroll
      for (int ri = 0; ri < 2; ++ri)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int64_t row = (qd >= 2 ? L1.mh : 0) + r2 + ri * L2.mh;
          const int64_t col = ((qd & 1) ? L1.kh : 0) + c2 + j * kq;
          q[qd][ri][j] = __ldg(reinterpret_cast<const uint2 *>(src + row * ld + col));
        }
    // inputs are read mod p: one packed max over the 128 values, the reducing path only if needed
    uint32_t mx = 0;
#pragma unroll
    for (int qd = 0; qd < 4; ++qd)
#pragma unroll
      for (int ri = 0; ri < 2; ++ri)
#pragma unroll
        for (int j = 0; j < 4; ++j) mx = __vmaxu2(mx, __vmaxu2(q[qd][ri][j].x, q[qd][ri][j].y));
    if (max(mx & 0xFFFF, mx >> 16) >= m.p) {
#pragma unroll
      for (int qd = 0; qd < 4; ++qd)
#pragma unroll
        for (int ri = 0; ri < 2; ++ri)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint32_t x[4];
            unpack4(q[qd][ri][j], x);
#pragma unroll
            for (int e = 0; e < 4; ++e) x[e] = mod_u32(x[e], m);
            q[qd][ri][j] = pack4(x);
          }
    }
    // level 1 at (r2 + ri mh2, c2 + j kq), j = 0, 1 (columns j + 2 are the Y partners, + kh1/2)
    uint2 s3[2][4];
#pragma unroll
    for (int ri = 0; ri < 2; ++ri)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        uint32_t x11a[4], x11b[4], x12a[4], x12b[4], x21a[4], x21b[4], x22a[4], x22b[4], sa[4], sb[4];
        unpack4(q[0][ri][j], x11a); unpack4(q[0][ri][j + 2], x11b);
        unpack4(q[1][ri][j], x12a); unpack4(q[1][ri][j + 2], x12b);
        unpack4(q[2][ri][j], x21a); unpack4(q[2][ri][j + 2], x21b);
        unpack4(q[3][ri][j], x22a); unpack4(q[3][ri][j + 2], x22b);
        k1_core<SCHEME, YK, true, D2 ? 4 : 0>(L1, N1, r2 + ri * L2.mh, c2 + j * kq, x11a, x11b, x12a, x12b, x21a, x21b, x22a, x22b,
                            sa, sb);
        s3[ri][j] = pack4(sa);
        s3[ri][j + 2] = pack4(sb);
      }
    // level 2: nodes X11 (A11), X12 (A12), S3 at (r2, c2); their quadrant quads: row ri, column j
#pragma unroll
    for (int n = 0; n < 3; ++n) {
      const uint2(&t)[2][4] = n == 0 ? q[0] : (n == 1 ? q[1] : s3);
      uint32_t x11a[4], x11b[4], x12a[4], x12b[4], x21a[4], x21b[4], x22a[4], x22b[4];
      unpack4(t[0][0], x11a); unpack4(t[0][1], x11b); unpack4(t[0][2], x12a); unpack4(t[0][3], x12b);
      unpack4(t[1][0], x21a); unpack4(t[1][1], x21b); unpack4(t[1][2], x22a); unpack4(t[1][3], x22b);
      k1_core<SCHEME, YK, true, D2 ? 7 : 0>(L2, L2.nodes[n], r2, c2, x11a, x11b, x12a, x12b, x21a, x21b, x22a, x22b);
    }
  }
}

cudaError_t launch_preadd2(const PreParams &l1, const PreParams &l2, cudaStream_t s) {
  Pre2Params p;
  p.l1 = l1;
  p.l2 = l2;
  const int64_t threads = l1.kh / 16;   // kq / 4 column groups
  dim3 grid((unsigned)((threads + 255) / 256), (unsigned)std::min<int64_t>(l2.mh, 65535), 1);
  // the depth-2 instance when the operand sets are exactly those (host-side check of the layout)
  bool d2 = l1.n_nodes == 1 && l2.n_nodes == 3 && l1.nodes[0].s3 == nullptr;
  for (int o = 0; o < OUT_N && d2; ++o) d2 = (l1.nodes[0].op_row[o] >= 0) == (o < 4);
  for (int n = 0; n < l2.n_nodes && d2; ++n) {
    d2 = l2.nodes[n].s3 == nullptr;
    for (int o = 0; o < OUT_N && d2; ++o) d2 = l2.nodes[n].op_row[o] >= 0;
  }
#define P2(S, Y)                                                                   \
  do {                                                                             \
    if (d2) preadd2_kernel<S, Y, true><<<grid, 256, 0, s>>>(p);                    \
    else preadd2_kernel<S, Y, false><<<grid, 256, 0, s>>>(p);                      \
  } while (0)
  if (l1.scheme == 0) { if (l1.ykind == 0) P2(0, 0); else P2(0, 1); }
  else if (l1.scheme == 1) { if (l1.ykind == 0) P2(1, 0); else P2(1, 1); }
  else if (l1.scheme == 2) { if (l1.ykind == 0) P2(2, 0); else P2(2, 1); }
  else return cudaErrorInvalidValue;
#undef P2
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
  const int64_t nrows = range_rows(P.row_ranges, P.rows_pad);
  for (int64_t j = blockIdx.y; j < nrows; j += gridDim.y) {
    const int64_t r = range_row(P.row_ranges, j);
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
            if (v.e16) {   // 4 uint16 components (ADJ_IN_U16)
              const uint16_t *src = static_cast<const uint16_t *>(v.ptr) + 4 * (r * v.ld + c + e);
              const uint2 h2 = vv.vec_ok ? __ldg(reinterpret_cast<const uint2 *>(src))
                                         : make_uint2((uint32_t)__ldg(src) | ((uint32_t)__ldg(src + 1) << 16),
                                                      (uint32_t)__ldg(src + 2) | ((uint32_t)__ldg(src + 3) << 16));
              w4 = make_uint4(h2.x & 0xFFFF, h2.x >> 16, h2.y & 0xFFFF, h2.y >> 16);
            } else {
              const uint32_t *src = static_cast<const uint32_t *>(v.ptr) + 4 * (r * v.ld + c + e);
              w4 = vv.vec_ok ? __ldg(reinterpret_cast<const uint4 *>(src))
                             : make_uint4(__ldg(src), __ldg(src + 1), __ldg(src + 2), __ldg(src + 3));
            }
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
__global__ void __launch_bounds__(256, 6) split_plain_kernel(const __grid_constant__ SplitParams P) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= P.kpad / 16) return;
  const int64_t c0 = g * 16;
  const int64_t ps = P.rows_pad * P.kpad;
  const InView &v = P.in;
  const int64_t nrows = range_rows(P.row_ranges, P.rows_pad);
  for (int64_t j = blockIdx.y; j < nrows; j += gridDim.y) {
    const int64_t r = range_row(P.row_ranges, j);
    InView vv = v;
    if (r >= P.rows) vv.rows_valid = 0;
    const bool fast = vv.vec_ok && r < vv.rows_valid && c0 + 15 < vv.cols_valid && c0 + 15 < P.cols;
    uint32_t x[4][4];
    if (fast && vv.type == IN_U16R && ((uintptr_t)v.ptr % 16 == 0) && (v.ld % 8 == 0)) {
      // ADJ_IN_U16: two 16-byte loads of 8 uint16 each
      const uint4 *src = reinterpret_cast<const uint4 *>(static_cast<const uint16_t *>(v.ptr) + r * v.ld + c0);
      const uint4 q0 = __ldg(src), q1 = __ldg(src + 1);
      const uint32_t w[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
      uint32_t mx = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        x[i >> 1][(i & 1) * 2] = w[i] & 0xFFFF;
        x[i >> 1][(i & 1) * 2 + 1] = w[i] >> 16;
        mx = max(mx, max(w[i] & 0xFFFF, w[i] >> 16));
      }
      if (mx >= P.mod.p) {
#pragma unroll
        for (int h = 0; h < 4; ++h)
#pragma unroll
          for (int e = 0; e < 4; ++e) x[h][e] = mod_u32(x[h][e], P.mod);
      }
    } else if (fast && vv.type == IN_U32) {
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
  const int64_t nrows = range_rows(p.row_ranges, p.rows_pad);
  const unsigned gy = (unsigned)(nrows < 65535 ? nrows : 65535);
  if (p.mode == 0) {
    dim3 g16((unsigned)((p.kpad / 16 + 255) / 256), gy);
    if (p.scheme == 0) split_plain_kernel<0><<<g16, 256, 0, s>>>(p);
    else if (p.scheme == 1) split_plain_kernel<1><<<g16, 256, 0, s>>>(p);
    else if (p.scheme == 2) split_plain_kernel<2><<<g16, 256, 0, s>>>(p);
    else split_plain_kernel<3><<<g16, 256, 0, s>>>(p);
    return cudaGetLastError();
  }
  dim3 grid((unsigned)((p.kpad / 8 + 255) / 256), gy);
  if (p.scheme == 0) split_kernel<0><<<grid, 256, 0, s>>>(p);
  else if (p.scheme == 1) split_kernel<1><<<grid, 256, 0, s>>>(p);
  else if (p.scheme == 2) split_kernel<2><<<grid, 256, 0, s>>>(p);
  else split_kernel<3><<<grid, 256, 0, s>>>(p);
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
__global__ void __launch_bounds__(256, 4) herk_preadd_kernel(const __grid_constant__ HerkPreParams P) {
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

}  // namespace adj
