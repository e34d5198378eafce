// Modular arithmetic and int8 limb splitting shared by the host planner and the kernels of
// the CUDA path (not shared with oracle/).
#pragma once
#include <cmath>
#include <cstdint>

#ifndef __CUDACC__
#define __host__
#define __device__
#define __forceinline__ inline
#endif

namespace adj {

// Barrett constants for an odd prime p < 2^18.  mulmod() needs residue products < 2^32
// (p <= 65521); mulmod_w() is the 64-bit version for the wide limb scheme.
struct ModP {
  uint32_t p;
  uint32_t mu;   // floor(2^32 / p)
  uint32_t c32;  // 2^32 mod p
  uint32_t half; // (p - 1) / 2 : centered representative threshold
  uint64_t mu64; // floor(2^64 / p) (computed as floor((2^64 - 1) / p); p is odd so it is the same)
};

inline ModP make_modp(uint32_t p) {
  ModP m;
  m.p = p;
  m.mu = (uint32_t)((1ull << 32) / p);
  m.c32 = (uint32_t)((1ull << 32) % p);
  m.half = (p - 1) / 2;
  m.mu64 = ~0ull / p;
  return m;
}

__host__ __device__ __forceinline__ uint32_t umin32(uint32_t a, uint32_t b) { return a < b ? a : b; }
// x mod p for any 32-bit x: q = umulhi(x, mu) underestimates floor(x/p) by at most 1.
__host__ __device__ __forceinline__ uint32_t mod_u32(uint32_t x, const ModP &m) {
#ifdef __CUDA_ARCH__
  uint32_t q = __umulhi(x, m.mu);
#else
  uint32_t q = (uint32_t)(((uint64_t)x * m.mu) >> 32);
#endif
  uint32_t r = x - q * m.p;
  return umin32(r, r - m.p);   // r < 2p: r - p wraps above r unless r >= p
}
// signed 32-bit -> [0, p): reduce the two's-complement bits, then remove 2^32 if x < 0
__host__ __device__ __forceinline__ uint32_t mod_s32(int32_t x, const ModP &m) {
  uint32_t r = mod_u32((uint32_t)x, m);
  if (x < 0) r = r >= m.c32 ? r - m.c32 : r + m.p - m.c32;
  return r;
}
__host__ __device__ __forceinline__ uint32_t mulmod(uint32_t a, uint32_t b, const ModP &m) {
  return mod_u32(a * b, m);  // a, b < p < 2^16
}
// a * b mod p for residues a, b < p < 2^32 (64-bit product, 64-bit Barrett, one correction)
__host__ __device__ __forceinline__ uint32_t mulmod_w(uint32_t a, uint32_t b, const ModP &m) {
  const uint64_t x = (uint64_t)a * b;
#ifdef __CUDA_ARCH__
  const uint64_t q = __umul64hi(x, m.mu64);
#else
  const uint64_t q = (uint64_t)(((unsigned __int128)x * m.mu64) >> 64);
#endif
  uint64_t r = x - q * m.p;
  return (uint32_t)(r >= m.p ? r - m.p : r);
}
// mulmod for any supported p (runtime choice; for cold paths)
__host__ __device__ __forceinline__ uint32_t mulmod_any(uint32_t a, uint32_t b, const ModP &m) {
  return m.p > 65535u ? mulmod_w(a, b, m) : mulmod(a, b, m);
}
// (unsigned-min forms: one VIMNMX instead of a compare and a select)
__host__ __device__ __forceinline__ uint32_t addmod(uint32_t a, uint32_t b, const ModP &m) {
  const uint32_t s = a + b;
  return umin32(s, s - m.p);
}
__host__ __device__ __forceinline__ uint32_t submod(uint32_t a, uint32_t b, const ModP &m) {
  const uint32_t d = a - b;
  return umin32(d, d + m.p);
}
// centered representative in [-(p-1)/2, (p-1)/2]
__host__ __device__ __forceinline__ int32_t centered(uint32_t x, const ModP &m) {
  return x > m.half ? (int32_t)x - (int32_t)m.p : (int32_t)x;
}

// Shoup multiplication by a fixed weight, fused with the accumulation into a residue partial.
// The weight is kept centered, wc in [-(p-1)/2, (p-1)/2], with wq = floor(wc * 2^32 / p) (floor
// toward -inf), so |wq| < 2^31.  For any int32 x: q = mulhi_s32(x, wq) is within 1 of
// floor(x wc / p) (|x (wc 2^32/p - wq)| / 2^32 < 1/2), so r = x wc - q p lies in [-p, 2p) and is
// computed exactly in wrapping 32-bit arithmetic.  acc_mulred returns (part + x w) mod p for a
// residue part < p: s = part + r + p in [0, 4p) (needs 4p < 2^32), then two unsigned min-subtracts.
struct ShoupW {
  int32_t wc, wq;
};
inline ShoupW make_shoup(uint32_t w, uint32_t p) {
  ShoupW s;
  w %= p;
  s.wc = w > (p - 1) / 2 ? (int32_t)w - (int32_t)p : (int32_t)w;
  const int64_t num = (int64_t)s.wc * ((int64_t)1 << 32);
  int64_t q = num / (int64_t)p;
  if (num % (int64_t)p != 0 && num < 0) --q;   // floor
  s.wq = (int32_t)q;
  return s;
}
__host__ __device__ __forceinline__ uint32_t acc_mulred(int32_t x, int32_t wc, int32_t wq, uint32_t part, uint32_t p) {
#ifdef __CUDA_ARCH__
  const int32_t q = __mulhi(x, wq);
#else
  const int32_t q = (int32_t)(((int64_t)x * (int64_t)wq) >> 32);
#endif
  const uint32_t r = (uint32_t)x * (uint32_t)wc - (uint32_t)q * p;
  uint32_t s = part + r + p;
  s = umin32(s, s - 2 * p);
  return umin32(s, s - p);
}

// The same Shoup step without the final corrections (part = 0): x w mod p + {0, p, 2p}, a value
// in [0, 3p) (r = x wc - q p lies in [-p, 2p)).  The wide leaf's intermediate Horner steps keep
// it in TMEM: the next unit accumulates on top of it (K segments bounded for a start < 3p,
// field.cpp limb_kmax_from_residue), and only the last step of a tile reduces fully.
__host__ __device__ __forceinline__ uint32_t mulred_lazy3(int32_t x, int32_t wc, int32_t wq, uint32_t p) {
#ifdef __CUDA_ARCH__
  const int32_t q = __mulhi(x, wq);
#else
  const int32_t q = (int32_t)(((int64_t)x * (int64_t)wq) >> 32);
#endif
  return (uint32_t)x * (uint32_t)wc - (uint32_t)q * p + p;
}

// ---- K1's lazy reduction of the Y products for p > 16763 (preadd.cu) ----------
// The products' sum v (|v| < 2 p^2 < 2^37 for p < 2^18) is carried exactly mod 2^32 (wrapping
// uint32 arithmetic) and approximately in float (vf, relative error a few 2^-24).  The float
// quotient estimate q = rn(vf / p) is then within ~0.6 of v / p, so u = v + h - q p, a value in
// (-p, 2p), is exact in wrapping 32-bit arithmetic and two unsigned mins give the offset residue
// (v + h) mod p in [0, p) (h = (p - 1) / 2: u - h is the centered residue of v).  Host-checked over
// extreme and random inputs of every scheme above 16763 (tests/test_host_modp.py).
__host__ __device__ __forceinline__ int32_t f2i_rn(float x) {
#ifdef __CUDA_ARCH__
  return __float2int_rn(x);
#else
  return (int32_t)std::nearbyintf(x);   // round half to even in the default FP environment
#endif
}
__host__ __device__ __forceinline__ float lazy_invp(uint32_t p) { return 1.0f / (float)p; }
__host__ __device__ __forceinline__ uint32_t lazy_off(uint32_t v_bits, float vf, float invp, uint32_t p, uint32_t h) {
  const int32_t q = f2i_rn(vf * invp);
  const uint32_t u = v_bits + h - (uint32_t)q * p;
  return umin32(umin32(u, u - p), u + p);
}
// K1 constants of one prime and skew-unitary Y (host-made, passed to the kernel)
struct K1Const {
  ModP mod;
  uint32_t ya, yb;     // Y = ya I (YK = 0) or Rot2(ya, yb) (YK = 1)
  uint32_t bias;       // p <= 16763: h + p (2p + 1) -- makes every exact int32 v of S1 / S2 non-negative
  float invp;          // p > 16763, Rot2: float quotient estimate
  ShoupW ya_w, nya_w;  // p > 16763, Y = ya I: Shoup weights of ya and -ya
};
inline K1Const make_k1const(uint32_t p, uint32_t ya, uint32_t yb) {
  K1Const k;
  k.mod = make_modp(p);
  k.ya = ya;
  k.yb = yb;
  k.bias = (uint32_t)((p - 1) / 2 + (uint64_t)p * (2ull * p + 1));
  k.invp = lazy_invp(p);
  k.ya_w = make_shoup(ya, p);
  k.nya_w = make_shoup((p - ya % p) % p, p);
  return k;
}

// S1 = (A21 - A11) Y and S2 = A22 - A21 Y as offset residues (v + h) mod p,
// h = (p - 1) / 2, for canonical inputs x < p: YK = 0, Y = ya I (the two lanes a / b
// independent); YK = 1, Y = Rot2(ya, yb) on the column pair (j, j + k/4): [X1 X2] Y =
// [a X1 - b X2, b X1 + a X2].  Three reductions, by prime range:
//   WIDE = false (p <= 16763, 2 p^2 + p < 2^30): v exact in int32, (v + bias) mod p by mod_u32
//     (bias = h + p (2p + 1) keeps v + bias in [0, 2^31));
//   WIDE, YK = 0: one Shoup step per output (acc_mulred: (part + x w) mod p for any int32 x);
//   WIDE, YK = 1: v exact mod 2^32 plus the float quotient estimate (lazy_off).
// Host-checked over extreme and random inputs (tests/test_host_modp.py).
template <bool WIDE, int YK>
__host__ __device__ __forceinline__ void k1_s1_s2(uint32_t x11a, uint32_t x11b, uint32_t x21a, uint32_t x21b,
                                                  uint32_t x22a, uint32_t x22b, const K1Const &kc, uint32_t &s1a,
                                                  uint32_t &s1b, uint32_t &s2a, uint32_t &s2b) {
  const uint32_t p = kc.mod.p, h = kc.mod.half, ya = kc.ya, yb = kc.yb;
  const int32_t d1 = (int32_t)x21a - (int32_t)x11a, d2 = (int32_t)x21b - (int32_t)x11b;
  const uint32_t ud1 = (uint32_t)d1, ud2 = (uint32_t)d2;
  if (!WIDE) {
    if (YK == 0) {
      s1a = mod_u32(ya * ud1 + kc.bias, kc.mod);
      s1b = mod_u32(ya * ud2 + kc.bias, kc.mod);
      s2a = mod_u32(x22a - ya * x21a + kc.bias, kc.mod);
      s2b = mod_u32(x22b - ya * x21b + kc.bias, kc.mod);
    } else {
      s1a = mod_u32(ya * ud1 - yb * ud2 + kc.bias, kc.mod);
      s1b = mod_u32(yb * ud1 + ya * ud2 + kc.bias, kc.mod);
      s2a = mod_u32(x22a - (ya * x21a - yb * x21b) + kc.bias, kc.mod);
      s2b = mod_u32(x22b - (yb * x21a + ya * x21b) + kc.bias, kc.mod);
    }
  } else if (YK == 0) {
    const uint32_t u22a = umin32(x22a + h, x22a + h - p), u22b = umin32(x22b + h, x22b + h - p);
    s1a = acc_mulred(d1, kc.ya_w.wc, kc.ya_w.wq, h, p);
    s1b = acc_mulred(d2, kc.ya_w.wc, kc.ya_w.wq, h, p);
    s2a = acc_mulred((int32_t)x21a, kc.nya_w.wc, kc.nya_w.wq, u22a, p);
    s2b = acc_mulred((int32_t)x21b, kc.nya_w.wc, kc.nya_w.wq, u22b, p);
  } else {
    const float invp = kc.invp;
    const float yaf = (float)ya, ybf = (float)yb, d1f = (float)d1, d2f = (float)d2;
    const float x21af = (float)x21a, x21bf = (float)x21b, x22af = (float)x22a, x22bf = (float)x22b;
    s1a = lazy_off(ya * ud1 - yb * ud2, fmaf(yaf, d1f, -(ybf * d2f)), invp, p, h);
    s1b = lazy_off(yb * ud1 + ya * ud2, fmaf(ybf, d1f, yaf * d2f), invp, p, h);
    const float trfa = fmaf(yaf, x21af, -(ybf * x21bf)), trfb = fmaf(ybf, x21af, yaf * x21bf);
    s2a = lazy_off(x22a - (ya * x21a - yb * x21b), x22af - trfa, invp, p, h);
    s2b = lazy_off(x22b - (yb * x21a + ya * x21b), x22bf - trfb, invp, p, h);
  }
}

// int8 limb split of a canonical residue:
//   scheme 0 (p <= 255)    : l0 = c                                    (s8)
//   scheme 1 (p <= 16763)  : hi = floor((c+64)/128), lo = c - 128 hi, mid = hi + lo  (all s8)
//   scheme 2 (p <= 65521)  : hi = floor(c/256) (s8), lo = c - 256 hi in [0,255] (u8)
// Returns limbs packed as bytes: byte0 = plane 0, byte1 = plane 1, byte2 = plane 2.
__host__ __device__ __forceinline__ uint32_t limb_split(uint32_t x, int scheme, const ModP &m) {
  int32_t c = centered(x, m);
  if (scheme == 0) return (uint32_t)(uint8_t)(int8_t)c;
  if (scheme == 1) {
    int32_t hi = (c + 64) >> 7;
    int32_t lo = c - (hi << 7);
    int32_t mid = hi + lo;
    return (uint32_t)(uint8_t)(int8_t)hi | ((uint32_t)(uint8_t)(int8_t)lo << 8) |
           ((uint32_t)(uint8_t)(int8_t)mid << 16);
  }
  int32_t hi = c >> 8;
  int32_t lo = c - (hi << 8);
  return (uint32_t)(uint8_t)(int8_t)hi | ((uint32_t)(uint8_t)lo << 8);
}

}  // namespace adj
