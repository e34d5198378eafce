// Host prime-field constants: Legendre symbol, Tonelli-Shanks, Alg. alg:sosmodp, the
// skew-unitary Y choice and the int8 limb scheme with its int32 overflow bound.
#include "field.hpp"

namespace adj {

bool is_prime_u32(uint32_t n) {
  if (n < 2) return false;
  if (n % 2 == 0) return n == 2;
  for (uint32_t d = 3; (uint64_t)d * d <= n; d += 2)
    if (n % d == 0) return false;
  return true;
}

uint32_t powmod(uint32_t b, uint64_t e, uint32_t p) {
  uint64_t r = 1 % p, x = b % p;
  while (e) {
    if (e & 1) r = r * x % p;
    x = x * x % p;
    e >>= 1;
  }
  return (uint32_t)r;
}

int legendre(uint32_t a, uint32_t p) {
  a %= p;
  if (a == 0) return 0;
  return powmod(a, (p - 1) / 2, p) == 1 ? 1 : -1;
}

bool sqrt_mod(uint32_t a, uint32_t p, uint32_t *out) {
  a %= p;
  if (a == 0) { *out = 0; return true; }
  if (legendre(a, p) != 1) return false;
  uint64_t q = p - 1;
  int s = 0;
  while ((q & 1) == 0) { q >>= 1; s++; }
  uint32_t z = 2;
  while (legendre(z, p) != -1) z++;
  uint64_t M = s, c = powmod(z, q, p), t = powmod(a, q, p), r = powmod(a, (q + 1) / 2, p);
  while (t != 1) {
    uint64_t i = 0, t2 = t;
    while (t2 != 1) { t2 = t2 * t2 % p; i++; }
    uint64_t b = powmod((uint32_t)c, 1ull << (M - i - 1), p);
    M = i;
    c = b * b % p;
    t = t * c % p;
    r = r * b % p;
  }
  uint32_t rr = (uint32_t)r;
  *out = rr < p - rr ? rr : p - rr;
  return true;
}

void sos(uint32_t k, uint32_t p, uint32_t *a, uint32_t *b) {
  k %= p;
  uint32_t r;
  if (k == 0 || legendre(k, p) == 1) {          // k is a square: (sqrt(k), 0)
    sqrt_mod(k, p, &r);
    *a = r; *b = 0;
    return;
  }
  uint32_t s = 2;                                // lowest quadratic non-residue
  while (legendre(s, p) == 1) s++;
  uint32_t c; sqrt_mod(s - 1, p, &c);            // s - 1 is a square
  uint32_t rr = (uint32_t)((uint64_t)k * powmod(s, p - 2, p) % p);   // k s^-1
  uint32_t aa; sqrt_mod(rr, p, &aa);             // k = a^2 (1 + c^2)
  *a = aa;
  *b = (uint32_t)((uint64_t)aa * c % p);
}

SkewY skew_unitary(uint32_t p) {
  SkewY y{0, 0, 0};
  if (p % 4 == 1) {                              // Prop. lem:lemsqrt
    sqrt_mod(p - 1, p, &y.a);
    y.kind = 0;
  } else {                                       // Prop. lem:pigeonhole + Alg. 2
    sos(p - 1, p, &y.a, &y.b);
    y.kind = 1;
  }
  return y;
}

LimbScheme limb_scheme(uint32_t p) {
  if (p <= 255) return LIMB_S8;
  if (p <= 16763) return LIMB_K7;
  if (p <= 65521) return LIMB_SU8;
  return LIMB_T6;
}

int limb_planes(LimbScheme s) { return s == LIMB_S8 ? 1 : (s == LIMB_K7 ? 3 : (s == LIMB_SU8 ? 2 : 6)); }
int limb_accs(LimbScheme s) { return s == LIMB_S8 ? 1 : (s == LIMB_T6 ? 6 : 3); }

static int64_t limb_kmax_lim(LimbScheme s, uint32_t p, int64_t lim);
int64_t limb_kmax(LimbScheme s, uint32_t p) { return limb_kmax_lim(s, p, 2147483647); }
// accumulations that start from a lazy Horner value < 3p (modp.cuh mulred_lazy3)
int64_t limb_kmax_from_residue(LimbScheme s, uint32_t p) { return limb_kmax_lim(s, p, 2147483647 - 3 * (int64_t)p); }

static int64_t limb_kmax_lim(LimbScheme s, uint32_t p, int64_t lim) {
  int64_t c = (p - 1) / 2;                       // centered |x| <= c
  if (s == LIMB_S8) return lim / (c * c);
  if (s == LIMB_K7) {
    int64_t hi = (c + 64) / 128 + 1, mid = hi + 64;   // |mid| <= hi + 64 (bound)
    int64_t t = mid * mid > 64 * 64 ? mid * mid : 64 * 64;
    return lim / t;
  }
  if (s == LIMB_T6) return lim / (64 * 64);   // digit pair sums in [-64, 63]
  // SU8: lo*lo <= 255^2, cross: |hi*lo| + |lo*hi| <= 2 * 128 * 255
  int64_t t = 2 * 128 * 255;
  if (255 * 255 > t) t = 255 * 255;
  return lim / t;
}

}  // namespace adj
