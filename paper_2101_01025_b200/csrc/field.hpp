// Host-side prime-field constants for the CUDA path (a0 "Plan").
// Independent of oracle/ (no shared code).
#pragma once
#include <cstdint>

namespace adj {

bool is_prime_u32(uint32_t n);
uint32_t powmod(uint32_t b, uint64_t e, uint32_t p);
int legendre(uint32_t a, uint32_t p);            // Euler's criterion
bool sqrt_mod(uint32_t a, uint32_t p, uint32_t *r); // Tonelli-Shanks, returns min(r, p-r)
// Alg. alg:sosmodp: a^2 + b^2 = k mod p
void sos(uint32_t k, uint32_t p, uint32_t *a, uint32_t *b);

// Skew-unitary Y: kind 0 = scalar i (Y = i I), kind 1 = Rot2 [[a,b],[-b,a]] (x) I.
struct SkewY {
  int kind;
  uint32_t a, b;
};
SkewY skew_unitary(uint32_t p);

// int8 limb schemes
enum LimbScheme : int {
  LIMB_S8 = 0,   // p <= 255: one signed limb, centered residue
  LIMB_K7 = 1,   // p <= 16763: balanced base 2^7 (hi, lo, mid = hi + lo), Karatsuba, 3 accumulators
  LIMB_SU8 = 2,  // p <= 65521: hi = floor(c/256) signed, lo = c - 256 hi unsigned; 4 MMAs, 3 accumulators
  LIMB_T6 = 3,   // p < 2^18: three balanced base-64 digits (d2, d1, d0) + the pair sums d2+d1, d1+d0,
                 // d2+d0 (all s8); 3-way Karatsuba: 6 MMAs, 6 accumulators
};
constexpr uint32_t kMaxModulus = 262139;   // largest prime below 2^18
LimbScheme limb_scheme(uint32_t p);
int limb_planes(LimbScheme s);       // int8 planes per operand
int limb_accs(LimbScheme s);         // TMEM accumulators per output tile
// largest inner dimension one int32 accumulation segment may take without overflow
int64_t limb_kmax(LimbScheme s, uint32_t p);
// the same bound when every accumulation starts from a residue < p (the wide-N leaf's Horner
// values in TMEM): k * max|term| + p <= 2^31 - 1
int64_t limb_kmax_from_residue(LimbScheme s, uint32_t p);

}  // namespace adj
