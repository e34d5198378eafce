// Launch-parameter structs shared by the host scheduler (api.cpp / plan.cpp) and the kernels.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "modp.cuh"

namespace adj {

constexpr int kMaxMaps = 4;        // one TMA map per operand arena (levels 0..3)
constexpr int kMaxProducts = 64;   // leaf products in one grouped launch (depth <= 3)
constexpr int kMaxNodes = 32;      // recursion nodes per level in one batched launch
constexpr int kMaxRowRanges = 8;   // output-tile sharding: row ranges a rank's K1 / split covers
constexpr int kBM = 128;           // UMMA M / tile rows
constexpr int kBK = 128;           // bytes of K per pipeline stage (one 128B swizzle atom)

// ---------------------------------------------------------------- leaf (K2/K3) products
struct LeafProduct {
  int32_t map;           // arena / tensor-map index
  int32_t a_row0;        // row of plane 0 of operand A inside the arena
  int32_t b_row0;        // row of plane 0 of operand B
  int32_t a_plane_rows;  // rows between consecutive limb planes of A
  int32_t b_plane_rows;
  int32_t kblocks;       // K / 128
  int32_t sym;           // 1: SYRK leaf, only tiles/elements with col <= row are written
  int32_t out_u32;       // 1: uint32 output, 0: uint16
  int32_t out_rows;      // writes masked to row < out_rows, col < out_cols
  int32_t out_cols;
  int32_t vec_ok;        // 16-byte vector stores allowed (alignment checked on host)
  int32_t kseg;          // k-blocks per int32 accumulation segment (>= kblocks: one segment)
  int64_t ldo;           // output leading dimension (elements)
  void *out;
  uint32_t alpha, beta;  // axpby: out <- alpha v + beta out (mod p), SYRK form (uint32 outputs only)
  int32_t axpby, pad2_;
};

struct LeafTerm {        // one tcgen05.mma operand pair accumulated into accumulator `acc`
  int8_t acc, a_plane, b_plane, a_signed, b_signed, pad_[3];
};

struct LeafParams {
  CUtensorMap maps[kMaxMaps];
  CUtensorMap maps_half[kMaxMaps];   // the same arenas with 64-row boxes: B operand of N = 128 tail jobs
  LeafProduct prod[kMaxProducts];
  // jobs: .x = product << 24 | I << 12 | J (longest-K products first);
  //       .y = 0 for a whole tile; kb0 | kb1 << 12 | piece << 24: a K-range piece of a tail
  //       tile whose residue partial goes to fixup slot piece-1 (summed by the fixup kernel);
  //       h << 24 | 0xFFFFFF: column half h (N = 128, whole K) of a tail tile, written directly
  const uint2 *tiles;
  int32_t n_tiles;
  void *fixup;             // 256 x 256 residue partials (u16, or u32 if fixup32), one slot per tail piece
  int32_t n_terms;
  int32_t acc_begin[8];    // terms [acc_begin[j], acc_begin[j+1]) accumulate into accumulator j
  LeafTerm terms[8];
  uint32_t weight[6];      // residue weight of each accumulator in the limb recombination
  ShoupW wshoup[6];        // the same weights as Shoup pairs (centered weight, floor(w 2^32 / p))
  ShoupW hshoup[6];        // wide-N leaf (Horner in TMEM): w_j / w_{j+1} mod p, the step to the next accumulator
  ShoupW one;              // Shoup pair of 1 (the step between K segments of one accumulator)
  int32_t fixup32;         // fixup slots hold uint32 residues (p > 2^16) instead of uint16
  int32_t *job_counter;    // dynamic scheduling: next job index (zeroed before the launch); null = static
  int32_t debug;           // diagnostics only (ADJ_LEAF_DEBUG): 1 no TMA, 2 no epilogue, 8 no math, 16 no tcgen05.ld,
                           // 32 no stores, 128 per-role cycle profile, 256 A operand only, 16384 cluster exit times
  int32_t gate;            // wide leaf, dynamic: claim-wave gate (api.cpp launch_leaf_all): 1000 + g = a job is
                           // claimed when it starts and claim wave w starts once g % of wave w - 1 has issued
                           // its loads (job_counter[1] counts them); 1..100 = the same with claims two ahead;
                           // -1 = claim at start without a gate; 0 = neither
  int32_t kalt;            // odd units of a job walk K backwards (a unit starts on the k-blocks the previous
                           // one loaded last, still in L2); api.cpp launch_leaf_all
  int32_t gate_pre;        // wide leaf: stages of a gated job issued before its gate wait (soft gate)
  int32_t pad_gp;
  ModP mod;
};

// tail tiles split along K into pieces (fixup_kernel sums them into the product output)
struct FixupTile {
  int32_t q, I, J, slot0, npieces, pad_;
};

// ---------------------------------------------------------------- K1 pre-addition
enum InType : int32_t { IN_U32 = 0, IN_U16 = 1, IN_PAIR_SUM = 2, IN_PAIR_RE = 3, IN_PAIR_IM = 4,
                        IN_QUAD_SUM = 5 /* quaternion x1 + x2 + x3 + x4 (Q6's W = U1 + U2, Alg. alg:2M3M) */,
                        IN_U16R = 6     /* caller's uint16 input (ADJ_IN_U16): reduced mod p like IN_U32 */ };

struct InView {          // a (possibly padded) view of a node's input matrix
  const void *ptr;
  int64_t ld;            // elements (pairs for IN_PAIR_*)
  int64_t rows_valid, cols_valid;
  int32_t type;
  int32_t vec_ok;        // 16-byte aligned rows -> vector loads allowed
  int32_t e16;           // IN_PAIR_*: (re, im) pairs of uint16 (ADJ_IN_U16) instead of uint32
  int32_t pad_;
};

// S1, S2, S4, X22 (GEMM operands), X11, X12, S3 (SYRK leaves when the level is the last)
enum PreOut : int { OUT_S1 = 0, OUT_S2, OUT_S4, OUT_X22, OUT_X11, OUT_X12, OUT_S3, OUT_N };

struct PreNode {
  InView in;
  int64_t op_row[OUT_N];   // arena row of plane 0 for each output operand; -1 = not produced
  int64_t op_off[OUT_N];   // the same as a byte offset, op_row * kpad (host-computed)
  void *s3;                // materialised S3 residues (when S3 recurses), else null (u16 / u32 if res32)
  int64_t s3_ld;
  // 2M side output (root node, IN_PAIR_SUM input): limb planes of X = Re(A) and Y = Im(A) for
  // the general product H = X Y^T, written from the same read of A as the pre-addition of T.
  int8_t *side;            // arena 0 or null
  int64_t side_kpad, side_rows_pad, side_x_row, side_y_row;
};

// rows [0, rows_pad) of the arena (n = 0) or only the listed ranges (output-tile sharding)
struct RowRanges {
  int32_t n, pad_;
  int64_t lo[kMaxRowRanges], hi[kMaxRowRanges];
};

struct PreParams {
  PreNode nodes[kMaxNodes];
  RowRanges rows;
  int32_t n_nodes;
  int32_t scheme, planes;
  int32_t ykind;           // 0: Y = i I ; 1: Y = [[a,b],[-b,a]] (x) I
  uint32_t ya, yb;
  int64_t mh, kh;          // half sizes (node input is 2 mh x 2 kh, zero padded)
  int64_t rows_pad;        // rows per plane in the arena (>= mh, multiple of 128)
  int64_t kpad;            // arena row length in bytes (>= kh, multiple of 128)
  int64_t plane_bytes;     // rows_pad * kpad (host-computed)
  int8_t *arena;
  int32_t res32;           // workspace residues are uint32 (p > 2^16)
  int32_t pad_;
  ModP mod;
  K1Const kc;              // S1 / S2 reduction constants (modp.cuh k1_s1_s2)
};

// plain limb split of a view into arena planes (depth 0, gemm_modp, 2M's X / Y)
struct SplitParams {
  InView in;
  RowRanges row_ranges;
  int64_t rows, cols;      // logical size (>= valid); padding written as zero
  int64_t rows_pad, kpad;
  int64_t op_row;
  int64_t op_row2, op_row3;  // mode 1 (2M): Y = Im(A) and T = Re + Im planes
  int8_t *arena;
  int32_t scheme, planes;
  int32_t mode;              // 0: plain split of `in`; 1: 2M split of interleaved pairs;
                             // 2: quaternion split (Alg. alg:2M3M operands A, B, C, D, U1, U2, W)
  int64_t qrow[7];           // mode 2: arena rows of the QuatOp operands (-1 = not written)
  ModP mod;
};

// ---------------------------------------------------------------- K4 recombination
struct CombNode {
  const void *P[5];        // P1..P5 (index 0..4), each rows_pad x rows_pad, ld = ldp (u16, or u32 if in32)
  void *out;
  int64_t ldo;
  int64_t out_valid;       // output is out_valid x out_valid (<= 2 mh); only Low written
};

struct CombParams {
  CombNode nodes[kMaxNodes];
  int32_t n_nodes;
  int32_t out_u32;
  int64_t mh, ldp;
  ModP mod;
  uint32_t alpha, beta;    // axpby on the final (uint32) output, SYRK form
  int32_t axpby;
  int32_t in32;            // P buffers hold uint32 residues (p > 2^16)
  const uint32_t *pairs;   // output-tile sharding: the (ti << 16 | tj) lower tile pairs to do (else all)
  int32_t n_pairs;
  int32_t inplace;         // low-memory schedule: P1, P3, P5 read from out's C11, C21, C22 blocks
};

// ---------------------------------------------------------------- GF(p^2) Alg. 1 (PLAN_HERK1)
// PLAN_HERK1: one level of Alg. alg:MIAHMM directly over GF(p^2) with Y = (a + ib) I (PAPER.md
// §4.4, 741-758); its Hermitian leaves P1, P2, P5 by 2M (G = T T^T, H = X Y^T) and its general
// leaves P3, P4 by 3M (t1 = Xr Yr^T, t2 = Xi Yi^T, t3 = (Xr + Xi)(Yr - Yi)^T).  Operands (one
// arena, in this order) and product buffers:
enum HerkOp : int {
  HO_T11 = 0, HO_X11, HO_Y11, HO_T12, HO_X12, HO_Y12, HO_T3, HO_X3, HO_Y3,   // A11, A12, S3: T = re + im, X = re, Y = im
  HO_X22, HO_Y22, HO_Z22, HO_X4, HO_Y4, HO_W4,                              // A22 (Z = re + im), S4 (W = re - im)
  HO_X1, HO_Y1, HO_Z1, HO_X2, HO_Y2, HO_W2,                                 // S1 (Z), S2 (W)
  HO_N
};
enum HerkBuf : int { HB_G1 = 0, HB_H1, HB_G2, HB_H2, HB_G5, HB_H5, HB_A1, HB_A2, HB_A3, HB_B1, HB_B2, HB_B3, HB_N };
// K1 over GF(p^2): S1 = y (A21 - A11), S2 = A22 - y A21, S3 = S1 - A22, S4 = S3 + A12 with the
// scalar y = ya + i yb (Y = y I, y conj(y) = -1), written as the 21 HerkOp limb operands.
struct HerkPreParams {
  InView in;               // A, IN_PAIR_RE type (interleaved (re, im) uint32 pairs), m x k valid
  int64_t mh, kh;          // half sizes (A is zero padded to 2 mh x 2 kh)
  int64_t rows_pad, kpad;
  int8_t *arena;
  int32_t scheme, planes;
  uint32_t ya, yb;
  ModP mod;
};
// K4 over GF(p^2) fused with the 2M / 3M leaf combinations (HerkBuf order in B[]).
struct HerkCombParams {
  const void *B[12];       // rows_pad x rows_pad residue buffers (u16, or u32 if in32), ld = ldp
  int64_t mh, ldp;
  uint32_t *C;             // interleaved (re, im) pairs, ldc in pairs
  int64_t ldc, out_valid;
  ModP mod;
  uint32_t alpha, beta;
  int32_t axpby, in32;
};

// ---------------------------------------------------------------- quaternion 6M combine (PLAN_QUAT)
struct QuatCombParams {
  const void *Q[6];        // Q1..Q5 (full), Q6 (Low): rows_pad x rows_pad residues (u16, or u32 if in32), ld = ldq
  int64_t m, ldq;
  uint32_t *C;             // 4 interleaved components per quaternion, ldc in quaternions
  int64_t ldc;
  ModP mod;
  uint32_t alpha, beta;
  int32_t axpby, in32;
  int32_t out16, pad_;     // ADJ_OUT_U16: C holds 4 uint16 components per quaternion
};

// ---------------------------------------------------------------- output-tile sharding: pack / unpack
struct RectDev {
  int64_t r0, c0, rows, cols;  // region of C (uint32 residues)
  int64_t off;                 // element offset of its rows x cols block in the packed buffer
  int32_t lower, pad_;         // lower: only col <= row is copied back into C
};

}  // namespace adj
