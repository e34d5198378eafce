// Recursion planner for Alg. alg:MIAHMM on the GPU (a0 "Plan" + a3 "Recurse").
//
// A plan is the static part of a call: level sizes, workspace layout, the list of leaf
// products (P3, P4 at every level; P1, P2, P5 at the last level) and the packed tile list of
// the single grouped leaf launch.  Pointers are bound per call (bind()).
#pragma once
#include <cstddef>
#include <cstdint>
#include <utility>
#include <vector>

#include "field.hpp"
#include "types.hpp"

namespace adj {

enum PlanKind : int { PLAN_SYRK_T = 0, PLAN_SYRK_H = 1, PLAN_GEMM = 2, PLAN_HERK1 = 3, PLAN_QUAT = 4,
                      PLAN_LOWMEM = 5 /* root level of the low-memory schedule (phi = T, ADJ_LOW_MEM) */ };

// PLAN_QUAT (phi = quaternion conjugate transpose, Alg. alg:2M3M): arena-0 operands
enum QuatOp : int { QO_A = 0, QO_B, QO_C, QO_D, QO_U1, QO_U2, QO_W, QO_N };


struct ShardRect {
  int64_t r0, c0, rows, cols;
  int lower;             // only elements with col <= row belong to the shard
};

struct ArenaPlan {
  int64_t kpad = 0;      // bytes per row (K padded to 128)
  int64_t n_rows = 0;    // total rows (all operands x planes)
  size_t offset = 0;     // byte offset in the workspace
  size_t bytes() const { return (size_t)kpad * (size_t)n_rows; }
};

struct LevelPlan {
  int64_t mh = 0, kh = 0;       // half sizes at this level
  int64_t rows_pad = 0, kpad = 0;
  int n_nodes = 0, n_ops = 0;   // nodes at this level, operands per node in the arena
  int arena = -1;
  size_t s3_offset = 0, s3_node_bytes = 0;   // materialised S3 (levels < depth)
  size_t p_offset = 0, p_buf_bytes = 0;      // P1..P5 per node, rows_pad^2 uint16 each
};

// leaf product whose output pointer is resolved at bind time
enum OutTarget : int { OUT_PBUF = 0, OUT_C = 1, OUT_HBUF = 2, OUT_GBUF = 3, OUT_QBUF = 4,
                       OUT_C21 = 5 /* low-memory root: P3 into C's C21 block */,
                       OUT_LMP4 = 6 /* low-memory root: P4 buffer */ };
struct ProductPlan {
  LeafProduct lp;        // everything except `out` (and ldo for OUT_C)
  int target;            // OutTarget
  int level, node, idx;  // for OUT_PBUF
};

struct Plan {
  PlanKind kind;
  int64_t m = 0, n = 0, k = 0;   // SYRK: A is m x k, C m x m; GEMM: A m x k, B n x k, C m x n
  uint32_t p = 0;
  int depth = 0;
  LimbScheme scheme;
  int planes = 1, nacc = 1, bn = 128;
  int tile_m = 256, tile_n = 256;  // CTA-pair output tile (leaf2_kernel)
  int kseg = 1;                    // k-blocks per int32 accumulation segment (limb k_max / 128)
  bool segmented = false;          // some leaf product needs more than one K segment
  bool res32 = false;              // workspace residues (P, S3, G, H, fixup) are uint32 (p > 2^16)
  int res_bytes() const { return res32 ? 4 : 2; }
  ModP mod;
  SkewY Y;
  std::vector<ArenaPlan> arenas;
  std::vector<LevelPlan> lv;      // lv[0] = the input level (mh = m, kh = k); lv[1..depth]
  // depth-0 / 2M / gemm operands living in arena 0
  int64_t rows_pad0 = 0, kpad0 = 0, rows_pad_b = 0;
  int64_t op0_row[3] = {-1, -1, -1};  // SYRK_T d=0: A; SYRK_H: X, Y, (T if d==0); GEMM: A, B
  size_t h_offset = 0, g_offset = 0;  // 2M buffers H, G (uint16 rows_pad0^2)
  size_t hb_offset = 0, hb_bytes = 0; // PLAN_HERK1: HB_N product buffers of lv[1].rows_pad^2 residues
  size_t q_offset = 0, q_bytes = 0;   // PLAN_QUAT: Q1..Q5 (rows_pad0^2 residues each); Q6 in g_offset
  int64_t q_row[QO_N] = {-1, -1, -1, -1, -1, -1, -1};   // PLAN_QUAT arena-0 operand rows
  size_t ws_bytes = 0;
  std::vector<ProductPlan> prods;
  std::vector<uint32_t> tiles;       // 2 words per leaf job (LeafParams::tiles)
  uint32_t *d_tiles = nullptr;       // device copy (owned by the plan cache)
  std::vector<FixupTile> fixups;     // tail tiles split along K into pieces
  FixupTile *d_fixups = nullptr;
  size_t fixup_offset = 0;           // workspace offset of the 256x256 u16 piece slots
  size_t counter_offset = 0;         // workspace offset of the leaf's dynamic job counter
  int n_pieces = 0;
  int grid = 1;
  bool dynamic = false;              // leaf jobs claimed with an atomic counter (long launches)
  bool wide = false;                 // 256 x 512 leaf tiles (leafw_kernel, Horner recombination in TMEM)
  int dev = 0;
  LeafParams leaf_template;           // terms, weights, mod (maps/outs bound per call)
  // output-tile sharding (adjprod_modp_shard): this plan computes only the tiles `shard_rank` owns
  int shard_rank = -1, shard_n = 0;
  std::vector<ShardRect> shard_rects;  // the regions of C it writes (Low part when `lower`)
  std::vector<std::pair<int64_t, int64_t>> shard_rows;   // [r0, r1) rows of the top level's operands its tiles read
  std::vector<uint32_t> comb_pairs;    // depth 1: K4 64 x 64 lower tile pairs (ti << 16 | tj)
  uint32_t *d_comb_pairs = nullptr;
  // PLAN_LOWMEM: the root level of Alg. alg:MIAHMM only (depth = 1 here; the call's
  // depth is lm_depth).  K1 writes S1, S2, S4, A22 and materialises S3; one leaf launch writes
  // P3 into C21 and P4 into a buffer; then the children X11, X12, S3 run as ordinary calls of
  // depth lm_depth - 1 whose Low results land in C11, a P2 buffer and C22; K4 runs in place.
  // Workspace: [S3 | P2 | P4 | region], the region holding the root's arena and then, reused,
  // the children's workspace.
  int lm_depth = 0;
  size_t lm_p2_off = 0, lm_p4_off = 0, lm_region_off = 0, lm_child_ws = 0;
};

// Build (host only, no CUDA calls).  Returns false with *err set if unsupported.
bool build_syrk_plan(Plan &P, int64_t m, int64_t k, uint32_t p, int phi, int depth, int num_sms,
                     const char **err, int shard_rank = -1, int shard_n = 0);
std::vector<int> shard_owners(int64_t T, int depth, int nranks);
bool build_gemm_plan(Plan &P, int64_t m, int64_t n, int64_t k, uint32_t p, int num_sms, const char **err);
bool build_herk1_plan(Plan &P, int64_t m, int64_t k, uint32_t p, int num_sms, const char **err);
bool build_lowmem_plan(Plan &P, int64_t m, int64_t k, uint32_t p, int depth, int num_sms, const char **err);
bool lowmem_shape_ok(int64_t m, int64_t k, int depth);
int auto_depth(int64_t m, int64_t k, uint32_t p, int phi);

}  // namespace adj
