// Recursion planner (host): level sizes with zero padding, workspace layout, leaf product list
// and the grouped, longest-K-first tile list of the single leaf launch.
#include "plan.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace adj {

static inline int64_t rup(int64_t x, int64_t a) { return (x + a - 1) / a * a; }
static inline int64_t cdiv(int64_t x, int64_t a) { return (x + a - 1) / a; }

static void fill_scheme(Plan &P, uint32_t p) {
  P.p = p;
  P.scheme = limb_scheme(p);
  P.planes = limb_planes(P.scheme);
  P.nacc = limb_accs(P.scheme);
  P.bn = 256;
  P.tile_m = P.tile_n = 256;
  P.kseg = (int)std::max<int64_t>(1, limb_kmax(P.scheme, p) / kBK);
  P.res32 = p > 65535;
  P.mod = make_modp(p);
  P.Y = skew_unitary(p);
  LeafParams &L = P.leaf_template;
  std::memset(&L, 0, sizeof(L));
  L.mod = P.mod;
  L.fixup32 = p > 65535;
  auto pw = [&](int e) { return (uint32_t)(((uint64_t)1 << e) % p); };
  if (P.scheme == LIMB_S8) {
    L.n_terms = 1;
    L.terms[0] = {0, 0, 0, 1, 1, {0, 0, 0}};
    L.acc_begin[0] = 0; L.acc_begin[1] = 1; L.acc_begin[2] = 1; L.acc_begin[3] = 1;
    L.weight[0] = 1;
  } else if (P.scheme == LIMB_K7) {
    // x y = 2^14 hh + 2^7 (hl + lh) + ll,  hl + lh = mm - hh - ll  (Karatsuba)
    //     = (2^14 - 2^7) hh + (1 - 2^7) ll + 2^7 mm
    L.n_terms = 3;
    L.terms[0] = {0, 0, 0, 1, 1, {0, 0, 0}};   // hh
    L.terms[1] = {1, 1, 1, 1, 1, {0, 0, 0}};   // ll
    L.terms[2] = {2, 2, 2, 1, 1, {0, 0, 0}};   // mm
    L.acc_begin[0] = 0; L.acc_begin[1] = 1; L.acc_begin[2] = 2; L.acc_begin[3] = 3;
    L.weight[0] = (pw(14) + p - pw(7)) % p;
    L.weight[1] = (1 + p - pw(7)) % p;
    L.weight[2] = pw(7);
  } else if (P.scheme == LIMB_T6) {
    // x = 2^12 d2 + 2^6 d1 + d0; with P_ij = (d_i + d_j)(e_i + e_j) (3-way Karatsuba):
    // x y = 2^24 P22 + 2^18 (P21 - P22 - P11) + 2^12 (P20 - P22 - P00 + P11) + 2^6 (P10 - P11 - P00) + P00
    // planes: 0 d2, 1 d1, 2 d0, 3 d2+d1, 4 d1+d0, 5 d2+d0; accumulator j = plane j x plane j
    L.n_terms = 6;
    for (int j = 0; j < 6; ++j) {
      L.terms[j] = {(int8_t)j, (int8_t)j, (int8_t)j, 1, 1, {0, 0, 0}};
      L.acc_begin[j] = j;
    }
    L.acc_begin[6] = 6;
    auto neg = [&](uint32_t x) { return (p - x % p) % p; };
    L.weight[0] = (uint32_t)(((uint64_t)pw(24) + neg(pw(18)) + neg(pw(12))) % p);   // P22
    L.weight[1] = (uint32_t)(((uint64_t)neg(pw(18)) + pw(12) + neg(pw(6))) % p);    // P11
    L.weight[2] = (uint32_t)(((uint64_t)neg(pw(12)) + neg(pw(6)) + 1) % p);         // P00
    L.weight[3] = pw(18);                                                             // P21
    L.weight[4] = pw(6);                                                              // P10
    L.weight[5] = pw(12);                                                             // P20
  } else {
    // x y = 2^16 hh + 2^8 (hl + lh) + ll ; hi signed, lo unsigned
    L.n_terms = 4;
    // accumulator order hh, (hl + lh), ll: with the K direction alternating per unit, the mixed
    // sweep (all four planes) starts on the hi planes hh just loaded and ll on the lo planes the
    // mixed sweep loaded last (c3 -0.95%); ADJ_ACC_ORDER=0 (diagnostics): hh, ll, mixed
    static const bool mixed_mid = !(getenv("ADJ_ACC_ORDER") && !atoi(getenv("ADJ_ACC_ORDER")));
    if (mixed_mid) {
      L.terms[0] = {0, 0, 0, 1, 1, {0, 0, 0}};   // hh  s8 x s8
      L.terms[1] = {1, 0, 1, 1, 0, {0, 0, 0}};   // hl  s8 x u8
      L.terms[2] = {1, 1, 0, 0, 1, {0, 0, 0}};   // lh  u8 x s8
      L.terms[3] = {2, 1, 1, 0, 0, {0, 0, 0}};   // ll  u8 x u8
      L.acc_begin[0] = 0; L.acc_begin[1] = 1; L.acc_begin[2] = 3; L.acc_begin[3] = 4;
      L.weight[0] = pw(16);
      L.weight[1] = pw(8);
      L.weight[2] = 1 % p;
    } else {
    L.terms[0] = {0, 0, 0, 1, 1, {0, 0, 0}};   // hh  s8 x s8
    L.terms[1] = {1, 1, 1, 0, 0, {0, 0, 0}};   // ll  u8 x u8
    L.terms[2] = {2, 0, 1, 1, 0, {0, 0, 0}};   // hl  s8 x u8
    L.terms[3] = {2, 1, 0, 0, 1, {0, 0, 0}};   // lh  u8 x s8
    L.acc_begin[0] = 0; L.acc_begin[1] = 1; L.acc_begin[2] = 2; L.acc_begin[3] = 4;
    L.weight[0] = pw(16);
    L.weight[1] = 1 % p;
    L.weight[2] = pw(8);
    }
  }
  for (int j = 0; j < 6; ++j) L.wshoup[j] = make_shoup(L.weight[j], p);
}

static ProductPlan make_prod(const Plan &P, int arena, int64_t arow, int64_t brow, int64_t a_pr, int64_t b_pr, int64_t kpad,
                             bool sym, int target, int level, int node, int idx, int64_t out_rows,
                             int64_t out_cols, bool out_u32, int64_t ldo) {
  ProductPlan pp;
  std::memset(&pp.lp, 0, sizeof(pp.lp));
  pp.lp.map = arena;
  pp.lp.a_row0 = (int32_t)arow;
  pp.lp.b_row0 = (int32_t)brow;
  pp.lp.a_plane_rows = (int32_t)a_pr;
  pp.lp.b_plane_rows = (int32_t)b_pr;
  pp.lp.kblocks = (int32_t)(kpad / kBK);
  pp.lp.sym = sym ? 1 : 0;
  pp.lp.out_u32 = (out_u32 || P.res32) ? 1 : 0;   // workspace residues are uint32 for p > 2^16
  pp.lp.out_rows = (int32_t)out_rows;
  pp.lp.out_cols = (int32_t)out_cols;
  pp.lp.vec_ok = 1;
  pp.lp.kseg = P.kseg;
  pp.lp.ldo = ldo;
  pp.target = target;
  pp.level = level;
  pp.node = node;
  pp.idx = idx;
  return pp;
}

// Grouped rasterisation: bands of 8 row tiles, column-major inside a band, so that the ~148
// concurrently running tiles share few A / B row panels in L2.
static void append_tiles(Plan &P) {
  std::stable_sort(P.prods.begin(), P.prods.end(),
                   [](const ProductPlan &a, const ProductPlan &b) { return a.lp.kblocks > b.lp.kblocks; });
  P.tiles.clear();
  static const int band = getenv("ADJ_BAND") ? std::max(1, atoi(getenv("ADJ_BAND"))) : 8;   // diagnostics
  for (size_t q = 0; q < P.prods.size(); ++q) {
    const LeafProduct &lp = P.prods[q].lp;
    const int64_t tm = cdiv(lp.out_rows, P.tile_m);
    const int64_t tn = cdiv(lp.out_cols, P.tile_n);
    for (int64_t b0 = 0; b0 < tm; b0 += band) {
      const int64_t b1 = std::min<int64_t>(tm, b0 + band);
      for (int64_t J = 0; J < tn; ++J)
        for (int64_t I = b0; I < b1; ++I) {
          if (lp.sym && J * P.tile_n > I * P.tile_m + P.tile_m - 1) continue;   // tile above the diagonal
          P.tiles.push_back(((uint32_t)q << 24) | ((uint32_t)I << 12) | (uint32_t)J);
          P.tiles.push_back(0u);   // whole tile
        }
    }
  }
}

// Tail balancing: jobs are dealt round-robin to the clusters, so with n tiles of equal cost the
// last wave holds n mod ncl tiles while the other clusters idle.  Those tail tiles are split
// along K into ~ncl / rem pieces each; every piece writes its residue partial to a fixup slot
// and fixup_kernel sums the pieces mod p (exact: < pieces * p < 2^32).
// When the last wave fills between a half and a quarter of the clusters, its tiles are split
// into two N = 128 column halves instead (no fixup: each half is written directly).
static void split_tail(Plan &P, int ncl) {
  P.fixups.clear();
  P.n_pieces = 0;
  const int64_t n = (int64_t)P.tiles.size() / 2;
  const int64_t rem = n % ncl;
  if (n == 0 || rem == 0 || rem * 2 > ncl) return;
  static const bool nsplit = !(getenv("ADJ_TAIL_KSPLIT") && atoi(getenv("ADJ_TAIL_KSPLIT")));   // diagnostics
  if (rem * 4 > ncl && nsplit) {
    for (int64_t t = n - rem; t < n; ++t) {
      P.tiles[2 * t + 1] = 0x00FFFFFFu;                  // column half 0 (kb0 = kb1 = 4095: no K piece)
      P.tiles.push_back(P.tiles[2 * t]);
      P.tiles.push_back(0x01FFFFFFu);                    // column half 1
    }
    return;
  }
  const int pieces = (int)(ncl / rem);
  std::vector<uint32_t> out(P.tiles.begin(), P.tiles.begin() + 2 * (n - rem));
  for (int64_t t = n - rem; t < n; ++t) {
    const uint32_t x = P.tiles[2 * t];
    const int q = (int)(x >> 24);
    const int kb = P.prods[q].lp.kblocks;
    const int np = std::min(pieces, kb);
    if (np < 2 || kb > 4095) { out.push_back(x); out.push_back(0u); continue; }
    FixupTile ft;
    ft.q = q; ft.I = (int)((x >> 12) & 0xFFF); ft.J = (int)(x & 0xFFF);
    ft.slot0 = P.n_pieces; ft.npieces = np; ft.pad_ = 0;
    for (int i = 0; i < np; ++i) {
      const uint32_t kb0 = (uint32_t)((int64_t)kb * i / np), kb1 = (uint32_t)((int64_t)kb * (i + 1) / np);
      out.push_back(x);
      out.push_back(kb0 | (kb1 << 12) | ((uint32_t)(P.n_pieces + i + 1) << 24));
    }
    P.n_pieces += np;
    P.fixups.push_back(ft);
  }
  P.tiles.swap(out);
}

// Wide-N leaf (leafw_kernel: 256 x 512 tiles, 25% fewer operand bytes per MAC, the limb
// recombination Horner-style in TMEM) for long launches (> 16 waves of wide jobs, where the
// static tail of the last wave is small without splitting).  Needs every limb weight invertible
// mod p (the Horner steps are w_j / w_{j+1}) and K segments bounded for accumulations that start
// from a residue < p.  Not for shard plans (their ownership is in 256 x 256 tiles).
static uint32_t powmod(uint64_t b, uint64_t e, uint32_t p) {
  uint64_t r = 1;
  b %= p;
  for (; e; e >>= 1, b = b * b % p)
    if (e & 1) r = r * b % p;
  return (uint32_t)r;
}
static void choose_wide(Plan &P, int num_sms) {
  P.wide = false;
  P.tile_n = 256;
  // ADJ_LEAF_WIDE (diagnostics, A/B): 0 off, 1 long launches (default), 2 always
  static const int env = getenv("ADJ_LEAF_WIDE") ? atoi(getenv("ADJ_LEAF_WIDE")) : 1;
  if (env == 0) return;
  LeafParams &L = P.leaf_template;
  for (int j = 0; j < P.nacc; ++j)
    if (L.weight[j] % P.p == 0) return;
  int64_t nt = 0, nt_n = 0;   // wide (256 x 512) and 256 x 256 jobs of the launch
  for (const ProductPlan &pp : P.prods) {
    const int64_t tm = cdiv(pp.lp.out_rows, 256), tn = cdiv(pp.lp.out_cols, 512), tn2 = cdiv(pp.lp.out_cols, 256);
    for (int64_t I = 0; I < tm; ++I) {
      for (int64_t J = 0; J < tn; ++J)
        if (!pp.lp.sym || J * 512 <= I * 256 + 255) ++nt;
      for (int64_t J = 0; J < tn2; ++J)
        if (!pp.lp.sym || J <= I) ++nt_n;
    }
  }
  // Long launches (> 16 waves) always; shorter ones when the wide makespan -- whole waves of jobs
  // costing 1.74 narrow jobs each (2 x the MACs at ~0.87 of the time per MAC, measured at c2) --
  // beats the narrow one, whose K-split tail balances to nt_n / clusters (c2 -1.8%, the 6-plane
  // x131071 -5.5%, c5 equal: profiles/r02/wide_short_launches.txt)
  const int64_t ncl = std::max(1, num_sms / 2);
  const bool short_ok = (double)cdiv(nt, ncl) * 1.74 < (double)nt_n / (double)ncl;
  if (env != 2 && nt <= 16 * ncl && !short_ok) return;
  const int kseg = (int)std::max<int64_t>(1, limb_kmax_from_residue((LimbScheme)P.scheme, P.p) / kBK);
  P.wide = true;
  P.tile_n = 512;
  P.kseg = kseg;
  for (ProductPlan &pp : P.prods) pp.lp.kseg = kseg;
  for (int j = 0; j + 1 < P.nacc; ++j)
    L.hshoup[j] = make_shoup((uint32_t)((uint64_t)L.weight[j] * powmod(L.weight[j + 1], P.p - 2, P.p) % P.p), P.p);
  L.one = make_shoup(1, P.p);
}

static void set_grid(Plan &P, int num_sms) {
  if (!P.wide) split_tail(P, num_sms / 2);
  P.fixup_offset = P.ws_bytes;
  // the tail never has more pieces than clusters (pieces = ncl / rem per tail tile): reserve the
  // worst case, so the size does not depend on the tile list (a shard's filtered list fits the
  // full plan's workspace)
  P.ws_bytes += (size_t)std::max(P.n_pieces, num_sms / 2) * 256 * 256 * P.res_bytes();
  P.ws_bytes = (P.ws_bytes + 255) / 256 * 256;
  P.counter_offset = P.ws_bytes;            // dynamic job counter of the leaf launch
  P.ws_bytes += 256;
  const int64_t nt = std::max<int64_t>(1, (int64_t)P.tiles.size() / 2);
  P.grid = 2 * (int)std::min<int64_t>(num_sms / 2, nt);   // CTA pairs
  // dynamic job claiming pays on long launches (clusters drift apart; in-order claiming keeps the
  // concurrent tiles a contiguous window: c3 / c4 -11..-17% time); for the 256 x 256 leaf static
  // round-robin was ~1% faster on launches of a dozen waves (c2, before the gate), and the
  // wide launches always claim dynamically, so the claim-wave gate keeps their tiles in step
  // (short ones too: c2 -1.2%, c5 -5.3%, x131071 -1.9% against static)
  P.dynamic = P.wide || nt > 16 * (int64_t)(num_sms / 2);
  P.segmented = false;
  for (const ProductPlan &pp : P.prods) P.segmented |= pp.lp.kblocks > pp.lp.kseg;
}

// Depth choice (R13), from measured B200 crossovers (profiles/r01/depth_crossover.txt):
// one level of Alg. alg:MIAHMM saves 1/8 of the leaf MMA work but adds a K1 and a K4 pass over
// HBM, and smaller leaves run the tcgen05 pipeline less efficiently.  It pays when the level's
// leaf products stay large -- (m/2)^2 (k/2) >= 2^38 MACs each: 16384^2 x 16384 (d = 1),
// 32768^2 x 32768 (d = 2) and 16384 x 131072 (d = 2) recurse, 8192^2 x 8192 does not (classical
// is 8% faster there).  Under the power cap of the large configs the saved MMAs also buy clock.
// phi = Q: Q6 is 1/11 of the 6M work; one level saves 1/8 of it -- never worth a K1 + K4 pass.
// Deeper levels are also used when the inner dimension exceeds the int32 accumulation bound
// of the limb scheme (K segmentation would handle it too; recursion also cuts the MMA work).
int auto_depth(int64_t m, int64_t k, uint32_t p, int phi) {
  int d = 0;
  while (phi != 2 && d < 3) {
    const double mh = (double)cdiv(m, (int64_t)1 << (d + 1)), kh = (double)cdiv(k, (int64_t)1 << (d + 1));
    if (mh * mh * kh < 274877906944.0) break;   // 2^38
    ++d;
  }
  const int64_t kmax = limb_kmax(limb_scheme(p), p);
  int64_t kh = k;
  for (int l = 1; l <= d; ++l) kh = 8 * cdiv(kh, 16);
  while (d < 3 && std::max<int64_t>(kBK, rup(kh, kBK)) > kmax) { ++d; kh = 8 * cdiv(kh, 16); }
  return d;
}

// ---------------------------------------------------------------- output-tile sharding
// Ownership unit: a pair {(I, J), (J, I)}, I >= J, of 256 x 256 tiles of the top-level product
// grid (depth 1: the (m/2) grid of P1..P5; depth 0: the grid of C).  Cost in leaf-tile units: a
// diagonal pair has its SYRK tile(s) and, at depth 1, the P3 / P4 tiles (I, I); an off-diagonal
// pair twice the GEMM tiles.
// A pair (I, J) reads the operand rows of tile bands I and J only, so a rank whose pairs touch
// few bands pre-adds (K1) only those rows.  The bands are cut into g contiguous groups and the
// triangle into the g (g + 1) / 2 blocks of group pairs (gi >= gj); whole blocks are dealt,
// largest first, to the least loaded rank (ties: the rank that already touches the block's
// groups).  g is chosen per (T, nranks) to minimise the modelled per-rank time
//   load_r / total + kK1Share * bands_r / T
// (kK1Share: K1's measured share of a depth-1 step); g = T degenerates to dealing
// single pairs.  Deterministic: every rank computes the same table.
static constexpr double kK1Share = 0.06;

std::vector<int> shard_owners(int64_t T, int depth, int nranks) {
  const int64_t npairs = T * (T + 1) / 2;
  auto cost = [&](int64_t I, int64_t J) -> int64_t { return depth == 0 ? 1 : (I == J ? 5 : 7); };
  std::vector<int> best_owner;
  double best_score = 1e30;
  std::vector<int64_t> cand;
  for (int64_t g = 1; g <= std::min<int64_t>(T, 24); ++g) cand.push_back(g);
  if (T > 24) cand.push_back(T);
  for (int64_t g : cand) {
    std::vector<int64_t> gb((size_t)g + 1);
    for (int64_t i = 0; i <= g; ++i) gb[(size_t)i] = T * i / g;
    struct Blk { int64_t gi, gj, cost; };
    std::vector<Blk> blks;
    for (int64_t gi = 0; gi < g; ++gi)
      for (int64_t gj = 0; gj <= gi; ++gj) {
        int64_t c = 0;
        for (int64_t I = gb[gi]; I < gb[gi + 1]; ++I)
          for (int64_t J = gb[gj]; J < std::min(gb[gj + 1], I + 1); ++J) c += cost(I, J);
        if (c > 0) blks.push_back({gi, gj, c});
      }
    if ((int64_t)blks.size() < nranks && g < T) continue;
    std::stable_sort(blks.begin(), blks.end(), [](const Blk &a, const Blk &b) { return a.cost > b.cost; });
    std::vector<int64_t> load((size_t)nranks, 0);
    std::vector<std::vector<char>> touch((size_t)nranks, std::vector<char>((size_t)g, 0));
    std::vector<int> blk_owner(blks.size(), 0);
    for (size_t b = 0; b < blks.size(); ++b) {
      int bestr = 0;
      int64_t bl = -1;
      int bn = 3;
      for (int r = 0; r < nranks; ++r) {
        const int fresh = (touch[r][(size_t)blks[b].gi] ? 0 : 1) + (blks[b].gi != blks[b].gj && !touch[r][(size_t)blks[b].gj] ? 1 : 0);
        if (bl < 0 || load[r] < bl || (load[r] == bl && fresh < bn)) { bestr = r; bl = load[r]; bn = fresh; }
      }
      blk_owner[b] = bestr;
      load[bestr] += blks[b].cost;
      touch[bestr][(size_t)blks[b].gi] = touch[bestr][(size_t)blks[b].gj] = 1;
    }
    int64_t total = 0;
    for (int64_t l : load) total += l;
    double score = 0;
    for (int r = 0; r < nranks; ++r) {
      int64_t bands = 0;
      for (int64_t q = 0; q < g; ++q) if (touch[r][(size_t)q]) bands += gb[q + 1] - gb[q];
      score = std::max(score, (double)load[r] / (double)std::max<int64_t>(1, total) + kK1Share * (double)bands / (double)T);
    }
    if (score < best_score - 1e-12) {
      best_score = score;
      best_owner.assign((size_t)npairs, 0);
      for (size_t b = 0; b < blks.size(); ++b)
        for (int64_t I = gb[blks[b].gi]; I < gb[blks[b].gi + 1]; ++I)
          for (int64_t J = gb[blks[b].gj]; J < std::min(gb[blks[b].gj + 1], I + 1); ++J)
            best_owner[(size_t)(I * (I + 1) / 2 + J)] = blk_owner[b];
    }
  }
  return best_owner;
}

bool apply_shard(Plan &P, int rank, int nranks, const char **err) {
  if (P.kind != PLAN_SYRK_T || P.depth > 1) { *err = "tile sharding supports phi = T at depth 0 or 1"; return false; }
  P.shard_rank = rank;
  P.shard_n = nranks;
  const int64_t grid_rows = P.depth == 0 ? P.rows_pad0 : P.lv[1].rows_pad;
  const int64_t T = (grid_rows + 255) / 256;
  const std::vector<int> owner = shard_owners(T, P.depth, nranks);
  auto owns = [&](int64_t I, int64_t J) {
    const int64_t a = std::max(I, J), b = std::min(I, J);
    return owner[(size_t)(a * (a + 1) / 2 + b)] == rank;
  };
  std::vector<uint32_t> kept;
  for (size_t t = 0; t + 1 < P.tiles.size(); t += 2) {
    const uint32_t x = P.tiles[t];
    if (owns((x >> 12) & 0xFFF, x & 0xFFF)) { kept.push_back(x); kept.push_back(P.tiles[t + 1]); }
  }
  P.tiles.swap(kept);
  // the tile bands this rank's pairs read: K1 (or the depth-0 split) pre-adds only their rows
  {
    std::vector<char> band((size_t)T, 0);
    for (int64_t I = 0; I < T; ++I)
      for (int64_t J = 0; J <= I; ++J)
        if (owns(I, J)) band[(size_t)I] = band[(size_t)J] = 1;
    P.shard_rows.clear();
    for (int64_t I = 0; I < T; ++I) {
      if (!band[(size_t)I]) continue;
      const int64_t r0 = 256 * I, r1 = std::min<int64_t>(256 * (I + 1), grid_rows);
      if (!P.shard_rows.empty() && P.shard_rows.back().second == r0) P.shard_rows.back().second = r1;
      else P.shard_rows.push_back({r0, r1});
    }
    if ((int)P.shard_rows.size() > kMaxRowRanges) P.shard_rows.assign(1, {0, grid_rows});   // too fragmented: all rows
  }
  // C regions this rank writes (for packing / gathering) and, at depth 1, the 64 x 64 lower tile
  // pairs of the K4 combine inside the owned 256-pairs
  P.shard_rects.clear();
  P.comb_pairs.clear();
  const int64_t m = P.m;
  auto rect = [&](int64_t r0, int64_t c0, int64_t nr, int64_t nc, int lower) {
    nr = std::min(nr, m - r0);
    nc = std::min(nc, m - c0);
    if (nr > 0 && nc > 0) P.shard_rects.push_back({r0, c0, nr, nc, lower});
  };
  if (P.depth == 0) {
    for (int64_t I = 0; I < T; ++I)
      for (int64_t J = 0; J <= I; ++J)
        if (owns(I, J)) rect(256 * I, 256 * J, 256, 256, I == J);
    return true;
  }
  const int64_t mh = P.lv[1].mh;
  for (int64_t I = 0; I < T; ++I)
    for (int64_t J = 0; J <= I; ++J) {
      if (!owns(I, J)) continue;
      for (int64_t ti = 4 * I; ti < 4 * I + 4; ++ti)
        for (int64_t tj = 4 * J; tj < 4 * J + 4; ++tj)
          if (ti >= tj && 64 * ti < mh && 64 * tj < mh) P.comb_pairs.push_back((uint32_t)(ti << 16 | tj));
      // rows/cols of the product grid clipped to mh, then placed in C's quadrants
      const int64_t r0 = 256 * I, c0 = 256 * J;
      const int64_t nr = std::min<int64_t>(256, mh - r0), nc = std::min<int64_t>(256, mh - c0);
      if (nr <= 0 || nc <= 0) continue;
      rect(r0, c0, nr, nc, I == J);                  // C11 = Low(U3)
      rect(mh + r0, c0, nr, nc, 0);                  // C21 = U4 on (I, J)
      if (I != J) rect(mh + c0, r0, nc, nr, 0);      // C21 = U4 on (J, I)
      rect(mh + r0, mh + c0, nr, nc, I == J);        // C22 = Low(U5)
    }
  return true;
}

bool build_syrk_plan(Plan &P, int64_t m, int64_t k, uint32_t p, int phi, int depth, int num_sms,
                     const char **err, int shard_rank, int shard_n) {
  P = Plan();
  P.kind = phi == 0 ? PLAN_SYRK_T : (phi == 1 ? PLAN_SYRK_H : PLAN_QUAT);
  P.m = m; P.n = m; P.k = k; P.depth = depth;
  fill_scheme(P, p);
  const int planes = P.planes;

  P.lv.resize(depth + 1);
  P.lv[0].mh = m; P.lv[0].kh = k;
  P.lv[0].rows_pad = rup(std::max<int64_t>(m, 1), kBM);
  P.lv[0].kpad = std::max<int64_t>(kBK, rup(k, kBK));
  int nn = 1;
  for (int l = 1; l <= depth; ++l) {
    LevelPlan &L = P.lv[l];
    L.mh = cdiv(P.lv[l - 1].mh, 2);
    L.kh = 8 * cdiv(P.lv[l - 1].kh, 16);          // kh multiple of 8, 2 kh >= previous (zero pad)
    L.rows_pad = rup(L.mh, kBM);
    L.kpad = std::max<int64_t>(kBK, rup(L.kh, kBK));
    L.n_nodes = nn;
    L.n_ops = (l == depth) ? OUT_N : 4;
    nn *= 3;
    if (L.n_nodes > kMaxNodes) { *err = "depth too large"; return false; }
  }
  size_t off = 0;
  auto alloc = [&](size_t bytes) { size_t o = off; off += (size_t)rup((int64_t)bytes, 256); return o; };

  P.rows_pad0 = P.lv[0].rows_pad;
  P.kpad0 = P.lv[0].kpad;
  int n0 = 0;
  if (P.kind == PLAN_SYRK_T && depth == 0) { P.op0_row[0] = 0; n0 = 1; }
  if (P.kind == PLAN_SYRK_H) {
    P.op0_row[0] = 0;
    P.op0_row[1] = (int64_t)planes * P.rows_pad0;
    n0 = 2;
    if (depth == 0) { P.op0_row[2] = 2 * (int64_t)planes * P.rows_pad0; n0 = 3; }
  }
  if (P.kind == PLAN_QUAT) {
    // Alg. alg:2M3M operands A, B, C, D, U1 = A + B, U2 = C + D (+ W = U1 + U2 for Q6 at depth 0)
    n0 = depth == 0 ? QO_N : QO_W;
    for (int o = 0; o < n0; ++o) P.q_row[o] = (int64_t)o * planes * P.rows_pad0;
  }
  if (n0 > 0) {
    ArenaPlan a;
    a.kpad = P.kpad0;
    a.n_rows = (int64_t)n0 * planes * P.rows_pad0;
    a.offset = alloc(a.bytes());
    P.arenas.push_back(a);
  }
  for (int l = 1; l <= depth; ++l) {
    LevelPlan &L = P.lv[l];
    ArenaPlan a;
    a.kpad = L.kpad;
    a.n_rows = (int64_t)L.n_nodes * L.n_ops * planes * L.rows_pad;
    a.offset = alloc(a.bytes());
    L.arena = (int)P.arenas.size();
    P.arenas.push_back(a);
  }
  if ((int)P.arenas.size() > kMaxMaps) { *err = "too many operand arenas"; return false; }
  for (int l = 1; l < depth; ++l) {
    LevelPlan &L = P.lv[l];
    L.s3_node_bytes = (size_t)rup(L.mh * L.kh * P.res_bytes(), 256);
    L.s3_offset = alloc(L.s3_node_bytes * L.n_nodes);
  }
  for (int l = 1; l <= depth; ++l) {
    LevelPlan &L = P.lv[l];
    L.p_buf_bytes = (size_t)rup(L.rows_pad * L.rows_pad * P.res_bytes(), 256);
    L.p_offset = alloc(L.p_buf_bytes * 5 * L.n_nodes);
  }
  if (P.kind == PLAN_SYRK_H) {
    P.h_offset = alloc((size_t)P.rows_pad0 * P.rows_pad0 * P.res_bytes());
    P.g_offset = alloc((size_t)P.rows_pad0 * P.rows_pad0 * P.res_bytes());
  }
  if (P.kind == PLAN_QUAT) {
    P.q_bytes = (size_t)rup(P.rows_pad0 * P.rows_pad0 * P.res_bytes(), 256);
    P.q_offset = alloc(P.q_bytes * 5);                                        // Q1..Q5
    P.g_offset = alloc((size_t)P.rows_pad0 * P.rows_pad0 * P.res_bytes());  // Q6 (Low)
  }
  P.ws_bytes = off;

  // the int32 accumulation bound per leaf product is met by K segmentation
  if (P.rows_pad0 >= (int64_t)4096 * P.tile_m) { *err = "m too large"; return false; }

  // leaf products
  P.prods.clear();
  if (P.kind == PLAN_SYRK_T && depth == 0)
    P.prods.push_back(make_prod(P, 0, 0, 0, P.rows_pad0, P.rows_pad0, P.kpad0, true, OUT_C, 0, 0, 0, m, m, true, 0));
  if (P.kind == PLAN_SYRK_H) {
    P.prods.push_back(make_prod(P, 0, P.op0_row[0], P.op0_row[1], P.rows_pad0, P.rows_pad0, P.kpad0, false, OUT_HBUF,
                                0, 0, 0, P.rows_pad0, P.rows_pad0, false, P.rows_pad0));     // H = X Y^T
    if (depth == 0)
      P.prods.push_back(make_prod(P, 0, P.op0_row[2], P.op0_row[2], P.rows_pad0, P.rows_pad0, P.kpad0, true, OUT_GBUF,
                                  0, 0, 0, P.rows_pad0, P.rows_pad0, false, P.rows_pad0)); // G = T T^T
  }
  if (P.kind == PLAN_QUAT) {
    // Q1 = C A^T, Q2 = D B^T, Q3 = U2 U1^T, Q4 = A B^T, Q5 = C D^T
    const int qa[5] = {QO_C, QO_D, QO_U2, QO_A, QO_C}, qb[5] = {QO_A, QO_B, QO_U1, QO_B, QO_D};
    for (int q = 0; q < 5; ++q)
      P.prods.push_back(make_prod(P, 0, P.q_row[qa[q]], P.q_row[qb[q]], P.rows_pad0, P.rows_pad0, P.kpad0, false,
                                  OUT_QBUF, 0, 0, q, P.rows_pad0, P.rows_pad0, false, P.rows_pad0));
    if (depth == 0)   // Q6 = (U1 + U2)(U1 + U2)^T, Low
      P.prods.push_back(make_prod(P, 0, P.q_row[QO_W], P.q_row[QO_W], P.rows_pad0, P.rows_pad0, P.kpad0, true,
                                  OUT_GBUF, 0, 0, 0, P.rows_pad0, P.rows_pad0, false, P.rows_pad0));
  }
  for (int l = 1; l <= depth; ++l) {
    const LevelPlan &L = P.lv[l];
    for (int n = 0; n < L.n_nodes; ++n) {
      auto row = [&](int o) { return ((int64_t)n * L.n_ops + o) * planes * L.rows_pad; };
      const int64_t rp = L.rows_pad;
      // P3 = A22 phi(S4), P4 = S1 phi(S2)   (general products)
      P.prods.push_back(make_prod(P, L.arena, row(OUT_X22), row(OUT_S4), rp, rp, L.kpad, false, OUT_PBUF, l, n, 2, rp, rp,
                                  false, rp));
      P.prods.push_back(make_prod(P, L.arena, row(OUT_S1), row(OUT_S2), rp, rp, L.kpad, false, OUT_PBUF, l, n, 3, rp, rp,
                                  false, rp));
      if (l == depth) {
        // P1 = A11 phi(A11), P2 = A12 phi(A12), P5 = S3 phi(S3) at the last level
        P.prods.push_back(make_prod(P, L.arena, row(OUT_X11), row(OUT_X11), rp, rp, L.kpad, true, OUT_PBUF, l, n, 0, rp,
                                    rp, false, rp));
        P.prods.push_back(make_prod(P, L.arena, row(OUT_X12), row(OUT_X12), rp, rp, L.kpad, true, OUT_PBUF, l, n, 1, rp,
                                    rp, false, rp));
        P.prods.push_back(make_prod(P, L.arena, row(OUT_S3), row(OUT_S3), rp, rp, L.kpad, true, OUT_PBUF, l, n, 4, rp,
                                    rp, false, rp));
      }
    }
  }
  if ((int)P.prods.size() > kMaxProducts) { *err = "too many leaf products"; return false; }
  if (shard_n == 0) choose_wide(P, num_sms);
  append_tiles(P);
  if (shard_n > 0 && !apply_shard(P, shard_rank, shard_n, err)) return false;
  set_grid(P, num_sms);
  return true;
}

bool build_herk1_plan(Plan &P, int64_t m, int64_t k, uint32_t p, int num_sms, const char **err) {
  P = Plan();
  P.kind = PLAN_HERK1;
  P.m = m; P.n = m; P.k = k; P.depth = 1;
  fill_scheme(P, p);
  P.lv.resize(2);
  P.lv[0].mh = m; P.lv[0].kh = k;
  P.lv[0].rows_pad = rup(std::max<int64_t>(m, 1), kBM);
  P.lv[0].kpad = std::max<int64_t>(kBK, rup(k, kBK));
  LevelPlan &L = P.lv[1];
  L.mh = cdiv(m, 2);
  L.kh = 8 * cdiv(k, 16);
  L.rows_pad = rup(L.mh, kBM);
  L.kpad = std::max<int64_t>(kBK, rup(L.kh, kBK));
  L.n_nodes = 1;
  L.n_ops = HO_N;
  P.rows_pad0 = P.lv[0].rows_pad;
  P.kpad0 = P.lv[0].kpad;
  if (L.rows_pad >= (int64_t)4096 * P.tile_m) { *err = "m too large"; return false; }
  size_t off = 0;
  ArenaPlan a;
  a.kpad = L.kpad;
  a.n_rows = (int64_t)HO_N * P.planes * L.rows_pad;
  a.offset = 0;
  off = (size_t)rup((int64_t)a.bytes(), 256);
  L.arena = 0;
  P.arenas.push_back(a);
  P.hb_bytes = (size_t)rup(L.rows_pad * L.rows_pad * P.res_bytes(), 256);
  P.hb_offset = off;
  off += P.hb_bytes * HB_N;
  L.p_offset = P.hb_offset;     // pbuf(P, ws, 1, 0, idx) addresses product buffer idx
  L.p_buf_bytes = P.hb_bytes;
  P.ws_bytes = off;
  const int64_t rp = L.rows_pad;
  auto row = [&](int o) { return (int64_t)o * P.planes * rp; };
  struct Q { int a, b; bool sym; int buf; };
  const Q qs[HB_N] = {{HO_T11, HO_T11, true, HB_G1}, {HO_X11, HO_Y11, false, HB_H1},
                      {HO_T12, HO_T12, true, HB_G2}, {HO_X12, HO_Y12, false, HB_H2},
                      {HO_T3, HO_T3, true, HB_G5},   {HO_X3, HO_Y3, false, HB_H5},
                      {HO_X22, HO_X4, false, HB_A1}, {HO_Y22, HO_Y4, false, HB_A2}, {HO_Z22, HO_W4, false, HB_A3},
                      {HO_X1, HO_X2, false, HB_B1},  {HO_Y1, HO_Y2, false, HB_B2},  {HO_Z1, HO_W2, false, HB_B3}};
  for (const Q &q : qs)
    P.prods.push_back(make_prod(P, 0, row(q.a), row(q.b), rp, rp, L.kpad, q.sym, OUT_PBUF, 1, 0, q.buf, rp, rp, false, rp));
  append_tiles(P);
  set_grid(P, num_sms);
  return true;
}

// ---------------------------------------------------------------- low-memory schedule (row N1)
// Applies to phi = T at depth >= 1 when the root's blocks are whole 64-row multiples (m even
// halves, 32 x 32 in-place K4 tiles stay inside C): m % 64 == 0.
bool lowmem_shape_ok(int64_t m, int64_t k, int depth) { return depth >= 1 && m >= 128 && m % 64 == 0 && k >= 1; }

bool build_lowmem_plan(Plan &P, int64_t m, int64_t k, uint32_t p, int depth, int num_sms, const char **err) {
  if (!lowmem_shape_ok(m, k, depth)) { *err = "low-memory schedule needs depth >= 1 and m % 64 == 0"; return false; }
  Plan child;
  const int64_t mh = m / 2, kh = 8 * cdiv(k, 16);
  if (!build_syrk_plan(child, mh, kh, p, 0, depth - 1, num_sms, err)) return false;
  P = Plan();
  P.kind = PLAN_LOWMEM;
  P.m = m; P.n = m; P.k = k; P.depth = 1; P.lm_depth = depth;
  fill_scheme(P, p);
  P.lv.resize(2);
  P.lv[0].mh = m; P.lv[0].kh = k;
  P.lv[0].rows_pad = rup(m, kBM);
  P.lv[0].kpad = std::max<int64_t>(kBK, rup(k, kBK));
  LevelPlan &L = P.lv[1];
  L.mh = mh; L.kh = kh;
  L.rows_pad = rup(mh, kBM);
  L.kpad = std::max<int64_t>(kBK, rup(kh, kBK));
  L.n_nodes = 1;
  L.n_ops = 4;                                   // S1, S2, S4, A22 (P1, P2, P5 are the children)
  P.rows_pad0 = P.lv[0].rows_pad;
  P.kpad0 = P.lv[0].kpad;
  if (L.rows_pad >= (int64_t)4096 * P.tile_m) { *err = "m too large"; return false; }
  size_t off = 0;
  auto alloc = [&](size_t bytes) { size_t o = off; off += (size_t)rup((int64_t)bytes, 256); return o; };
  L.s3_node_bytes = (size_t)rup(mh * kh * P.res_bytes(), 256);
  L.s3_offset = alloc(L.s3_node_bytes);
  const size_t pb = (size_t)L.rows_pad * L.rows_pad * P.res_bytes();
  P.lm_p2_off = alloc(pb);
  P.lm_p4_off = alloc(pb);
  P.lm_region_off = off;
  ArenaPlan a;
  a.kpad = L.kpad;
  a.n_rows = (int64_t)4 * P.planes * L.rows_pad;
  a.offset = alloc(a.bytes());
  L.arena = 0;
  P.arenas.push_back(a);
  P.ws_bytes = off;
  const int64_t rp = L.rows_pad;
  auto row = [&](int o) { return (int64_t)o * P.planes * rp; };
  // P3 = A22 phi(S4) into C21 (m - mh = mh rows), P4 = S1 phi(S2) into its buffer
  P.prods.push_back(make_prod(P, 0, row(OUT_X22), row(OUT_S4), rp, rp, L.kpad, false, OUT_C21, 1, 0, 2, mh, mh, true, 0));
  P.prods.push_back(make_prod(P, 0, row(OUT_S1), row(OUT_S2), rp, rp, L.kpad, false, OUT_LMP4, 1, 0, 3, rp, rp, false, rp));
  append_tiles(P);
  set_grid(P, num_sms);
  P.lm_child_ws = child.ws_bytes;
  P.ws_bytes = std::max(P.ws_bytes, P.lm_region_off + child.ws_bytes);
  P.ws_bytes = (P.ws_bytes + 255) / 256 * 256;
  return true;
}

bool build_gemm_plan(Plan &P, int64_t m, int64_t n, int64_t k, uint32_t p, int num_sms, const char **err) {
  P = Plan();
  P.kind = PLAN_GEMM;
  P.m = m; P.n = n; P.k = k; P.depth = 0;
  fill_scheme(P, p);
  P.rows_pad0 = rup(std::max<int64_t>(m, 1), kBM);
  P.rows_pad_b = rup(std::max<int64_t>(n, 1), kBM);
  P.kpad0 = std::max<int64_t>(kBK, rup(k, kBK));
  if (P.rows_pad0 >= (int64_t)4096 * P.tile_m || P.rows_pad_b >= (int64_t)4096 * P.tile_n) { *err = "m or n too large"; return false; }
  P.op0_row[0] = 0;
  P.op0_row[1] = (int64_t)P.planes * P.rows_pad0;
  ArenaPlan a;
  a.kpad = P.kpad0;
  a.n_rows = (int64_t)P.planes * (P.rows_pad0 + P.rows_pad_b);
  a.offset = 0;
  P.arenas.push_back(a);
  P.ws_bytes = (size_t)rup((int64_t)a.bytes(), 256);
  P.prods.push_back(make_prod(P, 0, P.op0_row[0], P.op0_row[1], P.rows_pad0, P.rows_pad_b, P.kpad0, false, OUT_C, 0, 0, 0,
                              m, n, true, 0));
  append_tiles(P);
  set_grid(P, num_sms);
  return true;
}

}  // namespace adj
