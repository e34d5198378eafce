// C ABI (include/adjprod.h): validation, plan cache, stream-ordered launch schedule.
//
// Schedule of one adjprod_modp call at depth d >= 1 (all on the caller's stream):
//   K1 level 1 .. d            pre-additions + limb planes, top-down (level l+1 reads S3 of level l)
//   grouped leaf launch        every P3/P4 of every level and P1/P2/P5 of level d, one persistent
//                              tcgen05 kernel, longest-K tiles first
//   K4 level d .. 1            recombination bottom-up into the parent's P buffers, then into C
// For phi = H (2M): split X, Y (and T = X + Y at depth 0); H = X Y^T joins the grouped leaf launch;
// G = Low(T T^T) runs the same tree; K5 forms Re/Im.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <dlfcn.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/adjprod.h"
#include "field.hpp"
#include "kernels.hpp"
#include "plan.hpp"

using namespace adj;

namespace {

thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

adj_status_t fail(adj_status_t st, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

#define CUDA_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess) return fail(ADJ_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(_e)); \
  } while (0)

// ------------------------------------------------------------------ per-class event timing
std::atomic<int> g_prof_on{0};
std::mutex g_prof_mu;
struct ProfRec { int cls; cudaEvent_t a, b; };
std::vector<ProfRec> g_prof;

struct ProfScope {
  int cls;
  cudaStream_t s;
  cudaEvent_t a = nullptr, b = nullptr;
  ProfScope(int c, cudaStream_t st) : cls(c), s(st) {
    if (!g_prof_on.load()) return;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
  }
  ~ProfScope() {
    if (!a) return;
    cudaEventRecord(b, s);
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof.push_back({cls, a, b});
  }
};

enum { CLS_LEAF = 0, CLS_PRE = 1, CLS_COMB = 2, CLS_OTHER = 3 };

#define LAUNCH_CLS(cls, expr)         \
  do {                                \
    ProfScope _ps(cls, s);            \
    CUDA_TRY(expr);                   \
    g_launches.fetch_add(1);          \
  } while (0)
#define LAUNCH(expr) LAUNCH_CLS(CLS_OTHER, expr)

// ------------------------------------------------------------------ device info
struct DevInfo {
  bool ok = false;
  int sms = 0;
};
std::mutex g_mu;
std::map<int, DevInfo> g_dev;

adj_status_t check_device(int *dev_out, int *sms_out) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_dev.find(dev);
  if (it == g_dev.end()) {
    DevInfo di;
    int major = 0, minor = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    CUDA_TRY(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev));
    CUDA_TRY(cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, dev));
    di.ok = (major == 10 && minor == 0);
    it = g_dev.emplace(dev, di).first;
  }
  if (!it->second.ok) return fail(ADJ_ERR_ARCH, "device %d is not sm_100 (B200); this library is sm_100a only", dev);
  *dev_out = dev;
  *sms_out = it->second.sms;
  return ADJ_OK;
}

// ------------------------------------------------------------------ workspace pool
// Calls without a caller workspace allocate it stream-ordered from a per-device pool that keeps
// its memory between calls (release threshold = max): the default pool returns freed memory at
// every synchronisation, which made each multi-GB workspace a fresh mapping (measured: a 32768^2
// call took several times its compute time).
std::mutex g_pool_mu;
std::map<int, cudaMemPool_t> g_pools;

}  // namespace
cudaError_t adj_pool_alloc(void **ptr, size_t bytes, cudaStream_t s) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  cudaMemPool_t pool;
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    auto it = g_pools.find(dev);
    if (it == g_pools.end()) {
      cudaMemPoolProps props = {};
      props.allocType = cudaMemAllocationTypePinned;
      props.handleTypes = cudaMemHandleTypeNone;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      if ((e = cudaMemPoolCreate(&pool, &props)) != cudaSuccess) return e;
      uint64_t thr = ~0ull;
      if ((e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr)) != cudaSuccess) return e;
      g_pools.emplace(dev, pool);
    } else {
      pool = it->second;
    }
  }
  return cudaMallocFromPoolAsync(ptr, bytes, pool, s);
}
namespace {

// ------------------------------------------------------------------ TMA descriptor encoding
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

adj_status_t get_encode() {
  if (g_encode) return ADJ_OK;
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (!fn || q != cudaDriverEntryPointSuccess) return fail(ADJ_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return ADJ_OK;
}

adj_status_t encode_arena(CUtensorMap *map, void *base, int64_t kpad, int64_t rows, int box_rows = kBM) {
  cuuint64_t dims[2] = {(cuuint64_t)kpad, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)kpad};
  cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ADJ_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return ADJ_OK;
}

// SM count of the current device for host-only queries (workspace size, shard layout); 148
// (B200) when no device is visible -- the plan's only SM dependence is the tail split and its
// fixup slots, which are sized for num_sms / 2 pieces
int query_sms() {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess &&
      sms > 0)
    return sms;
  cudaGetLastError();
  return 148;
}

// ------------------------------------------------------------------ plan cache
// dev, kind, m, n, k, p, phi, depth, shard rank, shard count.  Bounded (LRU over the plans no
// call holds, see PlanRef): an evicted plan's device tile arrays are released with cudaFree, which
// waits for the launches that read them.
using Key = std::tuple<int, int, int64_t, int64_t, int64_t, uint32_t, int, int, int, int>;
struct CachedPlan {
  std::unique_ptr<Plan> plan;
  uint64_t last_use = 0;
};
std::map<Key, CachedPlan> g_plans;
std::map<const Plan *, int> g_plan_pins;   // plans some call is using right now (guarded by g_mu)
uint64_t g_plan_clock = 0;
constexpr size_t kMaxCachedPlans = 64;

// What get_plan hands out: the plan stays pinned -- never evicted, whatever other host threads
// insert meanwhile -- until the PlanRef goes out of scope or is given another plan.
struct PlanRef {
  Plan *p = nullptr;
  PlanRef() = default;
  PlanRef(const PlanRef &) = delete;
  PlanRef &operator=(const PlanRef &) = delete;
  ~PlanRef() { reset(); }
  void reset() {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_plan_pins.find(p);
    if (it != g_plan_pins.end() && --it->second <= 0) g_plan_pins.erase(it);
    p = nullptr;
  }
  Plan *operator->() const { return p; }
  Plan &operator*() const { return *p; }
};

void free_plan_device(Plan &P) {
  if (P.d_tiles) cudaFree(P.d_tiles);
  if (P.d_comb_pairs) cudaFree(P.d_comb_pairs);
  if (P.d_fixups) cudaFree(P.d_fixups);
  P.d_tiles = nullptr;
  P.d_comb_pairs = nullptr;
  P.d_fixups = nullptr;
}

void evict_plans() {   // caller holds g_mu
  while (g_plans.size() >= kMaxCachedPlans) {
    auto lru = g_plans.end();
    for (auto it = g_plans.begin(); it != g_plans.end(); ++it)
      if (g_plan_pins.count(it->second.plan.get()) == 0 &&
          (lru == g_plans.end() || it->second.last_use < lru->second.last_use))
        lru = it;
    if (lru == g_plans.end()) return;   // every cached plan is in use: the cache grows past its bound
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(lru->second.plan->dev);
    free_plan_device(*lru->second.plan);
    cudaSetDevice(cur);
    g_plans.erase(lru);
  }
}

adj_status_t get_plan(PlanRef *out, int kind, int64_t m, int64_t n, int64_t k, uint32_t p, int phi, int depth, int dev,
                      int sms, int shard_rank = -1, int shard_n = 0) {
  out->reset();
  std::lock_guard<std::mutex> lk(g_mu);
  Key key{dev, kind, m, n, k, p, phi, depth, shard_rank, shard_n};
  auto it = g_plans.find(key);
  if (it != g_plans.end()) {
    it->second.last_use = ++g_plan_clock;
    out->p = it->second.plan.get();
    ++g_plan_pins[out->p];
    return ADJ_OK;
  }
  evict_plans();
  auto P = std::make_unique<Plan>();
  const char *err = nullptr;
  bool ok = kind == PLAN_GEMM     ? build_gemm_plan(*P, m, n, k, p, sms, &err)
            : kind == PLAN_HERK1  ? build_herk1_plan(*P, m, k, p, sms, &err)
            : kind == PLAN_LOWMEM ? build_lowmem_plan(*P, m, k, p, depth, sms, &err)
                                  : build_syrk_plan(*P, m, k, p, phi, depth, sms, &err, shard_rank, shard_n);
  if (!ok) return fail(ADJ_ERR_INVALID_VALUE, "plan: %s", err ? err : "unsupported");
  P->dev = dev;
  auto upload = [&](void **dst, const void *src, size_t bytes) -> cudaError_t {
    if (bytes == 0) return cudaSuccess;
    cudaError_t e = cudaMalloc(dst, bytes);
    return e != cudaSuccess ? e : cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice);
  };
  cudaError_t e = upload(reinterpret_cast<void **>(&P->d_tiles), P->tiles.data(), P->tiles.size() * sizeof(uint32_t));
  if (e == cudaSuccess)
    e = upload(reinterpret_cast<void **>(&P->d_comb_pairs), P->comb_pairs.data(), P->comb_pairs.size() * sizeof(uint32_t));
  if (e == cudaSuccess)
    e = upload(reinterpret_cast<void **>(&P->d_fixups), P->fixups.data(), P->fixups.size() * sizeof(FixupTile));
  if (e != cudaSuccess) {
    free_plan_device(*P);
    return fail(ADJ_ERR_CUDA, "plan upload: %s", cudaGetErrorString(e));
  }
  out->p = P.get();
  ++g_plan_pins[out->p];
  CachedPlan cp;
  cp.plan = std::move(P);
  cp.last_use = ++g_plan_clock;
  g_plans.emplace(key, std::move(cp));
  return ADJ_OK;
}

// ------------------------------------------------------------------ validation helpers
bool valid_modulus(uint32_t p) { return p >= 3 && p <= kMaxModulus && is_prime_u32(p); }
}  // namespace
// uint32 words per element: GF(p) 1, GF(p^2) 2, quaternions 4
int adj_phi_width(adj_phi_t phi) { return phi == ADJ_PHI_H ? 2 : (phi == ADJ_PHI_Q ? 4 : 1); }
namespace {

bool overlap(const void *a, size_t abytes, const void *b, size_t bbytes) {
  uintptr_t a0 = (uintptr_t)a, a1 = a0 + abytes, b0 = (uintptr_t)b, b1 = b0 + bbytes;
  return abytes && bbytes && a0 < b1 && b0 < a1;
}

size_t span_bytes(int64_t rows, int64_t cols, int64_t ld, int elem_bytes) {
  if (rows <= 0 || cols <= 0) return 0;
  return (size_t)((rows - 1) * ld + cols) * elem_bytes;
}

InView make_view(const void *ptr, int64_t ld, int64_t rows, int64_t cols, int type, bool e16 = false) {
  InView v;
  std::memset(&v, 0, sizeof(v));
  v.ptr = ptr;
  v.ld = ld;
  v.rows_valid = rows;
  v.cols_valid = cols;
  v.type = type;
  v.e16 = e16 ? 1 : 0;   // pair types only: (re, im) uint16 pairs
  uintptr_t a = (uintptr_t)ptr;
  if (type == IN_U16 || type == IN_U16R) v.vec_ok = (a % 8 == 0) && (ld % 4 == 0);
  else if (type == IN_U32) v.vec_ok = (a % 16 == 0) && (ld % 4 == 0);
  else if (e16) v.vec_ok = (a % 16 == 0) && (ld % 4 == 0);
  else v.vec_ok = (a % 16 == 0) && (ld % 2 == 0);
  return v;
}

InView child_view(const InView &pv, int c, const LevelPlan &Lp, void *s3, int64_t s3_ld, bool res32) {
  // children of a node at level l-1 (half sizes Lp.mh, Lp.kh): 0 = X11, 1 = X12, 2 = S3
  if (c == 2) return make_view(s3, s3_ld, Lp.mh, Lp.kh, res32 ? IN_U32 : IN_U16);
  const int64_t rows = std::min(pv.rows_valid, Lp.mh);
  if (c == 0) return make_view(pv.ptr, pv.ld, rows, std::min(pv.cols_valid, Lp.kh), pv.type, pv.e16);
  const int esz = (pv.type == IN_U16 || pv.type == IN_U16R) ? 2
                  : (pv.type == IN_U32 ? 4 : (pv.type == IN_QUAD_SUM ? (pv.e16 ? 8 : 16) : (pv.e16 ? 4 : 8)));
  const void *ptr = static_cast<const uint8_t *>(pv.ptr) + (size_t)Lp.kh * esz;
  int64_t cols = std::max<int64_t>(0, std::min(pv.cols_valid - Lp.kh, Lp.kh));
  return make_view(ptr, pv.ld, rows, cols, pv.type, pv.e16);
}

// ------------------------------------------------------------------ launch schedule
struct Ptrs {
  uint32_t alpha = 1, beta = 0;   // SYRK form on the final Low(C): alpha Low(A phi(A)) + beta Low(C)
  int axpby = 0;
  const uint32_t *A = nullptr; int64_t lda = 0;
  const uint32_t *B = nullptr; int64_t ldb = 0;
  uint32_t *C = nullptr; int64_t ldc = 0;
  uint8_t *ws = nullptr;
  bool res16 = false;   // write the final Low(C) as uint16 residues (adjprod_modp_partial, ADJ_OUT_U16)
  bool in16 = false;    // A holds uint16 values (ADJ_IN_U16)
};

void *pbuf(const Plan &P, uint8_t *ws, int l, int n, int idx) {
  const LevelPlan &L = P.lv[l];
  return ws + L.p_offset + ((size_t)n * 5 + idx) * L.p_buf_bytes;
}
void *s3buf(const Plan &P, uint8_t *ws, int l, int n) {
  const LevelPlan &L = P.lv[l];
  return ws + L.s3_offset + (size_t)n * L.s3_node_bytes;
}

adj_status_t launch_leaf_all(const Plan &P, const Ptrs &x, cudaStream_t s) {
  if (P.tiles.empty()) return ADJ_OK;
  adj_status_t st = get_encode();
  if (st != ADJ_OK) return st;
  LeafParams L = P.leaf_template;
  for (size_t a = 0; a < P.arenas.size(); ++a) {
    st = encode_arena(&L.maps[a], x.ws + P.arenas[a].offset, P.arenas[a].kpad, P.arenas[a].n_rows);
    if (st != ADJ_OK) return st;
    st = encode_arena(&L.maps_half[a], x.ws + P.arenas[a].offset, P.arenas[a].kpad, P.arenas[a].n_rows, kBM / 2);
    if (st != ADJ_OK) return st;
  }
  for (size_t a = P.arenas.size(); a < (size_t)kMaxMaps; ++a) {
    L.maps[a] = L.maps[0];
    L.maps_half[a] = L.maps_half[0];
  }
  for (size_t q = 0; q < P.prods.size(); ++q) {
    const ProductPlan &pp = P.prods[q];
    L.prod[q] = pp.lp;
    switch (pp.target) {
      case OUT_PBUF: L.prod[q].out = pbuf(P, x.ws, pp.level, pp.node, pp.idx); break;
      case OUT_HBUF: L.prod[q].out = x.ws + P.h_offset; break;
      case OUT_GBUF: L.prod[q].out = x.ws + P.g_offset; break;
      case OUT_QBUF: L.prod[q].out = x.ws + P.q_offset + (size_t)pp.idx * P.q_bytes; break;
      case OUT_LMP4: L.prod[q].out = x.ws + P.lm_p4_off; break;
      case OUT_C21: {   // low-memory root: P3 into C's C21 block, in C's element type
        const size_t eb = (x.res16 && !P.res32) ? 2 : 4;
        L.prod[q].out = reinterpret_cast<uint8_t *>(x.C) + (size_t)P.lv[1].mh * (size_t)x.ldc * eb;
        L.prod[q].ldo = x.ldc;
        L.prod[q].out_u32 = eb == 4 ? 1 : 0;
        L.prod[q].vec_ok = ((uintptr_t)L.prod[q].out % 16 == 0) && (x.ldc % (eb == 2 ? 8 : 4) == 0);
        break;
      }
      case OUT_C:
        L.prod[q].out = x.C;
        L.prod[q].ldo = x.ldc;
        L.prod[q].vec_ok = ((uintptr_t)x.C % 16 == 0) && (x.ldc % (x.res16 ? 8 : 4) == 0);
        if (x.res16) L.prod[q].out_u32 = 0;
        L.prod[q].alpha = x.alpha;
        L.prod[q].beta = x.beta;
        L.prod[q].axpby = x.axpby;
        break;
    }
  }
  L.tiles = reinterpret_cast<const uint2 *>(P.d_tiles);
  L.n_tiles = (int32_t)(P.tiles.size() / 2);
  L.fixup = x.ws + P.fixup_offset;
  if (const char *dbg = getenv("ADJ_LEAF_DEBUG")) L.debug = atoi(dbg);   // diagnostics only
  // K-direction alternation of a job's units, for the s8 / u8 scheme only, whose
  // consecutive accumulators share operand planes (c3 -1.2%; the K7 scheme's do not: c4 +0.3%);
  // ADJ_LEAF_KALT (diagnostics): 0 off, 2 every scheme
  static const int kalt = getenv("ADJ_LEAF_KALT") ? atoi(getenv("ADJ_LEAF_KALT")) : 1;
  L.kalt = (kalt == 2 || (kalt == 1 && P.scheme == LIMB_SU8)) ? 1 : 0;
  // soft claim-wave gate: a gated job issues its first gate_pre stages before it waits,
  // so its MMAs start as soon as the gate opens (2: c3 -0.7%, c4 -0.6%; ADJ_LEAF_GATE_PRE: diagnostics)
  static const int gate_pre = getenv("ADJ_LEAF_GATE_PRE") ? atoi(getenv("ADJ_LEAF_GATE_PRE")) : 2;
  L.gate_pre = std::max(0, gate_pre);
  // diagnostics: ADJ_LEAF_STATIC / ADJ_LEAF_DYNAMIC force the job scheduler (A/B measurements)
  static const bool force_static = getenv("ADJ_LEAF_STATIC") != nullptr;
  static const bool force_dynamic = getenv("ADJ_LEAF_DYNAMIC") != nullptr;
  if (force_dynamic || (P.dynamic && !force_static)) {
    L.job_counter = reinterpret_cast<int32_t *>(x.ws + P.counter_offset);
    CUDA_TRY(cudaMemsetAsync(L.job_counter, 0, 2 * sizeof(int32_t), s));   // claims, jobs loaded
    // Claim-wave gate of the dynamic leaf launch.  A job is claimed when its loads are about to
    // start, and the jobs of claim wave w (claim index / clusters) start only once every job of
    // wave w - 1 has issued its loads, so the tiles that run together walk K together and their
    // operand panels are read from DRAM about once (c3 -5.7%, c4 -11% under the power cap).
    // ADJ_LEAF_GATE (diagnostics, A/B): 0 = off (claims two ahead, no gate); 1..100 = gate % with
    // claims two ahead; 1000 + g = claim at start, gate g %; -1 = claim at start, no gate
    static const int gate = getenv("ADJ_LEAF_GATE") ? atoi(getenv("ADJ_LEAF_GATE")) : 1100;
    L.gate = gate;
  }
  // diagnostics: ADJ_LEAF_GRID caps the persistent grid (CTAs, even; power-regime A/B)
  static const int grid_cap = getenv("ADJ_LEAF_GRID") ? atoi(getenv("ADJ_LEAF_GRID")) & ~1 : 0;
  const int grid = grid_cap > 0 ? std::min(P.grid, grid_cap) : P.grid;
  if (P.wide) LAUNCH_CLS(CLS_LEAF, launch_leafw(L, P.nacc, grid, s));
  else LAUNCH_CLS(CLS_LEAF, launch_leaf2(L, P.nacc, P.segmented, grid, s));
  if (!P.fixups.empty()) LAUNCH_CLS(CLS_LEAF, launch_fixup(L, P.d_fixups, (int)P.fixups.size(), s));
  return ADJ_OK;
}

// output-tile sharding: the top level's pre-addition / split covers only the rows of the tile
// bands this rank's tiles read (plan.cpp apply_shard); otherwise every row
void set_shard_rows(const Plan &P, RowRanges &R) {
  std::memset(&R, 0, sizeof(R));
  if (P.shard_n <= 0) return;
  R.n = (int32_t)P.shard_rows.size();
  for (int i = 0; i < R.n; ++i) {
    R.lo[i] = P.shard_rows[(size_t)i].first;
    R.hi[i] = P.shard_rows[(size_t)i].second;
  }
}

adj_status_t run_split(const Plan &P, const InView &v, int64_t rows, int64_t cols, int64_t rows_pad, int64_t op_row,
                       uint8_t *arena, cudaStream_t s) {
  SplitParams sp;
  std::memset(&sp, 0, sizeof(sp));
  sp.in = v;
  sp.rows = rows;
  sp.cols = cols;
  sp.rows_pad = rows_pad;
  sp.kpad = P.kpad0;
  sp.op_row = op_row;
  sp.arena = reinterpret_cast<int8_t *>(arena);
  sp.scheme = P.scheme;
  sp.planes = P.planes;
  sp.mod = P.mod;
  set_shard_rows(P, sp.row_ranges);
  LAUNCH_CLS(CLS_PRE, launch_split(sp, s));
  return ADJ_OK;
}

// The fused K1 of levels 1 + 2 (preadd.cu preadd2_kernel) applies: phi = T, depth >= 2, uint16
// residues, a uint16 root view covering the whole m x k input, and both levels halve exactly
// with no padding rows or columns (m, k multiples of 512).
bool k1_fused_ok(const Plan &P, const InView &root, const uint8_t *side_arena) {
  static const bool off = getenv("ADJ_K1_UNFUSED") != nullptr;   // diagnostics (A/B)
  if (off || P.kind != PLAN_SYRK_T || P.depth < 2 || P.res32 || P.scheme > 2 ||
      side_arena != nullptr || P.shard_n > 0)
    return false;
  if ((root.type != IN_U16 && root.type != IN_U16R) || !root.vec_ok || root.rows_valid != P.m || root.cols_valid != P.k)
    return false;
  const LevelPlan &A = P.lv[1], &B = P.lv[2];
  return 2 * A.mh == P.m && 2 * A.kh == P.k && A.rows_pad == A.mh && A.kpad == A.kh && 2 * B.mh == A.mh &&
         2 * B.kh == A.kh && B.rows_pad == B.mh && B.kpad == B.kh && A.kh % 16 == 0 &&
         // 32-bit thread offsets into every level's planes (preadd.cu k1_core<O32>)
         (int64_t)P.planes * A.rows_pad * A.kpad <= (int64_t(1) << 32) &&
         (int64_t)P.planes * B.rows_pad * B.kpad <= (int64_t(1) << 32);
}

adj_status_t run_tree(const Plan &P, const InView &root, const Ptrs &x, cudaStream_t s,
                      uint8_t *side_arena = nullptr) {
  // top-down pre-additions
  const bool fused = k1_fused_ok(P, root, side_arena);
  PreParams pp1;
  std::vector<std::vector<InView>> views(P.depth + 1);
  views[1] = {root};
  for (int l = 1; l <= P.depth; ++l) {
    const LevelPlan &L = P.lv[l];
    if (l > 1) {
      const LevelPlan &Lp = P.lv[l - 1];
      views[l].resize(L.n_nodes);
      for (int n = 0; n < L.n_nodes; ++n) {
        const int parent = n / 3, c = n % 3;
        views[l][n] = child_view(views[l - 1][parent], c, Lp, c == 2 ? s3buf(P, x.ws, l - 1, parent) : nullptr, Lp.kh,
                                 P.res32);
      }
    }
    PreParams pp;
    std::memset(&pp, 0, sizeof(pp));
    pp.n_nodes = L.n_nodes;
    pp.scheme = P.scheme;
    pp.planes = P.planes;
    pp.ykind = P.Y.kind;
    pp.ya = P.Y.a;
    pp.yb = P.Y.b;
    pp.mh = L.mh;
    pp.kh = L.kh;
    pp.rows_pad = L.rows_pad;
    pp.kpad = L.kpad;
    pp.plane_bytes = L.rows_pad * L.kpad;
    pp.arena = reinterpret_cast<int8_t *>(x.ws + P.arenas[L.arena].offset);
    pp.res32 = P.res32 ? 1 : 0;
    pp.mod = P.mod;
    pp.kc = make_k1const(P.p, P.Y.a, P.Y.b);
    if (l == 1) set_shard_rows(P, pp.rows);
    for (int n = 0; n < L.n_nodes; ++n) {
      PreNode &N = pp.nodes[n];
      N.in = views[l][n];
      for (int o = 0; o < OUT_N; ++o) {
        N.op_row[o] = o < L.n_ops ? ((int64_t)n * L.n_ops + o) * P.planes * L.rows_pad : -1;
        N.op_off[o] = N.op_row[o] >= 0 ? N.op_row[o] * L.kpad : 0;
      }
      // fused levels 1 + 2 keep the level-1 S3 in registers -- unless level 3 exists: the X11 / X12
      // views of the level-2 S3 node's children point into it
      if ((l < P.depth || P.kind == PLAN_LOWMEM) && !(fused && l == 1 && P.depth == 2)) {
        N.s3 = s3buf(P, x.ws, l, n);
        N.s3_ld = L.kh;
      }
      if (l == 1 && side_arena != nullptr) {
        N.side = reinterpret_cast<int8_t *>(side_arena);
        N.side_kpad = P.kpad0;
        N.side_rows_pad = P.rows_pad0;
        N.side_x_row = P.op0_row[0];
        N.side_y_row = P.op0_row[1];
      }
    }
    if (fused && l == 1) { pp1 = pp; continue; }
    if (fused && l == 2) LAUNCH_CLS(CLS_PRE, launch_preadd2(pp1, pp, s));
    else LAUNCH_CLS(CLS_PRE, launch_preadd(pp, s));
  }
  return ADJ_OK;
}

// K1 of every level, then the grouped leaf launch
adj_status_t run_tree_leaf(const Plan &P, const InView &root, const Ptrs &x, cudaStream_t s,
                           uint8_t *side_arena = nullptr) {
  adj_status_t st = run_tree(P, root, x, s, side_arena);
  return st != ADJ_OK ? st : launch_leaf_all(P, x, s);
}

adj_status_t run_combine(const Plan &P, const Ptrs &x, void *final_out, int64_t final_ld, bool final_u32,
                         cudaStream_t s) {
  for (int l = P.depth; l >= 1; --l) {
    const LevelPlan &L = P.lv[l];
    CombParams cp;
    std::memset(&cp, 0, sizeof(cp));
    cp.n_nodes = L.n_nodes;
    cp.mh = L.mh;
    cp.ldp = L.rows_pad;
    cp.mod = P.mod;
    cp.out_u32 = (l == 1) ? (final_u32 ? 1 : 0) : 0;
    cp.in32 = P.res32 ? 1 : 0;
    if (P.res32) cp.out_u32 = 1;
    if (l == 1 && final_u32) {
      cp.alpha = x.alpha;
      cp.beta = x.beta;
      cp.axpby = x.axpby;
    }
    if (P.shard_n > 0) {          // output-tile sharding (depth 1): only this rank's tile pairs
      cp.pairs = P.d_comb_pairs;
      cp.n_pairs = (int32_t)P.comb_pairs.size();
    }
    for (int n = 0; n < L.n_nodes; ++n) {
      CombNode &N = cp.nodes[n];
      for (int i = 0; i < 5; ++i) N.P[i] = pbuf(P, x.ws, l, n, i);
      if (l == 1) {
        N.out = final_out;
        N.ldo = final_ld;
        N.out_valid = P.lv[0].mh;
      } else {
        static const int slot_of_child[3] = {0, 1, 4};   // X11 -> P1, X12 -> P2, S3 -> P5
        N.out = pbuf(P, x.ws, l - 1, n / 3, slot_of_child[n % 3]);
        N.ldo = P.lv[l - 1].rows_pad;
        N.out_valid = P.lv[l - 1].mh;
      }
    }
    LAUNCH_CLS(CLS_COMB, launch_combine(cp, s));
  }
  return ADJ_OK;
}

// phi = T through the grouped schedule: Low(x.C) = Low(V V^T) for the view `root` (m x k valid)
adj_status_t run_syrk_t(const Plan &P, const InView &root, const Ptrs &x, cudaStream_t s) {
  adj_status_t st;
  if (P.depth == 0) {
    st = run_split(P, root, P.m, P.k, P.rows_pad0, P.op0_row[0], x.ws + P.arenas[0].offset, s);
    if (st) return st;
    return launch_leaf_all(P, x, s);
  }
  st = run_tree_leaf(P, root, x, s);
  if (st) return st;
  return run_combine(P, x, x.C, x.ldc, !x.res16, s);
}

// Low-memory schedule (ADJ_LOW_MEM; plan.hpp PLAN_LOWMEM).  R is the root plan.
adj_status_t run_lowmem(const Plan &R, const InView &root, const Ptrs &x, int dev, int sms, cudaStream_t s) {
  adj_status_t st;
  const LevelPlan &L = R.lv[1];
  // K1 of the root: S1, S2, S4, A22 limb planes and S3
  if ((st = run_tree(R, root, x, s)) != ADJ_OK) return st;
  // P3 -> C21, P4 -> buffer (one grouped launch)
  if ((st = launch_leaf_all(R, x, s)) != ADJ_OK) return st;
  // the three recursive products, each an ordinary call one level shallower
  // whose workspace reuses the root's arena region: P1 = X11 X11^T -> C11, P2 = X12 X12^T ->
  // buffer, P5 = S3 S3^T -> C22 (Low parts only)
  PlanRef Q;
  if ((st = get_plan(&Q, PLAN_SYRK_T, L.mh, L.mh, L.kh, R.p, 0, R.lm_depth - 1, dev, sms)) != ADJ_OK) return st;
  if (Q->ws_bytes > R.lm_child_ws) return fail(ADJ_ERR_WORKSPACE, "low-memory child workspace");
  const size_t eb = (x.res16 && !R.res32) ? 2 : 4;
  for (int c = 0; c < 3; ++c) {
    const InView v = child_view(root, c, L, c == 2 ? x.ws + L.s3_offset : nullptr, L.kh, R.res32);
    Ptrs xc;
    xc.ws = x.ws + R.lm_region_off;
    if (c == 1) {
      xc.C = reinterpret_cast<uint32_t *>(x.ws + R.lm_p2_off);
      xc.ldc = L.rows_pad;
      xc.res16 = !R.res32;
    } else {
      const size_t off = c == 0 ? 0 : ((size_t)L.mh * (size_t)x.ldc + (size_t)L.mh) * eb;
      xc.C = reinterpret_cast<uint32_t *>(reinterpret_cast<uint8_t *>(x.C) + off);
      xc.ldc = x.ldc;
      xc.res16 = x.res16;
    }
    if ((st = run_syrk_t(*Q, v, xc, s)) != ADJ_OK) return st;
  }
  // root K4 in place (U1..U5)
  CombParams cp;
  std::memset(&cp, 0, sizeof(cp));
  cp.n_nodes = 1;
  cp.mh = L.mh;
  cp.ldp = L.rows_pad;
  cp.mod = R.mod;
  cp.in32 = R.res32 ? 1 : 0;
  cp.out_u32 = eb == 4 ? 1 : 0;
  cp.inplace = 1;
  CombNode &N = cp.nodes[0];
  N.P[1] = x.ws + R.lm_p2_off;
  N.P[3] = x.ws + R.lm_p4_off;
  N.out = x.C;
  N.ldo = x.ldc;
  N.out_valid = R.m;
  LAUNCH_CLS(CLS_COMB, launch_combine(cp, s));
  return ADJ_OK;
}

adj_status_t run_syrk(const Plan &P, const Ptrs &x, adj_phi_t phi, uint32_t flags, cudaStream_t s, int dev = 0,
                      int sms = 0) {
  adj_status_t st;
  const int64_t m = P.m, k = P.k;
  if (phi == ADJ_PHI_T) {
    InView root = make_view(x.A, x.lda, m, k, x.in16 ? IN_U16R : IN_U32);
    st = P.kind == PLAN_LOWMEM ? run_lowmem(P, root, x, dev, sms, s) : run_syrk_t(P, root, x, s);
    if (st) return st;
  } else {
    // 2M (Alg. alg:2M): A = X + iY; H = X phi(Y) = X Y^T; G = (X+Y) phi(X + eps Y), eps = 1.
    // X / Y limb planes come from the same pass over A as T (split mode 1 at depth 0, the
    // root pre-addition's side output at depth >= 1).
    uint8_t *arena0 = x.ws + P.arenas[0].offset;
    InView troot = make_view(x.A, x.lda, m, k, IN_PAIR_SUM, x.in16);
    void *G = x.ws + P.g_offset;
    void *H = x.ws + P.h_offset;
    if (P.depth == 0) {
      SplitParams sp;
      std::memset(&sp, 0, sizeof(sp));
      sp.in = troot;
      sp.rows = m; sp.cols = k;
      sp.rows_pad = P.rows_pad0; sp.kpad = P.kpad0;
      sp.op_row = P.op0_row[0]; sp.op_row2 = P.op0_row[1]; sp.op_row3 = P.op0_row[2];
      sp.arena = reinterpret_cast<int8_t *>(arena0);
      sp.scheme = P.scheme; sp.planes = P.planes; sp.mode = 1; sp.mod = P.mod;
      LAUNCH_CLS(CLS_PRE, launch_split(sp, s));
      st = launch_leaf_all(P, x, s);
      if (st) return st;
    } else {
      // arena-0 padding the root pre-addition does not cover: rows [2 mh, rows_pad0), columns [2 kh, kpad0)
      const int64_t mh = P.lv[1].mh, kh = P.lv[1].kh, rp0 = P.rows_pad0, kp0 = P.kpad0;
      for (int op = 0; op < 2; ++op)
        for (int pl = 0; pl < P.planes; ++pl) {
          uint8_t *base = arena0 + (size_t)(P.op0_row[op] + (int64_t)pl * rp0) * kp0;
          if (2 * mh < rp0) CUDA_TRY(cudaMemsetAsync(base + (size_t)(2 * mh) * kp0, 0, (size_t)(rp0 - 2 * mh) * kp0, s));
          if (2 * kh < kp0) CUDA_TRY(cudaMemset2DAsync(base + 2 * kh, kp0, 0, kp0 - 2 * kh, 2 * mh, s));
        }
      st = run_tree_leaf(P, troot, x, s, arena0);
      if (st) return st;
      st = run_combine(P, x, G, P.rows_pad0, false, s);
      if (st) return st;
    }
    LAUNCH_CLS(CLS_COMB, launch_twom(m, G, P.rows_pad0, H, P.rows_pad0, P.res32 ? 1 : 0, x.C, x.ldc, P.mod, x.alpha,
                                     x.beta, x.axpby, x.res16 ? 1 : 0, s));
  }
  if (flags & ADJ_FILL_UPPER) LAUNCH(launch_fill_upper(m, adj_phi_width(phi), x.C, x.ldc, P.mod, s));
  return ADJ_OK;
}

// phi = Q: Alg. alg:2M3M.  One read of M gives the limb planes of A, B, C,
// D, U1 = A + B, U2 = C + D (and W = U1 + U2 at depth 0); Q1..Q5 and Q6 = Low(W W^T) (through
// Alg. alg:MIAHMM when depth >= 1, its root pre-addition reading W = x1 + x2 + x3 + x4 from M)
// share one grouped leaf launch; the 6M combine forms H1..H4.
adj_status_t run_quat(const Plan &P, const Ptrs &x, uint32_t flags, cudaStream_t s) {
  const int64_t m = P.m, k = P.k;
  SplitParams sp;
  std::memset(&sp, 0, sizeof(sp));
  sp.in = make_view(x.A, x.lda, m, k, IN_QUAD_SUM, x.in16);
  sp.rows = m; sp.cols = k;
  sp.rows_pad = P.rows_pad0; sp.kpad = P.kpad0;
  sp.arena = reinterpret_cast<int8_t *>(x.ws + P.arenas[0].offset);
  sp.scheme = P.scheme; sp.planes = P.planes; sp.mode = 2; sp.mod = P.mod;
  for (int o = 0; o < QO_N; ++o) sp.qrow[o] = P.q_row[o];
  LAUNCH_CLS(CLS_PRE, launch_split(sp, s));
  adj_status_t st;
  void *G = x.ws + P.g_offset;
  st = P.depth >= 1 ? run_tree_leaf(P, make_view(x.A, x.lda, m, k, IN_QUAD_SUM, x.in16), x, s)
                    : launch_leaf_all(P, x, s);
  if (st) return st;
  if (P.depth >= 1) {
    st = run_combine(P, x, G, P.rows_pad0, false, s);
    if (st) return st;
  }
  QuatCombParams qp;
  std::memset(&qp, 0, sizeof(qp));
  for (int q = 0; q < 5; ++q) qp.Q[q] = x.ws + P.q_offset + (size_t)q * P.q_bytes;
  qp.Q[5] = G;
  qp.m = m; qp.ldq = P.rows_pad0;
  qp.C = x.C; qp.ldc = x.ldc;
  qp.mod = P.mod;
  qp.alpha = x.alpha; qp.beta = x.beta; qp.axpby = x.axpby;
  qp.in32 = P.res32 ? 1 : 0;
  qp.out16 = x.res16 ? 1 : 0;
  LAUNCH_CLS(CLS_COMB, launch_quat_combine(qp, s));
  if (flags & ADJ_FILL_UPPER) LAUNCH(launch_fill_upper(m, 4, x.C, x.ldc, P.mod, s));
  return ADJ_OK;
}

// phi = H by one level of Alg. alg:MIAHMM over GF(p^2) (ADJ_HERK_ALG1): K1 over GF(p^2), one
// grouped leaf launch (2M for P1, P2, P5; 3M for P3, P4), then the fused GF(p^2) K4.
adj_status_t run_herk1(const Plan &P, const Ptrs &x, uint32_t flags, cudaStream_t s) {
  const LevelPlan &L = P.lv[1];
  HerkPreParams hp;
  std::memset(&hp, 0, sizeof(hp));
  hp.in = make_view(x.A, x.lda, P.m, P.k, IN_PAIR_RE, x.in16);
  hp.mh = L.mh; hp.kh = L.kh;
  hp.rows_pad = L.rows_pad; hp.kpad = L.kpad;
  hp.arena = reinterpret_cast<int8_t *>(x.ws + P.arenas[0].offset);
  hp.scheme = P.scheme; hp.planes = P.planes;
  hp.ya = P.Y.a; hp.yb = P.Y.b;
  hp.mod = P.mod;
  LAUNCH_CLS(CLS_PRE, launch_herk_preadd(hp, s));
  adj_status_t st = launch_leaf_all(P, x, s);
  if (st) return st;
  HerkCombParams cp;
  std::memset(&cp, 0, sizeof(cp));
  for (int b = 0; b < HB_N; ++b) cp.B[b] = x.ws + P.hb_offset + (size_t)b * P.hb_bytes;
  cp.mh = L.mh; cp.ldp = L.rows_pad;
  cp.C = x.C; cp.ldc = x.ldc; cp.out_valid = P.m;
  cp.mod = P.mod;
  cp.alpha = x.alpha; cp.beta = x.beta; cp.axpby = x.axpby;
  cp.in32 = P.res32 ? 1 : 0;
  LAUNCH_CLS(CLS_COMB, launch_herk_combine(cp, s));
  if (flags & ADJ_FILL_UPPER) LAUNCH(launch_fill_upper(P.m, 2, x.C, x.ldc, P.mod, s));
  return ADJ_OK;
}

adj_status_t validate_syrk(int64_t m, int64_t k, uint32_t p, adj_phi_t phi, const uint32_t *A, int64_t lda,
                           const uint32_t *C, int64_t ldc, uint32_t flags = 0) {
  if (m < 0 || k < 0) return fail(ADJ_ERR_INVALID_VALUE, "negative dimension (m=%lld, k=%lld)", (long long)m, (long long)k);
  if (phi != ADJ_PHI_T && phi != ADJ_PHI_H && phi != ADJ_PHI_Q)
    return fail(ADJ_ERR_INVALID_VALUE, "phi must be ADJ_PHI_T, ADJ_PHI_H or ADJ_PHI_Q");
  if (!valid_modulus(p)) return fail(ADJ_ERR_UNSUPPORTED_MODULUS, "p=%u is not an odd prime in [3, 262139]", p);
  if (phi == ADJ_PHI_H && p % 4 != 3)
    return fail(ADJ_ERR_UNSUPPORTED_MODULUS, "phi=H needs p = 3 mod 4 (GF(p)[i]/(i^2+1)); p=%u", p);
  if (m == 0) return ADJ_OK;
  if (C == nullptr) return fail(ADJ_ERR_INVALID_VALUE, "C is null");
  if (k > 0 && A == nullptr) return fail(ADJ_ERR_INVALID_VALUE, "A is null");
  if (lda < k || (lda < 1 && k > 0)) return fail(ADJ_ERR_INVALID_VALUE, "lda=%lld < k=%lld", (long long)lda, (long long)k);
  if (ldc < m) return fail(ADJ_ERR_INVALID_VALUE, "ldc=%lld < m=%lld", (long long)ldc, (long long)m);
  const int w = adj_phi_width(phi);
  const int ea = (flags & ADJ_IN_U16) ? 2 * w : 4 * w, ec = (flags & ADJ_OUT_U16) ? 2 * w : 4 * w;
  if (overlap(A, span_bytes(m, k, lda, ea), C, span_bytes(m, m, ldc, ec)))
    return fail(ADJ_ERR_INVALID_VALUE, "A and C overlap");
  return ADJ_OK;
}

}  // namespace

// ==================================================================== C ABI
extern "C" {

const char *adj_status_string(adj_status_t s) {
  switch (s) {
    case ADJ_OK: return "ADJ_OK";
    case ADJ_ERR_INVALID_VALUE: return "ADJ_ERR_INVALID_VALUE";
    case ADJ_ERR_UNSUPPORTED_MODULUS: return "ADJ_ERR_UNSUPPORTED_MODULUS";
    case ADJ_ERR_WORKSPACE: return "ADJ_ERR_WORKSPACE";
    case ADJ_ERR_CUDA: return "ADJ_ERR_CUDA";
    case ADJ_ERR_NCCL: return "ADJ_ERR_NCCL";
    case ADJ_ERR_ARCH: return "ADJ_ERR_ARCH";
  }
  return "ADJ_ERR_UNKNOWN";
}

const char *adj_last_error(void) { return g_last_error.c_str(); }
uint64_t adj_launch_count(void) { return g_launches.load(); }

void adj_profile_enable(int on) { g_prof_on.store(on ? 1 : 0); }

adj_status_t adj_profile_read(double ms[4], uint64_t launches[4]) {
  if (!ms || !launches) return fail(ADJ_ERR_INVALID_VALUE, "null output");
  std::vector<ProfRec> recs;
  {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    recs.swap(g_prof);
  }
  for (int c = 0; c < 4; ++c) { ms[c] = 0; launches[c] = 0; }
  for (auto &r : recs) {
    float t = 0;
    CUDA_TRY(cudaEventSynchronize(r.b));
    CUDA_TRY(cudaEventElapsedTime(&t, r.a, r.b));
    ms[r.cls] += t;
    launches[r.cls] += 1;
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  return ADJ_OK;
}
void adj_launch_count_reset(void) { g_launches.store(0); }

adj_status_t adj_sos(uint32_t p, uint32_t k, uint32_t *a, uint32_t *b) {
  if (!a || !b) return fail(ADJ_ERR_INVALID_VALUE, "null output");
  if (p < 3 || !is_prime_u32(p)) return fail(ADJ_ERR_UNSUPPORTED_MODULUS, "p=%u is not an odd prime", p);
  sos(k, p, a, b);
  return ADJ_OK;
}

adj_status_t adj_skew_unitary(uint32_t p, adj_phi_t phi, int *kind, uint32_t *a, uint32_t *b) {
  if (!kind || !a || !b) return fail(ADJ_ERR_INVALID_VALUE, "null output");
  if (!valid_modulus(p)) return fail(ADJ_ERR_UNSUPPORTED_MODULUS, "p=%u is not an odd prime in [3, 262139]", p);
  if (phi == ADJ_PHI_H && p % 4 != 3) return fail(ADJ_ERR_UNSUPPORTED_MODULUS, "phi=H needs p = 3 mod 4");
  SkewY y = skew_unitary(p);
  *kind = y.kind;
  *a = y.a;
  *b = y.b;
  return ADJ_OK;
}

adj_status_t adjprod_modp_auto_depth(int64_t m, int64_t k, uint32_t p, adj_phi_t phi, int *depth) {
  if (!depth) return fail(ADJ_ERR_INVALID_VALUE, "null output");
  *depth = auto_depth(m, k, p, (int)phi);
  return ADJ_OK;
}

adj_status_t adjprod_modp_workspace_size(int64_t m, int64_t k, uint32_t p, adj_phi_t phi, const adj_opts_t *opts,
                                         size_t *bytes) {
  if (!bytes) return fail(ADJ_ERR_INVALID_VALUE, "null output");
  if (m < 0 || k < 0) return fail(ADJ_ERR_INVALID_VALUE, "negative dimension");
  if (!valid_modulus(p)) return fail(ADJ_ERR_UNSUPPORTED_MODULUS, "p=%u is not an odd prime in [3, 262139]", p);
  if (m == 0 || k == 0) { *bytes = 0; return ADJ_OK; }
  const bool herk1 = phi == ADJ_PHI_H && opts && (opts->flags & ADJ_HERK_ALG1);
  int depth = (opts && opts->depth >= 0) ? opts->depth : (herk1 ? 1 : auto_depth(m, k, p, (int)phi));
  if (herk1 && depth != 1) return fail(ADJ_ERR_INVALID_VALUE, "ADJ_HERK_ALG1 runs exactly one level (depth 1 or -1)");
  Plan P;
  const char *err = nullptr;
  const int sms = query_sms();
  const bool lowmem = opts && (opts->flags & ADJ_LOW_MEM) && phi == ADJ_PHI_T && lowmem_shape_ok(m, k, depth);
  if (!(herk1    ? build_herk1_plan(P, m, k, p, sms, &err)
        : lowmem ? build_lowmem_plan(P, m, k, p, depth, sms, &err)
                 : build_syrk_plan(P, m, k, p, (int)phi, depth, sms, &err)))
    return fail(ADJ_ERR_INVALID_VALUE, "plan: %s", err ? err : "unsupported");
  *bytes = P.ws_bytes;
  return ADJ_OK;
}

adj_status_t adjprod_modp_leaf_tile(int64_t m, int64_t k, uint32_t p, adj_phi_t phi, const adj_opts_t *opts,
                                    int *tile_n) {
  if (!tile_n) return fail(ADJ_ERR_INVALID_VALUE, "null output");
  if (m < 0 || k < 0) return fail(ADJ_ERR_INVALID_VALUE, "negative dimension");
  if (!valid_modulus(p)) return fail(ADJ_ERR_UNSUPPORTED_MODULUS, "p=%u is not an odd prime in [3, 262139]", p);
  *tile_n = 256;
  if (m == 0 || k == 0) return ADJ_OK;
  const bool herk1 = phi == ADJ_PHI_H && opts && (opts->flags & ADJ_HERK_ALG1);
  const int depth = (opts && opts->depth >= 0) ? opts->depth : (herk1 ? 1 : auto_depth(m, k, p, (int)phi));
  Plan P;
  const char *err = nullptr;
  const int sms = query_sms();
  const bool lowmem = opts && (opts->flags & ADJ_LOW_MEM) && phi == ADJ_PHI_T && lowmem_shape_ok(m, k, depth);
  if (!(herk1    ? build_herk1_plan(P, m, k, p, sms, &err)
        : lowmem ? build_lowmem_plan(P, m, k, p, depth, sms, &err)
                 : build_syrk_plan(P, m, k, p, (int)phi, depth, sms, &err)))
    return fail(ADJ_ERR_INVALID_VALUE, "plan: %s", err ? err : "unsupported");
  *tile_n = P.tile_n;
  return ADJ_OK;
}

static adj_status_t adjprod_impl(int64_t m, int64_t k, uint32_t p, adj_phi_t phi, uint32_t alpha, const uint32_t *A,
                                 int64_t lda, uint32_t beta, uint32_t *C, int64_t ldc, const adj_opts_t *opts,
                                 cudaStream_t s) {
  const uint32_t flags = opts ? opts->flags : 0;
  adj_status_t st = validate_syrk(m, k, p, phi, A, lda, C, ldc, flags);
  if (st != ADJ_OK) return st;
  alpha %= p;
  beta %= p;
  const int axpby = !(alpha == 1 && beta == 0);
  const bool in16 = flags & ADJ_IN_U16, out16 = flags & ADJ_OUT_U16;
  if ((in16 || out16) && p > 65535)
    return fail(ADJ_ERR_INVALID_VALUE, "ADJ_IN_U16 / ADJ_OUT_U16 need p < 2^16");
  if (out16 && (axpby || (flags & (ADJ_FILL_UPPER | ADJ_HERK_ALG1))))
    return fail(ADJ_ERR_INVALID_VALUE, "ADJ_OUT_U16 is the plain form: no alpha / beta, ADJ_FILL_UPPER or ADJ_HERK_ALG1");
  if (m == 0) return ADJ_OK;
  int dev, sms;
  if ((st = check_device(&dev, &sms)) != ADJ_OK) return st;
  const int w = adj_phi_width(phi);
  if (k == 0 || alpha == 0) {  // Low(C) = beta Low(C)
    if (out16) {
      LAUNCH(launch_zero_lower(m, C, ldc * w * 2, 2 * w, s));
      return ADJ_OK;
    }
    if (beta == 0) {
      LAUNCH(launch_zero_lower(m, C, ldc * w * 4, 4 * w, s));
    } else {
      LAUNCH(launch_scale_lower(m, w, C, ldc, beta, make_modp(p), s));
    }
    if (flags & ADJ_FILL_UPPER) LAUNCH(launch_fill_upper(m, w, C, ldc, make_modp(p), s));
    return ADJ_OK;
  }
  const bool herk1 = phi == ADJ_PHI_H && (flags & ADJ_HERK_ALG1);
  int depth = (opts && opts->depth >= 0) ? opts->depth : (herk1 ? 1 : auto_depth(m, k, p, (int)phi));
  if (depth > 3) return fail(ADJ_ERR_INVALID_VALUE, "depth %d > 3 unsupported", depth);
  if (herk1 && depth != 1) return fail(ADJ_ERR_INVALID_VALUE, "ADJ_HERK_ALG1 runs exactly one level (depth 1 or -1)");
  // low-memory schedule (ADJ_LOW_MEM): where it applies; the in-place K4 reads C with 16-byte loads
  const bool lm_applies = phi == ADJ_PHI_T && !axpby && lowmem_shape_ok(m, k, depth);
  const bool lm_aligned = (uintptr_t)C % 16 == 0 && ldc % 8 == 0;
  const bool lowmem = (flags & ADJ_LOW_MEM) && lm_applies;
  if (lowmem && !lm_aligned)
    return fail(ADJ_ERR_INVALID_VALUE, "ADJ_LOW_MEM needs C 16-byte aligned and ldc %% 8 == 0");
  PlanRef P;
  const int kind = herk1 ? PLAN_HERK1
                   : lowmem ? PLAN_LOWMEM
                   : (phi == ADJ_PHI_T ? PLAN_SYRK_T : (phi == ADJ_PHI_H ? PLAN_SYRK_H : PLAN_QUAT));
  if ((st = get_plan(&P, kind, m, m, k, p, (int)phi, depth, dev, sms)) != ADJ_OK) return st;
  // automatic fall-back to the low-memory schedule: a caller workspace too small for the grouped
  // schedule but large enough for it, or a failed library workspace allocation
  const bool lm_fallback = !lowmem && lm_applies && lm_aligned;
  auto to_lowmem = [&]() -> adj_status_t { return get_plan(&P, PLAN_LOWMEM, m, m, k, p, (int)phi, depth, dev, sms); };
  Ptrs x;
  x.A = A; x.lda = lda; x.C = C; x.ldc = ldc;
  x.alpha = alpha; x.beta = beta; x.axpby = axpby;
  x.in16 = in16;
  x.res16 = out16;
  void *ws = opts ? opts->workspace : nullptr;
  bool own = false;
  if (ws == nullptr) {
    cudaError_t e = adj_pool_alloc(&ws, P->ws_bytes, s);
    if (e != cudaSuccess && lm_fallback) {
      cudaGetLastError();
      if ((st = to_lowmem()) != ADJ_OK) return st;
      e = adj_pool_alloc(&ws, P->ws_bytes, s);
    }
    if (e != cudaSuccess) return fail(ADJ_ERR_WORKSPACE, "workspace allocation of %zu bytes: %s", P->ws_bytes,
                                      cudaGetErrorString(e));
    own = true;
  } else if (opts->workspace_bytes < P->ws_bytes) {
    if (lm_fallback && (st = to_lowmem()) != ADJ_OK) return st;
    if (opts->workspace_bytes < P->ws_bytes)
      return fail(ADJ_ERR_WORKSPACE, "workspace %zu bytes < required %zu", opts->workspace_bytes, P->ws_bytes);
  }
  x.ws = static_cast<uint8_t *>(ws);
  st = herk1 ? run_herk1(*P, x, flags, s)
              : (phi == ADJ_PHI_Q ? run_quat(*P, x, flags, s) : run_syrk(*P, x, phi, flags, s, dev, sms));
  if (own) {
    cudaError_t e = cudaFreeAsync(ws, s);
    if (st == ADJ_OK && e != cudaSuccess) return fail(ADJ_ERR_CUDA, "cudaFreeAsync: %s", cudaGetErrorString(e));
  }
  return st;
}

static adj_status_t shard_plan(PlanRef *out, int64_t m, int64_t k, uint32_t p, int depth, int rank, int nranks, int dev,
                               int sms) {
  return get_plan(out, PLAN_SYRK_T, m, m, std::max<int64_t>(k, 1), p, 0, depth, dev, sms, rank, nranks);
}

static int shard_depth(int64_t m, int64_t k, uint32_t p, const adj_opts_t *opts) {
  return (opts && opts->depth >= 0) ? opts->depth : std::min(1, auto_depth(m, std::max<int64_t>(k, 1), p, 0));
}

adj_status_t adjprod_modp_shard(int64_t m, int64_t k, uint32_t p, adj_phi_t phi, const uint32_t *A, int64_t lda,
                                uint32_t *C, int64_t ldc, int rank, int nranks, const adj_opts_t *opts,
                                adj_stream_t stream) {
  const uint32_t flags = opts ? opts->flags : 0;
  adj_status_t st = validate_syrk(m, k, p, phi, A, lda, C, ldc, flags & ADJ_IN_U16);
  if (st != ADJ_OK) return st;
  if (phi != ADJ_PHI_T) return fail(ADJ_ERR_INVALID_VALUE, "output-tile sharding supports phi = ADJ_PHI_T");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(ADJ_ERR_INVALID_VALUE, "rank %d of %d", rank, nranks);
  if (flags & ADJ_FILL_UPPER) return fail(ADJ_ERR_INVALID_VALUE, "ADJ_FILL_UPPER with sharding");
  if (flags & ADJ_OUT_U16) return fail(ADJ_ERR_INVALID_VALUE, "ADJ_OUT_U16 is an adjprod_modp_ex flag");
  if ((flags & ADJ_IN_U16) && p > 65535) return fail(ADJ_ERR_INVALID_VALUE, "ADJ_IN_U16 needs p < 2^16");
  if (m == 0) return ADJ_OK;
  const int depth = shard_depth(m, k, p, opts);
  if (depth > 1) return fail(ADJ_ERR_INVALID_VALUE, "output-tile sharding runs at depth 0 or 1 (got %d)", depth);
  int dev, sms;
  if ((st = check_device(&dev, &sms)) != ADJ_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  PlanRef P;
  if ((st = shard_plan(&P, m, k, p, depth, rank, nranks, dev, sms)) != ADJ_OK) return st;
  if (P->shard_rects.empty()) return ADJ_OK;   // more ranks than tile pairs: this rank owns nothing
  if (k == 0) {   // Low(C) = 0 on the owned regions: one launch over the region list
    if (P->shard_rects.empty()) return ADJ_OK;
    std::vector<RectDev> rd(P->shard_rects.size());
    int max_rows = 0;
    for (size_t i = 0; i < rd.size(); ++i) {
      const ShardRect &R = P->shard_rects[i];
      rd[i].r0 = R.r0; rd[i].c0 = R.c0; rd[i].rows = R.rows; rd[i].cols = R.cols;
      rd[i].lower = R.lower ? 1 : 0; rd[i].pad_ = 0; rd[i].off = 0;
      max_rows = std::max<int>(max_rows, (int)R.rows);
    }
    void *d = nullptr;
    CUDA_TRY(adj_pool_alloc(&d, rd.size() * sizeof(RectDev), s));
    CUDA_TRY(cudaMemcpyAsync(d, rd.data(), rd.size() * sizeof(RectDev), cudaMemcpyHostToDevice, s));
    LAUNCH(launch_rect_copy(static_cast<RectDev *>(d), (int)rd.size(), max_rows, C, ldc, d, 4, 2, s));
    CUDA_TRY(cudaFreeAsync(d, s));
    return ADJ_OK;
  }
  Ptrs x;
  x.A = A; x.lda = lda; x.C = C; x.ldc = ldc;
  x.in16 = (flags & ADJ_IN_U16) != 0;
  void *ws = opts ? opts->workspace : nullptr;
  bool own = false;
  if (ws == nullptr) {
    CUDA_TRY(adj_pool_alloc(&ws, P->ws_bytes, s));
    own = true;
  } else if (opts->workspace_bytes < P->ws_bytes) {
    return fail(ADJ_ERR_WORKSPACE, "workspace %zu bytes < required %zu", opts->workspace_bytes, P->ws_bytes);
  }
  x.ws = static_cast<uint8_t *>(ws);
  st = run_syrk(*P, x, phi, 0, s);
  if (own) {
    cudaError_t e = cudaFreeAsync(ws, s);
    if (st == ADJ_OK && e != cudaSuccess) return fail(ADJ_ERR_CUDA, "cudaFreeAsync: %s", cudaGetErrorString(e));
  }
  return st;
}

adj_status_t adjprod_modp_partial(int64_t m, int64_t k, uint32_t p, adj_phi_t phi, const uint32_t *A, int64_t lda,
                                  void *R, int64_t ldr, const adj_opts_t *opts, adj_stream_t stream) {
  const uint32_t flags = opts ? opts->flags : 0;
  // R holds uint16 residues for p < 2^16 (ADJ_OUT_U16's width for the overlap check), uint32 otherwise
  adj_status_t st = validate_syrk(m, k, p, phi, A, lda, static_cast<const uint32_t *>(R), ldr,
                                  (flags & ADJ_IN_U16) | (p < 65536 ? ADJ_OUT_U16 : 0u));
  if (st != ADJ_OK) return st;
  if (phi != ADJ_PHI_T) return fail(ADJ_ERR_INVALID_VALUE, "adjprod_modp_partial supports phi = ADJ_PHI_T");
  if (flags & ADJ_OUT_U16) return fail(ADJ_ERR_INVALID_VALUE, "ADJ_OUT_U16 is an adjprod_modp_ex flag");
  if ((flags & ADJ_IN_U16) && p > 65535) return fail(ADJ_ERR_INVALID_VALUE, "ADJ_IN_U16 needs p < 2^16");
  if (m == 0) return ADJ_OK;
  if (p > 65535) {   // residues need 32 bits: the ordinary call writes them
    adj_opts_t o = opts ? *opts : adj_opts_t{-1, 0, nullptr, 0};
    o.flags &= ~ADJ_FILL_UPPER;
    return adjprod_modp_ex(m, k, p, phi, A, lda, static_cast<uint32_t *>(R), ldr, &o, stream);
  }
  int dev, sms;
  if ((st = check_device(&dev, &sms)) != ADJ_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  uint16_t *R16 = static_cast<uint16_t *>(R);
  if (k == 0) {
    LAUNCH(launch_zero_lower(m, R16, ldr * 2, 2, s));
    return ADJ_OK;
  }
  const int depth = (opts && opts->depth >= 0) ? opts->depth : auto_depth(m, k, p, 0);
  if (depth > 3) return fail(ADJ_ERR_INVALID_VALUE, "depth %d > 3 unsupported", depth);
  PlanRef P;
  if ((st = get_plan(&P, PLAN_SYRK_T, m, m, k, p, 0, depth, dev, sms)) != ADJ_OK) return st;
  Ptrs x;
  x.A = A; x.lda = lda;
  x.C = static_cast<uint32_t *>(R); x.ldc = ldr;
  x.res16 = true;
  x.in16 = (flags & ADJ_IN_U16) != 0;
  void *ws = opts ? opts->workspace : nullptr;
  bool own = false;
  if (ws == nullptr) {
    CUDA_TRY(adj_pool_alloc(&ws, P->ws_bytes, s));
    own = true;
  } else if (opts->workspace_bytes < P->ws_bytes) {
    return fail(ADJ_ERR_WORKSPACE, "workspace %zu bytes < required %zu", opts->workspace_bytes, P->ws_bytes);
  }
  x.ws = static_cast<uint8_t *>(ws);
  st = run_syrk(*P, x, phi, 0, s);
  if (own) {
    cudaError_t e = cudaFreeAsync(ws, s);
    if (st == ADJ_OK && e != cudaSuccess) return fail(ADJ_ERR_CUDA, "cudaFreeAsync: %s", cudaGetErrorString(e));
  }
  return st;
}

adj_status_t adj_sum_partials(int64_t m, uint32_t p, const void *R, int64_t ldr, int64_t stride, int n, uint32_t *C,
                              int64_t ldc, adj_stream_t stream) {
  if (m < 0 || n < 0 || ldr < m || ldc < m || stride < 0) return fail(ADJ_ERR_INVALID_VALUE, "bad arguments");
  if (!valid_modulus(p)) return fail(ADJ_ERR_UNSUPPORTED_MODULUS, "p=%u is not an odd prime in [3, 262139]", p);
  if (m == 0) return ADJ_OK;
  if (!C || (n > 0 && !R)) return fail(ADJ_ERR_INVALID_VALUE, "null pointer");
  if ((uint64_t)n * (p - 1) >= (1ull << 32)) return fail(ADJ_ERR_INVALID_VALUE, "too many partials for exact uint32 sums");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  LAUNCH(launch_sum_partials(m, R, ldr, stride, n, p > 65535 ? 4 : 2, C, ldc, make_modp(p), s));
  return ADJ_OK;
}

adj_status_t adj_shard_layout(int64_t m, int64_t k, uint32_t p, int depth, int rank, int nranks, int64_t *rects,
                              int64_t max_rects, int64_t *n_rects, int64_t *n_elems) {
  if (!n_rects || !n_elems) return fail(ADJ_ERR_INVALID_VALUE, "null output");
  if (m < 0 || k < 0 || nranks < 1 || rank < 0 || rank >= nranks) return fail(ADJ_ERR_INVALID_VALUE, "bad arguments");
  if (!valid_modulus(p)) return fail(ADJ_ERR_UNSUPPORTED_MODULUS, "p=%u is not an odd prime in [3, 262139]", p);
  *n_rects = 0;
  *n_elems = 0;
  if (m == 0) return ADJ_OK;
  adj_opts_t o{depth, 0, nullptr, 0};
  const int d = shard_depth(m, k, p, &o);
  if (d > 1) return fail(ADJ_ERR_INVALID_VALUE, "output-tile sharding runs at depth 0 or 1 (got %d)", d);
  Plan P;
  const char *err = nullptr;
  if (!build_syrk_plan(P, m, std::max<int64_t>(k, 1), p, 0, d, query_sms(), &err, rank, nranks))
    return fail(ADJ_ERR_INVALID_VALUE, "plan: %s", err ? err : "unsupported");
  *n_rects = (int64_t)P.shard_rects.size();
  for (size_t i = 0; i < P.shard_rects.size(); ++i) {
    const ShardRect &R = P.shard_rects[i];
    *n_elems += R.rows * R.cols;
    if (rects && (int64_t)i < max_rects) {
      rects[5 * i] = R.r0; rects[5 * i + 1] = R.c0; rects[5 * i + 2] = R.rows; rects[5 * i + 3] = R.cols;
      rects[5 * i + 4] = R.lower;
    }
  }
  return ADJ_OK;
}

adj_status_t adj_shard_rows(int64_t m, int64_t k, uint32_t p, int depth, int rank, int nranks, int64_t *ranges,
                            int64_t max_ranges, int64_t *n_ranges) {
  if (!n_ranges) return fail(ADJ_ERR_INVALID_VALUE, "null output");
  if (m < 0 || k < 0 || nranks < 1 || rank < 0 || rank >= nranks) return fail(ADJ_ERR_INVALID_VALUE, "bad arguments");
  if (!valid_modulus(p)) return fail(ADJ_ERR_UNSUPPORTED_MODULUS, "p=%u is not an odd prime in [3, 262139]", p);
  *n_ranges = 0;
  if (m == 0) return ADJ_OK;
  adj_opts_t o{depth, 0, nullptr, 0};
  const int d = shard_depth(m, k, p, &o);
  if (d > 1) return fail(ADJ_ERR_INVALID_VALUE, "output-tile sharding runs at depth 0 or 1 (got %d)", d);
  Plan P;
  const char *err = nullptr;
  if (!build_syrk_plan(P, m, std::max<int64_t>(k, 1), p, 0, d, query_sms(), &err, rank, nranks))
    return fail(ADJ_ERR_INVALID_VALUE, "plan: %s", err ? err : "unsupported");
  *n_ranges = (int64_t)P.shard_rows.size();
  for (size_t i = 0; i < P.shard_rows.size(); ++i)
    if (ranges && (int64_t)i < max_ranges) {
      ranges[2 * i] = P.shard_rows[i].first;
      ranges[2 * i + 1] = P.shard_rows[i].second;
    }
  return ADJ_OK;
}

adj_status_t adjprod_modp_ex(int64_t m, int64_t k, uint32_t p, adj_phi_t phi, const uint32_t *A, int64_t lda,
                             uint32_t *C, int64_t ldc, const adj_opts_t *opts, adj_stream_t stream) {
  return adjprod_impl(m, k, p, phi, 1, A, lda, 0, C, ldc, opts, reinterpret_cast<cudaStream_t>(stream));
}

adj_status_t adjprod_modp_syrk(int64_t m, int64_t k, uint32_t p, adj_phi_t phi, uint32_t alpha, const uint32_t *A,
                               int64_t lda, uint32_t beta, uint32_t *C, int64_t ldc, const adj_opts_t *opts,
                               adj_stream_t stream) {
  return adjprod_impl(m, k, p, phi, alpha, A, lda, beta, C, ldc, opts, reinterpret_cast<cudaStream_t>(stream));
}

adj_status_t adjprod_modp(int64_t m, int64_t k, uint32_t p, adj_phi_t phi, const uint32_t *A, int64_t lda,
                          uint32_t *C, int64_t ldc, adj_stream_t stream) {
  return adjprod_modp_ex(m, k, p, phi, A, lda, C, ldc, nullptr, stream);
}

adj_status_t gemm_modp(int64_t m, int64_t n, int64_t k, uint32_t p, const uint32_t *A, int64_t lda,
                       const uint32_t *B, int64_t ldb, uint32_t *C, int64_t ldc, adj_stream_t stream) {
  if (m < 0 || n < 0 || k < 0) return fail(ADJ_ERR_INVALID_VALUE, "negative dimension");
  if (!valid_modulus(p)) return fail(ADJ_ERR_UNSUPPORTED_MODULUS, "p=%u is not an odd prime in [3, 262139]", p);
  if (m == 0 || n == 0) return ADJ_OK;
  if (!C || (k > 0 && (!A || !B))) return fail(ADJ_ERR_INVALID_VALUE, "null pointer");
  if (lda < k || ldb < k || ldc < n) return fail(ADJ_ERR_INVALID_VALUE, "leading dimension too small");
  if (overlap(A, span_bytes(m, k, lda, 4), C, span_bytes(m, n, ldc, 4)) ||
      overlap(B, span_bytes(n, k, ldb, 4), C, span_bytes(m, n, ldc, 4)))
    return fail(ADJ_ERR_INVALID_VALUE, "C overlaps an input");
  adj_status_t st;
  int dev, sms;
  if ((st = check_device(&dev, &sms)) != ADJ_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (k == 0) {
    CUDA_TRY(cudaMemset2DAsync(C, (size_t)ldc * 4, 0, (size_t)n * 4, (size_t)m, s));
    return ADJ_OK;
  }
  PlanRef P;
  if ((st = get_plan(&P, PLAN_GEMM, m, n, k, p, 0, 0, dev, sms)) != ADJ_OK) return st;
  void *ws = nullptr;
  CUDA_TRY(adj_pool_alloc(&ws, P->ws_bytes, s));
  Ptrs x;
  x.A = A; x.lda = lda; x.B = B; x.ldb = ldb; x.C = C; x.ldc = ldc;
  x.ws = static_cast<uint8_t *>(ws);
  uint8_t *arena = x.ws + P->arenas[0].offset;
  st = run_split(*P, make_view(A, lda, m, k, IN_U32), m, k, P->rows_pad0, P->op0_row[0], arena, s);
  if (st == ADJ_OK) st = run_split(*P, make_view(B, ldb, n, k, IN_U32), n, k, P->rows_pad_b, P->op0_row[1], arena, s);
  if (st == ADJ_OK) st = launch_leaf_all(*P, x, s);
  cudaError_t e = cudaFreeAsync(ws, s);
  if (st == ADJ_OK && e != cudaSuccess) return fail(ADJ_ERR_CUDA, "cudaFreeAsync: %s", cudaGetErrorString(e));
  return st;
}

adj_status_t adj_mod_lower(int64_t m, uint32_t p, adj_phi_t phi, uint32_t *X, int64_t ldx, adj_stream_t stream) {
  if (m < 0 || ldx < m) return fail(ADJ_ERR_INVALID_VALUE, "bad dimensions");
  if (!valid_modulus(p)) return fail(ADJ_ERR_UNSUPPORTED_MODULUS, "p=%u is not an odd prime in [3, 262139]", p);
  if (m == 0) return ADJ_OK;
  if (!X) return fail(ADJ_ERR_INVALID_VALUE, "X is null");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  LAUNCH(launch_mod_lower(m, adj_phi_width(phi), X, ldx, X, ldx, make_modp(p), s));
  return ADJ_OK;
}

}  // extern "C"
