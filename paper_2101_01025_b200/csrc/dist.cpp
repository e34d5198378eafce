// Multi-GPU split-K over NCCL: every rank computes Low(A_r phi(A_r)) on its
// column slice with the single-GPU path, the residue partials are summed exactly by an NCCL
// uint32 reduce (sum < G p < 2^32) and reduced mod p on the root.  NCCL is resolved with
// dlopen at first use (the torch-bundled libnccl.so.2 when running inside torch).
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/adjprod.h"
#include "kernels.hpp"

struct adj_comm_s {
  ncclComm_t comm;
  int nranks, rank;
  // ADJ_DIST_P2P exchange window: the root's G partial slots; the other ranks map it with CUDA
  // IPC (peer memory over NVLink) and write their partials into it from the final kernel
  void *win = nullptr;
  size_t win_bytes = 0;
  int win_root = -1;
  bool win_owned = false;        // root: cudaMalloc'ed; others: IPC-mapped
  void *d_scratch = nullptr;     // 128-byte device buffer: IPC record broadcast and barrier token
};

namespace {

struct NcclApi {
  bool loaded = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;
std::mutex g_nccl_mu;
thread_local std::string g_dist_err;

bool load_nccl() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.loaded) return true;
  void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) { g_dist_err = "libnccl.so.2 not found"; return false; }
#define SYM(name, field)                                                       \
  *reinterpret_cast<void **>(&g_nccl.field) = dlsym(h, name);                  \
  if (!g_nccl.field) { g_dist_err = "NCCL symbol missing: " name; return false; }
  SYM("ncclGetUniqueId", GetUniqueId)
  SYM("ncclCommInitRank", CommInitRank)
  SYM("ncclCommDestroy", CommDestroy)
  SYM("ncclReduce", Reduce)
  SYM("ncclSend", Send)
  SYM("ncclRecv", Recv)
  SYM("ncclGroupStart", GroupStart)
  SYM("ncclBroadcast", Broadcast)
  SYM("ncclAllReduce", AllReduce)
  SYM("ncclGroupEnd", GroupEnd)
  SYM("ncclGetErrorString", GetErrorString)
#undef SYM
  g_nccl.loaded = true;
  return true;
}

}  // namespace

namespace {
adj_status_t ensure_scratch(adj_comm_t comm) {
  if (!comm->d_scratch && cudaMalloc(&comm->d_scratch, 128) != cudaSuccess) return ADJ_ERR_CUDA;
  return ADJ_OK;
}

// every rank's status -> the worst one, on every rank (a 4-byte NCCL max all-reduce and a stream
// synchronisation), so that no rank enters a collective its peers skipped after a local failure
adj_status_t agree_status(adj_comm_t comm, adj_status_t st, cudaStream_t s) {
  if (comm->nranks == 1) return st;
  if (ensure_scratch(comm) != ADJ_OK) return ADJ_ERR_CUDA;   // (a peer then fails its all-reduce: NCCL error)
  int32_t v = (int32_t)st;
  if (cudaMemcpyAsync(comm->d_scratch, &v, 4, cudaMemcpyHostToDevice, s) != cudaSuccess) return ADJ_ERR_CUDA;
  if (g_nccl.AllReduce(comm->d_scratch, comm->d_scratch, 1, ncclInt32, ncclMax, comm->comm, s) != ncclSuccess)
    return ADJ_ERR_NCCL;
  if (cudaMemcpyAsync(&v, comm->d_scratch, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess) return ADJ_ERR_CUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return ADJ_ERR_CUDA;
  return (adj_status_t)v;
}

// a barrier over the communicator (4-byte all-reduce, then the stream is synchronised)
adj_status_t host_barrier(adj_comm_t comm, cudaStream_t s) {
  if (ensure_scratch(comm) != ADJ_OK) return ADJ_ERR_CUDA;
  if (g_nccl.AllReduce(comm->d_scratch, comm->d_scratch, 1, ncclInt32, ncclSum, comm->comm, s) != ncclSuccess)
    return ADJ_ERR_NCCL;
  return cudaStreamSynchronize(s) == cudaSuccess ? ADJ_OK : ADJ_ERR_CUDA;
}

// releases the exchange window in the order CUDA IPC requires: importers close their mappings,
// a barrier, then the root frees the exported allocation
adj_status_t release_window(adj_comm_t comm, cudaStream_t s) {
  if (!comm->win) return ADJ_OK;
  if (!comm->win_owned) cudaIpcCloseMemHandle(comm->win);
  adj_status_t st = comm->nranks > 1 ? host_barrier(comm, s) : ADJ_OK;
  if (comm->win_owned) cudaFree(comm->win);
  comm->win = nullptr;
  comm->win_bytes = 0;
  comm->win_root = -1;
  return st;
}

}  // namespace

int adj_phi_width(adj_phi_t phi);                                    // api.cpp
cudaError_t adj_pool_alloc(void **ptr, size_t bytes, cudaStream_t s);   // api.cpp: retained workspace pool

namespace {
// rank r's column slice of A starts k0 elements into each row: k0 x (uint16 | uint32 words) x
// phi's width bytes (adj_elem_bytes)
const uint32_t *kslice_ptr(const uint32_t *A, adj_phi_t phi, uint32_t flags, int64_t k0) {
  int64_t ea = 0;
  if (!A || adj_elem_bytes(phi, flags, &ea) != ADJ_OK) return A;
  return reinterpret_cast<const uint32_t *>(reinterpret_cast<const uint8_t *>(A) + k0 * ea);
}

// the packed regions (RectDev, buffer offsets) of `rank` for this problem
adj_status_t rank_rects(int64_t m, int64_t k, uint32_t p, int depth, int rank, int G, std::vector<adj::RectDev> &out,
                        int64_t *elems, int *max_rows) {
  int64_t n = 0, e = 0;
  adj_status_t st = adj_shard_layout(m, k, p, depth, rank, G, nullptr, 0, &n, &e);
  if (st != ADJ_OK) return st;
  std::vector<int64_t> raw((size_t)(5 * n));
  if ((st = adj_shard_layout(m, k, p, depth, rank, G, raw.data(), n, &n, &e)) != ADJ_OK) return st;
  out.resize((size_t)n);
  int64_t off = 0;
  *max_rows = 0;
  for (int64_t i = 0; i < n; ++i) {
    adj::RectDev &R = out[(size_t)i];
    R.r0 = raw[5 * i]; R.c0 = raw[5 * i + 1]; R.rows = raw[5 * i + 2]; R.cols = raw[5 * i + 3];
    R.lower = (int32_t)raw[5 * i + 4]; R.pad_ = 0;
    R.off = off;
    off += R.rows * R.cols;
    *max_rows = std::max<int>(*max_rows, (int)R.rows);
  }
  *elems = off;
  return ADJ_OK;
}

// output-tile sharding: every rank computes its regions of Low(C) with the full A, the root
// receives the other ranks' regions packed (only result tiles cross NVLink) and unpacks them
adj_status_t dist_tiles(int64_t m, int64_t k, uint32_t p, adj_phi_t phi, const uint32_t *A, int64_t lda, uint32_t *C,
                        int64_t ldc, int root, adj_comm_t comm, const adj_opts_t *opts, adj_stream_t stream) {
  const int G = comm->nranks, r = comm->rank;
  adj_status_t st = adjprod_modp_shard(m, k, p, phi, A, lda, C, ldc, r, G, opts, stream);
  if (G == 1) return st;
  if (!load_nccl()) return ADJ_ERR_NCCL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if ((st = agree_status(comm, st, s)) != ADJ_OK) return st;
  const int depth = opts ? opts->depth : -1;
  std::vector<std::vector<adj::RectDev>> rects((size_t)G);
  std::vector<int64_t> elems((size_t)G, 0);
  std::vector<int> max_rows((size_t)G, 0);
  for (int q = 0; q < G; ++q) {
    if (r != root && q != r) continue;
    if ((st = rank_rects(m, k, p, depth, q, G, rects[(size_t)q], &elems[(size_t)q], &max_rows[(size_t)q])) != ADJ_OK)
      return st;
  }
  // device copies of the region lists and the packed buffers
  std::vector<void *> allocs;
  auto dalloc = [&](size_t bytes) -> void * {
    void *ptr = nullptr;
    if (bytes && adj_pool_alloc(&ptr, bytes, s) == cudaSuccess) allocs.push_back(ptr);
    return ptr;
  };
  std::vector<adj::RectDev *> drects((size_t)G, nullptr);
  std::vector<void *> bufs((size_t)G, nullptr);
  const int esize = p < 65536 ? 2 : 4;   // residues travel as uint16 when they fit
  for (int q = 0; q < G; ++q) {
    if (rects[(size_t)q].empty() || q == root) continue;
    drects[(size_t)q] = static_cast<adj::RectDev *>(dalloc(rects[(size_t)q].size() * sizeof(adj::RectDev)));
    bufs[(size_t)q] = dalloc((size_t)elems[(size_t)q] * esize);
    if (!drects[(size_t)q] || !bufs[(size_t)q]) st = ADJ_ERR_CUDA;
    else if (cudaMemcpyAsync(drects[(size_t)q], rects[(size_t)q].data(), rects[(size_t)q].size() * sizeof(adj::RectDev),
                             cudaMemcpyHostToDevice, s) != cudaSuccess) st = ADJ_ERR_CUDA;
  }
  if (st == ADJ_OK && r != root && bufs[(size_t)r] &&
      adj::launch_rect_copy(drects[(size_t)r], (int)rects[(size_t)r].size(), max_rows[(size_t)r], C, ldc, bufs[(size_t)r],
                            esize, 1, s) != cudaSuccess)
    st = ADJ_ERR_CUDA;
  // a local failure (allocation, launch) on one rank must not leave its peers blocked in the
  // send / recv group: agree on the status first
  st = agree_status(comm, st, s);
  if (st == ADJ_OK) {
    g_nccl.GroupStart();
    for (int q = 0; q < G; ++q) {
      if (q == root || !bufs[(size_t)q]) continue;
      if (r == root) {
        if (g_nccl.Recv(bufs[(size_t)q], (size_t)elems[(size_t)q] * esize, ncclUint8, q, comm->comm, s) != ncclSuccess)
          st = ADJ_ERR_NCCL;
      } else if (q == r) {
        if (g_nccl.Send(bufs[(size_t)q], (size_t)elems[(size_t)q] * esize, ncclUint8, root, comm->comm, s) != ncclSuccess)
          st = ADJ_ERR_NCCL;
      }
    }
    if (g_nccl.GroupEnd() != ncclSuccess) st = ADJ_ERR_NCCL;
  }
  if (st == ADJ_OK && r == root)
    for (int q = 0; q < G; ++q)
      if (q != root && bufs[(size_t)q] &&
          adj::launch_rect_copy(drects[(size_t)q], (int)rects[(size_t)q].size(), max_rows[(size_t)q], C, ldc,
                                bufs[(size_t)q], esize, 0, s) != cudaSuccess)
        st = ADJ_ERR_CUDA;
  for (void *ptr : allocs) cudaFreeAsync(ptr, s);
  return st;
}

// the root's exchange window (G slots of m x m narrow residues), mapped on every rank
// (collective: every rank calls it with the same root and size, so all take the same branch)
adj_status_t setup_window(adj_comm_t comm, int root, size_t bytes, cudaStream_t s) {
  if (comm->win && comm->win_root == root && comm->win_bytes >= bytes) return ADJ_OK;
  adj_status_t st = release_window(comm, s);
  if (st != ADJ_OK) return st;
  if (ensure_scratch(comm) != ADJ_OK) return ADJ_ERR_CUDA;
  cudaIpcMemHandle_t h;
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  st = ADJ_OK;
  if (comm->rank == root) {
    if (cudaMalloc(&comm->win, bytes) != cudaSuccess) { comm->win = nullptr; st = ADJ_ERR_CUDA; }
    else {
      comm->win_owned = true;
      if (cudaIpcGetMemHandle(&h, comm->win) != cudaSuccess) st = ADJ_ERR_CUDA;
    }
  }
  // the root's allocation failing must not leave the other ranks waiting in the broadcast
  if ((st = agree_status(comm, st, s)) != ADJ_OK) {
    if (comm->win && comm->win_owned) cudaFree(comm->win);
    comm->win = nullptr;
    return st;
  }
  if (comm->rank == root &&
      cudaMemcpyAsync(comm->d_scratch, &h, 64, cudaMemcpyHostToDevice, s) != cudaSuccess) return ADJ_ERR_CUDA;
  if (g_nccl.Broadcast(comm->d_scratch, comm->d_scratch, 64, ncclUint8, root, comm->comm, s) != ncclSuccess)
    return ADJ_ERR_NCCL;
  if (cudaStreamSynchronize(s) != cudaSuccess) return ADJ_ERR_CUDA;
  if (comm->rank != root) {
    if (cudaMemcpy(&h, comm->d_scratch, 64, cudaMemcpyDeviceToHost) != cudaSuccess) return ADJ_ERR_CUDA;
    if (cudaIpcOpenMemHandle(&comm->win, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return ADJ_ERR_CUDA;
    comm->win_owned = false;
  }
  comm->win_root = root;
  comm->win_bytes = bytes;
  return ADJ_OK;
}

// split-K with the exchange fused into the compute (ADJ_DIST_P2P): every rank's final kernel
// (leaf epilogue at depth 0, K4 otherwise) stores its Low(A_r A_r^T) residues, 2 bytes each for
// p < 2^16, straight into slot r of the root's window over NVLink (adjprod_modp_partial with a
// peer pointer); two NCCL barriers order the window's reuse and the root's exact sum
// (adj_sum_partials).  NVLink carries m^2/2 narrow residues per rank instead of the m^2 uint32
// words of the reduce.
adj_status_t dist_p2p(int64_t m, int64_t k, uint32_t p, adj_phi_t phi, const uint32_t *A, int64_t lda, uint32_t *C,
                      int64_t ldc, int root, adj_comm_t comm, const adj_opts_t *opts, adj_stream_t stream) {
  if (!load_nccl()) return ADJ_ERR_NCCL;
  const int G = comm->nranks, r = comm->rank;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const size_t esize = p < 65536 ? 2 : 4;
  const size_t slot = (size_t)m * (size_t)m;
  adj_status_t st = setup_window(comm, root, slot * esize * (size_t)G, s);
  if (st != ADJ_OK) return st;
  // barrier 1: the root has finished reading the window of the previous call
  if (g_nccl.AllReduce(comm->d_scratch, comm->d_scratch, 1, ncclInt32, ncclSum, comm->comm, s) != ncclSuccess)
    return ADJ_ERR_NCCL;
  int64_t k0 = 0, k1 = 0;
  adj_dist_kslice(k, G, r, &k0, &k1);
  void *mine = static_cast<uint8_t *>(comm->win) + (size_t)r * slot * esize;
  adj_opts_t o = opts ? *opts : adj_opts_t{-1, 0, nullptr, 0};
  o.flags &= ADJ_IN_U16;
  const uint32_t *Ar = kslice_ptr(A, phi, o.flags, k0);
  st = adjprod_modp_partial(m, k1 - k0, p, phi, Ar, lda, mine, m, &o, stream);
  if (st != ADJ_OK) return st;
  // barrier 2: every rank's partial kernels (and their peer stores) have completed
  if (g_nccl.AllReduce(comm->d_scratch, comm->d_scratch, 1, ncclInt32, ncclSum, comm->comm, s) != ncclSuccess)
    return ADJ_ERR_NCCL;
  if (r == root) st = adj_sum_partials(m, p, comm->win, m, (int64_t)slot, G, C, ldc, stream);
  return st;
}

// output-tile sharding with the gather fused into the compute (ADJ_DIST_TILES | ADJ_DIST_P2P):
// the root exports its C (adj_ipc_export), the record and ldc are broadcast, every other rank
// maps the root's C and runs its share (adjprod_modp_shard) with the mapped pointer as its output:
// the final kernel of the share -- the leaf epilogue at depth 0 (tile by tile, under the MMAs of
// the following tiles), K4 at depth 1 -- stores the owned regions of Low(C) over NVLink straight
// into their place.  No pack, no NCCL data movement, no unpack on the root.
adj_status_t dist_tiles_p2p(int64_t m, int64_t k, uint32_t p, adj_phi_t phi, const uint32_t *A, int64_t lda,
                            uint32_t *C, int64_t ldc, int root, adj_comm_t comm, const adj_opts_t *opts,
                            adj_stream_t stream) {
  const int G = comm->nranks, r = comm->rank;
  if (G == 1) return adjprod_modp_shard(m, k, p, phi, A, lda, C, ldc, 0, 1, opts, stream);
  if (!load_nccl()) return ADJ_ERR_NCCL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  constexpr size_t kRec = ADJ_IPC_RECORD_BYTES + 8;   // handle, offset, ldc
  uint8_t rec[kRec] = {};
  adj_status_t st = ensure_scratch(comm);
  if (st == ADJ_OK && r == root) {
    st = adj_ipc_export(C, rec);
    std::memcpy(rec + ADJ_IPC_RECORD_BYTES, &ldc, 8);
  }
  if ((st = agree_status(comm, st, s)) != ADJ_OK) return st;
  if (r == root && cudaMemcpyAsync(comm->d_scratch, rec, kRec, cudaMemcpyHostToDevice, s) != cudaSuccess)
    st = ADJ_ERR_CUDA;   // (the peers then see garbage and fail to open: agreed below)
  if (g_nccl.Broadcast(comm->d_scratch, comm->d_scratch, kRec, ncclUint8, root, comm->comm, s) != ncclSuccess)
    return ADJ_ERR_NCCL;
  void *dst = nullptr;
  int64_t ldd = ldc;
  if (r != root && st == ADJ_OK) {
    if (cudaMemcpyAsync(rec, comm->d_scratch, kRec, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      st = ADJ_ERR_CUDA;
    else {
      std::memcpy(&ldd, rec + ADJ_IPC_RECORD_BYTES, 8);
      st = adj_ipc_open(rec, &dst);
    }
  }
  // every rank has its output pointer before any store
  if ((st = agree_status(comm, st, s)) == ADJ_OK)
    st = adjprod_modp_shard(m, k, p, phi, A, lda, r == root ? C : static_cast<uint32_t *>(dst), r == root ? ldc : ldd,
                            r, G, opts, stream);
  // barrier 1 (host-synchronised): every rank's share, and so every peer store, has completed
  st = agree_status(comm, st, s);
  if (dst) adj_ipc_close(dst);
  // barrier 2: the importers have unmapped C -- the root's caller may free it after the return
  const adj_status_t b = host_barrier(comm, s);
  return st != ADJ_OK ? st : b;
}
}  // namespace

extern "C" {

adj_status_t adj_comm_get_unique_id(uint8_t id[128]) {
  if (!id) return ADJ_ERR_INVALID_VALUE;
  if (!load_nccl()) return ADJ_ERR_NCCL;
  ncclUniqueId u;
  if (g_nccl.GetUniqueId(&u) != ncclSuccess) return ADJ_ERR_NCCL;
  static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id, &u, 128);
  return ADJ_OK;
}

adj_status_t adj_comm_init(int nranks, const uint8_t id[128], int rank, adj_comm_t *comm) {
  if (!id || !comm || nranks < 1 || rank < 0 || rank >= nranks) return ADJ_ERR_INVALID_VALUE;
  if (!load_nccl()) return ADJ_ERR_NCCL;
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  ncclComm_t c;
  ncclResult_t r = g_nccl.CommInitRank(&c, nranks, u, rank);
  if (r != ncclSuccess) return ADJ_ERR_NCCL;
  adj_comm_s *cm = new adj_comm_s;
  cm->comm = c;
  cm->nranks = nranks;
  cm->rank = rank;
  *comm = cm;
  return ADJ_OK;
}

adj_status_t adj_comm_destroy(adj_comm_t comm) {
  if (!comm) return ADJ_ERR_INVALID_VALUE;
  if (comm->win) {   // collective when a P2P window exists: importers close, barrier, the root frees
    cudaStream_t s = nullptr;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    release_window(comm, s);
    if (s) cudaStreamDestroy(s);
  }
  if (comm->d_scratch) cudaFree(comm->d_scratch);
  if (g_nccl.loaded) g_nccl.CommDestroy(comm->comm);
  delete comm;
  return ADJ_OK;
}

// ---- CUDA IPC of a pointer inside an allocation: the handle names the allocation's base, the
// record carries the offset (cuMemGetAddressRange through the runtime's driver entry point)
namespace {
std::mutex g_ipc_mu;
std::map<void *, void *> g_ipc_open;   // pointer handed out -> mapped base
}  // namespace

adj_status_t adj_ipc_export(const void *ptr, uint8_t rec[ADJ_IPC_RECORD_BYTES]) {
  if (!ptr || !rec) return ADJ_ERR_INVALID_VALUE;
  using range_fn = CUresult (*)(CUdeviceptr *, size_t *, CUdeviceptr);
  static range_fn get_range = nullptr;
  if (!get_range) {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn ||
        q != cudaDriverEntryPointSuccess)
      return ADJ_ERR_CUDA;
    get_range = reinterpret_cast<range_fn>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (get_range(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS) return ADJ_ERR_CUDA;
  cudaIpcMemHandle_t h;
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  if (cudaIpcGetMemHandle(&h, reinterpret_cast<void *>(base)) != cudaSuccess) {
    cudaGetLastError();
    return ADJ_ERR_CUDA;
  }
  const int64_t off = (int64_t)(reinterpret_cast<CUdeviceptr>(ptr) - base);
  std::memcpy(rec, &h, 64);
  std::memcpy(rec + 64, &off, 8);
  return ADJ_OK;
}

adj_status_t adj_ipc_open(const uint8_t rec[ADJ_IPC_RECORD_BYTES], void **ptr) {
  if (!rec || !ptr) return ADJ_ERR_INVALID_VALUE;
  cudaIpcMemHandle_t h;
  int64_t off = 0;
  std::memcpy(&h, rec, 64);
  std::memcpy(&off, rec + 64, 8);
  if (off < 0) return ADJ_ERR_INVALID_VALUE;
  void *base = nullptr;
  if (cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
    cudaGetLastError();
    return ADJ_ERR_CUDA;
  }
  *ptr = static_cast<uint8_t *>(base) + off;
  std::lock_guard<std::mutex> g(g_ipc_mu);
  g_ipc_open[*ptr] = base;
  return ADJ_OK;
}

adj_status_t adj_ipc_close(void *ptr) {
  void *base = nullptr;
  {
    std::lock_guard<std::mutex> g(g_ipc_mu);
    auto it = g_ipc_open.find(ptr);
    if (it == g_ipc_open.end()) return ADJ_ERR_INVALID_VALUE;
    base = it->second;
    g_ipc_open.erase(it);
  }
  return cudaIpcCloseMemHandle(base) == cudaSuccess ? ADJ_OK : ADJ_ERR_CUDA;
}

adj_status_t adj_dist_kslice(int64_t k, int nranks, int rank, int64_t *k0, int64_t *k1) {
  if (!k0 || !k1 || k < 0 || nranks < 1 || rank < 0 || rank >= nranks) return ADJ_ERR_INVALID_VALUE;
  const int64_t per = ((k + nranks - 1) / nranks + 7) / 8 * 8;
  *k0 = std::min<int64_t>(k, (int64_t)rank * per);
  *k1 = std::min<int64_t>(k, *k0 + per);
  return ADJ_OK;
}

adj_status_t adj_elem_bytes(adj_phi_t phi, uint32_t flags, int64_t *bytes) {
  if (!bytes || (phi != ADJ_PHI_T && phi != ADJ_PHI_H && phi != ADJ_PHI_Q)) return ADJ_ERR_INVALID_VALUE;
  *bytes = (int64_t)((flags & ADJ_IN_U16) ? 2 : 4) * adj_phi_width(phi);
  return ADJ_OK;
}

adj_status_t adjprod_modp_dist_partial(int64_t m, int64_t k, uint32_t p, adj_phi_t phi, const uint32_t *A, int64_t lda,
                                       uint32_t *R, int64_t ldr, int rank, int nranks, const adj_opts_t *opts,
                                       adj_stream_t stream) {
  if (m < 0 || k < 0 || nranks < 1 || rank < 0 || rank >= nranks) return ADJ_ERR_INVALID_VALUE;
  int64_t k0 = 0, k1 = 0;
  adj_dist_kslice(k, nranks, rank, &k0, &k1);
  return adjprod_modp_ex(m, k1 - k0, p, phi, kslice_ptr(A, phi, opts ? opts->flags : 0, k0), lda, R, ldr, opts, stream);
}

adj_status_t adjprod_modp_dist(int64_t m, int64_t k, uint32_t p, adj_phi_t phi, const uint32_t *A, int64_t lda,
                               uint32_t *C, int64_t ldc, int root, adj_comm_t comm, const adj_opts_t *opts,
                               adj_stream_t stream) {
  if (!comm || root < 0 || root >= comm->nranks) return ADJ_ERR_INVALID_VALUE;
  if (m < 0 || k < 0) return ADJ_ERR_INVALID_VALUE;
  if (opts && (opts->flags & ADJ_OUT_U16)) return ADJ_ERR_INVALID_VALUE;   // Low(C) on the root is uint32
  if (m == 0) return ADJ_OK;
  const int G = comm->nranks, r = comm->rank;
  if (opts && (opts->flags & ADJ_DIST_TILES) && (opts->flags & ADJ_DIST_P2P))
    return dist_tiles_p2p(m, k, p, phi, A, lda, C, ldc, root, comm, opts, stream);
  if (opts && (opts->flags & ADJ_DIST_TILES)) return dist_tiles(m, k, p, phi, A, lda, C, ldc, root, comm, opts, stream);
  if (opts && (opts->flags & ADJ_DIST_P2P) && phi == ADJ_PHI_T && G > 1)
    return dist_p2p(m, k, p, phi, A, lda, C, ldc, root, comm, opts, stream);
  if (G == 1) return adjprod_modp_dist_partial(m, k, p, phi, A, lda, C, ldc, 0, 1, opts, stream);
  if (!load_nccl()) return ADJ_ERR_NCCL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int w = adj_phi_width(phi);
  const uint32_t flags = opts ? opts->flags : 0;
  // the rank's partial Low(A_r phi(A_r)) in a dense m x m buffer (the caller's Up(C) stays
  // untouched): uint16 words when the residues fit (ADJ_OUT_U16), then its lower triangle packed
  // as uint32 words -- the reduce moves m (m + 1) / 2 words per element instead of m^2
  const bool narrow = p < 65536 && !(flags & (ADJ_HERK_ALG1 | ADJ_FILL_UPPER));
  adj_opts_t o = opts ? *opts : adj_opts_t{-1, 0, nullptr, 0};
  o.flags &= ~(ADJ_FILL_UPPER | ADJ_DIST_TILES | ADJ_DIST_P2P);
  if (narrow) o.flags |= ADJ_OUT_U16;
  const size_t dense = (size_t)m * (size_t)m * (size_t)w * (narrow ? 2 : 4);
  const size_t packed = (size_t)(m * (m + 1) / 2) * (size_t)w;
  void *W = nullptr, *Pk = nullptr;
  adj_status_t st = ADJ_OK;
  if (adj_pool_alloc(&W, dense, s) != cudaSuccess || adj_pool_alloc(&Pk, packed * 4, s) != cudaSuccess) st = ADJ_ERR_CUDA;
  if (st == ADJ_OK) st = adjprod_modp_dist_partial(m, k, p, phi, A, lda, static_cast<uint32_t *>(W), m, r, G, &o, stream);
  if (st == ADJ_OK &&
      adj::launch_pack_lower(m, w, W, m, narrow ? 2 : 4, static_cast<uint32_t *>(Pk), s) != cudaSuccess)
    st = ADJ_ERR_CUDA;
  // a local failure must not leave the peers blocked in the reduce
  st = agree_status(comm, st, s);
  if (st == ADJ_OK) {
    // exact: each word is a sum of G residues < G p < 2^32
    if (g_nccl.Reduce(Pk, Pk, packed, ncclUint32, ncclSum, root, comm->comm, s) != ncclSuccess) st = ADJ_ERR_NCCL;
  }
  if (st == ADJ_OK && r == root) {
    if (adj::launch_unpack_mod_lower(m, w, static_cast<uint32_t *>(Pk), C, ldc, adj::make_modp(p), s) != cudaSuccess)
      st = ADJ_ERR_CUDA;
    else if ((flags & ADJ_FILL_UPPER) && adj::launch_fill_upper(m, w, C, ldc, adj::make_modp(p), s) != cudaSuccess)
      st = ADJ_ERR_CUDA;
  }
  if (W) cudaFreeAsync(W, s);
  if (Pk) cudaFreeAsync(Pk, s);
  return st;
}

adj_status_t adj_shard_pack(int64_t m, int64_t k, uint32_t p, int depth, int rank, int nranks, uint32_t *C,
                            int64_t ldc, void *buf, int unpack, adj_stream_t stream) {
  if (m < 0 || ldc < m || !C || !buf) return ADJ_ERR_INVALID_VALUE;
  if (m == 0) return ADJ_OK;
  std::vector<adj::RectDev> rects;
  int64_t elems = 0;
  int max_rows = 0;
  adj_status_t st = rank_rects(m, k, p, depth, rank, nranks, rects, &elems, &max_rows);
  if (st != ADJ_OK || rects.empty()) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  void *d = nullptr;
  if (adj_pool_alloc(&d, rects.size() * sizeof(adj::RectDev), s) != cudaSuccess) return ADJ_ERR_CUDA;
  if (cudaMemcpyAsync(d, rects.data(), rects.size() * sizeof(adj::RectDev), cudaMemcpyHostToDevice, s) != cudaSuccess)
    st = ADJ_ERR_CUDA;
  if (st == ADJ_OK && adj::launch_rect_copy(static_cast<adj::RectDev *>(d), (int)rects.size(), max_rows, C, ldc, buf,
                                            p < 65536 ? 2 : 4, unpack ? 0 : 1, s) != cudaSuccess)
    st = ADJ_ERR_CUDA;
  cudaFreeAsync(d, s);
  return st;
}

}  // extern "C"
