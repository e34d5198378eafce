// Multi-GPU split-K over NCCL: every rank computes Low(A_r phi(A_r)) on its
// column slice with the single-GPU path, the residue partials are summed exactly by an NCCL
// uint32 reduce (sum < G p < 2^32) and reduced mod p on the root.  NCCL is resolved with
// dlopen at first use (the torch-bundled libnccl.so.2 when running inside torch).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/adjprod.h"
#include "kernels.hpp"

struct adj_comm_s {
  ncclComm_t comm;
  int nranks, rank;
};

namespace {

struct NcclApi {
  bool loaded = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
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
  SYM("ncclGetErrorString", GetErrorString)
#undef SYM
  g_nccl.loaded = true;
  return true;
}

}  // namespace

int adj_phi_width(adj_phi_t phi);   // api.cpp

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
  *comm = new adj_comm_s{c, nranks, rank};
  return ADJ_OK;
}

adj_status_t adj_comm_destroy(adj_comm_t comm) {
  if (!comm) return ADJ_ERR_INVALID_VALUE;
  if (g_nccl.loaded) g_nccl.CommDestroy(comm->comm);
  delete comm;
  return ADJ_OK;
}

adj_status_t adj_dist_kslice(int64_t k, int nranks, int rank, int64_t *k0, int64_t *k1) {
  if (!k0 || !k1 || k < 0 || nranks < 1 || rank < 0 || rank >= nranks) return ADJ_ERR_INVALID_VALUE;
  const int64_t per = ((k + nranks - 1) / nranks + 7) / 8 * 8;
  *k0 = std::min<int64_t>(k, (int64_t)rank * per);
  *k1 = std::min<int64_t>(k, *k0 + per);
  return ADJ_OK;
}

adj_status_t adjprod_modp_dist(int64_t m, int64_t k, uint32_t p, adj_phi_t phi, const uint32_t *A, int64_t lda,
                               uint32_t *C, int64_t ldc, int root, adj_comm_t comm, const adj_opts_t *opts,
                               adj_stream_t stream) {
  if (!comm || root < 0 || root >= comm->nranks) return ADJ_ERR_INVALID_VALUE;
  if (m < 0 || k < 0) return ADJ_ERR_INVALID_VALUE;
  if (m == 0) return ADJ_OK;
  const int G = comm->nranks, r = comm->rank;
  const int w = adj_phi_width(phi);
  int64_t k0 = 0, k1 = 0;
  adj_dist_kslice(k, G, r, &k0, &k1);
  const uint32_t *Ar = A ? A + k0 * w : nullptr;
  if (G == 1) return adjprod_modp_ex(m, k1 - k0, p, phi, Ar, lda, C, ldc, opts, stream);
  if (!load_nccl()) return ADJ_ERR_NCCL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // partial Low(A_r phi(A_r)) in a dense m x m buffer (the caller's Up(C) stays untouched)
  uint32_t *W = nullptr;
  const size_t count = (size_t)m * m * w;
  if (cudaMallocAsync(reinterpret_cast<void **>(&W), count * 4, s) != cudaSuccess) return ADJ_ERR_CUDA;
  adj_status_t st = adjprod_modp_ex(m, k1 - k0, p, phi, Ar, lda, W, m, opts, stream);
  if (st == ADJ_OK) {
    // exact: each entry is a sum of G residues < G p < 2^32
    if (g_nccl.Reduce(W, W, count, ncclUint32, ncclSum, root, comm->comm, s) != ncclSuccess) st = ADJ_ERR_NCCL;
  }
  if (st == ADJ_OK && r == root) {
    if (adj::launch_mod_lower(m, w, W, m, C, ldc, adj::make_modp(p), s) != cudaSuccess) st = ADJ_ERR_CUDA;
  }
  cudaFreeAsync(W, s);
  return st;
}

}  // extern "C"
