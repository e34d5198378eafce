/*
 * adjprod.h -- C ABI of the B200 (sm_100a) implementation of the hot path of
 * arXiv 2101.01025, "multiplication of a matrix by its adjoint":
 *
 *     Low(C) = Low(A . phi(A)) mod p
 *
 * computed with the paper's 5-product recursion (Alg. alg:MIAHMM) on
 * int8 tcgen05 tensor-core leaves, and, for phi = conjugate transpose over GF(p^2), with
 * the paper's 2M reduction (Alg. alg:2M).
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 * - Matrices are row-major.  A "leading dimension" (lda, ldb, ldc) counts ELEMENTS
 *   between consecutive rows (GF(p^2) elements for phi = ADJ_PHI_H).
 * - Device pointers unless a function says "host".  The caller owns A, B, C and any
 *   workspace; the library never frees caller memory.  Plans (tile lists, constants) are
 *   cached per device inside the library.
 * - GF(p) elements are uint32 residues.  Inputs are interpreted mod p (non-canonical input
 *   is reduced, not undefined).  Outputs are canonical, in [0, p).
 * - GF(p^2) = GF(p)[i]/(i^2 + 1) (requires p = 3 mod 4 so that x^2+1 is irreducible);
 *   an element x + i y is stored as an interleaved (x, y) uint32 pair.  Conjugation is the
 *   Frobenius map x + iy -> x - iy.
 * - Quaternions H_GF(p) (§6.2, 1532-1558): x1 + x2 i + x3 j + x4 k with
 *   i^2 = j^2 = k^2 = ijk = -1, stored as 4 interleaved uint32 (x1, x2, x3, x4); conjugation
 *   negates x2, x3, x4.  Leading dimensions count quaternions for phi = ADJ_PHI_Q.
 * - Low/Up: Low includes the diagonal.  Only Low(C) is written; the
 *   strict upper triangle of C is left untouched unless ADJ_FILL_UPPER is set, in which
 *   case Up(C) = phi(Low(C)) (Lemma lem:uplow).
 * - Supported moduli: odd primes 3 <= p <= 262139 (the largest prime below 2^18; this covers
 *   the paper's own moduli 131071 and 131041).  Limb schemes: p <= 255
 *   one signed int8 limb; 257 <= p <= 16763 two balanced base-2^7 limbs with Karatsuba;
 *   16787 <= p <= 65521 a signed-int8 high limb and an unsigned-int8 low limb; p > 2^16 three
 *   balanced base-2^6 digits with 3-way Karatsuba.
 * - Shapes need no alignment: odd or ragged dimensions are zero-padded internally, which
 *   leaves A phi(A) unchanged.
 * - Every call is asynchronous on `stream`, like cuBLAS.  Argument validation is
 *   synchronous and happens before any launch; an invalid call launches nothing and returns
 *   an error code (no abort, no exception crosses the ABI).  Asynchronous CUDA faults surface
 *   at a later synchronisation, as in cuBLAS.  adj_last_error() gives a thread-local detail
 *   string for the last failing call on the calling thread.
 * - Thread safety: entry points may be called concurrently from several host threads on
 *   different streams with different workspaces; the internal plan cache is locked, bounded
 *   (64 plans per process, least recently used first) and never evicts a plan a call is using.
 */
#ifndef ADJPROD_H
#define ADJPROD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *adj_stream_t; /* == cudaStream_t; NULL = legacy default stream */
typedef struct adj_comm_s *adj_comm_t;    /* opaque NCCL-backed communicator */

typedef enum {
  ADJ_PHI_T = 0, /* phi = transpose over GF(p)               (Examples ex:antih) */
  ADJ_PHI_H = 1, /* phi = conjugate transpose over GF(p^2)   (Examples ex:antih) */
  ADJ_PHI_Q = 2  /* phi = conjugate transpose over the quaternions H_GF(p), computed with
                    Alg. alg:2M3M (6M): five general
                    products and one product of a matrix by its transpose, Q6, which runs
                    through Alg. alg:MIAHMM at the requested depth */
} adj_phi_t;

typedef enum {
  ADJ_OK = 0,
  ADJ_ERR_INVALID_VALUE = 1,       /* negative/inconsistent sizes, null pointers, A/C overlap */
  ADJ_ERR_UNSUPPORTED_MODULUS = 2, /* p not an odd prime in [3, 262139]; phi=H with p != 3 mod 4 */
  ADJ_ERR_WORKSPACE = 3,           /* caller workspace too small / allocation failed */
  ADJ_ERR_CUDA = 4,                /* a CUDA runtime call failed */
  ADJ_ERR_NCCL = 5,                /* NCCL missing or a collective failed */
  ADJ_ERR_ARCH = 6                 /* current device is not sm_100 (B200) */
} adj_status_t;

/* option flags (adj_opts_t.flags)
 *   ADJ_FILL_UPPER : also write the strict upper triangle, Up(C) = phi(Low(C)) (Lemma lem:uplow).
 *   ADJ_HERK_ALG1  : phi = ADJ_PHI_H only -- run one level of Alg. alg:MIAHMM directly over
 *                    GF(p^2) with the scalar skew-unitary Y = (a + ib) I, a^2 + b^2 = -1
 *                    (§4.4, 750-758) instead of the 2M reduction
 *                    to GF(p) (Alg. alg:2M).  Its Hermitian leaves P1, P2, P5 use 2M, its
 *                    general leaves P3, P4 use 3M.  Requires depth 1 (or -1); the result is the
 *                    same Low(C).  Ignored for phi = ADJ_PHI_T.
 *   ADJ_DIST_TILES : adjprod_modp_dist only -- output-tile sharding instead of split-K.
 *   ADJ_DIST_P2P   : adjprod_modp_dist only, phi = ADJ_PHI_T -- split-K with the exchange fused
 *                    into the final kernel: each rank stores its partial (narrow residues)
 *                    straight into the root's window over NVLink (CUDA IPC peer memory), the root
 *                    sums exactly (adj_sum_partials); no NCCL data movement.
 *                    With ADJ_DIST_TILES as well: output-tile sharding with the gather fused into
 *                    the final kernel -- the root's C is mapped on every rank (adj_ipc_export /
 *                    adj_ipc_open), and each rank's last kernel (leaf epilogue at depth 0, K4 at
 *                    depth 1) stores its owned regions of Low(C) straight into it over NVLink;
 *                    no pack, no NCCL data movement, no unpack.
 *   ADJ_IN_U16     : p < 2^16 -- A holds uint16 values (phi = H: interleaved uint16 (re, im)
 *                    pairs; phi = Q: 4 uint16 components), read mod p; lda counts elements as
 *                    before: half the bytes to read and to ship over PCIe.  phi = T also through
 *                    adjprod_modp_shard, adjprod_modp_partial and adjprod_modp_dist.
 *   ADJ_OUT_U16    : p < 2^16 -- Low(C) written as uint16 residues (pairs / quadruples for
 *                    phi = H / Q); the plain form only (no alpha / beta, no ADJ_FILL_UPPER, not
 *                    with ADJ_HERK_ALG1).
 *   ADJ_LOW_MEM    : phi = ADJ_PHI_T, depth >= 1, m a multiple of 64, plain form (alpha = 1,
 *                    beta = 0) -- the low-memory temporary schedule (the GPU counterpart of the
 *                    in-place schedules of Table tab:schedule:AAT): the root
 *                    level's products P1, P3, P5 are formed in C's own blocks C11, C21, C22 and
 *                    only P2, P4 and S3 live in the workspace; the root's operand arena is
 *                    reused by its three children (ordinary calls one level shallower), and the
 *                    root recombination runs in place.  Same Low(C); Up(C) untouched.  Requires
 *                    C 16-byte aligned and ldc a multiple of 8 (INVALID_VALUE otherwise).
 *                    Ignored where it does not apply (other phi, depth 0, m % 64 != 0, SYRK
 *                    form); adjprod_modp_workspace_size honours it the same way.  Without the
 *                    flag a call falls back to this schedule by itself where it applies and C is
 *                    so aligned, when the caller's workspace is smaller than the grouped
 *                    schedule's size but not than this one's, or when the library's workspace
 *                    allocation fails. */
enum { ADJ_FILL_UPPER = 1u, ADJ_HERK_ALG1 = 2u, ADJ_DIST_TILES = 4u, ADJ_DIST_P2P = 8u, ADJ_IN_U16 = 16u,
       ADJ_OUT_U16 = 32u, ADJ_LOW_MEM = 64u };

typedef struct {
  int depth;              /* recursion levels of Alg. alg:MIAHMM; -1 = automatic; 0 = classical */
  uint32_t flags;         /* ADJ_* option flags above, or-ed */
  void *workspace;        /* device memory of >= workspace_bytes, or NULL (library allocates
                             stream-ordered from a per-device pool that retains its memory
                             between calls, cudaMallocFromPoolAsync / cudaFreeAsync) */
  size_t workspace_bytes;
} adj_opts_t;

/*
 * adjprod_modp -- Low(C) = Low(A phi(A)).
 *   Problem statement: Alg. alg:MIAHMM "Ensure Low(A phi(A))".
 *   m, k   : A is m x k (m output rows, k contracted columns); C is m x m.  m = 0 is a no-op;
 *            k = 0 writes Low(C) = 0.
 *   p      : odd prime, 3 <= p <= 262139 (phi = ADJ_PHI_H additionally needs p = 3 mod 4).
 *   phi    : ADJ_PHI_T (A, C uint32 residues), ADJ_PHI_H (A, C interleaved (re, im) pairs)
 *            or ADJ_PHI_Q (A, C interleaved quaternions (x1, x2, x3, x4)).
 *   A, lda : device, lda >= k.     C, ldc : device, ldc >= m.  A and C must not overlap.
 *   Uses default options (automatic depth, library-allocated workspace).
 */
adj_status_t adjprod_modp(int64_t m, int64_t k, uint32_t p, adj_phi_t phi,
                          const uint32_t *A, int64_t lda, uint32_t *C, int64_t ldc,
                          adj_stream_t stream);

/* adjprod_modp_ex -- as adjprod_modp with explicit options (depth, flags, workspace). */
adj_status_t adjprod_modp_ex(int64_t m, int64_t k, uint32_t p, adj_phi_t phi,
                             const uint32_t *A, int64_t lda, uint32_t *C, int64_t ldc,
                             const adj_opts_t *opts, adj_stream_t stream);

/*
 * adjprod_modp_syrk -- the SYRK / HERK form  Low(C) <- alpha Low(A phi(A)) + beta Low(C)
 *   (Table tab:schedule:AATpC, "C <- alpha A A^T + beta C").
 *   alpha, beta in GF(p) (reduced mod p; for phi = ADJ_PHI_H they scale the re and im parts
 *   alike, so the result stays Hermitian).  C is read (old values, interpreted mod p) and written
 *   on Low(C) only.  The paper's in-place schedule with one n/2 x n/2 temporary is replaced by the
 *   library workspace; the axpby is fused into the kernel that writes the final Low(C).
 *   alpha = 1, beta = 0 is adjprod_modp_ex.  Arguments otherwise as adjprod_modp_ex.
 */
adj_status_t adjprod_modp_syrk(int64_t m, int64_t k, uint32_t p, adj_phi_t phi, uint32_t alpha,
                               const uint32_t *A, int64_t lda, uint32_t beta, uint32_t *C, int64_t ldc,
                               const adj_opts_t *opts, adj_stream_t stream);

/* Workspace bytes adjprod_modp_ex needs for these arguments (host, no launch). */
adj_status_t adjprod_modp_workspace_size(int64_t m, int64_t k, uint32_t p, adj_phi_t phi,
                                         const adj_opts_t *opts, size_t *bytes);

/* Depth the automatic choice (opts->depth = -1) resolves to for this problem (host). */
adj_status_t adjprod_modp_auto_depth(int64_t m, int64_t k, uint32_t p, adj_phi_t phi,
                                     int *depth);

/* Output-tile width of the grouped leaf launch this call would use (host, no device work):
 * 512 for the wide-N leaf (256 x 512 CTA-pair tiles, Horner recombination in TMEM; launches of
 * more than 16 waves), 256 otherwise.  Same arguments and errors as the workspace query. */
adj_status_t adjprod_modp_leaf_tile(int64_t m, int64_t k, uint32_t p, adj_phi_t phi,
                                    const adj_opts_t *opts, int *tile_n);

/*
 * gemm_modp -- C = A B^T mod p over GF(p), all of C (m x n).  The paper's general product
 *   A phi(B) (P3, P4 of Alg. alg:MIAHMM) exposed on its own.
 *   A: m x k (lda >= k), B: n x k (ldb >= k), C: m x n (ldc >= n); device; C must not overlap
 *   A or B.  Library-allocated workspace.
 */
adj_status_t gemm_modp(int64_t m, int64_t n, int64_t k, uint32_t p,
                       const uint32_t *A, int64_t lda, const uint32_t *B, int64_t ldb,
                       uint32_t *C, int64_t ldc, adj_stream_t stream);

/*
 * adj_skew_unitary -- the skew-unitary Y the path uses (host, exact), Y phi(Y) = -I
 *   (Eq. eq:skewu).
 *   *kind = 0: Y = a I with a = sqrt(-1) mod p (p = 1 mod 4, Prop. lem:lemsqrt),
 *              smallest of the two roots; *b = 0.
 *   *kind = 1: Y = [[a, b], [-b, a]] (x) I with a^2 + b^2 = -1 (p = 3 mod 4,
 *              Prop. lem:pigeonhole; (a, b) from Alg. alg:sosmodp).
 *   For phi = ADJ_PHI_H the 2M reduction runs Alg. alg:MIAHMM over GF(p) for its G product,
 *   so the same GF(p) Y is returned.
 */
adj_status_t adj_skew_unitary(uint32_t p, adj_phi_t phi, int *kind, uint32_t *a, uint32_t *b);

/* adj_sos -- Alg. alg:sosmodp: (a, b) with a^2 + b^2 = k mod p (host). */
adj_status_t adj_sos(uint32_t p, uint32_t k, uint32_t *a, uint32_t *b);

/*
 * adj_mod_lower -- in place, x <- x mod p on Low(X) (m x m, ldx), device.  Used after an
 *   exact integer sum of residue partials (multi-GPU split-K reduce).
 */
adj_status_t adj_mod_lower(int64_t m, uint32_t p, adj_phi_t phi, uint32_t *X, int64_t ldx,
                           adj_stream_t stream);

/* ---------------- multi-GPU (one process per GPU; NCCL over NVLink) ---------------- */

/* rank 0 creates an id (host buffer of 128 bytes); ship it to the other ranks out of band */
adj_status_t adj_comm_get_unique_id(uint8_t id[128]);
adj_status_t adj_comm_init(int nranks, const uint8_t id[128], int rank, adj_comm_t *comm);
/* adj_comm_destroy -- releases the communicator.  Collective (every rank calls it) once an
 *   ADJ_DIST_P2P call has set up the exchange window: importers unmap it, a barrier follows, then
 *   the root frees it (CUDA IPC requires importers to close before the exporter frees). */
adj_status_t adj_comm_destroy(adj_comm_t comm);

/* CUDA IPC of a device pointer inside an allocation (the building blocks of ADJ_DIST_TILES |
 *   ADJ_DIST_P2P; host calls, synchronous).
 *   adj_ipc_export -- ptr: a device pointer anywhere inside a cudaMalloc allocation (e.g. a torch
 *     tensor's data pointer) of the current device.  Writes an ADJ_IPC_RECORD_BYTES record (the
 *     allocation's 64-byte cudaIpcMemHandle_t, then the byte offset of ptr from its base as a
 *     little-endian int64) to rec.  ADJ_ERR_INVALID_VALUE for a null ptr / rec, ADJ_ERR_CUDA
 *     when the memory cannot be exported (stream-ordered pool memory, host memory).
 *   adj_ipc_open -- maps the record's allocation in this process (another process; any device
 *     with peer access to the owner's, or the same device) and returns base + offset in *ptr.
 *   adj_ipc_close -- unmaps a pointer adj_ipc_open returned (after the work that uses it has
 *     completed).  The exporter must not free the allocation before every importer closed it. */
#define ADJ_IPC_RECORD_BYTES 72
adj_status_t adj_ipc_export(const void *ptr, uint8_t rec[ADJ_IPC_RECORD_BYTES]);
adj_status_t adj_ipc_open(const uint8_t rec[ADJ_IPC_RECORD_BYTES], void **ptr);
adj_status_t adj_ipc_close(void *ptr);

/* adj_dist_kslice -- the column slice [k0, k1) of A that rank `rank` of `nranks` owns in
 *   adjprod_modp_dist (host, no GPU): per = ceil(k / nranks) rounded up to a multiple of 8,
 *   k0 = min(k, rank * per), k1 = min(k, k0 + per).  Slices are disjoint and cover [0, k). */
adj_status_t adj_dist_kslice(int64_t k, int nranks, int rank, int64_t *k0, int64_t *k1);

/* adj_elem_bytes -- bytes of one element of A as the entry points read it (host, no GPU):
 *   (2 with ADJ_IN_U16 in `flags`, else 4) x the words per element of phi (T 1, H 2, Q 4).
 *   Rank r's k-slice of a row-major A starts at byte offset k0 * adj_elem_bytes(...) of each row
 *   (adjprod_modp_dist, split-K).  INVALID_VALUE for a null output or an unknown phi. */
adj_status_t adj_elem_bytes(adj_phi_t phi, uint32_t flags, int64_t *bytes);

/*
 * adjprod_modp_shard -- output-tile sharding, phi = ADJ_PHI_T, depth 0 or 1
 *   (-1: the automatic depth capped at 1).  The top-level product grid of Alg. alg:MIAHMM (the
 *   (m/2) grid of P1..P5 at depth 1; the grid of C at depth 0) is cut into 256 x 256 tiles;
 *   pairs {(I, J), (J, I)}, I >= J, are dealt to `nranks` owners in blocks of band groups (a
 *   pair reads the operand rows of tile bands I and J only; the blocks keep each rank's bands
 *   few; deterministic).  This call writes exactly the regions of Low(C) that `rank` owns
 *   (adj_shard_layout) and nothing else: the top-level pre-addition (or the depth-0 split) covers
 *   only the rows of the bands the rank's tiles read (adj_shard_rows), the grouped leaf launch
 *   runs only the owned tiles of P1..P5 and the recombination only the owned tile pairs.
 *   Running every rank's share, on one device or on several, writes all of Low(C).  A caller
 *   workspace of adjprod_modp_workspace_size(m, k, p, ADJ_PHI_T, depth) bytes (the same depth)
 *   suffices.  ADJ_FILL_UPPER is not supported here (INVALID_VALUE).
 */
adj_status_t adjprod_modp_shard(int64_t m, int64_t k, uint32_t p, adj_phi_t phi,
                                const uint32_t *A, int64_t lda, uint32_t *C, int64_t ldc,
                                int rank, int nranks, const adj_opts_t *opts, adj_stream_t stream);

/*
 * adjprod_modp_partial -- Low(A A^T) mod p (phi = ADJ_PHI_T) written as canonical residues in
 *   the narrowest width: uint16 for p < 2^16, uint32 otherwise.  R is m x m with leading
 *   dimension ldr ELEMENTS of that width (device, caller-owned; may be peer memory over
 *   NVLink).  The building block of the split-K exchange: partials of column slices are summed
 *   exactly by adj_sum_partials (2 bytes per residue moved instead of 4).
 */
adj_status_t adjprod_modp_partial(int64_t m, int64_t k, uint32_t p, adj_phi_t phi,
                                  const uint32_t *A, int64_t lda, void *R, int64_t ldr,
                                  const adj_opts_t *opts, adj_stream_t stream);

/*
 * adj_sum_partials -- Low(C) = (sum_{r < n} Low(R_r)) mod p, R_r = R + r * stride elements,
 *   elements uint16 for p < 2^16 else uint32 (as adjprod_modp_partial writes them), each a
 *   residue < p; exact while n (p - 1) < 2^32.  Device pointers, async on `stream`.
 */
adj_status_t adj_sum_partials(int64_t m, uint32_t p, const void *R, int64_t ldr, int64_t stride, int n,
                              uint32_t *C, int64_t ldc, adj_stream_t stream);

/*
 * adj_shard_layout -- (host, no GPU) the regions of C that `rank` of `nranks` writes in
 *   adjprod_modp_shard for this problem: *n_rects regions, each 5 int64 (row0, col0, rows,
 *   cols, lower) stored in rects[5*i..5*i+4] for i < max_rects (rects may be NULL); lower = 1
 *   means only the elements with col <= row belong to the rank.  *n_elems = sum rows*cols.
 *   The regions of all ranks partition Low(C).
 */
adj_status_t adj_shard_layout(int64_t m, int64_t k, uint32_t p, int depth, int rank, int nranks,
                              int64_t *rects, int64_t max_rects, int64_t *n_rects, int64_t *n_elems);

/*
 * adj_shard_rows -- (host, no GPU) the row ranges [lo, hi) of the top-level operands that `rank`
 *   pre-adds in adjprod_modp_shard (rows of the (m/2) quadrants at depth 1, of A at depth 0):
 *   *n_ranges ranges stored as ranges[2*i], ranges[2*i+1] for i < max_ranges (ranges may be NULL).
 */
adj_status_t adj_shard_rows(int64_t m, int64_t k, uint32_t p, int depth, int rank, int nranks,
                            int64_t *ranges, int64_t max_ranges, int64_t *n_ranges);

/*
 * adj_shard_pack -- pack (unpack = 0) the regions of C that `rank` of `nranks` owns
 *   (adj_shard_layout, region by region, row by row) into the contiguous buffer `buf`, as uint16
 *   residues for p < 2^16 and uint32 otherwise, or unpack them back into C (unpack = 1; only the
 *   elements col <= row of "lower" regions).  buf holds n_elems of adj_shard_layout.  Device
 *   pointers, async on `stream`.  The gather step of ADJ_DIST_TILES.
 */
adj_status_t adj_shard_pack(int64_t m, int64_t k, uint32_t p, int depth, int rank, int nranks,
                            uint32_t *C, int64_t ldc, void *buf, int unpack, adj_stream_t stream);

/*
 * adjprod_modp_dist -- collective; every rank of `comm` calls it with the same m, k, p, phi,
 *   root.  Default: split-K sharding: rank r computes Low(A_r phi(A_r)) on its
 *   column slice A_r = A[:, k_r0 : k_r1] (k_r0 = r*ceil(k/G) rounded to a multiple of 8) with
 *   the single-GPU path (adjprod_modp_dist_partial), packs the lower triangle (m (m+1) / 2
 *   elements, row by row) as uint32 words, the packed partials are summed exactly with an NCCL
 *   uint32 reduce to `root` (sum < G p < 2^32) and reduced mod p into Low(C) there.
 *   A: the full m x k matrix on every rank (only the rank's slice is read).  C: m x m on every
 *   rank; Low(C) is the result on `root` only.
 *   With opts->flags & ADJ_DIST_TILES (phi = ADJ_PHI_T): output-tile sharding instead -- every
 *   rank runs adjprod_modp_shard with the full A into its C, then the root gathers the other
 *   ranks' regions (packed, NCCL send/recv: only result tiles move).
 *   With ADJ_DIST_TILES | ADJ_DIST_P2P: the same sharding, each rank's final kernel storing its
 *   regions straight into the root's C over NVLink (the root exports C with adj_ipc_export and
 *   broadcasts the record and ldc; the other ranks' C arguments are not used).  The root's C
 *   must be cudaMalloc memory (ADJ_ERR_CUDA on every rank otherwise).  Two host-synchronised
 *   barriers: after the compute (every peer store has landed when the call returns on the root)
 *   and after the importers unmapped C (the caller may free C once the call returns).
 */
adj_status_t adjprod_modp_dist(int64_t m, int64_t k, uint32_t p, adj_phi_t phi,
                               const uint32_t *A, int64_t lda, uint32_t *C, int64_t ldc,
                               int root, adj_comm_t comm, const adj_opts_t *opts,
                               adj_stream_t stream);

/*
 * adjprod_modp_dist_partial -- rank `rank`'s share of the split-K sharding of adjprod_modp_dist:
 *   Low(A_r phi(A_r)) mod p of its column slice A_r = A[:, k0:k1) (adj_dist_kslice), read at byte
 *   offset k0 * adj_elem_bytes(phi, flags) of each row of A, written to R (m x m, leading
 *   dimension ldr, uint32 or, with ADJ_OUT_U16, uint16 words x phi's width).  Not collective:
 *   the partials of all ranks summed mod p give Low(A phi(A)).  Device pointers, async.
 */
adj_status_t adjprod_modp_dist_partial(int64_t m, int64_t k, uint32_t p, adj_phi_t phi,
                                       const uint32_t *A, int64_t lda, uint32_t *R, int64_t ldr,
                                       int rank, int nranks, const adj_opts_t *opts,
                                       adj_stream_t stream);

/* ---------------- diagnostics ---------------- */
const char *adj_status_string(adj_status_t status);
const char *adj_last_error(void); /* thread-local detail for the last failing call */

/* Number of kernels the library launched on this thread since the last reset (the
 * bench's gpu_launches claim) and a reset. */
uint64_t adj_launch_count(void);
void adj_launch_count_reset(void);

/* Per-kernel-class timing for measurement (bench.py).  When enabled, CUDA events are recorded
 * on the launch stream around every launch of class c (0 = grouped tcgen05 leaf, 1 = K1
 * pre-addition / limb split, 2 = K4 / K5 recombination, 3 = other); adj_profile_read
 * synchronises on them and returns, per class, the summed milliseconds and launch counts,
 * then clears the record.  Disabled by default (no events, no overhead). */
void adj_profile_enable(int on);
adj_status_t adj_profile_read(double ms[4], uint64_t launches[4]);

#ifdef __cplusplus
}
#endif
#endif /* ADJPROD_H */
