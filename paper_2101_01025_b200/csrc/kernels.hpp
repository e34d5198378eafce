// Host-callable launchers of the sm_100a kernels (leaf.cu, preadd.cu, combine.cu, misc.cu).
#pragma once
#include <cuda_runtime.h>

#include "types.hpp"

namespace adj {

cudaError_t launch_fixup(const LeafParams &p, const FixupTile *tiles, int n, cudaStream_t s);
cudaError_t launch_leaf2(const LeafParams &p, int nacc, bool segmented, int grid, cudaStream_t s);  // CTA-pair, 256x256 tiles
cudaError_t launch_leafw(const LeafParams &p, int nacc, int grid, cudaStream_t s);                  // CTA-pair, 256x512 tiles
cudaError_t launch_preadd(const PreParams &p, cudaStream_t s);
cudaError_t launch_preadd2(const PreParams &l1, const PreParams &l2, cudaStream_t s);   // fused K1 of levels 1 + 2
cudaError_t launch_split(const SplitParams &p, cudaStream_t s);
cudaError_t launch_combine(const CombParams &p, cudaStream_t s);
cudaError_t launch_herk_preadd(const HerkPreParams &p, cudaStream_t s);
cudaError_t launch_herk_combine(const HerkCombParams &p, cudaStream_t s);
cudaError_t launch_quat_combine(const QuatCombParams &p, cudaStream_t s);
cudaError_t launch_twom(int64_t m, const void *G, int64_t ldg, const void *H, int64_t ldh, int in32,
                        void *C, int64_t ldc, const ModP &mod, uint32_t alpha, uint32_t beta, int axpby,
                        int out16, cudaStream_t s);
cudaError_t launch_scale_lower(int64_t m, int w, uint32_t *X, int64_t ldx, uint32_t beta, const ModP &mod,
                               cudaStream_t s);
cudaError_t launch_mod_lower(int64_t m, int w, const uint32_t *src, int64_t lds, uint32_t *dst, int64_t ldd,
                             const ModP &mod, cudaStream_t s);
// split-K exchange: Low(src) (uint16 / uint32 words, esz 2 / 4, w per element) packed row by row
// into uint32 words (element offset i (i + 1) / 2 for row i), and the packed sum back into Low(C) mod p
cudaError_t launch_pack_lower(int64_t m, int w, const void *src, int64_t lds, int esz, uint32_t *dst, cudaStream_t s);
cudaError_t launch_unpack_mod_lower(int64_t m, int w, const uint32_t *src, uint32_t *C, int64_t ldc, const ModP &mod,
                                    cudaStream_t s);
// Low(X) <- 0, elements of esz bytes (even), one launch
cudaError_t launch_zero_lower(int64_t m, void *X, int64_t ld_bytes, int esz, cudaStream_t s);
// pack (to_buf = 1) / unpack (to_buf = 0) / zero (to_buf = 2) the listed regions of C into / from a contiguous buffer
// of esize-byte residues (2: uint16 for p < 2^16)
cudaError_t launch_rect_copy(const RectDev *rects, int n, int max_rows, uint32_t *C, int64_t ldc, void *buf,
                             int esize, int to_buf, cudaStream_t s);
// C[i][j] = (sum_r R_r[i][j]) mod p on Low, R_r = R + r * stride (elements of `esize` bytes)
cudaError_t launch_sum_partials(int64_t m, const void *R, int64_t ldr, int64_t stride, int n, int esize, uint32_t *C,
                                int64_t ldc, const ModP &mod, cudaStream_t s);
cudaError_t launch_fill_upper(int64_t m, int w, uint32_t *C, int64_t ldc, const ModP &mod, cudaStream_t s);

}  // namespace adj
