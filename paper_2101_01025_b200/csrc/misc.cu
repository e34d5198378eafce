// Small helpers: split-K finalisation (mod p of summed partials), SYRK-form scaling, optional
// Up(C) = phi(Low(C)), output-tile pack / unpack, exact sum of narrow partials.
#include <algorithm>
#include <cstdio>

#include "kernel_util.cuh"

namespace adj {

// ============================================================================ helpers
// dst[i][j] = src[i][j] mod p on the lower triangle (w = 1: uint32, w = 2: (re, im) pairs)
__global__ void mod_lower_kernel(int64_t row0, int w, const uint32_t *src, int64_t lds, uint32_t *dst,
                                 int64_t ldd, ModP mod) {
  const int64_t i = row0 + blockIdx.y;
  const uint32_t *a = src + i * lds * w;
  uint32_t *b = dst + i * ldd * w;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < (i + 1) * w;
       j += (int64_t)gridDim.x * blockDim.x)
    b[j] = mod_u32(a[j], mod);
}

cudaError_t launch_mod_lower(int64_t m, int w, const uint32_t *src, int64_t lds, uint32_t *dst, int64_t ldd,
                             const ModP &mod, cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  const int64_t per_row = (m * w + 255) / 256;
  for (int64_t r0 = 0; r0 < m; r0 += 65535) {
    const int64_t rows = (m - r0) < 65535 ? (m - r0) : 65535;
    mod_lower_kernel<<<dim3((unsigned)(per_row < 64 ? per_row : 64), (unsigned)rows), 256, 0, s>>>(
        r0, w, src, lds, dst, ldd, mod);
  }
  return cudaGetLastError();
}

// split-K exchange: Low(src) packed row by row (row i holds i + 1 elements of w words at
// element offset i (i + 1) / 2) as uint32 words; src words are uint16 (esz 2) or uint32
template <typename T>
__global__ void pack_lower_kernel(int64_t row0, int w, const T *src, int64_t lds, uint32_t *dst) {
  const int64_t i = row0 + blockIdx.y;
  const T *a = src + i * lds * w;
  uint32_t *b = dst + (i * (i + 1) / 2) * w;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < (i + 1) * w; j += (int64_t)gridDim.x * blockDim.x)
    b[j] = (uint32_t)a[j];
}
// and back: C = packed mod p on Low(C)
__global__ void unpack_mod_lower_kernel(int64_t row0, int w, const uint32_t *src, uint32_t *C, int64_t ldc, ModP mod) {
  const int64_t i = row0 + blockIdx.y;
  const uint32_t *a = src + (i * (i + 1) / 2) * w;
  uint32_t *b = C + i * ldc * w;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < (i + 1) * w; j += (int64_t)gridDim.x * blockDim.x)
    b[j] = mod_u32(a[j], mod);
}

cudaError_t launch_pack_lower(int64_t m, int w, const void *src, int64_t lds, int esz, uint32_t *dst, cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  const int64_t per_row = (m * w + 255) / 256;
  for (int64_t r0 = 0; r0 < m; r0 += 65535) {
    const int64_t rows = (m - r0) < 65535 ? (m - r0) : 65535;
    const dim3 grid((unsigned)(per_row < 64 ? per_row : 64), (unsigned)rows);
    if (esz == 2) pack_lower_kernel<uint16_t><<<grid, 256, 0, s>>>(r0, w, static_cast<const uint16_t *>(src), lds, dst);
    else pack_lower_kernel<uint32_t><<<grid, 256, 0, s>>>(r0, w, static_cast<const uint32_t *>(src), lds, dst);
  }
  return cudaGetLastError();
}

cudaError_t launch_unpack_mod_lower(int64_t m, int w, const uint32_t *src, uint32_t *C, int64_t ldc, const ModP &mod,
                                    cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  const int64_t per_row = (m * w + 255) / 256;
  for (int64_t r0 = 0; r0 < m; r0 += 65535) {
    const int64_t rows = (m - r0) < 65535 ? (m - r0) : 65535;
    unpack_mod_lower_kernel<<<dim3((unsigned)(per_row < 64 ? per_row : 64), (unsigned)rows), 256, 0, s>>>(
        r0, w, src, C, ldc, mod);
  }
  return cudaGetLastError();
}

// Low(X) <- beta Low(X) (SYRK form with k = 0)
__global__ void scale_lower_kernel(int64_t row0, int w, uint32_t *X, int64_t ldx, uint32_t beta, ModP mod) {
  const int64_t i = row0 + blockIdx.y;
  uint32_t *row = X + i * ldx * w;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < (i + 1) * w;
       j += (int64_t)gridDim.x * blockDim.x)
    row[j] = mulmod_any(beta, mod_u32(row[j], mod), mod);
}

cudaError_t launch_scale_lower(int64_t m, int w, uint32_t *X, int64_t ldx, uint32_t beta, const ModP &mod,
                               cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  const int64_t per_row = (m * w + 255) / 256;
  for (int64_t r0 = 0; r0 < m; r0 += 65535) {
    const int64_t rows = (m - r0) < 65535 ? (m - r0) : 65535;
    scale_lower_kernel<<<dim3((unsigned)(per_row < 64 ? per_row : 64), (unsigned)rows), 256, 0, s>>>(
        r0, w, X, ldx, beta, mod);
  }
  return cudaGetLastError();
}

// Low(X) <- 0 for esz-byte elements (esz even: uint16 / uint32 residues x phi's width); one launch
// for the whole triangle (k = 0 or alpha = 0), written as uint16 words
__global__ void zero_lower_kernel(int64_t row0, void *X, int64_t ld_bytes, int esz) {
  const int64_t i = row0 + blockIdx.y;
  uint16_t *row = reinterpret_cast<uint16_t *>(static_cast<uint8_t *>(X) + i * ld_bytes);
  const int64_t n = (i + 1) * (esz / 2);
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    row[j] = 0;
}

cudaError_t launch_zero_lower(int64_t m, void *X, int64_t ld_bytes, int esz, cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  const int64_t per_row = (m * (esz / 2) + 255) / 256;
  for (int64_t r0 = 0; r0 < m; r0 += 65535) {
    const int64_t rows = (m - r0) < 65535 ? (m - r0) : 65535;
    zero_lower_kernel<<<dim3((unsigned)(per_row < 64 ? per_row : 64), (unsigned)rows), 256, 0, s>>>(r0, X, ld_bytes,
                                                                                                     esz);
  }
  return cudaGetLastError();
}

// pack / unpack / zero (to_buf = 2) the listed regions of C: one block per (region row, region);
// threads over the columns.  The packed buffer holds
// uint16 residues when p < 2^16 (half the bytes on the wire), uint32 otherwise.
template <typename BT>
__global__ void __launch_bounds__(256) rect_copy_kernel(const RectDev *rects, uint32_t *C, int64_t ldc, BT *buf,
                                                        int to_buf) {
  const RectDev R = rects[blockIdx.y];
  const int64_t i = blockIdx.x;
  if (i >= R.rows) return;
  uint32_t *c = C + (R.r0 + i) * ldc + R.c0;
  BT *b = buf + R.off + i * R.cols;
  const int64_t ncol = R.lower ? min64(R.cols, R.r0 + i - R.c0 + 1) : R.cols;
  for (int64_t j = threadIdx.x; j < ncol; j += blockDim.x) {
    if (to_buf == 1) b[j] = (BT)c[j];
    else if (to_buf == 0) c[j] = b[j];
    else c[j] = 0;
  }
}

cudaError_t launch_rect_copy(const RectDev *rects, int n, int max_rows, uint32_t *C, int64_t ldc, void *buf,
                             int esize, int to_buf, cudaStream_t s) {
  if (n == 0 || max_rows == 0) return cudaSuccess;
  const dim3 grid((unsigned)max_rows, (unsigned)n);
  if (esize == 2) rect_copy_kernel<uint16_t><<<grid, 256, 0, s>>>(rects, C, ldc, static_cast<uint16_t *>(buf), to_buf);
  else rect_copy_kernel<uint32_t><<<grid, 256, 0, s>>>(rects, C, ldc, static_cast<uint32_t *>(buf), to_buf);
  return cudaGetLastError();
}

// exact residue sum of n partials (each < p, n (p - 1) < 2^32) then mod p, on Low; one block per row
template <typename T>
__global__ void __launch_bounds__(256) sum_partials_kernel(int64_t m, const T *R, int64_t ldr, int64_t stride, int n,
                                                           uint32_t *C, int64_t ldc, ModP mod) {
  const int64_t i = blockIdx.x;
  if (i >= m) return;
  for (int64_t j = threadIdx.x; j <= i; j += blockDim.x) {
    uint32_t acc = 0;
    for (int r = 0; r < n; ++r) acc += (uint32_t)R[(int64_t)r * stride + i * ldr + j];
    C[i * ldc + j] = mod_u32(acc, mod);
  }
}

cudaError_t launch_sum_partials(int64_t m, const void *R, int64_t ldr, int64_t stride, int n, int esize, uint32_t *C,
                                int64_t ldc, const ModP &mod, cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  if (esize == 2)
    sum_partials_kernel<uint16_t><<<(unsigned)m, 256, 0, s>>>(m, static_cast<const uint16_t *>(R), ldr, stride, n, C,
                                                               ldc, mod);
  else
    sum_partials_kernel<uint32_t><<<(unsigned)m, 256, 0, s>>>(m, static_cast<const uint32_t *>(R), ldr, stride, n, C,
                                                               ldc, mod);
  return cudaGetLastError();
}

// Up(C) = phi(Low(C)) (Lemma lem:uplow): C[j][i] = C[i][j] (conjugated for phi = H), i > j
__global__ void __launch_bounds__(256) fill_upper_kernel(int64_t m, int w, uint32_t *C, int64_t ldc, ModP mod) {
  const int ti = blockIdx.y, tj = blockIdx.x;
  if (ti < tj) return;
  const int tx = threadIdx.x, ty = threadIdx.y;
  __shared__ uint32_t s[32][33][4];
  const int64_t i0 = (int64_t)ti * 32, j0 = (int64_t)tj * 32;
  for (int y = ty; y < 32; y += 8) {
    const int64_t i = i0 + y, j = j0 + tx;
    if (i < m && j < m && j < i)
      for (int c = 0; c < w; ++c) s[y][tx][c] = C[(i * ldc + j) * w + c];
  }
  __syncthreads();
  for (int y = ty; y < 32; y += 8) {
    const int64_t r = j0 + y, c = i0 + tx;   // upper element (r, c) = phi(C[c][r]): conjugate, transposed
    if (r < m && c < m && r < c) {
      C[(r * ldc + c) * w] = s[tx][y][0];
      for (int q = 1; q < w; ++q) C[(r * ldc + c) * w + q] = submod(0, s[tx][y][q], mod);
    }
  }
}

cudaError_t launch_fill_upper(int64_t m, int w, uint32_t *C, int64_t ldc, const ModP &mod, cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  const unsigned nt = (unsigned)((m + 31) / 32);
  fill_upper_kernel<<<dim3(nt, nt), dim3(32, 8), 0, s>>>(m, w, C, ldc, mod);
  return cudaGetLastError();
}

}  // namespace adj
