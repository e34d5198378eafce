/* Plain C use of the boundary (include/adjprod.h), no Python or PyTorch: Low(A A^T) mod p for a
 * 300 x 257 A over GF(8191) at the automatic depth, a few entries checked against the definition
 * (C = A phi(A)), and the synchronous validation path.
 *
 *   gcc -std=c11 -I include -I /usr/local/cuda/include examples/c_abi_example.c \
 *       -L paper_2101_01025_b200 -ladjprod -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2101_01025_b200 -o c_abi_example && ./c_abi_example
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime.h>

#include "adjprod.h"

int main(void) {
  const int64_t m = 300, k = 257, lda = 260, ldc = 301;
  const uint32_t p = 8191;
  uint32_t *hA = malloc(sizeof(uint32_t) * m * lda), *hC = malloc(sizeof(uint32_t) * m * ldc);
  uint64_t s = 12345;
  for (int64_t i = 0; i < m * lda; ++i) {   /* any 32-bit values: the library reads them mod p */
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    hA[i] = (uint32_t)(s >> 32);
  }
  uint32_t *dA, *dC;
  if (cudaMalloc((void **)&dA, sizeof(uint32_t) * m * lda) != cudaSuccess ||
      cudaMalloc((void **)&dC, sizeof(uint32_t) * m * ldc) != cudaSuccess) {
    printf("no device\n");
    return 2;
  }
  cudaMemcpy(dA, hA, sizeof(uint32_t) * m * lda, cudaMemcpyHostToDevice);
  cudaMemset(dC, 0, sizeof(uint32_t) * m * ldc);

  adj_status_t st = adjprod_modp(m, k, p, ADJ_PHI_T, dA, lda, dC, ldc, NULL);
  if (st != ADJ_OK) {
    printf("adjprod_modp: %s (%s)\n", adj_status_string(st), adj_last_error());
    return 1;
  }
  cudaMemcpy(hC, dC, sizeof(uint32_t) * m * ldc, cudaMemcpyDeviceToHost);

  int bad = 0;
  const int64_t rows[4] = {0, 1, 150, 299};
  for (int r = 0; r < 4; ++r) {
    const int64_t i = rows[r];
    for (int64_t j = 0; j <= i; ++j) {   /* Low(C)[i][j] = sum_t A[i][t] A[j][t] mod p */
      uint64_t acc = 0;
      for (int64_t t = 0; t < k; ++t) acc = (acc + (uint64_t)(hA[i * lda + t] % p) * (hA[j * lda + t] % p)) % p;
      if (hC[i * ldc + j] != (uint32_t)acc) ++bad;
    }
  }
  /* validation is synchronous and needs no launch: 91 = 7 * 13 is not a prime */
  st = adjprod_modp(m, k, 91, ADJ_PHI_T, dA, lda, dC, ldc, NULL);
  const int refused = st == ADJ_ERR_UNSUPPORTED_MODULUS;
  printf("c_abi_example: %s (%d mismatches on 4 sampled rows; p = 91 refused: %s)\n", bad ? "FAIL" : "OK", bad,
         refused ? adj_status_string(st) : "NO");
  cudaFree(dA);
  cudaFree(dC);
  free(hA);
  free(hC);
  return bad || !refused;
}
