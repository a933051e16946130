/* fram_demo.c — the C ABI used from plain C (no CUDA headers, host buffers).
 *
 * Builds a seeded weighted random graph A (n nodes), its relabelled copy Ã = P·A·Pᵀ with a known
 * permutation σ (B[σ(i)][σ(j)] = A[i][j], R18), solves FRAM (Alg. 1) through fram_solve
 * with HOST pointers (the library stages them to the device), and checks that the matching found
 * is σ.  Exit code 0 = matched, 1 = wrong matching, 2 = library error (message printed; e.g. no
 * sm_100 GPU: FRAM_ERR_CUDA — there is no CPU fallback).
 *
 * Build (done by __graft_entry__.build()):
 *   gcc -O2 -Iinclude examples/fram_demo.c -Lpaper_2508_00887_b200 -lfram \
 *       -Wl,-rpath,'$ORIGIN/../paper_2508_00887_b200' -o examples/fram_demo
 * Usage: examples/fram_demo [n=64] [precision: 0 fp64 | 1 tf32 | 2 bf16 | 3 fp16]
 */
#include <stdio.h>
#include <stdlib.h>

#include "fram.h"

static uint64_t s_state = 0x9e3779b97f4a7c15ull;
static double urand(void) {                 /* splitmix64 → [0, 1) */
  uint64_t z = (s_state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  z ^= z >> 31;
  return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 64;
  const int prec = argc > 2 ? atoi(argv[2]) : FRAM_PREC_FP64;
  if (n < 2 || prec < 0 || prec > 3) {
    fprintf(stderr, "usage: %s [n>=2] [precision 0-3]\n", argv[0]);
    return 2;
  }
  double* A = calloc((size_t)n * n, sizeof(double));
  double* B = calloc((size_t)n * n, sizeof(double));
  int* sigma = malloc((size_t)n * sizeof(int));
  int32_t* perm = malloc((size_t)n * sizeof(int32_t));
  if (!A || !B || !sigma || !perm) return 2;
  for (int i = 0; i < n; ++i)                 /* weighted random graph, edge density 0.3 */
    for (int j = i + 1; j < n; ++j)
      if (urand() < 0.3) A[(size_t)i * n + j] = A[(size_t)j * n + i] = 0.1 + urand();
  for (int i = 0; i < n; ++i) sigma[i] = i;   /* Fisher–Yates */
  for (int i = n - 1; i > 0; --i) {
    const int k = (int)(urand() * (i + 1));
    const int t = sigma[i]; sigma[i] = sigma[k]; sigma[k] = t;
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) B[(size_t)sigma[i] * n + sigma[j]] = A[(size_t)i * n + j];

  fram_schedule s = {10.0, 0.95, 1e-3, 1e-4, 100, 1000, 0, FRAM_FLAG_CHECK_SYMMETRY, NULL, 0};
  fram_handle h = NULL;
  fram_status st = fram_create(n, 1.0, &s, 0, &h);
  if (st != FRAM_OK) {
    fprintf(stderr, "fram_create: status %d: %s\n", (int)st, fram_last_error());
    return 2;
  }
  fram_stats stats = {0};
  st = fram_solve(h, FRAM_DT_F64, A, B, NULL, NULL, (fram_precision)prec, NULL, NULL, perm, &stats);
  if (st != FRAM_OK && st != FRAM_NOT_CONVERGED) {
    fprintf(stderr, "fram_solve: status %d: %s\n", (int)st, fram_last_error());
    fram_destroy(h);
    return 2;
  }
  int correct = 0;
  for (int i = 0; i < n; ++i) correct += (perm[i] == sigma[i]);
  printf("n=%d precision=%d status=%d outer_iters=%d total_passes=%lld accuracy=%.4f\n", n, prec, (int)st,
         stats.outer_iters, (long long)stats.total_passes, (double)correct / n);
  fram_destroy(h);
  free(A); free(B); free(sigma); free(perm);
  return correct == n ? 0 : 1;
}
