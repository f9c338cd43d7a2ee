/* A C host calling the engine through the C ABI only (include/gridshift_cuda.h,
 * libgridshift_cuda.so): the binding a non-Python caller of the reference's
 * meanshiftpp (modeseek.py:125-146) would use.  Two Gaussian blobs in 2-D;
 * prints clusters, iterations and the first labels.
 *
 *   gcc -O2 -I include examples/c_host.c -L paper_2104_00303_b200 \
 *       -lgridshift_cuda -Wl,-rpath,$PWD/paper_2104_00303_b200 -lm -o c_host
 *   ./c_host            (needs a GPU; "--version" only loads the library)
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "gridshift_cuda.h"

static double gauss(uint64_t* s) {   /* Box-Muller on a splitmix64 stream */
  double u[2];
  for (int i = 0; i < 2; ++i) {
    uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    u[i] = ((double)(z >> 11) + 0.5) * 0x1p-53;
  }
  return sqrt(-2.0 * log(u[0])) * cos(6.283185307179586 * u[1]);
}

int main(int argc, char** argv) {
  printf("%s\n", gs_version());
  if (argc > 1 && strcmp(argv[1], "--version") == 0) return 0;
  const int64_t n = 20000;
  const int32_t d = 2, max_iters = 300;
  double* x = malloc(sizeof(double) * n * d);
  uint64_t seed = 7;
  for (int64_t i = 0; i < n; ++i) {
    const double cx = (i & 1) ? 8.0 : 2.0;
    x[i * d] = cx + 0.4 * gauss(&seed);
    x[i * d + 1] = 5.0 + 0.4 * gauss(&seed);
  }
  gs_ctx* ctx = NULL;
  if (gs_ctx_create(0, &ctx) != GS_OK) {
    fprintf(stderr, "context: %s\n", gs_last_error());
    return 1;
  }
  int64_t* labels = malloc(sizeof(int64_t) * n);
  double movement[300];
  int64_t k = 0;
  int32_t iters = 0, converged = 0;
  const double h = 0.5, eta = 1e-4 * (double)n * h;   /* ShiftConfig.resolve_eta default */
  const int rc = gs_meanshiftpp(ctx, x, n, d, h, eta, max_iters, labels, &k, &iters, movement, &converged);
  if (rc != GS_OK) {
    fprintf(stderr, "gs_meanshiftpp: %s\n", gs_last_error());
    return 1;
  }
  double* modes = malloc(sizeof(double) * k * d);
  gs_fetch_modes(ctx, modes, k);
  printf("k=%lld iterations=%d converged=%d\n", (long long)k, iters, converged);
  for (int64_t c = 0; c < k; ++c) printf("mode %lld: (%.6f, %.6f)\n", (long long)c, modes[c * d], modes[c * d + 1]);
  printf("labels[0..3] = %lld %lld %lld %lld\n", (long long)labels[0], (long long)labels[1],
         (long long)labels[2], (long long)labels[3]);
  gs_ctx_destroy(ctx);
  free(modes);
  free(labels);
  free(x);
  return 0;
}
