/* c_abi_demo.c — the MFP through the C ABI alone (include/mfp.h), no Python:
 * exact-subsolver solve of x^2 - y^2 (exactly discrete-harmonic) on a 65 x 65 grid,
 * checked against the closed form.
 *
 *   gcc -O2 -I include examples/c_abi_demo.c -L paper_2308_14258_b200 -lmfp \
 *       -I /usr/local/cuda/include -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_2308_14258_b200 -o /tmp/mfp_demo
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "mfp.h"

#define CHECK(x)                                                                            \
  do {                                                                                      \
    mfp_status s_ = (x);                                                                    \
    if (s_ != MFP_OK) {                                                                     \
      fprintf(stderr, "%s -> %d (%s)\n", #x, (int)s_, ctx ? mfp_last_error(ctx) : "");    \
      return 1;                                                                             \
    }                                                                                       \
  } while (0)

int main(void) {
  const int n = 64;
  mfp_ctx* ctx = NULL;
  mfp_config cfg = {MFP_ABI_VERSION, n, n, 32, 16, 1, 1, MFP_FP32, MFP_EXACT_LAPLACE, 4};
  mfp_sdnet_desc net = {2, {5, 5, 0, 0}, {1, 8, 1, 0, 0}, 128, 3, 0};
  size_t ws = 0;
  CHECK(mfp_workspace_size(&cfg, &net, 0, &ws));
  void* dws = NULL;
  if (cudaMalloc(&dws, ws) != cudaSuccess) { fprintf(stderr, "cudaMalloc failed\n"); return 1; }
  CHECK(mfp_init(&cfg, &net, NULL, 0, 0, NULL, dws, ws, NULL, &ctx));
  /* g walked counter-clockwise from (0,0): bottom x = 0..n-1, right y = 0..n-1,
   * top x = n..1, left y = n..1 (reading G6); f = x^2 - y^2 at h = 1/64 */
  const double h = 1.0 / 64.0;
  float* g = (float*)malloc(sizeof(float) * 4 * n);
  int k = 0;
  for (int x = 0; x < n; x++) g[k++] = (float)((x * h) * (x * h));
  for (int y = 0; y < n; y++) g[k++] = (float)((n * h) * (n * h) - (y * h) * (y * h));
  for (int x = n; x > 0; x--) g[k++] = (float)((x * h) * (x * h) - (n * h) * (n * h));
  for (int y = n; y > 0; y--) g[k++] = (float)(-(y * h) * (y * h));
  float* u = (float*)malloc(sizeof(float) * (n + 1) * (n + 1));
  mfp_report rep;
  mfp_status st = mfp_solve(ctx, g, 2000, 1e-7f, u, &rep);
  if (st != MFP_OK) { fprintf(stderr, "solve -> %d (%s)\n", (int)st, mfp_last_error(ctx)); return 1; }
  double err = 0.0;
  for (int y = 0; y <= n; y++)
    for (int x = 0; x <= n; x++) {
      const double f = (x * h) * (x * h) - (y * h) * (y * h);
      const double e = fabs(u[y * (n + 1) + x] - f);
      if (e > err) err = e;
    }
  printf("exact subsolver: %d iterations, converged %d, max |u - (x^2 - y^2)| = %.3e\n", rep.iterations,
         rep.converged, err);
  mfp_destroy(ctx);
  cudaFree(dws);
  free(g);
  free(u);
  return err < 1e-5 ? 0 : 2;
}
