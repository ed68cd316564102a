/* Minimal C client of libcwreco (include/cwreco.h): no Python, no torch.
 *
 * Builds a periodic 2-D mesh of n×n squares split into triangles, sets cell
 * averages of a smooth field, and runs the CWENO reconstruction (M = 3, 4
 * variables) end to end through cwreco_reconstruct_host (host buffers).  Without
 * a CUDA device the host setup still runs and the compute call reports ECUDA
 * (there is no CPU fallback); the program then exits 0 after printing it.
 *
 *   cc -O2 -I include examples/cwreco_example.c -L paper_1612_09335_b200 -lcwreco \
 *      -Wl,-rpath,$PWD/paper_1612_09335_b200 -lm -o /tmp/cwreco_example
 *   /tmp/cwreco_example [device]      (device < 0: host-only context)
 */
#define _USE_MATH_DEFINES
#include <math.h>
#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "cwreco.h"

#define CHECK(call)                                                                  \
  do {                                                                               \
    cwreco_status s_ = (call);                                                       \
    if (s_ != CWRECO_OK) {                                                           \
      fprintf(stderr, "%s -> status %d: %s\n", #call, (int)s_, cwreco_last_error()); \
      return s_ == CWRECO_ECUDA ? 0 : 1;                                             \
    }                                                                                \
  } while (0)

int main(int argc, char** argv) {
  const int device = argc > 1 ? atoi(argv[1]) : 0;
  const int n = 24, d = 2, M = 3, V = 4;
  const int64_t n_nodes = (int64_t)n * n, n_cells = 2LL * n * n;
  double* xyz = malloc(sizeof(double) * n_nodes * d);
  int64_t* cells = malloc(sizeof(int64_t) * n_cells * 3);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      xyz[(j * n + i) * 2 + 0] = (double)i / n;
      xyz[(j * n + i) * 2 + 1] = (double)j / n;
    }
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {  /* periodic torus: node indices wrap (R28 split) */
      const int64_t a = j * n + i, b = j * n + (i + 1) % n, c = ((j + 1) % n) * n + (i + 1) % n,
                    e = ((j + 1) % n) * n + i, t = 2 * (j * n + i);
      cells[3 * t + 0] = a; cells[3 * t + 1] = b; cells[3 * t + 2] = c;
      cells[3 * t + 3] = a; cells[3 * t + 4] = c; cells[3 * t + 5] = e;
    }
  const double period[2] = {1.0, 1.0};
  cwreco_params prm = {1e5, 1.0, 1e-14, 4};
  cwreco_ctx* ctx = NULL;
  CHECK(cwreco_create(d, M, V, &prm, device, &ctx));
  CHECK(cwreco_set_mesh(ctx, n_nodes, xyz, n_cells, cells, period));
  CHECK(cwreco_build_stencils(ctx));
  CHECK(cwreco_precompute(ctx));
  cwreco_info info;
  CHECK(cwreco_get_info(ctx, &info));
  printf("cells %lld, modes %d, stencil %d, tile cells %d, device bytes %lld\n", (long long)info.n_cells,
         info.n_modes, info.n_e, info.tile_cells, (long long)info.device_bytes);
  /* averages in SFC order: Q = (1, sin 2πx, cos 2πy, 2) at the barycentres (first-order averages) */
  int64_t* perm = malloc(sizeof(int64_t) * n_cells);
  CHECK(cwreco_get_permutation(ctx, perm));
  double* avgs = malloc(sizeof(double) * n_cells * V);
  for (int64_t s = 0; s < n_cells; ++s) {
    const int64_t c = perm[s];
    double bx = 0, by = 0;
    for (int k = 0; k < 3; ++k) {
      double x = xyz[cells[3 * c + k] * 2], y = xyz[cells[3 * c + k] * 2 + 1];
      if (k && x - xyz[cells[3 * c] * 2] < -0.5) x += 1.0;
      if (k && y - xyz[cells[3 * c] * 2 + 1] < -0.5) y += 1.0;
      bx += x / 3;
      by += y / 3;
    }
    avgs[s * V + 0] = 1.0;
    avgs[s * V + 1] = sin(2 * M_PI * bx);
    avgs[s * V + 2] = cos(2 * M_PI * by);
    avgs[s * V + 3] = 2.0;
  }
  double* coeffs = malloc(sizeof(double) * n_cells * V * info.n_modes);
  CHECK(cwreco_reconstruct_host(ctx, avgs, coeffs, 0, NULL));
  /* conservation: w[0]·ψ1 = Q for every cell and variable */
  double worst = 0, psi1 = sqrt(2.0);
  for (int64_t s = 0; s < n_cells; ++s)
    for (int v = 0; v < V; ++v) {
      const double e = fabs(coeffs[(s * V + v) * info.n_modes] * psi1 - avgs[s * V + v]);
      if (e > worst) worst = e;
    }
  printf("reconstructed %lld cells; conservation error %.3g\n", (long long)n_cells, worst);
  cwreco_destroy(ctx);
  free(xyz); free(cells); free(perm); free(avgs); free(coeffs);
  return worst <= 1e-14 ? 0 : 1;
}
