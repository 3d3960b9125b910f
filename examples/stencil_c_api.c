/*
 * examples/stencil_c_api.c -- the boundary used from plain C (no Python, no torch): create a seeded
 * 7-point variable-coefficient grid (Fig. 1c), run T steps on the GPU, read the newest level
 * back, print a checksum, and exercise the error paths of include/stencil.h.
 *
 *   cc -O2 -I include examples/stencil_c_api.c -L paper_1410_3060_b200 -lstencil \
 *      -Wl,-rpath,$PWD/paper_1410_3060_b200 -o build/stencil_c_api
 *   build/stencil_c_api [nx ny nz T]
 */
#include <stdio.h>
#include <stdlib.h>

#include "stencil.h"

#define CHECK(call)                                                                  \
  do {                                                                               \
    int rc_ = (call);                                                                \
    if (rc_ != ST_OK) {                                                              \
      fprintf(stderr, "%s failed: %d (%s)\n", #call, rc_, stencil_last_error());     \
      return 1;                                                                      \
    }                                                                                \
  } while (0)

int main(int argc, char **argv) {
  int64_t nx = argc > 1 ? atoll(argv[1]) : 64, ny = argc > 2 ? atoll(argv[2]) : 48;
  int64_t nz = argc > 3 ? atoll(argv[3]) : 40, T = argc > 4 ? atoll(argv[4]) : 10;
  printf("%s\n", stencil_version());

  /* host-only plan of a 4-way z-slab split (no device needed) */
  for (int r = 0; r < 4; ++r) {
    int64_t o0, o1, s0, s1;
    int bt;
    CHECK(stencil_plan_slab(nz, 1, 4, r, 2, &o0, &o1, &s0, &s1, &bt));
    printf("slab %d: owns planes [%lld,%lld), stores [%lld,%lld), bt %d\n", r, (long long)o0,
           (long long)o1, (long long)s0, (long long)s1, bt);
  }

  /* argument errors are reported, never fatal */
  stencil_ctx *bad = NULL;
  if (stencil_create_seeded(&bad, 9, nx, ny, nz, 1, NULL, NULL) != ST_E_INVAL) return 2;
  printf("bad kind -> ST_E_INVAL: %s\n", stencil_last_error());

  st_opts o;
  stencil_opts_default(&o);
  stencil_ctx *h = NULL;
  int rc = stencil_create_seeded(&h, ST_7PT_VAR, nx, ny, nz, 14103060ull, NULL, &o);
  if (rc == ST_E_CUDA) {  /* no GPU: the library has no CPU fallback */
    printf("no CUDA device: %s\n", stencil_last_error());
    return 0;
  }
  CHECK(rc);
  CHECK(stencil_run(h, T));
  st_info info;
  CHECK(stencil_info(h, &info));
  const int64_t n = (nx + 2) * (ny + 2) * (nz + 2);
  double *out = (double *)malloc((size_t)n * sizeof(double));
  CHECK(stencil_read(h, 0, out, n));
  double sum = 0.0;
  for (int64_t i = 0; i < n; ++i) sum += out[i];
  printf("7pt-var %lldx%lldx%lld T=%lld bt=%d launches=%lld checksum=%.17g\n", (long long)nx,
         (long long)ny, (long long)nz, (long long)T, info.bt, (long long)info.launches, sum);
  if (stencil_read(h, 1, out, n) != ST_E_INVAL) return 3; /* level 1 is scratch for Jacobi kinds */
  free(out);
  CHECK(stencil_destroy(h));
  return 0;
}
