/*
 * synth.c -- host fill of the seeded generator in synth.h (input synthesis only; see synth.h).
 * Built into synth/libsynth.so; used by tests/ and bench.py to build the oracle's inputs.
 */
#include "synth.h"
#include <stdint.h>

/*
 * Fill out[(z-z0)][(y-y0)][(x-x0)] for the sub-box [z0,z1) x [y0,y1) x [x0,x1) of a global padded
 * grid of extent (Z, Y, X) (x fastest).  dist 0 = U[-1,1), dist 1 = U[0,c).
 * Returns 0, or -1 on a bad box.
 */
int synth_fill_box(uint64_t seed, int stream, int dist, double c,
                   int64_t Z, int64_t Y, int64_t X,
                   int64_t z0, int64_t z1, int64_t y0, int64_t y1, int64_t x0, int64_t x1,
                   double *out) {
  if (z0 < 0 || y0 < 0 || x0 < 0 || z1 > Z || y1 > Y || x1 > X || z0 > z1 || y0 > y1 || x0 > x1)
    return -1;
  const uint64_t key = synth_key(seed, stream);
  const int64_t ny = y1 - y0, nx = x1 - x0;
#pragma omp parallel for schedule(static)
  for (int64_t z = z0; z < z1; ++z)
    for (int64_t y = y0; y < y1; ++y) {
      double *row = out + ((z - z0) * ny + (y - y0)) * nx;
      const uint64_t base = (uint64_t)((z * Y + y) * X);
      if (dist == 0)
        for (int64_t x = x0; x < x1; ++x) row[x - x0] = synth_sym(key, base + (uint64_t)x);
      else
        for (int64_t x = x0; x < x1; ++x) row[x - x0] = synth_scaled(key, base + (uint64_t)x, c);
    }
  return 0;
}
