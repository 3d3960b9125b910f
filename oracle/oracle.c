/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.  The plain, slow, obviously-correct CPU oracle of the
 * paper's stencil updates.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load or call this; the product path (paper_1410_3060_b200/) never does,
 * and shares no code, header or constant with it.
 *
 * What it computes (§3.1 "Definitions and terminology", lines 106-136, and Fig. 1,
 * lines 138-268): T Jacobi sweeps ("the stencil array ... is not written to during the same
 * sweep", line 130) of one of four star stencils over the interior of a padded grid
 * Omega[z][y][x], x fastest (lines 119-126).  The time index takes only the values 0 and 1:
 * each sweep writes the other buffer, then the buffers swap (lines 126-128).  The naive order is
 * one full sweep per time step (§4.1).
 *
 *   kind 1, 7-point constant  (Fig. 1b):
 *     O' = w1*O + w2*(O[x-1]+O[x+1]) + w2*(O[y-1]+O[y+1]) + w2*(O[z-1]+O[z+1])
 *   kind 2, 7-point variable  (Fig. 1c):
 *     O' = W0*O + W1*O[x-1] + W2*O[x+1] + W3*O[y-1] + W4*O[y+1] + W5*O[z-1] + W6*O[z+1]
 *   kind 3, 25-point constant wave, 2nd order in time (Fig. 1e), scalar alpha
 *     (reading Q2):
 *     O^{t+1} = 2*O^t - O^{t-1} + alpha*[w0*O^t + sum_{r=1..4} w_r*((x pair_r)+(y pair_r)+(z pair_r))]
 *     O^{t+1} overwrites the buffer that held O^{t-1} (line 126-128; each point reads its own
 *     O^{t-1} before writing it).
 *   kind 5, the same wave with the domain-sized alpha_{z,y,x} exactly as Fig. 1e prints it (
 *     SURVEY.md NEXT-1): alpha is one padded coefficient field, w0..w4 scalars.
 *   kind 4, 25-point variable, axis-symmetric (Fig. 1d):
 *     O' = W0*O + sum_{r=1..4} [ W_{3r-2}*(x pair_r) + W_{3r-1}*(y pair_r) + W_{3r}*(z pair_r) ]
 *
 * Every expression is evaluated left to right exactly as printed in Fig. 1 (each + and * one
 * IEEE-754 binary64 round-to-nearest operation); the file is compiled with -ffp-contract=off so
 * no FMA is formed.  Ghost cells (width R, the fixed boundary of reading Q1) are read, never
 * written.  OpenMP over z only: every point is computed independently, so the result does not
 * depend on the thread count (pin P10).
 *
 * Parity status: pinned (tests/test_oracle_pins.py, pins P1-P11 of DESIGN.md).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_OK 0
#define OR_EINVAL -1
#define OR_ENOMEM -2

static int radius_of(int kind) {
  switch (kind) {
    case 1: case 2: return 1;
    case 3: case 4: case 5: return 4;
    default: return -1;
  }
}

static int ncoef_of(int kind) { return kind == 2 ? 7 : kind == 4 ? 13 : kind == 5 ? 1 : 0; }
static int nscal_of(int kind) { return kind == 1 ? 2 : kind == 3 ? 6 : kind == 5 ? 5 : 0; }

/* One sweep of kind 1 (Fig. 1b): dst <- F(src) over the interior. */
static void sweep_7c(int64_t nx, int64_t ny, int64_t nz, const double *src, double *dst,
                     double w1, double w2) {
  const int64_t X = nx + 2, Y = ny + 2;
  const int64_t sy = X, sz = X * Y;
#pragma omp parallel for schedule(static)
  for (int64_t z = 1; z <= nz; ++z)
    for (int64_t y = 1; y <= ny; ++y)
      for (int64_t x = 1; x <= nx; ++x) {
        const int64_t p = z * sz + y * sy + x;
        dst[p] = w1 * src[p]
               + w2 * (src[p - 1] + src[p + 1])
               + w2 * (src[p - sy] + src[p + sy])
               + w2 * (src[p - sz] + src[p + sz]);
      }
}

/* One sweep of kind 2 (Fig. 1c). W[0..6] = centre, x-1, x+1, y-1, y+1, z-1, z+1. */
static void sweep_7v(int64_t nx, int64_t ny, int64_t nz, const double *src, double *dst,
                     const double *const *W) {
  const int64_t X = nx + 2, Y = ny + 2;
  const int64_t sy = X, sz = X * Y;
#pragma omp parallel for schedule(static)
  for (int64_t z = 1; z <= nz; ++z)
    for (int64_t y = 1; y <= ny; ++y)
      for (int64_t x = 1; x <= nx; ++x) {
        const int64_t p = z * sz + y * sy + x;
        dst[p] = W[0][p] * src[p]
               + W[1][p] * src[p - 1]
               + W[2][p] * src[p + 1]
               + W[3][p] * src[p - sy]
               + W[4][p] * src[p + sy]
               + W[5][p] * src[p - sz]
               + W[6][p] * src[p + sz];
      }
}

/* One step of kind 3 (Fig. 1e): cur = O^t, prev = O^{t-1}; prev <- O^{t+1} in place.
 * s[0] = w0, s[1..4] = w1..w4, s[5] = alpha. */
static void sweep_25w(int64_t nx, int64_t ny, int64_t nz, const double *cur, double *prev,
                      const double *s) {
  const int64_t X = nx + 8, Y = ny + 8;
  const int64_t sy = X, sz = X * Y;
  const double w0 = s[0], w1 = s[1], w2 = s[2], w3 = s[3], w4 = s[4], alpha = s[5];
#pragma omp parallel for schedule(static)
  for (int64_t z = 4; z < nz + 4; ++z)
    for (int64_t y = 4; y < ny + 4; ++y)
      for (int64_t x = 4; x < nx + 4; ++x) {
        const int64_t p = z * sz + y * sy + x;
        const double *c = cur;
        prev[p] = 2.0 * c[p] - prev[p] + alpha * (w0 * c[p]
          + w1 * ((c[p - 1] + c[p + 1]) + (c[p - sy] + c[p + sy]) + (c[p - sz] + c[p + sz]))
          + w2 * ((c[p - 2] + c[p + 2]) + (c[p - 2 * sy] + c[p + 2 * sy]) + (c[p - 2 * sz] + c[p + 2 * sz]))
          + w3 * ((c[p - 3] + c[p + 3]) + (c[p - 3 * sy] + c[p + 3 * sy]) + (c[p - 3 * sz] + c[p + 3 * sz]))
          + w4 * ((c[p - 4] + c[p + 4]) + (c[p - 4 * sy] + c[p + 4 * sy]) + (c[p - 4 * sz] + c[p + 4 * sz])));
      }
}

/* One step of kind 5 (Fig. 1e with alpha_{z,y,x}): as kind 3, alpha read from the field A at the point.
 * s[0] = w0, s[1..4] = w1..w4. */
static void sweep_25wa(int64_t nx, int64_t ny, int64_t nz, const double *cur, double *prev,
                       const double *s, const double *A) {
  const int64_t X = nx + 8, Y = ny + 8;
  const int64_t sy = X, sz = X * Y;
  const double w0 = s[0], w1 = s[1], w2 = s[2], w3 = s[3], w4 = s[4];
#pragma omp parallel for schedule(static)
  for (int64_t z = 4; z < nz + 4; ++z)
    for (int64_t y = 4; y < ny + 4; ++y)
      for (int64_t x = 4; x < nx + 4; ++x) {
        const int64_t p = z * sz + y * sy + x;
        const double *c = cur;
        prev[p] = 2.0 * c[p] - prev[p] + A[p] * (w0 * c[p]
          + w1 * ((c[p - 1] + c[p + 1]) + (c[p - sy] + c[p + sy]) + (c[p - sz] + c[p + sz]))
          + w2 * ((c[p - 2] + c[p + 2]) + (c[p - 2 * sy] + c[p + 2 * sy]) + (c[p - 2 * sz] + c[p + 2 * sz]))
          + w3 * ((c[p - 3] + c[p + 3]) + (c[p - 3 * sy] + c[p + 3 * sy]) + (c[p - 3 * sz] + c[p + 3 * sz]))
          + w4 * ((c[p - 4] + c[p + 4]) + (c[p - 4 * sy] + c[p + 4 * sy]) + (c[p - 4 * sz] + c[p + 4 * sz])));
      }
}

/* One sweep of kind 4 (Fig. 1d).  W[0] centre; W[1+3(r-1)+a] for radius r, axis a = x,y,z. */
static void sweep_25v(int64_t nx, int64_t ny, int64_t nz, const double *src, double *dst,
                      const double *const *W) {
  const int64_t X = nx + 8, Y = ny + 8;
  const int64_t sy = X, sz = X * Y;
#pragma omp parallel for schedule(static)
  for (int64_t z = 4; z < nz + 4; ++z)
    for (int64_t y = 4; y < ny + 4; ++y)
      for (int64_t x = 4; x < nx + 4; ++x) {
        const int64_t p = z * sz + y * sy + x;
        const double *o = src;
        dst[p] = W[0][p] * o[p]
               + W[1][p] * (o[p - 1] + o[p + 1])
               + W[2][p] * (o[p - sy] + o[p + sy])
               + W[3][p] * (o[p - sz] + o[p + sz])
               + W[4][p] * (o[p - 2] + o[p + 2])
               + W[5][p] * (o[p - 2 * sy] + o[p + 2 * sy])
               + W[6][p] * (o[p - 2 * sz] + o[p + 2 * sz])
               + W[7][p] * (o[p - 3] + o[p + 3])
               + W[8][p] * (o[p - 3 * sy] + o[p + 3 * sy])
               + W[9][p] * (o[p - 3 * sz] + o[p + 3 * sz])
               + W[10][p] * (o[p - 4] + o[p + 4])
               + W[11][p] * (o[p - 4 * sy] + o[p + 4 * sy])
               + W[12][p] * (o[p - 4 * sz] + o[p + 4 * sz]);
      }
}

/*
 * Advance (V, U) by T time steps.  V, U: padded arrays of (nz+2R)(ny+2R)(nx+2R) doubles.
 *   Jacobi kinds (1, 2, 4): V holds Omega^0; U's interior is scratch (its ghosts must equal V's).
 *   Wave kinds (3, 5):      V holds Omega^0, U holds Omega^{-1}.
 * On return V = Omega^T and U = Omega^{T-1}.  coef: ncoef padded fields (kinds 2, 4), else unused.
 * scalars: (w1, w2) for kind 1; (w0, w1, w2, w3, w4, alpha) for kind 3; (w0, .., w4) for kind 5,
 * whose coef[0] is the alpha field.
 * nthreads <= 0: OpenMP default.  Returns 0, -1 (bad argument), -2 (no memory).
 */
int oracle_run(int kind, int64_t nx, int64_t ny, int64_t nz, double *V, double *U,
               const double *const *coef, int ncoef, const double *scalars, int nscalars,
               int64_t T, int nthreads) {
  const int R = radius_of(kind);
  if (R < 0 || nx < 1 || ny < 1 || nz < 1 || T < 1 || !V || !U) return OR_EINVAL;
  if (ncoef != ncoef_of(kind) || nscalars != nscal_of(kind)) return OR_EINVAL;
  if (ncoef && !coef) return OR_EINVAL;
  if (nscalars && !scalars) return OR_EINVAL;
#ifdef _OPENMP
  int saved = omp_get_max_threads();
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  double *cur = V, *nxt = U;  /* cur = Omega^t, nxt = Omega^{t-1} (wave) or scratch */
  for (int64_t t = 0; t < T; ++t) {
    switch (kind) {
      case 1: sweep_7c(nx, ny, nz, cur, nxt, scalars[0], scalars[1]); break;
      case 2: sweep_7v(nx, ny, nz, cur, nxt, coef); break;
      case 3: sweep_25w(nx, ny, nz, cur, nxt, scalars); break;
      case 4: sweep_25v(nx, ny, nz, cur, nxt, coef); break;
      case 5: sweep_25wa(nx, ny, nz, cur, nxt, scalars, coef[0]); break;
    }
    double *tmp = cur; cur = nxt; nxt = tmp;  /* swap: t in {0,1} */
  }
  if (cur != V) {  /* odd T: newest level sits in U's storage; exchange contents */
    const int64_t n = (nx + 2 * R) * (ny + 2 * R) * (nz + 2 * R);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) { double a = V[i]; V[i] = U[i]; U[i] = a; }
  }
#ifdef _OPENMP
  omp_set_num_threads(saved);
#endif
  return OR_OK;
}

int oracle_radius(int kind) { return radius_of(kind); }
