// point.cuh -- the per-point update F_kind of PAPER.md Fig. 1, shared by EVERY device
// kernel of the library (naive, z-streaming, temporally blocked, slab edge kernels).
//
// Each function fixes one operation order with explicit round-to-nearest intrinsics (__dadd_rn,
// __dmul_rn, __fma_rn are never re-associated or contracted by nvcc), so all kernel variants
// produce bitwise-identical results regardless of how they gather the neighbours (DESIGN.md §4,
// test G4).  The order differs from the CPU oracle's textual order (the oracle forbids FMA);
// the parity tolerance in tests/ covers that.
#pragma once

namespace st {

enum Kind { K7C = 1, K7V = 2, K25W = 3, K25V = 4, K25WA = 5 };

template <int KIND> struct Traits;
template <> struct Traits<K7C>  { static constexpr int R = 1, NCOEF = 0, NSCAL = 2; static constexpr bool WAVE = false; };
template <> struct Traits<K7V>  { static constexpr int R = 1, NCOEF = 7, NSCAL = 0; static constexpr bool WAVE = false; };
template <> struct Traits<K25W> { static constexpr int R = 4, NCOEF = 0, NSCAL = 6; static constexpr bool WAVE = true; };
template <> struct Traits<K25V> { static constexpr int R = 4, NCOEF = 13, NSCAL = 0; static constexpr bool WAVE = false; };
// Fig. 1e with the domain-sized alpha_{z,y,x} as printed: one coefficient field.
template <> struct Traits<K25WA> { static constexpr int R = 4, NCOEF = 1, NSCAL = 5; static constexpr bool WAVE = true; };

// Neighbour access convention for all functions below: m[a][r-1] / p[a][r-1] are the values at
// distance r in the minus / plus direction of axis a (a = 0 x, 1 y, 2 z); c is the centre.

// Fig. 1b: w1*O + w2*((x-1 + x+1) + (y-1 + y+1) + (z-1 + z+1)).
__device__ __forceinline__ double point_7c(double c, const double (&m)[3][1], const double (&p)[3][1],
                                           double w1, double w2) {
  double s = __dadd_rn(__dadd_rn(__dadd_rn(m[0][0], p[0][0]), __dadd_rn(m[1][0], p[1][0])),
                       __dadd_rn(m[2][0], p[2][0]));
  return __fma_rn(w1, c, __dmul_rn(w2, s));
}

// Fig. 1c: W0*O + W1*O[x-1] + W2*O[x+1] + W3*O[y-1] + W4*O[y+1] + W5*O[z-1] + W6*O[z+1],
// summed as two independent FMA chains (x terms with the centre, y and z terms) added at the end, so
// the dependent-latency depth is 5 instead of 7 (the kernels are latency-bound at low occupancy).
__device__ __forceinline__ double point_7v(double c, const double (&m)[3][1], const double (&p)[3][1],
                                           const double (&W)[7]) {
  double a = __dmul_rn(W[0], c);
  double b = __dmul_rn(W[3], m[1][0]);
  a = __fma_rn(W[1], m[0][0], a);
  b = __fma_rn(W[4], p[1][0], b);
  a = __fma_rn(W[2], p[0][0], a);
  b = __fma_rn(W[5], m[2][0], b);
  b = __fma_rn(W[6], p[2][0], b);
  return __dadd_rn(a, b);
}

// Fig. 1d: W0*O + sum_{r=1..4} [W_{3r-2}(x pair) + W_{3r-1}(y pair) + W_{3r}(z pair)],
// as three independent FMA chains (one per axis; the centre term starts the x chain) added at the end,
// (x + y) + z: dependent-latency depth 6 instead of 13.  The two halves are separate functions because
// the two-level kernel (pipe25.cu) evaluates them at different steps of its z-stream: the x/y half when
// plane z is complete, the z chain one term per plane as planes z+1..z+4 arrive -- same operations.
// x chain (the centre term starts it) and y chain of Fig. 1d; point_25v_xy = x + y
__device__ __forceinline__ double point_25v_x(double c, const double (&m)[3][4], const double (&p)[3][4],
                                              const double (&W)[13]) {
  double a = __fma_rn(W[1], __dadd_rn(m[0][0], p[0][0]), __dmul_rn(W[0], c));
#pragma unroll
  for (int r = 1; r < 4; ++r) a = __fma_rn(W[1 + 3 * r], __dadd_rn(m[0][r], p[0][r]), a);
  return a;
}
__device__ __forceinline__ double point_25v_y(const double (&m)[3][4], const double (&p)[3][4], const double (&W)[13]) {
  double b = __dmul_rn(W[2], __dadd_rn(m[1][0], p[1][0]));
#pragma unroll
  for (int r = 1; r < 4; ++r) b = __fma_rn(W[2 + 3 * r], __dadd_rn(m[1][r], p[1][r]), b);
  return b;
}
__device__ __forceinline__ double point_25v_xy(double c, const double (&m)[3][4], const double (&p)[3][4],
                                               const double (&W)[13]) {
  return __dadd_rn(point_25v_x(c, m, p, W), point_25v_y(m, p, W));
}
// term r (1..4) of the z chain: W_{3r} * (V[z-r] + V[z+r]) (r = 1 starts the chain) added to z
__device__ __forceinline__ double point_25v_zterm(int r, double z, double w, double vm, double vp) {
  return r == 1 ? __dmul_rn(w, __dadd_rn(vm, vp)) : __fma_rn(w, __dadd_rn(vm, vp), z);
}
__device__ __forceinline__ double point_25v(double c, const double (&m)[3][4], const double (&p)[3][4],
                                            const double (&W)[13]) {
  const double xy = point_25v_xy(c, m, p, W);
  double z = 0.0;
#pragma unroll
  for (int r = 1; r <= 4; ++r) z = point_25v_zterm(r, z, W[3 * r], m[2][r - 1], p[2][r - 1]);
  return __dadd_rn(xy, z);
}

// Fig. 1e: 2*O^t - O^{t-1} + alpha*[w0*O^t + sum_r w_r*(x+y+z pairs_r)].
// s = {w0, w1, w2, w3, w4, *}; alpha = the scalar s[5] (kind 3) or the field value at the point
// (kind 5); u = O^{t-1} at the point.  The Laplacian is summed as an x/y chain (the centre term starts
// it) plus a z chain, L = xy + z (round 2: the two-level wave kernel, pipe25.cu, finishes the x/y chain
// of plane z in the step level 1 computes that plane and accumulates the z chain as planes z+1..z+4
// arrive -- the same operations as here).
__device__ __forceinline__ double point_25w_xy(double c, const double (&m)[3][4], const double (&p)[3][4],
                                               const double (&s)[6]) {
  double L = __dmul_rn(s[0], c);
#pragma unroll
  for (int r = 0; r < 4; ++r)
    L = __fma_rn(s[1 + r], __dadd_rn(__dadd_rn(m[0][r], p[0][r]), __dadd_rn(m[1][r], p[1][r])), L);
  return L;
}
// term r (1..4) of the wave's z chain: w_r * (O[z-r] + O[z+r]) (r = 1 starts the chain) added to z
__device__ __forceinline__ double point_25w_zterm(int r, double z, double w, double vm, double vp) {
  return r == 1 ? __dmul_rn(w, __dadd_rn(vm, vp)) : __fma_rn(w, __dadd_rn(vm, vp), z);
}
// the update from the two halves of the Laplacian
__device__ __forceinline__ double point_25w_final(double c, double u, double xy, double z, double alpha) {
  return __fma_rn(alpha, __dadd_rn(xy, z), __dsub_rn(__dmul_rn(2.0, c), u));
}
__device__ __forceinline__ double point_25w(double c, double u, const double (&m)[3][4],
                                            const double (&p)[3][4], const double (&s)[6], double alpha) {
  const double xy = point_25w_xy(c, m, p, s);
  double z = 0.0;
#pragma unroll
  for (int r = 1; r <= 4; ++r) z = point_25w_zterm(r, z, s[r], m[2][r - 1], p[2][r - 1]);
  return point_25w_final(c, u, xy, z, alpha);
}

// Dispatch on the kind; W = the coefficient values at the point (variable kinds), u = O^{t-1} (wave),
// ps = scalar weights.
template <int KIND, int R>
__device__ __forceinline__ double apply_point(double c, double u, const double (&m)[3][R],
                                              const double (&pl)[3][R], const double* W,
                                              const double (&ps)[6]) {
  if constexpr (KIND == K7C) {
    return point_7c(c, m, pl, ps[0], ps[1]);
  } else if constexpr (KIND == K7V) {
    double w[7];
#pragma unroll
    for (int i = 0; i < 7; ++i) w[i] = W[i];
    return point_7v(c, m, pl, w);
  } else if constexpr (KIND == K25V) {
    double w[13];
#pragma unroll
    for (int i = 0; i < 13; ++i) w[i] = W[i];
    return point_25v(c, m, pl, w);
  } else if constexpr (KIND == K25WA) {
    const double s[6] = {ps[0], ps[1], ps[2], ps[3], ps[4], 0.0};
    return point_25w(c, u, m, pl, s, W[0]);
  } else {
    const double s[6] = {ps[0], ps[1], ps[2], ps[3], ps[4], ps[5]};
    return point_25w(c, u, m, pl, s, s[5]);
  }
}

}  // namespace st
