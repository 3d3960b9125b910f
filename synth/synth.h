/*
 * synth.h -- seeded, counter-based synthetic-input generator (reading Q6).
 *
 * This module is shared INPUT SYNTHESIS only: it holds none of the stencil method's arithmetic.
 * The CUDA library (device fill kernel) and the test/bench harness (host fill that feeds the
 * oracle) both include it so that both sides see the same seeded numbers; nothing else is shared.
 *
 * The paper prints no input data (§6 line 974ff: "synthetic" grids only).  BASELINE.json
 * asks for "V0 and boundary uniform[-1,1] from seed", "7 coefficient arrays each uniform[0,1/7)",
 * "13 coefficient arrays uniform[0,1/25)".  The generator is a pure function of
 * (seed, stream, global padded linear index) so that any sub-box (a z-slab on one rank, a cone
 * sample for the oracle) is bitwise identical to the same cells of the global array.
 *
 * Definition (frozen; golden values in tests/golden/synth_golden.txt):
 *   mix(z):   z ^= z >> 30; z *= 0xBF58476D1CE4E5B9; z ^= z >> 27; z *= 0x94D049BB133111EB; z ^= z >> 31
 *   key     = mix(seed ^ (0x9E3779B97F4A7C15 * (stream + 1)))
 *   h       = mix(key + 0xD1B54A32D192ED03 * (idx + 1))          (all arithmetic mod 2^64)
 *   u       = (h >> 11) * 2^-53                                   in [0, 1), exact
 *   U[-1,1) = 2u - 1                                              (exact in binary64)
 *   U[0,c)  = u * c, c = 1.0/7.0 or 1.0/25.0 (one RN multiply)
 *
 * Stream ids: 0 = V^0 and all ghosts; 1 = interior of U^0 for the 25-point wave (Omega^{-1});
 *             2 + i = coefficient field W_i (Fig. 1c / 1d numbering).
 */
#ifndef SYNTH_H
#define SYNTH_H

#include <stdint.h>

#if defined(__CUDACC__)
#define SYNTH_HD __host__ __device__ __forceinline__
#else
#define SYNTH_HD static inline
#endif

#define SYNTH_STREAM_V 0
#define SYNTH_STREAM_U 1
#define SYNTH_STREAM_W(i) (2 + (i))

SYNTH_HD uint64_t synth_mix(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

SYNTH_HD uint64_t synth_key(uint64_t seed, int stream) {
  return synth_mix(seed ^ (0x9E3779B97F4A7C15ull * (uint64_t)(stream + 1)));
}

SYNTH_HD double synth_unit(uint64_t key, uint64_t idx) {
  uint64_t h = synth_mix(key + 0xD1B54A32D192ED03ull * (idx + 1ull));
  return (double)(h >> 11) * 0x1.0p-53;
}

/* U[-1,1): 2u - 1, exact. */
SYNTH_HD double synth_sym(uint64_t key, uint64_t idx) { return 2.0 * synth_unit(key, idx) - 1.0; }

/* U[0,c): u * c with c passed in (1.0/7.0 or 1.0/25.0). */
SYNTH_HD double synth_scaled(uint64_t key, uint64_t idx, double c) { return synth_unit(key, idx) * c; }

#endif
