// pipe25.cu -- the 25-point variable-coefficient stencil (Fig. 1d) with TWO fused
// time levels per launch (b_t = 2): the wavefront temporal blocking of P:569-602 for the kind whose 13
// coefficient fields made it capacity-bound on the paper's CPU (1WD needs 93 MiB of cache).
//
// Why a kernel of its own: in the generic pipe kernel, level k reads the coefficients of
// plane z at step z + k*R, so a fused block must keep each coefficient plane on chip for (b_t - 1)*R = 4
// steps: 5 planes x 13 fields x the level-1 extent >= 320 KB per CTA -- more than shared memory.  Here the
// update of a level-2 cell is split the way its arithmetic already is (point.cuh: point_25v_x / _y /
// _zterm):
//   * the x/y half (centre + 8 x-pair + 8 y-pair terms, 9 coefficients) needs level 1's plane z only; it
//     is computed in the SAME step that level 1 computes plane z, with the coefficient plane still in the
//     shared-memory ring -- so every coefficient plane crosses HBM once per block and leaves shared memory
//     after one step;
//   * the z chain's term r needs level-1 plane z + r, computed r steps later: it is accumulated one term
//     per step.  What a cell must carry between steps -- its pending x/y partial sums (4 planes), z chains
//     (3 planes) and the z-coefficients they still need (10 values) -- lives in TENSOR MEMORY (TMEM,
//     tcgen05.ld/st), as do both z-rings (level-0 and level-1 values of the last planes).  Registers hold
//     only the current step's operands.
// The operations are exactly point_25v's (same FMA chains, same final (x + y) + z adds), so the results
// are bitwise equal to every other variant (test G4).
//
// Per step s of a work item's z-stream (one CTA per SM, persistent; a producer warp + NW consumer warps):
//   producer: TMA loads into one ring slot (one full mbarrier): box A = plane s of Omega^t over the
//     level-1 extent E1 (TX x TY; its centre column is the z-ring's newest entry), box B = plane s-R with
//     an R-wide halo (x/y neighbours of level 1; its centre is the ring's middle entry), box C = the 13
//     coefficient fields of plane s-R over E1 (one 4-D box); and an L2 prefetch of step s+2's A and C
//     boxes (the ring is 2 slots deep);
//   level 1 (all consumer warps, 2x2 cells per thread): plane q = s-R of level 1 over E1 (full point_25v),
//     written to a shared plane;  named barrier;
//   level 2 (the warps whose rows hold output cells): x/y half of plane q, the z-chain terms of planes
//     q-1..q-4, and the finished output plane q-4 = s-2R, streamed to HBM.
// The output tile is (TX - 2R) x (TY - 2R) (overlapped tiles shrinking by R per level, as in pipe.cu).
//
// CLU > 1 (the GPU analog of the paper's thread groups sharing one cache block,
// P:735-764): a thread-block cluster of CLU CTAs stacked in y shares one TX x (CLU*TY) tile.  Each CTA
// computes level 1 on its own TY rows only; the R level-1 rows a CTA's level 2 needs from a neighbour are
// pushed to it through distributed shared memory (cp.async.bulk.shared::cluster, completion on the
// receiver's mbarrier), so the trapezoid shrinks only at the cluster's outer rows: level-1 work and
// coefficient-box traffic per output cell drop by (CLU*TY - 2R)/(CLU*(TY - 2R)).  The rows cross SMs
// while the next step runs: the warp next to a cluster neighbour ("boundary warp") finishes the y chain of
// its cells one step late, from the rows received meanwhile (x chain and the y-coefficients wait in
// shared memory for that step) -- no warp ever waits on the neighbour's current step.
#include "kernels.cuh"
#include "point.cuh"
#include "sm100.cuh"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

namespace st {

template <int KIND, int TX, int TY, int D, int CLU, int SKEW>
struct P25Cfg {
  // KIND = K25V (Fig. 1d, 13 coefficient fields) or K25W (Fig. 1e with a scalar alpha: box C carries
  // Omega^{t-1} instead of coefficients, and the carried state has no z-coefficients)
  static constexpr bool WAVE = KIND == K25W;
  static constexpr int R = 4, NC = WAVE ? 0 : 13, CX = 2, CY = 2, NCELL = CX * CY;
  static constexpr int CF = WAVE ? 1 : NC;  // fields of box C
  static constexpr int LPR = TX / CX;             // threads per block row
  static constexpr int NCONS = LPR * (TY / CY);   // consumer threads
  static constexpr int NW = NCONS / 32;           // consumer warps
  static constexpr int THREADS = NCONS + 32;      // + the producer warp
  // SKEW (parallelogram tiles in y): level 2 runs R rows below level 1 instead of
  // shrinking, so y-neighbouring tiles never compute the same cell; the 2R level-1 rows below the tile
  // come from the tile underneath through global memory (box I), and box C reaches R rows lower (CR)
  static constexpr int CR = SKEW ? R : 0;
  static constexpr int OX = TX - 2 * R;                     // output columns of a tile
  static constexpr int OYP = SKEW ? TY : CLU * TY - 2 * R;  // output rows of a (cluster) tile
  static constexpr int FX = TX + 2 * R, FY = TY + 2 * R;  // box B (level-1 footprint)
  static constexpr int AEL = TX * TY, BEL = FX * FY, CFIELD = TX * (TY + CR), CEL = CF * CFIELD;
  static constexpr int IEL = SKEW ? 2 * R * TX : 0;       // box I: level-1 rows -2R..-1 of plane q
  static constexpr int BOFF = (AEL + 15) / 16 * 16, COFF = BOFF + (BEL + 15) / 16 * 16;
  static constexpr int IOFF = COFF + (CEL + 15) / 16 * 16;
  static constexpr int SLOT = IOFF + (IEL + 15) / 16 * 16;  // doubles per ring slot (128-byte aligned parts)
  static constexpr int PEL = TX * TY;                       // one shared level-1 plane
  static constexpr int NPB = SKEW ? 2 : 3;                  // level-1 planes kept (boundary warps read q-1)
  static constexpr int RXEL = R * TX;                       // one pushed boundary strip (R rows)
  static constexpr int NRX = CLU > 1 ? 4 : 0;               // receive slots per side
  static constexpr int STASH = CLU > 1 ? 2 * 32 * NCELL * 5 : 0;  // boundary warps' carried x chain + Wy
  // CLU = 2: the warp without level-2 rows ("helper") finishes the boundary warp's y chains; it hands the
  // x/y halves back through a mailbox (double-buffered by step parity; the stash is too)
  static constexpr bool HELPER = CLU == 2;
  static constexpr int MBOX = HELPER ? 2 * 32 * NCELL : 0;
  static constexpr int WROWS = 32 / LPR * CY;               // E1 rows per consumer warp
  static constexpr uint32_t TX_BYTES_A = AEL * 8, TX_BYTES_B = BEL * 8, TX_BYTES_C = CEL * 8, RX_BYTES = RXEL * 8,
                            TX_BYTES_I = IEL * 8;
  static constexpr int XROW0 = TY - 2 * R;  // SKEW: the tile's level-1 rows the tile above imports
  static constexpr size_t SMEM = 8 * ((size_t)D * SLOT + (size_t)NPB * PEL + 2 * (size_t)NRX * RXEL + STASH + MBOX) +
                                 8 * (2 * D + 8 + 2 * NRX + 8) + 4 * 8 + 128;
  static_assert(TX % 16 == 0 && TY % CY == 0 && NCONS % 32 == 0 && 32 % LPR == 0, "thread layout");
  static_assert(TY % WROWS == 0 && WROWS == R, "one warp = R rows (the pushed strip)");
  static_assert(OX > 0 && TY > 2 * R && (OX & 3) == 0, "output tile (whole 32-byte sectors per row)");
  static_assert(CLU == 1 || CLU == 2 || CLU == 4, "clusters of 1, 2 or 4 CTAs along y");
  static_assert(!WAVE || CLU == 1, "wave: single-CTA tiles");
  static_assert(!SKEW || (CLU == 1 && !WAVE && TY >= 4 * R && (2 * R) % WROWS == 0),
                "skewed tiles: single CTA, 25v; the exporting rows are whole warps");
  static_assert(KIND == K25V || KIND == K25W, "25-point kinds");
  // TMEM (512 columns x 128 lanes; warp w reaches lanes 32*(w%4)..): warp w uses columns
  // [256*(w/4), +256): at most two warps per lane quadrant.
  static_assert(NW <= 8, "TMEM quadrants");
  static_assert(SMEM <= 227 * 1024, "shared memory");
  static_assert(SMEM > 116 * 1024, "one CTA per SM (the CTA allocates all 512 TMEM columns)");
  static_assert(FX <= 256 && FY <= 256 && TX <= 256, "TMA box dimension limit");
};

// TMEM column map of a consumer thread (32-bit columns of its lane, relative to its warp's 256)
constexpr uint32_t kColV1 = 0;    // level-1 z-ring: 2 parity regions x 4 cells x 4 planes   [0, 64)
constexpr uint32_t kColS1 = 64;   // carried state, 16 doubles per cell                       [64, 192)
constexpr uint32_t kColV0 = 192;  // level-0 z-ring: 2 rows x 2 cells x 7 planes, row j at 192 + 28j
constexpr uint32_t kColS2 = 248;  // carried state, 1 double per cell                         [248, 256)

__device__ __forceinline__ double dbl(uint32_t lo, uint32_t hi) { return __hiloint2double((int)hi, (int)lo); }
__device__ __forceinline__ void put(uint32_t* w, double v) {
  w[0] = (uint32_t)__double2loint(v);
  w[1] = (uint32_t)__double2hiint(v);
}
// one row's level-0 ring (28 columns) as aligned x16 / x8 / x4 pieces
template <int J>
__device__ __forceinline__ void v0ring_ld(uint32_t t, uint32_t (&w)[28]) {
  uint32_t a[16], b[8], c[4];
  if constexpr (J == 0) {
    tmem_ld16(t + kColV0, a); tmem_ld8(t + kColV0 + 16, b); tmem_ld4(t + kColV0 + 24, c);
  } else {
    tmem_ld4(t + kColV0 + 28, c); tmem_ld16(t + kColV0 + 32, a); tmem_ld8(t + kColV0 + 48, b);
  }
  tmem_wait_ld();
  if constexpr (J == 0) {
#pragma unroll
    for (int i = 0; i < 16; ++i) w[i] = a[i];
#pragma unroll
    for (int i = 0; i < 8; ++i) w[16 + i] = b[i];
#pragma unroll
    for (int i = 0; i < 4; ++i) w[24 + i] = c[i];
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = c[i];
#pragma unroll
    for (int i = 0; i < 16; ++i) w[4 + i] = a[i];
#pragma unroll
    for (int i = 0; i < 8; ++i) w[20 + i] = b[i];
  }
}
template <int J>
__device__ __forceinline__ void v0ring_st(uint32_t t, const uint32_t (&w)[28]) {
  uint32_t a[16], b[8], c[4];
  if constexpr (J == 0) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = w[i];
#pragma unroll
    for (int i = 0; i < 8; ++i) b[i] = w[16 + i];
#pragma unroll
    for (int i = 0; i < 4; ++i) c[i] = w[24 + i];
    tmem_st16(t + kColV0, a); tmem_st8(t + kColV0 + 16, b); tmem_st4(t + kColV0 + 24, c);
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) c[i] = w[i];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = w[4 + i];
#pragma unroll
    for (int i = 0; i < 8; ++i) b[i] = w[20 + i];
    tmem_st4(t + kColV0 + 28, c); tmem_st16(t + kColV0 + 32, a); tmem_st8(t + kColV0 + 48, b);
  }
}

template <int KIND, int TX, int TY, int D, int CLU, int SKEW>
__global__ void __launch_bounds__(P25Cfg<KIND, TX, TY, D, CLU, SKEW>::THREADS, 1)
    pipe25_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                  const __grid_constant__ CUtensorMap mapC, const __grid_constant__ CUtensorMap mapI,
                  const __grid_constant__ CUtensorMap mapS, const KParams p, int ntx, int nty, int items) {
  using C = P25Cfg<KIND, TX, TY, D, CLU, SKEW>;
  constexpr int R = C::R, NC = C::NC, NCONS = C::NCONS, FX = C::FX, CX = C::CX, CY = C::CY, NW = C::NW;
  constexpr bool WAVE = C::WAVE;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw);
  double* sP = ring + (size_t)D * C::SLOT;
  double* rxTop = sP + (size_t)C::NPB * C::PEL;      // rows -R..-1 (the CTA above, rank - 1), per slot
  double* rxBot = rxTop + (size_t)C::NRX * C::RXEL;  // rows TY..TY+R-1 (the CTA below, rank + 1)
  double* stash = rxBot + (size_t)C::NRX * C::RXEL;  // [boundary warp top/bottom | step parity][lane][cell][5]
  double* mbox = stash + C::STASH;                    // HELPER: [step parity][lane][cell]
  uint64_t* full = reinterpret_cast<uint64_t*>(mbox + C::MBOX);
  uint64_t* empty = full + D;
  uint64_t* itemFull = empty + D;
  uint64_t* itemEmpty = itemFull + 4;
  uint64_t* rxbTop = itemEmpty + 4;
  uint64_t* rxbBot = rxbTop + C::NRX;
  uint64_t* cfull = rxbBot + C::NRX;  // cluster work-item queue (rank 0 -> ranks 1..CLU-1)
  uint64_t* cempty = cfull + 4;
  volatile int* itemq = reinterpret_cast<volatile int*>(cempty + 4);
  volatile int* cid = itemq + 4;

  uint32_t crank = 0;
  if constexpr (CLU > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < D; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], NW); }
    for (int i = 0; i < 4; ++i) { mbar_init(&itemFull[i], 1); mbar_init(&itemEmpty[i], NW); }
    for (int i = 0; i < C::NRX; ++i) { mbar_init(&rxbTop[i], 1); mbar_init(&rxbBot[i], 1); }
    for (int i = 0; i < 4; ++i) { mbar_init(&cfull[i], 1); mbar_init(&cempty[i], CLU > 1 ? CLU - 1 : 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __shared__ uint32_t tmem_base;
  if (tid < 32) {  // consumer warp 0 allocates all 512 columns (one CTA per SM)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if constexpr (CLU > 1) cluster_sync_all();  // every CTA's barriers exist before any remote arrive / copy

  if (tid >= NCONS) {
    // ---------------------------------------------------------------- producer warp
    if (tid == NCONS) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mapC) : "memory");
      if constexpr (SKEW) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mapI) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mapS) : "memory");
      }
      uint32_t iv = 0;
      const uint64_t polA = l2_policy(p.l2h & 3), polB = l2_policy((p.l2h >> 2) & 3),
                     polC = l2_policy((p.l2h >> 4) & 3);
      for (uint32_t n = 0;; ++n) {
        const uint32_t qs = n & 3;
        mbar_wait(&itemEmpty[qs], ((n >> 2) & 1) ^ 1);
        int g;
        if (CLU > 1 && p.lockstep) {
          // static rounds of whole clusters: every CTA of cluster k takes item n * (G / CLU) + k
          g = (int)(n * (gridDim.x / CLU) + blockIdx.x / CLU);
          if (g >= items) g = -1;
        } else if constexpr (CLU > 1) {
          // every CTA of a cluster takes the same items: rank 0 draws from the global counter and passes
          // the id to the others through a 4-entry queue in their shared memory
          if (crank == 0) {
            mbar_wait(&cempty[qs], ((n >> 2) & 1) ^ 1);
            g = (int)atomicAdd(p.sched, 1u);
            if (g >= items) g = -1;
            for (uint32_t k = 1; k < (uint32_t)CLU; ++k) {
              asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(dsmem_addr((const void*)&cid[qs], k)), "r"(g)
                           : "memory");
              mbar_arrive_remote(dsmem_addr(&cfull[qs], k));
            }
          } else {
            mbar_wait_cluster(&cfull[qs], (n >> 2) & 1);
            g = cid[qs];
            mbar_arrive_remote(dsmem_addr(&cempty[qs], 0u));
          }
        } else if (p.lockstep) {
          // static rounds: CTA c takes item n * G + c; the tile order (decode, tblk_*) makes a round a
          // compact patch of tiles, and the rounds start together (below), so overlapping tiles stream the
          // same planes at the same time and their shared halo boxes hit L2
          g = (int)(n * gridDim.x + blockIdx.x);
          if (g >= items) g = -1;
        } else {
          g = (int)atomicAdd(p.sched, 1u);
          if (g >= items) g = -1;
        }
        itemq[qs] = g;
        mbar_arrive(&itemFull[qs]);  // release: the id is visible to the consumers' acquire
        if (g < 0) break;
        const bool skip = (p.dbg & 8) && g == 0;  // fault injection: item 0 never loaded (nor computed)
        Item it = decode<R, 1, C::OX, C::OYP>(g, ntx, nty, p);
        it.gy0 += (int)crank * TY + C::CR;  // SKEW: level-1 rows [R + ty*TY, +TY), level 2 R rows lower
        // SKEW: the flags of this tile (two exporting warps) and of the tile underneath
        const long long fme = 2ll * (((long long)it.zc * nty + it.ty) * ntx + it.tx);
        const long long fbelow = fme - 2ll * ntx;
        if constexpr (SKEW) {
          if (skip) {  // fault injection: the skipped item still releases the tile above (wrong planes, no hang)
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p.xflag + fme), "r"(p.xbase + 0xFFFFu) : "memory");
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p.xflag + fme + 1), "r"(p.xbase + 0xFFFFu) : "memory");
          }
        }
        const int xb = ((it.gx0 - R + p.xoff) & ~1) - (p.xoff & ~1);  // box B (footprint)
        const int xa = ((it.gx0 + p.xoff) & ~1) - (p.xoff & ~1);      // boxes A, C (level-1 extent)
        for (int s = it.s_begin; s <= it.s_end && !skip; ++s, ++iv) {
          const uint32_t sl = iv % D;
          mbar_wait(&empty[sl], ((iv / D) & 1) ^ 1);
          // level 1 computes plane q = s - R this step only once its z-neighbours are in the ring (then it
          // needs the coefficients); box B's centre enters the z-ring for every plane of the stream
          const int q = s - R;
          const bool needB = q >= it.s_begin;
          const bool need1 = needB && (it.s_begin == 0 || q >= it.s_begin + R);
          // SKEW: level 1's rows -2R..-1 of plane q, from the tile underneath (or the ghost rows, bottom tile)
          // (only planes whose level 1 is real: adjacent z-chunks write the same exchange planes, and a
          // chunk's fill planes hold its input instead)
          const bool needI = SKEW && need1 && q >= 0 && q < p.zl;
          mbar_expect_tx(&full[sl], C::TX_BYTES_A + (needB ? C::TX_BYTES_B : 0u) + (need1 ? C::TX_BYTES_C : 0u) +
                                        (needI ? C::TX_BYTES_I : 0u));
          double* slot = ring + (size_t)sl * C::SLOT;
          if constexpr (SKEW) {
            if (needI) {
              if (it.ty > 0 && !(p.dbg & 64)) {  // (STENCIL_DBG bit 64, experiment: no wait, wrong results)
                // wait until both exporting warps of the tile underneath stored plane q (bounded: a lost
                // producer makes wrong planes, not a hung GPU)
                const unsigned int want = p.xbase + (unsigned int)q + 1u;
                for (int w = 0; w < 2; ++w) {
                  unsigned int v;
                  for (long long spin = 0; spin < (1ll << 26); ++spin) {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.xflag + fbelow + w) : "memory");
                    if ((int)(v - want) >= 0) break;
                    __nanosleep(64);
                  }
                }
                // the generic-proxy stores just observed must be visible to the TMA (async proxy) load
                asm volatile("fence.proxy.async.global;" ::: "memory");
                tma_load_3d(slot + C::IOFF, &mapI, &full[sl], xa, it.gy0 - 2 * R, q);
              } else {
                tma_load_3d(slot + C::IOFF, &mapS, &full[sl], xa, it.gy0 - 2 * R, q);  // ghost rows of plane q
              }
            }
          }
          // (STENCIL_DBG bit 16, a DRAM-traffic diagnostic with wrong results: box B re-reads plane s)
          const int qb = (p.dbg & 16) ? s : q;
          if (p.l2h == 0) {
            tma_load_3d(slot, &mapA, &full[sl], xa, it.gy0, s);
            if (needB) tma_load_3d(slot + C::BOFF, &mapB, &full[sl], xb, it.gy0 - R, qb);
            if (need1) {
              if constexpr (WAVE) tma_load_3d(slot + C::COFF, &mapC, &full[sl], xa, it.gy0, q);  // Omega^{t-1}
              else tma_load_4d(slot + C::COFF, &mapC, &full[sl], xa, it.gy0 - C::CR, q, 0);
            }
          } else {  // experiment: L2 eviction priorities per box
            tma_load_3d_hint(slot, &mapA, &full[sl], xa, it.gy0, s, polA);
            if (needB) tma_load_3d_hint(slot + C::BOFF, &mapB, &full[sl], xb, it.gy0 - R, qb, polB);
            if (need1) {
              if constexpr (WAVE) tma_load_3d_hint(slot + C::COFF, &mapC, &full[sl], xa, it.gy0, q, polC);
              else tma_load_4d_hint(slot + C::COFF, &mapC, &full[sl], xa, it.gy0 - C::CR, q, 0, polC);
            }
          }
          if (p.pfd > 0 && s + p.pfd <= it.s_end) {  // warm L2 for the loads pfd steps ahead (beyond the ring)
            tma_prefetch_3d(&mapA, xa, it.gy0, s + p.pfd);
            if (q + p.pfd >= 0) {
              if constexpr (WAVE) tma_prefetch_3d(&mapC, xa, it.gy0, q + p.pfd);
              else tma_prefetch_4d(&mapC, xa, it.gy0, q + p.pfd, 0);
            }
          }
        }
        if (p.lockstep) {
          // round n issued: wait until every CTA with an item in round n has issued its loads too (all CTAs
          // are resident, one per SM, so this grid-wide wait cannot deadlock)
          const unsigned int want =
              (unsigned int)(CLU * min((long long)(n + 1) * (gridDim.x / CLU), (long long)items));
          __threadfence();
          atomicAdd(p.sched, 1u);
          unsigned int v;
          for (;;) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.sched) : "memory");
            if (v >= want) break;
            __nanosleep(128);
          }
        }
      }
      // every CTA has drawn its terminating id before the last one gets here: reset for the next launch
      __threadfence();
      if ((CLU == 1 || crank == 0) && atomicAdd(p.sched + 1, 1u) == gridDim.x / CLU - 1) {
        p.sched[0] = 0;
        p.sched[1] = 0;
        __threadfence();
      }
    }
    if constexpr (CLU > 1) cluster_sync_all();  // no CTA leaves while a neighbour may still push into it
    return;
  }

  // ---------------------------------------------------------------- consumers
  const int warp = tid >> 5, lane = tid & 31;
  const int x0 = (tid % C::LPR) * CX;   // first E1 column of this thread's 2x2 block
  const int ly0 = (tid / C::LPR) * CY;  // first E1 row
  // level-2 rows of this CTA (the trapezoid shrinks by R only at the cluster's outer rows)
  const int ylo = SKEW ? -R : (crank == 0 ? R : 0), yhi = SKEW ? TY - R : (crank == (uint32_t)CLU - 1 ? TY - R : TY);
  const int wr0 = warp * C::WROWS;  // the warp's first row (warp-uniform)
  // level 2 runs on the warps whose rows hold output cells, on the same 2x2 blocks as level 1 (an
  // output-only mapping measured no faster)
  // (SKEW: every warp; a thread's level-2 cells sit R rows below its level-1 cells)
  const bool lvl2 = SKEW || (wr0 + C::WROWS > ylo && wr0 < yhi);
  const int l2x = x0, l2y = ly0 - C::CR;
  const bool exporter = SKEW && ly0 >= C::XROW0;  // SKEW: level-1 rows the tile above imports
  const bool topB = CLU > 1 && warp == 0 && crank > 0;                        // needs rows of rank - 1
  const bool botB = CLU > 1 && warp == NW - 1 && crank < (uint32_t)CLU - 1;  // needs rows of rank + 1
  const bool bnd = topB || botB;
  // HELPER (pairs): rank 0's warp 0 / rank 1's last warp has no level-2 rows; it computes the delayed y
  // chains of the boundary warp (rank 0's last warp / rank 1's warp 0) -- same lanes, same columns
  const bool helper = C::HELPER && !lvl2;
  const int bwarp = crank == 0 ? NW - 1 : 0;                          // the boundary warp a helper serves
  const int hly0 = ((bwarp * 32 + lane) / C::LPR) * CY;               // its lane's first row
  const uint32_t tq = tmem_base + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 256);
  double* myst = stash + (size_t)((topB ? 0 : 1) * 32 + lane) * C::NCELL * 5;  // boundary warps (CLU = 4)
  const double ps[6] = {p.s[0], p.s[1], p.s[2], p.s[3], p.s[4], p.s[5]};  // the wave's w0, w1..w4, alpha
  uint32_t iv = 0;

  for (uint32_t n = 0;; ++n) {
    const uint32_t qs = n & 3;
    mbar_wait(&itemFull[qs], (n >> 2) & 1);
    const int g = itemq[qs];
    __syncwarp();
    if (lane == 0) mbar_arrive(&itemEmpty[qs]);
    if (g < 0) break;
    if ((p.dbg & 8) && g == 0) continue;  // fault injection: work item 0 never computed
    Item it = decode<R, 1, C::OX, C::OYP>(g, ntx, nty, p);
    it.gy0 += (int)crank * TY + C::CR;
    const long long fme = 2ll * (((long long)it.zc * nty + it.ty) * ntx + it.tx);
    bool act1[CY][CX], outc[CY][CX];
    long long col[CY];
#pragma unroll
    for (int j = 0; j < CY; ++j) {
      const int ly = ly0 + j, gy = it.gy0 + ly;
#pragma unroll
      for (int i = 0; i < CX; ++i) {
        const int gx = it.gx0 + x0 + i;
        act1[j][i] = gx >= R && gx < p.nx + R && gy >= R && gy < p.ny + R;
      }
      // level-2 cells: stored output columns / rows of the tile, interior of the grid
      const int ly2 = l2y + j, gy2 = it.gy0 + ly2;
      col[j] = (long long)gy2 * p.pitch + it.gx0 + l2x;
#pragma unroll
      for (int i = 0; i < CX; ++i) {
        const int lx = l2x + i, gx = it.gx0 + lx;
        outc[j][i] = gx >= R && gx < p.nx + R && gy2 >= R && gy2 < p.ny + R && lx >= R && lx < TX - R &&
                     ly2 >= ylo && ly2 < yhi;
      }
    }

    unsigned int xpend = 0;  // SKEW exporters: planes stored but not yet released (+1)
    for (int s = it.s_begin; s <= it.s_end; ++s, ++iv) {
      const uint32_t sl = iv % D;
      const double* slot = ring + (size_t)sl * C::SLOT;
      if constexpr (SKEW) {
        // release the exported planes every xg steps, at the start of a step: by now the stores of the
        // last step have long completed, so the fence costs little (every lane fences its own stores,
        // then lane 0 publishes the warp's flag)
        if (exporter && xpend && (int)(xpend % (unsigned int)p.xg) == 0 && !(p.dbg & 256)) {
          if (!(p.dbg & 128)) __threadfence();  // (STENCIL_DBG bit 128, experiment: no fence)
          __syncwarp();
          if (lane == 0)
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p.xflag + fme + (warp - C::XROW0 / C::WROWS)),
                         "r"(p.xbase + xpend)
                         : "memory");
          xpend = 0;
        }
      }
      mbar_wait(&full[sl], (iv / D) & 1);

      // ---------------- level 1: plane q = s - R over the level-1 extent (all consumer warps)
      const int q = s - R;
      const bool zv1 = !(p.dbg & 1) && q >= p.zi0 && q < p.zi1 && (it.s_begin == 0 || q >= it.s_begin + R);
      const double* Bb = slot + C::BOFF + R * FX + R;  // Bb[y * FX + x] = E1 cell (x, y) of plane q
      const double* Cs = slot + C::COFF;               // Cs[f * CFIELD + y * TX + x]: field f at E1 (x, y)
      double v1[CY][CX];
      double v0c4[CY][CX];  // the wave: level 0 of plane q - R, the Omega^t of level 2's output plane
      {
        double ys[CY + 2 * R][CX];
#pragma unroll
        for (int r = 0; r < CY + 2 * R; ++r) lds_row<CX, true>(Bb + (ly0 - R + r) * FX + x0, ys[r]);
#pragma unroll
        for (int j = 0; j < CY; ++j) {
          // level-0 z-ring of row j's two cells (TMEM): planes s-8+k, k in {0..3, 5..7} (7 entries);
          // k = 4 is plane q itself (the centre of box B), k = 8 plane s (box A)
          uint32_t zr[28];
          if (j == 0) v0ring_ld<0>(tq, zr); else v0ring_ld<1>(tq, zr);
          double vnew[CX];
          lds_row<CX, true>(slot + (ly0 + j) * TX + x0, vnew);
          double xr[R + CX + R];
          lds_row<R, true>(Bb + (ly0 + j) * FX + x0 - R, xr);
          lds_row<R, true>(Bb + (ly0 + j) * FX + x0 + CX, xr + R + CX);
#pragma unroll
          for (int i = 0; i < CX; ++i) xr[R + i] = ys[R + j][i];
          double Wr[NC > 0 ? NC : 1][CX];
#pragma unroll
          for (int f = 0; f < NC; ++f) lds_row<CX, true>(Cs + f * C::CFIELD + (ly0 + j + C::CR) * TX + x0, Wr[f]);
          double urow[CX];  // the wave: Omega^{t-1} of plane q (box C)
          if constexpr (WAVE) lds_row<CX, true>(Cs + (ly0 + j) * TX + x0, urow);
          auto V0 = [&](int k, int i) -> double {  // plane s - 8 + k of cell (j, i)
            if (k == 8) return vnew[i];
            if (k == R) return ys[R + j][i];
            const int e = k < R ? k : k - 1;
            return dbl(zr[14 * i + 2 * e], zr[14 * i + 2 * e + 1]);
          };
          uint32_t zn[28];
#pragma unroll
          for (int i = 0; i < CX; ++i) {
            double m[3][R], pl[3][R], W[NC > 0 ? NC : 1];
#pragma unroll
            for (int r = 1; r <= R; ++r) {
              m[0][r - 1] = xr[R + i - r];
              pl[0][r - 1] = xr[R + i + r];
              m[1][r - 1] = ys[R + j - r][i];
              pl[1][r - 1] = ys[R + j + r][i];
              m[2][r - 1] = V0(R - r, i);
              pl[2][r - 1] = V0(R + r, i);
            }
#pragma unroll
            for (int f = 0; f < NC; ++f) W[f] = Wr[f][i];
            const double c = V0(R, i);
            double v;
            if constexpr (WAVE) {
              v = point_25w(c, urow[i], m, pl, ps, ps[5]);
              v0c4[j][i] = V0(0, i);
            } else {
              v = point_25v(c, m, pl, W);
            }
            // ghosts, cells outside the grid and planes not computed at level 1 keep their input value
            v1[j][i] = (zv1 && act1[j][i]) ? v : c;
            // the ring moves on a plane: next step's entries are this step's k = 1..3, 4 (box B), 6, 7, 8
#pragma unroll
            for (int e = 0; e < 7; ++e) put(zn + 14 * i + 2 * e, V0(e < R ? e + 1 : e + 2, i));
          }
          if (j == 0) v0ring_st<0>(tq, zn); else v0ring_st<1>(tq, zn);
        }
      }
      double* P = sP + (size_t)(iv % C::NPB) * C::PEL;  // rotates with the CTA's step counter (pipe.cu)
#pragma unroll
      for (int j = 0; j < CY; ++j) sts_row<CX, true>(P + (ly0 + j) * TX + x0, v1[j]);
      if constexpr (SKEW) {
        // hand the top 2R level-1 rows of plane q to the tile above (plain stores: they should stay in L2
        // for its import a few steps later), then release them warp by warp -- only planes whose level 1
        // is computed (not a z-chunk's fill planes: the neighbouring chunk writes the same exchange plane)
        if (exporter && q >= it.s_begin && (it.s_begin == 0 || q >= it.s_begin + R) && q >= 0 && q < p.zl) {
#pragma unroll
          for (int j = 0; j < CY; ++j) {
            const int gy = it.gy0 + ly0 + j;
            if (gy >= p.ny + 2 * R) continue;
            double* dx = p.xch + (long long)q * p.plane + (long long)gy * p.pitch + it.gx0 + x0;
#pragma unroll
            for (int i = 0; i < CX; ++i) {
              const int gx = it.gx0 + x0 + i;
              if (gx >= 0 && gx < p.nx + 2 * R) dx[i] = v1[j][i];
            }
          }
          xpend = (unsigned int)q + 1u;  // released at the start of a later step (below), off this step's path
        }
      }
      if constexpr (CLU > 1) {
        // the push of two steps ago has read its rows before this barrier releases their rewrite (the
        // plane is rewritten NPB = 3 steps after it was pushed)
        if (bnd && lane == 0) bulk_wait_read<1>();
      }
      if (!(p.dbg & 2)) named_sync(1, NCONS);

      if constexpr (CLU > 1) {
        // push this CTA's outer R level-1 rows of plane q to the cluster neighbours, which finish their
        // boundary rows' y chains with them next step; arm this step's receive slot
        if (bnd && lane == 0) {
          const uint32_t k = iv % C::NRX;
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          if (topB) {
            mbar_expect_tx(&rxbTop[k], C::RX_BYTES);
            bulk_copy_to_peer(dsmem_addr(rxBot + (size_t)k * C::RXEL, crank - 1), P, C::RX_BYTES,
                              dsmem_addr(&rxbBot[k], crank - 1));
          } else {
            mbar_expect_tx(&rxbBot[k], C::RX_BYTES);
            bulk_copy_to_peer(dsmem_addr(rxTop + (size_t)k * C::RXEL, crank + 1), P + (TY - R) * TX, C::RX_BYTES,
                              dsmem_addr(&rxbTop[k], crank + 1));
          }
        }
      }

      // ---------------- level 2: x/y half of plane q, z-chain terms of planes q-1..q-4, output plane q-4
      if (lvl2) {
        const uint32_t colR = kColV1 + (uint32_t)(q & 1) * 32;  // level-1 z-ring of q's parity, per cell:
        uint32_t s2[8], s2n[8];                                  // V1(q-2), V1(q-4), V1(q-6), V1(q-8)
        if constexpr (!WAVE) tmem_ld8(tq + kColS2, s2);  // Z(q-2) of the 4 cells
        double ys[CY + 2 * R][CX];
        double Pprev[CY][CX];  // boundary warps: P(q-1), completed this step
        if (!bnd) {
#pragma unroll
          for (int r = 0; r < CY + 2 * R; ++r) {
            if constexpr (SKEW) {  // rows below the tile: box I (level-1 rows -2R..-1 of plane q)
              const int row = l2y - R + r;
              lds_row<CX, true>((row < 0 ? slot + C::IOFF + (row + 2 * R) * TX : P + row * TX) + l2x, ys[r]);
            } else {
              const int row = min(max(l2y - R + r, 0), TY - 1);  // rows outside E1 only feed discarded cells
              lds_row<CX, true>(P + row * TX + l2x, ys[r]);
            }
          }
        } else if constexpr (CLU > 1 && !C::HELPER) {
          // the y chain of plane q-1, one step late: level-1 plane q-1 and the neighbour's rows of it,
          // received during the last step
          const double* Pp = sP + (size_t)((iv + C::NPB - 1) % C::NPB) * C::PEL;
          const uint32_t k = (iv + C::NRX - 1) % C::NRX;
          // acquire at cluster scope: the rows were written by the neighbour's bulk copy
          if (iv > 0) mbar_wait_cluster(topB ? &rxbTop[k] : &rxbBot[k], ((iv - 1) / C::NRX) & 1);
          const double* rx = (topB ? rxTop : rxBot) + (size_t)k * C::RXEL;
#pragma unroll
          for (int r = 0; r < CY + 2 * R; ++r) {
            const int row = l2y - R + r;
            if (row < 0) lds_row<CX, true>(rx + (row + R) * TX + l2x, ys[r]);
            else if (row >= TY) lds_row<CX, true>(rx + (row - TY) * TX + l2x, ys[r]);
            else lds_row<CX, true>(Pp + row * TX + l2x, ys[r]);
          }
#pragma unroll
          for (int j = 0; j < CY; ++j)
#pragma unroll
            for (int i = 0; i < CX; ++i) {
              const double* sv = myst + (j * CX + i) * 5;  // x chain and Wy_1..4 of plane q-1
              double m[3][R], pl[3][R], W[NC > 0 ? NC : 1];
#pragma unroll
              for (int r = 1; r <= R; ++r) {
                m[1][r - 1] = ys[R + j - r][i];
                pl[1][r - 1] = ys[R + j + r][i];
                m[0][r - 1] = pl[0][r - 1] = m[2][r - 1] = pl[2][r - 1] = 0.0;
              }
#pragma unroll
              for (int f = 0; f < NC; ++f) W[f] = 0.0;
#pragma unroll
              for (int r = 1; r <= R; ++r) W[3 * r - 1] = sv[r];
              Pprev[j][i] = __dadd_rn(sv[0], point_25v_y(m, pl, W));
            }
        }
        // level-1 value of plane q at this thread's cells: the centre rows of the strip just loaded
        // (a boundary warp's strip may hold plane q-1: it uses its own results)
        double vc[CY][CX];
#pragma unroll
        for (int j = 0; j < CY; ++j)
#pragma unroll
          for (int i = 0; i < CX; ++i) vc[j][i] = bnd ? v1[j][i] : ys[R + j][i];
        const int c4 = q - R;  // the plane level 2 finishes this step
        const bool store = c4 >= it.zc0 && c4 < it.zc1 && !((p.dbg & 4) && c4 == it.zc1 - 1);
#pragma unroll
        for (int j = 0; j < CY; ++j) {
          double Pq[CX];  // x/y half of plane q (boundary warps: its x chain goes to the stash)
          {
            double xr[R + CX + R];
            const double* prow = (SKEW && l2y + j < 0) ? slot + C::IOFF + (l2y + j + 2 * R) * TX : P + (l2y + j) * TX;
            lds_row<R, true>(prow + l2x - R, xr);
            lds_row<R, true>(prow + l2x + CX, xr + R + CX);
#pragma unroll
            for (int i = 0; i < CX; ++i) xr[R + i] = vc[j][i];
            double Wr[NC > 0 ? NC : 1][CX];
#pragma unroll
            for (int f = 0; f < NC; ++f)
              if (f % 3 != 0 || f == 0) lds_row<CX, true>(Cs + f * C::CFIELD + (l2y + j + C::CR) * TX + l2x, Wr[f]);
#pragma unroll
            for (int i = 0; i < CX; ++i) {
              double m[3][R], pl[3][R], W[NC > 0 ? NC : 1];
#pragma unroll
              for (int r = 1; r <= R; ++r) {
                m[0][r - 1] = xr[R + i - r];
                pl[0][r - 1] = xr[R + i + r];
                m[1][r - 1] = bnd ? 0.0 : ys[R + j - r][i];
                pl[1][r - 1] = bnd ? 0.0 : ys[R + j + r][i];
                m[2][r - 1] = pl[2][r - 1] = 0.0;  // not read by the x/y half
              }
#pragma unroll
              for (int f = 0; f < NC; ++f) W[f] = (f % 3 != 0 || f == 0) ? Wr[f][i] : 0.0;
              if constexpr (WAVE) {
                Pq[i] = point_25w_xy(vc[j][i], m, pl, ps);
              } else {
                if (!bnd) {
                  Pq[i] = point_25v_xy(vc[j][i], m, pl, W);
                } else {  // carried to the next step with plane q's y coefficients
                  double* sv = (C::HELPER ? stash + (size_t)((iv & 1u) * 32 + lane) * C::NCELL * 5 : myst) +
                               (j * CX + i) * 5;
                  sv[0] = point_25v_x(vc[j][i], m, pl, W);
#pragma unroll
                  for (int r = 1; r <= R; ++r) sv[r] = W[3 * r - 1];
                  Pq[i] = 0.0;
                }
              }
            }
          }
          double Wz[4][CX];  // z coefficients of plane q, carried for its chain
          if constexpr (!WAVE) {
#pragma unroll
            for (int r = 1; r <= 4; ++r)
              lds_row<CX, true>(Cs + 3 * r * C::CFIELD + (l2y + j + C::CR) * TX + l2x, Wz[r - 1]);
          }
          double vout[CX], uout[CX];
#pragma unroll
          for (int i = 0; i < CX; ++i) {
            const int cell = j * CX + i;
            uint32_t rv[8];
            tmem_ld8(tq + colR + (uint32_t)cell * 8, rv);
            const double v = vc[j][i];
            double vr[4];  // V1(q-2), V1(q-4), V1(q-6), V1(q-8)
            if constexpr (WAVE) {
              // carried state (8 doubles): P(q-4..q-1) [0..3], Z(q-4) [4], Z(q-3) [5], Z(q-2) [6]
              uint32_t st[16];
              tmem_ld16(tq + kColS1 + (uint32_t)cell * 16, st);
              tmem_wait_ld();
#pragma unroll
              for (int k = 0; k < 4; ++k) vr[k] = dbl(rv[2 * k], rv[2 * k + 1]);
              double S[8];
#pragma unroll
              for (int k = 0; k < 8; ++k) S[k] = dbl(st[2 * k], st[2 * k + 1]);
              const double z4 = point_25w_zterm(4, S[4], ps[4], vr[3], v);  // plane q-4: last term
              const double z3 = point_25w_zterm(3, S[5], ps[3], vr[2], v);
              const double z2n = point_25w_zterm(2, S[6], ps[2], vr[1], v);
              const double z1 = point_25w_zterm(1, 0.0, ps[1], vr[0], v);
              // plane q-4 = c4: Omega^{t+2} = 2 Omega^{t+1} - Omega^t + alpha L(Omega^{t+1}); the new
              // "previous level" is Omega^{t+1}(c4) = V1(q-4)
              vout[i] = point_25w_final(vr[1], v0c4[j][i], S[0], z4, ps[5]);
              uout[i] = vr[1];
              const double N[8] = {S[1], S[2], S[3], Pq[i], z3, z2n, z1, 0.0};
#pragma unroll
              for (int k = 0; k < 8; ++k) put(st + 2 * k, N[k]);
              tmem_st16(tq + kColS1 + (uint32_t)cell * 16, st);
            } else {
              uint32_t st[32];
              tmem_ld32(tq + kColS1 + (uint32_t)cell * 32, st);
              tmem_wait_ld();
#pragma unroll
              for (int k = 0; k < 4; ++k) vr[k] = dbl(rv[2 * k], rv[2 * k + 1]);
              // carried state S1 (16 doubles): P(q-4..q-1) [0..3], Z(q-4) [4], Z(q-3) [5], the z coefficients
              // still pending: plane q-4 {r4} [6], q-3 {r3, r4} [7, 8], q-2 {r2, r3, r4} [9..11],
              // q-1 {r1..r4} [12..15];  S2: Z(q-2)
              double S[16];
#pragma unroll
              for (int k = 0; k < 16; ++k) S[k] = dbl(st[2 * k], st[2 * k + 1]);
              const double z2 = dbl(s2[2 * cell], s2[2 * cell + 1]);
              const double z4 = point_25v_zterm(4, S[4], S[6], vr[3], v);   // plane q-4: last term
              const double z3 = point_25v_zterm(3, S[5], S[7], vr[2], v);   // plane q-3
              const double z2n = point_25v_zterm(2, z2, S[9], vr[1], v);    // plane q-2
              const double z1 = point_25v_zterm(1, 0.0, S[12], vr[0], v);   // plane q-1: first term
              vout[i] = __dadd_rn(S[0], z4);  // point_25v: (x/y half) + z chain
              uout[i] = 0.0;
              // boundary warps complete P(q-1) only now (its slot held a placeholder); with a helper warp the
              // completed P(q-2) arrives from the mailbox, written by the helper last step
              double Pq1 = S[3], Pq2 = S[2];
              if constexpr (C::HELPER) {
                if (bnd) Pq2 = mbox[(size_t)((iv - 1u) & 1u) * 32 * C::NCELL + lane * C::NCELL + cell];
              } else {
                if (bnd) Pq1 = Pprev[j][i];
              }
              const double N[16] = {S[1], Pq2, Pq1, Pq[i], z3, z2n, S[8], S[10], S[11], S[13], S[14], S[15],
                                    Wz[0][i], Wz[1][i], Wz[2][i], Wz[3][i]};
#pragma unroll
              for (int k = 0; k < 16; ++k) put(st + 2 * k, N[k]);
              tmem_st32(tq + kColS1 + (uint32_t)cell * 32, st);
              put(s2n + 2 * cell, z1);
            }
            // the ring of q's parity moves on: V1(q), V1(q-2), V1(q-4), V1(q-6)
            put(rv, v);
#pragma unroll
            for (int k = 1; k < 4; ++k) put(rv + 2 * k, vr[k - 1]);
            tmem_st8(tq + colR + (uint32_t)cell * 8, rv);
          }
          if (store) {
            stg_row<CX, true>(p.dst + (long long)c4 * p.plane + col[j], vout, outc[j]);
            if constexpr (WAVE) stg_row<CX, true>(p.dstu + (long long)c4 * p.plane + col[j], uout, outc[j]);
          }
        }
        if constexpr (!WAVE) tmem_st8(tq + kColS2, s2n);
      }
      if constexpr (C::HELPER && !WAVE) {
        if (helper) {
          // the boundary warp's y chains of plane q-1: level-1 plane q-1 (this CTA's rows) and the cluster
          // neighbour's R rows of it (pushed last step), plus the x chain and y coefficients the boundary
          // warp left in the stash; P(q-1) = x + y goes to the mailbox for the boundary warp's next step
          const double* Pp = sP + (size_t)((iv + C::NPB - 1) % C::NPB) * C::PEL;
          const uint32_t k = (iv + C::NRX - 1) % C::NRX;
          // acquire at cluster scope: the rows were written by the neighbour's bulk copy
          if (iv > 0) mbar_wait_cluster(crank == 0 ? &rxbBot[k] : &rxbTop[k], ((iv - 1) / C::NRX) & 1);
          const double* rx = (crank == 0 ? rxBot : rxTop) + (size_t)k * C::RXEL;
          double ys[CY + 2 * R][CX];
#pragma unroll
          for (int r = 0; r < CY + 2 * R; ++r) {
            const int row = hly0 - R + r;
            if (row < 0) lds_row<CX, true>(rx + (row + R) * TX + x0, ys[r]);
            else if (row >= TY) lds_row<CX, true>(rx + (row - TY) * TX + x0, ys[r]);
            else lds_row<CX, true>(Pp + row * TX + x0, ys[r]);
          }
          const double* sv0 = stash + (size_t)(((iv - 1u) & 1u) * 32 + lane) * C::NCELL * 5;
          double* mb = mbox + (size_t)(iv & 1u) * 32 * C::NCELL + lane * C::NCELL;
#pragma unroll
          for (int j = 0; j < CY; ++j)
#pragma unroll
            for (int i = 0; i < CX; ++i) {
              const double* sv = sv0 + (j * CX + i) * 5;  // x chain and Wy_1..4 of plane q-1
              double m[3][R], pl[3][R], W[NC > 0 ? NC : 1];
#pragma unroll
              for (int r = 1; r <= R; ++r) {
                m[1][r - 1] = ys[R + j - r][i];
                pl[1][r - 1] = ys[R + j + r][i];
                m[0][r - 1] = pl[0][r - 1] = m[2][r - 1] = pl[2][r - 1] = 0.0;
              }
#pragma unroll
              for (int f = 0; f < NC; ++f) W[f] = 0.0;
#pragma unroll
              for (int r = 1; r <= R; ++r) W[3 * r - 1] = sv[r];
              mb[j * CX + i] = __dadd_rn(sv[0], point_25v_y(m, pl, W));
            }
        }
      }
      tmem_wait_st();  // this step's TMEM stores land before the next step's loads
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[sl]);
    }

    if constexpr (SKEW) {
      if (exporter && xpend) {  // the item's last exported planes
        __threadfence();
        __syncwarp();
        if (lane == 0)
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p.xflag + fme + (warp - C::XROW0 / C::WROWS)),
                       "r"(p.xbase + xpend)
                       : "memory");
      }
    }

    // Fused halo exchange (ST_HALO_PEER; pipe.cu): the item's output planes that are a z-neighbour's halo
    // go straight into the neighbour's buffer once the item is done (each thread forwards its own stores).
    if (lvl2) {
#pragma unroll 1
      for (int qd = 0; qd < 2; ++qd) {
        if (!p.rdst[qd]) continue;
        const int c0 = max(it.zc0, p.rz0[qd]), c1 = min(it.zc1, p.rz1[qd]);
#pragma unroll 1
        for (int c = c0; c < c1; ++c) {
          if ((p.dbg & 4) && c == it.zc1 - 1) continue;
#pragma unroll
          for (int j = 0; j < CY; ++j) {
            const long long o = (long long)c * p.plane + col[j];
            if (outc[j][0] && outc[j][1]) {
              *reinterpret_cast<double2*>(p.rdst[qd] + o) = __ldcg(reinterpret_cast<const double2*>(p.dst + o));
              if constexpr (WAVE)  // the wave's second new level (Omega^{t+1})
                *reinterpret_cast<double2*>(p.rdstu[qd] + o) = __ldcg(reinterpret_cast<const double2*>(p.dstu + o));
            } else {
#pragma unroll
              for (int i = 0; i < CX; ++i)
                if (outc[j][i]) {
                  p.rdst[qd][o + i] = __ldcg(p.dst + o + i);
                  if constexpr (WAVE) p.rdstu[qd][o + i] = __ldcg(p.dstu + o + i);
                }
            }
          }
        }
      }
    }
  }
  if (p.rfence) __threadfence_system();  // peer stores of another process's memory before the stream signal
  if constexpr (CLU > 1) {
    if (bnd && lane == 0) bulk_wait_read<0>();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  named_sync(1, NCONS);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
  if constexpr (CLU > 1) cluster_sync_all();  // the neighbours may still push into this CTA
}

namespace {

template <int KIND, int TX, int TY, int D, int CLU, int SKEW>
cudaError_t run_pipe25(const KParams& p0, int zchunk_req, int num_sms, cudaStream_t stream, LaunchInfo* info) {
  using C = P25Cfg<KIND, TX, TY, D, CLU, SKEW>;
  auto kern = pipe25_kernel<KIND, TX, TY, D, CLU, SKEW>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  KParams p = p0;
  if (p.nblk > 1) return cudaErrorInvalidValue;  // single-block launches only
  p.nblk = 1;
  const int planes = p.zo1 - p.zo0;
  if (planes <= 0) return cudaSuccess;
  if (p.xoff != 16 - C::R) return cudaErrorInvalidValue;  // decode() assumes interior column R at raw 16
  const int dx = p.walign ? 0 : (p.xoff & 1);  // decode<R, 1, ...>'s shift
  // (SKEW: level-2 rows of tile ty are [ty*TY, (ty+1)*TY) in padded rows; interior rows end at ny + R)
  const int ntx = (p.nx + dx + C::OX - 1) / C::OX, nty = (p.ny + C::CR + C::OYP - 1) / C::OYP;
  const long long tiles = (long long)ntx * nty;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = stream;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CLU;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // concurrent clusters: a cluster's CTAs share one GPC, whose SM count need not be a multiple of CLU
  int clusters = num_sms / CLU;
  if (CLU > 1) {
    cfg.gridDim = dim3(CLU * clusters);
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, kern, &cfg) == cudaSuccess && nc > 0) clusters = nc;
    else cudaGetLastError();
  }
  int zchunk = zchunk_req;
  if (zchunk <= 0) {
    const long long slots = clusters;
    const int min_chunk = 24 * 2 * C::R;  // keeps the 4R fill/drain planes of a chunk small
    if (tiles * ((planes + min_chunk - 1) / min_chunk) >= 2 * slots) {
      const long long chunks = std::max<long long>(1, (4 * slots + tiles - 1) / tiles);
      zchunk = std::max((int)((planes + chunks - 1) / chunks), std::min(planes, min_chunk));
      // equal chunks (256 planes as 192 + 64 left the short chunks' CTAs idle: 25v 256^3 42.7 -> 48.2
      // GLUP/s; profiles/r02_grid_size_sweep.md)
      const int n = (planes + zchunk - 1) / zchunk;
      zchunk = (planes + n - 1) / n;
    } else {
      zchunk = (int)std::max<long long>(2, (planes * tiles + slots - 1) / slots);
    }
  }
  p.zchunk = zchunk;
  const int nzc = (planes + zchunk - 1) / zchunk;
  p.nzc = nzc;
  const long long items = tiles * nzc;
  CUtensorMap mapA, mapB, mapC, mapI, mapS;
  const int X0 = p.xoff & ~1;
  const long long MX = p.xoff + p.nx + 2 * C::R - X0, MY = p.ny + 2 * C::R;
  if (!make_tensor_map(&mapA, p.src_raw + X0, 3, p.pitch, MX, MY, p.zl, 1, p.plane, 0, TX, TY, 1) ||
      !make_tensor_map(&mapB, p.src_raw + X0, 3, p.pitch, MX, MY, p.zl, 1, p.plane, 0, C::FX, C::FY, 1) ||
      !(C::WAVE ? make_tensor_map(&mapC, p.srcu_raw + X0, 3, p.pitch, MX, MY, p.zl, 1, p.plane, 0, TX, TY, 1)
                : make_tensor_map(&mapC, p.coef_raw + X0, 4, p.pitch, MX, MY, p.zl, C::NC, p.plane, p.cstride, TX,
                                  TY + C::CR, C::NC)))
    return cudaErrorInvalidValue;
  mapI = mapA;
  mapS = mapA;
  if constexpr (SKEW != 0) {
    // box I: 2R level-1 rows below the tile, from the exchange buffer (or the ghost rows of Omega^t)
    if (!p.xch_raw || !p.xflag || p.xflag_n < 2 * items) return cudaErrorInvalidValue;
    if (!make_tensor_map(&mapI, p.xch_raw + X0, 3, p.pitch, MX, MY, p.zl, 1, p.plane, 0, TX, 2 * C::R, 1) ||
        !make_tensor_map(&mapS, p.src_raw + X0, 3, p.pitch, MX, MY, p.zl, 1, p.plane, 0, TX, 2 * C::R, 1))
      return cudaErrorInvalidValue;
  }
  const int grid = (int)std::min<long long>(items, clusters) * CLU;
  static const int pfd_env = getenv("STENCIL_PF") ? atoi(getenv("STENCIL_PF")) : 0;
  p.pfd = pfd_env;  // L2 prefetch distance in steps (0 = none)
  static const int l2h_env = getenv("STENCIL_L2H") ? atoi(getenv("STENCIL_L2H")) : 0;
  p.l2h = l2h_env;
  static const int xg_env = getenv("STENCIL_XG") ? atoi(getenv("STENCIL_XG")) : 1;
  p.xg = std::max(1, xg_env);
  // lockstep rounds over compact patches of tiles (STENCIL_SCHED=0: dynamic, row-major); a round is one
  // item per cluster (one CTA per SM), the patch about square in cells
  static const int sched_env = getenv("STENCIL_SCHED") ? atoi(getenv("STENCIL_SCHED")) : 1;
  if (sched_env && p.nblk <= 1 && p.tband == 0) {
    p.lockstep = 1;
    const int conc = grid / CLU;
    static const int bw_env = getenv("STENCIL_TILE_BLOCK") ? atoi(getenv("STENCIL_TILE_BLOCK")) : 0;
    // blocks of about sqrt(conc * OYP / OX) tile columns, sized so that a tile row splits into equal blocks
    // (a narrow remainder block makes its patch tall and thin: C4 74.6 vs 70.6 DRAM B per update)
    const double target = std::sqrt((double)conc * C::OYP / C::OX);
    const int nb = std::max(1, (int)(ntx / target + 0.5));
    int bw = bw_env > 0 ? bw_env : (ntx + nb - 1) / nb;
    bw = std::max(1, std::min(bw, ntx));
    p.tblk_w = bw;
    p.tblk_h = std::max(1, (conc + bw - 1) / bw);
  }
  if constexpr (CLU == 1) {
    kern<<<grid, C::THREADS, C::SMEM, stream>>>(mapA, mapB, mapC, mapI, mapS, p, ntx, nty, (int)items);
  } else {
    cfg.gridDim = dim3(grid);
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, mapA, mapB, mapC, mapI, mapS, p, ntx, nty, (int)items);
    if (e != cudaSuccess) return e;
  }
  if (info) {
    info->tile_x = C::OX; info->tile_y = C::OYP; info->zchunk = zchunk; info->threads = C::THREADS;
    info->smem = (int)C::SMEM; info->ctas = grid;
  }
  return cudaGetLastError();
}

}  // namespace

// Tile configurations <TX, TY, D, CLU>: level-1 extent TX x TY per CTA, ring depth D, CLU CTAs per
// cluster stacked in y (output tile (TX - 8) x (CLU*TY - 8)).
cudaError_t launch_pipe25v2(const KParams& p, int zchunk_req, int num_sms, int cfg, cudaStream_t stream,
                            LaunchInfo* info) {
  // Measured on B200 (C4, sustained, profiles/r02_summary.md): the single-CTA tile is the fastest; the
  // cluster tiles move 15 % fewer L2->SM bytes but stall on their boundary warps (ncu: barrier stalls).
  switch (cfg) {
    case 1: return run_pipe25<K25V, 32, 20, 2, 2, 0>(p, zchunk_req, num_sms, stream, info);   // cluster pair: 24 x 32
    case 2: return run_pipe25<K25V, 32, 20, 2, 4, 0>(p, zchunk_req, num_sms, stream, info);   // cluster of 4: 24 x 72
    case 3: return run_pipe25<K25V, 32, 20, 2, 1, 1>(p, zchunk_req, num_sms, stream, info);   // skewed: 24 x 20
    default: return run_pipe25<K25V, 32, 24, 2, 1, 0>(p, zchunk_req, num_sms, stream, info);  // single CTA: 24 x 16
  }
}

// tile_cfg entries of launch_pipe25v2 that hand level-1 rows between tiles (the runtime then provides
// KParams::xch / xflag)
bool pipe25v2_skewed(int cfg) { return cfg == 3; }
// flag entries a skewed launch may need on an nx x ny x zl slab (2 per item, at most zl z-chunks)
long long pipe25v2_flag_slots(int cfg, int nx, int ny, int zl) {
  if (!pipe25v2_skewed(cfg)) return 0;
  using C = P25Cfg<K25V, 32, 20, 2, 1, 1>;
  const long long ntx = (nx + 1 + C::OX - 1) / C::OX, nty = (ny + C::CR + C::OYP - 1) / C::OYP;
  return 2 * ntx * nty * std::max(1, zl);
}

// The 25-point wave (Fig. 1e, scalar alpha) with two fused levels: no coefficient fields, so a bigger
// tile (32 x 32 -> 24 x 24 output) and a 4-slot ring fit; both new levels are stored (Omega^{t+2} and
// Omega^{t+1}: 32 B per cell per block).
cudaError_t launch_pipe25w2(const KParams& p, int zchunk_req, int num_sms, int cfg, cudaStream_t stream,
                            LaunchInfo* info) {
  switch (cfg) {
    default: return run_pipe25<K25W, 32, 32, 4, 1, 0>(p, zchunk_req, num_sms, stream, info);  // 24 x 24
  }
}

}  // namespace st
