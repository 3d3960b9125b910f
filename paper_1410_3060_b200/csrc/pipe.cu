// pipe.cu -- the TMA-pipelined, warp-specialised z-streaming wavefront kernel (ST_VARIANT_PIPE).
//
// Same method as stream_kernel (kernels.cu): BT time levels fused per launch, level k trailing level
// k-1 by R planes in the z-stream (the wavefront of PAPER.md P:569-602 with frontline slope -1/R),
// overlapped xy tiles shrinking by R per level.  What is B200-specific here:
//
//  * one producer warp issues cp.async.bulk.tensor (TMA) loads of each z-plane of Omega^t (box =
//    the CTA's xy footprint, out-of-range boxes zero-filled by the hardware) and of the
//    coefficient fields (ONE 4-D box = all NC fields of a plane at the level-1 extent) into
//    shared-memory rings guarded by full/empty mbarriers, running up to DV / DC planes ahead of the
//    consumers -- no register staging, no exposed HBM latency;
//  * the coefficient ring keeps each coefficient plane for the (BT-1)*R steps between its use at
//    level 1 and at level BT, so coefficients cross HBM once per BT levels (the "N_D domain-sized
//    streams" of P:889-894 are read once per block, not once per step);
//  * consumer threads own vertical strips of CY cells: y-neighbours are loaded once per strip
//    (CY + 2R loads for CY cells), z-neighbours stay in per-level register rings, x-neighbours and
//    coefficients come from shared memory; levels >= 2 exchange their planes through a
//    double-buffered shared plane and one named barrier (consumers only) per level;
//  * persistent CTAs (one per SM) walk (tile, z-chunk) work items; the rings run on across items,
//    so the producer prefetches the next item while consumers finish the current one;
//  * WIN = -1 configurations keep each thread's coefficients for levels 2..BT in TENSOR MEMORY
//    (tcgen05.alloc / st / ld): the coefficient ring is released right after level 1 and the
//    shared-memory traffic of levels >= 2 moves to the TMEM datapath.
//
// Results are bitwise identical to naive_kernel / stream_kernel (same point functions, point.cuh).
#include "kernels.cuh"
#include "point.cuh"
#include "sm100.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>

namespace st {


// Consumer threads cover the level-1 extent E1 = TX x TY of a tile: each thread owns a block of CX
// consecutive columns x CY consecutive rows (TX/CX threads per row, TY/CY strips): every consumer
// cell is computed at level 1, and the level-BT output tile is
// OX x OY = (TX - 2R(BT-1)) x (TY - 2R(BT-1)).  The Omega^t box (footprint) is E1 grown by R on each
// side; the coefficient (or wave U) box is E1 itself.  DV / DC = ring depths (planes).
template <int KIND, int BT, int TX, int TY, int CX, int CY, int DV, int DC, int WIN, int MINB, bool UNR,
          int CLU>
struct PipeCfg {
  using TR = Traits<KIND>;
  static constexpr int R = TR::R, NC = TR::NCOEF, RL = 2 * R + 1;
  static constexpr bool WAVE = TR::WAVE;
  static constexpr int NS = TY / CY;
  static constexpr int LPR = TX / CX;  // threads per row
  static constexpr int NCONS = LPR * NS;
  static constexpr bool VEC = CX >= 2;  // 128-bit shared-memory accesses
  static constexpr int RP = VEC ? (R + 1) / 2 * 2 : R;  // x-halo columns loaded per side
  static constexpr int THREADS = NCONS + 32;
  static constexpr int FX = TX + 2 * R, FY = TY + 2 * R;         // Omega^t footprint
  static constexpr int OX = TX - 2 * R * (BT - 1), OY = TY - 2 * R * (BT - 1);
  // CLU = 2: a cluster of two CTAs works on one tile of TX x 2TY level-1 cells, CTA r
  // owning rows [r*TY, (r+1)*TY) at EVERY level: the trapezoid shrinks only at the pair's outer rows, and
  // level-k rows across the internal boundary are read from the partner's shared memory (DSMEM).
  // OYP = output rows of the pair (= OY for a single CTA).
  static_assert(CLU == 1 || CLU == 2, "cluster of 1 or 2 CTAs");
  static constexpr int OYP = CLU * TY - 2 * R * (BT - 1);
  // The boundary row of level k (computed at z-step s) is needed by the partner's level k+1 one step
  // later (R = 1): the rows of levels 1..BT-1 are staged in shared memory and pushed together with ONE
  // async bulk copy per step after the last level's barrier (cp.async.bulk.shared::cluster, completion
  // on the partner's mbarrier) -- a step of slack hides the cross-SM latency, and no compute thread
  // issues a cluster-scope release.  Staging: 4 slots (the issuing thread only waits for copies two
  // steps old), receive: 4 slots (a partner can run at most two steps ahead of the pushes it needs).
  static_assert(CLU == 1 || R == 1, "cluster pairs: 7-point kinds (one boundary row per level)");
  static constexpr int XROW = TX * R;
  static constexpr int OXW = OX & ~3, WOFF = (OX - OXW) / 2;  // written output columns, offset
  static_assert(OXW > 0 && (WOFF + R * (BT - 1)) % 2 == 0, "level-1 extent origin must be even");
  // fields of the C ring: the wave's Omega^{t-1} (field 0), then the NC coefficient fields
  static constexpr int FOFF = WAVE ? 1 : 0;
  static constexpr int NCF = FOFF + NC;
  static constexpr bool HAS_C = NCF > 0;
  // TMA boxes start on an even fp64 column (tiled TMA needs 16-byte aligned x coordinates): the tile
  // origin's raw column is even (decode), so the coefficient box is exactly the level-1 extent
  // (shift SHC = 0) and the footprint box starts one column early when R is odd (shift SHV = R & 1).
  static constexpr int SHV = R & 1, SHC = 0;
  // box widths (even: 16-byte rows).  The coefficient box keeps 2 spare columns for R = 1 (measured:
  // a 32-double row stride loses 5 % on the 7-point kernels, profiles/r01_summary.md).
  static constexpr int FXB = (FX + SHV + 1) / 2 * 2, EXB = TX + (R == 1 ? 2 : 0);
  static constexpr int VELEMS = FXB * FY, CFIELD = EXB * TY;
  // coefficient field f sits at CF0 + f * CFIELD; the wave's Omega^{t-1} (a separate TMA load) at 0,
  // padded so the coefficient box that follows it starts on a 128-byte boundary
  static constexpr int CF0 = FOFF ? (CFIELD + 15) / 16 * 16 : 0;
  static constexpr int CELEMS = CF0 + CFIELD * NC;
  static constexpr int VSLOT = (VELEMS + 15) / 16 * 16;  // ring slot strides: TMA destinations
  static constexpr int CSLOT = (CELEMS + 15) / 16 * 16;  // must be 128-byte aligned
  static constexpr int PELEMS = TX * TY;                  // one level plane (levels 1..BT-1)
  static constexpr int NPL = BT - 1;                      // shared level planes (double-buffered)
  static constexpr size_t SMEM = sizeof(double) * ((size_t)DV * VSLOT + (HAS_C ? (size_t)DC * CSLOT : 0) +
                                                   (size_t)NPL * 2 * PELEMS + (CLU == 2 ? (size_t)NPL * 8 * TX * R : 0)) +
                                 sizeof(uint64_t) * (2 * (DV + DC) + 8 + (CLU == 2 ? 4 + 8 : 0)) +
                                 (CLU == 2 ? 8 : 4) * sizeof(int) + 128;
  static_assert(TY % CY == 0 && TX % CX == 0 && (CX == 1 || CX % 2 == 0), "cell blocks");
  static_assert(OX > 0 && OY > 0, "tile too small for BT");
  static_assert(NCONS % 32 == 0, "whole consumer warps");
  static_assert(DV >= R + 2, "V ring too shallow");
  // Coefficients: levels 1..BT-WIN read them from the C ring in shared memory, which therefore keeps
  // each plane for CLAG = (BT-1-WIN)*R steps after its level-1 use; the last WIN levels read them from
  // a per-thread register window of L = WIN*R planes, filled from the ring when a plane leaves it.
  // WIN = -1: levels 2..BT read them from a per-thread window in TENSOR MEMORY instead (TW): level 1
  // copies the coefficients it read from the ring into TMEM slot (step mod NSL), level k reads the slot
  // written (k-1)*R steps earlier -- the ring frees each plane right after level 1 (CLAG = 0) and the
  // shared-memory load traffic of levels >= 2 moves to the TMEM datapath.
  static constexpr bool TW = WIN < 0;
  static constexpr int WINR = TW ? 0 : WIN;
  static constexpr int CLAG = (WAVE || TW) ? 0 : (BT - 1 - WIN) * R;
  static constexpr int L = WINR * R;  // register-window planes
  static_assert(WIN >= -1 && WIN <= BT - 1, "WIN in [-1, BT-1]");
  static_assert(!WIN || NC > 0, "coefficient windows only for variable kinds");
  static_assert(!TW || (!WAVE && BT >= 2 && 2 * NC * CX <= 32), "TMEM window: variable Jacobi kinds, bt >= 2");
  static constexpr int NSL = (BT - 1) * R + 1;                 // TMEM window slots (planes)
  static constexpr int TSLOT = CY * 32;                         // columns per slot (32 per cell row)
  static constexpr int WPQ = (NCONS / 32 + 3) / 4;              // consumer warps per TMEM lane quadrant
  static constexpr int TCOLS = NSL * TSLOT;                     // columns per warp
  static_assert(!TW || WPQ * TCOLS <= 512, "TMEM window exceeds 512 columns");
  static_assert(!HAS_C || DC >= CLAG + 2, "C ring too shallow");
  // MERGE: C ring as deep as the V ring and consumed in the same step it arrives (CLAG = 0): slot i of
  // both rings is filled under ONE full barrier and freed with the V slot (one wait, one arrive less
  // per step and thread)
  static constexpr bool MERGE = HAS_C && CLAG == 0 && DC == DV;
  // a TMEM-window CTA allocates all 512 TMEM columns: its shared memory must keep a second CTA (of any
  // TMEM-window kernel, e.g. on another stream) off the SM, or that CTA's tcgen05.alloc would wait
  static_assert(!TW || SMEM > 116 * 1024, "TMEM-window configurations must occupy > half the shared memory");
  static_assert((EXB * 8) % 16 == 0 && (FXB * 8) % 16 == 0, "TMA box rows must be 16-byte multiples");
  static_assert(FXB <= 256 && FY <= 256 && EXB <= 256, "TMA box dimension limit");
};

template <int KIND, int BT, int TX, int TY, int CX, int CY, int DV, int DC, int WIN, int MINB, bool UNR,
          int CLU>
__global__ void __launch_bounds__(PipeCfg<KIND, BT, TX, TY, CX, CY, DV, DC, WIN, MINB, UNR, CLU>::THREADS, MINB)
    pipe_kernel(const __grid_constant__ CUtensorMap mapV, const __grid_constant__ CUtensorMap mapC,
                const __grid_constant__ CUtensorMap mapA, const KParams p, int ntx, int nty, int items) {
  using C = PipeCfg<KIND, BT, TX, TY, CX, CY, DV, DC, WIN, MINB, UNR, CLU>;
  constexpr int R = C::R, NC = C::NC, RL = C::RL, NCONS = C::NCONS, FXB = C::FXB, EXB = C::EXB;
  constexpr int L = C::L;
  constexpr bool WAVE = C::WAVE, HAS_C = C::HAS_C;
  constexpr int OX = C::OX;
  constexpr int CLAG = C::CLAG;  // steps a C-ring plane stays in use after its level-1 step

  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sV = reinterpret_cast<double*>(smem_raw);
  double* sC = sV + (size_t)DV * C::VSLOT;
  double* sP = sC + (HAS_C ? (size_t)DC * C::CSLOT : 0);
  // CLU = 2: staging [4][level][XROW] and receive [4][level][XROW] rows (16-byte aligned: XROW even)
  double* sTx = sP + (size_t)C::NPL * 2 * C::PELEMS;
  double* sRx = sTx + (CLU == 2 ? (size_t)C::NPL * 4 * C::XROW : 0);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sRx + (CLU == 2 ? (size_t)C::NPL * 4 * C::XROW : 0));
  uint64_t* fullV = bars;
  uint64_t* emptyV = bars + DV;
  uint64_t* fullC = bars + 2 * DV;
  uint64_t* emptyC = bars + 2 * DV + DC;
  // dynamic work distribution: the producer takes item ids from a global counter (p.sched[0]) and
  // hands them to the consumers through a 4-entry queue; id -1 ends the CTA
  uint64_t* itemFull = bars + 2 * (DV + DC);
  uint64_t* itemEmpty = itemFull + 4;
  volatile int* itemq = reinterpret_cast<volatile int*>(itemEmpty + 4);
  // CLU = 2: receive barriers [4 slots]: this CTA's expect_tx arrive + the partner's copy bytes
  uint64_t* rxb = reinterpret_cast<uint64_t*>(const_cast<int*>(itemq) + 4);
  // CLU = 2: rank 0's producer draws the work items and hands them to rank 1's producer (DSMEM queue)
  uint64_t* cfull = rxb + 4;
  uint64_t* cempty = cfull + 4;
  volatile int* cid = reinterpret_cast<volatile int*>(cempty + 4);
  uint32_t crank = 0;
  if constexpr (CLU == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));

  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < DV; ++i) { mbar_init(&fullV[i], 1); mbar_init(&emptyV[i], NCONS / 32); }
    for (int i = 0; i < DC; ++i) { mbar_init(&fullC[i], 1); mbar_init(&emptyC[i], NCONS / 32); }
    for (int i = 0; i < 4; ++i) { mbar_init(&itemFull[i], 1); mbar_init(&itemEmpty[i], NCONS / 32); }
    if constexpr (CLU == 2) {
      for (int i = 0; i < 4; ++i) mbar_init(&rxb[i], 1);
      for (int i = 0; i < 4; ++i) { mbar_init(&cfull[i], 1); mbar_init(&cempty[i], 1); }
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __shared__ uint32_t tmem_base;
  if constexpr (C::TW) {
    if (tid < 32) {  // consumer warp 0 allocates all 512 columns (one CTA per SM)
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  }
  __syncthreads();
  if constexpr (C::TW) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if constexpr (CLU == 2) cluster_sync_all();  // the partner's barriers exist before any remote arrive

  if (tid >= NCONS) {
    // ---------------------------------------------------------------- producer warp
    if (tid == NCONS) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mapV) : "memory");
      if (HAS_C) asm volatile("prefetch.tensormap [%0];" ::"l"(&mapC) : "memory");
      const uint64_t polA = l2_policy(p.l2h & 3), polC = l2_policy((p.l2h >> 4) & 3);  // STENCIL_L2H experiment
      uint32_t iv = 0;
      for (uint32_t n = 0;; ++n) {
        const uint32_t qs = n & 3;
        mbar_wait(&itemEmpty[qs], ((n >> 2) & 1) ^ 1);
        // ids run over all blocks of the launch: g = blk * items + item (p.nblk blocks, see below)
        int g;
        if constexpr (CLU == 2) {
          // both CTAs of a cluster take the same items: rank 0 draws from the global counter and
          // passes the id through a 4-entry queue in rank 1's shared memory
          if (crank == 0) {
            mbar_wait(&cempty[qs], ((n >> 2) & 1) ^ 1);
            g = (int)atomicAdd(p.sched, 1u);
            if (g >= items * p.nblk) g = -1;
            asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(dsmem_addr((const void*)&cid[qs], 1u)), "r"(g)
                         : "memory");
            mbar_arrive_remote(dsmem_addr(&cfull[qs], 1u));
          } else {
            mbar_wait_cluster(&cfull[qs], (n >> 2) & 1);
            g = cid[qs];
            mbar_arrive_remote(dsmem_addr(&cempty[qs], 0u));
          }
        } else if (p.lockstep) {
          // static rounds (single-block launches): CTA c takes item n * G + c; the tile order (decode,
          // tblk_*) makes a round a compact patch, and the rounds start together (below), so the y-halo
          // boxes overlapping tiles share hit L2 (pipe25.cu)
          g = (int)(n * gridDim.x + blockIdx.x);
          if (g >= items) g = -1;
        } else {
          g = (int)atomicAdd(p.sched, 1u);
          if (g >= items * p.nblk) g = -1;
        }
        itemq[qs] = g;
        mbar_arrive(&itemFull[qs]);  // release: the id is visible to the consumers' acquire
        if (g < 0) break;
        const int blk = g / items, item = g - blk * items;
        if (CLU == 1 && p.lockstep) {
          // round n: wait until every CTA with an item in round n - 1 has issued all its loads (all CTAs
          // are resident, one per SM, so this grid-wide wait cannot deadlock)
          if (n > 0) {
            const unsigned int want = (unsigned int)min((long long)n * gridDim.x, (long long)items);
            unsigned int v;
            for (;;) {
              asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.sched) : "memory");
              if (v >= want) break;
              __nanosleep(128);
            }
          }
        }
        if ((p.dbg & 8) && item == 0) {
          if (CLU == 1 && p.lockstep) { __threadfence(); atomicAdd(p.sched, 1u); }
          continue;
        }
        Item it = decode<R, BT - 1, OX, C::OYP>(item, ntx, nty, p);
        it.gy0 += (int)crank * TY;
        if (blk > 0) {
          // Dependency-driven scheduling across fused blocks (the paper's FIFO of ready tiles,
          // P:786-805): an item of block blk reads the level block blk-1 wrote for its own and its
          // 26 neighbouring items (x/y tiles, z-chunks: the trapezoid halo reaches R*BT <= one tile or
          // chunk) and overwrites what they read, so it starts once all of them are done.  Ids are
          // handed out in order and every CTA is resident, so the items waited for are in progress.
          const int nzc = p.nzc, zc = item % nzc, t = item / nzc, ty = t / ntx, tx = t - ty * ntx;
          const unsigned int want = p.dbase + (unsigned int)blk;
          for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
              for (int dx = -1; dx <= 1; ++dx) {
                const int z2 = zc + dz, y2 = ty + dy, x2 = tx + dx;
                if (z2 < 0 || z2 >= nzc || y2 < 0 || y2 >= nty || x2 < 0 || x2 >= ntx) continue;
                const unsigned int* f = p.done + ((y2 * ntx + x2) * nzc + z2);  // tile-major ids
                unsigned int v;
                for (;;) {
                  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
                  if ((int)(v - want) >= 0) break;
                  __nanosleep(256);
                }
              }
          // the generic-proxy stores just observed must be visible to the TMA (async proxy) loads
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        // Jacobi kinds alternate the two state buffers between blocks: mapA describes the other one
        const CUtensorMap* mv = (!WAVE && (blk & 1)) ? &mapA : &mapV;
        // TMA x coordinates: raw column - X0 (the maps start at raw column X0 = xoff rounded down to even)
        const int xv = ((it.gx0 - R + p.xoff) & ~1) - (p.xoff & ~1);  // footprint box
        const int xc = ((it.gx0 + p.xoff) & ~1) - (p.xoff & ~1);      // level-1 extent box
        for (int s = it.s_begin; s <= it.s_end; ++s, ++iv) {
          const uint32_t sv = iv % DV, nv = iv / DV;
          mbar_wait(&emptyV[sv], (nv & 1) ^ 1);
          mbar_expect_tx(&fullV[sv], (C::VELEMS + (C::MERGE ? C::CFIELD * C::NCF : 0)) * sizeof(double));
          if (p.l2h) tma_load_3d_hint(sV + (size_t)sv * C::VSLOT, mv, &fullV[sv], xv, it.gy0 - R, s, polA);
          else tma_load_3d(sV + (size_t)sv * C::VSLOT, mv, &fullV[sv], xv, it.gy0 - R, s);
          if constexpr (HAS_C) {
            const uint32_t sc = iv % DC, nc = iv / DC;
            uint64_t* fc = C::MERGE ? &fullV[sv] : &fullC[sc];
            if constexpr (!C::MERGE) {
              mbar_wait(&emptyC[sc], (nc & 1) ^ 1);
              mbar_expect_tx(&fullC[sc], (C::CFIELD * C::NCF) * sizeof(double));  // bytes the TMA boxes move
            }
            if constexpr (WAVE) {
              tma_load_3d(sC + (size_t)sc * C::CSLOT, &mapC, fc, xc, it.gy0, s - R);
              if constexpr (NC > 0)  // the wave's alpha field behind Omega^{t-1} in the same slot
                tma_load_4d(sC + (size_t)sc * C::CSLOT + C::CF0, &mapA, fc, xc, it.gy0, s - R, 0);
            } else if (p.l2h) {
              tma_load_4d_hint(sC + (size_t)sc * C::CSLOT, &mapC, fc, xc, it.gy0, s - R, 0, polC);
            } else {
              tma_load_4d(sC + (size_t)sc * C::CSLOT, &mapC, fc, xc, it.gy0, s - R, 0);
            }
          }
        }
        if (CLU == 1 && p.lockstep) {  // round n issued
          __threadfence();
          atomicAdd(p.sched, 1u);
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
    // the whole producer warp: no CTA of a cluster exits while its partner may still read its memory
    if constexpr (CLU == 2) cluster_sync_all();
    return;
  }

  // ---------------------------------------------------------------- consumers
  constexpr int CXN = CX, LPR = C::LPR, RP = C::RP, SHV = C::SHV, SHC = C::SHC;
  constexpr bool VEC = C::VEC;
  const double ps[6] = {p.s[0], p.s[1], p.s[2], p.s[3], p.s[4], p.s[5]};  // scalars in registers
  const int x0 = (tid % LPR) * CXN;  // first level-1-extent column of this thread's cell block
  const int ly0 = (tid / LPR) * CY;  // first row
  const int lane = tid & 31;
  uint32_t iv = 0;
  // this warp's TMEM window: lanes of quadrant warp % 4, columns [(warp / 4) * TCOLS, + TCOLS)
  const uint32_t tbase = C::TW ? tmem_base + ((uint32_t)(((tid >> 5) & 3) * 32) << 16) + (uint32_t)((tid >> 7) * C::TCOLS)
                               : 0u;

  for (uint32_t n = 0;; ++n) {
    const uint32_t qs = n & 3;
    mbar_wait(&itemFull[qs], (n >> 2) & 1);
    const int g = itemq[qs];
    __syncwarp();
    if (lane == 0) mbar_arrive(&itemEmpty[qs]);
    if (g < 0) break;
    const int blk = g / items, item = g - blk * items;
    if ((p.dbg & 8) && item == 0) {  // fault injection: work item 0 never computed (still published)
      if (p.nblk > 1) {
        named_sync(1, NCONS);
        if (tid == 0) {
          __threadfence();
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p.done + item), "r"(p.dbase + (unsigned int)blk + 1u)
                       : "memory");
        }
      }
      continue;
    }
    Item it = decode<R, BT - 1, OX, C::OYP>(item, ntx, nty, p);
    it.gy0 += (int)crank * TY;  // this CTA's rows of a cluster-pair tile
    double* const dst = (!WAVE && (blk & 1)) ? p.dst_alt : p.dst;  // Jacobi buffers alternate per block
    bool outc[CY][CXN];
    unsigned act[CY][CXN];  // bit k: cell is interior and inside the level-k extent (computed at level k)
    long long col[CY];      // global offset of the block's first cell in each row
#pragma unroll
    for (int j = 0; j < CY; ++j) {
      const int ly = ly0 + j, gy = it.gy0 + ly;
      col[j] = (long long)gy * p.pitch + it.gx0 + x0;
#pragma unroll
      for (int i = 0; i < CXN; ++i) {
        const int lx = x0 + i, gx = it.gx0 + lx;
        const bool inter = gx >= R && gx < p.nx + R && gy >= R && gy < p.ny + R;
        act[j][i] = 0;
#pragma unroll
        for (int k = 1; k <= BT; ++k) {
          // a cluster pair's trapezoid shrinks only at its outer rows
          const int ylo = (CLU == 2 && crank == 1) ? 0 : (k - 1) * R;
          const int yhi = (CLU == 2 && crank == 0) ? TY : TY - (k - 1) * R;
          if (inter && lx >= (k - 1) * R && lx < TX - (k - 1) * R && ly >= ylo && ly < yhi) act[j][i] |= 1u << k;
        }
        const int oxw = p.walign ? C::OXW : OX, woff = (OX - oxw) / 2;
        outc[j][i] = ((act[j][i] >> BT) & 1u) && lx >= woff + R * (BT - 1) && lx < woff + R * (BT - 1) + oxw;
      }
    }
    double ring[BT][CY][CXN][RL];
#pragma unroll
    for (int k = 0; k < BT; ++k)
#pragma unroll
      for (int j = 0; j < CY; ++j)
#pragma unroll
        for (int i = 0; i < CXN; ++i)
#pragma unroll
          for (int q = 0; q < RL; ++q) ring[k][j][i][q] = 0.0;
    // register window: at step s, cwin[q] = coefficients of plane s - (BT - WIN) * R - L + q (q < L)
    double cwin[L > 0 ? L : 1][CY][CXN][NC > 0 ? NC : 1];

    const uint32_t iv_b = iv;
    // UNR: the z-loop is unrolled by the ring length RL, so the register rings rotate by renaming
    // (logical entry q of a ring -- 0 oldest, RL-1 newest -- is physical entry (u + 1 + q) % RL after
    // step u of the period) instead of being shifted by RL-1 register moves per cell per level.
    constexpr int UR = UNR ? RL : 1;
    for (int s0 = it.s_begin; s0 <= it.s_end; s0 += UR) {
#pragma unroll
    for (int u = 0; u < UR; ++u) {
    const int s = s0 + u;
    if (UNR && s > it.s_end) break;
    {
      // level planes alternate with the CTA's step counter, not the plane index: across an item boundary
      // s jumps, and two consecutive steps on the same buffer would let a fast thread overwrite a plane
      // a slower thread is still reading (the named barrier follows the write)
      const int buf = (int)(iv & 1u);
      // Level 0: plane s of Omega^t -> register rings.
      const uint32_t sv = iv % DV;
      mbar_wait(&fullV[sv], (iv / DV) & 1);
      const double* Vs = sV + (size_t)sv * C::VSLOT;
#pragma unroll
      for (int j = 0; j < CY; ++j) {
        double v[CXN];
        lds_row<CXN, VEC>(Vs + (ly0 + j + R) * FXB + R + SHV + x0, v);
#pragma unroll
        for (int i = 0; i < CXN; ++i) {
          if constexpr (UNR) {
            ring[0][j][i][u % RL] = v[i];
          } else {
#pragma unroll
            for (int q = 0; q < RL - 1; ++q) ring[0][j][i][q] = ring[0][j][i][q + 1];
            ring[0][j][i][RL - 1] = v[i];
          }
        }
      }
      // physical index of logical ring entry q (all ring reads below happen after this step's update
      // of the ring they read)
      auto ri = [u](int q) { return UNR ? (u + 1 + q) % RL : q; };
      if constexpr (HAS_C && !C::MERGE) mbar_wait(&fullC[iv % DC], (iv / DC) & 1);

#pragma unroll
      for (int k = 1; k <= BT; ++k) {
        const int c = s - k * R;
        // planes below s_begin + k*R are not valid at level k (unless the stream starts at plane 0).
        // Invalid steps still run the same straight-line code (no divergent branches) but read only
        // slots this step has already waited for, and their results are discarded by the select.
        const bool zv = !(p.dbg & 1) && c >= p.zi0 && c < p.zi1 && (it.s_begin == 0 || c >= it.s_begin + k * R);
        // x/y neighbour source, addressed as Sb[y * SS + x] in level-1-extent coordinates: level 1
        // reads the footprint box of plane s - R, level k >= 2 a shared level plane (TX x TY).
        const double* Sb;
        int SS;
        if (k == 1) {
          Sb = sV + (size_t)((zv ? iv - R : iv) % DV) * C::VSLOT + R * FXB + R + SHV;
          SS = FXB;
        } else {
          double* P = sP + (size_t)((k - 2) * 2 + buf) * C::PELEMS;
#pragma unroll
          for (int j = 0; j < CY; ++j) {
            double v[CXN];
#pragma unroll
            for (int i = 0; i < CXN; ++i) v[i] = ring[k - 1][j][i][ri(R)];
            sts_row<CXN, VEC>(P + (ly0 + j) * TX + x0, v);
          }
          if (!(p.dbg & 2)) named_sync(1, NCONS);
          if constexpr (CLU == 2) {
            if (k == BT && tid == 0) {
              // the boundary rows of levels 1..BT-1 (computed this step, staged, ordered by the barrier
              // above) go to the partner in one copy; this CTA expects the partner's rows of this step
              const uint32_t slot = iv & 3u;
              constexpr uint32_t bytes = (uint32_t)(C::NPL * C::XROW * sizeof(double));
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              mbar_expect_tx(&rxb[slot], bytes);
              bulk_copy_to_peer(dsmem_addr(sRx + (size_t)slot * C::NPL * C::XROW, crank ^ 1u),
                                sTx + (size_t)slot * C::NPL * C::XROW, bytes, dsmem_addr(&rxb[slot], crank ^ 1u));
              bulk_wait_read<2>();  // copies of two steps ago have read their staging slots
            }
          }
          Sb = P;
          SS = TX;
        }
        const double* Ck = sC + (size_t)((zv ? iv - (k - 1) * R : iv) % DC) * C::CSLOT + SHC;
        // y-strip: rows ly0 - R .. ly0 + CY + R - 1 of this thread's columns
        double ys[CY + 2 * R][CXN];
#pragma unroll
        for (int q = 0; q < CY + 2 * R; ++q) {
          int row = ly0 - R + q;
          if (k > 1) {
            if (CLU == 2 && ((crank == 0 && row >= TY) || (crank == 1 && row < 0))) {
              // across the pair's internal boundary: the partner's level-(k-1) row of this plane,
              // computed and pushed by it one step ago (receive slot (iv - 1) % 4)
              if (iv > 0) {
                const uint32_t slot = (iv - 1u) & 3u;
                mbar_wait_cluster(&rxb[slot], ((iv - 1u) >> 2) & 1u);
                lds_row<CXN, VEC>(sRx + ((size_t)slot * C::NPL + (k - 2)) * C::XROW + x0, ys[q]);
              } else {
#pragma unroll
                for (int i = 0; i < CXN; ++i) ys[q][i] = 0.0;  // the kernel's first step: never a valid plane
              }
              continue;
            }
            row = min(max(row, 0), TY - 1);  // level planes have no halo rows (outer side: discarded)
          }
          lds_row<CXN, VEC>(Sb + row * SS + x0, ys[q]);
        }
#pragma unroll
        for (int j = 0; j < CY; ++j) {
          const int ly = ly0 + j;
          // this row's x-neighbourhood: RP halo columns | the block's CX cells | RP halo columns
          double xr[RP + CXN + RP];
          lds_row<RP, VEC>(Sb + ly * SS + x0 - RP, xr);  // in shared memory even at the plane edges
          lds_row<RP, VEC>(Sb + ly * SS + x0 + CXN, xr + RP + CXN);
#pragma unroll
          for (int i = 0; i < CXN; ++i) xr[RP + i] = ys[R + j][i];
          double Wrow[NC > 0 ? NC : 1][CXN];
          if constexpr (NC > 0) {
            if (C::TW && k >= 2) {
              // level k: the coefficients of plane s - k*R, stored by level 1 (k-1)*R steps ago
              uint32_t w[32];
              tmem_ld32(tbase + (uint32_t)(((iv - (uint32_t)((k - 1) * R)) % C::NSL) * C::TSLOT + j * 32), w);
              tmem_wait_ld();
#pragma unroll
              for (int f = 0; f < NC; ++f)
#pragma unroll
                for (int i = 0; i < CXN; ++i) Wrow[f][i] = __hiloint2double(w[2 * (f * CXN + i) + 1], w[2 * (f * CXN + i)]);
            } else if (!(C::WINR && k > BT - C::WINR)) {
#pragma unroll
              for (int f = 0; f < NC; ++f)
                lds_row<CXN, VEC>(Ck + C::CF0 + f * C::CFIELD + ly * EXB + x0, Wrow[f]);
              if (C::TW && k == 1) {  // keep them for levels 2..BT
                uint32_t w[32];
#pragma unroll
                for (int q = 0; q < 32; ++q) w[q] = 0u;
#pragma unroll
                for (int f = 0; f < NC; ++f)
#pragma unroll
                  for (int i = 0; i < CXN; ++i) {
                    w[2 * (f * CXN + i)] = (uint32_t)__double2loint(Wrow[f][i]);
                    w[2 * (f * CXN + i) + 1] = (uint32_t)__double2hiint(Wrow[f][i]);
                  }
                tmem_st32(tbase + (uint32_t)((iv % C::NSL) * C::TSLOT + j * 32), w);
              }
            }
          }
          double urow[CXN];
          if constexpr (WAVE) {
            if (k == 1) lds_row<CXN, VEC>(Ck + ly * EXB + x0, urow);
          }
          double vout[CXN], uout[CXN];  // last level: the row's results, stored after the loop
#pragma unroll
          for (int i = 0; i < CXN; ++i) {
            double m[3][R], pl[3][R];
#pragma unroll
            for (int r = 1; r <= R; ++r) {
              m[0][r - 1] = xr[RP + i - r];
              pl[0][r - 1] = xr[RP + i + r];
              m[1][r - 1] = ys[R + j - r][i];
              pl[1][r - 1] = ys[R + j + r][i];
              m[2][r - 1] = ring[k - 1][j][i][ri(R - r)];
              pl[2][r - 1] = ring[k - 1][j][i][ri(R + r)];
            }
            double W[NC > 0 ? NC : 1];
            if constexpr (NC > 0) {
#pragma unroll
              for (int f = 0; f < NC; ++f)
                W[f] = (C::WINR && k > BT - C::WINR) ? cwin[L > 0 ? (BT - k) * R : 0][j][i][f] : Wrow[f][i];
            }
            double uo = 0.0;
            if constexpr (WAVE) uo = (k == 1) ? urow[i] : ring[k >= 2 ? k - 2 : 0][j][i][ri(0)];
            const double vc = apply_point<KIND, R>(ring[k - 1][j][i][ri(R)], uo, m, pl, W, ps);
            // ghosts and cells outside the level-k extent keep their input value.  At the last level
            // the store predicate below already implies the select's condition (outc -> act bit BT,
            // c in [zc0, zc1) -> zv), so the select is skipped there.
            const double v = (k == BT) ? vc : (zv && ((act[j][i] >> k) & 1u)) ? vc : ring[k - 1][j][i][ri(R)];
            if (CLU == 2 && k < BT && (crank == 0 ? ly == TY - 1 : ly == 0))  // stage the boundary row
              sTx[((size_t)(iv & 3u) * C::NPL + (k - 1)) * C::XROW + x0 + i] = v;
            if (k < BT) {
              if constexpr (UNR) {
                ring[k < BT ? k : 0][j][i][u % RL] = v;
              } else {
#pragma unroll
                for (int q = 0; q < RL - 1; ++q)
                  ring[k < BT ? k : 0][j][i][q] = ring[k < BT ? k : 0][j][i][q + 1];
                ring[k < BT ? k : 0][j][i][RL - 1] = v;
              }
            } else {
              vout[i] = v;
              if constexpr (WAVE && BT >= 2) uout[i] = ring[BT - 1][j][i][ri(R)];
            }
          }
          if (k == BT && c >= it.zc0 && c < it.zc1 && !((p.dbg & 4) && c == it.zc1 - 1)) {
            const long long o = (long long)c * p.plane + col[j];
            stg_row<CXN, VEC>(dst + o, vout, outc[j]);
            if constexpr (WAVE && BT >= 2) stg_row<CXN, VEC>(p.dstu + o, uout, outc[j]);
          }
        }
        if (k == 1 && iv >= iv_b + R) {  // footprint plane of step iv - R fully consumed
          __syncwarp();
          if (lane == 0) mbar_arrive(&emptyV[(iv - R) % DV]);
        }
      }
      if constexpr (C::TW) tmem_wait_st();  // this step's TMEM stores complete before later steps read them
      if constexpr (L > 0) {  // slide the window: drop plane s - BT*R, append plane s - (BT-WIN)*R
        // (before the item's first CLAG steps the window entry is never used; read a waited slot)
        const double* C1 = sC + (size_t)((iv >= iv_b + CLAG ? iv - CLAG : iv) % DC) * C::CSLOT + SHC;
#pragma unroll
        for (int j = 0; j < CY; ++j)
#pragma unroll
          for (int f = 0; f < NC; ++f) {
            double w[CXN];
            lds_row<CXN, VEC>(C1 + C::CF0 + f * C::CFIELD + (ly0 + j) * EXB + x0, w);
#pragma unroll
            for (int i = 0; i < CXN; ++i) {
#pragma unroll
              for (int q = 0; q < L - 1; ++q) cwin[q][j][i][f] = cwin[q + 1][j][i][f];
              cwin[L - 1][j][i][f] = w[i];
            }
          }
      }
      if (HAS_C && !C::MERGE && iv >= iv_b + CLAG) {  // C plane of step iv - CLAG fully consumed
        __syncwarp();
        if (lane == 0) mbar_arrive(&emptyC[(iv - CLAG) % DC]);
      }
    }
    ++iv;
    }
    }
    // release ring slots of this item that the lags above did not reach
    __syncwarp();
    if (lane == 0) {
      for (uint32_t i = (iv >= iv_b + R ? iv - R : iv_b); i < iv; ++i) mbar_arrive(&emptyV[i % DV]);
      if (HAS_C && !C::MERGE)
        for (uint32_t i = (iv >= iv_b + CLAG ? iv - CLAG : iv_b); i < iv; ++i) mbar_arrive(&emptyC[i % DC]);
    }
    // Fused halo exchange (ST_HALO_PEER): the item's output planes that are a
    // z-neighbour's halo planes go straight into the neighbour's buffer (peer memory over NVLink, or
    // another slab on this device) as soon as the item is done -- each thread forwards the cells it
    // stored itself (program order: its own stores are visible to its loads; they hit L2), so the hot
    // z-loop above is the same code with or without the exchange.
#pragma unroll 1
    for (int q = 0; q < 2; ++q) {
      if (!p.rdst[q]) continue;
      const int c0 = max(it.zc0, p.rz0[q]), c1 = min(it.zc1, p.rz1[q]);
#pragma unroll 1
      for (int c = c0; c < c1; ++c) {
        if ((p.dbg & 4) && c == it.zc1 - 1) continue;  // fault injection: a plane never written
#pragma unroll
        for (int j = 0; j < CY; ++j) {
          const long long o = (long long)c * p.plane + col[j];
#pragma unroll
          for (int i = 0; i < CXN; i += (VEC ? 2 : 1)) {
            if (VEC && outc[j][i] && outc[j][i + 1 < CXN ? i + 1 : i]) {  // 16-byte aligned pair (see stg_row)
              *reinterpret_cast<double2*>(p.rdst[q] + o + i) = __ldcg(reinterpret_cast<const double2*>(dst + o + i));
              if constexpr (WAVE && BT >= 2)
                *reinterpret_cast<double2*>(p.rdstu[q] + o + i) =
                    __ldcg(reinterpret_cast<const double2*>(p.dstu + o + i));
              continue;
            }
#pragma unroll
            for (int e = 0; e < (VEC ? 2 : 1); ++e)
              if (i + e < CXN && outc[j][i + e]) {
                p.rdst[q][o + i + e] = __ldcg(dst + o + i + e);
                if constexpr (WAVE && BT >= 2) p.rdstu[q][o + i + e] = __ldcg(p.dstu + o + i + e);
              }
          }
        }
      }
    }
    if (p.nblk > 1) {  // publish: this item of block blk is complete (all consumers' stores)
      named_sync(1, NCONS);
      if (tid == 0) {
        __threadfence();
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p.done + item), "r"(p.dbase + (unsigned int)blk + 1u)
                     : "memory");
      }
    }
  }
  // peer stores of another process's memory are ordered before the stream's completion signal
  if (p.rfence) __threadfence_system();
  if constexpr (C::TW) {  // all consumers are done with TMEM; warp 0 frees it
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    named_sync(1, NCONS);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
  }
  if constexpr (CLU == 2) cluster_sync_all();  // the partner may still read this CTA's level planes
}

// ------------------------------------------------------------------------------------------------ host

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

// rank-3 (x, y, z) or rank-4 (x, y, z, field) map of fp64 padded arrays in the library's layout
// The map starts at raw column kX0 of each row and is X columns wide: the row padding beyond the padded
// extent is out of bounds (zero-filled by the TMA unit, no DRAM traffic), not loaded.
bool make_tensor_map(CUtensorMap* m, const double* base, int rank, long long pitch, long long X, long long Y, long long zl,
              long long nfields, long long plane, long long fstride, int bx, int by, int bf) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[4] = {(cuuint64_t)X, (cuuint64_t)Y, (cuuint64_t)zl, (cuuint64_t)nfields};
  cuuint64_t strides[3] = {(cuuint64_t)pitch * 8, (cuuint64_t)plane * 8, (cuuint64_t)fstride * 8};
  cuuint32_t box[4] = {(cuuint32_t)bx, (cuuint32_t)by, 1, (cuuint32_t)bf};
  cuuint32_t es[4] = {1, 1, 1, 1};
  // L2 promotion: experiment knob STENCIL_TMA_PROMO = 0 (none), 1 (64B), 2 (128B), 3 (256B)
  static int promo = [] {
    const char* e = getenv("STENCIL_TMA_PROMO");
    return e ? atoi(e) : 0;
  }();
  const CUtensorMapL2promotion pr = promo == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                   : promo == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                   : promo == 3 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                                                : CU_TENSOR_MAP_L2_PROMOTION_NONE;
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<double*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, pr, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

namespace {

template <int KIND, int BT, int TX, int TY, int CX, int CY, int DV, int DC, int WIN = 0, int MINB = 1, bool UNR = false,
          int CLU = 1>
cudaError_t run_pipe(const KParams& p0, int zchunk_req, int num_sms, cudaStream_t stream, LaunchInfo* info) {
  using C = PipeCfg<KIND, BT, TX, TY, CX, CY, DV, DC, WIN, MINB, UNR, CLU>;
  auto kern = pipe_kernel<KIND, BT, TX, TY, CX, CY, DV, DC, WIN, MINB, UNR, CLU>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  KParams p = p0;
  if (p.nblk < 1) p.nblk = 1;
  const int planes = p.zo1 - p.zo0;
  if (planes <= 0) return cudaSuccess;
  if (p.xoff != 16 - C::R) return cudaErrorInvalidValue;  // decode() assumes interior column R at raw 16
  const int oxw = p.walign ? C::OXW : C::OX;
  const int dx = p.walign ? 0 : ((C::R - C::R * (BT - 1) + p.xoff) & 1);
  const int ntx = (p.nx + dx + oxw - 1) / oxw, nty = (p.ny + C::OYP - 1) / C::OYP;
  const long long tiles = (long long)ntx * nty;
  int zchunk = zchunk_req;
  if (zchunk <= 0) {
    int occ0 = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ0, kern, C::THREADS, C::SMEM);
    const long long slots = (long long)std::max(1, occ0) * num_sms;
    const int min_chunk = 24 * BT * C::R;  // keeps the 2*BT*R fill/drain planes of a chunk < ~8 %
    if (tiles * ((planes + min_chunk - 1) / min_chunk) >= 2 * slots) {
      // large grid: ~4 work items per CTA for load balance (dynamic distribution), chunks >= min_chunk
      // planes (tools/tune.py, session 2: 4 items beat 8 for the 25-point kinds -- each chunk re-reads
      // its 2*BT*R halo planes -- and tie for the 7-point kinds)
      const long long chunks = std::max<long long>(1, (4 * slots + tiles - 1) / tiles);
      zchunk = std::max((int)((planes + chunks - 1) / chunks), std::min(planes, min_chunk));
    } else {
      // small grid (latency-bound): about one work item per CTA slot
      zchunk = (int)std::max<long long>(2, (planes * tiles + slots - 1) / slots);
    }
  }
  p.zchunk = zchunk;
  const int nzc = (planes + zchunk - 1) / zchunk;
  p.nzc = nzc;
  const long long items = tiles * nzc;
  CUtensorMap mapV, mapC, mapA;
  memset(&mapC, 0, sizeof mapC);
  memset(&mapA, 0, sizeof mapA);
  // TMA x coordinate 0 = raw column X0 (even, so the map base stays 16-byte aligned); the row's last
  // column is the padded extent's (raw xoff + nx + 2R - 1)
  const int X0 = p.xoff & ~1;
  const long long MX = p.xoff + p.nx + 2 * C::R - X0, MY = p.ny + 2 * C::R;
  if (!make_tensor_map(&mapV, p.src_raw + X0, 3, p.pitch, MX, MY, p.zl, 1, p.plane, 0, C::FXB, C::FY, 1))
    return cudaErrorInvalidValue;
  if (!C::WAVE && p.nblk > 1 &&  // multi-block launch: the V box of odd blocks comes from the other buffer
      !make_tensor_map(&mapA, p.dst_raw + X0, 3, p.pitch, MX, MY, p.zl, 1, p.plane, 0, C::FXB, C::FY, 1))
    return cudaErrorInvalidValue;
  if (C::HAS_C) {
    bool ok = C::WAVE ? make_tensor_map(&mapC, p.srcu_raw + X0, 3, p.pitch, MX, MY, p.zl, 1, p.plane, 0, C::EXB, TY, 1)
                      : make_tensor_map(&mapC, p.coef_raw + X0, 4, p.pitch, MX, MY, p.zl, C::NC, p.plane, p.cstride,
                                 C::EXB, TY, C::NC);
    if (ok && C::WAVE && C::NC > 0)
      ok = make_tensor_map(&mapA, p.coef_raw + X0, 4, p.pitch, MX, MY, p.zl, C::NC, p.plane, p.cstride, C::EXB, TY, C::NC);
    if (!ok) return cudaErrorInvalidValue;
  }
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::THREADS, C::SMEM);
  int grid = (int)std::min<long long>(items * std::max(1, p.nblk), (long long)std::max(1, occ) * num_sms);
  // single-block launches of single-CTA tiles: lockstep rounds over compact patches of tiles, so the
  // overlapping halo boxes of y-neighbours are streamed at the same time and hit L2 (STENCIL_SCHED=0:
  // dynamic work counter, row-major tiles)
  static const int l2h_env = getenv("STENCIL_L2H") ? atoi(getenv("STENCIL_L2H")) : 0;
  p.l2h = l2h_env;
  static const int sched_env = getenv("STENCIL_SCHED") ? atoi(getenv("STENCIL_SCHED")) : 1;
  if (CLU == 1 && sched_env && p.nblk <= 1 && p.tband == 0 && occ <= 1) {
    p.lockstep = 1;
    static const int bw_env = getenv("STENCIL_TILE_BLOCK") ? atoi(getenv("STENCIL_TILE_BLOCK")) : 0;
    // blocks of about sqrt(grid * OY / OX) tile columns, sized so that a tile row splits into equal blocks
    const double target = std::sqrt((double)grid * C::OYP / oxw);
    const int nb = std::max(1, (int)(ntx / target + 0.5));
    int bw = bw_env > 0 ? bw_env : (ntx + nb - 1) / nb;
    bw = std::max(1, std::min(bw, ntx));
    p.tblk_w = bw;
    p.tblk_h = std::max(1, (grid + bw - 1) / bw);
  }
  if (p.nblk > 1 && (C::WAVE || CLU != 1 || items > kMaxDoneItems || !p.done)) return cudaErrorInvalidValue;
  if constexpr (CLU == 1) {
    kern<<<grid, C::THREADS, C::SMEM, stream>>>(mapV, mapC, mapA, p, ntx, nty, (int)items);
  } else {
    // clusters of CLU CTAs along x of the grid (consecutive blockIdx.x), static item schedule per cluster
    grid = (int)std::min<long long>((long long)items * CLU, (long long)std::max(1, occ) * num_sms / CLU * CLU);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(C::THREADS);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CLU;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const int it32 = (int)items;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, mapV, mapC, mapA, p, ntx, nty, it32);
    if (e != cudaSuccess) return e;
  }
  if (info) {
    info->tile_x = oxw; info->tile_y = C::OYP; info->zchunk = zchunk; info->threads = C::THREADS;
    info->smem = (int)C::SMEM; info->ctas = grid;
  }
  return cudaGetLastError();
}

}  // namespace

int max_pipe_bt(int kind) {
  switch (kind) {
    case K7C: return 8;
    case K7V: return 5;
    case K25W: return 2;
    case K25WA: return 1;
    case K25V: return 2;  // bt = 2: pipe25.cu
    default: return 0;
  }
}

// Tile configurations <KIND, BT, TX, TY, CX, CY, DV, DC, WIN, MINB>: level-1 extent TX x TY, cell
// blocks of CX x CY per consumer thread, V / coefficient ring depths, coefficient window of the levels
// >= 2 (0: shared ring, k > 0: register window for the last k levels, -1: TMEM window), CTAs per SM.
// The last entry of each (kind, bt) is the default (tile_cfg 0); the others are the alternatives the
// sweeps in profiles/ compare (all bitwise equal, test G4).  Shared memory per CTA stays below the
// 227 KB opt-in limit (DESIGN.md §5 lists each budget).  At BT = 1 the coefficient box equals the output
// tile, and TX = 32 / 64 puts its rows on 128-byte lines (interior column x = R is 128-byte aligned).
cudaError_t launch_pipe(int kind, int b, const KParams& p, int zchunk_req, int num_sms, int cfg,
                        cudaStream_t stream, LaunchInfo* info) {
  // CFG(kind, BT, TX, TY, CX, CY, DV, DC, WIN, MINB)
#define CFG(K, B, TX, TY, CX, CY, DV, DC, W, M) \
  return run_pipe<K, B, TX, TY, CX, CY, DV, DC, W, M>(p, zchunk_req, num_sms, stream, info)
  // CFGU: the same with the z-loop unrolled by the ring length (rings rotate by renaming)
#define CFGU(K, B, TX, TY, CX, CY, DV, DC, W, M) \
  return run_pipe<K, B, TX, TY, CX, CY, DV, DC, W, M, true>(p, zchunk_req, num_sms, stream, info)
  // CFGC: unrolled, cluster pair (two CTAs share one TX x 2TY tile through DSMEM)
#define CFGC(K, B, TX, TY, CX, CY, DV, DC, W, M) \
  return run_pipe<K, B, TX, TY, CX, CY, DV, DC, W, M, true, 2>(p, zchunk_req, num_sms, stream, info)
  // Consumer-thread counts are kept at <= 224 (+ 32 producer = 256 threads) where registers matter:
  // ptxas budgets registers for blocks rounded up to 128 threads (288-thread blocks get 168).
  switch (kind) {
    case K7C:
      switch (b) {
        case 1: CFG(K7C, 1, 32, 28, 1, 4, 6, 2, 0, 1);
        case 2: CFG(K7C, 2, 32, 28, 1, 4, 6, 2, 0, 1);
        case 3: CFG(K7C, 3, 32, 28, 1, 4, 6, 2, 0, 1);
        case 4: CFG(K7C, 4, 32, 28, 1, 4, 6, 2, 0, 1);
        case 5: CFG(K7C, 5, 32, 28, 1, 4, 6, 2, 0, 1);
        case 6: CFG(K7C, 6, 32, 28, 1, 4, 6, 2, 0, 1);
        case 7: CFG(K7C, 7, 32, 28, 1, 4, 6, 2, 0, 1);
        case 8: CFG(K7C, 8, 32, 28, 1, 4, 6, 2, 0, 1);
      }
      break;
    case K7V:
      switch (b) {
        case 1:
          if (cfg == 1) CFG(K7V, 1, 32, 28, 2, 2, 4, 3, 0, 1);
          CFG(K7V, 1, 32, 32, 1, 4, 4, 3, 0, 1);
        case 2:
          if (cfg == 1) CFG(K7V, 2, 32, 28, 2, 2, 4, 3, 1, 1);
          if (cfg == 2) CFG(K7V, 2, 32, 28, 1, 4, 4, 3, 0, 1);
          if (cfg == 3) CFG(K7V, 2, 32, 28, 1, 4, 4, 3, 1, 1);  // round-1 default (rings shifted)
          if (cfg == 4) CFGU(K7V, 2, 32, 28, 2, 2, 4, 3, -1, 1);  // TMEM coefficient window
          CFGU(K7V, 2, 32, 28, 1, 4, 4, 3, 1, 1);                // C2: 148-151 -> 157-159 GLUP/s
        case 3:
          if (cfg == 1) CFG(K7V, 3, 32, 28, 1, 4, 4, 3, 1, 1);
          if (cfg == 2) CFG(K7V, 3, 32, 20, 1, 4, 4, 4, 0, 1);
          if (cfg == 3) CFGU(K7V, 3, 32, 28, 2, 2, 4, 3, 1, 1);
          if (cfg == 4) CFGU(K7V, 3, 32, 28, 1, 2, 4, 3, 1, 1);
          if (cfg == 5) CFG(K7V, 3, 32, 28, 1, 2, 4, 3, 1, 1);
          if (cfg == 6) CFGU(K7V, 3, 32, 24, 1, 2, 4, 3, 1, 1);
          if (cfg == 7) CFG(K7V, 3, 32, 28, 2, 2, 4, 3, 1, 1);   // session-1 default (register window)
          if (cfg == 8) CFG(K7V, 3, 32, 28, 2, 2, 4, 3, -1, 1);
          if (cfg == 9) CFGC(K7V, 3, 32, 28, 2, 2, 4, 3, -1, 1);  // cluster pair: 32 x 56 tile
          // TMEM coefficient window for levels 2..3 (WIN = -1): C2 bt=3 163-168 -> 184-192 GLUP/s
          CFGU(K7V, 3, 32, 28, 2, 2, 4, 3, -1, 1);
        case 4:  // TMEM coefficient window only (the ring would need (bt-1)*R more slots otherwise)
          if (cfg == 1) CFGU(K7V, 4, 32, 24, 2, 2, 4, 3, -1, 1);  // session-2 default
          if (cfg == 2) CFG(K7V, 4, 32, 24, 2, 2, 4, 3, -1, 1);
          if (cfg == 3) CFGC(K7V, 4, 32, 24, 2, 2, 4, 3, -1, 1);  // cluster pair: 32 x 48 tile
          if (cfg == 4) CFGC(K7V, 4, 32, 28, 2, 2, 4, 2, -1, 1);  // cluster pair: 32 x 56 tile
          // 7 consumer warps, 2-slot coefficient ring (lookahead 1): 199 -> 202 GLUP/s (session 3)
          CFGU(K7V, 4, 32, 28, 2, 2, 4, 2, -1, 1);
        case 5:  // TMEM window of 5 slots: 2x1 cells so that 3 warps per lane quadrant fit 480 columns
          if (cfg == 1) CFG(K7V, 5, 32, 24, 2, 1, 4, 2, -1, 1);
          CFGU(K7V, 5, 32, 24, 2, 1, 4, 2, -1, 1);
      }
      break;
    case K25W:
      if (b == 1) {
        if (cfg == 1) CFG(K25W, 1, 64, 14, 4, 1, 7, 3, 0, 1);
        if (cfg == 2) CFG(K25W, 1, 32, 28, 2, 2, 7, 3, 0, 1);
        if (cfg == 3) CFG(K25W, 1, 64, 16, 1, 4, 7, 3, 0, 1);
        if (cfg == 4) CFG(K25W, 1, 64, 14, 2, 2, 7, 3, 0, 1);  // round-1 default (rings shifted)
        if (cfg == 5) CFG(K25W, 1, 64, 14, 2, 2, 10, 6, 0, 1);
        if (cfg == 6) CFGU(K25W, 1, 64, 14, 2, 2, 10, 6, 0, 1);
        if (cfg == 7) CFGU(K25W, 1, 64, 20, 2, 2, 8, 4, 0, 1);
        if (cfg == 8) CFGU(K25W, 1, 64, 14, 2, 2, 8, 4, 0, 1);
        CFGU(K25W, 1, 64, 14, 2, 2, 8, 8, 0, 1);  // merged V/U rings; C3: 165-169 (round 1) -> 185-196 GLUP/s
      }
      if (b == 2) {  // the leapfrog with two fused levels: both time levels in, both out (32 B/cell)
        // round 2: the two-level kernel of pipe25.cu (TMEM z-rings, 24 x 24 tiles) by default; the
        // round-1 generic kernel (register rings, 24 x 16 tiles) as tile_cfg 1 / 2
        if (cfg == 1) CFGU(K25W, 2, 32, 24, 2, 2, 7, 3, 0, 1);
        if (cfg == 2) CFG(K25W, 2, 32, 24, 2, 2, 7, 3, 0, 1);
        return launch_pipe25w2(p, zchunk_req, num_sms, 0, stream, info);
      }
      break;
    case K25WA:
      if (b == 1) {
        if (cfg == 1) CFG(K25WA, 1, 64, 16, 1, 4, 7, 3, 0, 1);
        if (cfg == 2) CFG(K25WA, 1, 64, 14, 2, 2, 7, 3, 0, 1);  // round-1 default (rings shifted)
        if (cfg == 3) CFGU(K25WA, 1, 64, 20, 2, 2, 8, 4, 0, 1);
        if (cfg == 4) CFGU(K25WA, 1, 64, 14, 2, 2, 8, 4, 0, 1);
        CFGU(K25WA, 1, 64, 14, 2, 2, 8, 8, 0, 1);  // merged rings; C3A: 148-152 (round 1) -> 172-179 GLUP/s
      }
      break;
    case K25V:
      if (b == 1) {
        if (cfg == 1) CFG(K25V, 1, 64, 8, 1, 2, 6, 3, 0, 1);
        if (cfg == 2) CFG(K25V, 1, 64, 8, 4, 1, 6, 3, 0, 1);
        if (cfg == 3) CFGU(K25V, 1, 64, 8, 2, 2, 6, 3, 0, 1);
        CFG(K25V, 1, 64, 8, 2, 2, 6, 3, 0, 1);
      }
      if (b == 2) return launch_pipe25v2(p, zchunk_req, num_sms, cfg, stream, info);  // pipe25.cu
      break;
  }
#undef CFG
#undef CFGU
#undef CFGC
  return cudaErrorInvalidValue;
}

}  // namespace st
