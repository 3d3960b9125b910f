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
//    so the producer prefetches the next item while consumers finish the current one.
//
// Results are bitwise identical to naive_kernel / stream_kernel (same point functions, point.cuh).
#include "kernels.cuh"
#include "point.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

namespace st {

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n"
      "DONE:\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int x,
                                            int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int x,
                                            int y, int z, int w) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z), "r"(w)
      : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

struct Item {
  int gx0, gy0, zc0, zc1, s_begin, s_end;
};

template <int R, int BT, int OX, int OY>
__device__ __forceinline__ Item decode(int item, int ntx, int nty, const KParams& p) {
  const int per = ntx * nty;
  const int zc = item / per, t = item - zc * per;
  const int ty = t / ntx, tx = t - ty * ntx;
  Item it;
  it.gx0 = tx * OX + R - R * BT;
  it.gy0 = ty * OY + R - R * BT;
  it.zc0 = p.zo0 + zc * p.zchunk;
  it.zc1 = min(p.zo1, it.zc0 + p.zchunk);
  it.s_begin = max(0, it.zc0 - BT * R);
  it.s_end = it.zc1 - 1 + BT * R;
  return it;
}

}  // namespace

// FX x FY footprint, consumer threads own CY-cell vertical strips; DV / DC = ring depths.
template <int KIND, int BT, int FX, int FY, int CY, int DV, int DC>
struct PipeCfg {
  using TR = Traits<KIND>;
  static constexpr int R = TR::R, NC = TR::NCOEF, RL = 2 * R + 1;
  static constexpr bool WAVE = TR::WAVE;
  static constexpr int NS = FY / CY;
  static constexpr int NCONS = FX * NS;
  static constexpr int THREADS = NCONS + 32;
  static constexpr int EX = FX - 2 * R, EY = FY - 2 * R;
  static constexpr int OX = FX - 2 * R * BT, OY = FY - 2 * R * BT;
  static constexpr int NCF = WAVE ? 1 : NC;  // fields in the C ring (coefficients, or U for the wave)
  static constexpr bool HAS_C = NCF > 0;
  static constexpr int VELEMS = FX * FY, CELEMS = EX * EY * NCF;
  static constexpr int CSLOT = (CELEMS + 15) / 16 * 16;  // C-ring slot stride: 128-byte aligned
  static constexpr int NPL = BT - 1;  // shared level planes (double-buffered)
  static constexpr size_t SMEM = sizeof(double) * ((size_t)DV * VELEMS + (HAS_C ? (size_t)DC * CSLOT : 0) +
                                                   (size_t)NPL * 2 * VELEMS) +
                                 sizeof(uint64_t) * 2 * (DV + DC) + 128;
  static_assert(FY % CY == 0, "strips");
  static_assert(OX > 0 && OY > 0, "footprint too small for BT");
  static_assert(NCONS % 32 == 0, "whole consumer warps");
  static_assert(DV >= R + 2, "V ring too shallow");
  static_assert(!HAS_C || DC >= (WAVE ? 0 : (BT - 1) * R) + 2, "C ring too shallow");
  static_assert((EX * 8) % 16 == 0 && (FX * 8) % 16 == 0, "TMA box rows must be 16-byte multiples");
};

template <int KIND, int BT, int FX, int FY, int CY, int DV, int DC>
__global__ void __launch_bounds__(PipeCfg<KIND, BT, FX, FY, CY, DV, DC>::THREADS, 1)
    pipe_kernel(const __grid_constant__ CUtensorMap mapV, const __grid_constant__ CUtensorMap mapC,
                const KParams p, int ntx, int nty, int items) {
  using C = PipeCfg<KIND, BT, FX, FY, CY, DV, DC>;
  constexpr int R = C::R, NC = C::NC, RL = C::RL, EX = C::EX, NCONS = C::NCONS;
  constexpr bool WAVE = C::WAVE, HAS_C = C::HAS_C;
  constexpr int OX = C::OX, OY = C::OY;
  constexpr int CLAG = WAVE ? 0 : (BT - 1) * R;  // steps a C-ring plane stays in use

  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sV = reinterpret_cast<double*>(smem_raw);
  double* sC = sV + (size_t)DV * C::VELEMS;
  double* sP = sC + (HAS_C ? (size_t)DC * C::CSLOT : 0);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + (size_t)C::NPL * 2 * C::VELEMS);
  uint64_t* fullV = bars;
  uint64_t* emptyV = bars + DV;
  uint64_t* fullC = bars + 2 * DV;
  uint64_t* emptyC = bars + 2 * DV + DC;

  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < DV; ++i) { mbar_init(&fullV[i], 1); mbar_init(&emptyV[i], NCONS / 32); }
    for (int i = 0; i < DC; ++i) { mbar_init(&fullC[i], 1); mbar_init(&emptyC[i], NCONS / 32); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (tid >= NCONS) {
    // ---------------------------------------------------------------- producer warp
    if (tid == NCONS) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mapV) : "memory");
      if (HAS_C) asm volatile("prefetch.tensormap [%0];" ::"l"(&mapC) : "memory");
      uint32_t iv = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const Item it = decode<R, BT, OX, OY>(item, ntx, nty, p);
        for (int s = it.s_begin; s <= it.s_end; ++s, ++iv) {
          const uint32_t sv = iv % DV, nv = iv / DV;
          mbar_wait(&emptyV[sv], (nv & 1) ^ 1);
          mbar_expect_tx(&fullV[sv], C::VELEMS * sizeof(double));
          tma_load_3d(sV + (size_t)sv * C::VELEMS, &mapV, &fullV[sv], it.gx0 + p.xoff, it.gy0, s);
          if constexpr (HAS_C) {
            const uint32_t sc = iv % DC, nc = iv / DC;
            mbar_wait(&emptyC[sc], (nc & 1) ^ 1);
            mbar_expect_tx(&fullC[sc], C::CELEMS * sizeof(double));
            if constexpr (WAVE)
              tma_load_3d(sC + (size_t)sc * C::CSLOT, &mapC, &fullC[sc], it.gx0 + R + p.xoff, it.gy0 + R, s - R);
            else
              tma_load_4d(sC + (size_t)sc * C::CSLOT, &mapC, &fullC[sc], it.gx0 + R + p.xoff, it.gy0 + R, s - R, 0);
          }
        }
      }
    }
    return;
  }

  // ---------------------------------------------------------------- consumers
  const int lx = tid % FX;
  const int ly0 = (tid / FX) * CY;
  const int lane = tid & 31;
  const int X = p.nx + 2 * R, Y = p.ny + 2 * R;
  (void)X; (void)Y;
  uint32_t iv = 0;

  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    const Item it = decode<R, BT, OX, OY>(item, ntx, nty, p);
    const int gx = it.gx0 + lx;
    const bool xin = gx >= R && gx < p.nx + R;
    bool inter[CY], outc[CY];
    unsigned lvl[CY];
    long long col[CY];
#pragma unroll
    for (int j = 0; j < CY; ++j) {
      const int ly = ly0 + j, gy = it.gy0 + ly;
      inter[j] = xin && gy >= R && gy < p.ny + R;
      lvl[j] = 0;
#pragma unroll
      for (int k = 1; k <= BT; ++k)
        if (lx >= k * R && lx < FX - k * R && ly >= k * R && ly < FY - k * R) lvl[j] |= 1u << k;
      outc[j] = inter[j] && ((lvl[j] >> BT) & 1u);
      col[j] = (long long)gy * p.pitch + gx;
    }
    double ring[BT][CY][RL];
#pragma unroll
    for (int k = 0; k < BT; ++k)
#pragma unroll
      for (int j = 0; j < CY; ++j)
#pragma unroll
        for (int i = 0; i < RL; ++i) ring[k][j][i] = 0.0;

    const uint32_t iv_b = iv;
    for (int s = it.s_begin; s <= it.s_end; ++s, ++iv) {
      const int buf = s & 1;
      // Level 0: plane s of Omega^t -> register rings.
      const uint32_t sv = iv % DV;
      mbar_wait(&fullV[sv], (iv / DV) & 1);
      const double* Vs = sV + (size_t)sv * C::VELEMS;
#pragma unroll
      for (int j = 0; j < CY; ++j) {
        const double v = Vs[(ly0 + j) * FX + lx];
#pragma unroll
        for (int i = 0; i < RL - 1; ++i) ring[0][j][i] = ring[0][j][i + 1];
        ring[0][j][RL - 1] = v;
      }
      if constexpr (HAS_C) mbar_wait(&fullC[iv % DC], (iv / DC) & 1);

#pragma unroll
      for (int k = 1; k <= BT; ++k) {
        const int c = s - k * R;
        const double* Src;
        if (k == 1) {
          Src = sV + (size_t)((iv - R) % DV) * C::VELEMS;
        } else {
          double* P = sP + (size_t)((k - 2) * 2 + buf) * C::VELEMS;
#pragma unroll
          for (int j = 0; j < CY; ++j) P[(ly0 + j) * FX + lx] = ring[k - 1][j][R];
          named_sync(1, NCONS);
          Src = P;
        }
        // planes below s_begin + k*R are not valid at level k (unless the stream starts at plane 0)
        const bool zv = c >= p.zi0 && c < p.zi1 && (it.s_begin == 0 || c >= it.s_begin + k * R);
        const double* Ck = sC + (size_t)((iv - (k - 1) * R) % DC) * C::CSLOT;
        double ys[CY + 2 * R];
        if (zv) {
#pragma unroll
          for (int i = 0; i < CY + 2 * R; ++i) {
            const int row = min(max(ly0 - R + i, 0), FY - 1);
            ys[i] = Src[row * FX + lx];
          }
        }
#pragma unroll
        for (int j = 0; j < CY; ++j) {
          double v = ring[k - 1][j][R];
          if (zv && inter[j] && ((lvl[j] >> k) & 1u)) {
            const int ly = ly0 + j;
            double m[3][R], pl[3][R];
            const double* row = Src + ly * FX + lx;
#pragma unroll
            for (int r = 1; r <= R; ++r) {
              m[0][r - 1] = row[-r];
              pl[0][r - 1] = row[r];
              m[1][r - 1] = ys[R + j - r];
              pl[1][r - 1] = ys[R + j + r];
              m[2][r - 1] = ring[k - 1][j][R - r];
              pl[2][r - 1] = ring[k - 1][j][R + r];
            }
            const int ci = (ly - R) * EX + (lx - R);
            double W[NC > 0 ? NC : 1];
            if constexpr (NC > 0) {
#pragma unroll
              for (int f = 0; f < NC; ++f) W[f] = Ck[f * (C::CELEMS / C::NCF) + ci];
            }
            double u = 0.0;
            if constexpr (WAVE) u = (k == 1) ? Ck[ci] : ring[k >= 2 ? k - 2 : 0][j][0];
            v = apply_point<KIND, R>(ring[k - 1][j][R], u, m, pl, W, p.s);
          }
          if (k < BT) {
#pragma unroll
            for (int i = 0; i < RL - 1; ++i) ring[k < BT ? k : 0][j][i] = ring[k < BT ? k : 0][j][i + 1];
            ring[k < BT ? k : 0][j][RL - 1] = v;
          } else if (outc[j] && c >= it.zc0 && c < it.zc1) {
            const long long o = (long long)c * p.plane + col[j];
            __stcs(p.dst + o, v);
            if constexpr (WAVE && BT >= 2) __stcs(p.dstu + o, ring[BT - 1][j][R]);
          }
        }
        if (k == 1 && iv >= iv_b + R) {  // V plane of step iv - R fully consumed
          __syncwarp();
          if (lane == 0) mbar_arrive(&emptyV[(iv - R) % DV]);
        }
        if (HAS_C && k == BT && iv >= iv_b + CLAG) {  // C plane of step iv - CLAG fully consumed
          __syncwarp();
          if (lane == 0) mbar_arrive(&emptyC[(iv - CLAG) % DC]);
        }
      }
    }
    // release ring slots of this item that the lags above did not reach
    __syncwarp();
    if (lane == 0) {
      for (uint32_t i = (iv >= iv_b + R ? iv - R : iv_b); i < iv; ++i) mbar_arrive(&emptyV[i % DV]);
      if (HAS_C)
        for (uint32_t i = (iv >= iv_b + CLAG ? iv - CLAG : iv_b); i < iv; ++i) mbar_arrive(&emptyC[i % DC]);
    }
  }
}

// ------------------------------------------------------------------------------------------------ host
namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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
bool make_map(CUtensorMap* m, const double* base, int rank, long long pitch, long long Y, long long zl,
              long long nfields, long long plane, long long fstride, int bx, int by, int bf) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[4] = {(cuuint64_t)pitch, (cuuint64_t)Y, (cuuint64_t)zl, (cuuint64_t)nfields};
  cuuint64_t strides[3] = {(cuuint64_t)pitch * 8, (cuuint64_t)plane * 8, (cuuint64_t)fstride * 8};
  cuuint32_t box[4] = {(cuuint32_t)bx, (cuuint32_t)by, 1, (cuuint32_t)bf};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<double*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int KIND, int BT, int FX, int FY, int CY, int DV, int DC>
cudaError_t run_pipe(const KParams& p0, int zchunk_req, int num_sms, cudaStream_t stream, LaunchInfo* info) {
  using C = PipeCfg<KIND, BT, FX, FY, CY, DV, DC>;
  auto kern = pipe_kernel<KIND, BT, FX, FY, CY, DV, DC>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  KParams p = p0;
  const int planes = p.zo1 - p.zo0;
  if (planes <= 0) return cudaSuccess;
  const int ntx = (p.nx + C::OX - 1) / C::OX, nty = (p.ny + C::OY - 1) / C::OY;
  const long long tiles = (long long)ntx * nty;
  int zchunk = zchunk_req;
  if (zchunk <= 0) {
    // >= ~8 work items per CTA for load balance, chunks >= 12x the 2*BT*R fill/drain planes
    int occ0 = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ0, kern, C::THREADS, C::SMEM);
    const long long chunks = std::max<long long>(1, (8LL * std::max(1, occ0) * num_sms + tiles - 1) / tiles);
    zchunk = (int)((planes + chunks - 1) / chunks);
    zchunk = std::max(zchunk, std::min(planes, 24 * BT * C::R));
  }
  p.zchunk = zchunk;
  const int nzc = (planes + zchunk - 1) / zchunk;
  const long long items = tiles * nzc;
  CUtensorMap mapV, mapC;
  memset(&mapC, 0, sizeof mapC);
  if (!make_map(&mapV, p.src_raw, 3, p.pitch, p.ny + 2 * C::R, p.zl, 1, p.plane, 0, FX, FY, 1))
    return cudaErrorInvalidValue;
  if (C::HAS_C) {
    bool ok = C::WAVE ? make_map(&mapC, p.srcu_raw, 3, p.pitch, p.ny + 2 * C::R, p.zl, 1, p.plane, 0, C::EX, C::EY, 1)
                      : make_map(&mapC, p.coef_raw, 4, p.pitch, p.ny + 2 * C::R, p.zl, C::NC, p.plane, p.cstride,
                                 C::EX, C::EY, C::NC);
    if (!ok) return cudaErrorInvalidValue;
  }
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::THREADS, C::SMEM);
  const int grid = (int)std::min<long long>(items, (long long)std::max(1, occ) * num_sms);
  kern<<<grid, C::THREADS, C::SMEM, stream>>>(mapV, mapC, p, ntx, nty, (int)items);
  if (info) {
    info->tile_x = C::OX; info->tile_y = C::OY; info->zchunk = zchunk; info->threads = C::THREADS;
    info->smem = (int)C::SMEM; info->ctas = grid;
  }
  return cudaGetLastError();
}

}  // namespace

int max_pipe_bt(int kind) {
  switch (kind) {
    case K7C: return 8;
    case K7V: return 3;
    case K25W: return 1;
    case K25V: return 1;
    default: return 0;
  }
}

// Tile configurations: <KIND, BT, FX, FY, CY, DV, DC>.  Shared memory per CTA (see PipeCfg::SMEM)
// stays below the 227 KB opt-in limit; DESIGN.md §5 lists the budget of each.
cudaError_t launch_pipe(int kind, int b, const KParams& p, int zchunk_req, int num_sms, int cfg,
                        cudaStream_t stream, LaunchInfo* info) {
#define PIPE(K, B, FX, FY, CY, DV, DC) return run_pipe<K, B, FX, FY, CY, DV, DC>(p, zchunk_req, num_sms, stream, info)
  switch (kind) {
    case K7C:
      switch (b) {
        case 1: PIPE(K7C, 1, 32, 32, 4, 6, 2);
        case 2: PIPE(K7C, 2, 32, 32, 4, 6, 2);
        case 3: PIPE(K7C, 3, 32, 32, 4, 6, 2);
        case 4: PIPE(K7C, 4, 32, 32, 4, 6, 2);
        case 5: PIPE(K7C, 5, 32, 32, 4, 6, 2);
        case 6: PIPE(K7C, 6, 32, 32, 4, 6, 2);
        case 7: PIPE(K7C, 7, 32, 32, 4, 6, 2);
        case 8: PIPE(K7C, 8, 32, 32, 4, 6, 2);
      }
      break;
    case K7V:
      switch (b) {
        case 1:
          if (cfg == 1) PIPE(K7V, 1, 32, 32, 4, 4, 2);
          PIPE(K7V, 1, 32, 32, 4, 4, 3);
        case 2:
          if (cfg == 1) PIPE(K7V, 2, 32, 24, 4, 4, 4);
          PIPE(K7V, 2, 32, 32, 4, 4, 3);
        case 3:
          PIPE(K7V, 3, 32, 24, 4, 4, 4);
      }
      break;
    case K25W:
      if (b == 1) {
        if (cfg == 1) PIPE(K25W, 1, 64, 32, 8, 8, 4);
        PIPE(K25W, 1, 64, 16, 4, 6, 3);
      }
      break;
    case K25V:
      if (b == 1) PIPE(K25V, 1, 64, 16, 4, 8, 3);
      break;
  }
#undef PIPE
  return cudaErrorInvalidValue;
}

}  // namespace st
