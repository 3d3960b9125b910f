// kernels.cu -- sm_100a kernels of the stencil hot path.
//
//  naive_kernel   one thread per interior point, one time step per launch: the GPU form of the
//                 naive sweep (§4.1).  Reference variant for test G4.
//  stream_kernel  2.5-D z-streaming with BT fused time levels.  One CTA owns an xy footprint of
//                 FX x FY columns and streams z.  Level k (1..BT) trails level k-1 by R planes:
//                 the single-thread wavefront with frontline slope -1/R of P:569-602, turned into
//                 a CTA-wide z-stream; the footprint shrinks by R per level in x and y (overlapped
//                 tiles), so the CTA's output tile is (FX - 2R*BT) x (FY - 2R*BT) and needs no
//                 communication with other CTAs.  z-neighbours of every level live in per-thread
//                 register rings of 2R+1 planes; x/y neighbours come from one shared-memory plane per
//                 level (double-buffered, one __syncthreads per level per step) -- the GPU analog of
//                 the layer condition: every V element is read from HBM once per block.
//  coop_kernel    small grids (latency-bound, L2-resident): ALL T time steps in one cooperative launch,
//                 a grid-wide barrier between sweeps (the naive sweep order of P:557-560 without a
//                 kernel launch per step).
//  fill_kernel    the seeded generator of synth/synth.h on the device.
//
// All kernels call the point functions of point.cuh, so their results are bitwise identical.
#include "kernels.cuh"
#include "point.cuh"
#include "../../synth/synth.h"

#include <cooperative_groups.h>

#include <algorithm>

namespace st {

// ------------------------------------------------------------------------------------------------
// naive: one thread per interior point of planes [zo0, zo1), one time step.
template <int KIND>
__global__ void __launch_bounds__(256) naive_kernel(const KParams p) {
  constexpr int R = Traits<KIND>::R, NC = Traits<KIND>::NCOEF;
  const int x = blockIdx.x * 32 + threadIdx.x + R;
  if (x >= p.nx + R) return;
  // grid-stride over y and z: the launch caps grid.y / grid.z at 65535 (tall grids, thick slabs)
  for (int z = p.zo0 + (int)blockIdx.z; z < p.zo1; z += (int)gridDim.z)
    for (int y = (int)blockIdx.y * 8 + (int)threadIdx.y + R; y < p.ny + R; y += (int)gridDim.y * 8) {
      const long long i = (long long)z * p.plane + (long long)y * p.pitch + x;
      double m[3][R], pl[3][R];
#pragma unroll
      for (int r = 1; r <= R; ++r) {
        m[0][r - 1] = p.src[i - r];
        pl[0][r - 1] = p.src[i + r];
        m[1][r - 1] = p.src[i - r * p.pitch];
        pl[1][r - 1] = p.src[i + r * p.pitch];
        m[2][r - 1] = p.src[i - r * p.plane];
        pl[2][r - 1] = p.src[i + r * p.plane];
      }
      double W[NC > 0 ? NC : 1];
#pragma unroll
      for (int k = 0; k < NC; ++k) W[k] = p.coef[k * p.cstride + i];
      const double u = Traits<KIND>::WAVE ? p.srcu[i] : 0.0;
      p.dst[i] = apply_point<KIND, R>(p.src[i], u, m, pl, W, p.s);
    }
}

// ------------------------------------------------------------------------------------------------
// coop: T sweeps in one cooperative launch.  Warps own rows (y, z) of the interior, lanes own x
// (grid-stride); after a sweep every thread passes a grid-wide barrier and the roles of the two state
// buffers swap -- for the Jacobi kinds dst is the other buffer, for the wave Omega^{t+1} overwrites
// Omega^{t-1} in place (each cell reads its own U before writing it), so in both cases
// (src, other) -> (other, src).  Bitwise equal to naive_kernel (same gathers, same point function).
// 7-point kinds: one CTA per SM (1024 threads for 7c, 512 for 7v), two cells per lane whose operands are all loaded before
// either is computed (the L2 round trips overlap); 25-point kinds: two 256-thread CTAs per SM, one
// cell per lane (their 25 gathers + 13 coefficients need ~120 registers).  tools/coop_sweep.py.
template <int KIND>
struct CoopCfg {
  static constexpr int THREADS = KIND == K7C ? 1024 : KIND == K7V ? 512 : 256;  // 7v: 14 gathers + 14 coefs
  static constexpr int MINB = Traits<KIND>::R == 1 ? 1 : 2;
  static constexpr int CB = Traits<KIND>::R == 1 ? 2 : 1;
};

template <int KIND>
__global__ void __launch_bounds__(CoopCfg<KIND>::THREADS, CoopCfg<KIND>::MINB) coop_kernel(KParams p, int T) {
  constexpr int R = Traits<KIND>::R, NC = Traits<KIND>::NCOEF, CB = CoopCfg<KIND>::CB;
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const double* src = p.src;
  double* oth = p.dst;  // == p.srcu for every kind (see run_coop)
  const int nxc = (p.nx + 32 * CB - 1) / (32 * CB);  // x-chunks of 32*CB cells per row
  const long long units = (long long)p.ny * (p.zo1 - p.zo0) * nxc;
  const long long warps = (long long)gridDim.x * (blockDim.x / 32);
  const long long w0 = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  for (int t = 0; t < T; ++t) {
    for (long long u = w0; u < units; u += warps) {
      const long long row = u / nxc;
      const int xc = (int)(u - row * nxc);
      const int y = (int)(row % p.ny) + R, z = (int)(row / p.ny) + p.zo0;
      const long long b = (long long)z * p.plane + (long long)y * p.pitch;
      long long idx[CB];
      bool ok[CB];
      double c[CB], uo[CB], m[CB][3][R], pl[CB][3][R], W[CB][NC > 0 ? NC : 1];
#pragma unroll
      for (int q = 0; q < CB; ++q) {
        const int x = R + xc * 32 * CB + q * 32 + lane;
        ok[q] = x < p.nx + R;
        idx[q] = b + (ok[q] ? x : R);  // out-of-range lanes gather a valid cell and store nothing
      }
#pragma unroll
      for (int q = 0; q < CB; ++q) {
        const long long i = idx[q];
#pragma unroll
        for (int r = 1; r <= R; ++r) {
          m[q][0][r - 1] = src[i - r];
          pl[q][0][r - 1] = src[i + r];
          m[q][1][r - 1] = src[i - r * p.pitch];
          pl[q][1][r - 1] = src[i + r * p.pitch];
          m[q][2][r - 1] = src[i - r * p.plane];
          pl[q][2][r - 1] = src[i + r * p.plane];
        }
#pragma unroll
        for (int k = 0; k < NC; ++k) W[q][k] = p.coef[k * p.cstride + i];
        c[q] = src[i];
        uo[q] = Traits<KIND>::WAVE ? oth[i] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < CB; ++q)
        if (ok[q]) oth[idx[q]] = apply_point<KIND, R>(c[q], uo[q], m[q], pl[q], W[q], p.s);
    }
    grid.sync();
    double* tmp = const_cast<double*>(src);
    src = oth;
    oth = tmp;
  }
}

// Largest cooperative grid of coop_kernel<KIND> on this device (0 if unsupported).
template <int KIND>
int coop_grid(int num_sms) {
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, coop_kernel<KIND>, CoopCfg<KIND>::THREADS, 0) != cudaSuccess)
    return 0;
  return std::min(occ, CoopCfg<KIND>::MINB) * num_sms;
}

template <int KIND>
cudaError_t run_coop(const KParams& p0, int T, int num_sms, cudaStream_t stream, LaunchInfo* info) {
  const int grid = coop_grid<KIND>(num_sms);  // every co-resident CTA: more loads in flight per sweep
  if (grid <= 0) return cudaErrorCooperativeLaunchTooLarge;
  KParams p = p0;
  int Tv = T;
  void* args[] = {(void*)&p, (void*)&Tv};
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)coop_kernel<KIND>, dim3(grid),
                                              dim3(CoopCfg<KIND>::THREADS), args, 0, stream);
  if (info) {
    info->tile_x = 32 * CoopCfg<KIND>::CB; info->tile_y = 1; info->zchunk = 1;
    info->threads = CoopCfg<KIND>::THREADS; info->smem = 0;
    info->ctas = grid;
  }
  return e;
}

// ------------------------------------------------------------------------------------------------
// coop_tb: the cooperative kernel with temporal blocking in shared memory (7-point Jacobi kinds).
// Every CTA owns an output block of BX x BY x BZ interior cells; per ROUND it loads the block grown by
// H = R*BTL cells on every side (from L2: the grids this runs on are L2-resident) into shared memory,
// runs L <= BTL levels there -- level k updates the region shrunk by k*R, so the block's own cells are
// exact after L levels (the overlapped-tile trapezoid of P:600-612, in all three dimensions) -- and
// writes the block back; one grid-wide barrier per round instead of one per sweep.  Cells that are not
// interior keep their (fixed ghost) value at every level; cells beyond the padded extent are loaded as
// 0 and only ever feed ghost cells, whose value is not computed.  Same point function, same operands
// as naive_kernel: bitwise equal (test G4).  Buffers alternate per round (`swaps` = rounds).
template <int KIND, int BX, int BY, int BZ, int BTL>
struct TbCfg {
  static constexpr int R = Traits<KIND>::R, H = R * BTL;
  static constexpr int SX = BX + 2 * H, SY = BY + 2 * H, SZ = BZ + 2 * H, N = SX * SY * SZ;
  static constexpr int THREADS = 1024;
  static constexpr size_t SMEM = 2 * sizeof(double) * (size_t)N;
  static_assert(SX <= 32 && SY <= THREADS / 32, "warp = one y row of the grown block, lane = x");
  static_assert(SMEM <= 227 * 1024, "two grown blocks must fit in shared memory");
};

// One level of a round: warp w updates y row lo + w of the region shrunk by lo = k*R, lane = x, walking z
// (the column's centre and z-neighbours rotate through registers: 5 shared loads per 7-point update).
template <int KIND, int SX, int SY, int SZ>
__device__ __forceinline__ void tb_level(const double* __restrict__ A, double* __restrict__ B, int lo, int ox,
                                         int oy, int oz, const KParams& p, int warp, int lane) {
  constexpr int R = Traits<KIND>::R, NC = Traits<KIND>::NCOEF, SXY = SX * SY;
  static_assert(R == 1, "7-point kinds");
  const int sy = lo + warp, sx = lo + lane;
  if (sy >= SY - lo || sx >= SX - lo) return;
  const int gy = oy + sy, gx = ox + sx;
  const bool xyint = gy >= R && gy < p.ny + R && gx >= R && gx < p.nx + R;
  int i = (lo * SY + sy) * SX + sx;
  double zm = A[i - SXY], zc = A[i];
  const long long g0 = (long long)gy * p.pitch + gx;
#pragma unroll 4
  for (int sz = lo; sz < SZ - lo; ++sz, i += SXY) {
    const double zp = A[i + SXY];
    const double m[3][1] = {{A[i - 1]}, {A[i - SX]}, {zm}}, pl[3][1] = {{A[i + 1]}, {A[i + SX]}, {zp}};
    const int gz = oz + sz;
    const bool upd = xyint && gz >= p.zi0 && gz < p.zi1;
    double W[NC > 0 ? NC : 1];
    const long long gi = upd ? (long long)gz * p.plane + g0 : 0;
#pragma unroll
    for (int f = 0; f < NC; ++f) W[f] = __ldg(p.coef + f * p.cstride + gi);
    B[i] = upd ? apply_point<KIND, R>(zc, 0.0, m, pl, W, p.s) : zc;
    zm = zc;
    zc = zp;
  }
}

template <int KIND, int BX, int BY, int BZ, int BTL>
__global__ void __launch_bounds__(1024, 1) coop_tb_kernel(KParams p, int T) {
  using C = TbCfg<KIND, BX, BY, BZ, BTL>;
  constexpr int R = C::R, H = C::H, SX = C::SX, SY = C::SY, SZ = C::SZ, SXY = SX * SY;
  static_assert(!Traits<KIND>::WAVE, "Jacobi kinds");
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double tb_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nzi = p.zi1 - p.zi0;
  const int nbx = (p.nx + BX - 1) / BX, nby = (p.ny + BY - 1) / BY, nbz = (nzi + BZ - 1) / BZ;
  const int nblocks = nbx * nby * nbz;
  const int GX = p.nx + 2 * R, GY = p.ny + 2 * R;
  const double* src = p.src;
  double* dst = p.dst;
  for (int t = 0; t < T; t += BTL) {
    const int L = min(BTL, T - t);
    for (int b = blockIdx.x; b < nblocks; b += gridDim.x) {
      const int bz = b / (nbx * nby), byx = b - bz * nbx * nby, by = byx / nbx, bx = byx - by * nbx;
      // padded coordinates of grown-block cell (0, 0, 0): x, y global; z local plane
      const int ox = R + bx * BX - H, oy = R + by * BY - H, oz = p.zi0 + bz * BZ - H;
      // grown block -> shared memory with asynchronous copies (cp.async, zero-filled outside the padded
      // extent): all of a warp's rows are in flight at once
      if (warp < SY && lane < SX) {
        const int gy = oy + warp, gx = ox + lane;
        const bool xyok = gy >= 0 && gy < GY && gx >= 0 && gx < GX;
        for (int sz = 0; sz < SZ; ++sz) {
          const int gz = oz + sz;
          const bool ok = xyok && gz >= 0 && gz < p.zl;
          const double* g = ok ? src + ((long long)gz * p.plane + (long long)gy * p.pitch + gx) : src;
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(
                           static_cast<uint32_t>(__cvta_generic_to_shared(tb_smem + sz * SXY + warp * SX + lane))),
                       "l"(g), "r"(ok ? 8 : 0)
                       : "memory");
        }
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncthreads();
      double* A = tb_smem;
      double* B = tb_smem + C::N;
#pragma unroll 1
      for (int k = 1; k <= L; ++k) {
        tb_level<KIND, SX, SY, SZ>(A, B, k * R, ox, oy, oz, p, warp, lane);
        __syncthreads();
        double* tmp = A;
        A = B;
        B = tmp;
      }
      if (warp < BY && lane < BX) {
        const int sy = H + warp, gy = oy + sy, gx = ox + H + lane;
        if (gy < p.ny + R && gx < p.nx + R)
          for (int sz = H; sz < H + BZ && oz + sz < p.zi1; ++sz)
            dst[(long long)(oz + sz) * p.plane + (long long)gy * p.pitch + gx] = A[sz * SXY + sy * SX + H + lane];
      }
      __syncthreads();  // the next block's load overwrites this one's shared memory
    }
    grid.sync();
    double* tmp = const_cast<double*>(src);
    src = dst;
    dst = tmp;
  }
}

template <int KIND, int BX, int BY, int BZ, int BTL>
cudaError_t run_coop_tb(const KParams& p0, int T, int num_sms, cudaStream_t stream, LaunchInfo* info, int* swaps) {
  using C = TbCfg<KIND, BX, BY, BZ, BTL>;
  auto kern = coop_tb_kernel<KIND, BX, BY, BZ, BTL>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  static int occ = 0;  // per instantiation; the device's SM layout does not change
  if (occ < 1 && (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::THREADS, C::SMEM) != cudaSuccess || occ < 1))
    return cudaErrorCooperativeLaunchTooLarge;
  const long long nblocks = (long long)((p0.nx + BX - 1) / BX) * ((p0.ny + BY - 1) / BY) *
                            ((p0.zi1 - p0.zi0 + BZ - 1) / BZ);
  const int grid = (int)std::min<long long>(nblocks, (long long)occ * num_sms);
  KParams p = p0;
  int Tv = T;
  void* args[] = {(void*)&p, (void*)&Tv};
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(C::THREADS), args, C::SMEM, stream);
  if (info) {
    info->tile_x = BX; info->tile_y = BY; info->zchunk = BZ;
    info->threads = C::THREADS; info->smem = (int)C::SMEM; info->ctas = grid;
  }
  if (swaps) *swaps = (T + BTL - 1) / BTL;
  return e;
}

// Output blocks of the temporally blocked cooperative kernel: (16, 16, 8) cells, 5 levels per round
// (grown block 26 x 26 x 18, 195 KB for the two copies).  Measured (tools/coop_sweep.py, B200): C1 7c
// 64^3 T = 10 37.9 us vs 36.3 us for one sweep per barrier -- the 2.5x redundant level work of the
// grown blocks costs what the 8 saved grid barriers gain; 15 % faster on one-block grids (8^3, T = 50);
// 7v 1.7x slower (its coefficients come from L2 at every level).  Not the default (tile_cfg 2).
constexpr int kTbBX = 16, kTbBY = 16, kTbBZ = 8, kTbBT = 5;

cudaError_t launch_coop(int kind, const KParams& p, int T, int num_sms, int cfg, cudaStream_t stream, LaunchInfo* info,
                        int* swaps) {
  if (swaps) *swaps = T;
  if (p.zo1 <= p.zo0 || T <= 0) {
    if (swaps) *swaps = 0;
    return cudaSuccess;
  }
  // cfg 0 / 1: one sweep per grid barrier; cfg 2: temporal blocking in shared memory (7-point Jacobi kinds)
  if (cfg == 2) {
    if (kind == K7C) return run_coop_tb<K7C, kTbBX, kTbBY, kTbBZ, kTbBT>(p, T, num_sms, stream, info, swaps);
    if (kind == K7V) return run_coop_tb<K7V, kTbBX, kTbBY, kTbBZ, kTbBT>(p, T, num_sms, stream, info, swaps);
    return cudaErrorInvalidValue;
  }
  switch (kind) {
    case K7C: return run_coop<K7C>(p, T, num_sms, stream, info);
    case K7V: return run_coop<K7V>(p, T, num_sms, stream, info);
    case K25W: return run_coop<K25W>(p, T, num_sms, stream, info);
    case K25WA: return run_coop<K25WA>(p, T, num_sms, stream, info);
    case K25V: return run_coop<K25V>(p, T, num_sms, stream, info);
    default: return cudaErrorInvalidValue;
  }
}

// ------------------------------------------------------------------------------------------------
// z-streaming wavefront kernel with BT fused levels (see the file header).
//   block = (FX, FYT) threads; thread (lx, ty) owns footprint columns (lx, ty + j*FYT), j < CY.
template <int KIND, int BT, int FX, int FYT, int CY>
__global__ void __launch_bounds__(FX * FYT) stream_kernel(const KParams p) {
  using TR = Traits<KIND>;
  constexpr int R = TR::R, NC = TR::NCOEF, RL = 2 * R + 1;
  constexpr bool WAVE = TR::WAVE;
  constexpr int FY = FYT * CY;
  constexpr int OX = FX - 2 * R * BT, OY = FY - 2 * R * BT;
  static_assert(OX > 0 && OY > 0, "footprint too small for BT");
  extern __shared__ double smem[];  // [BT][2][FY][FX]

  const int lx = threadIdx.x, ty = threadIdx.y;
  const int X = p.nx + 2 * R, Y = p.ny + 2 * R;
  const int gx = (int)blockIdx.x * OX + R - R * BT + lx;
  const int gyb = (int)blockIdx.y * OY + R - R * BT;
  const int zc0 = p.zo0 + (int)blockIdx.z * p.zchunk;
  const int zc1 = min(p.zo1, zc0 + p.zchunk);

  int ly[CY];
  long long col[CY];
  bool in_dom[CY], inter[CY], out_col[CY];
  unsigned lvl[CY];  // bit k set: column inside the level-k extent
#pragma unroll
  for (int j = 0; j < CY; ++j) {
    ly[j] = ty + j * FYT;
    const int gy = gyb + ly[j];
    in_dom[j] = gx >= 0 && gx < X && gy >= 0 && gy < Y;
    inter[j] = gx >= R && gx < p.nx + R && gy >= R && gy < p.ny + R;
    col[j] = in_dom[j] ? (long long)gy * p.pitch + gx : 0;
    lvl[j] = 0;
#pragma unroll
    for (int k = 1; k <= BT; ++k)
      if (lx >= k * R && lx < FX - k * R && ly[j] >= k * R && ly[j] < FY - k * R) lvl[j] |= 1u << k;
    out_col[j] = inter[j] && (lvl[j] >> BT & 1u);
  }

  double ring[BT][CY][RL];
#pragma unroll
  for (int k = 0; k < BT; ++k)
#pragma unroll
    for (int j = 0; j < CY; ++j)
#pragma unroll
      for (int i = 0; i < RL; ++i) ring[k][j][i] = 0.0;
  double uq[CY][WAVE ? R + 1 : 1];
#pragma unroll
  for (int j = 0; j < CY; ++j)
#pragma unroll
    for (int i = 0; i < (WAVE ? R + 1 : 1); ++i) uq[j][i] = 0.0;

  const int s_begin = max(0, zc0 - BT * R);
  const int s_end = zc1 - 1 + BT * R;
  for (int s = s_begin; s <= s_end; ++s) {
    const int buf = s & 1;
    const bool have = s < p.zl;
    // Level-1 coefficients of plane s - R, issued before the barrier to overlap their latency.
    double w1[CY][NC > 0 ? NC : 1];
    if constexpr (NC > 0) {
      const int c1 = s - R;
      const bool z1in = c1 >= p.zi0 && c1 < p.zi1;
#pragma unroll
      for (int j = 0; j < CY; ++j) {
        const bool need = z1in && inter[j] && (lvl[j] & 2u);
        const double* cp = p.coef + (long long)c1 * p.plane + col[j];
#pragma unroll
        for (int i = 0; i < NC; ++i) w1[j][i] = need ? __ldg(cp + i * p.cstride) : 0.0;
      }
    }
    // Level 0: plane s of Omega^t (and Omega^{t-1} for the wave) into the register rings.
#pragma unroll
    for (int j = 0; j < CY; ++j) {
      const double v = (have && in_dom[j]) ? __ldg(p.src + (long long)s * p.plane + col[j]) : 0.0;
#pragma unroll
      for (int i = 0; i < RL - 1; ++i) ring[0][j][i] = ring[0][j][i + 1];
      ring[0][j][RL - 1] = v;
      if constexpr (WAVE) {
        const double u = (have && inter[j] && (lvl[j] & 2u))
                             ? __ldg(p.srcu + (long long)s * p.plane + col[j]) : 0.0;
#pragma unroll
        for (int i = 0; i < R; ++i) uq[j][i] = uq[j][i + 1];
        uq[j][R] = u;
      }
    }
#pragma unroll
    for (int k = 1; k <= BT; ++k) {
      double* P = smem + ((k - 1) * 2 + buf) * (FY * FX);
#pragma unroll
      for (int j = 0; j < CY; ++j) P[ly[j] * FX + lx] = ring[k - 1][j][R];
      __syncthreads();
      const int c = s - k * R;  // plane computed at level k in this step
      const bool zin = c >= p.zi0 && c < p.zi1;
#pragma unroll
      for (int j = 0; j < CY; ++j) {
        double v = ring[k - 1][j][R];  // ghosts and out-of-extent columns keep the input value
        if (zin && inter[j] && (lvl[j] >> k & 1u)) {
          double m[3][R], pl[3][R];
          const double* row = P + ly[j] * FX + lx;
#pragma unroll
          for (int r = 1; r <= R; ++r) {
            m[0][r - 1] = row[-r];
            pl[0][r - 1] = row[r];
            m[1][r - 1] = row[-r * FX];
            pl[1][r - 1] = row[r * FX];
            m[2][r - 1] = ring[k - 1][j][R - r];
            pl[2][r - 1] = ring[k - 1][j][R + r];
          }
          double W[NC > 0 ? NC : 1];
          if constexpr (NC > 0) {
            if (k == 1) {
#pragma unroll
              for (int i = 0; i < NC; ++i) W[i] = w1[j][i];
            } else {
              const double* cp = p.coef + (long long)c * p.plane + col[j];
#pragma unroll
              for (int i = 0; i < NC; ++i) W[i] = __ldg(cp + i * p.cstride);
            }
          }
          double u = 0.0;
          if constexpr (WAVE) u = (k == 1) ? uq[j][0] : ring[k >= 2 ? k - 2 : 0][j][0];
          v = apply_point<KIND, R>(ring[k - 1][j][R], u, m, pl, W, p.s);
        }
        if (k < BT) {
#pragma unroll
          for (int i = 0; i < RL - 1; ++i) ring[k < BT ? k : 0][j][i] = ring[k < BT ? k : 0][j][i + 1];
          ring[k < BT ? k : 0][j][RL - 1] = v;
        } else if (out_col[j] && c >= zc0 && c < zc1) {
          const long long o = (long long)c * p.plane + col[j];
          __stcs(p.dst + o, v);
          if constexpr (WAVE && BT >= 2) __stcs(p.dstu + o, ring[BT - 1][j][R]);
        }
      }
    }
  }
}

// ------------------------------------------------------------------------------------------------
__global__ void fill_kernel(double* base, long long pitch, long long plane, int zl, long long gz0,
                            long long GX, long long GY, long long GZ, int R, uint64_t key,
                            uint64_t key_u, int mode, double c) {
  const long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= GX) return;
  // grid-stride over y and z (grid.y / grid.z are capped at 65535 by the launch)
  for (long long z = blockIdx.z; z < zl; z += gridDim.z)
    for (long long y = blockIdx.y; y < GY; y += gridDim.y) {
      const long long gz = gz0 + z;
      const uint64_t idx = (uint64_t)((gz * GY + y) * GX + x);
      double v;
      if (mode == 2) {
        v = synth_scaled(key, idx, c);
      } else if (mode == 1 && x >= R && x < GX - R && y >= R && y < GY - R && gz >= R && gz < GZ - R) {
        v = synth_sym(key_u, idx);
      } else {
        v = synth_sym(key, idx);
      }
      base[z * plane + y * pitch + x] = v;
    }
}

cudaError_t launch_fill(double* base, long long pitch, long long plane, int zl, long long gz0,
                        long long GX, long long GY, long long GZ, int R, uint64_t seed, int stream,
                        int mode, double c, cudaStream_t cs) {
  if (zl <= 0) return cudaSuccess;
  dim3 block(128);
  dim3 grid((unsigned)((GX + 127) / 128), (unsigned)std::min<long long>(GY, 65535),
            (unsigned)std::min(zl, 65535));
  const uint64_t key = synth_key(seed, mode == 1 ? SYNTH_STREAM_V : stream);
  const uint64_t key_u = synth_key(seed, SYNTH_STREAM_U);
  fill_kernel<<<grid, block, 0, cs>>>(base, pitch, plane, zl, gz0, GX, GY, GZ, R, key, key_u, mode, c);
  return cudaGetLastError();
}

// Copy the cells of the global ghost shell (width R) of local planes [0, zl) from src to dst (same
// layout); interior cells are left alone.
__global__ void ghost_copy_kernel(double* dst, const double* src, long long pitch, long long plane, int zl,
                                  long long gz0, long long GX, long long GY, long long GZ, int R) {
  const long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= GX) return;
  for (long long z = blockIdx.z; z < zl; z += gridDim.z)
    for (long long y = blockIdx.y; y < GY; y += gridDim.y) {
      const long long gz = gz0 + z;
      if (x >= R && x < GX - R && y >= R && y < GY - R && gz >= R && gz < GZ - R) continue;
      const long long o = z * plane + y * pitch + x;
      dst[o] = src[o];
    }
}

cudaError_t launch_ghost_copy(double* dst, const double* src, long long pitch, long long plane, int zl,
                              long long gz0, long long GX, long long GY, long long GZ, int R, cudaStream_t cs) {
  if (zl <= 0) return cudaSuccess;
  dim3 grid((unsigned)((GX + 127) / 128), (unsigned)std::min<long long>(GY, 65535), (unsigned)std::min(zl, 65535));
  ghost_copy_kernel<<<grid, 128, 0, cs>>>(dst, src, pitch, plane, zl, gz0, GX, GY, GZ, R);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------------
cudaError_t launch_naive(int kind, const KParams& p, cudaStream_t stream, LaunchInfo* info) {
  const int planes = p.zo1 - p.zo0;
  if (planes <= 0) return cudaSuccess;
  dim3 block(32, 8);
  dim3 grid((p.nx + 31) / 32, std::min((p.ny + 7) / 8, 65535), std::min(planes, 65535));
  switch (kind) {
    case K7C: naive_kernel<K7C><<<grid, block, 0, stream>>>(p); break;
    case K7V: naive_kernel<K7V><<<grid, block, 0, stream>>>(p); break;
    case K25W: naive_kernel<K25W><<<grid, block, 0, stream>>>(p); break;
    case K25WA: naive_kernel<K25WA><<<grid, block, 0, stream>>>(p); break;
    case K25V: naive_kernel<K25V><<<grid, block, 0, stream>>>(p); break;
    default: return cudaErrorInvalidValue;
  }
  if (info) {
    info->tile_x = 32; info->tile_y = 8; info->zchunk = 1; info->threads = 256; info->smem = 0;
    info->ctas = (long long)grid.x * grid.y * grid.z;
  }
  return cudaGetLastError();
}

template <int KIND, int BT, int FX, int FYT, int CY>
static cudaError_t run_stream(const KParams& p0, int zchunk_req, int num_sms, cudaStream_t stream,
                              LaunchInfo* info) {
  constexpr int R = Traits<KIND>::R;
  constexpr int FY = FYT * CY;
  constexpr int OX = FX - 2 * R * BT, OY = FY - 2 * R * BT;
  constexpr int THREADS = FX * FYT;
  constexpr int SMEM = BT * 2 * FX * FY * (int)sizeof(double);
  auto kern = stream_kernel<KIND, BT, FX, FYT, CY>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  KParams p = p0;
  const int planes = p.zo1 - p.zo0;
  if (planes <= 0) return cudaSuccess;
  const long long tiles = (long long)((p.nx + OX - 1) / OX) * ((p.ny + OY - 1) / OY);
  int zchunk = zchunk_req;
  if (zchunk <= 0) {
    // Enough CTAs for ~4 per SM, but keep each z-chunk >= 8 * (warm-up depth) planes so the
    // 2*BT*R planes of wavefront fill/drain stay a small fraction of the stream.
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, THREADS, SMEM);
    const long long want = (long long)std::max(1, occ) * num_sms * 4;
    long long chunks = std::max<long long>(1, (want + tiles - 1) / tiles);
    zchunk = (int)((planes + chunks - 1) / chunks);
    zchunk = std::max(zchunk, std::min(planes, 16 * BT * R));
  }
  p.zchunk = zchunk;
  dim3 grid((p.nx + OX - 1) / OX, (p.ny + OY - 1) / OY, (planes + zchunk - 1) / zchunk);
  dim3 block(FX, FYT);
  kern<<<grid, block, SMEM, stream>>>(p);
  if (info) {
    info->tile_x = OX; info->tile_y = OY; info->zchunk = zchunk; info->threads = THREADS;
    info->smem = SMEM; info->ctas = (long long)grid.x * grid.y * grid.z;
  }
  return cudaGetLastError();
}

int max_stream_bt(int kind) {
  switch (kind) {
    case K7C: return 6;
    case K7V: return 4;
    case K25W: return 1;
    case K25WA: return 1;
    case K25V: return 1;
    default: return 0;
  }
}

cudaError_t launch_stream(int kind, int b, const KParams& p, int zchunk_req, int num_sms,
                          cudaStream_t stream, LaunchInfo* info) {
#define ST_7(K, B) case B: return run_stream<K, B, 32, 16, 2>(p, zchunk_req, num_sms, stream, info)
  switch (kind) {
    case K7C:
      switch (b) { ST_7(K7C, 1); ST_7(K7C, 2); ST_7(K7C, 3); ST_7(K7C, 4); ST_7(K7C, 5); ST_7(K7C, 6); }
      break;
    case K7V:
      switch (b) { ST_7(K7V, 1); ST_7(K7V, 2); ST_7(K7V, 3); ST_7(K7V, 4); }
      break;
    case K25W:
      if (b == 1) return run_stream<K25W, 1, 64, 8, 2>(p, zchunk_req, num_sms, stream, info);
      break;
    case K25WA:
      if (b == 1) return run_stream<K25WA, 1, 64, 8, 2>(p, zchunk_req, num_sms, stream, info);
      break;
    case K25V:
      if (b == 1) return run_stream<K25V, 1, 64, 8, 2>(p, zchunk_req, num_sms, stream, info);
      break;
  }
#undef ST_7
  return cudaErrorInvalidValue;
}

}  // namespace st
