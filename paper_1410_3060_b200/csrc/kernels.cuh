// kernels.cuh -- launch interface between the runtime (runtime.cu) and the device kernels.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace st {

// Arguments of one kernel launch.  Pointers are pre-offset so that element (z, y, x) of a padded
// array (local plane z, padded row y, padded column x) is ptr[z*plane + y*pitch + x].
struct KParams {
  const double* src;   // Omega^t at the start of the block (level 0 of the wavefront)
  const double* srcu;  // wave: Omega^{t-1}; else unused
  double* dst;         // Jacobi: Omega^{t+b}; wave: Omega^{t+b} (b = 1: in place over srcu)
  double* dstu;        // wave, b >= 2: Omega^{t+b-1}; else unused
  const double* coef;  // first coefficient field (variable kinds)
  long long cstride;   // elements between consecutive coefficient fields
  long long pitch;     // row pitch (elements)
  long long plane;     // plane stride (elements)
  int nx, ny;          // interior extents in x and y; padded columns are [0, nx + 2R)
  int zl;              // planes stored locally
  int zi0, zi1;        // local planes that are interior planes of the global grid: [zi0, zi1)
  int zo0, zo1;        // local planes this launch writes at the last level: [zo0, zo1)
  int zchunk;          // output planes per CTA along z (grid.z = ceil((zo1 - zo0) / zchunk))
  double s[6];         // scalar weights (7c: w1, w2; wave: w0, w1..w4, alpha)
  // TMA-pipelined kernel only: 16-byte-aligned allocation bases (element (z, y, x) of a padded array
  // is raw[z*plane + y*pitch + x + xoff]) for the tensor maps.
  const double* src_raw;
  const double* srcu_raw;
  const double* coef_raw;
  int xoff;
  int dbg;     // experiment knob (STENCIL_DBG): bit 0 = discard every level's results in the pipe
               // kernel (the straight-line arithmetic still runs: results are wrong), bit 1 = skip level
               // barriers; fault injection for the mutation tests (STENCIL_FAULT):
               // bit 2 = never write the last plane of a z-chunk, bit 3 = skip work item 0
               // (pipe25: bit 4 = box B re-reads plane s, a DRAM diagnostic with wrong results)
  unsigned int* sched;  // pipe kernel: 2 zeroed device counters (next work item, CTAs done)
  // Pipe kernel, several fused blocks in ONE launch (Jacobi kinds, single slab): nblk blocks; block i
  // reads the buffer block i-1 wrote (odd blocks: V from dst_raw, stores to dst_alt = the src buffer);
  // done[item] = dbase + i + 1 once item of block i is complete (dependency-driven scheduling).
  int nblk;
  int nzc;  // z-chunks per tile (set by the launcher)
  unsigned int* done;
  unsigned int dbase;
  double* dst_alt;
  const double* dst_raw;
  // Fused halo exchange (pipe kernel only): last-level output planes in local range
  // [rz0[q], rz1[q]) are also stored through rdst[q] (and rdstu[q], wave second level), a pointer into
  // a z-neighbour's buffer pre-offset so that the same element offset addresses the same global cell.
  // NULL = no remote target.  rfence: end with a system-scope fence (peer memory of another process).
  double* rdst[2];
  double* rdstu[2];
  int rz0[2], rz1[2];
  int rfence;
  int tband;   // pipe kernel, single-block launches: tile order within a z-chunk (STENCIL_TILE_BAND;
               // 0 = row-major, w > 0 = bands of w tile columns walked row by row, so y-neighbours are w
               // ids apart instead of ntx)
  int tblk_w, tblk_h;  // tile order in blocks of tblk_w x tblk_h tiles (0 = row-major; set by launchers)
  int lockstep;        // pipe kernels: static round-robin items, CTAs start each round together (launcher)
  int pfd;             // pipe25: TMA L2-prefetch distance in steps (launcher; STENCIL_PF)
  int l2h;             // pipe25 experiment (STENCIL_L2H): L2 priorities of boxes A/B/C, 2 bits each
                       // (0 = no hint, 1 = evict_first, 2 = evict_last, 3 = evict_normal)
  // pipe25 skewed tiles (SKEW): the level-1 rows a tile hands to the tile above go through
  // xch (a state-sized buffer, offset like dst; xch_raw its allocation base); xflag[2 * item slot + w] =
  // xbase + q + 1 once exporting warp w stored plane q (xflag_n entries); xbase grows by 65536 per launch
  double* xch;
  const double* xch_raw;
  unsigned int* xflag;
  long long xflag_n;
  unsigned int xbase;
  int xg;  // skewed tiles: exported planes are released every xg steps (launcher; STENCIL_XG)
  int walign;  // pipe kernel: tiles write sector-aligned output segments (STENCIL_WALIGN=1; default 0:
               // measured slower under the power cap for OX % 4 != 0, profiles/r01_summary.md)
};

struct LaunchInfo {
  int tile_x, tile_y;  // output tile of one CTA
  int zchunk;          // planes per CTA
  int threads;         // threads per CTA
  int smem;            // dynamic shared memory bytes
  long long ctas;      // CTAs launched
};

// One time step, one thread per interior point (ST_VARIANT_NAIVE).
cudaError_t launch_naive(int kind, const KParams& p, cudaStream_t stream, LaunchInfo* info);

// b fused time levels (1 <= b <= max_stream_bt(kind)) of the z-streaming wavefront kernel
// (ST_VARIANT_STREAM).  zchunk_req = 0 picks a default.
cudaError_t launch_stream(int kind, int b, const KParams& p, int zchunk_req, int num_sms,
                          cudaStream_t stream, LaunchInfo* info);
int max_stream_bt(int kind);

// b fused levels of the TMA-pipelined, warp-specialised z-streaming kernel (ST_VARIANT_PIPE):
// a producer warp streams planes of Omega^t and the coefficient fields into shared-memory rings
// with cp.async.bulk.tensor + mbarriers; consumer warps run the same wavefront as stream_kernel.
// cfg selects a tile configuration (0 = default for the kind and b).  Persistent: one CTA per SM.
constexpr long long kMaxDoneItems = 1 << 18;  // per-item completion counters of a multi-block launch
cudaError_t launch_pipe(int kind, int b, const KParams& p, int zchunk_req, int num_sms, int cfg,
                        cudaStream_t stream, LaunchInfo* info);
int max_pipe_bt(int kind);

// The 25-point variable-coefficient kind with two fused levels (pipe25.cu): same contract as
// launch_pipe for (K25V, b = 2); cfg selects a tile configuration (0 = default).
// tile_cfg entries of launch_pipe25v2 with skewed tiles (they need KParams::xch / xflag)
bool pipe25v2_skewed(int cfg);
long long pipe25v2_flag_slots(int cfg, int nx, int ny, int zl);
cudaError_t launch_pipe25v2(const KParams& p, int zchunk_req, int num_sms, int cfg, cudaStream_t stream,
                            LaunchInfo* info);
// The 25-point wave with two fused levels (pipe25.cu): contract of launch_pipe for (K25W, b = 2).
cudaError_t launch_pipe25w2(const KParams& p, int zchunk_req, int num_sms, int cfg, cudaStream_t stream,
                            LaunchInfo* info);

// Tensor map (cuTensorMapEncodeTiled) of fp64 padded arrays in the library's layout: rank 3 (x, y, z)
// or 4 (x, y, z, field); box bx x by x 1 (x bf).  The map covers columns [0, X) from `base` (the row
// padding beyond the padded extent is out of bounds: zero-filled by the TMA unit, never fetched).
bool make_tensor_map(CUtensorMap* m, const double* base, int rank, long long pitch, long long X, long long Y,
                     long long zl, long long nfields, long long plane, long long fstride, int bx, int by, int bf);

// T time steps of the whole slab in ONE cooperative launch with a grid-wide barrier between sweeps
// (ST_VARIANT_COOP, small latency-bound grids).  p.src = Omega^t, p.dst = p.srcu = the other buffer.
// cfg 0 / 1 = one sweep per grid barrier; 2 = temporal blocking in shared memory, one grid barrier per
// round of 5 levels (7-point Jacobi kinds; measured no faster at C1, kernels.cu).
// *swaps = how many times the two state buffers swapped roles (T, or the number of rounds).
cudaError_t launch_coop(int kind, const KParams& p, int T, int num_sms, int cfg, cudaStream_t stream, LaunchInfo* info,
                        int* swaps);

// Seeded fill of the local planes of one array (synth/synth.h).  mode 0: U[-1,1) from `stream`
// everywhere; mode 1: U[-1,1), interior cells from stream 1 and the rest from stream 0 (wave
// Omega^{-1}); mode 2: U[0, c) from `stream`.  gz0 = global padded index of local plane 0;
// (GX, GY, GZ) = global padded extents; R = ghost width.
cudaError_t launch_fill(double* base, long long pitch, long long plane, int zl, long long gz0,
                        long long GX, long long GY, long long GZ, int R, uint64_t seed, int stream,
                        int mode, double c, cudaStream_t cs);

// Copy the global ghost shell (width R) of local planes [0, zl) of one padded array into another of
// the same layout (stencil_write keeps every buffer's fixed boundary equal to level 0's).
cudaError_t launch_ghost_copy(double* dst, const double* src, long long pitch, long long plane, int zl,
                              long long gz0, long long GX, long long GY, long long GZ, int R, cudaStream_t cs);

}  // namespace st
