/*
 * stencil.h -- C ABI of libstencil.so, the B200 (sm_100a) engine for the hot path of
 * Malas et al., "Multicore-optimized wavefront diamond blocking for optimizing stencil updates"
 * (arXiv 1410.3060; /root/reference/PAPER.md, cited "P:<line>").
 *
 * What the library computes: T Jacobi-style sweeps of one
 * of four 3-D star stencils on a Cartesian fp64 grid (Fig. 1 at P:138-268):
 *
 *   ST_7PT_CONST  Fig. 1b: O' = w1*O + w2*sum of the 6 axis neighbours
 *   ST_7PT_VAR    Fig. 1c: O' = W0*O + W1*O[x-1] + W2*O[x+1] + W3*O[y-1] + W4*O[y+1]
 *                                           + W5*O[z-1] + W6*O[z+1]       (7 domain-sized fields)
 *   ST_25PT_WAVE  Fig. 1e: O^{t+1} = 2 O^t - O^{t-1}
 *                          + alpha*[w0*O^t + sum_{r=1..4} w_r*(x, y and z pairs at distance r)]
 *                 with a scalar alpha (reading Q2)
 *   ST_25PT_VAR   Fig. 1d: O' = W0*O + sum_{r=1..4} sum_{axis} W_{1+3(r-1)+axis}*(pair)
 *                                                                           (13 domain-sized fields)
 *   ST_25PT_WAVE_A  Fig. 1e with the domain-sized alpha_{z,y,x} as printed: one field
 *
 * Grid and layout: arrays are indexed [z][y][x], x fastest, over the PADDED extent
 * (nz+2R) x (ny+2R) x (nx+2R), R = 1 (7-point) or 4 (25-point).  The outer shell of width R is the
 * fixed boundary (reading Q1): read every step, never written, identical in both time
 * levels.  Host buffers crossing this ABI are dense and unpadded beyond that (row = nx+2R doubles).
 * The device layout is the library's own (pitched, 128-byte aligned interior rows) and never
 * crosses the ABI.
 *
 * Time levels: the library keeps Omega^t ("level 0", newest) and Omega^{t-1}
 * ("level 1").  For the Jacobi kinds level 1's interior is scratch; for the wave it is the
 * previous time step that Fig. 1e reads.
 *
 * Conventions for every function:
 *   - returns ST_OK (0) or a negative ST_E_* code; it never aborts or exits;
 *   - stencil_last_error() returns a thread-local message about the last failure on this thread;
 *   - after an ST_E_CUDA / ST_E_NCCL failure the handle is poisoned: every call except
 *     stencil_destroy returns ST_E_STATE;
 *   - one handle must not be used from two threads at once (not reentrant); distinct handles may be
 *     used concurrently;
 *   - work is enqueued on opts->stream (the caller's CUDA stream; the Python binding passes torch's
 *     current stream); stencil_run returns after enqueueing; stencil_read / stencil_sync synchronize.
 *   - there is no CPU fallback: without a usable CUDA device every creating call fails with
 *     ST_E_CUDA.
 */
#ifndef STENCIL_H
#define STENCIL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct stencil_ctx stencil_ctx; /* opaque; owned by the library */

typedef enum {
  ST_7PT_CONST = 1, /* Fig. 1b */
  ST_7PT_VAR = 2,   /* Fig. 1c */
  ST_25PT_WAVE = 3, /* Fig. 1e, scalar alpha */
  ST_25PT_VAR = 4,  /* Fig. 1d */
  ST_25PT_WAVE_A = 5 /* Fig. 1e exactly as printed: alpha_{z,y,x} a domain-sized field (SURVEY
                        NEXT-1); w0..w4 scalars */
} st_kind;

enum {
  ST_OK = 0,
  ST_E_INVAL = -1, /* bad argument: kind, extent < 1, count mismatch, NULL pointer, T < 1, ... */
  ST_E_NOMEM = -2, /* device allocation failed; the message states the requested bytes */
  ST_E_CUDA = -3,  /* CUDA runtime error (message appended); handle poisoned */
  ST_E_NCCL = -4,  /* NCCL error (message appended); handle poisoned */
  ST_E_STATE = -5  /* handle poisoned by an earlier failure, or used concurrently */
};

/* Kernel variants.  All variants evaluate the same per-point expression with the same
 * operation order, so their results are bitwise identical (test G4). */
enum {
  ST_VARIANT_AUTO = 0,   /* library's choice for the kind and shape (the benchmarked plan) */
  ST_VARIANT_NAIVE = 1,  /* one thread per point, one launch per time step (the GPU naive sweep) */
  ST_VARIANT_STREAM = 2, /* 2.5-D z-streaming; with bt > 1 the time-skewed wavefront of
                            bt fused levels over overlapped xy tiles (P:569-602 transposed);
                            loads through registers, one CTA per tile and z-chunk */
  ST_VARIANT_PIPE = 3,   /* the same wavefront with TMA-fed shared-memory rings: a producer warp
                            streams planes and coefficient fields ahead with cp.async.bulk.tensor +
                            mbarriers; persistent CTAs.  The default.  bt per kind:
                            7c <= 8, 7v <= 5, the 25-point kinds <= 2 (two fused levels of the
                            25-point stencils run the two-level kernel of DESIGN.md §5b, whose
                            z-chains are carried in tensor memory), the alpha-field wave 1.  Library
                            defaults: 7c 4, 7v 4, 25v 2, the waves 1 (the Python binding applies
                            tools/tune.py's measured plan for known shapes). */
  ST_VARIANT_COOP = 4    /* small, latency-bound grids (their arrays fit in L2): all T steps of a
                            stencil_run in ONE cooperative launch, a grid-wide barrier between
                            sweeps.  Single slab only.  Auto-selected below a size threshold.
                            tile_cfg 2 (7-point Jacobi kinds): temporal blocking in shared memory,
                            one grid barrier per round of 5 levels. */
};

/* Halo exchange between z-slabs. */
enum {
  ST_HALO_COPY = 0, /* after every fused block the R*bt boundary planes are copied (device copies
                       between the slabs of one handle; NCCL send/recv between processes on a comm
                       stream).  Bulk-synchronous by default (one launch per slab, then the copy);
                       STENCIL_OVERLAP=1: edge kernels first and the copy overlapping the interior
                       kernel ("halo-first").  The default mode. */
  ST_HALO_PEER = 1  /* fused: one kernel per slab and block; the kernel stores the planes that are a
                       z-neighbour's halo straight into the neighbour's buffer as it produces them
                       (another slab of this handle, or the neighbour process's GPU memory mapped over
                       NVLink with CUDA IPC), then a stream-ordered flag write in the neighbour's
                       memory tells it the block's halos have landed (cuStreamWriteValue64); before
                       its next block each rank's host polls its flags (timeout
                       STENCIL_PEER_TIMEOUT_MS, default 120 s -> ST_E_STATE), so no GPU stream waits
                       on another process.  No edge/interior split, no copy, no NCCL at all (no
                       nccl_id needed).  Pipe variant only.  With one slab per handle every rank must
                       call stencil_peer_export / stencil_peer_import after creating and before
                       running (ranks may also be several handles of one process: their descriptors
                       are then used without IPC). */
};

/* Device allocator: return a device pointer to >= bytes (256-byte aligned) or NULL. */
typedef void *(*st_alloc_fn)(size_t bytes, void *stream, void *user);
typedef void (*st_free_fn)(void *ptr, size_t bytes, void *stream, void *user);

typedef struct {
  int device;          /* CUDA ordinal; -1 = the current device */
  int variant;         /* ST_VARIANT_*; 0 = auto */
  int bt;              /* time-block depth (levels fused per launch); 0 = auto; >= 1 otherwise */
  int tile_cfg;        /* kernel tile configuration index of the variant (0 = default; an index the
                          pipe / stream variants do not define selects the default; ST_VARIANT_COOP
                          accepts 0, 1 and, for the 7-point Jacobi kinds, 2 -- else ST_E_INVAL).
                          25-point variable at bt = 2 (pipe25.cu): 0 = 32x24 overlapped tile, 1 / 2 =
                          cluster pair / quad, 3 = skewed tiles (non-redundant in y; the library then
                          allocates one more state-sized exchange buffer per slab) */
  int local_slabs;     /* z-slabs held by this handle: 1 (one slab per process and GPU; neighbours
                          exchange halos with NCCL), or nranks with rank = 0 ("loopback": all slabs
                          on this handle's device, halos exchanged by device copies -- the multi-GPU
                          plan on one GPU) */
  int zchunk;          /* planes per CTA z-chunk; 0 = auto */
  int rank, nranks;    /* z-slab decomposition over nranks processes (one GPU each); 1 = single */
  const void *nccl_id; /* nranks > 1: 128-byte ncclUniqueId made by rank 0 (stencil_nccl_unique_id)
                          and broadcast by the caller (the Python binding uses torch.distributed) */
  void *stream;        /* cudaStream_t to enqueue on; NULL = the legacy default stream */
  st_alloc_fn alloc;   /* NULL = cudaMalloc */
  st_free_fn free;     /* NULL = cudaFree */
  void *alloc_user;
  int halo;            /* ST_HALO_COPY (0) or ST_HALO_PEER; used when nranks > 1.  ST_HALO_PEER across
                          processes allocates the state buffers with cudaMalloc (CUDA IPC needs whole
                          allocations), ignoring alloc/free for them */
  int host_slab;       /* 0: host arrays of stencil_create / stencil_write are GLOBAL padded arrays.
                          1 (nranks > 1, local_slabs = 1, bt >= 1): they hold only this rank's stored
                          planes [store_z0, store_z1) of stencil_plan_slab(nz, R, nranks, rank, bt) --
                          a rank never needs the other ranks' inputs in host memory */
} st_opts;

typedef struct {
  int kind, R, bt, variant, rank, nranks, local_slabs;
  int tile_x, tile_y, zchunk;     /* output tile of the bt-deep launches; z planes per work item */
  int64_t nx, ny, nz;             /* global interior extents */
  int64_t own_z0, own_z1;         /* padded planes [own_z0, own_z1) this handle owns (global index) */
  int64_t pitch, plane;           /* device row pitch and plane stride, in doubles */
  int64_t local_planes;           /* padded planes stored by this handle (owned + halos) */
  int64_t device_bytes;           /* device memory held by the handle */
  int64_t steps_done;             /* time steps applied since creation (Omega^steps_done is level 0) */
  int64_t launches;               /* kernel launches enqueued since creation / last stats reset */
  int halo;                       /* ST_HALO_* in effect */
  int smem_bytes, threads;        /* dynamic shared memory and threads per CTA of the bt-deep launches */
} st_info;

/* Fill *o with defaults: device -1, auto variant/bt/tiles, single rank (local_slabs 1), NULL stream,
 * cudaMalloc. */
void stencil_opts_default(st_opts *o);

/*
 * Create a grid from host arrays.  Every pointer is a HOST pointer to a dense padded array of
 * (nz+2R)*(ny+2R)*(nx+2R) doubles in the GLOBAL layout (every rank passes the global arrays and
 * copies its slab; the library copies everything before returning; the caller keeps ownership) --
 * or, with opts->host_slab = 1, to the (store_z1-store_z0)*(ny+2R)*(nx+2R) doubles of this rank's
 * stored planes only (same layout, plane store_z0 first).
 *   v0      : Omega^0, ghosts included (fixed boundary values).
 *   u0      : wave kinds (3, 5) only: Omega^{-1}; only its interior is used (ghosts come from v0).
 *             Other kinds: must be NULL.
 *   coeff   : n_coeff pointers.  ST_7PT_CONST: 2 pointers to one double each (w1 centre, w2
 *             neighbour).  ST_25PT_WAVE: 6 pointers to one double each (w0, w1, w2, w3, w4, alpha).
 *             ST_7PT_VAR: 7 padded fields W0..W6.  ST_25PT_VAR: 13 padded fields W0..W12 in
 *             Fig. 1c / 1d numbering.  ST_25PT_WAVE_A: 6 pointers, w0..w4 (one double each) then
 *             the padded alpha field.  Only the interior cells of a field are read.
 *   opts    : NULL = defaults.
 * Errors: ST_E_INVAL (kind, extent < 1, n_coeff, NULL, nz < nranks, rank out of range),
 *         ST_E_NOMEM, ST_E_CUDA, ST_E_NCCL.
 */
int stencil_create(stencil_ctx **out, int kind, int64_t nx, int64_t ny, int64_t nz,
                   const double *const *coeff, int n_coeff, const double *v0, const double *u0,
                   const st_opts *opts);

/*
 * Create a grid whose inputs are drawn on the device by the seeded generator of synth/synth.h
 * (reading Q6): V^0 and ghosts ~ U[-1,1) (stream 0); wave
 * Omega^{-1} interior ~ U[-1,1) (stream 1); W_i ~ U[0,1/7) or U[0,1/25) (stream 2+i).  The draw is
 * a function of the global padded index, so every rank fills its own slab without communication.
 * ST_25PT_WAVE_A's alpha field ~ U[0, 0.2) (stream 2; the leapfrog is stable for alpha < 0.205).
 *   scalars : constant kinds: 2 (7-point) or 6 (wave) doubles in the order of stencil_create's coeff,
 *             ST_25PT_WAVE_A: 5 (w0..w4); NULL = the BASELINE.json values (0.4, 0.1) /
 *             (3*(-205/72), 8/5, -1/5, 8/315, -1/560, 0.1).  Variable kinds 2, 4: must be NULL.
 */
int stencil_create_seeded(stencil_ctx **out, int kind, int64_t nx, int64_t ny, int64_t nz,
                          uint64_t seed, const double *scalars, const st_opts *opts);

/*
 * Host copy of the seeded input a stencil_create_seeded handle draws on the device (synth/synth.h,
 * DESIGN.md readings Q6-Q9, Q21), same bits: writes the dense padded GLOBAL array
 * (nz+2R)(ny+2R)(nx+2R) of one input into out (HOST pointer, out_elems >= that size).  No device is
 * needed.  stream_id: 0 = V^0 (Omega^0 incl. ghosts, U[-1,1)); 1 = the wave's Omega^{-1} (interior
 * from stream 1, ghosts from stream 0; ST_25PT_WAVE / _A only); 2 + i = coefficient field W_i of the
 * variable kinds (U[0,1/7) / U[0,1/25)) or the alpha field of ST_25PT_WAVE_A (i = 0, U[0,0.2)).
 * ST_E_INVAL for a stream the kind does not have, extents < 1, NULL or short out.
 */
int stencil_generate(int kind, int64_t nx, int64_t ny, int64_t nz, uint64_t seed, int stream_id, double *out,
                     int64_t out_elems);

/* Enqueue T >= 1 time steps (T < 1 -> ST_E_INVAL).  Asynchronous on opts->stream.
 * Multi-rank: collective; every rank calls it with the same T. */
int stencil_run(stencil_ctx *h, int64_t T);

/* Block until the handle's enqueued work is done. */
int stencil_sync(stencil_ctx *h);

/*
 * Copy a time level to the host.  level 0 = Omega^t (newest), level 1 = Omega^{t-1} (wave kinds
 * only; ST_E_INVAL for the Jacobi kinds, whose level 1 is scratch).  out: HOST pointer to a dense
 * padded GLOBAL array of out_elems >= (nz+2R)(ny+2R)(nx+2R) doubles; this rank writes the padded
 * planes it owns ([own_z0, own_z1) of st_info; rank 0 owns the bottom R ghost planes, the last
 * rank the top R) and leaves the other planes untouched.  Synchronizes.
 */
int stencil_read(stencil_ctx *h, int level, double *out, int64_t out_elems);

/* Copy padded planes [z0, z1) (global indices, inside this rank's owned range) of a level to a dense
 * host array of (z1-z0)(ny+2R)(nx+2R) doubles.  Synchronizes. */
int stencil_read_planes(stencil_ctx *h, int level, int64_t z0, int64_t z1, double *out,
                        int64_t out_elems);

/* Overwrite a level from a dense padded GLOBAL host array (interior and ghosts of this rank's
 * stored planes) -- with opts->host_slab, from an array of this rank's stored planes only.  Used for
 * checkpoint/resume and the end-to-end upload path.  level 1 only for the wave.  The fixed boundary
 * is level 0's ghost shell: writing level 0 also resets the other buffers' ghosts to the new ghosts;
 * writing level 1 (wave) uses only the interior of `in` (its ghosts stay level 0's, as u0 in
 * stencil_create).  ST_E_INVAL if in_elems is too small. */
int stencil_write(stencil_ctx *h, int level, const double *in, int64_t in_elems);

/* Plan and state of a handle. */
int stencil_info(const stencil_ctx *h, st_info *out);

/* Per-launch device timing of the library's own kernels (CUDA events on opts->stream).
 * enable != 0: record an event pair around every kernel launch from now on.  stencil_kernel_time
 * synchronizes and returns the summed kernel milliseconds and the number of timed launches since
 * the last reset (reset != 0 clears both afterwards). */
int stencil_set_timing(stencil_ctx *h, int enable);
int stencil_kernel_time(stencil_ctx *h, double *ms, int64_t *launches, int reset);

/* Release all device memory and the NCCL communicator.  NULL is a no-op. */
int stencil_destroy(stencil_ctx *h);

/* Thread-local description of the last error on this thread ("" if none). */
const char *stencil_last_error(void);

/* Write a fresh 128-byte ncclUniqueId into out (rank 0 of a multi-rank run). */
int stencil_nccl_unique_id(void *out, size_t out_bytes);

/*
 * Host-side plan of the z-slab decomposition; pure function, no device needed.
 * The nz interior planes are split into nranks contiguous slabs, remainder planes to the lowest
 * ranks.  Outputs (global padded plane indices): [*own_z0, *own_z1) the planes rank owns (its
 * interior slab, plus the bottom / top R ghost planes on the first / last rank);
 * [*store_z0, *store_z1) the planes it stores (owned + halo of depth R*bt on internal sides).
 * With st_opts.host_slab the handle must run at exactly this bt: stencil_create returns ST_E_INVAL
 * when the kind / variant caps bt lower (the stored range would differ from the caller's arrays).
 * bt is clamped to max(1, min(bt, thinnest slab / R)) and returned in *bt_eff, so halo data always
 * comes from the adjacent rank only.  ST_E_INVAL if nz < nranks or (nranks > 1 and a slab is
 * thinner than R planes).
 */
int stencil_plan_slab(int64_t nz, int R, int nranks, int rank, int bt, int64_t *own_z0,
                      int64_t *own_z1, int64_t *store_z0, int64_t *store_z1, int *bt_eff);

/*
 * ST_HALO_PEER across processes (one slab per process): wire the z-neighbours' memory.
 * stencil_peer_export writes this rank's descriptor (CUDA IPC handles of its state buffers and of
 * its halo-arrival flags, plus its slab geometry) into desc[0 .. ST_PEER_DESC_BYTES).  The caller
 * moves the descriptors between processes (the Python binding all-gathers them with
 * torch.distributed) and every rank calls stencil_peer_import with the descriptors of rank-1
 * ("below", NULL on rank 0) and rank+1 ("above", NULL on the last rank).  Collective: all ranks must
 * import before any rank runs.  Errors: ST_E_INVAL (wrong mode, short buffer, descriptor of the
 * wrong rank / geometry, missing neighbour), ST_E_CUDA (IPC mapping failed, e.g. no peer access).
 */
#define ST_PEER_DESC_BYTES 512
int stencil_peer_export(stencil_ctx *h, void *desc, size_t desc_bytes);
int stencil_peer_import(stencil_ctx *h, const void *below, const void *above);

/*
 * Optional check after stencil_peer_import (collective, before the first run): every rank stores a
 * rank-tagged word into each neighbour's memory with a kernel (the fused halo stores' path) and
 * with a stream-ordered flag write (the block signal's path), then polls its own memory from the
 * host for the neighbours' words -- it never blocks the GPU.  ST_OK when both arrived, ST_E_STATE
 * after timeout_ms (the caller can then fall back to ST_HALO_COPY on every rank).
 */
int stencil_peer_handshake(stencil_ctx *h, int timeout_ms);

/* Library version string. */
const char *stencil_version(void);

#ifdef __cplusplus
}
#endif

#endif /* STENCIL_H */
