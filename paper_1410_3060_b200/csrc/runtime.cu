// runtime.cu -- libstencil.so: the C ABI of include/stencil.h and the runtime behind it.
//
// Plan (§8(e)): device layout, time-block schedule
// (ceil(T/bt) launches, last one T mod bt levels, reading Q16), buffer-role rotation of the
// two time levels, z-slab decomposition with R*bt-deep halos.
//
// A handle owns one or more consecutive z-slabs of the global grid ("slabs").  After every fused block
// of b levels the R*b boundary planes of the new level are exchanged between neighbouring slabs:
//   * slabs of the same handle (opts.local_slabs = nranks, one process, one GPU): device-to-device
//     copies on the handle's stream ("loopback"; the same plan as multi-GPU, testable on one GPU);
//   * slabs of different processes (one slab per process and GPU): NCCL send/recv in one group.
// With opts.halo = ST_HALO_PEER the exchange is fused into the kernel instead: one launch per slab
// and block stores the neighbours' halo planes straight into their buffers (pipe kernel, KParams
// rdst), and across processes a stream-ordered flag write into the neighbour's memory (CUDA IPC)
// announces the block; the neighbour's stream waits on that flag before its next block.
#include "../../include/stencil.h"
#include "kernels.cuh"
#include "../../synth/synth.h"

#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <mutex>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#ifndef STENCIL_VERSION
#define STENCIL_VERSION "0.2.0"
#endif

namespace {

thread_local std::string g_err;

void set_err(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
}

int radius_of(int kind) { return (kind == 1 || kind == 2) ? 1 : (kind >= 3 && kind <= 5) ? 4 : -1; }
int ncoef_of(int kind) { return kind == 2 ? 7 : kind == 4 ? 13 : kind == 5 ? 1 : 0; }  // domain-sized fields
int nscal_of(int kind) { return kind == 1 ? 2 : kind == 3 ? 6 : kind == 5 ? 5 : 0; }    // scalar weights
bool is_wave(int kind) { return kind == ST_25PT_WAVE || kind == ST_25PT_WAVE_A; }

// ---------------------------------------------------------------- NCCL, loaded at run time
// The Python binding imports torch first, so libnccl.so.2 (torch's) is normally already loaded;
// RTLD_NOLOAD picks that copy so the process never holds two NCCLs.
struct Nccl {
  bool ok = false;
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
};

Nccl* nccl() {
  static Nccl n;
  static bool tried = false;
  if (tried) return n.ok ? &n : nullptr;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
  if (!h) {
    const char* env = getenv("STENCIL_NCCL_LIB");
    if (env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
  }
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) { set_err("cannot load libnccl.so.2: %s", dlerror()); return nullptr; }
#define LOAD(f) n.f = (decltype(n.f))dlsym(h, "nccl" #f); if (!n.f) { set_err("nccl symbol nccl%s missing", #f); return nullptr; }
  LOAD(GetUniqueId) LOAD(CommInitRank) LOAD(CommDestroy) LOAD(Send) LOAD(Recv) LOAD(GroupStart)
  LOAD(GroupEnd) LOAD(GetErrorString)
#undef LOAD
  n.ok = true;
  return &n;
}

// ---------------------------------------------------------------- stream memory operations
// (driver API, resolved through the runtime so the library does not link libcuda directly)
using WaitValue64Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
using WriteValue64Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
struct MemOps {
  WaitValue64Fn wait = nullptr;
  WriteValue64Fn write = nullptr;
};
const MemOps& memops() {
  static MemOps m;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue64", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      m.wait = reinterpret_cast<WaitValue64Fn>(f);
    f = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue64", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      m.write = reinterpret_cast<WriteValue64Fn>(f);
  });
  return m;
}

// Descriptor of one rank's memory for ST_HALO_PEER (stencil_peer_export / import).
struct PeerDesc {
  uint64_t magic;
  int32_t rank, nranks, kind, nbuf, bt, pad;
  int64_t nx, ny, nz, pitch, plane, store_z0, zl;
  int64_t pid;                  // exporting process: a descriptor from this process is used directly
  uint64_t raw_buf[4], raw_flags;  // (the neighbour is another handle here, e.g. two ranks emulated
  int32_t device, pad2;            //  on one GPU in one process; CUDA IPC cannot open own handles)
  cudaIpcMemHandle_t buf[4];
  cudaIpcMemHandle_t flags;
};
constexpr uint64_t kPeerMagic = 0x3330363031343153ull;  // "S1410603"
static_assert(sizeof(PeerDesc) <= ST_PEER_DESC_BYTES, "peer descriptor too large");

// One z-slab: global padded planes [store_z0, store_z1) stored, [own_z0, own_z1) owned,
// interior planes [lo, hi) computed.
struct Slab {
  int rank = 0;
  int64_t own_z0 = 0, own_z1 = 0, store_z0 = 0, store_z1 = 0, zl = 0, lo = 0, hi = 0;
  double* buf[4] = {nullptr, nullptr, nullptr, nullptr};  // raw (un-offset) state buffers
  double* coef = nullptr;                                  // raw coefficient slab
  double* xch = nullptr;  // skewed 25v tiles: level-1 rows handed between tiles (raw, lazily allocated)
};

}  // namespace

// ---------------------------------------------------------------- the handle
struct stencil_ctx {
  int kind = 0, R = 0, ncoef = 0, nscal = 0;
  int64_t nx = 0, ny = 0, nz = 0;
  int rank = 0, nranks = 1, local = 1;  // first local slab's rank, total slabs, slabs on this handle
  int device = 0, num_sms = 148;
  int variant = ST_VARIANT_PIPE, bt = 1, zchunk_req = 0, tile_cfg = 0;
  cudaStream_t stream = nullptr;
  bool host_slab = false;  // host arrays hold only the stored planes (st_opts.host_slab)
  // global padded plane of host array plane 0
  int64_t host_z0() const { return host_slab ? slabs.front().store_z0 : 0; }
  st_alloc_fn alloc = nullptr;
  st_free_fn free_fn = nullptr;
  void* alloc_user = nullptr;

  // layout (elements), common to all slabs
  int64_t X = 0, Y = 0, pitch = 0, plane = 0, xoff = 0;
  std::vector<Slab> slabs;
  int nbuf = 2;
  int lv0 = 0, lv1 = 1;  // buffer index of Omega^t and Omega^{t-1} (same in every slab)
  double scal[6] = {0, 0, 0, 0, 0, 0};
  unsigned int* sched = nullptr;  // pipe kernel work counters (zero between launches)
  unsigned int* done = nullptr;   // per-item completion counters of multi-block launches (lazy)
  unsigned int* xflag = nullptr;  // skewed 25v tiles: per-item export flags (lazy), xflag_n entries
  long long xflag_n = 0;
  unsigned int xbase = 0;         // flag base of the last skewed launch (+65536 per launch)

  std::vector<std::pair<void*, size_t>> allocs;
  int64_t steps = 0;
  int64_t launches = 0;
  int64_t device_bytes = 0;
  bool poisoned = false;
  std::atomic<int> busy{0};
  st::LaunchInfo last_launch{};

  bool timing = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> events;
  size_t events_used = 0;

  ncclComm_t comm = nullptr;
  // halo-first overlap (nranks > 1): the exchange runs on comm_stream after the edge kernels
  // (ev_edge) while the interior kernels run on `stream`; ev_halo marks the exchange's completion.
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_edge = nullptr, ev_halo = nullptr;
  bool halo_pending = false;
  bool overlap = false;  // STENCIL_OVERLAP=1: halo-first schedule (edge kernels, exchange, interior kernel)

  // ST_HALO_PEER (fused halo exchange)
  int halo = ST_HALO_COPY;
  int64_t blocks = 0;            // fused blocks run since creation (the flag protocol's counter)
  bool peer_ready = false;       // neighbours wired (loopback: at create; processes: after import)
  bool ipc = false;              // peers are other processes (CUDA IPC)
  uint64_t* flags = nullptr;     // this rank's halo-arrival counters: [0] from below, [1] from above
  cudaStream_t poll_stream = nullptr;  // host-side polls of `flags` (peer_wait)
  struct Peer {
    bool on = false;
    bool opened = false;  // pointers come from cudaIpcOpenMemHandle (closed at release)
    double* buf[4] = {nullptr, nullptr, nullptr, nullptr};  // raw state buffers (IPC-mapped)
    uint64_t* flags = nullptr;                              // the neighbour's counters
    int64_t store_z0 = 0;
  } peer[2];                     // [0] below (rank - 1), [1] above (rank + 1)

  double* at(const Slab& s, int b) const { return s.buf[b] + xoff; }
  int64_t own_z0() const { return slabs.front().own_z0; }
  int64_t own_z1() const { return slabs.back().own_z1; }
};

namespace {

struct Guard {  // not reentrant: one thread at a time per handle
  stencil_ctx* h;
  bool ok;
  explicit Guard(stencil_ctx* hh) : h(hh), ok(false) {
    int z = 0;
    ok = h->busy.compare_exchange_strong(z, 1);
  }
  ~Guard() { if (ok) h->busy.store(0); }
};

int cuda_fail(stencil_ctx* h, cudaError_t e, const char* what) {
  set_err("%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
  if (h) h->poisoned = true;
  return ST_E_CUDA;
}

#define CK(expr, what)                                   \
  do {                                                   \
    cudaError_t _e = (expr);                             \
    if (_e != cudaSuccess) return cuda_fail(h, _e, what); \
  } while (0)

void* dev_alloc(stencil_ctx* h, size_t bytes) {
  void* p = nullptr;
  if (h->alloc) {
    p = h->alloc(bytes, (void*)h->stream, h->alloc_user);
  } else if (cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    p = nullptr;
  }
  if (p) {
    h->allocs.emplace_back(p, bytes);
    h->device_bytes += (int64_t)bytes;
  }
  return p;
}

void release(stencil_ctx* h) {
  cudaStreamSynchronize(h->stream);
  for (auto& pr : h->peer) {
    if (!h->ipc || !pr.on || !pr.opened) continue;
    for (auto* b : pr.buf)
      if (b) cudaIpcCloseMemHandle(b);
    if (pr.flags) cudaIpcCloseMemHandle(pr.flags);
    pr = stencil_ctx::Peer{};
  }
  for (auto& a : h->allocs) {
    if (h->free_fn) h->free_fn(a.first, a.second, (void*)h->stream, h->alloc_user);
    else cudaFree(a.first);
  }
  h->allocs.clear();
  for (auto& e : h->events) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
  h->events.clear();
  if (h->comm && nccl()) nccl()->CommDestroy(h->comm);
  h->comm = nullptr;
  if (h->comm_stream) cudaStreamSynchronize(h->comm_stream), cudaStreamDestroy(h->comm_stream);
  if (h->poll_stream) cudaStreamDestroy(h->poll_stream);
  h->poll_stream = nullptr;
  if (h->ev_edge) cudaEventDestroy(h->ev_edge);
  if (h->ev_halo) cudaEventDestroy(h->ev_halo);
  h->comm_stream = nullptr;
  h->ev_edge = h->ev_halo = nullptr;
}

// Debug / fault-injection knobs, read at every call so tests can toggle them (never set in production).
int env_int(const char* name) {
  const char* v = getenv(name);
  return v ? atoi(v) : 0;
}

// ST_VARIANT_AUTO picks the cooperative all-steps kernel for grids of at most this many padded cells
// (tools/coop_sweep.py on B200, T = 10: faster than the pipe kernel for every kind at 66^3-72^3, for
// 7c at 130^3 (214 vs 135 GLUP/s), 25w / 25v at 104^3; even with 7v at 130^3; slower for 7c at 194^3).
constexpr double kCoopAutoCells = 3.0e6;

int default_bt(int kind) {
  switch (kind) {
    case ST_7PT_CONST: return 4;  // tools/sweep.py on B200
    case ST_7PT_VAR: return 4;  // tools/tune.py (round 2, sustained): 196.1 vs 190.1 GLUP/s at bt = 3
    case ST_25PT_VAR: return 2;  // pipe25.cu (round 2): C4 57.8 vs 52.8 GLUP/s at bt = 1, same box
    default: return 1;
  }
}

int plan_slab(int64_t nz, int R, int nranks, int rank, int bt, Slab* s, int* bt_eff) {
  if (nz < 1 || R < 1 || nranks < 1 || rank < 0 || rank >= nranks || nz < nranks || bt < 0) {
    set_err("plan_slab: bad arguments (nz=%lld R=%d nranks=%d rank=%d bt=%d)", (long long)nz, R,
            nranks, rank, bt);
    return ST_E_INVAL;
  }
  const int64_t base = nz / nranks, rem = nz % nranks;
  const int64_t thin = base;  // thinnest slab
  if (nranks > 1 && thin < R) {
    set_err("plan_slab: slabs of %lld planes are thinner than the radius %d (nz=%lld, nranks=%d)",
            (long long)thin, R, (long long)nz, nranks);
    return ST_E_INVAL;
  }
  int b = std::max(1, bt);
  if (nranks > 1) b = (int)std::max<int64_t>(1, std::min<int64_t>(b, thin / R));
  const int64_t lo = R + rank * base + std::min<int64_t>(rank, rem);
  const int64_t hi = lo + base + (rank < rem ? 1 : 0);
  const int64_t H = (int64_t)R * b;
  s->rank = rank;
  s->lo = lo;
  s->hi = hi;
  s->own_z0 = rank == 0 ? 0 : lo;
  s->own_z1 = rank == nranks - 1 ? nz + 2 * R : hi;
  s->store_z0 = rank == 0 ? 0 : lo - H;
  s->store_z1 = rank == nranks - 1 ? nz + 2 * R : hi + H;
  s->zl = s->store_z1 - s->store_z0;
  if (bt_eff) *bt_eff = b;
  return ST_OK;
}

// Common part of both create calls: validation, device, plan, allocation, communicator.
int create_common(stencil_ctx** out, int kind, int64_t nx, int64_t ny, int64_t nz,
                  const st_opts* opts_in, stencil_ctx** hp) {
  if (!out) { set_err("out is NULL"); return ST_E_INVAL; }
  *out = nullptr;
  st_opts o;
  stencil_opts_default(&o);
  if (opts_in) o = *opts_in;
  const int R = radius_of(kind);
  if (R < 0) { set_err("bad kind %d", kind); return ST_E_INVAL; }
  if (nx < 1 || ny < 1 || nz < 1) { set_err("extents must be >= 1 (got %lld %lld %lld)", (long long)nx, (long long)ny, (long long)nz); return ST_E_INVAL; }
  if (nx > (1 << 30) || ny > (1 << 30)) { set_err("extent too large"); return ST_E_INVAL; }
  if (o.bt < 0 || o.variant < 0 || o.variant > ST_VARIANT_COOP || o.zchunk < 0 || o.tile_cfg < 0) {
    set_err("bad options (bt=%d variant=%d zchunk=%d tile_cfg=%d)", o.bt, o.variant, o.zchunk, o.tile_cfg);
    return ST_E_INVAL;
  }
  if (o.nranks < 1 || o.rank < 0 || o.rank >= o.nranks) { set_err("bad rank %d of %d", o.rank, o.nranks); return ST_E_INVAL; }
  const int local = o.local_slabs < 1 ? 1 : o.local_slabs;
  if (!(local == 1 || (local == o.nranks && o.rank == 0))) {
    set_err("local_slabs must be 1 (one slab per process) or nranks with rank 0 (got %d of %d)", local, o.nranks);
    return ST_E_INVAL;
  }
  if (nz < o.nranks) { set_err("nz=%lld < nranks=%d", (long long)nz, o.nranks); return ST_E_INVAL; }
  if (o.halo != ST_HALO_COPY && o.halo != ST_HALO_PEER) { set_err("bad halo mode %d", o.halo); return ST_E_INVAL; }
  if (o.host_slab && (o.nranks < 2 || o.local_slabs != 1 || o.bt < 1)) {
    set_err("host_slab needs nranks > 1, local_slabs = 1 and an explicit bt >= 1 (the stored range must be "
            "known to the caller: stencil_plan_slab)");
    return ST_E_INVAL;
  }
  if (o.variant == ST_VARIANT_COOP && o.nranks > 1) {
    set_err("ST_VARIANT_COOP runs a single slab (nranks = 1)");
    return ST_E_INVAL;
  }
  if (o.variant == ST_VARIANT_COOP &&
      (o.tile_cfg > 2 || (o.tile_cfg == 2 && kind != ST_7PT_CONST && kind != ST_7PT_VAR))) {
    set_err("ST_VARIANT_COOP: tile_cfg %d is not defined for kind %d (0, 1; 2 for the 7-point Jacobi kinds)",
            o.tile_cfg, kind);
    return ST_E_INVAL;
  }
  if (o.halo == ST_HALO_PEER && o.variant != ST_VARIANT_AUTO && o.variant != ST_VARIANT_PIPE) {
    set_err("halo mode ST_HALO_PEER needs the pipe variant (got variant %d)", o.variant);
    return ST_E_INVAL;
  }
  const bool one_slab = o.nranks > 1 && local == 1;           // one slab per process
  const bool use_nccl = one_slab && o.halo == ST_HALO_COPY;   // ST_HALO_PEER needs no communicator
  if (use_nccl && !o.nccl_id) { set_err("nranks > 1 with one slab per process needs nccl_id"); return ST_E_INVAL; }

  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev < 1) {
    cudaGetLastError();
    set_err("no CUDA device available (%s); libstencil has no CPU fallback",
            e != cudaSuccess ? cudaGetErrorString(e) : "0 devices");
    return ST_E_CUDA;
  }
  int dev = o.device;
  if (dev < 0) cudaGetDevice(&dev);
  if (dev >= ndev) { set_err("device %d >= device count %d", dev, ndev); return ST_E_INVAL; }

  stencil_ctx* h = new stencil_ctx();
  *hp = h;
  h->kind = kind; h->R = R; h->ncoef = ncoef_of(kind); h->nscal = nscal_of(kind);
  h->nx = nx; h->ny = ny; h->nz = nz;
  h->rank = o.rank; h->nranks = o.nranks; h->local = local;
  h->device = dev;
  h->stream = (cudaStream_t)o.stream;
  h->alloc = o.alloc; h->free_fn = o.free; h->alloc_user = o.alloc_user;
  h->zchunk_req = o.zchunk;
  h->tile_cfg = o.tile_cfg;
  h->halo = o.nranks > 1 ? o.halo : ST_HALO_COPY;
  h->host_slab = o.host_slab != 0;
  h->ipc = h->halo == ST_HALO_PEER && one_slab;
  if (h->ipc) {  // IPC maps whole allocations: state buffers and flags come straight from cudaMalloc
    h->alloc = nullptr;
    h->free_fn = nullptr;
  }
  CK(cudaSetDevice(dev), "cudaSetDevice");
  CK(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, dev), "device attribute");

  h->variant = o.variant == ST_VARIANT_AUTO ? ST_VARIANT_PIPE : o.variant;
  if (o.variant == ST_VARIANT_AUTO && o.nranks == 1 && o.bt == 0 && o.zchunk == 0 && o.tile_cfg == 0) {
    // small, latency-bound grids: one cooperative launch for all T steps
    const double cells = (double)(nx + 2 * R) * (double)(ny + 2 * R) * (double)(nz + 2 * R);
    if (cells <= kCoopAutoCells) h->variant = ST_VARIANT_COOP;
  }
  int bt = (h->variant == ST_VARIANT_NAIVE || h->variant == ST_VARIANT_COOP) ? 1 : (o.bt ? o.bt : default_bt(kind));
  const int bt_cap = h->variant == ST_VARIANT_PIPE ? st::max_pipe_bt(kind)
                   : h->variant == ST_VARIANT_STREAM ? st::max_stream_bt(kind) : 1;
  bt = std::min(bt, std::max(1, bt_cap));
  if (o.host_slab && bt != o.bt) {
    // the caller sized its host arrays with stencil_plan_slab(..., o.bt): a different depth would shift
    // every stored plane by R*(o.bt - bt) (the stored range is [lo - R*bt, hi + R*bt))
    set_err("host_slab: bt=%d is not available for kind %d with variant %d (at most %d); size the host arrays "
            "for an available bt", o.bt, kind, h->variant, bt);
    return ST_E_INVAL;
  }
  h->slabs.resize(local);
  for (int i = 0; i < local; ++i) {
    int bt_eff = 1;
    int rc = plan_slab(nz, R, o.nranks, o.rank + i, bt, &h->slabs[i], &bt_eff);
    if (rc) return rc;
    h->bt = bt_eff;
  }

  // Device layout: interior column x = R lands on a 128-byte boundary; rows padded to 16 doubles.
  h->X = nx + 2 * R;
  h->Y = ny + 2 * R;
  h->xoff = 16 - R;
  h->pitch = ((h->xoff + h->X) + 15) / 16 * 16;
  h->plane = h->pitch * h->Y;
  h->nbuf = (is_wave(kind) && h->bt >= 2) ? 4 : 2;
  for (auto& s : h->slabs) {
    const size_t bytes = (size_t)h->plane * (size_t)s.zl * sizeof(double);
    for (int b = 0; b < h->nbuf; ++b) {
      s.buf[b] = (double*)dev_alloc(h, bytes);
      if (!s.buf[b]) {
        set_err("device allocation of %zu bytes failed (state buffer %d of slab %d; %lld bytes held)", bytes,
                b, s.rank, (long long)h->device_bytes);
        return ST_E_NOMEM;
      }
    }
    if (h->ncoef) {
      const size_t cb = bytes * (size_t)h->ncoef;
      s.coef = (double*)dev_alloc(h, cb);
      if (!s.coef) {
        set_err("device allocation of %zu bytes failed (%d coefficient fields of slab %d; %lld bytes held)", cb,
                h->ncoef, s.rank, (long long)h->device_bytes);
        return ST_E_NOMEM;
      }
    }
  }
  h->lv0 = 0;
  h->lv1 = 1;
  if (h->halo == ST_HALO_PEER) {
    if (h->ipc) {
      h->flags = (uint64_t*)dev_alloc(h, 256);
      if (!h->flags) { set_err("device allocation of 256 bytes failed (halo flags)"); return ST_E_NOMEM; }
      CK(cudaMemsetAsync(h->flags, 0, 256, h->stream), "zero halo flags");
    } else {  // loopback: the neighbours are the handle's own slabs, stream-ordered
      h->peer_ready = true;
    }
  }
  h->sched = (unsigned int*)dev_alloc(h, 256);
  if (!h->sched) { set_err("device allocation of 256 bytes failed"); return ST_E_NOMEM; }
  CK(cudaMemsetAsync(h->sched, 0, 256, h->stream), "zero work counters");

  if (o.nranks > 1) {
    CK(cudaStreamCreateWithFlags(&h->comm_stream, cudaStreamNonBlocking), "comm stream");
    CK(cudaEventCreateWithFlags(&h->ev_edge, cudaEventDisableTiming), "event");
    CK(cudaEventCreateWithFlags(&h->ev_halo, cudaEventDisableTiming), "event");
    // Bulk-synchronous by default (one launch per slab and block, then the exchange): the halo-first
    // overlap's edge kernels stream R*bt-plane slabs through a z-stream that needs 2*R*bt fill/drain planes,
    // ~3x their output, which costs more than the exchange it hides over NVLink (C5 at bt = 2, 256-plane
    // slabs: ~12 % edge overhead vs a 0.2 ms exchange per 9 ms block).  STENCIL_OVERLAP=1
    // selects the halo-first schedule.
    const char* ov = getenv("STENCIL_OVERLAP");
    h->overlap = ov && atoi(ov);
  }
  if (use_nccl) {
    Nccl* n = nccl();
    if (!n) { h->poisoned = true; return ST_E_NCCL; }
    ncclUniqueId id;
    memcpy(&id, o.nccl_id, sizeof id);
    ncclResult_t r = n->CommInitRank(&h->comm, o.nranks, id, o.rank);
    if (r != ncclSuccess) {
      set_err("ncclCommInitRank: %s", n->GetErrorString(r));
      h->comm = nullptr;
      h->poisoned = true;
      return ST_E_NCCL;
    }
  }
  return ST_OK;
}

// Copy dense padded global host planes [store_z0, store_z1) of slab s into its device buffer raw.
// Staged: chunks of planes go host -> a dense device staging slot in one contiguous copy each (55 GB/s,
// the PCIe peak), then a device-to-device pitched copy into the library layout (a pitched cudaMemcpy2D
// straight from host memory ran at ~31 GB/s on B200; tools/pcie_probe.py).  Two slots: the repack of
// chunk i runs on an auxiliary stream while chunk i+1 crosses PCIe (on a busy GPU the repack competes
// with the kernels for HBM and would otherwise stall the upload).  Without staging memory (allocation
// failed, or STENCIL_NO_STAGE) the direct 2-D copy is used.
constexpr int64_t kStagePlanes = 32;
struct Stager {
  stencil_ctx* h;
  double* slot[2] = {nullptr, nullptr};
  size_t bytes = 0;
  cudaStream_t aux = nullptr;
  cudaEvent_t h2d[2] = {nullptr, nullptr}, d2d[2] = {nullptr, nullptr};
  int64_t n = 0;  // chunks issued

  explicit Stager(stencil_ctx* hh) : h(hh) {
    if (env_int("STENCIL_NO_STAGE")) return;  // experiment knob: direct pitched host copies
    bytes = (size_t)(kStagePlanes * h->X * h->Y) * sizeof(double);
    for (int i = 0; i < 2; ++i) slot[i] = alloc_one();
    if (slot[1] && (cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking) != cudaSuccess ||
                    cudaEventCreateWithFlags(&h2d[0], cudaEventDisableTiming) != cudaSuccess ||
                    cudaEventCreateWithFlags(&h2d[1], cudaEventDisableTiming) != cudaSuccess ||
                    cudaEventCreateWithFlags(&d2d[0], cudaEventDisableTiming) != cudaSuccess ||
                    cudaEventCreateWithFlags(&d2d[1], cudaEventDisableTiming) != cudaSuccess)) {
      cudaGetLastError();
      drop_aux();
    }
  }
  double* alloc_one() {
    void* p = nullptr;
    if (h->alloc) p = h->alloc(bytes, (void*)h->stream, h->alloc_user);
    else if (cudaMalloc(&p, bytes) != cudaSuccess) { cudaGetLastError(); p = nullptr; }
    return (double*)p;
  }
  void drop_aux() {
    for (int i = 0; i < 2; ++i) {
      if (h2d[i]) cudaEventDestroy(h2d[i]);
      if (d2d[i]) cudaEventDestroy(d2d[i]);
      h2d[i] = d2d[i] = nullptr;
    }
    if (aux) cudaStreamDestroy(aux);
    aux = nullptr;
  }
  cudaError_t upload(const Slab& s, double* raw, const double* host) {
    const double* src = host + (size_t)(s.store_z0 - h->host_z0()) * h->X * h->Y;
    if (!slot[0])
      return cudaMemcpy2DAsync(raw + h->xoff, h->pitch * sizeof(double), src, h->X * sizeof(double),
                               h->X * sizeof(double), (size_t)h->Y * s.zl, cudaMemcpyHostToDevice, h->stream);
    const int64_t hplane = h->X * h->Y;
    for (int64_t z0 = 0; z0 < s.zl; z0 += kStagePlanes, ++n) {
      const int64_t nz = std::min<int64_t>(kStagePlanes, s.zl - z0);
      const int k = aux ? (int)(n & 1) : 0;
      cudaError_t e = cudaSuccess;
      if (aux && n >= 2) e = cudaStreamWaitEvent(h->stream, d2d[k], 0);  // slot k's previous repack is done
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(slot[k], src + z0 * hplane, (size_t)(nz * hplane) * sizeof(double), cudaMemcpyHostToDevice,
                            h->stream);
      cudaStream_t rs = h->stream;
      if (e == cudaSuccess && aux) {
        e = cudaEventRecord(h2d[k], h->stream);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(aux, h2d[k], 0);
        rs = aux;
      }
      if (e == cudaSuccess)  // repack by the copy engine (~3.4 TB/s)
        e = cudaMemcpy2DAsync(raw + h->xoff + z0 * h->plane, h->pitch * sizeof(double), slot[k], h->X * sizeof(double),
                              h->X * sizeof(double), (size_t)(nz * h->Y), cudaMemcpyDeviceToDevice, rs);
      if (e == cudaSuccess && aux) e = cudaEventRecord(d2d[k], aux);
      if (e != cudaSuccess) return e;
    }
    return finish();  // later work on h->stream (and the caller's device copies) sees the planes
  }
  cudaError_t finish() {
    if (!aux) return cudaSuccess;
    for (int k = 0; k < 2 && k < n; ++k) {
      cudaError_t e = cudaStreamWaitEvent(h->stream, d2d[k], 0);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  ~Stager() {
    finish();  // the slots are released in h->stream order, after the last repack that reads them
    for (int i = 0; i < 2; ++i) {
      if (!slot[i]) continue;
      if (h->free_fn) h->free_fn(slot[i], bytes, (void*)h->stream, h->alloc_user);
      else { cudaStreamSynchronize(h->stream); cudaFree(slot[i]); }
    }
    drop_aux();  // destroying a stream / event with work pending is safe (released on completion)
  }
};

void fail_create(stencil_ctx* h) {
  if (!h) return;
  release(h);
  delete h;
}

st::KParams base_params(stencil_ctx* h, const Slab& s) {
  st::KParams p{};
  p.coef = s.coef ? s.coef + h->xoff : nullptr;
  p.cstride = h->plane * s.zl;
  p.pitch = h->pitch;
  p.plane = h->plane;
  p.nx = (int)h->nx;
  p.ny = (int)h->ny;
  p.zl = (int)s.zl;
  p.zi0 = (int)std::max<int64_t>(0, h->R - s.store_z0);
  p.zi1 = (int)std::min<int64_t>(s.zl, h->nz + h->R - s.store_z0);
  p.zo0 = (int)(s.lo - s.store_z0);
  p.zo1 = (int)(s.hi - s.store_z0);
  for (int i = 0; i < 6; ++i) p.s[i] = h->scal[i];
  p.coef_raw = s.coef;
  p.sched = h->sched;
  p.xoff = (int)h->xoff;
  p.dbg = env_int("STENCIL_DBG") | (env_int("STENCIL_FAULT") & 12);
  static const int walign = getenv("STENCIL_WALIGN") ? atoi(getenv("STENCIL_WALIGN")) : 0;
  p.walign = walign;
  p.tband = getenv("STENCIL_TILE_BAND") ? atoi(getenv("STENCIL_TILE_BAND")) : 0;
  p.nblk = 1;
  return p;
}

cudaEvent_t timing_begin(stencil_ctx* h, cudaEvent_t* end) {
  if (!h->timing) return nullptr;
  if (h->events_used == h->events.size()) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    h->events.emplace_back(a, b);
  }
  auto& pr = h->events[h->events_used++];
  cudaEventRecord(pr.first, h->stream);
  *end = pr.second;
  return pr.first;
}

// Halo exchange of `depth` planes of buffer b after a block.
int exchange(stencil_ctx* h, int b, int64_t depth, cudaStream_t cs) {
  if (env_int("STENCIL_FAULT") & 1) depth -= 1;  // fault injection: halo one plane too shallow
  if (h->nranks == 1 || depth <= 0) return ST_OK;
  const size_t cnt = (size_t)(depth * h->plane);
  if (h->local > 1) {
    // loopback: slabs i and i+1 of this handle share the boundary between slab i's top owned planes
    // [hi_i - depth, hi_i) and slab i+1's bottom owned planes [lo_{i+1}, lo_{i+1} + depth).
    for (size_t i = 0; i + 1 < h->slabs.size(); ++i) {
      Slab& a = h->slabs[i];
      Slab& c = h->slabs[i + 1];
      double* A = a.buf[b];
      double* Cb = c.buf[b];
      cudaError_t e = cudaMemcpyAsync(Cb + (c.lo - depth - c.store_z0) * h->plane,
                                      A + (a.hi - depth - a.store_z0) * h->plane, cnt * sizeof(double),
                                      cudaMemcpyDeviceToDevice, cs);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(A + (a.hi - a.store_z0) * h->plane, Cb + (c.lo - c.store_z0) * h->plane,
                            cnt * sizeof(double), cudaMemcpyDeviceToDevice, cs);
      if (e != cudaSuccess) return cuda_fail(h, e, "loopback halo copy");
    }
    return ST_OK;
  }
  Nccl* n = nccl();
  if (!n) { h->poisoned = true; return ST_E_NCCL; }
  Slab& s = h->slabs.front();
  const int64_t lo = s.lo - s.store_z0, hi = s.hi - s.store_z0;
  double* base = s.buf[b];
  ncclResult_t r = n->GroupStart();
  if (h->rank > 0 && r == ncclSuccess) {
    r = n->Send(base + lo * h->plane, cnt, ncclFloat64, h->rank - 1, h->comm, cs);
    if (r == ncclSuccess)
      r = n->Recv(base + (lo - depth) * h->plane, cnt, ncclFloat64, h->rank - 1, h->comm, cs);
  }
  if (h->rank < h->nranks - 1 && r == ncclSuccess) {
    r = n->Send(base + (hi - depth) * h->plane, cnt, ncclFloat64, h->rank + 1, h->comm, cs);
    if (r == ncclSuccess)
      r = n->Recv(base + hi * h->plane, cnt, ncclFloat64, h->rank + 1, h->comm, cs);
  }
  ncclResult_t r2 = n->GroupEnd();
  if (r == ncclSuccess) r = r2;
  if (r != ncclSuccess) {
    set_err("NCCL halo exchange: %s", n->GetErrorString(r));
    h->poisoned = true;
    return ST_E_NCCL;
  }
  return ST_OK;
}

// ST_HALO_PEER: the remote targets of slab s's output planes.  Side q = 0 (below) receives planes
// [lo, lo + H) of the new level(s), side 1 (above) planes [hi - H, hi): exactly the halo planes the
// neighbour stores (its store range reaches H = R*bt planes past its owned planes).
void peer_targets(stencil_ctx* h, const Slab& s, int d0, int d1, st::KParams& p) {
  const int64_t H = (int64_t)h->R * h->bt - ((env_int("STENCIL_FAULT") & 1) ? 1 : 0);  // fault: too shallow
  for (int q = 0; q < 2; ++q) {
    const Slab* n = nullptr;
    double* const* nbuf = nullptr;
    int64_t nz0 = 0;
    if (!h->ipc) {
      const int idx = (int)(&s - h->slabs.data()) + (q == 0 ? -1 : 1);
      if (idx < 0 || idx >= (int)h->slabs.size()) continue;
      n = &h->slabs[idx];
      nbuf = n->buf;
      nz0 = n->store_z0;
    } else {
      if (!h->peer[q].on) continue;
      nbuf = h->peer[q].buf;
      nz0 = h->peer[q].store_z0;
    }
    const int64_t shift = (s.store_z0 - nz0) * h->plane + h->xoff;  // same global cell, other slab
    p.rdst[q] = nbuf[d0] + shift;
    p.rdstu[q] = d1 >= 0 ? nbuf[d1] + shift : nullptr;
    const int64_t g0 = q == 0 ? s.lo : s.hi - H, g1 = q == 0 ? s.lo + H : s.hi;
    p.rz0[q] = (int)(g0 - s.store_z0);
    p.rz1[q] = (int)(g1 - s.store_z0);
  }
  p.rfence = h->ipc ? 1 : 0;
}

// Skewed two-level 25v tiles (pipe25.cu): the slab's exchange buffer (one state-sized
// array: a tile stores its top 2R level-1 rows of every plane there for the tile above) and the per-item
// flags, allocated at the first such launch; a fresh flag base per launch.
int skew_params(stencil_ctx* h, Slab& s, st::KParams& p) {
  if (!s.xch) {
    const size_t bytes = (size_t)h->plane * (size_t)s.zl * sizeof(double);
    s.xch = (double*)dev_alloc(h, bytes);
    if (!s.xch) { set_err("device allocation of %zu bytes failed (skewed-tile exchange buffer)", bytes); return ST_E_NOMEM; }
  }
  const long long need = st::pipe25v2_flag_slots(h->tile_cfg, (int)h->nx, (int)h->ny, (int)s.zl);
  if (h->xflag_n < need) {
    h->xflag = (unsigned int*)dev_alloc(h, (size_t)need * sizeof(unsigned int));
    if (!h->xflag) { set_err("device allocation failed (skewed-tile flags)"); return ST_E_NOMEM; }
    h->xflag_n = need;
    h->xbase = 0;
    CK(cudaMemsetAsync(h->xflag, 0, (size_t)need * sizeof(unsigned int), h->stream), "zero skewed-tile flags");
  }
  h->xbase += 65536u;
  if (h->xbase >= 0x80000000u) {  // flags are compared as (int)(v - want): restart before that wraps
    CK(cudaMemsetAsync(h->xflag, 0, (size_t)h->xflag_n * sizeof(unsigned int), h->stream), "zero skewed-tile flags");
    h->xbase = 65536u;
  }
  p.xch = s.xch + h->xoff;
  p.xch_raw = s.xch;
  p.xflag = h->xflag;
  p.xflag_n = h->xflag_n;
  p.xbase = h->xbase;
  return ST_OK;
}

// Launch the kernel of the handle's variant for b levels over output planes [z0, z1) (global padded
// indices) of slab s; peer = also store the neighbours' halo planes into their buffers.
int launch_range(stencil_ctx* h, Slab& s, int b, int d0, int d1, int64_t z0, int64_t z1, bool peer = false) {
  if (z1 <= z0) return ST_OK;
  st::KParams p = base_params(h, s);
  if (peer) peer_targets(h, s, d0, d1, p);
  p.zo0 = (int)(z0 - s.store_z0);
  p.zo1 = (int)(z1 - s.store_z0);
  p.src = h->at(s, h->lv0);
  p.srcu = h->at(s, h->lv1);
  p.dst = h->at(s, d0);
  p.dstu = d1 >= 0 ? h->at(s, d1) : nullptr;
  p.src_raw = s.buf[h->lv0];
  p.srcu_raw = s.buf[h->lv1];
  if (h->variant == ST_VARIANT_PIPE && h->kind == ST_25PT_VAR && b == 2 && st::pipe25v2_skewed(h->tile_cfg)) {
    const int rc = skew_params(h, s, p);
    if (rc) return rc;
  }
  cudaEvent_t ev_end = nullptr;
  cudaEvent_t ev_begin = timing_begin(h, &ev_end);
  cudaError_t e;
  st::LaunchInfo li{};
  if (h->variant == ST_VARIANT_NAIVE)
    e = st::launch_naive(h->kind, p, h->stream, &li);
  else if (h->variant == ST_VARIANT_STREAM)
    e = st::launch_stream(h->kind, b, p, h->zchunk_req, h->num_sms, h->stream, &li);
  else
    e = st::launch_pipe(h->kind, b, p, h->zchunk_req, h->num_sms, h->tile_cfg, h->stream, &li);
  if (ev_begin) cudaEventRecord(ev_end, h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "kernel launch");
  // st_info reports the plan's full-depth launches; a remainder block's plan only until one has run
  if (b == h->bt || h->last_launch.tile_x == 0) h->last_launch = li;
  h->launches++;
  return ST_OK;
}

int peer_wait(stencil_ctx* h, int64_t target);

// One block of b levels on every slab, then the halo exchange of the new level(s).
// Multi-slab schedule ("halo-first"): the edge kernels compute the R*b boundary planes of
// each slab that has a neighbour, the exchange of those planes starts on comm_stream, and the interior
// kernel (planes [lo + R*b, hi - R*b)) runs on the compute stream meanwhile.  The interior kernel reads
// only owned planes of the old level and writes only interior planes of the new one, so it touches
// neither the planes being sent nor the halo planes being received.  The next block waits for the
// exchange (ev_halo).
int run_block(stencil_ctx* h, int b) {
  const bool wave = is_wave(h->kind);
  int new0, new1, d0, d1 = -1;
  if (!wave) {
    d0 = h->lv1;
    new0 = h->lv1;
    new1 = h->lv0;
  } else if (b == 1) {
    d0 = h->lv1;  // Omega^{t+1} overwrites Omega^{t-1} in place
    new0 = h->lv1;
    new1 = h->lv0;
  } else {
    int spare[2], k = 0;
    for (int i = 0; i < 4; ++i)
      if (i != h->lv0 && i != h->lv1) spare[k++] = i;
    d0 = spare[0];
    d1 = spare[1];
    new0 = spare[0];
    new1 = spare[1];
  }
  int rc = ST_OK;
  // The halo exchanged after every block is the full stored depth H = R*bt, also after a shorter
  // remainder block (b = T mod bt): the next run's first block needs H planes of the new level.
  const int64_t depth = (int64_t)h->R * h->bt;
  if (h->nranks > 1 && h->halo == ST_HALO_PEER) {
    // Fused exchange: one launch per slab, the kernel stores the neighbours' halo planes itself.
    if (!h->peer_ready) {
      set_err("ST_HALO_PEER across processes: call stencil_peer_import on every rank before running");
      return ST_E_STATE;
    }
    const MemOps& m = memops();
    if (h->ipc) {
      // wait until both neighbours have stored block blocks-1's halos into this rank's buffers (and
      // thereby finished reading the buffers this block's remote stores overwrite)
      if (!m.write) { set_err("stream memory operations unavailable"); h->poisoned = true; return ST_E_CUDA; }
      if ((rc = peer_wait(h, h->blocks))) return rc;
    }
    for (auto& s : h->slabs)
      if ((rc = launch_range(h, s, b, d0, d1, s.lo, s.hi, true))) return rc;
    if (h->ipc) {
      // announce: neighbour below counts arrivals from above in its flags[1], neighbour above in [0]
      for (int q = 0; q < 2; ++q)
        if (h->peer[q].on) {
          CUresult r = m.write((CUstream)h->stream, (CUdeviceptr)(h->peer[q].flags + (1 - q)),
                               (cuuint64_t)(h->blocks + 1), CU_STREAM_WRITE_VALUE_DEFAULT);
          if (r != CUDA_SUCCESS) { set_err("cuStreamWriteValue64 failed (%d)", (int)r); h->poisoned = true; return ST_E_CUDA; }
        }
    }
  } else if (h->nranks == 1) {
    for (auto& s : h->slabs)
      if ((rc = launch_range(h, s, b, d0, d1, s.lo, s.hi))) return rc;
  } else {
    cudaError_t e = cudaSuccess;
    if (h->halo_pending) e = cudaStreamWaitEvent(h->stream, h->ev_halo, 0);  // previous block's halos
    if (e != cudaSuccess) return cuda_fail(h, e, "wait halo");
    if (!h->overlap) {
      for (auto& s : h->slabs)
        if ((rc = launch_range(h, s, b, d0, d1, s.lo, s.hi))) return rc;
    } else {
      // edge planes first (a slab thinner than two edges is computed whole)
      for (auto& s : h->slabs) {
        const bool below = s.rank > 0, above = s.rank < h->nranks - 1;
        const int64_t ilo = s.lo + (below ? depth : 0), ihi = s.hi - (above ? depth : 0);
        if (ilo >= ihi) {
          if ((rc = launch_range(h, s, b, d0, d1, s.lo, s.hi))) return rc;
          continue;
        }
        if (below && (rc = launch_range(h, s, b, d0, d1, s.lo, ilo))) return rc;
        if (above && (rc = launch_range(h, s, b, d0, d1, ihi, s.hi))) return rc;
      }
    }
    e = cudaEventRecord(h->ev_edge, h->stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(h->comm_stream, h->ev_edge, 0);
    if (e != cudaSuccess) return cuda_fail(h, e, "edge event");
    rc = exchange(h, new0, depth, h->comm_stream);
    if (!rc && wave) rc = exchange(h, new1, depth, h->comm_stream);
    if (rc) return rc;
    e = cudaEventRecord(h->ev_halo, h->comm_stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "halo event");
    h->halo_pending = true;
    if (h->overlap) {
      for (auto& s : h->slabs) {
        const bool below = s.rank > 0, above = s.rank < h->nranks - 1;
        const int64_t ilo = s.lo + (below ? depth : 0), ihi = s.hi - (above ? depth : 0);
        if (ilo < ihi && (rc = launch_range(h, s, b, d0, d1, ilo, ihi))) return rc;
      }
    }
  }
  h->lv0 = new0;
  h->lv1 = new1;
  h->steps += b;
  h->blocks++;
  return rc;
}

// Handshake kernel: plain device stores into the neighbours' flag blocks (peer memory), the same path
// the fused halo stores take.  Slot 2 / 3 of a flag block = word from the neighbour below / above.
__global__ void peer_poke_kernel(uint64_t* below_flags, uint64_t* above_flags, uint64_t magic) {
  if (below_flags) below_flags[3] = magic;  // I am the neighbour above of the rank below
  if (above_flags) above_flags[2] = magic;
  __threadfence_system();
}

uint64_t handshake_magic(int rank) { return 0x5EED000000000000ull + (uint64_t)rank; }

// ST_HALO_PEER across processes: wait until both neighbours' block counters (written into this rank's flag
// words by their streams after their kernels, cuStreamWriteValue64) reach `target`.  By default the HOST
// waits -- it polls the flag words with small device-to-host copies on a private stream, with a timeout --
// so no GPU stream ever blocks on another process (a neighbour that died or stalled becomes an ST_E_STATE
// error here instead of a hung stream; the profiling recipe warns against device-side cross-process waits
// on a shared GPU).  STENCIL_PEER_DEVICE_WAIT=1 enqueues cuStreamWaitValue64 on the handle's stream instead
// (asynchronous; the pre-round-2 behaviour).  Blocks last milliseconds, the poll microseconds.
int peer_wait(stencil_ctx* h, int64_t target) {
  if (env_int("STENCIL_PEER_DEVICE_WAIT")) {
    const MemOps& m = memops();
    if (!m.wait) { set_err("stream memory operations unavailable"); h->poisoned = true; return ST_E_CUDA; }
    for (int q = 0; q < 2; ++q)
      if (h->peer[q].on) {
        CUresult r = m.wait((CUstream)h->stream, (CUdeviceptr)(h->flags + q), (cuuint64_t)target,
                            CU_STREAM_WAIT_VALUE_GEQ);
        if (r != CUDA_SUCCESS) { set_err("cuStreamWaitValue64 failed (%d)", (int)r); h->poisoned = true; return ST_E_CUDA; }
      }
    return ST_OK;
  }
  if (!h->poll_stream) {
    cudaError_t e = cudaStreamCreateWithFlags(&h->poll_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return cuda_fail(h, e, "peer poll stream");
  }
  const int timeout_ms = env_int("STENCIL_PEER_TIMEOUT_MS") > 0 ? env_int("STENCIL_PEER_TIMEOUT_MS") : 120000;
  uint64_t got[2] = {0, 0};
  const auto t0 = std::chrono::steady_clock::now();
  for (int spins = 0;; ++spins) {
    cudaError_t e = cudaMemcpyAsync(got, h->flags, sizeof got, cudaMemcpyDeviceToHost, h->poll_stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->poll_stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "peer flag poll");
    if ((!h->peer[0].on || (int64_t)got[0] >= target) && (!h->peer[1].on || (int64_t)got[1] >= target)) return ST_OK;
    const auto ms = std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count();
    if (ms > timeout_ms) {
      set_err("ST_HALO_PEER: the neighbours' halos of block %lld did not arrive within %d ms (flags %llu %llu); "
              "a neighbour rank stopped or failed", (long long)target, timeout_ms, (unsigned long long)got[0],
              (unsigned long long)got[1]);
      h->poisoned = true;
      return ST_E_STATE;
    }
    if (spins > 16) usleep(spins > 1000 ? 1000 : 20);
  }
}

// Several full blocks of a single-slab Jacobi grid in ONE pipe-kernel launch (dependency-driven
// scheduling across blocks, pipe.cu): the tail of block i can overlap the start of block i+1.
// Opt-in (STENCIL_MULTIBLOCK=1): measured 1-7 % slower than one launch per block on B200 (C2 ~189 vs
// 193, C4 49 vs 52.5 GLUP/s): the kernels run at the 1 kW power cap, where the idle tails of per-block
// launches cost no throughput and filling them lowers the SM clock (profiles/r01_summary.md).
bool multiblock_ok(const stencil_ctx* h) {
  return env_int("STENCIL_MULTIBLOCK") == 1 && h->variant == ST_VARIANT_PIPE && h->nranks == 1 && !is_wave(h->kind) &&
         !(h->kind == ST_25PT_VAR && h->bt >= 2);  // the two-level 25-point kernel (pipe25.cu): one block per launch
}

int run_blocks_fused(stencil_ctx* h, int nblk, int b) {
  if (!h->done) {
    const size_t bytes = (size_t)st::kMaxDoneItems * sizeof(unsigned int);
    h->done = (unsigned int*)dev_alloc(h, bytes);
    if (!h->done) { set_err("device allocation of %zu bytes failed (block counters)", bytes); return ST_E_NOMEM; }
    CK(cudaMemsetAsync(h->done, 0, bytes, h->stream), "zero block counters");
  }
  Slab& s = h->slabs.front();
  st::KParams p = base_params(h, s);
  p.src = h->at(s, h->lv0);
  p.srcu = h->at(s, h->lv1);
  p.dst = h->at(s, h->lv1);
  p.dst_alt = h->at(s, h->lv0);
  p.src_raw = s.buf[h->lv0];
  p.srcu_raw = s.buf[h->lv1];
  p.dst_raw = s.buf[h->lv1];
  p.nblk = nblk;
  p.done = h->done;
  p.dbase = (unsigned int)h->blocks;
  cudaEvent_t ev_end = nullptr;
  cudaEvent_t ev_begin = timing_begin(h, &ev_end);
  const cudaError_t e = st::launch_pipe(h->kind, b, p, h->zchunk_req, h->num_sms, h->tile_cfg, h->stream,
                                        &h->last_launch);
  if (ev_begin) cudaEventRecord(ev_end, h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "multi-block kernel launch");
  h->launches++;
  if (nblk & 1) std::swap(h->lv0, h->lv1);
  h->steps += (int64_t)nblk * b;
  h->blocks += nblk;
  return ST_OK;
}

// ST_HALO_PEER across processes: enqueue a wait until both neighbours have delivered every block run
// so far (no remote store into this rank's memory is still in flight afterwards).
int wait_peers(stencil_ctx* h) {
  if (!h->ipc || !h->peer_ready) return ST_OK;
  return peer_wait(h, h->blocks);
}

int check_handle(stencil_ctx* h) {
  if (!h) { set_err("NULL handle"); return ST_E_INVAL; }
  if (h->poisoned) { set_err("handle poisoned by an earlier CUDA/NCCL failure"); return ST_E_STATE; }
  return ST_OK;
}

}  // namespace

// ================================================================ C ABI
extern "C" {

void stencil_opts_default(st_opts* o) {
  if (!o) return;
  memset(o, 0, sizeof *o);
  o->device = -1;
  o->variant = ST_VARIANT_AUTO;
  o->nranks = 1;
  o->local_slabs = 1;
}

const char* stencil_last_error(void) { return g_err.c_str(); }

const char* stencil_version(void) { return STENCIL_VERSION " (sm_100a)"; }

int stencil_plan_slab(int64_t nz, int R, int nranks, int rank, int bt, int64_t* own_z0,
                      int64_t* own_z1, int64_t* store_z0, int64_t* store_z1, int* bt_eff) {
  if (!own_z0 || !own_z1 || !store_z0 || !store_z1) { set_err("NULL output"); return ST_E_INVAL; }
  Slab s;
  int rc = plan_slab(nz, R, nranks, rank, bt, &s, bt_eff);
  if (rc) return rc;
  *own_z0 = s.own_z0;
  *own_z1 = s.own_z1;
  *store_z0 = s.store_z0;
  *store_z1 = s.store_z1;
  return ST_OK;
}

int stencil_create(stencil_ctx** out, int kind, int64_t nx, int64_t ny, int64_t nz,
                   const double* const* coeff, int n_coeff, const double* v0, const double* u0,
                   const st_opts* opts) {
  const int R = radius_of(kind);
  if (R < 0) { set_err("bad kind %d", kind); return ST_E_INVAL; }
  const int want = kind == 1 ? 2 : kind == 2 ? 7 : kind == 3 ? 6 : kind == 4 ? 13 : 6;
  if (n_coeff != want) { set_err("kind %d needs n_coeff=%d (got %d)", kind, want, n_coeff); return ST_E_INVAL; }
  if (!coeff || !v0) { set_err("NULL coeff or v0"); return ST_E_INVAL; }
  for (int i = 0; i < n_coeff; ++i)
    if (!coeff[i]) { set_err("coeff[%d] is NULL", i); return ST_E_INVAL; }
  if (is_wave(kind) && !u0) { set_err("wave kinds need u0"); return ST_E_INVAL; }
  if (!is_wave(kind) && u0) { set_err("u0 must be NULL for kind %d", kind); return ST_E_INVAL; }
  stencil_ctx* h = nullptr;
  int rc = create_common(out, kind, nx, ny, nz, opts, &h);
  if (rc) { fail_create(h); return rc; }
  const size_t hplane = (size_t)h->X * h->Y;
  cudaError_t e = cudaSuccess;
  {  // the staging slots are released (in stream order) before the synchronize below
  Stager stage(h);
  for (auto& s : h->slabs) {
    // V^0 once, then device copies into the other state buffers (same layout: ghosts and all)
    e = stage.upload(s, s.buf[0], v0);
    for (int b = 1; b < h->nbuf && e == cudaSuccess; ++b)
      e = cudaMemcpyAsync(s.buf[b], s.buf[0], (size_t)h->plane * s.zl * sizeof(double), cudaMemcpyDeviceToDevice,
                          h->stream);
    if (e == cudaSuccess && is_wave(kind)) {
      // level 1 = Omega^{-1}: interior from u0, ghosts from v0 (reading Q9).  Upload u0's
      // planes, then restore ghosts from v0: ghost planes wholesale, ghost rows/columns by 2-D copies.
      double* d = s.buf[h->lv1] + h->xoff;
      const size_t P = h->pitch * sizeof(double), HX = h->X * sizeof(double);
      for (int64_t z = 0; z < s.zl && e == cudaSuccess; ++z) {
        const int64_t gz = s.store_z0 + z;
        const bool zghost = gz < R || gz >= nz + R;
        const double* src = (zghost ? v0 : u0) + (size_t)(gz - h->host_z0()) * hplane;
        double* dz = d + z * h->plane;
        e = cudaMemcpy2DAsync(dz, P, src, HX, HX, h->Y, cudaMemcpyHostToDevice, h->stream);
        if (e == cudaSuccess && !zghost) {
          const double* g = v0 + (size_t)(gz - h->host_z0()) * hplane;
          e = cudaMemcpy2DAsync(dz, P, g, HX, HX, R, cudaMemcpyHostToDevice, h->stream);
          if (e == cudaSuccess)
            e = cudaMemcpy2DAsync(dz + (h->Y - R) * h->pitch, P, g + (h->Y - R) * h->X, HX, HX, R,
                                  cudaMemcpyHostToDevice, h->stream);
          if (e == cudaSuccess)
            e = cudaMemcpy2DAsync(dz, P, g, HX, R * sizeof(double), h->Y, cudaMemcpyHostToDevice, h->stream);
          if (e == cudaSuccess)
            e = cudaMemcpy2DAsync(dz + h->X - R, P, g + h->X - R, HX, R * sizeof(double), h->Y,
                                  cudaMemcpyHostToDevice, h->stream);
        }
      }
    }
    // coefficient fields follow the scalars in coeff[] (kind 5: w0..w4, then the alpha field)
    for (int i = 0; i < h->ncoef && e == cudaSuccess; ++i)
      e = stage.upload(s, s.coef + (size_t)i * h->plane * s.zl, coeff[h->nscal + i]);
  }
  }
  if (e != cudaSuccess) rc = cuda_fail(h, e, "upload");
  if (rc == ST_OK)
    for (int i = 0; i < h->nscal; ++i) h->scal[i] = *coeff[i];
  if (rc == ST_OK) {
    e = cudaStreamSynchronize(h->stream);  // host arrays may be freed by the caller after return
    if (e != cudaSuccess) rc = cuda_fail(h, e, "create synchronize");
  }
  if (rc) { fail_create(h); return rc; }
  *out = h;
  return ST_OK;
}

int stencil_create_seeded(stencil_ctx** out, int kind, int64_t nx, int64_t ny, int64_t nz,
                          uint64_t seed, const double* scalars, const st_opts* opts) {
  const int R = radius_of(kind);
  if (R < 0) { set_err("bad kind %d", kind); return ST_E_INVAL; }
  if (nscal_of(kind) == 0 && scalars) { set_err("variable kinds take no scalars"); return ST_E_INVAL; }
  stencil_ctx* h = nullptr;
  int rc = create_common(out, kind, nx, ny, nz, opts, &h);
  if (rc) { fail_create(h); return rc; }
  static const double d7c[2] = {0.4, 0.1};
  const double d25w[6] = {3.0 * (-205.0 / 72.0), 8.0 / 5.0, -1.0 / 5.0, 8.0 / 315.0, -1.0 / 560.0, 0.1};
  if (kind == ST_7PT_CONST) for (int i = 0; i < 2; ++i) h->scal[i] = scalars ? scalars[i] : d7c[i];
  if (kind == ST_25PT_WAVE) for (int i = 0; i < 6; ++i) h->scal[i] = scalars ? scalars[i] : d25w[i];
  if (kind == ST_25PT_WAVE_A) for (int i = 0; i < 5; ++i) h->scal[i] = scalars ? scalars[i] : d25w[i];
  const long long GZ = nz + 2 * R;
  // U[0, c): 1/7 (7v), 1/25 (25v), 0.2 for the wave's alpha field (stable below 0.205, synth/__init__.py)
  const double c = kind == ST_7PT_VAR ? 1.0 / 7.0 : kind == ST_25PT_VAR ? 1.0 / 25.0 : 0.2;
  cudaError_t e = cudaSuccess;
  for (auto& s : h->slabs) {
    for (int b = 0; b < h->nbuf && e == cudaSuccess; ++b) {
      const int mode = (is_wave(kind) && b == h->lv1) ? 1 : 0;
      e = st::launch_fill(s.buf[b] + h->xoff, h->pitch, h->plane, (int)s.zl, s.store_z0, h->X, h->Y, GZ, R,
                          seed, 0, mode, 0.0, h->stream);
    }
    for (int i = 0; i < h->ncoef && e == cudaSuccess; ++i)
      e = st::launch_fill(s.coef + (size_t)i * h->plane * s.zl + h->xoff, h->pitch, h->plane, (int)s.zl,
                          s.store_z0, h->X, h->Y, GZ, R, seed, 2 + i, 2, c, h->stream);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) {
    rc = cuda_fail(h, e, "seeded fill");
    fail_create(h);
    return rc;
  }
  *out = h;
  return ST_OK;
}

int stencil_run(stencil_ctx* h, int64_t T) {
  int rc = check_handle(h);
  if (rc) return rc;
  if (T < 1) { set_err("T must be >= 1 (got %lld)", (long long)T); return ST_E_INVAL; }
  Guard g(h);
  if (!g.ok) { set_err("handle used concurrently"); return ST_E_STATE; }
  const cudaError_t e = cudaSetDevice(h->device);
  if (e != cudaSuccess) return cuda_fail(h, e, "cudaSetDevice");
  if (h->variant == ST_VARIANT_COOP) {  // all T steps in one cooperative launch
    Slab& s = h->slabs.front();
    st::KParams p = base_params(h, s);
    p.src = h->at(s, h->lv0);
    p.srcu = h->at(s, h->lv1);
    p.dst = h->at(s, h->lv1);
    cudaEvent_t ev_end = nullptr;
    cudaEvent_t ev_begin = timing_begin(h, &ev_end);
    // one launch per 2^30 steps (the kernel's step counter is an int)
    for (int64_t left = T; left > 0;) {
      const int Tl = (int)std::min<int64_t>(left, 1 << 30);
      p.src = h->at(s, h->lv0);
      p.srcu = h->at(s, h->lv1);
      p.dst = h->at(s, h->lv1);
      int swaps = 0;
      const cudaError_t le = st::launch_coop(h->kind, p, Tl, h->num_sms, h->tile_cfg, h->stream, &h->last_launch, &swaps);
      if (le != cudaSuccess) return cuda_fail(h, le, "cooperative launch");
      h->launches++;
      if (swaps & 1) std::swap(h->lv0, h->lv1);
      h->steps += Tl;
      h->blocks += Tl;
      left -= Tl;
    }
    if (ev_begin) cudaEventRecord(ev_end, h->stream);
    return ST_OK;
  }
  const int bt = h->variant == ST_VARIANT_NAIVE ? 1 : h->bt;
  int64_t left = T;
  if (multiblock_ok(h) && bt >= 1) {
    // the leading run of full blocks (all but a merged remainder) in one launch
    int64_t nfull = left / bt;
    if (left % bt) nfull -= 1;  // the last full block is merged with the remainder (below)
    const int64_t cap = 1 << 20;
    while (nfull >= 2 && rc == ST_OK) {
      const int64_t n = std::min<int64_t>(nfull, cap);
      rc = run_blocks_fused(h, (int)n, bt);
      left -= n * bt;
      nfull -= n;
    }
  }
  while (left > 0 && rc == ST_OK) {
    // a remainder shorter than bt is merged with the last full block and split evenly (T = 100 at
    // bt = 3: ..., 3, 2, 2 instead of ..., 3, 3, 1): fewer levels in the least efficient launch
    const int b = (left > bt && left < 2 * (int64_t)bt) ? (int)((left + 1) / 2) : (int)std::min<int64_t>(bt, left);
    rc = run_block(h, b);
    left -= b;
  }
  if (rc == ST_OK && h->halo_pending) {  // later work on the caller's stream sees the halos
    const cudaError_t e2 = cudaStreamWaitEvent(h->stream, h->ev_halo, 0);
    if (e2 != cudaSuccess) return cuda_fail(h, e2, "join comm stream");
    h->halo_pending = false;
  }
  return rc;
}

int stencil_sync(stencil_ctx* h) {
  int rc = check_handle(h);
  if (rc) return rc;
  if ((rc = wait_peers(h))) return rc;
  cudaError_t e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "stream synchronize");
  return ST_OK;
}

int stencil_read_planes(stencil_ctx* h, int level, int64_t z0, int64_t z1, double* out, int64_t out_elems) {
  int rc = check_handle(h);
  if (rc) return rc;
  if (level < 0 || level > 1 || (level == 1 && !is_wave(h->kind))) {
    set_err("level %d not readable for kind %d", level, h->kind);
    return ST_E_INVAL;
  }
  if (!out || z0 < h->own_z0() || z1 > h->own_z1() || z0 > z1) {
    set_err("planes [%lld,%lld) outside owned [%lld,%lld) or NULL out", (long long)z0, (long long)z1,
            (long long)h->own_z0(), (long long)h->own_z1());
    return ST_E_INVAL;
  }
  const int64_t hplane = h->X * h->Y;
  if (out_elems < (z1 - z0) * hplane) {
    set_err("out_elems %lld < %lld", (long long)out_elems, (long long)((z1 - z0) * hplane));
    return ST_E_INVAL;
  }
  Guard g(h);
  if (!g.ok) { set_err("handle used concurrently"); return ST_E_STATE; }
  cudaError_t e = cudaSuccess;
  for (auto& s : h->slabs) {
    const int64_t a = std::max(z0, s.own_z0), b = std::min(z1, s.own_z1);
    if (a >= b) continue;
    const double* src = h->at(s, level == 0 ? h->lv0 : h->lv1) + (a - s.store_z0) * h->plane;
    e = cudaMemcpy2DAsync(out + (a - z0) * hplane, h->X * sizeof(double), src, h->pitch * sizeof(double),
                          h->X * sizeof(double), (size_t)h->Y * (b - a), cudaMemcpyDeviceToHost, h->stream);
    if (e != cudaSuccess) break;
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "read");
  return ST_OK;
}

int stencil_read(stencil_ctx* h, int level, double* out, int64_t out_elems) {
  int rc = check_handle(h);
  if (rc) return rc;
  const int64_t hplane = h->X * h->Y;
  const int64_t total = (h->nz + 2 * h->R) * hplane;
  if (!out || out_elems < total) { set_err("out must hold %lld doubles", (long long)total); return ST_E_INVAL; }
  return stencil_read_planes(h, level, h->own_z0(), h->own_z1(), out + h->own_z0() * hplane,
                             (h->own_z1() - h->own_z0()) * hplane);
}

int stencil_write(stencil_ctx* h, int level, const double* in, int64_t in_elems) {
  int rc = check_handle(h);
  if (rc) return rc;
  if (level < 0 || level > 1 || (level == 1 && !is_wave(h->kind))) {
    set_err("level %d not writable for kind %d", level, h->kind);
    return ST_E_INVAL;
  }
  const int64_t total = (h->host_slab ? h->slabs.front().store_z1 - h->slabs.front().store_z0 : h->nz + 2 * h->R) *
                        h->X * h->Y;
  if (!in || in_elems < total) { set_err("in must hold %lld doubles", (long long)total); return ST_E_INVAL; }
  Guard g(h);
  if (!g.ok) { set_err("handle used concurrently"); return ST_E_STATE; }
  if ((rc = wait_peers(h))) return rc;
  cudaError_t e = cudaSuccess;
  Stager stage(h);
  for (auto& s : h->slabs) {
    const int dstb = level == 0 ? h->lv0 : h->lv1;
    const size_t bytes = (size_t)h->plane * s.zl * sizeof(double);
    if (e == cudaSuccess) e = stage.upload(s, s.buf[dstb], in);
    if (e == cudaSuccess && level == 0 && !is_wave(h->kind))  // keep level 1's ghosts equal to the new ghosts
      e = cudaMemcpyAsync(s.buf[h->lv1], s.buf[dstb], bytes, cudaMemcpyDeviceToDevice, h->stream);
    if (is_wave(h->kind)) {
      // the fixed boundary is level 0's ghost shell in every buffer (reading Q9, as stencil_create does
      // with v0): a level-0 write hands its ghosts to level 1 (and the spare buffers), a level-1 write
      // keeps only its interior
      for (int b = 0; b < h->nbuf && e == cudaSuccess; ++b)
        if (b != h->lv0 && (level == 0 || b == h->lv1))
          e = st::launch_ghost_copy(s.buf[b] + h->xoff, s.buf[h->lv0] + h->xoff, h->pitch, h->plane, (int)s.zl,
                                    s.store_z0, h->X, h->Y, h->nz + 2 * h->R, h->R, h->stream);
    }
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "write");
  return ST_OK;
}

int stencil_info(const stencil_ctx* h, st_info* o) {
  if (!h || !o) { set_err("NULL handle or out"); return ST_E_INVAL; }
  memset(o, 0, sizeof *o);
  o->kind = h->kind; o->R = h->R; o->bt = (h->variant == ST_VARIANT_NAIVE || h->variant == ST_VARIANT_COOP) ? 1 : h->bt;
  o->variant = h->variant; o->rank = h->rank; o->nranks = h->nranks; o->local_slabs = h->local;
  o->tile_x = h->last_launch.tile_x; o->tile_y = h->last_launch.tile_y; o->zchunk = h->last_launch.zchunk;
  o->nx = h->nx; o->ny = h->ny; o->nz = h->nz;
  o->own_z0 = h->own_z0(); o->own_z1 = h->own_z1();
  o->pitch = h->pitch; o->plane = h->plane;
  int64_t zl = 0;
  for (auto& s : h->slabs) zl += s.zl;
  o->local_planes = zl;
  o->device_bytes = h->device_bytes; o->steps_done = h->steps; o->launches = h->launches;
  o->halo = h->halo;
  o->smem_bytes = h->last_launch.smem;
  o->threads = h->last_launch.threads;
  return ST_OK;
}

int stencil_peer_export(stencil_ctx* h, void* desc, size_t desc_bytes) {
  int rc = check_handle(h);
  if (rc) return rc;
  if (!desc || desc_bytes < ST_PEER_DESC_BYTES) { set_err("desc must hold %d bytes", ST_PEER_DESC_BYTES); return ST_E_INVAL; }
  if (!h->ipc) { set_err("stencil_peer_export: handle is not in ST_HALO_PEER mode across processes"); return ST_E_INVAL; }
  CK(cudaSetDevice(h->device), "cudaSetDevice");
  const Slab& s = h->slabs.front();
  PeerDesc d;
  memset(&d, 0, sizeof d);
  d.magic = kPeerMagic;
  d.rank = h->rank; d.nranks = h->nranks; d.kind = h->kind; d.nbuf = h->nbuf; d.bt = h->bt;
  d.nx = h->nx; d.ny = h->ny; d.nz = h->nz; d.pitch = h->pitch; d.plane = h->plane;
  d.store_z0 = s.store_z0; d.zl = s.zl;
  d.pid = (int64_t)getpid();
  d.device = h->device;
  for (int b = 0; b < h->nbuf; ++b) {
    CK(cudaIpcGetMemHandle(&d.buf[b], s.buf[b]), "cudaIpcGetMemHandle");
    d.raw_buf[b] = (uint64_t)(uintptr_t)s.buf[b];
  }
  CK(cudaIpcGetMemHandle(&d.flags, h->flags), "cudaIpcGetMemHandle");
  d.raw_flags = (uint64_t)(uintptr_t)h->flags;
  memset(desc, 0, ST_PEER_DESC_BYTES);
  memcpy(desc, &d, sizeof d);
  return ST_OK;
}

int stencil_peer_handshake(stencil_ctx* h, int timeout_ms) {
  int rc = check_handle(h);
  if (rc) return rc;
  if (!h->ipc || !h->peer_ready) { set_err("stencil_peer_handshake: import the neighbours first"); return ST_E_STATE; }
  CK(cudaSetDevice(h->device), "cudaSetDevice");
  const MemOps& m = memops();
  if (!m.write) { set_err("stream memory operations unavailable"); return ST_E_CUDA; }
  const uint64_t mine = handshake_magic(h->rank);
  // data path: a kernel's stores into peer memory; signal path: a stream-ordered flag write
  peer_poke_kernel<<<1, 1, 0, h->stream>>>(h->peer[0].on ? h->peer[0].flags : nullptr,
                                          h->peer[1].on ? h->peer[1].flags : nullptr, mine);
  CK(cudaGetLastError(), "handshake kernel");
  for (int q = 0; q < 2; ++q)
    if (h->peer[q].on) {
      CUresult r = m.write((CUstream)h->stream, (CUdeviceptr)(h->peer[q].flags + 5 - q), (cuuint64_t)mine,
                           CU_STREAM_WRITE_VALUE_DEFAULT);
      if (r != CUDA_SUCCESS) { set_err("cuStreamWriteValue64 failed (%d)", (int)r); return ST_E_CUDA; }
    }
  CK(cudaStreamSynchronize(h->stream), "handshake");
  // poll this rank's own flag block from the host (a private stream: nothing here can block forever)
  cudaStream_t ps = nullptr;
  CK(cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking), "handshake stream");
  uint64_t got[6] = {0, 0, 0, 0, 0, 0};
  bool ok = false;
  for (int waited = 0;; waited += 1) {
    cudaError_t e = cudaMemcpyAsync(got, h->flags, sizeof got, cudaMemcpyDeviceToHost, ps);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ps);
    if (e != cudaSuccess) { cudaStreamDestroy(ps); return cuda_fail(h, e, "handshake poll"); }
    ok = (!h->peer[0].on || (got[2] == handshake_magic(h->rank - 1) && got[4] == handshake_magic(h->rank - 1))) &&
         (!h->peer[1].on || (got[3] == handshake_magic(h->rank + 1) && got[5] == handshake_magic(h->rank + 1)));
    if (ok || waited >= timeout_ms) break;
    usleep(1000);
  }
  cudaStreamDestroy(ps);
  if (!ok) {
    set_err("stencil_peer_handshake: neighbour stores did not arrive within %d ms (got %llx %llx %llx %llx)",
            timeout_ms, (unsigned long long)got[2], (unsigned long long)got[3], (unsigned long long)got[4],
            (unsigned long long)got[5]);
    return ST_E_STATE;
  }
  return ST_OK;
}

int stencil_peer_import(stencil_ctx* h, const void* below, const void* above) {
  int rc = check_handle(h);
  if (rc) return rc;
  if (!h->ipc) { set_err("stencil_peer_import: handle is not in ST_HALO_PEER mode across processes"); return ST_E_INVAL; }
  if (h->peer_ready) { set_err("stencil_peer_import: already imported"); return ST_E_STATE; }
  if ((h->rank > 0) != (below != nullptr) || (h->rank < h->nranks - 1) != (above != nullptr)) {
    set_err("stencil_peer_import: rank %d of %d needs %s below and %s above", h->rank, h->nranks,
            h->rank > 0 ? "a descriptor" : "NULL", h->rank < h->nranks - 1 ? "a descriptor" : "NULL");
    return ST_E_INVAL;
  }
  CK(cudaSetDevice(h->device), "cudaSetDevice");
  const void* src[2] = {below, above};
  for (int q = 0; q < 2; ++q) {
    if (!src[q]) continue;
    PeerDesc d;
    memcpy(&d, src[q], sizeof d);
    const int want = h->rank + (q == 0 ? -1 : 1);
    if (d.magic != kPeerMagic || d.rank != want || d.nranks != h->nranks || d.kind != h->kind ||
        d.nbuf != h->nbuf || d.bt != h->bt || d.nx != h->nx || d.ny != h->ny || d.nz != h->nz ||
        d.pitch != h->pitch || d.plane != h->plane) {
      set_err("stencil_peer_import: descriptor %s does not describe rank %d of this grid", q ? "above" : "below", want);
      return ST_E_INVAL;
    }
    auto& pr = h->peer[q];
    if (d.pid == (int64_t)getpid()) {  // a handle of this process: its pointers are valid here
      if (d.device != h->device) {
        cudaError_t pe = cudaDeviceEnablePeerAccess(d.device, 0);
        if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) return cuda_fail(h, pe, "peer access");
        cudaGetLastError();
      }
      for (int b = 0; b < h->nbuf; ++b) pr.buf[b] = (double*)(uintptr_t)d.raw_buf[b];
      pr.flags = (uint64_t*)(uintptr_t)d.raw_flags;
      pr.opened = false;
    } else {
      for (int b = 0; b < h->nbuf; ++b) {
        void* ptr = nullptr;
        CK(cudaIpcOpenMemHandle(&ptr, d.buf[b], cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
        pr.buf[b] = (double*)ptr;
      }
      void* fp = nullptr;
      CK(cudaIpcOpenMemHandle(&fp, d.flags, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
      pr.flags = (uint64_t*)fp;
      pr.opened = true;
    }
    pr.store_z0 = d.store_z0;
    pr.on = true;
  }
  h->peer_ready = true;
  return ST_OK;
}

int stencil_set_timing(stencil_ctx* h, int enable) {
  int rc = check_handle(h);
  if (rc) return rc;
  h->timing = enable != 0;
  return ST_OK;
}

int stencil_kernel_time(stencil_ctx* h, double* ms, int64_t* launches, int reset) {
  int rc = check_handle(h);
  if (rc) return rc;
  cudaError_t e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "kernel_time synchronize");
  double tot = 0.0;
  for (size_t i = 0; i < h->events_used; ++i) {
    float t = 0.f;
    e = cudaEventElapsedTime(&t, h->events[i].first, h->events[i].second);
    if (e != cudaSuccess) return cuda_fail(h, e, "cudaEventElapsedTime");
    tot += t;
  }
  if (ms) *ms = tot;
  if (launches) *launches = (int64_t)h->events_used;
  if (reset) h->events_used = 0;
  return ST_OK;
}

int stencil_destroy(stencil_ctx* h) {
  if (!h) return ST_OK;
  cudaSetDevice(h->device);
  if (!h->poisoned) wait_peers(h);  // no neighbour may still be storing into this rank's buffers
  release(h);
  delete h;
  return ST_OK;
}

int stencil_generate(int kind, int64_t nx, int64_t ny, int64_t nz, uint64_t seed, int stream_id, double* out,
                     int64_t out_elems) {
  const int R = radius_of(kind);
  if (R < 0) { set_err("bad kind %d", kind); return ST_E_INVAL; }
  if (nx < 1 || ny < 1 || nz < 1) { set_err("extents must be >= 1"); return ST_E_INVAL; }
  const int64_t X = nx + 2 * R, Y = ny + 2 * R, Z = nz + 2 * R;
  if (!out || out_elems < X * Y * Z) { set_err("out must hold %lld doubles", (long long)(X * Y * Z)); return ST_E_INVAL; }
  const int nf = ncoef_of(kind);
  if (stream_id < 0 || (stream_id == 1 && !is_wave(kind)) || stream_id >= 2 + nf) {
    set_err("kind %d has no input stream %d", kind, stream_id);
    return ST_E_INVAL;
  }
  // the device fill's modes (st::launch_fill): 0 = U[-1,1) from the stream everywhere; 1 = wave
  // Omega^{-1} (interior stream 1, the rest stream 0); 2 = U[0, c) from the stream
  const int mode = stream_id == 0 ? 0 : stream_id == 1 ? 1 : 2;
  const double c = kind == ST_7PT_VAR ? 1.0 / 7.0 : kind == ST_25PT_VAR ? 1.0 / 25.0 : 0.2;
  const uint64_t key = synth_key(seed, mode == 1 ? SYNTH_STREAM_V : stream_id);
  const uint64_t key_u = synth_key(seed, SYNTH_STREAM_U);
  for (int64_t z = 0; z < Z; ++z)
    for (int64_t y = 0; y < Y; ++y)
      for (int64_t x = 0; x < X; ++x) {
        const uint64_t idx = (uint64_t)((z * Y + y) * X + x);
        double v;
        if (mode == 2) v = synth_scaled(key, idx, c);
        else if (mode == 1 && x >= R && x < X - R && y >= R && y < Y - R && z >= R && z < Z - R) v = synth_sym(key_u, idx);
        else v = synth_sym(key, idx);
        out[idx] = v;
      }
  return ST_OK;
}

int stencil_nccl_unique_id(void* out, size_t out_bytes) {
  if (!out || out_bytes < sizeof(ncclUniqueId)) { set_err("need %zu bytes", sizeof(ncclUniqueId)); return ST_E_INVAL; }
  Nccl* n = nccl();
  if (!n) return ST_E_NCCL;
  ncclUniqueId id;
  ncclResult_t r = n->GetUniqueId(&id);
  if (r != ncclSuccess) { set_err("ncclGetUniqueId: %s", n->GetErrorString(r)); return ST_E_NCCL; }
  memcpy(out, &id, sizeof id);
  return ST_OK;
}

}  // extern "C"
