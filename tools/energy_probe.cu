// energy_probe.cu -- kernels that each keep ONE data path of every SM busy for a given number of
// iterations, so that tools/energy_probe.py can read the board power while it runs and derive the
// energy per operation / per byte of that path (the coefficients of the power model in DESIGN.md §6):
//   0  FP64 FMA        independent DFMA chains                          (flops = 2 per FMA)
//   1  shared memory   conflict-free 128-bit loads                      (bytes)
//   2  L2              128-bit .cg loads of a buffer that fits in L2    (bytes)
//   3  HBM             128-bit streaming copy of buffers far larger than L2 (bytes read + written)
//   4  TMEM            tcgen05.ld 32x32b.x32                            (bytes)
// Built as a shared library (Makefile: build/libenergy_probe.so); ep_run(kind, iters, buf, n) launches
// the kernel synchronously and returns its device time in ms (negative on error) and the unit count.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

__global__ void __launch_bounds__(512, 1) k_fp64(double* out, long long iters) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = 0.999999, c = 1e-7;
  for (long long i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
      a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
  }
  const double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 1.2345) out[0] = s;
}

__global__ void __launch_bounds__(512, 1) k_smem(double* out, long long iters) {
  __shared__ double2 buf[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_double2(i, i + 1);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  int idx = threadIdx.x;
  for (long long i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double2 v = buf[(idx + u * 256) & 2047];  // 8 distinct addresses per iteration
      acc.x += v.x;
      acc.y += v.y;
    }
    idx += 32;
  }
  if (acc.x == 1.2345) out[0] = acc.x + acc.y;
}

__global__ void __launch_bounds__(512, 1) k_l2(const double2* __restrict__ buf, long long n2, double* out, long long iters) {
  double2 acc = make_double2(0, 0);
  long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = 0; i < iters; ++i) {
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldcg(buf + ((idx + u * stride) & (n2 - 1)));  // n2: a power of 2
#pragma unroll
    for (int u = 0; u < 4; ++u) { acc.x += v[u].x; acc.y += v[u].y; }
    idx += 4 * stride;
  }
  if (acc.x == 1.2345) out[0] = acc.x + acc.y;
}

__global__ void __launch_bounds__(512, 1) k_hbm(const double2* __restrict__ a, double2* __restrict__ b, long long n2,
                                               long long iters) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long it = 0; it < iters; ++it)
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride) __stcs(b + i, __ldcs(a + i));
}

__global__ void __launch_bounds__(256, 1) k_tmem(double* out, long long iters) {
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&taddr_s)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = taddr_s + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp / 4) * 64);
  uint32_t acc = 0, v[32];
  for (long long it = 0; it < iters; ++it) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(base + (uint32_t)((it & 1) * 32)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
    for (int i = 0; i < 32; ++i) acc += v[i];
  }
  if (acc == 0x12345678u) out[0] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr_s), "n"(512));
}

}  // namespace

extern "C" {

// kind as above; buf/n: a device buffer of n doubles (L2: the first n doubles are read; HBM: split in
// two halves, copied a -> b).  *units = operations (flops) or bytes moved.  Returns ms, < 0 on error.
double ep_run(int kind, long long iters, double* buf, long long n, double* units) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  double u = 0;
  switch (kind) {
    case 0: k_fp64<<<sms, 512>>>(buf, iters); u = 2.0 * 64 * 512.0 * sms * (double)iters; break;
    case 1: k_smem<<<sms, 512>>>(buf, iters); u = 16.0 * 8 * 512.0 * sms * (double)iters; break;
    case 2: k_l2<<<sms, 512>>>((const double2*)buf, n / 2, buf + n - 1, iters); u = 16.0 * 4 * 512.0 * sms * (double)iters; break;
    case 3: k_hbm<<<sms * 2, 512>>>((const double2*)buf, (double2*)(buf + n / 2), n / 4, iters);
            u = 2.0 * 8.0 * (double)(n / 2) * (double)iters; break;
    case 4: cudaFuncSetAttribute(k_tmem, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
            k_tmem<<<sms, 256, 120 * 1024>>>(buf, iters); u = 128.0 * 256.0 * sms * (double)iters; break;
    default: return -1.0;
  }
  cudaEventRecord(e1);
  if (cudaEventSynchronize(e1) != cudaSuccess || cudaGetLastError() != cudaSuccess) return -2.0;
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (units) *units = u;
  return ms;
}

}  // extern "C"
