// tmem_probe.cu -- measured tcgen05.ld (TMEM -> registers) and tcgen05.st throughput per SM, to decide
// whether TMEM can serve as a per-thread coefficient window for the temporally blocked 7-point kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/tmem_probe tools/tmem_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) tmem_kernel(unsigned* out, int iters, int do_st) {
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
  uint32_t acc = 0;
  uint32_t v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
    if (do_st) {
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
          "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(base),
          "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
          "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
          "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
          "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
      asm volatile("tcgen05.wait::st.sync.aligned;");
    } else {
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
  }
  if (acc == 0x12345678u) out[0] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr_s), "n"(512));
}

template <int WARPS>
void run(int sms, unsigned* out, int do_st) {
  const int iters = 1 << 14;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  tmem_kernel<WARPS><<<sms, WARPS * 32>>>(out, 16, do_st);
  cudaEventRecord(a);
  tmem_kernel<WARPS><<<sms, WARPS * 32>>>(out, iters, do_st);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double bytes = (double)sms * WARPS * 32 * 32 * 4 * iters;
  printf("{\"op\": \"%s\", \"warps_per_sm\": %d, \"GBps_total\": %.1f, \"bytes_per_clk_per_sm_at_max_clock\": %.1f, "
         "\"error\": \"%s\"}\n",
         do_st ? "tcgen05.st 32x32b.x32" : "tcgen05.ld 32x32b.x32", WARPS, bytes / (ms * 1e-3) / 1e9,
         bytes / (ms * 1e-3) / sms / (clk * 1e3), cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* out;
  cudaMalloc(&out, 4);
  for (int st = 0; st < 2; ++st) {
    run<4>(sms, out, st);
    run<8>(sms, out, st);
  }
  return 0;
}
