// fp64_peak.cu -- measured FP64 FMA throughput of this GPU (the second bound of BASELINE.json's
// roofline: "FP64 peak divided by flops per LUP").  Every thread runs 8 independent DFMA chains; the
// grid fills every SM several times over.  Prints one JSON line: {"fp64_tflops": ..., ...}.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double b, double c) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int n = 0; n < iters; ++n) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.678) out[0] = s;  // keeps the chains alive
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 8);
  const int threads = 256, blocks = sms * 8, iters = 1 << 16;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_kernel<<<blocks, threads>>>(out, 1024, 0.999999, 1e-9);  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 8 * (double)iters * threads * blocks;
  cudaError_t err = cudaGetLastError();
  printf("{\"fp64_tflops\": %.3f, \"ms\": %.3f, \"sms\": %d, \"max_clock_mhz\": %d, \"error\": \"%s\", "
         "\"how\": \"8 independent DFMA chains per thread, %d x %d threads, best of 5, CUDA events\"}\n",
         flops / (best * 1e-3) / 1e12, best, sms, clk / 1000, cudaGetErrorString(err), blocks, threads);
  return err == cudaSuccess ? 0 : 1;
}
