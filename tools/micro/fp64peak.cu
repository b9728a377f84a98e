// FP64 DFMA peak of this GPU (the double-double kernels and the
// batched dd GEPP are FP64-bound; their roofline needs a measured peak).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/micro/fp64peak.cu -o tools/micro/fp64peak
// Prints one JSON object: {"dfma_tflops": ..., "sm_count": ..., ...}
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void __launch_bounds__(256) k_dfma(double* out, int iters, double a, double b) {
  double x[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) x[i] = (double)(threadIdx.x + i) * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = __fma_rn(x[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 8);
  constexpr int ILP = 8;
  const int iters = 1 << 16;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best = 0.0;
  int best_ctas = 0;
  for (int per_sm : {2, 4, 8}) {
    const int grid = sms * per_sm;
    k_dfma<ILP><<<grid, 256>>>(out, iters, 0.999999, 1e-9);
    cudaDeviceSynchronize();
    float ms_best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      k_dfma<ILP><<<grid, 256>>>(out, iters, 0.999999, 1e-9);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < ms_best) ms_best = ms;
    }
    const double flop = 2.0 * (double)grid * 256 * ILP * iters;
    const double tf = flop / (ms_best * 1e-3) / 1e12;
    if (tf > best) best = tf, best_ctas = per_sm;
  }
  printf("{\"dfma_tflops\": %.3f, \"sm_count\": %d, \"clock_khz\": %d, \"ctas_per_sm\": %d, \"ilp\": %d, "
         "\"how\": \"%d independent DFMA chains per thread, 256 threads per CTA, best of 5 launches (CUDA events)\", "
         "\"flop_per_clk_per_sm\": %.1f}\n",
         best, sms, clk, best_ctas, ILP, ILP, best * 1e12 / ((double)sms * clk * 1e3));
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
