// dependent-latency of fp64 / fp32 ops and shared-memory round trips (one warp)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, float* outf, unsigned long long* t, int n) {
  double a = out[0], b = out[1], c = out[2];
  float af = outf[0], bf = outf[1], cf = outf[2];
  __shared__ double sh[64];
  sh[threadIdx.x] = a;
  __syncwarp();
  unsigned long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, c);
  unsigned long long t1 = clock64();
  for (int i = 0; i < n; ++i) af = fmaf(af, bf, cf);
  unsigned long long t2 = clock64();
  for (int i = 0; i < n; ++i) a = a + b;
  unsigned long long t3 = clock64();
  for (int i = 0; i < n; ++i) a = 1.0 / a;
  unsigned long long t4 = clock64();
  for (int i = 0; i < n; ++i) a = sqrt(a);
  unsigned long long t5 = clock64();
  int idx = threadIdx.x;
  double s = 0;
  for (int i = 0; i < n; ++i) { s = sh[idx]; idx = ((int)s & 31); }
  unsigned long long t6 = clock64();
  for (int i = 0; i < n; ++i) a = __shfl_xor_sync(0xffffffffu, a, 1) + c;
  unsigned long long t7 = clock64();
  out[threadIdx.x] = a + s; outf[threadIdx.x] = af;
  if (threadIdx.x == 0) { t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2; t[3] = t4 - t3; t[4] = t5 - t4; t[5] = t6 - t5; t[6] = t7 - t6; }
}
int main() {
  double* o; float* of; unsigned long long* t;
  cudaMalloc(&o, 8 * 64); cudaMalloc(&of, 4 * 64); cudaMalloc(&t, 64);
  double h[3] = {1.0, 0.999999, 1e-9}; float hf[3] = {1.f, 0.9999f, 1e-9f};
  cudaMemcpy(o, h, 24, cudaMemcpyHostToDevice); cudaMemcpy(of, hf, 12, cudaMemcpyHostToDevice);
  const int n = 4096;
  unsigned long long ht[7];
  for (int r = 0; r < 2; ++r) { k<<<1, 32>>>(o, of, t, n); cudaMemcpy(ht, t, 56, cudaMemcpyDeviceToHost); }
  const char* nm[7] = {"dfma", "ffma", "dadd", "drcp(1/x)", "dsqrt", "lds chain", "shfl+dadd"};
  for (int i = 0; i < 7; ++i) printf("%-10s %.1f cycles/op\n", nm[i], ht[i] / (double)n);
}
