// Microbenchmark: cross-CTA flag hand-off latency and per-tile arithmetic cost.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2201_09827_b200/csrc/gb_ops.cuh"
using namespace gb;

__global__ void chain(unsigned long long* ctr, int nlinks, int fence_mode, unsigned long long* tout) {
  // block b waits for counter == b, then publishes b+1 (one warp per CTA)
  const int b = blockIdx.x;
  if (threadIdx.x != 0) return;
  unsigned long long t0 = gtimer();
  for (int it = 0; it < nlinks; it += gridDim.x) {
    unsigned long long target = it + b;
    while (ld_relaxed64(ctr) < target) __nanosleep(8);
    if (fence_mode) fence_acq_rel();
    if (fence_mode) __threadfence();
    st_release64(ctr, target + 1);
  }
  if (b == 0) tout[0] = gtimer() - t0;
}

template <int M>
__global__ void tile_cost(double* out, int reps, unsigned long long* tout) {
  using Ar = Arith<M>;
  typename Ar::T acc = Ar::from(1.0 + threadIdx.x);
  __shared__ float tile[32 * 33];
  for (int i = threadIdx.x; i < 32 * 33; i += blockDim.x) tile[i] = 0.001f * (i % 97);
  __syncwarp();
  const int lane = threadIdx.x & 31;
  typename Ar::T yv = Ar::from(0.5 + lane);
  unsigned long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll 8
    for (int jj = 0; jj < 32; ++jj) {
      typename Ar::T yj = Ar::shfl(yv, jj);
      acc = Ar::sub_prod(acc, (double)tile[lane * 33 + jj], yj);
    }
  }
  unsigned long long t1 = clock64();
  out[threadIdx.x] = Ar::val(acc);
  if (threadIdx.x == 0) tout[0] = (t1 - t0) / reps;
}

__global__ void fp64_peak(double* out, int reps, unsigned long long* tout) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b = 1.0000001, c = 1e-9;
  unsigned long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
  }
  unsigned long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
  if (threadIdx.x == 0 && blockIdx.x == 0) tout[0] = t1 - t0;
}

template <int M>
__global__ void diag_cost(double* out, int reps, unsigned long long* tout) {
  using Ar = Arith<M>;
  __shared__ float tile[32 * 33];
  for (int i = threadIdx.x; i < 32 * 33; i += blockDim.x) tile[i] = 1.0f + 0.001f * (i % 97);
  __syncwarp();
  const int lane = threadIdx.x & 31;
  typename Ar::T acc = Ar::from(1.0 + lane);
  unsigned long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    for (int jj = 31; jj >= 0; --jj) {
      if (lane == jj) acc = Ar::div(acc, (double)tile[lane * 33 + lane]);
      const typename Ar::T yj = Ar::shfl(acc, jj);
      if (lane < jj) acc = Ar::sub_prod(acc, (double)tile[lane * 33 + jj], yj);
    }
  }
  unsigned long long t1 = clock64();
  out[threadIdx.x] = Ar::val(acc);
  if (threadIdx.x == 0) tout[0] = (t1 - t0) / reps;
}

int main() {
  unsigned long long *ctr, *t;
  double* o;
  cudaMalloc(&ctr, 8);
  cudaMalloc(&t, 64);
  cudaMalloc(&o, 8 * 1024);
  unsigned long long h;
  for (int grid : {2, 16, 64, 148}) {
    for (int fm : {0, 1}) {
      cudaMemset(ctr, 0, 8);
      chain<<<grid, 32>>>(ctr, 4096, fm, t);
      cudaDeviceSynchronize();
      cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
      printf("chain grid %3d fence %d: %.3f us per link\n", grid, fm, h / 1e3 / 4096);
    }
  }
  for (int w : {1, 2, 4, 8, 16}) {
    tile_cost<MODE_F64><<<1, 32 * w>>>(o, 100, t);
    cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
    printf("tile f64 with %d warps/CTA: %llu cycles per warp-tile\n", w, h);
  }
  tile_cost<MODE_DD><<<1, 32>>>(o, 100, t);
  cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
  printf("tile dd : %llu cycles\n", h);
  diag_cost<MODE_F64><<<1, 32>>>(o, 100, t);
  cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
  printf("diag f64 (upper, with div): %llu cycles\n", h);
  diag_cost<MODE_DD><<<1, 32>>>(o, 100, t);
  cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
  printf("diag dd (upper, with div): %llu cycles\n", h);
  {
    double* big;
    cudaMalloc(&big, 8 * 148 * 1024);
    fp64_peak<<<148, 1024>>>(big, 10000, t);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    fp64_peak<<<148, 1024>>>(big, 10000, t);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("fp64 FMA throughput: %.2f TFLOP/s\n", 148.0 * 1024 * 10000 * 4 * 2 / (ms * 1e-3) / 1e12);
  }
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("clock %d kHz; err %s\n", clk, cudaGetErrorString(cudaGetLastError()));
}
