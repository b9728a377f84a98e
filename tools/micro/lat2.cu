// dependent-latency probes: DFMA, DADD, FFMA, LDS, SHFL(f64), globaltimer resolution, L2 ping-pong handoff
#include <cuda_runtime.h>
#include <cstdio>
__global__ void k_lat(double* out, long long* cyc, int n) {
  __shared__ double sm[64];
  double a = out[0], b = out[1], c = out[2];
  float fa = (float)a, fb = (float)b;
  if (threadIdx.x < 64) sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = __fma_rn(a, b, c);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) a = __dadd_rn(a, b);
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) fa = __fmaf_rn(fa, fb, fa);
  long long t3 = clock64();
  int idx = threadIdx.x & 63;
  for (int i = 0; i < n; ++i) idx = (int)sm[idx] & 63;
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) a = __shfl_xor_sync(0xffffffffu, a, 1) + 1.0;
  long long t5 = clock64();
  unsigned long long g0, g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  int k = 0;
  do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1)); ++k; } while (g1 == g0);
  long long t6 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / n; cyc[1] = (t2 - t1) / n; cyc[2] = (t3 - t2) / n; cyc[3] = (t4 - t3) / n;
    cyc[4] = (t5 - t4) / n; cyc[5] = (long long)(g1 - g0); cyc[6] = k;
  }
  out[3] = a + fa + idx;
}
// ping-pong between two CTAs through L2: 64 tagged 16-B entries per hop
__global__ void k_pingpong(uint4* buf, int hops, long long* out) {
  const int me = blockIdx.x;  // 0 or 1
  uint4* mine = buf + me * 64;
  uint4* theirs = buf + (1 - me) * 64;
  long long t0 = clock64();
  unsigned long long g0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  for (int h = 0; h < hops; ++h) {
    const unsigned tag = 2 * h + 1 + me;  // partner writes tag 2h+1+(1-me)
    if ((h & 1) == me) {
      if (threadIdx.x < 64)
        asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(mine + threadIdx.x), "r"(h), "r"(tag), "r"(h), "r"(tag) : "memory");
    } else if (threadIdx.x < 32) {
      const unsigned want = 2 * h + 1 + (1 - me);
      bool ok0 = false, ok1 = false;
      while (true) {
        unsigned x, y, z, w;
        if (!ok0) { asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "l"(theirs + threadIdx.x) : "memory"); ok0 = (y == want && w == want); }
        if (!ok1) { asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "l"(theirs + 32 + threadIdx.x) : "memory"); ok1 = (y == want && w == want); }
        if (__all_sync(0xffffffffu, ok0 && ok1)) break;
      }
    }
    __syncthreads();
  }
  unsigned long long g1; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  if (threadIdx.x == 0 && me == 0) { out[0] = (clock64() - t0) / hops; out[1] = (long long)(g1 - g0) / hops; }
}
int main() {
  double* d; long long* c; uint4* buf;
  cudaMalloc(&d, 64); cudaMalloc(&c, 128); cudaMalloc(&buf, 128 * 16);
  double h[4] = {1.0, 1.0000001, 1e-9, 0}; cudaMemcpy(d, h, 32, cudaMemcpyHostToDevice);
  k_lat<<<1, 32>>>(d, c, 2000); cudaDeviceSynchronize();
  long long r[8]; cudaMemcpy(r, c, 64, cudaMemcpyDeviceToHost);
  printf("latency (cycles): DFMA %lld, DADD %lld, FFMA %lld, LDS %lld, SHFL.f64+DADD %lld; globaltimer step %lld ns (after %lld reads)\n", r[0], r[1], r[2], r[3], r[4], r[5], r[6]);
  for (int sep : {0, 1}) {
    cudaMemset(buf, 0, 128 * 16);
    // two CTAs; with 148 CTAs of filler? just 2
    k_pingpong<<<2, 256>>>(buf, 2000, c); cudaDeviceSynchronize();
    cudaMemcpy(r, c, 16, cudaMemcpyDeviceToHost);
    printf("L2 tagged hand-off (64 entries): %lld cycles, %lld ns per hop (%s)\n", r[0], r[1], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
