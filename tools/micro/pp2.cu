// L2 hand-off latency between CTA 0 and CTA `peer` of a 148-CTA grid, others idle or streaming
#include <cuda_runtime.h>
#include <cstdio>
__global__ void k_pp(uint4* buf, int hops, int peer, long long* out, const uint4* junk, size_t njunk, int* smid) {
  if (threadIdx.x == 0) { int s; asm("mov.u32 %0, %%smid;" : "=r"(s)); smid[blockIdx.x] = s; }
  const int me = blockIdx.x == 0 ? 0 : (blockIdx.x == peer ? 1 : -1);
  if (me < 0) {
    if (njunk == 0) return;
    unsigned acc = 0;
    for (size_t i = (blockIdx.x * 256 + threadIdx.x); i < njunk; i += gridDim.x * 256) acc ^= __ldcs(junk + i).x;
    if (acc == 0x123) buf[200] = make_uint4(acc, 0, 0, 0);
    return;
  }
  uint4* mine = buf + me * 64;
  uint4* theirs = buf + (1 - me) * 64;
  unsigned long long g0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  for (int h = 0; h < hops; ++h) {
    if ((h & 1) == me) {
      if (threadIdx.x < 64)
        asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(mine + threadIdx.x), "r"(h), "r"(h + 1), "r"(h), "r"(h + 1) : "memory");
    } else if (threadIdx.x < 32) {
      const unsigned want = h + 1;
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
  if (threadIdx.x == 0 && me == 0) out[0] = (long long)(g1 - g0) / hops;
}
int main() {
  uint4* buf; long long* o; int* sm; uint4* junk;
  const size_t nj = (512ull << 20) / 16;
  cudaMalloc(&buf, 256 * 16); cudaMalloc(&o, 16); cudaMalloc(&sm, 148 * 4); cudaMalloc(&junk, nj * 16);
  cudaMemset(junk, 1, nj * 16);
  int smid[148];
  for (int load = 0; load < 2; ++load)
    for (int peer : {1, 2, 3, 8, 37, 74, 75, 100, 147}) {
      cudaMemset(buf, 0, 256 * 16);
      k_pp<<<148, 256>>>(buf, 1000, peer, o, junk, load ? nj : 0, sm);
      cudaDeviceSynchronize();
      long long r; cudaMemcpy(&r, o, 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(smid, sm, 148 * 4, cudaMemcpyDeviceToHost);
      printf("%s peer %3d (sm %3d vs sm %3d): %lld ns per hop %s\n", load ? "streaming" : "idle     ", peer, smid[0], smid[peer], r, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
