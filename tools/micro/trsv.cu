// Microbenchmark of the team TRSV alone (synthetic unit-lower / upper factors).
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2201_09827_b200/csrc/gb_ops.cuh"
using namespace gb;

template <int M, bool kLower>
__global__ void __launch_bounds__(256) k_trsv(int n, const float* LU, size_t ld, typename Arith<M>::T* y,
                                              unsigned long long* ctr, unsigned long long epoch, GridCtl* ctl,
                                              double* partials, unsigned long long* tout, int use_rcp,
                                              const double* rh, const double* rl, unsigned long long* stamps) {
  extern __shared__ __align__(16) unsigned char smem[];
  GridTeam t{(int)gridDim.x, (int)blockIdx.x, ctl, partials, 64, 0u};
  TrsvSync ts{ctr, ctr + 1, epoch, PhaseLog{nullptr, 0}, stamps};
  t.sync();
  unsigned long long t0 = gtimer();
  trsv_blocks<M, GridTeam, float, kLower>(t, n, LU, ld, y, ts, smem, use_rcp ? rh : nullptr, use_rcp ? rl : nullptr);
  t.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) tout[0] = gtimer() - t0;
}

template <int M, bool kLower>
float run(int n, int G, int rcp) {
  using T = typename Arith<M>::T;
  size_t ld = (n + 31) & ~31;
  std::vector<float> h((size_t)n * ld);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) h[(size_t)i * ld + j] = (i == j) ? 2.0f : 0.5f / n;
  float* LU;
  T* y;
  unsigned long long *ctr, *tout;
  GridCtl* ctl;
  double *part, *rh, *rl;
  cudaMalloc(&LU, sizeof(float) * h.size());
  cudaMemcpy(LU, h.data(), sizeof(float) * h.size(), cudaMemcpyHostToDevice);
  cudaMalloc(&y, sizeof(T) * n);
  cudaMemset(y, 0, sizeof(T) * n);
  cudaMalloc(&ctr, 32);
  cudaMemset(ctr, 0, 32);
  cudaMalloc(&tout, 8);
  cudaMalloc(&ctl, sizeof(GridCtl));
  cudaMemset(ctl, 0, sizeof(GridCtl));
  cudaMalloc(&part, 8 * 2 * 64 * 256);
  cudaMalloc(&rh, 8 * n);
  unsigned long long* stamps;
  cudaMalloc(&stamps, 8 * 3 * 1024);
  cudaMemset(stamps, 0, 8 * 3 * 1024);
  cudaMalloc(&rl, 8 * n);
  cudaMemset(rh, 0, 8 * n);
  cudaMemset(rl, 0, 8 * n);
  size_t sm = 8 * 32 * 33 * sizeof(float);
  auto kern = k_trsv<M, kLower>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  unsigned long long epoch = 0, hout = 0;
  float best = 1e30f;
  for (int it = 0; it < 5; ++it) {
    void* args[] = {&n, &LU, &ld, &y, &ctr, &epoch, &ctl, &part, &tout, &rcp, &rh, &rl, &stamps};
    if (!kLower) {  // backward waits for a completed forward of this epoch
      unsigned long long v = (epoch + 1) * ((n + 31) / 32);
      cudaMemcpy(ctr, &v, 8, cudaMemcpyHostToDevice);
    }
    cudaLaunchCooperativeKernel((void*)kern, G, 256, args, sm, 0);
    cudaDeviceSynchronize();
    cudaMemcpy(&hout, tout, 8, cudaMemcpyDeviceToHost);
    best = std::min(best, hout / 1e3f);
    epoch++;
    cudaMemset(ctr, 0, 32);
    epoch = 0;
  }
  if (getenv("STAMPS")) {
    std::vector<unsigned long long> st(3 * 1024);
    cudaMemcpy(st.data(), stamps, 8 * 3 * 1024, cudaMemcpyDeviceToHost);
    int nb = (n + 31) / 32;
    printf("  block: deps_seen->published (us) | published->next deps_seen (us)\n  ");
    for (int s = 0; s < std::min(nb, 24); ++s) {
      double a = (st[3 * s + 1] - st[3 * s]) / 1e3;
      double b = s + 1 < nb ? ((double)st[3 * (s + 1) + 2] - (double)st[3 * s + 1]) / 1e3 : 0.0;
      double c = s + 1 < nb ? ((double)st[3 * (s + 1)] - (double)st[3 * (s + 1) + 2]) / 1e3 : 0.0;
      printf("[%d loc %.2f handoff %.2f lasttile %.2f] ", s, a, b, c);
    }
    printf("\n");
  }
  cudaFree(LU); cudaFree(y); cudaFree(ctr); cudaFree(tout); cudaFree(ctl); cudaFree(part); cudaFree(rh); cudaFree(rl);
  return best;
}

int main() {
  if (getenv("STAMPS")) {
    printf("f64 fwd n=1024 G=16: %.1f us\n", run<MODE_F64, true>(1024, 16, 0));
    return 0;
  }
  for (int n : {1024, 2048, 8192}) {
    for (int G : {16, 64, 148}) {
      if (G > n / 32) continue;
      printf("n %5d G %3d  f64 fwd %8.1f us  bwd %8.1f us | dd fwd %8.1f us  bwd %8.1f us (rcp bwd %8.1f)\n", n, G,
             run<MODE_F64, true>(n, G, 0), run<MODE_F64, false>(n, G, 0), run<MODE_DD, true>(n, G, 0),
             run<MODE_DD, false>(n, G, 0), run<MODE_DD, false>(n, G, 1));
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
