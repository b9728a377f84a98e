// Microbenchmark of trsv_cta (CTA-per-block F64 / DD triangular solve) alone.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -DGB_SPIN_NS=8 trsv_cta.cu -o trsv_cta
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2201_09827_b200/csrc/gb_ops.cuh"
using namespace gb;

template <int M, bool kLower>
__global__ void __launch_bounds__(256) k_trsv(int n, const float* LU, size_t ld, typename Arith<M>::T* y,
                                              unsigned long long* ctr, unsigned long long epoch, GridCtl* ctl,
                                              double* partials, unsigned long long* tout, const double* ih,
                                              const double* il, unsigned long long* stamps, uint4* yt) {
  extern __shared__ __align__(16) unsigned char smem[];
  GridTeam t{(int)gridDim.x, (int)blockIdx.x, ctl, partials, 64, 0u, gridDim.x > 1 && cluster_ncta() == gridDim.x};
  TrsvSync ts{ctr, ctr + 1, epoch, PhaseLog{nullptr, 0}, stamps, yt};
  if (t.clu) {  // tagged y in cluster shared memory (after the TRSV tiles)
    uint4* loc = reinterpret_cast<uint4*>(smem + 8 * 32 * 33 * sizeof(double) + 256 * 16);
    for (int i = threadIdx.x; i < 2 * n; i += blockDim.x) loc[i] = yt[i];  // same initial tags
    ts.ytag = loc;
    ts.dsm = t.size();
  }
  t.sync();
  unsigned long long t0 = gtimer();
  trsv_cta<M, GridTeam, float, kLower>(t, n, LU, ld, y, ts, smem, ih, il);
  t.sync();
  if (t.clu && (stamps != nullptr)) {}
  if (blockIdx.x == 0 && threadIdx.x == 0) tout[0] = gtimer() - t0;
}

template <int M, bool kLower>
float run(int n, int G, bool stamps_out, bool clu = false) {
  using T = typename Arith<M>::T;
  size_t ld = (n + 31) & ~31;
  int nb = (n + 31) / 32;
  std::vector<float> h((size_t)n * ld);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) h[(size_t)i * ld + j] = (i == j) ? 2.0f : 0.5f / n;
  std::vector<double> inv((size_t)nb * kInvStride, 0.0);
  for (int b = 0; b < nb; ++b)
    for (int i = 0; i < 32; ++i) inv[(size_t)b * kInvStride + i * 33] = 0.5;
  float* LU;
  T* y;
  unsigned long long *ctr, *tout, *stamps;
  GridCtl* ctl;
  double *part, *ih, *il;
  cudaMalloc(&LU, sizeof(float) * h.size());
  cudaMemcpy(LU, h.data(), sizeof(float) * h.size(), cudaMemcpyHostToDevice);
  cudaMalloc(&y, sizeof(T) * n);
  cudaMemset(y, 0, sizeof(T) * n);
  cudaMalloc(&ctr, 32);
  cudaMalloc(&tout, 8);
  cudaMalloc(&ctl, sizeof(GridCtl));
  cudaMemset(ctl, 0, sizeof(GridCtl));
  cudaMalloc(&part, 8 * 2 * 64 * 256);
  cudaMalloc(&ih, 8 * inv.size());
  cudaMalloc(&il, 8 * inv.size());
  cudaMemcpy(ih, inv.data(), 8 * inv.size(), cudaMemcpyHostToDevice);
  cudaMemset(il, 0, 8 * inv.size());
  uint4* yt;
  cudaMalloc(&yt, 32 * (size_t)n);
  cudaMemset(yt, 0, 32 * (size_t)n);
  cudaMalloc(&stamps, 8 * 3 * nb);
  cudaMemset(stamps, 0, 8 * 3 * nb);
  size_t sm = 8 * 32 * 33 * sizeof(double) + 256 * 16 + (clu ? 32 * (size_t)n : 0);
  auto kern = k_trsv<M, kLower>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  unsigned long long epoch = 0, hout = 0;
  float best = 1e30f;
  for (int it = 0; it < 5; ++it) {
    epoch = it;
    if (!kLower) {  // fake a finished forward sweep of this epoch
      std::vector<unsigned> w(8 * (size_t)n);
      for (size_t e = 0; e < w.size(); e += 2) { w[e] = 0; w[e + 1] = 2 * it + 1; }
      cudaMemcpy(yt, w.data(), 4 * w.size(), cudaMemcpyHostToDevice);
    }
    void* args[] = {&n, &LU, &ld, &y, &ctr, &epoch, &ctl, &part, &tout, &ih, &il, &stamps, &yt};
    if (clu) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(G);
      cfg.blockDim = dim3(256);
      cfg.dynamicSmemBytes = sm;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = G;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, kern, n, (const float*)LU, ld, y, ctr, epoch, ctl, part, tout, (const double*)ih,
                         (const double*)il, stamps, yt);
    } else {
      cudaLaunchCooperativeKernel((void*)kern, G, 256, args, sm, 0);
    }
    cudaDeviceSynchronize();
    cudaMemcpy(&hout, tout, 8, cudaMemcpyDeviceToHost);
    best = std::min(best, hout / 1e3f);
  }
  if (stamps_out) {
    std::vector<unsigned long long> st(3 * nb);
    cudaMemcpy(st.data(), stamps, 8 * 3 * nb, cudaMemcpyDeviceToHost);
    double hand = 0, slack = 0, pub = 0;
    int cnt = 0;
    for (int s = 1; s < nb; ++s) {
      hand += ((double)st[3 * s + 2] - (double)st[3 * (s - 1) + 1]) / 1e3;
      slack += ((double)st[3 * s + 2] - (double)st[3 * s]) / 1e3;
      pub += ((double)st[3 * s + 1] - (double)st[3 * s + 2]) / 1e3;
      ++cnt;
    }
    printf("   per link: stored->seen %.2f us, z ready before seen %.2f us, seen->stored %.2f us\n", hand / cnt,
           slack / cnt, pub / cnt);
  }
  cudaFree(LU); cudaFree(y); cudaFree(ctr); cudaFree(tout); cudaFree(ctl); cudaFree(part); cudaFree(ih);
  cudaFree(il); cudaFree(stamps); cudaFree(yt);
  return best;
}

int main() {
  for (int n : {1024, 8192}) {
    for (int G : {32, 148}) {
      if (G > n / 32) continue;
      printf("n %5d G %3d  f64 fwd %8.1f us  bwd %8.1f us | dd fwd %8.1f us  bwd %8.1f us\n", n, G,
             run<MODE_F64, true>(n, G, false), run<MODE_F64, false>(n, G, false), run<MODE_DD, true>(n, G, false),
             run<MODE_DD, false>(n, G, false));
    }
  }
  for (int G : {8, 16}) {
    printf("cluster n 1024 G %d: f64 fwd %8.1f us bwd %8.1f us | dd fwd %8.1f us bwd %8.1f us\n", G,
           run<MODE_F64, true>(1024, G, false, true), run<MODE_F64, false>(1024, G, false, true),
           run<MODE_DD, true>(1024, G, false, true), run<MODE_DD, false>(1024, G, false, true));
    printf("grid    n 1024 G %d: f64 fwd %8.1f us bwd %8.1f us | dd fwd %8.1f us bwd %8.1f us\n", G,
           run<MODE_F64, true>(1024, G, false, false), run<MODE_F64, false>(1024, G, false, false),
           run<MODE_DD, true>(1024, G, false, false), run<MODE_DD, false>(1024, G, false, false));
  }
  printf("dd fwd n=1024 G=16 cluster:\n");
  run<MODE_DD, true>(1024, 16, true, true);
  printf("dd bwd n=1024 G=16 cluster:\n");
  run<MODE_DD, false>(1024, 16, true, true);
  printf("f64 fwd n=1024 G=16 cluster:\n");
  run<MODE_F64, true>(1024, 16, true, true);
  printf("dd fwd n=1024 G=32:\n");
  run<MODE_DD, true>(1024, 32, true);
  printf("dd fwd n=8192 G=148:\n");
  run<MODE_DD, true>(8192, 148, true);
  printf("f64 fwd n=8192 G=148:\n");
  run<MODE_F64, true>(8192, 148, true);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
