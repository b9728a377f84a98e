// Micro-benchmark + check of the tcgen05 trailing update (csrc/gb_tcgemm.cuh)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include tools/micro/tcgemm.cu -o tools/micro/tcgemm
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <random>
#include "../../paper_2201_09827_b200/csrc/gb_tcgemm.cuh"
using namespace gb;
int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 8192;
  const int K = argc > 2 ? atoi(argv[2]) : 256;
  const int pairmode = argc > 3 ? atoi(argv[3]) : 1;  // 1: CTA-pair kernel (cta_group::2, C through smem + TMA when whole tiles), 2: pair kernel, register epilogue, 0: one-CTA kernel
  const size_t ld = (n + 31) & ~31;
  std::mt19937 rng(3);
  std::uniform_real_distribution<float> U(-1.f, 1.f);
  std::vector<__half> W((size_t)n * ld);
  for (auto& x : W) x = __float2half(U(rng));
  __half *dW, *dBt;
  cudaMalloc(&dW, W.size() * 2);
  cudaMalloc(&dBt, (size_t)n * K * 2);
  cudaMemcpy(dW, W.data(), W.size() * 2, cudaMemcpyHostToDevice);
  const int k0 = 0, r0 = K, c0 = K, M = n - K, N = n - K;
  int nsm = 148;
  auto upd = [&]() {
    return pairmode ? tcg2::tc_update(dW, ld, n, r0, c0, M, N, k0, K, dBt, 0, pairmode == 2 ? 0 : -1)
                    : tcg::tc_update(dW, ld, n, r0, c0, M, N, k0, K, dBt, nsm, 0);
  };
  if (pairmode) printf("co-resident CTA pairs: %d\n", tcg2::max_pairs());
  cudaError_t e = upd();
  cudaError_t e2 = cudaDeviceSynchronize();
  printf("n=%d K=%d launch: %s / %s\n", n, K, cudaGetErrorString(e), cudaGetErrorString(e2));
  std::vector<__half> R(W.size());
  cudaMemcpy(R.data(), dW, R.size() * 2, cudaMemcpyDeviceToHost);
  // check sampled rows against a double-precision accumulation
  int bad = 0, off1 = 0; long checked = 0;
  for (int t = 0; t < 48; ++t) {
    const int i = r0 + (int)(rng() % M);
    for (int j = c0; j < c0 + N; j += 7) {
      double acc = 0;
      for (int k = 0; k < K; ++k) acc += (double)__half2float(W[(size_t)i * ld + k0 + k]) * __half2float(W[(size_t)(k0 + k) * ld + j]);
      const float ref = __half2float(__float2half_rn((float)((double)__half2float(W[(size_t)i * ld + j]) - acc)));
      const float got = __half2float(R[(size_t)i * ld + j]);
      const float ulp = std::fabs(ref) < 6.1e-5f ? 6e-8f : std::ldexp(1.f, std::ilogb(ref) - 10);
      const float d = std::fabs(got - ref);
      if (d > 1.01f * ulp) ++bad; else if (d > 0) ++off1;
      ++checked;
    }
  }
  printf("check: %ld entries, %d beyond 1 fp16 ulp, %d at 1 ulp (fp32 accumulation order)\n", checked, bad, off1);
  // timing: repeated updates (values drift; only the time matters)
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 2; ++i) upd();
  const int reps = 10;
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) upd();
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); ms /= reps;
  const double fl = 2.0 * M * N * K;
  printf("update[%s] M=N=%d K=%d: %.1f us  %.1f TFLOP/s (%.1f%% of 1593.7)  [%s]\n", pairmode ? "pair" : "1cta", M, K, ms * 1e3, fl / (ms * 1e-3) / 1e12,
         100 * fl / (ms * 1e-3) / 1e12 / 1593.7, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
