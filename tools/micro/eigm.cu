// device warp_hqr (the leader eigensolve) on a matrix from disk (column-major fp64)
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cmath>
#include <cuda_runtime.h>
#include "../../paper_2201_09827_b200/csrc/gb_dense.cuh"
__global__ void k_hqr(const double* A, int p, double* out, int* ok) {
  extern __shared__ double sm[];
  double* H = sm; double* Z = H + p * p; double* wr = Z + p * p; double* wi = wr + p; double* ort = wi + p;
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) H[e] = A[e];
  __syncthreads();
  if (threadIdx.x < 64) { bool r = gb::warp_hqr(H, p, p, Z, p, wr, wi, ort); if (threadIdx.x == 0) *ok = r; }
  __syncthreads();
  for (int e = threadIdx.x; e < 2 * p; e += blockDim.x) out[e] = wr[e];
}
int main(int argc, char** argv) {
  int p = atoi(argv[2]);
  std::vector<double> a(p * p);
  FILE* f = fopen(argv[1], "rb"); fread(a.data(), 8, p * p, f); fclose(f);
  double *dA, *o; int* ok;
  cudaMalloc(&dA, 8 * p * p); cudaMalloc(&o, 16 * p); cudaMalloc(&ok, 4);
  cudaMemcpy(dA, a.data(), 8 * p * p, cudaMemcpyHostToDevice);
  size_t sm = 8 * (2 * p * p + 3 * p);
  cudaFuncSetAttribute(k_hqr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_hqr<<<1, 256, sm>>>(dA, p, o, ok);
  std::vector<double> w(2 * p); int hok;
  cudaMemcpy(w.data(), o, 16 * p, cudaMemcpyDeviceToHost); cudaMemcpy(&hok, ok, 4, cudaMemcpyDeviceToHost);
  std::vector<int> ord(p); for (int i = 0; i < p; ++i) ord[i] = i;
  std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return std::hypot(w[x], w[p + x]) < std::hypot(w[y], w[p + y]); });
  printf("ok %d\n", hok);
  for (int i = 0; i < 14; ++i) printf("%d %.16e %+.16e |%.16e|\n", ord[i], w[ord[i]], w[p + ord[i]], std::hypot(w[ord[i]], w[p + ord[i]]));
  return 0;
}
