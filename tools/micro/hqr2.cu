// A/B of the leader eigensolve (warp_hqr): the current gb_dense.cuh against
// the previous version (old_dense.cuh, namespace gbold) -- bitwise-equal
// Schur form, Schur vectors and eigenvalues, and cycles.
//   old_dense.cuh = a previous gb_dense.cuh moved into namespace gbold:
//     git show <rev>:paper_2201_09827_b200/csrc/gb_dense.cuh | sed 's/namespace gb {/namespace gbold {\nusing namespace gb;/;
//       s/^}  \/\/ namespace gb/}  \/\/ namespace gbold/; s|#include "gb_common.cuh"|#include "../../paper_2201_09827_b200/csrc/gb_common.cuh"|' > old_dense.cuh
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a hqr2.cu -o hqr2
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2201_09827_b200/csrc/gb_dense.cuh"
#include "old_dense.cuh"

template <int V>
__global__ void k_hqr(const double* A, int p, double* out, unsigned long long* cyc, int* ok) {
  extern __shared__ double sm[];
  double* H = sm;
  double* Z = H + p * p;
  double* wr = Z + p * p;
  double* wi = wr + p;
  double* ort = wi + p;
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) H[e] = A[e];
  __syncthreads();
  unsigned long long t0 = clock64();
  if (threadIdx.x < 64) {
    bool r = V == 0 ? gbold::warp_hqr(H, p, p, Z, p, wr, wi, ort) : gb::warp_hqr(H, p, p, Z, p, wr, wi, ort);
    if (threadIdx.x == 0) *ok = r;
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  for (int e = threadIdx.x; e < 2 * p * p + 2 * p; e += blockDim.x) out[e] = sm[e];
}

int main() {
  for (int p : {40, 50, 60, 64}) {
    std::vector<double> a(p * p);
    srand(p);
    for (auto& x : a) x = (rand() / (double)RAND_MAX) - 0.5;
    double *dA, *o0, *o1;
    unsigned long long* cyc;
    int* ok;
    size_t nout = 2 * p * p + 2 * p;
    cudaMalloc(&dA, 8 * p * p);
    cudaMalloc(&o0, 8 * nout);
    cudaMalloc(&o1, 8 * nout);
    cudaMalloc(&cyc, 16);
    cudaMalloc(&ok, 8);
    cudaMemcpy(dA, a.data(), 8 * p * p, cudaMemcpyHostToDevice);
    size_t sm = 8 * (2 * p * p + 3 * p);
    cudaFuncSetAttribute(k_hqr<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(k_hqr<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    unsigned long long c0 = ~0ull, c1 = ~0ull, c;
    for (int it = 0; it < 3; ++it) {
      k_hqr<0><<<1, 256, sm>>>(dA, p, o0, cyc, ok);
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      c0 = c < c0 ? c : c0;
      k_hqr<1><<<1, 256, sm>>>(dA, p, o1, cyc + 1, ok + 1);
      cudaMemcpy(&c, cyc + 1, 8, cudaMemcpyDeviceToHost);
      c1 = c < c1 ? c : c1;
    }
    std::vector<double> h0(nout), h1(nout);
    int hok[2];
    cudaMemcpy(h0.data(), o0, 8 * nout, cudaMemcpyDeviceToHost);
    cudaMemcpy(h1.data(), o1, 8 * nout, cudaMemcpyDeviceToHost);
    cudaMemcpy(hok, ok, 8, cudaMemcpyDeviceToHost);
    printf("p %3d ok %d/%d old %llu cyc new %llu cyc (x%.2f) bitwise-equal %s\n", p, hok[0], hok[1], c0, c1,
           (double)c0 / c1, memcmp(h0.data(), h1.data(), 8 * nout) == 0 ? "yes" : "NO");
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
