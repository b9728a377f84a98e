// Microbenchmark of the leader's nonsymmetric eigen-solve (warp_hqr) on a
// random p x p matrix held in shared memory.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a hqr.cu -o hqr
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2201_09827_b200/csrc/gb_dense.cuh"
using namespace gb;

#ifndef NOZ
#define NOZ 0
#endif
namespace gb {

GB_DEVICE double frcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  // two Newton steps: r <- r (2 - x r)
  double e = __fma_rn(-x, r, 1.0);
  r = __fma_rn(r, e, r);
  e = __fma_rn(-x, r, 1.0);
  return __fma_rn(r, e, r);
}
GB_DEVICE double fsqrt(double t) {
  // sqrt via rsqrt + Newton (t > 0)
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(t));
  double h = 0.5 * y;
  double g = t * y;
  double r = __fma_rn(-g, h, 0.5);
  g = __fma_rn(g, r, g);
  h = __fma_rn(h, r, h);
  r = __fma_rn(-g, h, 0.5);
  g = __fma_rn(g, r, g);
  double d = __fma_rn(-g, g, t);
  return __fma_rn(d, h, g);
}
static __device__ __noinline__ bool warp_hqr_dbg(double* H, int ld, int p, double* Z, int ldz, double* wr, double* wi,
                                double* ort, unsigned long long* st) {
  unsigned long long c0 = clock64();
  const int lane = threadIdx.x & 31;
  const int nn = p, low = 0, high = p - 1;
  // --- orthes: Householder reduction to Hessenberg form ---
  for (int m = low + 1; m <= high - 1; ++m) {
    double scale = 0.0;
    for (int i = m + lane; i <= high; i += 32) scale += fabs(H[IX(i, m - 1, ld)]);
    scale = warp_sum(scale);
    if (scale == 0.0) continue;
    double hh = 0.0;
    for (int i = m + lane; i <= high; i += 32) {
      double o = H[IX(i, m - 1, ld)] / scale;
      ort[i] = o;
      hh = __fma_rn(o, o, hh);
    }
    hh = warp_sum(hh);
    __syncwarp();
    double om = ort[m];
    double g = sqrt(hh);
    if (om > 0) g = -g;
    hh = hh - om * g;
    __syncwarp();
    if (lane == 0) ort[m] = om - g;
    __syncwarp();
    for (int j = m + lane; j < nn; j += 32) {
      double f = 0.0;
      for (int i = high; i >= m; --i) f = __fma_rn(ort[i], H[IX(i, j, ld)], f);
      f = f / hh;
      for (int i = m; i <= high; ++i) H[IX(i, j, ld)] = __fma_rn(-f, ort[i], H[IX(i, j, ld)]);
    }
    __syncwarp();
    for (int i = lane; i <= high; i += 32) {
      double f = 0.0;
      for (int j = high; j >= m; --j) f = __fma_rn(ort[j], H[IX(i, j, ld)], f);
      f = f / hh;
      for (int j = m; j <= high; ++j) H[IX(i, j, ld)] = __fma_rn(-f, ort[j], H[IX(i, j, ld)]);
    }
    __syncwarp();
    if (lane == 0) {
      ort[m] = scale * ort[m];
      H[IX(m, m - 1, ld)] = scale * g;
    }
    __syncwarp();
  }
  for (int e = lane; e < nn * nn; e += 32) Z[IX(e % nn, e / nn, ldz)] = (e % nn == e / nn) ? 1.0 : 0.0;
  __syncwarp();
  for (int m = high - 1; m >= low + 1; --m) {
    double hm = H[IX(m, m - 1, ld)];
    if (hm == 0.0) continue;
    for (int i = m + 1 + lane; i <= high; i += 32) ort[i] = H[IX(i, m - 1, ld)];
    __syncwarp();
    for (int j = m + lane; j <= high; j += 32) {
      double g = 0.0;
      for (int i = m; i <= high; ++i) g = __fma_rn(ort[i], Z[IX(i, j, ldz)], g);
      g = (g / ort[m]) / hm;
      for (int i = m; i <= high; ++i) Z[IX(i, j, ldz)] = __fma_rn(g, ort[i], Z[IX(i, j, ldz)]);
    }
    __syncwarp();
  }
  // clear below the subdiagonal
  for (int e = lane; e < nn * nn; e += 32) {
    int i = e % nn, j = e / nn;
    if (i > j + 1) H[IX(i, j, ld)] = 0.0;
  }
  __syncwarp();

  unsigned long long c1 = clock64();
  unsigned long long nsteps = 0, nsweeps = 0;
  // --- hqr2: Francis double-shift QR with accumulation ---
  int n = nn - 1;
  const double eps = kEps52;
  double exshift = 0.0, p_ = 0, q = 0, r = 0, s = 0, z = 0, t, w, x, y;
  double norm = 0.0;
  for (int i = lane; i < nn; i += 32)
    for (int j = max(i - 1, 0); j < nn; ++j) norm += fabs(H[IX(i, j, ld)]);
  norm = warp_sum(norm);
  int iter = 0, total = 0;
  const int itmax = 40 * max(10, nn);
  while (n >= low) {
    int l = n;
    while (l > low) {
      s = fabs(H[IX(l - 1, l - 1, ld)]) + fabs(H[IX(l, l, ld)]);
      if (s == 0.0) s = norm;
      if (fabs(H[IX(l, l - 1, ld)]) < eps * s) break;
      l--;
    }
    if (l == n) {
      __syncwarp();
      if (lane == 0) {
        H[IX(n, n, ld)] = H[IX(n, n, ld)] + exshift;
        wr[n] = H[IX(n, n, ld)];
        wi[n] = 0.0;
      }
      __syncwarp();
      n--;
      iter = 0;
    } else if (l == n - 1) {
      w = H[IX(n, n - 1, ld)] * H[IX(n - 1, n, ld)];
      p_ = (H[IX(n - 1, n - 1, ld)] - H[IX(n, n, ld)]) / 2.0;
      q = p_ * p_ + w;
      z = sqrt(fabs(q));
      double hnn = H[IX(n, n, ld)] + exshift;
      double hn1 = H[IX(n - 1, n - 1, ld)] + exshift;
      __syncwarp();
      if (lane == 0) {
        H[IX(n, n, ld)] = hnn;
        H[IX(n - 1, n - 1, ld)] = hn1;
      }
      __syncwarp();
      x = hnn;
      if (q >= 0) {
        z = (p_ >= 0) ? p_ + z : p_ - z;
        double d1 = x + z, d2 = d1;
        if (z != 0.0) d2 = x - w / z;
        if (lane == 0) {
          wr[n - 1] = d1;
          wr[n] = d2;
          wi[n - 1] = 0.0;
          wi[n] = 0.0;
        }
        x = H[IX(n, n - 1, ld)];
        s = fabs(x) + fabs(z);
        p_ = x / s;
        q = z / s;
        r = sqrt(p_ * p_ + q * q);
        p_ = p_ / r;
        q = q / r;
        __syncwarp();
        for (int j = n - 1 + lane; j < nn; j += 32) {
          double zz = H[IX(n - 1, j, ld)];
          H[IX(n - 1, j, ld)] = q * zz + p_ * H[IX(n, j, ld)];
          H[IX(n, j, ld)] = q * H[IX(n, j, ld)] - p_ * zz;
        }
        __syncwarp();
        for (int i = lane; i <= n; i += 32) {
          double zz = H[IX(i, n - 1, ld)];
          H[IX(i, n - 1, ld)] = q * zz + p_ * H[IX(i, n, ld)];
          H[IX(i, n, ld)] = q * H[IX(i, n, ld)] - p_ * zz;
        }
        for (int i = low + lane; i <= high; i += 32) {
          double zz = Z[IX(i, n - 1, ldz)];
          Z[IX(i, n - 1, ldz)] = q * zz + p_ * Z[IX(i, n, ldz)];
          Z[IX(i, n, ldz)] = q * Z[IX(i, n, ldz)] - p_ * zz;
        }
        __syncwarp();
      } else {
        if (lane == 0) {
          wr[n - 1] = x + p_;
          wr[n] = x + p_;
          wi[n - 1] = z;
          wi[n] = -z;
        }
        __syncwarp();
      }
      n = n - 2;
      iter = 0;
    } else {
      x = H[IX(n, n, ld)];
      y = 0.0;
      w = 0.0;
      if (l < n) {
        y = H[IX(n - 1, n - 1, ld)];
        w = H[IX(n, n - 1, ld)] * H[IX(n - 1, n, ld)];
      }
      if (iter == 10) {
        exshift += x;
        __syncwarp();
        for (int i = low + lane; i <= n; i += 32) H[IX(i, i, ld)] -= x;
        __syncwarp();
        s = fabs(H[IX(n, n - 1, ld)]) + fabs(H[IX(n - 1, n - 2, ld)]);
        x = y = 0.75 * s;
        w = -0.4375 * s * s;
      }
      if (iter == 30) {
        s = (y - x) / 2.0;
        s = s * s + w;
        if (s > 0) {
          s = sqrt(s);
          if (y < x) s = -s;
          s = x - w / ((y - x) / 2.0 + s);
          __syncwarp();
          for (int i = low + lane; i <= n; i += 32) H[IX(i, i, ld)] -= s;
          __syncwarp();
          exshift += s;
          x = y = w = 0.964;
        }
      }
      iter++;
      if (++total > itmax) return false;
      int m = n - 2;
      while (m >= l) {
        z = H[IX(m, m, ld)];
        r = x - z;
        s = y - z;
        p_ = (r * s - w) / H[IX(m + 1, m, ld)] + H[IX(m, m + 1, ld)];
        q = H[IX(m + 1, m + 1, ld)] - z - r - s;
        r = H[IX(m + 2, m + 1, ld)];
        s = fabs(p_) + fabs(q) + fabs(r);
        p_ = p_ / s;
        q = q / s;
        r = r / s;
        if (m == l) break;
        if (fabs(H[IX(m, m - 1, ld)]) * (fabs(q) + fabs(r)) <
            eps * (fabs(p_) * (fabs(H[IX(m - 1, m - 1, ld)]) + fabs(z) + fabs(H[IX(m + 1, m + 1, ld)]))))
          break;
        m--;
      }
      __syncwarp();
      for (int i = m + 2 + lane; i <= n; i += 32) {
        H[IX(i, i - 2, ld)] = 0.0;
        if (i > m + 2) H[IX(i, i - 3, ld)] = 0.0;
      }
      __syncwarp();
      ++nsweeps;
      for (int k = m; k <= n - 1; ++k) {
        ++nsteps;
        bool notlast = (k != n - 1);
        if (k != m) {
          p_ = H[IX(k, k - 1, ld)];
          q = H[IX(k + 1, k - 1, ld)];
          r = notlast ? H[IX(k + 2, k - 1, ld)] : 0.0;
          x = fabs(p_) + fabs(q) + fabs(r);
          if (x == 0.0) continue;
          const double rx = frcp(x);  // one division instead of three
          p_ = p_ * rx;
          q = q * rx;
          r = r * rx;
        }
        s = fsqrt(p_ * p_ + q * q + r * r);
        if (p_ < 0) s = -s;
        if (s != 0) {
          __syncwarp();
          if (lane == 0) {
            if (k != m) H[IX(k, k - 1, ld)] = -s * x;
            else if (l != m) H[IX(k, k - 1, ld)] = -H[IX(k, k - 1, ld)];
          }
          __syncwarp();
          p_ = p_ + s;
          const double rs = frcp(s), rp = frcp(p_);
          x = p_ * rs;
          y = q * rs;
          z = r * rs;
          q = q * rp;
          r = r * rp;
          for (int j = k + lane; j < nn; j += 32) {
            double pp = H[IX(k, j, ld)] + q * H[IX(k + 1, j, ld)];
            if (notlast) {
              pp = pp + r * H[IX(k + 2, j, ld)];
              H[IX(k + 2, j, ld)] = H[IX(k + 2, j, ld)] - pp * z;
            }
            H[IX(k, j, ld)] = H[IX(k, j, ld)] - pp * x;
            H[IX(k + 1, j, ld)] = H[IX(k + 1, j, ld)] - pp * y;
          }
          __syncwarp();
          const int iend = min(n, k + 3);
          for (int i = lane; i <= iend; i += 32) {
            double pp = x * H[IX(i, k, ld)] + y * H[IX(i, k + 1, ld)];
            if (notlast) {
              pp = pp + z * H[IX(i, k + 2, ld)];
              H[IX(i, k + 2, ld)] = H[IX(i, k + 2, ld)] - pp * r;
            }
            H[IX(i, k, ld)] = H[IX(i, k, ld)] - pp;
            H[IX(i, k + 1, ld)] = H[IX(i, k + 1, ld)] - pp * q;
          }
          if (!NOZ) for (int i = low + lane; i <= high; i += 32) {
            double pp = x * Z[IX(i, k, ldz)] + y * Z[IX(i, k + 1, ldz)];
            if (notlast) {
              pp = pp + z * Z[IX(i, k + 2, ldz)];
              Z[IX(i, k + 2, ldz)] = Z[IX(i, k + 2, ldz)] - pp * r;
            }
            Z[IX(i, k, ldz)] = Z[IX(i, k, ldz)] - pp;
            Z[IX(i, k + 1, ldz)] = Z[IX(i, k + 1, ldz)] - pp * q;
          }
          __syncwarp();
        }
      }
    }
  }
  __syncwarp();
  if ((threadIdx.x & 31) == 0) { st[0] = c1 - c0; st[1] = clock64() - c1; st[2] = nsweeps; st[3] = nsteps; }
  return true;
}

}  // namespace gb

__global__ void k_hqr(const double* A, int p, int ld, double* wr_out, double* wi_out, unsigned long long* cyc, int* ok) {
  __shared__ unsigned long long st[4];
  extern __shared__ double sm[];
  double* H = sm;
  double* Z = H + ld * p;
  double* wr = Z + ld * p;
  double* wi = wr + p;
  double* ort = wi + p;
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) H[(e % p) + (e / p) * ld] = A[e];
  __syncthreads();
  unsigned long long t0 = clock64();
  if (threadIdx.x < 32) {
    bool r = warp_hqr_dbg(H, ld, p, Z, ld, wr, wi, ort, st);
    if (threadIdx.x == 0) *ok = r;
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; for (int i = 0; i < 4; ++i) cyc[1 + i] = st[i]; }
  for (int i = threadIdx.x; i < p; i += blockDim.x) {
    wr_out[i] = wr[i];
    wi_out[i] = wi[i];
  }
}

int main() {
  for (int pl : {40, 60, 100, 1040, 1060, 1100}) {
    const int p = pl % 1000, ld = pl > 1000 ? (p | 1) : p;
    std::vector<double> a(p * p);
    srand(1);
    for (auto& x : a) x = (rand() / (double)RAND_MAX) - 0.5;
    double *dA, *wr, *wi;
    unsigned long long* cyc;
    int* ok;
    cudaMalloc(&dA, 8 * p * p);
    cudaMalloc(&wr, 8 * p);
    cudaMalloc(&wi, 8 * p);
    cudaMalloc(&cyc, 40);
    cudaMalloc(&ok, 4);
    cudaMemcpy(dA, a.data(), 8 * p * p, cudaMemcpyHostToDevice);
    size_t sm = 8 * (2 * ld * p + 3 * p);
    cudaFuncSetAttribute(k_hqr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    unsigned long long best = ~0ull, stv[5];
    for (int it = 0; it < 3; ++it) {
      k_hqr<<<1, 256, sm>>>(dA, p, ld, wr, wi, cyc, ok);
      unsigned long long c;
      cudaMemcpy(stv, cyc, 40, cudaMemcpyDeviceToHost);
      c = stv[0];
      best = c < best ? c : best;
    }
    std::vector<double> hr(p), hi(p);
    int hok;
    cudaMemcpy(hr.data(), wr, 8 * p, cudaMemcpyDeviceToHost);
    cudaMemcpy(hi.data(), wi, 8 * p, cudaMemcpyDeviceToHost);
    cudaMemcpy(&hok, ok, 4, cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 0; i < p; ++i) s += hr[i] * hr[i] + hi[i] * hi[i];
    printf("orthes %llu hqr %llu sweeps %llu steps %llu (%.0f cyc/step) | ", stv[1], stv[2], stv[3], stv[4], (double)stv[2] / stv[4]);
    printf("ld %4d p %4d ok %d cycles %llu (%.1f us @1.9GHz) sum|l|^2 %.12e\n", ld, p, hok, best, best / 1.9e3, s);
    cudaFree(dA); cudaFree(wr); cudaFree(wi); cudaFree(cyc); cudaFree(ok);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
