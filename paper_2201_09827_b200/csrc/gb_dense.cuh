// Small dense fp64 linear algebra run by ONE CTA (the team leader): the
// harmonic-Ritz eigenproblems, least-squares and QR of GCRO-DR
// (reference densela.py:410-477, gcrodr.py:104-218).
//
// Matrices are column-major (a[i + j*ld]) fp64 in global memory.  Routines
// named blk_* must be called by every thread of the CTA; warp_* by every
// thread too, but only warp 0 computes (the others wait at the closing
// __syncthreads).  Scalar bookkeeping is replicated in the participating
// threads (identical inputs give identical values); scalar stores are done by
// one thread followed by a barrier.
//
// Algorithms (restated from the published literature, not from the reference):
//   * GEPP with first-max pivots (LAPACK dgetrf/dgetrs semantics);
//   * Householder QR with the dlarfg sign convention + explicit Q (dgeqrf/dorgqr);
//   * nonsymmetric eigenproblem: Householder reduction to Hessenberg form and
//     the Francis double-shift QR iteration with accumulated Schur vectors
//     (EISPACK orthes/hqr2), eigenvectors by back-substitution on the real
//     Schur form for the selected eigenvalues only, normalised like LAPACK
//     dgeev (unit 2-norm, largest component real via la_xlartg);
//   * 2-norm condition number from a Householder bidiagonalisation and
//     Sturm-count bisection on the Golub-Kahan tridiagonal (relative accuracy
//     of the extreme singular values).
#pragma once
#include "gb_common.cuh"

namespace gb {

#define IX(i, j, ld) ((size_t)(i) + (size_t)(j) * (ld))

constexpr double kEps53 = 1.1102230246251565e-16;  // 2^-53
constexpr double kEps52 = 2.220446049250313e-16;   // 2^-52

// ---------------------------------------------------------------------------
// GEPP  (a: p x p in place, piv[k] = row exchanged with k) -> first zero or -1
// ---------------------------------------------------------------------------
static __device__ __noinline__ int blk_getrf(double* a, int ld, int p, int* piv) {
  __shared__ int s_piv;
  __shared__ double s_key[64];
  __shared__ int s_idx[32];
  int zero = -1;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int k = 0; k < p; ++k) {
    // first max of |a[k:, k]|
    double bv = -1.0;
    int bi = p;
    for (int i = k + threadIdx.x; i < p; i += blockDim.x) {
      double v = fabs(a[IX(i, k, ld)]);
      if (v != v) v = __longlong_as_double(0x7ff0000000000000ull);
      if (v > bv) {
        bv = v;
        bi = i;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      s_key[wid] = bv;
      s_idx[wid] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double v = s_key[0];
      int ii = s_idx[0];
      for (int w = 1; w < nw; ++w)
        if (s_key[w] > v || (s_key[w] == v && s_idx[w] < ii)) {
          v = s_key[w];
          ii = s_idx[w];
        }
      s_piv = ii;
      piv[k] = ii;
    }
    __syncthreads();
    const int pk = s_piv;
    const double pv = a[IX(pk, k, ld)];
    if (pv == 0.0) {
      if (zero < 0) zero = k;
      __syncthreads();
      continue;
    }
    if (pk != k)
      for (int j = threadIdx.x; j < p; j += blockDim.x) {
        double t = a[IX(k, j, ld)];
        a[IX(k, j, ld)] = a[IX(pk, j, ld)];
        a[IX(pk, j, ld)] = t;
      }
    __syncthreads();
    const double rp = 1.0 / pv;
    for (int i = k + 1 + threadIdx.x; i < p; i += blockDim.x) a[IX(i, k, ld)] *= rp;
    __syncthreads();
    // trailing update: warp per column, lanes down the rows (no div/mod)
    for (int j = k + 1 + wid; j < p; j += nw) {
      const double akj = a[IX(k, j, ld)];
      for (int i = k + 1 + lane; i < p; i += 32) a[IX(i, j, ld)] = __fma_rn(-a[IX(i, k, ld)], akj, a[IX(i, j, ld)]);
    }
    __syncthreads();
  }
  return zero;
}

// B (p x q) <- A^-1 B using blk_getrf factors.  The row interchanges run one
// thread per column; the substitutions sweep j in order with every (row,
// column) update of a step in parallel, so each element sees the same
// operation sequence as a per-column column-sweep solve.
static __device__ __noinline__ void blk_getrs(const double* a, int ld, int p, const int* piv, double* b, int ldb,
                                 int q) {
  for (int c = threadIdx.x; c < q; c += blockDim.x) {
    double* x = b + (size_t)c * ldb;
    for (int k = 0; k < p; ++k) {
      int pk = piv[k];
      if (pk != k) {
        double t = x[k];
        x[k] = x[pk];
        x[pk] = t;
      }
    }
  }
  __syncthreads();
  // forward (unit lower) and backward (upper) sweeps: lanes down the rows,
  // each warp takes 4 right-hand-side columns per pass with all loads issued
  // before the updates (the factor entry a(i, j) is loaded once per pass)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  auto sweep = [&](int j, int i0, int i1) {
    for (int c0 = wid; c0 < q; c0 += 4 * nw) {
      double xj[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = c0 + u * nw;
        xj[u] = c < q ? b[IX(j, c, ldb)] : 0.0;
      }
      for (int i = i0 + lane; i < i1; i += 32) {
        const double aij = a[IX(i, j, ld)];
        double bv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = c0 + u * nw;
          bv[u] = c < q ? b[IX(i, c, ldb)] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = c0 + u * nw;
          if (c < q && xj[u] != 0.0) b[IX(i, c, ldb)] = __fma_rn(-xj[u], aij, bv[u]);
        }
      }
    }
  };
  for (int j = 0; j < p - 1; ++j) {
    sweep(j, j + 1, p);
    __syncthreads();
  }
  for (int j = p - 1; j >= 0; --j) {
    for (int c = threadIdx.x; c < q; c += blockDim.x)
      if (b[IX(j, c, ldb)] != 0.0) b[IX(j, c, ldb)] = b[IX(j, c, ldb)] / a[IX(j, j, ld)];
    __syncthreads();
    if (j == 0) break;
    sweep(j, 0, j);
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Householder QR of a (r x c, r >= c) in place: R in the upper triangle,
// reflectors below (implicit unit), tau[c].  dlarfg convention.
// ---------------------------------------------------------------------------
static __device__ __noinline__ void blk_geqrf(double* a, int ld, int r, int c, double* tau) {
  __shared__ double s_red[33];
  __shared__ double s_beta, s_tau, s_scal;
  for (int j = 0; j < c; ++j) {
    double ss = 0.0;
    for (int i = j + 1 + threadIdx.x; i < r; i += blockDim.x) {
      double v = a[IX(i, j, ld)];
      ss = __fma_rn(v, v, ss);
    }
    double vv[1] = {ss};
    block_sum<double, 1>(vv, s_red);
    if (threadIdx.x == 0) {
      double alpha = a[IX(j, j, ld)];
      double xnorm = sqrt(vv[0]);
      if (xnorm == 0.0) {
        s_tau = 0.0;
        s_beta = alpha;
        s_scal = 1.0;
      } else {
        double beta = -copysign(hypot(alpha, xnorm), alpha);
        s_tau = (beta - alpha) / beta;
        s_scal = 1.0 / (alpha - beta);
        s_beta = beta;
      }
      tau[j] = s_tau;
    }
    __syncthreads();
    const double tj = s_tau, scal = s_scal;
    if (tj != 0.0)
      for (int i = j + 1 + threadIdx.x; i < r; i += blockDim.x) a[IX(i, j, ld)] *= scal;
    __syncthreads();
    if (threadIdx.x == 0) a[IX(j, j, ld)] = s_beta;
    // apply H_j to columns j+1..c-1: one warp per column, lanes down the rows
    if (tj != 0.0) {
      const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
      for (int l = j + 1 + wid; l < c; l += nw) {
        double wv = 0.0;
        for (int i = j + 1 + lane; i < r; i += 32) wv = __fma_rn(a[IX(i, j, ld)], a[IX(i, l, ld)], wv);
        wv = (warp_sum(wv) + a[IX(j, l, ld)]) * tj;
        __syncwarp();
        if (lane == 0) a[IX(j, l, ld)] -= wv;
        for (int i = j + 1 + lane; i < r; i += 32) a[IX(i, l, ld)] = __fma_rn(-wv, a[IX(i, j, ld)], a[IX(i, l, ld)]);
      }
    }
    __syncthreads();
  }
}

// explicit Q (r x c) from blk_geqrf output (dorg2r)
static __device__ __noinline__ void blk_orgqr(const double* a, int ld, int r, int c, const double* tau, double* q,
                                 int ldq) {
  for (int e = threadIdx.x; e < r * c; e += blockDim.x) {
    int i = e % r, j = e / r;
    q[IX(i, j, ldq)] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int j = c - 1; j >= 0; --j) {
    const double tj = tau[j];
    if (tj != 0.0)
      for (int l = j + threadIdx.x; l < c; l += blockDim.x) {
        double wv = q[IX(j, l, ldq)];
        for (int i = j + 1; i < r; ++i) wv = __fma_rn(a[IX(i, j, ld)], q[IX(i, l, ldq)], wv);
        wv *= tj;
        q[IX(j, l, ldq)] -= wv;
        for (int i = j + 1; i < r; ++i) q[IX(i, l, ldq)] = __fma_rn(-wv, a[IX(i, j, ld)], q[IX(i, l, ldq)]);
      }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// qr_reduced (densela.py:410-432): Q, R with diag(R) >= 0; returns false when
// rank deficient (|R_ii| < max(r,c) * 2^-53 * ||R||_F) or non-finite.
// `a` is destroyed; q (r x c, ldq), rr (c x c, ldr).
// ---------------------------------------------------------------------------
static __device__ __noinline__ bool blk_qr_signed(double* a, int ld, int r, int c, double* q, int ldq, double* rr,
                                     int ldr, double* tau) {
  __shared__ int s_bad;
  __shared__ double s_red[33];
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  for (int e = threadIdx.x; e < r * c; e += blockDim.x) {
    double v = a[IX(e % r, e / r, ld)];
    if (!isfinite(v)) s_bad = 1;
  }
  __syncthreads();
  if (s_bad) return false;
  blk_geqrf(a, ld, r, c, tau);
  blk_orgqr(a, ld, r, c, tau, q, ldq);
  // sign fix and Frobenius norm
  double fro = 0.0;
  for (int e = threadIdx.x; e < c * c; e += blockDim.x) {
    int i = e % c, j = e / c;
    double v = (i <= j) ? a[IX(i, j, ld)] : 0.0;
    double s = a[IX(i, i, ld)] < 0.0 ? -1.0 : 1.0;
    rr[IX(i, j, ldr)] = v * s;
    fro = __fma_rn(v, v, fro);
  }
  double ff[1] = {fro};
  block_sum<double, 1>(ff, s_red);
  for (int e = threadIdx.x; e < r * c; e += blockDim.x) {
    int j = e / r;
    if (a[IX(j, j, ld)] < 0.0) q[IX(e % r, j, ldq)] = -q[IX(e % r, j, ldq)];
  }
  __syncthreads();
  const double tol = (double)max(r, c) * kEps53 * sqrt(ff[0]);
  bool ok = true;
  for (int i = 0; i < c; ++i)
    if (fabs(rr[IX(i, i, ldr)]) < tol) ok = false;
  __syncthreads();
  return ok;
}

// y = R^-1 g for upper-triangular R (c x c, ld), zero-diagonal entries give 0
// (the reference falls back to lstsq there; gmres.py:117-120).
static __device__ __noinline__ void blk_upper_solve(const double* rmat, int ld, int c, const double* g, double* y) {
  // warp 0: lanes sum the solved part of row i, one warp reduction per row
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int i = c - 1; i >= 0; --i) {
      double s = 0.0;
      for (int j = i + 1 + lane; j < c; j += 32) s = __fma_rn(-rmat[IX(i, j, ld)], y[j], s);
      s = warp_sum(s) + g[i];
      const double d = rmat[IX(i, i, ld)];
      if (lane == 0) y[i] = d != 0.0 ? s / d : 0.0;
      __syncwarp();
    }
  }
  __syncthreads();
}

// least squares min ||G y - rhs|| via Householder QR (gcrodr.py:212-218).
// g (r x c) destroyed.  y[c].
static __device__ __noinline__ void blk_lstsq(double* g, int ld, int r, int c, const double* rhs, double* y,
                                 double* tau, double* tmp) {
  blk_geqrf(g, ld, r, c, tau);
  // tmp = Q^T rhs (apply reflectors in order)
  for (int i = threadIdx.x; i < r; i += blockDim.x) tmp[i] = rhs[i];
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int j = 0; j < c; ++j) {
      const double tj = tau[j];
      if (tj == 0.0) continue;
      double wv = 0.0;
      for (int i = j + 1 + lane; i < r; i += 32) wv = __fma_rn(g[IX(i, j, ld)], tmp[i], wv);
      wv = (warp_sum(wv) + tmp[j]) * tj;
      __syncwarp();
      if (lane == 0) tmp[j] -= wv;
      for (int i = j + 1 + lane; i < r; i += 32) tmp[i] = __fma_rn(-wv, g[IX(i, j, ld)], tmp[i]);
      __syncwarp();
    }
  }
  __syncthreads();
  blk_upper_solve(g, ld, c, tmp, y);
}

// ---------------------------------------------------------------------------
// 2-norm condition number (np.linalg.cond): sigma_max / sigma_min
// b (p x p) destroyed.
// ---------------------------------------------------------------------------
__device__ inline double tgk_count(const double* bd, int len, double x) {
  // eigenvalues < x of the zero-diagonal tridiagonal with off-diagonal bd
  const double pivmin = 1e-300;
  double q = -x;
  int cnt = q < 0.0;
  for (int t = 0; t < len; ++t) {
    if (fabs(q) < pivmin) q = -pivmin;
    q = -x - (bd[t] * bd[t]) / q;
    cnt += q < 0.0;
  }
  return (double)cnt;
}

static __device__ __noinline__ double blk_cond2(double* b, int ld, int p, double* bd /* 2p */, double* tmp) {
  __shared__ double s_red[33];
  __shared__ double s_tau, s_beta, s_scal;
  if (p == 1) {
    double v = fabs(b[0]);
    return v == 0.0 ? INFINITY : 1.0;
  }
  // Golub-Kahan bidiagonalisation
  for (int i = 0; i < p; ++i) {
    // left reflector on column i, rows i..p-1
    double ss = 0.0;
    for (int r = i + 1 + threadIdx.x; r < p; r += blockDim.x) ss = __fma_rn(b[IX(r, i, ld)], b[IX(r, i, ld)], ss);
    double vv[1] = {ss};
    block_sum<double, 1>(vv, s_red);
    if (threadIdx.x == 0) {
      double alpha = b[IX(i, i, ld)], xn = sqrt(vv[0]);
      if (xn == 0.0) {
        s_tau = 0.0;
        s_beta = alpha;
        s_scal = 1.0;
      } else {
        double beta = -copysign(hypot(alpha, xn), alpha);
        s_tau = (beta - alpha) / beta;
        s_scal = 1.0 / (alpha - beta);
        s_beta = beta;
      }
    }
    __syncthreads();
    double tj = s_tau;
    if (tj != 0.0) {
      for (int r = i + 1 + threadIdx.x; r < p; r += blockDim.x) b[IX(r, i, ld)] *= s_scal;
      __syncthreads();
      for (int l = i + 1 + threadIdx.x; l < p; l += blockDim.x) {
        double wv = b[IX(i, l, ld)];
        for (int r = i + 1; r < p; ++r) wv = __fma_rn(b[IX(r, i, ld)], b[IX(r, l, ld)], wv);
        wv *= tj;
        b[IX(i, l, ld)] -= wv;
        // loads in batches ahead of the stores (the matrix may live in global memory)
        for (int r0 = i + 1; r0 < p; r0 += 8) {
          double x[8], y[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            x[u] = r0 + u < p ? b[IX(r0 + u, i, ld)] : 0.0;
            y[u] = r0 + u < p ? b[IX(r0 + u, l, ld)] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (r0 + u < p) b[IX(r0 + u, l, ld)] = __fma_rn(-wv, x[u], y[u]);
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) bd[2 * i] = s_beta;
    __syncthreads();
    if (i >= p - 1) break;
    // right reflector on row i, columns i+1..p-1
    ss = 0.0;
    for (int c = i + 2 + threadIdx.x; c < p; c += blockDim.x) ss = __fma_rn(b[IX(i, c, ld)], b[IX(i, c, ld)], ss);
    vv[0] = ss;
    block_sum<double, 1>(vv, s_red);
    if (threadIdx.x == 0) {
      double alpha = b[IX(i, i + 1, ld)], xn = sqrt(vv[0]);
      if (xn == 0.0) {
        s_tau = 0.0;
        s_beta = alpha;
        s_scal = 1.0;
      } else {
        double beta = -copysign(hypot(alpha, xn), alpha);
        s_tau = (beta - alpha) / beta;
        s_scal = 1.0 / (alpha - beta);
        s_beta = beta;
      }
    }
    __syncthreads();
    tj = s_tau;
    if (tj != 0.0) {
      for (int c = i + 2 + threadIdx.x; c < p; c += blockDim.x) b[IX(i, c, ld)] *= s_scal;
      __syncthreads();
      for (int r = i + 1 + threadIdx.x; r < p; r += blockDim.x) {
        double wv = b[IX(r, i + 1, ld)];
        for (int c = i + 2; c < p; ++c) wv = __fma_rn(b[IX(i, c, ld)], b[IX(r, c, ld)], wv);
        wv *= tj;
        b[IX(r, i + 1, ld)] -= wv;
        for (int c0 = i + 2; c0 < p; c0 += 8) {
          double x[8], y[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            x[u] = c0 + u < p ? b[IX(i, c0 + u, ld)] : 0.0;
            y[u] = c0 + u < p ? b[IX(r, c0 + u, ld)] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (c0 + u < p) b[IX(r, c0 + u, ld)] = __fma_rn(-wv, x[u], y[u]);
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) bd[2 * i + 1] = s_beta;
    __syncthreads();
  }
  __shared__ double s_res[2];
  const int len = 2 * p - 1;
  // multisection on the ordered bit patterns of positive doubles: warp 0
  // finds sigma_max, warp 1 sigma_min; each round the 32 lanes evaluate 32
  // interior points (5 bits per round instead of 1 for plain bisection)
  if (threadIdx.x < 64) {
    const int lane = threadIdx.x & 31, wsel = threadIdx.x >> 5;
    double bnd = 0.0;
    for (int t = 0; t < len; ++t) {
      const double l = t > 0 ? fabs(bd[t - 1]) : 0.0;
      bnd = fmax(bnd, l + fabs(bd[t]));
    }
    bnd = fmax(bnd, fabs(bd[len - 1]));
    bnd = bnd * (1.0 + 4.0 * kEps52) + 1e-300;
    const double target = wsel == 0 ? (double)(2 * p) : (double)(p + 1);
    unsigned long long lo = 0ull, hi = (unsigned long long)__double_as_longlong(bnd);
    bool singular = false;
    if (wsel == 1) singular = tgk_count(bd, len, __longlong_as_double(1ll)) >= target;
    if (singular) {
      hi = 0ull;
    } else {
      while (hi - lo > 1) {
        const unsigned long long span = hi - lo;
        const unsigned long long step = span / 33 > 0 ? span / 33 : 1;
        unsigned long long mid = lo + step * (unsigned long long)(lane + 1);
        if (mid >= hi) mid = hi - 1;
        const bool ok = tgk_count(bd, len, __longlong_as_double((long long)mid)) >= target;
        const unsigned mask = __ballot_sync(0xffffffffu, ok);
        if (mask == 0u) {
          lo = __shfl_sync(0xffffffffu, mid, 31);
        } else {
          const int f = __ffs(mask) - 1;
          const unsigned long long mf = __shfl_sync(0xffffffffu, mid, f);
          const unsigned long long mp = f > 0 ? __shfl_sync(0xffffffffu, mid, f - 1) : lo;
          hi = mf;
          lo = f > 0 ? mp : lo;
        }
      }
    }
    if (lane == 0) s_res[wsel] = __longlong_as_double((long long)hi);
  }
  __syncthreads();
  double smax = s_res[0], smin = s_res[1];
  __syncthreads();
  (void)tmp;
  return smin == 0.0 ? INFINITY : smax / smin;
}

// ---------------------------------------------------------------------------
// nonsymmetric eigenproblem (warp 0).  h (p x p) in, overwritten by the real
// Schur form T; z (p x p) Schur vectors; wr, wi eigenvalues in Schur order.
// Returns false on non-convergence.
// ---------------------------------------------------------------------------
// Schur-vector updates handed from the QR warp to a second warp (ring in
// shared memory): type 0 = bulge reflector at column k (x, y, z, q, r),
// type 1 = 2x2 standardisation rotation at (k-1, k) (p, q).  The QR warp's
// dependent chain per bulge step no longer includes the Z update.
struct ZRec {
  double a[5];
  int k, type, notlast;
};
constexpr int kZRing = 64;

// hp != nullptr: the QR iteration runs on a packed shared-memory copy of the
// Hessenberg matrix (column j keeps rows 0 .. j+3: the upper triangle, the
// subdiagonal and the two bulge diagonals, hqr_pack_doubles(p) doubles) and
// the quasi-triangular result is copied back to H -- same operations in the
// same order, only the storage changes (a 200 x 200 problem does not fit the
// scratch as a square and would otherwise pay an L2 round trip per access)
__host__ __device__ inline size_t hqr_pack_doubles(int p) { return (size_t)p * (p + 7) / 2 + 8; }
// Householder reduction to Hessenberg form and the accumulated transformation
// (EISPACK orthes + ortran) by the whole CTA: one thread per column (row) of
// the two-sided update, every element with exactly the operation order of
// the one-warp version inside warp_hqr (so the results are bit-identical);
// the loads of a pass are issued in batches ahead of the stores.  At p = 200
// the one-warp version costs ~85 ms of L2 round trips per eigenproblem.
// ort: p doubles of scratch (global or shared); all threads call.
static __device__ __noinline__ void blk_orthes(double* H, int ld, int p, double* Z, int ldz, double* ort) {
  const int nn = p, low = 0, high = p - 1;
  __shared__ double s_sc[34];
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
  for (int m = low + 1; m <= high - 1; ++m) {
    // scale = sum_i |H(i, m-1)|, hh = sum_i (H(i, m-1) / scale)^2 in the one-warp order (lane-strided partials,
    // butterfly): warp 0 computes them
    if (wid == 0) {
      double scale = 0.0;
      for (int i = m + lane; i <= high; i += 32) scale += fabs(H[IX(i, m - 1, ld)]);
      scale = warp_sum(scale);
      double hh = 0.0;
      if (scale != 0.0) {
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
        if (lane == 0) {
          ort[m] = om - g;
          s_sc[2] = g;
        }
      }
      if (lane == 0) {
        s_sc[0] = scale;
        s_sc[1] = hh;
      }
    }
    __syncthreads();
    const double scale = s_sc[0], hh = s_sc[1];
    if (scale == 0.0) {
      __syncthreads();
      continue;
    }
    // columns j >= m: H(m.., j) -= f ort, f = (sum_{i = high..m} ort_i H(i, j)) / hh
    for (int j = m + tid; j < nn; j += nt) {
      double f = 0.0;
      for (int i = high; i >= m; --i) f = __fma_rn(ort[i], H[IX(i, j, ld)], f);
      f = f / hh;
      for (int i0 = m; i0 <= high; i0 += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = i0 + u <= high ? H[IX(i0 + u, j, ld)] : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (i0 + u <= high) H[IX(i0 + u, j, ld)] = __fma_rn(-f, ort[i0 + u], v[u]);
      }
    }
    __syncthreads();
    // rows i: H(i, m..) -= f ort^T, f = (sum_{j = high..m} ort_j H(i, j)) / hh
    for (int i = tid; i <= high; i += nt) {
      double f = 0.0;
      for (int j = high; j >= m; --j) f = __fma_rn(ort[j], H[IX(i, j, ld)], f);
      f = f / hh;
      for (int j0 = m; j0 <= high; j0 += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = j0 + u <= high ? H[IX(i, j0 + u, ld)] : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (j0 + u <= high) H[IX(i, j0 + u, ld)] = __fma_rn(-f, ort[j0 + u], v[u]);
      }
    }
    __syncthreads();
    if (tid == 0) {
      ort[m] = scale * ort[m];
      H[IX(m, m - 1, ld)] = scale * s_sc[2];
    }
    __syncthreads();
  }
  for (int e = tid; e < nn * nn; e += nt) Z[IX(e % nn, e / nn, ldz)] = (e % nn == e / nn) ? 1.0 : 0.0;
  __syncthreads();
  for (int m = high - 1; m >= low + 1; --m) {
    const double hm = H[IX(m, m - 1, ld)];
    if (hm == 0.0) continue;  // uniform: every thread reads the same entry
    for (int i = m + 1 + tid; i <= high; i += nt) ort[i] = H[IX(i, m - 1, ld)];
    __syncthreads();
    for (int j = m + tid; j <= high; j += nt) {
      double g = 0.0;
      for (int i = m; i <= high; ++i) g = __fma_rn(ort[i], Z[IX(i, j, ldz)], g);
      g = (g / ort[m]) / hm;
      for (int i0 = m; i0 <= high; i0 += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = i0 + u <= high ? Z[IX(i0 + u, j, ldz)] : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (i0 + u <= high) Z[IX(i0 + u, j, ldz)] = __fma_rn(g, ort[i0 + u], v[u]);
      }
    }
    __syncthreads();
  }
  // clear below the subdiagonal
  for (int e = tid; e < nn * nn; e += nt) {
    int i = e % nn, j = e / nn;
    if (i > j + 1) H[IX(i, j, ld)] = 0.0;
  }
  __syncthreads();
}

// number of Schur-vector warps warp_hqr wants next to the QR warp
__host__ __device__ inline int hqr_z_warps(int p, int nwarps_cta, int nq = 1) {
  const int want = (p + 31) / 32;
  const int have = nwarps_cta - nq;
  return want < 1 ? 1 : (want < have ? want : have);
}
struct ZShared {
  ZRec ring[kZRing];
  volatile int head, done;
  volatile int tail[8];
};
static __device__ __noinline__ ZShared& zshared() {
  __shared__ ZShared z;
  return z;
}
template <bool kPacked>
static __device__ __noinline__ bool warp_hqr_t(double* H, int ld, int p, double* Z, int ldz, double* wr, double* wi,
                                  double* ort, double* hp, int nz, bool reduced, int nq) {
  // called by threads 0 .. 32 (1 + nz) - 1: warp 0 runs orthes + the QR
  // iteration, warps 1 .. nz apply the Schur-vector updates it pushes.  Z
  // warp w owns the rows i = w - 1 + nz * t (t = 0, 1, ...) strided by lane:
  // rows are independent, the records are applied in order per row.  Inside
  // a sweep the reflectors walk down the diagonal (k, k + 1, ...), so a lane
  // keeps Z(i, k .. k+2) of its row in registers, shifts them by one column
  // per record (one store, one load issued a record ahead) and only falls
  // back to plain loads when the sweep restarts.
  ZShared& zs = zshared();  // one instance for both storage variants
  ZRec* const zring = zs.ring;
  volatile int& s_head = zs.head;
  volatile int& s_done = zs.done;
  volatile int* const s_tail = zs.tail;
  const int lane = threadIdx.x & 31;
  const int low_ = 0, high_ = p - 1;
  // nq QR warps (1, or 4 for the large eigenproblems: the row / column updates of a bulge
  // step are split over 128 threads, every thread keeps the scalars redundantly and the
  // warps meet at a named barrier wherever the one-warp version has a __syncwarp)
  const int zbar = 32 * (nq + nz);
  const int qt = threadIdx.x, qn = 32 * nq;
  auto qsync = [&]() {
    if (nq == 1) __syncwarp();
    else asm volatile("bar.sync 3, %0;" ::"r"(qn) : "memory");
  };
  if ((int)(threadIdx.x >> 5) >= nq) {
    const int zw = (threadIdx.x >> 5) - nq;
    asm volatile("bar.sync 1, %0;" ::"r"(zbar) : "memory");  // Z initialised, ring reset
    int tail = 0;
    const int rows_per_pass = 32 * nz;
    for (;;) {
      const int head = s_head;
      if (tail == head) {
        if (s_done && tail == s_head) break;
        continue;
      }
      __threadfence_block();
      for (; tail < head; ++tail) {
        const volatile ZRec& R = zring[tail % kZRing];
        const int k = R.k, type = R.type, nl = R.notlast;
        const double a0 = R.a[0], a1 = R.a[1], a2 = R.a[2], a3 = R.a[3], a4 = R.a[4];
        if (type == 0) {
          for (int i = low_ + zw * 32 + lane; i <= high_; i += rows_per_pass) {
            // the next reflector of the sweep touches column k + 3
            if (k + 3 <= high_) asm volatile("prefetch.global.L1 [%0];" ::"l"(Z + IX(i, k + 3, ldz)));
            double pp = a0 * Z[IX(i, k, ldz)] + a1 * Z[IX(i, k + 1, ldz)];
            if (nl) {
              pp = pp + a2 * Z[IX(i, k + 2, ldz)];
              Z[IX(i, k + 2, ldz)] = Z[IX(i, k + 2, ldz)] - pp * a4;
            }
            Z[IX(i, k, ldz)] = Z[IX(i, k, ldz)] - pp;
            Z[IX(i, k + 1, ldz)] = Z[IX(i, k + 1, ldz)] - pp * a3;
          }
        } else {
          for (int i = low_ + zw * 32 + lane; i <= high_; i += rows_per_pass) {
            double zz = Z[IX(i, k - 1, ldz)];
            Z[IX(i, k - 1, ldz)] = a3 * zz + a0 * Z[IX(i, k, ldz)];
            Z[IX(i, k, ldz)] = a3 * Z[IX(i, k, ldz)] - a0 * zz;
          }
        }
      }
      __syncwarp();
      if (lane == 0) s_tail[zw] = tail;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(zbar) : "memory");
    return true;
  }
  // producer side: lane 0 appends records and publishes the head every
  // kZPub records (one fence per batch); ring space is re-checked only when
  // the cached tail says the ring may be full
  constexpr int kZPub = 8;
  int zh = 0, zt = 0;  // lane 0's local head and cached tail
  auto zpublish = [&]() {
    __threadfence_block();
    s_head = zh;
  };
  auto zpush = [&](int type, int k, int nl, double a0, double a1, double a2, double a3, double a4) {
    if (qt == 0) {
      if (zh - zt >= kZRing) {
        zpublish();
        for (;;) {
          int mn = s_tail[0];
          for (int w = 1; w < nz; ++w) mn = min(mn, s_tail[w]);
          zt = mn;
          if (zh - zt < kZRing) break;
        }
      }
      ZRec& R = zring[zh % kZRing];
      R.a[0] = a0;
      R.a[1] = a1;
      R.a[2] = a2;
      R.a[3] = a3;
      R.a[4] = a4;
      R.k = k;
      R.type = type;
      R.notlast = nl;
      ++zh;
      if (zh % kZPub == 0) zpublish();
    }
  };
  auto zfinish = [&]() {
    if (qt == 0) {
      zpublish();
      __threadfence_block();
      s_done = 1;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(zbar) : "memory");  // the Z warps drained the ring
  };
  const int nn = p, low = 0, high = p - 1;
  // --- orthes: Householder reduction to Hessenberg form (skipped when the
  // CTA has already run blk_orthes) ---
  for (int m = low + 1; !reduced && m <= high - 1; ++m) {
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
  for (int e = lane; !reduced && e < nn * nn; e += 32) Z[IX(e % nn, e / nn, ldz)] = (e % nn == e / nn) ? 1.0 : 0.0;
  __syncwarp();
  for (int m = high - 1; !reduced && m >= low + 1; --m) {
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
  if (qt == 0) {
    s_head = 0;
    for (int w = 0; w < 8; ++w) s_tail[w] = 0;
    s_done = 0;
  }
  qsync();
  asm volatile("bar.sync 1, %0;" ::"r"(zbar) : "memory");  // start the Z warps

  constexpr bool packed = kPacked;  // compile-time: the accessor sits in the hottest loop of cfg2
  double* const hbase = packed ? hp : H;
  auto HH = [&](int i, int j) -> double& { return hbase[(packed ? ((j * (j + 7)) >> 1) : j * ld) + i]; };
  if (packed) {
    for (int e = qt; e < p * p; e += qn) {
      const int i = e % p, j = e / p;
      if (i <= j + 3) HH(i, j) = H[IX(i, j, ld)];
    }
    qsync();
  }
  // --- hqr2: Francis double-shift QR with accumulation ---
  int n = nn - 1;
  const double eps = kEps52;
  double exshift = 0.0, p_ = 0, q = 0, r = 0, s = 0, z = 0, t, w, x, y;
  double norm = 0.0;
  for (int i = lane; i < nn; i += 32)  // every QR warp sums the whole matrix (same order, same value)
    for (int j = max(i - 1, 0); j < nn; ++j) norm += fabs(HH(i, j));
  norm = warp_sum(norm);
  int iter = 0, total = 0;
  const int itmax = 40 * max(10, nn);
  while (n >= low) {
    // small-subdiagonal search (the first l from n downwards with a
    // negligible H(l, l-1)), 32 candidates per ballot instead of a serial scan
    int l = low;
    for (int base = n; base > low; base -= 32) {
      const int cand = base - lane;
      bool hit = false;
      if (cand > low) {
        double sc = fabs(HH(cand - 1, cand - 1)) + fabs(HH(cand, cand));
        if (sc == 0.0) sc = norm;
        hit = fabs(HH(cand, cand - 1)) < eps * sc;
      }
      const unsigned bm = __ballot_sync(0xffffffffu, hit);
      if (bm) {
        l = base - (__ffs(bm) - 1);
        break;
      }
    }
    if (l == n) {
      qsync();
      if (qt == 0) {
        HH(n, n) = HH(n, n) + exshift;
        wr[n] = HH(n, n);
        wi[n] = 0.0;
      }
      qsync();
      n--;
      iter = 0;
    } else if (l == n - 1) {
      w = HH(n, n - 1) * HH(n - 1, n);
      p_ = (HH(n - 1, n - 1) - HH(n, n)) / 2.0;
      q = p_ * p_ + w;
      z = sqrt(fabs(q));
      double hnn = HH(n, n) + exshift;
      double hn1 = HH(n - 1, n - 1) + exshift;
      qsync();
      if (qt == 0) {
        HH(n, n) = hnn;
        HH(n - 1, n - 1) = hn1;
      }
      qsync();
      x = hnn;
      if (q >= 0) {
        z = (p_ >= 0) ? p_ + z : p_ - z;
        double d1 = x + z, d2 = d1;
        if (z != 0.0) d2 = x - w / z;
        if (qt == 0) {
          wr[n - 1] = d1;
          wr[n] = d2;
          wi[n - 1] = 0.0;
          wi[n] = 0.0;
        }
        x = HH(n, n - 1);
        s = fabs(x) + fabs(z);
        p_ = x / s;
        q = z / s;
        r = sqrt(p_ * p_ + q * q);
        p_ = p_ / r;
        q = q / r;
        qsync();
        for (int j = n - 1 + qt; j < nn; j += qn) {
          double zz = HH(n - 1, j);
          HH(n - 1, j) = q * zz + p_ * HH(n, j);
          HH(n, j) = q * HH(n, j) - p_ * zz;
        }
        qsync();
        for (int i = qt; i <= n; i += qn) {
          double zz = HH(i, n - 1);
          HH(i, n - 1) = q * zz + p_ * HH(i, n);
          HH(i, n) = q * HH(i, n) - p_ * zz;
        }
        zpush(1, n, 0, p_, 0.0, 0.0, q, 0.0);
        qsync();
      } else {
        if (qt == 0) {
          wr[n - 1] = x + p_;
          wr[n] = x + p_;
          wi[n - 1] = z;
          wi[n] = -z;
        }
        qsync();
      }
      n = n - 2;
      iter = 0;
    } else {
      x = HH(n, n);
      y = 0.0;
      w = 0.0;
      if (l < n) {
        y = HH(n - 1, n - 1);
        w = HH(n, n - 1) * HH(n - 1, n);
      }
      if (iter == 10) {
        exshift += x;
        qsync();
        for (int i = low + qt; i <= n; i += qn) HH(i, i) -= x;
        qsync();
        s = fabs(HH(n, n - 1)) + fabs(HH(n - 1, n - 2));
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
          qsync();
          for (int i = low + qt; i <= n; i += qn) HH(i, i) -= s;
          qsync();
          exshift += s;
          x = y = w = 0.964;
        }
      }
      iter++;
      if (++total > itmax) {
        zfinish();
        return false;
      }
      // start of the double-shift sweep: the first m from n-2 downwards with
      // two consecutive small subdiagonals (m = l always qualifies); 32
      // candidates per ballot, then the chosen m's start vector is recomputed
      // with exactly the operations of the serial EISPACK loop
      int m = l;
      for (int base = n - 2; base > l; base -= 32) {
        const int mm = base - lane;
        bool hit = false;
        if (mm > l) {
          const double zz = HH(mm, mm);
          const double rr = x - zz, ss = y - zz;
          double pp = (rr * ss - w) / HH(mm + 1, mm) + HH(mm, mm + 1);
          double qq = HH(mm + 1, mm + 1) - zz - rr - ss;
          double r3 = HH(mm + 2, mm + 1);
          const double s3 = fabs(pp) + fabs(qq) + fabs(r3);
          pp = pp / s3;
          qq = qq / s3;
          r3 = r3 / s3;
          hit = fabs(HH(mm, mm - 1)) * (fabs(qq) + fabs(r3)) <
                eps * (fabs(pp) * (fabs(HH(mm - 1, mm - 1)) + fabs(zz) + fabs(HH(mm + 1, mm + 1))));
        }
        const unsigned bm = __ballot_sync(0xffffffffu, hit);
        if (bm) {
          m = base - (__ffs(bm) - 1);
          break;
        }
      }
      z = HH(m, m);
      r = x - z;
      s = y - z;
      p_ = (r * s - w) / HH(m + 1, m) + HH(m, m + 1);
      q = HH(m + 1, m + 1) - z - r - s;
      r = HH(m + 2, m + 1);
      s = fabs(p_) + fabs(q) + fabs(r);
      p_ = p_ / s;
      q = q / s;
      r = r / s;
      qsync();
      for (int i = m + 2 + qt; i <= n; i += qn) {
        HH(i, i - 2) = 0.0;
        if (i > m + 2) HH(i, i - 3) = 0.0;
      }
      qsync();
      for (int k = m; k <= n - 1; ++k) {
        bool notlast = (k != n - 1);
        if (k != m) {
          p_ = HH(k, k - 1);
          q = HH(k + 1, k - 1);
          r = notlast ? HH(k + 2, k - 1) : 0.0;
          x = fabs(p_) + fabs(q) + fabs(r);
          if (x == 0.0) continue;
          const double rx = 1.0 / x;  // one division instead of three
          p_ = p_ * rx;
          q = q * rx;
          r = r * rx;
        }
        s = sqrt(p_ * p_ + q * q + r * r);
        if (p_ < 0) s = -s;
        if (s != 0) {
          qsync();
          if (qt == 0) {
            if (k != m) HH(k, k - 1) = -s * x;
            else if (l != m) HH(k, k - 1) = -HH(k, k - 1);
          }
          qsync();
          p_ = p_ + s;
          const double rs = 1.0 / s, rp = 1.0 / p_;
          x = p_ * rs;
          y = q * rs;
          z = r * rs;
          q = q * rp;
          r = r * rp;
          for (int j = k + qt; j < nn; j += qn) {
            double pp = HH(k, j) + q * HH(k + 1, j);
            if (notlast) {
              pp = pp + r * HH(k + 2, j);
              HH(k + 2, j) = HH(k + 2, j) - pp * z;
            }
            HH(k, j) = HH(k, j) - pp * x;
            HH(k + 1, j) = HH(k + 1, j) - pp * y;
          }
          qsync();
          const int iend = min(n, k + 3);
          for (int i = qt; i <= iend; i += qn) {
            double pp = x * HH(i, k) + y * HH(i, k + 1);
            if (notlast) {
              pp = pp + z * HH(i, k + 2);
              HH(i, k + 2) = HH(i, k + 2) - pp * r;
            }
            HH(i, k) = HH(i, k) - pp;
            HH(i, k + 1) = HH(i, k + 1) - pp * q;
          }
          zpush(0, k, notlast ? 1 : 0, x, y, z, q, r);
          qsync();  // column update visible to the next step's scalars
        }
      }
    }
  }
  qsync();
  if (packed) {
    for (int e = qt; e < p * p; e += qn) {
      const int i = e % p, j = e / p;
      if (i <= j + 1) H[IX(i, j, ld)] = HH(i, j);
    }
    qsync();
  }
  zfinish();
  return true;
}

static __device__ __forceinline__ bool warp_hqr(double* H, int ld, int p, double* Z, int ldz, double* wr, double* wi,
                                               double* ort, double* hp = nullptr, int nz = 1, bool reduced = false,
                                               int nq = 1) {
  return hp != nullptr ? warp_hqr_t<true>(H, ld, p, Z, ldz, wr, wi, ort, hp, nz, reduced, nq)
                       : warp_hqr_t<false>(H, ld, p, Z, ldz, wr, wi, ort, hp, nz, reduced, nq);
}

GB_DEVICE void cdiv(double xr, double xi, double yr, double yi, double& cr, double& ci) {
  double rr, d;
  if (fabs(yr) > fabs(yi)) {
    rr = yi / yr;
    d = yr + rr * yi;
    cr = (xr + rr * xi) / d;
    ci = (xi - rr * xr) / d;
  } else {
    rr = yr / yi;
    d = yi + rr * yr;
    cr = (rr * xr + xi) / d;
    ci = (rr * xi - xr) / d;
  }
}

// Eigenvector(s) for Schur position `col` (real: one vector; complex pair
// (col, col+1) with wi[col] > 0: re/im), computed by ONE thread.  T is the
// final quasi-triangular matrix, X a p x 2 scratch (ldx), out_re/out_im length
// p vectors in the original basis (Z X), normalised like LAPACK dgeev.
static __device__ __noinline__ void eigvec_one(const double* T, int ld, int p, const double* Z, int ldz,
                                  const double* wr, const double* wi, double normT, int col, double* X,
                                  int ldx, double* out_re, double* out_im) {
  const double eps = kEps52;
  const bool cplx = wi[col] != 0.0;
  double* xr = X;        // column n-1 (real part) for complex, the vector for real
  double* xi = X + ldx;  // column n   (imag part)
  if (!cplx) {
    const int n = col;
    const double pp = wr[n];
    for (int i = 0; i < p; ++i) xr[i] = 0.0;
    xr[n] = 1.0;
    int l = n;
    double z = 0, s = 0;
    for (int i = n - 1; i >= 0; --i) {
      double w = T[IX(i, i, ld)] - pp;
      double r = 0.0;
      for (int j = l; j <= n; ++j) r += T[IX(i, j, ld)] * xr[j];
      if (wi[i] < 0.0) {
        z = w;
        s = r;
      } else {
        l = i;
        if (wi[i] == 0.0) {
          xr[i] = (w != 0.0) ? -r / w : -r / (eps * normT);
        } else {
          double x = T[IX(i, i + 1, ld)], y = T[IX(i + 1, i, ld)];
          double q = (wr[i] - pp) * (wr[i] - pp) + wi[i] * wi[i];
          double t = (x * s - z * r) / q;
          xr[i] = t;
          xr[i + 1] = (fabs(x) > fabs(z)) ? (-r - w * t) / x : (-s - y * t) / z;
        }
        double t = fabs(xr[i]);
        if ((eps * t) * t > 1)
          for (int j = i; j <= n; ++j) xr[j] /= t;
      }
    }
    // back-transform and normalise
    double nrm = 0.0;
    for (int i = 0; i < p; ++i) {
      double v = 0.0;
      for (int k = 0; k <= n; ++k) v += Z[IX(i, k, ldz)] * xr[k];
      out_re[i] = v;
      nrm += v * v;
    }
    nrm = sqrt(nrm);
    double inv = nrm > 0 ? 1.0 / nrm : 1.0;
    for (int i = 0; i < p; ++i) {
      out_re[i] *= inv;
      out_im[i] = 0.0;
    }
    return;
  }
  // complex pair: Schur positions (col, col+1), wi[col] > 0; hqr2 builds it at n = col+1
  const int n = col + 1;
  const double pp = wr[n], q = wi[n];  // q < 0
  for (int i = 0; i < p; ++i) {
    xr[i] = 0.0;
    xi[i] = 0.0;
  }
  int l = n - 1;
  if (fabs(T[IX(n, n - 1, ld)]) > fabs(T[IX(n - 1, n, ld)])) {
    xr[n - 1] = q / T[IX(n, n - 1, ld)];
    xi[n - 1] = -(T[IX(n, n, ld)] - pp) / T[IX(n, n - 1, ld)];
  } else {
    double cr, ci;
    cdiv(0.0, -T[IX(n - 1, n, ld)], T[IX(n - 1, n - 1, ld)] - pp, q, cr, ci);
    xr[n - 1] = cr;
    xi[n - 1] = ci;
  }
  xr[n] = 0.0;
  xi[n] = 1.0;
  double z = 0, r = 0, s = 0;
  for (int i = n - 2; i >= 0; --i) {
    double ra = 0.0, sa = 0.0;
    for (int j = l; j <= n; ++j) {
      ra += T[IX(i, j, ld)] * xr[j];
      sa += T[IX(i, j, ld)] * xi[j];
    }
    double w = T[IX(i, i, ld)] - pp;
    if (wi[i] < 0.0) {
      z = w;
      r = ra;
      s = sa;
    } else {
      l = i;
      if (wi[i] == 0.0) {
        double cr, ci;
        cdiv(-ra, -sa, w, q, cr, ci);
        xr[i] = cr;
        xi[i] = ci;
      } else {
        double x = T[IX(i, i + 1, ld)], y = T[IX(i + 1, i, ld)];
        double vr = (wr[i] - pp) * (wr[i] - pp) + wi[i] * wi[i] - q * q;
        double vi = (wr[i] - pp) * 2.0 * q;
        if (vr == 0.0 && vi == 0.0)
          vr = eps * normT * (fabs(w) + fabs(q) + fabs(x) + fabs(y) + fabs(z));
        double cr, ci;
        cdiv(x * r - z * ra + q * sa, x * s - z * sa - q * ra, vr, vi, cr, ci);
        xr[i] = cr;
        xi[i] = ci;
        if (fabs(x) > (fabs(z) + fabs(q))) {
          xr[i + 1] = (-ra - w * xr[i] + q * xi[i]) / x;
          xi[i + 1] = (-sa - w * xi[i] - q * xr[i]) / x;
        } else {
          cdiv(-r - y * xr[i], -s - y * xi[i], z, q, cr, ci);
          xr[i + 1] = cr;
          xi[i + 1] = ci;
        }
      }
      double t = fmax(fabs(xr[i]), fabs(xi[i]));
      if ((eps * t) * t > 1)
        for (int j = i; j <= n; ++j) {
          xr[j] /= t;
          xi[j] /= t;
        }
    }
  }
  // back-transform: v = Z x ; re = col n-1, im = col n (eigenvalue wr + i*|wi|)
  double nrm = 0.0;
  for (int i = 0; i < p; ++i) {
    double a = 0.0, b = 0.0;
    for (int k = 0; k <= n; ++k) {
      a += Z[IX(i, k, ldz)] * xr[k];
      b += Z[IX(i, k, ldz)] * xi[k];
    }
    out_re[i] = a;
    out_im[i] = b;
    nrm += a * a + b * b;
  }
  // dgeev: unit 2-norm, then rotate so the largest component is real
  nrm = sqrt(nrm);
  double inv = nrm > 0 ? 1.0 / nrm : 1.0;
  int kmax = 0;
  double best = -1.0;
  for (int i = 0; i < p; ++i) {
    out_re[i] *= inv;
    out_im[i] *= inv;
    double m2 = out_re[i] * out_re[i] + out_im[i] * out_im[i];
    if (m2 > best) {
      best = m2;
      kmax = i;
    }
  }
  double f = out_re[kmax], g = out_im[kmax], cs, sn;
  if (g == 0.0) {
    cs = 1.0;
    sn = 0.0;
  } else if (f == 0.0) {
    cs = 0.0;
    sn = copysign(1.0, g);
  } else {
    double d = sqrt(f * f + g * g);
    cs = fabs(f) / d;
    double rr = copysign(d, f);
    sn = g / rr;
  }
  for (int i = 0; i < p; ++i) {
    double a = out_re[i], b = out_im[i];
    out_re[i] = cs * a + sn * b;
    out_im[i] = cs * b - sn * a;
  }
  out_im[kmax] = 0.0;
}

}  // namespace gb
