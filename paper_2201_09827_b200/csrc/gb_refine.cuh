// One refinement step and its surroundings (reference refine.py):
//   residual in u_r + nbe/cbe      check_convergence  refine.py:172-229
//   x0 = LU substitution in u_f    refine.py:317-321  (+ densela.py:235-261)
//   xref                           _reference_solution refine.py:236-258
//                                  (dd GEPP quad_solve densela.py:368-407 for
//                                   n <= 600, else fp64 LU + 4 dd refinements)
//   the step body                  refine.py:362-394
//   full loop (batched mode only)  refine.py:362-421 incl. the decision rules
#pragma once
#include "gb_krylov.cuh"
#include "gb_lu.cuh"

namespace gb {

enum { UR_F32 = 0, UR_F64 = 1, UR_DD = 2 };

// status bits of a refinement step (beyond the inner-solve bits)
enum : int { RS_NU_ZERO = 256, RS_NU_NONFINITE = 512 };

struct ResidOut {
  double nbe, cbe, xinf, rinf;
};

// r = b - A x accumulated in u_r, cden = |A||x| + |b|; nbe, cbe as in
// check_convergence.  r is written in fp64 (the carrier the reference keeps).
template <class Team, class TA, class TW, class TB>
__device__ ResidOut residual_check(Team& t, const TA* A, size_t lda, int n, const TW* x, const TB* b,
                                   double* r, int ur, double normA, double normB, double* red) {
  int lo, hi;
  t.rows(n, lo, hi);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double rmax = 0.0, cmax = -1.0;
  for (int i = lo + wid; i < hi; i += nw) {
    const TA* ar = A + (size_t)i * lda;
    double ca = 0.0;
    double ri;
    // grid teams (n > 1024): long rows stream from HBM, 8 x 16 B in flight per lane
    constexpr int kU = Team::kTB == kTrsvB ? 8 : 4;
    if (ur == UR_DD) {
      dd acc = row_dot_ex<MODE_DD, true, TA, TW, kU>(ar, x, n, &ca);
      dd rr = dd_add(dd{(double)b[i], 0.0}, dd_neg(acc));
      ri = dd_val(rr);
    } else if (ur == UR_F64) {
      double acc = row_dot_ex<MODE_F64, true, TA, TW, kU>(ar, x, n, &ca);
      ri = __dsub_rn((double)b[i], acc);
    } else {
      float acc = row_dot_ex<MODE_F32, true, TA, TW, kU>(ar, x, n, &ca);
      ri = (double)__fsub_rn((float)b[i], acc);
    }
    const double cd = ca + fabs((double)b[i]);
    if (lane == 0) r[i] = ri;
    rmax = nan_max(rmax, fabs(ri));
    const double ratio = fabs(ri) / cd;
    if (isfinite(ratio)) cmax = fmax(cmax, ratio);
  }
  // block reductions (NaN-propagating for rmax)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    rmax = nan_max(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
    cmax = fmax(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
  }
  __syncthreads();
  if (lane == 0) {
    red[wid] = rmax;
    red[32 + wid] = cmax;
  }
  __syncthreads();
  rmax = lane < nw ? red[lane] : 0.0;
  cmax = lane < nw ? red[32 + lane] : -1.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    rmax = nan_max(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
    cmax = fmax(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
  }
  __syncthreads();
  rmax = t.finish_max(rmax);
  cmax = t.finish_max(cmax);
  const double xinf = team_amax<TW>(t, x, n, red);
  ResidOut o;
  const double denom = normA * xinf + normB;
  o.nbe = denom > 0 ? rmax / denom : INFINITY;
  o.cbe = cmax >= 0.0 ? cmax : o.nbe;
  o.xinf = xinf;
  o.rinf = rmax;
  return o;
}

// forward error ||x - xref||_inf / ||xref||_inf  (refine.py:424-430)
template <class Team, class TW>
__device__ double forward_error(Team& t, const TW* x, const double* xref, int n, double* red) {
  int lo, hi;
  t.rows(n, lo, hi);
  double e = 0.0, d = 0.0;
  for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    e = nan_max(e, fabs((double)x[i] - xref[i]));
    d = nan_max(d, fabs(xref[i]));
  }
  e = block_max(e, red);
  d = block_max(d, red);
  e = t.finish_max(e);
  d = t.finish_max(d);
  return d == 0.0 ? e : e / d;
}

// ---------------------------------------------------------------------------
// double-double GEPP solve by one CTA (quad_solve, densela.py:368-407).
// ah/al: n x n row-major scratch (global), x out.  Returns false on an
// exact zero pivot (the reference returns no reference solution then).
// ---------------------------------------------------------------------------
template <class TA, class TW>
__device__ bool dd_gepp_solve(const TA* A, size_t lda, const TW* b, int n, double* ah, double* al,
                              double* yh, double* yl, int* perm, double* xout, PivKey* pscr) {
  for (size_t e = threadIdx.x; e < (size_t)n * n; e += blockDim.x) {
    ah[e] = (double)A[(e / n) * lda + e % n];
    al[e] = 0.0;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) perm[i] = i;
  __syncthreads();
  __shared__ int s_zero;
  if (threadIdx.x == 0) s_zero = 0;
  for (int k = 0; k < n - 1; ++k) {
    PivKey key{0.0, -1, 0};
    for (int i = k + threadIdx.x; i < n; i += blockDim.x) {
      PivKey c = make_key(ah[(size_t)i * n + k], i);
      if (piv_better(c, key)) key = c;
    }
    key = block_pivot(key, pscr);
    const int p = key.i;
    const bool isz = ah[(size_t)p * n + k] == 0.0 && al[(size_t)p * n + k] == 0.0;
    // all threads have read the pivot before the interchange rewrites row p
    __syncthreads();
    if (isz) {
      if (threadIdx.x == 0) s_zero = 1;
      __syncthreads();
      return false;
    }
    if (p != k) {
      for (int j = threadIdx.x; j < n; j += blockDim.x) {
        double t1 = ah[(size_t)k * n + j];
        ah[(size_t)k * n + j] = ah[(size_t)p * n + j];
        ah[(size_t)p * n + j] = t1;
        t1 = al[(size_t)k * n + j];
        al[(size_t)k * n + j] = al[(size_t)p * n + j];
        al[(size_t)p * n + j] = t1;
      }
      if (threadIdx.x == 0) {
        int t2 = perm[k];
        perm[k] = perm[p];
        perm[p] = t2;
      }
    }
    __syncthreads();
    const dd pv{ah[(size_t)k * n + k], al[(size_t)k * n + k]};
    for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x) {
      dd m = dd_div(dd{ah[(size_t)i * n + k], al[(size_t)i * n + k]}, pv);
      ah[(size_t)i * n + k] = m.hi;
      al[(size_t)i * n + k] = m.lo;
    }
    __syncthreads();
    const int mm = n - k - 1;
    for (int e = threadIdx.x; e < mm * mm; e += blockDim.x) {
      int i = k + 1 + e / mm, j = k + 1 + e % mm;
      dd m{ah[(size_t)i * n + k], al[(size_t)i * n + k]};
      dd u{ah[(size_t)k * n + j], al[(size_t)k * n + j]};
      dd a{ah[(size_t)i * n + j], al[(size_t)i * n + j]};
      dd r = dd_sub(a, dd_mul(m, u));
      ah[(size_t)i * n + j] = r.hi;
      al[(size_t)i * n + j] = r.lo;
    }
    __syncthreads();
  }
  if (ah[(size_t)(n - 1) * n + n - 1] == 0.0 && al[(size_t)(n - 1) * n + n - 1] == 0.0) return false;
  // substitution: column sweeps as in the reference, parallel over rows
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    yh[i] = (double)b[perm[i]];
    yl[i] = 0.0;
  }
  __syncthreads();
  for (int i = 0; i < n - 1; ++i) {
    const dd yi{yh[i], yl[i]};
    for (int r = i + 1 + threadIdx.x; r < n; r += blockDim.x) {
      dd tt = dd_mul(dd{ah[(size_t)r * n + i], al[(size_t)r * n + i]}, yi);
      dd y = dd_sub(dd{yh[r], yl[r]}, tt);
      yh[r] = y.hi;
      yl[r] = y.lo;
    }
    __syncthreads();
  }
  for (int i = n - 1; i >= 0; --i) {
    if (threadIdx.x == 0) {
      dd y = dd_div(dd{yh[i], yl[i]}, dd{ah[(size_t)i * n + i], al[(size_t)i * n + i]});
      yh[i] = y.hi;
      yl[i] = y.lo;
    }
    __syncthreads();
    const dd yi{yh[i], yl[i]};
    for (int r = threadIdx.x; r < i; r += blockDim.x) {
      dd tt = dd_mul(dd{ah[(size_t)r * n + i], al[(size_t)r * n + i]}, yi);
      dd y = dd_sub(dd{yh[r], yl[r]}, tt);
      yh[r] = y.hi;
      yl[r] = y.lo;
    }
    __syncthreads();
  }
  bool fin = true;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double v = __dadd_rn(yh[i], yl[i]);
    xout[i] = v;
  }
  __syncthreads();
  for (int i = 0; i < n; ++i)
    if (!isfinite(xout[i])) fin = false;
  __syncthreads();
  return fin;
}

}  // namespace gb
