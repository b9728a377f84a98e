// Team-distributed operators: residual, preconditioned operator, LU
// substitution and the format-faithful BLAS-1 of the Krylov loop.
//
// Reference semantics (paths relative to /root/reference/pkg/src/irkit):
//   residual(a, x, b, ctx)              densela.py:340-361
//   apply_preconditioned(a, f, v, ...)  densela.py:268-299
//   precond_rhs(f, r, ...)              densela.py:314-333
//   lu_solve / _sub_*                   densela.py:175-261
//   vdot/vnorm2/vscale/vaxpy/mat_tvec   precision.py:513-587
//
// Layout: A is row-major n x n at u width (TA = float for u=single, double for
// u=double); LU is packed row-major at u_f width (TF = __half/float/double);
// perm[i] is the original row of pivot position i.  Rows are processed in
// blocks of 32 (kRB).  In a GridTeam, row block b of the forward solve is owned
// by CTA b % G (backward: (nb-1-b) % G); a monotone 64-bit progress counter
// published with st.release lets later blocks consume earlier ones without a
// grid barrier.  Inside a block each lane owns one row and walks the columns
// in order, so with one warp (exact modes) the per-element operation order is
// exactly the reference's column sweep.
#pragma once
#include "gb_team.cuh"

namespace gb {

constexpr int kRB = 32;  // rows per TRSV / GEMV block

enum Mode { MODE_F32 = 0, MODE_F64 = 1, MODE_DD = 2, MODE_H16 = 3 };

template <class T>
GB_DEVICE double to_d(T x) { return (double)x; }
template <>
GB_DEVICE double to_d<__half>(__half x) { return (double)__half2float(x); }
template <class T>
GB_DEVICE float to_f(T x) { return (float)x; }
template <>
GB_DEVICE float to_f<__half>(__half x) { return __half2float(x); }

// ---------------------------------------------------------------------------
// accumulator arithmetic per operator mode
// ---------------------------------------------------------------------------
template <int M>
struct Arith;

template <>
struct Arith<MODE_F64> {
  using T = double;
  static constexpr bool kExactOrder = false;
  GB_DEVICE static T zero() { return 0.0; }
  GB_DEVICE static T from(double x) { return x; }
  GB_DEVICE static T sub_prod(T acc, double l, T y) { return __fma_rn(-l, y, acc); }
  GB_DEVICE static T mac(T acc, double a, double v) { return __fma_rn(a, v, acc); }
  GB_DEVICE static T add(T a, T b) { return __dadd_rn(a, b); }
  GB_DEVICE static T sub(T a, T b) { return __dsub_rn(a, b); }
  GB_DEVICE static T div(T y, double u) { return __ddiv_rn(y, u); }
  GB_DEVICE static double val(T x) { return x; }
  GB_DEVICE static T shfl(T x, int src) { return __shfl_sync(0xffffffffu, x, src); }
  GB_DEVICE static T ld(const T* p) { return __ldcg(p); }
};

template <>
struct Arith<MODE_F32> {
  using T = float;
  static constexpr bool kExactOrder = false;
  GB_DEVICE static T zero() { return 0.f; }
  GB_DEVICE static T from(double x) { return __double2float_rn(x); }
  GB_DEVICE static T sub_prod(T acc, double l, T y) { return __fmaf_rn(-(float)l, y, acc); }
  GB_DEVICE static T mac(T acc, double a, double v) { return __fmaf_rn((float)a, (float)v, acc); }
  GB_DEVICE static T add(T a, T b) { return __fadd_rn(a, b); }
  GB_DEVICE static T sub(T a, T b) { return __fsub_rn(a, b); }
  GB_DEVICE static T div(T y, double u) { return __fdiv_rn(y, (float)u); }
  GB_DEVICE static double val(T x) { return (double)x; }
  GB_DEVICE static T shfl(T x, int src) { return __shfl_sync(0xffffffffu, x, src); }
  GB_DEVICE static T ld(const T* p) { return __ldcg(p); }
};

// half simulated: every multiply and subtract rounded (densela.py:201-217)
template <>
struct Arith<MODE_H16> {
  using T = float;
  static constexpr bool kExactOrder = true;
  GB_DEVICE static T zero() { return 0.f; }
  GB_DEVICE static T from(double x) { return __half2float(__double2half(x)); }
  GB_DEVICE static T sub_prod(T acc, double l, T y) { return h_sub(acc, h_mul((float)l, y)); }
  GB_DEVICE static T mac(T acc, double a, double v) { return h_add(acc, h_mul((float)a, (float)v)); }
  GB_DEVICE static T add(T a, T b) { return h_add(a, b); }
  GB_DEVICE static T sub(T a, T b) { return h_sub(a, b); }
  GB_DEVICE static T div(T y, double u) { return h_div(y, (float)u); }
  GB_DEVICE static double val(T x) { return (double)x; }
  GB_DEVICE static T shfl(T x, int src) { return __shfl_sync(0xffffffffu, x, src); }
  GB_DEVICE static T ld(const T* p) { return __ldcg(p); }
};

template <>
struct Arith<MODE_DD> {
  using T = dd;
  static constexpr bool kExactOrder = false;
  GB_DEVICE static T zero() { return dd{0.0, 0.0}; }
  GB_DEVICE static T from(double x) { return dd{x, 0.0}; }
  GB_DEVICE static T sub_prod(T acc, double l, T y) { return dd_sub(acc, dd_scale(l, y)); }
  GB_DEVICE static T mac(T acc, double a, double v) { return dd_add(acc, two_prod(a, v)); }
  GB_DEVICE static T add(T a, T b) { return dd_add(a, b); }
  GB_DEVICE static T sub(T a, T b) { return dd_sub(a, b); }
  GB_DEVICE static T div(T y, double u) { return dd_div(y, dd{u, 0.0}); }
  GB_DEVICE static double val(T x) { return dd_val(x); }
  GB_DEVICE static T shfl(T x, int src) {
    return dd{__shfl_sync(0xffffffffu, x.hi, src), __shfl_sync(0xffffffffu, x.lo, src)};
  }
  GB_DEVICE static T ld(const T* p) {
    double2 v = __ldcg(reinterpret_cast<const double2*>(p));
    return dd{v.x, v.y};
  }
};

// tile element type: factors held at u_f width fit a float tile exactly
template <class TF>
struct TileT {
  using T = float;
};
template <>
struct TileT<double> {
  using T = double;
};

// ---------------------------------------------------------------------------
// system view
// ---------------------------------------------------------------------------
template <class TA, class TF>
struct SysView {
  int n;
  size_t lda;
  const TA* A;
  size_t ldf;
  const TF* LU;
  const int* perm;
};

// progress counters of the flag-based TRSV (one per direction)
struct TrsvSync {
  unsigned long long* fwd;
  unsigned long long* bwd;
  unsigned long long epoch;  // call index; identical in all CTAs
};

GB_DEVICE unsigned long long ld_acquire64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
GB_DEVICE void st_release64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <class Team>
GB_DEVICE void wait_progress(const unsigned long long* ctr, unsigned long long target,
                             unsigned long long* cache) {
  if constexpr (Team::kGrid) {
    if (*cache >= target) return;
    unsigned long long v;
    while ((v = ld_acquire64(ctr)) < target) __nanosleep(32);
    *cache = v;
  }
}

// ---------------------------------------------------------------------------
// triangular solves over row blocks.
//   y (in: right-hand side in accumulator type, out: solution), length n.
//   Lower: unit diagonal, column order 0..i-1.  Upper: columns n-1..i+1 then
//   divide by U_ii.  kSplit: number of warps that split the off-diagonal
//   columns of a row block (1 keeps the exact per-element order).
// ---------------------------------------------------------------------------
template <int M, class Team, class TF, bool kLower>
__device__ void trsv_blocks(Team& t, int n, const TF* LU, size_t ldf,
                            typename Arith<M>::T* y, const TrsvSync& ts, void* smem_raw) {
  using Ar = Arith<M>;
  using T = typename Ar::T;
  const int nb = (n + kRB - 1) / kRB;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const int split = Ar::kExactOrder ? 1 : nw;
  // smem: per warp a 32x33 tile (fp64 factors keep a double tile) + partials
  using TT = typename TileT<TF>::T;
  TT* tiles = reinterpret_cast<TT*>(smem_raw);
  T* parts = reinterpret_cast<T*>(tiles + nw * 32 * 33);
  TT* tile = tiles + wid * 32 * 33;
  unsigned long long* ctr = kLower ? ts.fwd : ts.bwd;
  const unsigned long long base = ts.epoch * (unsigned long long)nb;
  __shared__ unsigned long long cache;
  if (threadIdx.x == 0) {
    cache = 0;
    // the backward sweep starts from the bottom of the forward result
    if (!kLower) {
      unsigned long long c2 = 0;
      wait_progress<Team>(ts.fwd, base + (unsigned long long)nb, &c2);
    }
  }
  __syncthreads();

  const int G = t.size(), r = t.rank();
  for (int s = r; s < nb; s += G) {
    const int b = kLower ? s : nb - 1 - s;
    const int row = b * kRB + lane;
    const bool rv = row < n;
    T acc = Ar::zero();
    if (wid < split) {
      if (wid == 0 && rv) acc = Ar::ld(y + row);
      // off-diagonal column blocks handled by this warp, in order
      const int ncb = kLower ? b : nb - 1 - b;  // number of off-diagonal blocks
      for (int q = wid; q < ncb; q += split) {
        const int cb = kLower ? q : nb - 1 - q;
        // wait until column block cb is final
        if (lane == 0) wait_progress<Team>(ctr, base + (unsigned long long)(q + 1), &cache);
        __syncwarp();
        // stage the 32x32 tile (rows of this block, columns of cb) coalesced
        const int c0 = cb * kRB;
        for (int rr = 0; rr < 32; ++rr) {
          int gr = b * kRB + rr, gc = c0 + lane;
          TT v = TT(0);
          if (gr < n && gc < n) v = (TT)to_d(LU[(size_t)gr * ldf + gc]);
          tile[rr * 33 + lane] = v;
        }
        T yv = (c0 + lane < n) ? Ar::ld(y + c0 + lane) : Ar::zero();
        __syncwarp();
        if (kLower) {
          for (int jj = 0; jj < 32; ++jj) {
            T yj = Ar::shfl(yv, jj);
            if (rv && c0 + jj < n) acc = Ar::sub_prod(acc, (double)tile[lane * 33 + jj], yj);
          }
        } else {
          for (int jj = 31; jj >= 0; --jj) {
            T yj = Ar::shfl(yv, jj);
            if (rv && c0 + jj < n) acc = Ar::sub_prod(acc, (double)tile[lane * 33 + jj], yj);
          }
        }
        __syncwarp();
      }
      if (split > 1) parts[wid * 32 + lane] = acc;
    }
    __syncthreads();
    if (wid == 0) {
      if (split > 1) {
        acc = parts[lane];
        for (int w = 1; w < split; ++w) acc = Ar::add(acc, parts[w * 32 + lane]);
      }
      // diagonal block
      for (int rr = 0; rr < 32; ++rr) {
        int gr = b * kRB + rr, gc = b * kRB + lane;
        TT v = TT(0);
        if (gr < n && gc < n) v = (TT)to_d(LU[(size_t)gr * ldf + gc]);
        tile[rr * 33 + lane] = v;
      }
      __syncwarp();
      if (kLower) {
        for (int jj = 0; jj < 32; ++jj) {
          T yj = Ar::shfl(acc, jj);
          if (rv && lane > jj) acc = Ar::sub_prod(acc, (double)tile[lane * 33 + jj], yj);
        }
      } else {
        for (int jj = 31; jj >= 0; --jj) {
          if (lane == jj && rv) acc = Ar::div(acc, (double)tile[lane * 33 + lane]);
          T yj = Ar::shfl(acc, jj);
          if (rv && lane < jj && b * kRB + jj < n)
            acc = Ar::sub_prod(acc, (double)tile[lane * 33 + jj], yj);
        }
      }
      if (rv) y[row] = acc;
      __syncwarp();
      if constexpr (Team::kGrid) {
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release64(ctr, base + (unsigned long long)(s + 1));
      }
    }
    __syncthreads();
  }
}

template <int M, class TF>
__host__ __device__ inline size_t trsv_smem_bytes(int nthreads) {
  return (size_t)(nthreads / 32) * 32 * 33 * sizeof(typename TileT<TF>::T) +
         (size_t)(nthreads / 32) * 32 * sizeof(typename Arith<M>::T);
}

// ---------------------------------------------------------------------------
// GEMV rows into the accumulator: y[i] = sum_j A[src(i), j] * v[j]
// One warp per row; rows of a block distributed over the CTA's warps.
// ---------------------------------------------------------------------------
// 16-byte vector of row elements
template <class T>
struct alignas(16) Vec16 {
  static constexpr int N = 16 / sizeof(T);
  T v[N];
};

// One warp computes sum_j a[j] * v[j] (mode M) and optionally sum |a||v|.
// 128-bit loads, kU independent accumulators per lane (memory-level
// parallelism), deterministic combine and warp tree.
template <int M, bool kAbs, class TA, class TV>
__device__ __forceinline__ typename Arith<M>::T row_dot_ex(const TA* __restrict__ arow, const TV* __restrict__ v,
                                                           int n, double* absdot) {
  using Ar = Arith<M>;
  using T = typename Ar::T;
  constexpr int VW = Vec16<TA>::N;
  constexpr int kU = 4;
  const int lane = threadIdx.x & 31;
  T acc[kU];
  double ab[kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    acc[u] = Ar::zero();
    ab[u] = 0.0;
  }
  const int nv = n / VW;
  const Vec16<TA>* av = reinterpret_cast<const Vec16<TA>*>(arow);
  int base = lane;
  for (; base + 32 * (kU - 1) < nv; base += 32 * kU) {
    Vec16<TA> a[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) a[u] = av[base + 32 * u];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
#pragma unroll
      for (int e = 0; e < VW; ++e) {
        const double x = (double)a[u].v[e];
        const double y = to_d(v[(base + 32 * u) * VW + e]);
        acc[u] = Ar::mac(acc[u], x, y);
        if (kAbs) ab[u] = __fma_rn(fabs(x), fabs(y), ab[u]);
      }
    }
  }
  for (; base < nv; base += 32) {
    Vec16<TA> a0 = av[base];
#pragma unroll
    for (int e = 0; e < VW; ++e) {
      const double x = (double)a0.v[e];
      const double y = to_d(v[base * VW + e]);
      acc[0] = Ar::mac(acc[0], x, y);
      if (kAbs) ab[0] = __fma_rn(fabs(x), fabs(y), ab[0]);
    }
  }
  for (int j = nv * VW + lane; j < n; j += 32) {
    const double x = (double)arow[j];
    const double y = to_d(v[j]);
    acc[1] = Ar::mac(acc[1], x, y);
    if (kAbs) ab[1] = __fma_rn(fabs(x), fabs(y), ab[1]);
  }
  T s = Ar::add(Ar::add(acc[0], acc[1]), Ar::add(acc[2], acc[3]));
  if constexpr (M == MODE_DD) {
    s = warp_sum_dd(s);
  } else {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s = Ar::add(s, __shfl_xor_sync(0xffffffffu, s, o));
  }
  if (kAbs) *absdot = warp_sum((ab[0] + ab[1]) + (ab[2] + ab[3]));
  return s;
}

template <int M, class TA, class TV>
__device__ __forceinline__ typename Arith<M>::T row_dot(const TA* __restrict__ arow, const TV* __restrict__ v, int n) {
  return row_dot_ex<M, false>(arow, v, n, nullptr);
}

// ---------------------------------------------------------------------------
// w = fl_u( U^-1 L^-1 ( (A v)[perm] ) )    (apply_preconditioned)
// or, with v == nullptr, the precond_rhs variant on r:
// w = fl_u( U^-1 L^-1 r[perm] )             (r pre-rounded by the caller)
// ---------------------------------------------------------------------------
template <int M, class Team, class TA, class TF, class TV, class TR, class TW>
__device__ void op_apply(Team& t, const SysView<TA, TF>& s, const TV* v, const TR* rvec,
                         TW* w, typename Arith<M>::T* ybuf, TrsvSync& ts, void* smem) {
  using Ar = Arith<M>;
  const int n = s.n;
  const int nb = (n + kRB - 1) / kRB;
  const int G = t.size(), r = t.rank();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // 1. right-hand side in permuted order, blocks owned as in the forward solve
  for (int b = r; b < nb; b += G) {
    for (int rr = wid; rr < kRB; rr += nw) {
      int i = b * kRB + rr;
      if (i >= n) break;
      int src = s.perm[i];
      typename Ar::T val;
      if (v != nullptr) {
        val = row_dot<M>(s.A + (size_t)src * s.lda, v, n);
      } else {
        val = Ar::from(to_d(rvec[src]));
      }
      if (lane == 0) ybuf[i] = val;
    }
  }
  __syncthreads();
  // 2. forward (unit lower) then backward (upper)
  trsv_blocks<M, Team, TF, true>(t, n, s.LU, s.ldf, ybuf, ts, smem);
  trsv_blocks<M, Team, TF, false>(t, n, s.LU, s.ldf, ybuf, ts, smem);
  ts.epoch++;
  // 3. round to u: each CTA writes the rows it finalised in the backward pass
  for (int q = r; q < nb; q += G) {
    int b = nb - 1 - q;
    for (int rr = threadIdx.x; rr < kRB; rr += blockDim.x) {
      int i = b * kRB + rr;
      if (i < n) w[i] = (TW)Ar::val(Ar::ld(ybuf + i));
    }
  }
  t.sync();
}

// ---------------------------------------------------------------------------
// format-faithful BLAS-1 over a team (precision.py:513-587)
// ---------------------------------------------------------------------------
template <class TW>
struct Fmt;
// u = single: native fp32 arithmetic, multiply and add rounded separately
template <>
struct Fmt<float> {
  GB_DEVICE static float rnd(double x) { return __double2float_rn(x); }
  GB_DEVICE static float scale(double a, float x) { return __fmul_rn((float)a, x); }
  GB_DEVICE static float axpy(double a, float x, float y) { return __fadd_rn(y, __fmul_rn((float)a, x)); }
  using Acc = float;
  GB_DEVICE static float mac(float acc, float x, float y) { return __fmaf_rn(x, y, acc); }
  GB_DEVICE static double sqrt_(double s) { return (double)sqrtf((float)s); }
  static constexpr double u = 5.9604644775390625e-08;  // 2^-24
};
template <>
struct Fmt<double> {
  GB_DEVICE static double rnd(double x) { return x; }
  GB_DEVICE static double scale(double a, double x) { return __dmul_rn(a, x); }
  GB_DEVICE static double axpy(double a, double x, double y) { return __dadd_rn(y, __dmul_rn(a, x)); }
  using Acc = double;
  GB_DEVICE static double mac(double acc, double x, double y) { return __fma_rn(x, y, acc); }
  GB_DEVICE static double sqrt_(double s) { return sqrt(s); }
  static constexpr double u = 1.1102230246251565e-16;  // 2^-53
};

// K simultaneous dot products x_i . y over the team; result in every thread
template <class TW, int K, class Team>
__device__ void team_dots(Team& t, const TW* const (&x)[K], const TW* y, int n, double (&out)[K],
                          void* red) {
  using Acc = typename Fmt<TW>::Acc;
  int lo, hi;
  t.rows(n, lo, hi);
  Acc a[K];
#pragma unroll
  for (int i = 0; i < K; ++i) a[i] = Acc(0);
  for (int j = lo + threadIdx.x; j < hi; j += blockDim.x) {
    TW yj = y[j];
#pragma unroll
    for (int i = 0; i < K; ++i) a[i] = Fmt<TW>::mac(a[i], x[i][j], yj);
  }
  block_sum<Acc, K>(a, reinterpret_cast<Acc*>(red));
  t.template finish_sum<Acc, K>(a);
#pragma unroll
  for (int i = 0; i < K; ++i) out[i] = (double)a[i];
}

template <class TW, class Team>
__device__ double team_dot(Team& t, const TW* x, const TW* y, int n, void* red) {
  const TW* xs[1] = {x};
  double o[1];
  team_dots<TW, 1>(t, xs, y, n, o, red);
  return o[0];
}

template <class TW, class Team>
__device__ double team_nrm2(Team& t, const TW* x, int n, void* red) {
  return Fmt<TW>::sqrt_(team_dot<TW>(t, x, x, n, red));
}

// infinity norm of a u-valued vector (NaN propagates like numpy max)
template <class TW, class Team>
__device__ double team_amax(Team& t, const TW* x, int n, double* red) {
  int lo, hi;
  t.rows(n, lo, hi);
  double m = 0.0;
  for (int j = lo + threadIdx.x; j < hi; j += blockDim.x) m = nan_max(m, fabs((double)x[j]));
  // block max with NaN propagation
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = nan_max(m, __shfl_xor_sync(0xffffffffu, m, o));
  __syncthreads();
  if (lane == 0) red[wid] = m;
  __syncthreads();
  m = lane < nw ? red[lane] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = nan_max(m, __shfl_xor_sync(0xffffffffu, m, o));
  __syncthreads();
  return t.finish_max(m);
}

// y <- y + alpha * x  (local rows only; caller syncs when others need y)
template <class TW, class Team>
GB_DEVICE void team_axpy(Team& t, double alpha, const TW* x, TW* y, int n) {
  int lo, hi;
  t.rows(n, lo, hi);
  for (int j = lo + threadIdx.x; j < hi; j += blockDim.x) y[j] = Fmt<TW>::axpy(alpha, x[j], y[j]);
}
template <class TW, class Team>
GB_DEVICE void team_scale(Team& t, double alpha, const TW* x, TW* y, int n) {
  int lo, hi;
  t.rows(n, lo, hi);
  for (int j = lo + threadIdx.x; j < hi; j += blockDim.x) y[j] = Fmt<TW>::scale(alpha, x[j]);
}
template <class TW, class Team>
GB_DEVICE void team_copy(Team& t, const TW* x, TW* y, int n) {
  int lo, hi;
  t.rows(n, lo, hi);
  for (int j = lo + threadIdx.x; j < hi; j += blockDim.x) y[j] = x[j];
}
template <class TW, class Team>
GB_DEVICE void team_zero(Team& t, TW* y, int n) {
  int lo, hi;
  t.rows(n, lo, hi);
  for (int j = lo + threadIdx.x; j < hi; j += blockDim.x) y[j] = TW(0);
}

// out[i] = X_i . y  for i < K (runtime K), X columns of length n with stride ld.
// Every entry is a native dot in the work format (mat_tvec, precision.py:577-587).
// Results land in smem `out` (K entries) identical in all CTAs.
template <class TW, class Team>
__device__ void team_tvec(Team& t, const TW* X, size_t ld, int K, const TW* y, int n, double* out,
                          double* tmp) {
  using Acc = typename Fmt<TW>::Acc;
  int lo, hi;
  t.rows(n, lo, hi);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // one warp per column, lanes over rows, deterministic tree
  for (int i = wid; i < K; i += nw) {
    Acc a = Acc(0);
    const TW* xi = X + (size_t)i * ld;
    for (int j = lo + lane; j < hi; j += 32) a = Fmt<TW>::mac(a, xi[j], y[j]);
    a = warp_sum(a);
    if (lane == 0) tmp[i] = (double)a;
  }
  __syncthreads();
  if constexpr (Team::kGrid) {
    t.template sum_vec<double>(tmp, out, K);
    // sum_vec summed in double; re-round to the work format's accumulation
    for (int i = threadIdx.x; i < K; i += blockDim.x) out[i] = (double)(Acc)out[i];
    __syncthreads();
  } else {
    for (int i = threadIdx.x; i < K; i += blockDim.x) out[i] = tmp[i];
    __syncthreads();
  }
}

}  // namespace gb
