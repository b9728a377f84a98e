// GEPP LU factorisation in u_f (reference densela.py:124-168).
//
//   MODE_H16: the reference's simulated half GEPP -- multiplier fl16(a/p),
//             update fl16(a - fl16(l*u)), first-max pivot, whole-row swaps.
//             Every element receives its updates in increasing k, so the
//             blocked right-looking variant below (panel, row swaps, TRSM,
//             trailing update applying k in order) is bit-identical to the
//             unblocked reference loop.
//   MODE_F32 / MODE_F64: LAPACK-style GEPP (?getrf): FMA updates, multipliers
//             by the reciprocal pivot, zero pivots skipped and reported.
//
// Storage: row-major, leading dimension ld.  perm[i] = original row at pivot
// position i (densela.py:137-140 converts LAPACK ipiv the same way).
#pragma once
#include "gb_team.cuh"
#include "gb_ops.cuh"
#include "gb_tc.cuh"

namespace gb {

template <int M>
struct LuT;
template <>
struct LuT<MODE_H16> {
  using S = __half;  // global storage
  using C = float;   // compute carrier (half-valued)
  GB_DEVICE static S st(C x) { return __float2half_rn(x); }
  GB_DEVICE static C ld(S x) { return __half2float(x); }
  GB_DEVICE static S from_u(double x) { return __double2half(x); }
  GB_DEVICE static C mult(C a, C p) { return h_div(a, p); }
  GB_DEVICE static C upd(C a, C l, C u) { return h_sub(a, h_mul(l, u)); }
  static constexpr bool kLapack = false;
};
template <>
struct LuT<MODE_F32> {
  using S = float;
  using C = float;
  GB_DEVICE static S st(C x) { return x; }
  GB_DEVICE static C ld(S x) { return x; }
  GB_DEVICE static S from_u(double x) { return __double2float_rn(x); }
  GB_DEVICE static C mult(C a, C p) { return __fmul_rn(a, __frcp_rn(p)); }
  GB_DEVICE static C upd(C a, C l, C u) { return __fmaf_rn(-l, u, a); }
  static constexpr bool kLapack = true;
};
template <>
struct LuT<MODE_F64> {
  using S = double;
  using C = double;
  GB_DEVICE static S st(C x) { return x; }
  GB_DEVICE static C ld(S x) { return x; }
  GB_DEVICE static S from_u(double x) { return x; }
  GB_DEVICE static C mult(C a, C p) { return __dmul_rn(a, __drcp_rn(p)); }
  GB_DEVICE static C upd(C a, C l, C u) { return __fma_rn(-l, u, a); }
  static constexpr bool kLapack = true;
};

// (|value|, index) pivot key: NaN beats everything (numpy argmax returns the
// first NaN), then larger |value|, then the lower index.
struct PivKey {
  double v;
  int i;
  int nan;
};
GB_DEVICE bool piv_better(const PivKey& a, const PivKey& b) {
  if (a.i < 0) return false;
  if (b.i < 0) return true;
  if (a.nan != b.nan) return a.nan > b.nan;
  if (a.v != b.v) return a.v > b.v;
  return a.i < b.i;
}
GB_DEVICE PivKey piv_shfl(const PivKey& k, int o) {
  return PivKey{__shfl_xor_sync(0xffffffffu, k.v, o), __shfl_xor_sync(0xffffffffu, k.i, o),
                __shfl_xor_sync(0xffffffffu, k.nan, o)};
}
// block-wide pivot search; every thread gets the result. scratch: 32 PivKey.
__device__ inline PivKey block_pivot(PivKey k, PivKey* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    PivKey q = piv_shfl(k, o);
    if (piv_better(q, k)) k = q;
  }
  __syncthreads();
  if (lane == 0) scratch[wid] = k;
  __syncthreads();
  k = lane < nw ? scratch[lane] : PivKey{0.0, -1, 0};
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    PivKey q = piv_shfl(k, o);
    if (piv_better(q, k)) k = q;
  }
  __syncthreads();
  return k;
}
GB_DEVICE PivKey make_key(double x, int i) {
  PivKey k;
  k.nan = (x != x);
  k.v = k.nan ? 0.0 : fabs(x);
  k.i = i;
  return k;
}

// ---------------------------------------------------------------------------
// one-CTA in-place GEPP on a buffer of carrier type C (smem or global).
// Returns the first zero-pivot column, or -1.
// ---------------------------------------------------------------------------
template <int M>
__device__ int lu_cta(typename LuT<M>::C* a, int n, int lda, int* perm, PivKey* scratch) {
  using L = LuT<M>;
  using C = typename L::C;
  __shared__ int s_p;
  int zero = -1;
  for (int i = threadIdx.x; i < n; i += blockDim.x) perm[i] = i;
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    PivKey key{0.0, -1, 0};
    for (int i = k + threadIdx.x; i < n; i += blockDim.x) {
      PivKey c = make_key((double)a[(size_t)i * lda + k], i);
      if (piv_better(c, key)) key = c;
    }
    key = block_pivot(key, scratch);
    const int p = key.i;
    const C piv = a[(size_t)p * lda + k];
    const bool isz = (piv == C(0));
    // every thread holds the pivot before the row interchange below may
    // overwrite a[p][k] (thread k % blockDim swaps that entry)
    __syncthreads();
    if (isz && zero < 0) zero = k;
    if (isz && L::kLapack) continue;  // LAPACK: column already zero below
    if (p != k) {
      for (int j = threadIdx.x; j < n; j += blockDim.x) {
        C t = a[(size_t)k * lda + j];
        a[(size_t)k * lda + j] = a[(size_t)p * lda + j];
        a[(size_t)p * lda + j] = t;
      }
      if (threadIdx.x == 0) {
        int t = perm[k];
        perm[k] = perm[p];
        perm[p] = t;
      }
    }
    __syncthreads();
    for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x)
      a[(size_t)i * lda + k] = L::mult(a[(size_t)i * lda + k], piv);
    __syncthreads();
    const int m = n - k - 1;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
      int i = k + 1 + e / m, j = k + 1 + e % m;
      a[(size_t)i * lda + j] = L::upd(a[(size_t)i * lda + j], a[(size_t)i * lda + k], a[(size_t)k * lda + j]);
    }
    __syncthreads();
  }
  (void)s_p;
  return zero;
}

// ---------------------------------------------------------------------------
// blocked GEPP kernels (large n)
// ---------------------------------------------------------------------------
struct LuStatus {
  int zero_col;  // first zero pivot (or INT_MAX)
  int pad;
  unsigned long long amax_bits;  // max|A_uf| as ordered bits
  unsigned long long umax_bits;  // max|U|
};

GB_DEVICE void atomic_max_abs(unsigned long long* p, double v) {
  v = fabs(v);
  if (v != v) v = __longlong_as_double(0x7ff0000000000000ull);  // NaN -> inf
  atomicMax(p, (unsigned long long)__double_as_longlong(v));
}

// W = fl_uf(A) and the amax of the rounded matrix
template <int M, class TA>
__global__ void k_lu_convert(const TA* __restrict__ A, size_t lda, typename LuT<M>::S* W, size_t ldw,
                             int n, LuStatus* st) {
  using L = LuT<M>;
  double m = 0.0;
  size_t total = (size_t)n * n;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total;
       e += (size_t)gridDim.x * blockDim.x) {
    size_t i = e / n, j = e % n;
    typename L::S s = L::from_u((double)A[i * lda + j]);
    W[i * ldw + j] = s;
    double v = fabs((double)L::ld(s));
    m = (v > m || v != v) ? v : m;
  }
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) atomic_max_abs(&st->amax_bits, m);
}

// dd-exact reciprocals of diag(U): 1/U_ii = rh + rl
template <class S>
__global__ void k_lu_rcp(const S* W, size_t ld, int n, double* rh, double* rl) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double d = to_d(W[(size_t)i * ld + i]);
    dd q = dd_div(dd{1.0, 0.0}, dd{d, 0.0});
    rh[i] = q.hi;
    rl[i] = q.lo;
  }
}

// dd-accurate inverses of the 32x32 diagonal blocks (for the non-exact
// substitution modes): one warp per block, lane c builds column c.
// Layout: element (i, j) of block b at b*1024 + j*32 + i; L part strictly
// lower (unit diagonal implied), U part upper including the diagonal.
template <class S>
__device__ void diag_inv_block(const S* W, size_t ld, int n, int b, double* lh, double* ll, double* uh,
                               double* ul) {
  const int c = threadIdx.x & 31;
  const int r0 = b * 32;
  const int m = min(32, n - r0);
  dd x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = dd{0.0, 0.0};
  if (c < m) {
    x[c] = dd{1.0, 0.0};
    for (int i = c + 1; i < m; ++i) {
      dd s{0.0, 0.0};
      for (int j = c; j < i; ++j) s = dd_add(s, dd_scale(to_d(W[(size_t)(r0 + i) * ld + r0 + j]), x[j]));
      x[i] = dd_neg(s);
    }
  }
  for (int i = 0; i < 32; ++i) {
    lh[(size_t)b * kInvStride + c * 32 + i] = (i > c && c < m) ? x[i].hi : 0.0;
    ll[(size_t)b * kInvStride + c * 32 + i] = (i > c && c < m) ? x[i].lo : 0.0;
    x[i] = dd{0.0, 0.0};
  }
  if (c < m) {
    x[c] = dd_div(dd{1.0, 0.0}, dd{to_d(W[(size_t)(r0 + c) * ld + r0 + c]), 0.0});
    for (int i = c - 1; i >= 0; --i) {
      dd s{0.0, 0.0};
      for (int j = i + 1; j <= c; ++j) s = dd_add(s, dd_scale(to_d(W[(size_t)(r0 + i) * ld + r0 + j]), x[j]));
      const dd ri = dd_div(dd{1.0, 0.0}, dd{to_d(W[(size_t)(r0 + i) * ld + r0 + i]), 0.0});
      x[i] = dd_neg(dd_mul(s, ri));
    }
  }
  for (int i = 0; i < 32; ++i) {
    uh[(size_t)b * kInvStride + c * 32 + i] = (i <= c && c < m) ? x[i].hi : 0.0;
    ul[(size_t)b * kInvStride + c * 32 + i] = (i <= c && c < m) ? x[i].lo : 0.0;
  }
}

// Folded off-diagonal blocks for trsv_cta (second half of each block record,
// row-major, element (i, j) at b*kInvStride + 1024 + i*32 + j):
//   lower b >= 1:      D_b^-1 L_{b,b-1}   (D_b unit lower diagonal block)
//   upper b <= nb - 2: U_bb^-1 U_{b,b+1}
// so the block solve becomes y_b = D_b^-1 t' - M_b y_adjacent with t' free of
// the adjacent block: only one 32-term product waits on the neighbour.
template <class S>
__device__ void diag_fold_block(const S* W, size_t ld, int n, int b, double* lh, double* ll, double* uh,
                                double* ul) {
  const int j = threadIdx.x & 31;
  const int nb = (n + 31) / 32;
  const int r0 = b * 32;
  const int m = min(32, n - r0);
  double* fl_h = lh + (size_t)b * kInvStride + 1024;
  double* fl_l = ll + (size_t)b * kInvStride + 1024;
  double* fu_h = uh + (size_t)b * kInvStride + 1024;
  double* fu_l = ul + (size_t)b * kInvStride + 1024;
  const double* Li_h = lh + (size_t)b * kInvStride;
  const double* Li_l = ll + (size_t)b * kInvStride;
  const double* Ui_h = uh + (size_t)b * kInvStride;
  const double* Ui_l = ul + (size_t)b * kInvStride;
  for (int i = 0; i < 32; ++i) {
    dd sl{0.0, 0.0}, su{0.0, 0.0};
    if (i < m) {
      if (b >= 1) {
        const int c = (b - 1) * 32 + j;
        sl = dd{to_d(W[(size_t)(r0 + i) * ld + c]), 0.0};
        for (int k = 0; k < i; ++k)
          sl = dd_add(sl, dd_scale(to_d(W[(size_t)(r0 + k) * ld + c]), dd{Li_h[k * 32 + i], Li_l[k * 32 + i]}));
      }
      if (b + 1 < nb) {
        const int c = (b + 1) * 32 + j;
        if (c < n)
          for (int k = i; k < m; ++k)
            su = dd_add(su, dd_scale(to_d(W[(size_t)(r0 + k) * ld + c]), dd{Ui_h[k * 32 + i], Ui_l[k * 32 + i]}));
      }
    }
    fl_h[i * 32 + j] = sl.hi;
    fl_l[i * 32 + j] = sl.lo;
    fu_h[i * 32 + j] = su.hi;
    fu_l[i * 32 + j] = su.lo;
  }
}

template <class S>
__global__ void k_diag_fold(const S* W, size_t ld, int n, double* lh, double* ll, double* uh, double* ul) {
  const int wpb = blockDim.x / 32;
  const int nb = (n + 31) / 32;
  for (int b = blockIdx.x * wpb + (threadIdx.x >> 5); b < nb; b += gridDim.x * wpb)
    diag_fold_block(W, ld, n, b, lh, ll, uh, ul);
}

template <class S>
__global__ void k_diag_inv(const S* W, size_t ld, int n, double* lh, double* ll, double* uh, double* ul) {
  const int wpb = blockDim.x / 32;
  const int nb = (n + 31) / 32;
  for (int b = blockIdx.x * wpb + (threadIdx.x >> 5); b < nb; b += gridDim.x * wpb)
    diag_inv_block(W, ld, n, b, lh, ll, uh, ul);
}

// B-row versions of the two record builders above for the grid-team
// substitution (trsv_cta_g): B threads per block, thread c builds column c;
// record stride 2 B^2, inverse column-major then folded block row-major.
template <int B, class S>
__device__ void diag_inv_block_b(const S* W, size_t ld, int n, int b, double* lh, double* ll, double* uh,
                               double* ul) {
  constexpr int RS = inv_stride<B>();
  const int c = threadIdx.x % B;
  const int r0 = b * B;
  const int m = min(B, n - r0);
  dd x[B];
#pragma unroll
  for (int i = 0; i < B; ++i) x[i] = dd{0.0, 0.0};
  if (c < m) {
    x[c] = dd{1.0, 0.0};
    for (int i = c + 1; i < m; ++i) {
      dd s{0.0, 0.0};
      for (int j = c; j < i; ++j) s = dd_add(s, dd_scale(to_d(W[(size_t)(r0 + i) * ld + r0 + j]), x[j]));
      x[i] = dd_neg(s);
    }
  }
  for (int i = 0; i < B; ++i) {
    lh[(size_t)b * RS + c * B + i] = (i > c && c < m) ? x[i].hi : 0.0;
    ll[(size_t)b * RS + c * B + i] = (i > c && c < m) ? x[i].lo : 0.0;
    x[i] = dd{0.0, 0.0};
  }
  if (c < m) {
    x[c] = dd_div(dd{1.0, 0.0}, dd{to_d(W[(size_t)(r0 + c) * ld + r0 + c]), 0.0});
    for (int i = c - 1; i >= 0; --i) {
      dd s{0.0, 0.0};
      for (int j = i + 1; j <= c; ++j) s = dd_add(s, dd_scale(to_d(W[(size_t)(r0 + i) * ld + r0 + j]), x[j]));
      const dd ri = dd_div(dd{1.0, 0.0}, dd{to_d(W[(size_t)(r0 + i) * ld + r0 + i]), 0.0});
      x[i] = dd_neg(dd_mul(s, ri));
    }
  }
  for (int i = 0; i < B; ++i) {
    uh[(size_t)b * RS + c * B + i] = (i <= c && c < m) ? x[i].hi : 0.0;
    ul[(size_t)b * RS + c * B + i] = (i <= c && c < m) ? x[i].lo : 0.0;
  }
}

// Folded off-diagonal blocks (second half of each block record, row-major,
// element (i, j) at b*2B^2 + B^2 + i*B + j):
//   lower b >= 1:      D_b^-1 L_{b,b-1}   (D_b unit lower diagonal block)
//   upper b <= nb - 2: U_bb^-1 U_{b,b+1}
// so the block solve becomes y_b = D_b^-1 t' - M_b y_adjacent with t' free of
// the adjacent block: only one B-term product waits on the neighbour.
template <int B, class S>
__device__ void diag_fold_block_b(const S* W, size_t ld, int n, int b, double* lh, double* ll, double* uh,
                                double* ul) {
  constexpr int RS = inv_stride<B>();
  const int j = threadIdx.x % B;
  const int nb = (n + B - 1) / B;
  const int r0 = b * B;
  const int m = min(B, n - r0);
  double* fl_h = lh + (size_t)b * RS + B * B;
  double* fl_l = ll + (size_t)b * RS + B * B;
  double* fu_h = uh + (size_t)b * RS + B * B;
  double* fu_l = ul + (size_t)b * RS + B * B;
  const double* Li_h = lh + (size_t)b * RS;
  const double* Li_l = ll + (size_t)b * RS;
  const double* Ui_h = uh + (size_t)b * RS;
  const double* Ui_l = ul + (size_t)b * RS;
  for (int i = 0; i < B; ++i) {
    dd sl{0.0, 0.0}, su{0.0, 0.0};
    if (i < m) {
      if (b >= 1) {
        const int c = (b - 1) * B + j;
        sl = dd{to_d(W[(size_t)(r0 + i) * ld + c]), 0.0};
        for (int k = 0; k < i; ++k)
          sl = dd_add(sl, dd_scale(to_d(W[(size_t)(r0 + k) * ld + c]), dd{Li_h[k * B + i], Li_l[k * B + i]}));
      }
      if (b + 1 < nb) {
        const int c = (b + 1) * B + j;
        if (c < n)
          for (int k = i; k < m; ++k)
            su = dd_add(su, dd_scale(to_d(W[(size_t)(r0 + k) * ld + c]), dd{Ui_h[k * B + i], Ui_l[k * B + i]}));
      }
    }
    fl_h[i * B + j] = sl.hi;
    fl_l[i * B + j] = sl.lo;
    fu_h[i * B + j] = su.hi;
    fu_l[i * B + j] = su.lo;
  }
}

template <int B, class S>
__global__ void k_diag_fold_b(const S* W, size_t ld, int n, double* lh, double* ll, double* uh, double* ul) {
  const int bpc = blockDim.x / B;
  const int nb = (n + B - 1) / B;
  for (int b = blockIdx.x * bpc + (int)(threadIdx.x / B); b < nb; b += gridDim.x * bpc)
    diag_fold_block_b<B>(W, ld, n, b, lh, ll, uh, ul);
}

template <int B, class S>
__global__ void k_diag_inv_b(const S* W, size_t ld, int n, double* lh, double* ll, double* uh, double* ul) {
  const int bpc = blockDim.x / B;
  const int nb = (n + B - 1) / B;
  for (int b = blockIdx.x * bpc + (int)(threadIdx.x / B); b < nb; b += gridDim.x * bpc)
    diag_inv_block_b<B>(W, ld, n, b, lh, ll, uh, ul);
}

// max |U| over the upper triangle
template <int M>
__global__ void k_lu_umax(const typename LuT<M>::S* W, size_t ld, int n, LuStatus* st) {
  using L = LuT<M>;
  double m = 0.0;
  for (int i = blockIdx.x; i < n; i += gridDim.x)
    for (int j = i + threadIdx.x; j < n; j += blockDim.x) {
      double v = fabs((double)L::ld(W[(size_t)i * ld + j]));
      m = (v > m || v != v) ? v : m;
    }
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) atomic_max_abs(&st->umax_bits, m);
}

// ---------------------------------------------------------------------------
// persistent team LU: the whole blocked GEPP in ONE cooperative launch.
//   per panel of 32 columns:
//     P  distributed panel factorisation: the panel rows live in the CTAs'
//        shared memory; per column one grid barrier (candidate pivots and the
//        candidate rows are staged in global memory, parity double-buffered)
//     S  row interchanges of the columns outside the panel
//     T  U12 = L11^-1 A12 (exact per-element order)
//     G  A22 -= L21 U12 (k applied in order per element; LAPACK modes sum the
//        32-term block product first, like sgemm/dgemm)
// ---------------------------------------------------------------------------
struct LuWork {
  PivKey* ckey;  // [2][G]
  double* crow;  // [2][G][32]
  double* rowk;  // [2][32]
  int* piv;      // [32]
};

constexpr int kLuNB = 32;

template <int M>
__device__ __forceinline__ void lu_gemm_tile(typename LuT<M>::S* W, size_t ld, int n, int nc, int k0, int i0, int j0,
                                             typename LuT<M>::C* ls, typename LuT<M>::C* us) {
  using L = LuT<M>;
  using C = typename L::C;
  constexpr int NB = kLuNB, TM = 64, TN = 64;
  for (int e = threadIdx.x; e < TM * NB; e += blockDim.x) {
    int r = e / NB, c = e % NB;
    ls[r * (NB + 1) + c] = (i0 + r < n) ? L::ld(W[(size_t)(i0 + r) * ld + k0 + c]) : C(0);
  }
  for (int e = threadIdx.x; e < NB * TN; e += blockDim.x) {
    int r = e / TN, c = e % TN;
    us[r * (TN + 1) + c] = (j0 + c < nc) ? L::ld(W[(size_t)(k0 + r) * ld + j0 + c]) : C(0);
  }
  __syncthreads();
  const int tr = threadIdx.x / 16, tc = threadIdx.x % 16;
  C acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      int i = i0 + tr + 16 * a, j = j0 + tc + 16 * b;
      acc[a][b] = (i < n && j < nc) ? L::ld(W[(size_t)i * ld + j]) : C(0);
    }
  if constexpr (L::kLapack) {
    C s[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) s[a][b] = C(0);
#pragma unroll 8
    for (int k = 0; k < NB; ++k) {
      C lv[4], uv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) lv[a] = ls[(tr + 16 * a) * (NB + 1) + k];
#pragma unroll
      for (int b = 0; b < 4; ++b) uv[b] = us[k * (TN + 1) + tc + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) s[a][b] = L::upd(s[a][b], -lv[a], uv[b]);
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = acc[a][b] - s[a][b];
  } else if constexpr (M == MODE_H16) {
    // exact fp16 GEPP update fl16(a - fl16(l u)) on packed half2 pairs:
    // __hmul2_rn / __hsub2_rn round each product and difference to fp16 and
    // are never contracted into an fma, so every element sees the same
    // operation sequence as the fp32-carried L::upd (double rounding through
    // fp32 is innocuous: 24 >= 2*11 + 2) at a quarter of the instructions
    __half2 acc2[4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int p = 0; p < 2; ++p) acc2[a][p] = __floats2half2_rn(acc[a][2 * p], acc[a][2 * p + 1]);
#pragma unroll 4
    for (int k = 0; k < NB; ++k) {
      __half2 l2[4], u2[2];
#pragma unroll
      for (int a = 0; a < 4; ++a) l2[a] = __float2half2_rn(ls[(tr + 16 * a) * (NB + 1) + k]);
#pragma unroll
      for (int p = 0; p < 2; ++p)
        u2[p] = __floats2half2_rn(us[k * (TN + 1) + tc + 16 * (2 * p)], us[k * (TN + 1) + tc + 16 * (2 * p + 1)]);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int p = 0; p < 2; ++p) acc2[a][p] = __hsub2_rn(acc2[a][p], __hmul2_rn(l2[a], u2[p]));
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        acc[a][2 * p] = __low2float(acc2[a][p]);
        acc[a][2 * p + 1] = __high2float(acc2[a][p]);
      }
  } else {
#pragma unroll 4
    for (int k = 0; k < NB; ++k) {
      C lv[4], uv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) lv[a] = ls[(tr + 16 * a) * (NB + 1) + k];
#pragma unroll
      for (int b = 0; b < 4; ++b) uv[b] = us[k * (TN + 1) + tc + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = L::upd(acc[a][b], lv[a], uv[b]);
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      int i = i0 + tr + 16 * a, j = j0 + tc + 16 * b;
      if (i < n && j < nc) W[(size_t)i * ld + j] = L::st(acc[a][b]);
    }
  __syncthreads();
}

template <int M>
__host__ __device__ inline size_t lu_team_smem(int n, int G) {
  using C = typename LuT<M>::C;
  const int sl = (n + G - 1) / G;
  const size_t simt = sizeof(C) * ((size_t)sl * 33 + 64 + 32 * 33 + 64 * 33 + 32 * 65) + 64;
  // tensor-core tiles (A 128x32, B 256x32 fp16, 1024-B aligned) + barrier
  return ((simt + 1023) & ~(size_t)1023) + 8192 + 16384 + 64;
}

// ---------------------------------------------------------------------------
// tensor-core mode of the fp16 trailing update (lu_mode = 1):
//   A22[i0:i0+128, j0:j0+256] = fl16(A22 - L21 U12) with the 32-wide panel
//   product on tcgen05 (fp16 operands, fp32 accumulator in TMEM).  Results are
//   rounded to u_f once per panel (north_star (1)); pivots then agree with the
//   exact mode up to near-ties.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void lu_tc_tile(__half* W, size_t ld, int n, int nc, int k0, int i0, int j0, unsigned char* sA,
                                           unsigned char* sB, uint64_t* mbar, uint32_t tmem, uint32_t& phase) {
  // Operands are staged with 16-byte shared-space stores (st.shared.v4 on
  // the 32-bit shared address: the aligned staging pointer has lost its
  // address space, so plain stores would be generic 2-byte ST.E).
  const uint32_t sa = tc::smem_u32(sA), sb = tc::smem_u32(sB);
  // A: L21 rows [i0, i0+128), panel columns [k0, k0+32): K-major already
  for (int e = threadIdx.x; e < 128 * 4; e += blockDim.x) {
    const int r = e >> 2, c = e & 3;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    const int gi = i0 + r;
    if (gi < n) v = *reinterpret_cast<const uint4*>(W + (size_t)gi * ld + k0 + c * 8);
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(sa + tc::sw64_off(r, c * 8)), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
  }
  // B: U12 rows [k0, k0+32), columns [j0, j0+256) transposed to K-major:
  // item (column nn, k-chunk kc) gathers the 8 panel rows kc*8..kc*8+7 of one
  // column (lanes take consecutive columns: coalesced 2-byte loads) into one
  // 16-byte K-major store
  for (int e = threadIdx.x; e < 256 * 4; e += blockDim.x) {
    const int nn = e & 255, kc = e >> 8;
    const int gj = j0 + nn;
    __align__(16) __half h[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) h[q] = gj < nc ? W[(size_t)(k0 + kc * 8 + q) * ld + gj] : __float2half(0.f);
    const uint4 v = *reinterpret_cast<const uint4*>(h);
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(sb + tc::sw64_off(nn, kc * 8)), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
  }
  tc::fence_proxy_async();
  __syncthreads();
  if (threadIdx.x == 0) {
    tc::fence_after();
    constexpr uint32_t idesc = tc::idesc_f16_f32(128, 256);
    const uint64_t ad = tc::desc_k64(tc::smem_u32(sA)), bd = tc::desc_k64(tc::smem_u32(sB));
    tc::mma_f16(tmem, ad, bd, idesc, 0u);
    tc::mma_f16(tmem, ad + 2, bd + 2, idesc, 1u);  // K = 16..31: +32 bytes inside the swizzle atom
    tc::commit(mbar);
  }
  tc::mbar_wait(mbar, phase);
  phase ^= 1u;
  tc::fence_after();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = (w & 3) * 32 + lane, gi = i0 + row;
  const int cbase = (w >> 2) * 128;
#pragma unroll 1
  for (int ch = 0; ch < 4; ++ch) {
    float acc[32];
    tc::tmem_ld32(tmem + ((uint32_t)((w & 3) * 32) << 16) + (uint32_t)(cbase + ch * 32), acc);
    const int gj = j0 + cbase + ch * 32;
    if (gi < n && gj < nc) {
      __half* p = W + (size_t)gi * ld + gj;
      if (gj + 32 <= nc) {
        __align__(16) __half h[32];
#pragma unroll
        for (int q = 0; q < 4; ++q) reinterpret_cast<uint4*>(h)[q] = reinterpret_cast<const uint4*>(p)[q];
#pragma unroll
        for (int q = 0; q < 32; ++q) h[q] = __float2half_rn(__half2float(h[q]) - acc[q]);
#pragma unroll
        for (int q = 0; q < 4; ++q) reinterpret_cast<uint4*>(p)[q] = reinterpret_cast<const uint4*>(h)[q];
      } else {
        for (int q = 0; q < 32 && gj + q < nc; ++q) p[q] = __float2half_rn(__half2float(p[q]) - acc[q]);
      }
    }
  }
  tc::fence_before();
  __syncthreads();
}

template <int M, class Team, class TA>
__device__ void lu_team(Team& t, const TA* A, size_t lda, typename LuT<M>::S* W, size_t ld, int n, int* perm,
                        LuStatus* st, LuWork wk, void* smem_raw, int tcmode = 0, int cbeg = 0, int cend = -1,
                        int* ipiv_all = nullptr) {
  // Column window [cbeg, cend) (multiples of 32, or cend = n): the blocked
  // tensor mode factors one wide panel per launch -- interchanges, U12 and the
  // rank-32 updates stay inside the window, the pivot rows are recorded in
  // ipiv_all for the host-side pass over the other columns.  The default
  // window is the whole matrix (one launch = the whole factorisation).
  if (cend < 0) cend = n;
  using L = LuT<M>;
  using C = typename L::C;
  constexpr int NB = kLuNB;
  const int G = t.size(), r = t.rank();
  const int sl_max = (n + G - 1) / G;
  C* P = reinterpret_cast<C*>(smem_raw);
  C* pivrow = P + (size_t)sl_max * 33;
  C* rowkv = pivrow + 32;
  C* l11 = rowkv + 32;
  C* ls = l11 + 32 * 33;
  C* us = ls + 64 * 33;
  __shared__ PivKey pscr[32];
  __shared__ int s_p, s_win;
  __shared__ double s_red[32];
  __shared__ uint32_t s_tmem;
  // tensor-core staging (TC mode, fp16 only)
  const size_t simt_bytes = sizeof(C) * ((size_t)sl_max * 33 + 64 + 32 * 33 + 64 * 33 + 32 * 65) + 64;
  unsigned char* tcbase = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + ((simt_bytes + 1023) & ~(size_t)1023) + 1023) & ~(uintptr_t)1023);
  unsigned char* sA = tcbase;
  unsigned char* sB = tcbase + 8192;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(tcbase + 8192 + 16384);
  const bool use_tc = (M == MODE_H16) && tcmode != 0;
  uint32_t tphase = 0;
  if (use_tc) {
    if (threadIdx.x < 32) tc::tmem_alloc(&s_tmem, 256);
    if (threadIdx.x == 0) tc::mbar_init(mbar, 1);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
  }
  const int nthr = G * blockDim.x;
  const int gtid = r * blockDim.x + threadIdx.x;
  // W = fl_uf(A), amax, identity permutation
  if (cbeg == 0) {
    int lo, hi;
    t.rows(n, lo, hi);
    double m = 0.0;
    for (int i = lo; i < hi; ++i)
      for (int j = threadIdx.x; j < n; j += blockDim.x) {
        typename L::S s = L::from_u((double)A[(size_t)i * lda + j]);
        W[(size_t)i * ld + j] = s;
        const double v = fabs((double)L::ld(s));
        m = (v > m || v != v) ? v : m;
      }
    m = block_max(m, s_red);
    if (threadIdx.x == 0) atomic_max_abs(&st->amax_bits, m);
    for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) perm[i] = i;
  }
  t.sync();
  for (int k0 = cbeg; k0 < cend; k0 += NB) {
    const int kend = min(cend, k0 + NB), pw = kend - k0;
    const int sl = (n - k0 + G - 1) / G;
    const int p0 = min(n, k0 + r * sl), p1 = min(n, p0 + sl);
    // ---- P: panel rows into shared memory
    for (int e = threadIdx.x; e < (p1 - p0) * pw; e += blockDim.x) {
      const int rr = e / pw, c = e % pw;
      P[rr * 33 + c] = L::ld(W[(size_t)(p0 + rr) * ld + k0 + c]);
    }
    __syncthreads();
    for (int c = 0; c < pw; ++c) {
      const int k = k0 + c, par = c & 1;
      PivKey key{0.0, -1, 0};
      for (int i = max(p0, k) + threadIdx.x; i < p1; i += blockDim.x) {
        PivKey cand = make_key((double)P[(i - p0) * 33 + c], i);
        if (piv_better(cand, key)) key = cand;
      }
      key = block_pivot(key, pscr);
      if (threadIdx.x == 0) wk.ckey[par * G + r] = key;
      if (key.i >= 0)
        for (int cc = threadIdx.x; cc < pw; cc += blockDim.x)
          wk.crow[((size_t)par * G + r) * 32 + cc] = (double)P[(key.i - p0) * 33 + cc];
      if (k >= p0 && k < p1)
        for (int cc = threadIdx.x; cc < pw; cc += blockDim.x) wk.rowk[par * 32 + cc] = (double)P[(k - p0) * 33 + cc];
      t.sync();
      if (threadIdx.x < 32) {
        PivKey best{0.0, -1, 0};
        int bw = -1;
        for (int g = threadIdx.x; g < G; g += 32) {
          PivKey q = key;
          if constexpr (Team::kGrid) {
            const PivKey* src = wk.ckey + par * G + g;
            q.v = __ldcg(&src->v);
            q.i = __ldcg(&src->i);
            q.nan = __ldcg(&src->nan);
          }
          if (piv_better(q, best)) {
            best = q;
            bw = g;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          PivKey q = piv_shfl(best, o);
          int qw = __shfl_xor_sync(0xffffffffu, bw, o);
          if (piv_better(q, best)) {
            best = q;
            bw = qw;
          }
        }
        if (threadIdx.x == 0) {
          s_p = best.i;
          s_win = bw;
        }
      }
      __syncthreads();
      const int p = s_p, win = s_win;
      for (int cc = threadIdx.x; cc < pw; cc += blockDim.x) {
        pivrow[cc] = (C)__ldcg(wk.crow + ((size_t)par * G + win) * 32 + cc);
        rowkv[cc] = (C)__ldcg(wk.rowk + par * 32 + cc);
      }
      __syncthreads();
      const C pv = pivrow[c];
      const bool isz = (pv == C(0));
      if (t.leader() && threadIdx.x == 0) {
        if (isz) atomicMin(&st->zero_col, k);
        const bool swap = (p != k) && !(isz && L::kLapack);
        wk.piv[c] = swap ? p : k;
        if (ipiv_all != nullptr) ipiv_all[k] = swap ? p : k;
        if (swap) {
          int tmp = perm[k];
          perm[k] = perm[p];
          perm[p] = tmp;
        }
      }
      if (isz && L::kLapack) {
        __syncthreads();
        continue;
      }
      if (p != k) {
        if (p >= p0 && p < p1)
          for (int cc = threadIdx.x; cc < pw; cc += blockDim.x) P[(p - p0) * 33 + cc] = rowkv[cc];
        if (k >= p0 && k < p1)
          for (int cc = threadIdx.x; cc < pw; cc += blockDim.x) P[(k - p0) * 33 + cc] = pivrow[cc];
      }
      __syncthreads();
      for (int i = max(p0, k + 1) + threadIdx.x; i < p1; i += blockDim.x) {
        C* row = P + (i - p0) * 33;
        const C lm = L::mult(row[c], pv);
        row[c] = lm;
        for (int j = c + 1; j < pw; ++j) row[j] = L::upd(row[j], lm, pivrow[j]);
      }
      __syncthreads();
    }
    for (int e = threadIdx.x; e < (p1 - p0) * pw; e += blockDim.x) {
      const int rr = e / pw, c = e % pw;
      W[(size_t)(p0 + rr) * ld + k0 + c] = L::st(P[rr * 33 + c]);
    }
    t.sync();
    // ---- S: interchanges outside the panel
    for (int idx = gtid; idx < cend - cbeg - pw; idx += nthr) {
      const int j = cbeg + idx < k0 ? cbeg + idx : cbeg + idx + pw;
      for (int c = 0; c < pw; ++c) {
        const int p = __ldcg(wk.piv + c);
        if (p != k0 + c) {
          auto tmp = W[(size_t)(k0 + c) * ld + j];
          W[(size_t)(k0 + c) * ld + j] = W[(size_t)p * ld + j];
          W[(size_t)p * ld + j] = tmp;
        }
      }
    }
    t.sync();
    if (kend >= cend) break;
    // ---- T: U12 = L11^-1 A12
    for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
      const int rr = e / NB, c = e % NB;
      l11[rr * 33 + c] = (rr < pw && c < pw) ? L::ld(W[(size_t)(k0 + rr) * ld + k0 + c]) : C(0);
    }
    __syncthreads();
    for (int j = kend + gtid; j < cend; j += nthr) {
      C col[NB];
#pragma unroll
      for (int rr = 0; rr < NB; ++rr) col[rr] = rr < pw ? L::ld(W[(size_t)(k0 + rr) * ld + j]) : C(0);
#pragma unroll
      for (int rr = 1; rr < NB; ++rr) {
#pragma unroll
        for (int i = 0; i < rr; ++i) col[rr] = L::upd(col[rr], l11[rr * 33 + i], col[i]);
      }
#pragma unroll
      for (int rr = 0; rr < NB; ++rr)
        if (rr < pw) W[(size_t)(k0 + rr) * ld + j] = L::st(col[rr]);
    }
    t.sync();
    // ---- G: trailing update over the team
    const int rest = n - kend, crest = cend - kend;
    if constexpr (M == MODE_H16) {
      if (use_tc && pw == NB) {
        const int ntr = (rest + 127) / 128, ntc = (crest + 255) / 256;
        for (int tt = r; tt < ntr * ntc; tt += G)
          lu_tc_tile(reinterpret_cast<__half*>(W), ld, n, cend, k0, kend + (tt / ntc) * 128, kend + (tt % ntc) * 256,
                     sA, sB, mbar, s_tmem, tphase);
        t.sync();
        continue;
      }
    }
    const int ntr = (rest + 63) / 64, ntc = (crest + 63) / 64;
    for (int tt = r; tt < ntr * ntc; tt += G) {
      const int ti = tt / ntc, tj = tt % ntc;
      lu_gemm_tile<M>(W, ld, n, cend, k0, kend + ti * 64, kend + tj * 64, ls, us);
    }
    t.sync();
  }
  if (use_tc) {
    tc::fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tc::tmem_dealloc(s_tmem, 256);
  }
  // growth numerator max|U| over this CTA's rows
  if (cend >= n) {
    int lo, hi;
    t.rows(n, lo, hi);
    double m = 0.0;
    for (int i = lo; i < hi; ++i)
      for (int j = i + threadIdx.x; j < n; j += blockDim.x) {
        const double v = fabs((double)L::ld(W[(size_t)i * ld + j]));
        m = (v > m || v != v) ? v : m;
      }
    m = block_max(m, s_red);
    if (threadIdx.x == 0) atomic_max_abs(&st->umax_bits, m);
  }
}

template <int M, class TA, class Team>
__global__ void __launch_bounds__(256) k_lu_team(const TA* A, size_t lda, typename LuT<M>::S* W, size_t ld, int n,
                                                 int* perm, LuStatus* st, LuWork wk, GridCtl* ctl, double* part,
                                                 int tcmode, int cbeg, int cend, int* ipiv_all) {
  extern __shared__ __align__(1024) unsigned char smem_lu[];
  Team t;
  if constexpr (Team::kGrid) t = Team{(int)gridDim.x, (int)blockIdx.x, ctl, part, 64, 0u};
  lu_team<M>(t, A, lda, W, ld, n, perm, st, wk, smem_lu, tcmode, cbeg, cend, ipiv_all);
}

// ---------------------------------------------------------------------------
// blocked tensor mode, host-driven (gb_solver.cuh lu_run_blocked): after a
// wide panel [c0, c0 + w) has been factored in its window,
//   k_lu_apply_pivots   the panel's row interchanges on the columns outside it
//   k_lu_trsm32         the 32-row base case of U12 = L11^-1 A12 (exact
//                       per-element order, as phase T above); the levels above
//                       it and the trailing update run on tcgen05
//                       (gb_tcgemm.cuh)
// ---------------------------------------------------------------------------
template <class S>
__global__ void k_lu_apply_pivots(S* W, size_t ld, int n, int c0, int w, const int* __restrict__ ipiv) {
  const int nout = n - w;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < nout; idx += gridDim.x * blockDim.x) {
    const int j = idx < c0 ? idx : idx + w;
    for (int k = c0; k < c0 + w; ++k) {
      const int p = __ldg(ipiv + k);
      if (p != k) {
        const S a = W[(size_t)k * ld + j];
        W[(size_t)k * ld + j] = W[(size_t)p * ld + j];
        W[(size_t)p * ld + j] = a;
      }
    }
  }
}

// rows [r0, r0 + 32) of columns [c0, c0 + N): X = L11^-1 X with the unit lower
// 32 x 32 block L11 = W[r0:r0+32, r0:r0+32]
template <int M>
__global__ void __launch_bounds__(256) k_lu_trsm32(typename LuT<M>::S* W, size_t ld, int r0, int c0, int N) {
  using L = LuT<M>;
  using C = typename L::C;
  constexpr int NB = 32;
  __shared__ C l11[NB * 33];
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int rr = e / NB, c = e % NB;
    l11[rr * 33 + c] = L::ld(W[(size_t)(r0 + rr) * ld + r0 + c]);
  }
  __syncthreads();
  for (int j = c0 + blockIdx.x * blockDim.x + threadIdx.x; j < c0 + N; j += gridDim.x * blockDim.x) {
    C col[NB];
#pragma unroll
    for (int rr = 0; rr < NB; ++rr) col[rr] = L::ld(W[(size_t)(r0 + rr) * ld + j]);
#pragma unroll
    for (int rr = 1; rr < NB; ++rr) {
#pragma unroll
      for (int i = 0; i < rr; ++i) col[rr] = L::upd(col[rr], l11[rr * 33 + i], col[i]);
    }
#pragma unroll
    for (int rr = 0; rr < NB; ++rr) W[(size_t)(r0 + rr) * ld + j] = L::st(col[rr]);
  }
}

}  // namespace gb
