// Solver object, kernels and the per-variant implementation (Impl).  Each
// precision variant is instantiated in its own translation unit
// (gb_var_*.cu) so the variants compile in parallel; gb_capi.cu holds the
// extern "C" entry points and the dispatch.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "gb_refine.cuh"
#pragma once

using namespace gb;

static thread_local std::string g_err;

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      g_err = std::string(#x) + ": " + cudaGetErrorString(e_);                 \
      return GB_ERR_CUDA;                                                      \
    }                                                                          \
  } while (0)

static gb_status fail(gb_status s, const std::string& m) {
  g_err = m;
  return s;
}

namespace {

constexpr int kThreads = 256;
constexpr int kSmallN = 256;  // <= : one CTA per system

template <class TF>
struct UfMode;
template <>
struct UfMode<__half> {
  static constexpr int M = MODE_H16;
};
template <>
struct UfMode<float> {
  static constexpr int M = MODE_F32;
};
template <>
struct UfMode<double> {
  static constexpr int M = MODE_F64;
};

template <class TW>
GB_DEVICE TW fl_add(TW a, TW b);
template <>
GB_DEVICE float fl_add<float>(float a, float b) { return __fadd_rn(a, b); }
template <>
GB_DEVICE double fl_add<double>(double a, double b) { return __dadd_rn(a, b); }

enum { METH_SIR = 0, METH_GMRES = 1, METH_GCRODR = 2 };

template <class TW, class TF, int MV>
struct Prob {
  Krylov<TW, TW, TF, MV> K;
  const TW* b;
  TW* xs;
  double* r;
  double* xref;
  int* has_xref;
  double normA, normB;
  int ur, method;
  unsigned long long* ctr;    // [2]
  unsigned long long* epoch;  // [1]
  GridCtl* ctl;
  double* partials;
  int kmax;
  gb_step_info* out;
  int* flags;  // [0] x0_reset
  // xref (large n): fp64 factors
  const double* LUx;
  const int* permx;
  double* rtmp;
  double* dtmp;
};

template <class Team>
struct MakeTeam;
template <>
struct MakeTeam<CtaTeam> {
  template <class P>
  GB_DEVICE static CtaTeam make(const P&) { return CtaTeam{}; }
};
template <>
struct MakeTeam<GridTeam> {
  template <class P>
  GB_DEVICE static GridTeam make(const P& p) {
    return GridTeam{(int)gridDim.x, (int)blockIdx.x, p.ctl, p.partials, p.kmax, 0u};
  }
};

__host__ __device__ inline size_t sm_doubles(int m, int k) { return (size_t)5 * m + 2 * k + 512; }

template <class TW, class TF, int MV>
__host__ __device__ inline size_t ops_bytes() {
  size_t a = trsv_smem_bytes<MV, TF>(kThreads);
  size_t b = trsv_smem_bytes<UfMode<TF>::M, TF>(kThreads);
  size_t c = trsv_smem_bytes<MODE_F64, double>(kThreads);
  return std::max(a, std::max(b, c));
}

// ---------------------------------------------------------------------------
// device bodies
// ---------------------------------------------------------------------------
template <class TW, class TF, int MV, class Team>
__device__ void x0_body(Team& t, Prob<TW, TF, MV>& P, double* sm, void* ops) {
  constexpr int UM = UfMode<TF>::M;
  auto& K = P.K;
  TrsvSync ts{P.ctr, P.ctr + 1, *P.epoch};
  double* red = sm + 4 * K.m + 4;
  t.sync();
  op_apply<UM>(t, K.sys, (const TW*)nullptr, P.b, P.xs, reinterpret_cast<typename Arith<UM>::T*>(K.ybuf), ts,
               ops);
  int lo, hi;
  t.rows(K.n, lo, hi);
  double bad = 0.0;
  for (int i = lo + threadIdx.x; i < hi; i += blockDim.x)
    if (!isfinite((double)P.xs[i])) bad = 1.0;
  bad = block_max(bad, red);
  bad = t.finish_max(bad);
  if (bad != 0.0) {
    for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) P.xs[i] = TW(0);
  }
  t.sync();
  residual_check(t, K.sys.A, K.sys.lda, K.n, (const TW*)P.xs, P.b, P.r, P.ur, P.normA, P.normB, red);
  if (t.leader() && threadIdx.x == 0) {
    P.flags[0] = bad != 0.0;
    *P.epoch = ts.epoch;
  }
}

template <class TW, class TF, int MV, class Team>
__device__ void step_body(Team& t, Prob<TW, TF, MV>& P, double* sm, void* ops) {
  using F = Fmt<TW>;
  constexpr int UM = UfMode<TF>::M;
  auto& K = P.K;
  TrsvSync ts{P.ctr, P.ctr + 1, *P.epoch};
  double* red = sm + 4 * K.m + 4;
  const int n = K.n;
  int lo, hi;
  t.rows(n, lo, hi);
  gb_step_info info;
  memset(&info, 0, sizeof(info));
  t.sync();
  const double nu = team_amax<double>(t, P.r, n, red);
  info.nu = nu;
  if (nu == 0.0 || !isfinite(nu)) {
    info.status = (nu == 0.0) ? RS_NU_ZERO : RS_NU_NONFINITE;
    info.ferr = P.has_xref[0] ? forward_error(t, (const TW*)P.xs, P.xref, n, red) : NAN;
    if (t.leader() && threadIdx.x == 0) *P.out = info;
    return;
  }
  for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) K.rhat[i] = (TW)F::rnd(P.r[i] / nu);
  StepScalars st{0, KS_CONVERGED, 0, 0};
  if (P.method == METH_SIR) {
    t.sync();
    op_apply<UM>(t, K.sys, (const TW*)nullptr, (const TW*)K.rhat, K.x,
                 reinterpret_cast<typename Arith<UM>::T*>(K.ybuf), ts, ops);
    st.ncycles = 1;
    if (t.leader() && threadIdx.x == 0) K.cycle_iters[0] = 1;
  } else {
    st = inner_solve(t, K, ts, sm, ops);
  }
  int its = 0;
  if (P.method == METH_SIR) {
    its = 1;
  } else {
    // sum of per-cycle steps (leader wrote them; broadcast through global)
    t.sync();
    for (int c = 0; c < st.ncycles; ++c) its += __ldcg(K.cycle_iters + c);
  }
  for (int i = lo + threadIdx.x; i < hi; i += blockDim.x)
    P.xs[i] = fl_add<TW>(P.xs[i], F::scale(nu, K.x[i]));
  t.sync();
  info.ferr = P.has_xref[0] ? forward_error(t, (const TW*)P.xs, P.xref, n, red) : NAN;
  ResidOut ro = residual_check(t, K.sys.A, K.sys.lda, n, (const TW*)P.xs, P.b, P.r, P.ur, P.normA, P.normB, red);
  info.nbe = ro.nbe;
  info.cbe = ro.cbe;
  info.inner_iters = its;
  info.ncycles = st.ncycles;
  info.status = st.status;
  info.applies = st.applies;
  info.keff = st.keff;
  if (t.leader() && threadIdx.x == 0) {
    *P.out = info;
    *P.epoch = ts.epoch;
  }
}

// xref for n > 600 (refine.py:251-256): fp64 LU solve + 4 dd-residual sweeps
template <class TW, class TF, int MV, class Team>
__device__ void xref_refine_body(Team& t, Prob<TW, TF, MV>& P, double* sm, void* ops) {
  auto& K = P.K;
  TrsvSync ts{P.ctr, P.ctr + 1, *P.epoch};
  double* red = sm + 4 * K.m + 4;
  const int n = K.n;
  SysView<TW, double> sx{n, K.sys.lda, K.sys.A, K.sys.lda, P.LUx, P.permx};
  auto* yb = reinterpret_cast<double*>(K.ybuf);
  t.sync();
  op_apply<MODE_F64>(t, sx, (const TW*)nullptr, P.b, P.xref, yb, ts, ops);
  int lo, hi;
  t.rows(n, lo, hi);
  for (int it = 0; it < 4; ++it) {
    residual_check(t, K.sys.A, K.sys.lda, n, (const double*)P.xref, P.b, P.rtmp, UR_DD, 1.0, 1.0, red);
    t.sync();
    op_apply<MODE_F64>(t, sx, (const TW*)nullptr, (const double*)P.rtmp, P.dtmp, yb, ts, ops);
    for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) P.xref[i] = __dadd_rn(P.xref[i], P.dtmp[i]);
    t.sync();
  }
  double bad = 0.0;
  for (int i = lo + threadIdx.x; i < hi; i += blockDim.x)
    if (!isfinite(P.xref[i])) bad = 1.0;
  bad = block_max(bad, red);
  bad = t.finish_max(bad);
  if (t.leader() && threadIdx.x == 0) {
    P.has_xref[0] = bad == 0.0;
    *P.epoch = ts.epoch;
  }
}

// kernel-level debug ops (one vector): what 0 = apply, 1 = precond_rhs,
// 2 = residual (ur in P.ur), 3 = lu_solve (u_f); input in rtmp (fp64)
template <int M, class TW, class TF, int MV, class Team>
__device__ void debug_body(Team& t, Prob<TW, TF, MV>& P, double* sm, void* ops, int what) {
  auto& K = P.K;
  TrsvSync ts{P.ctr, P.ctr + 1, *P.epoch};
  double* red = sm + 4 * K.m + 4;
  const int n = K.n;
  int lo, hi;
  t.rows(n, lo, hi);
  auto* yb = reinterpret_cast<typename Arith<M>::T*>(K.ybuf);
  // input rounded to u as the reference's callers hold it
  for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) K.rhat[i] = (TW)P.rtmp[i];
  t.sync();
  if (what == 0) {
    op_apply<M>(t, K.sys, (const TW*)K.rhat, (const TW*)nullptr, K.w, yb, ts, ops);
  } else if (what == 1 || what == 3) {
    op_apply<M>(t, K.sys, (const TW*)nullptr, (const TW*)K.rhat, K.w, yb, ts, ops);
  } else {
    residual_check(t, K.sys.A, K.sys.lda, n, (const TW*)K.rhat, P.b, P.dtmp, P.ur, 1.0, 1.0, red);
  }
  t.sync();
  if (what != 2)
    for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) P.dtmp[i] = (double)K.w[i];
  if (t.leader() && threadIdx.x == 0) *P.epoch = ts.epoch;
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
template <class TW, class TF, int MV, class Team>
__global__ void __launch_bounds__(kThreads) k_x0(Prob<TW, TF, MV> Pin) {
  extern __shared__ __align__(16) unsigned char smem[];
  Prob<TW, TF, MV> P = Pin;
  Team t = MakeTeam<Team>::make(P);
  double* sm = reinterpret_cast<double*>(smem);
  void* ops = smem + sm_doubles(P.K.m, P.K.k) * sizeof(double);
  x0_body(t, P, sm, ops);
}

template <class TW, class TF, int MV, class Team>
__global__ void __launch_bounds__(kThreads) k_step(Prob<TW, TF, MV> Pin) {
  extern __shared__ __align__(16) unsigned char smem[];
  Prob<TW, TF, MV> P = Pin;
  Team t = MakeTeam<Team>::make(P);
  double* sm = reinterpret_cast<double*>(smem);
  void* ops = smem + sm_doubles(P.K.m, P.K.k) * sizeof(double);
  step_body(t, P, sm, ops);
  if (t.leader() && threadIdx.x == 0) P.K.keff_io[1] = (P.K.U == Pin.K.U) ? 0 : 1;
}

template <class TW, class TF, int MV, class Team>
__global__ void __launch_bounds__(kThreads) k_xref_refine(Prob<TW, TF, MV> Pin) {
  extern __shared__ __align__(16) unsigned char smem[];
  Prob<TW, TF, MV> P = Pin;
  Team t = MakeTeam<Team>::make(P);
  double* sm = reinterpret_cast<double*>(smem);
  void* ops = smem + sm_doubles(P.K.m, P.K.k) * sizeof(double);
  xref_refine_body(t, P, sm, ops);
}

template <int M, class TW, class TF, int MV, class Team>
__global__ void __launch_bounds__(kThreads) k_debug(Prob<TW, TF, MV> Pin, int what) {
  extern __shared__ __align__(16) unsigned char smem[];
  Prob<TW, TF, MV> P = Pin;
  Team t = MakeTeam<Team>::make(P);
  double* sm = reinterpret_cast<double*>(smem);
  void* ops = smem + sm_doubles(P.K.m, P.K.k) * sizeof(double);
  debug_body<M>(t, P, sm, ops, what);
}

// dd GEPP xref (n <= 600) by one CTA
template <class TW>
__global__ void __launch_bounds__(kThreads) k_xref_small(const TW* A, size_t lda, const TW* b, int n, double* ah,
                                                      double* al, double* yh, double* yl, int* perm, double* xref,
                                                      int* ok) {
  __shared__ PivKey pscr[32];
  bool r = dd_gepp_solve(A, lda, b, n, ah, al, yh, yl, perm, xref, pscr);
  if (threadIdx.x == 0) *ok = r ? 1 : 0;
}

// A_u = fl_u(a), b_u = fl_u(b); row sums of |A_u| and max|b_u|
template <class TW>
__global__ void k_set_system(const double* __restrict__ a, int n, TW* A, size_t lda, const double* bsrc, TW* b,
                             unsigned long long* norms) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  double rowmax = 0.0, bmax = 0.0;
  for (int i = warp; i < n; i += nwarps) {
    double s = 0.0;
    for (int j = lane; j < n; j += 32) {
      TW v = (TW)a[(size_t)i * n + j];
      A[(size_t)i * lda + j] = v;
      s += fabs((double)v);
    }
    s = warp_sum(s);
    rowmax = (s > rowmax || s != s) ? s : rowmax;
    if (lane == 0) {
      TW bv = (TW)bsrc[i];
      b[i] = bv;
      double ab = fabs((double)bv);
      bmax = (ab > bmax || ab != ab) ? ab : bmax;
    }
  }
  if (lane == 0) {
    atomic_max_abs(&norms[0], rowmax);
    atomic_max_abs(&norms[1], bmax);
  }
}

template <class TF>
__global__ void k_copy_lu_to_f64(const TF* W, size_t ld, int n, double* out) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < (size_t)n * n; e += (size_t)gridDim.x * blockDim.x)
    out[e] = to_d(W[(e / n) * ld + e % n]);
}

template <class TW>
__global__ void k_to_f64(const TW* x, int n, double* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = (double)x[i];
}

// one-CTA LU for small n (smem carrier), then stored at u_f width
template <int M, class TW>
__global__ void __launch_bounds__(kThreads) k_lu_small(const TW* A, size_t lda, typename LuT<M>::S* W, size_t ldw,
                                                    int n, int* perm, LuStatus* st) {
  using L = LuT<M>;
  using C = typename L::C;
  extern __shared__ __align__(16) unsigned char smem[];
  C* a = reinterpret_cast<C*>(smem);
  __shared__ PivKey pscr[32];
  double am = 0.0;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    C v = L::ld(L::from_u((double)A[(size_t)(e / n) * lda + e % n]));
    a[e] = v;
    double x = fabs((double)v);
    am = (x > am || x != x) ? x : am;
  }
  am = warp_max(am);
  if ((threadIdx.x & 31) == 0) atomic_max_abs(&st->amax_bits, am);
  __syncthreads();
  int z = lu_cta<M>(a, n, n, perm, pscr);
  double um = 0.0;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    int i = e / n, j = e % n;
    W[(size_t)i * ldw + j] = L::st(a[e]);
    if (j >= i) {
      double x = fabs((double)a[e]);
      um = (x > um || x != x) ? x : um;
    }
  }
  um = warp_max(um);
  if ((threadIdx.x & 31) == 0) atomic_max_abs(&st->umax_bits, um);
  if (threadIdx.x == 0 && z >= 0) atomicMin(&st->zero_col, z);
}

// ---------------------------------------------------------------------------
// arena
// ---------------------------------------------------------------------------
struct Arena {
  char* base = nullptr;
  size_t off = 0, cap = 0;
  template <class T>
  T* take(size_t count) {
    size_t bytes = count * sizeof(T);
    off = (off + 255) & ~size_t(255);
    T* p = reinterpret_cast<T*>(base + off);
    off += bytes;
    return p;
  }
};

}  // namespace

// ---------------------------------------------------------------------------
// solver object
// ---------------------------------------------------------------------------
struct VariantOps;

struct gb_solver {
  int n = 0, ldv = 0, lda = 0, G = 1;
  gb_options o{};
  cudaStream_t stream = nullptr;
  void* mem = nullptr;
  size_t mem_bytes = 0;
  const VariantOps* ops = nullptr;
  // typed pointers stored type-erased
  void *A = nullptr, *b = nullptr, *LU = nullptr, *xs = nullptr;
  double* stage = nullptr;
  int *perm = nullptr, *piv = nullptr;
  LuStatus* lust = nullptr;
  double *r = nullptr, *xref = nullptr, *rtmp = nullptr, *dtmp = nullptr;
  void *V = nullptr, *w = nullptr, *xk = nullptr, *res = nullptr, *s = nullptr, *rhat = nullptr;
  void *C = nullptr, *U = nullptr, *Cn = nullptr, *Un = nullptr, *Ut = nullptr, *Yt = nullptr;
  double *Wd = nullptr, *Qd = nullptr, *H = nullptr, *R = nullptr, *B = nullptr, *bc = nullptr, *dense = nullptr,
         *gram = nullptr;
  size_t gram_stride = 0;
  void* ybuf = nullptr;
  unsigned long long *ctr = nullptr, *epoch = nullptr, *norms = nullptr;
  GridCtl* ctl = nullptr;
  double* partials = nullptr;
  int kmax = 0;
  int *cycle_iters = nullptr, *cycle_keff = nullptr, *keff_io = nullptr, *flags = nullptr, *has_xref = nullptr;
  gb_step_info* out = nullptr;
  // xref workspace
  double *xa = nullptr, *xb = nullptr, *xyh = nullptr, *xyl = nullptr;
  int *xperm = nullptr, *xpiv = nullptr;
  LuStatus* xst = nullptr;
  double normA = 0, normB = 0;
  int parity = 0;
  bool have_system = false, have_lu = false, have_x0 = false;
  float last_step_ms = 0, last_factor_ms = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};

struct VariantOps {
  gb_status (*setup)(gb_solver*);
  gb_status (*set_system)(gb_solver*, const double*, const double*);
  gb_status (*factor)(gb_solver*, int*, double*);
  gb_status (*x0)(gb_solver*, int*);
  gb_status (*xref)(gb_solver*, int*);
  gb_status (*step)(gb_solver*, gb_step_info*);
  gb_status (*debug)(gb_solver*, const double*, double*, int what, int fmt);
  gb_status (*get_x)(gb_solver*, double*);
  gb_status (*get_lu)(gb_solver*, double*, long long*);
};

namespace {

template <class K>
gb_status set_smem(K kern, size_t bytes) {
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  return GB_OK;
}

template <class TW, class TF, int MV>
struct Impl {
  using P_t = Prob<TW, TF, MV>;
  static constexpr int UM = UfMode<TF>::M;

  static P_t make(gb_solver* s) {
    P_t P;
    memset(&P, 0, sizeof(P));
    auto& K = P.K;
    K.n = s->n;
    K.ldv = s->ldv;
    K.m = s->o.m;
    K.k = s->o.k;
    K.max_cycles = s->o.max_cycles;
    K.tau = s->o.tau;
    K.reorth = s->o.reorthogonalize;
    K.recycling = (s->o.method == GB_RGMRES_IR || s->o.method == GB_RSGMRES_IR);
    K.sys = SysView<TW, TF>{s->n, (size_t)s->lda, (const TW*)s->A, (size_t)s->lda, (const TF*)s->LU, s->perm};
    K.V = (TW*)s->V;
    K.w = (TW*)s->w;
    K.x = (TW*)s->xk;
    K.res = (TW*)s->res;
    K.s = (TW*)s->s;
    K.rhat = (TW*)s->rhat;
    K.C = (TW*)s->C;
    K.U = (TW*)s->U;
    K.Cn = (TW*)s->Cn;
    K.Un = (TW*)s->Un;
    if (s->parity) {
      std::swap(K.C, K.Cn);
      std::swap(K.U, K.Un);
    }
    K.Ut = (TW*)s->Ut;
    K.Yt = (TW*)s->Yt;
    K.Wd = s->Wd;
    K.Qd = s->Qd;
    K.H = s->H;
    K.R = s->R;
    K.B = s->B;
    K.bc = s->bc;
    K.dense = s->dense;
    K.gram = s->gram;
    K.gram_stride = s->gram_stride;
    K.ybuf = (typename Arith<MV>::T*)s->ybuf;
    K.cycle_iters = s->cycle_iters;
    K.cycle_keff = s->cycle_keff;
    K.keff_io = s->keff_io;
    P.b = (const TW*)s->b;
    P.xs = (TW*)s->xs;
    P.r = s->r;
    P.xref = s->xref;
    P.has_xref = s->has_xref;
    P.normA = s->normA;
    P.normB = s->normB;
    P.ur = s->o.ur == GB_QUAD ? UR_DD : (s->o.ur == GB_DOUBLE ? UR_F64 : UR_F32);
    P.method = s->o.method == GB_SIR ? METH_SIR
               : (s->o.method == GB_GMRES_IR || s->o.method == GB_SGMRES_IR) ? METH_GMRES
                                                                              : METH_GCRODR;
    P.ctr = s->ctr;
    P.epoch = s->epoch;
    P.ctl = s->ctl;
    P.partials = s->partials;
    P.kmax = s->kmax;
    P.out = s->out;
    P.flags = s->flags;
    P.LUx = s->xa;
    P.permx = s->xperm;
    P.rtmp = s->rtmp;
    P.dtmp = s->dtmp;
    return P;
  }

  static size_t smem_bytes(gb_solver* s) {
    return sm_doubles(s->o.m, s->o.k) * sizeof(double) + ops_bytes<TW, TF, MV>();
  }

  template <class KernT, class... Args>
  static gb_status launch(gb_solver* s, KernT kern, Args... args) {
    size_t sm = smem_bytes(s);
    gb_status st = set_smem(kern, sm);
    if (st != GB_OK) return st;
    if (s->G == 1) {
      kern<<<1, kThreads, sm, s->stream>>>(args...);
      CK(cudaGetLastError());
    } else {
      void* argv[] = {(void*)&args...};
      CK(cudaLaunchCooperativeKernel((void*)kern, dim3(s->G), dim3(kThreads), argv, sm, s->stream));
    }
    return GB_OK;
  }

  static gb_status setup(gb_solver* s) {
    const int n = s->n, m = s->o.m, k = s->o.k, ldv = s->ldv, lda = s->lda;
    const int S = m + k + 2;
    s->gram_stride = (size_t)S * S;
    s->kmax = S + 64;
    Arena a;
    auto plan = [&](bool commit) {
      a.off = 0;
      s->A = a.take<TW>((size_t)n * lda);
      s->stage = a.take<double>((size_t)n * n);
      s->b = a.take<TW>(ldv);
      s->LU = a.take<TF>((size_t)n * lda);
      s->perm = a.take<int>(ldv);
      s->piv = a.take<int>(64);
      s->lust = a.take<LuStatus>(1);
      s->xs = a.take<TW>(ldv);
      s->r = a.take<double>(ldv);
      s->xref = a.take<double>(ldv);
      s->rtmp = a.take<double>(ldv);
      s->dtmp = a.take<double>(ldv);
      s->V = a.take<TW>((size_t)(m + 1) * ldv);
      s->w = a.take<TW>(ldv);
      s->xk = a.take<TW>(ldv);
      s->res = a.take<TW>(ldv);
      s->s = a.take<TW>(ldv);
      s->rhat = a.take<TW>(ldv);
      s->C = a.take<TW>((size_t)(k + 1) * ldv);
      s->U = a.take<TW>((size_t)(k + 1) * ldv);
      s->Cn = a.take<TW>((size_t)(k + 1) * ldv);
      s->Un = a.take<TW>((size_t)(k + 1) * ldv);
      s->Ut = a.take<TW>((size_t)(k + 1) * ldv);
      s->Yt = a.take<TW>((size_t)(k + 1) * ldv);
      s->Wd = a.take<double>((size_t)(k + 1) * ldv);
      s->Qd = a.take<double>((size_t)(k + 1) * ldv);
      s->H = a.take<double>((size_t)(m + 1) * m);
      s->R = a.take<double>((size_t)(m + 1) * m);
      s->B = a.take<double>((size_t)(k + 1) * m);
      s->bc = a.take<double>((size_t)3 * S + 2 * (size_t)S * (k + 2) + 2 * (size_t)(k + 1) * (k + 1) + 64);
      s->dense = a.take<double>((size_t)10 * S * S + 24 * (size_t)S * (k + 3) + 4096);
      s->gram = a.take<double>((size_t)(s->G + 1) * S * S);
      s->ybuf = a.take<double2>(ldv);
      s->ctr = a.take<unsigned long long>(4);
      s->epoch = a.take<unsigned long long>(2);
      s->norms = a.take<unsigned long long>(2);
      s->ctl = a.take<GridCtl>(1);
      s->partials = a.take<double>((size_t)2 * s->G * s->kmax);
      s->cycle_iters = a.take<int>(m * 0 + s->o.max_cycles + 4);
      s->cycle_keff = a.take<int>(s->o.max_cycles + 4);
      s->keff_io = a.take<int>(4);
      s->flags = a.take<int>(4);
      s->has_xref = a.take<int>(4);
      s->out = a.take<gb_step_info>(1);
      if (n <= 600) {
        s->xa = a.take<double>((size_t)n * n);
        s->xb = a.take<double>((size_t)n * n);
        s->xyh = a.take<double>(ldv);
        s->xyl = a.take<double>(ldv);
        s->xperm = a.take<int>(ldv);
      } else {
        s->xa = a.take<double>((size_t)n * lda);
        s->xperm = a.take<int>(ldv);
        s->xpiv = a.take<int>(64);
        s->xst = a.take<LuStatus>(1);
      }
      (void)commit;
    };
    a.base = nullptr;
    plan(false);
    size_t bytes = a.off + 4096;
    CK(cudaMalloc(&s->mem, bytes));
    s->mem_bytes = bytes;
    a.base = (char*)s->mem;
    plan(true);
    CK(cudaMemsetAsync(s->mem, 0, bytes, s->stream));
    return GB_OK;
  }

  static gb_status set_system(gb_solver* s, const double* a, const double* b) {
    const int n = s->n;
    double* bstage = s->rtmp;  // n doubles
    CK(cudaMemcpyAsync(s->stage, a, sizeof(double) * (size_t)n * n, cudaMemcpyHostToDevice, s->stream));
    CK(cudaMemcpyAsync(bstage, b, sizeof(double) * n, cudaMemcpyHostToDevice, s->stream));
    CK(cudaMemsetAsync(s->norms, 0, 2 * sizeof(unsigned long long), s->stream));
    int blocks = std::min(1184, std::max(1, (n + 7) / 8));
    k_set_system<TW><<<blocks, 256, 0, s->stream>>>(s->stage, n, (TW*)s->A, s->lda, bstage, (TW*)s->b, s->norms);
    CK(cudaGetLastError());
    unsigned long long nb[2];
    CK(cudaMemcpyAsync(nb, s->norms, sizeof(nb), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    memcpy(&s->normA, &nb[0], 8);
    memcpy(&s->normB, &nb[1], 8);
    // fresh recycle state / counters for a new system
    CK(cudaMemsetAsync(s->keff_io, 0, 4 * sizeof(int), s->stream));
    s->parity = 0;
    return GB_OK;
  }

  template <int M, class TA, class S>
  static gb_status lu_run(gb_solver* s, const TA* A, size_t lda, S* W, int* perm, int* piv, LuStatus* st) {
    const int n = s->n;
    LuStatus init{0x7fffffff, 0, 0ull, 0ull};
    CK(cudaMemcpyAsync(st, &init, sizeof(init), cudaMemcpyHostToDevice, s->stream));
    if (n <= 128 && M != MODE_F64) {
      size_t sm = (size_t)n * n * sizeof(typename LuT<M>::C);
      gb_status e = set_smem(k_lu_small<M, TA>, sm);
      if (e != GB_OK) return e;
      k_lu_small<M, TA><<<1, kThreads, sm, s->stream>>>(A, lda, W, s->lda, n, perm, st);
      CK(cudaGetLastError());
      return GB_OK;
    }
    constexpr int NB = 32;
    k_lu_convert<M, TA><<<1184, 256, 0, s->stream>>>(A, lda, W, s->lda, n, st);
    CK(cudaGetLastError());
    // identity permutation
    std::vector<int> id(n);
    for (int i = 0; i < n; ++i) id[i] = i;
    CK(cudaMemcpyAsync(perm, id.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    for (int k0 = 0; k0 < n; k0 += NB) {
      k_lu_panel<M><<<1, 1024, 0, s->stream>>>(W, s->lda, n, k0, NB, perm, piv, st);
      int outside = n - std::min(NB, n - k0);
      if (outside > 0) k_lu_laswp<M><<<(outside + 255) / 256, 256, 0, s->stream>>>(W, s->lda, n, k0, NB, piv);
      int rest = n - (k0 + NB);
      if (rest > 0) {
        k_lu_trsm<M, NB><<<std::min(1184, (rest + 127) / 128), 128, 0, s->stream>>>(W, s->lda, n, k0);
        dim3 g((rest + 63) / 64, (rest + 63) / 64);
        k_lu_gemm<M, NB><<<g, 256, 0, s->stream>>>(W, s->lda, n, k0);
      }
    }
    CK(cudaGetLastError());
    k_lu_umax<M><<<std::min(n, 1184), 256, 0, s->stream>>>(W, s->lda, n, st);
    CK(cudaGetLastError());
    return GB_OK;
  }

  static gb_status factor(gb_solver* s, int* zero_col, double* growth) {
    CK(cudaEventRecord(s->ev0, s->stream));
    gb_status e = lu_run<UM>(s, (const TW*)s->A, (size_t)s->lda, (typename LuT<UM>::S*)s->LU, s->perm, s->piv, s->lust);
    if (e != GB_OK) return e;
    CK(cudaEventRecord(s->ev1, s->stream));
    LuStatus h;
    CK(cudaMemcpyAsync(&h, s->lust, sizeof(h), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    CK(cudaEventElapsedTime(&s->last_factor_ms, s->ev0, s->ev1));
    *zero_col = h.zero_col == 0x7fffffff ? -1 : h.zero_col;
    double amax, umax;
    memcpy(&amax, &h.amax_bits, 8);
    memcpy(&umax, &h.umax_bits, 8);
    *growth = amax != 0.0 ? umax / amax : NAN;
    return GB_OK;
  }

  static gb_status x0(gb_solver* s, int* reset) {
    P_t P = make(s);
    gb_status e = s->G == 1 ? launch(s, k_x0<TW, TF, MV, CtaTeam>, P) : launch(s, k_x0<TW, TF, MV, GridTeam>, P);
    if (e != GB_OK) return e;
    int f = 0;
    CK(cudaMemcpyAsync(&f, s->flags, sizeof(int), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    *reset = f;
    return GB_OK;
  }

  static gb_status xref(gb_solver* s, int* ok) {
    const int n = s->n;
    if (n <= 600) {
      k_xref_small<TW><<<1, kThreads, 0, s->stream>>>((const TW*)s->A, s->lda, (const TW*)s->b, n, s->xa, s->xb,
                                                     s->xyh, s->xyl, s->xperm, s->xref, s->has_xref);
      CK(cudaGetLastError());
    } else {
      // fp64 GEPP of A (lu_factor(a, DOUBLE)) then the dd-residual refinement
      gb_status e = lu_run<MODE_F64>(s, (const TW*)s->A, (size_t)s->lda, s->xa, s->xperm, s->xpiv, s->xst);
      if (e != GB_OK) return e;
      LuStatus h;
      CK(cudaMemcpyAsync(&h, s->xst, sizeof(h), cudaMemcpyDeviceToHost, s->stream));
      CK(cudaStreamSynchronize(s->stream));
      if (h.zero_col != 0x7fffffff) {
        int z = 0;
        CK(cudaMemcpyAsync(s->has_xref, &z, sizeof(int), cudaMemcpyHostToDevice, s->stream));
        *ok = 0;
        return GB_OK;
      }
      P_t P = make(s);
      e = s->G == 1 ? launch(s, k_xref_refine<TW, TF, MV, CtaTeam>, P)
                    : launch(s, k_xref_refine<TW, TF, MV, GridTeam>, P);
      if (e != GB_OK) return e;
    }
    int f = 0;
    CK(cudaMemcpyAsync(&f, s->has_xref, sizeof(int), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    *ok = f;
    return GB_OK;
  }

  static gb_status step(gb_solver* s, gb_step_info* info) {
    P_t P = make(s);
    CK(cudaEventRecord(s->ev0, s->stream));
    gb_status e = s->G == 1 ? launch(s, k_step<TW, TF, MV, CtaTeam>, P) : launch(s, k_step<TW, TF, MV, GridTeam>, P);
    if (e != GB_OK) return e;
    CK(cudaEventRecord(s->ev1, s->stream));
    int kio[4];
    CK(cudaMemcpyAsync(info, s->out, sizeof(gb_step_info), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaMemcpyAsync(kio, s->keff_io, sizeof(kio), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    CK(cudaEventElapsedTime(&s->last_step_ms, s->ev0, s->ev1));
    if (kio[1]) s->parity ^= 1;
    return GB_OK;
  }

  static constexpr int op_format() {
    return MV == MODE_DD ? GB_QUAD : (MV == MODE_F64 ? GB_DOUBLE : (MV == MODE_F32 ? GB_SINGLE : GB_HALF));
  }

  static gb_status debug(gb_solver* s, const double* in, double* out, int what, int fmt) {
    const int n = s->n;
    CK(cudaMemcpyAsync(s->rtmp, in, sizeof(double) * n, cudaMemcpyHostToDevice, s->stream));
    P_t P = make(s);
    gb_status e = GB_OK;
    auto go = [&](auto kc, auto kg) { return s->G == 1 ? launch(s, kc, P, what) : launch(s, kg, P, what); };
    if (what == 2) {
      // residual(a, x, b, ctx): the mode template is irrelevant for it
      P.ur = fmt == GB_QUAD ? UR_DD : (fmt == GB_DOUBLE ? UR_F64 : UR_F32);
      e = go(k_debug<MV, TW, TF, MV, CtaTeam>, k_debug<MV, TW, TF, MV, GridTeam>);
    } else if (what == 3) {
      e = go(k_debug<UM, TW, TF, MV, CtaTeam>, k_debug<UM, TW, TF, MV, GridTeam>);
    } else if (fmt == op_format()) {
      e = go(k_debug<MV, TW, TF, MV, CtaTeam>, k_debug<MV, TW, TF, MV, GridTeam>);
    } else {
      return fail(GB_ERR_UNSUPPORTED, "operator context differs from this solver's matvec format");
    }
    if (e != GB_OK) return e;
    CK(cudaMemcpyAsync(out, s->dtmp, sizeof(double) * n, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    return GB_OK;
  }

  static gb_status get_x(gb_solver* s, double* x) {
    k_to_f64<TW><<<64, 256, 0, s->stream>>>((const TW*)s->xs, s->n, s->dtmp);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(x, s->dtmp, sizeof(double) * s->n, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    return GB_OK;
  }

  static gb_status get_lu(gb_solver* s, double* lu, long long* perm) {
    const int n = s->n;
    double* tmp = nullptr;
    CK(cudaMalloc(&tmp, sizeof(double) * (size_t)n * n));
    k_copy_lu_to_f64<TF><<<1184, 256, 0, s->stream>>>((const TF*)s->LU, s->lda, n, tmp);
    CK(cudaMemcpyAsync(lu, tmp, sizeof(double) * (size_t)n * n, cudaMemcpyDeviceToHost, s->stream));
    std::vector<int> p(n);
    CK(cudaMemcpyAsync(p.data(), s->perm, sizeof(int) * n, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    CK(cudaFree(tmp));
    for (int i = 0; i < n; ++i) perm[i] = p[i];
    return GB_OK;
  }

  static const VariantOps* table() {
    static const VariantOps t{setup, set_system, factor, x0, xref, step, debug, get_x, get_lu};
    return &t;
  }
};

}  // namespace
