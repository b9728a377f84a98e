// Solver object, kernels and the per-variant implementation (Impl).  Each
// precision variant is instantiated in its own translation unit
// (gb_var_*.cu) so the variants compile in parallel; gb_capi.cu holds the
// extern "C" entry points and the dispatch.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "gb_refine.cuh"
#include "gb_tcgemm.cuh"
#pragma once

using namespace gb;

// one definition (gb_capi.cu) shared by every precision-variant translation unit,
// so gb_last_error() reports failures raised inside the variants
extern thread_local std::string g_err;
// kernels launched by this library (gb_launch_count); counted at launch sites
extern long long* gb_launch_counter();
static inline void count_launch(long long k = 1) { __atomic_fetch_add(gb_launch_counter(), k, __ATOMIC_RELAXED); }

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
  int inner_only;  // gb_debug_inner_solve: the inner solver alone on fl_u(rtmp), d -> dtmp
  double normA, normB;
  int ur, method;
  unsigned long long* ctr;    // [2]
  unsigned long long* epoch;  // [1]
  uint4* ytag = nullptr;      // tagged y of trsv_cta (2 x 16 B per entry)
  int ytag_dsm = 0;           // > 0: ytag is the CTA's shared-memory copy (cluster of that many CTAs)
  unsigned ytag_smem_off = 0;    // cluster launch: byte offset of the copy in dynamic smem
  unsigned ytag_smem_bytes = 0;  // 0 = keep ytag in global memory
  unsigned part_smem_off = 0;    // cluster launch: shared copy of the team partials (0 = none)
  GridCtl* ctl;
  double* partials;
  int kmax;
  gb_step_info* out;
  PhaseLog log;
  int* flags;  // [0] x0_reset
  // xref (large n): fp64 factors
  const double* LUx;
  const int* permx;
  const double* xrcph;
  const double* xrcpl;
  const double *xlinvh, *xlinvl, *xuinvh, *xuinvl;
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
    GridTeam t{(int)gridDim.x, (int)blockIdx.x, p.ctl, p.partials, p.kmax, 0u,
               gridDim.x > 1 && cluster_ncta() == gridDim.x};
    t.links_begin();
    return t;
  }
};
template <>
struct MakeTeam<ClusterTeam> {
  template <class P>
  GB_DEVICE static ClusterTeam make(const P& p) {
    ClusterTeam t;
    static_cast<GridTeam&>(t) = MakeTeam<GridTeam>::make(p);
    return t;
  }
};

__host__ __device__ inline size_t sm_doubles(int m, int k) { return (size_t)5 * m + 2 * k + 512; }

// cluster team: move the tagged y of the CTA-per-block TRSV into shared memory
// (zeroed here; the bodies' first team barrier orders it before any push).
template <class Team, class P_t>
__device__ void ytag_setup(Team& t, P_t& P, unsigned char* smem) {
  if constexpr (Team::kGrid) {
    if (t.clu && P.ytag_smem_bytes > 0) {
      uint4* yt = reinterpret_cast<uint4*>(smem + P.ytag_smem_off);
      for (unsigned i = threadIdx.x; i < P.ytag_smem_bytes / 16; i += blockDim.x) yt[i] = make_uint4(0u, 0u, 0u, 0u);
      P.ytag = yt;
      P.ytag_dsm = t.size();
    }
    if (t.clu && P.part_smem_off > 0) t.spart = reinterpret_cast<double*>(smem + P.part_smem_off);
  }
}
// a CTA of the cluster must not exit while peers may still push into its copy
template <class Team, class P_t>
__device__ void ytag_finish(Team& t, const P_t& P) {
  if constexpr (Team::kGrid) {
    if (P.ytag_dsm > 0) t.sync();
    t.links_end();
  }
}

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
  ts.ytag = P.ytag;
  ts.dsm = P.ytag_dsm;
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
  TrsvSync ts{P.ctr, P.ctr + 1, *P.epoch, P.log};
  ts.ytag = P.ytag;
  ts.dsm = P.ytag_dsm;
  mark(ts.log, 30);
  double* red = sm + 4 * K.m + 4;
  const int n = K.n;
  int lo, hi;
  t.rows(n, lo, hi);
  gb_step_info info;
  memset(&info, 0, sizeof(info));
  t.sync();
  const double nu = P.inner_only ? 1.0 : team_amax<double>(t, P.r, n, red);
  info.nu = nu;
  if (nu == 0.0 || !isfinite(nu)) {
    info.status = (nu == 0.0) ? RS_NU_ZERO : RS_NU_NONFINITE;
    info.ferr = P.has_xref[0] ? forward_error(t, (const TW*)P.xs, P.xref, n, red) : NAN;
    if (t.leader() && threadIdx.x == 0) *P.out = info;
    return;
  }
  if (P.inner_only) {
    // gmres_solve / gcrodr_solve on a caller's right-hand side (gmres.py:235, gcrodr.py:221)
    for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) K.rhat[i] = (TW)P.rtmp[i];
  } else {
    for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) K.rhat[i] = (TW)F::rnd(P.r[i] / nu);
  }
  StepScalars st{0, KS_CONVERGED, 0, 0};
  mark(ts.log, 31);
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
  mark(ts.log, 33);
  if (P.method == METH_SIR) {
    its = 1;
  } else {
    // sum of per-cycle steps (leader wrote them; broadcast through global)
    t.sync();
    for (int c = 0; c < st.ncycles; ++c) its += __ldcg(K.cycle_iters + c);
  }
  if (P.inner_only) {
    for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) P.dtmp[i] = (double)K.x[i];
    info.ferr = info.nbe = info.cbe = NAN;
    info.inner_iters = its;
    info.ncycles = st.ncycles;
    info.status = st.status;
    info.applies = st.applies;
    info.keff = st.keff;
    if (t.leader() && threadIdx.x == 0) {
      *P.out = info;
      *P.epoch = ts.epoch;
    }
    return;
  }
  for (int i = lo + threadIdx.x; i < hi; i += blockDim.x)
    P.xs[i] = fl_add<TW>(P.xs[i], F::scale(nu, K.x[i]));
  t.sync();
  mark(ts.log, 34);
  info.ferr = P.has_xref[0] ? forward_error(t, (const TW*)P.xs, P.xref, n, red) : NAN;
  mark(ts.log, 35);
  ResidOut ro = residual_check(t, K.sys.A, K.sys.lda, n, (const TW*)P.xs, P.b, P.r, P.ur, P.normA, P.normB, red);
  info.nbe = ro.nbe;
  info.cbe = ro.cbe;
  info.inner_iters = its;
  info.ncycles = st.ncycles;
  info.status = st.status;
  info.applies = st.applies;
  info.keff = st.keff;
  mark(ts.log, 39);
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
  ts.ytag = P.ytag;
  ts.dsm = P.ytag_dsm;
  double* red = sm + 4 * K.m + 4;
  const int n = K.n;
  SysView<TW, double> sx{n,       K.sys.lda, K.sys.A,  K.sys.lda, P.LUx,    P.permx,
                         P.xrcph, P.xrcpl,   P.xlinvh, P.xlinvl,  P.xuinvh, P.xuinvl};
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
  ts.ytag = P.ytag;
  ts.dsm = P.ytag_dsm;
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
  } else if (what == 5) {
    // check_convergence's residual and backward errors (refine.py:194-208)
    ResidOut ro = residual_check(t, K.sys.A, K.sys.lda, n, (const TW*)K.rhat, P.b, P.dtmp, P.ur, P.normA, P.normB, red);
    if (t.leader() && threadIdx.x == 0) {
      P.out->nbe = ro.nbe;
      P.out->cbe = ro.cbe;
    }
  } else {
    residual_check(t, K.sys.A, K.sys.lda, n, (const TW*)K.rhat, P.b, P.dtmp, P.ur, 1.0, 1.0, red);
  }
  t.sync();
  if (what != 2 && what != 5)
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
  ytag_setup(t, P, smem);
  x0_body(t, P, sm, ops);
  ytag_finish(t, P);
}

template <class TW, class TF, int MV, class Team>
__global__ void __launch_bounds__(kThreads) k_step(Prob<TW, TF, MV> Pin) {
  extern __shared__ __align__(16) unsigned char smem[];
  Prob<TW, TF, MV> P = Pin;
  Team t = MakeTeam<Team>::make(P);
  double* sm = reinterpret_cast<double*>(smem);
  void* ops = smem + sm_doubles(P.K.m, P.K.k) * sizeof(double);
  P.K.fast = P.K.fast_cap > 0 ? reinterpret_cast<double*>(ops) : nullptr;
  P.K.pack = reinterpret_cast<double*>(ops);
  ytag_setup(t, P, smem);
  step_body(t, P, sm, ops);
  if (t.leader() && threadIdx.x == 0) P.K.keff_io[1] = (P.K.U == Pin.K.U) ? 0 : 1;
  ytag_finish(t, P);
}

template <class TW, class TF, int MV, class Team>
__global__ void __launch_bounds__(kThreads) k_xref_refine(Prob<TW, TF, MV> Pin) {
  extern __shared__ __align__(16) unsigned char smem[];
  Prob<TW, TF, MV> P = Pin;
  Team t = MakeTeam<Team>::make(P);
  double* sm = reinterpret_cast<double*>(smem);
  void* ops = smem + sm_doubles(P.K.m, P.K.k) * sizeof(double);
  ytag_setup(t, P, smem);
  xref_refine_body(t, P, sm, ops);
  ytag_finish(t, P);
}

template <int M, class TW, class TF, int MV, class Team>
__global__ void __launch_bounds__(kThreads) k_debug(Prob<TW, TF, MV> Pin, int what) {
  extern __shared__ __align__(16) unsigned char smem[];
  Prob<TW, TF, MV> P = Pin;
  Team t = MakeTeam<Team>::make(P);
  double* sm = reinterpret_cast<double*>(smem);
  void* ops = smem + sm_doubles(P.K.m, P.K.k) * sizeof(double);
  ytag_setup(t, P, smem);
  debug_body<M>(t, P, sm, ops, what);
  ytag_finish(t, P);
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
    bool odd = false;
    for (int j = lane; j < n; j += 32) {
      TW v = (TW)a[(size_t)i * n + j];
      A[(size_t)i * lda + j] = v;
      s += fabs((double)v);
      const double av = fabs((double)v);
      odd |= !(av >= (sizeof(TW) == 4 ? 1.1754943508222875e-38 : 2.2250738585072014e-308) && av <= 1.7976931348623157e308);
    }
    if (__any_sync(0xffffffffu, odd) && lane == 0) atomicOr(&norms[2], 1ull);
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
// batched mode: one CTA per system, the whole refinement loop on the device
// (refine.py:277-421 including the decision rules of check_convergence).
// ---------------------------------------------------------------------------
struct SlotLayout {
  size_t stride;
  size_t A, b, LU, lubuf, perm, rcph, rcpl, linvh, linvl, uinvh, uinvl, xs, r, xref, rtmp, dtmp, V, w, xk, res, s, rhat, C, U, Cn, Un, Ut, Yt, Wd, Qd, H, R,
      B, bc, dense, gram, ybuf, ctr, epoch, cyc_it, cyc_ke, keff_io, flags, has_xref, out, xa, xb, xyh, xyl, xperm;
};

struct BatchArgs {
  int count, n, i_max;
  double c_conv, u_unit;
  const double* a;  // count x n x n
  const double* b;  // count x n
  char* slots;
  SlotLayout L;
  int* next;  // work counter
  // outputs
  int *converged, *steps, *reason, *inner, *flags;
  double *nbe, *ferr, *x, *growth;
  // options
  int m, k, max_cycles, reorth, explicit_res, method, ur, fast_cap;
  double tau;
};

template <class TW, class TF, int MV>
__global__ void __launch_bounds__(kThreads) k_batched(BatchArgs B) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int UM = UfMode<TF>::M;
  using L = LuT<UM>;
  double* sm = reinterpret_cast<double*>(smem);
  void* ops = smem + sm_doubles(B.m, B.k) * sizeof(double);
  __shared__ int s_sys;
  __shared__ PivKey pscr[32];
  __shared__ double s_norm[2];
  char* base = B.slots + (size_t)blockIdx.x * B.L.stride;
  const SlotLayout& Ly = B.L;
  const int fcap = B.fast_cap;
  const int n = B.n, ldv = (n + 31) & ~31;
  Prob<TW, TF, MV> P;
  memset(&P, 0, sizeof(P));
  auto& K = P.K;
  K.n = n;
  K.ldv = ldv;
  K.m = B.m;
  K.k = B.k;
  K.max_cycles = B.max_cycles;
  K.tau = B.tau;
  K.reorth = B.reorth;
  K.explicit_res = B.explicit_res;
  K.recycling = B.method == METH_GCRODR;
  TW* A = (TW*)(base + Ly.A);
  K.sys = SysView<TW, TF>{n,
                          (size_t)ldv,
                          A,
                          (size_t)ldv,
                          (const TF*)(base + Ly.LU),
                          (const int*)(base + Ly.perm),
                          (const double*)(base + Ly.rcph),
                          (const double*)(base + Ly.rcpl),
                          (const double*)(base + Ly.linvh),
                          (const double*)(base + Ly.linvl),
                          (const double*)(base + Ly.uinvh),
                          (const double*)(base + Ly.uinvl)};
  K.V = (TW*)(base + Ly.V);
  K.w = (TW*)(base + Ly.w);
  K.x = (TW*)(base + Ly.xk);
  K.res = (TW*)(base + Ly.res);
  K.s = (TW*)(base + Ly.s);
  K.rhat = (TW*)(base + Ly.rhat);
  K.C = (TW*)(base + Ly.C);
  K.U = (TW*)(base + Ly.U);
  K.Cn = (TW*)(base + Ly.Cn);
  K.Un = (TW*)(base + Ly.Un);
  K.Ut = (TW*)(base + Ly.Ut);
  K.Yt = (TW*)(base + Ly.Yt);
  K.Wd = (double*)(base + Ly.Wd);
  K.Qd = (double*)(base + Ly.Qd);
  K.H = (double*)(base + Ly.H);
  K.R = (double*)(base + Ly.R);
  K.B = (double*)(base + Ly.B);
  K.bc = (double*)(base + Ly.bc);
  K.dense = (double*)(base + Ly.dense);
  K.gram = (double*)(base + Ly.gram);
  K.gram_stride = (size_t)(B.m + B.k + 2) * (B.m + B.k + 2);
  K.ybuf = (typename Arith<MV>::T*)(base + Ly.ybuf);
  K.cycle_iters = (int*)(base + Ly.cyc_it);
  K.cycle_keff = (int*)(base + Ly.cyc_ke);
  K.keff_io = (int*)(base + Ly.keff_io);
  K.fast = fcap > 0 ? reinterpret_cast<double*>(ops) : nullptr;
  K.fast_cap = fcap;
  K.ops_bytes = 0;  // batched mode: the op region holds the system (no staging)
  P.b = (const TW*)(base + Ly.b);
  P.xs = (TW*)(base + Ly.xs);
  P.r = (double*)(base + Ly.r);
  P.xref = (double*)(base + Ly.xref);
  P.has_xref = (int*)(base + Ly.has_xref);
  P.ur = B.ur;
  P.method = B.method;
  P.ctr = (unsigned long long*)(base + Ly.ctr);
  P.epoch = (unsigned long long*)(base + Ly.epoch);
  P.out = (gb_step_info*)(base + Ly.out);
  P.flags = (int*)(base + Ly.flags);
  CtaTeam t;
  while (true) {
    if (threadIdx.x == 0) s_sys = atomicAdd(B.next, 1);
    __syncthreads();
    const int sys = s_sys;
    __syncthreads();
    if (sys >= B.count) break;
    const double* a = B.a + (size_t)sys * n * n;
    const double* bb = B.b + (size_t)sys * n;
    // A_u, b_u and the inf-norms (refine.py:285-300)
    double rmax = 0.0, bmax = 0.0;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int i = wid; i < n; i += nw) {
      double rs = 0.0;
      for (int j = lane; j < n; j += 32) {
        TW v = (TW)a[(size_t)i * n + j];
        A[(size_t)i * ldv + j] = v;
        rs += fabs((double)v);
      }
      rs = warp_sum(rs);
      rmax = (rs > rmax || rs != rs) ? rs : rmax;
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      TW v = (TW)bb[i];
      ((TW*)P.b)[i] = v;
      double ab = fabs((double)v);
      bmax = (ab > bmax || ab != ab) ? ab : bmax;
    }
    rmax = block_max(rmax, sm);
    bmax = block_max(bmax, sm);
    if (threadIdx.x == 0) {
      s_norm[0] = rmax;
      s_norm[1] = bmax;
      K.keff_io[0] = 0;
      K.keff_io[1] = 0;
    }
    __syncthreads();
    P.normA = s_norm[0];
    P.normB = s_norm[1];
    // LU in u_f (densela.py:124-168) on the slot carrier buffer
    typename L::C* lub = (typename L::C*)(base + Ly.lubuf);
    double am = 0.0;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      typename L::C v = L::ld(L::from_u((double)A[(size_t)(e / n) * ldv + e % n]));
      lub[e] = v;
      double x = fabs((double)v);
      am = (x > am || x != x) ? x : am;
    }
    am = block_max(am, sm);
    __syncthreads();
    int* perm = (int*)(base + Ly.perm);
    const int zero = lu_cta<UM>(lub, n, n, perm, pscr);
    double um = 0.0;
    TF* LUo = (TF*)(base + Ly.LU);
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      int i = e / n, j = e % n;
      LUo[(size_t)i * ldv + j] = (TF)L::st(lub[e]);
      if (j >= i) {
        double x = fabs((double)lub[e]);
        um = (x > um || x != x) ? x : um;
      }
    }
    um = block_max(um, sm);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      dd q = dd_div(dd{1.0, 0.0}, dd{(double)lub[(size_t)i * n + i], 0.0});
      ((double*)(base + Ly.rcph))[i] = q.hi;
      ((double*)(base + Ly.rcpl))[i] = q.lo;
    }
    __syncthreads();
    for (int bk = threadIdx.x >> 5; bk < (n + 31) / 32; bk += blockDim.x >> 5)
      diag_inv_block(LUo, (size_t)ldv, n, bk, (double*)(base + Ly.linvh), (double*)(base + Ly.linvl),
                     (double*)(base + Ly.uinvh), (double*)(base + Ly.uinvl));
    __syncthreads();
    int flags = 0;
    if (zero >= 0) {
      if (threadIdx.x == 0) {
        B.converged[sys] = 0;
        B.steps[sys] = 0;
        B.reason[sys] = 2;  // InnerStagnation
        B.flags[sys] = 4;   // lu_failed
        B.growth[sys] = NAN;
      }
      for (int i = threadIdx.x; i < n; i += blockDim.x) B.x[(size_t)sys * n + i] = NAN;
      __syncthreads();
      continue;
    }
    // x0 (refine.py:317-321)
    x0_body(t, P, sm, ops);
    __syncthreads();
    if (P.flags[0]) flags |= 1;
    // xref: double-double GEPP (n <= 600)
    bool okx = dd_gepp_solve((const TW*)A, (size_t)ldv, P.b, n, (double*)(base + Ly.xa), (double*)(base + Ly.xb),
                             (double*)(base + Ly.xyh), (double*)(base + Ly.xyl), (int*)(base + Ly.xperm), P.xref,
                             pscr);
    if (threadIdx.x == 0) P.has_xref[0] = okx ? 1 : 0;
    __syncthreads();
    if (!okx) flags |= 2;
    // refinement loop with the reference's decision rules
    int steps = 0, conv = 0, reason = 1, grow = 0;
    double prev = 0.0;
    for (int it = 0; it < B.i_max; ++it) {
      step_body(t, P, sm, ops);
      __syncthreads();
      gb_step_info info = *P.out;
      __syncthreads();
      const size_t o = (size_t)sys * B.i_max + steps;
      if (info.status & (RS_NU_ZERO | RS_NU_NONFINITE)) {
        if (info.status & RS_NU_ZERO) {
          if (threadIdx.x == 0) {
            B.inner[o] = 0;
            B.nbe[o] = 0.0;
            B.ferr[o] = info.ferr;
          }
          steps++;
          conv = 1;
          reason = 0;
        } else {
          reason = 3;
        }
        break;
      }
      if (threadIdx.x == 0) {
        B.inner[o] = info.inner_iters;
        B.nbe[o] = info.nbe;
        B.ferr[o] = info.ferr;
      }
      steps++;
      // check_convergence (refine.py:210-229); Python max() semantics
      double worst = info.nbe;
      if (info.cbe > worst) worst = info.cbe;
      const double f = isfinite(info.ferr) ? info.ferr : 0.0;
      if (f > worst) worst = f;
      const bool stag = (info.status & KS_STAGNATED) && B.method != METH_SIR;
      if (isfinite(worst) && worst <= B.c_conv * B.u_unit) {
        conv = 1;
        reason = 0;
        break;
      }
      if (stag) {
        reason = 2;
        break;
      }
      if (it > 0) {
        if (!isfinite(info.nbe) || (isfinite(prev) && info.nbe >= 2.0 * prev)) grow++;
        else grow = 0;
      }
      prev = info.nbe;
      if (grow >= 3) {
        reason = 3;
        break;
      }
    }
    if (threadIdx.x == 0) {
      B.converged[sys] = conv;
      B.steps[sys] = steps;
      B.reason[sys] = conv ? 0 : reason;
      B.flags[sys] = flags;
      B.growth[sys] = am != 0.0 ? um / am : NAN;
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) B.x[(size_t)sys * n + i] = (double)P.xs[i];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// arena
// ---------------------------------------------------------------------------
// grow-only device buffers of the batched entry point (one pool per variant)
struct BatchPool {
  std::mutex mu;
  void* ptr[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  size_t cap[5] = {0, 0, 0, 0, 0};
  char* get(int i, size_t bytes) {
    if (bytes > cap[i]) {
      if (ptr[i]) cudaFree(ptr[i]);
      ptr[i] = nullptr;
      cap[i] = 0;
      if (cudaMalloc(&ptr[i], bytes) != cudaSuccess) return nullptr;
      cap[i] = bytes;
    }
    return reinterpret_cast<char*>(ptr[i]);
  }
};
inline BatchPool& batch_pool() {
  static BatchPool* p = new BatchPool();  // never destroyed: outlives the CUDA context teardown
  return *p;
}

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
  bool cluster = false;  // the G-CTA team is launched as one thread-block cluster
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
  double *rcph = nullptr, *rcpl = nullptr, *xrcph = nullptr, *xrcpl = nullptr;
  double *linvh = nullptr, *linvl = nullptr, *uinvh = nullptr, *uinvl = nullptr;
  double *xlinvh = nullptr, *xlinvl = nullptr, *xuinvh = nullptr, *xuinvl = nullptr;
  // grid teams with an fp64 operator: inverses of the big diagonal blocks
  // (gb_opseg.cuh sweep_bsp), GEMV bulk-copy stages, A entries all normal
  double *bigl = nullptr, *bigu = nullptr;
  int nbig = 0, gemv_ns = 0, a_normal = 0, sweep_la = 0;
  int inner_only = 0;      // next step launch runs the inner solver alone (gb_debug_inner_solve)
  int max_cycles_cap = 0;  // o.max_cycles at creation (workspace size); o.max_cycles may be lowered
  PivKey* lu_ckey = nullptr;
  double *lu_crow = nullptr, *lu_rowk = nullptr;
  int* lu_piv = nullptr;
  int* lu_ipiv = nullptr;  // blocked tensor LU: pivot row of every column (LAPACK ipiv)
  // blocked tensor LU statistics of the last factorisation (gb_lu_tc_stats)
  double tc_update_ms = 0.0, tc_update_flop = 0.0, tc_trsm_ms = 0.0, tc_panel_ms = 0.0;
  std::vector<cudaEvent_t> tc_events;
  double *r = nullptr, *xref = nullptr, *rtmp = nullptr, *dtmp = nullptr;
  void *V = nullptr, *w = nullptr, *xk = nullptr, *res = nullptr, *s = nullptr, *rhat = nullptr;
  void *C = nullptr, *U = nullptr, *Cn = nullptr, *Un = nullptr, *Ut = nullptr, *Yt = nullptr;
  double *Wd = nullptr, *Qd = nullptr, *H = nullptr, *R = nullptr, *B = nullptr, *bc = nullptr, *dense = nullptr,
         *gram = nullptr;
  size_t gram_stride = 0;
  void* ybuf = nullptr;
  unsigned long long *ctr = nullptr, *epoch = nullptr, *norms = nullptr;
  uint4* ytag = nullptr;
  unsigned long long* plog = nullptr;  // phase log (diagnostics), 1 + 2 * cap
  int plog_cap = 0;
  bool plog_host = false;  // GB_PLOG_HOST=1: mapped pinned host memory (readable after a fault)
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
  gb_status (*set_system)(gb_solver*, const double*, const double*, int);
  gb_status (*factor)(gb_solver*, int*, double*);
  gb_status (*x0)(gb_solver*, int*);
  gb_status (*xref)(gb_solver*, int*);
  gb_status (*step)(gb_solver*, gb_step_info*);
  gb_status (*debug)(gb_solver*, const double*, double*, int what, int fmt);
  gb_status (*get_x)(gb_solver*, double*);
  gb_status (*get_lu)(gb_solver*, double*, long long*);
  gb_status (*time_op)(gb_solver*, int what, int reps, double* ms);
  gb_status (*batched)(int, int, const gb_options*, int, double, const double*, const double*, int, gb_batch_out*,
                       double*, cudaStream_t);
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
    K.explicit_res = s->o.explicit_residual;
    K.recycling = (s->o.method == GB_RGMRES_IR || s->o.method == GB_RSGMRES_IR);
    K.sys = SysView<TW, TF>{s->n,     (size_t)s->lda, (const TW*)s->A, (size_t)s->lda, (const TF*)s->LU, s->perm,
                            s->rcph,  s->rcpl,        s->linvh,        s->linvl,        s->uinvh,          s->uinvl};
    if (s->bigl != nullptr && s->gemv_ns > 0) {
      K.sys.bigl = s->bigl;
      K.sys.bigu = s->bigu;
      K.sys.nbig = s->nbig;
      K.sys.gemv_ns = s->gemv_ns;
      K.sys.a_normal = s->a_normal;
      K.sys.sweep_la = s->sweep_la;
    }
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
    K.fast = nullptr;
    K.pack = nullptr;
    K.fast_cap = fast_cap(s->o.m, s->o.k);
    K.ops_bytes = (int)(smem_bytes(s) - sm_doubles(s->o.m, s->o.k) * sizeof(double));
    P.b = (const TW*)s->b;
    P.xs = (TW*)s->xs;
    P.r = s->r;
    P.xref = s->xref;
    P.has_xref = s->has_xref;
    P.inner_only = s->inner_only;
    P.normA = s->normA;
    P.normB = s->normB;
    P.ur = s->o.ur == GB_QUAD ? UR_DD : (s->o.ur == GB_DOUBLE ? UR_F64 : UR_F32);
    P.method = s->o.method == GB_SIR ? METH_SIR
               : (s->o.method == GB_GMRES_IR || s->o.method == GB_SGMRES_IR) ? METH_GMRES
                                                                              : METH_GCRODR;
    P.ctr = s->ctr;
    P.epoch = s->epoch;
    P.ytag = s->ytag;
    if (s->cluster) {
      P.ytag_smem_off = (unsigned)((smem_bytes(s) + 15) & ~(size_t)15);
      P.ytag_smem_bytes = (unsigned)(32 * (size_t)s->ldv);
      P.part_smem_off = P.ytag_smem_off + P.ytag_smem_bytes;
    }
    P.ctl = s->ctl;
    P.partials = s->partials;
    P.kmax = s->kmax;
    P.out = s->out;
    P.flags = s->flags;
    P.LUx = s->xa;
    P.permx = s->xperm;
    P.xrcph = s->xrcph;
    P.xrcpl = s->xrcpl;
    P.xlinvh = s->xlinvh;
    P.xlinvl = s->xlinvl;
    P.xuinvh = s->xuinvh;
    P.xuinvl = s->xuinvl;
    P.rtmp = s->rtmp;
    P.dtmp = s->dtmp;
    P.log = PhaseLog{s->plog, s->plog_cap, s->plog_host ? s->plog + 1 + 2 * (size_t)s->plog_cap : nullptr};
    return P;
  }

  // dynamic smem: the sm region + max(TRSV tiles, leader fast scratch when it fits)
  static int fast_cap(int m, int k) {
    const size_t need = (size_t)leader_fast_need(m + k + 2, k) * sizeof(double);
    const size_t base = sm_doubles(m, k) * sizeof(double);
    return (base + std::max(need, ops_bytes<TW, TF, MV>()) <= 190 * 1024) ? (int)(need / sizeof(double)) : 0;
  }
  static size_t smem_bytes_for(int m, int k) {
    const int fc = fast_cap(m, k);
    return sm_doubles(m, k) * sizeof(double) + std::max(ops_bytes<TW, TF, MV>(), (size_t)fc * sizeof(double));
  }
  // grid teams with kTrsvB-row blocks also stage a block record in the op
  // region (trsv_cta_g); one-CTA and cluster teams keep the 32-row scheme
  static int trsv_block(const gb_solver* s) { return (s->G > 1 && !s->cluster) ? kTrsvB : 32; }
  static size_t smem_bytes(gb_solver* s) {
    size_t b = smem_bytes_for(s->o.m, s->o.k);
    if (s->bigl != nullptr && s->gemv_ns > 0) {
      // bulk-copy GEMV (v as fp64 + a ring filling the rest of 227 KB) and the
      // big-block substitution's staged vector (sweep_bsp)
      const size_t base = sm_doubles(s->o.m, s->o.k) * sizeof(double);
      b = std::max(b, base + std::max(seg::gemv_smem(s->n, s->gemv_ns), (size_t)s->nbig * 16 + 64));
    }
    if (s->G > 1 && !s->cluster && fast_cap(s->o.m, s->o.k) == 0) {
      // packed Hessenberg storage of the harmonic-Ritz eigenproblem (dimension <= m)
      const size_t need = sm_doubles(s->o.m, s->o.k) * sizeof(double) + hqr_pack_doubles(s->o.m) * sizeof(double);
      if (need <= 227 * 1024 - 8192) b = std::max(b, need);
    }
    if (trsv_block(s) == kTrsvB) {
      const size_t need = sm_doubles(s->o.m, s->o.k) * sizeof(double) +
                          std::max(trsv_cta_smem<MV, kTrsvB>(), trsv_cta_smem<MODE_F64, kTrsvB>());
      b = std::max(b, need);
    }
    return b;
  }

  // can G CTAs of this kernel (with `sm` bytes of smem each) run as one cluster?
  template <class KernT>
  static bool cluster_fits(gb_solver* s, KernT kern, size_t sm) {
    if (cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(s->G);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = sm;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = s->G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nclu = 0;
    if (cudaOccupancyMaxActiveClusters(&nclu, (const void*)kern, &cfg) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return nclu >= 1;
  }

  template <class KernT, class... Args>
  static gb_status launch(gb_solver* s, KernT kern, Args... args) {
    size_t sm = smem_bytes(s);
    if (s->G == 1) {
      gb_status st = set_smem(kern, sm);
      if (st != GB_OK) return st;
      count_launch();
      kern<<<1, kThreads, sm, s->stream>>>(args...);
      CK(cudaGetLastError());
      return GB_OK;
    }
    // cluster team: + shared tagged y and the shared copy of the team
    // partials (ytag_setup); otherwise the cooperative grid (the kernel sees
    // no cluster and keeps both in global memory)
    const size_t smc = ((sm + 15) & ~(size_t)15) + 32 * (size_t)s->ldv + 2 * sizeof(double) * s->G * s->kmax;
    if (s->cluster && smc <= 227 * 1024 && set_smem(kern, smc) == GB_OK && cluster_fits(s, kern, smc)) {
      count_launch();
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(s->G);
      cfg.blockDim = dim3(kThreads);
      cfg.dynamicSmemBytes = smc;
      cfg.stream = s->stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = s->G;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      CK(cudaLaunchKernelEx(&cfg, kern, args...));
      return GB_OK;
    }
    cudaGetLastError();
    gb_status st = set_smem(kern, sm);
    if (st != GB_OK) return st;
    count_launch();
    void* argv[] = {(void*)&args...};
    CK(cudaMemsetAsync(&s->ctl->count, 0, sizeof(unsigned), s->stream));  // GridTeam::sync arrival counter
    CK(cudaLaunchCooperativeKernel((void*)kern, dim3(s->G), dim3(kThreads), argv, sm, s->stream));
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
      const size_t ninv = std::max((size_t)((n + 31) / 32) * kInvStride,
                                   (size_t)((n + kTrsvB - 1) / kTrsvB) * inv_stride<kTrsvB>());
      s->linvh = a.take<double>(ninv);
      s->linvl = a.take<double>(ninv);
      s->uinvh = a.take<double>(ninv);
      s->uinvl = a.take<double>(ninv);
      s->xlinvh = a.take<double>(ninv);
      s->xlinvl = a.take<double>(ninv);
      s->xuinvh = a.take<double>(ninv);
      s->xuinvl = a.take<double>(ninv);
      if (s->G > 1 && !s->cluster && MV == MODE_F64) {
        s->nbig = n >= 8192 ? 2048 : 1024;
        const size_t nk = (size_t)((n + s->nbig - 1) / s->nbig);
        s->bigl = a.take<double>(nk * s->nbig * s->nbig);
        s->bigu = a.take<double>(nk * s->nbig * s->nbig);
      }
      s->lu_ckey = a.take<PivKey>(2 * 160);
      s->lu_crow = a.take<double>(2 * 160 * 32);
      s->lu_rowk = a.take<double>(64);
      s->lu_piv = a.take<int>(64);
      s->lu_ipiv = a.take<int>(ldv);
      s->rcph = a.take<double>(ldv);
      s->rcpl = a.take<double>(ldv);
      s->xrcph = a.take<double>(ldv);
      s->xrcpl = a.take<double>(ldv);
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
      s->ytag = a.take<uint4>(2 * (size_t)ldv);
      s->norms = a.take<unsigned long long>(4);
      s->ctl = a.take<GridCtl>(1 + (kCtlExtraBytes + sizeof(GridCtl) - 1) / sizeof(GridCtl));  // + reduce1 slots, broadcast
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
    if (s->bigl != nullptr) {
      const char* la = std::getenv("GB_SWEEP_LA");
      s->sweep_la = (la && la[0] == '1') ? 1 : 0;
      // 227 KB per CTA = dynamic + static: the step kernels declare 7 KB of
      // static shared memory (reduction / pivot scratch), reserve 8 KB for it
      const size_t budget = 227 * 1024 - sm_doubles(s->o.m, s->o.k) * sizeof(double) - 8192;
      s->gemv_ns = (budget > seg::gemv_vbytes(n) + 4608 + 2 * seg::GCH) ? seg::gemv_stages(n, budget) : 0;
    }
    CK(cudaMemsetAsync(s->mem, 0, bytes, s->stream));
    return GB_OK;
  }

  static gb_status set_system(gb_solver* s, const double* a, const double* b, int on_device) {
    const int n = s->n;
    const double* asrc = a;
    const double* bsrc = b;
    if (!on_device) {
      double* bstage = s->rtmp;  // n doubles
      CK(cudaMemcpyAsync(s->stage, a, sizeof(double) * (size_t)n * n, cudaMemcpyHostToDevice, s->stream));
      CK(cudaMemcpyAsync(bstage, b, sizeof(double) * n, cudaMemcpyHostToDevice, s->stream));
      asrc = s->stage;
      bsrc = bstage;
    }
    CK(cudaMemsetAsync(s->norms, 0, 3 * sizeof(unsigned long long), s->stream));
    int blocks = std::min(1184, std::max(1, (n + 7) / 8));
    count_launch();
    k_set_system<TW><<<blocks, 256, 0, s->stream>>>(asrc, n, (TW*)s->A, s->lda, bsrc, (TW*)s->b, s->norms);
    CK(cudaGetLastError());
    unsigned long long nb[3];
    CK(cudaMemcpyAsync(nb, s->norms, sizeof(nb), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    memcpy(&s->normA, &nb[0], 8);
    memcpy(&s->normB, &nb[1], 8);
    s->a_normal = nb[2] == 0 ? 1 : 0;  // no zero / subnormal / inf / NaN entry in fl_u(A)
    // fresh recycle state / counters for a new system
    CK(cudaMemsetAsync(s->keff_io, 0, 4 * sizeof(int), s->stream));
    s->parity = 0;
    return GB_OK;
  }

  template <int M, class TA, class S>
  static gb_status lu_run(gb_solver* s, const TA* A, size_t lda, S* W, int* perm, int* piv, LuStatus* st,
                          double* rh, double* rl, double* ilh, double* ill, double* iuh, double* iul,
                          int tcmode = 0, bool big = false) {
    gb_status e = lu_run_core<M>(s, A, lda, W, perm, piv, st, tcmode);
    if (e != GB_OK) return e;
    if (big && s->bigl != nullptr) {
      // inverses of the big diagonal blocks for the grid-team fp64 operator
      const size_t smb = (size_t)8 * s->nbig * sizeof(double);
      gb_status e2 = set_smem(seg::k_bigblock_inverse<S, true>, smb);
      if (e2 == GB_OK) e2 = set_smem(seg::k_bigblock_inverse<S, false>, smb);
      if (e2 != GB_OK) return e2;
      count_launch(2);
      seg::k_bigblock_inverse<S, true><<<148 * 4, 256, smb, s->stream>>>(W, (size_t)s->lda, s->n, s->nbig, s->bigl);
      seg::k_bigblock_inverse<S, false><<<148 * 4, 256, smb, s->stream>>>(W, (size_t)s->lda, s->n, s->nbig, s->bigu);
      CK(cudaGetLastError());
    }
    count_launch(2);
    k_lu_rcp<S><<<std::max(1, std::min(1184, (s->n + 255) / 256)), 256, 0, s->stream>>>(W, s->lda, s->n, rh, rl);
    if (trsv_block(s) == kTrsvB) {
      // grid teams: kTrsvB-row block records for trsv_cta_g
      const int nbk = (s->n + kTrsvB - 1) / kTrsvB;
      k_diag_inv_b<kTrsvB, S><<<std::max(1, (nbk + 1) / 2), 2 * kTrsvB, 0, s->stream>>>(W, s->lda, s->n, ilh, ill,
                                                                                      iuh, iul);
      count_launch();
      k_diag_fold_b<kTrsvB, S><<<std::max(1, (nbk + 1) / 2), 2 * kTrsvB, 0, s->stream>>>(W, s->lda, s->n, ilh, ill,
                                                                                       iuh, iul);
    } else {
      const int nbk = (s->n + 31) / 32;
      k_diag_inv<S><<<std::max(1, (nbk + 3) / 4), 128, 0, s->stream>>>(W, s->lda, s->n, ilh, ill, iuh, iul);
      count_launch();
      k_diag_fold<S><<<std::max(1, (nbk + 3) / 4), 128, 0, s->stream>>>(W, s->lda, s->n, ilh, ill, iuh, iul);
    }
    CK(cudaGetLastError());
    return GB_OK;
  }

  template <int M, class TA, class S>
  static gb_status lu_run_core(gb_solver* s, const TA* A, size_t lda, S* W, int* perm, int* piv, LuStatus* st,
                               int tcmode = 0) {
    const int n = s->n;
    LuStatus init{0x7fffffff, 0, 0ull, 0ull};
    CK(cudaMemcpyAsync(st, &init, sizeof(init), cudaMemcpyHostToDevice, s->stream));
    if (n <= 128 && M == MODE_H16 && tcmode == 0) {
      size_t sm = (size_t)n * n * sizeof(typename LuT<M>::C);
      gb_status e = set_smem(k_lu_small<M, TA>, sm);
      if (e != GB_OK) return e;
      count_launch();
      k_lu_small<M, TA><<<1, kThreads, sm, s->stream>>>(A, lda, W, s->lda, n, perm, st);
      CK(cudaGetLastError());
      return GB_OK;
    }
    // one persistent cooperative launch for the whole blocked factorisation
    int dev = 0, sms = 148;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int G = n <= 256 ? 1 : std::min(sms, (n + 63) / 64);
    const size_t smb = lu_team_smem<M>(n, G);
    LuWork wk{s->lu_ckey, s->lu_crow, s->lu_rowk, s->lu_piv};
    count_launch();
    if (G == 1) {
      auto kern = k_lu_team<M, TA, CtaTeam>;
      gb_status e = set_smem(kern, smb);
      if (e != GB_OK) return e;
      kern<<<1, 256, smb, s->stream>>>(A, lda, W, (size_t)s->lda, n, perm, st, wk, s->ctl, s->partials, tcmode, 0, n,
                                       (int*)nullptr);
      CK(cudaGetLastError());
    } else {
      auto kern = k_lu_team<M, TA, GridTeam>;
      gb_status e = set_smem(kern, smb);
      if (e != GB_OK) return e;
      size_t ldw = (size_t)s->lda;
      GridCtl* ctl = s->ctl;
      double* part = s->partials;
      if constexpr (M == MODE_H16) {
        if (tcmode != 0 && n >= 2048) return lu_run_blocked<TA>(s, A, lda, W, perm, st, wk, G, smb);
      }
      int cbeg = 0, cend = n;
      int* ipiv = nullptr;
      void* argv[] = {(void*)&A,   (void*)&lda,  (void*)&W,      (void*)&ldw,  (void*)&n,    (void*)&perm, (void*)&st,
                      (void*)&wk,  (void*)&ctl,  (void*)&part,   (void*)&tcmode, (void*)&cbeg, (void*)&cend,
                      (void*)&ipiv};
      CK(cudaMemsetAsync(&s->ctl->count, 0, sizeof(unsigned), s->stream));  // GridTeam::sync arrival counter
      CK(cudaLaunchCooperativeKernel((void*)kern, dim3(G), dim3(256), argv, smb, s->stream));
    }
    (void)piv;
    return GB_OK;
  }

  // U12 = L11^-1 A12 for the w x w unit lower block at (r0, r0) and the columns
  // [c0, c0 + N): recursive halving; the off-diagonal products run on tcgen05
  static cudaError_t trsm_rec(gb_solver* s, __half* W, int r0, int w, int c0, int N, __half* Bt) {
    if (w <= 32) {
      count_launch();
      k_lu_trsm32<MODE_H16><<<std::max(1, std::min(296, (N + 255) / 256)), 256, 0, s->stream>>>(W, (size_t)s->lda,
                                                                                                 r0, c0, N);
      return cudaGetLastError();
    }
    const int h = ((w / 2 + 31) / 32) * 32;
    cudaError_t e = trsm_rec(s, W, r0, h, c0, N, Bt);
    if (e != cudaSuccess) return e;
    count_launch(2);
    e = tcg2::tc_update(W, (size_t)s->lda, s->n, r0 + h, c0, w - h, N, r0, h, Bt, s->stream);
    if (e != cudaSuccess) return e;
    return trsm_rec(s, W, r0 + h, w - h, c0, N, Bt);
  }

  // Blocked tensor-mode LU (north_star (1)): panels of kLuWide columns are
  // factored by the team kernel in a column window (pivot search, interchanges
  // and rank-32 tcgen05 updates inside the panel); then the interchanges are
  // applied to the other columns, U12 = L11^-1 A12 (recursive, tcgen05 below
  // the 32-row base case) and the trailing matrix takes ONE rank-kLuWide
  // update A22 = fl16(A22 - fp32(L21 U12)) on the CTA-pair tcgen05 kernel fed
  // by TMA (gb_tcgemm.cuh), i.e. n / kLuWide passes over the trailing matrix.
  static constexpr int kLuWide = 1024;
  template <class TA>
  static gb_status lu_run_blocked(gb_solver* s, const TA* A, size_t lda, __half* W, int* perm, LuStatus* st,
                                  LuWork wk, int G, size_t smb) {
    const int n = s->n;
    auto kern = k_lu_team<MODE_H16, TA, GridTeam>;
    size_t ldw = (size_t)s->lda;
    GridCtl* ctl = s->ctl;
    double* part = s->partials;
    int tcmode = 1;
    int* ipiv = s->lu_ipiv;
    __half* Bt = reinterpret_cast<__half*>(s->stage);  // host-upload staging area: free during the factorisation
    const int npanel = (n + kLuWide - 1) / kLuWide;
    while ((int)s->tc_events.size() < 4 * npanel) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      s->tc_events.push_back(e);
    }
    s->tc_update_flop = 0.0;
    int done = 0;
    for (int c0 = 0, ip = 0; c0 < n; c0 += kLuWide, ++ip) {
      int cbeg = c0, cend = std::min(n, c0 + kLuWide);
      const int w = cend - cbeg, rest = n - cend;
      void* argv[] = {(void*)&A,   (void*)&lda,  (void*)&W,      (void*)&ldw,  (void*)&n,    (void*)&perm, (void*)&st,
                      (void*)&wk,  (void*)&ctl,  (void*)&part,   (void*)&tcmode, (void*)&cbeg, (void*)&cend,
                      (void*)&ipiv};
      CK(cudaEventRecord(s->tc_events[4 * ip], s->stream));
      CK(cudaMemsetAsync(&s->ctl->count, 0, sizeof(unsigned), s->stream));
      count_launch();
      CK(cudaLaunchCooperativeKernel((void*)kern, dim3(G), dim3(256), argv, smb, s->stream));
      count_launch();
      k_lu_apply_pivots<__half><<<148, 256, 0, s->stream>>>(W, ldw, n, cbeg, w, ipiv);
      CK(cudaGetLastError());
      CK(cudaEventRecord(s->tc_events[4 * ip + 1], s->stream));
      if (rest > 0) {
        CK(trsm_rec(s, W, cbeg, w, cend, rest, Bt));
        CK(cudaEventRecord(s->tc_events[4 * ip + 2], s->stream));
        count_launch(2);
        CK(tcg2::tc_update(W, ldw, n, cend, cend, rest, rest, cbeg, w, Bt, s->stream));
        s->tc_update_flop += 2.0 * (double)rest * rest * w;
      } else {
        CK(cudaEventRecord(s->tc_events[4 * ip + 2], s->stream));
      }
      CK(cudaEventRecord(s->tc_events[4 * ip + 3], s->stream));
      done = ip + 1;
    }
    CK(cudaStreamSynchronize(s->stream));
    s->tc_update_ms = s->tc_trsm_ms = s->tc_panel_ms = 0.0;
    for (int ip = 0; ip < done; ++ip) {
      float a = 0.f, b = 0.f, c = 0.f;
      CK(cudaEventElapsedTime(&a, s->tc_events[4 * ip], s->tc_events[4 * ip + 1]));
      CK(cudaEventElapsedTime(&b, s->tc_events[4 * ip + 1], s->tc_events[4 * ip + 2]));
      CK(cudaEventElapsedTime(&c, s->tc_events[4 * ip + 2], s->tc_events[4 * ip + 3]));
      s->tc_panel_ms += a;
      s->tc_trsm_ms += b;
      s->tc_update_ms += c;
    }
    return GB_OK;
  }

  static gb_status factor(gb_solver* s, int* zero_col, double* growth) {
    CK(cudaEventRecord(s->ev0, s->stream));
    gb_status e = lu_run<UM>(s, (const TW*)s->A, (size_t)s->lda, (typename LuT<UM>::S*)s->LU, s->perm, s->piv, s->lust,
                             s->rcph, s->rcpl, s->linvh, s->linvl, s->uinvh, s->uinvl, s->o.lu_mode, true);
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
    gb_status e = s->G == 1   ? launch(s, k_x0<TW, TF, MV, CtaTeam>, P)
                  : s->cluster ? launch(s, k_x0<TW, TF, MV, ClusterTeam>, P)
                               : launch(s, k_x0<TW, TF, MV, GridTeam>, P);
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
      count_launch();
      k_xref_small<TW><<<1, kThreads, 0, s->stream>>>((const TW*)s->A, s->lda, (const TW*)s->b, n, s->xa, s->xb,
                                                     s->xyh, s->xyl, s->xperm, s->xref, s->has_xref);
      CK(cudaGetLastError());
    } else {
      // fp64 GEPP of A (lu_factor(a, DOUBLE)) then the dd-residual refinement
      gb_status e = lu_run<MODE_F64>(s, (const TW*)s->A, (size_t)s->lda, s->xa, s->xperm, s->xpiv, s->xst, s->xrcph,
                                     s->xrcpl, s->xlinvh, s->xlinvl, s->xuinvh, s->xuinvl);
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
                    : s->cluster ? launch(s, k_xref_refine<TW, TF, MV, ClusterTeam>, P)
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
    gb_status e = s->G == 1   ? launch(s, k_step<TW, TF, MV, CtaTeam>, P)
                  : s->cluster ? launch(s, k_step<TW, TF, MV, ClusterTeam>, P)
                               : launch(s, k_step<TW, TF, MV, GridTeam>, P);
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
    auto go = [&](auto kc, auto kcl, auto kg) {
      return s->G == 1 ? launch(s, kc, P, what) : s->cluster ? launch(s, kcl, P, what) : launch(s, kg, P, what);
    };
    if (what == 2 || what == 5) {
      // residual(a, x, b, ctx): the mode template is irrelevant for it
      P.ur = fmt == GB_QUAD ? UR_DD : (fmt == GB_DOUBLE ? UR_F64 : UR_F32);
      e = go(k_debug<MV, TW, TF, MV, CtaTeam>, k_debug<MV, TW, TF, MV, ClusterTeam>, k_debug<MV, TW, TF, MV, GridTeam>);
    } else if (what == 3) {
      e = go(k_debug<UM, TW, TF, MV, CtaTeam>, k_debug<UM, TW, TF, MV, ClusterTeam>, k_debug<UM, TW, TF, MV, GridTeam>);
    } else if (fmt == op_format()) {
      e = go(k_debug<MV, TW, TF, MV, CtaTeam>, k_debug<MV, TW, TF, MV, ClusterTeam>, k_debug<MV, TW, TF, MV, GridTeam>);
    } else {
      return fail(GB_ERR_UNSUPPORTED, "operator context differs from this solver's matvec format");
    }
    if (e != GB_OK) return e;
    CK(cudaMemcpyAsync(out, s->dtmp, sizeof(double) * n, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    return GB_OK;
  }

  // device time of one kernel-level op launch (what as in debug(), operator
  // in this solver's matvec format), averaged over `reps` back-to-back
  // launches on device-resident data (the vector left in rtmp)
  static gb_status time_op(gb_solver* s, int what, int reps, double* ms) {
    P_t P = make(s);
    if (what == 2) P.ur = s->o.ur == GB_QUAD ? UR_DD : (s->o.ur == GB_DOUBLE ? UR_F64 : UR_F32);
    auto one = [&]() -> gb_status {
      auto go = [&](auto kc, auto kcl, auto kg) {
        return s->G == 1 ? launch(s, kc, P, what) : s->cluster ? launch(s, kcl, P, what) : launch(s, kg, P, what);
      };
      if (what == 3)
        return go(k_debug<UM, TW, TF, MV, CtaTeam>, k_debug<UM, TW, TF, MV, ClusterTeam>,
                  k_debug<UM, TW, TF, MV, GridTeam>);
      return go(k_debug<MV, TW, TF, MV, CtaTeam>, k_debug<MV, TW, TF, MV, ClusterTeam>,
                k_debug<MV, TW, TF, MV, GridTeam>);
    };
    gb_status e = one();  // warm-up
    if (e != GB_OK) return e;
    CK(cudaEventRecord(s->ev0, s->stream));
    for (int i = 0; i < reps; ++i) {
      e = one();
      if (e != GB_OK) return e;
    }
    CK(cudaEventRecord(s->ev1, s->stream));
    CK(cudaEventSynchronize(s->ev1));
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, s->ev0, s->ev1));
    *ms = (double)t / reps;
    return GB_OK;
  }

  static gb_status get_x(gb_solver* s, double* x) {
    count_launch();
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

  static gb_status batched(int count, int n, const gb_options* o, int i_max, double c_conv, const double* a,
                           const double* b, int on_device, gb_batch_out* out, double* device_ms, cudaStream_t st) {
    if (n > 600) return fail(GB_ERR_UNSUPPORTED, "batched mode needs n <= 600 (dd GEPP reference solution)");
    const int m = o->m, k = o->k, ldv = (n + 31) & ~31, S = m + k + 2;
    SlotLayout Ly;
    size_t off = 0;
    auto take = [&](size_t bytes) {
      off = (off + 255) & ~size_t(255);
      size_t r = off;
      off += bytes;
      return r;
    };
    Ly.A = take(sizeof(TW) * (size_t)n * ldv);
    Ly.b = take(sizeof(TW) * ldv);
    Ly.LU = take(sizeof(TF) * (size_t)n * ldv);
    Ly.lubuf = take(sizeof(double) * (size_t)n * n);
    Ly.perm = take(sizeof(int) * ldv);
    Ly.rcph = take(sizeof(double) * ldv);
    Ly.rcpl = take(sizeof(double) * ldv);
    Ly.linvh = take(sizeof(double) * (size_t)ldv * (kInvStride / 32));
    Ly.linvl = take(sizeof(double) * (size_t)ldv * (kInvStride / 32));
    Ly.uinvh = take(sizeof(double) * (size_t)ldv * (kInvStride / 32));
    Ly.uinvl = take(sizeof(double) * (size_t)ldv * (kInvStride / 32));
    Ly.xs = take(sizeof(TW) * ldv);
    Ly.r = take(sizeof(double) * ldv);
    Ly.xref = take(sizeof(double) * ldv);
    Ly.rtmp = take(sizeof(double) * ldv);
    Ly.dtmp = take(sizeof(double) * ldv);
    Ly.V = take(sizeof(TW) * (size_t)(m + 1) * ldv);
    Ly.w = take(sizeof(TW) * ldv);
    Ly.xk = take(sizeof(TW) * ldv);
    Ly.res = take(sizeof(TW) * ldv);
    Ly.s = take(sizeof(TW) * ldv);
    Ly.rhat = take(sizeof(TW) * ldv);
    Ly.C = take(sizeof(TW) * (size_t)(k + 1) * ldv);
    Ly.U = take(sizeof(TW) * (size_t)(k + 1) * ldv);
    Ly.Cn = take(sizeof(TW) * (size_t)(k + 1) * ldv);
    Ly.Un = take(sizeof(TW) * (size_t)(k + 1) * ldv);
    Ly.Ut = take(sizeof(TW) * (size_t)(k + 1) * ldv);
    Ly.Yt = take(sizeof(TW) * (size_t)(k + 1) * ldv);
    Ly.Wd = take(sizeof(double) * (size_t)(k + 1) * ldv);
    Ly.Qd = take(sizeof(double) * (size_t)(k + 1) * ldv);
    Ly.H = take(sizeof(double) * (size_t)(m + 1) * m);
    Ly.R = take(sizeof(double) * (size_t)(m + 1) * m);
    Ly.B = take(sizeof(double) * (size_t)(k + 1) * m);
    Ly.bc = take(sizeof(double) * ((size_t)3 * S + 2 * (size_t)S * (k + 2) + 2 * (size_t)(k + 1) * (k + 1) + 64));
    Ly.dense = take(sizeof(double) * ((size_t)10 * S * S + 24 * (size_t)S * (k + 3) + 4096));
    Ly.gram = take(sizeof(double) * (size_t)2 * S * S);
    Ly.ybuf = take(16 * (size_t)ldv);
    Ly.ctr = take(32);
    Ly.epoch = take(16);
    Ly.cyc_it = take(sizeof(int) * (o->max_cycles + 4));
    Ly.cyc_ke = take(sizeof(int) * (o->max_cycles + 4));
    Ly.keff_io = take(16);
    Ly.flags = take(16);
    Ly.has_xref = take(16);
    Ly.out = take(sizeof(gb_step_info));
    Ly.xa = take(sizeof(double) * (size_t)n * n);
    Ly.xb = take(sizeof(double) * (size_t)n * n);
    Ly.xyh = take(sizeof(double) * ldv);
    Ly.xyl = take(sizeof(double) * ldv);
    Ly.xperm = take(sizeof(int) * ldv);
    Ly.stride = (off + 255) & ~size_t(255);

    const size_t sm = smem_bytes_for(m, k);
    gb_status e = set_smem(k_batched<TW, TF, MV>, sm);
    if (e != GB_OK) return e;
    int dev = 0, sms = 148, per = 1;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_batched<TW, TF, MV>, kThreads, sm));
    const int grid = std::max(1, std::min(count, sms * std::max(per, 1)));
    // device buffers: a grow-only per-process pool (no cudaMalloc/cudaFree on
    // the per-batch path once warm), guarded for concurrent callers
    std::lock_guard<std::mutex> guard(batch_pool().mu);
    const size_t na = (size_t)count * n * n, nb = (size_t)count * n;
    const size_t ints = (size_t)count * (5 + i_max) + 1, dbls = (size_t)count * (2 * i_max + n + 1);
    char* slots = batch_pool().get(0, Ly.stride * grid);
    int* ibuf = reinterpret_cast<int*>(batch_pool().get(1, sizeof(int) * ints));
    double* dbuf = reinterpret_cast<double*>(batch_pool().get(2, sizeof(double) * dbls));
    if (!slots || !ibuf || !dbuf) return fail(GB_ERR_CUDA, "batched workspace allocation failed");
    CK(cudaMemsetAsync(slots, 0, Ly.stride * grid, st));
    const double *da = a, *db = b;
    if (!on_device) {
      double* ta = reinterpret_cast<double*>(batch_pool().get(3, sizeof(double) * na));
      double* tb = reinterpret_cast<double*>(batch_pool().get(4, sizeof(double) * nb));
      if (!ta || !tb) return fail(GB_ERR_CUDA, "batched input allocation failed");
      CK(cudaMemcpyAsync(ta, a, sizeof(double) * na, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(tb, b, sizeof(double) * nb, cudaMemcpyHostToDevice, st));
      da = ta;
      db = tb;
    }
    CK(cudaMemsetAsync(ibuf, 0, sizeof(int) * ints, st));
    BatchArgs A;
    A.count = count;
    A.n = n;
    A.i_max = i_max;
    A.c_conv = c_conv;
    A.u_unit = sizeof(TW) == 4 ? 5.9604644775390625e-08 : 1.1102230246251565e-16;
    A.a = da;
    A.b = db;
    A.slots = slots;
    A.L = Ly;
    A.next = ibuf;
    A.converged = ibuf + 1;
    A.steps = A.converged + count;
    A.reason = A.steps + count;
    A.flags = A.reason + count;
    A.inner = A.flags + count;
    A.nbe = dbuf;
    A.ferr = A.nbe + (size_t)count * i_max;
    A.x = A.ferr + (size_t)count * i_max;
    A.growth = A.x + (size_t)count * n;
    A.m = m;
    A.k = k;
    A.max_cycles = o->max_cycles;
    A.reorth = o->reorthogonalize;
    A.explicit_res = o->explicit_residual;
    A.method = o->method == GB_SIR ? METH_SIR
               : (o->method == GB_GMRES_IR || o->method == GB_SGMRES_IR) ? METH_GMRES
                                                                          : METH_GCRODR;
    A.ur = o->ur == GB_QUAD ? UR_DD : (o->ur == GB_DOUBLE ? UR_F64 : UR_F32);
    A.tau = o->tau;
    A.fast_cap = fast_cap(m, k);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, st));
    count_launch();
    k_batched<TW, TF, MV><<<grid, kThreads, sm, st>>>(A);
    CK(cudaGetLastError());
    CK(cudaEventRecord(e1, st));
    // outputs
    CK(cudaMemcpyAsync(out->converged, A.converged, sizeof(int) * count, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(out->steps, A.steps, sizeof(int) * count, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(out->reason, A.reason, sizeof(int) * count, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(out->flags, A.flags, sizeof(int) * count, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(out->inner, A.inner, sizeof(int) * count * i_max, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(out->nbe, A.nbe, sizeof(double) * count * i_max, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(out->ferr, A.ferr, sizeof(double) * count * i_max, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(out->x, A.x, sizeof(double) * count * n, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(out->growth, A.growth, sizeof(double) * count, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (device_ms) *device_ms = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return GB_OK;
  }

  static const VariantOps* table() {
    static const VariantOps t{setup, set_system, factor, x0, xref, step, debug, get_x, get_lu, time_op, batched};
    return &t;
  }
};

}  // namespace
