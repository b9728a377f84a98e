// Restarted GMRES(m) and GCRO-DR(m, k) on a Team, plus one refinement step.
//
// Reference (paths under /root/reference/pkg/src/irkit):
//   arnoldi_cycle           gmres.py:123-215   (MGS, selective reorth, Givens)
//   _recurrence_residual    gmres.py:218-232
//   gmres_solve             gmres.py:235-311
//   harmonic_ritz_first     gcrodr.py:140-168
//   harmonic_ritz_recycle   gcrodr.py:171-197
//   _real_basis_smallest    gcrodr.py:104-137
//   gcrodr_solve            gcrodr.py:221-419
//   _refine loop body       refine.py:362-407 (host loop; one step per launch)
//
// All CTAs of a GridTeam execute the same control flow on bit-identical
// scalars.  Long vectors are sliced by rows across CTAs; small dense work
// (Givens least squares, harmonic-Ritz eigenproblems, QR of small matrices)
// is done by the leader CTA and broadcast through global memory.
#pragma once
#include "gb_dense.cuh"
#include "gb_ops.cuh"

namespace gb {

// leader-only orthogonalisation for n <= kLeaderOrthRows (w in registers)
constexpr int kThreadsPerCta = 256;
constexpr int kLeaderOrthRows = 2048;

// status bits reported per inner solve
enum : int { KS_CONVERGED = 1, KS_STAGNATED = 2, KS_BREAKDOWN = 4 };

template <class TW, class TA, class TF, int MV>
struct Krylov {
  using Y = typename Arith<MV>::T;
  // sizes / options
  int n, ldv, m, k, max_cycles;
  double tau;
  int reorth, recycling;
  int explicit_res;  // restart_residual / cycle_residual == "explicit"
  // problem
  SysView<TA, TF> sys;
  // long vectors (ldv stride)
  TW *V, *w, *x, *res, *s, *rhat;
  TW *C, *U, *Cn, *Un, *Ut, *Yt;  // (k + 1) columns each
  double *Wd, *Qd;                // fp64 tall (k + 1) columns
  // small dense (column-major fp64)
  double *H, *R, *B;  // (m+1) x m, (m+1) x m, (k+1) x m
  double* bc;         // broadcast area
  double* dense;      // leader scratch
  double* gram;       // G * gram_stride partials
  size_t gram_stride;
  Y* ybuf;
  // per-solve outputs
  int* cycle_iters;  // [max_cycles + 1]
  int* cycle_keff;   // [max_cycles + 1]
  // recycle state carried across solves
  int* keff_io;  // [1]
  // leader fast scratch in shared memory (reuses the TRSV tile region while
  // no substitution is running); nullptr -> global scratch only
  double* fast;
  int fast_cap;  // doubles
  int ops_bytes;  // size of the shared op region (TRSV tiles / leader scratch)
  // the op region itself: packed Hessenberg storage for eigenproblems whose
  // dense scratch does not fit it (gb_dense.cuh warp_hqr)
  double* pack;
};

// shared-memory need (doubles) of the leader's dense work at dimension p
__host__ __device__ inline int leader_fast_need(int p, int kk) { return 3 * p * p + 5 * p * (kk + 2) + 8 * p + 64; }

struct StepScalars {
  int ncycles, status, applies, keff;
};

// --------------------------------------------------------------------------
// helpers
// --------------------------------------------------------------------------
template <class T>
GB_DEVICE T* colp(T* base, int ldv, int i) { return base + (size_t)i * ldv; }

// out[i] = X_i . y over two column groups (X1: K1 cols, X2: K2 cols)
template <class TW, class Team>
__device__ void team_tvec2(Team& t, const TW* X1, int K1, const TW* X2, int K2, int ldv, const TW* y,
                           int n, double* out, double* tmp) {
  using Acc = typename Fmt<TW>::Acc;
  int lo, hi;
  t.rows(n, lo, hi);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int K = K1 + K2;
  for (int i = wid; i < K; i += nw) {
    const TW* xi = i < K1 ? X1 + (size_t)i * ldv : X2 + (size_t)(i - K1) * ldv;
    Acc a = Acc(0);
    for (int j = lo + lane; j < hi; j += 32) a = Fmt<TW>::mac(a, xi[j], y[j]);
    a = warp_sum(a);
    if (lane == 0) tmp[i] = (double)a;
  }
  __syncthreads();
  if constexpr (Team::kGrid) {
    t.template sum_vec<double>(tmp, out, K);
    for (int i = threadIdx.x; i < K; i += blockDim.x) out[i] = (double)(Acc)out[i];
  } else {
    for (int i = threadIdx.x; i < K; i += blockDim.x) out[i] = tmp[i];
  }
  __syncthreads();
}

// column norms ||X_i|| in the work format
template <class TW, class Team>
__device__ void team_colnorms(Team& t, const TW* X, int K, int ldv, int n, double* out, double* tmp) {
  using Acc = typename Fmt<TW>::Acc;
  int lo, hi;
  t.rows(n, lo, hi);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = wid; i < K; i += nw) {
    const TW* xi = X + (size_t)i * ldv;
    Acc a = Acc(0);
    for (int j = lo + lane; j < hi; j += 32) a = Fmt<TW>::mac(a, xi[j], xi[j]);
    a = warp_sum(a);
    if (lane == 0) tmp[i] = (double)a;
  }
  __syncthreads();
  if constexpr (Team::kGrid) {
    t.template sum_vec<double>(tmp, out, K);
    for (int i = threadIdx.x; i < K; i += blockDim.x) out[i] = Fmt<TW>::sqrt_((double)(Acc)out[i]);
  } else {
    for (int i = threadIdx.x; i < K; i += blockDim.x) out[i] = Fmt<TW>::sqrt_(tmp[i]);
  }
  __syncthreads();
}

// leader writes, everybody reads: barrier + invalidate
template <class Team>
GB_DEVICE void bcast_sync(Team& t) { t.sync(); }

// --------------------------------------------------------------------------
// operator application  w = fl_u(U^-1 L^-1 (A v)[perm])
// --------------------------------------------------------------------------
template <class TW, class TA, class TF, int MV, class Team>
__device__ void apply_A(Team& t, Krylov<TW, TA, TF, MV>& K, TrsvSync& ts, const TW* v, TW* out,
                        void* smem, int& applies) {
  t.sync();  // v complete
  op_apply<MV>(t, K.sys, v, (const TW*)nullptr, out, K.ybuf, ts, smem);
  ++applies;
}

// --------------------------------------------------------------------------
// one Arnoldi cycle (gmres.py:123-215).  V_0 from r0/beta; H, R (rotated), B
// written by the leader; returns steps, flags; the Givens LS solution y is
// written to K.bc[0..steps) when want_y.
// smem layout (doubles): cs[m], sn[m], g[m+1], col[m+2], red[64], tmp[...]
// --------------------------------------------------------------------------
struct CycleOut {
  int steps;
  bool converged, breakdown;
};

// Givens update of column j (gmres.py:99-114, 182-190) by thread 0: each
// product and sum rounded to u.  col[0..j+1] in, rotated column in rot.
template <class TW>
GB_DEVICE void givens_update(int j, const double* col, double* rot, double* cs, double* sn, double* g) {
  using F = Fmt<TW>;
  for (int i = 0; i <= j + 1; ++i) rot[i] = col[i];
  for (int i = 0; i < j; ++i) {
    double a = rot[i], b = rot[i + 1];
    rot[i] = F::rnd(F::rnd(cs[i] * a) + F::rnd(sn[i] * b));
    rot[i + 1] = F::rnd(F::rnd(cs[i] * b) - F::rnd(sn[i] * a));
  }
  double hh = hypot(rot[j], rot[j + 1]);
  double c = 1.0, s2 = 0.0;
  if (hh != 0.0) {
    c = F::rnd(rot[j] / hh);
    s2 = F::rnd(rot[j + 1] / hh);
  }
  cs[j] = c;
  sn[j] = s2;
  rot[j] = F::rnd(F::rnd(c * rot[j]) + F::rnd(s2 * rot[j + 1]));
  rot[j + 1] = 0.0;
  double gj = g[j];
  g[j] = F::rnd(F::rnd(c * gj) + F::rnd(s2 * 0.0));
  g[j + 1] = F::rnd(F::rnd(c * 0.0) - F::rnd(s2 * gj));
}

// spare broadcast slots after the recycle matrices in K.bc (64 doubles)
template <class TW, class TA, class TF, int MV>
GB_DEVICE double* bc_orth(const Krylov<TW, TA, TF, MV>& K) {
  const size_t S = (size_t)K.m + K.k + 2;
  return K.bc + 3 * S + 2 * S * (K.k + 2) + 2 * (size_t)(K.k + 1) * (K.k + 1);
}

// block-wide sum of this thread's partial (all threads get it)
template <class A>
GB_DEVICE A blk_sum1(A v, double* red) {
  A a[1] = {v};
  block_sum<A, 1>(a, reinterpret_cast<A*>(red));
  return a[0];
}

// Leader-only orthogonalisation of w against C (one CGS projection) and V
// (MGS with selective reorthogonalisation), the Givens update and the next
// basis vector -- the whole of gmres.py:150-201 for one step, run by the
// leader CTA over all n <= kLeaderOrthRows rows.  w lives in registers (QW
// rows per thread) and the next basis column is loaded into registers before
// each block reduction, so every dot costs one block reduction and no team
// barrier: a step takes two team barriers instead of j + 4.  Results through
// bc_orth: [0] = ||w|| after orthogonalisation, [1] = |g_{j+1}|.
template <class TW, class TA, class TF, int MV>
__device__ __noinline__ void leader_orth(Krylov<TW, TA, TF, MV>& K, int j, int kc, double* cs, double* sn, double* g,
                            double* col, double* red, double* tmp) {
  using F = Fmt<TW>;
  using Acc = typename F::Acc;
  constexpr int QW = kLeaderOrthRows / kThreadsPerCta;
  const int n = K.n, ldv = K.ldv, M = K.m;
  const int tid = threadIdx.x, bd = blockDim.x;
  TW wr[QW], cur[QW], prv[QW];
  auto ld_col = [&](const TW* base, TW (&d)[QW]) {
#pragma unroll
    for (int q = 0; q < QW; ++q) {
      const int r = tid + q * bd;
      d[q] = r < n ? base[r] : TW(0);
    }
  };
#pragma unroll
  for (int q = 0; q < QW; ++q) {
    const int r = tid + q * bd;
    wr[q] = r < n ? __ldcg(K.w + r) : TW(0);
  }
  if (kc > 0) {
    // cc = C^T w (each dot in the work format), then w -= cc_i C_i in order
    ld_col(K.C, cur);
    for (int i = 0; i < kc; ++i) {
      Acc a = Acc(0);
#pragma unroll
      for (int q = 0; q < QW; ++q) a = F::mac(a, cur[q], wr[q]);
      if (i + 1 < kc) ld_col(K.C + (size_t)(i + 1) * ldv, cur);
      a = blk_sum1<Acc>(a, red);
      if (tid == 0) tmp[i] = (double)a;
    }
    __syncthreads();
    for (int i = 0; i < kc; ++i) {
      ld_col(K.C + (size_t)i * ldv, cur);
      const double ci = tmp[i];
#pragma unroll
      for (int q = 0; q < QW; ++q) wr[q] = F::axpy(-ci, cur[q], wr[q]);
    }
    for (int i = tid; i < kc; i += bd) K.B[IX(i, j, K.k + 1)] = tmp[i];
    __syncthreads();
  }
  auto nrm2 = [&]() {
    Acc a = Acc(0);
#pragma unroll
    for (int q = 0; q < QW; ++q) a = F::mac(a, wr[q], wr[q]);
    return F::sqrt_((double)blk_sum1<Acc>(a, red));
  };
  const double wnorm0 = nrm2();
  // MGS: h_i = v_i . w ; w -= h_i v_i  (axpy fused with the next dot)
  auto mgs = [&](bool accumulate) {
    double hprev = 0.0;
    ld_col(K.V, cur);
    for (int i = 0; i <= j; ++i) {
      Acc a = Acc(0);
#pragma unroll
      for (int q = 0; q < QW; ++q) {
        if (i > 0) wr[q] = F::axpy(-hprev, prv[q], wr[q]);
        a = F::mac(a, cur[q], wr[q]);
      }
#pragma unroll
      for (int q = 0; q < QW; ++q) prv[q] = cur[q];
      if (i < j) ld_col(K.V + (size_t)(i + 1) * ldv, cur);
      hprev = (double)blk_sum1<Acc>(a, red);
      if (tid == 0) col[i] = accumulate ? F::rnd(col[i] + hprev) : hprev;
    }
#pragma unroll
    for (int q = 0; q < QW; ++q) wr[q] = F::axpy(-hprev, prv[q], wr[q]);
  };
  mgs(false);
  double hlast = nrm2();
  if (K.reorth && hlast < sqrt(F::u) * wnorm0) {
    mgs(true);
    hlast = nrm2();
  }
  if (tid == 0) {
    col[j + 1] = hlast;
    givens_update<TW>(j, col, tmp, cs, sn, g);
  }
  __syncthreads();
  for (int i = tid; i <= j + 1; i += bd) {
    K.H[IX(i, j, M + 1)] = col[i];
    K.R[IX(i, j, M + 1)] = tmp[i];
  }
  if (hlast != 0.0) {
    TW* vn = K.V + (size_t)(j + 1) * ldv;
    const double rh = 1.0 / hlast;
#pragma unroll
    for (int q = 0; q < QW; ++q) {
      const int r = tid + q * bd;
      if (r < n) vn[r] = F::scale(rh, wr[q]);
    }
  }
  if (tid == 0) {
    double* o = bc_orth(K);
    o[0] = hlast;
    o[1] = fabs(g[j + 1]);
  }
}

template <class TW, class TA, class TF, int MV, class Team>
__device__ CycleOut arnoldi_cycle(Team& t, Krylov<TW, TA, TF, MV>& K, TrsvSync& ts, const TW* r0,
                                  double beta, int mb, double tol_abs, int kc, bool want_y,
                                  double* sm, void* smem_ops, int& applies) {
  using F = Fmt<TW>;
  const int n = K.n, ldv = K.ldv, M = K.m;
  double* cs = sm;
  double* sn = cs + M;
  double* g = sn + M;
  double* col = g + M + 1;
  double* red = col + M + 2;
  double* tmp = red + 64;  // >= k + 2 + m
  const double sqrt_u = sqrt(F::u);
  if (threadIdx.x == 0) g[0] = beta;
  team_scale(t, 1.0 / beta, r0, K.V, n);
  CycleOut co{0, false, false};
  int lo, hi;
  t.rows(n, lo, hi);
  for (int j = 0; j < mb; ++j) {
    TW* vj = colp(K.V, ldv, j);
    mark(ts.log, 20);
    apply_A(t, K, ts, vj, K.w, smem_ops, applies);
    if (Team::kGrid && n <= kLeaderOrthRows && blockDim.x == kThreadsPerCta) {
      t.sync();  // w complete
      if (t.leader()) leader_orth(K, j, kc, cs, sn, g, col, red, tmp);
      t.sync();
      const double* o = bc_orth(K);
      const double hlast = __ldcg(o), estimate = __ldcg(o + 1);
      co.steps = j + 1;
      mark(ts.log, 25);
      if (hlast == 0.0) {
        co.breakdown = co.converged = true;
        break;
      }
      if (estimate <= tol_abs) {
        co.converged = true;
        break;
      }
      continue;
    }
    // deflation against C: one CGS projection, sequential subtraction
    if (kc > 0) {
      team_tvec2<TW>(t, K.C, kc, (const TW*)nullptr, 0, ldv, K.w, n, tmp, red);
      for (int r = lo + threadIdx.x; r < hi; r += blockDim.x) {
        TW wr = K.w[r];
        for (int i = 0; i < kc; ++i) wr = F::axpy(-tmp[i], K.C[(size_t)i * ldv + r], wr);
        K.w[r] = wr;
      }
      if (t.leader())
        for (int i = threadIdx.x; i < kc; i += blockDim.x) K.B[IX(i, j, K.k + 1)] = tmp[i];
      __syncthreads();
    }
    mark(ts.log, 21);
    const double wnorm0 = team_nrm2<TW>(t, K.w, n, red);
    mark(ts.log, 22);
    // MGS: h_i = v_i . w ; w -= h_i v_i  (axpy fused with the next dot).
    // This thread's rows of w stay in registers for the whole sweep and the
    // next basis column is loaded before each reduction (the loads do not
    // depend on it), so one team reduction is the only latency per i.
    double hprev = 0.0;
    // Large cooperative grids run the sweep on a sub-team of T CTAs (1024 rows
    // each): every link is one exchange through global memory, and T = 16
    // slots are polled in a fraction of the time 148 take.  The other CTAs
    // wait at the barrier below; the h column is broadcast through colbuf.
    bool sub_done = false;
    // (cooperative-grid team type only: the cluster kernel must not carry this code, its
    // register budget is what the cfg2 step time hangs on)
    if constexpr (Team::kGrid && Team::kTB == kTrsvB) {
      int T = 0;
      if (!t.clu && t.spart == nullptr && t.size() > 32 && j + 2 <= kColBuf && n <= 32 * 1024) T = (n + 1023) / 1024;
      if (T > 0) {
      sub_done = true;
      constexpr int QW = 4;
      if (t.rank() < T) {
        const int per = (((n + T - 1) / T) + 31) & ~31;  // <= 1024 rows
        const int slo = min(n, t.rank() * per), shi = min(n, slo + per);
        TW wr[QW], vc[QW], vn[QW];
#pragma unroll
        for (int q = 0; q < QW; ++q) {
          const int r = slo + threadIdx.x + q * blockDim.x;
          wr[q] = r < shi ? __ldcg(K.w + r) : TW(0);
          vc[q] = r < shi ? K.V[r] : TW(0);
        }
        for (int i = 0; i <= j; ++i) {
          typename F::Acc a = typename F::Acc(0);
#pragma unroll
          for (int q = 0; q < QW; ++q) {
            const int r = slo + threadIdx.x + q * blockDim.x;
            if (r < shi) {
              if (i > 0) wr[q] = F::axpy(-hprev, vn[q], wr[q]);
              a = F::mac(a, vc[q], wr[q]);
            }
          }
#pragma unroll
          for (int q = 0; q < QW; ++q) {
            const int r = slo + threadIdx.x + q * blockDim.x;
            vn[q] = vc[q];
            vc[q] = (r < shi && i < j) ? K.V[(size_t)(i + 1) * ldv + r] : TW(0);
          }
          a = t.template reduce1_sub<typename F::Acc>(a, reinterpret_cast<typename F::Acc*>(red), T);
          hprev = (double)a;
          if (threadIdx.x == 0) col[i] = hprev;
        }
#pragma unroll
        for (int q = 0; q < QW; ++q) {
          const int r = slo + threadIdx.x + q * blockDim.x;
          if (r < shi) K.w[r] = F::axpy(-hprev, vn[q], wr[q]);
        }
        __syncthreads();
        if (t.leader())
          for (int i = threadIdx.x; i <= j; i += blockDim.x) t.colbuf()[i] = col[i];
      }
      t.sync();
      for (int i = threadIdx.x; i <= j; i += blockDim.x) col[i] = __ldcg(t.colbuf() + i);
      hprev = __ldcg(t.colbuf() + j);
      __syncthreads();
      }
    }
    if (!sub_done) {
      constexpr int QW = 4;  // rows per thread: a CTA slice has <= 4 * blockDim rows
      TW wr[QW], vc[QW], vn[QW];
#pragma unroll
      for (int q = 0; q < QW; ++q) {
        const int r = lo + threadIdx.x + q * blockDim.x;
        wr[q] = r < hi ? K.w[r] : TW(0);
        vc[q] = r < hi ? K.V[r] : TW(0);
      }
      for (int i = 0; i <= j; ++i) {
        typename F::Acc a[1] = {typename F::Acc(0)};
#pragma unroll
        for (int q = 0; q < QW; ++q) {
          const int r = lo + threadIdx.x + q * blockDim.x;
          if (r < hi) {
            if (i > 0) wr[q] = F::axpy(-hprev, vn[q], wr[q]);  // vn = v_{i-1}
            a[0] = F::mac(a[0], vc[q], wr[q]);
          }
        }
        // v_{i-1} <- v_i ; prefetch v_{i+1}
#pragma unroll
        for (int q = 0; q < QW; ++q) {
          const int r = lo + threadIdx.x + q * blockDim.x;
          vn[q] = vc[q];
          vc[q] = (r < hi && i < j) ? K.V[(size_t)(i + 1) * ldv + r] : TW(0);
        }
        if constexpr (Team::kGrid && Team::kTB == kTrsvB)
          a[0] = t.template reduce1<typename F::Acc>(a[0], reinterpret_cast<typename F::Acc*>(red));
        else
          t.template reduce<typename F::Acc, 1>(a, reinterpret_cast<typename F::Acc*>(red));
        hprev = (double)a[0];
        if (threadIdx.x == 0) col[i] = hprev;
      }
#pragma unroll
      for (int q = 0; q < QW; ++q) {
        const int r = lo + threadIdx.x + q * blockDim.x;
        if (r < hi) K.w[r] = F::axpy(-hprev, vn[q], wr[q]);  // vn = v_j
      }
    }
    mark(ts.log, 23);
    double hlast = team_nrm2<TW>(t, K.w, n, red);
    mark(ts.log, 24);
    if (K.reorth && hlast < sqrt_u * wnorm0) {
      for (int i = 0; i <= j; ++i) {
        const TW* vi = colp(K.V, ldv, i);
        const TW* vp = i > 0 ? colp(K.V, ldv, i - 1) : nullptr;
        typename F::Acc a[1] = {typename F::Acc(0)};
        for (int r = lo + threadIdx.x; r < hi; r += blockDim.x) {
          TW wr = K.w[r];
          if (i > 0) {
            wr = F::axpy(-hprev, vp[r], wr);
            K.w[r] = wr;
          }
          a[0] = F::mac(a[0], vi[r], wr);
        }
        t.template reduce<typename F::Acc, 1>(a, reinterpret_cast<typename F::Acc*>(red));
        hprev = (double)a[0];
        if (threadIdx.x == 0) col[i] = F::rnd(col[i] + hprev);
      }
      const TW* vp = colp(K.V, ldv, j);
      for (int r = lo + threadIdx.x; r < hi; r += blockDim.x) K.w[r] = F::axpy(-hprev, vp[r], K.w[r]);
      hlast = team_nrm2<TW>(t, K.w, n, red);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      col[j + 1] = hlast;
      givens_update<TW>(j, col, tmp, cs, sn, g);
    }
    __syncthreads();
    if (t.leader()) {
      for (int i = threadIdx.x; i <= j + 1; i += blockDim.x) {
        K.H[IX(i, j, M + 1)] = col[i];
        K.R[IX(i, j, M + 1)] = tmp[i];
      }
    }
    const double estimate = fabs(g[j + 1]);
    co.steps = j + 1;
    mark(ts.log, 25);
    __syncthreads();
    if (hlast == 0.0) {
      co.breakdown = co.converged = true;
      break;
    }
    team_scale(t, 1.0 / hlast, K.w, colp(K.V, ldv, j + 1), n);
    if (estimate <= tol_abs) {
      co.converged = true;
      break;
    }
  }
  if (want_y) {
    // y = fl_u(R^-1 g) on the leader (gmres.py:203-204)
    t.sync();
    if (t.leader()) {
      blk_upper_solve(K.R, M + 1, co.steps, g, tmp);
      for (int i = threadIdx.x; i < co.steps; i += blockDim.x) K.bc[i] = F::rnd(tmp[i]);
    }
  }
  t.sync();
  return co;
}

// x += sum_i y_i V_i  (sequential, u arithmetic); y from K.bc
template <class TW, class Team>
__device__ void update_x(Team& t, TW* x, const TW* V, int ldv, const double* y, int cnt, int n) {
  int lo, hi;
  t.rows(n, lo, hi);
  for (int r = lo + threadIdx.x; r < hi; r += blockDim.x) {
    TW xr = x[r];
    for (int i = 0; i < cnt; ++i) xr = Fmt<TW>::axpy(__ldcg(y + i), V[(size_t)i * ldv + r], xr);
    x[r] = xr;
  }
}

// res = V (beta e1 - Hbar y) with t rounded (gmres.py:218-232); y at K.bc
template <class TW, class TA, class TF, int MV, class Team>
__device__ void recurrence_res(Team& t, Krylov<TW, TA, TF, MV>& K, int steps, double beta) {
  using F = Fmt<TW>;
  double* tv = K.bc + 2 * (K.m + K.k + 2);
  if (t.leader()) {
    for (int i = threadIdx.x; i <= steps; i += blockDim.x) {
      double acc = 0.0;
      for (int c = 0; c < steps; ++c) acc = __fma_rn(K.H[IX(i, c, K.m + 1)], K.bc[c], acc);
      double v = -acc;
      if (i == 0) v += beta;
      tv[i] = F::rnd(v);
    }
  }
  t.sync();
  int lo, hi;
  t.rows(K.n, lo, hi);
  for (int r = lo + threadIdx.x; r < hi; r += blockDim.x) {
    TW acc = TW(0);
    for (int i = 0; i <= steps; ++i) acc = F::axpy(__ldcg(tv + i), K.V[(size_t)i * K.ldv + r], acc);
    K.res[r] = acc;
  }
}

// res = fl_u(s - A~ x): the explicit boundary residual (gmres.py:294-295,
// gcrodr.py:301-304 and 376-379); one operator application, counted
template <class TW, class TA, class TF, int MV, class Team>
__device__ void explicit_residual(Team& t, Krylov<TW, TA, TF, MV>& K, TrsvSync& ts, void* smem_ops, int& applies) {
  apply_A(t, K, ts, K.x, K.w, smem_ops, applies);
  t.sync();
  int lo, hi;
  t.rows(K.n, lo, hi);
  for (int r = lo + threadIdx.x; r < hi; r += blockDim.x) K.res[r] = K.s[r] - K.w[r];
  t.sync();
}

// --------------------------------------------------------------------------
// harmonic Ritz selection on the leader.  M (p x p) column-major, destroyed.
// Writes P (p x keff, ldp) normalised columns; returns keff or -1 on failure.
// scratch: Z p*p, X 2p per thread-vector, wr, wi, ort, ord.
// --------------------------------------------------------------------------
static __device__ __noinline__ int leader_ritz_basis(double* Mx, int p, int kreq, double* P, int ldp, double* scr,
                                                     double* hp = nullptr) {
  double* Z = scr;
  double* wr = Z + (size_t)p * p;
  double* wi = wr + p;
  double* ort = wi + p;
  double* absv = ort + p;
  int* ord = reinterpret_cast<int*>(absv + p);
  int* sel = ord + p;  // selection: schur index per chosen eigen-slot
  int* kind = sel + (kreq + 2);
  double* X = reinterpret_cast<double*>(kind + (kreq + 2) + 2);
  X = reinterpret_cast<double*>(((uintptr_t)X + 15) & ~(uintptr_t)15);
  double* vre = X + 2 * (size_t)p * (kreq + 2);
  double* vim = vre + (size_t)p * (kreq + 2);
  __shared__ int s_ok, s_cnt;
  // non-finite check (eig_small: NoConvergence)
  if (threadIdx.x == 0) s_ok = 1;
  __syncthreads();
  for (int e = threadIdx.x; e < p * p; e += blockDim.x)
    if (!isfinite(Mx[e])) s_ok = 0;
  __syncthreads();
  if (!s_ok) return -1;
  const int nq = (p >= 128 && blockDim.x >= 256) ? 4 : 1;  // QR warps (reduced problems only, see below)
  const int nz = hqr_z_warps(p, (int)(blockDim.x >> 5), nq);
  // large problems (cfg5: p = 200): Hessenberg form + accumulated transformation by the whole
  // CTA; small ones (cfg2: p = 50, in shared memory) stay on the QR warp, where the CTA
  // barriers would cost more than they save.  Same arithmetic either way.
  const bool wide = p >= 128;
  if (wide) blk_orthes(Mx, p, p, Z, p, ort);
  if ((int)threadIdx.x < 32 * (nq + nz)) {  // warps 0 .. nq-1: QR iteration, then nz warps of Schur-vector updates
    bool ok = warp_hqr(Mx, p, p, Z, p, wr, wi, ort, hp, nz, wide, nq);
    if (threadIdx.x == 0) s_ok = ok ? 1 : 0;
  }
  __syncthreads();
  if (!s_ok) return -1;
  // stable sort by |lambda|
  for (int i = threadIdx.x; i < p; i += blockDim.x) absv[i] = hypot(wr[i], wi[i]);
  __syncthreads();
  for (int i = threadIdx.x; i < p; i += blockDim.x) {
    int rk = 0;
    for (int j = 0; j < p; ++j) rk += (absv[j] < absv[i]) || (absv[j] == absv[i] && j < i);
    ord[rk] = i;
  }
  __syncthreads();
  // _real_basis_smallest (gcrodr.py:104-137): choose Schur indices
  if (threadIdx.x == 0) {
    const int kk = min(kreq, p);
    const int allow = (kk + 1 <= p - 1) ? kk + 1 : kk;
    int cnt = 0, i = 0, nsel = 0;
    while (i < p && cnt < kk) {
      int si = ord[i];
      if (wi[si] == 0.0) {
        sel[nsel] = si;
        kind[nsel] = 0;  // real
        nsel++;
        cnt++;
        i++;
      } else if (cnt + 2 <= allow) {
        sel[nsel] = si;
        kind[nsel] = 1;  // re + im
        nsel++;
        cnt += 2;
        i += 2;
      } else if (cnt == 0) {
        sel[nsel] = si;
        kind[nsel] = 2;  // re only
        nsel++;
        cnt++;
        i++;
      } else {
        break;
      }
    }
    s_cnt = nsel;
    kind[kreq + 1] = cnt;
  }
  __syncthreads();
  const int nsel = s_cnt, keff = kind[kreq + 1];
  // Schur-form norm for the back-substitution safeguard
  __shared__ double s_norm;
  if (threadIdx.x == 0) {
    double nn = 0.0;
    for (int i = 0; i < p; ++i)
      for (int j = max(i - 1, 0); j < p; ++j) nn += fabs(Mx[IX(i, j, p)]);
    s_norm = nn;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < nsel; q += blockDim.x) {
    int si = sel[q];
    int schur_col = si;
    if (wi[si] != 0.0 && wi[si] < 0.0) schur_col = si - 1;  // pair start
    eigvec_one(Mx, p, p, Z, p, wr, wi, s_norm, schur_col, X + (size_t)q * 2 * p, p,
               vre + (size_t)q * p, vim + (size_t)q * p);
    if (wi[si] < 0.0) {  // conjugate requested: flip the imaginary part
      for (int i = 0; i < p; ++i) vim[(size_t)q * p + i] = -vim[(size_t)q * p + i];
    }
  }
  __syncthreads();
  // assemble P columns and normalise (reference re-normalises the complex
  // vector first: eig_small divides by its 2-norm, which is ~1)
  if (threadIdx.x == 0) {
    int c = 0;
    for (int q = 0; q < nsel; ++q) {
      const double* re = vre + (size_t)q * p;
      const double* im = vim + (size_t)q * p;
      double nn = 0.0;
      for (int i = 0; i < p; ++i) nn += re[i] * re[i] + im[i] * im[i];
      nn = sqrt(nn);
      if (nn == 0.0) nn = 1.0;
      for (int i = 0; i < p; ++i) P[IX(i, c, ldp)] = re[i] / nn;
      c++;
      if (kind[q] == 1) {
        for (int i = 0; i < p; ++i) P[IX(i, c, ldp)] = im[i] / nn;
        c++;
      }
    }
    for (int cc = 0; cc < c; ++cc) {
      double s = 0.0;
      for (int i = 0; i < p; ++i) s += P[IX(i, cc, ldp)] * P[IX(i, cc, ldp)];
      s = sqrt(s);
      if (s == 0.0) s = 1.0;
      for (int i = 0; i < p; ++i) P[IX(i, cc, ldp)] /= s;
    }
  }
  __syncthreads();
  return keff;
}

// C[r x c] = A[r x q] B[q x c] (column-major, fp64) by the CTA
static __device__ __noinline__ void blk_gemm(const double* A, int lda, const double* Bm, int ldb, double* Cm, int ldc,
                                int r, int q, int c, bool transA = false) {
  for (int e = threadIdx.x; e < r * c; e += blockDim.x) {
    int i = e % r, j = e / r;
    double acc = 0.0;
    for (int l = 0; l < q; ++l) {
      double a = transA ? A[IX(l, i, lda)] : A[IX(i, l, lda)];
      acc = __fma_rn(a, Bm[IX(l, j, ldb)], acc);
    }
    Cm[IX(i, j, ldc)] = acc;
  }
  __syncthreads();
}

// --------------------------------------------------------------------------
// distributed rebuild of the recycle space from small-matrix results at bc:
//   Yt = fl(Vh P)   Cn = fl(W Q)   Un = fl(Yt R^-1)
// Vh columns: [X1 (K1 cols), X2 (K2 cols)], W columns: [Y1 (K1), Y2 (K2 + 1)]
// --------------------------------------------------------------------------
template <class TW, class TA, class TF, int MV, class Team>
__device__ void rebuild_space(Team& t, Krylov<TW, TA, TF, MV>& K, const TW* X1, const TW* X2,
                              const TW* Y1, const TW* Y2, int K1, int K2, int kn, const double* P,
                              int ldp, const double* Q, int ldq, const double* Rm, int ldr) {
  using F = Fmt<TW>;
  int lo, hi;
  t.rows(K.n, lo, hi);
  const int ldv = K.ldv;
  const int pdim = K1 + K2;  // Vh columns
  for (int r = lo + threadIdx.x; r < hi; r += blockDim.x) {
    double yt[33];
    for (int c = 0; c < kn; ++c) {
      double a = 0.0, b = 0.0;
      for (int i = 0; i < pdim; ++i) {
        double v = i < K1 ? (double)X1[(size_t)i * ldv + r] : (double)X2[(size_t)(i - K1) * ldv + r];
        a = __fma_rn(v, __ldcg(P + IX(i, c, ldp)), a);
      }
      for (int i = 0; i <= pdim; ++i) {
        double v = i < K1 ? (double)Y1[(size_t)i * ldv + r] : (double)Y2[(size_t)(i - K1) * ldv + r];
        b = __fma_rn(v, __ldcg(Q + IX(i, c, ldq)), b);
      }
      yt[c] = F::rnd(a);
      K.Yt[(size_t)c * ldv + r] = (TW)yt[c];
      K.Cn[(size_t)c * ldv + r] = (TW)F::rnd(b);
    }
    // U = Yt R^-1  (row vector solve  u R = yt)
    for (int c = 0; c < kn; ++c) {
      double s = yt[c];
      for (int i = 0; i < c; ++i) s = __fma_rn(-yt[i], __ldcg(Rm + IX(i, c, ldr)), s);
      yt[c] = s / __ldcg(Rm + IX(c, c, ldr));
      K.Un[(size_t)c * ldv + r] = (TW)F::rnd(yt[c]);
    }
  }
}

template <class TW, class TA, class TF, int MV>
GB_DEVICE void swap_space(Krylov<TW, TA, TF, MV>& K) {
  TW* a = K.C;
  K.C = K.Cn;
  K.Cn = a;
  a = K.U;
  K.U = K.Un;
  K.Un = a;
}


// --------------------------------------------------------------------------
// bc layout (doubles), S = m + k + 2:
//   [0, S)           y (Givens or block LS solution); bc[S-1] = status word
//   [S, 2S)          gy
//   [2S, 3S)         recurrence coefficients t
//   [3S, ...)        P (S x (k+2)), Q (S x (k+2)), R ((k+1) x (k+1))
//   then             warm-start R ((k+1) x (k+1))
// --------------------------------------------------------------------------
template <class TW, class TA, class TF, int MV>
GB_DEVICE int bc_S(const Krylov<TW, TA, TF, MV>& K) { return K.m + K.k + 2; }
template <class TW, class TA, class TF, int MV>
GB_DEVICE double* bc_P(const Krylov<TW, TA, TF, MV>& K) { return K.bc + 3 * (size_t)bc_S(K); }
template <class TW, class TA, class TF, int MV>
GB_DEVICE double* bc_Q(const Krylov<TW, TA, TF, MV>& K) { return bc_P(K) + (size_t)bc_S(K) * (K.k + 2); }
template <class TW, class TA, class TF, int MV>
GB_DEVICE double* bc_R(const Krylov<TW, TA, TF, MV>& K) { return bc_Q(K) + (size_t)bc_S(K) * (K.k + 2); }
template <class TW, class TA, class TF, int MV>
GB_DEVICE double* bc_Rw(const Krylov<TW, TA, TF, MV>& K) { return bc_R(K) + (size_t)(K.k + 1) * (K.k + 1); }

// --------------------------------------------------------------------------
// distributed Householder QR of the tall fp64 matrix Wd (n x c): Q -> Qd,
// R -> bc_Rw (ld k+1), sign-fixed, rank-tested (densela.py:410-432).
// --------------------------------------------------------------------------
template <class TW, class TA, class TF, int MV, class Team>
__device__ bool team_qr_tall(Team& t, Krylov<TW, TA, TF, MV>& K, int c, double* sm) {
  const int n = K.n, ldv = K.ldv, ldr = K.k + 1;
  double* A = K.Wd;
  double* Q = K.Qd;
  double* Rm = bc_Rw(K);
  double* red = sm + 4 * K.m + 4;
  double* loc = red + 64;       // c + 2
  double* tot = loc + 40;       // c + 2
  double* taus = tot + 40;      // c
  __shared__ double s_beta, s_tau, s_scal;
  int lo, hi;
  t.rows(n, lo, hi);
  // non-finite entries -> RankDeficient
  double bad = 0.0;
  for (int r = lo + threadIdx.x; r < hi; r += blockDim.x)
    for (int j = 0; j < c; ++j)
      if (!isfinite(A[(size_t)j * ldv + r])) bad = 1.0;
  {
    double b2 = block_max(bad, red);
    b2 = t.finish_max(b2);
    if (b2 != 0.0) return false;
  }
  for (int j = 0; j < c; ++j) {
    double* aj = A + (size_t)j * ldv;
    double pp[2] = {0.0, 0.0};
    for (int r = max(lo, j + 1) + threadIdx.x; r < hi; r += blockDim.x) pp[0] = __fma_rn(aj[r], aj[r], pp[0]);
    if (threadIdx.x == 0 && j >= lo && j < hi) pp[1] = aj[j];
    block_sum<double, 2>(pp, red);
    t.template finish_sum<double, 2>(pp);
    if (threadIdx.x == 0) {
      double alpha = pp[1], xn = sqrt(pp[0]);
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
      taus[j] = s_tau;
    }
    __syncthreads();
    const double tj = s_tau, scal = s_scal, beta = s_beta;
    if (tj != 0.0)
      for (int r = max(lo, j + 1) + threadIdx.x; r < hi; r += blockDim.x) aj[r] *= scal;
    __syncthreads();
    if (threadIdx.x == 0 && j >= lo && j < hi) aj[j] = beta;
    __syncthreads();
    const int nl = c - j - 1;
    if (nl > 0 && tj != 0.0) {
      // w_l = A[j,l] + sum_{r>j} v_r A[r,l]
      for (int l = threadIdx.x; l < nl; l += blockDim.x) loc[l] = 0.0;
      __syncthreads();
      const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
      for (int l = wid; l < nl; l += nw) {
        const double* al = A + (size_t)(j + 1 + l) * ldv;
        double acc = 0.0;
        for (int r = max(lo, j + 1) + lane; r < hi; r += 32) acc = __fma_rn(aj[r], al[r], acc);
        acc = warp_sum(acc);
        if (lane == 0) loc[l] = acc + ((j >= lo && j < hi) ? al[j] : 0.0);
      }
      __syncthreads();
      t.template sum_vec<double>(loc, tot, nl);
      for (int l = 0; l < nl; ++l) {
        double* al = A + (size_t)(j + 1 + l) * ldv;
        const double wl = tj * tot[l];
        for (int r = max(lo, j + 1) + threadIdx.x; r < hi; r += blockDim.x) al[r] = __fma_rn(-wl, aj[r], al[r]);
        if (threadIdx.x == 0 && j >= lo && j < hi) al[j] -= wl;
      }
      __syncthreads();
    }
  }
  // R (owned by the CTA holding rows < c) -> broadcast
  if (lo == 0 && hi > 0) {
    for (int e = threadIdx.x; e < c * c; e += blockDim.x) {
      int i = e % c, jj = e / c;
      Rm[IX(i, jj, ldr)] = (i <= jj) ? A[(size_t)jj * ldv + i] : 0.0;
    }
  }
  // explicit Q
  for (int jj = 0; jj < c; ++jj)
    for (int r = lo + threadIdx.x; r < hi; r += blockDim.x) Q[(size_t)jj * ldv + r] = (r == jj) ? 1.0 : 0.0;
  __syncthreads();
  for (int j = c - 1; j >= 0; --j) {
    const double tj = taus[j];
    if (tj == 0.0) continue;
    const double* aj = A + (size_t)j * ldv;
    const int nl = c - j;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int l = wid; l < nl; l += nw) {
      const double* ql = Q + (size_t)(j + l) * ldv;
      double acc = 0.0;
      for (int r = max(lo, j + 1) + lane; r < hi; r += 32) acc = __fma_rn(aj[r], ql[r], acc);
      acc = warp_sum(acc);
      if (lane == 0) loc[l] = acc + ((j >= lo && j < hi) ? ql[j] : 0.0);
    }
    __syncthreads();
    t.template sum_vec<double>(loc, tot, nl);
    for (int l = 0; l < nl; ++l) {
      double* ql = Q + (size_t)(j + l) * ldv;
      const double wl = tj * tot[l];
      for (int r = max(lo, j + 1) + threadIdx.x; r < hi; r += blockDim.x) ql[r] = __fma_rn(-wl, aj[r], ql[r]);
      if (threadIdx.x == 0 && j >= lo && j < hi) ql[j] -= wl;
    }
    __syncthreads();
  }
  t.sync();
  // sign fix + rank test, identical in all CTAs
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    double fro = 0.0;
    for (int jj = 0; jj < c; ++jj)
      for (int i = 0; i <= jj; ++i) {
        double v = __ldcg(Rm + IX(i, jj, ldr));
        fro = __fma_rn(v, v, fro);
      }
    const double tol = (double)max(n, c) * kEps53 * sqrt(fro);
    int ok = 1;
    for (int i = 0; i < c; ++i) {
      double d = __ldcg(Rm + IX(i, i, ldr));
      loc[i] = d < 0.0 ? -1.0 : 1.0;
      if (fabs(d) < tol) ok = 0;
    }
    s_ok = ok;
  }
  __syncthreads();
  const int ok = s_ok;
  for (int jj = 0; jj < c; ++jj) {
    const double sg = loc[jj];
    if (sg < 0.0)
      for (int r = lo + threadIdx.x; r < hi; r += blockDim.x) Q[(size_t)jj * ldv + r] = -Q[(size_t)jj * ldv + r];
  }
  t.sync();
  if (t.leader()) {
    for (int e = threadIdx.x; e < c * c; e += blockDim.x) {
      int i = e % c, jj = e / c;
      Rm[IX(i, jj, ldr)] = (i <= jj) ? Rm[IX(i, jj, ldr)] * loc[i] : 0.0;
    }
  }
  t.sync();
  return ok != 0;
}

// --------------------------------------------------------------------------
// Gram W^T Vh (gr x gc) in the work format (gcrodr.py:187):
//   W = [C (keff), V (j+1)], Vh = [Ut (keff), V (j)].
// Per-CTA partials, then a rank-ordered distributed reduction; the final
// matrix (ld gr) is at gram_final(K, t).
// --------------------------------------------------------------------------
template <class TW, class TA, class TF, int MV, class Team>
GB_DEVICE double* gram_final(const Krylov<TW, TA, TF, MV>& K, const Team& t) {
  return K.gram + (size_t)t.size() * K.gram_stride;
}

template <class TW, class TA, class TF, int MV, class Team>
__device__ void team_gram(Team& t, Krylov<TW, TA, TF, MV>& K, int keff, int j, double* sm, void* smem_ops) {
  using Acc = typename Fmt<TW>::Acc;
  const int gr = keff + j + 1, gc = keff + j, ldv = K.ldv;
  int lo, hi;
  t.rows(K.n, lo, hi);
  double* part = Team::kGrid ? K.gram + (size_t)t.rank() * K.gram_stride : gram_final(K, t);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int total = gr * gc;
  const int nr = hi - lo;
  if ((size_t)nr * (gr + gc) * sizeof(TW) <= (size_t)K.ops_bytes) {
    // stage this CTA's rows of W = [C, V] and Vh = [Ut, V] in shared memory
    // (row-major, one coalesced pass), then every thread forms whole Gram
    // entries from shared memory: no per-entry warp reduction on the path
    TW* Ws = reinterpret_cast<TW*>(smem_ops);
    TW* Vs = Ws + (size_t)nr * gr;
    for (int c = wid; c < gr + gc; c += nw) {
      const bool isw = c < gr;
      const int cc = isw ? c : c - gr;
      const int kk = keff;
      const TW* col = isw ? (cc < kk ? K.C + (size_t)cc * ldv : K.V + (size_t)(cc - kk) * ldv)
                          : (cc < kk ? K.Ut + (size_t)cc * ldv : K.V + (size_t)(cc - kk) * ldv);
      TW* dst = isw ? Ws + cc : Vs + cc;
      const int ld = isw ? gr : gc;
      for (int r = lane; r < nr; r += 32) dst[(size_t)r * ld] = col[lo + r];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
      const int a = e % gr, b = e / gr;
      Acc acc = Acc(0);
      for (int r = 0; r < nr; ++r) acc = Fmt<TW>::mac(acc, Ws[(size_t)r * gr + a], Vs[(size_t)r * gc + b]);
      part[e] = (double)acc;
    }
    __syncthreads();
  } else
  for (int e = wid; e < total; e += nw) {
    const int a = e % gr, b = e / gr;
    const TW* wa = a < keff ? K.C + (size_t)a * ldv : K.V + (size_t)(a - keff) * ldv;
    const TW* vb = b < keff ? K.Ut + (size_t)b * ldv : K.V + (size_t)(b - keff) * ldv;
    Acc acc = Acc(0);
    for (int r = lo + lane; r < hi; r += 32) acc = Fmt<TW>::mac(acc, wa[r], vb[r]);
    acc = warp_sum(acc);
    if (lane == 0) part[e] = (double)acc;
  }
  if constexpr (Team::kGrid) {
    t.sync();
    double* fin = gram_final(K, t);
    const int G = t.size();
    const int chunk = (total + G - 1) / G;
    const int e0 = t.rank() * chunk, e1 = min(total, e0 + chunk);
    for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
      Acc acc = Acc(0);
      for (int g = 0; g < G; ++g) acc += (Acc)__ldcg(K.gram + (size_t)g * K.gram_stride + e);
      fin[e] = (double)acc;
    }
  }
  t.sync();
}

// --------------------------------------------------------------------------
// harmonic_ritz_recycle + QR(Ghat P) on the leader (gcrodr.py:171-197, 383-390).
// Ghat (gr x gc, ld gr) is at K.dense (kept from the LS).  Returns kn (> 0)
// with P, Q, R written to bc, or -1 (keep the previous space).
// --------------------------------------------------------------------------
template <class TW, class TA, class TF, int MV, class Team>
__device__ int leader_recycle(const Team& t, Krylov<TW, TA, TF, MV>& K, int keff, int j, const PhaseLog& lg) {
  const int S = bc_S(K), kk = K.k;
  const int gr = keff + j + 1, gc = keff + j;
  double* Gm = K.dense;
  double* base = K.dense + 2 * (size_t)S * S + 3 * (size_t)S;
  double* a1 = base;
  double* b1 = a1 + (size_t)S * S;
  double* b1c = b1 + (size_t)S * S;
  double* rd = b1c + (size_t)S * S;
  double* bd = rd + (size_t)S * S;
  int* piv = reinterpret_cast<int*>(bd + 2 * S);
  double* P = bd + 3 * (size_t)S;
  double* GP = P + (size_t)S * (kk + 2);
  double* Qs = GP + (size_t)S * (kk + 2);
  double* Rs = Qs + (size_t)S * (kk + 2);
  double* tau = Rs + (size_t)(kk + 2) * (kk + 2);
  double* scr = tau + S;
  const double* wtv = gram_final(K, t);
  __shared__ int s_flag;
  __shared__ double s_red[33];
  // a1 = G^T G, b1 = G^T (W^T Vh)
  for (int e = threadIdx.x; e < gc * gc; e += blockDim.x) {
    int a = e % gc, b = e / gc;
    double x = 0.0, y = 0.0;
    for (int l = 0; l < gr; ++l) {
      double g = Gm[IX(l, a, gr)];
      x = __fma_rn(g, Gm[IX(l, b, gr)], x);
      y = __fma_rn(g, __ldcg(wtv + IX(l, b, gr)), y);
    }
    a1[IX(a, b, gc)] = x;
    b1[IX(a, b, gc)] = y;
  }
  if (threadIdx.x == 0) s_flag = 0;
  __syncthreads();
  for (int e = threadIdx.x; e < gc * gc; e += blockDim.x) {
    if (!isfinite(a1[e])) atomicOr(&s_flag, 1);
    if (!isfinite(b1[e])) atomicOr(&s_flag, 2);
  }
  __syncthreads();
  if (s_flag) return -1;  // NoConvergence / SingularB propagate -> keep space
  // shared-memory staging when it fits (the factorisation, the eigen
  // iteration and the bidiagonalisation are latency bound: every scalar step
  // touches the matrix).  fast layout: [emat p^2 | lu p^2 | inv p^2 | ...]
  const bool fast = K.fast != nullptr && leader_fast_need(gc, kk) <= K.fast_cap;
  const size_t pp = (size_t)gc * gc;
  double* emat = fast ? K.fast : rd;        // b1^-1 a1 (eig input)
  double* lu = fast ? K.fast + pp : b1;     // LU factors of b1
  double* escr = fast ? K.fast + pp : scr;  // eig scratch (after the solves)
  for (int e = threadIdx.x; e < gc * gc; e += blockDim.x) {
    emat[e] = a1[e];
    if (fast) lu[e] = b1[e];
  }
  __syncthreads();
  mark(lg, 60);
  // SingularB screen (eig_generalized, densela.py:460-477: cond2(b1) > 2^53).
  // cond2 <= p * cond1, so an exactly computed ||b1||_1 ||b1^-1||_1 below
  // 2^53 / (4 p) proves the pencil regular without the SVD; otherwise (and
  // without the fast staging) the 2-norm condition number decides.
  bool need_cond2 = true;
  if (!fast) {
    // large pencils (cfg5: gc = 200) run the same screen in global memory: b1 is kept in
    // b1c, factored in place, inverted into the eig scratch; the bidiagonalisation-based
    // cond2 (18 ms at gc = 200, against ~5 ms for the inverse) only runs if the screen fails
    for (int e = threadIdx.x; e < gc * gc; e += blockDim.x) b1c[e] = b1[e];
    __syncthreads();
  }
  int zero = blk_getrf(lu, gc, gc, piv);  // lu == b1 without the fast staging
  bool screened = false;
  if (zero < 0) {
    double* inv = fast ? K.fast + 2 * pp : scr;
    const double* b1orig = fast ? b1 : b1c;
    for (int e = threadIdx.x; e < gc * gc; e += blockDim.x) inv[e] = (e % gc == e / gc) ? 1.0 : 0.0;
    __syncthreads();
    blk_getrs(lu, gc, gc, piv, inv, gc, gc);
    __shared__ double s_n1[2];
    if (threadIdx.x < 64) {
      const int lane = threadIdx.x & 31;
      // column sums: warp 0 over b1, warp 1 over the inverse
      const double* m = threadIdx.x < 32 ? b1orig : inv;
      double best = 0.0;
      for (int c = lane; c < gc; c += 32) {
        double cs = 0.0;
        for (int r0 = 0; r0 < gc; ++r0) cs += fabs(m[IX(r0, c, gc)]);
        best = nan_max(best, cs);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) best = nan_max(best, __shfl_xor_sync(0xffffffffu, best, o));
      if (lane == 0) s_n1[threadIdx.x >> 5] = best;
    }
    __syncthreads();
    const double c1 = s_n1[0] * s_n1[1];
    need_cond2 = !(c1 * 4.0 * gc < 1.0 / kEps53);
    screened = !need_cond2;
    __syncthreads();
  }
  if (!fast && !screened) {
    // the screen did not decide: restore b1 and take the cond2 path below unchanged
    for (int e = threadIdx.x; e < gc * gc; e += blockDim.x) b1[e] = b1c[e];
    __syncthreads();
    zero = -1;
  }
  if (need_cond2) {
    double* cmat = fast ? K.fast + 2 * pp : b1c;
    for (int e = threadIdx.x; e < gc * gc; e += blockDim.x) cmat[e] = b1[e];
    __syncthreads();
    double cnd = blk_cond2(cmat, gc, gc, bd, scr);
    if (!(cnd <= 1.0 / kEps53)) {
      // shift by sqrt(u) * ||b1||_F and retry once (gcrodr.py:192-196)
      double f = 0.0;
      for (int e = threadIdx.x; e < gc * gc; e += blockDim.x) f = __fma_rn(b1[e], b1[e], f);
      double ff[1] = {f};
      block_sum<double, 1>(ff, s_red);
      const double shift = sqrt(kEps53) * sqrt(ff[0]);
      for (int e = threadIdx.x; e < gc; e += blockDim.x) b1[IX(e, e, gc)] += shift;
      __syncthreads();
      for (int e = threadIdx.x; e < gc * gc; e += blockDim.x) cmat[e] = b1[e];
      __syncthreads();
      cnd = blk_cond2(cmat, gc, gc, bd, scr);
      if (!(cnd <= 1.0 / kEps53)) return -1;
      // refactor the shifted pencil
      for (int e = threadIdx.x; e < gc * gc; e += blockDim.x) lu[e] = b1[e];
      __syncthreads();
      zero = blk_getrf(lu, gc, gc, piv);
    } else if (!fast) {
      zero = blk_getrf(lu, gc, gc, piv);  // lu == b1 (cond2 worked on a copy)
    }
  }
  mark(lg, 61);
  // reduced = b1^-1 a1
  if (zero >= 0) return -1;
  mark(lg, 62);
  blk_getrs(lu, gc, gc, piv, emat, gc, gc);
  mark(lg, 63);
  double* hp = (!fast && K.pack != nullptr && hqr_pack_doubles(gc) * sizeof(double) <= (size_t)K.ops_bytes)
                   ? K.pack
                   : nullptr;
  const int kn = leader_ritz_basis(emat, gc, kk, P, gc, escr, hp);
  mark(lg, 64);
  if (kn <= 0) return -1;
  for (int e = threadIdx.x; e < gr * kn; e += blockDim.x) {
    int a = e % gr, b = e / gr;
    double acc = 0.0;
    for (int l = 0; l < gc; ++l) acc = __fma_rn(Gm[IX(a, l, gr)], P[IX(l, b, gc)], acc);
    GP[IX(a, b, gr)] = acc;
  }
  __syncthreads();
  if (!blk_qr_signed(GP, gr, gr, kn, Qs, gr, Rs, kk + 1, tau)) return -1;
  mark(lg, 65);
  double* bP = bc_P(K);
  double* bQ = bc_Q(K);
  double* bR = bc_R(K);
  for (int e = threadIdx.x; e < gc * kn; e += blockDim.x) bP[IX(e % gc, e / gc, S)] = P[IX(e % gc, e / gc, gc)];
  for (int e = threadIdx.x; e < gr * kn; e += blockDim.x) bQ[IX(e % gr, e / gr, S)] = Qs[IX(e % gr, e / gr, gr)];
  for (int e = threadIdx.x; e < kn * kn; e += blockDim.x) bR[IX(e % kn, e / kn, kk + 1)] = Rs[IX(e % kn, e / kn, kk + 1)];
  __syncthreads();
  return kn;
}

// --------------------------------------------------------------------------
// the inner solve: GMRES (recycling == 0) or GCRO-DR.  Input K.rhat (u-valued),
// output K.x.  Returns scalars identical in all CTAs.
// --------------------------------------------------------------------------
template <class TW, class TA, class TF, int MV, class Team>
__device__ StepScalars inner_solve(Team& t, Krylov<TW, TA, TF, MV>& K, TrsvSync& ts, double* sm,
                                   void* smem_ops) {
  using F = Fmt<TW>;
  const int n = K.n, ldv = K.ldv, M = K.m, kk = K.k;
  double* red = sm + 4 * M + 4;
  double* tmp = red + 64;
  StepScalars out{0, 0, 0, 0};
  int applies = 0;
  // s = U^-1 L^-1 rhat[perm] at u^2, stored in u
  t.sync();
  mark(ts.log, 36);
  op_apply<MV>(t, K.sys, (const TW*)nullptr, K.rhat, K.s, K.ybuf, ts, smem_ops);
  mark(ts.log, 37);
  const double snorm = team_nrm2<TW>(t, K.s, n, red);
  team_zero(t, K.x, n);
  mark(ts.log, 38);
  int keff = K.recycling ? *K.keff_io : 0;
  if (snorm == 0.0) {
    out.status = KS_CONVERGED;
    out.keff = keff;
    t.sync();
    return out;
  }
  const double tol = K.tau * snorm;
  team_copy(t, K.s, K.res, n);
  int cycles = 0;
  bool have_space = false, breakdown = false;
  int lo, hi;
  t.rows(n, lo, hi);

  // ---- warm start from an incoming recycle space (gcrodr.py:268-285) ----
  if (K.recycling && keff > 0) {
    for (int i = 0; i < keff; ++i) {
      apply_A(t, K, ts, colp(K.U, ldv, i), K.w, smem_ops, applies);
      for (int r = lo + threadIdx.x; r < hi; r += blockDim.x) K.Wd[(size_t)i * ldv + r] = (double)K.w[r];
    }
    t.sync();
    // distributed Householder QR of Wd (n x keff)
    bool ok = team_qr_tall(t, K, keff, sm);
    if (ok) {
      // C = fl(Q); U = fl(Yk R^-1) in place (Yk = U)
      const double* Rm = bc_Rw(K);
      for (int r = lo + threadIdx.x; r < hi; r += blockDim.x) {
        double yt[33];
        for (int c = 0; c < keff; ++c) yt[c] = (double)K.U[(size_t)c * ldv + r];
        for (int c = 0; c < keff; ++c) {
          double s = yt[c];
          for (int i = 0; i < c; ++i) s = __fma_rn(-yt[i], __ldcg(Rm + IX(i, c, kk + 1)), s);
          yt[c] = s / __ldcg(Rm + IX(c, c, kk + 1));
          K.U[(size_t)c * ldv + r] = (TW)F::rnd(yt[c]);
          K.C[(size_t)c * ldv + r] = (TW)F::rnd(K.Qd[(size_t)c * ldv + r]);
        }
      }
      t.sync();
      team_tvec2<TW>(t, K.C, keff, (const TW*)nullptr, 0, ldv, K.res, n, tmp, red);
      for (int r = lo + threadIdx.x; r < hi; r += blockDim.x) {
        TW xr = K.x[r], rr = K.res[r];
        for (int i = 0; i < keff; ++i) {
          xr = F::axpy(tmp[i], K.U[(size_t)i * ldv + r], xr);
          rr = F::axpy(-tmp[i], K.C[(size_t)i * ldv + r], rr);
        }
        K.x[r] = xr;
        K.res[r] = rr;
      }
      have_space = true;
    } else {
      keff = 0;
    }
  } else {
    keff = 0;
  }

  bool converged = false;
  bool first = true;
  while (true) {
    const double beta = team_nrm2<TW>(t, K.res, n, red);
    if (!first || !K.recycling || have_space) {
      if (beta <= tol) {
        converged = true;
        break;
      }
      if (cycles >= K.max_cycles) break;
    }
    if (!K.recycling || !have_space) {
      // ---- plain GMRES(m) cycle (+ harvest for GCRO-DR) ----
      mark(ts.log, 40);
      CycleOut co = arnoldi_cycle(t, K, ts, K.res, beta, M, tol, 0, true, sm, smem_ops, applies);
      mark(ts.log, 41);
      const int j = co.steps;
      if (threadIdx.x == 0 && t.leader() && cycles <= K.max_cycles) {
        K.cycle_iters[cycles] = j;
        K.cycle_keff[cycles] = 0;
      }
      cycles++;
      breakdown = breakdown || co.breakdown;
      update_x(t, K.x, K.V, ldv, K.bc, j, n);
      if (co.converged || !K.explicit_res)
        recurrence_res(t, K, j, beta);
      else
        explicit_residual(t, K, ts, smem_ops, applies);
      if (!K.recycling) {
        if (co.converged) {
          converged = true;
          break;
        }
        first = false;
        continue;
      }
      first = false;
      if (j >= kk) {
        // harmonic_ritz_first on the leader (gcrodr.py:140-168, 305-315)
        if (t.leader()) {
          double* D = K.dense;
          const int ldd = M + kk + 2;
          double* Hm = D;                       // j x j
          double* HT = Hm + (size_t)ldd * ldd;  // j x j
          double* wv = HT + (size_t)ldd * ldd;  // j
          int* piv = reinterpret_cast<int*>(wv + ldd);
          double* P = wv + 2 * ldd;                 // j x (k+1)
          double* HP = P + (size_t)ldd * (kk + 2);  // (j+1) x keff
          double* Qs = HP + (size_t)ldd * (kk + 2);
          double* Rs = Qs + (size_t)ldd * (kk + 2);
          double* tau = Rs + (size_t)(kk + 2) * (kk + 2);
          double* scr = tau + ldd;
          for (int e = threadIdx.x; e < j * j; e += blockDim.x) {
            int a = e % j, b = e / j;
            Hm[IX(a, b, j)] = K.H[IX(a, b, M + 1)];
            HT[IX(a, b, j)] = K.H[IX(b, a, M + 1)];
          }
          for (int e = threadIdx.x; e < j; e += blockDim.x) wv[e] = (e == j - 1) ? 1.0 : 0.0;
          __syncthreads();
          const double hsub = K.H[IX(j, j - 1, M + 1)];
          if (hsub != 0.0) {
            int z = blk_getrf(HT, j, j, piv);
            if (z < 0) {
              blk_getrs(HT, j, j, piv, wv, j, 1);
              __shared__ int s_fin;
              if (threadIdx.x == 0) {
                s_fin = 1;
                for (int e = 0; e < j; ++e)
                  if (!isfinite(wv[e])) s_fin = 0;
              }
              __syncthreads();
              if (s_fin)
                for (int e = threadIdx.x; e < j; e += blockDim.x)
                  Hm[IX(e, j - 1, j)] += (hsub * hsub) * wv[e];
              __syncthreads();
            }
          }
          int kn;
          if (K.fast != nullptr && leader_fast_need(j, kk) <= K.fast_cap) {
            for (int e = threadIdx.x; e < j * j; e += blockDim.x) K.fast[e] = Hm[e];
            __syncthreads();
            kn = leader_ritz_basis(K.fast, j, kk, P, j, K.fast + (size_t)j * j);
          } else {
            double* hp = (K.pack != nullptr && hqr_pack_doubles(j) * sizeof(double) <= (size_t)K.ops_bytes)
                             ? K.pack
                             : nullptr;
            kn = leader_ritz_basis(Hm, j, kk, P, j, scr, hp);
          }
          int status = -1;
          if (kn > 0) {
            // Hbar P  ((j+1) x kn)
            for (int e = threadIdx.x; e < (j + 1) * kn; e += blockDim.x) {
              int a = e % (j + 1), b = e / (j + 1);
              double acc = 0.0;
              for (int l = 0; l < j; ++l) acc = __fma_rn(K.H[IX(a, l, M + 1)], P[IX(l, b, j)], acc);
              HP[IX(a, b, j + 1)] = acc;
            }
            __syncthreads();
            bool ok = blk_qr_signed(HP, j + 1, j + 1, kn, Qs, j + 1, Rs, kk + 1, tau);
            if (ok) status = kn;
          }
          // broadcast P (j x kn), Q ((j+1) x kn), R (kn x kn)
          double* bP = K.bc + 3 * (M + kk + 2);
          double* bQ = bP + (size_t)(M + kk + 2) * (kk + 2);
          double* bR = bQ + (size_t)(M + kk + 2) * (kk + 2);
          if (status > 0) {
            for (int e = threadIdx.x; e < j * kn; e += blockDim.x) bP[IX(e % j, e / j, M + kk + 2)] = P[IX(e % j, e / j, j)];
            for (int e = threadIdx.x; e < (j + 1) * kn; e += blockDim.x)
              bQ[IX(e % (j + 1), e / (j + 1), M + kk + 2)] = Qs[IX(e % (j + 1), e / (j + 1), j + 1)];
            for (int e = threadIdx.x; e < kn * kn; e += blockDim.x)
              bR[IX(e % kn, e / kn, kk + 1)] = Rs[IX(e % kn, e / kn, kk + 1)];
          }
          if (threadIdx.x == 0) K.bc[M + kk + 1] = (double)status;
          __syncthreads();
        }
        t.sync();
        const int status = (int)__ldcg(K.bc + M + kk + 1);
        if (status > 0) {
          double* bP = K.bc + 3 * (M + kk + 2);
          double* bQ = bP + (size_t)(M + kk + 2) * (kk + 2);
          double* bR = bQ + (size_t)(M + kk + 2) * (kk + 2);
          rebuild_space(t, K, (const TW*)nullptr, K.V, (const TW*)nullptr, K.V, 0, j, status, bP, M + kk + 2,
                        bQ, M + kk + 2, bR, kk + 1);
          swap_space(K);
          keff = status;
          have_space = true;
        } else {
          have_space = false;
          keff = 0;
        }
        if (threadIdx.x == 0 && t.leader()) K.cycle_keff[cycles - 1] = keff;
      }
      continue;
    }
    // ---- deflated cycle (gcrodr.py:342-390) ----
    const int budget = M - keff;
    mark(ts.log, 50);
    CycleOut co = arnoldi_cycle(t, K, ts, K.res, beta, budget, tol, keff, false, sm, smem_ops, applies);
    mark(ts.log, 51);
    const int j = co.steps;
    if (threadIdx.x == 0 && t.leader() && cycles <= K.max_cycles) K.cycle_iters[cycles] = j;
    cycles++;
    breakdown = breakdown || co.breakdown;
    // D = diag(1 / ||U_i||) rounded to u; Ut = fl(U_i * d_i)
    team_colnorms<TW>(t, K.U, keff, ldv, n, tmp, red);
    double dk[33];
    for (int i = 0; i < keff; ++i) {
      double d = tmp[i] == 0.0 ? 1.0 : tmp[i];
      dk[i] = F::rnd(1.0 / d);
    }
    for (int r = lo + threadIdx.x; r < hi; r += blockDim.x)
      for (int i = 0; i < keff; ++i)
        K.Ut[(size_t)i * ldv + r] = (TW)F::rnd((double)K.U[(size_t)i * ldv + r] * dk[i]);
    const int gr = keff + j + 1, gc = keff + j;
    // rhs = W^T res, W = [C, V(:, :j+1)]
    team_tvec2<TW>(t, K.C, keff, K.V, j + 1, ldv, K.res, n, tmp, red);
    // least squares on the leader; y and gy broadcast
    double* by = K.bc;                 // y  (gc)
    double* bgy = K.bc + (M + kk + 2);  // gy (gr)
    if (t.leader()) {
      double* D = K.dense;
      const int ldg = gr;
      double* Gm = D;                               // gr x gc
      double* G2 = Gm + (size_t)(M + kk + 2) * (M + kk + 2);
      double* tau = G2 + (size_t)(M + kk + 2) * (M + kk + 2);
      double* tv = tau + (M + kk + 2);
      double* yv = tv + (M + kk + 2);
      for (int e = threadIdx.x; e < gr * gc; e += blockDim.x) {
        int a = e % gr, b = e / gr;
        double v = 0.0;
        if (a < keff && b < keff) v = (a == b) ? dk[a] : 0.0;
        else if (a < keff) v = K.B[IX(a, b - keff, kk + 1)];
        else if (b >= keff) v = K.H[IX(a - keff, b - keff, M + 1)];
        Gm[IX(a, b, ldg)] = v;
        G2[IX(a, b, ldg)] = v;
      }
      __syncthreads();
      blk_lstsq(G2, ldg, gr, gc, tmp, yv, tau, tv);
      for (int e = threadIdx.x; e < gc; e += blockDim.x) by[e] = F::rnd(yv[e]);
      __syncthreads();
      for (int e = threadIdx.x; e < gr; e += blockDim.x) {
        double acc = 0.0;
        for (int l = 0; l < gc; ++l) acc = __fma_rn(Gm[IX(e, l, ldg)], by[l], acc);
        bgy[e] = F::rnd(acc);
      }
      __syncthreads();
    }
    t.sync();
    // x += Vh y ; res -= W gy   (Vh = [Ut, V(:, :j)])
    for (int r = lo + threadIdx.x; r < hi; r += blockDim.x) {
      TW xr = K.x[r];
      for (int i = 0; i < gc; ++i) {
        const TW* col = i < keff ? K.Ut + (size_t)i * ldv : K.V + (size_t)(i - keff) * ldv;
        xr = F::axpy(__ldcg(by + i), col[r], xr);
      }
      K.x[r] = xr;
      TW rr = K.res[r];
      for (int i = 0; i < gr; ++i) {
        const TW* col = i < keff ? K.C + (size_t)i * ldv : K.V + (size_t)(i - keff) * ldv;
        rr = F::axpy(-__ldcg(bgy + i), col[r], rr);
      }
      K.res[r] = rr;
    }
    if (K.explicit_res && !co.converged) explicit_residual(t, K, ts, smem_ops, applies);
    mark(ts.log, 52);
    if (j >= 1) {
      // W^T Vh (gr x gc) in the work format: per-CTA partial Grams
      team_gram(t, K, keff, j, sm, smem_ops);
      mark(ts.log, 53);
      if (t.leader()) {
        int kn = leader_recycle(t, K, keff, j, ts.log);
        if (threadIdx.x == 0) K.bc[M + kk + 1] = (double)kn;
        __syncthreads();
      }
      t.sync();
      const int kn = (int)__ldcg(K.bc + M + kk + 1);
      if (kn > 0) {
        double* bP = K.bc + 3 * (M + kk + 2);
        double* bQ = bP + (size_t)(M + kk + 2) * (kk + 2);
        double* bR = bQ + (size_t)(M + kk + 2) * (kk + 2);
        rebuild_space(t, K, K.Ut, K.V, K.C, K.V, keff, j, kn, bP, M + kk + 2, bQ, M + kk + 2, bR, kk + 1);
        swap_space(K);
        keff = kn;
      }
    }
    if (threadIdx.x == 0 && t.leader() && cycles - 1 <= K.max_cycles) K.cycle_keff[cycles - 1] = keff;
    mark(ts.log, 55);
    first = false;
  }
  t.sync();
  if (t.leader() && threadIdx.x == 0 && K.recycling) *K.keff_io = have_space ? keff : 0;
  out.ncycles = cycles;
  out.status = (converged ? KS_CONVERGED : KS_STAGNATED) | (breakdown ? KS_BREAKDOWN : 0);
  out.applies = applies;
  out.keff = have_space ? keff : 0;
  return out;
}

}  // namespace gb
