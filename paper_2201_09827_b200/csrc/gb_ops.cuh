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
#include "gb_opseg.cuh"

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
  GB_DEVICE static T mul_rcp(T y, double rh, double) { return __dmul_rn(y, rh); }
  GB_DEVICE static T mac_t(T s, double l, T y) { return __fma_rn(l, y, s); }
  GB_DEVICE static T mac_inv(T s, double ih, double, T t) { return __fma_rn(ih, t, s); }
  static constexpr bool kInv = true;
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
  GB_DEVICE static T mul_rcp(T y, double rh, double) { return __fmul_rn(y, (float)rh); }
  GB_DEVICE static T mac_t(T s, double l, T y) { return __fmaf_rn((float)l, y, s); }
  GB_DEVICE static T mac_inv(T s, double ih, double, T t) { return s; }
  static constexpr bool kInv = false;
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
  GB_DEVICE static T mul_rcp(T y, double, double) { return y; }  // never used (exact order)
  GB_DEVICE static T mac_t(T s, double, T) { return s; }           // never used (exact order)
  GB_DEVICE static T mac_inv(T s, double, double, T) { return s; }
  static constexpr bool kInv = false;
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
  GB_DEVICE static T mul_rcp(T y, double rh, double rl) { return dd_mul(y, dd{rh, rl}); }
  GB_DEVICE static T mac_t(T s, double l, T y) { return dd_add(s, dd_scale(l, y)); }
  GB_DEVICE static T mac_inv(T s, double ih, double il, T t) { return dd_add(s, dd_mul(dd{ih, il}, t)); }
  static constexpr bool kInv = true;
  GB_DEVICE static double val(T x) { return dd_val(x); }
  GB_DEVICE static T shfl(T x, int src) {
    return dd{__shfl_sync(0xffffffffu, x.hi, src), __shfl_sync(0xffffffffu, x.lo, src)};
  }
  GB_DEVICE static T ld(const T* p) {
    double2 v = __ldcg(reinterpret_cast<const double2*>(p));
    return dd{v.x, v.y};
  }
};

template <class T>
GB_DEVICE T sel(bool c, T a, T b) { return c ? a : b; }
template <>
GB_DEVICE dd sel<dd>(bool c, dd a, dd b) { return dd{c ? a.hi : b.hi, c ? a.lo : b.lo}; }

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
  // reciprocals of diag(U) (dd-exact hi/lo), used by the non-exact modes to
  // keep divisions off the substitution's critical path; nullptr -> divide
  const double* rcp_hi;
  const double* rcp_lo;
  // dd-accurate inverses of the 32x32 diagonal blocks of L (strictly lower
  // part, unit diagonal implied) and U; element (i, j) of block b at
  // b*kInvStride + j*32 + i, followed by the folded off-diagonal block
  // (diag_fold_block).  nullptr -> sequential substitution.
  const double* linv_hi;
  const double* linv_lo;
  const double* uinv_hi;
  const double* uinv_lo;
  // grid teams, fp64 operator (gb_opseg.cuh): inverses of the nbig x nbig
  // diagonal blocks of L and U (row-major fp64 per block), the GEMV's bulk-copy
  // stages and whether every entry of A is a normal number (integer-pipe
  // conversion); bigl == nullptr -> the CTA-per-block substitution
  const double* bigl = nullptr;
  const double* bigu = nullptr;
  int nbig = 0;
  int gemv_ns = 0;
  int a_normal = 0;
  int sweep_la = 0;  // look-ahead form of the big-block sweeps (seg::sweep_la)
};

// progress counters of the flag-based TRSV (one per direction)
struct TrsvSync {
  unsigned long long* fwd;
  unsigned long long* bwd;
  unsigned long long epoch;  // call index; identical in all CTAs
  PhaseLog log;              // optional phase timers
  unsigned long long* stamps = nullptr;  // diagnostics: per block (deps seen, published)
  uint4* ytag = nullptr;  // tagged copy of y for trsv_cta (2 x 16 B per entry)
  int dsm = 0;            // > 0: ytag is this CTA's shared-memory copy in a cluster of dsm CTAs
};

GB_DEVICE unsigned long long ld_acquire64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
GB_DEVICE unsigned long long ld_relaxed64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
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
    while ((v = ld_relaxed64(ctr)) < target) __nanosleep(16);
    fence_acq_rel();
    *cache = v;
  }
}

// ---------------------------------------------------------------------------
// triangular solves: warp-owned 32-row blocks, wavefront over the whole team.
//   Row block b (32 rows) belongs to warp b mod W of the team (W = CTAs x
//   warps), processed in the sweep order; each lane owns one row and walks the
//   columns of its row in the reference's column-sweep order (lower: 0..i-1,
//   upper: n-1..i+1 then the division), so the exact modes (H16) reproduce the
//   reference bit for bit.  A block is published with one monotone progress
//   counter per direction (st.release; consumers poll relaxed + one fence);
//   the next tile's loads are issued before the wait (software pipelining).
//   y: in = right-hand side (accumulator type), out = solution.
// ---------------------------------------------------------------------------
template <class TT, class TF>
GB_DEVICE void tile_regs(TT (&v)[32], const TF* __restrict__ LU, size_t ldf, int n, int r0, int c0) {
  const int gc = c0 + (threadIdx.x & 31);
#pragma unroll
  for (int rr = 0; rr < 32; ++rr) {
    const int gr = r0 + rr;
    v[rr] = (gr < n && gc < n) ? (TT)to_d(LU[(size_t)gr * ldf + gc]) : TT(0);
  }
}
template <class TT>
GB_DEVICE void tile_store(TT* tile, const TT (&v)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int rr = 0; rr < 32; ++rr) tile[rr * 33 + lane] = v[rr];
}

// intra-CTA progress (CtaTeam): shared-memory counter
struct CtaProgress {
  volatile unsigned long long v;
};


template <class Team>
GB_DEVICE void wait_ctr(unsigned long long* gctr, volatile unsigned long long* sctr, unsigned long long target,
                        unsigned long long& cache) {
  if (cache >= target) return;
  unsigned long long v;
  if constexpr (Team::kGrid) {
#ifndef GB_SPIN_NS
#define GB_SPIN_NS 8
#endif
    while ((v = ld_relaxed64(gctr)) < target) {
      if (GB_SPIN_NS > 0) __nanosleep(GB_SPIN_NS);
    }
    fence_acq_rel();
  } else {
    while ((v = *sctr) < target) {
    }
    __threadfence_block();
  }
  cache = v;
}

template <int M, class Team, class TF, bool kLower>
__device__ void trsv_blocks(Team& t, int n, const TF* LU, size_t ldf, typename Arith<M>::T* y,
                            const TrsvSync& ts, void* smem_raw, const double* rcph = nullptr,
                            const double* rcpl = nullptr, const double* inv_h = nullptr,
                            const double* inv_l = nullptr) {
  using Ar = Arith<M>;
  using T = typename Ar::T;
  using TT = typename TileT<TF>::T;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const int nb = (n + 31) / 32;
  TT* tile = reinterpret_cast<TT*>(smem_raw) + wid * 32 * 33;
  unsigned long long* gctr = kLower ? ts.fwd : ts.bwd;
  __shared__ CtaProgress sprog[2];
  volatile unsigned long long* sctr = &sprog[kLower ? 0 : 1].v;
  const unsigned long long base = Team::kGrid ? ts.epoch * (unsigned long long)nb : 0ull;
  if constexpr (!Team::kGrid) {
    if (threadIdx.x == 0) *sctr = 0ull;
  }
  __syncthreads();
  unsigned long long cache = 0;
  if (!kLower && Team::kGrid) {
    // the backward sweep starts from the bottom of the forward result
    if (lane == 0) wait_ctr<Team>(ts.fwd, nullptr, base + (unsigned long long)nb, cache);
    cache = 0;
    __syncwarp();
  }
  const int W = t.size() * nw;
  const int gw = t.rank() * nw + wid;
  for (int s = gw; s < nb; s += W) {
    const int b = kLower ? s : nb - 1 - s;
    const int row0 = b * 32;
    const int row = row0 + lane;
    const bool rv = row < n;
    T acc = rv ? Ar::ld(y + row) : Ar::zero();
    const int noff = kLower ? b : nb - 1 - b;
    TT v[32];
    // first off-diagonal tile (or the diagonal tile) prefetched into registers;
    // each iteration stores the current tile and prefetches the next one
    tile_regs(v, LU, ldf, n, row0, noff > 0 ? (kLower ? 0 : nb - 1) * 32 : row0);
    for (int q = 0; q < noff; ++q) {
      const int cb = kLower ? q : nb - 1 - q;
      const int c0 = cb * 32;
      __syncwarp();
      tile_store(tile, v);
      tile_regs(v, LU, ldf, n, row0, q + 1 < noff ? (kLower ? q + 1 : nb - 2 - q) * 32 : row0);
      // every lane polls: a single spinning lane costs ~9 us of warp
      // reconvergence per wait on sm_100a (measured, tools/micro/trsv.cu)
      wait_ctr<Team>(gctr, sctr, base + (unsigned long long)(q + 1), cache);
      if (ts.stamps != nullptr && lane == 0 && q + 1 == noff) ts.stamps[3 * s + 2] = gtimer();
      __syncwarp();
      const T yv = (c0 + lane < n) ? Ar::ld(y + c0 + lane) : Ar::zero();
      if constexpr (!Ar::kExactOrder) {
        // four independent partial sums (entries beyond n are zero)
        T s0 = Ar::zero(), s1 = Ar::zero(), s2 = Ar::zero(), s3 = Ar::zero();
#pragma unroll
        for (int jj = 0; jj < 32; jj += 4) {
          s0 = Ar::mac_t(s0, (double)tile[lane * 33 + jj], Ar::shfl(yv, jj));
          s1 = Ar::mac_t(s1, (double)tile[lane * 33 + jj + 1], Ar::shfl(yv, jj + 1));
          s2 = Ar::mac_t(s2, (double)tile[lane * 33 + jj + 2], Ar::shfl(yv, jj + 2));
          s3 = Ar::mac_t(s3, (double)tile[lane * 33 + jj + 3], Ar::shfl(yv, jj + 3));
        }
        acc = Ar::sub(acc, Ar::add(Ar::add(s0, s1), Ar::add(s2, s3)));
      } else if (kLower) {
        // exact column-sweep order, branch-free: divergence inside these
        // loops costs a warp reconvergence per step on sm_100a
#pragma unroll 8
        for (int jj = 0; jj < 32; ++jj) {
          const T yj = Ar::shfl(yv, jj);
          acc = sel(c0 + jj < n, Ar::sub_prod(acc, (double)tile[lane * 33 + jj], yj), acc);
        }
      } else {
#pragma unroll 8
        for (int jj = 31; jj >= 0; --jj) {
          const T yj = Ar::shfl(yv, jj);
          acc = sel(c0 + jj < n, Ar::sub_prod(acc, (double)tile[lane * 33 + jj], yj), acc);
        }
      }
    }
    if (ts.stamps != nullptr && lane == 0) ts.stamps[3 * s] = gtimer();
    if constexpr (Ar::kInv) {
      if (inv_h != nullptr) {
        // y_b = inv(D_b) t_b as a 32-term dot per lane (no sequential chain);
        // lower: unit diagonal implied (strictly lower part stored)
        const double* ih = inv_h + (size_t)b * kInvStride + lane;
        const double* il = inv_l != nullptr ? inv_l + (size_t)b * kInvStride + lane : nullptr;
        T s0 = kLower ? acc : Ar::zero(), s1 = Ar::zero(), s2 = Ar::zero(), s3 = Ar::zero();
#pragma unroll
        for (int jj = 0; jj < 32; jj += 4) {
          const T t0 = Ar::shfl(acc, jj), t1 = Ar::shfl(acc, jj + 1), t2 = Ar::shfl(acc, jj + 2),
                  t3 = Ar::shfl(acc, jj + 3);
          s0 = Ar::mac_inv(s0, __ldg(ih + (jj)*32), il ? __ldg(il + (jj)*32) : 0.0, t0);
          s1 = Ar::mac_inv(s1, __ldg(ih + (jj + 1) * 32), il ? __ldg(il + (jj + 1) * 32) : 0.0, t1);
          s2 = Ar::mac_inv(s2, __ldg(ih + (jj + 2) * 32), il ? __ldg(il + (jj + 2) * 32) : 0.0, t2);
          s3 = Ar::mac_inv(s3, __ldg(ih + (jj + 3) * 32), il ? __ldg(il + (jj + 3) * 32) : 0.0, t3);
        }
        acc = Ar::add(Ar::add(s0, s1), Ar::add(s2, s3));
        if (rv) y[row] = acc;
        goto published;
      }
    }
    // diagonal block (its tile is already in v)
    __syncwarp();
    tile_store(tile, v);
    __syncwarp();
    if (kLower) {
      for (int jj = 0; jj < 32; ++jj) {
        const T yj = Ar::shfl(acc, jj);
        acc = sel(lane > jj, Ar::sub_prod(acc, (double)tile[lane * 33 + jj], yj), acc);
      }
    } else {
      const bool use_rcp = !Ar::kExactOrder && rcph != nullptr;
      double rh = 0.0, rl = 0.0;
      if (use_rcp && rv) {
        rh = __ldg(rcph + row);
        rl = rcpl != nullptr ? __ldg(rcpl + row) : 0.0;
      }
      const double dg = (double)tile[lane * 33 + lane];
      for (int jj = 31; jj >= 0; --jj) {
        const T dv = use_rcp ? Ar::mul_rcp(acc, rh, rl) : Ar::div(acc, dg);
        acc = sel(lane == jj && rv, dv, acc);
        const T yj = Ar::shfl(acc, jj);
        acc = sel(lane < jj && row0 + jj < n, Ar::sub_prod(acc, (double)tile[lane * 33 + jj], yj), acc);
      }
    }
    if (rv) y[row] = acc;
  published:
    if (ts.stamps != nullptr && lane == 0) ts.stamps[3 * s + 1] = gtimer();
    __syncwarp();
    if (lane == 0) {
      if constexpr (Team::kGrid) {
        __threadfence();
        st_release64(gctr, base + (unsigned long long)(s + 1));
      } else {
        __threadfence();  // y goes through L2: consumers read it with ld.cg
        *sctr = (unsigned long long)(s + 1);
      }
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// super-block triangular solve for the non-exact modes (F64 / DD): a CTA owns
// 256 rows (warp w: rows 32w..32w+31).  Off-diagonal super-blocks are consumed
// as the grid-wide progress counter publishes them (8 tiles per warp, ILP
// sums); the diagonal super-block is an in-CTA warp chain through shared
// memory (diagonal 32x32 blocks applied through their dd inverses).  One
// global hand-off per 256 rows instead of per 32 rows.
// ---------------------------------------------------------------------------
template <int M, class Team, class TF, bool kLower>
__device__ void trsv_super(Team& t, int n, const TF* LU, size_t ldf, typename Arith<M>::T* y, const TrsvSync& ts,
                           void* smem_raw, const double* inv_h, const double* inv_l) {
  using Ar = Arith<M>;
  using T = typename Ar::T;
  using TT = typename TileT<TF>::T;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const int SB = nw * 32;
  const int nsb = (n + SB - 1) / SB;
  TT* tile = reinterpret_cast<TT*>(smem_raw) + wid * 32 * 33;
  T* ysb = reinterpret_cast<T*>(reinterpret_cast<TT*>(smem_raw) + nw * 32 * 33);  // SB entries
  __shared__ volatile int s_cnt;  // sub-blocks of the current super-block finalised
  unsigned long long* gctr = kLower ? ts.fwd : ts.bwd;
  // same epoch base as trsv_blocks (32-row units) so the counters stay
  // monotone when the two solvers alternate on one TrsvSync
  const unsigned long long base = ts.epoch * (unsigned long long)((n + 31) / 32);
  unsigned long long cache = 0;
  if (!kLower && Team::kGrid) {
    // the backward sweep starts from the bottom of the completed forward result
    wait_ctr<Team>(ts.fwd, nullptr, base + (unsigned long long)nsb, cache);
    cache = 0;
  }
  const int G = t.size(), r = t.rank();
  for (int s = r; s < nsb; s += G) {
    const int b = kLower ? s : nsb - 1 - s;
    const int row0 = b * SB + wid * 32;
    const int row = row0 + lane;
    const bool rv = row < n;
    T acc = rv ? Ar::ld(y + row) : Ar::zero();
    if (threadIdx.x == 0) s_cnt = 0;
    // off-diagonal super-blocks in sweep order, nw tiles each
    const int noff = kLower ? b : nsb - 1 - b;
    const int ntiles = noff * nw;
    TT v[32];
    auto tile_col = [&](int q) {
      const int sbi = q / nw, tt = q % nw;
      const int cb = kLower ? sbi : nsb - 1 - sbi;
      return cb * SB + (kLower ? tt : nw - 1 - tt) * 32;
    };
    if (ntiles > 0 && row0 < n) tile_regs(v, LU, ldf, n, row0, tile_col(0));
    for (int q = 0; q < ntiles; ++q) {
      const int c0 = tile_col(q);
      __syncwarp();
      if (row0 < n) tile_store(tile, v);
      if (q + 1 < ntiles && row0 < n) tile_regs(v, LU, ldf, n, row0, tile_col(q + 1));
      if (q % nw == 0) wait_ctr<Team>(gctr, nullptr, base + (unsigned long long)(q / nw + 1), cache);
      __syncwarp();
      if (row0 >= n || c0 >= n) continue;
      const T yv = (c0 + lane < n) ? Ar::ld(y + c0 + lane) : Ar::zero();
      T s0 = Ar::zero(), s1 = Ar::zero(), s2 = Ar::zero(), s3 = Ar::zero();
#pragma unroll
      for (int jj = 0; jj < 32; jj += 4) {
        s0 = Ar::mac_t(s0, (double)tile[lane * 33 + jj], Ar::shfl(yv, jj));
        s1 = Ar::mac_t(s1, (double)tile[lane * 33 + jj + 1], Ar::shfl(yv, jj + 1));
        s2 = Ar::mac_t(s2, (double)tile[lane * 33 + jj + 2], Ar::shfl(yv, jj + 2));
        s3 = Ar::mac_t(s3, (double)tile[lane * 33 + jj + 3], Ar::shfl(yv, jj + 3));
      }
      acc = Ar::sub(acc, Ar::add(Ar::add(s0, s1), Ar::add(s2, s3)));
    }
    __syncthreads();
    // diagonal super-block: in-CTA chain over the sub-blocks
    const int nvalid = min(nw, (n - b * SB + 31) / 32);  // sub-blocks with rows < n
    for (int st = 0; st < nvalid; ++st) {
      const int w = kLower ? st : nvalid - 1 - st;  // sub-block finalised at this step
      const int d0 = b * SB + w * 32;
      if (row0 >= n) continue;
      if (wid == w) {
        // y_w = inv(D_w) t_w  (lower: unit diagonal implied)
        const double* ih = inv_h + (size_t)(b * nw + w) * kInvStride + lane;
        const double* il = inv_l != nullptr ? inv_l + (size_t)(b * nw + w) * kInvStride + lane : nullptr;
        T q0 = kLower ? acc : Ar::zero(), q1 = Ar::zero(), q2 = Ar::zero(), q3 = Ar::zero();
#pragma unroll
        for (int jj = 0; jj < 32; jj += 4) {
          q0 = Ar::mac_inv(q0, __ldg(ih + jj * 32), il ? __ldg(il + jj * 32) : 0.0, Ar::shfl(acc, jj));
          q1 = Ar::mac_inv(q1, __ldg(ih + (jj + 1) * 32), il ? __ldg(il + (jj + 1) * 32) : 0.0,
                           Ar::shfl(acc, jj + 1));
          q2 = Ar::mac_inv(q2, __ldg(ih + (jj + 2) * 32), il ? __ldg(il + (jj + 2) * 32) : 0.0,
                           Ar::shfl(acc, jj + 2));
          q3 = Ar::mac_inv(q3, __ldg(ih + (jj + 3) * 32), il ? __ldg(il + (jj + 3) * 32) : 0.0,
                           Ar::shfl(acc, jj + 3));
        }
        acc = Ar::add(Ar::add(q0, q1), Ar::add(q2, q3));
        ysb[w * 32 + lane] = acc;
        if (rv) y[row] = acc;
        __syncwarp();
        __threadfence_block();
        if (lane == 0) s_cnt = st + 1;
      } else if (kLower ? (wid > w) : (wid < w)) {
        // tile (wid, w) is independent of y_w: load it before waiting
        tile_regs(v, LU, ldf, n, row0, d0);
        tile_store(tile, v);
        while (s_cnt < st + 1) {
        }
        __threadfence_block();
        __syncwarp();
        const T yv = ysb[w * 32 + lane];
        T s0 = Ar::zero(), s1 = Ar::zero(), s2 = Ar::zero(), s3 = Ar::zero();
#pragma unroll
        for (int jj = 0; jj < 32; jj += 4) {
          s0 = Ar::mac_t(s0, (double)tile[lane * 33 + jj], Ar::shfl(yv, jj));
          s1 = Ar::mac_t(s1, (double)tile[lane * 33 + jj + 1], Ar::shfl(yv, jj + 1));
          s2 = Ar::mac_t(s2, (double)tile[lane * 33 + jj + 2], Ar::shfl(yv, jj + 2));
          s3 = Ar::mac_t(s3, (double)tile[lane * 33 + jj + 3], Ar::shfl(yv, jj + 3));
        }
        acc = Ar::sub(acc, Ar::add(Ar::add(s0, s1), Ar::add(s2, s3)));
        __syncwarp();
      }
    }
    __syncthreads();
    if constexpr (Team::kGrid) {
      if (threadIdx.x < 32) {
        __threadfence();
        if (threadIdx.x == 0) st_release64(gctr, base + (unsigned long long)(s + 1));
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// CTA-per-block triangular solve for the non-exact modes (F64 / DD) on a grid
// team: 32-row block b is owned by one CTA; warp w holds rows 4w..4w+3 of the
// block, lane = column inside a 32-column tile.  Products accumulate per
// thread over all off-diagonal tiles (no per-tile reduction), so only the
// last tile, one butterfly sum and the 32x32 inverse apply sit on the
// dependency chain between blocks.  A dd tile owned by one lane per row costs
// ~3.4k cycles of dependent dd arithmetic on sm_100a; here a link is one MAC
// plus two 5-level butterflies.
// ---------------------------------------------------------------------------
template <int M>
GB_DEVICE typename Arith<M>::T ar_warp_sum(typename Arith<M>::T v) {
  if constexpr (M == MODE_DD) {
    return warp_sum_dd(v);
  } else {
    return warp_sum(v);
  }
}

// Tagged y entries: every 8-byte word carries 32 payload bits and a 32-bit
// tag (sweep id), so a consumer that sees the tag in both words of an entry
// has its value -- no progress counter, no fence, one round trip.
//   dsm == 0: the tagged copy lives in global memory (L2 round trip per poll);
//   dsm == G: the team is one thread-block cluster and every CTA holds its own
//             copy in shared memory -- producers push each entry into all G
//             copies (st.shared::cluster), consumers poll their local copy
//             (measured on B200: polling a producer's copy over DSMEM instead
//             is ~3x slower per link under contention).
// (q0, qs): this thread pushes into cluster CTAs q0, q0 + qs, ... (the
// producers of one entry split the G remote stores between them)
GB_DEVICE void ytag_put1(uint4* p, double v, unsigned tag, int dsm, int q0 = 0, int qs = 1) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  if (dsm == 0) {
    if (q0 == 0)
      asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"((unsigned)b), "r"(tag),
                   "r"((unsigned)(b >> 32)), "r"(tag)
                   : "memory");
    return;
  }
  const unsigned la = (unsigned)__cvta_generic_to_shared(p);
  for (int q = q0; q < dsm; q += qs) {
    unsigned ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(q));
    asm volatile("st.relaxed.cluster.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(ra), "r"((unsigned)b),
                 "r"(tag), "r"((unsigned)(b >> 32)), "r"(tag)
                 : "memory");
  }
}
GB_DEVICE bool ytag_get1(const uint4* p, unsigned tag, double& v, int dsm) {
  unsigned x, y, z, w;
  if (dsm == 0) {
    asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(x), "=r"(y), "=r"(z), "=r"(w)
                 : "l"(p)
                 : "memory");
  } else {
    asm volatile("ld.relaxed.cluster.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(x), "=r"(y), "=r"(z), "=r"(w)
                 : "r"((unsigned)__cvta_generic_to_shared(p))
                 : "memory");
  }
  v = __longlong_as_double((long long)(((unsigned long long)z << 32) | x));
  return y == tag && w == tag;
}
GB_DEVICE void ytag_put(uint4* yt, int i, double v, unsigned tag, int dsm, int q0 = 0, int qs = 1) {
  ytag_put1(yt + 2 * i, v, tag, dsm, q0, qs);
}
GB_DEVICE void ytag_put(uint4* yt, int i, dd v, unsigned tag, int dsm, int q0 = 0, int qs = 1) {
  ytag_put1(yt + 2 * i, v.hi, tag, dsm, q0, qs);
  ytag_put1(yt + 2 * i + 1, v.lo, tag, dsm, q0, qs);
}
GB_DEVICE bool ytag_get(const uint4* yt, int i, unsigned tag, double& v, int dsm) {
  return ytag_get1(yt + 2 * i, tag, v, dsm);
}
GB_DEVICE bool ytag_get(const uint4* yt, int i, unsigned tag, dd& v, int dsm) {
  const bool a = ytag_get1(yt + 2 * i, tag, v.hi, dsm);
  const bool b = ytag_get1(yt + 2 * i + 1, tag, v.lo, dsm);
  return a && b;
}
// warp-uniform poll: every lane waits for its own entry (invalid lanes: zero)
template <int M>
GB_DEVICE typename Arith<M>::T ytag_wait(const uint4* yt, int i, bool valid, unsigned tag, int dsm) {
  typename Arith<M>::T v = Arith<M>::zero();
  bool ok = !valid || ytag_get(yt, i, tag, v, dsm);
  while (!__all_sync(0xffffffffu, ok)) {
    if (!ok) ok = ytag_get(yt, i, tag, v, dsm);
  }
  return valid ? v : Arith<M>::zero();
}

// Compensated accumulation of products (Ogita-Rump-Oishi Dot2 for the DD
// mode): the exact product error and the two_sum error of every step are
// summed in a running double, so the result carries the accuracy of
// dd arithmetic (error <= u^2-level relative to sum |a_i y_i|) at ~10 fp64
// operations per term instead of a full dd_add; F64: a plain fma chain.
template <int M>
struct CAcc;
template <>
struct CAcc<MODE_F64> {
  double s = 0.0;
  GB_DEVICE void add(double a, double y) { s = __fma_rn(a, y, s); }
  // (ih, il) * t: the F64 mode keeps only the high part of dd records
  GB_DEVICE void add_inv(double ih, double, double t) { s = __fma_rn(ih, t, s); }
  GB_DEVICE void merge(const CAcc& o) { s = __dadd_rn(s, o.s); }
  GB_DEVICE CAcc xor_shfl(int o) const {
    CAcc r;
    r.s = __shfl_xor_sync(0xffffffffu, s, o);
    return r;
  }
  GB_DEVICE double get() const { return s; }
};
template <>
struct CAcc<MODE_DD> {
  double s = 0.0, c = 0.0;
  GB_DEVICE void add(double a, double y) {
    const double p = __dmul_rn(a, y);
    const double e = __fma_rn(a, y, -p);
    const double t = __dadd_rn(s, p);
    const double v = __dsub_rn(t, s);
    const double q = __dadd_rn(__dsub_rn(s, __dsub_rn(t, v)), __dsub_rn(p, v));
    s = t;
    c = __dadd_rn(c, __dadd_rn(q, e));
  }
  GB_DEVICE void add(double a, dd y) {
    const double p = __dmul_rn(a, y.hi);
    const double e = __fma_rn(a, y.lo, __fma_rn(a, y.hi, -p));
    const double t = __dadd_rn(s, p);
    const double v = __dsub_rn(t, s);
    const double q = __dadd_rn(__dsub_rn(s, __dsub_rn(t, v)), __dsub_rn(p, v));
    s = t;
    c = __dadd_rn(c, __dadd_rn(q, e));
  }
  // (ih + il) * (t.hi + t.lo): exact leading product, first-order cross terms
  GB_DEVICE void add_inv(double ih, double il, dd t) {
    const double p = __dmul_rn(ih, t.hi);
    const double e = __fma_rn(il, t.hi, __fma_rn(ih, t.lo, __fma_rn(ih, t.hi, -p)));
    const double u = __dadd_rn(s, p);
    const double v = __dsub_rn(u, s);
    const double q = __dadd_rn(__dsub_rn(s, __dsub_rn(u, v)), __dsub_rn(p, v));
    s = u;
    c = __dadd_rn(c, __dadd_rn(q, e));
  }
  // symmetric in (this, o): every lane of a butterfly ends with the same bits
  GB_DEVICE void merge(const CAcc& o) {
    const double u = __dadd_rn(s, o.s);
    const double v = __dsub_rn(u, s);
    const double q = __dadd_rn(__dsub_rn(s, __dsub_rn(u, v)), __dsub_rn(o.s, v));
    s = u;
    c = __dadd_rn(__dadd_rn(c, o.c), q);
  }
  GB_DEVICE CAcc xor_shfl(int o) const {
    CAcc r;
    r.s = __shfl_xor_sync(0xffffffffu, s, o);
    r.c = __shfl_xor_sync(0xffffffffu, c, o);
    return r;
  }
  GB_DEVICE dd get() const { return fast_two_sum(s, c); }
};

template <int M>
GB_DEVICE CAcc<M> cbfly8(CAcc<M> a) {
#pragma unroll
  for (int o = 1; o < 8; o <<= 1) a.merge(a.xor_shfl(o));
  return a;
}

// xor-butterfly over the 8 lanes of a row group (every lane ends with the same
// bits: the per-mode add is commutative bit for bit)
template <int M>
GB_DEVICE typename Arith<M>::T bfly8(typename Arith<M>::T v) {
#pragma unroll
  for (int o = 1; o < 8; o <<= 1) {
    if constexpr (M == MODE_DD) {
      dd w{__shfl_xor_sync(0xffffffffu, v.hi, o), __shfl_xor_sync(0xffffffffu, v.lo, o)};
      v = dd_add(v, w);
    } else {
      v = Arith<M>::add(v, __shfl_xor_sync(0xffffffffu, v, o));
    }
  }
  return v;
}

// four consecutive factor entries of one row (zero past n), vectorised when
// the run is in range (rows are padded to 32 entries, runs start at 4k)
template <class TF>
GB_DEVICE void load4(const TF* __restrict__ p, int c, int n, bool rowok, double (&d)[4]) {
  if (rowok && c + 3 < n) {
    if constexpr (sizeof(TF) == 4) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(p));
      d[0] = v.x, d[1] = v.y, d[2] = v.z, d[3] = v.w;
    } else if constexpr (sizeof(TF) == 2) {
      const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
      const __half2 a = *reinterpret_cast<const __half2*>(&v.x), b = *reinterpret_cast<const __half2*>(&v.y);
      d[0] = __low2float(a), d[1] = __high2float(a), d[2] = __low2float(b), d[3] = __high2float(b);
    } else {
      const double2 a = __ldg(reinterpret_cast<const double2*>(p)), b = __ldg(reinterpret_cast<const double2*>(p) + 1);
      d[0] = a.x, d[1] = a.y, d[2] = b.x, d[3] = b.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) d[j] = (rowok && c + j < n) ? to_d(p[j]) : 0.0;
  }
}

template <int M, class Team, class TF, bool kLower>
__device__ void trsv_cta(Team& t, int n, const TF* __restrict__ LU, size_t ldf, typename Arith<M>::T* y,
                         const TrsvSync& ts, void* smem_raw, const double* __restrict__ inv_h,
                         const double* __restrict__ inv_l) {
  // Lane layout: warp w owns rows 4w..4w+3 of the 32-row block; inside the
  // warp, lane = 8 * (row - 4w) + cg and lane cg covers the four columns
  // 4cg..4cg+3 of every 32-column tile.  Every row sum is then four MACs per
  // lane plus a 3-level butterfly over the row's 8 lanes, so the chain
  // between blocks is 4 MACs + 3 shuffle levels (instead of one 5-level warp
  // reduction per row).
  using Ar = Arith<M>;
  using T = typename Ar::T;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int rq = lane >> 3, cg = lane & 7, c4 = cg * 4;
  const int ri = wid * 4 + rq;  // row inside the block
  const int nb = (n + 31) / 32;
  T* tsh = reinterpret_cast<T*>(smem_raw);  // [2][32]: the block's reduced right-hand side
  uint4* yt = ts.ytag;
  const unsigned tag = (unsigned)(2ull * ts.epoch + (kLower ? 1ull : 2ull));
  const unsigned ftag = (unsigned)(2ull * ts.epoch + 1ull);
  const int G = t.size();
  int it = 0;
  for (int s = t.rank(); s < nb; s += G, ++it) {
    const int b = kLower ? s : nb - 1 - s;
    const int r = b * 32 + ri;
    const bool rowok = r < n;
    const int noff = kLower ? b : nb - 1 - b;
    const int nfar = noff > 0 ? noff - 1 : 0;  // tiles before the adjacent block
    // block inverse (column-major, [c * 32 + ri]) and folded neighbour block
    // (row-major, [1024 + ri * 32 + c]) for this lane's four columns
    double ih[4], il[4], mh[4], ml[4];
    const double* rec_h = inv_h + (size_t)b * kInvStride;
    const double* rec_l = inv_l + (size_t)b * kInvStride;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      ih[j] = __ldg(rec_h + (c4 + j) * 32 + ri);
      il[j] = __ldg(rec_l + (c4 + j) * 32 + ri);
      mh[j] = -__ldg(rec_h + 1024 + ri * 32 + c4 + j);
      ml[j] = -__ldg(rec_l + 1024 + ri * 32 + c4 + j);
    }
    // own row's input: lower -> permuted right-hand side; upper -> forward result
    T y0 = kLower ? (rowok ? Ar::ld(y + r) : Ar::zero()) : ytag_wait<M>(yt, r, rowok, ftag, ts.dsm);
    CAcc<M> ca0, ca1;
    double lv[4], ln[4];
    const TF* lrow = LU + (size_t)(rowok ? r : 0) * ldf;
    auto tile_col = [&](int q) { return (kLower ? q : nb - 1 - q) * 32; };
    if (nfar > 0) load4<TF>(lrow + tile_col(0) + c4, tile_col(0) + c4, n, rowok, lv);
    for (int q = 0; q < nfar; ++q) {
      const int tc = tile_col(q);
      if (q + 1 < nfar) load4<TF>(lrow + tile_col(q + 1) + c4, tile_col(q + 1) + c4, n, rowok, ln);
      const T yl = ytag_wait<M>(yt, tc + lane, tc + lane < n, tag, ts.dsm);
      ca0.add(lv[0], Ar::shfl(yl, c4 + 0));
      ca1.add(lv[1], Ar::shfl(yl, c4 + 1));
      ca0.add(lv[2], Ar::shfl(yl, c4 + 2));
      ca1.add(lv[3], Ar::shfl(yl, c4 + 3));
#pragma unroll
      for (int j = 0; j < 4; ++j) lv[j] = ln[j];
    }
    // t' = y0 - (far tiles) for this row (all 8 lanes of the row hold it)
    T acc = Ar::zero();
    if (nfar > 0) {
      ca0.merge(ca1);
      acc = T(cbfly8<M>(ca0).get());
    }
    const T tp = Ar::sub(y0, acc);
    T* tb = tsh + (it & 1) * 32;
    if (cg == 0) tb[ri] = tp;
    __syncthreads();
    // partial of D_b^-1 t' over this lane's columns (lower: unit diagonal
    // implied), carried as a compensated pair through the chain below
    CAcc<M> pa, pb;
    pa.add_inv(ih[0], il[0], tb[c4 + 0]);
    pb.add_inv(ih[1], il[1], tb[c4 + 1]);
    pa.add_inv(ih[2], il[2], tb[c4 + 2]);
    pb.add_inv(ih[3], il[3], tb[c4 + 3]);
    if (ts.stamps != nullptr && threadIdx.x == 0) ts.stamps[3 * s] = gtimer();
    // y_b = D_b^-1 t' - M_b y_adjacent  (critical chain: 2 products deep,
    // one pair merge, 3 butterfly merges)
    if (noff > 0) {
      const int tc = (kLower ? b - 1 : b + 1) * 32;
      const T yl = ytag_wait<M>(yt, tc + lane, tc + lane < n, tag, ts.dsm);
      if (ts.stamps != nullptr && threadIdx.x == 0) ts.stamps[3 * s + 2] = gtimer();
      pa.add_inv(mh[0], ml[0], Ar::shfl(yl, c4 + 0));
      pb.add_inv(mh[1], ml[1], Ar::shfl(yl, c4 + 1));
      pa.add_inv(mh[2], ml[2], Ar::shfl(yl, c4 + 2));
      pb.add_inv(mh[3], ml[3], Ar::shfl(yl, c4 + 3));
    }
    pa.merge(pb);
    T z = T(cbfly8<M>(pa).get());
    if (kLower) z = Ar::add(z, tp);
    if (rowok) {
      ytag_put(yt, r, z, tag, ts.dsm, cg, 8);  // the row's 8 lanes share the cluster pushes
      if (cg == 0) y[r] = z;
    }
    if (ts.stamps != nullptr && threadIdx.x == 0) ts.stamps[3 * s + 1] = gtimer();
  }
}

// ---------------------------------------------------------------------------
// Grid-team substitution with B-row blocks (B = kTrsvB = 64, n > 1024): the
// same scheme as trsv_cta with larger blocks (half the links of the chain);
// the block records are staged in shared memory while the far tiles are
// accumulated.  Out of line so its registers do not burden k_step.
// ---------------------------------------------------------------------------
// xor-butterfly of compensated pairs over L lanes (L a power of two)
template <int M, int L>
GB_DEVICE CAcc<M> cbfly(CAcc<M> a) {
#pragma unroll
  for (int o = 1; o < L; o <<= 1) a.merge(a.xor_shfl(o));
  return a;
}

// shared memory of trsv_cta<B>: tsh [2][B] T | ystage [8][B] T | block
// record stage (D_b^-1 and M_b: 2 B^2 hi, + 2 B^2 lo in the dd mode)
template <int M, int B>
__host__ __device__ constexpr size_t trsv_cta_smem() {
  return (2 + 8) * (size_t)B * sizeof(typename Arith<M>::T) + 2 * (size_t)B * (B + 1) * 8 * (M == MODE_DD ? 2 : 1);
}

template <int M, class Team, class TF, bool kLower, int B = kTrsvB>
__device__ __noinline__ void trsv_cta_g(Team& t, int n, const TF* __restrict__ LU, size_t ldf, typename Arith<M>::T* y,
                         const TrsvSync& ts, void* smem_raw, const double* __restrict__ inv_h,
                         const double* __restrict__ inv_l) {
  // Block b (B rows) is owned by CTA b mod G.  Lane layout: warp w owns rows
  // RPW*w .. RPW*w+RPW-1 of the block; the LPR lanes of a row each cover CPL
  // columns of every B-column tile, in runs of 4: column 4*LPR*g + 4*cg + e
  // (vector loads from the factors, conflict-free shared-memory reads).  Every row sum is CPL MACs
  // per lane (two compensated chains) plus a log2(LPR)-level butterfly, so
  // the chain between blocks is: stage the neighbour's B entries, CPL MACs
  // against the folded neighbour block M_b (staged in shared memory while
  // the far tiles are accumulated), the butterfly and the push.
  using Ar = Arith<M>;
  using T = typename Ar::T;
  constexpr int NW = 8;  // warps per CTA (blockDim 256)
  constexpr int RPW = B / NW, LPR = 32 / RPW, CPL = B / LPR, YPL = B / 32;
  constexpr int RS = inv_stride<B>();
  static_assert(RPW * NW == B && LPR * RPW == 32 && CPL % 4 == 0, "unsupported TRSV block");
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int rq = lane / LPR, cg = lane % LPR;
  constexpr int S = B + 1;  // padded row stride of the staged records
  // column of this lane's j-th product (j = 4 g + e)
  auto colj = [&](int j) { return (j >> 2) * 4 * LPR + 4 * cg + (j & 3); };
  const int ri = wid * RPW + rq;  // row inside the block
  const int nb = (n + B - 1) / B;
  T* tsh = reinterpret_cast<T*>(smem_raw);        // [2][B]
  T* ystage = tsh + 2 * B + wid * B;              // this warp's [B]
  // staged record, row-major with stride S: D_b^-1 rows [0, B), M_b rows [B, 2B)
  double* rst_h = reinterpret_cast<double*>(tsh + (2 + NW) * B);
  double* rst_l = rst_h + 2 * B * S;  // dd mode only
  uint4* yt = ts.ytag;
  const unsigned tag = (unsigned)(2ull * ts.epoch + (kLower ? 1ull : 2ull));
  const unsigned ftag = (unsigned)(2ull * ts.epoch + 1ull);
  const int G = t.size();
  // stage the B entries of tile column tc (warp-wide poll) into ystage
  auto stage_tile = [&](int tc) {
    __syncwarp();
    // poll all YPL entries of this lane together (one round trip per poll)
    T v[YPL];
    bool ok[YPL];
#pragma unroll
    for (int h = 0; h < YPL; ++h) {
      const int c = tc + h * 32 + lane;
      v[h] = Ar::zero();
      ok[h] = !(c < n) || ytag_get(yt, c, tag, v[h], ts.dsm);
    }
    for (;;) {
      bool all = true;
#pragma unroll
      for (int h = 0; h < YPL; ++h) all = all && ok[h];
      if (__all_sync(0xffffffffu, all)) break;
#pragma unroll
      for (int h = 0; h < YPL; ++h)
        if (!ok[h]) ok[h] = ytag_get(yt, tc + h * 32 + lane, tag, v[h], ts.dsm);
    }
#pragma unroll
    for (int h = 0; h < YPL; ++h) ystage[h * 32 + lane] = (tc + h * 32 + lane < n) ? v[h] : Ar::zero();
    __syncwarp();
  };
  int it = 0;
  for (int s = t.rank(); s < nb; s += G, ++it) {
    const int b = kLower ? s : nb - 1 - s;
    const int r = b * B + ri;
    const bool rowok = r < n;
    const int noff = kLower ? b : nb - 1 - b;
    const int nfar = noff > 0 ? noff - 1 : 0;  // tiles before the adjacent block
    const double* rec_h = inv_h + (size_t)b * RS;
    const double* rec_l = inv_l + (size_t)b * RS;
    __syncthreads();  // previous block's readers of the record stage are done
    {
      // stage D_b^-1 (and M_b when a neighbour exists): the loads overlap the
      // far-tile accumulation; the chain then reads only shared memory
      // D^-1 is column-major in the record: transpose into rows
      for (int e = threadIdx.x; e < B * B; e += blockDim.x) {
        const int i = e % B, c = e / B;
        rst_h[i * S + c] = __ldg(rec_h + e);
        if constexpr (M == MODE_DD) rst_l[i * S + c] = __ldg(rec_l + e);
      }
      if (noff > 0)
        for (int e = threadIdx.x; e < B * B; e += blockDim.x) {
          const int i = e / B, c = e % B;
          rst_h[(B + i) * S + c] = __ldg(rec_h + B * B + e);
          if constexpr (M == MODE_DD) rst_l[(B + i) * S + c] = __ldg(rec_l + B * B + e);
        }
    }
    // own row's input: lower -> permuted right-hand side; upper -> forward result
    T y0 = kLower ? (rowok ? Ar::ld(y + r) : Ar::zero()) : ytag_wait<M>(yt, r, rowok, ftag, ts.dsm);
    CAcc<M> ca0, ca1;
    double lv[CPL], ln[CPL];
    const TF* lrow = LU + (size_t)(rowok ? r : 0) * ldf;
    auto tile_col = [&](int q) { return (kLower ? q : nb - 1 - q) * B; };
    auto load_row = [&](int tc, double (&d)[CPL]) {
#pragma unroll
      for (int g = 0; g < CPL / 4; ++g) {
        double q4[4];
        const int c = tc + colj(4 * g);
        load4<TF>(lrow + c, c, n, rowok, q4);
#pragma unroll
        for (int e = 0; e < 4; ++e) d[4 * g + e] = q4[e];
      }
    };
    if (nfar > 0) load_row(tile_col(0), lv);
    for (int q = 0; q < nfar; ++q) {
      const int tc = tile_col(q);
      if (q + 1 < nfar) load_row(tile_col(q + 1), ln);
      stage_tile(tc);
#pragma unroll
      for (int j = 0; j < CPL; j += 2) {
        ca0.add(lv[j], ystage[colj(j)]);
        ca1.add(lv[j + 1], ystage[colj(j + 1)]);
      }
#pragma unroll
      for (int j = 0; j < CPL; ++j) lv[j] = ln[j];
    }
    // t' = y0 - (far tiles) for this row (all LPR lanes of the row hold it)
    T acc = Ar::zero();
    if (nfar > 0) {
      ca0.merge(ca1);
      acc = T(cbfly<M, LPR>(ca0).get());
    }
    const T tp = Ar::sub(y0, acc);
    T* tb = tsh + (it & 1) * B;
    if (cg == 0) tb[ri] = tp;
    __syncthreads();
    // partial of D_b^-1 t' over this lane's columns (lower: unit diagonal
    // implied), carried as a compensated pair through the chain below
    CAcc<M> pa, pb;
#pragma unroll
    for (int j = 0; j < CPL; j += 2) {
      const int e0 = ri * S + colj(j), e1 = ri * S + colj(j + 1);
      pa.add_inv(rst_h[e0], M == MODE_DD ? rst_l[e0] : 0.0, tb[colj(j)]);
      pb.add_inv(rst_h[e1], M == MODE_DD ? rst_l[e1] : 0.0, tb[colj(j + 1)]);
    }
    if (ts.stamps != nullptr && threadIdx.x == 0) ts.stamps[3 * s] = gtimer();
    // y_b = D_b^-1 t' - M_b y_adjacent
    if (noff > 0) {
      stage_tile((kLower ? b - 1 : b + 1) * B);
      if (ts.stamps != nullptr && threadIdx.x == 0) ts.stamps[3 * s + 2] = gtimer();
#pragma unroll
      for (int j = 0; j < CPL; j += 2) {
        const int e0 = (B + ri) * S + colj(j), e1 = (B + ri) * S + colj(j + 1);
        pa.add_inv(-rst_h[e0], M == MODE_DD ? -rst_l[e0] : 0.0, ystage[colj(j)]);
        pb.add_inv(-rst_h[e1], M == MODE_DD ? -rst_l[e1] : 0.0, ystage[colj(j + 1)]);
      }
    }
    pa.merge(pb);
    T z = T(cbfly<M, LPR>(pa).get());
    if (kLower) z = Ar::add(z, tp);
    if (rowok) {
      ytag_put(yt, r, z, tag, ts.dsm, cg, LPR);  // grid team: the cg == 0 lane stores
      if (cg == 0) y[r] = z;
    }
    if (ts.stamps != nullptr && threadIdx.x == 0) ts.stamps[3 * s + 1] = gtimer();
  }
}

template <int M, class TF>
__host__ __device__ inline size_t trsv_smem_bytes(int nthreads) {
  return (size_t)(nthreads / 32) * 32 * 33 * sizeof(typename TileT<TF>::T) +
         (size_t)nthreads * sizeof(typename Arith<M>::T);
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
template <int M, bool kAbs, class TA, class TV, int kU = 4>
__device__ __forceinline__ typename Arith<M>::T row_dot_ex(const TA* __restrict__ arow, const TV* __restrict__ v,
                                                           int n, double* absdot) {
  using Ar = Arith<M>;
  using T = typename Ar::T;
  constexpr int VW = Vec16<TA>::N;
  const int lane = threadIdx.x & 31;
  if constexpr (M == MODE_DD) {
    // compensated (Dot2) accumulation: exact products, two_sum errors summed
    CAcc<MODE_DD> ca[kU];
    double ab[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) ab[u] = 0.0;
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
          ca[u].add(x, y);
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
        ca[0].add(x, y);
        if (kAbs) ab[0] = __fma_rn(fabs(x), fabs(y), ab[0]);
      }
    }
    for (int j = nv * VW + lane; j < n; j += 32) {
      const double x = (double)arow[j];
      const double y = to_d(v[j]);
      ca[1].add(x, y);
      if (kAbs) ab[1] = __fma_rn(fabs(x), fabs(y), ab[1]);
    }
    dd s;
    if constexpr (kU == 4) {
      s = dd_add(dd_add(ca[0].get(), ca[1].get()), dd_add(ca[2].get(), ca[3].get()));
    } else {
#pragma unroll
      for (int h = kU / 2; h > 0; h >>= 1)
#pragma unroll
        for (int u = 0; u < h; ++u) ca[u].merge(ca[u + h]);
      s = ca[0].get();
    }
    s = warp_sum_dd(s);
    if (kAbs) {
#pragma unroll
      for (int h = kU / 2; h > 2; h >>= 1)
#pragma unroll
        for (int u = 0; u < h; ++u) ab[u] += ab[u + h];
      *absdot = warp_sum((ab[0] + ab[1]) + (ab[2] + ab[3]));
    }
    return s;
  }
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
#pragma unroll
  for (int h = kU / 2; h > 2; h >>= 1)
#pragma unroll
    for (int u = 0; u < h; ++u) {
      acc[u] = Ar::add(acc[u], acc[u + h]);
      ab[u] += ab[u + h];
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
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  mark(ts.log, 10);
  if constexpr (Team::kGrid && Team::kTB == kTrsvB && M == MODE_F64) {
    if (s.bigl != nullptr) {
      // grid team, fp64 operator: bulk-copy GEMV + big-block substitutions
      double* yb = reinterpret_cast<double*>(ybuf);
      double* ysol = yb + s.lda;  // ybuf holds 2 ldv doubles
      if (v != nullptr) {
        if (s.a_normal)
          seg::gemv_perm<TA, TV, true>(t, n, s.A, s.lda, s.perm, v, yb, smem, s.gemv_ns, ts.log);
        else
          seg::gemv_perm<TA, TV, false>(t, n, s.A, s.lda, s.perm, v, yb, smem, s.gemv_ns, ts.log);
      } else {
        int lo, hi;
        t.rows(n, lo, hi);
        for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) yb[i] = to_d(rvec[s.perm[i]]);
      }
      t.sync();
      mark(ts.log, 11);
      if (s.sweep_la) {
        seg::sweep_la<TF, true>(t, n, s.nbig, s.LU, s.ldf, s.bigl, yb, ysol, seg::OutNone{}, smem);
        mark(ts.log, 12);
        seg::sweep_la<TF, false>(t, n, s.nbig, s.LU, s.ldf, s.bigu, ysol, yb, seg::OutTo<TW>{w}, smem);
      } else {
        seg::sweep_bsp<TF, true>(t, n, s.nbig, s.LU, s.ldf, s.bigl, yb, ysol, seg::OutNone{}, smem);
        mark(ts.log, 12);
        seg::sweep_bsp<TF, false>(t, n, s.nbig, s.LU, s.ldf, s.bigu, ysol, yb, seg::OutTo<TW>{w}, smem);
      }
      mark(ts.log, 13);
      ts.epoch++;
      return;
    }
  }
  // 1. right-hand side in permuted order over the team's row slices
  int lo, hi;
  t.rows(n, lo, hi);
  for (int i = lo + wid; i < hi; i += nw) {
    const int src = s.perm[i];
    typename Ar::T val;
    if (v != nullptr) {
      if constexpr (Team::kTB == kTrsvB)  // grid teams (n > 1024): rows stream from HBM, 8 x 16 B in flight per lane
        val = row_dot_ex<M, false, TA, TV, 8>(s.A + (size_t)src * s.lda, v, n, nullptr);
      else
        val = row_dot<M>(s.A + (size_t)src * s.lda, v, n);
    } else {
      val = Ar::from(to_d(rvec[src]));
    }
    if (lane == 0) ybuf[i] = val;
  }
  t.sync();
  mark(ts.log, 11);
  // 2. forward (unit lower) then backward (upper)
  bool done = false;
  if constexpr (Team::kGrid && Arith<M>::kInv) {
    if (s.linv_hi != nullptr && s.uinv_hi != nullptr && ts.ytag != nullptr) {
      if constexpr (Team::kTB == kTrsvB) {
        trsv_cta_g<M, Team, TF, true, kTrsvB>(t, n, s.LU, s.ldf, ybuf, ts, smem, s.linv_hi, s.linv_lo);
        mark(ts.log, 12);
        trsv_cta_g<M, Team, TF, false, kTrsvB>(t, n, s.LU, s.ldf, ybuf, ts, smem, s.uinv_hi, s.uinv_lo);
      } else {
        trsv_cta<M, Team, TF, true>(t, n, s.LU, s.ldf, ybuf, ts, smem, s.linv_hi, s.linv_lo);
        mark(ts.log, 12);
        trsv_cta<M, Team, TF, false>(t, n, s.LU, s.ldf, ybuf, ts, smem, s.uinv_hi, s.uinv_lo);
      }
      done = true;
    }
  }
  if constexpr (!Team::kGrid && Arith<M>::kInv) {
    if (s.linv_hi != nullptr && s.uinv_hi != nullptr) {
      trsv_super<M, Team, TF, true>(t, n, s.LU, s.ldf, ybuf, ts, smem, s.linv_hi, s.linv_lo);
      mark(ts.log, 12);
      trsv_super<M, Team, TF, false>(t, n, s.LU, s.ldf, ybuf, ts, smem, s.uinv_hi, s.uinv_lo);
      done = true;
    }
  }
  if (!done) {
    trsv_blocks<M, Team, TF, true>(t, n, s.LU, s.ldf, ybuf, ts, smem, nullptr, nullptr, s.linv_hi, s.linv_lo);
    mark(ts.log, 12);
    trsv_blocks<M, Team, TF, false>(t, n, s.LU, s.ldf, ybuf, ts, smem, s.rcp_hi, s.rcp_lo, s.uinv_hi, s.uinv_lo);
  }
  mark(ts.log, 13);
  ts.epoch++;
  // 3. round to u (rows of this CTA's slice; the backward sweep is complete
  // once the whole team passed the barrier)
  t.sync();
  for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) w[i] = (TW)Ar::val(Ar::ld(ybuf + i));
  t.sync();
  mark(ts.log, 14);
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
  t.template reduce<Acc, K>(a, reinterpret_cast<Acc*>(red));
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
