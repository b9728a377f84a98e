// Segment-pipelined preconditioned operator for grid teams (n > 1024, F64
// operator mode: u^2 = double, densela.py:268-333).
//
//   w = fl_u( U^-1 L^-1 ( (A v)[perm] ) )        (apply_preconditioned)
//   w = fl_u( U^-1 L^-1 r[perm] )                (precond_rhs, v == nullptr)
//
// Phase G (GEMV): every warp of the grid streams rows of A in perm order,
// 16 x 16 B loads in flight per lane, v staged once per CTA in shared memory.
//
// Phases L / U (substitutions): the sweep's 64-row blocks are grouped into
// segments of K consecutive blocks (sweep order); segment s is owned by CTA
// s mod G.  An owner
//   * accumulates the far field of its K*64 rows tile column by tile column
//     as the earlier blocks are published (tagged 16-byte words, no fences:
//     ytag_put/ytag_get), with the factor tiles streamed ahead of the wait;
//   * when the last earlier block lands, solves its K blocks back to back on
//     the SM: y_i = D_i^-1 (t_i - acc_i) with the block inverses held in
//     registers, each solved block updating the later blocks of the segment
//     from a shared-memory copy of the intra-segment tiles.
// The dependency chain therefore crosses SMs once per K blocks instead of
// once per block (trsv_cta_g), and the hand-off is one L2 round trip.
//
// All sums are plain fp64 fma chains in a fixed order (deterministic; the
// reference's dgemv / dtrsv accumulate in fp64 too).
#pragma once
#include "gb_common.cuh"
#include "gb_team.cuh"

namespace gb {
namespace seg {

constexpr int B = 64;    // block rows
constexpr int NT = 256;  // threads per CTA

// ---------------------------------------------------------------------------
// tagged entries: 16 B per value = {lo32, tag, hi32, tag}
// ---------------------------------------------------------------------------
GB_DEVICE void tput(uint4* p, double v, unsigned tag) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"((unsigned)b), "r"(tag),
               "r"((unsigned)(b >> 32)), "r"(tag)
               : "memory");
}
GB_DEVICE bool tget(const uint4* p, unsigned tag, double& v) {
  unsigned x, y, z, w;
  asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(x), "=r"(y), "=r"(z), "=r"(w)
               : "l"(p)
               : "memory");
  v = __longlong_as_double((long long)(((unsigned long long)z << 32) | x));
  return y == tag && w == tag;
}

// float -> double on the integer pipe (the F2F.F64.F32 conversion runs on
// the XU pipe, which a GEMV at HBM speed would saturate): exact for zero,
// normal, inf and NaN inputs; subnormal floats take the conversion unit
GB_DEVICE double f2d_int(float f) {
  const unsigned x = __float_as_uint(f);
  const unsigned mag = x & 0x7fffffffu;
  const unsigned e = (mag >> 3) + 0x38000000u;
  unsigned hi = mag >= 0x7f800000u ? ((mag >> 3) | 0x7ff00000u) : e;
  hi = (x & 0x80000000u) | (mag ? hi : 0u);
  double d = __hiloint2double((int)hi, (int)(x << 29));
  if (mag - 1u < 0x007fffffu) d = (double)f;  // subnormal (rare)
  return d;
}
// float -> double for a normal float (4 integer ops): sign and exponent are
// re-biased in place; callers check once per system that A has no zero,
// subnormal, inf or NaN entry (gemv_normal flag), else use f2d_int
GB_DEVICE double f2d_normal(float f) {
  const unsigned x = __float_as_uint(f);
  const unsigned hi = ((unsigned)(((int)x) >> 3) & 0x8fffffffu) + 0x38000000u;
  return __hiloint2double((int)hi, (int)(x << 29));
}
// half -> double: the half -> float step is exact and always lands on a
// normal float (or zero), so the integer path needs no subnormal branch
GB_DEVICE double h2d_int(float fh) {
  const unsigned x = __float_as_uint(fh);
  const unsigned mag = x & 0x7fffffffu;
  unsigned hi = mag >= 0x7f800000u ? ((mag >> 3) | 0x7ff00000u) : ((mag >> 3) + 0x38000000u);
  hi = (x & 0x80000000u) | (mag ? hi : 0u);
  return __hiloint2double((int)hi, (int)(x << 29));
}

template <class TF>
GB_DEVICE double f2d(TF x) {
  if constexpr (sizeof(TF) == 2) {
    return (double)__half2float(x);
  } else {
    return (double)x;
  }
}
// the same conversion (exact) on the integer pipe: F2F.F64.F32 issues at a
// quarter of the FMA rate and would cap a sweep that converts every factor
// entry once
template <class TF>
GB_DEVICE double f2d_fast(TF x) {
  if constexpr (sizeof(TF) == 2) {
    return h2d_int(__half2float(x));
  } else if constexpr (sizeof(TF) == 4) {
    return f2d_int(x);
  } else {
    return (double)x;
  }
}

// 8 consecutive factor entries (16 B of fp16, 32 B of fp32, 64 B of fp64)
template <class TF>
struct Pack8 {
  uint4 q[sizeof(TF) / 2];
};
template <class TF>
GB_DEVICE Pack8<TF> ld8(const TF* p) {
  Pack8<TF> r;
#pragma unroll
  for (int i = 0; i < (int)(sizeof(TF) / 2); ++i)
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.q[i].x), "=r"(r.q[i].y), "=r"(r.q[i].z), "=r"(r.q[i].w)
                 : "l"(reinterpret_cast<const uint4*>(p) + i));
  return r;
}
template <class TF>
GB_DEVICE void unpack8(const Pack8<TF>& p, double (&d)[8]) {
  if constexpr (sizeof(TF) == 2) {
    const __half2* h = reinterpret_cast<const __half2*>(&p.q[0]);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __half22float2(h[i]);
      d[2 * i] = h2d_int(f.x);
      d[2 * i + 1] = h2d_int(f.y);
    }
  } else if constexpr (sizeof(TF) == 4) {
    const float* f = reinterpret_cast<const float*>(&p.q[0]);
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i] = f2d_int(f[i]);
  } else {
    const double* f = reinterpret_cast<const double*>(&p.q[0]);
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i] = f[i];
  }
}

// ---------------------------------------------------------------------------
// async-copy helpers (cp.async 16 B, bulk copies with an mbarrier)
// ---------------------------------------------------------------------------
GB_DEVICE unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
GB_DEVICE void cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
GB_DEVICE void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
GB_DEVICE void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
GB_DEVICE void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
GB_DEVICE void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
GB_DEVICE void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
GB_DEVICE void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
GB_DEVICE void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// padded row stride of the staged intra-segment tiles: 68 doubles = 8 banks
// mod 32, so the 16 lanes of a half-warp (4 rows x 4 column phases) are
// conflict-free
constexpr int TP = 68;
constexpr int PD = 6;   // factor tile columns in flight (cp.async ring)
constexpr int PY = 16;  // staged published blocks (ring)
#ifndef GB_SEG_FAR_NS
#define GB_SEG_FAR_NS 128
#endif
#ifndef GB_SEG_PB
#define GB_SEG_PB 1
#endif
constexpr int PB = GB_SEG_PB;  // blocks polled per round trip
#ifndef GB_SEG_SLEEP
#define GB_SEG_SLEEP 1000
#endif

// shared memory of one sweep: Yring [PY][B] | T [R] | S [R] | intra tiles
// [K(K-1)/2][B][TP] | block inverses [K][B][TP] (fp64) | factor ring
// [PD][R][B] (TF) | counters
template <int K, class TF>
__host__ __device__ constexpr size_t sweep_smem() {
  return (size_t)(PY * B + 2 * K * B + (K * (K - 1) / 2) * B * TP + K * B * TP) * sizeof(double) +
         (size_t)PD * K * B * B * sizeof(TF) + 64;
}
// GEMV: v staged as fp64 (one conversion per element of A), then a bulk-copy
// ring of GCH-byte stages filling the rest of the budget (<= GNS_MAX)
constexpr int GCH = 16 * 1024;  // bytes per stage
constexpr int GNS_MAX = 8;
__host__ __device__ constexpr size_t gemv_vbytes(int n) { return ((size_t)n * 8 + 127) & ~(size_t)127; }
__host__ __device__ constexpr int gemv_stages(int n, size_t budget) {
  return (int)((budget - gemv_vbytes(n) - 512 - 4096) / GCH) < GNS_MAX
             ? (int)((budget - gemv_vbytes(n) - 512 - 4096) / GCH)
             : GNS_MAX;
}
constexpr int GROWS_MAX = 1024;  // rows per CTA (team slices are <= 1024 rows)
__host__ __device__ constexpr size_t gemv_smem(int n, int stages) {
  return gemv_vbytes(n) + (size_t)stages * GCH + 512 + GROWS_MAX * 4;
}

// output functors of the sweeps: nothing (forward) or w[i] = fl_u(y_i)
struct OutNone {
  GB_DEVICE void operator()(int, double) const {}
};
template <class TW>
struct OutTo {
  TW* w;
  GB_DEVICE void operator()(int i, double v) const { w[i] = (TW)v; }
};

struct SweepIO {
  int n;
  const void* LU;  // TF, row-major, leading dimension ldf
  size_t ldf;
  const double* inv;  // block records: b * 2 B^2 + c * B + i = (D_b^-1)_{ic} (hi)
  const double* rhs;  // lower: right-hand side (plain, perm order); upper: nullptr (read tagged fwd)
  uint4* tin;         // upper: tagged forward result (tag tin_tag)
  unsigned tin_tag;
  uint4* tout;  // tagged solution of this sweep
  unsigned tag;
  unsigned long long* stamps = nullptr;  // diagnostics: 4 globaltimer stamps per segment
};

// ---------------------------------------------------------------------------
// one sweep (lower: unit L forward, upper: U backward) over a grid team
// ---------------------------------------------------------------------------
template <class TF, bool kLower, int K, class Team, class Out>
__device__ __noinline__ void sweep(Team& t, const SweepIO io, void* smem_raw, Out out) {
  constexpr int R = K * B;     // rows per segment
  constexpr int RIT = R / 32;  // row iterations per warp (8 lanes per row, 4 rows per warp instr)
  constexpr int EPR = B * sizeof(TF) / 16;  // 16-B pieces per tile row
  const int n = io.n;
  const int nb = (n + B - 1) / B;
  const int nseg = (nb + K - 1) / K;
  const int G = t.size();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int rg = lane >> 3, cg = lane & 7;  // row-in-quad, column group (8 columns)
  const TF* LU = reinterpret_cast<const TF*>(io.LU);
  double* Yr = reinterpret_cast<double*>(smem_raw);  // [PY][B]
  double* T = Yr + PY * B;                            // [R]
  double* S = T + R;                                  // [R]
  double* TI = S + R;                                 // [K(K-1)/2][B][TP]
  double* DI = TI + (K * (K - 1) / 2) * B * TP;                     // [K][B][TP] row-major D^-1
  TF* Lr = reinterpret_cast<TF*>(DI + K * B * TP);                   // [PD][R][B]
  int* ycount = reinterpret_cast<int*>(Lr + (size_t)PD * R * B);
  auto blk = [&](int q) { return kLower ? q : nb - 1 - q; };  // sweep index -> block
  for (int s = t.rank(); s < nseg; s += G) {
    const int q0 = s * K;
    auto grow_of = [&](int slot) { return blk(min(q0 + slot / B, nb - 1)) * B + (slot % B); };
    const int kb = min(K, nb - q0);  // blocks in this segment
    const int rr = threadIdx.x >> 2, qq = threadIdx.x & 3;
    // ---- block inverses of the segment into shared memory, transposed to
    // row-major (the records are column-major): DI[i][row][col]
    for (int i = 0; i < kb; ++i) {
      const double* rec = io.inv + (size_t)blk(q0 + i) * 2 * B * B;
      for (int e = threadIdx.x; e < B * B; e += NT) DI[(size_t)i * B * TP + (e % B) * TP + e / B] = __ldg(rec + e);
    }
    // ---- intra-segment tiles (i' > i in sweep order): TI[p][row][col] fp64
    {
      int p = 0;
#pragma unroll
      for (int i = 0; i < K; ++i)
#pragma unroll
        for (int i2 = i + 1; i2 < K; ++i2, ++p) {
          if (i2 >= kb) continue;
          const int rb = blk(q0 + i2) * B, cb = blk(q0 + i) * B;
          for (int e = threadIdx.x; e < B * B; e += NT) {
            const int r = e / B, c = e % B;
            const int gr = rb + r, gc = cb + c;
            TI[(size_t)p * B * TP + r * TP + c] = (gr < n && gc < n) ? f2d<TF>(LU[(size_t)gr * io.ldf + gc]) : 0.0;
          }
        }
    }
    // ---- right-hand side of the segment rows (before the far field: off the chain)
    if (kLower) {
      for (int sl = threadIdx.x; sl < R; sl += NT) {
        const int gr = grow_of(sl);
        T[sl] = ((sl / B) < kb && gr < n) ? io.rhs[gr] : 0.0;
      }
    } else if (wid < K) {
      // forward result of block wid of the segment (published tagged)
      const int i = wid;
      double v0 = 0.0, v1 = 0.0;
      if (i < kb) {
        const int rb = blk(q0 + i) * B;
        const int c0 = rb + lane, c1 = rb + 32 + lane;
        bool ok0 = c0 >= n, ok1 = c1 >= n;
        while (true) {
          if (!ok0) ok0 = tget(io.tin + c0, io.tin_tag, v0);
          if (!ok1) ok1 = tget(io.tin + c1, io.tin_tag, v1);
          if (__all_sync(0xffffffffu, ok0 && ok1)) break;
        }
        if (c0 >= n) v0 = 0.0;
        if (c1 >= n) v1 = 0.0;
      }
      T[i * B + lane] = v0;
      T[i * B + 32 + lane] = v1;
    }
    if (threadIdx.x == 0) *ycount = 0;
    if (io.stamps != nullptr && threadIdx.x == 0) io.stamps[8 * s] = gtimer();
    // ---- factor tiles of earlier blocks: cp.async ring, PD - 1 columns ahead
    auto issue_col = [&](int qc) {
      if (qc < q0) {
        TF* dst = Lr + (size_t)(qc % PD) * R * B;
        const int cb = blk(qc) * B;
        for (int e = threadIdx.x; e < R * EPR; e += NT) {
          const int sl = e / EPR, pc = e % EPR;
          const int gr = grow_of(sl);
          void* d = dst + (size_t)sl * B + pc * (16 / sizeof(TF));
          if ((sl / B) < kb && gr < n)
            cp16(d, LU + (size_t)gr * io.ldf + cb + pc * (16 / sizeof(TF)));
          else
            *reinterpret_cast<uint4*>(d) = make_uint4(0, 0, 0, 0);
        }
      }
      cp_commit();
    };
#pragma unroll
    for (int p = 0; p < PD - 1; ++p) issue_col(p);
    double acc[RIT], acc2[RIT];
#pragma unroll
    for (int it = 0; it < RIT; ++it) acc[it] = acc2[it] = 0.0;
    __syncthreads();
    for (int qc = 0; qc < q0; ++qc) {
      // stage published blocks: warp 0 polls up to PB blocks per round trip
      if (wid == 0 && *((volatile int*)ycount) <= qc) {
        // at most PB blocks per round trip while catching up; at the frontier
        // only the next block is polled, and owners whose own segment is far
        // ahead back off in proportion (the frontier's tags are polled by
        // every owner ahead of it: keep that L2 traffic low)
        int have = qc, width = PB;
        for (;;) {
          const int nq = min(width, q0 - have);
          double v[PB][2];
          bool ok[PB];
#pragma unroll
          for (int j = 0; j < PB; ++j) {
            ok[j] = true;
            if (j < nq) {
              const int cb = blk(have + j) * B;
              const int c0 = cb + lane, c1 = cb + 32 + lane;
              bool a = c0 >= n || tget(io.tout + c0, io.tag, v[j][0]);
              bool b = c1 >= n || tget(io.tout + c1, io.tag, v[j][1]);
              if (c0 >= n) v[j][0] = 0.0;
              if (c1 >= n) v[j][1] = 0.0;
              ok[j] = a && b;
            }
          }
          int got = 0;
#pragma unroll
          for (int j = 0; j < PB; ++j) {
            const bool all = __all_sync(0xffffffffu, ok[j]) && j < nq;
            if (all && got == j) {
              double* ys = Yr + (size_t)((have + j) % PY) * B;
              ys[lane] = v[j][0];
              ys[32 + lane] = v[j][1];
              got = j + 1;
            }
          }
          have += got;
          if (got > 0) break;
          width = 1;
          const int dist = q0 - have;  // blocks between the frontier and this segment
          if (dist > K) __nanosleep(GB_SEG_SLEEP);
        }
        __syncwarp();
        if (lane == 0) *((volatile int*)ycount) = have;
        if (io.stamps != nullptr && lane == 0 && have == q0) io.stamps[8 * s + 4] = gtimer();  // last block seen
      }
      cp_wait<PD - 2>();
      __syncthreads();
      if (io.stamps != nullptr && threadIdx.x == 0 && qc == q0 - 1) io.stamps[8 * s + 5] = gtimer();
      issue_col(qc + PD - 1);  // into the slot consumed at qc - 1
      const double* ys = Yr + (size_t)(qc % PY) * B;
      const TF* tile = Lr + (size_t)(qc % PD) * R * B;
      double yv[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) yv[e] = ys[8 * cg + e];
#pragma unroll
      for (int it = 0; it < RIT; ++it) {
        const int sl = (it * 8 + wid) * 4 + rg;
        Pack8<TF> pk;
#pragma unroll
        for (int z = 0; z < (int)(sizeof(TF) / 2); ++z)
          pk.q[z] = reinterpret_cast<const uint4*>(tile + (size_t)sl * B + 8 * cg)[z];
        double d[8];
        unpack8<TF>(pk, d);
#pragma unroll
        for (int e = 0; e < 8; e += 2) {
          acc[it] = __fma_rn(d[e], yv[e], acc[it]);
          acc2[it] = __fma_rn(d[e + 1], yv[e + 1], acc2[it]);
        }
      }
    }
    cp_wait<0>();
    if (io.stamps != nullptr && threadIdx.x == 0) io.stamps[8 * s + 1] = gtimer();
    // ---- row sums over the 8 lanes of a row (fixed butterfly)
#pragma unroll
    for (int it = 0; it < RIT; ++it) {
      double a = __dadd_rn(acc[it], acc2[it]);
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) a = __dadd_rn(a, __shfl_xor_sync(0xffffffffu, a, o));
      if (cg == 0) S[(it * 8 + wid) * 4 + rg] = a;
    }
    __syncthreads();
    if (io.stamps != nullptr && threadIdx.x == 0) io.stamps[8 * s + 2] = gtimer();
    // ---- local solve of the K blocks
    double* Y = Yr;  // reuse ring slot 0 for the block just solved
#pragma unroll
    for (int i = 0; i < K; ++i) {
      if (i >= kb) break;
      // x = t - S over the block's 64 rows (smem), then y = D^-1 x: thread
      // (rr, qq) sums columns 4 cc + qq in four short chains
      const double* drow = DI + (size_t)i * B * TP + rr * TP;
      double a[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int cc = 0; cc < 16; ++cc) {
        const int c = 4 * cc + qq;
        a[cc & 3] = __fma_rn(drow[c], __dsub_rn(T[i * B + c], S[i * B + c]), a[cc & 3]);
      }
      double yv = __dadd_rn(__dadd_rn(a[0], a[1]), __dadd_rn(a[2], a[3]));
      yv = __dadd_rn(yv, __shfl_xor_sync(0xffffffffu, yv, 1));
      yv = __dadd_rn(yv, __shfl_xor_sync(0xffffffffu, yv, 2));
      if (kLower) yv = __dadd_rn(yv, __dsub_rn(T[i * B + rr], S[i * B + rr]));  // unit diagonal
      const int gr = blk(q0 + i) * B + rr;
      if (qq == 0) {
        Y[rr] = yv;
        if (gr < n) {
          tput(io.tout + gr, yv, io.tag);
          out(gr, yv);
        }
      }
      if (i + 1 >= kb) {
        if (io.stamps != nullptr && threadIdx.x == 0) io.stamps[8 * s + 3] = gtimer();
        break;
      }
      __syncthreads();
      // update the later blocks of the segment: S[i2] += L_{i2, i} y_i
      int p = 0;
#pragma unroll
      for (int ia = 0; ia < K; ++ia)
#pragma unroll
        for (int ib = ia + 1; ib < K; ++ib, ++p) {
          if (ia != i || ib >= kb) continue;
          const double* tile = TI + (size_t)p * B * TP + rr * TP;
          double u4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
          for (int cc = 0; cc < 16; ++cc) {
            const int c = 4 * cc + qq;
            u4[cc & 3] = __fma_rn(tile[c], Y[c], u4[cc & 3]);
          }
          double u = __dadd_rn(__dadd_rn(u4[0], u4[1]), __dadd_rn(u4[2], u4[3]));
          u = __dadd_rn(u, __shfl_xor_sync(0xffffffffu, u, 1));
          u = __dadd_rn(u, __shfl_xor_sync(0xffffffffu, u, 2));
          if (qq == 0) S[ib * B + rr] = __dadd_rn(S[ib * B + rr], u);
        }
      __syncthreads();
    }
    __syncthreads();
  }
}


// ---------------------------------------------------------------------------
// One block per owner, two-deep look-ahead (y_b of a 64-row block b, sweep
// order q; "b-1", "b-2" are the previous blocks in sweep order):
//   y_b = D_b^-1 (t_b - far_b - P_{b-2 -> b}) - M_b y_{b-1}
//   * far_b: products of every earlier block but the last two, pulled by
//     this owner tile column by tile column as they are published;
//   * P_{b-2 -> b} = L_{b, b-2} y_{b-2}: computed and pushed by the owner of
//     b-2 right after it published y_{b-2};
//   * M_b = D_b^-1 L_{b, b-1}: the folded neighbour block (k_diag_fold_b).
// After y_{b-1} lands the chain is one 64 x 64 product and the publish; the
// owner's far field and the pushed product both have one extra link of slack.
// ---------------------------------------------------------------------------
__host__ __device__ constexpr size_t sweep2_smem(size_t tf_bytes) {
  return (size_t)(PY * B + 3 * B + 3 * B * TP) * sizeof(double) + (size_t)PD * B * B * tf_bytes + 64;
}

struct SweepIO2 {
  SweepIO io;
  uint4* pout;  // tagged pushed products P_{b-2 -> b}, indexed by the rows of b (this sweep's tag)
};

template <class TF, bool kLower, class Team, class Out>
__device__ __noinline__ void sweep2(Team& t, const SweepIO2 io2, void* smem_raw, Out out) {
  const SweepIO& io = io2.io;
  constexpr int RIT = B / 32;
  constexpr int EPR = B * sizeof(TF) / 16;
  const int n = io.n;
  const int nb = (n + B - 1) / B;
  const int G = t.size();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int rg = lane >> 3, cg = lane & 7;
  const int rr = threadIdx.x >> 2, qq = threadIdx.x & 3;
  const TF* LU = reinterpret_cast<const TF*>(io.LU);
  double* Yr = reinterpret_cast<double*>(smem_raw);  // [PY][B]
  double* T = Yr + PY * B;                            // [B] rhs
  double* S = T + B;                                  // [B] far-field row sums
  double* Y = S + B;                                  // [B] this block's solution
  double* DI = Y + B;                                 // [B][TP] D^-1 (row-major)
  double* MI = DI + B * TP;                           // [B][TP] M
  double* P2 = MI + B * TP;                           // [B][TP] L_{b+2, b} (rows of the block two ahead)
  TF* Lr = reinterpret_cast<TF*>(P2 + B * TP);        // [PD][B][B]
  int* ycount = reinterpret_cast<int*>(Lr + (size_t)PD * B * B);
  auto blk = [&](int q) { return kLower ? q : nb - 1 - q; };
  for (int q0 = t.rank(); q0 < nb; q0 += G) {
    const int b = blk(q0);
    const int r0 = b * B;
    const double* rec = io.inv + (size_t)b * 2 * B * B;
    const bool ahead = q0 + 2 < nb;
    const int ra = ahead ? blk(q0 + 2) * B : 0;  // rows of the block two ahead
    for (int e = threadIdx.x; e < B * B; e += NT) {
      DI[(e % B) * TP + e / B] = __ldg(rec + e);
      MI[(e / B) * TP + e % B] = q0 > 0 ? __ldg(rec + B * B + e) : 0.0;
      const int r = e / B, c = e % B;
      P2[r * TP + c] = (ahead && ra + r < n && r0 + c < n) ? f2d<TF>(LU[(size_t)(ra + r) * io.ldf + r0 + c]) : 0.0;
    }
    if (kLower) {
      for (int r = threadIdx.x; r < B; r += NT) T[r] = (r0 + r < n) ? io.rhs[r0 + r] : 0.0;
    } else if (wid == 0) {
      double v0 = 0.0, v1 = 0.0;
      const int c0 = r0 + lane, c1 = r0 + 32 + lane;
      bool ok0 = c0 >= n, ok1 = c1 >= n;
      while (!__all_sync(0xffffffffu, ok0 && ok1)) {
        if (!ok0) ok0 = tget(io.tin + c0, io.tin_tag, v0);
        if (!ok1) ok1 = tget(io.tin + c1, io.tin_tag, v1);
      }
      T[lane] = c0 < n ? v0 : 0.0;
      T[32 + lane] = c1 < n ? v1 : 0.0;
    }
    if (threadIdx.x == 0) *ycount = 0;
    if (io.stamps != nullptr && threadIdx.x == 0) io.stamps[8 * q0] = gtimer();
    const int nfar = q0 > 1 ? q0 - 2 : 0;  // pulled columns: all but the last two blocks
    auto issue_col = [&](int qc) {
      if (qc < nfar) {
        TF* dst = Lr + (size_t)(qc % PD) * B * B;
        const int cb = blk(qc) * B;
        for (int e = threadIdx.x; e < B * EPR; e += NT) {
          const int sl = e / EPR, pc = e % EPR;
          void* d = dst + (size_t)sl * B + pc * (16 / sizeof(TF));
          if (r0 + sl < n)
            cp16(d, LU + (size_t)(r0 + sl) * io.ldf + cb + pc * (16 / sizeof(TF)));
          else
            *reinterpret_cast<uint4*>(d) = make_uint4(0, 0, 0, 0);
        }
      }
      cp_commit();
    };
#pragma unroll
    for (int p = 0; p < PD - 1; ++p) issue_col(p);
    double acc[RIT], acc2[RIT];
#pragma unroll
    for (int it = 0; it < RIT; ++it) acc[it] = acc2[it] = 0.0;
    __syncthreads();
    for (int qc = 0; qc < nfar; ++qc) {
      if (wid == 0 && *((volatile int*)ycount) <= qc) {
        int have = qc, width = PB;
        for (;;) {
          const int nq = min(width, nfar - have);
          double v[PB][2];
          bool ok[PB];
#pragma unroll
          for (int j = 0; j < PB; ++j) {
            ok[j] = true;
            if (j < nq) {
              const int cb = blk(have + j) * B;
              const int c0 = cb + lane, c1 = cb + 32 + lane;
              bool a = c0 >= n || tget(io.tout + c0, io.tag, v[j][0]);
              bool bb = c1 >= n || tget(io.tout + c1, io.tag, v[j][1]);
              if (c0 >= n) v[j][0] = 0.0;
              if (c1 >= n) v[j][1] = 0.0;
              ok[j] = a && bb;
            }
          }
          int got = 0;
#pragma unroll
          for (int j = 0; j < PB; ++j) {
            const bool all = __all_sync(0xffffffffu, ok[j]) && j < nq;
            if (all && got == j) {
              double* ys = Yr + (size_t)((have + j) % PY) * B;
              ys[lane] = v[j][0];
              ys[32 + lane] = v[j][1];
              got = j + 1;
            }
          }
          have += got;
          if (got > 0) break;
          width = 1;
          __nanosleep(min(GB_SEG_SLEEP, GB_SEG_FAR_NS * (q0 - have - 2)));
        }
        __syncwarp();
        if (lane == 0) *((volatile int*)ycount) = have;
      }
      cp_wait<PD - 2>();
      __syncthreads();
      issue_col(qc + PD - 1);
      const double* ys = Yr + (size_t)(qc % PY) * B;
      const TF* tile = Lr + (size_t)(qc % PD) * B * B;
      double yv[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) yv[e] = ys[8 * cg + e];
#pragma unroll
      for (int it = 0; it < RIT; ++it) {
        const int sl = (it * 8 + wid) * 4 + rg;
        Pack8<TF> pk;
#pragma unroll
        for (int z = 0; z < (int)(sizeof(TF) / 2); ++z)
          pk.q[z] = reinterpret_cast<const uint4*>(tile + (size_t)sl * B + 8 * cg)[z];
        double d[8];
        unpack8<TF>(pk, d);
#pragma unroll
        for (int e = 0; e < 8; e += 2) {
          acc[it] = __fma_rn(d[e], yv[e], acc[it]);
          acc2[it] = __fma_rn(d[e + 1], yv[e + 1], acc2[it]);
        }
      }
    }
    cp_wait<0>();
#pragma unroll
    for (int it = 0; it < RIT; ++it) {
      double a = __dadd_rn(acc[it], acc2[it]);
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) a = __dadd_rn(a, __shfl_xor_sync(0xffffffffu, a, o));
      if (cg == 0) S[(it * 8 + wid) * 4 + rg] = a;
    }
    __syncthreads();
    if (io.stamps != nullptr && threadIdx.x == 0) io.stamps[8 * q0 + 5] = gtimer();
    // the product pushed by the owner of b-2: warp 0 polls, the CTA reads smem
    // (ring slots PY-1 / PY-2 are not used by the far field of this block)
    double* Pp = Yr + (size_t)(PY - 1) * B;
    double* Yp = Yr + (size_t)(PY - 2) * B;
    if (wid == 0) {
      double p0 = 0.0, p1 = 0.0;
      if (q0 >= 2) {
        const int c0 = r0 + lane, c1 = r0 + 32 + lane;
        bool ok0 = c0 >= n, ok1 = c1 >= n;
        while (!__all_sync(0xffffffffu, ok0 && ok1)) {
          if (!ok0) ok0 = tget(io2.pout + c0, io.tag, p0);
          if (!ok1) ok1 = tget(io2.pout + c1, io.tag, p1);
        }
      }
      Pp[lane] = p0;
      Pp[32 + lane] = p1;
    }
    __syncthreads();
    // pre = D^-1 (t - far - P) (+ the unit diagonal in the lower sweep)
    double pre;
    {
      const double* drow = DI + rr * TP;
      double a[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int cc = 0; cc < 16; ++cc) {
        const int c = 4 * cc + qq;
        a[cc & 3] = __fma_rn(drow[c], __dsub_rn(__dsub_rn(T[c], S[c]), Pp[c]), a[cc & 3]);
      }
      pre = __dadd_rn(__dadd_rn(a[0], a[1]), __dadd_rn(a[2], a[3]));
      pre = __dadd_rn(pre, __shfl_xor_sync(0xffffffffu, pre, 1));
      pre = __dadd_rn(pre, __shfl_xor_sync(0xffffffffu, pre, 2));
      if (kLower) {
        pre = __dadd_rn(pre, __dsub_rn(__dsub_rn(T[rr], S[rr]), Pp[rr]));
      }
    }
    if (io.stamps != nullptr && threadIdx.x == 0) io.stamps[8 * q0 + 1] = gtimer();
    double yb = pre;
    if (q0 > 0) {
      // the hand-off: warp 0 polls the previous block, the CTA reads smem
      if (wid == 0) {
        const int cb = blk(q0 - 1) * B;
        double v0 = 0.0, v1 = 0.0;
        const int c0 = cb + lane, c1 = cb + 32 + lane;
        bool ok0 = c0 >= n, ok1 = c1 >= n;
        while (!__all_sync(0xffffffffu, ok0 && ok1)) {
          if (!ok0) ok0 = tget(io.tout + c0, io.tag, v0);
          if (!ok1) ok1 = tget(io.tout + c1, io.tag, v1);
        }
        Yp[lane] = v0;
        Yp[32 + lane] = v1;
        if (io.stamps != nullptr && lane == 0) io.stamps[8 * q0 + 4] = gtimer();
      }
      __syncthreads();
      const double* mrow = MI + rr * TP;
      double a[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int cc = 0; cc < 16; ++cc) {
        const int c = 4 * cc + qq;
        a[cc & 3] = __fma_rn(mrow[c], Yp[c], a[cc & 3]);
      }
      double z = __dadd_rn(__dadd_rn(a[0], a[1]), __dadd_rn(a[2], a[3]));
      z = __dadd_rn(z, __shfl_xor_sync(0xffffffffu, z, 1));
      z = __dadd_rn(z, __shfl_xor_sync(0xffffffffu, z, 2));
      yb = __dsub_rn(pre, z);
    }
    if (qq == 0) {
      Y[rr] = yb;
      if (r0 + rr < n) {
        tput(io.tout + r0 + rr, yb, io.tag);
        out(r0 + rr, yb);
      }
    }
    if (io.stamps != nullptr && threadIdx.x == 0) io.stamps[8 * q0 + 3] = gtimer();
    __syncthreads();
    // push P_{b -> b+2} = L_{b+2, b} y_b to the owner of the block two ahead
    if (ahead) {
      const double* prow = P2 + rr * TP;
      double a[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int cc = 0; cc < 16; ++cc) {
        const int c = 4 * cc + qq;
        a[cc & 3] = __fma_rn(prow[c], Y[c], a[cc & 3]);
      }
      double z = __dadd_rn(__dadd_rn(a[0], a[1]), __dadd_rn(a[2], a[3]));
      z = __dadd_rn(z, __shfl_xor_sync(0xffffffffu, z, 1));
      z = __dadd_rn(z, __shfl_xor_sync(0xffffffffu, z, 2));
      if (qq == 0 && ra + rr < n) tput(io2.pout + ra + rr, z, io.tag);
    }
    __syncthreads();
  }
}


// ---------------------------------------------------------------------------
// Bulk-synchronous blocked substitution with explicit inverses of large
// diagonal blocks (NB rows, e.g. 1024): per block K of the sweep
//   (1) y_K = D_K^-1 s_K          one warp per row, fp64 row of D_K^-1
//   (2) s_J -= F_{J,K} y_K         every later block J (rows of the factor,
//                                  one warp per row, u_f entries)
// with a team barrier after each phase.  The dependency chain is n / NB
// links of two barriers instead of n / 64 cross-SM hand-offs; the inverse
// rows (NB x NB fp64 per block, built once per factorisation by
// k_bigblock_inverse) add NB / (2 b_f n) ... (NB / n) * 8 / b_f of the factor
// traffic.  ybuf: in = right-hand side, scratch for s; ysol: the solution.
// ---------------------------------------------------------------------------
template <class TF, bool kLower, class Team, class Out>
__device__ __noinline__ void sweep_bsp(Team& t, int n, int NB, const TF* __restrict__ LU, size_t ldf,
                                      const double* __restrict__ dinv, double* ybuf, double* ysol, Out out,
                                      void* smem_raw) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int W = t.size() * (NT / 32);
  const int gw = t.rank() * (NT / 32) + wid;
  const int nK = (n + NB - 1) / NB;
  double* vs = reinterpret_cast<double*>(smem_raw);  // [NB]: s_K, then y_K
  for (int it = 0; it < nK; ++it) {
    const int K = kLower ? it : nK - 1 - it;
    const int r0 = K * NB, m = min(NB, n - r0);
    const double* D = dinv + (size_t)K * NB * NB;
    // (1) y_K = D_K^-1 s_K (triangular: lower rows use c <= r, upper c >= r)
    for (int c = threadIdx.x; c < NB; c += NT) vs[c] = c < m ? __ldcg(ybuf + r0 + c) : 0.0;
    __syncthreads();
    for (int r = gw; r < m; r += W) {
      const double2* drow = reinterpret_cast<const double2*>(D + (size_t)r * NB);
      const int v0 = kLower ? 0 : (r >> 1), v1 = kLower ? (r >> 1) + 1 : (m + 1) >> 1;  // double2 range
      double a[4] = {0.0, 0.0, 0.0, 0.0};
      for (int base = v0 + lane; base < v1; base += 32 * 16) {
        double2 d2[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int v = base + 32 * u;
          d2[u] = v < v1 ? __ldg(drow + v) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int v = base + 32 * u;
          if (v < v1) {
            a[u & 1] = __fma_rn(d2[u].x, vs[2 * v], a[u & 1]);
            a[2 + (u & 1)] = __fma_rn(d2[u].y, vs[2 * v + 1], a[2 + (u & 1)]);
          }
        }
      }
      double s = __dadd_rn(__dadd_rn(a[0], a[1]), __dadd_rn(a[2], a[3]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
      if (lane == 0) {
        ysol[r0 + r] = s;
        out(r0 + r, s);
      }
    }
    t.sync();
    if (it + 1 == nK) break;
    // (2) every later row: s_r -= sum_c F[r][r0 + c] y_K[c], c over the block
    for (int c = threadIdx.x; c < NB; c += NT) vs[c] = c < m ? __ldcg(ysol + r0 + c) : 0.0;
    __syncthreads();
    const int lo = kLower ? r0 + m : 0, hi = kLower ? n : r0;
    constexpr int VW = 16 / sizeof(TF);
    const int nv = (m + VW - 1) / VW;
    // two rows per warp pass, up to 8 x 16 B per row and lane in flight
    if (nv <= 32 * 8) {
      // one batch per row pair: software-pipelined, the next pair's 16 loads
      // per lane are issued before this pair's conversions and FMAs (a pass
      // is ~1.8 us of issue time on top of ~2 us of DRAM latency otherwise)
      uint4 q0[8], q1[8];
      auto load_pair = [&](int r, uint4 (&x0)[8], uint4 (&x1)[8]) {
        const bool two = r + W < hi;
        const uint4* f0 = reinterpret_cast<const uint4*>(LU + (size_t)r * ldf + r0);
        const uint4* f1 = reinterpret_cast<const uint4*>(LU + (size_t)(two ? r + W : r) * ldf + r0);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int v = lane + 32 * u;
          x0[u] = v < nv ? __ldg(f0 + v) : make_uint4(0, 0, 0, 0);
          x1[u] = (v < nv && two) ? __ldg(f1 + v) : make_uint4(0, 0, 0, 0);
        }
      };
      int r = lo + gw;
      if (r < hi) load_pair(r, q0, q1);
      for (; r < hi; r += 2 * W) {
        const bool two = r + W < hi;
        uint4 n0[8], n1[8];
        const bool more = r + 2 * W < hi;
        if (more) load_pair(r + 2 * W, n0, n1);
        double a[4] = {0.0, 0.0, 0.0, 0.0}, b[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int v = lane + 32 * u;
          if (v < nv) {
            const TF* e0 = reinterpret_cast<const TF*>(&q0[u]);
            const TF* e1 = reinterpret_cast<const TF*>(&q1[u]);
#pragma unroll
            for (int j = 0; j < VW; ++j) {
              const double y = vs[v * VW + j];
              a[j & 3] = __fma_rn(f2d<TF>(e0[j]), y, a[j & 3]);
              b[j & 3] = __fma_rn(f2d<TF>(e1[j]), y, b[j & 3]);
            }
          }
        }
        double s0 = __dadd_rn(__dadd_rn(a[0], a[1]), __dadd_rn(a[2], a[3]));
        double s1 = __dadd_rn(__dadd_rn(b[0], b[1]), __dadd_rn(b[2], b[3]));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          s0 = __dadd_rn(s0, __shfl_xor_sync(0xffffffffu, s0, o));
          s1 = __dadd_rn(s1, __shfl_xor_sync(0xffffffffu, s1, o));
        }
        if (lane == 0) {
          ybuf[r] = __dsub_rn(ybuf[r], s0);
          if (two) ybuf[r + W] = __dsub_rn(ybuf[r + W], s1);
        }
        if (more) {
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            q0[u] = n0[u];
            q1[u] = n1[u];
          }
        }
      }
    } else
    for (int r = lo + gw; r < hi; r += 2 * W) {
      const bool two = r + W < hi;
      const uint4* f0 = reinterpret_cast<const uint4*>(LU + (size_t)r * ldf + r0);
      const uint4* f1 = reinterpret_cast<const uint4*>(LU + (size_t)(two ? r + W : r) * ldf + r0);
      double a[4] = {0.0, 0.0, 0.0, 0.0}, b[4] = {0.0, 0.0, 0.0, 0.0};
      for (int base = lane; base < nv; base += 32 * 8) {
        uint4 q0[8], q1[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int v = base + 32 * u;
          q0[u] = v < nv ? __ldg(f0 + v) : make_uint4(0, 0, 0, 0);
          q1[u] = (v < nv && two) ? __ldg(f1 + v) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int v = base + 32 * u;
          if (v < nv) {
            const TF* e0 = reinterpret_cast<const TF*>(&q0[u]);
            const TF* e1 = reinterpret_cast<const TF*>(&q1[u]);
#pragma unroll
            for (int j = 0; j < VW; ++j) {
              const double y = vs[v * VW + j];
              a[j & 3] = __fma_rn(f2d<TF>(e0[j]), y, a[j & 3]);
              b[j & 3] = __fma_rn(f2d<TF>(e1[j]), y, b[j & 3]);
            }
          }
        }
      }
      double s0 = __dadd_rn(__dadd_rn(a[0], a[1]), __dadd_rn(a[2], a[3]));
      double s1 = __dadd_rn(__dadd_rn(b[0], b[1]), __dadd_rn(b[2], b[3]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        s0 = __dadd_rn(s0, __shfl_xor_sync(0xffffffffu, s0, o));
        s1 = __dadd_rn(s1, __shfl_xor_sync(0xffffffffu, s1, o));
      }
      if (lane == 0) {
        ybuf[r] = __dsub_rn(ybuf[r], s0);
        if (two) ybuf[r + W] = __dsub_rn(ybuf[r + W], s1);
      }
    }
    t.sync();
  }
}

// ---------------------------------------------------------------------------
// Look-ahead form of sweep_bsp (same arithmetic, same per-row summation order,
// so bit-identical results): after y_K is known only the rows of the NEXT
// block are updated before the barrier (phase A, NB rows); the solve of that
// block, y_{K+1} = D_{K+1}^-1 s_{K+1}, then runs in the same phase as the
// update of all the later rows with y_K (phase B), which hides the
// latency-bound triangular product behind the streamed panel.
// smem: 2 NB doubles (y_K | s_{K+1}).
// ---------------------------------------------------------------------------
template <bool kLower>
GB_DEVICE double bsp_diag_row(const double* __restrict__ D, int NB, int r, int m, const double* vs, int lane) {
  const double2* drow = reinterpret_cast<const double2*>(D + (size_t)r * NB);
  const int v0 = kLower ? 0 : (r >> 1), v1 = kLower ? (r >> 1) + 1 : (m + 1) >> 1;  // double2 range
  double a[4] = {0.0, 0.0, 0.0, 0.0};
  for (int base = v0 + lane; base < v1; base += 32 * 16) {
    double2 d2[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int v = base + 32 * u;
      d2[u] = v < v1 ? __ldg(drow + v) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int v = base + 32 * u;
      if (v < v1) {
        a[u & 1] = __fma_rn(d2[u].x, vs[2 * v], a[u & 1]);
        a[2 + (u & 1)] = __fma_rn(d2[u].y, vs[2 * v + 1], a[2 + (u & 1)]);
      }
    }
  }
  double s = __dadd_rn(__dadd_rn(a[0], a[1]), __dadd_rn(a[2], a[3]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
  return s;
}

// s[r] -= F[r][c0 .. c0+m) . y  for rows r and (two ? r2 : none); vs = y in smem
template <class TF>
GB_DEVICE void bsp_update_rows(const TF* __restrict__ LU, size_t ldf, int c0, int m, int r, int r2, bool two,
                               const double* vs, double* ybuf, int lane) {
  constexpr int VW = 16 / sizeof(TF);
  const int nv = (m + VW - 1) / VW;
  const uint4* f0 = reinterpret_cast<const uint4*>(LU + (size_t)r * ldf + c0);
  const uint4* f1 = reinterpret_cast<const uint4*>(LU + (size_t)(two ? r2 : r) * ldf + c0);
  double a[4] = {0.0, 0.0, 0.0, 0.0}, b[4] = {0.0, 0.0, 0.0, 0.0};
  for (int base = lane; base < nv; base += 32 * 8) {
    uint4 q0[8], q1[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int v = base + 32 * u;
      q0[u] = v < nv ? __ldg(f0 + v) : make_uint4(0, 0, 0, 0);
      q1[u] = (v < nv && two) ? __ldg(f1 + v) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int v = base + 32 * u;
      if (v < nv) {
        const TF* e0 = reinterpret_cast<const TF*>(&q0[u]);
        const TF* e1 = reinterpret_cast<const TF*>(&q1[u]);
#pragma unroll
        for (int j = 0; j < VW; ++j) {
          const double y = vs[v * VW + j];
          a[j & 3] = __fma_rn(f2d<TF>(e0[j]), y, a[j & 3]);
          b[j & 3] = __fma_rn(f2d<TF>(e1[j]), y, b[j & 3]);
        }
      }
    }
  }
  double s0 = __dadd_rn(__dadd_rn(a[0], a[1]), __dadd_rn(a[2], a[3]));
  double s1 = __dadd_rn(__dadd_rn(b[0], b[1]), __dadd_rn(b[2], b[3]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s0 = __dadd_rn(s0, __shfl_xor_sync(0xffffffffu, s0, o));
    s1 = __dadd_rn(s1, __shfl_xor_sync(0xffffffffu, s1, o));
  }
  if (lane == 0) {
    ybuf[r] = __dsub_rn(ybuf[r], s0);
    if (two) ybuf[r2] = __dsub_rn(ybuf[r2], s1);
  }
}

template <class TF, bool kLower, class Team, class Out>
__device__ __noinline__ void sweep_la(Team& t, int n, int NB, const TF* __restrict__ LU, size_t ldf,
                                     const double* __restrict__ dinv, double* ybuf, double* ysol, Out out,
                                     void* smem_raw) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int W = t.size() * (NT / 32);
  const int gw = t.rank() * (NT / 32) + wid;
  const int nK = (n + NB - 1) / NB;
  double* vy = reinterpret_cast<double*>(smem_raw);  // [NB]: y_K
  double* vs = vy + NB;                              // [NB]: s_{K+1}
  auto blk = [&](int it) { return kLower ? it : nK - 1 - it; };
  auto solve_block = [&](int K) {
    const int r0 = K * NB, m = min(NB, n - r0);
    const double* D = dinv + (size_t)K * NB * NB;
    for (int r = gw; r < m; r += W) {
      const double s = bsp_diag_row<kLower>(D, NB, r, m, vs, lane);
      if (lane == 0) {
        ysol[r0 + r] = s;
        out(r0 + r, s);
      }
    }
  };
  // prologue: first block of the sweep
  {
    const int K = blk(0), r0 = K * NB, m = min(NB, n - r0);
    for (int c = threadIdx.x; c < NB; c += NT) vs[c] = c < m ? __ldcg(ybuf + r0 + c) : 0.0;
    __syncthreads();
    solve_block(K);
    t.sync();
  }
  for (int it = 0; it + 1 < nK; ++it) {
    const int K = blk(it), K1 = blk(it + 1);
    const int r0 = K * NB, m = min(NB, n - r0);
    const int q0 = K1 * NB, mq = min(NB, n - q0);
    for (int c = threadIdx.x; c < NB; c += NT) vy[c] = c < m ? __ldcg(ysol + r0 + c) : 0.0;
    __syncthreads();
    // phase A: the next block's rows
    for (int r = gw; r < mq; r += 2 * W) {
      const bool two = r + W < mq;
      bsp_update_rows<TF>(LU, ldf, r0, m, q0 + r, q0 + r + W, two, vy, ybuf, lane);
    }
    t.sync();
    // phase B: solve the next block | update every later row with y_K
    for (int c = threadIdx.x; c < NB; c += NT) vs[c] = c < mq ? __ldcg(ybuf + q0 + c) : 0.0;
    __syncthreads();
    solve_block(K1);
    const int lo = kLower ? q0 + mq : 0, hi = kLower ? n : q0;
    // rotate the warp numbering past the warps that took a second solve row
    const int rot = mq % W;
    const int gw2 = (gw + W - rot) % W;
    for (int r = lo + gw2; r < hi; r += 2 * W) {
      const bool two = r + W < hi;
      bsp_update_rows<TF>(LU, ldf, r0, m, r, r + W, two, vy, ybuf, lane);
    }
    t.sync();
  }
}

// D_K^-1 for the NB x NB diagonal blocks of the unit lower (kLower) or upper
// factor, row-major fp64, one warp per column: forward (backward)
// substitution of e_c with warp-parallel dot products, the column kept in
// shared memory.  Launch: grid = any, 256 threads, smem = 8 warps * NB * 8 B.
template <class TF, bool kLower>
__global__ void __launch_bounds__(256) k_bigblock_inverse(const TF* __restrict__ LU, size_t ldf, int n, int NB,
                                                          double* dinv) {
  extern __shared__ double colbuf[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* x = colbuf + (size_t)wid * NB;
  const int nK = (n + NB - 1) / NB;
  const long total = (long)nK * NB;
  for (long job = (long)blockIdx.x * 8 + wid; job < total; job += (long)gridDim.x * 8) {
    const int K = (int)(job / NB), c = (int)(job % NB);
    const int r0 = K * NB, m = min(NB, n - r0);
    double* D = dinv + (size_t)K * NB * NB;
    if (c >= m) {
      for (int r = lane; r < NB; r += 32) D[(size_t)r * NB + c] = 0.0;
      continue;
    }
    for (int r = lane; r < NB; r += 32) x[r] = 0.0;
    __syncwarp();
    if (kLower) {
      if (lane == 0) x[c] = 1.0;
      __syncwarp();
      for (int r = c + 1; r < m; ++r) {
        const TF* frow = LU + (size_t)(r0 + r) * ldf + r0;
        double a = 0.0;
        for (int k = c + lane; k < r; k += 32) a = __fma_rn(f2d<TF>(frow[k]), x[k], a);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a = __dadd_rn(a, __shfl_xor_sync(0xffffffffu, a, o));
        if (lane == 0) x[r] = -a;
        __syncwarp();
      }
    } else {
      if (lane == 0) x[c] = 1.0 / f2d<TF>(LU[(size_t)(r0 + c) * ldf + r0 + c]);
      __syncwarp();
      for (int r = c - 1; r >= 0; --r) {
        const TF* frow = LU + (size_t)(r0 + r) * ldf + r0;
        double a = 0.0;
        for (int k = r + 1 + lane; k <= c; k += 32) a = __fma_rn(f2d<TF>(frow[k]), x[k], a);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a = __dadd_rn(a, __shfl_xor_sync(0xffffffffu, a, o));
        if (lane == 0) x[r] = -a / f2d<TF>(frow[r]);
        __syncwarp();
      }
    }
    for (int r = lane; r < NB; r += 32) D[(size_t)r * NB + c] = x[r];
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// GEMV phase: t[i] = sum_j A[perm[i], j] v[j] (fp64 accumulation), rows in
// perm order dealt round-robin over the team's CTAs.  Each CTA streams its
// rows through an NS-stage ring of GCH-byte bulk copies (one thread issues;
// one mbarrier per stage, expect_tx), v is staged once as fp64 in shared
// memory.  Thread q owns the 16-B vectors q, q + 256, ... of every chunk; its
// partial sums are reduced per row in a fixed order (deterministic).
// ---------------------------------------------------------------------------
// LDG variant: one warp per row (perm order over all warps of the team),
// U 16-B loads in flight per lane, v staged as fp64 in shared memory
template <class TA, class TV, int kConv, int U = 8, bool kSkew = false, class Team>
__device__ __noinline__ void gemv_ldg(Team& t, int n, const TA* __restrict__ A, size_t lda,
                                      const int* __restrict__ perm, const TV* __restrict__ v, double* out,
                                      void* smem_raw) {
  constexpr int VW = 16 / sizeof(TA);
  double* vs = reinterpret_cast<double*>(smem_raw);
  for (int j = threadIdx.x; j < (int)(gemv_vbytes(n) / 8); j += NT) vs[j] = j < n ? (double)v[j] : 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int W = t.size() * (NT / 32);
  const int nv = (n + VW - 1) / VW;  // rows are padded to lda (zeros) and v to 16 entries
  for (int i = t.rank() * (NT / 32) + wid; i < n; i += W) {
    const uint4* row = reinterpret_cast<const uint4*>(A + (size_t)perm[i] * lda);
    double acc0 = 0.0, acc1 = 0.0;
    // rows start at staggered offsets (whole 32-vector groups), so the warps'
    // concurrent requests spread over the DRAM channels instead of marching
    // through the same row offsets in lock step
    const int ngr = (nv + 31) / 32;
    const int skew = kSkew ? (int)(((unsigned)i * 2654435761u) % (unsigned)ngr) : 0;
    for (int base = lane; base < nv; base += 32 * U) {
      uint4 q[U];
      int ix[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        int g = (base >> 5) + u + skew;
        g = g >= ngr ? g - ngr : g;
        ix[u] = (base + 32 * u < nv) ? g * 32 + lane : nv;
        const int idx = ix[u];
        if (idx < nv)
          asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(q[u].x), "=r"(q[u].y), "=r"(q[u].z), "=r"(q[u].w)
                       : "l"(row + idx));
        else
          q[u] = make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = ix[u];
        if (idx < nv) {
          if constexpr (sizeof(TA) == 4) {
            const float* a = reinterpret_cast<const float*>(&q[u]);
            const double2* vv = reinterpret_cast<const double2*>(vs + idx * VW);
            const double2 w0 = vv[0], w1 = vv[1];
            if (kConv == 1) {
              acc0 = __fma_rn(f2d_normal(a[0]), w0.x, acc0);
              acc1 = __fma_rn(f2d_normal(a[1]), w0.y, acc1);
              acc0 = __fma_rn(f2d_normal(a[2]), w1.x, acc0);
              acc1 = __fma_rn(f2d_normal(a[3]), w1.y, acc1);
            } else if (kConv == 0) {
              acc0 = __fma_rn((double)a[0], w0.x, acc0);
              acc1 = __fma_rn((double)a[1], w0.y, acc1);
              acc0 = __fma_rn((double)a[2], w1.x, acc0);
              acc1 = __fma_rn((double)a[3], w1.y, acc1);
            } else if (kConv == 3) {
              // mixed: half the elements through the conversion unit, half on the integer pipe
              acc0 = __fma_rn((double)a[0], w0.x, acc0);
              acc1 = __fma_rn(f2d_normal(a[1]), w0.y, acc1);
              acc0 = __fma_rn((double)a[2], w1.x, acc0);
              acc1 = __fma_rn(f2d_normal(a[3]), w1.y, acc1);
            } else if (kConv == 2) {
              // timing probe only (wrong values): no conversion
              const double2 b = *reinterpret_cast<const double2*>(&q[u]);
              acc0 = __fma_rn(b.x, w0.x, acc0);
              acc1 = __fma_rn(b.y, w0.y, acc1);
              acc0 = __fma_rn(b.x, w1.x, acc0);
              acc1 = __fma_rn(b.y, w1.y, acc1);
            } else {
              acc0 = __fma_rn(f2d_int(a[0]), w0.x, acc0);
              acc1 = __fma_rn(f2d_int(a[1]), w0.y, acc1);
              acc0 = __fma_rn(f2d_int(a[2]), w1.x, acc0);
              acc1 = __fma_rn(f2d_int(a[3]), w1.y, acc1);
            }
          } else {
            const double* a = reinterpret_cast<const double*>(&q[u]);
            const double2 w0 = *reinterpret_cast<const double2*>(vs + idx * VW);
            acc0 = __fma_rn(a[0], w0.x, acc0);
            acc1 = __fma_rn(a[1], w0.y, acc1);
          }
        }
      }
    }
    double s = __dadd_rn(acc0, acc1);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
    if (lane == 0) out[i] = s;
  }
}

template <class TA, class TV, bool kNormal, class Team>
__device__ __noinline__ void gemv_perm(Team& t, int n, const TA* __restrict__ A, size_t lda,
                                       const int* __restrict__ perm, const TV* __restrict__ v, double* out,
                                       void* smem_raw, int NS, const PhaseLog lg = PhaseLog{nullptr, 0, nullptr}) {
  constexpr int EPC = GCH / sizeof(TA);  // elements per chunk
  double* vs = reinterpret_cast<double*>(smem_raw);
  unsigned char* ring = reinterpret_cast<unsigned char*>(smem_raw) + gemv_vbytes(n);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(ring + (size_t)NS * GCH);
  double* red = reinterpret_cast<double*>(full + GNS_MAX);  // [8]
  int* rows = reinterpret_cast<int*>(red + 8);               // perm of this CTA's rows
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int G = t.size(), r = t.rank();
  const int nrows = min(GROWS_MAX, n > r ? (n - r + G - 1) / G : 0);  // rows r, r + G, ...
  const size_t rowbytes = ((size_t)n * sizeof(TA) + 15) & ~(size_t)15;
  const int cpr = (int)((rowbytes + GCH - 1) / GCH);  // chunks per row
  const int total = nrows * cpr;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(full + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int j = threadIdx.x; j < n; j += NT) vs[j] = (double)v[j];  // once per apply
  for (int j = n + threadIdx.x; j < (int)(gemv_vbytes(n) / 8); j += NT) vs[j] = 0.0;
  for (int i = threadIdx.x; i < nrows; i += NT) rows[i] = perm[r + i * G];
  __syncthreads();
  mark(lg, 14);
  // producer state (thread 0): next chunk to issue as (row, chunk-in-row)
  int pr = 0, pc = 0, pn = 0;
  auto issue_next = [&]() {
    const size_t off = (size_t)pc * GCH;
    const unsigned bytes = (unsigned)min((size_t)GCH, rowbytes - off);
    unsigned long long* bar = full + (pn % NS);
    mbar_expect_tx(bar, bytes);
    bulk_g2s(ring + (size_t)(pn % NS) * GCH,
             reinterpret_cast<const unsigned char*>(A + (size_t)rows[pr] * lda) + off, bytes, bar);
    ++pn;
    if (++pc == cpr) pc = 0, ++pr;
  };
  if (threadIdx.x == 0) {
    fence_async_smem();  // earlier generic-proxy accesses of the ring before the async writes
    while (pn < min(NS, total)) issue_next();
  }
  double acc0 = 0.0, acc1 = 0.0;
  int ri = 0, ci = 0, st = 0;
  unsigned ph = 0;
  for (int c = 0; c < total; ++c) {
    mbar_wait(full + st, ph);
    const int e0 = ci * EPC;
    const int ne = min(EPC, n - e0);
    if constexpr (sizeof(TA) == 4) {
      // element pairs: 8 B of A and 16 B of v per lane, contiguous across the warp
      const float2* ch = reinterpret_cast<const float2*>(ring + (size_t)st * GCH);
      const double2* vv = reinterpret_cast<const double2*>(vs + e0);
      const int np = (ne + 1) / 2;  // v is zero-padded past n
      // a full chunk is 8 pairs per thread: all 16 shared-memory loads are
      // issued before the first conversion (the warp's only latency hiding
      // at 8 warps per SM is its own ILP)
      if (np == EPC / 2) {
        float2 a2[8];
        double2 w2[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          a2[u] = ch[threadIdx.x + u * NT];
          w2[u] = vv[threadIdx.x + u * NT];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          acc0 = __fma_rn(kNormal ? f2d_normal(a2[u].x) : f2d_int(a2[u].x), w2[u].x, acc0);
          acc1 = __fma_rn(kNormal ? f2d_normal(a2[u].y) : f2d_int(a2[u].y), w2[u].y, acc1);
        }
      } else {
#pragma unroll 4
        for (int q = threadIdx.x; q < np; q += NT) {
          const float2 a2 = ch[q];
          const double2 w2 = vv[q];
          acc0 = __fma_rn(kNormal ? f2d_normal(a2.x) : f2d_int(a2.x), w2.x, acc0);
          acc1 = __fma_rn(kNormal ? f2d_normal(a2.y) : f2d_int(a2.y), w2.y, acc1);
        }
      }
    } else {
      const double* ch = reinterpret_cast<const double*>(ring + (size_t)st * GCH);
#pragma unroll 4
      for (int q = threadIdx.x; q < ne; q += NT) acc0 = __fma_rn(ch[q], vs[e0 + q], acc0);
    }
    __syncthreads();  // stage consumed by every thread
    if (threadIdx.x == 0 && pn < total) {
      fence_async_smem();
      issue_next();
    }
    if (++st == NS) st = 0, ph ^= 1u;
    if (++ci == cpr) {
      // row done: fixed-order block reduction
      double s = __dadd_rn(acc0, acc1);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
      if (lane == 0) red[wid] = s;
      __syncthreads();
      if (threadIdx.x == 0) {
        double z = 0.0;
#pragma unroll
        for (int w = 0; w < NT / 32; ++w) z = __dadd_rn(z, red[w]);
        out[r + ri * G] = z;
      }
      acc0 = acc1 = 0.0;
      ci = 0;
      ++ri;
      mark(lg, 15);
    }
  }
  __syncthreads();
  // the ring's barriers are re-initialised by the next call (the region is
  // shared with the sweeps' staging and the leader's scratch in between):
  // invalidate them first -- re-initialising a live mbarrier is undefined,
  // and a stage that has completed an odd number of phases did fault the
  // next call's first wait at n = 16384 (111 rows x 4 chunks on 5 stages)
  if (threadIdx.x == 0)
    for (int i = 0; i < NS; ++i)
      asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(full + i)) : "memory");
  __syncthreads();
  mark(lg, 16);
}

}  // namespace seg
}  // namespace gb
