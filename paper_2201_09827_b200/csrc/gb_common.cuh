// Common device helpers: formats, format-faithful rounding, double-double
// arithmetic and warp/block reductions.
//
// Semantics follow reference precision.py:
//   * round to half/single: RNE with subnormals kept (precision.py:206-232);
//     a double->float->half chain is used where the reference rounds u then u_f
//     (refine.py:285 + densela.py:131);
//   * half arithmetic: every op rounded (precision.py:9-17); done in fp32 then
//     rounded to fp16 -- fp32 has 24 >= 2*11+2 bits so the double rounding is
//     innocuous for + - * / (SURVEY F1);
//   * double-double: the accurate two-two-sum dd_add and Dekker products of
//     precision.py:239-341 (two_prod via FMA gives the identical exact error).
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

#include "../../include/gcrodr_b200.h"

#ifndef GB_DEVICE
#define GB_DEVICE __device__ __forceinline__
#endif
#define GB_HD __host__ __device__ __forceinline__

namespace gb {

// per-32-row-block record of the TRSV helpers: the dd inverse of the diagonal
// block (1024 doubles) followed by the folded neighbour block (1024 doubles)
constexpr int kInvStride = 2048;
// row-block size of the grid-team substitution trsv_cta_g
constexpr int kTrsvB = 64;
// doubles per block record of B-row blocks: inverse (B^2) + folded neighbour (B^2)
template <int B>
__host__ __device__ constexpr int inv_stride() { return 2 * B * B; }

// optional phase timers (globaltimer ns, CTA 0 thread 0); enabled per launch
// by a non-null pointer.  slot 0 = count, then pairs (tag, t).
struct PhaseLog {
  unsigned long long* buf;
  int cap;
  // post-mortem mode (host-mapped log): last[b] = (count << 32 | tag) of CTA b's latest mark
  unsigned long long* last = nullptr;
};
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void mark(const PhaseLog& L, int tag) {
  if (L.last != nullptr && threadIdx.x == 0 && blockIdx.x < 256) {
    const unsigned long long prev = L.last[blockIdx.x];
    L.last[blockIdx.x] = ((prev >> 32) + 1ull) << 32 | (unsigned long long)(unsigned)tag;
  }
  if (L.buf != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long i = L.buf[0];
    if ((int)i < L.cap) {
      L.buf[1 + 2 * i] = (unsigned long long)tag;
      L.buf[2 + 2 * i] = gtimer();
      L.buf[0] = i + 1;
    }
  }
}

// ---------------------------------------------------------------------------
// rounding
// ---------------------------------------------------------------------------

GB_DEVICE double fl32(double x) { return (double)__double2float_rn(x); }
// fp64 -> fp16 directly (numpy astype(float16) from float64 rounds once)
GB_DEVICE __half h_from_d(double x) { return __double2half(x); }
GB_DEVICE double fl16(double x) { return (double)__half2float(__double2half(x)); }
GB_DEVICE float fl16f(float x) { return __half2float(__float2half_rn(x)); }

// half-simulated elementary ops (exact IEEE binary16 results, no FMA)
GB_DEVICE float h_mul(float a, float b) { return fl16f(__fmul_rn(a, b)); }
GB_DEVICE float h_sub(float a, float b) { return fl16f(__fsub_rn(a, b)); }
GB_DEVICE float h_add(float a, float b) { return fl16f(__fadd_rn(a, b)); }
GB_DEVICE float h_div(float a, float b) { return fl16f(__fdiv_rn(a, b)); }

// ---------------------------------------------------------------------------
// double-double (precision.py:239-341)
// ---------------------------------------------------------------------------

struct dd {
  double hi, lo;
};

GB_DEVICE dd two_sum(double a, double b) {
  double s = __dadd_rn(a, b);
  double v = __dsub_rn(s, a);
  double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, v)), __dsub_rn(b, v));
  return {s, e};
}
GB_DEVICE dd fast_two_sum(double a, double b) {
  double s = __dadd_rn(a, b);
  return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
GB_DEVICE dd two_prod(double a, double b) {
  double p = __dmul_rn(a, b);
  return {p, __fma_rn(a, b, -p)};
}
GB_DEVICE dd dd_add(dd x, dd y) {
  dd s = two_sum(x.hi, y.hi);
  dd t = two_sum(x.lo, y.lo);
  s = fast_two_sum(s.hi, __dadd_rn(s.lo, t.hi));
  return fast_two_sum(s.hi, __dadd_rn(s.lo, t.lo));
}
GB_DEVICE dd dd_neg(dd x) { return {-x.hi, -x.lo}; }
GB_DEVICE dd dd_sub(dd x, dd y) { return dd_add(x, dd_neg(y)); }
GB_DEVICE dd dd_mul(dd x, dd y) {
  dd p = two_prod(x.hi, y.hi);
  return fast_two_sum(p.hi, __dadd_rn(p.lo, __dadd_rn(__dmul_rn(x.hi, y.lo), __dmul_rn(x.lo, y.hi))));
}
// (d, 0) * x  (precision.py:287-291)
GB_DEVICE dd dd_scale(double d, dd x) {
  dd p = two_prod(d, x.hi);
  return fast_two_sum(p.hi, __dadd_rn(p.lo, __dmul_rn(d, x.lo)));
}
GB_DEVICE dd dd_div(dd x, dd y) {
  double q1 = __ddiv_rn(x.hi, y.hi);
  dd r = dd_sub(x, dd_scale(q1, y));
  double q2 = __ddiv_rn(r.hi, y.hi);
  r = dd_sub(r, dd_scale(q2, y));
  double q3 = __ddiv_rn(r.hi, y.hi);
  dd q = fast_two_sum(q1, q2);
  return dd_add(q, dd{q3, 0.0});
}
GB_DEVICE double dd_val(dd x) { return __dadd_rn(x.hi, x.lo); }

// ---------------------------------------------------------------------------
// reductions
// ---------------------------------------------------------------------------

template <class T>
GB_DEVICE T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
GB_DEVICE dd warp_sum_dd(dd v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dd w{__shfl_xor_sync(0xffffffffu, v.hi, o), __shfl_xor_sync(0xffffffffu, v.lo, o)};
    // dd_add is commutative bit for bit (two_sum's error term is exact), so
    // every lane ends with the same bits without a divergent pairing
    v = dd_add(v, w);
  }
  return v;
}
template <class T>
GB_DEVICE T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum of K values per thread; every thread receives the totals.
// Deterministic: fixed warp trees then a fixed-order sum over warps.
// `scratch` must hold K * 32 elements of T.
template <class T, int K>
__device__ void block_sum(T (&v)[K], T* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int i = 0; i < K; ++i) v[i] = warp_sum(v[i]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < K; ++i) scratch[i * 32 + wid] = v[i];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < K; ++i) {
    T t = lane < nw ? scratch[i * 32 + lane] : T(0);
    v[i] = warp_sum(t);
  }
  __syncthreads();
}

__device__ inline void block_sum_dd(dd& v, double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum_dd(v);
  __syncthreads();
  if (lane == 0) {
    scratch[wid] = v.hi;
    scratch[32 + wid] = v.lo;
  }
  __syncthreads();
  dd t = lane < nw ? dd{scratch[lane], scratch[32 + lane]} : dd{0.0, 0.0};
  v = warp_sum_dd(t);
  __syncthreads();
}

template <class T>
__device__ T block_max(T v, T* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  T t = lane < nw ? scratch[lane] : T(-1.0);
  v = warp_max(t);
  __syncthreads();
  return v;
}

// NaN-propagating |x| max used for nu = max|r| (numpy max propagates NaN)
GB_DEVICE double nan_max(double a, double b) {
  if (a != a) return a;
  if (b != b) return b;
  return a > b ? a : b;
}

}  // namespace gb
