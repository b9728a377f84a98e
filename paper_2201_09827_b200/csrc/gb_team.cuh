// Execution teams.
//
// Every solver routine is written once against a Team:
//   * CtaTeam  -- one CTA owns a whole system (batched mode, config 3 and the
//                 small single systems); sync() is __syncthreads().
//   * GridTeam -- every CTA of a cooperative (co-resident) grid works on one
//                 large system; rows of length-n vectors are sliced across
//                 CTAs, sync() is a grid barrier, and cross-CTA sums are
//                 deterministic (per-CTA partials summed in rank order, so all
//                 CTAs hold bit-identical scalars and take identical branches).
#pragma once
#include "gb_common.cuh"

namespace gb {

// GridCtl::count must be zero when a grid-team kernel starts (the host
// resets it before every launch, see gb_solver.cuh: grid_ctl_reset)
struct GridCtl {
  unsigned int count;
  unsigned int gen;
  unsigned int pad[30];
};

GB_DEVICE unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// relaxed (strong, no L1 invalidation) poll; pair with one fence_acquire()
GB_DEVICE unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
GB_DEVICE void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
GB_DEVICE void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct CtaTeam {
  static constexpr bool kGrid = false;
  static constexpr int kTB = 32;
  GB_DEVICE int size() const { return 1; }
  GB_DEVICE int rank() const { return 0; }
  GB_DEVICE bool leader() const { return true; }
  GB_DEVICE void sync() { __syncthreads(); }
  // rows [lo, hi) of a length-n vector owned by this CTA
  GB_DEVICE void rows(int n, int& lo, int& hi) const {
    lo = 0;
    hi = n;
  }
  // after a block-level reduction of K values (all threads hold them), make
  // them team-wide.  Nothing to do for a single CTA.
  template <class T, int K>
  GB_DEVICE void finish_sum(T (&v)[K]) {}
  // every thread holds its partials; on return every thread holds the team sums
  template <class T, int K>
  __device__ void reduce(T (&v)[K], T* scratch) {
    block_sum<T, K>(v, scratch);
  }
  GB_DEVICE double finish_max(double v) { return v; }
  // vector variant: local[K] in smem (this CTA's partials) -> out[K] in smem
  template <class T>
  __device__ void sum_vec(const T* local, T* out, int K) {
    for (int i = threadIdx.x; i < K; i += blockDim.x) out[i] = local[i];
    __syncthreads();
  }
};

// number of CTAs in this thread-block cluster (1 without a cluster launch)
GB_DEVICE unsigned cluster_ncta() {
  unsigned v;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(v));
  return v;
}

struct GridTeam {
  static constexpr bool kGrid = true;
  static constexpr int kTB = kTrsvB;  // substitution row block (trsv_cta_g)
  int G, r;
  GridCtl* ctl;
  double* partials;  // 2 buffers of G * kMaxK doubles
  int kmax;
  unsigned phase;
  // the whole team is one thread-block cluster (G <= 16 CTAs): sync() is the
  // hardware cluster barrier (release/acquire at cluster scope) instead of
  // the global-memory grid barrier
  bool clu = false;
  // cluster teams: per-CTA shared-memory copy of the partials buffers (same
  // layout as `partials`); producers push their values into every CTA's copy
  double* spart = nullptr;
  unsigned nsync = 0;  // grid barriers passed in this launch (identical in every CTA)

  GB_DEVICE int size() const { return G; }
  GB_DEVICE int rank() const { return r; }
  GB_DEVICE bool leader() const { return r == 0; }

  __device__ void sync() {
    if (clu) {
      asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
      return;
    }
    // monotone arrival counter (reset by the host before every launch): each
    // CTA adds 1 with a fire-and-forget release reduction and waits until all
    // G arrivals of this barrier are in.  A returning atomicAdd from every CTA
    // serialises at the L2 atomic unit (~2.6 us for 148 CTAs on B200); the
    // reductions pipeline (~0.5 us).
    __syncthreads();
    if (threadIdx.x < 32) {
      // the whole warp 0 spins uniformly (a lone spinning lane pays a large
      // reconvergence penalty on sm_100a, see tools/micro/trsv.cu)
      ++nsync;
      const unsigned target = nsync * (unsigned)G;
      if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&ctl->count) : "memory");
      while ((int)(ld_acquire(&ctl->count) - target) < 0) {
      }
    }
    __syncthreads();
  }
  GB_DEVICE void rows(int n, int& lo, int& hi) const {
    int per = (n + G - 1) / G;
    per = (per + 31) & ~31;
    lo = min(n, r * per);
    hi = min(n, lo + per);
  }
  GB_DEVICE double* buf() { return partials + (size_t)(phase & 1) * G * kmax; }
  GB_DEVICE double* sbuf() { return spart + (size_t)(phase & 1) * G * kmax; }
  // store v at offset idx of the current shared buffer of cluster CTA q
  GB_DEVICE static void push(double* local, int q, double v) {
    unsigned ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                 : "=r"(ra)
                 : "r"((unsigned)__cvta_generic_to_shared(local)), "r"(q));
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
  }

  // every thread holds its partials; on return every thread of every CTA
  // holds the team sums (bit-identical: fixed summation order).  Cluster
  // teams skip the block reduction: each warp pushes its warp sum straight
  // into every CTA's shared copy and one cluster barrier publishes them all.
  template <class T, int K>
  __device__ void reduce(T (&v)[K], T* scratch) {
    if (spart == nullptr) {
      block_sum<T, K>(v, scratch);
      finish_sum<T, K>(v);
      return;
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int i = 0; i < K; ++i) v[i] = warp_sum(v[i]);
    double* p = sbuf();
    if (lane < G) {
#pragma unroll
      for (int i = 0; i < K; ++i) push(p + ((size_t)(r * nw + wid)) * K + i, lane, (double)v[i]);
    }
    sync();
    const int tot = G * nw;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      T acc = T(0);
      for (int e = lane; e < tot; e += 32) acc += (T)p[(size_t)e * K + i];
      v[i] = warp_sum(acc);
    }
    ++phase;
  }

  // v[] holds this CTA's block-reduced values in every thread.
  template <class T, int K>
  __device__ void finish_sum(T (&v)[K]) {
    if (spart != nullptr) {
      // lane q of warp 0 pushes this CTA's K values into CTA q; the cluster
      // barrier orders the pushes; then every CTA sums its local copy
      double* p = sbuf();
      if (threadIdx.x < G) {
#pragma unroll
        for (int i = 0; i < K; ++i) push(p + (size_t)r * K + i, threadIdx.x, (double)v[i]);
      }
      sync();
      const int lane = threadIdx.x & 31;
#pragma unroll
      for (int i = 0; i < K; ++i) {
        T acc = T(0);
        for (int g = lane; g < G; g += 32) acc += (T)p[(size_t)g * K + i];
        v[i] = warp_sum(acc);
      }
      ++phase;
      return;
    }
    double* p = buf();
    if (threadIdx.x == 0) {
#pragma unroll
      for (int i = 0; i < K; ++i) p[(size_t)r * K + i] = (double)v[i];
    }
    sync();
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      T acc = T(0);
      for (int g = lane; g < G; g += 32) acc += (T)__ldcg(p + (size_t)g * K + i);
      v[i] = warp_sum(acc);
    }
    ++phase;
  }
  __device__ double finish_max(double v) {
    if (spart != nullptr) {
      double* p = sbuf();
      if (threadIdx.x < G) push(p + r, threadIdx.x, v);
      sync();
      const int lane = threadIdx.x & 31;
      double acc = -1.0;
      for (int g = lane; g < G; g += 32) acc = nan_max(acc, p[g]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc = nan_max(acc, __shfl_xor_sync(0xffffffffu, acc, o));
      ++phase;
      return acc;
    }
    double* p = buf();
    if (threadIdx.x == 0) p[r] = v;
    sync();
    const int lane = threadIdx.x & 31;
    double acc = -1.0;
    for (int g = lane; g < G; g += 32) acc = nan_max(acc, __ldcg(p + g));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = nan_max(acc, __shfl_xor_sync(0xffffffffu, acc, o));
    ++phase;
    return acc;
  }
  // local[K] (smem, this CTA's partials) -> out[K] (smem) summed in rank order.
  template <class T>
  __device__ void sum_vec(const T* local, T* out, int K) {
    if (spart != nullptr) {
      double* p = sbuf();
      for (int e = threadIdx.x; e < K * G; e += blockDim.x) {
        const int i = e / G, q = e % G;
        push(p + (size_t)r * K + i, q, (double)local[i]);
      }
      sync();
      for (int i = threadIdx.x; i < K; i += blockDim.x) {
        T acc = T(0);
        for (int g = 0; g < G; ++g) acc += (T)p[(size_t)g * K + i];
        out[i] = acc;
      }
      __syncthreads();
      ++phase;
      return;
    }
    double* p = buf();
    for (int i = threadIdx.x; i < K; i += blockDim.x) p[(size_t)r * K + i] = (double)local[i];
    sync();
    for (int i = threadIdx.x; i < K; i += blockDim.x) {
      T acc = T(0);
      for (int g = 0; g < G; ++g) acc += (T)__ldcg(p + (size_t)g * K + i);
      out[i] = acc;
    }
    __syncthreads();
    ++phase;
  }
};

// A grid team of <= 16 CTAs launched as one thread-block cluster (the cfg2
// size, n <= 1024): same protocol as GridTeam (sync() picks the cluster
// barrier at run time), but its own type so its kernels use the 32-row
// substitution and carry none of the 64-row code (register pressure).
struct ClusterTeam : GridTeam {
  static constexpr int kTB = 32;
};

}  // namespace gb
