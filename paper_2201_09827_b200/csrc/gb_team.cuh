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
  // one value per thread -> the team sum in every thread
  template <class T>
  __device__ T reduce1(T v, T* scratch) {
    T a[1] = {v};
    block_sum<T, 1>(a, scratch);
    return a[0];
  }
  // vector variant: local[K] in smem (this CTA's partials) -> out[K] in smem
  template <class T>
  __device__ void sum_vec(const T* local, T* out, int K) {
    for (int i = threadIdx.x; i < K; i += blockDim.x) out[i] = local[i];
    __syncthreads();
  }
};

// tagged 16-byte words {lo32, tag, hi32, tag}: a reader that sees the tag in
// both 8-byte halves has the value (no counters, no fences)
GB_DEVICE void team_tput(uint4* p, double v, unsigned tag) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"((unsigned)b), "r"(tag),
               "r"((unsigned)(b >> 32)), "r"(tag)
               : "memory");
}
GB_DEVICE bool team_tget(const uint4* p, unsigned tag, double& v) {
  unsigned x, y, z, w;
  asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(x), "=r"(y), "=r"(z), "=r"(w)
               : "l"(p)
               : "memory");
  v = __longlong_as_double((long long)(((unsigned long long)z << 32) | x));
  return y == tag && w == tag;
}
constexpr int kLinkSlots = 160;  // >= the largest grid team (148 CTAs)
constexpr int kSubSlots = 32;    // sub-team of the Gram-Schmidt sweep (reduce1_sub)
constexpr int kColBuf = 256;     // doubles broadcast from the sub-team to the grid
// bytes that follow the GridCtl word in global memory: full-team slots (2 sets),
// sub-team slots (2 sets), broadcast buffer
constexpr size_t kCtlExtraBytes = 2 * kLinkSlots * 16 + 2 * kSubSlots * 16 + kColBuf * 8;

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
  // tagged single-value reductions (reduce1, cooperative grids): links done by
  // this launch and the count carried over from earlier launches (the tags
  // must not repeat while a slot still holds an old one); slots follow *ctl
  unsigned long long link_base = 0, sub_base = 0;
  unsigned nlink = 0, nsub = 0;

  GB_DEVICE void links_begin() {
    if (ctl != nullptr) {
      link_base = *reinterpret_cast<volatile unsigned long long*>(&ctl->pad[0]);
      sub_base = *reinterpret_cast<volatile unsigned long long*>(&ctl->pad[2]);
    }
  }
  GB_DEVICE void links_end() {
    if (ctl != nullptr && r == 0 && threadIdx.x == 0) {
      if (nlink != 0) *reinterpret_cast<volatile unsigned long long*>(&ctl->pad[0]) = link_base + nlink;
      if (nsub != 0) *reinterpret_cast<volatile unsigned long long*>(&ctl->pad[2]) = sub_base + nsub;
    }
  }
  GB_DEVICE uint4* sub_slots() { return reinterpret_cast<uint4*>(ctl + 1) + 2 * kLinkSlots; }
  GB_DEVICE double* colbuf() { return reinterpret_cast<double*>(sub_slots() + 2 * kSubSlots); }
  // reduce1 over the first T <= 32 CTAs only (the others do not call): one
  // tagged slot per CTA, a single poll per lane.  The Gram-Schmidt sweep of a
  // large grid team runs on such a sub-team: its links are pure exchange
  // latency, and polling 16 slots is faster than polling 148.
  template <class T_>
  __device__ T_ reduce1_sub(T_ v, T_* scratch, int T) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    if (wid == 0) {
      T_ tsum = lane < nw ? scratch[lane] : T_(0);
      tsum = warp_sum(tsum);
      const unsigned tag = (unsigned)((sub_base + nsub) % 0xffffffffull) + 1u;
      uint4* slots = sub_slots() + (size_t)(nsub & 1u) * kSubSlots;
      if (lane == 0) team_tput(slots + r, (double)tsum, tag);
      double x = 0.0;
      bool ok = lane >= T;
      do {
        if (!ok) ok = team_tget(slots + lane, tag, x);
      } while (!__all_sync(0xffffffffu, ok));
      T_ acc = lane < T ? (T_)x : T_(0);
      acc = warp_sum(acc);
      if (lane == 0) scratch[32] = acc;
    }
    __syncthreads();
    ++nsub;
    return scratch[32];
  }
  // One value per thread -> the team sum in every thread of every CTA, as
  // reduce<T, 1> but in ONE global round trip for cooperative grids: the
  // CTA's block sum goes into its tagged slot, warp 0 polls the G slots of
  // this link (two slot sets alternate: a CTA can be at most one link ahead
  // of the slowest one) and sums them in rank order, so the result is
  // bit-identical in every CTA.  Used by the Gram-Schmidt sweep, whose
  // j + 1 dependent dots per Arnoldi step are pure reduction latency.
  template <class T>
  __device__ T reduce1(T v, T* scratch) {
    if (clu || spart != nullptr || G > kLinkSlots) {
      T a[1] = {v};
      reduce<T, 1>(a, scratch);
      return a[0];
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    if (wid == 0) {
      T tsum = lane < nw ? scratch[lane] : T(0);
      tsum = warp_sum(tsum);
      const unsigned tag = (unsigned)((link_base + nlink) % 0xffffffffull) + 1u;
      uint4* slots = reinterpret_cast<uint4*>(ctl + 1) + (size_t)(nlink & 1u) * kLinkSlots;
      if (lane == 0) team_tput(slots + r, (double)tsum, tag);
      constexpr int PL = kLinkSlots / 32;
      double x[PL];
      bool ok[PL];
#pragma unroll
      for (int j = 0; j < PL; ++j) {
        x[j] = 0.0;
        ok[j] = lane + 32 * j >= G;
      }
      bool all;
      do {
        all = true;
#pragma unroll
        for (int j = 0; j < PL; ++j) {
          if (!ok[j]) ok[j] = team_tget(slots + lane + 32 * j, tag, x[j]);
          all = all && ok[j];
        }
      } while (!__all_sync(0xffffffffu, all));
      T acc = T(0);
#pragma unroll
      for (int j = 0; j < PL; ++j)
        if (lane + 32 * j < G) acc += (T)x[j];
      acc = warp_sum(acc);
      if (lane == 0) scratch[32] = acc;
    }
    __syncthreads();
    ++nlink;
    return scratch[32];
  }

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
