// Tensor-core trailing update of the blocked fp16 LU (tensor mode, SURVEY
// §8(a) a6, densela.py:148-168 restated as a blocked GEPP):
//
//   C <- fl16( C - fp32( A * Bt^T ) )      A = L21 (M x K), Bt = U12^T (N x K)
//
// with K = the panel width (a multiple of 32).  One persistent,
// warp-specialised kernel per panel:
//   warp 0  TMA producer: 2-D tensor-map loads (SWIZZLE_64B, K-major 32-wide
//           slabs) of A (128 x 32) and Bt (256 x 32) into an STAGES-deep
//           ring of shared-memory stages, one mbarrier (expect_tx) per stage;
//   warp 1  MMA issuer: one thread issues tcgen05.mma kind::f16 (128 x 256 x
//           16, fp32 accumulator in TMEM), tcgen05.commit frees the stage;
//   warp 2  TMEM allocator (512 columns = two 128 x 256 fp32 accumulators);
//   warps 4-7  epilogue: tcgen05.ld of the accumulator (warp 4+q reads TMEM
//           lanes 32q..32q+31 = rows of the tile), C read, fl16(C - acc),
//           store; the accumulator buffer is handed back through an mbarrier,
//           so the epilogue of tile t overlaps the MMAs of tile t+1.
// Tiles (128 x 256 of C) are dealt round-robin over the persistent CTAs.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <algorithm>

#include "gb_tc.cuh"

namespace gb {
namespace tcg {

constexpr int BM = 128, BN = 256, BK = 32;        // tile and K slab (64-byte K-major rows)
constexpr int STAGES = 6;
constexpr int A_BYTES = BM * BK * 2;              // 8 KB
constexpr int B_BYTES = BN * BK * 2;              // 16 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;    // 24 KB
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;  // + alignment + barriers
constexpr int NTHREADS = 256;

__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(b)) : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(tc::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(tc::smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// C rows [r0, r0 + M), columns [c0, c0 + N) of W (row-major, leading dim ld);
// A via map_a at (column k0, row r0 + ...), Bt via map_b (row = C column - c0)
static __global__ void __launch_bounds__(NTHREADS, 1)
    k_tc_update(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b, __half* W,
                size_t ld, int r0, int c0, int M, int N, int k0, int K) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tm = (M + BM - 1) / BM, tn = (N + BN - 1) / BN;
  const int ntiles = tm * tn;
  const int nslab = K / BK;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      tc::mbar_init(full + i, 1);
      tc::mbar_init(empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(tfull + i, 1);
      tc::mbar_init(tempty + i, 4);  // one elected arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_map(&map_a);
    prefetch_map(&map_b);
  }
  if (warp == 2) tc::tmem_alloc(tmem_slot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---- TMA producer
    int st = 0;
    uint32_t ph = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int ti = t / tn, tj = t % tn;
      for (int s = 0; s < nslab; ++s) {
        tc::mbar_wait(empty + st, ph ^ 1u);
        unsigned char* sa = smem + st * STAGE_BYTES;
        unsigned char* sb = sa + A_BYTES;
        mbar_expect_tx(full + st, STAGE_BYTES);
        tma_2d(sa, &map_a, k0 + s * BK, r0 + ti * BM, full + st);
        tma_2d(sb, &map_b, s * BK, tj * BN, full + st);
        if (++st == STAGES) st = 0, ph ^= 1u;
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer (single thread)
    constexpr uint32_t idesc = tc::idesc_f16_f32(BM, BN);
    int st = 0;
    uint32_t ph = 0;
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int acc = it & 1;
      const uint32_t aph = (uint32_t)((it >> 1) & 1);
      tc::mbar_wait(tempty + acc, aph ^ 1u);  // the epilogue drained this accumulator
      tc::fence_after();
      const uint32_t dt = tmem + (uint32_t)(acc * BN);
      for (int s = 0; s < nslab; ++s) {
        tc::mbar_wait(full + st, ph);
        tc::fence_after();
        const unsigned char* sa = smem + st * STAGE_BYTES;
        const uint64_t ad = tc::desc_k64(tc::smem_u32(sa)), bd = tc::desc_k64(tc::smem_u32(sa + A_BYTES));
        tc::mma_f16(dt, ad, bd, idesc, s > 0 ? 1u : 0u);
        tc::mma_f16(dt, ad + 2, bd + 2, idesc, 1u);  // K = 16..31: +32 bytes inside the swizzle atom
        tc::commit(empty + st);                       // frees the stage once these MMAs completed
        if (++st == STAGES) st = 0, ph ^= 1u;
      }
      tc::commit(tfull + acc);  // accumulator complete
    }
  } else if (warp >= 4) {
    // ---- epilogue: row = TMEM lane
    const int q = warp - 4;
    const int row_in_tile = q * 32 + lane;
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int ti = t / tn, tj = t % tn;
      const int acc = it & 1;
      tc::mbar_wait(tfull + acc, (uint32_t)((it >> 1) & 1));
      tc::fence_after();
      const int gi = ti * BM + row_in_tile;  // row inside the update
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
#pragma unroll 1
      for (int ch = 0; ch < BN / 32; ++ch) {
        float v[32];
        tc::tmem_ld32(tbase + (uint32_t)(ch * 32), v);
        const int gj = tj * BN + ch * 32;
        if (gi < M && gj < N) {
          __half* p = W + (size_t)(r0 + gi) * ld + c0 + gj;
          if (gj + 32 <= N) {
            __align__(16) __half h[32];
#pragma unroll
            for (int z = 0; z < 4; ++z) reinterpret_cast<uint4*>(h)[z] = reinterpret_cast<const uint4*>(p)[z];
#pragma unroll
            for (int z = 0; z < 32; ++z) h[z] = __float2half_rn(__half2float(h[z]) - v[z]);
#pragma unroll
            for (int z = 0; z < 4; ++z) reinterpret_cast<uint4*>(p)[z] = reinterpret_cast<const uint4*>(h)[z];
          } else {
            for (int z = 0; z < 32 && gj + z < N; ++z) p[z] = __float2half_rn(__half2float(p[z]) - v[z]);
          }
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + acc);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 2) tc::tmem_dealloc(tmem, 512);
}

// Bt[j][k] = U12[k][j] (K x N of W at rows [k0, k0 + K), columns [c0, c0 + N))
// into the K-major scratch (row stride K)
static __global__ void k_transpose_u12(const __half* __restrict__ W, size_t ld, int k0, int c0, int K, int N,
                                __half* __restrict__ Bt) {
  __shared__ __half tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;  // bx: column (N), by: row (K)
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int k = by + i, j = bx + threadIdx.x;
    tile[i][threadIdx.x] = (k < K && j < N) ? W[(size_t)(k0 + k) * ld + c0 + j] : __float2half(0.f);
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int j = bx + i, k = by + threadIdx.x;
    if (j < N && k < K) Bt[(size_t)j * K + k] = tile[threadIdx.x][i];
  }
}

// ---------------------------------------------------------------------------
// host: tensor maps through the driver entry point (no libcuda link needed)
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (fn == nullptr) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D fp16 map over a row-major matrix (rows x cols, row pitch in elements),
// box = box_rows x 32 columns, SWIZZLE_64B (the UMMA K-major SW64 atom)
inline bool make_map(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t pitch_elems,
                     uint32_t box_rows, uint32_t box_cols = BK, bool swizzle128 = false) {
  EncodeTiledFn fn = encode_fn();
  if (fn == nullptr) return false;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {pitch_elems * 2};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// W[r0:r0+M, c0:c0+N] -= W[r0:r0+M, k0:k0+K] * W[k0:k0+K, c0:c0+N]  (fp32
// accumulation, one fl16 rounding); Bt: scratch of N * K halves
inline cudaError_t tc_update(__half* W, size_t ld, int nrows, int r0, int c0, int M, int N, int k0, int K,
                             __half* Bt, int nsm, cudaStream_t st) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  dim3 tb(32, 8), tg((N + 31) / 32, (K + 31) / 32);
  k_transpose_u12<<<tg, tb, 0, st>>>(W, ld, k0, c0, K, N, Bt);
  CUtensorMap ma, mb;
  if (!make_map(&ma, W, (uint64_t)nrows, ld, ld, BM) || !make_map(&mb, Bt, (uint64_t)N, (uint64_t)K, K, BN))
    return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_tc_update, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    attr = true;
  }
  const int ntiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  k_tc_update<<<ntiles < nsm ? ntiles : nsm, NTHREADS, SMEM_BYTES, st>>>(ma, mb, W, ld, r0, c0, M, N, k0, K);
  return cudaGetLastError();
}

}  // namespace tcg

// ---------------------------------------------------------------------------
// CTA-pair form of the same update (cta_group::2): a cluster of two CTAs on
// one TPC owns a 256 x 256 tile of C.  Each CTA stages its own 128 rows of A
// and its own 128 of the 256 Bt rows (16 KB per 32-wide K slab instead of the
// 24 KB of the one-CTA kernel, which the L2 -> SM path caps at ~44 % of the
// tensor peak: ~42 B/clk/SM against the 96 B/clk/SM a 128 x 256 tile needs);
// the leader's elected thread issues tcgen05.mma.cta_group::2 (M = 256,
// N = 256), which reads the B halves out of both CTAs' shared memory and
// leaves rows 128 r .. 128 r + 127 of the accumulator in CTA r's TMEM.
//   full[s]    lives in the leader: its producer arms 2 x 16 KB, both CTAs'
//              TMA loads complete_tx on it (cta_group::2 form);
//   empty[s], tfull[a]  are signalled in both CTAs by the multicast commit;
//   tempty[a]  lives in the leader: the 16 epilogue warps of the pair arrive.
// ---------------------------------------------------------------------------
namespace tcg2 {

constexpr int BM = 128, PM = 256, BN = 256, HN = 128, BK = 32;
constexpr int A_BYTES = BM * BK * 2;            // 8 KB
constexpr int B_BYTES = HN * BK * 2;            // 8 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;  // 16 KB per CTA
// kTmaC: the CTA's 128 x 256 tile of C is staged in shared memory (four
// 128 x 64 boxes, SWIZZLE_128B) by TMA under the tile's MMAs, updated in
// place by the epilogue warps and written back by TMA stores -- all global
// traffic of the epilogue is bulk and coalesced (row-per-lane global accesses
// cost 32 LSU wavefronts per instruction).  Needs M, N multiples of 256 (a
// TMA store cannot mask the rows / columns of a partial tile).
constexpr int C_BOX_COLS = 64;
constexpr int C_BOX_BYTES = BM * C_BOX_COLS * 2;  // 16 KB
constexpr int C_BYTES = 4 * C_BOX_BYTES;          // 64 KB
template <bool kTmaC>
struct Cfg {
  static constexpr int STAGES = kTmaC ? 8 : 12;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + (kTmaC ? C_BYTES : 0) + 1024 + 512;
};
constexpr int NTHREADS = 384;  // TMA, MMA, TMEM, C loader, 8 epilogue warps

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// address of the leader CTA's copy of a shared-memory object, in the cluster window
__device__ __forceinline__ uint32_t leader_addr(const void* p) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(tc::smem_u32(p)));
  return r;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void tma_2d_pair(void* dst, const CUtensorMap* map, int c0, int c1, uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(tc::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar_cluster)
      : "memory");
}
__device__ __forceinline__ void mma_f16_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// completion of all prior MMAs of the pair -> the barrier at this offset in both CTAs
__device__ __forceinline__ void commit_pair(uint64_t* mbar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          tc::smem_u32(mbar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(dst_smem)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int c0, int c1, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(tc::smem_u32(src))
               : "memory");
}

template <bool kTmaC>
static __global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTHREADS, 1)
    k_tc_update2(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                 const __grid_constant__ CUtensorMap map_c, __half* W, size_t ld, int r0, int c0, int M, int N, int k0,
                 int K) {
  constexpr int STAGES = Cfg<kTmaC>::STAGES;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // the same offset in both CTAs (the dynamic window starts at the same address)
  unsigned char* smem = reinterpret_cast<unsigned char*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* csm = smem + STAGES * STAGE_BYTES;  // C tile (kTmaC), 1024-byte aligned
  uint64_t* full = reinterpret_cast<uint64_t*>(csm + (kTmaC ? C_BYTES : 0));
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint64_t* cfull = tempty + 2;      // C tile landed
  uint64_t* cfree = cfull + 1;       // C tile written back, buffer reusable
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cfree + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int tm = (M + PM - 1) / PM, tn = (N + BN - 1) / BN;
  const int ntiles = tm * tn;
  const int nslab = K / BK;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      tc::mbar_init(full + i, 1);
      tc::mbar_init(empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(tfull + i, 1);
      tc::mbar_init(tempty + i, 16);  // one elected arrive per epilogue warp of the pair
    }
    tc::mbar_init(cfull, 1);
    tc::mbar_init(cfree, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    tcg::prefetch_map(&map_a);
    tcg::prefetch_map(&map_b);
    if (kTmaC) tcg::prefetch_map(&map_c);
  }
  if (warp == 2) tmem_alloc_pair(tmem_slot, 512);
  tc::fence_before();
  cluster_sync_all();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---- TMA producer (both CTAs): own 128 rows of A, own 128 rows of Bt
    int st = 0;
    uint32_t ph = 0;
    for (int t = pair; t < ntiles; t += npairs) {
      const int ti = t / tn, tj = t % tn;
      for (int s = 0; s < nslab; ++s) {
        tc::mbar_wait(empty + st, ph ^ 1u);
        unsigned char* sa = smem + st * STAGE_BYTES;
        unsigned char* sb = sa + A_BYTES;
        if (rank == 0) tcg::mbar_expect_tx(full + st, 2 * STAGE_BYTES);
        const uint32_t bar = leader_addr(full + st);
        tma_2d_pair(sa, &map_a, k0 + s * BK, r0 + ti * PM + (int)rank * BM, bar);
        tma_2d_pair(sb, &map_b, s * BK, tj * BN + (int)rank * HN, bar);
        if (++st == STAGES) st = 0, ph ^= 1u;
      }
    }
  } else if (warp == 1 && lane == 0 && rank == 0) {
    // ---- MMA issuer: one thread of the leader CTA for the pair
    constexpr uint32_t idesc = tc::idesc_f16_f32(PM, BN);
    int st = 0;
    uint32_t ph = 0;
    int it = 0;
    for (int t = pair; t < ntiles; t += npairs, ++it) {
      const int acc = it & 1;
      const uint32_t aph = (uint32_t)((it >> 1) & 1);
      tc::mbar_wait(tempty + acc, aph ^ 1u);  // both CTAs' epilogues drained this accumulator
      tc::fence_after();
      const uint32_t dt = tmem + (uint32_t)(acc * BN);
      for (int s = 0; s < nslab; ++s) {
        tc::mbar_wait(full + st, ph);
        tc::fence_after();
        const unsigned char* sa = smem + st * STAGE_BYTES;
        const uint64_t ad = tc::desc_k64(tc::smem_u32(sa)), bd = tc::desc_k64(tc::smem_u32(sa + A_BYTES));
        mma_f16_pair(dt, ad, bd, idesc, s > 0 ? 1u : 0u);
        mma_f16_pair(dt, ad + 2, bd + 2, idesc, 1u);
        commit_pair(empty + st);
        if (++st == STAGES) st = 0, ph ^= 1u;
      }
      commit_pair(tfull + acc);
    }
  } else if (kTmaC && warp == 3 && lane == 0) {
    // ---- C loader (both CTAs): this CTA's 128 x 256 tile of C, as soon as the
    // previous tile has been written back
    int it = 0;
    for (int t = pair; t < ntiles; t += npairs, ++it) {
      const int ti = t / tn, tj = t % tn;
      if (it > 0) tc::mbar_wait(cfree, (uint32_t)((it - 1) & 1));
      tcg::mbar_expect_tx(cfull, C_BYTES);
#pragma unroll
      for (int b = 0; b < 4; ++b)
        tcg::tma_2d(csm + b * C_BOX_BYTES, &map_c, c0 + tj * BN + b * C_BOX_COLS, r0 + ti * PM + (int)rank * BM, cfull);
    }
  } else if (kTmaC && warp >= 4) {
    // ---- epilogue, C through shared memory: thread = (row 32 q + lane, column
    // half hc); element (row, 16-byte chunk c) of a box sits at
    // row * 128 + ((c ^ (row & 7)) << 4) (SWIZZLE_128B)
    const int q = warp & 3, hc = (warp - 4) >> 2;
    const int row = q * 32 + lane;
    int it = 0;
    for (int t = pair; t < ntiles; t += npairs, ++it) {
      const int ti = t / tn, tj = t % tn;
      const int acc = it & 1;
      tc::mbar_wait(cfull, (uint32_t)(it & 1));
      tc::mbar_wait(tfull + acc, (uint32_t)((it >> 1) & 1));
      tc::fence_after();
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + hc * 128);
      auto upd = [](unsigned c, float a, float b) -> unsigned {
        __half2 h = *reinterpret_cast<__half2*>(&c);
        const float2 f = __half22float2(h);
        h = __floats2half2_rn(f.x - a, f.y - b);
        return *reinterpret_cast<unsigned*>(&h);
      };
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        float v[32];
        tc::tmem_ld32(tbase + (uint32_t)(ch * 32), v);
        unsigned char* box = csm + (hc * 2 + (ch >> 1)) * C_BOX_BYTES + row * 128;
#pragma unroll
        for (int z = 0; z < 4; ++z) {
          const int c = (ch & 1) * 4 + z;
          uint4* p = reinterpret_cast<uint4*>(box + ((c ^ (row & 7)) << 4));
          const uint4 cc = *p;
          uint4 o;
          o.x = upd(cc.x, v[8 * z + 0], v[8 * z + 1]);
          o.y = upd(cc.y, v[8 * z + 2], v[8 * z + 3]);
          o.z = upd(cc.z, v[8 * z + 4], v[8 * z + 5]);
          o.w = upd(cc.w, v[8 * z + 6], v[8 * z + 7]);
          *p = o;
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(leader_addr(tempty + acc));  // accumulator drained
      tc::fence_proxy_async();                                       // smem writes -> async proxy
      asm volatile("bar.sync 2, 256;" ::: "memory");                 // the 8 epilogue warps
      if (warp == 4 && lane == 0) {
#pragma unroll
        for (int b = 0; b < 4; ++b)
          tma_store_2d(&map_c, c0 + tj * BN + b * C_BOX_COLS, r0 + ti * PM + (int)rank * BM, csm + b * C_BOX_BYTES);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        tcg::mbar_arrive(cfree);
      }
    }
    if (warp == 4 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores complete
  } else if (warp >= 4) {
    // ---- epilogue (both CTAs, 8 warps): warp 4 + q + 4 h owns TMEM lanes
    // 32 q .. 32 q + 31 (rows 128 rank + 32 q + lane of the pair tile) and the
    // column half h.  The 256 bytes of C a thread updates are loaded BEFORE
    // the wait on the accumulator, i.e. under the MMAs of the same tile.
    const int q = warp & 3, hc = (warp - 4) >> 2;
    const int row_in_tile = (int)rank * BM + q * 32 + lane;
    int it = 0;
    for (int t = pair; t < ntiles; t += npairs, ++it) {
      const int ti = t / tn, tj = t % tn;
      const int acc = it & 1;
      const int gi = ti * PM + row_in_tile;
      const int gj0 = tj * BN + hc * 128;
      const bool rowok = gi < M;
      const bool fullw = rowok && gj0 + 128 <= N;
      __half* prow = W + (size_t)(r0 + (rowok ? gi : 0)) * ld + c0 + gj0;
      uint4 cpre[16];
      if (fullw) {
#pragma unroll
        for (int z = 0; z < 16; ++z) cpre[z] = reinterpret_cast<const uint4*>(prow)[z];
      }
      tc::mbar_wait(tfull + acc, (uint32_t)((it >> 1) & 1));
      tc::fence_after();
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + hc * 128);
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        float v[32];
        tc::tmem_ld32(tbase + (uint32_t)(ch * 32), v);
        const int gj = gj0 + ch * 32;
        if (fullw) {
          auto upd = [](unsigned c, float a, float b) -> unsigned {
            __half2 h = *reinterpret_cast<__half2*>(&c);
            const float2 f = __half22float2(h);
            h = __floats2half2_rn(f.x - a, f.y - b);
            return *reinterpret_cast<unsigned*>(&h);
          };
#pragma unroll
          for (int z = 0; z < 4; ++z) {
            const uint4 cc = cpre[4 * ch + z];
            uint4 o;
            o.x = upd(cc.x, v[8 * z + 0], v[8 * z + 1]);
            o.y = upd(cc.y, v[8 * z + 2], v[8 * z + 3]);
            o.z = upd(cc.z, v[8 * z + 4], v[8 * z + 5]);
            o.w = upd(cc.w, v[8 * z + 6], v[8 * z + 7]);
            reinterpret_cast<uint4*>(prow + ch * 32)[z] = o;
          }
        } else if (rowok && gj < N) {
          __half* p = prow + ch * 32;
          for (int z = 0; z < 32 && gj + z < N; ++z) p[z] = __float2half_rn(__half2float(p[z]) - v[z]);
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(leader_addr(tempty + acc));
    }
  }
  tc::fence_before();
  cluster_sync_all();  // the leader's MMAs read the peer's shared memory; remote arrives target the leader
  if (warp == 2) tmem_dealloc_pair(tmem, 512);
}

// pairs that can be co-resident (148 SMs = 74 TPCs unless a GPC is short)
template <bool kTmaC>
inline int max_pairs_t() {
  static int pairs = -1;
  if (pairs < 0) {
    cudaFuncSetAttribute(k_tc_update2<kTmaC>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<kTmaC>::SMEM_BYTES);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * 74);
    cfg.blockDim = dim3(NTHREADS);
    cfg.dynamicSmemBytes = Cfg<kTmaC>::SMEM_BYTES;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, (const void*)k_tc_update2<kTmaC>, &cfg) != cudaSuccess || n < 1) {
      cudaGetLastError();
      n = 64;
    }
    pairs = n;
  }
  return pairs;
}
inline int max_pairs() { return max_pairs_t<true>(); }

// same contract as tcg::tc_update; tma_c = -1 picks the shared-memory C path
// whenever the update is made of whole 256 x 256 tiles
inline cudaError_t tc_update(__half* W, size_t ld, int nrows, int r0, int c0, int M, int N, int k0, int K,
                             __half* Bt, cudaStream_t st, int tma_c = -1) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  dim3 tb(32, 8), tg((N + 31) / 32, (K + 31) / 32);
  tcg::k_transpose_u12<<<tg, tb, 0, st>>>(W, ld, k0, c0, K, N, Bt);
  const bool whole = M % PM == 0 && N % BN == 0 && c0 % 8 == 0;
  const bool use_c = tma_c < 0 ? whole : (tma_c != 0 && whole);
  CUtensorMap ma, mb, mc;
  if (!tcg::make_map(&ma, W, (uint64_t)nrows, ld, ld, BM) || !tcg::make_map(&mb, Bt, (uint64_t)N, (uint64_t)K, K, HN) ||
      !tcg::make_map(&mc, W, (uint64_t)nrows, ld, ld, BM, C_BOX_COLS, true))
    return cudaErrorInvalidValue;
  const int ntiles = ((M + PM - 1) / PM) * ((N + BN - 1) / BN);
  if (use_c) {
    const int pairs = std::min(ntiles, max_pairs_t<true>());
    k_tc_update2<true><<<2 * pairs, NTHREADS, Cfg<true>::SMEM_BYTES, st>>>(ma, mb, mc, W, ld, r0, c0, M, N, k0, K);
  } else {
    const int pairs = std::min(ntiles, max_pairs_t<false>());
    k_tc_update2<false><<<2 * pairs, NTHREADS, Cfg<false>::SMEM_BYTES, st>>>(ma, mb, mc, W, ld, r0, c0, M, N, k0, K);
  }
  return cudaGetLastError();
}

}  // namespace tcg2
}  // namespace gb
