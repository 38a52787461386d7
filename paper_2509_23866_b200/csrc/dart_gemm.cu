// dart_gemm.cu -- the plain GEMM steps of the LM-head backward (SURVEY §8(f)
// NEXT #3): C[M, N] (+)= A[M, K] * B[N, K]^T, bf16 operands, fp32 accumulation
// on the 5th-generation tensor cores (sm_100a).
//
// Either operand may be K-major (row-major [rows, K]) or MN-major (row-major
// [K, rows], i.e. the transpose is stored), so the three products of the
// LM head need no transposed copies:
//    logits  z  = h  W^T    A = h  [T, d] K-major,   B = W [V, d] K-major
//    dh         = dz W      A = dz [T, V] K-major,   B = W [V, d] MN-major (N = d contiguous)
//    dW        += dz^T h    A = dz [T, V] MN-major,  B = h [T, d] MN-major
//
// Same machinery as the LM-head forward kernel (dart_lmhead.cu): persistent
// CTAs, warp 0 = TMA producer into a 4-stage ring of 128-byte-swizzled tiles
// (K-major: one 64 x rows box; MN-major: 64 x 64 boxes 8 KB apart along MN),
// warp 1 = TMEM allocator + tcgen05.mma issuer (M = 128, N = 256, K = 16 per
// instruction), warps 2..5 = epilogue from two TMEM accumulators (fp32 store,
// bf16 store or fp32 read-add-write).  Tiles are rastered in groups of
// GM_GROUP row blocks for L2 reuse of the B panel.
#include <cstdio>
#include <cstdlib>

#include "dart_common.cuh"
#include "dart_internal.h"
#include "dart_tc.cuh"

namespace dart {
namespace {

constexpr int GM_BM = 128, GM_BN = 256, GM_BK = 64, GM_STAGES = 4, GM_ACC = 2, GM_THREADS = 192;
constexpr uint32_t GM_A_BYTES = GM_BM * GM_BK * 2;   // 16 KB
constexpr uint32_t GM_B_BYTES = GM_BN * GM_BK * 2;   // 32 KB
constexpr uint32_t GM_STAGE_BYTES = GM_A_BYTES + GM_B_BYTES;
constexpr size_t GM_SMEM = 1024 + (size_t)GM_STAGES * GM_STAGE_BYTES + 256;
constexpr uint32_t GM_TMEM_COLS = GM_ACC * GM_BN;
constexpr int GM_GROUP = 16;                        // row blocks per raster group

struct GemmParams {
  int M, N, K;
  int n_mt, n_nt;
  int64_t n_tiles;
  int c_mode;          // DART_GEMM_STORE_F32 / _STORE_BF16 / _ACCUM_F32
  void* C;
  int64_t ldc;         // elements
};

__device__ __forceinline__ void gm_tile(const GemmParams& p, int64_t t, int& mt, int& nt) {
  const int64_t per_group = (int64_t)GM_GROUP * p.n_nt;
  const int g = (int)(t / per_group);
  const int r = (int)(t - (int64_t)g * per_group);
  const int m0 = g * GM_GROUP;
  const int gm = min(GM_GROUP, p.n_mt - m0);
  mt = m0 + r % gm;
  nt = r / gm;
}

template <bool A_MN, bool B_MN>
__global__ void __launch_bounds__(GM_THREADS, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + GM_STAGES * GM_A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + GM_STAGES * GM_STAGE_BYTES);
  uint64_t* empty = full + GM_STAGES;
  uint64_t* tfull = empty + GM_STAGES;
  uint64_t* tempty = tfull + GM_ACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + GM_ACC);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < GM_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < GM_ACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_mbar_init();
    tc::tma_prefetch_desc(&tmA);
    tc::tma_prefetch_desc(&tmB);
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, GM_TMEM_COLS);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  const int KB = (p.K + GM_BK - 1) / GM_BK;

  if (warp == 0) {
    // ---------------------------------------------------------- TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t ph = 0;
      for (int64_t t = blockIdx.x; t < p.n_tiles; t += gridDim.x) {
        int mt, nt;
        gm_tile(p, t, mt, nt);
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&empty[stage], ph ^ 1u);
          mbar_arrive_expect_tx(&full[stage], GM_STAGE_BYTES);
          uint8_t* a = sA + stage * GM_A_BYTES;
          uint8_t* b = sB + stage * GM_B_BYTES;
          if (A_MN) {
            tc::tma_load_2d(a, &tmA, &full[stage], mt * GM_BM, kb * GM_BK);
            tc::tma_load_2d(a + 8192, &tmA, &full[stage], mt * GM_BM + 64, kb * GM_BK);
          } else {
            tc::tma_load_2d(a, &tmA, &full[stage], kb * GM_BK, mt * GM_BM);
          }
          if (B_MN) {
#pragma unroll
            for (int q = 0; q < GM_BN / 64; ++q)
              tc::tma_load_2d(b + q * 8192, &tmB, &full[stage], nt * GM_BN + 64 * q, kb * GM_BK);
          } else {
            tc::tma_load_2d(b, &tmB, &full[stage], kb * GM_BK, nt * GM_BN);
          }
          if (++stage == GM_STAGES) {
            stage = 0;
            ph ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_bf16_f32(GM_BM, GM_BN, A_MN, B_MN);
      constexpr uint32_t a_lbo = A_MN ? 8192u : 16u, b_lbo = B_MN ? 8192u : 16u;
      constexpr uint64_t a_kstep = A_MN ? (2048u >> 4) : (32u >> 4);   // one K step of 16
      constexpr uint64_t b_kstep = B_MN ? (2048u >> 4) : (32u >> 4);
      int stage = 0, acc = 0;
      uint32_t ph = 0, aph = 0;
      for (int64_t t = blockIdx.x; t < p.n_tiles; t += gridDim.x) {
        mbar_wait(&tempty[acc], aph ^ 1u);
        tc::fence_after();
        const uint32_t d_tmem = tmem + (uint32_t)(acc * GM_BN);
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&full[stage], ph);
          tc::fence_after();
          const uint64_t da = tc::smem_desc_sw128(smem_u32(sA + stage * GM_A_BYTES), a_lbo, 1024);
          const uint64_t db = tc::smem_desc_sw128(smem_u32(sB + stage * GM_B_BYTES), b_lbo, 1024);
#pragma unroll
          for (int k = 0; k < GM_BK / 16; ++k)
            tc::umma_bf16(d_tmem, da + a_kstep * k, db + b_kstep * k, idesc, (kb | k) != 0 ? 1u : 0u);
          tc::umma_commit(&empty[stage]);
          if (++stage == GM_STAGES) {
            stage = 0;
            ph ^= 1u;
          }
        }
        tc::umma_commit(&tfull[acc]);
        if (++acc == GM_ACC) {
          acc = 0;
          aph ^= 1u;
        }
      }
    }
  } else {
    // ---------------------------------------------------------- epilogue
    const int q = warp & 3;
    const int r = q * 32 + lane;
    int acc = 0;
    uint32_t aph = 0;
    for (int64_t t = blockIdx.x; t < p.n_tiles; t += gridDim.x) {
      int mt, nt;
      gm_tile(p, t, mt, nt);
      mbar_wait(&tfull[acc], aph);
      tc::fence_after();
      const int64_t m = (int64_t)mt * GM_BM + r;
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * GM_BN);
#pragma unroll 1
      for (int j = 0; j < GM_BN / 32; ++j) {
        float x[32];
        tc::tmem_ld32(tbase + (uint32_t)(j * 32), x);
        const int64_t n0 = (int64_t)nt * GM_BN + j * 32;
        if (m >= p.M || n0 >= p.N) continue;
        if (p.c_mode == DART_GEMM_STORE_BF16) {
          __nv_bfloat16* c = reinterpret_cast<__nv_bfloat16*>(p.C) + m * p.ldc + n0;
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            if (n0 + i + 8 <= p.N) {
              *reinterpret_cast<uint4*>(c + i) = make_uint4(pack_bf16x2(x[i], x[i + 1]), pack_bf16x2(x[i + 2], x[i + 3]),
                                                            pack_bf16x2(x[i + 4], x[i + 5]),
                                                            pack_bf16x2(x[i + 6], x[i + 7]));
            }
          }
        } else {
          float* c = reinterpret_cast<float*>(p.C) + m * p.ldc + n0;
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            if (n0 + i + 4 <= p.N) {
              float4 v = make_float4(x[i], x[i + 1], x[i + 2], x[i + 3]);
              if (p.c_mode == DART_GEMM_ACCUM_F32) {
                const float4 o = *reinterpret_cast<const float4*>(c + i);
                v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
              }
              *reinterpret_cast<float4*>(c + i) = v;
            }
          }
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive1(&tempty[acc]);
      if (++acc == GM_ACC) {
        acc = 0;
        aph ^= 1u;
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after();
    tc::tmem_dealloc(tmem, GM_TMEM_COLS);
  }
}

// ---------------------------------------------------------------- CTA-pair variant
// cta_group::2: a 2-CTA cluster computes a 256 x 256 tile -- each CTA stages
// its 128 rows of A and its 128 rows of B (K-major, 6 stages of 32 KB), the
// pair leader issues tcgen05.mma.cta_group::2 (M = 256, N = 256) and each CTA
// reads its 128 accumulator rows from its own TMEM.  Per SM this halves the
// shared-memory / L2 operand traffic of the B panel.
// DART_GEMM_CST = 1: the epilogue transposes each warp's 32 rows x 32 columns
// through shared memory and writes whole 128-byte row segments (8 lanes per
// row) instead of one 16-byte piece of 32 different rows per store -- the
// thread-per-row stores touched every L2 sector twice (ncu: 2x the output
// bytes crossed L1 -> L2) and, for the single-accumulator 256 x 512 tile,
// kept the tensor pipe idle 40% of the time.
#ifndef DART_GEMM_CST
#define DART_GEMM_CST 1
#endif
// NW = 2 ("wide"): the pair computes a 256 x 512 tile -- each CTA stages 128
// rows of A and 2 x 128 rows of B per stage, the leader issues two N = 256
// MMAs per K step into the two halves of one 512-column accumulator -- so a
// tile moves (256 + 512) K rows from L2 per 2x the flops: 3/4 of the NW = 1
// operand traffic (ncu: our 256 x 256 pair kernel reads the theoretical
// 70 GB through L2 for z = h W^T, cuBLAS 52 GB), at the price of a single
// accumulator (the epilogue no longer overlaps the next tile's MMAs).
template <int NW> struct G2 {
  static constexpr int STAGES = NW == 1 ? 6 : 4;
  static constexpr int ACC = NW == 1 ? 2 : 1;
  static constexpr int BN = 256 * NW;                       // tile N (pair)
  static constexpr uint32_t A_BYTES = 128 * GM_BK * 2;      // per CTA per stage
  static constexpr uint32_t B_HALF = 128 * GM_BK * 2;       // one N = 256 MMA's share of B per CTA
  static constexpr uint32_t B_BYTES = B_HALF * NW;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr size_t SMEM = 1024 + (size_t)STAGES * STAGE_BYTES + 256;
  // epilogue warps: 4 per 256 accumulator columns (NW = 2: two groups drain
  // the two halves of the single accumulator at the same time); with the
  // coalesced epilogue (DART_GEMM_CST) 4 warps that stage each 32 x 32 block
  // through shared memory (4.5 KB per warp)
  static constexpr int EPI_WARPS = DART_GEMM_CST ? 4 : 4 * NW;
  static constexpr int THREADS = 64 + 32 * EPI_WARPS;
  static constexpr uint32_t EPI_STRIDE = 36;                          // floats per staged row (16 B aligned)
  static constexpr size_t EPI_BYTES = DART_GEMM_CST ? (size_t)EPI_WARPS * 32 * EPI_STRIDE * 4 : 0;
  static constexpr size_t SMEM_ALL = SMEM + EPI_BYTES;
};

__device__ __forceinline__ uint32_t g2_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t g2_cluster_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t g2_cluster_count() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void g2_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void g2_tile(const GemmParams& p, int64_t t, int& mt, int& nt) {
  // p.n_mt counts 256-row pair tiles here
  gm_tile(p, t, mt, nt);
}

// MC = 2: a 4-CTA cluster = two CTA pairs on adjacent N tiles of the same M
// tile; each 128-row A block is loaded once for both pairs (each pair's CTA
// loads 64 of its rows and multicasts them to its counterpart in the other
// pair), so a pair reads (128 + 256) instead of (256 + 256) rows per stage
// from L2.  Stage slots are freed only when BOTH pairs' MMAs have read them
// (empty barriers count the two leaders' commits).
template <bool A_MN, bool B_MN, int NW, int MC = 1>
__global__ void __launch_bounds__(G2<NW>::THREADS, 1)
    gemm_bf16_2sm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                         const GemmParams p) {
  static_assert(MC == 1 || NW == 1, "multicast pairs use 256 x 256 tiles");
  // MC = 3: the same with the roles swapped -- the two pairs sit on adjacent
  // M tiles of the same N tile and the B block is the one multicast
  using C2 = G2<NW>;
  constexpr int G2_STAGES = C2::STAGES, G2_ACC = C2::ACC, G2_BN = C2::BN;
  constexpr uint32_t G2_A_BYTES = C2::A_BYTES, G2_B_BYTES = C2::B_BYTES, G2_STAGE_BYTES = C2::STAGE_BYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + G2_STAGES * G2_A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + G2_STAGES * G2_STAGE_BYTES);
  uint64_t* empty = full + G2_STAGES;
  uint64_t* tfull = empty + G2_STAGES;
  uint64_t* tempty = tfull + G2_ACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + G2_ACC);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = g2_rank();
  const uint32_t rank = crank & 1u;            // rank within the CTA pair
  const uint32_t pr = crank >> 1;              // pair index within the cluster (MC = 2)
  const bool leader = rank == 0;
  const uint16_t pair_mask = (uint16_t)(0x3u << (2 * pr));
  if (threadIdx.x == 0) {
    for (int s = 0; s < G2_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MC >= 2 ? 2 : 1);   // one commit per pair that reads the slot
    }
    for (int a = 0; a < G2_ACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * C2::EPI_WARPS);   // epilogue warps x 2 CTAs (leader's copy is the one used)
    }
    fence_mbar_init();
    tc::tma_prefetch_desc(&tmA);
    tc::tma_prefetch_desc(&tmB);
  }
  if (warp == 1) tc::tmem_alloc_2sm(tmem_slot, GM_TMEM_COLS);
  tc::fence_before();
  __syncthreads();
  g2_cluster_sync();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  const int KB = (p.K + GM_BK - 1) / GM_BK;
  const int64_t cid = g2_cluster_id(), ncl = g2_cluster_count();

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t ph = 0;
      for (int64_t t = cid; t < p.n_tiles; t += ncl) {
        int mt, nt;
        g2_tile(p, t, mt, nt);
        if (MC == 2) nt = 2 * nt + (int)pr;      // p.n_nt counts pairs of N tiles here
        if (MC == 3) mt = 2 * mt + (int)pr;      // p.n_mt counts pairs of M tiles here
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&empty[stage], ph ^ 1u);
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * G2_STAGE_BYTES);   // both CTAs' bytes
          uint8_t* a = sA + stage * G2_A_BYTES;
          uint8_t* b = sB + stage * G2_B_BYTES;
          const int m0 = mt * 256 + 128 * (int)rank;
          if (MC == 2) {                         // this CTA's 64-row half of the block, to both pairs
            const uint16_t mmask = (uint16_t)((1u << rank) | (1u << (rank + 2)));
            if (A_MN)
              tc::tma_load_2d_2sm_mc(a + 8192 * pr, &tmA, &full[stage], m0 + 64 * (int)pr, kb * GM_BK, mmask);
            else
              tc::tma_load_2d_2sm_mc(a + 8192 * pr, &tmA, &full[stage], kb * GM_BK, m0 + 64 * (int)pr, mmask);
          } else if (A_MN) {
            tc::tma_load_2d_2sm(a, &tmA, &full[stage], m0, kb * GM_BK);
            tc::tma_load_2d_2sm(a + 8192, &tmA, &full[stage], m0 + 64, kb * GM_BK);
          } else {
            tc::tma_load_2d_2sm(a, &tmA, &full[stage], kb * GM_BK, m0);
          }
#pragma unroll
          for (int hh = 0; hh < NW; ++hh) {   // B rows of MMA hh: [nt*BN + 256 hh, +256), this CTA's 128
            const int n0 = nt * G2_BN + 256 * hh + 128 * (int)rank;
            uint8_t* bh = b + hh * C2::B_HALF;
            if (MC == 3) {                       // this CTA's 64-row half of the B block, to both pairs
              const uint16_t mmask = (uint16_t)((1u << rank) | (1u << (rank + 2)));
              if (B_MN)
                tc::tma_load_2d_2sm_mc(bh + 8192 * pr, &tmB, &full[stage], n0 + 64 * (int)pr, kb * GM_BK, mmask);
              else
                tc::tma_load_2d_2sm_mc(bh + 8192 * pr, &tmB, &full[stage], kb * GM_BK, n0 + 64 * (int)pr, mmask);
            } else if (B_MN) {
              tc::tma_load_2d_2sm(bh, &tmB, &full[stage], n0, kb * GM_BK);
              tc::tma_load_2d_2sm(bh + 8192, &tmB, &full[stage], n0 + 64, kb * GM_BK);
            } else {
              tc::tma_load_2d_2sm(bh, &tmB, &full[stage], kb * GM_BK, n0);
            }
          }
          if (++stage == G2_STAGES) {
            stage = 0;
            ph ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      constexpr uint32_t idesc = tc::idesc_bf16_f32(256, 256, A_MN, B_MN);
      constexpr uint32_t a_lbo = A_MN ? 8192u : 16u, b_lbo = B_MN ? 8192u : 16u;
      constexpr uint64_t a_kstep = A_MN ? (2048u >> 4) : (32u >> 4);
      constexpr uint64_t b_kstep = B_MN ? (2048u >> 4) : (32u >> 4);
      int stage = 0, acc = 0;
      uint32_t ph = 0, aph = 0;
      for (int64_t t = cid; t < p.n_tiles; t += ncl) {
        mbar_wait(&tempty[acc], aph ^ 1u);
        tc::fence_after();
        const uint32_t d_tmem = tmem + (uint32_t)(acc * G2_BN);
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&full[stage], ph);
          tc::fence_after();
          const uint64_t da = tc::smem_desc_sw128(smem_u32(sA + stage * G2_A_BYTES), a_lbo, 1024);
#pragma unroll
          for (int hh = 0; hh < NW; ++hh) {
            const uint64_t db = tc::smem_desc_sw128(smem_u32(sB + stage * G2_B_BYTES + hh * C2::B_HALF), b_lbo, 1024);
#pragma unroll
            for (int k = 0; k < GM_BK / 16; ++k)
              tc::umma_bf16_2sm(d_tmem + 256 * hh, da + a_kstep * k, db + b_kstep * k, idesc,
                                (kb | k) != 0 ? 1u : 0u);
          }
          tc::umma_commit_2sm(&empty[stage], MC >= 2 ? (uint16_t)0xF : pair_mask);
          if (++stage == G2_STAGES) {
            stage = 0;
            ph ^= 1u;
          }
        }
        tc::umma_commit_2sm(&tfull[acc], pair_mask);
        if (++acc == G2_ACC) {
          acc = 0;
          aph ^= 1u;
        }
      }
    }
  } else {
    const int q = warp & 3;                     // TMEM lane quadrant this warp may access
    const int half = DART_GEMM_CST ? 0 : (warp - 2) >> 2;   // column group: [256 half, 256 half + 256)
    constexpr int EPI_COLS = DART_GEMM_CST ? G2_BN : 256;   // columns this warp drains per tile
    const int r = q * 32 + lane;
    float* T = reinterpret_cast<float*>(smem + G2_STAGES * G2_STAGE_BYTES + 256) + (warp - 2) * (32 * C2::EPI_STRIDE);
    int acc = 0;
    uint32_t aph = 0;
    for (int64_t t = cid; t < p.n_tiles; t += ncl) {
      int mt, nt;
      g2_tile(p, t, mt, nt);
      if (MC == 2) nt = 2 * nt + (int)pr;
      if (MC == 3) mt = 2 * mt + (int)pr;
      mbar_wait(&tfull[acc], aph);
      tc::fence_after();
      const int64_t m = (int64_t)mt * 256 + 128 * rank + r;
      const int64_t mrow0 = (int64_t)mt * 256 + 128 * rank + q * 32;   // this warp's first row
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * G2_BN + 256 * half);
#pragma unroll 1
      for (int j = 0; j < EPI_COLS / 32; ++j) {
        float x[32];
        tc::tmem_ld32(tbase + (uint32_t)(j * 32), x);
        const int64_t n0 = (int64_t)nt * G2_BN + 256 * half + j * 32;
        if (DART_GEMM_CST) {
          if (n0 >= p.N) continue;
          // stage: lane = row
#pragma unroll
          for (int g = 0; g < 8; ++g)
            *reinterpret_cast<float4*>(T + lane * C2::EPI_STRIDE + 4 * g) =
                make_float4(x[4 * g], x[4 * g + 1], x[4 * g + 2], x[4 * g + 3]);
          __syncwarp();
          // write: 8 lanes per row (4 columns each), 4 rows per instruction
          const int col = 4 * (lane & 7);
          const int64_t n = n0 + col;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int ri = 4 * k + (lane >> 3);
            const int64_t mm = mrow0 + ri;
            if (mm < p.M && n + 4 <= p.N) {
              float4 v = *reinterpret_cast<const float4*>(T + ri * C2::EPI_STRIDE + col);
              if (p.c_mode == DART_GEMM_STORE_BF16) {
                *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(p.C) + mm * p.ldc + n) =
                    make_uint2(pack_bf16x2(v.x, v.y), pack_bf16x2(v.z, v.w));
              } else {
                float* c = reinterpret_cast<float*>(p.C) + mm * p.ldc + n;
                if (p.c_mode == DART_GEMM_ACCUM_F32) {
                  const float4 o = *reinterpret_cast<const float4*>(c);
                  v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
                }
                *reinterpret_cast<float4*>(c) = v;
              }
            }
          }
          __syncwarp();
          continue;
        }
        if (m >= p.M || n0 >= p.N) continue;
        if (p.c_mode == DART_GEMM_STORE_BF16) {
          __nv_bfloat16* c = reinterpret_cast<__nv_bfloat16*>(p.C) + m * p.ldc + n0;
#pragma unroll
          for (int i = 0; i < 32; i += 8)
            if (n0 + i + 8 <= p.N)
              *reinterpret_cast<uint4*>(c + i) = make_uint4(pack_bf16x2(x[i], x[i + 1]), pack_bf16x2(x[i + 2], x[i + 3]),
                                                            pack_bf16x2(x[i + 4], x[i + 5]),
                                                            pack_bf16x2(x[i + 6], x[i + 7]));
        } else {
          float* c = reinterpret_cast<float*>(p.C) + m * p.ldc + n0;
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            if (n0 + i + 4 <= p.N) {
              float4 v = make_float4(x[i], x[i + 1], x[i + 2], x[i + 3]);
              if (p.c_mode == DART_GEMM_ACCUM_F32) {
                const float4 o = *reinterpret_cast<const float4*>(c + i);
                v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
              }
              *reinterpret_cast<float4*>(c + i) = v;
            }
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_remote(&tempty[acc], crank & ~1u);   // the pair leader's accumulator-empty barrier
      if (++acc == G2_ACC) {
        acc = 0;
        aph ^= 1u;
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  g2_cluster_sync();
  if (warp == 1) {
    tc::fence_after();
    tc::tmem_dealloc_2sm(tmem, GM_TMEM_COLS);
  }
}

template <bool A_MN, bool B_MN, int NW, int MC = 1>
cudaError_t launch_gemm_2sm(const CUtensorMap& ta, const CUtensorMap& tb, GemmParams p, int num_sms,
                            cudaStream_t st) {
  auto kern = gemm_bf16_2sm_kernel<A_MN, B_MN, NW, MC>;
  constexpr size_t smem = G2<NW>::SMEM_ALL;
  constexpr int CL = MC >= 2 ? 4 : 2;        // CTAs per cluster
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  p.n_mt = (p.M + 255) / 256;
  p.n_nt = (p.N + G2<NW>::BN - 1) / G2<NW>::BN;
  if (MC == 2) p.n_nt = (p.n_nt + 1) / 2;    // cluster items: pairs of N tiles
  if (MC == 3) p.n_mt = (p.n_mt + 1) / 2;    // cluster items: pairs of M tiles
  p.n_tiles = (int64_t)p.n_mt * p.n_nt;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(G2<NW>::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int64_t clusters = num_sms / CL;
  cfg.gridDim = dim3((unsigned)(CL * clusters));
  int nclu = 0;   // persistent clusters: never more than can be co-resident
  if (cudaOccupancyMaxActiveClusters(&nclu, kern, &cfg) == cudaSuccess && nclu > 0 && nclu < clusters) clusters = nclu;
  (void)cudaGetLastError();
  if (clusters > p.n_tiles) clusters = p.n_tiles;
  cfg.gridDim = dim3((unsigned)(CL * clusters));
  return cudaLaunchKernelEx(&cfg, kern, ta, tb, p);
}

template <bool A_MN, bool B_MN>
cudaError_t launch_gemm_t(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p, int num_sms,
                          cudaStream_t st) {
  auto kern = gemm_bf16_kernel<A_MN, B_MN>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GM_SMEM);
  if (e != cudaSuccess) return e;   // (per call: the attribute is per device)
  const int64_t grid = p.n_tiles < num_sms ? p.n_tiles : num_sms;
  kern<<<(unsigned)grid, GM_THREADS, GM_SMEM, st>>>(ta, tb, p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_gemm_bf16(const void* A, bool a_mn, int64_t lda, const void* B, bool b_mn, int64_t ldb, void* C,
                             int c_mode, int64_t ldc, int64_t M, int64_t N, int64_t K, int num_sms, cudaStream_t st) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  CUtensorMap ta, tb;
  const bool ok_a = a_mn ? tc::make_map_bf16(&ta, A, K, M, lda, 64, 64) : tc::make_map_bf16(&ta, A, M, K, lda, 64, GM_BM);
  const bool ok_b = b_mn ? tc::make_map_bf16(&tb, B, K, N, ldb, 64, 64) : tc::make_map_bf16(&tb, B, N, K, ldb, 64, GM_BN);
  if (!ok_a || !ok_b) return cudaErrorInvalidValue;
  GemmParams p;
  p.M = (int)M; p.N = (int)N; p.K = (int)K;
  p.n_mt = (int)((M + GM_BM - 1) / GM_BM);
  p.n_nt = (int)((N + GM_BN - 1) / GM_BN);
  p.n_tiles = (int64_t)p.n_mt * p.n_nt;
  p.c_mode = c_mode;
  p.C = C;
  p.ldc = ldc;
  const char* e2 = getenv("DART_GEMM_2SM");
  if (!(e2 && e2[0] == '0')) {   // default: CTA-pair kernel (each CTA stages 128 rows of A and of B);
                                 // 1264-1285 vs 1135 TFLOP/s sustained on [8192 x 3584] x [3584 x 152064]
    CUtensorMap ta2, tb2;
    const bool ok2a = a_mn ? tc::make_map_bf16(&ta2, A, K, M, lda, 64, 64) : tc::make_map_bf16(&ta2, A, M, K, lda, 64, 128);
    const bool ok2b = b_mn ? tc::make_map_bf16(&tb2, B, K, N, ldb, 64, 64) : tc::make_map_bf16(&tb2, B, N, K, ldb, 64, 128);
    if (!ok2a || !ok2b) return cudaErrorInvalidValue;
    // default: 4-CTA multicast clusters for narrow N (the LM head's dh = dz W and
    // dW = dz^T h: N = d), CTA pairs otherwise (z = h W^T, N = V) -- measured per
    // shape in a sustained loop (profiles/r01_gemm_vs_cublas.md)
    const int64_t n_nt_pair = (N + 255) / 256;
    const bool use_mc = (e2 && e2[0] == '4') || (!e2 && n_nt_pair <= 64 && M >= 1024);
    if (use_mc) {                 // 4-CTA clusters: A blocks multicast to two pairs (see MC)
      CUtensorMap ta4;
      if (!(a_mn ? tc::make_map_bf16(&ta4, A, K, M, lda, 64, 64) : tc::make_map_bf16(&ta4, A, M, K, lda, 64, 64)))
        return cudaErrorInvalidValue;
      if (a_mn && b_mn) return launch_gemm_2sm<true, true, 1, 2>(ta4, tb2, p, num_sms, st);
      if (a_mn) return launch_gemm_2sm<true, false, 1, 2>(ta4, tb2, p, num_sms, st);
      if (b_mn) return launch_gemm_2sm<false, true, 1, 2>(ta4, tb2, p, num_sms, st);
      return launch_gemm_2sm<false, false, 1, 2>(ta4, tb2, p, num_sms, st);
    }
    if (e2 && e2[0] == '5') {     // 4-CTA clusters: B blocks multicast to two pairs (opt-in, MC = 3)
      CUtensorMap tb4;
      if (!(b_mn ? tc::make_map_bf16(&tb4, B, K, N, ldb, 64, 64) : tc::make_map_bf16(&tb4, B, N, K, ldb, 64, 64)))
        return cudaErrorInvalidValue;
      if (a_mn && b_mn) return launch_gemm_2sm<true, true, 1, 3>(ta2, tb4, p, num_sms, st);
      if (a_mn) return launch_gemm_2sm<true, false, 1, 3>(ta2, tb4, p, num_sms, st);
      if (b_mn) return launch_gemm_2sm<false, true, 1, 3>(ta2, tb4, p, num_sms, st);
      return launch_gemm_2sm<false, false, 1, 3>(ta2, tb4, p, num_sms, st);
    }
    if (e2 && e2[0] == '2') {     // 256 x 512 pair tiles (opt-in, see G2<2>)
      if (a_mn && b_mn) return launch_gemm_2sm<true, true, 2>(ta2, tb2, p, num_sms, st);
      if (a_mn) return launch_gemm_2sm<true, false, 2>(ta2, tb2, p, num_sms, st);
      if (b_mn) return launch_gemm_2sm<false, true, 2>(ta2, tb2, p, num_sms, st);
      return launch_gemm_2sm<false, false, 2>(ta2, tb2, p, num_sms, st);
    }
    if (a_mn && b_mn) return launch_gemm_2sm<true, true, 1>(ta2, tb2, p, num_sms, st);
    if (a_mn) return launch_gemm_2sm<true, false, 1>(ta2, tb2, p, num_sms, st);
    if (b_mn) return launch_gemm_2sm<false, true, 1>(ta2, tb2, p, num_sms, st);
    return launch_gemm_2sm<false, false, 1>(ta2, tb2, p, num_sms, st);
  }
  if (a_mn && b_mn) return launch_gemm_t<true, true>(ta, tb, p, num_sms, st);
  if (a_mn) return launch_gemm_t<true, false>(ta, tb, p, num_sms, st);
  if (b_mn) return launch_gemm_t<false, true>(ta, tb, p, num_sms, st);
  return launch_gemm_t<false, false>(ta, tb, p, num_sms, st);
}

}  // namespace dart
