// dart_lmhead.cu -- SURVEY §8(f) NEXT #3: the LM head fused into the loss
// pass's forward sweep.
//
// z_{t,v} = sum_k h_{t,k} W_{v,k} (the logits whose softmax / T is
// pi_theta(a|h,s), Eq. 1) is computed on the 5th-generation
// tensor cores: tcgen05.mma (bf16 x bf16 -> fp32) with both operands staged
// into shared memory by TMA (128-byte swizzle) and the accumulator in TMEM.
// The epilogue reads each 128 x 256 accumulator tile back with tcgen05.ld and
// folds it straight into the per-row online softmax statistics (m, s, u) of
// the log2 domain (the same (m, s, u) algebra as the logits sweep
// entropy) plus the target's logit -- the [T, V] logits never touch memory.
//
// Work item = (128-row block mb, vocabulary chunk nc of LM_NT_PER_CHUNK
// 256-column tiles); each item leaves one (m, s, u) partial per row, folded in
// chunk order by lmhead_combine_kernel (dart_fwd.cu).  Persistent CTAs (one
// per SM) walk the items in a super-column raster: LM_GROUP_NC chunks x all
// row blocks, chunks innermost, so the ~148 concurrently active items touch
// ~37 hidden blocks and ~4 weight chunks at a time (L2 resident).
//
// Warp roles (192 threads): warp 0 = TMA producer (one lane), warp 1 = TMEM
// allocator + MMA issuer (one lane), warps 2..5 = epilogue (warp w reads TMEM
// lanes 32*(w%4) .. +31, i.e. accumulator rows).  Pipelines: LM_STAGES smem
// stages (full/empty mbarriers), two TMEM accumulators of 256 fp32 columns
// (tfull/tempty), so the epilogue of tile i overlaps the MMAs of tile i+1.
#include <cstdio>
#include <cstdlib>

#include "dart_common.cuh"
#include "dart_internal.h"
#include "dart_tc.cuh"

namespace dart {
namespace {

constexpr int LM_BM = 128, LM_BN = 256, LM_BK = 64, LM_STAGES = 4, LM_ACC = 2;
constexpr int LM_THREADS = 192;
constexpr uint32_t LM_A_BYTES = LM_BM * LM_BK * 2;   // 16 KB
constexpr uint32_t LM_B_BYTES = LM_BN * LM_BK * 2;   // 32 KB
constexpr uint32_t LM_STAGE_BYTES = LM_A_BYTES + LM_B_BYTES;
constexpr size_t LM_SMEM = 1024 + (size_t)LM_STAGES * LM_STAGE_BYTES + 256;
constexpr uint32_t LM_TMEM_COLS = LM_ACC * LM_BN;     // 512: the whole TMEM of the SM
constexpr float LM_MASKED = -1.0e30f;                 // raw logit for columns >= V
// CTA-pair mode (cta_group::2): 256-row items, each CTA stages 128 rows of h
// and 128 of the 256 W rows of a tile, 6 stages of 32 KB
constexpr int LM2_STAGES = 6;
constexpr uint32_t LM2_A_BYTES = 128 * LM_BK * 2, LM2_B_BYTES = 128 * LM_BK * 2;
constexpr uint32_t LM2_STAGE_BYTES = LM2_A_BYTES + LM2_B_BYTES;
constexpr size_t LM2_SMEM = 1024 + (size_t)LM2_STAGES * LM2_STAGE_BYTES + 256;

using tc::fence_after;
using tc::fence_before;
using tc::tma_load_2d;
using tc::tma_prefetch_desc;
using tc::tmem_ld32;
using tc::umma_commit;

constexpr uint32_t LM_IDESC = tc::idesc_bf16_f32(LM_BM, LM_BN, false, false);

__device__ __forceinline__ uint64_t sw128_kmajor_desc(uint32_t saddr) { return tc::smem_desc_sw128(saddr, 16, 1024); }
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
  tc::umma_bf16(tmem_d, da, db, LM_IDESC, accumulate);
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) { tc::mbar_arrive1(bar); }
__device__ __forceinline__ void tc_fence_after() { fence_after(); }
__device__ __forceinline__ void tc_fence_before() { fence_before(); }

// work item -> (row block, vocabulary chunk): super-columns of group_nc chunks,
// row blocks outer, chunks inner
__device__ __forceinline__ void lm_item(const LmParams& p, int64_t it, int& mb, int& nc) {
  const int64_t per_sc = (int64_t)p.n_mb * p.group_nc;
  const int sc = (int)(it / per_sc);
  const int rem = (int)(it - (int64_t)sc * per_sc);
  const int gn = min(p.group_nc, p.n_nc - sc * p.group_nc);
  mb = rem / gn;
  nc = sc * p.group_nc + rem % gn;
}

__device__ __forceinline__ uint32_t lm_cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t lm_cluster_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t lm_cluster_count() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void lm_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// PAIR = false: one CTA per 128-row item (cta_group::1).  PAIR = true: a 2-CTA
// cluster per 256-row item (cta_group::2; p.n_mb counts 256-row blocks).
template <bool PAIR>
__global__ void __launch_bounds__(LM_THREADS, 1)
    lmhead_fwd_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const LmParams p) {
  constexpr int STAGES = PAIR ? LM2_STAGES : LM_STAGES;
  constexpr uint32_t A_BYTES = PAIR ? LM2_A_BYTES : LM_A_BYTES, B_BYTES = PAIR ? LM2_B_BYTES : LM_B_BYTES;
  constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr int IBM = PAIR ? 256 : LM_BM;           // rows per item
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + LM_ACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + LM_ACC);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = PAIR ? lm_cluster_rank() : 0u;
  const bool leader = rank == 0;
  const int64_t unit0 = PAIR ? (int64_t)lm_cluster_id() : (int64_t)blockIdx.x;
  const int64_t nunits = PAIR ? (int64_t)lm_cluster_count() : (int64_t)gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < LM_ACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], PAIR ? 8 : 4);   // epilogue warps (x 2 CTAs in pair mode, leader's copy used)
    }
    fence_mbar_init();
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1) {
    if (PAIR) tc::tmem_alloc_2sm(tmem_slot, LM_TMEM_COLS);
    else tc::tmem_alloc(tmem_slot, LM_TMEM_COLS);
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) lm_cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int KB = (p.K + LM_BK - 1) / LM_BK;

  if (warp == 0) {
    // ---------------------------------------------------------- TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t ph = 0;
      for (int64_t it = unit0; it < p.n_items; it += nunits) {
        int mb, nc;
        lm_item(p, it, mb, nc);
        const int nt0 = nc * p.nt_per_chunk, nt1 = min(nt0 + p.nt_per_chunk, p.n_nt);
        for (int nt = nt0; nt < nt1; ++nt) {
          for (int kb = 0; kb < KB; ++kb) {
            mbar_wait(&empty[stage], ph ^ 1u);
            if (PAIR) {
              if (leader) mbar_arrive_expect_tx(&full[stage], 2 * STAGE_BYTES);   // both CTAs' bytes
              tc::tma_load_2d_2sm(sA + stage * A_BYTES, &tmA, &full[stage], kb * LM_BK, mb * IBM + 128 * (int)rank);
              tc::tma_load_2d_2sm(sB + stage * B_BYTES, &tmB, &full[stage], kb * LM_BK, nt * LM_BN + 128 * (int)rank);
            } else {
              mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
              tma_load_2d(sA + stage * A_BYTES, &tmA, &full[stage], kb * LM_BK, mb * LM_BM);
              tma_load_2d(sB + stage * B_BYTES, &tmB, &full[stage], kb * LM_BK, nt * LM_BN);
            }
            if (++stage == STAGES) {
              stage = 0;
              ph ^= 1u;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    if (lane == 0 && leader) {
      int stage = 0, acc = 0;
      uint32_t ph = 0, aph = 0;
      for (int64_t it = unit0; it < p.n_items; it += nunits) {
        int mb, nc;
        lm_item(p, it, mb, nc);
        const int nt0 = nc * p.nt_per_chunk, nt1 = min(nt0 + p.nt_per_chunk, p.n_nt);
        for (int nt = nt0; nt < nt1; ++nt) {
          mbar_wait(&tempty[acc], aph ^ 1u);
          tc_fence_after();
          const uint32_t d_tmem = tmem + (uint32_t)(acc * LM_BN);
          for (int kb = 0; kb < KB; ++kb) {
            mbar_wait(&full[stage], ph);
            tc_fence_after();
            const uint64_t da = sw128_kmajor_desc(smem_u32(sA + stage * A_BYTES));
            const uint64_t db = sw128_kmajor_desc(smem_u32(sB + stage * B_BYTES));
#pragma unroll
            for (int k = 0; k < LM_BK / 16; ++k) {  // UMMA_K = 16 bf16 = 32 B along the swizzled row
              if (PAIR)
                tc::umma_bf16_2sm(d_tmem, da + (uint64_t)(2 * k), db + (uint64_t)(2 * k),
                                  tc::idesc_bf16_f32(256, LM_BN, false, false), (kb | k) != 0 ? 1u : 0u);
              else
                umma_bf16(d_tmem, da + (uint64_t)(2 * k), db + (uint64_t)(2 * k), (kb | k) != 0 ? 1u : 0u);
            }
            if (PAIR) tc::umma_commit_2sm(&empty[stage], 0x3);   // frees the smem stage in both CTAs
            else umma_commit(&empty[stage]);        // frees the smem stage when these MMAs retire
            if (++stage == STAGES) {
              stage = 0;
              ph ^= 1u;
            }
          }
          if (PAIR) tc::umma_commit_2sm(&tfull[acc], 0x3);
          else umma_commit(&tfull[acc]);            // accumulator tile complete
          if (++acc == LM_ACC) {
            acc = 0;
            aph ^= 1u;
          }
        }
      }
    }
  } else {
    // ---------------------------------------------------------- epilogue
    const int q = warp & 3;            // TMEM lane quarter this warp may access
    const int r = q * 32 + lane;       // accumulator row of this thread
    const float c2 = p.c2;
    int acc = 0;
    uint32_t aph = 0;
    for (int64_t it = unit0; it < p.n_items; it += nunits) {
      int mb, nc;
      lm_item(p, it, mb, nc);
      const int nt0 = nc * p.nt_per_chunk, nt1 = min(nt0 + p.nt_per_chunk, p.n_nt);
      const int64_t row = (int64_t)mb * IBM + 128 * (int64_t)rank + r;
      const bool valid = row < p.T_loc;
      const int64_t y = valid ? (int64_t)p.target[row] : -1;
      float m_run = LM_MASKED;         // running max of z*c2 (log2 units); any real logit exceeds it
      double S = 0.0, U = 0.0;         // sum 2^(x-m), sum 2^(x-m)(x-m)
      float zy = 0.0f;
      for (int nt = nt0; nt < nt1; ++nt) {
        mbar_wait(&tfull[acc], aph);
        tc_fence_after();
        const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * LM_BN);
#pragma unroll 1
        for (int j = 0; j < LM_BN / 32; ++j) {
          float x[32];
          tmem_ld32(tbase + (uint32_t)(j * 32), x);
          const int64_t col0 = (int64_t)nt * LM_BN + j * 32;
          if (col0 + 32 > p.V) {       // vocabulary tail (TMA zero-filled columns >= V)
            const int nv = (int)max((int64_t)0, p.V - col0);
#pragma unroll
            for (int i = 0; i < 32; ++i) x[i] = (i < nv) ? x[i] : LM_MASKED;
          }
          float mx = x[0];
#pragma unroll
          for (int i = 1; i < 32; ++i) mx = fmaxf(mx, x[i]);
          const float gm = mx * c2;
          if (gm > m_run) {              // exact rescale of (S, U) to the new max
            const float dm = m_run - gm;
            const double f = (double)ex2(dm);
            U = f * (U + S * (double)dm);
            S *= f;
            m_run = gm;
          }
          float s0 = 0.f, s1 = 0.f, u0 = 0.f, u1 = 0.f;
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const float d0 = fmaf(x[i], c2, -m_run), d1 = fmaf(x[i + 1], c2, -m_run);
            const float e0 = ex2(d0), e1 = ex2(d1);
            s0 += e0;
            s1 += e1;
            u0 = fmaf(e0, d0, u0);
            u1 = fmaf(e1, d1, u1);
          }
          S += (double)(s0 + s1);
          U += (double)(u0 + u1);
          const int64_t jy = y - col0;
          if ((uint64_t)jy < 32u) {
            // binary select tree on the bits of jy (a plain x[jy] would put x in local memory)
            float t[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) t[i] = (jy & 16) ? x[i + 16] : x[i];
#pragma unroll
            for (int i = 0; i < 8; ++i) t[i] = (jy & 8) ? t[i + 8] : t[i];
#pragma unroll
            for (int i = 0; i < 4; ++i) t[i] = (jy & 4) ? t[i + 4] : t[i];
#pragma unroll
            for (int i = 0; i < 2; ++i) t[i] = (jy & 2) ? t[i + 2] : t[i];
            zy = (jy & 1) ? t[1] : t[0];
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (PAIR) tc::mbar_arrive_remote(&tempty[acc], 0);   // the leader's accumulator-empty barrier
          else mbar_arrive(&tempty[acc]);
        }
        if (++acc == LM_ACC) {
          acc = 0;
          aph ^= 1u;
        }
      }
      if (valid) {
        const int64_t idx = row * p.n_nc + nc;
        p.part_m[idx] = m_run;
        p.part_s[idx] = S;
        p.part_u[idx] = U;
        if (y >= (int64_t)nt0 * LM_BN && y < (int64_t)nt1 * LM_BN) p.zy[row] = zy;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (PAIR) lm_cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    if (PAIR) tc::tmem_dealloc_2sm(tmem, LM_TMEM_COLS);
    else tc::tmem_dealloc(tmem, LM_TMEM_COLS);
  }
}

}  // namespace

cudaError_t launch_lmhead(const void* hidden, int64_t ld_h, const void* weight, int64_t ld_w, const LmParams& p,
                          int num_sms, cudaStream_t st) {
  if (p.T_loc <= 0 || p.n_items <= 0) return cudaSuccess;
  CUtensorMap tmA, tmB;
  const char* e2 = getenv("DART_LMHEAD_2SM");
  if (e2 && e2[0] == '1') {
    // opt-in: CTA pairs (cta_group::2), 256-row items, 128-row boxes for h and W.  Correct
    // (tests pass) but measured slower in the bench loop: 60-63 ms vs 50 ms, the SM clock
    // falling to 1.0-1.1 GHz under the power cap (vs 1.37 GHz for the 1-CTA kernel)
    if (!tc::make_map_bf16(&tmA, hidden, p.T_loc, p.K, ld_h, LM_BK, 128)) return cudaErrorInvalidValue;
    if (!tc::make_map_bf16(&tmB, weight, p.V, p.K, ld_w, LM_BK, 128)) return cudaErrorInvalidValue;
    auto kern = lmhead_fwd_kernel<true>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LM2_SMEM);
    if (e != cudaSuccess) return e;
    LmParams q = p;
    q.n_mb = (int)((p.T_loc + 255) / 256);
    q.n_items = (int64_t)q.n_mb * q.n_nc;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(LM_THREADS);
    cfg.dynamicSmemBytes = LM2_SMEM;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int64_t pairs = num_sms / 2;
    cfg.gridDim = dim3((unsigned)(2 * pairs));
    int nclu = 0;   // persistent pairs: never more clusters than can be co-resident
    if (cudaOccupancyMaxActiveClusters(&nclu, kern, &cfg) == cudaSuccess && nclu > 0 && nclu < pairs) pairs = nclu;
    (void)cudaGetLastError();
    if (pairs > q.n_items) pairs = q.n_items;
    cfg.gridDim = dim3((unsigned)(2 * pairs));
    return cudaLaunchKernelEx(&cfg, kern, tmA, tmB, q);
  }
  if (!tc::make_map_bf16(&tmA, hidden, p.T_loc, p.K, ld_h, LM_BK, LM_BM)) return cudaErrorInvalidValue;
  if (!tc::make_map_bf16(&tmB, weight, p.V, p.K, ld_w, LM_BK, LM_BN)) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(lmhead_fwd_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)LM_SMEM);
  if (e != cudaSuccess) return e;   // (per call: the attribute is per device)
  const int64_t grid = p.n_items < num_sms ? p.n_items : num_sms;
  lmhead_fwd_kernel<false><<<(unsigned)grid, LM_THREADS, LM_SMEM, st>>>(tmA, tmB, p);
  return cudaGetLastError();
}

}  // namespace dart
