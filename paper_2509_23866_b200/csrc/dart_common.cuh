// dart_common.cuh -- sm_100a device helpers and the internal workspace layout
// shared by the DART kernels (fwd sweep, select, bwd sweep).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/dart_loss.h"

namespace dart {

// ---------------------------------------------------------------- constants
constexpr int KSEG = 8;                 // canonical segments per row (fwd reduction order)
constexpr int CH_BYTES = 4096;          // bulk-copy chunk (one mbarrier transaction)
constexpr int CH_VEC = CH_BYTES / 16;   // 16-byte vectors per chunk
constexpr int VPL = CH_VEC / 32;        // vectors per lane per chunk
constexpr int SPLIT_MAX_ROWS = 16384;   // split-row mode only below this many local rows
// -inf logits are clamped here (exp underflows to 0 and 0*(-1e30) = 0, where
// 0*(-inf) would be NaN); the value is exactly representable in bf16 (0xF14A).
constexpr uint32_t NEG_CLAMP_BF16 = 0xF14Au;
constexpr float NEG_CLAMP = -1.0002555517425873e+30f;  // == bf16 0xF14A as fp32 (0xF14A0000)

constexpr double LOG2E_D = 1.4426950408889634073599;
constexpr double LN2_D = 0.6931471805599453094172;

// ---------------------------------------------------------------- workspace
// Sub-buffers (256 B aligned), identical layout in every call of one pass.
struct WsLayout {
  size_t tok_adv, tok_step, lse2, aux_w, aux_kl, aux_flags, rec, klq;   // [T_loc] (rec: 32 B)
  size_t step_stats;                                                    // [S_loc * NSTAT] f64
  size_t step_cost;                                                     // [S_loc+1] i64
  size_t step_scale;                                                    // [S_loc] f64
  size_t step_chunk;                                                    // [S_loc+1] i64
  size_t part_m, part_s, part_u, row_cnt;                               // split mode [T_loc*KSEG]
  size_t H_glob;                                                        // [S] f32
  size_t grp_traj;                                                      // [G+1] i64 (trajectory CSR of groups)
  size_t grp_keep_step, grp_keep_tok;                                   // [G] i64
  size_t fused_rec;                                                     // [T_loc] 32 B (dart_loss_fused)
  size_t bwd_misc;                                                      // small scratch
  size_t total;
  bool split_alloc;
};

constexpr int NSTAT = 7;  // per-step: sum_w, sum_clip, sum_trunc, sum_adv, sum_adv2, sum_kl, sum_H

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

// 1-D bulk copy global -> shared (TMA engine, SASS UBLKCP), completion counted on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
      "%4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE_%=;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ uint4 lds128(const void* p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(smem_u32(p)));
  return v;
}

// A ring slot is handed back (to the producer warp, or to this warp's own next
// bulk copy) right after the shared loads that read it.  Those loads are
// generic-proxy reads and the refill is an async-proxy (bulk copy) write, so
// the hand-back is preceded by fence.proxy.async: it orders this thread's
// earlier shared accesses before the async proxy's later ones.  (An empty-asm
// "use" of the loaded words does not: ptxas deletes it, and without an
// ordering the refill raced the loads -- seen as rare run-to-run lse jitter
// of the fused update once extra stores congested the MIO queue.  A real
// data dependency also closes it but stalls every chunk on the load latency,
// 2-3% on the sweeps; the fence costs nothing measurable, A/B in
// profiles/r02_ring_fence.md.)
// Start value of a per-lane running maximum (log2 domain) when padding and
// -inf logits are clamped to NEG_CLAMP: NEG_CLAMP * c2 rounded TOWARD ZERO.
// A lane that only ever sees clamped values then gets
// 2^fma(NEG_CLAMP, c2, -m0) = 2^(<= 0) instead of 2^(+half an ulp of ~1.4e30)
// = inf (the round-to-nearest product can sit below the exact one), whose
// product with the fold's zero weight was a NaN row.
__device__ __forceinline__ float clamp_max0(float c2) { return __fmul_rz(NEG_CLAMP, c2); }

__device__ __forceinline__ void fence_reads_before_refill() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void stg128_cs(void* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// packed bf16x2 max (NaN-propagating) -- raw-bit domain, 2 logits per op
__device__ __forceinline__ uint32_t bmax2_nan(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("max.NaN.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t bmax2(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("max.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);  // cvt.rn.bf16x2.f32 (RNE)
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ void status_or(uint32_t* status, uint32_t bits) {
  if (bits) atomicOr(status, bits);
}

// deterministic warp sums (xor butterfly; every lane ends with the same value)
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ uint32_t warp_or(uint32_t v) { return __reduce_or_sync(0xffffffffu, v); }

// (m, s, u) partial of a softmax row in the log2 domain: s = sum 2^(x-m),
// u = sum 2^(x-m) (x-m).  m == -inf means "empty".
struct Part {
  double m, s, u;
};

// Canonical combine (left fold order is fixed by the callers).
__device__ __forceinline__ Part part_fold(Part a, Part b) {
  if (b.m == -INFINITY) return a;
  if (a.m == -INFINITY) return b;
  double m = fmax(a.m, b.m);
  double da = a.m - m, db = b.m - m;
  // rescale factors via MUFU.EX2 (rel. error ~2^-22, far inside the 1e-5 bar;
  // both split and unsplit rows use this same code, so bits stay canonical)
  float fa_f, fb_f;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(fa_f) : "f"((float)da));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(fb_f) : "f"((float)db));
  double fa = fa_f, fb = fb_f;
  Part r;
  r.m = m;
  r.s = a.s * fa + b.s * fb;
  r.u = (a.u + a.s * da) * fa + (b.u + b.s * db) * fb;
  return r;
}

// first index i in [lo, hi) with a[i] > key  (upper bound), a non-decreasing
__device__ __forceinline__ int64_t upper_bound_i64(const int64_t* a, int64_t lo, int64_t hi, int64_t key) {
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] > key) hi = mid; else lo = mid + 1;
  }
  return lo;
}
__device__ __forceinline__ int64_t lower_bound_i32(const int32_t* a, int64_t lo, int64_t hi, int64_t key) {
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

}  // namespace dart
