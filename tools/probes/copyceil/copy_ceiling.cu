// Read+write ceiling of SM-issued copies on B200 (tools only, not product code):
// how fast can a kernel move a logits-sized buffer (read N bytes, write N bytes)?
#include <cstdint>
#include <cuda_runtime.h>

template <int U, bool CS>
__global__ void __launch_bounds__(256) k_ldst(const uint4* __restrict__ s, uint4* __restrict__ d, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * U;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x * U + threadIdx.x; base < n; base += stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + (int64_t)u * blockDim.x;
      if (i < n) {
        if (CS) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(s + i));
        else v[u] = s[i];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + (int64_t)u * blockDim.x;
      if (i < n) {
        if (CS) asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(d + i), "r"(v[u].x), "r"(v[u].y),
                             "r"(v[u].z), "r"(v[u].w) : "memory");
        else d[i] = v[u];
      }
    }
  }
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// TMA bulk ring: each warp streams chunks g2s into its ring and writes them back
// with bulk s2g stores (no registers touch the data).  contiguous: CTA-contiguous
// range split over its warps (chunk w, w+W, ...), else grid-wide interleave.
template <int STAGES, int CH>
__global__ void k_bulk(const uint8_t* s, uint8_t* d, int64_t nbytes, int contiguous) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, W = blockDim.x / 32;
  uint8_t* ring = sm + (size_t)warp * STAGES * CH;
  __shared__ __align__(8) uint64_t bars[32 * STAGES];
  uint64_t* b = bars + warp * STAGES;
  const int64_t nch = nbytes / CH;
  int64_t j0, j1, step;
  if (contiguous) {
    const int64_t per = (nch + gridDim.x - 1) / gridDim.x;
    j0 = blockIdx.x * per + warp; j1 = min(nch, (int64_t)(blockIdx.x + 1) * per); step = W;
  } else {
    j0 = (int64_t)blockIdx.x * W + warp; j1 = nch; step = (int64_t)gridDim.x * W;
  }
  if (lane != 0) return;
  for (int i = 0; i < STAGES; ++i)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&b[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  int64_t jl = j0;   // next chunk to load
  int issued = 0;
  for (int i = 0; i < STAGES && jl < j1; ++i, jl += step, ++issued) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&b[i])), "r"(CH) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su32(ring + i * CH)), "l"(s + jl * CH), "r"(CH), "r"(su32(&b[i])) : "memory");
  }
  uint32_t phase = 0;
  int slot = 0;
  for (int64_t j = j0; j < j1; j += step) {
    asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}"
                 ::"r"(su32(&b[slot])), "r"(phase) : "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d + j * CH),
                 "r"(su32(ring + slot * CH)), "r"(CH) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (jl < j1) {
      // the slot about to be refilled is the oldest store's source: wait until it has been read
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&b[slot])), "r"(CH) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(su32(ring + slot * CH)), "l"(s + jl * CH), "r"(CH), "r"(su32(&b[slot])) : "memory");
      jl += step;
    }
    if (++slot == STAGES) { slot = 0; phase ^= 1u; }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void k_spin(int64_t cycles) {
  const int64_t t0 = clock64();
  while (clock64() - t0 < cycles) {}
}

extern "C" int probe(int which, const void* s, void* d, int64_t nbytes, int grid, int block, int arg,
                     cudaStream_t st) {
  const int64_t n = nbytes / 16;
  switch (which) {
    case 0: k_ldst<1, false><<<grid, 256, 0, st>>>((const uint4*)s, (uint4*)d, n); break;
    case 1: k_ldst<4, false><<<grid, 256, 0, st>>>((const uint4*)s, (uint4*)d, n); break;
    case 2: k_ldst<8, false><<<grid, 256, 0, st>>>((const uint4*)s, (uint4*)d, n); break;
    case 3: k_ldst<4, true><<<grid, 256, 0, st>>>((const uint4*)s, (uint4*)d, n); break;
    case 4: k_ldst<8, true><<<grid, 256, 0, st>>>((const uint4*)s, (uint4*)d, n); break;
    case 5: {
      const size_t sm = (size_t)(block / 32) * 4 * 4096;
      cudaFuncSetAttribute(k_bulk<4, 4096>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      k_bulk<4, 4096><<<grid, block, sm, st>>>((const uint8_t*)s, (uint8_t*)d, nbytes, arg);
      break;
    }
    case 6: {
      const size_t sm = (size_t)(block / 32) * 6 * 4096;
      cudaFuncSetAttribute(k_bulk<6, 4096>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      k_bulk<6, 4096><<<grid, block, sm, st>>>((const uint8_t*)s, (uint8_t*)d, nbytes, arg);
      break;
    }
    case 7: return (int)cudaMemcpyAsync(d, s, nbytes, cudaMemcpyDeviceToDevice, st);
    case 8: k_spin<<<grid, block, 0, st>>>((int64_t)arg * 1000); break;
  }
  return (int)cudaGetLastError();
}
