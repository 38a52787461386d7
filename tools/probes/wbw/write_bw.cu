// Write-only / read-only / copy bandwidth probes (tools only, not product code).
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_st128(uint4* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(0, 0, 0, 0);
}
__global__ void k_st128cs(uint4* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%1,%1,%1};" ::"l"(p + i), "r"(0) : "memory");
}
__global__ void k_st256(uint4* p, int64_t n) {   // n in 32-byte units
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p + 2 * i), "r"(0) : "memory");
}
// per-CTA contiguous range, like the bwd sweep's write stream
__global__ void k_st128_range(uint4* p, int64_t n) {
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t a = blockIdx.x * per, b = min(n, a + per);
  for (int64_t i = a + threadIdx.x; i < b; i += blockDim.x)
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%1,%1,%1};" ::"l"(p + i), "r"(0) : "memory");
}
__global__ void k_bulkst(uint8_t* p, int64_t nbytes) {   // TMA bulk store of a zeroed smem page
  __shared__ __align__(128) uint8_t z[4096];
  for (int i = threadIdx.x; i < 4096 / 16; i += blockDim.x) reinterpret_cast<uint4*>(z)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x % 32 != 0) return;
  const int64_t nch = nbytes / 4096;
  const int64_t w = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, W = (int64_t)gridDim.x * (blockDim.x / 32);
  int k = 0;
  for (int64_t c = w; c < nch; c += W) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 4096;" ::"l"(p + c * 4096),
                 "r"((uint32_t)__cvta_generic_to_shared(z)) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (++k == 8) { asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory"); k = 4; }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
extern "C" int probe(int which, void* p, int64_t nbytes, int grid, int block, cudaStream_t s) {
  switch (which) {
    case 0: k_st128<<<grid, block, 0, s>>>((uint4*)p, nbytes / 16); break;
    case 1: k_st128cs<<<grid, block, 0, s>>>((uint4*)p, nbytes / 16); break;
    case 2: k_st256<<<grid, block, 0, s>>>((uint4*)p, nbytes / 32); break;
    case 3: k_st128_range<<<grid, block, 0, s>>>((uint4*)p, nbytes / 16); break;
    case 4: k_bulkst<<<grid, block, 0, s>>>((uint8_t*)p, nbytes); break;
    case 5: return (int)cudaMemsetAsync(p, 0, nbytes, s);
  }
  return (int)cudaGetLastError();
}
