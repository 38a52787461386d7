// dart_select.cu -- high-entropy step selection (sm_100a).
//
//   K3a unpack_kernel  all-gather layout [world * S_pad] -> global order [S]
//   K3b select_kernel  one CTA per task group g: exact order statistic of the
//                      group's step entropies by 4-pass radix select on
//                      order-preserving uint32 keys (integer counting, so
//                      bit-exact and identical on every rank), the keep mask
//                      I[H_t >= tau_g] (Eq. 2; "top 80%",
//                      PAPER.md:235; threshold per group),
//                      and the group's kept step / token counts.
//   K3c norm_kernel    global N_keep and the normaliser.
#include "dart_common.cuh"
#include "dart_internal.h"

namespace dart {

__global__ void unpack_kernel(UnpackParams p) {
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < p.S; s += nthreads) {
    int r = 0;
    while (r + 1 < p.world && p.rank_step_off[r + 1] <= s) ++r;
    p.H[s] = p.gathered[(int64_t)r * p.S_pad + (s - p.rank_step_off[r])];
  }
}

// order-preserving map float -> uint32 (both zeros map to +0's key)
__device__ __forceinline__ uint32_t fkey(float h) {
  uint32_t b = __float_as_uint(h == 0.0f ? 0.0f : h);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float ikey(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// k-th smallest (0-based) of H[sa, sa+n) -- all threads of the block call it.
__device__ float radix_select(const float* H, int64_t sa, int64_t n, uint32_t kk, uint32_t* hist,
                              uint32_t* s_shared) {
  uint32_t prefix = 0, mask = 0;
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    for (int b = threadIdx.x; b < 256; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const uint32_t key = fkey(H[sa + i]);
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      uint32_t c = 0;
#pragma unroll
      for (int b = 0; b < 8; ++b) c += hist[lane * 8 + b];
      uint32_t cum = c;  // inclusive warp scan
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, cum, o);
        if (lane >= o) cum += y;
      }
      const uint32_t ball = __ballot_sync(0xffffffffu, cum > kk);
      const int L = __ffs(ball) - 1;  // first lane whose bins contain rank kk
      if (lane == L) {
        uint32_t e = cum - c;
        uint32_t digit = 0;
        for (int b = 0; b < 8; ++b) {
          const uint32_t h = hist[lane * 8 + b];
          if (e + h > kk) { digit = (uint32_t)(lane * 8 + b); break; }
          e += h;
        }
        s_shared[0] = prefix | (digit << shift);
        s_shared[1] = kk - e;
      }
    }
    __syncthreads();
    prefix = s_shared[0];
    kk = s_shared[1];
    mask |= 255u << shift;
    __syncthreads();
  }
  return ikey(prefix);
}

__global__ void __launch_bounds__(256) select_kernel(SelectParams p) {
  __shared__ uint32_t hist[256];
  __shared__ uint32_t s_shared[2];
  __shared__ unsigned long long cnt[2];
  for (int64_t g = blockIdx.x; g < p.G; g += gridDim.x) {
    const int64_t i0 = p.grp_traj[g], i1 = p.grp_traj[g + 1];
    const int64_t sa = p.traj_step_off[i0], sb = p.traj_step_off[i1];
    const int64_t n = sb - sa;
    if (n <= 0) {
      if (threadIdx.x == 0) {
        p.tau[g] = __int_as_float(0x7fc00000);
        p.grp_keep_step[g] = 0;
        p.grp_keep_tok[g] = 0;
      }
      continue;
    }
    const bool ok = p.group_ok[g] != 0;
    const double q = (double)p.q;
    bool use_double = false;
    float tau_f = -INFINITY;
    double tau_d = -INFINITY;
    if (p.rule == DART_SEL_FLOOR || p.rule == DART_SEL_CEIL) {
      int64_t k = (p.rule == DART_SEL_FLOOR) ? (int64_t)floor(q * (double)n) : (int64_t)ceil(q * (double)n);
      if (k > n - 1) k = n - 1;
      if (k < 0) k = 0;
      tau_f = radix_select(p.H, sa, n, (uint32_t)k, hist, s_shared);
    } else if (p.rule == DART_SEL_LINEAR) {
      const double pos = q * (double)(n - 1);
      int64_t lo = (int64_t)floor(pos);
      if (lo > n - 1) lo = n - 1;
      const int64_t hi = lo + 1 < n ? lo + 1 : n - 1;
      const double frac = pos - (double)lo;
      const double slo = (double)radix_select(p.H, sa, n, (uint32_t)lo, hist, s_shared);
      const double shi = (double)radix_select(p.H, sa, n, (uint32_t)hi, hist, s_shared);
      tau_d = slo + frac * (shi - slo);
      use_double = true;
    }
    // keep mask and counts
    if (threadIdx.x < 2) cnt[threadIdx.x] = 0ull;
    __syncthreads();
    unsigned long long ks = 0, kt = 0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const int64_t s = sa + i;
      const float h = p.H[s];
      bool keep;
      if (p.rule == DART_SEL_OFF) keep = true;
      else if (use_double) keep = (double)h >= tau_d;
      else keep = h >= tau_f;
      keep = keep && ok;
      p.keep[s] = keep ? 1 : 0;
      if (keep) {
        ks += 1;
        kt += (unsigned long long)(p.step_tok_off[s + 1] - p.step_tok_off[s]);
      }
    }
    atomicAdd(&cnt[0], ks);
    atomicAdd(&cnt[1], kt);
    __syncthreads();
    if (threadIdx.x == 0) {
      p.tau[g] = (p.rule == DART_SEL_OFF) ? -INFINITY : (use_double ? (float)tau_d : tau_f);
      p.grp_keep_step[g] = (int64_t)cnt[0];
      p.grp_keep_tok[g] = (int64_t)cnt[1];
    }
    __syncthreads();
  }
}

__global__ void norm_kernel(NormParams p) {
  __shared__ unsigned long long tot[2];
  if (threadIdx.x < 2) tot[threadIdx.x] = 0ull;
  __syncthreads();
  unsigned long long ks = 0, kt = 0;
  for (int64_t g = threadIdx.x; g < p.G; g += blockDim.x) {
    ks += (unsigned long long)p.grp_keep_step[g];
    kt += (unsigned long long)p.grp_keep_tok[g];
  }
  atomicAdd(&tot[0], ks);
  atomicAdd(&tot[1], kt);
  __syncthreads();
  if (threadIdx.x == 0) {
    dart_norm* n = reinterpret_cast<dart_norm*>(p.norm);
    n->n_keep_step = (int64_t)tot[0];
    n->n_keep_tok = (int64_t)tot[1];
    n->n_tok = p.T;
    n->n_step = p.S;
    double N = 0.0;
    switch (p.norm_mode) {
      case DART_NORM_TOKEN_MEAN_KEPT: N = (double)tot[1]; break;
      case DART_NORM_STEP_MEAN_KEPT: N = (double)tot[0]; break;
      case DART_NORM_TOKEN_MEAN_ALL: N = (double)p.T; break;
      case DART_NORM_STEP_MEAN_ALL: N = (double)p.S; break;
      default: N = 1.0; break;  // SUM
    }
    n->inv_norm = N > 0.0 ? 1.0 / N : 0.0;
  }
}

cudaError_t launch_unpack(const UnpackParams& p, cudaStream_t st) {
  int64_t blocks = (p.S + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  if (blocks < 1) blocks = 1;
  unpack_kernel<<<(unsigned)blocks, 256, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_select(const SelectParams& p, cudaStream_t st) {
  if (p.G <= 0) return cudaSuccess;
  int64_t blocks = p.G < 65535 ? p.G : 65535;
  select_kernel<<<(unsigned)blocks, 256, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_norm(const NormParams& p, cudaStream_t st) {
  norm_kernel<<<1, 256, 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace dart
