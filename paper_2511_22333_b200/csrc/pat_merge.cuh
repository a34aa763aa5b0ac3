// Merge of per-unit partials (o / l, log2-sum-exp) into the output: one warp
// per (query, head), online-softmax fold in slot (= unit) order
// (_merge_batch_into, attention.py:187-199).  Queries covered by one unit are
// written by the forward kernels directly and never reach the merge.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "pat_plan.cuh"

namespace pat {

template <typename T> struct MergeOut;
template <> struct MergeOut<__half> {
  static __device__ __forceinline__ uint32_t pack(float a, float b) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
};
template <> struct MergeOut<__nv_bfloat16> {
  static __device__ __forceinline__ uint32_t pack(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
};

// Warp `gw` of `nw` folds (query, head) pairs gw, gw + nw, ...  Latency-bound,
// so lanes fetch up to 32 slot LSEs at once, weights are shuffled, and the
// weighted O rows are independent loads issued 4 at a time.  Loads bypass L1
// (ld.global.cg): the partials were written by another grid.  The first
// descriptor (plan data, final before the forward started) and the row count
// are loaded by the caller before it waits for the forward.
template <int D, typename T>
__device__ __forceinline__ void merge_rows(const DevPlan& plan, const float* __restrict__ part_o,
                                           const float* __restrict__ part_lse, T* __restrict__ out, int gw, int nw,
                                           int nq, int4 md0) {
  const int H = plan.H;
  const int lane = threadIdx.x & 31;
  constexpr int PER = D / 32;
  int4 md_next = md0;
  for (int w = gw; w < nq * H; w += nw) {
    // this row's descriptor was fetched with the previous row; the next one's
    // goes out now, so a warp's rows cost one dependent round trip each
    const int4 md = md_next;
    if (w + nw < nq * H) md_next = __ldg(plan.merge_desc + (w + nw) / H);
    const int q = md.x, head = w % H, base = md.y, n = md.z;
    if (n <= 8) {
      // common case: every slot's LSE and O row are loaded at once (one round
      // trip after the descriptor), then folded
      const float lse = lane < n ? __ldcg(part_lse + (int64_t)(base + lane) * H + head) : -INFINITY;
      float v[8][PER];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (u < n) {
          const float* src = part_o + ((int64_t)(base + u) * H + head) * D + lane * PER;
          if constexpr (PER == 4) {
            const float4 x = __ldcg(reinterpret_cast<const float4*>(src));
            v[u][0] = x.x, v[u][1] = x.y, v[u][2] = x.z, v[u][3] = x.w;
          } else {
            const float2 x = __ldcg(reinterpret_cast<const float2*>(src));
            v[u][0] = x.x, v[u][1] = x.y;
          }
        }
      }
      float M = lse;
#pragma unroll
      for (int off = 4; off; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
      M = __shfl_sync(0xffffffffu, M, 0);
      const float f = lane < n ? exp2f(lse - M) : 0.f;
      float L = f;
#pragma unroll
      for (int off = 4; off; off >>= 1) L += __shfl_xor_sync(0xffffffffu, L, off);
      L = __shfl_sync(0xffffffffu, L, 0);
      float acc[PER];
#pragma unroll
      for (int e = 0; e < PER; ++e) acc[e] = 0.f;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float fu = __shfl_sync(0xffffffffu, f, u);
        if (u < n)
#pragma unroll
          for (int e = 0; e < PER; ++e) acc[e] += fu * v[u][e];
      }
      const float inv = 1.f / L;
      T* dst = out + ((int64_t)q * H + head) * D + lane * PER;
#pragma unroll
      for (int e = 0; e < PER; e += 2)
        *reinterpret_cast<uint32_t*>(dst + e) = MergeOut<T>::pack(acc[e] * inv, acc[e + 1] * inv);
      continue;
    }
    float acc[PER];
#pragma unroll
    for (int e = 0; e < PER; ++e) acc[e] = 0.f;
    float M = -INFINITY, L = 0.f;
    for (int c0 = 0; c0 < n; c0 += 32) {
      const int cn = min(32, n - c0);
      const float lse = lane < cn ? __ldcg(part_lse + (int64_t)(base + c0 + lane) * H + head) : -INFINITY;
      float cm = lse;
#pragma unroll
      for (int off = 16; off; off >>= 1) cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, off));
      const float Mn = fmaxf(M, cm);
      const float a = exp2f(M - Mn);  // rescale what was accumulated so far
#pragma unroll
      for (int e = 0; e < PER; ++e) acc[e] *= a;
      L *= a;
      M = Mn;
      const float f = lane < cn ? exp2f(lse - M) : 0.f;
      float fs = f;
#pragma unroll
      for (int off = 16; off; off >>= 1) fs += __shfl_xor_sync(0xffffffffu, fs, off);
      L += fs;
      for (int i = 0; i < cn; i += 4) {
        float v[4][PER];
        float fi[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          fi[u] = __shfl_sync(0xffffffffu, f, min(i + u, 31));
          const float* src = part_o + ((int64_t)(base + c0 + min(i + u, cn - 1)) * H + head) * D + lane * PER;
          if constexpr (PER == 4) {
            const float4 x = __ldcg(reinterpret_cast<const float4*>(src));
            v[u][0] = x.x, v[u][1] = x.y, v[u][2] = x.z, v[u][3] = x.w;
          } else {
            const float2 x = __ldcg(reinterpret_cast<const float2*>(src));
            v[u][0] = x.x, v[u][1] = x.y;
          }
          if (i + u >= cn) fi[u] = 0.f;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int e = 0; e < PER; ++e) acc[e] += fi[u] * v[u][e];
      }
    }
    const float inv = 1.f / L;
    T* dst = out + ((int64_t)q * H + head) * D + lane * PER;
#pragma unroll
    for (int e = 0; e < PER; e += 2) {
      uint32_t pk = MergeOut<T>::pack(acc[e] * inv, acc[e + 1] * inv);
      *reinterpret_cast<uint32_t*>(dst + e) = pk;
    }
  }
}

}  // namespace pat
