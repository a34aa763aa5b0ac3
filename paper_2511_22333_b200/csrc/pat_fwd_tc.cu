// Tensor-core (tcgen05 + TMEM + TMA) forward kernel for WIDE packs: a pack whose
// query tile (queries x G heads of one kv head) fills >= 64 rows forms a real
// dense contraction, so S = Q K^T and O += P V run on the 5th-gen tensor cores.
//
// One CTA (8 warps, one per SM) processes work items (unit, kv head, 128-row block):
//   warp 0      TMA producer: each 16-token page slice of K and V is loaded ONCE
//               per CTA into a 4-stage ring (64 tokens / stage), 128B swizzle,
//               straight from the paged cache (4-D tensor map over
//               [blocks][page][KVH][d]);
//   warp 1      MMA issuer (one thread): S_j = Q K_j^T (M=128, N=64, K=d) into a
//               double-buffered TMEM S, then O += P_{j-1} V_{j-1} (M=128, N=d,
//               K=64, V as an MN-major operand) into TMEM O;
//   warp 2      TMEM allocator;
//   warps 4..7  softmax (thread = row = TMEM lane): tcgen05.ld S, online softmax
//               in log2 units with lazy O rescale (only when the running max
//               grows by > 8, FA4-style), P -> smem (bf16/fp16) for the PV MMA,
//               and the epilogue (O / l -> output row, or fp32 partial + lse).
// Numerics follow cta_partial (attention.py:140-163): fp32 scores/accumulators.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include "pat_plan.cuh"
#include "pat_sm100.cuh"

namespace pat {

namespace tc {

constexpr int kThreads = 256;
constexpr int kM = 128;      // rows per tile (TMEM lanes)
constexpr int kN = 64;       // tokens per KV tile
constexpr uint32_t kTmemCols = 256;  // S0 [0,64) S1 [64,128) O [128, 128+D)
constexpr float kRescaleThreshold = 8.0f;  // log2 units

template <typename T> struct Fmt;

// kSplit: bf16 P is stored as hi + lo bf16 planes (two PV MMAs per k-step).
template <int D, bool kSplit>
struct Layout {
  static constexpr int KB = D / 64;                 // 64-element (128 B) column blocks
  static constexpr int kStages = kSplit ? 3 : 4;    // KV ring depth
  static constexpr int kQBytes = KB * kM * 128;     // [KB][128 rows][64]
  static constexpr int kPBytes = kM * 128;          // [128 rows][64 tokens]
  static constexpr int kPPlanes = kSplit ? 2 : 1;
  static constexpr int kTileBytes = KB * kN * 128;  // one K or V tile: [KB][64 tok][64]
  static constexpr int kOffQ = 0;
  static constexpr int kOffP = kOffQ + kQBytes;     // [buffer 2][plane][128][64]
  static constexpr int kOffKV = kOffP + 2 * kPPlanes * kPBytes;
  static constexpr int kOffBar = kOffKV + kStages * 2 * kTileBytes;
  static constexpr int kBytes = kOffBar + 1024;
  static constexpr int kAlloc = kBytes + 1024;  // manual 1024-B alignment slack
};

// barrier slots (8 B each) inside the barrier block
constexpr int kMaxStages = 4;
enum Bar : int {
  KV_FULL = 0,
  KV_EMPTY = KV_FULL + kMaxStages,
  S_FULL = KV_EMPTY + kMaxStages,
  S_EMPTY = S_FULL + 2,
  P_FULL = S_EMPTY + 2,
  P_EMPTY = P_FULL + 2,
  O_DONE = P_EMPTY + 2,
  O_EMPTY = O_DONE + 1,
  Q_FULL = O_EMPTY + 1,
  Q_EMPTY = Q_FULL + 1,
  NUM_BARS = Q_EMPTY + 1
};

template <> struct Fmt<__half> {
  static constexpr int ab = 0;
  static constexpr bool kSplit = false;
  static __device__ __forceinline__ uint32_t pack(float a, float b) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
  static __device__ __forceinline__ uint32_t pack_lo(float, float, uint32_t) { return 0u; }
};
template <> struct Fmt<__nv_bfloat16> {
  static constexpr int ab = 1;
  static constexpr bool kSplit = true;
  static __device__ __forceinline__ uint32_t pack(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
  static __device__ __forceinline__ uint32_t pack_lo(float a, float b, uint32_t hi) {
    __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162*>(&hi);
    float2 f = __bfloat1622float2(h);
    return pack(a - f.x, b - f.y);
  }
};

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

template <int D, typename T>
__global__ void __launch_bounds__(kThreads, 1)
    fwd_tc_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv, DevPlan plan,
                  int var, const T* __restrict__ qg, T* __restrict__ out, float* __restrict__ part_o,
                  float* __restrict__ part_lse, float scale_log2) {
  using L = Layout<D, Fmt<T>::kSplit>;
  constexpr int kStages = L::kStages;
  using namespace sm100;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sb = smem_u32(smem);
  const uint32_t sQ = sb + L::kOffQ, sP = sb + L::kOffP, sKV = sb + L::kOffKV;
  const uint32_t bars = sb + L::kOffBar;
  uint32_t* tmem_slot = (uint32_t*)(smem + L::kOffBar + NUM_BARS * 8);
  auto bar = [&](int i) { return bars + 8u * (uint32_t)i; };
  auto sK = [&](int s) { return sKV + (uint32_t)(s * 2 * L::kTileBytes); };
  auto sV = [&](int s) { return sKV + (uint32_t)(s * 2 * L::kTileBytes + L::kTileBytes); };

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int H = plan.H, G = plan.G, bs = plan.bs;
  const int n_items = plan.n_items[var];
  const Item* items = plan.items[var];

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(bar(KV_FULL + s), 1);
      mbar_init(bar(KV_EMPTY + s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar(S_FULL + b), 1);
      mbar_init(bar(S_EMPTY + b), 4);
      mbar_init(bar(P_FULL + b), 4);
      mbar_init(bar(P_EMPTY + b), 1);
    }
    mbar_init(bar(O_DONE), 1);
    mbar_init(bar(O_EMPTY), 4);
    mbar_init(bar(Q_FULL), 4);
    mbar_init(bar(Q_EMPTY), 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmk);
    tma_prefetch(&tmv);
  }
  if (warp == 2) tmem_alloc<kTmemCols>(smem_u32(tmem_slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tO = tmem + 128;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    // whole warp walks the items: lanes prefetch 32 block ids per load, lane 0
    // waits on the ring and issues the TMA boxes
    uint32_t g = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      const Item item = items[it];
      const int u = item.unit, h = item.kvh, p = plan.unit_pack[u];
      const int ntok = plan.unit_ntok[u];
      const int32_t* blist = plan.pack_blk + plan.pack_blk_off[p] + plan.unit_page0[u];
      const int npages = (ntok + bs - 1) / bs;
      const int ntiles = (ntok + kN - 1) / kN;
      int base = -1024, blk_reg = 0;
      for (int j = 0; j < ntiles; ++j, ++g) {
        const int s = g % kStages;
        const int rem = ntok - j * kN;
        const int ngrp = rem >= kN ? kN / 16 : (rem + 15) / 16;
        if (lane == 0) {
          mbar_wait(bar(KV_EMPTY + s), ((g / kStages) & 1) ^ 1);
          mbar_expect_tx(bar(KV_FULL + s), (uint32_t)(ngrp * L::KB * 2048 * 2));
        }
        for (int gr = 0; gr < ngrp; ++gr) {
          const int tok = j * kN + gr * 16;
          const int pg = tok / bs;
          if (pg >= base + 32) {
            base = pg;
            blk_reg = base + lane < npages ? __ldg(blist + base + lane) : 0;
          }
          const int blk = __shfl_sync(0xffffffffu, blk_reg, pg - base);
          if (lane == 0) {
            const int off = tok % bs;
#pragma unroll
            for (int kb = 0; kb < L::KB; ++kb) {
              tma_load_4d(sK(s) + kb * (kN * 128) + gr * 2048, &tmk, bar(KV_FULL + s), kb * 64, h, off, blk);
              tma_load_4d(sV(s) + kb * (kN * 128) + gr * 2048, &tmv, bar(KV_FULL + s), kb * 64, h, off, blk);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_qk = umma_idesc_f16(kM, kN, Fmt<T>::ab, 0);
      constexpr uint32_t idesc_pv = umma_idesc_f16(kM, D, Fmt<T>::ab, 1);
      uint32_t g = 0, n = 0;
      auto issue_pv = [&](uint32_t gp, bool first) {
        const int b = gp & 1, s = gp % kStages;
        if (first) mbar_wait(bar(O_EMPTY), (n & 1) ^ 1);
        mbar_wait(bar(P_FULL + b), (gp >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < kN / 16; ++k) {
          const uint32_t pb = sP + (b * L::kPPlanes) * L::kPBytes + k * 32;
          uint64_t bd = umma_desc_sw128(sV(s) + k * 16 * 128, kN * 128, 1024);
          umma_f16_ss(tO, umma_desc_sw128(pb, 16, 1024), bd, idesc_pv, (first && k == 0) ? 0u : 1u);
          if constexpr (L::kPPlanes == 2) umma_f16_ss(tO, umma_desc_sw128(pb + L::kPBytes, 16, 1024), bd, idesc_pv, 1u);
        }
        umma_commit(bar(KV_EMPTY + s));
        umma_commit(bar(P_EMPTY + b));
        umma_commit(bar(O_DONE));
      };
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const Item item = items[it];
        const int ntok = plan.unit_ntok[item.unit];
        const int ntiles = (ntok + kN - 1) / kN;
        mbar_wait(bar(Q_FULL), n & 1);
        tc_fence_after();
        for (int j = 0; j < ntiles; ++j) {
          const uint32_t gg = g + j;
          const int s = gg % kStages, b = gg & 1;
          mbar_wait(bar(KV_FULL + s), (gg / kStages) & 1);
          mbar_wait(bar(S_EMPTY + b), ((gg >> 1) & 1) ^ 1);
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const int kb = k >> 2, kk = k & 3;
            uint64_t a = umma_desc_sw128(sQ + kb * (kM * 128) + kk * 32, 16, 1024);
            uint64_t bd = umma_desc_sw128(sK(s) + kb * (kN * 128) + kk * 32, 16, 1024);
            umma_f16_ss(tS + b * kN, a, bd, idesc_qk, k > 0 ? 1u : 0u);
          }
          umma_commit(bar(S_FULL + b));
          if (j == ntiles - 1) umma_commit(bar(Q_EMPTY));
          if (j > 0) issue_pv(gg - 1, j == 1);
        }
        issue_pv(g + ntiles - 1, ntiles == 1);
        g += ntiles;
        ++n;
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax / epilogue
    const int t = tid - 128;  // row == TMEM lane
    const int wg = warp - 4;  // lane quarter owned by this warp
    const uint32_t lane_base = (uint32_t)(wg * 32) << 16;
    uint32_t g = 0, n = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      const Item item = items[it];
      const int u = item.unit, h = item.kvh, p = plan.unit_pack[u];
      const int ntok = plan.unit_ntok[u];
      const int ntiles = (ntok + kN - 1) / kN;
      const int qoff = plan.pack_q_off[p];
      const bool live = t < item.nrows;
      const int row = item.row0 + t;
      const int qi = live ? row / G : 0;
      const int qid = live ? plan.pack_q[qoff + qi] : 0;
      const int head = h * G + (live ? row % G : 0);

      // Q row -> smem (after the previous item's last QK MMA consumed it)
      mbar_wait(bar(Q_EMPTY), (n & 1) ^ 1);
      {
        const uint4* src = reinterpret_cast<const uint4*>(qg + ((int64_t)qid * H + head) * D);
#pragma unroll
        for (int ch = 0; ch < D / 8; ++ch) {
          uint4 v = live ? __ldg(src + ch) : make_uint4(0, 0, 0, 0);
          st_shared_v4(sQ + (ch >> 3) * (kM * 128) + t * 128 + (((ch & 7) ^ (t & 7)) << 4), v);
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(Q_FULL));

      float m_ref = -INFINITY, l = 0.f;
      for (int j = 0; j < ntiles; ++j) {
        const uint32_t gg = g + j;
        const int b = gg & 1;
        mbar_wait(bar(S_FULL + b), (gg >> 1) & 1);
        tc_fence_after();
        uint32_t sr[kN];
        tmem_ld32(tS + lane_base + b * kN, sr);
        tmem_ld32(tS + lane_base + b * kN + 32, sr + 32);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar(S_EMPTY + b));

        const int valid = ntok - j * kN;  // tokens of this tile that exist (>= 1)
        float mx = -INFINITY;
#pragma unroll
        for (int c = 0; c < kN; ++c) {
          float v = c < valid ? __uint_as_float(sr[c]) * scale_log2 : -INFINITY;
          sr[c] = __float_as_uint(v);
          mx = fmaxf(mx, v);
        }
        const bool need = mx > m_ref + kRescaleThreshold;
        if (__any_sync(0xffffffffu, need)) {
          const float m_new = need ? mx : m_ref;
          const float alpha = exp2f(m_ref - m_new);
          if (j > 0) {
            mbar_wait(bar(O_DONE), (gg - 1) & 1);
            tc_fence_after();
#pragma unroll
            for (int c = 0; c < D / 32; ++c) {
              uint32_t o[32];
              tmem_ld32(tO + lane_base + c * 32, o);
              tmem_wait_ld();
#pragma unroll
              for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
              tmem_st32(tO + lane_base + c * 32, o);
            }
            tmem_wait_st();
          }
          l *= alpha;
          m_ref = m_new;
        }
        // P = exp2(s - m_ref) -> smem row t (K-major A operand of the PV MMA)
        mbar_wait(bar(P_EMPTY + b), ((gg >> 1) & 1) ^ 1);
        const uint32_t prow = sP + (b * L::kPPlanes) * L::kPBytes + t * 128;
#pragma unroll
        for (int ch = 0; ch < kN / 8; ++ch) {
          float e[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            e[k] = exp2f(__uint_as_float(sr[ch * 8 + k]) - m_ref);
            l += e[k];
          }
          uint4 v = make_uint4(Fmt<T>::pack(e[0], e[1]), Fmt<T>::pack(e[2], e[3]), Fmt<T>::pack(e[4], e[5]),
                               Fmt<T>::pack(e[6], e[7]));
          st_shared_v4(prow + ((ch ^ (t & 7)) << 4), v);
          if constexpr (L::kPPlanes == 2) {
            uint4 w = make_uint4(Fmt<T>::pack_lo(e[0], e[1], v.x), Fmt<T>::pack_lo(e[2], e[3], v.y),
                                 Fmt<T>::pack_lo(e[4], e[5], v.z), Fmt<T>::pack_lo(e[6], e[7], v.w));
            st_shared_v4(prow + L::kPBytes + ((ch ^ (t & 7)) << 4), w);
          }
        }
        if (valid < kN) {
          // tail tile: zero V rows past the span (pages past the unit were not
          // loaded; a partial page may hold anything) so 0 * garbage cannot be NaN
          const int s = gg % kStages;
          mbar_wait(bar(KV_FULL + s), (gg / kStages) & 1);
          const int nz = (kN - valid) * L::KB * 8;  // 16-byte chunks to clear
          for (int c = t; c < nz; c += 128) {
            const int r = valid + c / (L::KB * 8);
            const int kb = (c / 8) % L::KB, ch = c % 8;
            st_shared_v4(sV(s) + kb * (kN * 128) + r * 128 + (ch << 4), make_uint4(0, 0, 0, 0));
          }
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar(P_FULL + b));
      }

      // epilogue: O / l
      const uint32_t glast = g + ntiles - 1;
      mbar_wait(bar(O_DONE), glast & 1);
      tc_fence_after();
      const float inv = 1.f / l;
      int slot = -1;
      if (live) slot = plan.unit_slot[plan.unit_slot_off[u] + qi];
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t o[32];
        tmem_ld32(tO + lane_base + c * 32, o);
        tmem_wait_ld();
        if (live) {
          if (slot < 0) {
            uint4* dst = reinterpret_cast<uint4*>(out + ((int64_t)qid * H + head) * D + c * 32);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float* f = reinterpret_cast<const float*>(o + k * 8);
              dst[k] = make_uint4(Fmt<T>::pack(f[0] * inv, f[1] * inv), Fmt<T>::pack(f[2] * inv, f[3] * inv),
                                  Fmt<T>::pack(f[4] * inv, f[5] * inv), Fmt<T>::pack(f[6] * inv, f[7] * inv));
            }
          } else {
            float4* dst = reinterpret_cast<float4*>(part_o + ((int64_t)slot * H + head) * D + c * 32);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const float* f = reinterpret_cast<const float*>(o + k * 4);
              dst[k] = make_float4(f[0] * inv, f[1] * inv, f[2] * inv, f[3] * inv);
            }
          }
        }
      }
      if (live && slot >= 0) part_lse[(int64_t)slot * H + head] = m_ref + log2f(l);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(O_EMPTY));
      g += ntiles;
      ++n;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
}

}  // namespace tc

// ------------------------------------------------------------------------------------------
// host side: tensor maps + launch
// ------------------------------------------------------------------------------------------

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

// 4-D map over a paged cache [num_blocks][bs][KVH][D]: box (64 d, 1 head, 16 tokens, 1 block).
int make_kv_tensor_map(CUtensorMap* map, const void* base, int64_t num_blocks, int bs, int kvh, int d, int dtype) {
  auto enc = get_encode();
  if (!enc) return -1;
  cuuint64_t dims[4] = {(cuuint64_t)d, (cuuint64_t)kvh, (cuuint64_t)bs, (cuuint64_t)num_blocks};
  cuuint64_t strides[3] = {(cuuint64_t)d * 2, (cuuint64_t)kvh * d * 2, (cuuint64_t)bs * kvh * d * 2};
  cuuint32_t box[4] = {64, 1, 16, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, dtype == PAT_DTYPE_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                   4, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)r;
}

template <int D, typename T>
static cudaError_t launch_tc_t(const CUtensorMap& tmk, const CUtensorMap& tmv, const DevPlan& plan, int var, int grid,
                               const void* q, void* out, float* po, float* pl, float scale_log2, cudaStream_t st) {
  constexpr int smem = tc::Layout<D, tc::Fmt<T>::kSplit>::kAlloc;
  static bool init = false;
  if (!init) {
    cudaError_t e = cudaFuncSetAttribute(tc::fwd_tc_kernel<D, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    init = true;
  }
  tc::fwd_tc_kernel<D, T><<<grid, tc::kThreads, smem, st>>>(tmk, tmv, plan, var, (const T*)q, (T*)out, po, pl,
                                                            scale_log2);
  return cudaGetLastError();
}

cudaError_t launch_forward_tc(const CUtensorMap& tmk, const CUtensorMap& tmv, const DevPlan& plan, int var, int grid,
                              int dtype, int d, const void* q, void* out, float* po, float* pl, float scale_log2,
                              cudaStream_t st) {
  if (dtype == PAT_DTYPE_F16) {
    if (d == 128) return launch_tc_t<128, __half>(tmk, tmv, plan, var, grid, q, out, po, pl, scale_log2, st);
    return launch_tc_t<64, __half>(tmk, tmv, plan, var, grid, q, out, po, pl, scale_log2, st);
  }
  if (d == 128) return launch_tc_t<128, __nv_bfloat16>(tmk, tmv, plan, var, grid, q, out, po, pl, scale_log2, st);
  return launch_tc_t<64, __nv_bfloat16>(tmk, tmv, plan, var, grid, q, out, po, pl, scale_log2, st);
}

}  // namespace pat
