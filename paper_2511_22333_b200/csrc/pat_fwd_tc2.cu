// Tensor-core (tcgen05 + TMEM + TMA) forward kernel: one persistent CTA per SM
// pulls work items (unit x kv head x up-to-128 rows) from a global counter in
// the scheduler's longest-first order and streams each item's KV span once
// through a 5-stage TMA ring.  Every pack goes through it: a narrow pack (a few
// queries x G heads) still runs QK^T / PV on the tensor core (M = 128 rows, the
// padding rows are free: the kernel is HBM- or softmax-bound, never MMA-bound).
//
//   warp 0      producer: claims items (atomic counter), resolves per-row
//               (query id, partial slot) into a 2-slot shared item ring, and
//               issues TMA boxes of 16-token page slices of K and V (64-token
//               stages, 128B swizzle) straight from the paged cache;
//   warp 1      TMEM allocator + MMA issuer (whole warp, one elected lane):
//                 S[c&1] = Q K_c^T     (TS: Q from TMEM, K K-major smem, M=128 N=64)
//                 O     += P[c-1] V    (TS: P from TMEM, V MN-major smem, N=d)
//               QK of tile c is issued before PV of tile c-1, S and P are
//               double-buffered, so softmax(c) overlaps PV(c-1) and QK(c+1);
//   warps 2-17  softmax / epilogue: 4 warps per TMEM lane quarter, each owning
//               16 of the 64 score columns (row max exchanged through smem).
// TMEM: S[2] (64 cols each), P[2] (64 cols: hi 32 + lo 32 packed 16-bit pairs),
// O (d cols fp32), Q (d/2 cols, packed 16-bit pairs) = 448 of 512 columns.
// Numerics follow cta_partial (attention.py:140-163): fp32 scores and
// accumulators, log2-domain online softmax with lazy O rescale (only when the
// running max grows by > 8), bf16 P = hi + lo (two PV MMAs).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include "pat_plan.cuh"
#include "pat_sm100.cuh"

namespace pat {
namespace tc2 {

#ifdef PAT_TC_TRACE
// Debug timeline (tools/tc_trace.py): CTA 0 records clock64 per (role, event, step).
// roles: 0 producer, 1 MMA issuer, 2 softmax (warp 2 lane 0), 3 softmax epilogue.
constexpr int kTraceSteps = 256;
__device__ long long g_tc_trace[4][8][kTraceSteps];
__device__ int g_trace_cta;  // the CTA traced (pat_debug_trace_cta)
__device__ unsigned long long g_span_tc[1][kSpanCtas][2];
#define TC_TRACE(role, ev, step)                                                         \
  do {                                                                                   \
    if (blockIdx.x == g_trace_cta && (step) < kTraceSteps) g_tc_trace[role][ev][step] = clock64(); \
  } while (0)
#else
#define TC_TRACE(role, ev, step) \
  do {                           \
  } while (0)
#endif
constexpr int kThreads = 576;  // producer, MMA issuer (+TMEM alloc), 16 softmax warps
constexpr int kSoftWarps = 16;
constexpr int kM = 128;        // rows per item tile (TMEM lanes)
constexpr int kN = 64;         // tokens per KV tile
#ifndef PAT_TC_STAGES
#define PAT_TC_STAGES 5
#endif
constexpr int kStages = PAT_TC_STAGES;  // KV ring depth: 4-6 measure the same; 5 is ~1% faster on c3 / c4
constexpr uint32_t kTmemCols = 512;
#ifndef PAT_TC_RESCALE_THRESHOLD
#define PAT_TC_RESCALE_THRESHOLD 8.0f
#endif
constexpr float kRescaleThreshold = PAT_TC_RESCALE_THRESHOLD;  // log2 units

// TMEM column map
constexpr uint32_t kColS = 0;    // S[b] at 64 b
constexpr uint32_t kColP = 128;  // P[b] at 128 + 64 b (hi 0-31, lo 32-63)
constexpr uint32_t kColO = 256;
constexpr uint32_t kColQ = 384;

// One slot of the work-item ring: the item and, per row, the query id and
// partial slot resolved by the producer warp (so consumers never chase the
// pack_q / unit_slot indirections at an item boundary).
struct ItemSlot {
  int32_t idx;
  int32_t pad[7];
  Item item;
  int2 meta[kM];  // (qid, slot) per row
};
static_assert(sizeof(ItemSlot) == 64 + 8 * kM, "ItemSlot layout");
constexpr uint32_t kSlotBytes = sizeof(ItemSlot);
constexpr uint32_t kFIdx = 0, kFKvh = 32 + 4, kFRow0 = 32 + 8, kFNrows = 32 + 12, kFNtok = 32 + 20, kFMeta = 64;

template <int D>
struct Layout {
  static constexpr int KB = D / 64;
  static constexpr int kTileBytes = KB * kN * 128;   // K or V stage tile: [KB][64][64]
  static constexpr int kOffKV = 0;
  static constexpr int kOffBar = kOffKV + kStages * 2 * kTileBytes;
  static constexpr int kOffRed = kOffBar + 512;                    // [2 parity][4 cq][128 rows] floats
  static constexpr int kOffRing = kOffRed + 2 * 4 * kM * 4;        // 2 x ItemSlot
  static constexpr int kBytes = kOffRing + 2 * (int)sizeof(ItemSlot);
  static constexpr int kAlloc = kBytes + 1024;
};

enum Bar : int {
  KV_FULL = 0,
  KV_EMPTY = KV_FULL + kStages,
  S_FULL = KV_EMPTY + kStages,  // [buffer] QK done
  S_EMPTY = S_FULL + 2,         // [buffer] softmax has read S
  P_FULL = S_EMPTY + 2,         // [buffer] P written to TMEM
  P_FREE = P_FULL + 2,          // [buffer] the PV reading P[b] completed (O updated)
  O_EMPTY = P_FREE + 2,         // epilogue has read O
  Q_FULL = O_EMPTY + 1,         // Q written to TMEM
  Q_EMPTY = Q_FULL + 1,         // last QK of the item completed
  ITEM_FULL = Q_EMPTY + 1,      // [slot] work item published by the producer
  ITEM_EMPTY = ITEM_FULL + 2,   // [slot] released by the MMA warp and the 16 softmax warps
  NUM_BARS = ITEM_EMPTY + 2
};
constexpr int kItemReaders = 1 + kSoftWarps;

template <typename T> struct Fmt;
template <> struct Fmt<__half> {
  static constexpr int ab = 0;
  static constexpr bool kSplit = false;
  static __device__ __forceinline__ uint32_t pack(float a, float b) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
  static __device__ __forceinline__ float2 unpack(uint32_t v) {
    return __half22float2(*reinterpret_cast<__half2*>(&v));
  }
};
template <> struct Fmt<__nv_bfloat16> {
  static constexpr int ab = 1;
#ifdef PAT_TC_NO_SPLIT
  static constexpr bool kSplit = false;
#else
  static constexpr bool kSplit = true;
#endif
  static __device__ __forceinline__ uint32_t pack(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
  static __device__ __forceinline__ float2 unpack(uint32_t v) {
    return make_float2(__uint_as_float(v << 16), __uint_as_float(v & 0xffff0000u));
  }
};

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float ex2_approx(float v) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}
// shared-space accesses by 32-bit address (the dynamic-smem base is re-aligned
// through an integer, so C++ pointers into it lose the shared address space)
__device__ __forceinline__ int lds_s32(uint32_t a) {
  int v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ int2 lds_v2(uint32_t a) {
  int2 v;
  asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ float lds_f32(uint32_t a) { return __int_as_float(lds_s32(a)); }
__device__ __forceinline__ void sts_f32(uint32_t a, float v) {
  asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ Item load_item(const Item* p) {
  const int4* q = reinterpret_cast<const int4*>(p);
  int4 a = __ldg(q), b = __ldg(q + 1);
  return Item{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
}

template <int D, typename T>
__global__ void __launch_bounds__(kThreads, 1)
    fwd_tc2_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv, DevPlan plan,
                   int var, const T* __restrict__ qg, T* __restrict__ out, float* __restrict__ part_o,
                   float* __restrict__ part_lse, float scale_log2) {
  using L = Layout<D>;
  using namespace sm100;
  constexpr bool kSplit = Fmt<T>::kSplit;
  constexpr int kQCols = D / 8;   // Q columns per softmax warp (its quarter of d, packed pairs)
  constexpr int kOCols = D / 4;   // O columns per softmax warp
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sb = smem_u32(smem);
  const uint32_t bars = sb + L::kOffBar;
  uint32_t* tmem_slot = (uint32_t*)(smem + L::kOffBar + NUM_BARS * 8);
  ItemSlot* ring = reinterpret_cast<ItemSlot*>(smem + L::kOffRing);
  auto bar = [&](int i) { return bars + 8u * (uint32_t)i; };
  auto sK = [&](int s) { return sb + L::kOffKV + (uint32_t)(s * 2 * L::kTileBytes); };
  auto sV = [&](int s) { return sb + L::kOffKV + (uint32_t)(s * 2 * L::kTileBytes + L::kTileBytes); };

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
      mbar_init(bar(S_EMPTY + b), kSoftWarps);
      mbar_init(bar(P_FULL + b), kSoftWarps);
      mbar_init(bar(P_FREE + b), 1);
      mbar_init(bar(ITEM_FULL + b), 32);
      mbar_init(bar(ITEM_EMPTY + b), kItemReaders);
    }
    mbar_init(bar(O_EMPTY), kSoftWarps);
    mbar_init(bar(Q_FULL), kSoftWarps);
    mbar_init(bar(Q_EMPTY), 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(smem_u32(tmem_slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  PAT_SPAN_BEGIN(g_span_tc, 0);

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    // Whole warp: lane i fetches the block id of page group i of a stage,
    // broadcast by shuffle (warp-uniform TMA operands), one elected lane issues.
    if (elect_one()) {
      tma_prefetch(&tmk);
      tma_prefetch(&tmv);
    }
    uint32_t g = 0;
    for (uint32_t n = 0;; ++n) {
      const uint32_t slot = n & 1;
      mbar_wait(bar(ITEM_EMPTY + slot), ((n >> 1) & 1) ^ 1);
      // the first item of CTA b is item b (no claim latency at kernel start),
      // later ones come from the counter, offset by the grid
      int it = (int)blockIdx.x;
      if (n > 0 && lane == 0) it = atomicAdd(plan.sched, 1) + (int)gridDim.x;
      it = __shfl_sync(0xffffffffu, it, 0);
      if (it >= n_items) it = -1;
      Item item{};
      if (it >= 0) {
        item = load_item(items + it);
        for (int r = lane; r < item.nrows; r += 32) {
          const int qi = (item.row0 + r) / G;
          ring[slot].meta[r] =
              make_int2(__ldg(plan.pack_q + item.qoff + qi), __ldg(plan.unit_slot + item.slot_off + qi));
        }
        if (lane == 0) ring[slot].item = item;
      }
      if (lane == 0) ring[slot].idx = it;
      __syncwarp();
      mbar_arrive(bar(ITEM_FULL + slot));
      if (it < 0) break;
      const int h = item.kvh, ntok = item.ntok;
      const int32_t* blist = plan.pack_blk + item.blk;
      const int ntiles = (ntok + kN - 1) / kN;
      for (int j = 0; j < ntiles; ++j, ++g) {
        const int s = g % kStages;
        const int rem = ntok - j * kN;
        const int ngrp = rem >= kN ? kN / 16 : (rem + 15) / 16;
        int my_blk = 0, my_off = 0;
        if (lane < ngrp) {
          const int tok = j * kN + lane * 16;
          const int pg = bs == 16 ? (tok >> 4) : tok / bs;
          my_blk = __ldg(blist + pg);
          my_off = bs == 16 ? 0 : tok - pg * bs;
        }
        mbar_wait(bar(KV_EMPTY + s), ((g / kStages) & 1) ^ 1);
        TC_TRACE(0, 0, g);
        if (elect_one()) mbar_expect_tx(bar(KV_FULL + s), (uint32_t)(ngrp * L::KB * 2048 * 2));
        __syncwarp();
        for (int gr = 0; gr < ngrp; ++gr) {
          const int blk = __shfl_sync(0xffffffffu, my_blk, gr);
          const int off = __shfl_sync(0xffffffffu, my_off, gr);
          if (elect_one()) {
#pragma unroll
            for (int kb = 0; kb < L::KB; ++kb) {
              tma_load_4d(sK(s) + kb * (kN * 128) + gr * 2048, &tmk, bar(KV_FULL + s), kb * 64, h, off, blk);
              tma_load_4d(sV(s) + kb * (kN * 128) + gr * 2048, &tmv, bar(KV_FULL + s), kb * 64, h, off, blk);
            }
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // The whole warp runs the loop so descriptors and TMEM addresses stay
    // warp-uniform (uniform datapath); one elected lane issues each
    // tcgen05.mma / commit (the same lane every time: all lanes are active).
    constexpr uint32_t idesc_qk = umma_idesc_f16(kM, kN, Fmt<T>::ab, 0);
    constexpr uint32_t idesc_pv = umma_idesc_f16(kM, D, Fmt<T>::ab, 1);
    uint32_t g = 0;  // KV tiles consumed (ring position)
    uint32_t c = 0;  // KV tiles processed (S / P buffer sequence)
    auto commit = [&](int b) {
      if (elect_one()) umma_commit(bar(b));
      __syncwarp();
    };
    auto issue_pv = [&](uint32_t cc, int s, bool first) {
      const uint32_t b = cc & 1;
      mbar_wait(bar(P_FULL + b), (cc >> 1) & 1);
      if (b == 0) TC_TRACE(1, 4, g);
      tc_fence_after();
      const uint64_t v0 = umma_desc_sw128(sV(s), kN * 128, 1024);
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < kN / 16; ++k) {
          const uint64_t bd = v0 + (uint64_t)((k * 16 * 128) >> 4);
          // P(m, k) is packed two per column: a k-step of 16 tokens = 8 columns
          const uint32_t tp = tmem + kColP + 64u * b + (uint32_t)(k * 8);
          umma_f16_ts(tmem + kColO, tp, bd, idesc_pv, (first && k == 0) ? 0u : 1u);
          if constexpr (kSplit) umma_f16_ts(tmem + kColO, tp + 32, bd, idesc_pv, 1u);
        }
        umma_commit(bar(P_FREE + b));
        umma_commit(bar(KV_EMPTY + s));
      }
      __syncwarp();
    };
    uint32_t n_items_done = 0;
    for (uint32_t n = 0;; ++n) {
      mbar_wait(bar(ITEM_FULL + (n & 1)), (n >> 1) & 1);
      const uint32_t rs = sb + L::kOffRing + (n & 1) * kSlotBytes;
      const int it = lds_s32(rs + kFIdx);
      const int ntok = it >= 0 ? lds_s32(rs + kFNtok) : 0;
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(ITEM_EMPTY + (n & 1)));
      if (it < 0) break;
      const int ntiles = (ntok + kN - 1) / kN;
      mbar_wait(bar(Q_FULL), n_items_done & 1);
      TC_TRACE(1, 5, g);
      tc_fence_after();
      int sprev = 0;
      for (int j = 0; j < ntiles; ++j, ++g, ++c) {
        const int s = g % kStages;
        const uint32_t b = c & 1;
        mbar_wait(bar(KV_FULL + s), (g / kStages) & 1);
        TC_TRACE(1, 0, g);
        mbar_wait(bar(S_EMPTY + b), ((c >> 1) & 1) ^ 1);  // softmax read S[b] (tile c-2)
        TC_TRACE(1, 3, g);
        tc_fence_after();
        const uint64_t k0 = umma_desc_sw128(sK(s), 16, 1024);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const int kb = k >> 2, kk = k & 3;
            // Q(m, k) packed two per column: a k-step of 16 = 8 columns
            umma_f16_ts(tmem + kColS + 64u * b, tmem + kColQ + (uint32_t)(k * 8),
                        k0 + (uint64_t)((kb * (kN * 128) + kk * 32) >> 4), idesc_qk, k > 0 ? 1u : 0u);
          }
          umma_commit(bar(S_FULL + b));
          if (j == ntiles - 1) umma_commit(bar(Q_EMPTY));
        }
        __syncwarp();
        TC_TRACE(1, 1, g);
        if (j > 0) {
          if (j == 1) mbar_wait(bar(O_EMPTY), (n_items_done & 1) ^ 1);
          issue_pv(c - 1, sprev, j == 1);
          TC_TRACE(1, 2, g);
        }
        sprev = s;
      }
      if (ntiles == 1) mbar_wait(bar(O_EMPTY), (n_items_done & 1) ^ 1);
      issue_pv(c - 1, sprev, ntiles == 1);
      ++n_items_done;
    }
  } else {
    // ------------------------------------------------------------ softmax / epilogue
    // warps 2-17: lane quarter wq = warp % 4 (the TMEM lanes the warp may
    // access), column quarter cq: 16 of the 64 score columns, 16 tokens' P,
    // d/4 of O and Q.  The 4 warps of a lane quarter exchange partial row
    // maxima through shared memory every KV tile (named barrier per quarter).
    const int wq = warp & 3, cq = (warp - 2) >> 2;
    const int t = wq * 32 + lane;                 // row in the item == TMEM lane
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    const uint32_t quarter_bar = 1 + wq;          // named barrier of the 4 warps of a lane quarter
    const uint32_t red = sb + L::kOffRed;  // [2 parity][4 cq][128] floats
    auto red_at = [&](uint32_t par, int q) { return red + (uint32_t)(((par * 4 + q) * kM + t) * 4); };
    const uint32_t ring_s = sb + L::kOffRing;
    auto fld = [&](uint32_t n, uint32_t off) { return lds_s32(ring_s + (n & 1) * kSlotBytes + off); };
    const bool tr = (t == 0 && cq == 0);          // trace thread
    uint32_t c = 0, g = 0, xc = 0, ni = 0;        // xc: exchange-buffer uses

    auto wait_item = [&](uint32_t n) { mbar_wait(bar(ITEM_FULL + (n & 1)), (n >> 1) & 1); };
    auto release_item = [&](uint32_t n) {
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(ITEM_EMPTY + (n & 1)));
    };
    // this thread's quarter of its Q row of the slot's item (zero past the item)
    auto load_q = [&](uint32_t n, uint32_t* qv) {
      const bool lv = t < fld(n, kFNrows);
      if (lv) {
        const int head = fld(n, kFKvh) * G + (fld(n, kFRow0) + t) % G;
        const int qid = fld(n, kFMeta + 8 * t);
        const uint4* src = reinterpret_cast<const uint4*>(qg + ((int64_t)qid * H + head) * D + cq * (D / 4));
#pragma unroll
        for (int i = 0; i < kQCols / 4; ++i) {
          const uint4 v = __ldg(src + i);
          qv[4 * i] = v.x, qv[4 * i + 1] = v.y, qv[4 * i + 2] = v.z, qv[4 * i + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < kQCols; ++i) qv[i] = 0u;
      }
    };
    auto store_q = [&](const uint32_t* qv) {
      const uint32_t ta = tmem + kColQ + lane_base + (uint32_t)(cq * kQCols);
      if constexpr (kQCols == 16) tmem_st16(ta, qv);
      else tmem_st8(ta, qv);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(Q_FULL));
    };

    wait_item(0);
    if (fld(0, kFIdx) >= 0) {
      uint32_t qv[kQCols];
      load_q(0, qv);
      store_q(qv);  // the Q region is free at kernel start
    }
    for (uint32_t n = 0;; ++n) {
      if (fld(n, kFIdx) < 0) break;  // ITEM_FULL(n) already waited
      const int ntok = fld(n, kFNtok);
      const int ntiles = (ntok + kN - 1) / kN;
      float m_ref = -INFINITY;  // running max, log2 units
      float2 l2 = make_float2(0.f, 0.f);
      bool have_next = false;
      uint32_t qn[kQCols];
      for (int j = 0; j < ntiles; ++j, ++c, ++g) {
        const uint32_t b = c & 1;
        mbar_wait(bar(S_FULL + b), (c >> 1) & 1);
        if (tr) TC_TRACE(2, 0, g);
        tc_fence_after();
        uint32_t sr[16];
        tmem_ld16(tmem + kColS + 64u * b + lane_base + (uint32_t)(16 * cq), sr);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar(S_EMPTY + b));
        if (tr) TC_TRACE(2, 6, g);
        if (j == ntiles - 1) {
          // last KV tile: fetch the next item and start loading its Q rows
          wait_item(n + 1);
          have_next = fld(n + 1, kFIdx) >= 0;
          if (have_next) load_q(n + 1, qn);
        }

        const int valid = ntok - j * kN - 16 * cq;  // valid columns of this quarter
        if (valid < 16) {
#pragma unroll
          for (int k = 0; k < 16; ++k)
            if (k >= valid) sr[k] = __float_as_uint(-INFINITY);
        }
        float pm[6];
#pragma unroll
        for (int k = 0; k < 5; ++k)
          pm[k] = fmax3(__uint_as_float(sr[3 * k]), __uint_as_float(sr[3 * k + 1]), __uint_as_float(sr[3 * k + 2]));
        pm[5] = __uint_as_float(sr[15]);
        const float pmx = fmax3(fmax3(pm[0], pm[1], pm[2]), pm[3], fmaxf(pm[4], pm[5]));
        sts_f32(red_at(xc & 1, cq), pmx);
        named_bar_sync(quarter_bar, 128);
        const float mx = fmaxf(fmax3(lds_f32(red_at(xc & 1, 0)), lds_f32(red_at(xc & 1, 1)), lds_f32(red_at(xc & 1, 2))),
                               lds_f32(red_at(xc & 1, 3))) *
                         scale_log2;
        ++xc;
        if (tr) TC_TRACE(2, 7, g);
        const bool need = mx > m_ref + kRescaleThreshold;
        if (__any_sync(0xffffffffu, need)) {
          const float m_new = need ? mx : m_ref;
          const float alpha = ex2_approx(m_ref - m_new);
          if (j > 0) {
            // O must hold PV(c-1): wait for the PV that read P[(c-1)&1]
            mbar_wait(bar(P_FREE + ((c - 1) & 1)), ((c - 1) >> 1) & 1);
            tc_fence_after();
#pragma unroll
            for (int q = 0; q < kOCols / 16; ++q) {
              uint32_t o[16];
              const uint32_t ta = tmem + kColO + lane_base + (uint32_t)(cq * kOCols + q * 16);
              tmem_ld16(ta, o);
#pragma unroll
              for (int e = 0; e < 16; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
              tmem_st16_wait(ta, o);
            }
          }
          l2.x *= alpha;
          l2.y *= alpha;
          m_ref = m_new;
        }
        // P = exp2(s * scale - m_ref) for this quarter's 16 tokens, packed pairs
        const float2 sc2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-m_ref, -m_ref);
        uint32_t ph[8], pl[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          float2 a = __ffma2_rn(make_float2(__uint_as_float(sr[2 * k]), __uint_as_float(sr[2 * k + 1])), sc2, nm2);
          a.x = ex2_approx(a.x);
          a.y = ex2_approx(a.y);
          ph[k] = Fmt<T>::pack(a.x, a.y);
          if constexpr (kSplit) {
            const float2 hf = Fmt<T>::unpack(ph[k]);
            const float2 lo = __fadd2_rn(a, make_float2(-hf.x, -hf.y));
            pl[k] = Fmt<T>::pack(lo.x, lo.y);
            l2 = __fadd2_rn(l2, a);
          } else {
            // normalise by the sum of the ROUNDED weights the MMA actually uses:
            // the output is then an exact weighted average of V rows
            l2 = __fadd2_rn(l2, Fmt<T>::unpack(ph[k]));
          }
        }
        if (tr) TC_TRACE(2, 1, g);
        // P[b] is free once the PV of tile c-2 completed
        mbar_wait(bar(P_FREE + b), ((c >> 1) & 1) ^ 1);
        tc_fence_after();
        if (tr) TC_TRACE(2, 2, g);
        const uint32_t tp = tmem + kColP + 64u * b + lane_base + (uint32_t)(8 * cq);
        tmem_st8(tp, ph);
        if constexpr (kSplit) tmem_st8(tp + 32, pl);
        if (j * kN + kN > ntok) {
          // tail tile: zero V rows past the span (stale / uninitialised smem)
          const int vt = ntok - j * kN;
          const int s = g % kStages;
          mbar_wait(bar(KV_FULL + s), (g / kStages) & 1);
          const int nz = (kN - vt) * L::KB * 8;
          for (int q = cq * kM + t; q < nz; q += 4 * kM) {
            const int rr = vt + q / (L::KB * 8);
            const int kb = (q / 8) % L::KB, ch = q % 8;
            st_shared_v4(sV(s) + kb * (kN * 128) + rr * 128 + (ch << 4), make_uint4(0, 0, 0, 0));
          }
          fence_proxy_async_smem();
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar(P_FULL + b));
        if (tr) TC_TRACE(2, 3, g);
      }

      // next item's Q -> TMEM once this item's last QK completed, so its first
      // QK overlaps this epilogue
      if (have_next) {
        mbar_wait(bar(Q_EMPTY), ni & 1);
        tc_fence_after();
        store_q(qn);
        if (tr) TC_TRACE(2, 4, g);
      }
      // epilogue: O / l; the 4 column quarters exchange their partial l
      const float lh = l2.x + l2.y;
      sts_f32(red_at(xc & 1, cq), lh);
      named_bar_sync(quarter_bar, 128);
      const float l = (lds_f32(red_at(xc & 1, 0)) + lds_f32(red_at(xc & 1, 1))) +
                      (lds_f32(red_at(xc & 1, 2)) + lds_f32(red_at(xc & 1, 3)));
      ++xc;
      if (tr) TC_TRACE(3, 0, g - 1);
      const bool live = t < fld(n, kFNrows);
      const int2 meta = live ? lds_v2(ring_s + (n & 1) * kSlotBytes + kFMeta + 8 * t) : make_int2(0, -1);
      const int head = fld(n, kFKvh) * G + (live ? (fld(n, kFRow0) + t) % G : 0);
      mbar_wait(bar(P_FREE + ((c - 1) & 1)), ((c - 1) >> 1) & 1);  // last PV done
      tc_fence_after();
      if (tr) TC_TRACE(3, 1, g - 1);
      const float inv = 1.f / l;
#pragma unroll
      for (int q = 0; q < kOCols / 16; ++q) {
        uint32_t o[16];
        const int col = cq * kOCols + q * 16;
        tmem_ld16(tmem + kColO + lane_base + (uint32_t)col, o);
        if (live) {
          if (meta.y < 0) {
            uint4* dst = reinterpret_cast<uint4*>(out + ((int64_t)meta.x * H + head) * D + col);
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              const float* f = reinterpret_cast<const float*>(o + k * 8);
              dst[k] = make_uint4(Fmt<T>::pack(f[0] * inv, f[1] * inv), Fmt<T>::pack(f[2] * inv, f[3] * inv),
                                  Fmt<T>::pack(f[4] * inv, f[5] * inv), Fmt<T>::pack(f[6] * inv, f[7] * inv));
            }
          } else {
            float4* dst = reinterpret_cast<float4*>(part_o + ((int64_t)meta.y * H + head) * D + col);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float* f = reinterpret_cast<const float*>(o + k * 4);
              dst[k] = make_float4(f[0] * inv, f[1] * inv, f[2] * inv, f[3] * inv);
            }
          }
        }
      }
      if (live && meta.y >= 0 && cq == 0) part_lse[(int64_t)meta.y * H + head] = m_ref + log2f(l);
      if (tr) TC_TRACE(3, 2, g - 1);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(O_EMPTY));
      if (tr) TC_TRACE(2, 5, g - 1);
      release_item(n);
      ++ni;
    }
  }
  PAT_SPAN_END(g_span_tc, 0);
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
  if (tid == 0) {
    // the last CTA out re-arms the item counter for the next launch
    __threadfence();
    if (atomicAdd(plan.sched + 1, 1) == (int)gridDim.x - 1) {
      plan.sched[0] = 0;
      plan.sched[1] = 0;
      __threadfence();
    }
  }
}

}  // namespace tc2

// ------------------------------------------------------------------------------------------
// host side: TMA descriptors over the paged cache + launch
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
static cudaError_t launch_tc2_t(const CUtensorMap& tmk, const CUtensorMap& tmv, const DevPlan& plan, int var,
                                int grid, const void* q, void* out, float* po, float* pl, float scale_log2,
                                cudaStream_t st) {
  constexpr int smem = tc2::Layout<D>::kAlloc;
  static bool init = false;
  if (!init) {
    cudaError_t e = cudaFuncSetAttribute(tc2::fwd_tc2_kernel<D, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    init = true;
  }
  tc2::fwd_tc2_kernel<D, T><<<grid, tc2::kThreads, smem, st>>>(tmk, tmv, plan, var, (const T*)q, (T*)out, po, pl,
                                                               scale_log2);
  return cudaGetLastError();
}

#ifdef PAT_TC_TRACE
extern "C" int pat_debug_tc_trace(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, tc2::g_tc_trace, sizeof(tc2::g_tc_trace));
}
extern "C" int pat_debug_trace_cta(int cta) {
  static long long zero[4][8][tc2::kTraceSteps];
  cudaMemcpyToSymbol(tc2::g_tc_trace, zero, sizeof(zero));
  return (int)cudaMemcpyToSymbol(tc2::g_trace_cta, &cta, sizeof(int));
}
extern "C" int pat_debug_spans_tc(unsigned long long* host) {
  int e = (int)cudaMemcpyFromSymbol(host, tc2::g_span_tc, sizeof(tc2::g_span_tc));
  static unsigned long long zero[1][kSpanCtas][2];
  cudaMemcpyToSymbol(tc2::g_span_tc, zero, sizeof(zero));
  return e;
}
#endif

cudaError_t launch_forward_tc(const CUtensorMap& tmk, const CUtensorMap& tmv, const DevPlan& plan, int var, int grid,
                              int dtype, int d, const void* q, void* out, float* po, float* pl, float scale_log2,
                              cudaStream_t st) {
  if (dtype == PAT_DTYPE_F16) {
    if (d == 128) return launch_tc2_t<128, __half>(tmk, tmv, plan, var, grid, q, out, po, pl, scale_log2, st);
    return launch_tc2_t<64, __half>(tmk, tmv, plan, var, grid, q, out, po, pl, scale_log2, st);
  }
  if (d == 128) return launch_tc2_t<128, __nv_bfloat16>(tmk, tmv, plan, var, grid, q, out, po, pl, scale_log2, st);
  return launch_tc2_t<64, __nv_bfloat16>(tmk, tmv, plan, var, grid, q, out, po, pl, scale_log2, st);
}

}  // namespace pat
