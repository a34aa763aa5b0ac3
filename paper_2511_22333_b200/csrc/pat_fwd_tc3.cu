// Tensor-core (tcgen05 + TMEM + TMA) forward kernel, two softmax warpgroups.
//
// One persistent CTA per SM pulls work items (unit x kv head x up to 256 rows)
// from a global counter in the scheduler's longest-first order and streams each
// item's KV span once through a 4-stage TMA ring.  Every pack goes through it.
//
//   warp 0      producer: claims items, resolves per-row (query id, partial
//               slot) into a 2-slot item ring, warms L2 with the item's Q rows,
//               issues TMA boxes of 16-token page slices of K and V (64-token
//               stages, 128B swizzle) straight from the paged vLLM cache;
//   warp 1      TMEM allocator + MMA issuer (one elected lane):
//                 S[g]  = Q_g K^T   (TS: Q from TMEM, K from smem, M=128 N=64)
//                 O[g] += P[g] V     (TS: P from TMEM over S[g], V from smem)
//   warps 4-7   softmax group 0, warps 8-11 softmax group 1: one thread per
//               TMEM lane (row), one lane quarter per warp (warps 2-3 idle:
//               setmaxnreg works on whole warpgroups).
//
// An item runs in one of two modes (the item's row count decides):
//   * PP (129-256 rows): group g owns rows [128 g, 128 g + 128); every KV stage
//     feeds both groups (two QK / PV per stage, 256 rows per KV byte read);
//   * EO (<= 128 rows): the groups take alternate KV tiles of the item (even /
//     odd), each with its own running max, sum and O accumulator; rows are also
//     replicated R = 4 / 2 / 1 times over the lane quarters (<= 32 / <= 64 /
//     <= 128 rows) so a narrow item's tile is split into R column slices of
//     64 / R tokens.  The 2R partial states of a row are combined (the
//     merge_partials fold) in the epilogue.
// Two softmax warps per SM sub-partition on independent tiles keep the
// per-tile exp / max chain of one warp from pacing the kernel.
//
// TMEM (512 columns): group g at 256 g: S/P at +0 (P = hi 32 + lo 32 columns
// of packed 16-bit pairs written over the consumed S), Q at +64 (packed
// pairs, the A operand of QK: shared-memory operand bandwidth is the scarce
// resource of tcgen05, so only K and V are read from shared memory), O at +128.
// The next EO item's Q rows are staged in shared memory with cp.async while
// the current item runs (two buffers; the item's buffer is the epilogue
// scratch once its rows are in TMEM).
// Numerics follow cta_partial (attention.py:140-163): fp32 scores and
// accumulators, log2-domain online softmax with lazy O rescale (only when the
// running max grows by > 8), bf16 P = hi + lo (two PV MMAs), fp16 P single.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <type_traits>

#include "pat_mma_sync.cuh"
#include "pat_plan.cuh"
#include "pat_sm100.cuh"

namespace pat {
namespace tc3 {

#ifdef PAT_TC_TRACE
// Debug timeline (tools/tc_trace.py): CTA g_trace_cta records clock64 per (role, event, step).
constexpr int kTraceSteps = 256;
__device__ long long g_tc_trace[4][8][kTraceSteps];
__device__ int g_trace_cta;
__device__ unsigned long long g_span_tc[1][kSpanCtas][2];
// per-item log (all CTAs): cta, item, rows, tiles, t_start, t_first_data, t_tiles_done, t_epilogue_done
constexpr int kItemLog = 32768;
__device__ long long g_item_log[kItemLog][8];
__device__ int g_item_n;
__device__ __forceinline__ long long gtime() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define ITEM_T(var) \
  do {              \
    var = gtime();  \
  } while (0)
#define TC_TRACE(role, ev, step)                                                                  \
  do {                                                                                            \
    if (blockIdx.x == g_trace_cta && (step) < kTraceSteps) g_tc_trace[role][ev][step] = clock64(); \
  } while (0)
#else
#define ITEM_T(var) \
  do {              \
  } while (0)
#define TC_TRACE(role, ev, step) \
  do {                           \
  } while (0)
#endif

constexpr int kThreads = 384;   // warpgroup 0: producer, MMA issuer (+TMEM alloc), 2 idle; warpgroups 1, 2: softmax
constexpr int kSoftWarps = 8;
constexpr int kM = 128;         // rows per group tile (TMEM lanes)
constexpr int kMaxRows = 2 * kM;
constexpr int kNarrow = 16;      // items of <= 16 rows run on the mma.sync path (NS)
constexpr int kN = 64;          // tokens per KV tile
#ifndef PAT_TC3_STAGES
#define PAT_TC3_STAGES 4
#endif
constexpr int kStages = PAT_TC3_STAGES;
constexpr uint32_t kTmemCols = 512;
constexpr float kRescaleThreshold = 8.0f;  // log2 units

struct ItemSlot {
  int32_t idx;
  int32_t pad[7];
  Item item;
  int2 meta[kMaxRows];  // (qid, slot) per row
};
static_assert(sizeof(ItemSlot) == 64 + 8 * kMaxRows, "ItemSlot layout");
constexpr uint32_t kSlotBytes = sizeof(ItemSlot);
constexpr uint32_t kFIdx = 0, kFKvh = 32 + 4, kFRow0 = 32 + 8, kFNrows = 32 + 12, kFNtok = 32 + 20, kFMeta = 64;

template <int D>
struct Layout {
  static constexpr int KB = D / 64;
  static constexpr int kTileBytes = KB * kN * 128;  // K or V stage tile: [KB][64 tok][128 B]
  static constexpr int kQBytes = KB * kM * 128;     // Q buffer: [KB][128 rows][128 B]
  static constexpr int kPW = D / 4;                 // epilogue combine: head-dim columns per pass
  static constexpr int kOffKV = 0;
  static constexpr int kOffQ = kOffKV + kStages * 2 * kTileBytes;
  static constexpr int kOffBar = kOffQ + 2 * kQBytes;
  static constexpr int kOffRing = kOffBar + 512;
  static constexpr int kOffX = kOffRing + 2 * (int)sizeof(ItemSlot);  // [m, l][8 warps][32] floats
  static constexpr int kBytes = kOffX + 2 * kSoftWarps * 32 * 4;
  static constexpr int kAlloc = kBytes + 1024;
  static_assert(kSoftWarps * 32 * kPW * 4 == kQBytes, "combine pass fills one Q buffer");
};

enum Bar : int {
  KV_FULL = 0,
  KV_EMPTY = KV_FULL + kStages,
  S_FULL = KV_EMPTY + kStages,  // [g] QK done
  P_FULL = S_FULL + 2,          // [g] P written over S (4 warps)
  SP_FREE = P_FULL + 2,         // [g] the PV reading P[g] completed (O[g] updated, S/P[g] free)
  O_EMPTY = SP_FREE + 2,        // [g] epilogue has read O[g] (4 warps)
  QT_FULL = O_EMPTY + 2,        // [g] the item's Q rows stored in group g's TMEM (4 warps)
  ITEM_FULL = QT_FULL + 2,      // [slot] published by the producer (32 lanes)
  ITEM_EMPTY = ITEM_FULL + 2,   // [slot] released by the MMA warp and the 8 softmax warps
  NUM_BARS = ITEM_EMPTY + 2
};
static_assert(NUM_BARS * 8 + 8 <= 512, "barrier area");

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
__device__ __forceinline__ float4 lds_v4f(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a)
               : "memory");
  return v;
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
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ Item load_item(const Item* p) {
  const int4* q = reinterpret_cast<const int4*>(p);
  int4 a = __ldg(q), b = __ldg(q + 1);
  return Item{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
}
__device__ __forceinline__ int rep_of(int nrows) { return nrows <= 32 ? 4 : (nrows <= 64 ? 2 : 1); }

template <int D, typename T>
// 12 warps launch with 168 registers; setmaxnreg then moves registers from the
// control warpgroup (56) to the two softmax warpgroups (224): 128 x 56 + 256 x 224 <= 64K
__global__ void __launch_bounds__(kThreads, 1)
    fwd_tc3_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv, DevPlan plan,
                   int var, const T* __restrict__ qg, T* __restrict__ out, float* __restrict__ part_o,
                   float* __restrict__ part_lse, float scale_log2, int32_t* __restrict__ sched) {
  using L = Layout<D>;
  using namespace sm100;
  constexpr bool kSplit = Fmt<T>::kSplit;
  constexpr int KB = L::KB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sb = smem_u32(smem);
  const uint32_t bars = sb + L::kOffBar;
  uint32_t* tmem_slot = (uint32_t*)(smem + L::kOffBar + NUM_BARS * 8);
  ItemSlot* ring = reinterpret_cast<ItemSlot*>(smem + L::kOffRing);
  auto bar = [&](int i) { return bars + 8u * (uint32_t)i; };
  auto sK = [&](int s) { return sb + L::kOffKV + (uint32_t)(s * 2 * L::kTileBytes); };
  auto sV = [&](int s) { return sb + L::kOffKV + (uint32_t)(s * 2 * L::kTileBytes + L::kTileBytes); };
  auto sQ = [&](int qb) { return sb + L::kOffQ + (uint32_t)(qb * L::kQBytes); };

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int H = plan.H, G = plan.G, bs = plan.bs;
  const int n_items = plan.n_items[var];
  const Item* items = plan.items[var];

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(bar(KV_FULL + s), 1);
      mbar_init(bar(KV_EMPTY + s), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(S_FULL + i), 1);
      mbar_init(bar(P_FULL + i), 4);
      mbar_init(bar(SP_FREE + i), 1);
      mbar_init(bar(O_EMPTY + i), 4);
      mbar_init(bar(QT_FULL + i), 4);
      mbar_init(bar(ITEM_FULL + i), 32);
      mbar_init(bar(ITEM_EMPTY + i), 1 + kSoftWarps);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(smem_u32(tmem_slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (elect_one()) {
      tma_prefetch(&tmk);
      tma_prefetch(&tmv);
    }
    uint32_t gt = 0;
    for (uint32_t n = 0;; ++n) {
      const uint32_t slot = n & 1;
      mbar_wait(bar(ITEM_EMPTY + slot), ((n >> 1) & 1) ^ 1);
      // the first item of CTA b is item b (no claim latency at kernel start),
      // later ones come from the counter, offset by the grid
      int it = (int)blockIdx.x;
      if (n > 0 && lane == 0) it = atomicAdd(sched, 1) + (int)gridDim.x;
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
        // warm L2 with the item's Q rows (the softmax warps copy them into
        // shared memory at the previous item's end): one bulk prefetch per query
        const int i0 = item.row0 / G, i1 = (item.row0 + item.nrows - 1) / G;
        for (int i = i0 + lane; i <= i1; i += 32) {
          const int qid = __ldg(plan.pack_q + item.qoff + i);
          const int a = max(i * G, item.row0), e = min((i + 1) * G, item.row0 + item.nrows);
          bulk_prefetch_l2(qg + ((int64_t)qid * H + item.kvh * G + (a - i * G)) * D, (uint32_t)((e - a) * D * 2));
        }
      }
      if (lane == 0) ring[slot].idx = it;
      __syncwarp();
      mbar_arrive(bar(ITEM_FULL + slot));
      if (it < 0) break;
      const int h = item.kvh, ntok = item.ntok;
      const int32_t* blist = plan.pack_blk + item.blk;
      const int ntiles = (ntok + kN - 1) / kN;
      for (int j = 0; j < ntiles; ++j, ++gt) {
        const int s = gt % kStages;
        const int rem = ntok - j * kN;
        const int ngrp = rem >= kN ? kN / 16 : (rem + 15) / 16;
        int my_blk = 0, my_off = 0;
        if (lane < ngrp) {
          const int tok = j * kN + lane * 16;
          const int pg = bs == 16 ? (tok >> 4) : tok / bs;
          my_blk = __ldg(blist + pg);
          my_off = bs == 16 ? 0 : tok - pg * bs;
        }
        mbar_wait(bar(KV_EMPTY + s), ((gt / kStages) & 1) ^ 1);
        TC_TRACE(0, 0, gt);
        if (elect_one()) mbar_expect_tx(bar(KV_FULL + s), (uint32_t)(ngrp * KB * 2048 * 2));
        __syncwarp();
        for (int gr = 0; gr < ngrp; ++gr) {
          const int blk = __shfl_sync(0xffffffffu, my_blk, gr);
          const int off = __shfl_sync(0xffffffffu, my_off, gr);
          if (elect_one()) {
#pragma unroll
            for (int kb = 0; kb < KB; ++kb) {
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
    // Per group g one S/P buffer: QK(g) may overwrite it once the PV that
    // read the previous P of g completed (SP_FREE), so each group's chain is
    // softmax -> PV -> QK -> softmax, and the two groups interleave on the
    // tensor pipe.
    constexpr uint32_t idesc_qk = umma_idesc_f16(kM, kN, Fmt<T>::ab, 0);
    constexpr uint32_t idesc_pv = umma_idesc_f16(kM, D, Fmt<T>::ab, 1);
    uint32_t gt = 0;                  // KV tiles consumed (ring position)
    // per-group counters, scalars (a group index known at compile time picks
    // the register): QKs issued, PVs issued, Q stores consumed, items that
    // accumulated into O[g]
    uint32_t cq0 = 0, cq1 = 0, cv0 = 0, cv1 = 0, qu0 = 0, qu1 = 0, ou0 = 0, ou1 = 0;
    auto commit = [&](int b) {
      if (elect_one()) umma_commit(bar(b));
      __syncwarp();
    };
    for (uint32_t n = 0;; ++n) {
      mbar_wait(bar(ITEM_FULL + (n & 1)), (n >> 1) & 1);
      const uint32_t rs = sb + L::kOffRing + (n & 1) * kSlotBytes;
      const int it = lds_s32(rs + kFIdx);
      const int ntok = it >= 0 ? lds_s32(rs + kFNtok) : 0;
      const int nrows = it >= 0 ? lds_s32(rs + kFNrows) : 0;
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(ITEM_EMPTY + (n & 1)));
      if (it < 0) break;
      const bool pp = nrows > kM;
      const int ntiles = (ntok + kN - 1) / kN;
      if (nrows <= kNarrow) {  // the softmax warps run it on mma.sync
        gt += (uint32_t)ntiles;
        continue;
      }
      auto stage_of = [&](int t) { return (int)((gt + (uint32_t)t) % kStages); };
      auto kv_wait = [&](int t) {
        const uint32_t gg = gt + (uint32_t)t;
        mbar_wait(bar(KV_FULL + gg % kStages), (gg / kStages) & 1);
        TC_TRACE(1, 0, gg);
      };
      auto qk = [&](auto g_tag, int s, bool first) {
        constexpr int g = decltype(g_tag)::value;
        uint32_t& cq = g ? cq1 : cq0;
        uint32_t& qu = g ? qu1 : qu0;
        mbar_wait(bar(SP_FREE + g), (cq & 1) ^ 1);  // previous PV of g done: S/P[g] free
        if (first) mbar_wait(bar(QT_FULL + g), qu++ & 1);
        tc_fence_after();
        const uint64_t k0 = umma_desc_sw128(sK(s), 16, 1024);
        const uint32_t tg = tmem + (uint32_t)(g * 256);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const int kb = k >> 2, kk = k & 3;
            // Q(m, k) packed two per column: a k-step of 16 = 8 columns
            umma_f16_ts(tg, tg + 64u + (uint32_t)(k * 8), k0 + (uint64_t)((kb * (kN * 128) + kk * 32) >> 4),
                        idesc_qk, k > 0 ? 1u : 0u);
          }
          umma_commit(bar(S_FULL + g));
        }
        __syncwarp();
        ++cq;
      };
      auto pv = [&](auto g_tag, int s, bool first) {
        constexpr int g = decltype(g_tag)::value;
        uint32_t& cv = g ? cv1 : cv0;
        mbar_wait(bar(P_FULL + g), cv & 1);
        if (first) mbar_wait(bar(O_EMPTY + g), ((g ? ou1 : ou0) & 1) ^ 1);
        tc_fence_after();
        const uint64_t v0 = umma_desc_sw128(sV(s), kN * 128, 1024);
        const uint32_t tg = tmem + (uint32_t)(g * 256);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < kN / 16; ++k) {
            const uint64_t bd = v0 + (uint64_t)((k * 16 * 128) >> 4);
            // P(m, k) is packed two per column: a k-step of 16 tokens = 8 columns
            umma_f16_ts(tg + 128u, tg + (uint32_t)(k * 8), bd, idesc_pv, (first && k == 0) ? 0u : 1u);
            if constexpr (kSplit) umma_f16_ts(tg + 128u, tg + 32u + (uint32_t)(k * 8), bd, idesc_pv, 1u);
          }
          umma_commit(bar(SP_FREE + g));
        }
        __syncwarp();
        ++cv;
      };
      const std::integral_constant<int, 0> G0{};
      const std::integral_constant<int, 1> G1{};
      TC_TRACE(1, 5, gt);
      if (pp) {
        kv_wait(0);
        qk(G0, stage_of(0), true);
        qk(G1, stage_of(0), true);
        TC_TRACE(1, 1, gt);
        for (int t = 0; t < ntiles; ++t) {
          const int s = stage_of(t);
          TC_TRACE(1, 4, gt + t);
          pv(G0, s, t == 0);
          if (t + 1 < ntiles) {
            kv_wait(t + 1);
            qk(G0, stage_of(t + 1), false);
          }
          pv(G1, s, t == 0);
          commit(KV_EMPTY + s);
          if (t + 1 < ntiles) qk(G1, stage_of(t + 1), false);
          TC_TRACE(1, 2, gt + t);
        }
        ++ou0, ++ou1;
      } else {
        kv_wait(0);
        qk(G0, stage_of(0), true);
        if (ntiles > 1) {
          kv_wait(1);
          qk(G1, stage_of(1), true);
        }
        TC_TRACE(1, 1, gt);
        for (int t = 0; t < ntiles; ++t) {
          const int s = stage_of(t);
          TC_TRACE(1, 4, gt + t);
          if (t & 1) pv(G1, s, t < 2);
          else pv(G0, s, t < 2);
          commit(KV_EMPTY + s);
          if (t + 2 < ntiles) {
            kv_wait(t + 2);
            if (t & 1) qk(G1, stage_of(t + 2), false);
            else qk(G0, stage_of(t + 2), false);
          }
          TC_TRACE(1, 2, gt + t);
        }
        ++ou0;
        if (ntiles >= 2) ++ou1;
      }
      gt += (uint32_t)ntiles;
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n" ::: "memory");
    // ------------------------------------------------------------ softmax / epilogue
    const int g = (warp - 4) >> 2;     // softmax group (warpgroup 1 or 2)
    const int wq = warp & 3;           // TMEM lane quarter
    const int ws = warp - 4;           // 0..7: slot in the exchange arrays
    const int tid8 = ws * 32 + lane;   // 0..255 over both groups
    const int ln = wq * 32 + lane;     // TMEM lane
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    const uint32_t tg = tmem + (uint32_t)(g * 256);  // this group's TMEM columns
    const uint32_t ring_s = sb + L::kOffRing;
    auto fld = [&](uint32_t n, uint32_t off) { return lds_s32(ring_s + (n & 1) * kSlotBytes + off); };
    const bool tr = (g == 0 && wq == 0 && lane == 0);
    uint32_t gt = 0, cs = 0;
    const uint32_t xml = sb + L::kOffX;  // [2: m, l][8 warps][32] floats

    auto wait_item = [&](uint32_t n) { mbar_wait(bar(ITEM_FULL + (n & 1)), (n >> 1) & 1); };
    auto tiles_of = [&](uint32_t n) {  // this group's KV tiles in item n
      const int nt = (fld(n, kFNtok) + kN - 1) / kN;
      return fld(n, kFNrows) > kM ? nt : (nt + 1 - g) / 2;
    };
    auto tc_item = [&](uint32_t n) { return fld(n, kFNrows) > kNarrow; };  // runs on tcgen05
    // the row this thread holds for item n: EO = the R-replicated layout, PP = 128 g + lane
    auto row_of = [&](uint32_t n) {
      const int nr = fld(n, kFNrows);
      return nr > kM ? g * kM + ln : (wq % (4 / rep_of(nr))) * 32 + lane;
    };
    auto q_src = [&](uint32_t n, int r, bool& live) {
      live = r < fld(n, kFNrows);
      const int qid = live ? fld(n, kFMeta + 8 * r) : 0;
      const int head = fld(n, kFKvh) * G + (live ? (fld(n, kFRow0) + r) % G : 0);
      return reinterpret_cast<const uint8_t*>(qg + ((int64_t)qid * H + head) * D);
    };
    // EO item n: cp.async this thread's Q row into staging buffer n & 1 (row =
    // TMEM lane, 128B-swizzled 16-byte chunks; both groups write the same rows)
    auto stage_q = [&](uint32_t n) {
      bool live;
      const uint8_t* src = q_src(n, row_of(n), live);
      const uint32_t dq = sQ((int)(n & 1)) + (uint32_t)(ln * 128);
#pragma unroll
      for (int ch = 0; ch < D / 8; ++ch)
        cp_async16(dq + (uint32_t)((ch >> 3) * (kM * 128) + (((ch & 7) ^ (ln & 7)) << 4)), src + ch * 16,
                   live ? 16u : 0u);
      cp_async_commit();
    };
    auto read_staged = [&](uint32_t n, uint32_t* qv) {
      const uint32_t dq = sQ((int)(n & 1)) + (uint32_t)(ln * 128);
#pragma unroll
      for (int ch = 0; ch < D / 8; ++ch) {
        const float4 v = lds_v4f(dq + (uint32_t)((ch >> 3) * (kM * 128) + (((ch & 7) ^ (ln & 7)) << 4)));
        qv[4 * ch] = __float_as_uint(v.x), qv[4 * ch + 1] = __float_as_uint(v.y);
        qv[4 * ch + 2] = __float_as_uint(v.z), qv[4 * ch + 3] = __float_as_uint(v.w);
      }
    };
    auto load_q_global = [&](uint32_t n, uint32_t* qv) {
      bool live;
      const uint4* src = reinterpret_cast<const uint4*>(q_src(n, row_of(n), live));
#pragma unroll
      for (int i = 0; i < D / 8; ++i) {
        const uint4 v = live ? __ldg(src + i) : make_uint4(0, 0, 0, 0);
        qv[4 * i] = v.x, qv[4 * i + 1] = v.y, qv[4 * i + 2] = v.z, qv[4 * i + 3] = v.w;
      }
    };
    auto store_q = [&](const uint32_t* qv) {
#pragma unroll
      for (int i = 0; i < D / 64; ++i) tmem_st32_nowait(tg + 64u + lane_base + 32u * i, qv + 32 * i);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(QT_FULL + g));
    };

    // ---------------------------------------------------------- narrow items (NS)
    // An item of <= 16 rows (a query or two x G) would waste a 128-lane tcgen05
    // tile; it runs on mma.sync m16n8k16 instead: the two groups take
    // alternate KV tiles, each warp 16 tokens of a tile (QK, online softmax,
    // PV, all in registers, reading the same TMA stage layout the tcgen05
    // path uses), and the 8 warps' partial states are folded at the end.
    auto narrow_item = [&](uint32_t n, long long& t_first, long long& t_done) {
      (void)t_first, (void)t_done;
      const int ntok = fld(n, kFNtok), nrows = fld(n, kFNrows);
      const int kvh = fld(n, kFKvh), row0 = fld(n, kFRow0);
      const int ntiles = (ntok + kN - 1) / kN;
      const uint32_t meta_s = ring_s + (n & 1) * kSlotBytes + kFMeta;
      const int r_lo = lane >> 2, r_hi = r_lo + 8, tq = (lane & 3) * 2;
      // Q fragments (A operand): rows r_lo / r_hi, 16-element k-steps
      uint32_t qa[D / 16][4];
      {
        auto qrow = [&](int r) -> const uint32_t* {
          if (r >= nrows) return nullptr;
          const int qid = lds_s32(meta_s + 8 * r);
          return reinterpret_cast<const uint32_t*>(qg + ((int64_t)qid * H + kvh * G + (row0 + r) % G) * D);
        };
        const uint32_t* p0 = qrow(r_lo);
        const uint32_t* p1 = qrow(r_hi);
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const int c = (ks * 16 + tq) >> 1;  // 32-bit word of the pair
          qa[ks][0] = p0 ? __ldg(p0 + c) : 0u;
          qa[ks][1] = p1 ? __ldg(p1 + c) : 0u;
          qa[ks][2] = p0 ? __ldg(p0 + c + 4) : 0u;
          qa[ks][3] = p1 ? __ldg(p1 + c + 4) : 0u;
        }
      }
      float o[D / 8][4];
#pragma unroll
      for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
      float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
      const int t0w = wq * 16;  // this warp's first token inside a tile
      for (int t = g; t < ntiles; t += 2) {
        const uint32_t gg = gt + (uint32_t)t;
        const int s = gg % kStages;
        mbar_wait(bar(KV_FULL + s), (gg / kStages) & 1);
        if (tr && t == g) ITEM_T(t_first);
        const uint32_t tk = sK(s), tv = sV(s);
        const int valid = ntok - t * kN - t0w;  // valid tokens of this warp's 16
        if (valid < 16) {
          // rows past the span hold stale bytes: zero this warp's V rows so P == 0 cannot meet a NaN
          for (int c = lane; c < 16 * (D / 8); c += 32) {
            const int tt = t0w + c / (D / 8), ch = c % (D / 8);
            if (tt - t0w >= valid)
              st_shared_v4(tv + (uint32_t)((ch >> 3) * (kN * 128) + tt * 128 + (((ch & 7) ^ (tt & 7)) << 4)),
                           make_uint4(0, 0, 0, 0));
          }
          __syncwarp();
        }
        float sc[2][4];
#pragma unroll
        for (int j = 0; j < 2; ++j) sc[j][0] = sc[j][1] = sc[j][2] = sc[j][3] = 0.f;
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          uint32_t b[4];
          const int tt = t0w + (lane & 7) + (lane >> 4) * 8;
          const int ch = ks * 2 + ((lane >> 3) & 1);
          ldsm_x4(b, tk + (uint32_t)((ch >> 3) * (kN * 128) + tt * 128 + (((ch & 7) ^ (tt & 7)) << 4)));
          mma16816<T>(sc[0], qa[ks], b[0], b[1]);
          mma16816<T>(sc[1], qa[ks], b[2], b[3]);
        }
        float mx[2] = {mrow[0], mrow[1]};
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int tok = j * 8 + tq + (e & 1);
            const float v = tok < valid ? sc[j][e] * scale_log2 : -INFINITY;
            sc[j][e] = v;
            mx[e >> 1] = fmaxf(mx[e >> 1], v);
          }
        float muse[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
          mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
          muse[r] = mx[r] == -INFINITY ? 0.f : mx[r];
          const float alpha = ex2_approx(mrow[r] - muse[r]);  // -inf -> 0
          mrow[r] = mx[r];
          lrow[r] *= alpha;
#pragma unroll
          for (int i = 0; i < D / 8; ++i) {
            o[i][2 * r] *= alpha;
            o[i][2 * r + 1] *= alpha;
          }
        }
        uint32_t pa[4], pl[4];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const float p0 = ex2_approx(sc[j][0] - muse[0]), p1 = ex2_approx(sc[j][1] - muse[0]);
          const float p2 = ex2_approx(sc[j][2] - muse[1]), p3 = ex2_approx(sc[j][3] - muse[1]);
          const uint32_t h01 = Fmt<T>::pack(p0, p1), h23 = Fmt<T>::pack(p2, p3);
          pa[2 * j] = h01;
          pa[2 * j + 1] = h23;
          if constexpr (kSplit) {
            const float2 f01 = Fmt<T>::unpack(h01), f23 = Fmt<T>::unpack(h23);
            pl[2 * j] = Fmt<T>::pack(p0 - f01.x, p1 - f01.y);
            pl[2 * j + 1] = Fmt<T>::pack(p2 - f23.x, p3 - f23.y);
            lrow[0] += p0 + p1;
            lrow[1] += p2 + p3;
          } else {
            const float2 f01 = Fmt<T>::unpack(h01), f23 = Fmt<T>::unpack(h23);
            lrow[0] += f01.x + f01.y;
            lrow[1] += f23.x + f23.y;
          }
        }
#pragma unroll
        for (int dn = 0; dn < D / 16; ++dn) {
          uint32_t b[4];
          const int tt = t0w + (lane & 7) + ((lane >> 3) & 1) * 8;
          const int ch = dn * 2 + (lane >> 4);
          ldsm_x4_t(b, tv + (uint32_t)((ch >> 3) * (kN * 128) + tt * 128 + (((ch & 7) ^ (tt & 7)) << 4)));
          mma16816<T>(o[dn * 2], pa, b[0], b[1]);
          mma16816<T>(o[dn * 2 + 1], pa, b[2], b[3]);
          if constexpr (kSplit) {
            mma16816<T>(o[dn * 2], pl, b[0], b[1]);
            mma16816<T>(o[dn * 2 + 1], pl, b[2], b[3]);
          }
        }
        // the group's four warps have read the stage: release it
        named_bar_sync(2 + g, 128);
        if (wq == 0 && lane == 0) mbar_arrive(bar(KV_EMPTY + s));
      }
      if (tr) ITEM_T(t_done);
      // ---- fold the 8 warps' partial states (merge_partials) through smem
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 1);
        lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 2);
      }
      if ((lane & 3) == 0) {  // [m, l][8 warps][16 rows]
        sts_f32(xml + (uint32_t)(ws * 16 + r_lo) * 4, mrow[0]);
        sts_f32(xml + (uint32_t)(ws * 16 + r_hi) * 4, mrow[1]);
        sts_f32(xml + (uint32_t)(128 + ws * 16 + r_lo) * 4, lrow[0]);
        sts_f32(xml + (uint32_t)(128 + ws * 16 + r_hi) * 4, lrow[1]);
      }
      constexpr int PWN = L::kQBytes / (kSoftWarps * 16 * 4);  // head-dim columns per pass
      const uint32_t xs = sQ((int)(n & 1));                    // this item's staging buffer
      // the summing thread: row rs_ of the item, 4 columns c4_ of the pass
      const int rs_ = tid8 / (PWN / 4), c4_ = tid8 % (PWN / 4);
      float wgt[kSoftWarps], M = -INFINITY, Lsum = 0.f;
#pragma unroll  // static indices into o[]
      for (int q = 0; q < D / PWN; ++q) {
        // [8 warps][16 rows][PWN] floats, unscaled partial O
        const uint32_t wb = xs + (uint32_t)(ws * 16 * PWN * 4);
#pragma unroll
        for (int i = 0; i < PWN / 8; ++i) {
          const int ii = q * (PWN / 8) + i;
          const int col = i * 8 + tq;
          asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(wb + (uint32_t)((r_lo * PWN + col) * 4)),
                       "f"(o[ii][0]), "f"(o[ii][1])
                       : "memory");
          asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(wb + (uint32_t)((r_hi * PWN + col) * 4)),
                       "f"(o[ii][2]), "f"(o[ii][3])
                       : "memory");
        }
        named_bar_sync(1, 256);
        if (q == 0 && rs_ < 16) {
#pragma unroll
          for (int w = 0; w < kSoftWarps; ++w) M = fmaxf(M, lds_f32(xml + (uint32_t)(w * 16 + rs_) * 4));
#pragma unroll
          for (int w = 0; w < kSoftWarps; ++w) {
            const float mw = lds_f32(xml + (uint32_t)(w * 16 + rs_) * 4);
            wgt[w] = mw == -INFINITY ? 0.f : ex2_approx(mw - M);
            Lsum += wgt[w] * lds_f32(xml + (uint32_t)(128 + w * 16 + rs_) * 4);
          }
          const float inv = 1.f / Lsum;
#pragma unroll
          for (int w = 0; w < kSoftWarps; ++w) wgt[w] *= inv;
        }
        if (rs_ < nrows) {
          float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int w = 0; w < kSoftWarps; ++w) {
            const float4 v = lds_v4f(xs + (uint32_t)(((w * 16 + rs_) * PWN + c4_ * 4) * 4));
            acc.x += wgt[w] * v.x, acc.y += wgt[w] * v.y, acc.z += wgt[w] * v.z, acc.w += wgt[w] * v.w;
          }
          const int2 meta = lds_v2(meta_s + 8 * rs_);
          const int head = kvh * G + (row0 + rs_) % G;
          const int col = q * PWN + c4_ * 4;
          if (meta.y < 0) {
            uint2* dst = reinterpret_cast<uint2*>(out + ((int64_t)meta.x * H + head) * D + col);
            *dst = make_uint2(Fmt<T>::pack(acc.x, acc.y), Fmt<T>::pack(acc.z, acc.w));
          } else {
            *reinterpret_cast<float4*>(part_o + ((int64_t)meta.y * H + head) * D + col) = acc;
            if (q == 0 && c4_ == 0) part_lse[(int64_t)meta.y * H + head] = M + log2f(Lsum);
          }
        }
        named_bar_sync(1, 256);
      }
    };

    wait_item(0);
    if (fld(0, kFIdx) >= 0 && tc_item(0) && tiles_of(0) > 0) {
      uint32_t qv[D / 2];
      load_q_global(0, qv);
      store_q(qv);
    }
    for (uint32_t n = 0;; ++n) {
      if (fld(n, kFIdx) < 0) break;  // ITEM_FULL(n) already waited
      const int ntok = fld(n, kFNtok);
      const int nrows = fld(n, kFNrows);
      const int kvh = fld(n, kFKvh), row0 = fld(n, kFRow0);
      const bool pp = nrows > kM;
      const int ntiles = (ntok + kN - 1) / kN;
      const int R = pp ? 1 : rep_of(nrows);
      const int QPC = 4 / R;                                  // lane quarters per copy
      const int kc = pp ? 0 : wq / QPC;                       // column slice of this warp
      const int row = pp ? g * kM + ln : (wq % QPC) * 32 + lane;
      const bool wlive = pp ? (g * kM + wq * 32 < nrows) : ((wq % QPC) * 32 < nrows);
      const int my_tiles = tiles_of(n);
      float m_ref = -INFINITY;  // running max, log2 units
      float2 l2 = make_float2(0.f, 0.f);
      int next_state = 0;  // 0 unknown, 1 staged (EO next), 2 known (no staging)
      long long it0 = 0, it1 = 0, it2 = 0, it3 = 0;
      (void)it0, (void)it1, (void)it2, (void)it3;
      if (tr) ITEM_T(it0);

      // one KV tile with NC score columns per thread
      auto tile = [&](auto nc_tag, int t, int k_mine) {
        constexpr int NC = decltype(nc_tag)::value;
        const uint32_t gg = gt + (uint32_t)t;
        if (next_state == 0 && mbar_test(bar(ITEM_FULL + ((n + 1) & 1)), ((n + 1) >> 1) & 1)) {
          // the next item is published: stage its Q rows now (EO), hidden behind this item
          const bool nx = fld(n + 1, kFIdx) >= 0 && fld(n + 1, kFNrows) <= kM && tc_item(n + 1);
          if (nx) stage_q(n + 1);
          next_state = nx ? 1 : 2;
        }
        mbar_wait(bar(S_FULL + g), cs & 1);
        if (tr) TC_TRACE(2, 0, gg);
        if (tr && k_mine == 0) ITEM_T(it1);
        tc_fence_after();
        const uint32_t sp = tg + lane_base;
        if (wlive) {
          uint32_t sr[NC];
          tmem_ld_n<NC>(sp + (uint32_t)(kc * NC), sr);
          if (tr) TC_TRACE(2, 6, gg);
          const int valid = ntok - t * kN - kc * NC;  // valid columns of this slice
          if (valid < NC) {
#pragma unroll
            for (int k = 0; k < NC; ++k)
              if (k >= valid) sr[k] = __float_as_uint(-INFINITY);
          }
          float pm[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
          for (int k = 0; k < NC / 8; ++k)
            pm[k & 3] = fmax3(pm[k & 3],
                              fmax3(__uint_as_float(sr[8 * k]), __uint_as_float(sr[8 * k + 1]),
                                    __uint_as_float(sr[8 * k + 2])),
                              fmax3(__uint_as_float(sr[8 * k + 3]), __uint_as_float(sr[8 * k + 4]),
                                    fmax3(__uint_as_float(sr[8 * k + 5]), __uint_as_float(sr[8 * k + 6]),
                                          __uint_as_float(sr[8 * k + 7]))));
          const float mx = fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])) * scale_log2;
          if (tr) TC_TRACE(2, 7, gg);
          const bool need = mx > m_ref + kRescaleThreshold;
          if (__any_sync(0xffffffffu, need)) {
            const float m_new = need ? mx : m_ref;
            const float alpha = m_new == -INFINITY ? 1.f : ex2_approx(m_ref - m_new);
            if (k_mine > 0) {
              // O[g] holds this group's previous PV (it completed before this QK was issued)
#pragma unroll 1
              for (int q = 0; q < D / 16; ++q) {
                uint32_t o[16];
                const uint32_t ta = tg + 128u + lane_base + (uint32_t)(q * 16);
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
          // P = exp2(s * scale - m_ref) for the slice, packed pairs (a slice
          // with no valid column so far keeps m_ref = -inf: reference 0, P = 0)
          const float mu = m_ref == -INFINITY ? 0.f : m_ref;
          const float2 sc2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-mu, -mu);
          // (in chunks of at most 32 columns: keeps the P registers of a
          // 64-column slice from piling up on top of S)
          constexpr int CH = NC < 32 ? NC : 32;
#pragma unroll
          for (int c0 = 0; c0 < NC; c0 += CH) {
            uint32_t ph[CH / 2], pl[CH / 2];
#pragma unroll
            for (int k = 0; k < CH / 2; ++k) {
              float2 a = __ffma2_rn(make_float2(__uint_as_float(sr[c0 + 2 * k]), __uint_as_float(sr[c0 + 2 * k + 1])),
                                    sc2, nm2);
              a.x = ex2_approx(a.x);
              a.y = ex2_approx(a.y);
              ph[k] = Fmt<T>::pack(a.x, a.y);
              if constexpr (kSplit) {
                const float2 hf = Fmt<T>::unpack(ph[k]);
                const float2 lo = __fadd2_rn(a, make_float2(-hf.x, -hf.y));
                pl[k] = Fmt<T>::pack(lo.x, lo.y);
                l2 = __fadd2_rn(l2, a);
              } else {
                // normalise by the sum of the ROUNDED weights the MMA actually uses
                l2 = __fadd2_rn(l2, Fmt<T>::unpack(ph[k]));
              }
            }
            // P over the consumed S: this slice, zeros in the other slices' columns
            if constexpr (NC == kN) {
              tmem_st_n<CH / 2>(sp + (uint32_t)(c0 / 2), ph);
              if constexpr (kSplit) tmem_st_n<CH / 2>(sp + 32u + (uint32_t)(c0 / 2), pl);
            } else {
#pragma unroll
              for (int gi = 0; gi < kN / NC; ++gi) {
                uint32_t vh[NC / 2], vl[NC / 2];
#pragma unroll
                for (int e = 0; e < NC / 2; ++e) {
                  vh[e] = gi == kc ? ph[e] : 0u;
                  if constexpr (kSplit) vl[e] = gi == kc ? pl[e] : 0u;
                }
                tmem_st_n<NC / 2>(sp + (uint32_t)(gi * (NC / 2)), vh);
                if constexpr (kSplit) tmem_st_n<NC / 2>(sp + 32u + (uint32_t)(gi * (NC / 2)), vl);
              }
            }
          }
          if (tr) TC_TRACE(2, 1, gg);
        }
        if (t * kN + kN > ntok && (!pp || g == 0)) {
          // tail tile: zero V rows past the span (stale / uninitialised smem)
          const int vt = ntok - t * kN;
          const int s = gg % kStages;
          mbar_wait(bar(KV_FULL + s), (gg / kStages) & 1);
          const int nz = (kN - vt) * KB * 8;
          for (int q = ln; q < nz; q += kM) {
            const int rr = vt + q / (KB * 8);
            const int kb = (q / 8) % KB, ch = q % 8;
            st_shared_v4(sV(s) + kb * (kN * 128) + rr * 128 + (ch << 4), make_uint4(0, 0, 0, 0));
          }
          fence_proxy_async_smem();
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar(P_FULL + g));
        if (tr) TC_TRACE(2, 3, gg);
        ++cs;
      };
      auto run_tiles = [&](auto nc_tag) {
        const int t0 = pp ? 0 : g, dt = pp ? 1 : 2;
        int k = 0;
        for (int t = t0; t < ntiles; t += dt, ++k) tile(nc_tag, t, k);
      };
      const bool ns = nrows <= kNarrow;
      if (ns) narrow_item(n, it1, it2);
      else if (R == 4) run_tiles(std::integral_constant<int, 16>{});
      else if (R == 2) run_tiles(std::integral_constant<int, 32>{});
      else run_tiles(std::integral_constant<int, 64>{});

      if (tr && !ns) ITEM_T(it2);
      // The next item's Q into this group's TMEM (its QKs for this item are
      // done), so the next item's first QK overlaps this epilogue.
      wait_item(n + 1);
      const bool have_next = fld(n + 1, kFIdx) >= 0;
      if (have_next && tc_item(n + 1)) {
        const bool next_eo = fld(n + 1, kFNrows) <= kM;
        if (next_eo && next_state != 1) stage_q(n + 1);
        uint32_t qv[D / 2];
        if (next_eo) {
          cp_async_wait_all();
          if (tiles_of(n + 1) > 0) read_staged(n + 1, qv);
        } else if (tiles_of(n + 1) > 0) {
          load_q_global(n + 1, qv);
        }
        if (tiles_of(n + 1) > 0) store_q(qv);
      }

      if (!ns) {
      // last PV of this group done
      if (my_tiles > 0) {
        mbar_wait(bar(SP_FREE + g), (cs - 1) & 1);
        tc_fence_after();
      }
      if (tr) TC_TRACE(3, 1, gt);
      const uint32_t meta_s = ring_s + (n & 1) * kSlotBytes + kFMeta;
      if (pp) {
        // one row per thread, written directly
        const float l = l2.x + l2.y;
        const bool live = row < nrows;
        const int2 meta = live ? lds_v2(meta_s + 8 * row) : make_int2(0, -1);
        const int head = kvh * G + (live ? (row0 + row) % G : 0);
        if (wlive) {
          const float inv = 1.f / l;
#pragma unroll 1
          for (int q = 0; q < D / 32; ++q) {
            uint32_t o[32];
            tmem_ld32(tg + 128u + lane_base + (uint32_t)(q * 32), o);
            if (live) {
              const float* f = reinterpret_cast<const float*>(o);
              if (meta.y < 0) {
                uint4* dst = reinterpret_cast<uint4*>(out + ((int64_t)meta.x * H + head) * D + q * 32);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  dst[k] = make_uint4(Fmt<T>::pack(f[8 * k] * inv, f[8 * k + 1] * inv),
                                      Fmt<T>::pack(f[8 * k + 2] * inv, f[8 * k + 3] * inv),
                                      Fmt<T>::pack(f[8 * k + 4] * inv, f[8 * k + 5] * inv),
                                      Fmt<T>::pack(f[8 * k + 6] * inv, f[8 * k + 7] * inv));
              } else {
                float4* dst = reinterpret_cast<float4*>(part_o + ((int64_t)meta.y * H + head) * D + q * 32);
#pragma unroll
                for (int k = 0; k < 8; ++k)
                  dst[k] = make_float4(f[4 * k] * inv, f[4 * k + 1] * inv, f[4 * k + 2] * inv, f[4 * k + 3] * inv);
              }
            }
          }
          if (live && meta.y >= 0) part_lse[(int64_t)meta.y * H + head] = m_ref + log2f(l);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar(O_EMPTY + g));
      } else {
        // combine the 2R partial states of each row (online-softmax fold, as
        // merge_partials) through shared memory; this item's Q staging buffer
        // (copied to TMEM before the item started) is the scratch.
        const bool had = my_tiles > 0;
        sts_f32(xml + (uint32_t)(ws * 32 + lane) * 4, had ? m_ref : -INFINITY);
        sts_f32(xml + (uint32_t)((kSoftWarps + ws) * 32 + lane) * 4, had ? l2.x + l2.y : 0.f);
        named_bar_sync(1, 256);
        // copy (group gg, copy i) of row `row` lives in warp slot gg * 4 + q, q = (row >> 5) + i * QPC
        float M = -INFINITY, Lsum = 0.f;
        for (int gg = 0; gg < 2; ++gg)
          for (int i = 0; i < R; ++i) {
            const int sl = gg * 4 + ((row >> 5) + i * QPC);
            M = fmaxf(M, lds_f32(xml + (uint32_t)(sl * 32 + lane) * 4));
          }
        for (int gg = 0; gg < 2; ++gg)
          for (int i = 0; i < R; ++i) {
            const int sl = gg * 4 + ((row >> 5) + i * QPC);
            const float mi = lds_f32(xml + (uint32_t)(sl * 32 + lane) * 4);
            const float li = lds_f32(xml + (uint32_t)((kSoftWarps + sl) * 32 + lane) * 4);
            Lsum += mi == -INFINITY ? 0.f : li * ex2_approx(mi - M);
          }
        const bool mine_live = had && m_ref != -INFINITY;
        const float f = mine_live ? ex2_approx(m_ref - M) / Lsum : 0.f;
        if (g == 0 && kc == 0 && row < nrows) {
          const int2 meta = lds_v2(meta_s + 8 * row);
          if (meta.y >= 0) part_lse[(int64_t)meta.y * H + kvh * G + (row0 + row) % G] = M + log2f(Lsum);
        }
        constexpr int PW = L::kPW, PC = PW / 4;  // columns per pass, 16-byte chunks per row per pass
        const uint32_t xs = sQ((int)(n & 1));
#pragma unroll 1
        for (int q = 0; q < D / PW; ++q) {
          uint32_t o[PW];
          if (had) {
            tmem_ld_n<PW>(tg + 128u + lane_base + (uint32_t)(q * PW), o);
            if (q == D / PW - 1) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(bar(O_EMPTY + g));
            }
          }
          const uint32_t rowp = xs + (uint32_t)((ws * 32 + lane) * PW * 4);
#pragma unroll
          for (int k = 0; k < PC; ++k) {
            uint4 v = make_uint4(0, 0, 0, 0);
            if (mine_live)
              v = make_uint4(__float_as_uint(__uint_as_float(o[4 * k]) * f),
                             __float_as_uint(__uint_as_float(o[4 * k + 1]) * f),
                             __float_as_uint(__uint_as_float(o[4 * k + 2]) * f),
                             __float_as_uint(__uint_as_float(o[4 * k + 3]) * f));
            st_shared_v4(rowp + (uint32_t)((k ^ (lane & (PC - 1))) << 4), v);
          }
          named_bar_sync(1, 256);
          for (int pr = tid8; pr < nrows * PC; pr += 256) {
            const int rr = pr / PC, ch = pr % PC;
            const int lr = rr & 31;
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int gg = 0; gg < 2; ++gg)
              for (int i = 0; i < R; ++i) {
                const int sl = gg * 4 + ((rr >> 5) + i * QPC);
                const float4 v = lds_v4f(xs + (uint32_t)((sl * 32 + lr) * PW * 4 + ((ch ^ (lr & (PC - 1))) << 4)));
                acc.x += v.x, acc.y += v.y, acc.z += v.z, acc.w += v.w;
              }
            const int2 meta = lds_v2(meta_s + 8 * rr);
            const int head = kvh * G + (row0 + rr) % G;
            const int col = q * PW + ch * 4;
            if (meta.y < 0) {
              uint2* dst = reinterpret_cast<uint2*>(out + ((int64_t)meta.x * H + head) * D + col);
              *dst = make_uint2(Fmt<T>::pack(acc.x, acc.y), Fmt<T>::pack(acc.z, acc.w));
            } else {
              *reinterpret_cast<float4*>(part_o + ((int64_t)meta.y * H + head) * D + col) = acc;
            }
          }
          named_bar_sync(1, 256);
        }
      }
      }  // tcgen05 epilogue
      if (tr) TC_TRACE(3, 2, gt);
#ifdef PAT_TC_TRACE
      if (tr) {
        ITEM_T(it3);
        const int k = atomicAdd(&g_item_n, 1);
        if (k < kItemLog) {
          long long* e = g_item_log[k];
          e[0] = blockIdx.x, e[1] = fld(n, kFIdx), e[2] = nrows, e[3] = ntiles;
          e[4] = it0, e[5] = it1, e[6] = it2, e[7] = it3;
        }
      }
#endif
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(ITEM_EMPTY + (n & 1)));
      gt += (uint32_t)ntiles;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
  if (tid == 0) {
    // the last CTA out re-arms the item counter for the next launch
    __threadfence();
    if (atomicAdd(sched + 1, 1) == (int)gridDim.x - 1) {
      sched[0] = 0;
      sched[1] = 0;
      __threadfence();
    }
  }
}

}  // namespace tc3

template <int D, typename T>
static cudaError_t launch_tc3_t(const CUtensorMap& tmk, const CUtensorMap& tmv, const DevPlan& plan, int var,
                                int grid, const void* q, void* out, float* po, float* pl, float scale_log2,
                                int32_t* sched, cudaStream_t st) {
  constexpr int smem = tc3::Layout<D>::kAlloc;
  // the opt-in is per device; setting it is cheap and idempotent
  cudaError_t e = cudaFuncSetAttribute(tc3::fwd_tc3_kernel<D, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  tc3::fwd_tc3_kernel<D, T><<<grid, tc3::kThreads, smem, st>>>(tmk, tmv, plan, var, (const T*)q, (T*)out, po, pl,
                                                               scale_log2, sched);
  return cudaGetLastError();
}

#ifdef PAT_TC_TRACE
extern "C" int pat_debug_tc_trace(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, tc3::g_tc_trace, sizeof(tc3::g_tc_trace));
}
extern "C" int pat_debug_trace_cta(int cta) {
  static long long zero[4][8][tc3::kTraceSteps];
  cudaMemcpyToSymbol(tc3::g_tc_trace, zero, sizeof(zero));
  return (int)cudaMemcpyToSymbol(tc3::g_trace_cta, &cta, sizeof(int));
}
extern "C" int pat_debug_item_log(long long* host, int* n) {
  int e = (int)cudaMemcpyFromSymbol(n, tc3::g_item_n, sizeof(int));
  if (e) return e;
  e = (int)cudaMemcpyFromSymbol(host, tc3::g_item_log, sizeof(tc3::g_item_log));
  int zero = 0;
  cudaMemcpyToSymbol(tc3::g_item_n, &zero, sizeof(int));
  return e;
}
extern "C" int pat_debug_spans_tc(unsigned long long* host) {
  int e = (int)cudaMemcpyFromSymbol(host, tc3::g_span_tc, sizeof(tc3::g_span_tc));
  static unsigned long long zero[1][kSpanCtas][2];
  cudaMemcpyToSymbol(tc3::g_span_tc, zero, sizeof(zero));
  return e;
}
#endif

cudaError_t launch_forward_tc(const CUtensorMap& tmk, const CUtensorMap& tmv, const DevPlan& plan, int var, int grid,
                              int dtype, int d, const void* q, void* out, float* po, float* pl, float scale_log2,
                              int32_t* sched, cudaStream_t st) {
  if (dtype == PAT_DTYPE_F16) {
    if (d == 128) return launch_tc3_t<128, __half>(tmk, tmv, plan, var, grid, q, out, po, pl, scale_log2, sched, st);
    return launch_tc3_t<64, __half>(tmk, tmv, plan, var, grid, q, out, po, pl, scale_log2, sched, st);
  }
  if (d == 128)
    return launch_tc3_t<128, __nv_bfloat16>(tmk, tmv, plan, var, grid, q, out, po, pl, scale_log2, sched, st);
  return launch_tc3_t<64, __nv_bfloat16>(tmk, tmv, plan, var, grid, q, out, po, pl, scale_log2, sched, st);
}

}  // namespace pat
