// Tensor-core (tcgen05 + TMEM + TMA) forward kernel: two independent item
// pipelines ("lanes") per CTA.
//
// One persistent CTA per SM runs two lanes.  Each lane claims its own work items
// (unit x kv head x up to 128 rows) from the global counter in the scheduler's
// longest-first order and streams each item's KV span once through its own TMA
// ring, so one lane's item boundary (Q load, last PV, O read-out and stores)
// overlaps the other lane's tiles instead of stalling the SM:
//
//   warps 0 / 3  producer of lane 0 / 1: claims items, resolves per-row (query
//                id, partial slot) into a 2-slot item ring, warms L2 with the
//                item's Q rows, issues TMA boxes of 16-token page slices of K
//                and V (32-token stages, 128B swizzle) straight from the paged
//                vLLM cache;
//   warps 1 / 4  QK issuer of lane 0 / 1 (warp 1 also allocates TMEM):
//                  S[b] = Q K^T   (TS: Q from TMEM, K from smem, M=128 N=32)
//   warps 2 / 5  PV issuer of lane 0 / 1:
//                  O   += P[b] V  (TS: P from TMEM over S[b], V from smem)
//                S/P are double-buffered (b = tile & 1): QK(t) waits only for
//                PV(t-2), so it runs a tile ahead of the softmax;
//   warps 6-9    softmax / epilogue of lane 0, warps 10-13 of lane 1: one thread
//                per TMEM lane = one row of the item (query x GQA head), the
//                whole 32-column tile per thread, so a row's running max, sum
//                and O never leave its thread: no cross-warp fold, no CTA-wide
//                barrier anywhere in the steady state.
//
// TMEM (512 columns): lane L at 256 L: S/P[b] at +32 b (P = hi 16 + lo 16
// columns of packed 16-bit pairs written over the consumed S), Q at +64
// (packed pairs, the A operand of QK), O at +128.
// KV tiles are 32 tokens (16 KB stages, 6 per lane): a stage is released as
// soon as its PV completes, so more of the ring is in flight.  The ring is laid
// out as K and V planes ([64 d][6 stages x 32 tokens] x 128 B each), so two
// consecutive stages hold 64 contiguous token rows.
//
// Narrow items (<= 16 rows: the unshared suffixes of a batch) would leave 112
// of the 128 MMA rows idle.  They run transposed instead, on 64-token tiles
// (an even/odd stage pair; the producer aligns them):
//   S^T[b] = K Q^T     (SS: M = 128 token rows -- 64 live --, N = 16 rows, K = d)
//   O^T   += V^T P^T   (SS: M = d, N = 16 rows, K = tokens; P^T in smem)
// a thread per token for the softmax (per-row maxima shared through a
// barrier-reduction vote and, when a row's max grows, shared memory) and a
// thread per head-dim lane for the epilogue: ~6x fewer tensor cycles per token.
// Numerics follow cta_partial (attention.py:140-163): fp32 scores and
// accumulators, log2-domain online softmax with lazy O rescale (only when the
// running max grows by > 8), bf16 P = hi + lo (two PV MMAs), fp16 P single and
// normalised by the sum of the rounded weights the MMA used.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include "pat_plan.cuh"
#include "pat_sm100.cuh"

namespace pat {
namespace tc4 {

#ifdef PAT_TC_TRACE
// Debug timeline (tools/tc_trace.py, tools/item_log.py).
constexpr int kTraceSteps = 256;
__device__ long long g_tc_trace[4][8][kTraceSteps];
__device__ int g_trace_cta;
__device__ unsigned long long g_span_tc[1][kSpanCtas][2];
// per-item log (all CTAs, both lanes): cta*2+lane, item, rows, tiles, t_start, t_first_data, t_tiles_done, t_epi_done
constexpr int kItemLog = 32768;
__device__ long long g_item_log[kItemLog][12];  // + [8] Q stored, [9] last PV done, [10] O read
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
#define TC_TRACE(role, ev, step)                                                   \
  do {                                                                             \
    if (traced && (step) < kTraceSteps) g_tc_trace[role][ev][step] = clock64(); \
  } while (0)
#else
#define ITEM_T(var) \
  do {              \
  } while (0)
#define TC_TRACE(role, ev, step) \
  do {                           \
  } while (0)
#endif

#ifndef PAT_TRACE_LANE
#define PAT_TRACE_LANE 0  // item pipeline whose per-tile events tools/tc_trace.py records
#endif
constexpr int kThreads = 448;  // per lane: producer, QK issuer, PV issuer; 2 x 4 softmax warps
constexpr int kCtl = 6;        // control warps
constexpr int kM = 128;  // rows per item (TMEM lanes)
constexpr int kN = 32;   // tokens per KV tile
#ifndef PAT_TC4_STAGES
#define PAT_TC4_STAGES 6
#endif
constexpr int kStages = PAT_TC4_STAGES;  // per lane
constexpr uint32_t kTmemCols = 512;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
constexpr int kNarrow = 16;                // items of <= 16 rows run transposed (N = 16)
#ifndef PAT_TC4_NSTG
#define PAT_TC4_NSTG 2
#endif
constexpr int kNStg = PAT_TC4_NSTG;        // ring stages per narrow tile (1 or 2)
constexpr int kNN = kNStg * kN;            // tokens per narrow tile
static_assert((kNStg == 1 || kNStg == 2) && kStages % kNStg == 0, "narrow tiles are aligned stage groups");

struct ItemSlot {
  int32_t idx;
  int32_t pad[7];  // [0] joined pair item (tiles from lane 0's ring), [1] its first ring position
  Item item;
  int2 meta[kM];  // (qid, slot) per row
};
static_assert(sizeof(ItemSlot) == 64 + 8 * kM, "ItemSlot layout");
constexpr uint32_t kSlotBytes = sizeof(ItemSlot);
constexpr uint32_t kFIdx = 0, kFShared = 4, kFG0 = 8, kFKvh = 32 + 4, kFRow0 = 32 + 8, kFNrows = 32 + 12, kFNtok = 32 + 20, kFMeta = 64;

template <int D>
struct Layout {
  static constexpr int KB = D / 64;
  static constexpr int kPlane = kStages * kN * 128;  // one 64-d plane of K or V: [6 x 32 tokens][128 B]
  static constexpr int kLaneRing = 2 * KB * kPlane;  // K planes, then V planes
  static constexpr int kOffKV = 0;                   // lane L ring at L * kLaneRing
  static constexpr int kOffBar = 2 * kLaneRing;
  static constexpr int kOffRing = kOffBar + 1024;  // item slots [lane][2]
  // narrow items, per lane: Q rows [KB][16][128 B], P^T [2 buffers][hi, lo][16 rows][64 tokens x 2 B]
  static constexpr int kNarQ = KB * kNarrow * 128;
  static constexpr int kNarLane = kNarQ + 4 * kNarrow * 128;
  static constexpr int kOffNar = (kOffRing + 4 * (int)sizeof(ItemSlot) + 1023) / 1024 * 1024;
  static constexpr int kOffX = kOffNar + 2 * kNarLane;  // [lane][max, sum][2 warps][16] floats
  static constexpr int kBytes = kOffX + 2 * 2 * 2 * kNarrow * 4;
  static constexpr int kAlloc = kBytes + 1024;
  static_assert(kAlloc <= 227 * 1024, "shared memory budget");
  static_assert(kNarQ % 1024 == 0, "SW128 operands are 1024-byte aligned");
};

enum Bar : int {
  KV_FULL = 0,
  KV_EMPTY = KV_FULL + kStages,
  // Two S/P buffers per lane (TMEM columns 32b .. 32b + 31, b = tile & 1): the
  // softmax writes P(c) over the S(c) it has loaded (hi at +0, lo at +16), so
  // QK(c) waits only for PV(c-2) -- the last reader of its buffer -- and runs a
  // whole tile ahead of the softmax, which never waits for a PV before writing
  // P.  Every barrier of the chain is per buffer: an arrival for tile c + 2
  // needs PV(c), so no arrival can land in another tile's phase.
  S_FULL = KV_EMPTY + kStages,  // [b] QK(c) done
  P_FULL = S_FULL + 2,          // [b] softmax(c) wrote P (4 warps)
  P_FREE = P_FULL + 2,          // [b] PV(c) completed: O updated, buffer b free
  O_EMPTY = P_FREE + 2,         // epilogue has read O (one arrival after the lane's named barrier)
  QT_FULL = O_EMPTY + 1,        // the item's Q rows stored in TMEM (4 warps)
  ITEM_FULL = QT_FULL + 1,      // [slot] published by the producer (32 lanes)
  ITEM_EMPTY = ITEM_FULL + 2,   // [slot] released by the MMA warp and the 4 softmax warps
  XKV_EMPTY = ITEM_EMPTY + 2,   // [stage] lane 0 only: lane 1 released a pair tile of lane 0's ring
  JOIN_FULL = XKV_EMPTY + kStages,  // [2] lane 0 only: join mailbox entry posted
  JOIN_EMPTY = JOIN_FULL + 2,       // [2] lane 0 only: join mailbox entry read by lane 1
  BARS_PER_LANE = JOIN_EMPTY + 2
};
static_assert(2 * BARS_PER_LANE * 8 + 32 <= 1024, "barrier area");

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
  static __device__ __forceinline__ __half cvt(float a) { return __float2half_rn(a); }
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
  static __device__ __forceinline__ __nv_bfloat16 cvt(float a) { return __float2bfloat16_rn(a); }
};

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
// streaming store (evict-first): outputs and partials are read once, by the merge
__device__ __forceinline__ void st_cs_v4(uint4* p, uint4 v) {
  asm volatile("st.global.cs.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
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
#ifdef PAT_EXP_FAKE  // timing experiment only: no MUFU work (wrong results)
  return fmaf(v, 0.001f, 0.5f);
#else
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
#endif
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
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void sts_u16(uint32_t a, uint16_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"(v) : "memory");
}
__device__ __forceinline__ void sts_f32(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
// named barrier of n threads that ORs a predicate across them
__device__ __forceinline__ bool bar_red_or(uint32_t id, uint32_t n, bool v) {
  uint32_t r;
  asm volatile(
      "{\n .reg .pred p, q;\n setp.ne.u32 q, %3, 0;\n bar.red.or.pred p, %1, %2, q;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(r)
      : "r"(id), "r"(n), "r"((uint32_t)v)
      : "memory");
  return r != 0;
}
// Instruction descriptor, kind::f16, fp32 accumulate, with both operand majors.
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N, int ab_fmt, int a_mn_major, int b_mn_major) {
  return (1u << 4) | ((uint32_t)ab_fmt << 7) | ((uint32_t)ab_fmt << 10) | ((uint32_t)a_mn_major << 15) |
         ((uint32_t)b_mn_major << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ uint16_t bits16(uint32_t packed_lo) { return (uint16_t)(packed_lo & 0xffffu); }
// shared-memory descriptor of an MN-major operand, SWIZZLE_32B (layout type 6):
// 16-element (32 B) atoms along N `lbo` bytes apart, 8-row K groups 256 B apart (SBO)
__device__ __forceinline__ uint64_t desc_sw32(uint32_t saddr, uint32_t lbo = 256u) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;  // LBO: next 16 N-elements
  d |= (uint64_t)((256u >> 4) & 0x3FFF) << 32;  // SBO
  d |= (uint64_t)1 << 46;                        // descriptor version (sm_100)
  d |= (uint64_t)6 << 61;                        // SWIZZLE_32B
  return d;
}

__device__ __forceinline__ Item load_item(const Item* p) {
  const int4* q = reinterpret_cast<const int4*>(p);
  int4 a = __ldg(q), b = __ldg(q + 1);
  return Item{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
}

template <int D, typename T>
// 12 warps x 168 registers (no setmaxnreg: a 56-register control warpgroup
// spilled the MMA issuer's loop state to local memory)
__global__ void __launch_bounds__(kThreads, 1)
    fwd_tc4_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv, DevPlan plan,
                   int var, const T* __restrict__ qg, T* __restrict__ out, float* __restrict__ part_o,
                   float* __restrict__ part_lse, float scale_log2, int32_t* __restrict__ sched) {
  using L = Layout<D>;
  using namespace sm100;
  constexpr bool kSplit = Fmt<T>::kSplit;
  constexpr int KB = L::KB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sb = smem_u32(smem);
  uint32_t* tmem_slot = (uint32_t*)(smem + L::kOffBar + 2 * BARS_PER_LANE * 8);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
#ifdef PAT_TC_TRACE
  const bool traced = (int)blockIdx.x == g_trace_cta;
  if (tid == 0 && blockIdx.x < kSpanCtas) g_span_tc[0][blockIdx.x][0] = (unsigned long long)gtime();
#endif
  // lane (pipeline) of this warp: control warps 0-2 -> 0 and 3-5 -> 1 (role = warp % 3:
  // producer, QK issuer, PV issuer); softmax 6-9 -> 0, 10-13 -> 1
  const int pl = warp < kCtl ? warp / 3 : ((warp - kCtl) >> 2);
  const int role = warp < kCtl ? warp % 3 : 3;
  auto barL = [&](int l, int i) { return sb + L::kOffBar + (uint32_t)((l * BARS_PER_LANE + i) * 8); };
  auto bar = [&](int i) { return barL(pl, i); };
  // stage s of lane l's KV ring: K at sK(l, s) + kb * kPlane, V likewise
  auto sK = [&](int l, int s) { return sb + L::kOffKV + (uint32_t)(l * L::kLaneRing + s * kN * 128); };
  auto sV = [&](int l, int s) { return sK(l, s) + (uint32_t)(KB * L::kPlane); };
  // narrow items: Q rows (B of S^T = K Q^T), P^T (B of O^T = V^T P^T), row max / sum exchange
  const uint32_t sQn = sb + L::kOffNar + (uint32_t)(pl * L::kNarLane);
  auto sPn = [&](uint32_t b, int h) { return sQn + (uint32_t)(L::kNarQ + (int)(b * 2 + h) * kNarrow * 128); };
  const uint32_t xch = sb + L::kOffX + (uint32_t)(pl * 2 * 2 * kNarrow * 4);
  int2* join = reinterpret_cast<int2*>(smem + L::kOffBar + 2 * BARS_PER_LANE * 8 + 16);  // [2] mailbox
  const uint32_t ring_s = sb + L::kOffRing + (uint32_t)(pl * 2 * kSlotBytes);
  ItemSlot* ring = reinterpret_cast<ItemSlot*>(smem + L::kOffRing) + pl * 2;
  auto fld = [&](uint32_t n, uint32_t off) { return lds_s32(ring_s + (n & 1) * kSlotBytes + off); };

  const int H = plan.H, G = plan.G, bs = plan.bs;
  const int n_items = plan.n_items[var];
  const Item* items = plan.items[var];

  if (tid < 2) {
    const uint32_t b0 = sb + L::kOffBar + (uint32_t)(tid * BARS_PER_LANE * 8);
    auto ib = [&](int i) { return b0 + 8u * (uint32_t)i; };
    for (int s = 0; s < kStages; ++s) {
      mbar_init(ib(KV_FULL + s), 1);
      mbar_init(ib(KV_EMPTY + s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(ib(S_FULL + b), 1);
      mbar_init(ib(P_FULL + b), 4);
      mbar_init(ib(P_FREE + b), 1);
    }
    mbar_init(ib(O_EMPTY), 1);
    mbar_init(ib(QT_FULL), 4);
    for (int i = 0; i < 2; ++i) {
      mbar_init(ib(ITEM_FULL + i), 32);
      mbar_init(ib(ITEM_EMPTY + i), 2 + 4);
      mbar_init(ib(JOIN_FULL + i), 1);
      mbar_init(ib(JOIN_EMPTY + i), 1);
    }
    for (int s = 0; s < kStages; ++s) mbar_init(ib(XKV_EMPTY + s), 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(smem_u32(tmem_slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tg = tmem + (uint32_t)(pl * 256);  // this lane's TMEM columns
  // the merge kernel (a programmatic dependent) may be scheduled now: its CTAs
  // take SMs as this grid's CTAs exit and wait for the whole grid there
  asm volatile("griddepcontrol.launch_dependents;");

  if (warp < kCtl) {
    if (role == 0) {
      // ------------------------------------------------------------ producer
      if (elect_one()) {
        tma_prefetch(&tmk);
        tma_prefetch(&tmv);
      }
      // Phase 1 (pair items, > 128 rows): lane 0 claims them, posts each to the
      // CTA's join mailbox with the ring position of its first tile and
      // streams its tiles once; lane 1 takes rows 128.. of the same item and
      // reads lane 0's ring (each stage is released by both lanes).  A "done"
      // entry ends phase 1; then both lanes claim the other items
      // independently.
      const int n_pair = plan.n_pair[var];
      bool pair_phase = n_pair > 0, first_claim = true;
      uint32_t gt = 0, jn = 0, pair_upto = 0;
      for (uint32_t n = 0;; ++n) {
        const uint32_t slot = n & 1;
        mbar_wait(bar(ITEM_EMPTY + slot), ((n >> 1) & 1) ^ 1);
        int it = -1, shared = 0;
        uint32_t g0 = 0;
        if (pair_phase) {
          if (pl == 0) {
            int c = 0;
            if (lane == 0) c = atomicAdd(sched + 0, 1);
            c = __shfl_sync(0xffffffffu, c, 0);
            if (c < n_pair) it = c;
            else pair_phase = false;
            mbar_wait(barL(0, JOIN_EMPTY + (jn & 1)), ((jn >> 1) & 1) ^ 1);
            if (lane == 0) {
              join[jn & 1] = make_int2(it, (int)gt);
              mbar_arrive(barL(0, JOIN_FULL + (jn & 1)));
            }
            __syncwarp();
          } else {
            mbar_wait(barL(0, JOIN_FULL + (jn & 1)), (jn >> 1) & 1);
            const int2 e = lds_v2(smem_u32(&join[jn & 1]));
            __syncwarp();
            if (lane == 0) mbar_arrive(barL(0, JOIN_EMPTY + (jn & 1)));
            if (e.x >= 0) it = e.x, shared = 1, g0 = (uint32_t)e.y;
            else pair_phase = false;
          }
          ++jn;
        }
        if (!pair_phase) {
          // the first claim of every lane is static (lane L of CTA b takes the
          // (b + L * grid)-th item: no 296-way atomic at kernel start), later
          // ones come from the counter, offset by the 2 * grid static claims
          int c = 0;
          if (n_pair == 0 && first_claim) c = (int)blockIdx.x + pl * (int)gridDim.x;
          else if (lane == 0) c = atomicAdd(sched + 2, 1) + (n_pair == 0 ? 2 * (int)gridDim.x : 0);
          first_claim = false;
          it = n_pair + __shfl_sync(0xffffffffu, c, 0);
          if (it >= n_items) it = -1;
        }
        Item item{};
        if (it >= 0) {
          item = load_item(items + it);
          if (it < n_pair) {  // pair item: lane 0 rows [0, 128), lane 1 the rest
            if (pl == 0) item.nrows = kM;
            else item.row0 += kM, item.nrows -= kM;
          }
          for (int r = lane; r < item.nrows; r += 32) {
            const int qi = (item.row0 + r) / G;
            ring[slot].meta[r] =
                make_int2(__ldg(plan.pack_q + item.qoff + qi), __ldg(plan.unit_slot + item.slot_off + qi));
          }
          if (lane == 0) ring[slot].item = item;
          // warm L2 with the item's Q rows (the softmax warps load them into
          // TMEM at the previous item's end): one bulk prefetch per query
          const int i0 = item.row0 / G, i1 = (item.row0 + item.nrows - 1) / G;
          for (int i = i0 + lane; i <= i1; i += 32) {
            const int qid = __ldg(plan.pack_q + item.qoff + i);
            const int a = max(i * G, item.row0), e = min((i + 1) * G, item.row0 + item.nrows);
            bulk_prefetch_l2(qg + ((int64_t)qid * H + item.kvh * G + (a - i * G)) * D, (uint32_t)((e - a) * D * 2));
          }
        }
        // first ring position of the item: narrow items start on an even stage
        // (their 64-token tiles are stage pairs); the odd one is skipped
        const bool narrow = it >= 0 && !shared && item.nrows <= kNarrow;
        if (!shared) g0 = narrow ? ((gt + kNStg - 1) & ~(uint32_t)(kNStg - 1)) : gt;
        if (lane == 0) {
          ring[slot].idx = it;
          ring[slot].pad[0] = shared;
          ring[slot].pad[1] = (int)g0;
        }
        __syncwarp();
        mbar_arrive(bar(ITEM_FULL + slot));
        if (it < 0) break;
        if (shared) continue;  // the tiles come through lane 0's ring
        if (g0 != gt) {  // skipped stage: an empty phase (no bytes), released by the MMA warp
          const int s = gt % kStages;
          mbar_wait(bar(KV_EMPTY + s), ((gt / kStages) & 1) ^ 1);
          if (gt >= (uint32_t)kStages && gt - kStages < pair_upto)
            mbar_wait(bar(XKV_EMPTY + s), ((gt / kStages) & 1) ^ 1);
          if (elect_one()) mbar_arrive(bar(KV_FULL + s));
          __syncwarp();
          ++gt;
        }
        const int h = item.kvh, ntok = item.ntok;
        const int32_t* blist = plan.pack_blk + item.blk;
        const int ntiles = (ntok + kN - 1) / kN;
        if (it < n_pair) pair_upto = gt + (uint32_t)ntiles;
        for (int j = 0; j < ntiles; ++j, ++gt) {
          const int s = gt % kStages;
          const int rem = ntok - j * kN;
          const int ngrp = rem >= kN ? kN / 16 : (rem + 15) / 16;  // 16-token page slices
          int my_blk = 0, my_off = 0;
          if (lane < ngrp) {
            const int tok = j * kN + lane * 16;
            const int pg = bs == 16 ? (tok >> 4) : tok / bs;
            my_blk = __ldg(blist + pg);
            my_off = bs == 16 ? 0 : tok - pg * bs;
          }
          mbar_wait(bar(KV_EMPTY + s), ((gt / kStages) & 1) ^ 1);
          // the previous occupant of this stage was a pair tile: lane 1 read it
          // too (pair tiles are a prefix of lane 0's ring, so every earlier use
          // of the stage was one: same parity as KV_EMPTY)
          if (gt >= (uint32_t)kStages && gt - kStages < pair_upto)
            mbar_wait(bar(XKV_EMPTY + s), ((gt / kStages) & 1) ^ 1);
          if (pl == PAT_TRACE_LANE) TC_TRACE(0, 0, gt);
          if (elect_one()) mbar_expect_tx(bar(KV_FULL + s), (uint32_t)(ngrp * KB * 2048 * 2));
          __syncwarp();
          for (int gr = 0; gr < ngrp; ++gr) {
            const int blk = __shfl_sync(0xffffffffu, my_blk, gr);
            const int off = __shfl_sync(0xffffffffu, my_off, gr);
            if (elect_one()) {
#pragma unroll
              for (int kb = 0; kb < KB; ++kb) {
                tma_load_4d(sK(pl, s) + kb * L::kPlane + gr * 2048, &tmk, bar(KV_FULL + s), kb * 64, h, off, blk);
                tma_load_4d(sV(pl, s) + kb * L::kPlane + gr * 2048, &tmv, bar(KV_FULL + s), kb * 64, h, off, blk);
              }
            }
            __syncwarp();
          }
        }
      }
    } else {
      // ------------------------------------------------------------ MMA issuers
      // Two warps per lane: one issues the QK products, the other the PV
      // products.  A single thread's tcgen05.mma stream completes one M = 128
      // instruction per ~65 cycles whatever N (tools/tmem_bench.cu), so one
      // issuer per lane capped a 32-token tile at 12 x 65 cycles; with QK and
      // PV on separate issuers they overlap and the tensor pipe approaches its
      // floor.  QK(c) needs its KV stage(s) and PV(c-2) done (it overwrites
      // S/P[c & 1]); PV(c) needs the softmax's P(c) and releases the stage(s).
      // The stage of ring position g is g % kStages of the lane's own ring, or
      // of lane 0's ring for a joined pair item.
      constexpr uint32_t idesc_qk = umma_idesc_f16(kM, kN, Fmt<T>::ab, 0);
      constexpr uint32_t idesc_pv = umma_idesc_f16(kM, D, Fmt<T>::ab, 1);
      constexpr uint32_t idesc_qkn = idesc_f16(kM, kNarrow, Fmt<T>::ab, 0, 0);  // S^T = K Q^T
      // O^T = V^T P^T; for bf16 the hi and lo P^T tiles (2 KB apart) are the two
      // 16-column halves of ONE N = 32 operand: V^T is read once per k-step and
      // O^T = [V^T P_hi^T | V^T P_lo^T] is summed in the epilogue
      constexpr int kNO = kSplit ? 2 * kNarrow : kNarrow;
      constexpr uint32_t idesc_pvn = idesc_f16(kM, kNO, Fmt<T>::ab, 1, 1);
      const bool is_qk = role == 1;
      uint32_t tcnt = 0, rpos = 0, qu = 0, ou = 0;
      for (uint32_t n = 0;; ++n) {
        mbar_wait(bar(ITEM_FULL + (n & 1)), (n >> 1) & 1);
        const int it = fld(n, kFIdx);
        const int ntok = it >= 0 ? fld(n, kFNtok) : 0;
        const bool narrow = it >= 0 && !fld(n, kFShared) && fld(n, kFNrows) <= kNarrow;
        const int src = it >= 0 && fld(n, kFShared) ? 0 : pl;  // ring the tiles come from
        const uint32_t base = it >= 0 ? (uint32_t)fld(n, kFG0) : 0u;
        __syncwarp();
        if (lane == 0) mbar_arrive(bar(ITEM_EMPTY + (n & 1)));
        if (it < 0) break;
        const int ntiles = narrow ? (ntok + kNN - 1) / kNN : (ntok + kN - 1) / kN;
        if (is_qk) {
          for (int t = 0; t < ntiles; ++t) {
            const uint32_t c = tcnt + (uint32_t)t;
            const uint32_t g = narrow ? base + (uint32_t)(kNStg * t) : base + (uint32_t)t;
            const int s = (int)(g % kStages);
            if (pl == PAT_TRACE_LANE) TC_TRACE(1, 2, c);
            mbar_wait(barL(src, KV_FULL + s), (g / kStages) & 1);
            if (kNStg == 2 && narrow && ntok - t * kNN > kN)
              mbar_wait(barL(src, KV_FULL + s + 1), ((g + 1) / kStages) & 1);
            if (pl == PAT_TRACE_LANE) TC_TRACE(1, 3, c);
            // buffer c & 1 was last read by PV(c - 2)
            mbar_wait(bar(P_FREE + (c & 1)), ((c >> 1) & 1) ^ 1);
            if (t == 0) mbar_wait(bar(QT_FULL), qu++ & 1);
            const uint32_t sbuf = tg + 32u * (c & 1);
            tc_fence_after();
            if (pl == PAT_TRACE_LANE) TC_TRACE(1, 0, c);
            if (elect_one()) {
              if (narrow) {
#pragma unroll
                for (int k = 0; k < D / 16; ++k) {
                  const int kb = k >> 2, kk = k & 3;
                  const uint64_t ad = umma_desc_sw128(sK(src, s) + (uint32_t)(kb * L::kPlane + kk * 32), 16, 1024);
                  const uint64_t bd = umma_desc_sw128(sQn + (uint32_t)(kb * kNarrow * 128 + kk * 32), 16, 1024);
                  umma_f16_ss(sbuf, ad, bd, idesc_qkn, k > 0 ? 1u : 0u);
                }
              } else {
                const uint64_t k0 = umma_desc_sw128(sK(src, s), 16, 1024);
#pragma unroll
                for (int k = 0; k < D / 16; ++k) {
                  const int kb = k >> 2, kk = k & 3;
                  // Q(m, k) packed two per column: a k-step of 16 = 8 columns
                  umma_f16_ts(sbuf, tg + 64u + (uint32_t)(k * 8),
                              k0 + (uint64_t)((kb * L::kPlane + kk * 32) >> 4), idesc_qk, k > 0 ? 1u : 0u);
                }
              }
              umma_commit(bar(S_FULL + (c & 1)));
            }
            __syncwarp();
          }
        } else {
          if (src == pl && base != rpos) {  // a stage the producer skipped to align a narrow item
            const int s = (int)(rpos % kStages);
            mbar_wait(bar(KV_FULL + s), (rpos / kStages) & 1);
            if (elect_one()) mbar_arrive(bar(KV_EMPTY + s));
            __syncwarp();
            rpos = base;
          }
          for (int t = 0; t < ntiles; ++t) {
            const uint32_t c = tcnt + (uint32_t)t, b = c & 1;
            const uint32_t g = narrow ? base + (uint32_t)(kNStg * t) : base + (uint32_t)t;
            const int s = (int)(g % kStages);
            if (pl == PAT_TRACE_LANE) TC_TRACE(1, 4, c);
            mbar_wait(bar(P_FULL + b), (c >> 1) & 1);
            if (t == 0) mbar_wait(bar(O_EMPTY), (ou & 1) ^ 1);
            tc_fence_after();
            if (elect_one()) {
              const uint32_t rel = src != pl ? barL(0, XKV_EMPTY + s) : bar(KV_EMPTY + s);
              if (narrow) {
                const int vt = min(kNN, ntok - t * kNN);
                const int nk = (vt + 15) / 16;
                for (int j = 0; j < nk; ++j) {
                  const uint64_t ad = umma_desc_sw128(sV(src, s) + (uint32_t)(j * 16 * 128), L::kPlane, 1024);
                  umma_f16_ss(tg + 128u, ad, desc_sw32(sPn(b, 0) + (uint32_t)(j * 512), kNarrow * 128), idesc_pvn,
                              (t == 0 && j == 0) ? 0u : 1u);
                }
                umma_commit(bar(P_FREE + b));
                umma_commit(rel);
                if (vt > kN) umma_commit(bar(KV_EMPTY + s + 1));
              } else {
                const uint64_t v0 = umma_desc_sw128(sV(src, s), L::kPlane, 1024);
#pragma unroll
                for (int k = 0; k < kN / 16; ++k) {
                  const uint64_t bd = v0 + (uint64_t)((k * 16 * 128) >> 4);
                  // P(m, k) is packed two per column: a k-step of 16 tokens = 8 columns
                  umma_f16_ts(tg + 128u, tg + 32u * b + (uint32_t)(k * 8), bd, idesc_pv, (t == 0 && k == 0) ? 0u : 1u);
                  if constexpr (kSplit)
                    umma_f16_ts(tg + 128u, tg + 32u * b + 16u + (uint32_t)(k * 8), bd, idesc_pv, 1u);
                }
                umma_commit(bar(P_FREE + b));
                umma_commit(rel);
              }
            }
            __syncwarp();
            if (pl == PAT_TRACE_LANE) TC_TRACE(1, 1, c);
          }
          ++ou;
          if (src == pl) rpos = base + (uint32_t)((ntok + kN - 1) / kN);
        }
        tcnt += (uint32_t)ntiles;
      }
      (void)qu;
    }
  } else {
    // ------------------------------------------------------------ softmax / epilogue
    const int wq = warp & 3;          // TMEM lane quarter
    const int ln = wq * 32 + lane;    // TMEM lane: row of a regular item, token of a narrow tile
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    const uint32_t sp = tg + lane_base;
    const uint32_t nbar = 1 + (uint32_t)pl;  // named barrier of the lane's 128 softmax threads
    constexpr int CPT = D / 64;              // 16-byte chunks of a narrow item's Q tile per thread
#ifdef PAT_TC_TRACE
    const bool tr = (wq == 0 && lane == 0);
#endif
    uint32_t tcnt = 0;  // tiles consumed by this lane (S/P phases)

    auto wait_item = [&](uint32_t n) { mbar_wait(bar(ITEM_FULL + (n & 1)), (n >> 1) & 1); };
    auto q_row = [&](uint32_t n, int r) {
      const int qid = fld(n, kFMeta + 8 * r);
      const int head = fld(n, kFKvh) * G + (fld(n, kFRow0) + r) % G;
      return reinterpret_cast<const uint4*>(qg + ((int64_t)qid * H + head) * D);
    };
    // narrow (transposed) items: <= 16 rows, tiles from the lane's own ring
    auto is_narrow = [&](uint32_t n) { return fld(n, kFNrows) <= kNarrow && !fld(n, kFShared); };
    // Q of item n (zeros past its rows) into TMEM -- a regular item's row `ln`,
    // the A operand of QK, 32 columns at a time -- or into shared memory -- CPT
    // 16-byte chunks of a narrow item's 16-row tile, the 128B-swizzled K-major
    // B operand of S^T = K Q^T
    // a narrow item's Q chunks of this thread (CPT x 16 B), loaded ahead of the
    // store: at the start of the previous item's last tile (8 registers)
    auto load_qn = [&](uint32_t n, uint4* qn) {
      const int r = ln >> 3;
      const uint4* src = r < fld(n, kFNrows) ? q_row(n, r) : nullptr;
#pragma unroll
      for (int i = 0; i < CPT; ++i) qn[i] = src ? __ldg(src + (ln & 7) * CPT + i) : make_uint4(0, 0, 0, 0);
    };
    auto store_qn = [&](const uint4* qn) {
      const int r = ln >> 3;
#pragma unroll
      for (int i = 0; i < CPT; ++i) {
        const int ch = (ln & 7) * CPT + i, kb = ch >> 3, cc = ch & 7;
        st_shared_v4(sQn + (uint32_t)(kb * kNarrow * 128 + r * 128 + ((cc ^ (r & 7)) << 4)), qn[i]);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(QT_FULL));
    };
    auto put_q = [&](uint32_t n) {
      const int nr = fld(n, kFNrows);
      if (is_narrow(n)) {
        uint4 qn[CPT];
        load_qn(n, qn);
        store_qn(qn);
        return;
      } else if (wq * 32 < nr) {
        const uint4* src = ln < nr ? q_row(n, ln) : nullptr;
#pragma unroll
        for (int i = 0; i < D / 64; ++i) {
          uint32_t qv[32];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint4 v = src ? __ldg(src + 8 * i + j) : make_uint4(0, 0, 0, 0);
            qv[4 * j] = v.x, qv[4 * j + 1] = v.y, qv[4 * j + 2] = v.z, qv[4 * j + 3] = v.w;
          }
          tmem_st32_nowait(sp + 64u + 32u * i, qv);
        }
        tmem_wait_st();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(QT_FULL));
    };
    // tail of an item's span inside stage(s) from ring position g0 on: zero V rows
    // [vt, vt rounded up to the stage) (stale / uninitialised smem; P == 0 there
    // must not meet a NaN)
    auto zero_v_tail = [&](int src, int s0, int vt) {
      const int nz = (((vt + kN - 1) / kN) * kN - vt) * KB * 8;
      for (int q = ln; q < nz; q += kM) {
        const int rr = vt + q / (KB * 8);
        const int kb = (q / 8) % KB, ch = q % 8;
        st_shared_v4(sV(src, s0) + (uint32_t)(kb * L::kPlane + rr * 128 + (ch << 4)), make_uint4(0, 0, 0, 0));
      }
      fence_proxy_async_smem();
    };

    wait_item(0);
    if (fld(0, kFIdx) >= 0) put_q(0);
    for (uint32_t n = 0;; ++n) {
      if (fld(n, kFIdx) < 0) break;  // ITEM_FULL(n) already waited
      const int ntok = fld(n, kFNtok);
      const int nrows = fld(n, kFNrows);
      const int src = fld(n, kFShared) ? 0 : pl;  // ring the item's tiles come from
      const uint32_t base = (uint32_t)fld(n, kFG0);
      const int kvh = fld(n, kFKvh), row0 = fld(n, kFRow0);
      const bool narrow = is_narrow(n);
      const int ntiles = narrow ? (ntok + kNN - 1) / kNN : (ntok + kN - 1) / kN;
      const uint32_t meta_s = ring_s + (n & 1) * kSlotBytes + kFMeta;
      bool have_next = false;
      long long it0 = 0, it1 = 0, it2 = 0, it3 = 0, it4 = 0, it5 = 0, it6 = 0;
      (void)it0, (void)it1, (void)it2, (void)it3, (void)it4, (void)it5, (void)it6;
#ifdef PAT_TC_TRACE
      if (tr) ITEM_T(it0);
#endif
      // next item: known at the start of this item's last tile; its Q rows
      // (L2-warm: the producer prefetched them at claim time) are loaded once
      // this item's last S is consumed.  (Holding them in registers across the
      // tile cost 64 registers; an L1 prefetch stalled the softmax warps: c4
      // 201 -> 197 us without it.)
      auto prefetch_next_q = [&]() {
        wait_item(n + 1);
        have_next = fld(n + 1, kFIdx) >= 0;

      };

      if (!narrow) {
        // ================================================= regular item: thread = row
        const bool wlive = wq * 32 < nrows;  // warp has live rows (warp-uniform)
        float m_ref = -INFINITY;             // running max, log2 units
        float2 l2 = make_float2(0.f, 0.f);
        for (int t = 0; t < ntiles; ++t) {
          const uint32_t c = tcnt + (uint32_t)t;
          const uint32_t sb_c = sp + 32u * (c & 1);  // this tile's S/P buffer
          if (t == ntiles - 1) prefetch_next_q();
          mbar_wait(bar(S_FULL + (c & 1)), (c >> 1) & 1);
#ifdef PAT_TC_TRACE
          if (tr && t == 0) ITEM_T(it1);
          if (tr && pl == PAT_TRACE_LANE) TC_TRACE(2, 0, c);
#endif
          tc_fence_after();
          if (wlive) {
            uint32_t sr[kN];
            tmem_ld32(sb_c, sr);
            const int valid = ntok - t * kN;
            if (valid < kN) {
#pragma unroll
              for (int k = 0; k < kN; ++k)
                if (k >= valid) sr[k] = __float_as_uint(-INFINITY);
            }
            float pm[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
            for (int k = 0; k < kN / 8; ++k)
              pm[k & 3] = fmax3(pm[k & 3],
                                fmax3(__uint_as_float(sr[8 * k]), __uint_as_float(sr[8 * k + 1]),
                                      __uint_as_float(sr[8 * k + 2])),
                                fmax3(__uint_as_float(sr[8 * k + 3]), __uint_as_float(sr[8 * k + 4]),
                                      fmax3(__uint_as_float(sr[8 * k + 5]), __uint_as_float(sr[8 * k + 6]),
                                            __uint_as_float(sr[8 * k + 7]))));
            const float mx = fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])) * scale_log2;
            const bool need = mx > m_ref + kRescaleThreshold;
            if (__any_sync(0xffffffffu, need)) {
              const float m_new = need ? mx : m_ref;
              const float alpha = m_new == -INFINITY ? 1.f : ex2_approx(m_ref - m_new);
              if (t > 0) {
                // O must hold the previous tile's PV before it is rescaled
                mbar_wait(bar(P_FREE + ((c - 1) & 1)), ((c - 1) >> 1) & 1);
                tc_fence_after();
#pragma unroll 1
                for (int q = 0; q < D / 16; ++q) {
                  uint32_t o[16];
                  const uint32_t ta = sp + 128u + (uint32_t)(q * 16);
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
            // P = exp2(s * scale - m_ref), packed pairs (a row with no valid
            // column so far keeps m_ref = -inf: reference 0, P = 0)
            const float mu = m_ref == -INFINITY ? 0.f : m_ref;
            const float2 sc2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-mu, -mu);
            uint32_t ph[kN / 2], plo[kN / 2];
#pragma unroll
            for (int k = 0; k < kN / 2; ++k) {
              float2 a =
                  __ffma2_rn(make_float2(__uint_as_float(sr[2 * k]), __uint_as_float(sr[2 * k + 1])), sc2, nm2);
              a.x = ex2_approx(a.x);
              a.y = ex2_approx(a.y);
              ph[k] = Fmt<T>::pack(a.x, a.y);
              if constexpr (kSplit) {
                const float2 hf = Fmt<T>::unpack(ph[k]);
                const float2 lo = __fadd2_rn(a, make_float2(-hf.x, -hf.y));
                plo[k] = Fmt<T>::pack(lo.x, lo.y);
                l2 = __fadd2_rn(l2, a);
              } else {
                // normalise by the sum of the ROUNDED weights the MMA actually uses
                l2 = __fadd2_rn(l2, Fmt<T>::unpack(ph[k]));
              }
            }
            // P over this tile's S (already in registers: tmem_ld32 waited)
            tmem_st_n<kN / 2>(sb_c, ph);
            if constexpr (kSplit) tmem_st_n<kN / 2>(sb_c + 16u, plo);
          }
          if (t * kN + kN > ntok) zero_v_tail(src, (int)((base + (uint32_t)t) % kStages), ntok - t * kN);
          if (wlive) tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(bar(P_FULL + (c & 1)));
#ifdef PAT_TC_TRACE
          if (tr && pl == PAT_TRACE_LANE) TC_TRACE(2, 1, c);
#endif
        }
#ifdef PAT_TC_TRACE
        if (tr) ITEM_T(it2);
#endif
        // The item's last QK completed (its S was consumed above): the next
        // item's Q goes in now, so its first QK overlaps this epilogue.
        if (have_next) put_q(n + 1);
#ifdef PAT_TC_TRACE
        if (tr) ITEM_T(it4);
#endif

        // ---- epilogue: the last PV of the item done -> O / l of this row
        const uint32_t gl = tcnt + (uint32_t)ntiles - 1;
        mbar_wait(bar(P_FREE + (gl & 1)), (gl >> 1) & 1);
#ifdef PAT_TC_TRACE
        if (tr) ITEM_T(it5);
#endif
        tc_fence_after();
        const bool live = ln < nrows;
        const float l = l2.x + l2.y;
        const int2 meta = live ? lds_v2(meta_s + 8 * ln) : make_int2(0, -1);
        const int head = kvh * G + (live ? (row0 + ln) % G : 0);
        if (wlive) {
          // (staging O through shared memory for coalesced 128-byte row writes
          // measured slower: c4 epilogue 5.3 -> 8.3 us per 128-row item)
          const float inv = 1.f / l;
#pragma unroll 1
          for (int q = 0; q < D / 32; ++q) {
            uint32_t o[32];
            tmem_ld32(sp + 128u + (uint32_t)(q * 32), o);
            if (live) {
              const float* f = reinterpret_cast<const float*>(o);
              if (meta.y < 0) {
                uint4* dst = reinterpret_cast<uint4*>(out + ((int64_t)meta.x * H + head) * D + q * 32);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  st_cs_v4(dst + k, make_uint4(Fmt<T>::pack(f[8 * k] * inv, f[8 * k + 1] * inv),
                                               Fmt<T>::pack(f[8 * k + 2] * inv, f[8 * k + 3] * inv),
                                               Fmt<T>::pack(f[8 * k + 4] * inv, f[8 * k + 5] * inv),
                                               Fmt<T>::pack(f[8 * k + 6] * inv, f[8 * k + 7] * inv)));
              } else {
                float4* dst = reinterpret_cast<float4*>(part_o + ((int64_t)meta.y * H + head) * D + q * 32);
#pragma unroll
                for (int k = 0; k < 8; ++k)
                  st_cs_v4(reinterpret_cast<uint4*>(dst + k),
                           make_uint4(__float_as_uint(f[4 * k] * inv), __float_as_uint(f[4 * k + 1] * inv),
                                      __float_as_uint(f[4 * k + 2] * inv), __float_as_uint(f[4 * k + 3] * inv)));
              }
            }
          }
          if (live && meta.y >= 0) part_lse[(int64_t)meta.y * H + head] = m_ref + log2f(l);
        }
        // O read by the lane's four warps: the next item's first PV may overwrite it
        tc_fence_before();
        named_bar_sync(nbar, 128);
        if (wq == 0 && lane == 0) mbar_arrive(bar(O_EMPTY));
      } else {
        // ================================================= narrow item: thread = token
        // S^T tile: lanes 0-63 = the tile's tokens (warps 0, 1), columns = the 16 rows
        float m_ref[kNarrow], lsum[kNarrow];
#pragma unroll
        for (int r = 0; r < kNarrow; ++r) m_ref[r] = -INFINITY, lsum[r] = 0.f;
        const bool tw = wq < 2;  // warp holds tokens
        // the next narrow item's Q chunks, loaded at the start of the last tile
        // and stored once its S^T is consumed (8 registers)
        uint4 qn[CPT];
        bool qn_pre = false;
        for (int t = 0; t < ntiles; ++t) {
          const uint32_t c = tcnt + (uint32_t)t, b = c & 1;
          const int s0 = (int)((base + (uint32_t)(kNStg * t)) % kStages);
          const int vt = min(kNN, ntok - t * kNN);  // valid tokens of the tile
          if (t == ntiles - 1) {
            prefetch_next_q();
            qn_pre = have_next && is_narrow(n + 1);
            if (qn_pre) load_qn(n + 1, qn);
          }
          mbar_wait(bar(S_FULL + b), (c >> 1) & 1);
#ifdef PAT_TC_TRACE
          if (tr && t == 0) ITEM_T(it1);
          if (tr && pl == PAT_TRACE_LANE) TC_TRACE(2, 0, c);
#endif
          tc_fence_after();
          float x[kNarrow];
          bool need = false;
          if (tw) {
            uint32_t sr[kNarrow];
            tmem_ld16(sp + 32u * b, sr);
            const bool tv = ln < vt;
#pragma unroll
            for (int r = 0; r < kNarrow; ++r) {
              x[r] = tv && r < nrows ? __uint_as_float(sr[r]) * scale_log2 : -INFINITY;
              need |= x[r] > m_ref[r] + kRescaleThreshold;
            }
          }
          if (bar_red_or(nbar, 128, need)) {
            // a row's max grew (always on the first tile): exact tile maxima
            // through shared memory, O^T / sums rescaled
            if (tw) {
#pragma unroll
              for (int r = 0; r < kNarrow; ++r) {
                float v = x[r];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
                if (lane == 0) sts_f32(xch + (uint32_t)((wq * kNarrow + r) * 4), v);
              }
            }
            named_bar_sync(nbar, 128);
            float alpha[kNarrow];
#pragma unroll
            for (int r = 0; r < kNarrow; ++r) {
              const float tm = fmaxf(lds_f32(xch + (uint32_t)(r * 4)), lds_f32(xch + (uint32_t)((kNarrow + r) * 4)));
              const float mn = fmaxf(m_ref[r], tm);
              alpha[r] = mn == -INFINITY ? 1.f : ex2_approx(m_ref[r] - mn);
              lsum[r] *= alpha[r];
              m_ref[r] = mn;
            }
            if (t > 0) {
              // O^T must hold the previous tile's PV before it is rescaled
              mbar_wait(bar(P_FREE + (b ^ 1u)), ((c - 1) >> 1) & 1);
              tc_fence_after();
#pragma unroll 1
              for (int h = 0; h < (kSplit ? 2 : 1); ++h) {  // the hi and lo halves of O^T
                uint32_t o[kNarrow];
                tmem_ld16(sp + 128u + (uint32_t)(h * kNarrow), o);
#pragma unroll
                for (int r = 0; r < kNarrow; ++r) o[r] = __float_as_uint(__uint_as_float(o[r]) * alpha[r]);
                tmem_st16_wait(sp + 128u + (uint32_t)(h * kNarrow), o);
              }
            }
            named_bar_sync(nbar, 128);  // exchange slots read before they are reused
          }
          if (tw) {
            // P^T into the MN-major 32B-swizzled B operand ([64 tokens][16 rows] x 2 B):
            // this thread's token row is 32 contiguous bytes, two 16-byte stores
            // (hi, and lo for bf16) instead of 16 scattered 2-byte ones
            uint32_t ph[kNarrow / 2], pq[kNarrow / 2];
#pragma unroll
            for (int r = 0; r < kNarrow; r += 2) {
              const float mu0 = m_ref[r] == -INFINITY ? 0.f : m_ref[r];
              const float mu1 = m_ref[r + 1] == -INFINITY ? 0.f : m_ref[r + 1];
              const float p0 = ex2_approx(x[r] - mu0), p1 = ex2_approx(x[r + 1] - mu1);
              ph[r / 2] = Fmt<T>::pack(p0, p1);
              const float2 hv = Fmt<T>::unpack(ph[r / 2]);
              if constexpr (kSplit) {
                pq[r / 2] = Fmt<T>::pack(p0 - hv.x, p1 - hv.y);
                lsum[r] += p0;
                lsum[r + 1] += p1;
              } else {
                lsum[r] += hv.x;
                lsum[r + 1] += hv.y;
              }
            }
            // P^T buffer b: its last reader PV(c - 2) completed before QK(c) was issued
            const uint32_t sw = (uint32_t)((ln >> 2) & 1);  // 32B swizzle: 16-byte chunk ^= bit 7 of the address
            const uint32_t a0 = (uint32_t)(ln * 32) + (sw << 4), a1 = (uint32_t)(ln * 32) + ((sw ^ 1u) << 4);
            st_shared_v4(sPn(b, 0) + a0, make_uint4(ph[0], ph[1], ph[2], ph[3]));
            st_shared_v4(sPn(b, 0) + a1, make_uint4(ph[4], ph[5], ph[6], ph[7]));
            if constexpr (kSplit) {
              st_shared_v4(sPn(b, 1) + a0, make_uint4(pq[0], pq[1], pq[2], pq[3]));
              st_shared_v4(sPn(b, 1) + a1, make_uint4(pq[4], pq[5], pq[6], pq[7]));
            }
          }
          if (vt < kNN && (vt % kN) != 0) zero_v_tail(pl, s0, vt);
          fence_proxy_async_smem();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(bar(P_FULL + b));
#ifdef PAT_TC_TRACE
          if (tr && pl == PAT_TRACE_LANE) TC_TRACE(2, 1, c);
#endif
        }
#ifdef PAT_TC_TRACE
        if (tr) ITEM_T(it2);
#endif
        if (qn_pre) store_qn(qn);
        else if (have_next) put_q(n + 1);
#ifdef PAT_TC_TRACE
        if (tr) ITEM_T(it4);
#endif

        // ---- epilogue: row sums over the 64 token threads, then thread = head-dim lane
        const uint32_t gl = tcnt + (uint32_t)ntiles - 1;
        if (tw) {
#pragma unroll
          for (int r = 0; r < kNarrow; ++r) {
            if (r >= nrows) break;
            float v = lsum[r];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) sts_f32(xch + (uint32_t)((2 * kNarrow + wq * kNarrow + r) * 4), v);
          }
        }
        mbar_wait(bar(P_FREE + (gl & 1)), (gl >> 1) & 1);
#ifdef PAT_TC_TRACE
        if (tr) ITEM_T(it5);
#endif
        tc_fence_after();
        uint32_t o[kNarrow];
        tmem_ld16(sp + 128u, o);
        if constexpr (kSplit) {
          uint32_t o2[kNarrow];
          tmem_ld16(sp + 128u + kNarrow, o2);
#pragma unroll
          for (int r = 0; r < kNarrow; ++r) o[r] = __float_as_uint(__uint_as_float(o[r]) + __uint_as_float(o2[r]));
        }
        tc_fence_before();
        named_bar_sync(nbar, 128);  // sums published, O^T read by all four warps
#ifdef PAT_TC_TRACE
        if (tr) ITEM_T(it6);
#endif
        if (wq == 0 && lane == 0) mbar_arrive(bar(O_EMPTY));
        // per-row scalars in parallel (thread = row): 1 / sum into the (now free)
        // maxima slots, the partial's log-sum-exp straight to global memory
        if (ln < nrows) {
          const float Ls = lds_f32(xch + (uint32_t)((2 * kNarrow + ln) * 4)) +
                           lds_f32(xch + (uint32_t)((3 * kNarrow + ln) * 4));
          sts_f32(xch + (uint32_t)(ln * 4), __frcp_rn(Ls));
          const int2 meta = lds_v2(meta_s + 8 * ln);
          if (meta.y >= 0) {
            float mr = m_ref[0];  // m_ref[ln] without dynamic register indexing
#pragma unroll
            for (int r = 1; r < kNarrow; ++r) mr = ln == r ? m_ref[r] : mr;
            part_lse[(int64_t)meta.y * H + kvh * G + (row0 + ln) % G] = mr + log2f(Ls);
          }
        }
        named_bar_sync(nbar, 128);
        if (ln < D) {
          // then thread = head-dim lane: every row's scalars loaded up front, one
          // coalesced row store each
          float inv[kNarrow];
          int2 mt[kNarrow];
#pragma unroll
          for (int r = 0; r < kNarrow; ++r) {
            inv[r] = lds_f32(xch + (uint32_t)(r * 4));
            mt[r] = lds_v2(meta_s + 8 * r);
          }
          int gh = row0 % G;  // GQA head of row r within the kv head's group
#pragma unroll
          for (int r = 0; r < kNarrow; ++r) {
            if (r >= nrows) break;
            const int head = kvh * G + gh;
            gh = gh + 1 == G ? 0 : gh + 1;
            const float v = __uint_as_float(o[r]) * inv[r];
            if (mt[r].y < 0)
              out[((int64_t)mt[r].x * H + head) * D + ln] = Fmt<T>::cvt(v);
            else
              part_o[((int64_t)mt[r].y * H + head) * D + ln] = v;
          }
        }
      }
#ifdef PAT_TC_TRACE
      if (tr) {
        ITEM_T(it3);
        const int k = atomicAdd(&g_item_n, 1);
        if (k < kItemLog) {
          long long* e = g_item_log[k];
          e[0] = blockIdx.x * 2 + pl, e[1] = fld(n, kFIdx), e[2] = nrows, e[3] = ntiles;
          e[4] = it0, e[5] = it1, e[6] = it2, e[7] = it3, e[8] = it4, e[9] = it5, e[10] = it6;
        }
      }
#endif
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(ITEM_EMPTY + (n & 1)));
      tcnt += (uint32_t)ntiles;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
#ifdef PAT_TC_TRACE
  if (tid == 0 && blockIdx.x < kSpanCtas) g_span_tc[0][blockIdx.x][1] = (unsigned long long)gtime();
#endif
  if (tid == 0) {
    // the last CTA out re-arms the item counter for the next launch
    __threadfence();
    if (atomicAdd(sched + 1, 1) == (int)gridDim.x - 1) {
      sched[0] = 0;
      sched[1] = 0;
      sched[2] = 0;
      __threadfence();
    }
  }
}

}  // namespace tc4

template <int D, typename T>
static cudaError_t launch_tc4_t(const CUtensorMap& tmk, const CUtensorMap& tmv, const DevPlan& plan, int var,
                                int grid, const void* q, void* out, float* po, float* pl, float scale_log2,
                                int32_t* sched, cudaStream_t st) {
  constexpr int smem = tc4::Layout<D>::kAlloc;
  // the opt-in is per device; setting it is cheap and idempotent
  cudaError_t e = cudaFuncSetAttribute(tc4::fwd_tc4_kernel<D, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  tc4::fwd_tc4_kernel<D, T><<<grid, tc4::kThreads, smem, st>>>(tmk, tmv, plan, var, (const T*)q, (T*)out, po, pl,
                                                               scale_log2, sched);
  return cudaGetLastError();
}

#ifdef PAT_TC_TRACE
extern "C" int pat_debug_tc_trace(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, tc4::g_tc_trace, sizeof(tc4::g_tc_trace));
}
extern "C" int pat_debug_trace_cta(int cta) {
  static long long zero[4][8][tc4::kTraceSteps];
  cudaMemcpyToSymbol(tc4::g_tc_trace, zero, sizeof(zero));
  return (int)cudaMemcpyToSymbol(tc4::g_trace_cta, &cta, sizeof(int));
}
extern "C" int pat_debug_item_log(long long* host, int* n) {
  int e = (int)cudaMemcpyFromSymbol(n, tc4::g_item_n, sizeof(int));
  if (e) return e;
  e = (int)cudaMemcpyFromSymbol(host, tc4::g_item_log, sizeof(tc4::g_item_log));
  int zero = 0;
  cudaMemcpyToSymbol(tc4::g_item_n, &zero, sizeof(int));
  return e;
}
extern "C" int pat_debug_spans_tc(unsigned long long* host) {
  int e = (int)cudaMemcpyFromSymbol(host, tc4::g_span_tc, sizeof(tc4::g_span_tc));
  static unsigned long long zero[1][kSpanCtas][2];
  cudaMemcpyToSymbol(tc4::g_span_tc, zero, sizeof(zero));
  return e;
}
#endif

cudaError_t launch_forward_tc(const CUtensorMap& tmk, const CUtensorMap& tmv, const DevPlan& plan, int var, int grid,
                              int dtype, int d, const void* q, void* out, float* po, float* pl, float scale_log2,
                              int32_t* sched, cudaStream_t st) {
  if (dtype == PAT_DTYPE_F16) {
    if (d == 128) return launch_tc4_t<128, __half>(tmk, tmv, plan, var, grid, q, out, po, pl, scale_log2, sched, st);
    return launch_tc4_t<64, __half>(tmk, tmv, plan, var, grid, q, out, po, pl, scale_log2, sched, st);
  }
  if (d == 128)
    return launch_tc4_t<128, __nv_bfloat16>(tmk, tmv, plan, var, grid, q, out, po, pl, scale_log2, sched, st);
  return launch_tc4_t<64, __nv_bfloat16>(tmk, tmv, plan, var, grid, q, out, po, pl, scale_log2, sched, st);
}

}  // namespace pat
