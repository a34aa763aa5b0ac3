// Tensor-core (tcgen05 + TMEM + TMA) forward kernel for WIDE packs, two
// 128-row query tiles per CTA (FA4-style ping-pong).
//
// A pack whose query tile (queries x G heads of one kv head) fills >= 64 rows
// forms a real dense contraction: S = Q K^T and O += P V run on the 5th-gen
// tensor cores.  One CTA (12 warps, one per SM) owns work items of
// (unit, kv head, 256 rows) = tiles A (rows 0-127) and B (rows 128-255) and
// streams the unit's KV span ONCE for both:
//   warp 0      TMA producer: 16-token page slices of K and V, 5-stage ring of
//               64-token stages, 128B swizzle, from the paged cache;
//   warp 1      MMA issuer (one thread), per KV tile j:
//                 S_A(j) = Q_A K_j^T, S_B(j) = Q_B K_j^T   (SS, M=128 N=64 K=d)
//                 O_A += P_A(j-1) V_{j-1}, O_B += P_B(j-1) V_{j-1}
//                 (TS: P read straight from TMEM, V an MN-major smem operand)
//               so the tensor core works on one tile while the other tile's
//               softmax runs;
//   warp 2      TMEM allocator (512 columns: S_A x2, S_B x2, O_A, O_B);
//   warps 4-7   softmax / epilogue of tile A (thread = row = TMEM lane);
//   warps 8-11  softmax / epilogue of tile B.
// Softmax: tcgen05.ld S, scale/mask in log2 units, lazy O rescale (only when the
// running max grows by > 8), P packed to 16-bit and tcgen05.st back over S
// (bf16: P = hi + lo, two PV MMAs, ~16-bit P).  Numerics follow cta_partial
// (attention.py:140-163): fp32 scores and accumulators.
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
// roles: 0 producer, 1 MMA issuer, 2 softmax tile A (warp 4 lane 0), 3 softmax tile B.
constexpr int kTraceSteps = 256;
__device__ long long g_tc_trace[4][8][kTraceSteps];
__device__ unsigned long long g_span_tc[1][kSpanCtas][2];
#define TC_TRACE(role, ev, step)                                        \
  do {                                                                  \
    if (blockIdx.x == 0 && (step) < kTraceSteps) g_tc_trace[role][ev][step] = clock64(); \
  } while (0)
#else
#define TC_TRACE(role, ev, step) \
  do {                           \
  } while (0)
#endif
constexpr int kThreads = 576;  // producer, MMA issuer (+TMEM alloc), 16 softmax warps
constexpr int kM = 128;       // rows per tile
constexpr int kN = 64;        // tokens per KV tile
constexpr int kStages = 4;
constexpr uint32_t kTmemCols = 512;
#ifndef PAT_TC_RESCALE_THRESHOLD
#define PAT_TC_RESCALE_THRESHOLD 8.0f
#endif
constexpr float kRescaleThreshold = PAT_TC_RESCALE_THRESHOLD;  // log2 units

template <int D>
struct Layout {
  static constexpr int KB = D / 64;
  static constexpr int kQBytes = KB * kM * 128;      // one tile's Q: [KB][128][64]
  static constexpr int kTileBytes = KB * kN * 128;   // K or V stage tile: [KB][64][64]
  static constexpr int kOffQ = 0;                    // Q_A, Q_B
  static constexpr int kOffKV = 2 * kQBytes;
  static constexpr int kOffBar = kOffKV + kStages * 2 * kTileBytes;
  static constexpr int kOffRed = kOffBar + 512;         // row-max / row-sum exchange
  static constexpr int kOffRing = kOffRed + 2 * 2 * 2 * kM * 4;  // 2 x ItemSlot
  static constexpr int kBytes = kOffRing + 2 * 2112;
  static constexpr int kAlloc = kBytes + 1024;
};

enum Bar : int {
  KV_FULL = 0,
  KV_EMPTY = KV_FULL + kStages,
  S_FULL = KV_EMPTY + kStages,  // [tile] QK done
  S_EMPTY = S_FULL + 2,         // [tile] softmax has read S
  P_FULL = S_EMPTY + 2,         // [tile] P written to TMEM
  O_DONE = P_FULL + 2,          // [tile] PV done (O updated, P region free)
  O_EMPTY = O_DONE + 2,         // [tile]
  Q_FULL = O_EMPTY + 2,         // [tile]
  Q_EMPTY = Q_FULL + 2,         // [tile]
  ITEM_FULL = Q_EMPTY + 2,      // [slot] work-item index published by the producer
  ITEM_EMPTY = ITEM_FULL + 2,   // [slot] read by the MMA warp and the 16 softmax warps
  NUM_BARS = ITEM_EMPTY + 2
};
constexpr int kItemReaders = 17;

// One slot of the work-item ring: the item and, per row, the query id and
// partial slot resolved by the producer warp (so consumers never chase the
// pack_q / unit_slot indirections at an item boundary).
struct ItemSlot {
  int32_t idx;
  int32_t pad[7];
  Item item;
  int2 meta[2 * 128];  // (qid, slot) per row
};
static_assert(sizeof(ItemSlot) == 2112, "ItemSlot layout");

template <typename T> struct Fmt;
template <> struct Fmt<__half> {
  static constexpr int ab = 0;
  static constexpr bool kSplit = false;
  static __device__ __forceinline__ uint32_t pack(float a, float b) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
  static __device__ __forceinline__ uint32_t pack_lo(float, float, uint32_t) { return 0u; }
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
  static __device__ __forceinline__ uint32_t pack_lo(float a, float b, uint32_t hi) {
    __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162*>(&hi);
    float2 f = __bfloat1622float2(h);
    return pack(a - f.x, b - f.y);
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
// 16-byte global -> shared async copy; src_size 0 zero-fills the destination
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
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
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sb = smem_u32(smem);
  const uint32_t sKV = sb + L::kOffKV;
  const uint32_t bars = sb + L::kOffBar;
  uint32_t* tmem_slot = (uint32_t*)(smem + L::kOffBar + NUM_BARS * 8);
  ItemSlot* ring = reinterpret_cast<ItemSlot*>(smem + L::kOffRing);
  auto bar = [&](int i) { return bars + 8u * (uint32_t)i; };
  auto sQ = [&](int x) { return sb + L::kOffQ + (uint32_t)(x * L::kQBytes); };
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
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(S_FULL + i), 1);
      mbar_init(bar(S_EMPTY + i), 8);
      mbar_init(bar(P_FULL + i), 8);
    }
    for (int x = 0; x < 2; ++x) {
      mbar_init(bar(O_DONE + x), 1);
      mbar_init(bar(O_EMPTY + x), 8);
      mbar_init(bar(Q_FULL + x), 8);
      mbar_init(bar(Q_EMPTY + x), 1);
      mbar_init(bar(ITEM_FULL + x), 32);
      mbar_init(bar(ITEM_EMPTY + x), kItemReaders);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(smem_u32(tmem_slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  PAT_SPAN_BEGIN(g_span_tc, 0);
  // TMEM columns: S[x] at 128x, P[x] at 128x + 64 (hi: +0..31, lo: +32..63),
  // O[x] at 256 + 128x.  P has its own columns: a PV MMA reading P from TMEM
  // must never share columns with a later QK MMA's accumulator (measured WAR
  // hazard when P lived inside the double-buffered S region).
  // Dynamic work distribution: the producer claims items (in the scheduler's
  // longest-first order) from a global counter one item ahead and publishes
  // the index through a 2-slot shared ring; the MMA warp and the softmax
  // warps follow the same sequence.  -1 ends the loop.
  // Returns the item index (-1 = done), the item and, for row `r` (< 0: none),
  // its (qid, slot) metadata.
  auto next_item = [&](uint32_t n, Item& itm, int r, int2& meta) -> int {
    const uint32_t slot = n & 1;
    mbar_wait(bar(ITEM_FULL + slot), (n >> 1) & 1);
    const ItemSlot* rs = ring + slot;  // plain loads: ordered by the mbarrier wait (asm memory clobber)
    const int it = rs->idx;
    if (it >= 0) {
      itm = rs->item;
      if (r >= 0 && r < itm.nrows) meta = rs->meta[r];
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(bar(ITEM_EMPTY + slot));
    return it;
  };
  auto tS = [&](int x) { return tmem + (uint32_t)(128 * x); };
  auto tP = [&](int x) { return tmem + (uint32_t)(128 * x + 64); };
  auto tO = [&](int x) { return tmem + 256u + (uint32_t)(128 * x); };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    // Whole warp: lane i fetches the block id of page group i of the stage,
    // broadcast by shuffle (warp-uniform operands), one elected lane issues.
    {
      if (elect_one()) {
        tma_prefetch(&tmk);
        tma_prefetch(&tmv);
      }
      uint32_t g = 0;
      for (uint32_t n = 0;; ++n) {
        const uint32_t slot = n & 1;
        mbar_wait(bar(ITEM_EMPTY + slot), ((n >> 1) & 1) ^ 1);
        int it = 0;
        if (lane == 0) {
          it = atomicAdd(plan.sched, 1);
          if (it >= n_items) it = -1;
        }
        it = __shfl_sync(0xffffffffu, it, 0);
        Item item{};
        if (it >= 0) {
          item = load_item(items + it);
          for (int r = lane; r < item.nrows; r += 32) {
            const int qi = (item.row0 + r) / G;
            ring[slot].meta[r] = make_int2(__ldg(plan.pack_q + item.qoff + qi), __ldg(plan.unit_slot + item.slot_off + qi));
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
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // The whole warp runs the loop so descriptors and TMEM addresses stay
    // warp-uniform (uniform datapath, no per-MMA waterfall); one elected lane
    // issues each tcgen05.mma / commit (CUTLASS's elect_one_sync pattern).
    {
      constexpr uint32_t idesc_qk = umma_idesc_f16(kM, kN, Fmt<T>::ab, 0);
      constexpr uint32_t idesc_pv = umma_idesc_f16(kM, D, Fmt<T>::ab, 1);
      uint32_t g = 0;           // KV tiles consumed
      uint32_t c[2] = {0, 0};   // KV tiles processed per query tile (S/P buffer index)
      uint32_t ni[2] = {0, 0};  // items processed per query tile
      auto commit = [&](int b) {
        if (elect_one()) umma_commit(bar(b));
        __syncwarp();
      };
      auto issue_qk = [&](int x, int s, uint32_t ci) {
        // S[x] is single-buffered: wait until the softmax has read tile ci-1
        mbar_wait(bar(S_EMPTY + x), (ci & 1) ^ 1);
        if (x == 0) TC_TRACE(1, 3, g);
        tc_fence_after();
        const uint64_t a0 = umma_desc_sw128(sQ(x), 16, 1024), b0 = umma_desc_sw128(sK(s), 16, 1024);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const int kb = k >> 2, kk = k & 3;
            // descriptor start address is in 16-byte units (bits 0-13)
            umma_f16_ss(tS(x), a0 + (uint64_t)((kb * (kM * 128) + kk * 32) >> 4),
                        b0 + (uint64_t)((kb * (kN * 128) + kk * 32) >> 4), idesc_qk, k > 0 ? 1u : 0u);
          }
        }
        __syncwarp();
      };
      auto issue_pv = [&](int x, int s, uint32_t ci, bool first) {
        if (first) mbar_wait(bar(O_EMPTY + x), (ni[x] & 1) ^ 1);
        mbar_wait(bar(P_FULL + x), ci & 1);
        if (x == 0) TC_TRACE(1, 4, g);
        tc_fence_after();
        const uint64_t v0 = umma_desc_sw128(sV(s), kN * 128, 1024);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < kN / 16; ++k) {
            const uint64_t bd = v0 + (uint64_t)((k * 16 * 128) >> 4);
            // P(m, k) is packed two per column: a k-step of 16 tokens = 8 columns
            umma_f16_ts(tO(x), tP(x) + k * 8, bd, idesc_pv, (first && k == 0) ? 0u : 1u);
            if constexpr (kSplit) umma_f16_ts(tO(x), tP(x) + 32 + k * 8, bd, idesc_pv, 1u);
          }
          umma_commit(bar(O_DONE + x));
        }
        __syncwarp();
      };
      for (uint32_t n = 0;; ++n) {
        Item item;
        int2 unused;
        if (next_item(n, item, -1, unused) < 0) break;
        const bool liveB = item.nrows > kM;
        const int ntiles = (item.ntok + kN - 1) / kN;
        mbar_wait(bar(Q_FULL + 0), ni[0] & 1);
        if (liveB) mbar_wait(bar(Q_FULL + 1), ni[1] & 1);
        TC_TRACE(1, 5, g);
        tc_fence_after();
        int sprev = 0;
        for (int j = 0; j < ntiles; ++j, ++g) {
          const int s = g % kStages;
          mbar_wait(bar(KV_FULL + s), (g / kStages) & 1);
          TC_TRACE(1, 0, g);
          tc_fence_after();
          // Both tiles' S MMAs are issued before either S_FULL is signalled:
          // a softmax must not read/write its S region while the OTHER tile's
          // QK MMA is in flight (measured: corrupted S/P when the two S
          // regions are 128 or 256 TMEM columns apart; tools/tc_debug.py).
          issue_qk(0, s, c[0] + j);
          if (liveB) issue_qk(1, s, c[1] + j);
          commit(S_FULL + 0);
          if (liveB) commit(S_FULL + 1);
          if (j == ntiles - 1) {
            commit(Q_EMPTY + 0);
            if (liveB) commit(Q_EMPTY + 1);
          }
          TC_TRACE(1, 1, g);
          if (j > 0) {
            issue_pv(0, sprev, c[0] + j - 1, j == 1);
            TC_TRACE(1, 2, g);
            if (liveB) issue_pv(1, sprev, c[1] + j - 1, j == 1);
            commit(KV_EMPTY + sprev);
          }
          sprev = s;
        }
        issue_pv(0, sprev, c[0] + ntiles - 1, ntiles == 1);
        if (liveB) issue_pv(1, sprev, c[1] + ntiles - 1, ntiles == 1);
        commit(KV_EMPTY + sprev);
        c[0] += ntiles;
        ++ni[0];
        if (liveB) {
          c[1] += ntiles;
          ++ni[1];
        }
      }
    }
  } else {
    // ------------------------------------------------------------ softmax / epilogue
    // 16 warps (2-17): tile x = sw >> 3, column half h = (sw >> 2) & 1, lane
    // quarter wq = warp % 4 (the TMEM lanes the warp may access).  The two
    // halves of a row (same lanes, same SMSP) exchange their partial row max
    // through shared memory each KV tile, so both keep the same running max.
    const int sw = warp - 2;
    const int x = sw >> 3, h = (sw >> 2) & 1, wq = warp & 3;
    const int t = wq * 32 + lane;                 // row in the tile == TMEM lane
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    const uint32_t pair_bar = 1 + x * 4 + wq;     // named barrier of the two half-warps
    float* red = reinterpret_cast<float*>(smem + L::kOffRed);  // [2 parity][2 tile][2 half][128]
    auto red_at = [&](uint32_t par, int hh) { return red + ((par * 2 + x) * 2 + hh) * kM + t; };
    uint32_t c = 0, ni = 0, g = 0, xc = 0;  // xc: exchange-buffer uses
    const int r = x * kM + t;                // row within an item
    constexpr int kCh = D / 16;              // 16-byte chunks per half row
    // Item n stays in its ring slot until this warp releases it after the
    // epilogue, so per-item fields are re-read from shared memory where used
    // instead of occupying registers across the KV loop.
    auto wait_item = [&](uint32_t n) -> const ItemSlot* {
      mbar_wait(bar(ITEM_FULL + (n & 1)), (n >> 1) & 1);
      return ring + (n & 1);
    };
    auto release_item = [&](uint32_t n) {
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(ITEM_EMPTY + (n & 1)));
    };
    auto x_live = [&](const ItemSlot* s) { return x == 0 || s->item.nrows > kM; };
    // cp.async this thread's half Q row of the slot's item into the swizzled
    // Q tile (zero-filled for rows past the item).
    auto issue_q = [&](const ItemSlot* s) {
      const bool lv = r < s->item.nrows;
      const int head = s->item.kvh * G + (lv ? (s->item.row0 + r) % G : 0);
      const T* srcq = qg + ((int64_t)(lv ? s->meta[r].x : 0) * H + head) * D;
#pragma unroll
      for (int i = 0; i < kCh; ++i) {
        const int ch = h * kCh + i;
        cp_async16(sQ(x) + (ch >> 3) * (kM * 128) + t * 128 + (((ch & 7) ^ (t & 7)) << 4), srcq + ch * 8, lv);
      }
    };
    auto finish_q = [&]() {
      cp_async_wait_all();
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(Q_FULL + x));
      if (t == 0 && h == 0) TC_TRACE(2 + x, 4, g);
    };
    bool q_pending = false;  // Q of the next x-live item issued, Q_FULL not yet arrived
    {
      const ItemSlot* s0 = wait_item(0);
      if (s0->idx >= 0 && x_live(s0)) {
        mbar_wait(bar(Q_EMPTY + x), (ni & 1) ^ 1);
        issue_q(s0);
        q_pending = true;
      }
    }
    for (uint32_t n = 0;; ++n) {
      const ItemSlot* cs = ring + (n & 1);  // ITEM_FULL(n) already waited
      if (cs->idx < 0) break;
      const int ntok = cs->item.ntok;
      const int ntiles = (ntok + kN - 1) / kN;
      if (!x_live(cs)) {
        // tile B idle for this item; prefetch Q if the next item uses it
        g += ntiles;
        const ItemSlot* ns = wait_item(n + 1);
        if (ns->idx >= 0 && x_live(ns)) {
          mbar_wait(bar(Q_EMPTY + x), (ni & 1) ^ 1);
          issue_q(ns);
          q_pending = true;
        }
        release_item(n);
        continue;
      }
      if (q_pending) {
        finish_q();
        q_pending = false;
      }

      float m_ref = -INFINITY;  // running max, log2 units
      float2 l2 = make_float2(0.f, 0.f);
      for (int j = 0; j < ntiles; ++j, ++c, ++g) {
        mbar_wait(bar(S_FULL + x), c & 1);
        if (t == 0 && h == 0) TC_TRACE(2 + x, 0, g);
        tc_fence_after();
        uint32_t sr[32];
        tmem_ld32(tS(x) + lane_base + 32 * h, sr);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar(S_EMPTY + x));
        if (j == ntiles - 1) {
          // last KV tile: this item's last QK is done, so the Q tile is free --
          // start copying the next item's Q rows now
          const ItemSlot* ns = wait_item(n + 1);
          if (ns->idx >= 0 && x_live(ns)) {
            mbar_wait(bar(Q_EMPTY + x), ni & 1);
            issue_q(ns);
            q_pending = true;
          }
        }

        const int valid = ntok - j * kN - 32 * h;  // valid columns of this half
        if (valid < 32) {
#pragma unroll
          for (int k = 0; k < 32; ++k)
            if (k >= valid) sr[k] = __float_as_uint(-INFINITY);
        }
        float pm[11];
#pragma unroll
        for (int k = 0; k < 10; ++k)
          pm[k] = fmax3(__uint_as_float(sr[3 * k]), __uint_as_float(sr[3 * k + 1]), __uint_as_float(sr[3 * k + 2]));
        pm[10] = fmaxf(__uint_as_float(sr[30]), __uint_as_float(sr[31]));
        float pmx = fmax3(fmax3(pm[0], pm[1], pm[2]), fmax3(pm[3], pm[4], pm[5]),
                          fmax3(fmax3(pm[6], pm[7], pm[8]), pm[9], pm[10]));
        *red_at(xc & 1, h) = pmx;
        named_bar_sync(pair_bar, 64);
        const float mx = fmaxf(pmx, *red_at(xc & 1, h ^ 1)) * scale_log2;
        ++xc;
        const bool need = mx > m_ref + kRescaleThreshold;
        if (__any_sync(0xffffffffu, need)) {
          const float m_new = need ? mx : m_ref;
          const float alpha = ex2_approx(m_ref - m_new);
          if (j > 0) {
            mbar_wait(bar(O_DONE + x), (c - 1) & 1);
            tc_fence_after();
#pragma unroll
            for (int q = 0; q < D / 32; ++q) {
              uint32_t o[16];
              const uint32_t ta = tO(x) + lane_base + (uint32_t)(h * (D / 2) + q * 16);
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
        // P = exp2(s * scale - m_ref), packed 16-bit pairs (hi: 16 cols, lo: 16
        // cols), computed and stored in two chunks of 16 columns
        const float2 sc2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-m_ref, -m_ref);
#pragma unroll
        for (int q2 = 0; q2 < 2; ++q2) {
          uint32_t ph[8], pl[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int kk = q2 * 8 + k;
            float2 a = __ffma2_rn(make_float2(__uint_as_float(sr[2 * kk]), __uint_as_float(sr[2 * kk + 1])), sc2, nm2);
            a.x = ex2_approx(a.x);
            a.y = ex2_approx(a.y);
            ph[k] = Fmt<T>::pack(a.x, a.y);
            if constexpr (kSplit) {
              const float2 hf = make_float2(__uint_as_float(ph[k] << 16), __uint_as_float(ph[k] & 0xffff0000u));
              const float2 lo = __fadd2_rn(a, make_float2(-hf.x, -hf.y));
              pl[k] = Fmt<T>::pack(lo.x, lo.y);
              l2 = __fadd2_rn(l2, a);
            } else {
              // normalise by the sum of the ROUNDED weights the MMA actually uses:
              // the output is then an exact weighted average of V rows
              l2 = __fadd2_rn(l2, Fmt<T>::unpack(ph[k]));
            }
          }
          if (q2 == 0) {
            if (t == 0 && h == 0) TC_TRACE(2 + x, 1, g);
            // the P columns are free once PV of the previous tile completed
            if (j > 0) {
              mbar_wait(bar(O_DONE + x), (c - 1) & 1);
              tc_fence_after();
            }
            if (t == 0 && h == 0) TC_TRACE(2 + x, 2, g);
          }
          tmem_st8(tP(x) + lane_base + 16 * h + 8 * q2, ph);
          if constexpr (kSplit) tmem_st8(tP(x) + lane_base + 32 + 16 * h + 8 * q2, pl);
        }
        if (j * kN + kN > ntok) {
          // tail tile: zero V rows past the span (both tiles may do it: same zeros)
          const int vt = ntok - j * kN;
          const int s = g % kStages;
          mbar_wait(bar(KV_FULL + s), (g / kStages) & 1);
          const int nz = (kN - vt) * L::KB * 8;
          for (int q = h * kM + t; q < nz; q += 2 * kM) {
            const int rr = vt + q / (L::KB * 8);
            const int kb = (q / 8) % L::KB, ch = q % 8;
            st_shared_v4(sV(s) + kb * (kN * 128) + rr * 128 + (ch << 4), make_uint4(0, 0, 0, 0));
          }
          fence_proxy_async_smem();
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar(P_FULL + x));
        if (t == 0 && h == 0) TC_TRACE(2 + x, 3, g);
      }

      // the next item's first QK can now overlap this epilogue
      if (q_pending) {
        finish_q();
        q_pending = false;
      }
      // epilogue: O / l; the halves exchange their partial l
      float lh = l2.x + l2.y;
      *red_at(xc & 1, h) = lh;
      named_bar_sync(pair_bar, 64);
      const float l = lh + *red_at(xc & 1, h ^ 1);
      ++xc;
      const bool live = r < cs->item.nrows;
      const int2 meta = live ? cs->meta[r] : make_int2(0, -1);
      const int head = cs->item.kvh * G + (live ? (cs->item.row0 + r) % G : 0);
      mbar_wait(bar(O_DONE + x), (c - 1) & 1);
      tc_fence_after();
      const float inv = 1.f / l;
#pragma unroll
      for (int q = 0; q < D / 32; ++q) {
        uint32_t o[16];
        const int col = h * (D / 2) + q * 16;
        tmem_ld16(tO(x) + lane_base + (uint32_t)col, o);
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
      if (live && meta.y >= 0 && h == 0) part_lse[(int64_t)meta.y * H + head] = m_ref + log2f(l);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(O_EMPTY + x));
      if (t == 0 && h == 0) TC_TRACE(2 + x, 5, g - 1);
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
