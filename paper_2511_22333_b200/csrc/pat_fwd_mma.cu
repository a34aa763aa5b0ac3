// Streaming forward kernel for packs whose query tile is narrow (rows = q*G <= 64
// per CTA) and the online-softmax merge kernel.
//
// One CTA (4 warps) owns one work item = (forward unit, kv head, row block) and
// computes, for each of its rows (query i of the pack, head kvh*G+g), the
// partial (max, exp-sum, weighted V sum) of cta_partial (attention.py:140-163)
// over the unit's KV span -- online, in 64-token stages:
//   * every K/V page of the stage is copied ONCE per CTA into shared memory
//     (16-byte cp.async, 128B-swizzled rows, 3-stage ring) and shared by all
//     rows of the pack (this is what packing buys: one load of a shared prefix
//     for all its queries);
//   * S = Q K^T and O += P V run on tensor cores with mma.sync m16n8k16
//     (Q rows padded to 16); fp32 accumulate, P rounded to the input dtype;
//   * the warps of one 16-row tile split the stage's tokens and are combined
//     at the end in shared memory.
// A row whose query is covered by this unit only is normalised and written to
// the output directly; otherwise (o/l, log2-sum-exp) goes to its fp32 slot and
// the merge kernel folds the slots (_merge_batch_into, attention.py:187-199).
#include <atomic>
#include <algorithm>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "pat_merge.cuh"
#include "pat_mma_sync.cuh"
#include "pat_plan.cuh"
#include "pat_sm100.cuh"

namespace pat {

constexpr int kStageTok = 64;

template <typename T> struct Vec2;
template <> struct Vec2<__half> {
  // fp16 P keeps 11 significant bits: one PV pass is exact enough
  static constexpr bool kSplitP = false;
  static __device__ __forceinline__ uint32_t pack(float a, float b) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
  static __device__ __forceinline__ uint32_t pack_lo(float, float, uint32_t) { return 0u; }
};
template <> struct Vec2<__nv_bfloat16> {
  // bf16 P keeps 8 significant bits (2^-9 relative error, visible on peaked
  // softmax rows): P = hi + lo, both bf16, two PV passes -> ~16-bit P
  static constexpr bool kSplitP = true;
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

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Shared-memory tiles hold 16-bit rows split into 64-element (128-byte) lines:
// a K/V stage is [page][D/64 halves][16 tokens][64], the Q tile [D/64][rows][64].
// The 16-byte chunk c of a line is stored at c ^ (row & 7) -- the TMA/UMMA
// 128B swizzle pattern (line index mod 8 == row mod 8 in these layouts), which
// makes every ldmatrix phase (8 consecutive rows, same chunk) conflict-free.
template <int D>
__device__ __forceinline__ uint32_t swz_kv(int t, int ch) {
  int line = (t >> 4) * (D / 64) * 16 + (ch >> 3) * 16 + (t & 15);
  return (uint32_t)(line * 128 + (((ch & 7) ^ (t & 7)) << 4));
}
template <int ROWS>
__device__ __forceinline__ uint32_t swz_q(int r, int ch) {
  int line = (ch >> 3) * ROWS + r;
  return (uint32_t)(line * 128 + (((ch & 7) ^ (r & 7)) << 4));
}

#ifdef PAT_TC_TRACE
__device__ unsigned long long g_span_mma[2][kSpanCtas][2];  // [stream, merge][cta][start, end]
#endif

template <int WM, int D>
struct StreamSmem {
  static constexpr int KB = D / 64;
  static constexpr int kTileBytes = kStageTok * D * 2;  // one K or V stage tile
  static constexpr int kStageBytes = 2 * kTileBytes;
  // K+V ring: as deep as the 227 KB budget allows next to Q (x2) and the scratch
  static constexpr int kNumStages = D == 128 ? (WM == 4 ? 4 : (WM == 2 ? 5 : 6)) : 8;
  static constexpr int kQBytes = WM * 16 * D * 2;       // linear [rows][D] (bulk-copied)
  // epilogue: per-warp O for half of head_dim at a time (two passes), m, l
  static constexpr int kScratchBytes = 4 * 16 * (D / 2) * 4 + 2 * 4 * 16 * 4;
  static constexpr int kOffQ = kNumStages * kStageBytes;  // two Q buffers
  static constexpr int kOffScratch = kOffQ + 2 * kQBytes;
  static constexpr int kOffBar = kOffScratch + kScratchBytes;
  static constexpr int kNumBars = 2 * kNumStages + 4;
  static constexpr int kBytes = kOffBar + kNumBars * 8;
  static constexpr int kAlloc = kBytes + 1024;
};

// warps 0-3 consumers (mma.sync), warp 4 producer (one thread)
constexpr int kStreamThreads = 160;

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const void* tmap, uint32_t bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];\n" ::"r"(dst),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n)); }

__device__ __forceinline__ Item load_item(const Item* p) {
  const int4* q = reinterpret_cast<const int4*>(p);
  int4 a = __ldg(q), b = __ldg(q + 1);
  return Item{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
}

// Streaming forward: one producer warp runs ahead through the CTA's items --
// TMA boxes for every 16-token page slice of K and V (5-stage ring) and a bulk
// copy of the item's Q rows into a double-buffered Q tile -- while four mma.sync
// consumer warps compute.  The producer prefetches the next item's descriptor
// and block ids, so item boundaries never drain the ring.
template <int WM, int D, typename T>
__global__ void __launch_bounds__(kStreamThreads, 1)
    fwd_stream_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                      DevPlan plan, int var, const T* __restrict__ qg, T* __restrict__ out,
                      float* __restrict__ part_o, float* __restrict__ part_lse, float scale_log2) {
  using S = StreamSmem<WM, D>;
  constexpr int NS = S::kNumStages;
  constexpr int WN = 4 / WM;          // warps sharing one row tile
  constexpr int TW = kStageTok / WN;  // tokens per warp per stage
  constexpr int NT = TW / 8;          // score n-tiles per warp
  constexpr int KS = D / 16;          // k-steps over head_dim
  constexpr int CH = D / 8;           // 16-byte chunks per token row
  constexpr int ROWS = WM * 16;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t full0 = sbase + S::kOffBar, empty0 = full0 + NS * 8;
  const uint32_t qfull0 = empty0 + NS * 8, qempty0 = qfull0 + 16;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int H = plan.H, G = plan.G, bs = plan.bs;
  const int n_items = plan.n_items[var];
  const Item* items = plan.items[var];

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 4);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(qfull0 + 8 * b, 1);
      mbar_init(qempty0 + 8 * b, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  PAT_SPAN_BEGIN(g_span_mma, 0);

  if (warp == 4) {
    // ------------------------------------------------------------ producer
    // One thread: item descriptors one item ahead, block ids one stage ahead
    // (independent loads, latency hidden behind the ring wait), Q rows by bulk
    // copy, K/V page slices by TMA.
    // Whole warp (warp-uniform TMA operands: lane i fetches page group i's
    // block id, broadcast by shuffle); lane 0 issues.
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmk) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmv) : "memory");
    }
    uint32_t g = 0, n = 0;
    int it = blockIdx.x;
    Item item;
    if (it < n_items) item = load_item(items + it);
    for (; it < n_items; it += gridDim.x, ++n) {
      const int nxt = it + gridDim.x;
      Item next_item = item;
      if (nxt < n_items) next_item = load_item(items + nxt);
      const int h = item.kvh, ntok = item.ntok;
      const int32_t* blist = plan.pack_blk + item.blk;
      const int nst = (ntok + kStageTok - 1) / kStageTok;
#if !(defined(PAT_STREAM_NOCOMPUTE) && PAT_STREAM_NOCOMPUTE >= 2)
      {
        const uint32_t qb = n & 1;
        const uint32_t dq = sbase + S::kOffQ + qb * S::kQBytes;
        const int r_end = item.row0 + item.nrows;
        const int i0 = item.row0 / G, i1 = (r_end - 1) / G;
        mbar_wait(qempty0 + 8 * qb, ((n >> 1) & 1) ^ 1);
        if (lane == 0) mbar_expect_tx(qfull0 + 8 * qb, (uint32_t)(item.nrows * D * 2));
        __syncwarp();
        for (int i = i0 + lane; i <= i1; i += 32) {
          const int a = max(i * G, item.row0), e = min((i + 1) * G, r_end);
          const int qid = __ldg(plan.pack_q + item.qoff + i);
          const T* src = qg + ((int64_t)qid * H + h * G + (a - i * G)) * D;
          bulk_load(dq + (a - item.row0) * D * 2, src, (uint32_t)((e - a) * D * 2), qfull0 + 8 * qb);
        }
      }
#endif
      for (int st = 0; st < nst; ++st, ++g) {
        const int s = g % NS;
        const int rem = ntok - st * kStageTok;
        const int ngrp = rem >= kStageTok ? kStageTok / 16 : (rem + 15) / 16;
        const uint32_t dk = sbase + s * S::kStageBytes, dv = dk + S::kTileBytes;
        int my_blk = 0, my_off = 0;
        if (lane < ngrp) {
          const int tok = st * kStageTok + lane * 16;
          const int pg = bs == 16 ? (tok >> 4) : tok / bs;
          my_blk = __ldg(blist + pg);
          my_off = bs == 16 ? 0 : tok - pg * bs;
        }
        mbar_wait(empty0 + 8 * s, ((g / NS) & 1) ^ 1);
        if (lane == 0) mbar_expect_tx(full0 + 8 * s, (uint32_t)(ngrp * S::KB * 2048 * 2));
        __syncwarp();
        for (int gr = 0; gr < ngrp; ++gr) {
          const int blk = __shfl_sync(0xffffffffu, my_blk, gr);
          const int off = __shfl_sync(0xffffffffu, my_off, gr);
          if (sm100::elect_one()) {
#pragma unroll
            for (int kb = 0; kb < S::KB; ++kb) {
              const uint32_t o = (uint32_t)((gr * S::KB + kb) * 2048);
              tma_load_4d(dk + o, &tmk, full0 + 8 * s, kb * 64, h, off, blk);
              tma_load_4d(dv + o, &tmv, full0 + 8 * s, kb * 64, h, off, blk);
            }
          }
          __syncwarp();
        }
      }
      item = next_item;
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int mt = warp / WN, wn = warp % WN;
  // epilogue metadata: warp w writes rows w, w+4, ...; lane k holds (qid, slot)
  // of row w + 4k.  Loaded one item ahead so item boundaries cost no latency.
  auto load_meta = [&](const Item& itm, int& mq, int& ms) {
    mq = 0;
    ms = -1;
    if (lane < ROWS / 4) {
      const int r = warp + 4 * lane;
      if (r < itm.nrows) {
        const int i = (itm.row0 + r) / G;
        mq = __ldg(plan.pack_q + itm.qoff + i);
        ms = __ldg(plan.unit_slot + itm.slot_off + i);
      }
    }
  };
  uint32_t g = 0, n = 0;
  Item item;
  int meta_qid = 0, meta_slot = -1;
  if ((int)blockIdx.x < n_items) {
    item = load_item(items + blockIdx.x);
    load_meta(item, meta_qid, meta_slot);
  }
  for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++n) {
    const int nxt = it + gridDim.x;
    Item next_item = item;
    if (nxt < n_items) next_item = load_item(items + nxt);
    const int h = item.kvh, ntok = item.ntok;
    const int nst = (ntok + kStageTok - 1) / kStageTok;

    // Q fragments (A operand) from the bulk-copied tile, then release the buffer
    const uint32_t qb = n & 1;
    const uint32_t sq = sbase + S::kOffQ + qb * S::kQBytes;
#if defined(PAT_STREAM_NOCOMPUTE) && PAT_STREAM_NOCOMPUTE >= 2
    for (int st = 0; st < nst; ++st, ++g) {
      const int s = g % NS;
      mbar_wait(full0 + 8 * s, (g / NS) & 1);
      __syncwarp();
      if (lane == 0) mbar_arrive(empty0 + 8 * s);
    }
    item = next_item;
    continue;
#endif
    mbar_wait(qfull0 + 8 * qb, (n >> 1) & 1);
    uint32_t qa[KS][4];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      int r = mt * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
      int ch = ks * 2 + (lane >> 4);
      ldsm_x4(qa[ks], sq + r * (D * 2) + ch * 16);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(qempty0 + 8 * qb);

    float o[D / 8][4];
#pragma unroll
    for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};

    for (int st = 0; st < nst; ++st, ++g) {
      const int s = g % NS;
      mbar_wait(full0 + 8 * s, (g / NS) & 1);
      const uint32_t tk = sbase + s * S::kStageBytes;
      const uint32_t tv = tk + S::kTileBytes;
      const int t0 = wn * TW;  // warp's first token inside the stage
      const int valid = ntok - st * kStageTok;
      if (valid < t0 + TW) {
        // tail: rows past the span hold stale/garbage bytes; zero this warp's V rows
        // so that P == 0 cannot meet a NaN
        for (int c = lane; c < TW * CH; c += 32) {
          int t = t0 + c / CH, ch = c % CH;
          if (t >= valid)
            asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};\n" ::"r"(tv + swz_kv<D>(t, ch)), "r"(0)
                         : "memory");
        }
        __syncwarp();
      }
#ifdef PAT_STREAM_NOCOMPUTE
      if (true) {
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 8 * s);
        continue;
      }
#endif
      float sc[NT][4];
#pragma unroll
      for (int j = 0; j < NT; ++j) sc[j][0] = sc[j][1] = sc[j][2] = sc[j][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
        for (int j = 0; j < NT; j += 2) {
          uint32_t b[4];
          int t = t0 + j * 8 + (lane & 7) + (lane >> 4) * 8;
          int ch = ks * 2 + ((lane >> 3) & 1);
          ldsm_x4(b, tk + swz_kv<D>(t, ch));
          mma16816<T>(sc[j], qa[ks], b[0], b[1]);
          mma16816<T>(sc[j + 1], qa[ks], b[2], b[3]);
        }
      }
      const int tbase = t0 + 2 * (lane & 3);
      float mx[2] = {mrow[0], mrow[1]};
#pragma unroll
      for (int j = 0; j < NT; ++j) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          int tok = tbase + j * 8 + (e & 1);
          float v = tok < valid ? sc[j][e] * scale_log2 : -INFINITY;
          sc[j][e] = v;
          mx[e >> 1] = fmaxf(mx[e >> 1], v);
        }
      }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
        mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
      }
      float alpha[2], muse[2];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        muse[r] = mx[r] == -INFINITY ? 0.f : mx[r];
        alpha[r] = exp2f(mrow[r] - muse[r]);
        mrow[r] = mx[r];
        lrow[r] *= alpha[r];
      }
#pragma unroll
      for (int i = 0; i < D / 8; ++i) {
        o[i][0] *= alpha[0];
        o[i][1] *= alpha[0];
        o[i][2] *= alpha[1];
        o[i][3] *= alpha[1];
      }
      constexpr bool kSplit = Vec2<T>::kSplitP;
      uint32_t pa[NT / 2][4], pl[kSplit ? NT / 2 : 1][4];
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        float p0 = exp2f(sc[j][0] - muse[0]), p1 = exp2f(sc[j][1] - muse[0]);
        float p2 = exp2f(sc[j][2] - muse[1]), p3 = exp2f(sc[j][3] - muse[1]);
        lrow[0] += p0 + p1;
        lrow[1] += p2 + p3;
        const uint32_t h01 = Vec2<T>::pack(p0, p1), h23 = Vec2<T>::pack(p2, p3);
        pa[j >> 1][(j & 1) * 2 + 0] = h01;
        pa[j >> 1][(j & 1) * 2 + 1] = h23;
        if constexpr (kSplit) {
          pl[j >> 1][(j & 1) * 2 + 0] = Vec2<T>::pack_lo(p0, p1, h01);
          pl[j >> 1][(j & 1) * 2 + 1] = Vec2<T>::pack_lo(p2, p3, h23);
        }
      }
#pragma unroll
      for (int kk = 0; kk < NT / 2; ++kk) {
#pragma unroll
        for (int dn = 0; dn < D / 16; ++dn) {
          uint32_t b[4];
          int t = t0 + kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
          int ch = dn * 2 + (lane >> 4);
          ldsm_x4_t(b, tv + swz_kv<D>(t, ch));
          mma16816<T>(o[dn * 2], pa[kk], b[0], b[1]);
          mma16816<T>(o[dn * 2 + 1], pa[kk], b[2], b[3]);
          if constexpr (kSplit) {
            mma16816<T>(o[dn * 2], pl[kk], b[0], b[1]);
            mma16816<T>(o[dn * 2 + 1], pl[kk], b[2], b[3]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty0 + 8 * s);
    }

    // ---- epilogue: combine the WN warps of each row tile through scratch ----
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 1);
      lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 2);
    }
    int next_qid = 0, next_slot = -1;
    if (nxt < n_items) load_meta(next_item, next_qid, next_slot);  // overlaps the epilogue
    constexpr int DH = D / 2;  // head-dim columns combined per pass
    float* so = reinterpret_cast<float*>(smem + S::kOffScratch);  // [4 warps][16][D / 2]
    float* sm = so + 4 * 16 * DH;                                 // [4][16]
    float* sl = sm + 4 * 16;                                      // [4][16]
#pragma unroll
    for (int pass = 0; pass < 2; ++pass) {
      named_sync(1, 128);  // previous scratch reads are done
      {
        const int ra = lane >> 2, rb = ra + 8, cb = 2 * (lane & 3);
        float* wo = so + warp * 16 * DH;
#pragma unroll
        for (int i = 0; i < D / 16; ++i) {
          const int ii = pass * (D / 16) + i;
          *reinterpret_cast<float2*>(wo + ra * DH + i * 8 + cb) = make_float2(o[ii][0], o[ii][1]);
          *reinterpret_cast<float2*>(wo + rb * DH + i * 8 + cb) = make_float2(o[ii][2], o[ii][3]);
        }
        if (pass == 0 && (lane & 3) == 0) {
          sm[warp * 16 + ra] = mrow[0];
          sm[warp * 16 + rb] = mrow[1];
          sl[warp * 16 + ra] = lrow[0];
          sl[warp * 16 + rb] = lrow[1];
        }
      }
      named_sync(1, 128);
#pragma unroll
      for (int k = 0; k < ROWS / 4; ++k) {
        const int r = warp + 4 * k;
        const int qid = __shfl_sync(0xffffffffu, meta_qid, k);
        const int slot = __shfl_sync(0xffffffffu, meta_slot, k);
        if (r >= item.nrows || lane * 2 >= DH) continue;
        const int x = lane * 2;  // within the pass's half
        const int tile = r / 16, rr = r % 16;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < WN; ++w) M = fmaxf(M, sm[(tile * WN + w) * 16 + rr]);
        float L = 0.f;
        float2 acc = make_float2(0.f, 0.f);
#pragma unroll
        for (int w = 0; w < WN; ++w) {
          const int ww = tile * WN + w;
          const float f = exp2f(sm[ww * 16 + rr] - M);
          L += sl[ww * 16 + rr] * f;
          const float2 v = *reinterpret_cast<const float2*>(so + (ww * 16 + rr) * DH + x);
          acc.x += v.x * f;
          acc.y += v.y * f;
        }
        const float inv = 1.f / L;
        const int head = h * G + (item.row0 + r) % G;
        const int xd = pass * DH + x;
        if (slot < 0) {
          T* dst = out + ((int64_t)qid * H + head) * D + xd;
          *reinterpret_cast<uint32_t*>(dst) = Vec2<T>::pack(acc.x * inv, acc.y * inv);
        } else {
          float* dst = part_o + ((int64_t)slot * H + head) * D + xd;
          *reinterpret_cast<float2*>(dst) = make_float2(acc.x * inv, acc.y * inv);
          if (pass == 0 && lane == 0) part_lse[(int64_t)slot * H + head] = M + log2f(L);
        }
      }
    }
    item = next_item;
    meta_qid = next_qid;
    meta_slot = next_slot;
  }
  PAT_SPAN_END(g_span_mma, 0);
}

// One warp per (query, head): fold the query's slots with online softmax
// (_merge_batch_into, attention.py:187-199); see pat_merge.cuh.
template <int D, typename T>
__global__ void __launch_bounds__(256, 3) merge_kernel(DevPlan plan, const float* __restrict__ part_o,
                                                    const float* __restrict__ part_lse, T* __restrict__ out) {
  // launched as a programmatic dependent of the forward (launch_merge): the
  // CTAs are resident when the forward drains.  The row count and this warp's
  // first descriptor (plan data) are fetched before waiting for its partials.
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nq = *plan.n_merge;
  const int4 md0 = gw < nq * plan.H ? __ldg(plan.merge_desc + gw / plan.H) : make_int4(0, 0, 0, 0);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  PAT_SPAN_BEGIN(g_span_mma, 1);
  merge_rows<D, T>(plan, part_o, part_lse, out, gw, (gridDim.x * blockDim.x) >> 5, nq, md0);
  PAT_SPAN_END(g_span_mma, 1);
}

#ifdef PAT_TC_TRACE
extern "C" int pat_debug_spans_mma(unsigned long long* host) {
  int e = (int)cudaMemcpyFromSymbol(host, g_span_mma, sizeof(g_span_mma));
  static unsigned long long zero[2][kSpanCtas][2];
  cudaMemcpyToSymbol(g_span_mma, zero, sizeof(zero));
  return e;
}
#endif

// ------------------------------------------------------------------------------------------
// launchers
// ------------------------------------------------------------------------------------------

template <int WM, int D, typename T>
static cudaError_t launch_fwd_t(const CUtensorMap& tmk, const CUtensorMap& tmv, const DevPlan& plan, int var,
                                int grid, const void* q, void* out, float* po, float* pl, float scale_log2,
                                cudaStream_t st) {
  constexpr int smem = StreamSmem<WM, D>::kAlloc;
  // the opt-in is per device; setting it on every launch is cheap and idempotent
  cudaError_t e = cudaFuncSetAttribute(fwd_stream_kernel<WM, D, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  fwd_stream_kernel<WM, D, T><<<grid, kStreamThreads, smem, st>>>(tmk, tmv, plan, var, (const T*)q, (T*)out, po,
                                                                  pl, scale_log2);
  return cudaGetLastError();
}

template <int D, typename T>
static cudaError_t launch_fwd_d(const CUtensorMap& tmk, const CUtensorMap& tmv, const DevPlan& plan, int var,
                                int grid, const void* q, void* out, float* po, float* pl, float scale_log2,
                                cudaStream_t st) {
  switch (var) {
    case VAR_R16: return launch_fwd_t<1, D, T>(tmk, tmv, plan, var, grid, q, out, po, pl, scale_log2, st);
    case VAR_R32: return launch_fwd_t<2, D, T>(tmk, tmv, plan, var, grid, q, out, po, pl, scale_log2, st);
    default: return launch_fwd_t<4, D, T>(tmk, tmv, plan, var, grid, q, out, po, pl, scale_log2, st);
  }
}

cudaError_t launch_forward_variant(const CUtensorMap& tmk, const CUtensorMap& tmv, const DevPlan& plan, int var,
                                   int grid, int dtype, int d, const void* q, void* out, float* po, float* pl,
                                   float scale_log2, cudaStream_t st) {
  if (dtype == PAT_DTYPE_F16) {
    if (d == 128) return launch_fwd_d<128, __half>(tmk, tmv, plan, var, grid, q, out, po, pl, scale_log2, st);
    return launch_fwd_d<64, __half>(tmk, tmv, plan, var, grid, q, out, po, pl, scale_log2, st);
  }
  if (d == 128) return launch_fwd_d<128, __nv_bfloat16>(tmk, tmv, plan, var, grid, q, out, po, pl, scale_log2, st);
  return launch_fwd_d<64, __nv_bfloat16>(tmk, tmv, plan, var, grid, q, out, po, pl, scale_log2, st);
}

template <int D, typename T>
static cudaError_t launch_merge_t(const DevPlan& plan, int grid, const float* po, const float* pl, void* out,
                                  cudaStream_t st) {
  // programmatic dependent launch: the merge grid is scheduled while the
  // forward drains (its CTAs block in griddepcontrol.wait until the forward
  // grid completed and flushed), hiding the launch gap between the two kernels
  // a persistent grid: at most the CTAs that are resident at once (warps loop
  // over rows), so no row waits for a second wave
  static std::atomic<int> resident[64];
  int dev = 0;
  cudaGetDevice(&dev);
  int cap = dev < 64 ? resident[dev].load(std::memory_order_relaxed) : 0;
  if (cap == 0) {
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, merge_kernel<D, T>, 256, 0);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cap = std::max(1, per_sm * sms);
    if (dev < 64) resident[dev].store(cap, std::memory_order_relaxed);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(std::min(grid, cap));
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, merge_kernel<D, T>, plan, po, pl, (T*)out);
}

cudaError_t launch_merge(const DevPlan& plan, int grid, int dtype, int d, const float* po, const float* pl,
                         void* out, cudaStream_t st) {
  if (dtype == PAT_DTYPE_F16)
    return d == 128 ? launch_merge_t<128, __half>(plan, grid, po, pl, out, st)
                    : launch_merge_t<64, __half>(plan, grid, po, pl, out, st);
  return d == 128 ? launch_merge_t<128, __nv_bfloat16>(plan, grid, po, pl, out, st)
                  : launch_merge_t<64, __nv_bfloat16>(plan, grid, po, pl, out, st);
}

}  // namespace pat
