// Microbenchmark: stream a paged KV cache [blocks][16][KVH][128] bf16 (c5-like,
// 65536 blocks, random block order) into shared memory with different copy
// engines / box shapes and report GB/s.  No compute: measures the delivery rate
// available to the narrow-pack streaming kernel.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o kv_stream_probe tools/kv_stream_probe.cu
//   ./kv_stream_probe
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int BS = 16, KVH = 8, D = 128;

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
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma4(uint32_t dst, const void* m, uint32_t bar, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n"
               ::"r"(dst), "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar) : "memory");
}
__device__ __forceinline__ void tma5(uint32_t dst, const void* m, uint32_t bar, int c0, int c1, int c2, int c3, int c4) {
  asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n"
               ::"r"(dst), "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar) : "memory");
}

// mode 0: 4D box (64 d, 1 head, 16 tok, 1 blk) x 2 halves  = 2 KB / op
// mode 1: 5D box (64 d_lo, 16 tok, 2 d_hi, 1 head, 1 blk)  = 4 KB / op
// mode 2: 5D box (64 d_lo, 16 tok, 2 d_hi, HPC heads, 1)    = 4*HPC KB / op (HPC heads per item)
// Each item: one head group, `pages` pages of K and V.  Stage = 4 pages.
template <int MODE, int HPC, int NS>
__global__ void __launch_bounds__(160, 1) tma_stream(const __grid_constant__ CUtensorMap mk, const __grid_constant__ CUtensorMap mv,
                                                     const int* blocks, int pages_per_item, int n_items, int* sink) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm);
  constexpr int STAGE = 4 * 4096 * HPC * 2;  // 4 pages x (16 tok x 256 B) x heads x (K,V)
  const uint32_t full0 = sb + NS * STAGE, empty0 = full0 + NS * 8;
  int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) { mbar_init(full0 + 8 * s, 1); mbar_init(empty0 + 8 * s, 4); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int nst = pages_per_item / 4;
  if (warp == 4) {
    if (lane == 0) {
      uint32_t g = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int hg = it % (KVH / HPC);
        const int* bl = blocks + (it / (KVH / HPC)) * pages_per_item;
        for (int st = 0; st < nst; ++st, ++g) {
          int s = g % NS;
          mbar_wait(empty0 + 8 * s, ((g / NS) & 1) ^ 1);
          mbar_expect_tx(full0 + 8 * s, STAGE);
          uint32_t dk = sb + s * STAGE, dv = dk + STAGE / 2;
          for (int pg = 0; pg < 4; ++pg) {
            int blk = bl[st * 4 + pg];
            if (MODE == 0) {
              for (int hh = 0; hh < HPC; ++hh)
                for (int kb = 0; kb < 2; ++kb) {
                  uint32_t o = ((pg * HPC + hh) * 2 + kb) * 2048;
                  tma4(dk + o, &mk, full0 + 8 * s, kb * 64, hg * HPC + hh, 0, blk);
                  tma4(dv + o, &mv, full0 + 8 * s, kb * 64, hg * HPC + hh, 0, blk);
                }
            } else {
              uint32_t o = pg * HPC * 4096;
              tma5(dk + o, &mk, full0 + 8 * s, 0, 0, 0, hg * HPC, blk);
              tma5(dv + o, &mv, full0 + 8 * s, 0, 0, 0, hg * HPC, blk);
            }
          }
        }
      }
    }
    return;
  }
  uint32_t g = 0;
  int acc = 0;
  for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
    for (int st = 0; st < nst; ++st, ++g) {
      int s = g % NS;
      mbar_wait(full0 + 8 * s, (g / NS) & 1);
      acc += sm[s * STAGE + threadIdx.x * 16];
      __syncwarp();
      if (lane == 0) mbar_arrive(empty0 + 8 * s);
    }
  }
  if (acc == 123456789) sink[0] = acc;
}

// cp.async 16B per thread, 2 CTAs/SM style (NS stages of 4 pages), block ids in smem
template <int NS>
__global__ void __launch_bounds__(128, 2) cpasync_stream(const uint16_t* kc, const uint16_t* vc, const int* blocks, int pages_per_item,
                                                       int n_items, int* sink) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm);
  constexpr int STAGE = 4 * 4096 * 2;
  int* sblk = (int*)(sm + NS * STAGE);
  const int nst = pages_per_item / 4;
  int acc = 0;
  for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
    const int h = it % KVH;
    const int* bl = blocks + (it / KVH) * pages_per_item;
    __syncthreads();
    for (int i = threadIdx.x; i < pages_per_item; i += 128) sblk[i] = bl[i];
    __syncthreads();
    auto load = [&](int st) {
      if (st < nst) {
        uint32_t dk = sb + (st % NS) * STAGE, dv = dk + STAGE / 2;
        for (int i = 0; i < 8; ++i) {
          int c = threadIdx.x + i * 128;  // 1024 chunks of 16B per K
          int t = c / 16, ch = c % 16;
          int blk = sblk[st * 4 + t / 16];
          size_t off = (((size_t)blk * BS + t % 16) * KVH + h) * D + ch * 8;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dk + c * 16), "l"(kc + off));
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dv + c * 16), "l"(vc + off));
        }
      }
      asm volatile("cp.async.commit_group;\n");
    };
    for (int s = 0; s < NS - 1; ++s) load(s);
    for (int st = 0; st < nst; ++st) {
      asm volatile("cp.async.wait_group %0;\n" ::"n"(NS - 2));
      __syncthreads();
      load(st + NS - 1);
      acc += sm[(st % NS) * STAGE + threadIdx.x * 16];
    }
    asm volatile("cp.async.wait_group 0;\n");
  }
  if (acc == 123456789) sink[0] = acc;
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  return (PFN_cuTensorMapEncodeTiled_v12000)p;
}

int main() {
  const int NB = 65536, PAGES = 256;  // c5: 256 queries x 4096 tokens
  size_t elems = (size_t)NB * BS * KVH * D;
  uint16_t *kc, *vc;
  CK(cudaMalloc(&kc, elems * 2));
  CK(cudaMalloc(&vc, elems * 2));
  {
    // random bf16 bit patterns (finite): a zero-filled cache streams faster than real data
    std::vector<uint16_t> h(elems);
    std::mt19937 rng(1);
    for (size_t i = 0; i < elems; ++i) h[i] = (uint16_t)((rng() & 0x7fff) | 0x3c00) & 0xbfff;
    CK(cudaMemcpy(kc, h.data(), elems * 2, cudaMemcpyHostToDevice));
    for (size_t i = 0; i < elems; ++i) h[i] = (uint16_t)((rng() & 0x7fff) | 0x3c00) & 0xbfff;
    CK(cudaMemcpy(vc, h.data(), elems * 2, cudaMemcpyHostToDevice));
  }
  std::vector<int> blocks(NB);
  for (int i = 0; i < NB; ++i) blocks[i] = i;
  int* dblk;
  CK(cudaMalloc(&dblk, NB * 4));
  CK(cudaMemcpy(dblk, blocks.data(), NB * 4, cudaMemcpyHostToDevice));
  int* sink;
  CK(cudaMalloc(&sink, 4));
  void* flush;
  CK(cudaMalloc(&flush, 512 << 20));
  auto E = enc();
  CUtensorMap m4k, m4v, m5k, m5v;
  {
    cuuint64_t dims[4] = {D, KVH, BS, (cuuint64_t)NB};
    cuuint64_t str[3] = {D * 2, KVH * D * 2, BS * KVH * D * 2};
    cuuint32_t box[4] = {64, 1, 16, 1}, es[4] = {1, 1, 1, 1};
    CUtensorMapL2promotion prom = getenv("PROMO") ? (CUtensorMapL2promotion)atoi(getenv("PROMO")) : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    E(&m4k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, kc, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, prom, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    E(&m4v, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, vc, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, prom, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  auto mk5 = [&](CUtensorMap* m, void* base, int hpc) {
    // dims: d_lo(64), tok(16), d_hi(2), head(KVH), block
    cuuint64_t dims[5] = {64, BS, 2, KVH, (cuuint64_t)NB};
    cuuint64_t str[4] = {KVH * D * 2, 128, D * 2, BS * KVH * D * 2};
    cuuint32_t box[5] = {64, 16, 2, (cuuint32_t)hpc, 1}, es[5] = {1, 1, 1, 1, 1};
    CUresult r = E(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) printf("encode5 failed %d\n", r);
  };
  int nsm = 148;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const double bytes = 2.0 * elems * 2;
  auto timeit = [&](const char* name, auto launch) {
    float best = 1e9;
    for (int r = 0; r < 4; ++r) {
      CK(cudaMemset(flush, r, 512 << 20));
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (r) best = std::min(best, ms);
    }
    CK(cudaGetLastError());
    printf("%-44s %8.1f us  %7.1f GB/s\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9);
  };
#define TMA_CASE(MODE, HPC, NS, NAME)                                                                   \
  {                                                                                                     \
    int smem = NS * 4 * 4096 * HPC * 2 + 2 * NS * 8 + 2048;                                              \
    CK(cudaFuncSetAttribute(tma_stream<MODE, HPC, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); \
    int n_items = 256 * (KVH / HPC);                                                                    \
    if (MODE == 2 || MODE == 1) { mk5(&m5k, kc, HPC); mk5(&m5v, vc, HPC); }                              \
    const CUtensorMap& K = MODE ? m5k : m4k; const CUtensorMap& V = MODE ? m5v : m4v;                   \
    timeit(NAME, [&] { tma_stream<MODE, HPC, NS><<<nsm, 160, smem>>>(K, V, dblk, PAGES, n_items, sink); }); \
  }
  TMA_CASE(0, 1, 5, "TMA 4D 2KB box, 1 head/item, 5 stages");
  TMA_CASE(0, 1, 6, "TMA 4D 2KB box, 1 head/item, 6 stages");
  TMA_CASE(1, 1, 5, "TMA 5D 4KB box, 1 head/item, 5 stages");
  TMA_CASE(1, 1, 6, "TMA 5D 4KB box, 1 head/item, 6 stages");
  TMA_CASE(2, 2, 3, "TMA 5D 8KB box, 2 heads/item, 3 stages");
  TMA_CASE(2, 2, 2, "TMA 5D 8KB box, 2 heads/item, 2 stages");
  TMA_CASE(2, 4, 1, "TMA 5D 16KB box, 4 heads/item, 1 stage");
  {
    int smem = 3 * 4 * 4096 * 2 + 4096 + 1024;
    CK(cudaFuncSetAttribute(cpasync_stream<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    timeit("cp.async 16B, 2 CTA/SM, 3 stages", [&] { cpasync_stream<3><<<2 * nsm, 128, smem>>>(kc, vc, dblk, PAGES, 256 * KVH, sink); });
    smem = 6 * 4 * 4096 * 2 + 4096 + 1024;
    CK(cudaFuncSetAttribute(cpasync_stream<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    timeit("cp.async 16B, 1 CTA/SM, 6 stages", [&] { cpasync_stream<6><<<nsm, 128, smem>>>(kc, vc, dblk, PAGES, 256 * KVH, sink); });
  }
  return 0;
}
