// Micro-benchmark of the tcgen05 resources the 128-row forward tiles share
// (one CTA, clock64): MMA rate for A in TMEM (TS) vs shared memory (SS) at
// M = 128 and N = 32 / 64 / 128, tcgen05.ld throughput (32x32b.x32, 4 and 8
// warps), and MMAs running while the warps load.  A debugging tool:
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2511_22333_b200/csrc \
//        tools/tmem_bench.cu -o tools/tmem_bench && tools/tmem_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "pat_sm100.cuh"

using namespace pat::sm100;

constexpr int kIters = 512;

struct Res {
  long long mma_cyc;
  long long ld_cyc[8];
};

// mode bits: 1 = run MMAs (warp 0 issues), 2 = warps load TMEM, 4 = A from smem (SS),
// 8 / 16 = rotate over 2 / 4 independent accumulators (N <= 64)
template <int N, int M = 128, int BMN = 0>
__global__ void __launch_bounds__(256, 1) bench(int mode, int ld_warps, Res* res, int issuers = 1) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sb = smem_u32(smem);
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bars[4];
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(smem_u32(&bars[i]), 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(smem_u32(&tslot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tslot;
  // TMEM: D at columns [0, N), A (TS) at [256, 320), loads from [384, 416)
  constexpr uint32_t idesc = umma_idesc_f16(M, N, 1, BMN);
  if (warp < issuers && (mode & 1)) {
    const uint32_t bar = smem_u32(&bars[warp]);
    const uint32_t dbase = (uint32_t)warp * 64u;  // issuer w: its own accumulator columns
    const long long t0 = clock64();
    if (elect_one()) {
      for (int i = 0; i < kIters; ++i) {
        const int k = i & 7;
        const uint64_t bd = umma_desc_sw128(sb + 32768u + (uint32_t)((k & 3) * 32 + (k >> 2) * 32768), 16, 1024);
        const int nacc = (mode & 16) ? 4 : (mode & 8) ? 2 : 1;
        const uint32_t dcol = issuers > 1 ? dbase : (uint32_t)((i % nacc) * N);
        if (mode & 4) {
          const uint64_t ad = umma_desc_sw128(sb + (uint32_t)((k & 3) * 32 + (k >> 2) * 16384), 16, 1024);
          umma_f16_ss(tm + dcol, ad, bd, idesc, i >= nacc ? 1u : 0u);
        } else {
          umma_f16_ts(tm + dcol, tm + 256u + (uint32_t)(k * 8), bd, idesc, i >= nacc ? 1u : 0u);
        }
      }
      umma_commit(bar);
    }
    __syncwarp();
    mbar_wait(bar, 0);
    const long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) atomicMax((unsigned long long*)&res->mma_cyc, (unsigned long long)(t1 - t0));
  }
  if ((mode & 2) && warp >= 4 - (ld_warps > 4 ? 4 : 0) && warp < 4 + ld_warps) {
    // warps 4.. (and 0-3 when 8 load): quarter = warp & 3
    const uint32_t ta = tm + 384u + ((uint32_t)((warp & 3) * 32) << 16);
    uint32_t r[32], acc = 0;
    const long long t0 = clock64();
    for (int i = 0; i < kIters; ++i) {
      tmem_ld32(ta, r);  // includes wait::ld
#pragma unroll
      for (int j = 0; j < 32; ++j) acc += r[j];
    }
    const long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) res->ld_cyc[warp] = t1 - t0 + (acc == 12345 ? 1 : 0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tm);
  }
}

template <int N, int M = 128, int BMN = 0>
void run(const char* name, int mode, int ld_warps, int issuers = 1) {
  Res* d;
  cudaMalloc(&d, sizeof(Res));
  cudaMemset(d, 0, sizeof(Res));
  const int smem = 32768 + 65536 + 1024;
  cudaFuncSetAttribute(bench<N, M, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int w = 0; w < 3; ++w) { cudaMemset(d, 0, sizeof(Res)); bench<N, M, BMN><<<1, 256, smem>>>(mode, ld_warps, d, issuers); }
  cudaError_t e = cudaDeviceSynchronize();
  Res h;
  cudaMemcpy(&h, d, sizeof(Res), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) {
    printf("%s: %s\n", name, cudaGetErrorString(e));
    return;
  }
  printf("%-34s", name);
  if (mode & 1) {
    const double per = (double)h.mma_cyc / kIters / issuers;
    const double floor = 128.0 * N / 256.0;
    (void)M;
    printf(" mma %6.1f cyc (floor %5.1f)  A+B operand bytes/cyc %6.1f", per, floor, (4096.0 + N * 32.0) / per);
  }
  if (mode & 2) {
    long long mx = 0;
    for (int w = 0; w < 8; ++w) mx = h.ld_cyc[w] > mx ? h.ld_cyc[w] : mx;
    const double per = (double)mx / kIters;
    printf(" ld32 x%d warps: %6.1f cyc/iter  %6.1f B/cyc", ld_warps, per, ld_warps * 4096.0 / per);
  }
  printf("\n");
}

int main() {
  run<32>("TS N=32", 1, 0);
  run<64>("TS N=64", 1, 0);
  run<128>("TS N=128", 1, 0);
  run<256>("TS N=256", 1, 0);
  run<32>("SS N=32", 5, 0);
  run<64>("SS N=64", 5, 0);
  run<128>("SS N=128", 5, 0);
  run<32>("ld only", 2, 4);
  run<32>("ld only", 2, 8);
  run<32>("TS N=32 + ld", 3, 4);
  run<128>("TS N=128 + ld", 3, 4);
  run<32>("TS N=32 2 acc", 9, 0);
  run<32>("TS N=32 4 acc", 17, 0);
  run<64>("TS N=64 2 acc", 9, 0);
  run<64>("TS N=64 4 acc", 17, 0);
  run<32>("SS N=32 2 acc", 13, 0);
  run<32>("SS N=32 4 acc", 21, 0);
  run<64>("SS N=64 4 acc", 21, 0);
  run<16, 128>("TS M=128 N=16", 1, 0);
  run<16, 128>("SS M=128 N=16", 5, 0);
  run<32, 64>("TS M=64 N=32", 1, 0);
  run<128, 64>("TS M=64 N=128", 1, 0);
  run<32, 64>("SS M=64 N=32", 5, 0);
  run<128, 64>("SS M=64 N=128", 5, 0);
  run<16, 64>("SS M=64 N=16", 5, 0);
  run<128, 128, 1>("TS M=128 N=128 B MN-major", 1, 0);
  run<32, 128, 1>("TS M=128 N=32 B MN-major", 1, 0);
  run<32>("TS N=32 x2 issuers (per MMA)", 1, 0, 2);
  run<32>("TS N=32 x4 issuers (per MMA)", 1, 0, 4);
  run<64>("TS N=64 x2 issuers (per MMA)", 1, 0, 2);
  run<32>("SS N=32 x2 issuers (per MMA)", 5, 0, 2);
  run<32>("SS N=32 x4 issuers (per MMA)", 5, 0, 4);
  run<32>("SS N=32 + ld", 7, 4);
  run<64>("SS N=64 + ld", 7, 4);
  return 0;
}
