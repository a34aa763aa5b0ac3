// Microbenchmark: tcgen05.mma issue/execute rate for the decode kernel's shapes
// (kind::f16, cta_group::1, K=16 per instruction):
//   QK  SS  M=128 N=64   (A = Q tile K-major, B = K tile K-major, SW128)
//   PV  TS  M=128 N=128  (A = P from TMEM, B = V tile MN-major, SW128)
//   QK  SS  M=128 N=128
// One CTA per SM (grid = 148), one elected thread issues `reps` x `per` MMAs
// back to back and commits; reports cycles per MMA.  Operand contents are
// garbage (throughput only).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2511_22333_b200/csrc -o tools/mma_probe tools/mma_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "pat_sm100.cuh"

using namespace pat::sm100;

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e = (x);                                                   \
    if (e != cudaSuccess) {                                                \
      printf("%s: %s\n", #x, cudaGetErrorString(e));                       \
      exit(1);                                                             \
    }                                                                      \
  } while (0)

template <int MODE>
__global__ void __launch_bounds__(128, 1) probe(int reps, long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sb = smem_u32(sm);
  const uint32_t bar = sb + 96 * 1024;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(smem_u32(&tslot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    constexpr uint32_t id_qk64 = umma_idesc_f16(128, 64, 1, 0);
    constexpr uint32_t id_qk128 = umma_idesc_f16(128, 128, 1, 0);
    constexpr uint32_t id_pv = umma_idesc_f16(128, 128, 1, 1);
    t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int kb = k >> 2, kk = k & 3;
        if (MODE == 0) {
          uint64_t a = umma_desc_sw128(sb + kb * 16384 + kk * 32, 16, 1024);
          uint64_t b = umma_desc_sw128(sb + 32768 + kb * 8192 + kk * 32, 16, 1024);
          umma_f16_ss(tmem, a, b, id_qk64, 1u);
        } else if (MODE == 1) {
          uint64_t b = umma_desc_sw128(sb + 49152 + (k & 3) * 16 * 128, 64 * 128, 1024);
          umma_f16_ts(tmem + 256, tmem + 128 + k * 8, b, id_pv, 1u);
        } else if (MODE == 2) {
          uint64_t a = umma_desc_sw128(sb + kb * 16384 + kk * 32, 16, 1024);
          uint64_t b = umma_desc_sw128(sb + 32768 + kb * 16384 + kk * 32, 16, 1024);
          umma_f16_ss(tmem, a, b, id_qk128, 1u);
        } else if (MODE == 3) {
          uint64_t b = umma_desc_sw128(sb + 49152 + (k & 3) * 16 * 128, 64 * 128, 1024);
          umma_f16_ts(tmem + 256, tmem + 128 + k * 8, b, umma_idesc_f16(64, 128, 1, 1), 1u);
        } else if (MODE == 4) {
          uint64_t a = umma_desc_sw128(sb + kb * 16384 + kk * 32, 16, 1024);
          uint64_t b = umma_desc_sw128(sb + 32768 + kb * 8192 + kk * 32, 16, 1024);
          umma_f16_ss(tmem, a, b, umma_idesc_f16(64, 64, 1, 0), 1u);
        } else {
          uint64_t a = umma_desc_sw128(sb + kb * 16384 + kk * 32, 16, 1024);
          uint64_t b = umma_desc_sw128(sb + 49152 + (k & 3) * 16 * 128, 64 * 128, 1024);
          umma_f16_ss(tmem + 256, a, b, umma_idesc_f16(64, 128, 1, 1), 1u);
        }
      }
    }
    umma_commit(bar);
    mbar_wait(bar, 0);
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int MODE>
void run(const char* name, int grid) {
  long long* d;
  CK(cudaMalloc(&d, grid * sizeof(long long)));
  const int smem = 100 * 1024;
  CK(cudaFuncSetAttribute(probe<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  for (int reps : {1, 4, 64}) {
    probe<MODE><<<grid, 128, smem>>>(reps, d);
    CK(cudaDeviceSynchronize());
    long long h[148];
    CK(cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost));
    double mx = 0, mean = 0;
    for (int i = 0; i < grid; ++i) {
      mx = h[i] > mx ? h[i] : mx;
      mean += h[i];
    }
    mean /= grid;
    printf("%-22s grid %3d reps %3d: %8.0f cycles total, %6.1f cycles/MMA (mean), %6.1f (max)\n", name, grid, reps,
           mean, mean / (reps * 8), mx / (reps * 8));
  }
  CK(cudaFree(d));
}

int main() {
  for (int grid : {1, 148}) {
    run<0>("QK SS M128 N64", grid);
    run<1>("PV TS M128 N128", grid);
    run<2>("QK SS M128 N128", grid);
    run<4>("QK SS M64 N64", grid);
    run<5>("PV SS M64 N128", grid);
    run<3>("PV TS M64 N128", grid);
  }
  return 0;
}
