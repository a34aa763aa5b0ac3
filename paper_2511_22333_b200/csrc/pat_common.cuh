// Shared definitions for the PAT (pack -> forward -> merge) native library.
#pragma once

#include <cstdint>
#include <cstddef>
#include <cuda_runtime.h>

#include "../../include/pat.h"

#define PAT_HD __host__ __device__ __forceinline__

namespace pat {

// Thread-local error message for pat_last_error().
void set_error(const char* fmt, ...);

// Rows view: row q is blk[row_begin(q) .. row_begin(q) + nblk[q]); the last
// block holds valid[q] tokens.  Either CSR (off != nullptr) or fixed stride.
struct RowsView {
  const int32_t* blk;
  const int64_t* off;   // CSR offsets (B+1) or nullptr
  int64_t stride;       // used when off == nullptr
  const int32_t* nblk;  // blocks per row
  const int32_t* valid; // valid tokens in the last block, in [1, bs]
  int B;
  int bs;

  PAT_HD int64_t row_begin(int q) const { return off ? off[q] : (int64_t)q * stride; }
  PAT_HD int32_t block(int q, int p) const { return blk[row_begin(q) + p]; }
  PAT_HD int32_t tokens_at(int q, int p) const { return p == nblk[q] - 1 ? valid[q] : bs; }
  PAT_HD bool same_unit(int q, int r, int p) const {
    return block(q, p) == block(r, p) && tokens_at(q, p) == tokens_at(r, p);
  }
  // tokens covered by positions [a, b) of row q
  PAT_HD int64_t span_tokens(int q, int a, int b) const {
    int64_t t = (int64_t)(b - a) * bs;
    if (b == nblk[q] && b > a) t -= (bs - valid[q]);
    return t;
  }
};

PAT_HD int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Debug builds (-DPAT_TC_TRACE, tools/layer_trace.py): per-CTA [start, end]
// globaltimer spans of a kernel, one array per translation unit.
#ifdef PAT_TC_TRACE
constexpr int kSpanCtas = 1024;
__device__ __forceinline__ unsigned long long pat_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define PAT_SPAN_BEGIN(arr, k)                                                \
  do {                                                                        \
    if (threadIdx.x == 0 && blockIdx.x < pat::kSpanCtas) arr[k][blockIdx.x][0] = pat::pat_gtime(); \
  } while (0)
#define PAT_SPAN_END(arr, k)                                                  \
  do {                                                                        \
    if ((threadIdx.x & 31) == 0 && blockIdx.x < pat::kSpanCtas)               \
      atomicMax(&arr[k][blockIdx.x][1], pat::pat_gtime());                    \
  } while (0)
#else
#define PAT_SPAN_BEGIN(arr, k) \
  do {                         \
  } while (0)
#define PAT_SPAN_END(arr, k) \
  do {                       \
  } while (0)
#endif

}  // namespace pat
