// GPU pack scheduler: pack_batch (packer.py:224-242) as a pass of data-parallel
// kernels over DEVICE block tables (vLLM layout: block_tables[B][stride],
// seq_lens[B]).  Same formulation as the host packer (pat_packer_host.cpp):
//   K1 rows      : blocks / valid tokens per row, validation (InvalidSpec)
//   K2 dup       : repeated block id inside a row (one CTA per row, smem sort)
//   K3 lcp       : pairwise longest common prefix over (block, tokens) units
//   K4 levels    : per query, the sorted distinct lcp values = its internal
//                  node ends; node sizes, minimum member, terminal counts
//   K5 decide    : TreeHeuristic replayed along each query's own path
//                  (merge iff 2*(s_c + terminal_c) > span, packer.py:153)
//   K6 rank      : DFS rank pi(q) = lexicographic rank of the child-slot key
//   K7 nodes     : node ids (owned by their minimum query), subtree pi range,
//                  member counts
//   K8 order     : pack emission order = (last pi in subtree, deeper first)
//   K9 members   : queries inside a pack in pi order, produces_partial
// Output (device): packs as (rep query, first block, end block, kv_len,
// query list, partial) in reference order; bit-exact with pack_batch.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <mutex>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "pat_plan_host.h"

namespace pat {
namespace dev {

struct Ws {
  // inputs
  const int32_t* bt;
  int64_t stride;
  const int32_t* seq;
  int B, bs, maxb, D;  // D = level capacity per query
  const int32_t* run;  // device flag: the table changed, re-plan (nullptr = always run)
  // per query
  int32_t* nblk;
  int32_t* valid;
  int32_t* err;     // [0] status, [1] row
  int32_t* lcp;     // [B*B]
  unsigned long long* hs;  // [B * hs_n] prefix hashes of each row's 32-position segments
  int hs_n;                // segments per row (ceil(maxb / 32))
  int32_t* K;       // internal levels
  int32_t* hasleaf;
  int32_t* end;     // [B*D]
  int32_t* nq;
  int32_t* minq;
  int32_t* term;
  int32_t* start;   // [B*(D+1)] (levels incl. leaf)
  int32_t* stop;
  int32_t* span;
  int32_t* anchor;
  int32_t* member;
  int32_t* nmemb;   // [B]
  int32_t* k0;      // [B]
  int32_t* cnt_own; // [B]
  int32_t* pi;      // [B]
  int32_t* order;   // [B]
  int32_t* base;    // [B+1]
  // nodes [2B]
  int32_t* n_hi;
  int32_t* n_lo;
  int32_t* n_cnt;
  int32_t* n_depth;
  int32_t* n_rep;
  int32_t* n_a0;
  int32_t* n_a1;
  int32_t* n_span;
  int32_t* n_pack;
  // packs [2B]
  int32_t* npacks;  // [1]
  int32_t* p_node;
  int32_t* p_qoff;  // [2B+1]
  int32_t* p_q;     // [B*(D+1)]
  int32_t* p_partial;
};

// Exclusive prefix sum of one value per thread over the block (blockDim a
// multiple of 32, <= 1024): warp shuffles, then the 32 warp totals.  All
// threads must call it; *total gets the block sum.
__device__ __forceinline__ int block_excl_scan(int v, int* total) {
  __shared__ int wsum[32];
  __shared__ int s_total;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int z = lane < nw ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, z, o);
      if (lane >= o) z += y;
    }
    if (lane < nw) wsum[lane] = z;  // inclusive over warps
    if (lane == 31) s_total = z;
  }
  __syncthreads();
  const int r = x - v + (wid > 0 ? wsum[wid - 1] : 0);
  *total = s_total;
  __syncthreads();
  return r;
}

__device__ __forceinline__ int tok_at(const Ws& w, int q, int p) { return p == w.nblk[q] - 1 ? w.valid[q] : w.bs; }
__device__ __forceinline__ int blk_at(const Ws& w, int q, int p) { return w.bt[(int64_t)q * w.stride + p]; }

// Each phase is a __device__ function written for any grid (grid-stride /
// block-stride loops, block-uniform control flow), launched either as its own
// kernel (pat_plan_create_device) or inside the persistent planner kernel of
// the device decoder, separated by grid barriers.
#define PAT_GRID_LOOP(i, n) for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += gridDim.x * blockDim.x)

__device__ void ph_rows(const Ws& w) {
  PAT_GRID_LOOP(q, w.B) {
    int s = w.seq[q];
    int n = s > 0 ? (s + w.bs - 1) / w.bs : 0;
    w.nblk[q] = n;
    w.valid[q] = s - (n - 1) * w.bs;
    if (n <= 0 || n > w.maxb) {
      if (atomicCAS(&w.err[0], 0, PAT_ERR_INVALID_SPEC) == 0) w.err[1] = q;
    }
  }
}
__global__ void k_rows(Ws w) {
  if (w.run && !*w.run) return;
  ph_rows(w);
}

__device__ __forceinline__ uint64_t lcp_mix(uint64_t z) {  // splitmix64 finaliser
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// hash term of (position, block id, tokens) of a row
__device__ __forceinline__ uint64_t lcp_term(const Ws& w, int q, int p) {
  return lcp_mix(lcp_mix(((uint64_t)(uint32_t)p << 32) | (uint32_t)blk_at(w, q, p)) + (uint64_t)(uint32_t)tok_at(w, q, p));
}

// one CTA per row: the row's segment prefix hashes (for the LCP phase), then a
// bitonic sort of its block ids in smem, adjacent compare
__device__ void ph_dup(const Ws& w, int32_t* sbuf) {
  for (int q = blockIdx.x; q < w.B; q += gridDim.x) {
  const int n = min(w.nblk[q], w.maxb);
  {
    // hs[q][s] = sum of the terms of positions [0, 32 (s + 1)) (order-free sum
    // of position-keyed terms: equal prefixes give equal values)
    const int S = (n + 31) / 32, lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    unsigned long long* seg = reinterpret_cast<unsigned long long*>(sbuf);
    for (int sg = wid; sg < S; sg += nw) {
      const int p = 32 * sg + lane;
      uint64_t x = p < n ? lcp_term(w, q, p) : 0;
#pragma unroll
      for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane == 0) seg[sg] = x;
    }
    __syncthreads();
    if (wid == 0) {
      uint64_t carry = 0;
      for (int s0 = 0; s0 < S; s0 += 32) {
        uint64_t x = s0 + lane < S ? seg[s0 + lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (s0 + lane < S) w.hs[(int64_t)q * w.hs_n + s0 + lane] = x + carry;
        carry += __shfl_sync(0xffffffffu, x, 31);
      }
    }
    __syncthreads();
  }
  if (n <= 1) continue;
  int P = 1;
  while (P < n) P <<= 1;
  for (int i = threadIdx.x; i < P; i += blockDim.x) sbuf[i] = i < n ? blk_at(w, q, i) : 0x7fffffff;
  __syncthreads();
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        int l = i ^ j;
        if (l > i) {
          bool up = (i & k) == 0;
          int a = sbuf[i], b = sbuf[l];
          if ((a > b) == up) {
            sbuf[i] = b;
            sbuf[l] = a;
          }
        }
      }
      __syncthreads();
    }
  for (int i = threadIdx.x; i + 1 < n; i += blockDim.x)
    if (sbuf[i] == sbuf[i + 1]) {
      if (atomicCAS(&w.err[0], 0, PAT_ERR_INVALID_SPEC) == 0) w.err[1] = q;
    }
  __syncthreads();
  }
}
__global__ void k_dup(Ws w) {
  if (w.run && !*w.run) return;
  extern __shared__ int32_t sbuf[];
  ph_dup(w, sbuf);
}

// one warp per (q, r) pair with q < r
__device__ void ph_lcp(const Ws& w) {
  const int lane = threadIdx.x & 31;
  const int64_t npairs = (int64_t)w.B * w.B;
  for (int64_t pr = (int64_t)(blockIdx.x * blockDim.x + threadIdx.x) / 32; pr < npairs;
       pr += (int64_t)gridDim.x * blockDim.x / 32) {
    const int q = (int)(pr / w.B), r = (int)(pr % w.B);
    if (r < q) continue;
    if (r == q) {
      if (lane == 0) w.lcp[(int64_t)q * w.B + q] = w.nblk[q];
      continue;
    }
    const int n = min(w.nblk[q], w.nblk[r]);
    // coarse: the first 32-position segment whose prefix hashes differ (the
    // segments before the last one lie inside both rows); then position by
    // position from there (a hash difference the positions do not confirm
    // cannot happen, but would only make the scan continue)
    const int S = (n + 31) / 32;
    int s_first = S > 0 ? S - 1 : 0;
    const unsigned long long* hq = w.hs + (int64_t)q * w.hs_n;
    const unsigned long long* hr = w.hs + (int64_t)r * w.hs_n;
    for (int s0 = 0; s0 < S - 1; s0 += 32) {
      const int sg = s0 + lane;
      const unsigned m = __ballot_sync(0xffffffffu, sg < S - 1 && hq[sg] != hr[sg]);
      if (m) {
        s_first = s0 + __ffs(m) - 1;
        break;
      }
    }
    int l = n;
    for (int p0 = 32 * s_first; p0 < n; p0 += 32) {
      const int p = p0 + lane;
      bool diff = false;
      if (p < n) diff = blk_at(w, q, p) != blk_at(w, r, p) || tok_at(w, q, p) != tok_at(w, r, p);
      unsigned m = __ballot_sync(0xffffffffu, diff);
      if (m) {
        l = p0 + __ffs(m) - 1;
        break;
      }
    }
    if (lane == 0) w.lcp[(int64_t)q * w.B + r] = w.lcp[(int64_t)r * w.B + q] = l;
  }
}
__global__ void k_lcp(Ws w) {
  if (w.run && !*w.run) return;
  ph_lcp(w);
}

// one CTA per query: sort (lcp, r) keys, derive the internal levels
__device__ void ph_levels(const Ws& w, unsigned long long* skey) {
  for (int q = blockIdx.x; q < w.B; q += gridDim.x) {
  int P = 1;
  while (P < w.B) P <<= 1;
  const int32_t* L = w.lcp + (int64_t)q * w.B;
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    unsigned long long k = ~0ull;
    if (i < w.B && i != q && L[i] >= 1) k = ((unsigned long long)(unsigned)L[i] << 32) | (unsigned)i;
    skey[i] = k;
  }
  __syncthreads();
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        int l = i ^ j;
        if (l > i) {
          bool up = (i & k) == 0;
          unsigned long long a = skey[i], b = skey[l];
          if ((a > b) == up) {
            skey[i] = b;
            skey[l] = a;
          }
        }
      }
      __syncthreads();
    }
  // The sorted entries (lcp value v, query r) group into levels, one per
  // distinct v (ascending).  Everything per level is a parallel scan over the
  // entries: level index (inclusive count of group starts), members at or past
  // the level (M - start + 1), terminal members (r ends exactly at v, summed
  // per level) and the smallest member id (suffix minimum of r from the start).
  int32_t* tflag = reinterpret_cast<int32_t*>(skey + P);  // [P] terminal flag
  int32_t* lvl = tflag + P;                              // [P] level index (scan)
  int32_t* suf = lvl + P;                                // [P] suffix min of r
  int32_t* tcnt = suf + P;                               // [P] terminal count per level
  __shared__ int s_m;
  if (threadIdx.x == 0) s_m = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    const unsigned long long k = skey[i];
    const bool valid = k != ~0ull;
    const int v = (int)(k >> 32);
    tflag[i] = valid && w.nblk[(int)(k & 0xffffffffu)] == v;
    lvl[i] = valid && (i == 0 || (int)(skey[i - 1] >> 32) != v);
    suf[i] = valid ? (int)(k & 0xffffffffu) : 0x7fffffff;
    tcnt[i] = 0;
    if (valid) atomicAdd(&s_m, 1);
  }
  __syncthreads();
  const int M = s_m;
  for (int off = 1; off < P; off <<= 1) {  // inclusive scan (levels), suffix min (members)
    int a[4], m[4];
    int n = 0;
    for (int i = threadIdx.x; i < P; i += blockDim.x, ++n) {
      if (n < 4) {
        a[n] = i >= off ? lvl[i - off] : 0;
        m[n] = i + off < P ? suf[i + off] : 0x7fffffff;
      }
    }
    __syncthreads();
    n = 0;
    for (int i = threadIdx.x; i < P; i += blockDim.x, ++n) {
      if (n < 4) {
        lvl[i] += a[n];
        suf[i] = min(suf[i], m[n]);
      }
    }
    __syncthreads();
  }
  const int Kq = M > 0 ? lvl[M - 1] : 0;
  const bool over = Kq > w.D;
  const int nbq = w.nblk[q];
  for (int i = threadIdx.x; i < M; i += blockDim.x)
    if (tflag[i]) atomicAdd(&tcnt[lvl[i] - 1], 1);
  __syncthreads();
  if (over) {
    if (threadIdx.x == 0 && atomicCAS(&w.err[0], 0, PAT_ERR_NO_FEASIBLE_CONFIG) == 0) w.err[1] = q;
  } else {
    for (int i = threadIdx.x; i < M; i += blockDim.x) {
      const int v = (int)(skey[i] >> 32);
      if (i == 0 || (int)(skey[i - 1] >> 32) != v) {  // the first entry of level k
        const int k = lvl[i] - 1;
        w.end[(int64_t)q * w.D + k] = v;
        w.nq[(int64_t)q * w.D + k] = 1 + (M - i);
        w.term[(int64_t)q * w.D + k] = tcnt[k] + (nbq == v ? 1 : 0);
        w.minq[(int64_t)q * w.D + k] = min(q, suf[i]);
      }
    }
  }
  if (threadIdx.x == 0) {
    const int K = over ? 0 : Kq;
    w.K[q] = K;
    w.hasleaf[q] = K == 0 || (int)(skey[M - 1] >> 32) < nbq;
  }
  __syncthreads();
  }
}
__global__ void k_levels(Ws w) {
  if (w.run && !*w.run) return;
  extern __shared__ unsigned long long skey[];
  ph_levels(w, skey);
}

__device__ __forceinline__ int levels_of(const Ws& w, int q) { return w.K[q] + (w.hasleaf[q] ? 1 : 0); }
__device__ __forceinline__ int owner_of(const Ws& w, int q, int k) {
  return k < w.K[q] ? w.minq[(int64_t)q * w.D + k] : q;
}

__device__ __forceinline__ int64_t span_tokens(const Ws& w, int q, int a, int b) {
  int64_t t = (int64_t)(b - a) * w.bs;
  if (b == w.nblk[q] && b > a) t -= (w.bs - w.valid[q]);
  return t;
}

// thread per query: TreeHeuristic decisions along the path + ownership
__device__ void ph_decide(const Ws& w) {
  PAT_GRID_LOOP(q, w.B) {
  const int K = w.K[q], Lv = levels_of(w, q), D1 = w.D + 1;
  int span = 0, anchor = 0, nm = 0;
  for (int k = 0; k < Lv; ++k) {
    const int st = k == 0 ? 0 : w.end[(int64_t)q * w.D + k - 1];
    const int sp = k < K ? w.end[(int64_t)q * w.D + k] : w.nblk[q];
    const int tok = (int)span_tokens(w, q, st, sp);
    if (k == 0) {
      span = tok;
      anchor = 0;
    } else {
      const int s_c = k < K ? w.nq[(int64_t)q * w.D + k] : 1;
      const int t_c = k < K ? w.term[(int64_t)q * w.D + k] : 1;
      const bool merged = 2 * (int64_t)(s_c + t_c) > span;
      // the member flag of level k-1 depends on this decision
      w.member[(int64_t)q * D1 + k - 1] = merged ? 0 : 1;
      nm += merged ? 0 : 1;
      span = merged ? span + tok : tok;
      anchor = merged ? anchor : st;
    }
    w.start[(int64_t)q * D1 + k] = st;
    w.stop[(int64_t)q * D1 + k] = sp;
    w.span[(int64_t)q * D1 + k] = span;
    w.anchor[(int64_t)q * D1 + k] = anchor;
  }
  w.member[(int64_t)q * D1 + Lv - 1] = 1;
  w.nmemb[q] = nm + 1;
  int k0 = 0;
  while (k0 < Lv && owner_of(w, q, k0) != q) ++k0;
  w.k0[q] = k0;
  w.cnt_own[q] = Lv - k0;
  }
}
__global__ void k_decide(Ws w) {
  if (w.run && !*w.run) return;
  ph_decide(w);
}

// lexicographic key element e of query q: e=0 root group min, e=1+k slot at level k
__device__ __forceinline__ int key_at(const Ws& w, int q, int e) {
  const int K = w.K[q];
  if (e == 0) return K > 0 ? w.minq[(int64_t)q * w.D] : q;
  const int k = e - 1;
  if (w.end[(int64_t)q * w.D + k] == w.nblk[q]) return q;
  return w.B + (k + 1 < K ? w.minq[(int64_t)q * w.D + k + 1] : q);
}

// warp per query: pi(q) = #{r : key(r) < key(q)}
__device__ void ph_rank(const Ws& w) {
  const int lane = threadIdx.x & 31;
  for (int q = (blockIdx.x * blockDim.x + threadIdx.x) / 32; q < w.B; q += gridDim.x * blockDim.x / 32) {
  const int lq = w.K[q] + 1;
  int cnt = 0;
  for (int r = lane; r < w.B; r += 32) {
    if (r == q) continue;
    const int lr = w.K[r] + 1;
    int e = 0;
    int less = 0;
    for (;; ++e) {
      if (e == lq || e == lr) {
        less = lr < lq;  // a proper prefix sorts first (never happens for distinct keys)
        break;
      }
      const int a = key_at(w, r, e), b = key_at(w, q, e);
      if (a != b) {
        less = a < b;
        break;
      }
    }
    cnt += less;
  }
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if (lane == 0) {
    w.pi[q] = cnt;
    w.order[cnt] = q;
  }
  }
}
__global__ void k_rank(Ws w) {
  if (w.run && !*w.run) return;
  ph_rank(w);
}

// single CTA exclusive scan of cnt_own -> base
__device__ void ph_scan_nodes(const Ws& w) {
  if (blockIdx.x != 0) return;  // one CTA of up to 1024 threads
  const int t = threadIdx.x, n = w.B;
  const int per = (n + blockDim.x - 1) / blockDim.x;
  int s = 0;
  for (int i = t * per; i < min(n, (t + 1) * per); ++i) s += w.cnt_own[i];
  int total;
  int acc = block_excl_scan(s, &total);
  if (t == 0) w.base[n] = total;
  for (int i = t * per; i < min(n, (t + 1) * per); ++i) {
    w.base[i] = acc;
    acc += w.cnt_own[i];
  }
}
__global__ void k_scan_nodes(Ws w) {
  if (w.run && !*w.run) return;
  ph_scan_nodes(w);
}

__device__ __forceinline__ int node_id(const Ws& w, int q, int k) {
  const int m = owner_of(w, q, k);
  return w.base[m] + k - w.k0[m];
}

__device__ void ph_nodes_init(const Ws& w) {
  const int N = w.base[w.B];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    w.n_hi[i] = 0;
    w.n_lo[i] = 0x7fffffff;
    w.n_cnt[i] = 0;
    w.n_pack[i] = -1;
  }
}
__global__ void k_nodes_init(Ws w) {
  if (w.run && !*w.run) return;
  ph_nodes_init(w);
}

// thread per query: every level it passes through
__device__ void ph_nodes(const Ws& w) {
  PAT_GRID_LOOP(q, w.B) {
  const int Lv = levels_of(w, q), D1 = w.D + 1;
  const int pq = w.pi[q];
  for (int k = 0; k < Lv; ++k) {
    const int id = node_id(w, q, k);
    atomicMax(&w.n_hi[id], pq + 1);
    atomicMin(&w.n_lo[id], pq);
    if (w.member[(int64_t)q * D1 + k]) atomicAdd(&w.n_cnt[id], 1);
    if (owner_of(w, q, k) == q) {
      w.n_depth[id] = k;
      w.n_rep[id] = q;
      w.n_a0[id] = w.anchor[(int64_t)q * D1 + k];
      w.n_a1[id] = w.stop[(int64_t)q * D1 + k];
      w.n_span[id] = w.span[(int64_t)q * D1 + k];
    }
  }
  }
}
__global__ void k_nodes(Ws w) {
  if (w.run && !*w.run) return;
  ph_nodes(w);
}

// thread per node: rank among emitting nodes by (hi asc, depth desc)
__device__ void ph_order(const Ws& w, int4* snode, int cap) {
  const int N = w.base[w.B];
  // (hi, depth, emitting) of every node, staged once per CTA when it fits
  const bool st = N <= cap;
  if (st) {
    for (int j = threadIdx.x; j < N; j += blockDim.x) snode[j] = make_int4(w.n_hi[j], w.n_depth[j], w.n_cnt[j] > 0, 0);
    __syncthreads();
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    if (w.n_cnt[i] == 0) continue;
    const int hi = w.n_hi[i], dp = w.n_depth[i];
    int r = 0;
    for (int j = 0; j < N; ++j) {
      const int4 nj = st ? snode[j] : make_int4(w.n_hi[j], w.n_depth[j], w.n_cnt[j] > 0, 0);
      if (j == i || !nj.z) continue;
      r += (nj.x < hi) || (nj.x == hi && nj.y > dp);
    }
    w.n_pack[i] = r;
    w.p_node[r] = i;
    atomicAdd(w.npacks, 1);
  }
}
__global__ void k_order(Ws w) {
  if (w.run && !*w.run) return;
  ph_order(w, nullptr, 0);
}

// single thread: query offsets per pack (packs <= 2B)
// CTA 0: exclusive scan of the packs' member counts (any block size)
__device__ void ph_pack_offsets(const Ws& w) {
  if (blockIdx.x != 0) return;
  const int np = *w.npacks, t = threadIdx.x, nt = blockDim.x;
  const int per = (np + nt - 1) / nt;
  int sum = 0;
  for (int p = t * per; p < min(np, (t + 1) * per); ++p) sum += w.n_cnt[w.p_node[p]];
  int total;
  int acc = block_excl_scan(sum, &total);
  if (t == 0) w.p_qoff[np] = total;
  for (int p = t * per; p < min(np, (t + 1) * per); ++p) {
    w.p_qoff[p] = acc;
    acc += w.n_cnt[w.p_node[p]];
    w.p_partial[p] = 0;
  }
}
__global__ void k_pack_offsets(Ws w) {
  if (w.run && !*w.run) return;
  ph_pack_offsets(w);
}

// thread per query: place it in each pack it belongs to, in pi order
__device__ void ph_members(const Ws& w) {
  PAT_GRID_LOOP(q, w.B) {
  const int Lv = levels_of(w, q), D1 = w.D + 1;
  const int pq = w.pi[q];
  for (int k = 0; k < Lv; ++k) {
    if (!w.member[(int64_t)q * D1 + k]) continue;
    const int id = node_id(w, q, k);
    const int p = w.n_pack[id];
    int pos = 0;
    for (int i = w.n_lo[id]; i < pq; ++i) {
      const int r = w.order[i];
      // r lies in this node's subtree (pi range is contiguous), so its level-k node is id
      pos += w.member[(int64_t)r * D1 + k];
    }
    w.p_q[w.p_qoff[p] + pos] = q;
    if (w.nmemb[q] > 1) atomicOr(&w.p_partial[p], 1);
  }
  }
}
__global__ void k_members(Ws w) {
  if (w.run && !*w.run) return;
  ph_members(w);
}

}  // namespace dev

// Runs the GPU pass and returns the packs on the host (block ids gathered from a
// host copy of the table).  One synchronisation: the pack count is needed to
// size the schedule.
int device_pack(const int32_t* d_bt, int64_t stride, const int32_t* d_seq, int B, int maxb, int bs,
                cudaStream_t st, HostPacks* out, std::vector<int32_t>* h_nblk, std::vector<int32_t>* h_valid,
                std::vector<int32_t>* h_rows) {
  out->clear();
  if (B == 0) return PAT_OK;
  if (B > 4096) {
    set_error("device packer supports up to 4096 queries (got %d)", B);
    return PAT_ERR_NO_FEASIBLE_CONFIG;
  }
  const int D = std::min(B, maxb + 1) + 1;
  const int D1 = D + 1;
  // one arena for the whole workspace
  std::vector<std::pair<int32_t**, size_t>> fields;
  dev::Ws w{};
  w.bt = d_bt;
  w.stride = stride;
  w.seq = d_seq;
  w.B = B;
  w.bs = bs;
  w.maxb = maxb;
  w.D = D;
  const size_t BB = (size_t)B * B, BD = (size_t)B * D, BD1 = (size_t)B * D1, N2 = 2 * (size_t)B + 2;
  w.hs_n = (maxb + 31) / 32;
  fields = {{&w.nblk, (size_t)B}, {&w.valid, (size_t)B}, {&w.err, 2}, {&w.lcp, BB},
            {reinterpret_cast<int32_t**>(&w.hs), (size_t)B * w.hs_n * 2}, {&w.K, (size_t)B},
            {&w.hasleaf, (size_t)B}, {&w.end, BD}, {&w.nq, BD}, {&w.minq, BD}, {&w.term, BD},
            {&w.start, BD1}, {&w.stop, BD1}, {&w.span, BD1}, {&w.anchor, BD1}, {&w.member, BD1},
            {&w.nmemb, (size_t)B}, {&w.k0, (size_t)B}, {&w.cnt_own, (size_t)B}, {&w.pi, (size_t)B},
            {&w.order, (size_t)B}, {&w.base, (size_t)B + 1}, {&w.n_hi, N2}, {&w.n_lo, N2}, {&w.n_cnt, N2},
            {&w.n_depth, N2}, {&w.n_rep, N2}, {&w.n_a0, N2}, {&w.n_a1, N2}, {&w.n_span, N2},
            {&w.n_pack, N2}, {&w.npacks, 1}, {&w.p_node, N2}, {&w.p_qoff, N2 + 1}, {&w.p_q, BD1},
            {&w.p_partial, N2}};
  size_t total = 0;
  for (auto& f : fields) total += (f.second + 63) & ~size_t(63);
  int32_t* arena = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&arena, total * 4, st);
  if (e != cudaSuccess) {
    set_error("device packer workspace (%zu B): %s", total * 4, cudaGetErrorString(e));
    return PAT_ERR_CUDA;
  }
  size_t off = 0;
  for (auto& f : fields) {
    *f.first = arena + off;
    off += (f.second + 63) & ~size_t(63);
  }
  cudaMemsetAsync(w.err, 0, 8, st);
  cudaMemsetAsync(w.npacks, 0, 4, st);
  cudaMemsetAsync(w.member, 0, BD1 * 4, st);
  // node records are copied back whole; unused entries stay defined (initcheck)
  for (int32_t* a : {w.n_rep, w.n_a0, w.n_a1, w.n_span}) cudaMemsetAsync(a, 0, N2 * 4, st);
  const int TB = 128;
  const int gq = (B + TB - 1) / TB;
  dev::k_rows<<<gq, TB, 0, st>>>(w);
  int P = 1;
  while (P < std::max(B, maxb)) P <<= 1;
  const int dup_smem = std::max(P * 4, 256);  // also the row's segment sums (8 B per 32 blocks)
  if (dup_smem > 48 * 1024) cudaFuncSetAttribute(dev::k_dup, cudaFuncAttributeMaxDynamicSharedMemorySize, dup_smem);
  dev::k_dup<<<B, 256, dup_smem, st>>>(w);
  {
    int64_t warps = (int64_t)B * B;
    int grid = (int)std::min<int64_t>((warps * 32 + 255) / 256, 148 * 16);
    dev::k_lcp<<<grid, 256, 0, st>>>(w);
  }
  int PB = 1;
  while (PB < B) PB <<= 1;
  if (PB * 24 > 48 * 1024) cudaFuncSetAttribute(dev::k_levels, cudaFuncAttributeMaxDynamicSharedMemorySize, PB * 24);
  dev::k_levels<<<B, 1024, PB * 24, st>>>(w);
  dev::k_decide<<<gq, TB, 0, st>>>(w);
  dev::k_rank<<<(B * 32 + 255) / 256, 256, 0, st>>>(w);
  dev::k_scan_nodes<<<1, 1024, 0, st>>>(w);
  dev::k_nodes_init<<<64, 256, 0, st>>>(w);
  dev::k_nodes<<<gq, TB, 0, st>>>(w);
  dev::k_order<<<64, 256, 0, st>>>(w);
  dev::k_pack_offsets<<<1, 1024, 0, st>>>(w);
  dev::k_members<<<gq, TB, 0, st>>>(w);
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    cudaFreeAsync(arena, st);
    set_error("device packer launch: %s", cudaGetErrorString(e));
    return PAT_ERR_CUDA;
  }
  // bring back status, counts and packs
  int32_t err[2], np = 0;
  cudaMemcpyAsync(err, w.err, 8, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&np, w.npacks, 4, cudaMemcpyDeviceToHost, st);
  h_nblk->resize(B);
  h_valid->resize(B);
  cudaMemcpyAsync(h_nblk->data(), w.nblk, B * 4, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(h_valid->data(), w.valid, B * 4, cudaMemcpyDeviceToHost, st);
  h_rows->resize((size_t)B * stride);
  cudaMemcpyAsync(h_rows->data(), d_bt, (size_t)B * stride * 4, cudaMemcpyDeviceToHost, st);
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    set_error("device packer: %s", cudaGetErrorString(e));
    return PAT_ERR_CUDA;
  }
  if (err[0]) {
    cudaFreeAsync(arena, st);
    if (err[0] == PAT_ERR_INVALID_SPEC) set_error("row %d: empty, too long, or repeats a block ID", err[1]);
    else set_error("query %d: prefix forest deeper than the device packer capacity", err[1]);
    return err[0];
  }
  std::vector<int32_t> node(np), qoff(np + 1), partial(np), rep(2 * B + 2), a0(2 * B + 2), a1(2 * B + 2),
      span(2 * B + 2);
  cudaMemcpyAsync(node.data(), w.p_node, np * 4, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(qoff.data(), w.p_qoff, (np + 1) * 4, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(partial.data(), w.p_partial, np * 4, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(rep.data(), w.n_rep, (2 * B + 2) * 4, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(a0.data(), w.n_a0, (2 * B + 2) * 4, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(a1.data(), w.n_a1, (2 * B + 2) * 4, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(span.data(), w.n_span, (2 * B + 2) * 4, cudaMemcpyDeviceToHost, st);
  std::vector<int32_t> q(np ? qoff[0] : 0);
  e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) {
    q.resize(qoff[np]);
    cudaMemcpyAsync(q.data(), w.p_q, qoff[np] * 4, cudaMemcpyDeviceToHost, st);
    e = cudaStreamSynchronize(st);
  }
  cudaFreeAsync(arena, st);
  if (e != cudaSuccess) {
    set_error("device packer copy-back: %s", cudaGetErrorString(e));
    return PAT_ERR_CUDA;
  }
  out->q = q;
  out->q_off.assign(qoff.begin(), qoff.end());
  for (int p = 0; p < np; ++p) {
    const int id = node[p];
    out->kv.push_back(span[id]);
    out->partial.push_back((uint8_t)partial[p]);
    out->rep.push_back(rep[id]);
    out->blk_begin.push_back(a0[id]);
    for (int j = a0[id]; j < a1[id]; ++j) out->blk.push_back((*h_rows)[(size_t)rep[id] * stride + j]);
    out->blk_off.push_back((int32_t)out->blk.size());
  }
  return PAT_OK;
}

// ------------------------------------------------------------------------------------------
// Device table hash for the lazy update (PackCache keyed by a device fingerprint,
// packer.py:189-221): 64-bit, order-sensitive over rows and positions, computed as
// a sum of splitmix64-mixed terms so the reduction order does not matter.
// ------------------------------------------------------------------------------------------
namespace {
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// one warp per row: (row, position, block id) terms and (row, seq_len)
__global__ void k_table_hash(const int32_t* __restrict__ bt, int64_t stride, const int32_t* __restrict__ seq, int B,
                             int bs, unsigned long long* out) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  uint64_t acc = 0;
  for (int q = w; q < B; q += nw) {
    const int len = __ldg(seq + q);
    const int nb = len > 0 ? (len + bs - 1) / bs : 0;
    const uint64_t rowk = mix64(((uint64_t)q << 32) ^ 0xA5A5A5A5ull);
    for (int j = lane; j < nb; j += 32)
      acc += mix64(rowk ^ ((uint64_t)j << 32) ^ (uint32_t)__ldg(bt + (int64_t)q * stride + j));
    if (lane == 0) acc += mix64(rowk + 0x5151ull + (uint64_t)(uint32_t)len);
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0 && acc) atomicAdd(out, (unsigned long long)acc);
}
}  // namespace

}  // namespace pat

extern "C" int pat_table_hash_device(int32_t B, const int32_t* block_tables, int64_t bt_stride,
                                     const int32_t* seq_lens, int32_t block_size, uint64_t* out_hash,
                                     void* stream) {
  if (!out_hash || B < 0 || block_size <= 0 || (B > 0 && (!block_tables || !seq_lens))) {
    pat::set_error("bad arguments to pat_table_hash_device");
    return PAT_ERR_SHAPE_MISMATCH;
  }
  cudaStream_t st = (cudaStream_t)stream;
  // seed with (B, block_size) so the empty table and different page sizes differ
  const uint64_t seed = ((uint64_t)(uint32_t)B << 32) ^ (uint64_t)(uint32_t)block_size ^ 0x7A7A000000000000ull;
  cudaError_t e = cudaMemcpyAsync(out_hash, &seed, sizeof(seed), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && B > 0) {
    const int blocks = std::min(148 * 4, (B + 7) / 8);
    pat::k_table_hash<<<blocks, 256, 0, st>>>(block_tables, bt_stride, seq_lens, B, block_size,
                                             (unsigned long long*)out_hash);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) {
    pat::set_error("pat_table_hash_device: %s", cudaGetErrorString(e));
    return PAT_ERR_CUDA;
  }
  return PAT_OK;
}

// ------------------------------------------------------------------------------------------
// Device-resident planner (pat_decoder): fingerprint -> compare -> GPU packer ->
// on-device schedule -> forward + merge, all stream-ordered with no host
// synchronisation and no allocation, so a serving step (or a CUDA graph of it)
// re-plans only when the block table changed (packer.py:189-221 lazy update,
// PAPER.md:433 "scheduler run asynchronously").
// ------------------------------------------------------------------------------------------
namespace pat {

cudaError_t launch_forward_tc(const CUtensorMap& tmk, const CUtensorMap& tmv, const DevPlan& plan, int var, int grid,
                              int dtype, int d, const void* q, void* out, float* po, float* pl, float scale_log2,
                              int32_t* sched, cudaStream_t st);
cudaError_t launch_merge(const DevPlan& plan, int grid, int dtype, int d, const float* po, const float* pl, void* out,
                         cudaStream_t st);
int make_kv_tensor_map(CUtensorMap* map, const void* base, int64_t num_blocks, int bs, int kvh, int d, int dtype);

namespace dev {

__global__ void k_reset(Ws w, int N2) {
  if (w.run && !*w.run) return;
  const int BD1 = w.B * (w.D + 1);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < BD1; i += gridDim.x * blockDim.x) w.member[i] = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N2; i += gridDim.x * blockDim.x)
    w.n_rep[i] = w.n_a0[i] = w.n_a1[i] = w.n_span[i] = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) w.err[0] = w.err[1] = *w.npacks = 0;
}

// table fingerprint seed, then compare with the last one: run = changed
__global__ void k_hash_seed(unsigned long long* h, int B, int bs) {
  *h = ((unsigned long long)(unsigned)B << 32) ^ (unsigned long long)(unsigned)bs ^ 0x7A7A000000000000ull;
}
__global__ void k_hash_check(const unsigned long long* h_new, unsigned long long* h_old, int32_t* run, int32_t* nrun) {
  const bool changed = *h_new != *h_old;
  *run = changed ? 1 : 0;
  if (changed) {
    *h_old = *h_new;
    atomicAdd(nrun, 1);
  }
}

struct Sched {
  Ws w;
  // outputs (the DevPlan points at these)
  int32_t* pack_blk_off;  // [2B+2]
  int32_t* pack_blk;      // [cap_blk]
  int32_t* unit_pack;     // [cap_units]
  int32_t* unit_page0;
  int32_t* unit_ntok;
  int32_t* unit_slot_off; // [cap_units+1]
  int32_t* unit_slot;     // [cap_members]
  Item* items;            // [cap_items]
  int32_t* n_items;       // [NUM_VARIANTS]
  int32_t* n_pair;        // [NUM_VARIANTS]
  int4* merge_desc;       // [B]
  int32_t* n_merge;       // [1]
  // scratch
  int32_t* parts;         // [2B+2]
  int32_t* ubase;         // [2B+3]
  int32_t* qcnt;          // [B]
  int32_t* qoff;          // [B]
  int32_t* qlist_n;       // [B]
  int2* qlist;            // [B][D+1] (pack, member index)
  int32_t* prior;         // [pack members] units of the member's query in earlier packs
  unsigned long long* ukey;  // [cap_units] sort keys
  // capacities
  int cap_blk, cap_units, cap_members, cap_items, cap_slots;
  // model
  float item_ns, row_ns, step_ns, hbm_bpns;
  int lanes, H, KVH, d, G;
};

// exclusive scan over n values produced by `val(i)` with one CTA; returns the total
template <typename F, typename O>
__device__ int cta_scan(int n, F val, O put) {
  const int t = threadIdx.x, nt = blockDim.x;
  const int per = (n + nt - 1) / nt;
  int s = 0;
  for (int i = t * per; i < min(n, (t + 1) * per); ++i) s += val(i);
  int total;
  int acc = block_excl_scan(s, &total);
  for (int i = t * per; i < min(n, (t + 1) * per); ++i) {
    put(i, acc);
    acc += val(i);
  }
  __syncthreads();
  return total;
}

__device__ __forceinline__ float sched_item_ns(const Sched& S, int rows, int ntok) {
  const float steps = (float)((ntok + 63) / 64);
  return S.item_ns + S.row_ns * rows / 128.f + steps * S.step_ns * (0.5f + 0.5f * S.d / 128.f);
}

// One CTA: split (chunk chosen by a makespan estimate over the lanes), units,
// partial slots in unit order, longest-first work items, merge descriptors.
#ifdef PAT_TC_TRACE
__device__ long long g_sched_stamp[16];
#define SCHED_STAMP(i)                                        \
  do {                                                        \
    if (threadIdx.x == 0) {                                   \
      long long t_;                                           \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));  \
      g_sched_stamp[i] = t_;                                  \
    }                                                         \
  } while (0)
#else
#define SCHED_STAMP(i) \
  do {                 \
  } while (0)
#endif
__device__ void ph_schedule(const Sched& S, uint8_t* smem, int smem_bytes) {
  if (blockIdx.x != 0) return;  // one CTA of 1024 threads
  SCHED_STAMP(0);
  const Ws& w = S.w;
  const int t = threadIdx.x, nt = blockDim.x;
  __shared__ int s_np, s_err, s_chunk;
  if (t == 0) {
    s_np = *w.npacks;
    s_err = w.err[0];
  }
  __syncthreads();
  const int NP = s_np;
  if (s_err || NP == 0) {  // invalid table: nothing runs (pat_decoder_status reports it)
    if (t < NUM_VARIANTS) S.n_items[t] = S.n_pair[t] = 0;
    if (t == 0) *S.n_merge = 0;
    return;
  }
  auto pk_node = [&](int p) { return w.p_node[p]; };
  // per-pack (pages, rows, kv) staged in shared memory when it fits (every
  // phase below reads them many times)
  int3* spk = reinterpret_cast<int3*>(smem);
  const bool pk_smem = NP * (int)sizeof(int3) <= smem_bytes;
  if (pk_smem) {
    for (int p = t; p < NP; p += nt) {
      const int id = pk_node(p);
      spk[p] = make_int3(w.n_a1[id] - w.n_a0[id], (w.p_qoff[p + 1] - w.p_qoff[p]) * S.G, w.n_span[id]);
    }
    __syncthreads();
  }
  auto pk_pages = [&](int p) { if (pk_smem) return spk[p].x; const int id = pk_node(p); return w.n_a1[id] - w.n_a0[id]; };
  auto pk_rows = [&](int p) { return pk_smem ? spk[p].y : (w.p_qoff[p + 1] - w.p_qoff[p]) * S.G; };
  auto pk_kv = [&](int p) { return pk_smem ? spk[p].z : w.n_span[pk_node(p)]; };

  // pack spans: the rep query's row [a0, a1)
  const int nblk = cta_scan(NP, pk_pages, [&](int i, int v) { S.pack_blk_off[i] = v; });
  if (t == 0) S.pack_blk_off[NP] = nblk;
  const int wp = t >> 5, ln = t & 31, nwp = nt >> 5;  // warp per pack / unit below
  for (int p = wp; p < NP; p += nwp) {
    const int id = pk_node(p), rep = w.n_rep[id], a0 = w.n_a0[id], n = w.n_a1[id] - a0;
    const int o = S.pack_blk_off[p];
    for (int j = ln; j < n; j += 32)
      if (o + j < S.cap_blk) S.pack_blk[o + j] = w.bt[(int64_t)rep * w.stride + a0 + j];
  }

  SCHED_STAMP(1);
  // chunk (pages, power of two): minimise the makespan estimate
  // over the candidates whose units, member slots and items fit the capacities
  int maxp = 1;
  {
    __shared__ int s_maxp;
    if (t == 0) s_maxp = 1;
    __syncthreads();
    for (int p = t; p < NP; p += nt) atomicMax(&s_maxp, pk_pages(p));
    __syncthreads();
    maxp = s_maxp;
  }
  if (t == 0) s_chunk = maxp;
  __syncthreads();
  {
    __shared__ float s_work, s_worst, s_bytes;
    __shared__ int s_units, s_memb, s_items;
    // longest-first claims over the lanes finish near max(work / lanes, longest
    // item) plus about half a mean item of tail
    float best = 3.0e38f;
    int best_c = maxp;
    for (int c = 1;; c *= 2) {
      const int cc = min(c, maxp);
      if (t == 0) s_work = s_worst = s_bytes = 0.f, s_units = s_memb = s_items = 0;
      __syncthreads();
      float work = 0.f, worst = 0.f, bytes = 0.f;
      int units = 0, memb = 0, its = 0;
      for (int p = t; p < NP; p += nt) {
        const int pages = pk_pages(p), rows = pk_rows(p), kv = pk_kv(p);
        const int parts = (pages + cc - 1) / cc;
        const int rb = (rows + 127) / 128;
        const int big = (pages + parts - 1) / parts;
        const float it = sched_item_ns(S, min(rows, 128), min(big * w.bs, kv));
        work += it * rb * parts * S.KVH;
        worst = fmaxf(worst, it);
        bytes += (float)kv * S.KVH * S.d * 4.f;
        if (parts > 1) bytes += (float)parts * (rows / S.G) * S.H * S.d * 8.f;
        units += parts;
        memb += parts * (rows / S.G);
        its += parts * rb * S.KVH;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {  // warp sums first: one shared atomic per warp
        work += __shfl_xor_sync(0xffffffffu, work, o);
        bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
        worst = fmaxf(worst, __shfl_xor_sync(0xffffffffu, worst, o));
        units += __shfl_xor_sync(0xffffffffu, units, o);
        memb += __shfl_xor_sync(0xffffffffu, memb, o);
        its += __shfl_xor_sync(0xffffffffu, its, o);
      }
      if ((t & 31) == 0) {
        atomicAdd(&s_work, work);
        atomicAdd(&s_bytes, bytes);
        atomicMax((int*)&s_worst, __float_as_int(worst));  // non-negative floats order as ints
        atomicAdd(&s_units, units);
        atomicAdd(&s_memb, memb);
        atomicAdd(&s_items, its);
      }
      __syncthreads();
      const float mean = s_items > 0 ? s_work / s_items : 0.f;
      const float est = fmaxf(s_bytes / S.hbm_bpns, fmaxf(s_work / S.lanes, s_worst) + 0.5f * mean);
      const bool fits = s_units <= S.cap_units && s_memb <= S.cap_members && s_items <= S.cap_items &&
                        s_memb <= S.cap_slots;
      if (fits && est <= best * 1.02f) {
        if (est < best) best = est;
        best_c = cc;
      }
      __syncthreads();
      if (cc >= maxp) break;
    }
    if (t == 0) s_chunk = best_c;
    __syncthreads();
  }
  const int chunk = s_chunk;

  SCHED_STAMP(2);
  // units: pack p -> parts[p] near-equal page runs, larger first, the last
  // carrying the partial block (simulator.py:137-154)
  for (int p = t; p < NP; p += nt) S.parts[p] = (pk_pages(p) + chunk - 1) / chunk;
  __syncthreads();
  const int NU = cta_scan(NP, [&](int p) { return S.parts[p]; }, [&](int i, int v) { S.ubase[i] = v; });
  if (t == 0) S.ubase[NP] = NU;
  __syncthreads();
  for (int p = wp; p < NP; p += nwp) {
    const int parts = S.parts[p], pages = pk_pages(p), kv = pk_kv(p), u0 = S.ubase[p];
    const int base = pages / parts, extra = pages % parts;
    for (int i = ln; i < parts; i += 32) {
      const int take = base + (i < extra ? 1 : 0);
      const int pos = i * base + min(i, extra);
      S.unit_pack[u0 + i] = p;
      S.unit_page0[u0 + i] = pos;
      S.unit_ntok[u0 + i] = min(take * w.bs, kv - pos * w.bs);
    }
  }
  __syncthreads();
  // member CSR of the units: unit u of pack p has the pack's members
  const int NM = cta_scan(NU, [&](int u) { const int p = S.unit_pack[u]; return w.p_qoff[p + 1] - w.p_qoff[p]; },
                          [&](int i, int v) { S.unit_slot_off[i] = v; });
  if (t == 0) S.unit_slot_off[NU] = NM;

  SCHED_STAMP(3);
  // slots: a query covered by more than one unit gets one slot per unit, in
  // unit order (the reference fold order, attention.py:228-235)
  for (int q = t; q < w.B; q += nt) S.qcnt[q] = 0, S.qlist_n[q] = 0;
  __syncthreads();
  const int D1 = w.D + 1;
  for (int p = wp; p < NP; p += nwp)
    for (int j = w.p_qoff[p] + ln; j < w.p_qoff[p + 1]; j += 32) {
      const int q = w.p_q[j];
      atomicAdd(&S.qcnt[q], S.parts[p]);
      const int k = atomicAdd(&S.qlist_n[q], 1);
      if (k < D1) S.qlist[(int64_t)q * D1 + k] = make_int2(p, j);
    }
  __syncthreads();
  for (int q = t; q < w.B; q += nt) {  // this query's packs in pack order -> units before each
    int2* L = S.qlist + (int64_t)q * D1;
    const int n = min(S.qlist_n[q], D1);
    for (int i = 1; i < n; ++i) {
      const int2 x = L[i];
      int k = i - 1;
      while (k >= 0 && L[k].x > x.x) L[k + 1] = L[k], --k;
      L[k + 1] = x;
    }
    int acc = 0;
    for (int i = 0; i < n; ++i) {
      S.prior[L[i].y] = acc;
      acc += S.parts[L[i].x];
    }
  }
  __syncthreads();
  const int NS = cta_scan(w.B, [&](int q) { return S.qcnt[q] > 1 ? S.qcnt[q] : 0; },
                          [&](int i, int v) { S.qoff[i] = v; });
  (void)NS;
  const int NMQ = cta_scan(w.B, [&](int q) { return S.qcnt[q] > 1 ? 1 : 0; }, [&](int q, int v) {
    if (S.qcnt[q] > 1) S.merge_desc[v] = make_int4(q, S.qoff[q], S.qcnt[q], 0);
  });
  if (t == 0) *S.n_merge = NMQ;
  for (int u = wp; u < NU; u += nwp) {
    const int p = S.unit_pack[u], m0 = w.p_qoff[p], m1 = w.p_qoff[p + 1];
    const int i = u - S.ubase[p];  // split index
    for (int j = m0 + ln; j < m1; j += 32) {
      const int q = w.p_q[j];
      S.unit_slot[S.unit_slot_off[u] + (j - m0)] = S.qcnt[q] > 1 ? S.qoff[q] + S.prior[j] + i : -1;
    }
  }
  __syncthreads();

  SCHED_STAMP(4);
  // work items (unit x 128-row block x kv head), longest (estimated) first:
  // units sorted by cost, descending (bitonic sort over the units in global memory)
  int P2 = 1;
  while (P2 < NU) P2 <<= 1;
  // the sort keys in shared memory (after the pack records) when they fit
  const int koff = pk_smem ? ((NP * (int)sizeof(int3) + 15) & ~15) : 0;
  unsigned long long* ukey =
      koff + P2 * 8 <= smem_bytes ? reinterpret_cast<unsigned long long*>(smem + koff) : S.ukey;
  for (int u = t; u < P2; u += nt) {
    unsigned long long key = ~0ull;
    if (u < NU) {
      const int p = S.unit_pack[u];
      const float c = sched_item_ns(S, min(pk_rows(p), 128), S.unit_ntok[u]) * ((pk_rows(p) + 127) / 128);
      key = ((unsigned long long)(0xFFFFFFFFu - (unsigned)fminf(c, 4.0e9f)) << 32) | (unsigned)u;
    }
    ukey[u] = key;
  }
  __syncthreads();
  for (int k = 2; k <= P2; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = t; i < P2; i += nt) {
        const int l = i ^ j;
        if (l > i) {
          const bool up = (i & k) == 0;
          const unsigned long long a = ukey[i], b = ukey[l];
          if ((a > b) == up) ukey[i] = b, ukey[l] = a;
        }
      }
      __syncthreads();
    }
  SCHED_STAMP(5);
  const int NI = cta_scan(NU, [&](int r) {
    const int u = (int)(ukey[r] & 0xFFFFFFFFu);
    return ((pk_rows(S.unit_pack[u]) + 127) / 128) * S.KVH;
  }, [&](int r, int v) {
    const int u = (int)(ukey[r] & 0xFFFFFFFFu), p = S.unit_pack[u], rows = pk_rows(p);
    int k = v;
    for (int r0 = 0; r0 < rows; r0 += 128)
      for (int h = 0; h < S.KVH; ++h, ++k)
        S.items[k] = Item{u, h, r0, min(128, rows - r0), S.pack_blk_off[p] + S.unit_page0[u], S.unit_ntok[u],
                          w.p_qoff[p], S.unit_slot_off[u]};
  });
  if (t < NUM_VARIANTS) {
    S.n_items[t] = t == VAR_TC ? NI : 0;
    S.n_pair[t] = 0;
  }
  SCHED_STAMP(6);
}

// grid barrier of the persistent planner (every CTA resident: cooperative
// launch).  The gpu-scope fence after the wait also invalidates the SM's L1,
// so the next phase reads what other SMs wrote.
__device__ void grid_sync(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1) == gridDim.x - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1);
    } else {
      while (*gen == g) __nanosleep(64);
    }
    __threadfence();
  }
  __syncthreads();
}

// fingerprint terms of (block_tables, seq_lens), summed (order-free); a warp per row
__device__ void ph_hash(const int32_t* __restrict__ bt, int64_t stride, const int32_t* __restrict__ seq, int B,
                        int bs, unsigned long long* acc_out) {
  const int lane = threadIdx.x & 31;
  const int wi = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  uint64_t acc = 0;
  for (int q = wi; q < B; q += nw) {
    const int len = seq[q];
    const int nb = len > 0 ? (len + bs - 1) / bs : 0;
    const uint64_t rowk = mix64(((uint64_t)q << 32) ^ 0xA5A5A5A5ull);
    for (int j = lane; j < nb; j += 32) acc += mix64(rowk ^ ((uint64_t)j << 32) ^ (uint32_t)bt[(int64_t)q * stride + j]);
    if (lane == 0) acc += mix64(rowk + 0x5151ull + (uint64_t)(uint32_t)len);
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  // one atomic per CTA, not per warp
  __shared__ unsigned long long wacc[32];
  if (lane == 0) wacc[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint64_t a = threadIdx.x < (blockDim.x >> 5) ? wacc[threadIdx.x] : 0;
#pragma unroll
    for (int off = 16; off; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
    if (threadIdx.x == 0 && a) atomicAdd(acc_out, (unsigned long long)a);
  }
}

#ifdef PAT_TC_TRACE
__device__ long long g_plan_stamp[32];
#define PLAN_STAMP(i)                                                        \
  do {                                                                       \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                               \
      long long t_;                                                          \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                 \
      g_plan_stamp[i] = t_;                                                  \
    }                                                                        \
  } while (0)
#else
#define PLAN_STAMP(i) \
  do {                \
  } while (0)
#endif

struct PlanState {
  unsigned long long* h_acc;  // fingerprint accumulator (left at 0 between calls)
  unsigned long long* h_old;  // fingerprint of the planned table
  int32_t* run;
  int32_t* nrun;
  unsigned* bar;  // [2] grid barrier
  int32_t* fwd_sched;  // [4] the forward's claim counters, zeroed here
};

// The whole planner in ONE launch: fingerprint -> compare -> (only when the
// table changed) reset, rows, duplicates, pairwise prefixes, levels, decisions,
// DFS rank, nodes, pack order and members, then the schedule on CTA 0.
__global__ void __launch_bounds__(1024, 1) k_plan(Ws w, Sched S, PlanState ps, int N2, int dyn_bytes) {
  extern __shared__ __align__(16) uint8_t dsm[];
  if (blockIdx.x == 0 && threadIdx.x < 4) ps.fwd_sched[threadIdx.x] = 0;
  ph_hash(w.bt, w.stride, w.seq, w.B, w.bs, ps.h_acc);
  // one barrier for fingerprint + compare: the last CTA to arrive compares
  // the fingerprint and publishes the decision before releasing the others
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned* bar = ps.bar;
    volatile unsigned* gen = bar + 1;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1) == gridDim.x - 1) {
      __threadfence();
      const unsigned long long h = *(volatile unsigned long long*)ps.h_acc +
          (((unsigned long long)(unsigned)w.B << 32) ^ (unsigned long long)(unsigned)w.bs ^ 0x7A7A000000000000ull);
      *ps.h_acc = 0;
      const bool changed = h != *ps.h_old;
      *ps.run = changed ? 1 : 0;
      if (changed) {
        *ps.h_old = h;
        atomicAdd(ps.nrun, 1);
      }
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1);
    } else {
      while (*gen == g) __nanosleep(64);
    }
    __threadfence();
  }
  __syncthreads();
  PLAN_STAMP(0);
  PLAN_STAMP(1);
  if (!*(volatile int32_t*)ps.run) return;
  {
    const int BD1 = w.B * (w.D + 1);
    PAT_GRID_LOOP(i, BD1) w.member[i] = 0;
    PAT_GRID_LOOP(i, N2) w.n_rep[i] = w.n_a0[i] = w.n_a1[i] = w.n_span[i] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) w.err[0] = w.err[1] = *w.npacks = 0;
  }
  grid_sync(ps.bar);
  PLAN_STAMP(2);
  ph_rows(w);
  grid_sync(ps.bar);
  PLAN_STAMP(3);
  ph_dup(w, (int32_t*)dsm);
  grid_sync(ps.bar);
  PLAN_STAMP(4);
  ph_lcp(w);
  grid_sync(ps.bar);
  PLAN_STAMP(5);
  ph_levels(w, (unsigned long long*)dsm);
  grid_sync(ps.bar);
  PLAN_STAMP(6);
  ph_decide(w);
  grid_sync(ps.bar);
  PLAN_STAMP(7);
  ph_rank(w);
  grid_sync(ps.bar);
  PLAN_STAMP(8);
  ph_scan_nodes(w);
  grid_sync(ps.bar);
  PLAN_STAMP(9);
  ph_nodes_init(w);
  grid_sync(ps.bar);
  PLAN_STAMP(10);
  ph_nodes(w);
  grid_sync(ps.bar);
  PLAN_STAMP(11);
  ph_order(w, reinterpret_cast<int4*>(dsm), dyn_bytes / 16);
  grid_sync(ps.bar);
  PLAN_STAMP(12);
  ph_pack_offsets(w);
  grid_sync(ps.bar);
  PLAN_STAMP(13);
  ph_members(w);
  grid_sync(ps.bar);
  PLAN_STAMP(14);
  ph_schedule(S, dsm, dyn_bytes);
  __syncthreads();
  PLAN_STAMP(15);
}

}  // namespace dev
}  // namespace pat

// dynamic shared memory of the planner kernel: the largest phase need (row
// sort, per-query key sort + flags, node records, pack records + unit keys)
static int plan_smem(int P, int PB, int n2) {
  const int want = std::max({P * 4, PB * 24, n2 * 16, n2 * 12 + 8 * 4096});
  return std::min(want, 190 * 1024);
}

struct pat_decoder {
  int Bmax = 0, maxb = 0, bs = 16, H = 0, KVH = 0, d = 0, D = 0, num_sms = 148, device = -1;
  void* arena = nullptr;
  pat::dev::Ws w{};
  pat::dev::Sched S{};
  pat::DevPlan plan{};
  unsigned long long* h_new = nullptr;  // fingerprint accumulator of the planner kernel
  unsigned long long* h_old = nullptr;
  int32_t* run = nullptr;
  int32_t* nrun = nullptr;
  unsigned* bar = nullptr;  // grid barrier of the planner kernel
  int plan_grid = 0;
  // TMA descriptors of the last (k_cache, v_cache) pair, under mu
  std::mutex mu;
  CUtensorMap tmk, tmv;
  const void* tm_k = nullptr;
  const void* tm_v = nullptr;
  int64_t tm_blocks = -1;
  int tm_dtype = -1;
};

extern "C" {

int pat_decoder_create(const pat_plan_options* opt, int32_t max_batch, int32_t max_blocks, int32_t block_size,
                       pat_decoder** out) {
  using namespace pat;
  if (!out || !opt) return PAT_ERR_INVALID_SPEC;
  *out = nullptr;
  if (max_batch < 1 || max_batch > 4096 || max_blocks < 1 || block_size < 16 || block_size % 16 ||
      opt->num_heads <= 0 || opt->num_kv_heads <= 0 || opt->num_heads % opt->num_kv_heads ||
      (opt->head_dim != 64 && opt->head_dim != 128)) {
    set_error("pat_decoder_create: need 1 <= max_batch <= 4096, block_size a multiple of 16, head_dim 64/128, "
              "H a multiple of KVH");
    return PAT_ERR_INVALID_SPEC;
  }
  pat_decoder* Dc = new pat_decoder();
  Dc->Bmax = max_batch;
  Dc->maxb = max_blocks;
  Dc->bs = block_size;
  Dc->H = opt->num_heads;
  Dc->KVH = opt->num_kv_heads;
  Dc->d = opt->head_dim;
  cudaGetDevice(&Dc->device);
  int nsm = 0;
  if (opt->num_sms > 0) nsm = opt->num_sms;
  else if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, Dc->device) != cudaSuccess || nsm <= 0)
    nsm = 148;
  Dc->num_sms = nsm;
  const int B = max_batch, D = std::min(B, max_blocks + 1) + 1, D1 = D + 1;
  const size_t Bz = (size_t)B;
  Dc->D = D;
  const size_t BB = (size_t)B * B, BD = (size_t)B * D, BD1 = (size_t)B * D1, N2 = 2 * (size_t)B + 2;
  const int G = Dc->H / Dc->KVH;
  // capacities of the schedule (the chunk choice keeps the plan inside them)
  const size_t cap_blk = (size_t)B * max_blocks;
  const size_t cap_units = N2 + (size_t)B * max_blocks / 8 + 64;
  const size_t cap_members = BD1 * 4 + 64;
  const size_t cap_slots = (size_t)B * 16;
  const size_t cap_items = cap_units * ((size_t)(B * G + 127) / 128) * Dc->KVH;
  const size_t cap_items_c = std::min<size_t>(cap_items, (size_t)1 << 20);
  size_t P2 = 1;
  while (P2 < cap_units) P2 <<= 1;
  struct F { void** p; size_t bytes; };
  dev::Ws& w = Dc->w;
  dev::Sched& S = Dc->S;
  std::vector<F> f = {
      {(void**)&w.nblk, Bz * 4}, {(void**)&w.valid, Bz * 4}, {(void**)&w.err, 8}, {(void**)&w.lcp, BB * 4},
      {(void**)&w.hs, Bz * ((max_blocks + 31) / 32) * 8},
      {(void**)&w.K, Bz * 4}, {(void**)&w.hasleaf, Bz * 4}, {(void**)&w.end, BD * 4}, {(void**)&w.nq, BD * 4},
      {(void**)&w.minq, BD * 4}, {(void**)&w.term, BD * 4}, {(void**)&w.start, BD1 * 4}, {(void**)&w.stop, BD1 * 4},
      {(void**)&w.span, BD1 * 4}, {(void**)&w.anchor, BD1 * 4}, {(void**)&w.member, BD1 * 4},
      {(void**)&w.nmemb, Bz * 4}, {(void**)&w.k0, Bz * 4}, {(void**)&w.cnt_own, Bz * 4}, {(void**)&w.pi, Bz * 4},
      {(void**)&w.order, Bz * 4}, {(void**)&w.base, (Bz + 1) * 4}, {(void**)&w.n_hi, N2 * 4},
      {(void**)&w.n_lo, N2 * 4}, {(void**)&w.n_cnt, N2 * 4}, {(void**)&w.n_depth, N2 * 4},
      {(void**)&w.n_rep, N2 * 4}, {(void**)&w.n_a0, N2 * 4}, {(void**)&w.n_a1, N2 * 4},
      {(void**)&w.n_span, N2 * 4}, {(void**)&w.n_pack, N2 * 4}, {(void**)&w.npacks, 4},
      {(void**)&w.p_node, N2 * 4}, {(void**)&w.p_qoff, (N2 + 1) * 4}, {(void**)&w.p_q, BD1 * 4},
      {(void**)&w.p_partial, N2 * 4},
      {(void**)&S.pack_blk_off, (N2 + 1) * 4}, {(void**)&S.pack_blk, cap_blk * 4},
      {(void**)&S.unit_pack, cap_units * 4}, {(void**)&S.unit_page0, cap_units * 4},
      {(void**)&S.unit_ntok, cap_units * 4}, {(void**)&S.unit_slot_off, (cap_units + 1) * 4},
      {(void**)&S.unit_slot, cap_members * 4}, {(void**)&S.items, cap_items_c * sizeof(Item)},
      {(void**)&S.n_items, 16}, {(void**)&S.n_pair, 16}, {(void**)&S.merge_desc, Bz * 16},
      {(void**)&S.n_merge, 4}, {(void**)&S.parts, N2 * 4}, {(void**)&S.ubase, (N2 + 1) * 4},
      {(void**)&S.qcnt, Bz * 4}, {(void**)&S.qoff, Bz * 4}, {(void**)&S.qlist_n, Bz * 4},
      {(void**)&S.qlist, BD1 * 8}, {(void**)&S.prior, BD1 * 4}, {(void**)&S.ukey, P2 * 8},
      {(void**)&Dc->h_new, 8}, {(void**)&Dc->h_old, 8}, {(void**)&Dc->run, 4}, {(void**)&Dc->nrun, 4},
      {(void**)&Dc->bar, 8}};
  size_t total = 0;
  for (auto& x : f) total += (x.bytes + 255) & ~size_t(255);
  if (cudaMalloc(&Dc->arena, total) != cudaSuccess) {
    set_error("pat_decoder_create: %zu bytes of device state", total);
    delete Dc;
    return PAT_ERR_CUDA;
  }
  cudaMemset(Dc->arena, 0, total);
  size_t off = 0;
  for (auto& x : f) {
    *x.p = (uint8_t*)Dc->arena + off;
    off += (x.bytes + 255) & ~size_t(255);
  }
  cudaMemset(Dc->h_old, 0xFF, 8);  // never equal to a real fingerprint's first value
  // the planner kernel runs one CTA per SM (all resident: cooperative launch)
  {
    int P = 1;
    while (P < std::max(B, max_blocks)) P <<= 1;
    int PB = 1;
    while (PB < B) PB <<= 1;
    const int dyn = plan_smem(P, PB, 2 * B + 2);
    cudaFuncSetAttribute(dev::k_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dev::k_plan, 1024, dyn);
    Dc->plan_grid = std::max(1, std::min(per_sm, 1)) * nsm;
    if (per_sm < 1) {
      set_error("pat_decoder_create: the planner kernel does not fit an SM");
      cudaFree(Dc->arena);
      delete Dc;
      return PAT_ERR_CUDA;
    }
  }
  w.D = D;
  w.bs = block_size;
  w.run = Dc->run;
  w.hs_n = (max_blocks + 31) / 32;
  S.cap_blk = (int)cap_blk;
  S.cap_units = (int)cap_units;
  S.cap_members = (int)cap_members;
  S.cap_items = (int)cap_items_c;
  S.cap_slots = (int)cap_slots;
  const pat_cost_model cm = cost_model();
  S.item_ns = (float)cm.tc_item_ns;
  S.row_ns = (float)cm.tc_item_row_ns;
  S.step_ns = (float)cm.tc_step_ns;
  S.hbm_bpns = (float)cm.hbm_bytes_per_ns;
  S.lanes = 2 * Dc->num_sms;
  S.H = Dc->H;
  S.KVH = Dc->KVH;
  S.d = Dc->d;
  S.G = G;
  DevPlan& P = Dc->plan;
  P.pack_q_off = w.p_qoff;
  P.pack_q = w.p_q;
  P.pack_blk_off = S.pack_blk_off;
  P.pack_blk = S.pack_blk;
  P.unit_pack = S.unit_pack;
  P.unit_page0 = S.unit_page0;
  P.unit_ntok = S.unit_ntok;
  P.unit_slot_off = S.unit_slot_off;
  P.unit_slot = S.unit_slot;
  for (int v = 0; v < NUM_VARIANTS; ++v) P.items[v] = S.items;
  P.n_items = S.n_items;
  P.n_pair = S.n_pair;
  P.merge_desc = S.merge_desc;
  P.n_merge = S.n_merge;
  P.H = Dc->H;
  P.KVH = Dc->KVH;
  P.d = Dc->d;
  P.G = G;
  P.bs = block_size;
  if (cudaDeviceSynchronize() != cudaSuccess) {
    set_error("pat_decoder_create: device initialisation failed");
    cudaFree(Dc->arena);
    delete Dc;
    return PAT_ERR_CUDA;
  }
  *out = Dc;
  return PAT_OK;
}

size_t pat_decoder_workspace_bytes(const pat_decoder* Dc) {
  if (!Dc) return 0;
  const size_t so = (size_t)Dc->S.cap_slots * Dc->H * Dc->d * 4, sl = (size_t)Dc->S.cap_slots * Dc->H * 4;
  return ((so + 255) & ~size_t(255)) + ((sl + 255) & ~size_t(255)) + 256;
}

int pat_decoder_forward(pat_decoder* Dc, const int32_t* block_tables, int64_t bt_stride, const int32_t* seq_lens,
                        int32_t B, int32_t max_blocks, const void* q, const void* k_cache, const void* v_cache,
                        int64_t num_pool_blocks, void* out, void* workspace, size_t workspace_bytes, int32_t dtype,
                        float scale, int32_t flags, void* stream) {
  using namespace pat;
  if (!Dc) return PAT_ERR_INVALID_SPEC;
  if (B < 0 || B > Dc->Bmax || max_blocks < 1 || max_blocks > Dc->maxb || bt_stride < max_blocks ||
      (B > 0 && (!block_tables || !seq_lens || !q || !k_cache || !v_cache || !out))) {
    set_error("pat_decoder_forward: table of %d x %d exceeds the decoder's %d x %d (or null pointers)", B, max_blocks,
              Dc->Bmax, Dc->maxb);
    return PAT_ERR_SHAPE_MISMATCH;
  }
  if (dtype != PAT_DTYPE_F16 && dtype != PAT_DTYPE_BF16) {
    set_error("dtype must be f16 or bf16");
    return PAT_ERR_NO_FEASIBLE_CONFIG;
  }
  if (workspace_bytes < pat_decoder_workspace_bytes(Dc)) {
    set_error("workspace %zu < required %zu", workspace_bytes, pat_decoder_workspace_bytes(Dc));
    return PAT_ERR_WORKSPACE;
  }
  if (B == 0) return PAT_OK;
  cudaStream_t st = (cudaStream_t)stream;
  CUtensorMap tmk, tmv;
  {
    std::lock_guard<std::mutex> lk(Dc->mu);
    if (Dc->tm_k != k_cache || Dc->tm_v != v_cache || Dc->tm_blocks != num_pool_blocks || Dc->tm_dtype != dtype) {
      const int e1 = make_kv_tensor_map(&Dc->tmk, k_cache, num_pool_blocks, Dc->bs, Dc->KVH, Dc->d, dtype);
      const int e2 = make_kv_tensor_map(&Dc->tmv, v_cache, num_pool_blocks, Dc->bs, Dc->KVH, Dc->d, dtype);
      if (e1 || e2) {
        Dc->tm_k = nullptr;
        set_error("cuTensorMapEncodeTiled failed (%d, %d)", e1, e2);
        return PAT_ERR_CUDA;
      }
      Dc->tm_k = k_cache;
      Dc->tm_v = v_cache;
      Dc->tm_blocks = num_pool_blocks;
      Dc->tm_dtype = dtype;
    }
    tmk = Dc->tmk;
    tmv = Dc->tmv;
  }
  dev::Ws w = Dc->w;
  w.bt = block_tables;
  w.stride = bt_stride;
  w.seq = seq_lens;
  w.B = B;
  w.maxb = max_blocks;
  dev::Sched S = Dc->S;
  S.w = w;
  const int N2 = 2 * B + 2;
  float* po = (float*)workspace;
  const size_t so = ((size_t)Dc->S.cap_slots * Dc->H * Dc->d * 4 + 255) & ~size_t(255);
  float* pl = (float*)((uint8_t*)workspace + so);
  int32_t* sched = (int32_t*)((uint8_t*)workspace + pat_decoder_workspace_bytes(Dc) - 256);
  if (!(flags & PAT_DECODE_SAME_TABLE)) {
    // fingerprint, compare, and (only when the table changed) GPU packer +
    // device schedule: ONE cooperative launch (grid barriers between phases);
    // it also zeroes the forward's claim counters
    int P = 1;
    while (P < std::max(B, max_blocks)) P <<= 1;
    int PB = 1;
    while (PB < B) PB <<= 1;
    const int dyn = plan_smem(P, PB, 2 * Dc->Bmax + 2);
    dev::PlanState ps{Dc->h_new, Dc->h_old, Dc->run, Dc->nrun, Dc->bar, sched};
    int n2 = N2, dynb = dyn;
    void* args[] = {(void*)&w, (void*)&S, (void*)&ps, (void*)&n2, (void*)&dynb};
    cudaError_t le = cudaLaunchCooperativeKernel((const void*)dev::k_plan, dim3(Dc->plan_grid), dim3(1024), args,
                                                 (size_t)dyn, st);
    if (le != cudaSuccess) {
      set_error("pat_decoder_forward: planner launch: %s", cudaGetErrorString(le));
      return PAT_ERR_CUDA;
    }
  } else if (cudaMemsetAsync(sched, 0, 16, st) != cudaSuccess) {
    set_error("pat_decoder_forward: counter reset failed");
    return PAT_ERR_CUDA;
  }
  // forward + merge over the device plan (counts read on the device)
  if (scale <= 0.f) scale = 1.0f / sqrtf((float)Dc->d);
  const float scale_log2 = scale * 1.4426950408889634f;
  cudaError_t e = launch_forward_tc(tmk, tmv, Dc->plan, VAR_TC, Dc->num_sms, dtype, Dc->d, q, out, po, pl, scale_log2,
                                    sched, st);
  if (e == cudaSuccess) e = launch_merge(Dc->plan, Dc->num_sms * 8, dtype, Dc->d, po, pl, out, st);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("pat_decoder_forward: %s", cudaGetErrorString(e));
    return PAT_ERR_CUDA;
  }
  return PAT_OK;
}

int pat_decoder_status(pat_decoder* Dc, void* stream, int32_t* replans) {
  if (!Dc) return PAT_ERR_INVALID_SPEC;
  int32_t err[2] = {0, 0}, n = 0;
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemcpyAsync(err, Dc->w.err, 8, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&n, Dc->nrun, 4, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) {
    pat::set_error("pat_decoder_status: %s", cudaGetErrorString(cudaGetLastError()));
    return PAT_ERR_CUDA;
  }
  if (replans) *replans = n;
  if (err[0] == PAT_ERR_INVALID_SPEC) pat::set_error("row %d: empty, too long, or repeats a block ID", err[1]);
  else if (err[0]) pat::set_error("query %d: prefix forest deeper than the device packer capacity", err[1]);
  return err[0];
}

void pat_decoder_destroy(pat_decoder* Dc) {
  if (!Dc) return;
  if (Dc->arena) cudaFree(Dc->arena);
  delete Dc;
}

}  // extern "C"

// Debug / test export of the device plan (synchronising copy of one array).
//  what: 0 npacks[1] 1 p_qoff 2 p_q 3 pack_blk_off 4 pack_blk 5 unit_pack 6 unit_page0
//        7 unit_ntok 8 unit_slot_off 9 unit_slot 10 items (8 ints each) 11 n_items[4]
//        12 merge_desc (4 ints each) 13 n_merge[1] 14 p_node 15 parts
#ifdef PAT_TC_TRACE
extern "C" int pat_debug_plan_stamps(long long* host) {
  int e = (int)cudaMemcpyFromSymbol(host, pat::dev::g_plan_stamp, sizeof(pat::dev::g_plan_stamp));
  if (!e) e = (int)cudaMemcpyFromSymbol(host + 32, pat::dev::g_sched_stamp, sizeof(pat::dev::g_sched_stamp));
  return e;
}
#endif

extern "C" int pat_decoder_debug_export(pat_decoder* Dc, int32_t what, int32_t* host, int64_t n_ints) {
  if (!Dc || !host) return PAT_ERR_INVALID_SPEC;
  const void* src = nullptr;
  switch (what) {
    case 0: src = Dc->w.npacks; break;
    case 1: src = Dc->w.p_qoff; break;
    case 2: src = Dc->w.p_q; break;
    case 3: src = Dc->S.pack_blk_off; break;
    case 4: src = Dc->S.pack_blk; break;
    case 5: src = Dc->S.unit_pack; break;
    case 6: src = Dc->S.unit_page0; break;
    case 7: src = Dc->S.unit_ntok; break;
    case 8: src = Dc->S.unit_slot_off; break;
    case 9: src = Dc->S.unit_slot; break;
    case 10: src = Dc->S.items; break;
    case 11: src = Dc->S.n_items; break;
    case 12: src = Dc->S.merge_desc; break;
    case 13: src = Dc->S.n_merge; break;
    case 14: src = Dc->w.p_node; break;
    case 15: src = Dc->S.parts; break;
    default: return PAT_ERR_INVALID_SPEC;
  }
  return cudaMemcpy(host, src, (size_t)n_ints * 4, cudaMemcpyDeviceToHost) == cudaSuccess ? PAT_OK : PAT_ERR_CUDA;
}
