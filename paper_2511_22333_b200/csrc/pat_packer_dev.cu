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
#include <cstdio>
#include <vector>

#include "pat_plan_host.h"

namespace pat {
namespace dev {

struct Ws {
  // inputs
  const int32_t* bt;
  int64_t stride;
  const int32_t* seq;
  int B, bs, maxb, D;  // D = level capacity per query
  // per query
  int32_t* nblk;
  int32_t* valid;
  int32_t* err;     // [0] status, [1] row
  int32_t* lcp;     // [B*B]
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

__device__ __forceinline__ int tok_at(const Ws& w, int q, int p) { return p == w.nblk[q] - 1 ? w.valid[q] : w.bs; }
__device__ __forceinline__ int blk_at(const Ws& w, int q, int p) { return w.bt[(int64_t)q * w.stride + p]; }

__global__ void k_rows(Ws w) {
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= w.B) return;
  int s = w.seq[q];
  int n = s > 0 ? (s + w.bs - 1) / w.bs : 0;
  w.nblk[q] = n;
  w.valid[q] = s - (n - 1) * w.bs;
  if (n <= 0 || n > w.maxb) {
    if (atomicCAS(&w.err[0], 0, PAT_ERR_INVALID_SPEC) == 0) w.err[1] = q;
  }
}

// one CTA per row: bitonic sort of the row's block ids in smem, adjacent compare
__global__ void k_dup(Ws w) {
  extern __shared__ int32_t sbuf[];
  const int q = blockIdx.x;
  const int n = min(w.nblk[q], w.maxb);
  if (n <= 1) return;
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
}

// one warp per (q, r) pair with q < r
__global__ void k_lcp(Ws w) {
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
    int l = n;
    for (int p0 = 0; p0 < n; p0 += 32) {
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

// one CTA per query: sort (lcp, r) keys, derive the internal levels
__global__ void k_levels(Ws w) {
  extern __shared__ unsigned long long skey[];
  const int q = blockIdx.x;
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
  // serial pass over the (few) entries by one thread keeps this simple and exact
  if (threadIdx.x == 0) {
    int M = 0;
    while (M < w.B && skey[M] != ~0ull) ++M;
    int Kq = 0;
    const int nbq = w.nblk[q];
    int sufmin = q;
    // distinct lcp values front to back (ascending): one internal level each
    int i = 0;
    while (i < M) {
      const int v = (int)(skey[i] >> 32);
      int j = i;
      int tcount = 0;
      while (j < M && (int)(skey[j] >> 32) == v) {
        const int r = (int)(skey[j] & 0xffffffffu);
        if (w.nblk[r] == v) ++tcount;
        ++j;
      }
      if (Kq >= w.D) {
        if (atomicCAS(&w.err[0], 0, PAT_ERR_NO_FEASIBLE_CONFIG) == 0) w.err[1] = q;
        return;
      }
      w.end[(int64_t)q * w.D + Kq] = v;
      w.nq[(int64_t)q * w.D + Kq] = 1 + (M - i);
      w.term[(int64_t)q * w.D + Kq] = tcount + (nbq == v ? 1 : 0);
      w.minq[(int64_t)q * w.D + Kq] = i;  // placeholder: group start, resolved below
      ++Kq;
      i = j;
    }
    // resolve minimum member of {r : lcp >= end_k} u {q} via a backward suffix min
    int k = Kq - 1;
    for (int e = M - 1; e >= 0 && k >= 0; --e) {
      sufmin = min(sufmin, (int)(skey[e] & 0xffffffffu));
      while (k >= 0 && w.minq[(int64_t)q * w.D + k] == e) {
        w.minq[(int64_t)q * w.D + k] = sufmin;
        --k;
      }
    }
    w.K[q] = Kq;
    w.hasleaf[q] = (Kq == 0) || w.end[(int64_t)q * w.D + Kq - 1] < nbq;
  }
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
__global__ void k_decide(Ws w) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= w.B) return;
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

// lexicographic key element e of query q: e=0 root group min, e=1+k slot at level k
__device__ __forceinline__ int key_at(const Ws& w, int q, int e) {
  const int K = w.K[q];
  if (e == 0) return K > 0 ? w.minq[(int64_t)q * w.D] : q;
  const int k = e - 1;
  if (w.end[(int64_t)q * w.D + k] == w.nblk[q]) return q;
  return w.B + (k + 1 < K ? w.minq[(int64_t)q * w.D + k + 1] : q);
}

// warp per query: pi(q) = #{r : key(r) < key(q)}
__global__ void k_rank(Ws w) {
  const int q = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x & 31;
  if (q >= w.B) return;
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

// single CTA exclusive scan of cnt_own -> base
__global__ void k_scan_nodes(Ws w) {
  __shared__ int32_t part[1024];
  const int t = threadIdx.x, n = w.B;
  const int per = (n + blockDim.x - 1) / blockDim.x;
  int s = 0;
  for (int i = t * per; i < min(n, (t + 1) * per); ++i) s += w.cnt_own[i];
  part[t] = s;
  __syncthreads();
  if (t == 0) {
    int acc = 0;
    for (int i = 0; i < (int)blockDim.x; ++i) {
      int v = part[i];
      part[i] = acc;
      acc += v;
    }
    w.base[n] = acc;
  }
  __syncthreads();
  int acc = part[t];
  for (int i = t * per; i < min(n, (t + 1) * per); ++i) {
    w.base[i] = acc;
    acc += w.cnt_own[i];
  }
}

__device__ __forceinline__ int node_id(const Ws& w, int q, int k) {
  const int m = owner_of(w, q, k);
  return w.base[m] + k - w.k0[m];
}

__global__ void k_nodes_init(Ws w) {
  const int N = w.base[w.B];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    w.n_hi[i] = 0;
    w.n_lo[i] = 0x7fffffff;
    w.n_cnt[i] = 0;
    w.n_pack[i] = -1;
  }
}

// thread per query: every level it passes through
__global__ void k_nodes(Ws w) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= w.B) return;
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

// thread per node: rank among emitting nodes by (hi asc, depth desc)
__global__ void k_order(Ws w) {
  const int N = w.base[w.B];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    if (w.n_cnt[i] == 0) continue;
    const int hi = w.n_hi[i], dp = w.n_depth[i];
    int r = 0;
    for (int j = 0; j < N; ++j) {
      if (j == i || w.n_cnt[j] == 0) continue;
      const int hj = w.n_hi[j], dj = w.n_depth[j];
      r += (hj < hi) || (hj == hi && dj > dp);
    }
    w.n_pack[i] = r;
    w.p_node[r] = i;
    atomicAdd(w.npacks, 1);
  }
}

// single thread: query offsets per pack (packs <= 2B)
__global__ void k_pack_offsets(Ws w) {
  const int np = *w.npacks;
  int acc = 0;
  for (int p = 0; p < np; ++p) {
    w.p_qoff[p] = acc;
    acc += w.n_cnt[w.p_node[p]];
    w.p_partial[p] = 0;
  }
  w.p_qoff[np] = acc;
}

// thread per query: place it in each pack it belongs to, in pi order
__global__ void k_members(Ws w) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= w.B) return;
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
  fields = {{&w.nblk, (size_t)B}, {&w.valid, (size_t)B}, {&w.err, 2}, {&w.lcp, BB}, {&w.K, (size_t)B},
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
  const int dup_smem = std::max(P, 1) * 4;
  if (dup_smem > 48 * 1024) cudaFuncSetAttribute(dev::k_dup, cudaFuncAttributeMaxDynamicSharedMemorySize, dup_smem);
  dev::k_dup<<<B, 256, dup_smem, st>>>(w);
  {
    int64_t warps = (int64_t)B * B;
    int grid = (int)std::min<int64_t>((warps * 32 + 255) / 256, 148 * 16);
    dev::k_lcp<<<grid, 256, 0, st>>>(w);
  }
  int PB = 1;
  while (PB < B) PB <<= 1;
  dev::k_levels<<<B, 256, PB * 8, st>>>(w);
  dev::k_decide<<<gq, TB, 0, st>>>(w);
  dev::k_rank<<<(B * 32 + 255) / 256, 256, 0, st>>>(w);
  dev::k_scan_nodes<<<1, 1024, 0, st>>>(w);
  dev::k_nodes_init<<<64, 256, 0, st>>>(w);
  dev::k_nodes<<<gq, TB, 0, st>>>(w);
  dev::k_order<<<64, 256, 0, st>>>(w);
  dev::k_pack_offsets<<<1, 1, 0, st>>>(w);
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
