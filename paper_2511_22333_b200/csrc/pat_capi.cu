// C ABI: plan creation (host packer / explicit units / device packer), export,
// and the forward launcher (multi-stream, one stream per kernel variant).
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "pat_plan_host.h"

namespace pat {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

cudaError_t launch_forward_variant(const CUtensorMap& tmk, const CUtensorMap& tmv, const DevPlan& plan, int var,
                                   int grid, int dtype, int d, const void* q, void* out, float* po, float* pl,
                                   float scale_log2, cudaStream_t st);
cudaError_t launch_merge(const DevPlan& plan, int grid, int dtype, int d, const float* po, const float* pl,
                         void* out, cudaStream_t st);
cudaError_t launch_forward_tc(const CUtensorMap& tmk, const CUtensorMap& tmv, const DevPlan& plan, int var, int grid,
                              int dtype, int d, const void* q, void* out, float* po, float* pl, float scale_log2,
                              int32_t* sched, cudaStream_t st);
int device_pack(const int32_t* d_bt, int64_t stride, const int32_t* d_seq, int B, int maxb, int bs, cudaStream_t st,
                HostPacks* out, std::vector<int32_t>* h_nblk, std::vector<int32_t>* h_valid,
                std::vector<int32_t>* h_rows);

// ------------------------------------------------------------------------------------------
// TMA descriptors over the paged cache
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

}  // namespace pat

using namespace pat;

#define CUDA_TRY(expr)                                                              \
  do {                                                                              \
    cudaError_t e_ = (expr);                                                        \
    if (e_ != cudaSuccess) {                                                        \
      set_error("%s failed: %s", #expr, cudaGetErrorString(e_));                    \
      return PAT_ERR_CUDA;                                                          \
    }                                                                               \
  } while (0)

struct pat_plan {
  int B = 0, bs = 16, H = 0, KVH = 0, d = 0, split_mode = 0, num_sms = 148, tc_min_rows = 64;
  bool tc_auto = false;  // tc_min_rows left to the library (options value 0)
  bool forward_only = false;  // PAT_PLAN_FORWARD_ONLY
  bool on_device = false;
  HostPacks packs;
  HostSchedule sched;
  int64_t unique_tokens = 0;
  int32_t n_items_total = 0, n_slots = 0, n_merge = 0;
  int32_t items_cap[NUM_VARIANTS] = {};
  // device
  void* dmem = nullptr;
  DevPlan dev{};
  int device = -1;
  // Host-side caches of pat_forward (the plan itself is immutable after
  // creation): the fork/join streams of a multi-variant plan and the TMA
  // descriptors of the last (k_cache, v_cache) pair, both under `mu`, so one
  // plan may be launched from several threads / streams concurrently.
  std::mutex mu;
  cudaStream_t streams[NUM_VARIANTS] = {};
  cudaEvent_t ev_fork = nullptr, ev_join[NUM_VARIANTS] = {};
  CUtensorMap tmk, tmv;
  const void* tm_k = nullptr;
  const void* tm_v = nullptr;
  int64_t tm_blocks = -1;
  int tm_dtype = -1;
};

namespace {

int check_opts(const pat_plan_options* opt) {
  if (!opt) {
    set_error("options are required");
    return PAT_ERR_INVALID_SPEC;
  }
  if (opt->num_kv_heads <= 0 || opt->num_heads <= 0 || opt->num_heads % opt->num_kv_heads != 0) {
    set_error("num_heads must be a positive multiple of num_kv_heads");
    return PAT_ERR_INVALID_SPEC;
  }
  if (opt->head_dim <= 0) {
    set_error("head_dim must be positive");
    return PAT_ERR_INVALID_SPEC;
  }
  if (opt->split_mode < PAT_SPLIT_NONE || opt->split_mode > PAT_SPLIT_NATIVE) {
    set_error("unknown split mode %d", opt->split_mode);
    return PAT_ERR_INVALID_SPEC;
  }
  return PAT_OK;
}

void init_plan(pat_plan* P, int B, int bs, const pat_plan_options* opt) {
  P->B = B;
  P->bs = bs;
  P->H = opt->num_heads;
  P->KVH = opt->num_kv_heads;
  P->d = opt->head_dim;
  P->split_mode = opt->split_mode;
  P->num_sms = opt->num_sms;
  P->tc_auto = opt->tc_min_rows == 0;
  P->forward_only = (opt->flags & PAT_PLAN_FORWARD_ONLY) != 0;
  P->tc_min_rows = opt->tc_min_rows == 0 ? 1 : (opt->tc_min_rows < 0 ? 0 : opt->tc_min_rows);
  if (P->d != 64 && P->d != 128) P->tc_min_rows = 0;
  if (P->num_sms <= 0) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0)
      P->num_sms = n;
    else
      P->num_sms = 148;
    cudaGetLastError();
  }
}

// Concatenate host arrays into one device allocation.
struct Blob {
  std::vector<uint8_t> bytes;
  size_t add(const void* p, size_t n) {
    size_t off = (bytes.size() + 255) & ~size_t(255);
    bytes.resize(off + std::max<size_t>(n, 4));
    if (n) memcpy(bytes.data() + off, p, n);
    return off;
  }
  template <typename V>
  size_t addv(const V& v) { return add(v.data(), v.size() * sizeof(v[0])); }
};

int upload(pat_plan* P) {
  const HostPacks& pk = P->packs;
  const HostSchedule& s = P->sched;
  Blob b;
  size_t o_pq_off = b.addv(pk.q_off), o_pq = b.addv(pk.q), o_pb_off = b.addv(pk.blk_off), o_pb = b.addv(pk.blk);
  size_t o_up = b.addv(s.unit_pack), o_u0 = b.addv(s.unit_page0), o_ut = b.addv(s.unit_ntok);
  size_t o_uso = b.addv(s.unit_slot_off), o_us = b.addv(s.unit_slot);
  size_t o_it[NUM_VARIANTS];
  int32_t nit[NUM_VARIANTS];
  for (int v = 0; v < NUM_VARIANTS; ++v) {
    o_it[v] = b.addv(s.items[v]);
    nit[v] = (int32_t)s.items[v].size();
    P->items_cap[v] = nit[v];
  }
  size_t o_nit = b.add(nit, sizeof(nit));
  size_t o_npr = b.add(s.n_pair, sizeof(s.n_pair));
  size_t o_mq = b.addv(s.merge_q), o_qso = b.addv(s.q_slot_off), o_qn = b.addv(s.q_nslot);
  std::vector<int32_t> mdesc;
  for (int32_t q : s.merge_q) mdesc.insert(mdesc.end(), {q, s.q_slot_off[q], s.q_nslot[q], 0});
  size_t o_md = b.addv(mdesc);
  int32_t nm = (int32_t)s.merge_q.size();
  size_t o_nm = b.add(&nm, sizeof(nm));
  const int32_t zeros[16] = {};
  size_t o_sched = b.add(zeros, sizeof(zeros));
  CUDA_TRY(cudaGetDevice(&P->device));
  CUDA_TRY(cudaMalloc(&P->dmem, b.bytes.size()));
  CUDA_TRY(cudaMemcpy(P->dmem, b.bytes.data(), b.bytes.size(), cudaMemcpyHostToDevice));
  uint8_t* base = (uint8_t*)P->dmem;
  DevPlan& D = P->dev;
  D.pack_q_off = (const int32_t*)(base + o_pq_off);
  D.pack_q = (const int32_t*)(base + o_pq);
  D.pack_blk_off = (const int32_t*)(base + o_pb_off);
  D.pack_blk = (const int32_t*)(base + o_pb);
  D.unit_pack = (const int32_t*)(base + o_up);
  D.unit_page0 = (const int32_t*)(base + o_u0);
  D.unit_ntok = (const int32_t*)(base + o_ut);
  D.unit_slot_off = (const int32_t*)(base + o_uso);
  D.unit_slot = (const int32_t*)(base + o_us);
  for (int v = 0; v < NUM_VARIANTS; ++v) D.items[v] = (const Item*)(base + o_it[v]);
  D.n_items = (const int32_t*)(base + o_nit);
  D.n_pair = (const int32_t*)(base + o_npr);
  D.merge_q = (const int32_t*)(base + o_mq);
  D.merge_desc = (const int4*)(base + o_md);
  D.q_slot_off = (const int32_t*)(base + o_qso);
  D.q_nslot = (const int32_t*)(base + o_qn);
  D.n_merge = (const int32_t*)(base + o_nm);
  D.sched = (int32_t*)(base + o_sched);
  D.H = P->H;
  D.KVH = P->KVH;
  D.d = P->d;
  D.G = P->H / P->KVH;
  D.bs = P->bs;
  P->on_device = true;
  return PAT_OK;
}

int finish_plan(pat_plan* P, const RowsView& R, int flags) {
  // Kernel choice (options value 0): every pack goes to the tcgen05 kernel --
  // one persistent kernel with dynamic load balance, narrow packs transposed.
  // (Round 1 kept the mma.sync streaming kernel for plans without a pack wider
  // than 16 rows; the round-2 narrow path is faster there too: c5 622 vs 688 us.)
  if (P->tc_auto) P->tc_min_rows = 1;
  ScheduleParams sp{P->B, P->bs, P->H, P->KVH, P->d, P->split_mode, P->num_sms, P->tc_min_rows};
  sp.pair_items = (flags & PAT_PLAN_PAIR_ITEMS) != 0;
  sp.all_partials = (flags & PAT_PLAN_ALL_PARTIALS) != 0;
  int st = host_schedule(P->packs, sp, &P->sched);
  if (st) return st;
  P->n_slots = P->sched.n_slots;
  P->n_merge = (int32_t)P->sched.merge_q.size();
  P->n_items_total = 0;
  for (int v = 0; v < NUM_VARIANTS; ++v) P->n_items_total += (int32_t)P->sched.items[v].size();
  P->unique_tokens = distinct_tokens(R);
  if (!(flags & PAT_PLAN_HOST_ONLY)) return upload(P);
  return PAT_OK;
}

std::vector<int32_t> nblk_from_off(int B, const int64_t* off) {
  std::vector<int32_t> n(B);
  for (int q = 0; q < B; ++q) n[q] = (int32_t)(off[q + 1] - off[q]);
  return n;
}

}  // namespace

extern "C" {

const char* pat_last_error(void) { return g_err; }

const char* pat_version(void) { return "patb200 0.1.0 (sm_100a)"; }

int pat_plan_create_host(int32_t B, const int64_t* row_off, const int32_t* row_blk, const int32_t* valid_last,
                         int32_t block_size, const pat_plan_options* opt, pat_plan** out) {
  if (!out) return PAT_ERR_INVALID_SPEC;
  *out = nullptr;
  int st = check_opts(opt);
  if (st) return st;
  if (B < 0 || (B > 0 && (!row_off || !row_blk || !valid_last))) {
    set_error("bad table arguments");
    return PAT_ERR_SHAPE_MISMATCH;
  }
  std::vector<int32_t> nb = nblk_from_off(B, row_off);
  RowsView R{row_blk, row_off, 0, nb.data(), valid_last, B, block_size};
  pat_plan* P = new pat_plan();
  init_plan(P, B, block_size, opt);
  st = host_pack(R, &P->packs);
  if (!st) st = finish_plan(P, R, opt->flags);
  if (st) {
    pat_plan_destroy(P);
    return st;
  }
  *out = P;
  return PAT_OK;
}

int pat_plan_create_units(int32_t B, const int64_t* row_off, const int32_t* row_blk, const int32_t* valid_last,
                          int32_t block_size, int32_t n_units, const int64_t* unit_q_off, const int32_t* unit_q,
                          const int64_t* unit_blk_off, const int32_t* unit_blk, const int32_t* unit_kv,
                          const pat_plan_options* opt, pat_plan** out) {
  if (!out) return PAT_ERR_INVALID_SPEC;
  *out = nullptr;
  int st = check_opts(opt);
  if (st) return st;
  std::vector<int32_t> nb = nblk_from_off(B, row_off);
  RowsView R{row_blk, row_off, 0, nb.data(), valid_last, B, block_size};
  st = validate_rows(R);
  if (st) return st;
  // Coverage (attention.py:258-269): per query, the multiset of unit blocks equals
  // its row and the unit tokens sum to kv_len.
  std::vector<std::vector<int32_t>> got(B);
  std::vector<int64_t> tok(B, 0);
  for (int u = 0; u < n_units; ++u) {
    if (unit_kv[u] < 1) {
      set_error("unit %d covers zero tokens", u);
      return PAT_ERR_EMPTY_SPAN;
    }
    for (int64_t i = unit_q_off[u]; i < unit_q_off[u + 1]; ++i) {
      int q = unit_q[i];
      if (q < 0 || q >= B) {
        set_error("unknown query %d", q);
        return PAT_ERR_COVERAGE_GAP;
      }
      got[q].insert(got[q].end(), unit_blk + unit_blk_off[u], unit_blk + unit_blk_off[u + 1]);
      tok[q] += unit_kv[u];
    }
  }
  for (int q = 0; q < B; ++q) {
    std::vector<int32_t> row(row_blk + row_off[q], row_blk + row_off[q + 1]);
    std::sort(row.begin(), row.end());
    std::sort(got[q].begin(), got[q].end());
    int64_t kv = (int64_t)(nb[q] - 1) * block_size + valid_last[q];
    if (row != got[q] || tok[q] != kv) {
      set_error("query %d: KV span not exactly covered", q);
      return PAT_ERR_COVERAGE_GAP;
    }
  }
  pat_plan* P = new pat_plan();
  init_plan(P, B, block_size, opt);
  HostPacks& pk = P->packs;
  pk.clear();
  std::vector<int32_t> memb(B, 0);
  for (int u = 0; u < n_units; ++u)
    for (int64_t i = unit_q_off[u]; i < unit_q_off[u + 1]; ++i) memb[unit_q[i]]++;
  for (int u = 0; u < n_units; ++u) {
    uint8_t partial = 0;
    for (int64_t i = unit_q_off[u]; i < unit_q_off[u + 1]; ++i) {
      pk.q.push_back(unit_q[i]);
      partial |= memb[unit_q[i]] > 1;
    }
    pk.q_off.push_back((int32_t)pk.q.size());
    pk.blk.insert(pk.blk.end(), unit_blk + unit_blk_off[u], unit_blk + unit_blk_off[u + 1]);
    pk.blk_off.push_back((int32_t)pk.blk.size());
    pk.kv.push_back(unit_kv[u]);
    pk.partial.push_back(partial);
    pk.rep.push_back(-1);
    pk.blk_begin.push_back(-1);
  }
  st = finish_plan(P, R, opt->flags);
  if (st) {
    pat_plan_destroy(P);
    return st;
  }
  *out = P;
  return PAT_OK;
}

int pat_plan_info_get(const pat_plan* P, pat_plan_info* info) {
  if (!P || !info) return PAT_ERR_INVALID_SPEC;
  info->num_queries = P->B;
  info->block_size = P->bs;
  info->n_packs = P->packs.n_packs();
  info->n_pack_q = (int32_t)P->packs.q.size();
  info->n_pack_blk = (int32_t)P->packs.blk.size();
  info->n_units = (int32_t)P->sched.unit_pack.size();
  info->n_items = P->n_items_total;
  info->n_slots = P->n_slots;
  info->n_merge_q = P->n_merge;
  info->on_device = P->on_device ? 1 : 0;
  info->unique_tokens = P->unique_tokens;
  info->n_fwd_kernels = 0;
  for (int v = 0; v < NUM_VARIANTS; ++v) info->n_fwd_kernels += P->sched.items[v].empty() ? 0 : 1;
  info->n_launches = info->n_fwd_kernels + (P->n_merge > 0 ? 1 : 0);
  return PAT_OK;
}

int pat_plan_export_packs(const pat_plan* P, int32_t* q_off, int32_t* q_ids, int32_t* blk_off, int32_t* blk_ids,
                          int32_t* kv_len, uint8_t* partial) {
  if (!P) return PAT_ERR_INVALID_SPEC;
  const HostPacks& pk = P->packs;
  if (q_off) memcpy(q_off, pk.q_off.data(), pk.q_off.size() * 4);
  if (q_ids) memcpy(q_ids, pk.q.data(), pk.q.size() * 4);
  if (blk_off) memcpy(blk_off, pk.blk_off.data(), pk.blk_off.size() * 4);
  if (blk_ids) memcpy(blk_ids, pk.blk.data(), pk.blk.size() * 4);
  if (kv_len) memcpy(kv_len, pk.kv.data(), pk.kv.size() * 4);
  if (partial) memcpy(partial, pk.partial.data(), pk.partial.size());
  return PAT_OK;
}

int pat_plan_export_units(const pat_plan* P, int32_t* pack, int32_t* page0, int32_t* npages, int32_t* ntok,
                          int32_t* split_index, int32_t* split_of) {
  if (!P) return PAT_ERR_INVALID_SPEC;
  const HostSchedule& s = P->sched;
  size_t n = s.unit_pack.size() * 4;
  if (pack) memcpy(pack, s.unit_pack.data(), n);
  if (page0) memcpy(page0, s.unit_page0.data(), n);
  if (npages) memcpy(npages, s.unit_npages.data(), n);
  if (ntok) memcpy(ntok, s.unit_ntok.data(), n);
  if (split_index) memcpy(split_index, s.unit_split_idx.data(), n);
  if (split_of) memcpy(split_of, s.unit_split_of.data(), n);
  return PAT_OK;
}

size_t pat_workspace_bytes(const pat_plan* P) {
  if (!P) return 0;
  size_t so = (size_t)P->n_slots * P->H * P->d * sizeof(float);
  size_t sl = (size_t)P->n_slots * P->H * sizeof(float);
  // fp32 partials (o / l, log2-sum-exp), then 256 bytes of per-launch item
  // counters (zeroed by pat_forward on the caller's stream)
  return ((so + 255) & ~size_t(255)) + ((sl + 255) & ~size_t(255)) + 256;
}

int pat_forward(const pat_plan* Pc, const void* q, const void* k_cache, const void* v_cache, int64_t num_pool_blocks,
                void* out, void* workspace, size_t workspace_bytes, int32_t dtype, float scale, void* stream) {
  pat_plan* P = const_cast<pat_plan*>(Pc);
  if (!P || !P->on_device) {
    set_error("plan is not on the device");
    return PAT_ERR_INVALID_SPEC;
  }
  if (P->d != 128 && P->d != 64) {
    set_error("no forward kernel for head_dim %d (have 64, 128)", P->d);
    return PAT_ERR_NO_FEASIBLE_CONFIG;
  }
  if (P->bs % 16 != 0) {
    set_error("block_size %d must be a multiple of 16", P->bs);
    return PAT_ERR_NO_FEASIBLE_CONFIG;
  }
  if (dtype != PAT_DTYPE_F16 && dtype != PAT_DTYPE_BF16) {
    set_error("dtype must be f16 or bf16");
    return PAT_ERR_NO_FEASIBLE_CONFIG;
  }
  if (P->B == 0) return PAT_OK;
  if (workspace_bytes < pat_workspace_bytes(P)) {
    set_error("workspace %zu < required %zu", workspace_bytes, pat_workspace_bytes(P));
    return PAT_ERR_WORKSPACE;
  }
  (void)num_pool_blocks;
  cudaStream_t st = (cudaStream_t)stream;
  float* po = (float*)workspace;
  size_t so = ((size_t)P->n_slots * P->H * P->d * sizeof(float) + 255) & ~size_t(255);
  float* pl = (float*)((uint8_t*)workspace + so);
  if (scale <= 0.f) scale = 1.0f / sqrtf((float)P->d);
  const float scale_log2 = scale * 1.4426950408889634f;

  int active[NUM_VARIANTS], na = 0;
  for (int v = 0; v < NUM_VARIANTS; ++v)
    if (P->items_cap[v] > 0) active[na++] = v;
  // the dynamic item counters of this launch live in the caller's workspace:
  // launches on different streams with different workspaces never share them
  int32_t* sched = (int32_t*)((uint8_t*)workspace + pat_workspace_bytes(P) - 256);
  CUDA_TRY(cudaMemsetAsync(sched, 0, 16, st));
  CUtensorMap tmk, tmv;
  {
    std::lock_guard<std::mutex> lk(P->mu);
    if ((P->tm_k != k_cache || P->tm_v != v_cache || P->tm_blocks != num_pool_blocks || P->tm_dtype != dtype)) {
      int e1 = make_kv_tensor_map(&P->tmk, k_cache, num_pool_blocks, P->bs, P->KVH, P->d, dtype);
      int e2 = make_kv_tensor_map(&P->tmv, v_cache, num_pool_blocks, P->bs, P->KVH, P->d, dtype);
      if (e1 || e2) {
        P->tm_k = nullptr;
        set_error("cuTensorMapEncodeTiled failed (%d, %d)", e1, e2);
        return PAT_ERR_CUDA;
      }
      P->tm_k = k_cache;
      P->tm_v = v_cache;
      P->tm_blocks = num_pool_blocks;
      P->tm_dtype = dtype;
    }
    tmk = P->tmk;
    tmv = P->tmv;
    if (na > 1 && !P->ev_fork) {
      CUDA_TRY(cudaEventCreateWithFlags(&P->ev_fork, cudaEventDisableTiming));
      for (int v = 0; v < NUM_VARIANTS; ++v) {
        CUDA_TRY(cudaStreamCreateWithFlags(&P->streams[v], cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreateWithFlags(&P->ev_join[v], cudaEventDisableTiming));
      }
    }
  }
  // Concurrent variants get disjoint SM shares proportional to their estimated
  // work (every forward kernel is persistent with one CTA per SM, and the
  // tcgen05 and streaming CTAs cannot share an SM's shared memory).
  double wsum = 0;
  for (int i = 0; i < na; ++i) wsum += P->sched.work[active[i]];
  auto grid_of = [&](int v) {
    double share = na > 1 && wsum > 0 ? P->sched.work[v] / wsum : 1.0;
    int g = (int)(P->num_sms * share + 0.5);
    return std::max(1, std::min(std::max(g, 1), P->items_cap[v]));
  };
  auto launch = [&](int v, cudaStream_t sv) -> cudaError_t {
    const int grid = grid_of(v);
    if (v == VAR_TC)
      return launch_forward_tc(tmk, tmv, P->dev, v, grid, dtype, P->d, q, out, po, pl, scale_log2, sched, sv);
    return launch_forward_variant(tmk, tmv, P->dev, v, grid, dtype, P->d, q, out, po, pl, scale_log2, sv);
  };
  if (na == 1) {
    CUDA_TRY(launch(active[0], st));
  } else if (na > 1) {
    // multi-stream forward (section 6): one stream per kernel config,
    // forked from and joined back into the caller's stream (the plan's fork /
    // join objects: concurrent multi-variant launches of ONE plan serialise on
    // them through the stream order of their records, as CUDA events do).
    CUDA_TRY(cudaEventRecord(P->ev_fork, st));
    for (int i = 0; i < na; ++i) {
      int v = active[i];
      cudaStream_t sv = i == 0 ? st : P->streams[v];
      if (i) CUDA_TRY(cudaStreamWaitEvent(sv, P->ev_fork, 0));
      CUDA_TRY(launch(v, sv));
      if (i) CUDA_TRY(cudaEventRecord(P->ev_join[v], sv));
    }
    for (int i = 1; i < na; ++i) CUDA_TRY(cudaStreamWaitEvent(st, P->ev_join[active[i]], 0));
  }
  if (P->n_merge > 0 && !P->forward_only) {
    int warps = P->n_merge * P->H;
    int grid = std::max(1, std::min((warps + 7) / 8, P->num_sms * 8));
    CUDA_TRY(launch_merge(P->dev, grid, dtype, P->d, po, pl, out, st));
  }
  return PAT_OK;
}

void pat_plan_destroy(pat_plan* P) {
  if (!P) return;
  if (P->dmem) cudaFree(P->dmem);
  for (int v = 0; v < NUM_VARIANTS; ++v) {
    if (P->streams[v]) cudaStreamDestroy(P->streams[v]);
    if (P->ev_join[v]) cudaEventDestroy(P->ev_join[v]);
  }
  if (P->ev_fork) cudaEventDestroy(P->ev_fork);
  delete P;
}

int pat_plan_create_device(int32_t B, const int32_t* block_tables, int64_t bt_stride, const int32_t* seq_lens,
                           int32_t max_blocks, int32_t block_size, const pat_plan_options* opt, void* stream,
                           pat_plan** out) {
  if (!out) return PAT_ERR_INVALID_SPEC;
  *out = nullptr;
  int st = check_opts(opt);
  if (st) return st;
  if (B < 0 || max_blocks < 1 || bt_stride < max_blocks || block_size <= 0 || (B > 0 && (!block_tables || !seq_lens))) {
    set_error("bad block-table arguments");
    return PAT_ERR_SHAPE_MISMATCH;
  }
  pat_plan* P = new pat_plan();
  init_plan(P, B, block_size, opt);
  std::vector<int32_t> nblk, valid, rows;
  st = device_pack(block_tables, bt_stride, seq_lens, B, max_blocks, block_size, (cudaStream_t)stream, &P->packs,
                   &nblk, &valid, &rows);
  if (!st) {
    RowsView R{rows.data(), nullptr, bt_stride, nblk.data(), valid.data(), B, block_size};
    st = finish_plan(P, R, opt->flags);
  }
  if (st) {
    pat_plan_destroy(P);
    return st;
  }
  *out = P;
  return PAT_OK;
}

}  // extern "C"
