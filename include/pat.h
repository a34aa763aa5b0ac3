/*
 * pat.h -- C ABI of the B200-native PAT decode-attention library
 * (pack -> multi-tile forward -> merge), libpatb200.so.
 *
 * Plain pointers and sizes only; device pointers are CUDA device addresses,
 * streams are cudaStream_t passed as void*.  Every function returns a status
 * code (PAT_OK = 0); pat_last_error() returns the thread-local message of the
 * last failure on the calling thread.
 *
 * Reference interfaces replaced (all paths under /root/reference/pkg/src/prefixpack):
 *   pat_plan_create_host     <- packer.py:224  pack_batch(table, cache=None) -> Partition
 *                               (build_forest workload.py:245, tree_heuristic packer.py:124,
 *                                assemble_partition workload.py:377) + split_long_kv
 *                                simulator.py:117 when split_mode == PAT_SPLIT_REFERENCE
 *   pat_plan_create_device   <- the same pack_batch, as a GPU pass over device block tables
 *   pat_plan_create_units    <- run_packed_attention(table, partition_or_tasks, ...)
 *                               attention.py:202 with an explicit Partition / [CtaTask] /
 *                               [CtaPack] (coverage check attention.py:258-269)
 *   pat_plan_info / pat_plan_export_packs / pat_plan_export_units
 *                            <- Partition.packs (workload.py:337-362) / CtaTask list
 *                               (simulator.py:99-114)
 *   pat_forward              <- run_packed_attention attention.py:202-239: per-unit
 *                               cta_partial (attention.py:140) + _merge_batch_into
 *                               (attention.py:187) + normalisation (attention.py:237-239)
 *   status codes             <- errors.py:4-45 exception classes
 */
#ifndef PAT_H_
#define PAT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One status code per prefixpack exception class (errors.py). */
enum pat_status {
  PAT_OK = 0,
  PAT_ERR_INVALID_SPEC = 1,       /* InvalidSpec             workload.py:120-132 */
  PAT_ERR_COVERAGE_GAP = 2,       /* CoverageGap             attention.py:258-269 */
  PAT_ERR_EMPTY_SPAN = 3,         /* EmptySpan               attention.py:147-148 */
  PAT_ERR_NON_POSITIVE_DENOM = 4, /* NonPositiveDenominator  attention.py:237-238 */
  PAT_ERR_SHAPE_MISMATCH = 5,     /* ShapeMismatch           attention.py:149-150, 219-220 */
  PAT_ERR_EMPTY_PARTIAL_LIST = 6, /* EmptyPartialList        attention.py:173-174 */
  PAT_ERR_NO_FEASIBLE_CONFIG = 7, /* NoFeasibleConfig: no kernel for this head_dim/page/dtype */
  PAT_ERR_WORKSPACE = 8,          /* workspace smaller than pat_workspace_bytes() */
  PAT_ERR_CUDA = 9,               /* CUDA runtime / driver failure */
  PAT_ERR_INTERNAL = 10
};

enum pat_dtype { PAT_DTYPE_F16 = 0, PAT_DTYPE_BF16 = 1 };

/* KV split policy applied to packs before the forward. */
enum pat_split_mode {
  PAT_SPLIT_NONE = 0,      /* one forward unit per pack */
  PAT_SPLIT_REFERENCE = 1, /* split_long_kv (simulator.py:117-155) exactly: mean over packs */
  PAT_SPLIT_NATIVE = 2     /* B200: chunks sized to fill 148 SMs, capped by merge traffic */
};

enum pat_plan_flags {
  PAT_PLAN_HOST_ONLY = 1,   /* build and keep the plan on the host only (no device upload) */
  PAT_PLAN_FORWARD_ONLY = 2, /* timing aid: pat_forward launches the forward kernel(s) but not
                               the merge (multi-unit queries' outputs are left unwritten) */
  PAT_PLAN_PAIR_ITEMS = 4,   /* tcgen05: run packs wider than 128 rows as 256-row items that both
                               item pipelines of a CTA consume from one KV stream (half the
                               L2 -> SM bytes per row; measured neutral on c4, so opt-in) */
  PAT_PLAN_ALL_PARTIALS = 8  /* every (unit, query) gets an fp32 partial slot (o / l, log2-sum-exp)
                               in the workspace, even for queries covered by one unit; with
                               FORWARD_ONLY this exposes the per-unit partials (cta_partial) */
};

typedef struct pat_plan pat_plan;

typedef struct pat_plan_options {
  int32_t num_heads;    /* H   (query heads)            WorkloadSpec.num_heads    workload.py:27 */
  int32_t num_kv_heads; /* KVH (GQA: head h reads h / (H/KVH)) attention.py:61-67 */
  int32_t head_dim;     /* d */
  int32_t split_mode;   /* pat_split_mode */
  int32_t num_sms;      /* 0 = query the current device */
  int32_t flags;        /* pat_plan_flags */
  int32_t tc_min_rows;  /* packs with >= this many rows (queries x G) use the tcgen05 kernel,
                           the others the mma.sync streaming kernel; 0 = library default
                           (every pack on the tcgen05 kernel, unless no pack has more than
                           16 rows: then all on the streaming kernel), < 0 = never */
} pat_plan_options;

typedef struct pat_plan_info {
  int32_t num_queries;  /* B */
  int32_t block_size;
  int32_t n_packs;      /* Partition.pack_count */
  int32_t n_pack_q;     /* sum of pack query counts */
  int32_t n_pack_blk;   /* sum of pack block counts */
  int32_t n_units;      /* forward units after the KV split */
  int32_t n_items;      /* CTA work items (unit x kv head x row block) */
  int32_t n_slots;      /* fp32 partial slots (queries covered by > 1 unit) */
  int32_t n_merge_q;    /* queries that need the merge kernel */
  int32_t on_device;    /* 1 when the plan lives in device memory */
  int64_t unique_tokens;/* distinct_block_census total tokens (simulator.py:68-75) */
  int32_t n_fwd_kernels;/* forward kernel launches per pat_forward (one per non-empty variant) */
  int32_t n_launches;   /* all kernel launches per pat_forward (forward + merge) */
} pat_plan_info;

/* Host C++ packer (the paper's async pack scheduler). Row q of the block table is
 * row_blk[row_off[q] .. row_off[q+1]); its last block holds valid_last[q] tokens. */
int pat_plan_create_host(int32_t B, const int64_t* row_off, const int32_t* row_blk,
                         const int32_t* valid_last, int32_t block_size,
                         const pat_plan_options* opt, pat_plan** out);

/* GPU packer: block_tables[B][bt_stride] and seq_lens[B] are DEVICE int32 arrays
 * (vLLM layout); blocks per row = ceil(seq_len / block_size).  Stream-ordered. */
int pat_plan_create_device(int32_t B, const int32_t* block_tables, int64_t bt_stride,
                           const int32_t* seq_lens, int32_t max_blocks, int32_t block_size,
                           const pat_plan_options* opt, void* stream, pat_plan** out);

/* Device table fingerprint for the lazy plan update (PackCache, packer.py:189-221):
 * 64-bit hash of (B, block_size, seq_lens, the used block ids of every row) written
 * to out_hash (device-accessible).  Stream-ordered; one small kernel. */
int pat_table_hash_device(int32_t B, const int32_t* block_tables, int64_t bt_stride,
                          const int32_t* seq_lens, int32_t block_size, uint64_t* out_hash,
                          void* stream);

/* Explicit partition: unit u has queries unit_q[unit_q_off[u] .. unit_q_off[u+1]),
 * blocks unit_blk[unit_blk_off[u] .. unit_blk_off[u+1]) and unit_kv[u] tokens.
 * Coverage against the table is checked (PAT_ERR_COVERAGE_GAP). */
int pat_plan_create_units(int32_t B, const int64_t* row_off, const int32_t* row_blk,
                          const int32_t* valid_last, int32_t block_size, int32_t n_units,
                          const int64_t* unit_q_off, const int32_t* unit_q,
                          const int64_t* unit_blk_off, const int32_t* unit_blk,
                          const int32_t* unit_kv, const pat_plan_options* opt, pat_plan** out);

int pat_plan_info_get(const pat_plan* plan, pat_plan_info* info);

/* Packs in reference order: q_off[n_packs+1], q_ids[n_pack_q], blk_off[n_packs+1],
 * blk_ids[n_pack_blk], kv_len[n_packs], partial[n_packs]. Synchronises on device plans. */
int pat_plan_export_packs(const pat_plan* plan, int32_t* q_off, int32_t* q_ids, int32_t* blk_off,
                          int32_t* blk_ids, int32_t* kv_len, uint8_t* partial);

/* Forward units after the split: pack index, first page within the pack, page count,
 * tokens, split_index, split_of (CtaTask fields simulator.py:99-110). */
int pat_plan_export_units(const pat_plan* plan, int32_t* pack, int32_t* page0, int32_t* npages,
                          int32_t* ntok, int32_t* split_index, int32_t* split_of);

/* Scheduler cost model (ns): the native KV split and the longest-first item
 * order estimate a work item of `rows` rows over `steps` 64-token KV spans as
 *   tcgen05:   tc_item_ns + tc_item_row_ns * rows / 128 + steps * tc_step_ns * (0.5 + 0.5 * d / 128)
 *              (per item pipeline; two pipelines per SM; the split simulates the
 *              kernel's longest-first claims over 2 x num_sms pipelines)
 *   streaming: stream_item_ns + steps * 64 * d * 4 / (hbm_bytes_per_ns / num_sms)
 * and the layer's byte floor as bytes / hbm_bytes_per_ns.  Process-wide; read
 * when a plan is created.  Defaults are measured B200 constants;
 * tools/calibrate.py measures the B200 values (profiles/b200_calibration.json,
 * loaded by paper_2511_22333_b200.calibration.load_profile).  Replaces the
 * reference's A100 tile cost tables (tiles.py). */
typedef struct pat_cost_model {
  double tc_item_ns;
  double tc_item_row_ns;
  double tc_step_ns;
  double stream_item_ns;
  double hbm_bytes_per_ns;
} pat_cost_model;

/* PAT_ERR_INVALID_SPEC on a NULL pointer or a non-positive step / bandwidth. */
int pat_set_cost_model(const pat_cost_model* model);
int pat_get_cost_model(pat_cost_model* model);

/* Bytes of device workspace pat_forward needs (fp32 partials + counters). */
size_t pat_workspace_bytes(const pat_plan* plan);

/* out[B][H][d] = attention of q[B][H][d] over the paged cache
 * k_cache/v_cache[num_pool_blocks][block_size][KVH][d] (vLLM NHD layout), dtype f16/bf16.
 * scale <= 0 selects 1/sqrt(d) (attention.py:152-153).  Stream-ordered, no host sync. */
int pat_forward(const pat_plan* plan, const void* q, const void* k_cache, const void* v_cache,
                int64_t num_pool_blocks, void* out, void* workspace, size_t workspace_bytes,
                int32_t dtype, float scale, void* stream);

void pat_plan_destroy(pat_plan* plan);

/* ---------------------------------------------------------------------------------
 * Device-resident decoder: the serving path with planning on the GPU.
 * Replaces packer.py:189-266 (PackCache + pack_batch_async) and the per-step
 * pack_batch -> run_packed_attention of a serving engine.
 * pat_decoder_forward enqueues on `stream`, with no host synchronisation and no
 * allocation: a 64-bit fingerprint of (block_tables, seq_lens), a comparison with
 * the last one on the device, the GPU packer and the device scheduler (both skip
 * at once when the table is unchanged), then the forward and merge kernels over
 * the device plan.  A CUDA graph of it stays valid while the table contents change.
 * max_batch <= 4096; a table outside the decoder's capacity is rejected.  An
 * invalid table (empty row, repeated block) makes the step a no-op on the device;
 * pat_decoder_status (synchronising) reports it and the re-plan count. */
typedef struct pat_decoder pat_decoder;
enum pat_decode_flags {
  PAT_DECODE_SAME_TABLE = 1  /* the caller guarantees the table is the one of the previous call
                               (e.g. the other layers of a decode step): forward + merge only */
};
int pat_decoder_create(const pat_plan_options* opt, int32_t max_batch, int32_t max_blocks,
                       int32_t block_size, pat_decoder** out);
size_t pat_decoder_workspace_bytes(const pat_decoder* dec);
int pat_decoder_forward(pat_decoder* dec, const int32_t* block_tables, int64_t bt_stride,
                        const int32_t* seq_lens, int32_t B, int32_t max_blocks, const void* q,
                        const void* k_cache, const void* v_cache, int64_t num_pool_blocks, void* out,
                        void* workspace, size_t workspace_bytes, int32_t dtype, float scale,
                        int32_t flags, void* stream);
int pat_decoder_status(pat_decoder* dec, void* stream, int32_t* replans);
void pat_decoder_destroy(pat_decoder* dec);

const char* pat_last_error(void);

/* Library version string. */
const char* pat_version(void);

#ifdef __cplusplus
}
#endif

#endif /* PAT_H_ */
