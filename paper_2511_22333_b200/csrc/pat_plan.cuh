// Plan layout shared by the planner (host or device) and the forward/merge kernels.
//
// A plan is the reference Partition (packs in pack_batch order, workload.py:337)
// refined into forward *units* (a pack, or one KV part of it after the split,
// simulator.py:117-155) and CTA *work items* (unit x kv head x row block).
#pragma once

#include "pat_common.cuh"

namespace pat {

// Kernel variants: rows of a work item = (#queries x G) rounded to a row tile.
//   V16 / V32 / V64: mma.sync m16n8k16 streaming kernel with 1 / 2 / 4 row tiles
//   of 16 rows per CTA (4 warps; the warps of a row tile split the KV tile);
//   TC: tcgen05 kernel, items of up to 128 rows (one TMEM lane per row).
enum Variant : int { VAR_R16 = 0, VAR_R32 = 1, VAR_R64 = 2, VAR_TC = 3, NUM_VARIANTS = 4 };

PAT_HD int variant_rows(int v) {
  return v == VAR_R16 ? 16 : (v == VAR_R32 ? 32 : (v == VAR_R64 ? 64 : 128));
}
// Packs with at least `tc_min_rows` rows go to the tensor-core kernel.
PAT_HD int choose_variant(int rows, int tc_min_rows) {
  if (tc_min_rows > 0 && rows >= tc_min_rows) return VAR_TC;
  return rows <= 16 ? VAR_R16 : (rows <= 32 ? VAR_R32 : VAR_R64);
}

// Work item: unit, kv head, first row, row count (rows = query_in_pack * G + g),
// plus everything a kernel needs at item start, resolved by the scheduler so a
// CTA issues ONE 32-byte load per item instead of a chain of dependent loads.
struct __align__(16) Item {
  int32_t unit;
  int32_t kvh;
  int32_t row0;
  int32_t nrows;
  int32_t blk;      // index into pack_blk of the unit's first page
  int32_t ntok;     // tokens of the unit
  int32_t qoff;     // index into pack_q of the pack's first query
  int32_t slot_off; // index into unit_slot of the unit's first member
};

// Device view of a plan (all pointers are device addresses).
struct DevPlan {
  const int32_t* pack_q_off;    // [n_packs+1]
  const int32_t* pack_q;        // [n_pack_q]   query ids, reference order
  const int32_t* pack_blk_off;  // [n_packs+1]
  const int32_t* pack_blk;      // [n_pack_blk] block ids of the pack's span
  const int32_t* unit_pack;     // [n_units]
  const int32_t* unit_page0;    // [n_units] first page (index into the pack's block list)
  const int32_t* unit_ntok;     // [n_units] tokens of the unit
  const int32_t* unit_slot_off; // [n_units+1] CSR over pack members
  const int32_t* unit_slot;     // slot id per (unit, member) or -1 = write output directly
  const Item* items[NUM_VARIANTS];
  const int32_t* n_items;       // [NUM_VARIANTS] (device counts)
  const int32_t* n_pair;        // [NUM_VARIANTS] leading items of > 128 rows (tcgen05: run by both
                                //     item pipelines of a CTA on one KV stream)
  const int32_t* merge_q;       // [n_merge_q] queries with > 1 unit
  const int4* merge_desc;       // [n_merge_q] (query, first slot, slots, 0): one load per merge row
  const int32_t* q_slot_off;    // [B] first slot of the query
  const int32_t* q_nslot;       // [B] slots of the query (0 or >= 2)
  const int32_t* n_merge;       // [1]
  int32_t* sched;               // [4] dynamic item counters (pair items, finished CTAs, other
                                //     items; tcgen05 kernel; zero between launches: the last CTA
                                //     resets them)
  int32_t H, KVH, d, G, bs;
};

}  // namespace pat
