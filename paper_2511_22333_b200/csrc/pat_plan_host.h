// Host-side plan structures (packs, units, items) and planner entry points.
#pragma once

#include <vector>

#include "pat_plan.cuh"

namespace pat {

// Packs in reference order (Partition.packs, workload.py:337).
struct HostPacks {
  std::vector<int32_t> q_off, q, blk_off, blk, kv;
  std::vector<uint8_t> partial;
  std::vector<int32_t> rep, blk_begin;  // pack span = row[rep][blk_begin : blk_begin + n)
  void clear() {
    q_off.assign(1, 0);
    blk_off.assign(1, 0);
    q.clear(); blk.clear(); kv.clear(); partial.clear(); rep.clear(); blk_begin.clear();
  }
  int n_packs() const { return (int)kv.size(); }
};

// Forward units, slots and work items derived from the packs.
struct HostSchedule {
  std::vector<int32_t> unit_pack, unit_page0, unit_npages, unit_ntok, unit_split_idx, unit_split_of;
  std::vector<int32_t> unit_slot_off, unit_slot;
  std::vector<int32_t> q_slot_off, q_nslot, merge_q;
  std::vector<Item> items[NUM_VARIANTS];
  int32_t n_pair[NUM_VARIANTS] = {0, 0, 0, 0};  // leading pair items (> 128 rows, tcgen05)
  double work[NUM_VARIANTS] = {0, 0, 0, 0};  // estimated SM-ns per kernel variant
  int32_t n_slots = 0;
};

int validate_rows(const RowsView& R);
int host_pack(const RowsView& R, HostPacks* out);
int64_t distinct_tokens(const RowsView& R);

struct ScheduleParams {
  int B, bs, H, KVH, d, split_mode, num_sms;
  int tc_min_rows;  // rows threshold of the tcgen05 variant (0 = off)
  bool pair_items = false;  // PAT_PLAN_PAIR_ITEMS
  bool all_partials = false;  // PAT_PLAN_ALL_PARTIALS
  pat_cost_model cm{};      // snapshot of the cost model (host_schedule takes it)
};
int host_schedule(const HostPacks& P, const ScheduleParams& sp, HostSchedule* out);
// process-wide scheduler cost model (pat_set_cost_model)
pat_cost_model cost_model();  // a copy taken under the model's lock

}  // namespace pat
