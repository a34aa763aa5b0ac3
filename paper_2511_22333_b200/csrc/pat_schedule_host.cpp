// Host scheduler: packs -> forward units (KV split) -> partial slots -> CTA work items.
//
// Reference mode reproduces split_long_kv (simulator.py:117-155) on the packs
// taken as tasks (the plan_tasks query pre-split, simulator.py:185-202, is not
// applied: a wide pack is tiled over rows inside the kernel instead of
// re-reading its KV per query group).  Native mode sizes parts for 148 SMs.
#include <algorithm>
#include <cmath>
#include <numeric>

#include "pat_plan_host.h"

namespace pat {

namespace {

struct Part {
  int page0, npages, ntok;
};

void split_pack(int npages, int kv, int bs, int parts, std::vector<Part>& out) {
  // near-equal block counts, larger parts first; the last part carries the
  // partial block (simulator.py:137-154)
  int base = npages / parts, extra = npages % parts, pos = 0, used = 0;
  for (int i = 0; i < parts; ++i) {
    int take = base + (i < extra ? 1 : 0);
    int tok = std::min(take * bs, kv - used);
    out.push_back({pos, take, tok});
    pos += take;
    used += tok;
  }
}


// Native KV split for B200.  Picks one chunk size (pages) for all packs by
// minimising a makespan estimate over candidate chunks:
//   max( bytes(chunk) / HBM_BW,                 -- KV + extra fp32 partials
//        work(chunk) / num_SMs,                 -- all items spread over SMs
//        max item cost )                        -- the critical CTA
// + per-item fixed cost.  An item's cost is pages x per-page time of its
// kernel (streaming: its HBM share per SM; tcgen05: per 128-row block).
// per-page cost (ns) of a work item of variant v (same constants as native_parts)
double page_cost(const ScheduleParams& sp, int v) {
  const double bw = 6.0e3;
  const double page_bytes = 16.0 * sp.d * 4;
  return v == VAR_TC ? 500.0 : page_bytes / (bw / std::max(sp.num_sms, 1));
}

void native_parts(const HostPacks& P, const ScheduleParams& sp, std::vector<int>& nparts) {
  const int NP = P.n_packs();
  const int G = sp.H / sp.KVH;
  const double bw = 6.0e3;                // bytes per ns (HBM, sustained)
  const double t_item = 1500.0;           // ns fixed cost per item (Q load, pipeline fill, epilogue)
  std::vector<int> rows(NP), pages(NP), rb(NP);
  int maxpages = 1;
  double kv_bytes = 0;
  for (int p = 0; p < NP; ++p) {
    rows[p] = (P.q_off[p + 1] - P.q_off[p]) * G;
    pages[p] = P.blk_off[p + 1] - P.blk_off[p];
    int v = choose_variant(rows[p], sp.tc_min_rows);
    rb[p] = (int)ceil_div(rows[p], variant_rows(v));
    maxpages = std::max(maxpages, pages[p]);
    kv_bytes += (double)P.kv[p] * sp.KVH * sp.d * 4;
  }
  std::vector<std::pair<int, double>> cand;
  for (int chunk = 1; ; chunk *= 2) {
    const int c = std::min(chunk, maxpages);
    double work = 0, worst = 0, extra = 0;
    double vwork[NUM_VARIANTS] = {0, 0, 0, 0};
    int64_t vitems[NUM_VARIANTS] = {0, 0, 0, 0};
    for (int p = 0; p < NP; ++p) {
      int parts = (int)ceil_div(pages[p], c);
      int v = choose_variant(rows[p], sp.tc_min_rows);
      double item = std::min(c, pages[p]) * page_cost(sp, v) + t_item;
      int64_t n = (int64_t)parts * rb[p] * sp.KVH;
      vitems[v] += n;
      vwork[v] += item * n;
      work += item * n;
      worst = std::max(worst, item);
      if (parts > 1) extra += (double)parts * (P.q_off[p + 1] - P.q_off[p]) * sp.H * sp.d * 8;
    }
    // each variant runs on an SM share proportional to its work (pat_forward);
    // its time is the number of item waves on that share x the mean item
    double tv = 0;
    for (int v = 0; v < NUM_VARIANTS; ++v) {
      if (!vitems[v]) continue;
      int sms = std::max(1, (int)(sp.num_sms * vwork[v] / work + 0.5));
      tv = std::max(tv, (double)ceil_div(vitems[v], sms) * (vwork[v] / vitems[v]));
    }
    double est = std::max({(kv_bytes + extra) / bw, tv, worst});
    cand.emplace_back(c, est);
    if (c >= maxpages) break;
  }
  double best = 1e300;
  for (auto& ce : cand) best = std::min(best, ce.second);
  int best_chunk = maxpages;  // the largest chunk within 2% of the best estimate: fewest splits
  for (auto& ce : cand)
    if (ce.second <= best * 1.02) best_chunk = std::max(best_chunk == maxpages ? 0 : best_chunk, ce.first);
  if (best_chunk <= 0) best_chunk = maxpages;
  for (int p = 0; p < NP; ++p) nparts[p] = (int)ceil_div(pages[p], best_chunk);
}

}  // namespace

int host_schedule(const HostPacks& P, const ScheduleParams& sp, HostSchedule* S) {
  const int NP = P.n_packs();
  const int G = sp.H / sp.KVH;
  *S = HostSchedule();
  S->q_slot_off.assign(sp.B, 0);
  S->q_nslot.assign(sp.B, 0);
  S->unit_slot_off.assign(1, 0);

  // 1. parts per pack
  std::vector<int> nparts(NP, 1);
  if (sp.split_mode == PAT_SPLIT_REFERENCE && NP > 0) {
    int64_t tot = 0;
    for (int p = 0; p < NP; ++p) tot += P.kv[p];
    const double mean = (double)tot / (double)NP;
    for (int p = 0; p < NP; ++p) {
      if ((double)P.kv[p] <= mean) continue;
      int parts = (int)std::ceil((double)P.kv[p] / mean);
      int nblocks = std::max(P.blk_off[p + 1] - P.blk_off[p], (int)ceil_div(P.kv[p], sp.bs));
      nparts[p] = std::min(parts, nblocks);
    }
  } else if (sp.split_mode == PAT_SPLIT_NATIVE && NP > 0) {
    native_parts(P, sp, nparts);
  }

  // 2. units
  std::vector<Part> parts;
  std::vector<int> unit_begin(NP + 1, 0);
  for (int p = 0; p < NP; ++p) {
    parts.clear();
    int pages = P.blk_off[p + 1] - P.blk_off[p];
    split_pack(pages, P.kv[p], sp.bs, nparts[p], parts);
    unit_begin[p + 1] = unit_begin[p] + (int)parts.size();
    for (int i = 0; i < (int)parts.size(); ++i) {
      S->unit_pack.push_back(p);
      S->unit_page0.push_back(parts[i].page0);
      S->unit_npages.push_back(parts[i].npages);
      S->unit_ntok.push_back(parts[i].ntok);
      S->unit_split_idx.push_back(i);
      S->unit_split_of.push_back((int)parts.size());
    }
  }
  const int NU = (int)S->unit_pack.size();

  // 3. slots: a query covered by more than one unit gets one fp32 partial slot
  // per unit, in unit order (the reference fold order, attention.py:228-235).
  std::vector<int32_t> qcnt(sp.B, 0);
  for (int p = 0; p < NP; ++p)
    for (int i = P.q_off[p]; i < P.q_off[p + 1]; ++i) qcnt[P.q[i]] += nparts[p];
  int32_t next = 0;
  for (int q = 0; q < sp.B; ++q) {
    if (qcnt[q] > 1) {
      S->q_slot_off[q] = next;
      S->q_nslot[q] = qcnt[q];
      next += qcnt[q];
      S->merge_q.push_back(q);
    } else {
      S->q_slot_off[q] = -1;
    }
  }
  S->n_slots = next;
  std::vector<int32_t> qcur(sp.B, 0);
  for (int u = 0; u < NU; ++u) {
    int p = S->unit_pack[u];
    for (int i = P.q_off[p]; i < P.q_off[p + 1]; ++i) {
      int q = P.q[i];
      S->unit_slot.push_back(qcnt[q] > 1 ? S->q_slot_off[q] + qcur[q]++ : -1);
    }
    S->unit_slot_off.push_back((int32_t)S->unit_slot.size());
  }

  // 4. work items, longest first within each kernel variant
  std::vector<int> order(NU);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return S->unit_npages[a] > S->unit_npages[b]; });
  for (int u : order) {
    int p = S->unit_pack[u];
    int rows = (P.q_off[p + 1] - P.q_off[p]) * G;
    int v = choose_variant(rows, sp.tc_min_rows);
    int R = variant_rows(v);
    for (int r0 = 0; r0 < rows; r0 += R)
      for (int h = 0; h < sp.KVH; ++h) {
        S->items[v].push_back({u, h, r0, std::min(R, rows - r0), P.blk_off[p] + S->unit_page0[u], S->unit_ntok[u],
                               P.q_off[p], S->unit_slot_off[u]});
        S->work[v] += S->unit_npages[u] * page_cost(sp, v) + 1500.0;
      }
  }
  (void)unit_begin;
  return PAT_OK;
}

}  // namespace pat
