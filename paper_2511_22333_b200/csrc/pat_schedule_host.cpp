// Host scheduler: packs -> forward units (KV split) -> partial slots -> CTA work items.
//
// Reference mode reproduces split_long_kv (simulator.py:117-155) on the packs
// taken as tasks (the plan_tasks query pre-split, simulator.py:185-202, is not
// applied: a wide pack is tiled over rows inside the kernel instead of
// re-reading its KV per query group).  Native mode sizes parts for 148 SMs.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <queue>

#include "pat_plan_host.h"

namespace pat {

// Measured on B200 for the two-lane tcgen05 kernel (tools/item_log.py: ~0.72 us
// per 32-token tile per lane with every SM streaming; an item boundary -- start
// latency + epilogue -- of ~3-4 us for a narrow item and ~6 us for a 128-row
// one), the per-item constant chosen by tools/cm_sweep.py over c1-c5 (3.6 us:
// c4 keeps its 8k root unsplit, 196.6 -> 184.3 us; c1-c3, c5 unchanged); see
// DESIGN.md §7.
static pat_cost_model g_cost_model = {3600.0, 2000.0, 1440.0, 1500.0, 6.5e3};
constexpr int kTcLanesPerSm = 2;  // independent item pipelines per tcgen05 CTA
static std::mutex g_cost_mu;

pat_cost_model cost_model() {
  std::lock_guard<std::mutex> lk(g_cost_mu);
  return g_cost_model;
}

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


// Estimated time (ns) of one work item of variant v with `rows` rows over
// `ntok` tokens, measured on B200: a tcgen05 lane streams a 64-token span of up
// to 128 rows in ~1.4 us when every SM streams (two lanes per SM share the
// chip's ~7 TB/s L2 -> SM bandwidth) plus the item boundary (Q load, last PV,
// epilogue stores); the mma.sync streaming kernel is HBM-paced.
double item_ns(const ScheduleParams& sp, int v, int rows, int ntok) {
  const pat_cost_model& cm = sp.cm;
  const double steps = (double)ceil_div(ntok, 64);
  const double dscale = sp.d / 128.0;
  if (v == VAR_TC)
    return cm.tc_item_ns + cm.tc_item_row_ns * rows / 128.0 + steps * cm.tc_step_ns * (0.5 + 0.5 * dscale);
  return cm.stream_item_ns + steps * 64.0 * sp.d * 4 / (cm.hbm_bytes_per_ns / std::max(sp.num_sms, 1));
}

// Makespan of greedy longest-first list scheduling of `costs` over `lanes`
// identical workers -- what the tcgen05 kernel's dynamic claims do.
double lpt_makespan(std::vector<double>& costs, int lanes) {
  std::sort(costs.begin(), costs.end(), std::greater<double>());
  std::priority_queue<double, std::vector<double>, std::greater<double>> free_at;
  for (int i = 0; i < lanes; ++i) free_at.push(0.0);
  double mk = 0;
  for (double c : costs) {
    double t = free_at.top() + c;
    free_at.pop();
    free_at.push(t);
    mk = std::max(mk, t);
  }
  return mk;
}

// Native KV split for B200.  Picks one chunk size (pages) for all packs by
// minimising a makespan estimate over candidate chunks:
//   max( bytes(chunk) / HBM_BW,                 -- KV + extra fp32 partials
//        sum(item cost) / SMs per variant,      -- dynamic (tcgen05) or wave-
//                                                  quantised (static) scheduling
//        max item cost )                        -- the critical CTA
void native_parts(const HostPacks& P, const ScheduleParams& sp, std::vector<int>& nparts) {
  const int NP = P.n_packs();
  const int G = sp.H / sp.KVH;
  const double bw = sp.cm.hbm_bytes_per_ns;
  std::vector<int> rows(NP), pages(NP);
  int maxpages = 1;
  double kv_bytes = 0;
  for (int p = 0; p < NP; ++p) {
    rows[p] = (P.q_off[p + 1] - P.q_off[p]) * G;
    pages[p] = P.blk_off[p + 1] - P.blk_off[p];
    maxpages = std::max(maxpages, pages[p]);
    kv_bytes += (double)P.kv[p] * sp.KVH * sp.d * 4;
  }
  std::vector<std::pair<int, double>> cand;
  std::vector<double> worsts;
  int64_t total_row_blocks_pages = 0;
  for (int p = 0; p < NP; ++p)
    total_row_blocks_pages += (int64_t)pages[p] * ceil_div(rows[p], variant_rows(choose_variant(rows[p], sp.tc_min_rows)));
  const int64_t max_items = (int64_t)64 * kTcLanesPerSm * std::max(sp.num_sms, 1);
  std::vector<double> tc_costs;
  for (int chunk = 1;; chunk *= 2) {
    const int c = std::min(chunk, maxpages);
    // far more items than lanes can balance only costs item boundaries
    if (c < maxpages && total_row_blocks_pages * sp.KVH / c > max_items) continue;
    double work = 0, worst = 0, extra = 0;
    double vwork[NUM_VARIANTS] = {0, 0, 0, 0};
    int64_t vitems[NUM_VARIANTS] = {0, 0, 0, 0};
    tc_costs.clear();
    for (int p = 0; p < NP; ++p) {
      const int parts = (int)ceil_div(pages[p], c);
      const int v = choose_variant(rows[p], sp.tc_min_rows);
      const int R = variant_rows(v);
      for (int r0 = 0; r0 < rows[p]; r0 += R) {
        // near-equal parts (split_pack): the larger ones carry ceil(pages / parts)
        const int big = (int)ceil_div(pages[p], parts);
        const double item = item_ns(sp, v, std::min(R, rows[p] - r0), std::min(big * sp.bs, P.kv[p]));
        const int64_t n = (int64_t)parts * sp.KVH;
        vitems[v] += n;
        vwork[v] += item * n;
        work += item * n;
        worst = std::max(worst, item);
        if (v == VAR_TC)
          for (int64_t i = 0; i < n; ++i) tc_costs.push_back(item);
      }
      if (parts > 1) extra += (double)parts * (P.q_off[p + 1] - P.q_off[p]) * sp.H * sp.d * 8;
    }
    // each variant runs on an SM share proportional to its work (pat_forward)
    double tv = 0;
    for (int v = 0; v < NUM_VARIANTS; ++v) {
      if (!vitems[v]) continue;
      const int sms = std::max(1, (int)(sp.num_sms * vwork[v] / work + 0.5));
      const double mean = vwork[v] / vitems[v];
      if (v == VAR_TC)  // dynamic longest-first claims over the kernel's lanes
        tv = std::max(tv, lpt_makespan(tc_costs, sms * kTcLanesPerSm));
      else
        tv = std::max(tv, (double)ceil_div(vitems[v], sms) * mean);
    }
    const double est = std::max({(kv_bytes + extra) / bw, tv, vitems[VAR_TC] ? 0.0 : worst});
    cand.emplace_back(c, est);
    worsts.push_back(vitems[VAR_TC] ? 0.0 : worst);
    if (getenv("PAT_DEBUG_SPLIT")) fprintf(stderr, "chunk %d bytes %.1f tv %.1f worst %.1f est %.1f\n", c, (kv_bytes + extra) / bw / 1e3, tv / 1e3, worst / 1e3, est / 1e3);
    if (c >= maxpages) break;
  }
  double best = 1e300;
  for (auto& ce : cand) best = std::min(best, ce.second);
  // the largest chunk within 2% of the best estimate (fewest splits) whose
  // longest item stays under half the makespan (robust to cost-model error;
  // the tcgen05 estimate simulates the claims, so its tail is already in it)
  int best_chunk = 0;
  for (size_t i = 0; i < cand.size(); ++i)
    if (cand[i].second <= best * 1.02 && worsts[i] <= 0.5 * cand[i].second)
      best_chunk = std::max(best_chunk, cand[i].first);
  if (best_chunk <= 0)
    for (auto& ce : cand)
      if (ce.second == best) best_chunk = ce.first;
  for (int p = 0; p < NP; ++p) nparts[p] = (int)ceil_div(pages[p], best_chunk);
}

}  // namespace

int host_schedule(const HostPacks& P, const ScheduleParams& sp_in, HostSchedule* S) {
  ScheduleParams sp = sp_in;
  sp.cm = cost_model();  // one consistent snapshot for the whole schedule
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
    if (qcnt[q] > 1 || (sp.all_partials && qcnt[q] > 0)) {
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
      S->unit_slot.push_back(S->q_slot_off[q] >= 0 && qcnt[q] > 0 ? S->q_slot_off[q] + qcur[q]++ : -1);
    }
    S->unit_slot_off.push_back((int32_t)S->unit_slot.size());
  }

  // 4. work items (unit x row block x kv head), longest (estimated) first
  // within each kernel variant: the tcgen05 kernel hands them out dynamically,
  // so this is longest-processing-time-first list scheduling.
  struct Cand {
    Item it;
    double ns;
    int v;
  };
  std::vector<Cand> cands;
  for (int u = 0; u < NU; ++u) {
    int p = S->unit_pack[u];
    int rows = (P.q_off[p + 1] - P.q_off[p]) * G;
    int v = choose_variant(rows, sp.tc_min_rows);
    // tcgen05: rows of a wide pack go in 256-row pair items (both item
    // pipelines of a CTA share one KV stream: half the L2 -> SM bytes per row)
    int R = sp.pair_items && v == VAR_TC && rows > variant_rows(v) ? 2 * variant_rows(v) : variant_rows(v);
    for (int r0 = 0; r0 < rows; r0 += R) {
      const int n = std::min(R, rows - r0);
      const double ns = item_ns(sp, v, std::min(n, variant_rows(v)), S->unit_ntok[u]);
      for (int h = 0; h < sp.KVH; ++h)
        cands.push_back({{u, h, r0, n, P.blk_off[p] + S->unit_page0[u], S->unit_ntok[u], P.q_off[p],
                          S->unit_slot_off[u]},
                         ns, v});
    }
  }
  // pair items first (the kernel runs them in a first phase), then longest first
  auto is_pair = [](const Cand& c) { return c.v == VAR_TC && c.it.nrows > variant_rows(VAR_TC); };
  std::stable_sort(cands.begin(), cands.end(), [&](const Cand& a, const Cand& b) {
    if (is_pair(a) != is_pair(b)) return is_pair(a);
    return a.ns > b.ns;
  });
  for (const Cand& c : cands) {
    S->items[c.v].push_back(c.it);
    S->work[c.v] += c.ns * (is_pair(c) ? 2 : 1);
    if (is_pair(c)) S->n_pair[c.v]++;
  }
  (void)unit_begin;
  return PAT_OK;
}

}  // namespace pat

extern "C" int pat_set_cost_model(const pat_cost_model* m) {
  if (!m || !(m->tc_step_ns > 0) || !(m->hbm_bytes_per_ns > 0) || m->tc_item_ns < 0 || m->tc_item_row_ns < 0 ||
      m->stream_item_ns < 0)
    return PAT_ERR_INVALID_SPEC;
  std::lock_guard<std::mutex> lk(pat::g_cost_mu);
  pat::g_cost_model = *m;
  return PAT_OK;
}

extern "C" int pat_get_cost_model(pat_cost_model* m) {
  if (!m) return PAT_ERR_INVALID_SPEC;
  std::lock_guard<std::mutex> lk(pat::g_cost_mu);
  *m = pat::g_cost_model;
  return PAT_OK;
}
