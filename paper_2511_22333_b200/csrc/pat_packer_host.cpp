// Host C++ pack scheduler -- the paper's "async pack scheduler (C++)"
// (PAPER.md:742), bit-exact with the reference pack_batch (packer.py:224-242):
// rows -> unit trie -> maximal-run prefix forest (workload.py:245-297) ->
// TreeHeuristic packs (packer.py:124-168) -> Partition with produces_partial
// (workload.py:377-393), linear in the number of (block, tokens) units.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <unordered_map>
#include <vector>

#include "pat_plan_host.h"

namespace pat {

int validate_rows(const RowsView& R) {
  if (R.bs <= 0) {
    set_error("block_size must be positive");
    return PAT_ERR_INVALID_SPEC;
  }
  int32_t maxb = -1;
  for (int q = 0; q < R.B; ++q) {
    int n = R.nblk[q];
    if (n <= 0) {
      set_error("row %d is empty", q);
      return PAT_ERR_INVALID_SPEC;
    }
    int v = R.valid[q];
    if (v < 1 || v > R.bs) {
      set_error("row %d valid-token count %d outside [1, block_size]", q, v);
      return PAT_ERR_INVALID_SPEC;
    }
    for (int p = 0; p < n; ++p) {
      const int32_t b = R.block(q, p);
      if (b < 0) {
        set_error("row %d has a negative block ID", q);
        return PAT_ERR_INVALID_SPEC;
      }
      maxb = std::max(maxb, b);
    }
  }
  // a repeated block inside a row: last row that used each block id (linear)
  std::vector<int32_t> seen((size_t)maxb + 1, -1);
  for (int q = 0; q < R.B; ++q)
    for (int p = 0; p < R.nblk[q]; ++p) {
      int32_t& s = seen[R.block(q, p)];
      if (s == q) {
        set_error("row %d repeats a block ID", q);
        return PAT_ERR_INVALID_SPEC;
      }
      s = q;
    }
  return PAT_OK;
}

namespace {

// Unit trie over the rows: node = a (block, tokens) unit at a row position;
// children in creation order (rows inserted by query id = first appearance).
struct TNode {
  int32_t first_kid = -1, last_kid = -1, next_sib = -1, n_kids = 0;
  int32_t blk = 0, tok = 0;           // the unit
  int32_t nq = 0, first_q = -1;      // queries passing through; the smallest of them
  int32_t ends_head = -1, ends_tail = -1, n_ends = 0;  // queries whose row ends here
  int32_t depth = 0;                  // row position of the unit
};
struct UKey {
  int32_t node, blk, tok;
  bool operator==(const UKey& o) const { return node == o.node && blk == o.blk && tok == o.tok; }
};
struct UKeyHash {
  size_t operator()(const UKey& k) const {
    uint64_t h = (uint64_t)(uint32_t)k.node * 0x9E3779B97F4A7C15ull;
    h ^= ((uint64_t)(uint32_t)k.blk + 0x632BE59BD9B4E019ull) * 0xC2B2AE3D27D4EB4Full;
    h ^= (uint64_t)(uint32_t)k.tok * 0x165667B19E3779F9ull;
    return (size_t)(h ^ (h >> 29));
  }
};

struct TriePacker {
  const RowsView& R;
  std::vector<TNode> T;
  std::vector<int32_t> next_end;  // per query: next query ending at the same trie node
  // emitted packs: queries (flattened), rep query, [a, b) row positions, tokens
  std::vector<int32_t> pq, pq_off{0}, prep, pa, pb, pkv;

  explicit TriePacker(const RowsView& r) : R(r) {}

  void build() {
    size_t total = 0;
    for (int q = 0; q < R.B; ++q) total += (size_t)R.nblk[q];
    T.reserve(total + 1);
    T.emplace_back();  // virtual root above the first units
    // children are found by scanning the sibling list; a node whose fan-out
    // passes kHashFrom moves its children into the hash map (a branch point
    // of B rows costs O(B), not O(B^2))
    constexpr int kHashFrom = 8;
    std::unordered_map<UKey, int32_t, UKeyHash> kid;
    next_end.assign(R.B, -1);
    for (int q = 0; q < R.B; ++q) {
      int32_t t = 0;
      for (int p = 0; p < R.nblk[q]; ++p) {
        const int32_t blk = R.block(q, p), tok = R.tokens_at(q, p);
        int32_t c = -1;
        if (T[t].n_kids < kHashFrom) {
          for (int32_t k = T[t].first_kid; k >= 0; k = T[k].next_sib)
            if (T[k].blk == blk && T[k].tok == tok) {
              c = k;
              break;
            }
        } else {
          auto it = kid.find(UKey{t, blk, tok});
          if (it != kid.end()) c = it->second;
        }
        if (c < 0) {
          c = (int32_t)T.size();
          T.emplace_back();
          T[c].depth = p;
          T[c].first_q = q;
          T[c].blk = blk;
          T[c].tok = tok;
          if (T[t].last_kid < 0) T[t].first_kid = c;
          else T[T[t].last_kid].next_sib = c;
          T[t].last_kid = c;
          if (++T[t].n_kids == kHashFrom)
            for (int32_t k = T[t].first_kid; k >= 0; k = T[k].next_sib) kid.emplace(UKey{t, T[k].blk, T[k].tok}, k);
          else if (T[t].n_kids > kHashFrom)
            kid.emplace(UKey{t, blk, tok}, c);
        }
        T[c].nq++;
        t = c;
      }
      if (T[t].ends_tail < 0) T[t].ends_head = q;
      else next_end[T[t].ends_tail] = q;
      T[t].ends_tail = q;
      T[t].n_ends++;
    }
  }

  // The forest node whose run starts at trie node c (workload.py:245-297): a
  // single-query group is a leaf with the whole remaining suffix; otherwise the
  // run extends while nobody ends and every row takes the same next unit.
  struct FNode {
    bool leaf;
    int32_t q, a, b;  // rep query, run positions [a, b) of its row
    int32_t tail;     // trie node of the run's last unit (internal nodes)
    int32_t nq;
    int64_t tokens;
  };
  FNode grow(int32_t c) const {
    FNode f{};
    f.q = T[c].first_q;
    f.a = T[c].depth;
    f.nq = T[c].nq;
    if (T[c].nq == 1) {
      f.leaf = true;
      f.b = R.nblk[f.q];
    } else {
      int32_t t = c;
      while (T[t].n_ends == 0 && T[t].first_kid >= 0 && T[T[t].first_kid].next_sib < 0) t = T[t].first_kid;
      f.leaf = false;
      f.tail = t;
      f.b = T[t].depth + 1;
    }
    f.tokens = R.span_tokens(f.q, f.a, f.b);
    return f;
  }
  // queries of a forest node's subtree, leaves in DFS order (empty leaves first)
  void subtree(int32_t c, std::vector<int32_t>& out) const {
    const FNode f = grow(c);
    if (f.leaf) {
      out.push_back(f.q);
      return;
    }
    for (int32_t q = T[f.tail].ends_head; q >= 0; q = next_end[q]) out.push_back(q);
    for (int32_t k = T[f.tail].first_kid; k >= 0; k = T[k].next_sib) subtree(k, out);
  }
  void emit(const std::vector<int32_t>& qs, int32_t rep, int32_t a, int32_t b, int64_t kv) {
    pq.insert(pq.end(), qs.begin(), qs.end());
    pq_off.push_back((int32_t)pq.size());
    prep.push_back(rep);
    pa.push_back(a);
    pb.push_back(b);
    pkv.push_back((int32_t)kv);
  }
  // TreeHeuristic (packer.py:124-161): a child is merged into the pack being
  // built iff 2 (s_child + terminal_child) > span; children's packs come first.
  void visit(int32_t c, bool inherit, int32_t anchor, int64_t span_in) {
    const FNode f = grow(c);
    const int32_t a = inherit ? anchor : f.a;
    const int64_t span = (inherit ? span_in : 0) + f.tokens;
    if (f.leaf) {
      if (span > 0) emit({f.q}, f.q, a, f.b, span);
      return;
    }
    std::vector<int32_t> rest;
    for (int32_t q = T[f.tail].ends_head; q >= 0; q = next_end[q]) rest.push_back(q);
    for (int32_t k = T[f.tail].first_kid; k >= 0; k = T[k].next_sib) {
      const FNode g = grow(k);
      const int32_t terminal = g.leaf ? 1 : T[g.tail].n_ends;
      if (2 * (int64_t)(g.nq + terminal) > span) {
        visit(k, true, a, span);  // merged: its queries leave this pack
      } else {
        visit(k, false, 0, 0);
        subtree(k, rest);
      }
    }
    if (!rest.empty() && span > 0) emit(rest, f.q, a, f.b, span);
  }
};

}  // namespace

// Linear in the table size: a unit trie (hash map keyed by (node, block,
// tokens)), compressed into the maximal-run forest on the fly, with the
// TreeHeuristic emitting packs in post-order.  (The GPU pass in
// pat_packer_dev.cu derives the same partition from pairwise prefixes.)
int host_pack(const RowsView& R, HostPacks* out) {
  const int B = R.B;
  out->clear();
  if (B == 0) return PAT_OK;
  int st = validate_rows(R);
  if (st) return st;
  TriePacker tp(R);
  tp.build();
  for (int32_t k = tp.T[0].first_kid; k >= 0; k = tp.T[k].next_sib) tp.visit(k, false, 0, 0);
  const int NP = (int)tp.pkv.size();
  std::vector<int32_t> cnt(B, 0);
  for (int32_t q : tp.pq) cnt[q]++;
  out->q = tp.pq;
  out->q_off = tp.pq_off;
  out->blk_off.assign(1, 0);
  for (int p = 0; p < NP; ++p) {
    uint8_t part = 0;
    for (int i = tp.pq_off[p]; i < tp.pq_off[p + 1]; ++i) part |= cnt[tp.pq[i]] > 1;
    out->partial.push_back(part);
    out->kv.push_back(tp.pkv[p]);
    out->rep.push_back(tp.prep[p]);
    out->blk_begin.push_back(tp.pa[p]);
    for (int j = tp.pa[p]; j < tp.pb[p]; ++j) out->blk.push_back(R.block(tp.prep[p], j));
    out->blk_off.push_back((int32_t)out->blk.size());
  }
  return PAT_OK;
}

int64_t distinct_tokens(const RowsView& R) {
  // fullest use of every block id (simulator.py:68-75), one pass
  int32_t maxb = -1;
  for (int q = 0; q < R.B; ++q)
    for (int p = 0; p < R.nblk[q]; ++p) maxb = std::max(maxb, R.block(q, p));
  std::vector<int32_t> best((size_t)maxb + 1, 0);
  for (int q = 0; q < R.B; ++q)
    for (int p = 0; p < R.nblk[q]; ++p) {
      int32_t& b = best[R.block(q, p)];
      b = std::max(b, R.tokens_at(q, p));
    }
  int64_t tot = 0;
  for (int32_t t : best) tot += t;
  return tot;
}

}  // namespace pat
