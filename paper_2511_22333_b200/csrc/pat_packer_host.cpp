// Host C++ pack scheduler -- the paper's "async pack scheduler (C++)"
// (PAPER.md:742), bit-exact with the reference pack_batch (packer.py:224-242).
//
// The algorithm is NOT the reference's recursive tree walk.  It derives the
// whole prefix forest from the pairwise longest-common-prefix matrix of the
// rows (as (block, tokens) units, workload.py:111-118), so that every phase is
// a data-parallel map/reduce that the GPU packer (pat_packer_dev.cu) runs as
// kernels; this file is the serial host driver of the same phases and is what
// the CPU tests check against the oracle.
//
// For query q let D_q = sorted distinct values of lcp(q, r) >= 1 over r != q.
//  * The internal forest nodes on q's root->leaf path end exactly at D_q
//    (workload.py:268-273 extends a run while every member continues equally,
//    i.e. up to the minimum lcp inside the group); level k spans
//    [D_q[k-1], D_q[k]) and holds S_k(q) = {q} u {r : lcp(q,r) >= D_q[k]}.
//  * If max(D_q) < len(q) (or D_q is empty) q ends in its own leaf holding the
//    remaining suffix (workload.py:258-266); otherwise q is an empty leaf of
//    its last internal node (workload.py:275-280).
//  * terminal(child) (packer.py:105-110) = #members ending exactly at the
//    child's end.
//  * TreeHeuristic's merge rule 2*(s_c + terminal_c) > span (packer.py:153)
//    only reads the node and its accumulated span, so each query can replay
//    every decision on its own path independently.
//  * q is in the pack of its path node k iff k is its last node or node k+1
//    was split (packer.py:154-160: merged children's queries leave the
//    parent's pack).
//  * Children are ordered [empty leaves by qid] + [groups by min qid]
//    (workload.py:275-294) and packs are emitted in post-order
//    (packer.py:150-161), so the DFS rank pi(q) is the lexicographic rank of
//    the key [min(root group), slot_0, slot_1, ...] with slot_k = q if q ends
//    at level k else B + min(group at level k+1); packs are ordered by
//    (last pi in the node's subtree, deeper first) and the queries inside a
//    pack by pi.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <vector>

#include "pat_plan_host.h"

namespace pat {

int validate_rows(const RowsView& R) {
  if (R.bs <= 0) {
    set_error("block_size must be positive");
    return PAT_ERR_INVALID_SPEC;
  }
  std::vector<int32_t> tmp;
  for (int q = 0; q < R.B; ++q) {
    int n = R.nblk[q];
    if (n <= 0) {
      set_error("row %d is empty", q);
      return PAT_ERR_INVALID_SPEC;
    }
    tmp.assign(R.blk + R.row_begin(q), R.blk + R.row_begin(q) + n);
    std::sort(tmp.begin(), tmp.end());
    if (std::adjacent_find(tmp.begin(), tmp.end()) != tmp.end()) {
      set_error("row %d repeats a block ID", q);
      return PAT_ERR_INVALID_SPEC;
    }
    int v = R.valid[q];
    if (v < 1 || v > R.bs) {
      set_error("row %d valid-token count %d outside [1, block_size]", q, v);
      return PAT_ERR_INVALID_SPEC;
    }
  }
  return PAT_OK;
}

// Per-query path through the forest.
struct QPath {
  std::vector<int32_t> end;    // internal level ends (D_q)
  std::vector<int32_t> nq;     // |S_k|
  std::vector<int32_t> minq;   // min S_k
  std::vector<int32_t> term;   // members ending exactly at end[k]
  bool has_leaf = false;
  // per level (internal levels, then the leaf if any)
  std::vector<int32_t> start, stop, span, anchor;
  std::vector<uint8_t> member;
  int levels() const { return (int)end.size() + (has_leaf ? 1 : 0); }
};

int host_pack(const RowsView& R, HostPacks* out) {
  const int B = R.B;
  out->clear();
  if (B == 0) return PAT_OK;
  int st = validate_rows(R);
  if (st) return st;

  // Phase 1: pairwise lcp over units.
  std::vector<int32_t> lcp((size_t)B * B);
  for (int q = 0; q < B; ++q) {
    lcp[(size_t)q * B + q] = R.nblk[q];
    for (int r = q + 1; r < B; ++r) {
      int n = std::min(R.nblk[q], R.nblk[r]);
      int p = 0;
      while (p < n && R.same_unit(q, r, p)) ++p;
      lcp[(size_t)q * B + r] = lcp[(size_t)r * B + q] = p;
    }
  }

  // Phase 2: per-query levels.
  std::vector<QPath> P(B);
  std::vector<int32_t> vals;
  for (int q = 0; q < B; ++q) {
    QPath& qp = P[q];
    const int32_t* L = &lcp[(size_t)q * B];
    vals.clear();
    for (int r = 0; r < B; ++r)
      if (r != q && L[r] >= 1) vals.push_back(L[r]);
    std::sort(vals.begin(), vals.end());
    vals.erase(std::unique(vals.begin(), vals.end()), vals.end());
    qp.end = vals;
    const int K = (int)vals.size();
    qp.nq.assign(K, 1);
    qp.minq.assign(K, q);
    qp.term.assign(K, 0);
    for (int k = 0; k < K; ++k) {
      int e = vals[k];
      if (R.nblk[q] == e) qp.term[k] += 1;
      for (int r = 0; r < B; ++r) {
        if (r == q || L[r] < e) continue;
        qp.nq[k] += 1;
        qp.minq[k] = std::min(qp.minq[k], r);
        if (L[r] == e && R.nblk[r] == e) qp.term[k] += 1;
      }
    }
    qp.has_leaf = (K == 0) || vals[K - 1] < R.nblk[q];
  }

  // Phase 3: replay TreeHeuristic decisions along each path.
  std::vector<int32_t> nmemb(B, 0);
  for (int q = 0; q < B; ++q) {
    QPath& qp = P[q];
    const int K = (int)qp.end.size();
    const int Lv = qp.levels();
    qp.start.resize(Lv);
    qp.stop.resize(Lv);
    qp.span.resize(Lv);
    qp.anchor.resize(Lv);
    qp.member.assign(Lv, 0);
    std::vector<uint8_t> merged(Lv, 0);
    for (int k = 0; k < Lv; ++k) {
      qp.start[k] = k == 0 ? 0 : qp.end[k - 1];
      qp.stop[k] = k < K ? qp.end[k] : R.nblk[q];
      int64_t tok = R.span_tokens(q, qp.start[k], qp.stop[k]);
      if (k == 0) {
        qp.span[k] = (int32_t)tok;
        qp.anchor[k] = 0;
      } else {
        int s_c = k < K ? qp.nq[k] : 1;
        int t_c = k < K ? qp.term[k] : 1;
        merged[k] = 2 * (int64_t)(s_c + t_c) > qp.span[k - 1];
        qp.span[k] = merged[k] ? qp.span[k - 1] + (int32_t)tok : (int32_t)tok;
        qp.anchor[k] = merged[k] ? qp.anchor[k - 1] : qp.start[k];
      }
    }
    for (int k = 0; k < Lv; ++k) {
      qp.member[k] = (k == Lv - 1) || !merged[k + 1];
      nmemb[q] += qp.member[k];
    }
  }

  // Phase 4: DFS rank pi(q) = lexicographic rank of the child-slot key.
  std::vector<std::vector<int32_t>> key(B);
  for (int q = 0; q < B; ++q) {
    const QPath& qp = P[q];
    const int K = (int)qp.end.size();
    key[q].push_back(K > 0 ? qp.minq[0] : q);
    for (int k = 0; k < K; ++k) {
      if (qp.end[k] == R.nblk[q]) key[q].push_back(q);
      else key[q].push_back(B + (k + 1 < K ? qp.minq[k + 1] : q));
    }
  }
  std::vector<int32_t> order(B);
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int a, int b) { return key[a] < key[b]; });
  std::vector<int32_t> pi(B);
  for (int i = 0; i < B; ++i) pi[order[i]] = i;

  // Phase 5: nodes.  Node (owner m, level k) where owner = min of the level's set
  // (the query itself at its leaf).  m owns a contiguous suffix of its levels.
  auto owner = [&](int q, int k) { return k < (int)P[q].end.size() ? P[q].minq[k] : q; };
  std::vector<int32_t> k0(B), base(B + 1, 0);
  for (int m = 0; m < B; ++m) {
    int Lv = P[m].levels(), k = 0;
    while (k < Lv && owner(m, k) != m) ++k;
    k0[m] = k;
    base[m + 1] = base[m] + (Lv - k);
  }
  const int N = base[B];
  std::vector<int32_t> hi(N, 0), cnt(N, 0), depth(N), rep(N), a0(N), a1(N), span(N);
  for (int m = 0; m < B; ++m)
    for (int k = k0[m]; k < P[m].levels(); ++k) {
      int id = base[m] + k - k0[m];
      depth[id] = k;
      rep[id] = m;
      a0[id] = P[m].anchor[k];
      a1[id] = P[m].stop[k];
      span[id] = P[m].span[k];
    }
  for (int q = 0; q < B; ++q)
    for (int k = 0; k < P[q].levels(); ++k) {
      int m = owner(q, k);
      int id = base[m] + k - k0[m];
      hi[id] = std::max(hi[id], pi[q] + 1);
      cnt[id] += P[q].member[k];
    }

  // Phase 6: emission order = (hi ascending, deeper first); queries by pi.
  std::vector<int32_t> nodes;
  for (int i = 0; i < N; ++i)
    if (cnt[i] > 0) nodes.push_back(i);
  std::sort(nodes.begin(), nodes.end(), [&](int a, int b) {
    return hi[a] != hi[b] ? hi[a] < hi[b] : depth[a] > depth[b];
  });
  std::vector<int32_t> pack_of(N, -1);
  for (size_t i = 0; i < nodes.size(); ++i) pack_of[nodes[i]] = (int)i;
  const int NP = (int)nodes.size();
  out->q_off.assign(NP + 1, 0);
  out->blk_off.assign(NP + 1, 0);
  out->kv.resize(NP);
  out->partial.assign(NP, 0);
  out->rep.resize(NP);
  out->blk_begin.resize(NP);
  for (int p = 0; p < NP; ++p) {
    int id = nodes[p];
    out->q_off[p + 1] = out->q_off[p] + cnt[id];
    out->blk_off[p + 1] = out->blk_off[p] + (a1[id] - a0[id]);
    out->kv[p] = span[id];
    out->rep[p] = rep[id];
    out->blk_begin[p] = a0[id];
  }
  out->q.assign(out->q_off[NP], -1);
  out->blk.resize(out->blk_off[NP]);
  std::vector<int32_t> cursor(out->q_off.begin(), out->q_off.end() - 1);
  for (int i = 0; i < B; ++i) {
    int q = order[i];
    for (int k = 0; k < P[q].levels(); ++k) {
      if (!P[q].member[k]) continue;
      int m = owner(q, k);
      int p = pack_of[base[m] + k - k0[m]];
      out->q[cursor[p]++] = q;
      if (nmemb[q] > 1) out->partial[p] = 1;
    }
  }
  for (int p = 0; p < NP; ++p) {
    int id = nodes[p];
    for (int j = a0[id]; j < a1[id]; ++j) out->blk[out->blk_off[p] + j - a0[id]] = R.block(rep[id], j);
  }
  return PAT_OK;
}

int64_t distinct_tokens(const RowsView& R) {
  std::vector<std::pair<int32_t, int32_t>> u;
  for (int q = 0; q < R.B; ++q)
    for (int p = 0; p < R.nblk[q]; ++p) u.emplace_back(R.block(q, p), R.tokens_at(q, p));
  std::sort(u.begin(), u.end());
  int64_t tot = 0;
  for (size_t i = 0; i < u.size(); ++i)
    if (i + 1 == u.size() || u[i + 1].first != u[i].first) tot += u[i].second;  // max fill per block
  return tot;
}

}  // namespace pat
