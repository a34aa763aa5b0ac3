"""CPU ORACLE (test infrastructure only) -- restatement of the reference packer.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU baseline.  The product path never routes through it.

Restates, in plain Python integer code, the reference's Pack stage:

* units of a row                      ``workload.py:111-118`` (``row_units``)
* table validation                    ``workload.py:120-132``
* sha256 fingerprint                  ``workload.py:134-143``
* prefix forest                       ``workload.py:245-297`` (``build_forest``)
* TreeHeuristic merge/split packing   ``packer.py:105-168``
* produces_partial marking            ``workload.py:377-393``
* pack_batch                          ``packer.py:224-242``
* naive per-node ablation             ``packer.py:171-186``
* query-centric baseline              ``simulator.py:85-96``
* long-KV split (reference mode)      ``simulator.py:117-155``
* distinct-token census / floor bytes ``simulator.py:25-27, 68-82``

Parity pinned: ``tests/test_oracle_golden.py`` checks every function here
against fixtures produced by the real reference (``tests/golden/make_golden.py``).

A pack is represented as a plain tuple ``(query_ids, block_ids, kv_len,
produces_partial)`` -- the field order of ``CtaPack`` (``workload.py:317-324``).
"""

from __future__ import annotations

import hashlib
import math


class OracleInvalid(ValueError):
    """Mirrors ``InvalidSpec`` for the oracle (``errors.py``)."""


# --------------------------------------------------------------------------
# table helpers
# --------------------------------------------------------------------------

def units(rows, valid_last, bs, q):
    """(block, tokens) per position; only the last may be partial (workload.py:111)."""
    r = rows[q]
    out = [(b, bs) for b in r]
    if out:
        out[-1] = (r[-1], valid_last[q])
    return out


def kv_len(rows, valid_last, bs, q):
    return (len(rows[q]) - 1) * bs + valid_last[q]


def validate(rows, valid_last, bs):
    """Same checks, same order, as ``BlockTable.validate`` (workload.py:120-132)."""
    if len(valid_last) != len(rows):
        raise OracleInvalid("valid_tokens_last_block must have one entry per row")
    if bs <= 0:
        raise OracleInvalid("block_size must be positive")
    for i, r in enumerate(rows):
        if len(r) == 0:
            raise OracleInvalid(f"row {i} is empty")
        if len(set(r)) != len(r):
            raise OracleInvalid(f"row {i} repeats a block ID")
        if not 1 <= valid_last[i] <= bs:
            raise OracleInvalid(f"row {i} valid-token count {valid_last[i]} outside [1, block_size]")


def fingerprint(rows, valid_last, bs):
    """Byte stream: str(bs), then per row b'|' + comma-joined ids + ';' + valid
    (workload.py:134-143)."""
    parts = [str(bs).encode()]
    for r, v in zip(rows, valid_last):
        parts.append(b"|" + ",".join(str(b) for b in r).encode() + f";{v}".encode())
    return hashlib.sha256(b"".join(parts)).hexdigest()


# --------------------------------------------------------------------------
# forest (workload.py:245-297)
# --------------------------------------------------------------------------

class Node:
    __slots__ = ("blocks", "tokens", "nq", "kids", "qids")

    def __init__(self, blocks, tokens, nq, kids=None, qids=()):
        self.blocks = tuple(blocks)
        self.tokens = tokens
        self.nq = nq
        self.kids = kids or []
        self.qids = tuple(qids)

    @property
    def leaf(self):
        return not self.kids

    def queries(self):
        """DFS query order (workload.py:219-225)."""
        if self.leaf:
            return list(self.qids)
        acc = []
        for k in self.kids:
            acc += k.queries()
        return acc


def forest(rows, valid_last, bs):
    validate(rows, valid_last, bs)
    U = [units(rows, valid_last, bs, q) for q in range(len(rows))]

    def groups_at(qs, pos):
        # first-appearance order of the unit at ``pos`` (dict insertion order in
        # the reference, workload.py:290-294)
        order, by = [], {}
        for q in qs:
            key = U[q][pos]
            if key not in by:
                by[key] = []
                order.append(key)
            by[key].append(q)
        return [by[k] for k in order]

    def make(qs, pos):
        if len(qs) == 1:
            q = qs[0]
            tail = U[q][pos:]
            return Node([b for b, _ in tail], sum(t for _, t in tail), 1, qids=(q,))
        end = pos
        while all(end < len(U[q]) for q in qs) and len({U[q][end] for q in qs}) == 1:
            end += 1
        run = U[qs[0]][pos:end]
        kids = [Node((), 0, 1, qids=(q,)) for q in qs if len(U[q]) == end]
        live = [q for q in qs if len(U[q]) > end]
        kids += [make(g, end) for g in groups_at(live, end)]
        return Node([b for b, _ in run], sum(t for _, t in run), len(qs), kids)

    if not rows:
        return []
    return [make(g, 0) for g in groups_at(list(range(len(rows))), 0)]


def flatten(roots):
    out = {}

    def walk(n, pre):
        path = pre + list(n.blocks)
        if n.leaf:
            for q in n.qids:
                out[q] = path
        for k in n.kids:
            walk(k, path)

    for r in roots:
        walk(r, [])
    return out


# --------------------------------------------------------------------------
# TreeHeuristic (packer.py:105-168)
# --------------------------------------------------------------------------

def _terminal(n):
    """1 for a leaf, else the number of empty-suffix leaf children (packer.py:105-110)."""
    if n.leaf:
        return 1
    return sum(1 for k in n.kids if k.leaf and k.tokens == 0)


def _pack_tree(node, blocks, span, out):
    # degenerate single-query chains fold into their child (packer.py:113-121)
    while not node.leaf and node.nq == 1:
        node = node.kids[0]
        blocks = blocks + node.blocks
        span += node.tokens
    if node.leaf:
        if span > 0:
            out.append((node.qids, blocks, span))
        return
    absorbed = set()
    for kid in node.kids:
        if kid.leaf and kid.tokens == 0:
            continue
        # strict inequality: ties split (packer.py:153)
        if 2 * (kid.nq + _terminal(kid)) > span:
            _pack_tree(kid, blocks + kid.blocks, span + kid.tokens, out)
            absorbed.update(kid.queries())
        else:
            _pack_tree(kid, kid.blocks, kid.tokens, out)
    rest = tuple(q for q in node.queries() if q not in absorbed)
    if rest and span > 0:
        out.append((rest, blocks, span))


def tree_packs(root):
    out = []
    _pack_tree(root, root.blocks, root.tokens, out)
    return out


def mark_partials(raw):
    """produces_partial = a member query appears in more than one pack
    (workload.py:377-393)."""
    seen = {}
    for qs, _, _ in raw:
        for q in qs:
            seen[q] = seen.get(q, 0) + 1
    return [(tuple(qs), tuple(b), int(kv), any(seen[q] > 1 for q in qs)) for qs, b, kv in raw]


def pack_batch(rows, valid_last, bs):
    """Ordered packs of ``pack_batch`` (packer.py:224-242)."""
    if len(rows) == 0:
        return []
    raw = []
    for root in forest(rows, valid_last, bs):
        raw += tree_packs(root)
    return mark_partials(raw)


def naive_per_node(rows, valid_last, bs):
    """One pack per forest node with tokens, pre-order (packer.py:171-186)."""
    raw = []

    def pre(n):
        if n.tokens > 0:
            raw.append((tuple(n.queries()), n.blocks, n.tokens))
        for k in n.kids:
            pre(k)

    for r in forest(rows, valid_last, bs):
        pre(r)
    return mark_partials(raw)


def query_centric(rows, valid_last, bs):
    """simulator.py:85-96."""
    raw = [((q,), tuple(rows[q]), kv_len(rows, valid_last, bs, q)) for q in range(len(rows))]
    return mark_partials(raw)


# --------------------------------------------------------------------------
# long-KV split, reference mode (simulator.py:117-155)
# --------------------------------------------------------------------------

def split_long_kv(tasks, bs):
    """``tasks``: list of (queries, block_ids, kv_len).  Returns a list of
    (queries, block_ids, kv_len, split_index, split_of)."""
    if not tasks:
        return []
    mean = sum(t[2] for t in tasks) / len(tasks)
    out = []
    for qs, blocks, kv in tasks:
        if kv <= mean:
            out.append((qs, blocks, kv, 0, 1))
            continue
        nblk = max(len(blocks), math.ceil(kv / bs))
        parts = min(math.ceil(kv / mean), nblk)
        base, extra = divmod(nblk, parts)
        pos = used = 0
        for i in range(parts):
            n = base + (1 if i < extra else 0)
            tok = min(n * bs, kv - used)
            out.append((qs, tuple(blocks[pos:pos + n]) if blocks else (), tok, i, parts))
            pos += n
            used += tok
    return out


# --------------------------------------------------------------------------
# traffic floor (simulator.py:25-27, 68-82)
# --------------------------------------------------------------------------

def distinct_census(rows, valid_last, bs):
    best = {}
    for q in range(len(rows)):
        for b, t in units(rows, valid_last, bs, q):
            if best.get(b, 0) < t:
                best[b] = t
    return len(best), sum(best.values())


def theoretical_min_kv_bytes(rows, valid_last, bs, num_kv_heads, head_dim, kv_bytes=2):
    return distinct_census(rows, valid_last, bs)[1] * head_dim * kv_bytes * 2 * num_kv_heads


def check_coverage(rows, valid_last, bs, unit_list):
    """attention.py:258-269 / workload.py:396-413: every query's unit blocks
    (sorted) equal its row, tokens equal kv_len."""
    blocks = {q: [] for q in range(len(rows))}
    toks = {q: 0 for q in range(len(rows))}
    for qs, bl, kv in unit_list:
        for q in qs:
            if q not in blocks:
                return False
            blocks[q] += list(bl)
            toks[q] += kv
    return all(sorted(blocks[q]) == sorted(rows[q]) and toks[q] == kv_len(rows, valid_last, bs, q)
               for q in range(len(rows)))
