"""Prefix forest and the top-down pack heuristic as inspectable Python objects
(drop-in names of ``prefixpack.workload`` / ``prefixpack.packer``).

The hot path never builds these: ``pack_batch`` runs the native packer
(``csrc/pat_packer_host.cpp``, GPU pass ``csrc/pat_packer_dev.cu``), which
derives the same partition without materialising a tree.  They exist for
callers that walk the forest (reports, ablations, tests), with the reference's
types and semantics:

* ``build_forest`` (reference ``workload.py:245-297``): maximal shared runs
  over (block, tokens) units; a single-query group is one leaf holding its
  whole remaining suffix; queries ending where a run ends are empty leaves
  listed before the child groups, groups in first-appearance order.  Built
  here from a unit trie (rows inserted in query order, so child order is first
  appearance) compressed into runs -- linear in the table size.
* ``tree_heuristic`` / ``pack_forest`` (reference ``packer.py:105-168``): a
  child is merged into its parent's pack iff 2 (s_child + terminal_child) >
  span, span being the accumulated inherited tokens; ties split.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Iterator, Optional, Sequence

from .workload import BlockTable, CtaPack


@dataclass
class PrefixNode:
    """A run of KV blocks shared by every query below it (``workload.py:200-227``);
    ``query_ids`` is set on leaves only."""

    block_ids: tuple
    token_len: int
    num_queries: int
    children: list = field(default_factory=list)
    query_ids: tuple = ()

    @property
    def is_leaf(self) -> bool:
        return not self.children

    def subtree_queries(self) -> list:
        out, stack = [], [self]
        while stack:
            n = stack.pop()
            if n.is_leaf:
                out.extend(n.query_ids)
            else:
                stack.extend(reversed(n.children))
        return out


@dataclass
class PrefixForest:
    roots: list
    block_size: int

    def iter_nodes(self) -> Iterator[PrefixNode]:
        stack = list(reversed(self.roots))
        while stack:
            n = stack.pop()
            yield n
            stack.extend(reversed(n.children))

    @property
    def node_count(self) -> int:
        return sum(1 for _ in self.iter_nodes())


class _Trie:
    __slots__ = ("kids", "ends", "queries")

    def __init__(self):
        self.kids: dict = {}     # unit -> _Trie, insertion (= first appearance) order
        self.ends: list = []     # queries whose row ends at this trie node
        self.queries: list = []  # queries passing through (in query order)


def build_forest(table: BlockTable) -> PrefixForest:
    table.validate()
    units = [table.row_units(q) for q in range(table.num_queries)]
    top = _Trie()
    for q, row in enumerate(units):
        t = top
        for u in row:
            t = t.kids.setdefault(u, _Trie())
            t.queries.append(q)
        t.ends.append(q)

    def grow(t: _Trie, first_unit, depth: int) -> PrefixNode:
        # t is the trie node reached by `first_unit` at row position `depth`
        qs = t.queries
        if len(qs) == 1:
            suffix = units[qs[0]][depth:]
            return PrefixNode(tuple(b for b, _ in suffix), sum(n for _, n in suffix), 1, query_ids=(qs[0],))
        run = [first_unit]
        # the run continues while nobody ends here and all rows take the same next unit
        while not t.ends and len(t.kids) == 1:
            (u, nxt), = t.kids.items()
            run.append(u)
            t = nxt
            depth += 1
        children = [PrefixNode((), 0, 1, query_ids=(q,)) for q in t.ends]
        children += [grow(k, u, depth + 1) for u, k in t.kids.items()]
        return PrefixNode(tuple(b for b, _ in run), sum(n for _, n in run), len(qs), children=children)

    roots = [grow(k, u, 0) for u, k in top.kids.items()]
    return PrefixForest(roots=roots, block_size=table.block_size)


def flatten_forest(forest: PrefixForest) -> dict:
    """Every query's block row from its root-to-leaf path (``workload.py:300-314``)."""
    rows: dict = {}
    stack = [(r, ()) for r in reversed(forest.roots)]
    while stack:
        node, prefix = stack.pop()
        path = prefix + tuple(node.block_ids)
        if node.is_leaf:
            for q in node.query_ids:
                rows[q] = list(path)
        stack.extend((c, path) for c in reversed(node.children))
    return rows


def _terminal(node: PrefixNode) -> int:
    """Queries whose KV ends at the node's run (``packer.py:105-110``)."""
    if node.is_leaf:
        return 1
    return sum(1 for c in node.children if c.is_leaf and c.token_len == 0)


def tree_heuristic(root: PrefixNode, inherited_blocks: Optional[Sequence[int]] = None,
                   inherited_tokens: Optional[int] = None) -> list:
    """Top-down pack of one prefix tree (``packer.py:124-161``): returns CtaPacks
    in emission order (children before the node's own remaining pack)."""
    blocks = tuple(inherited_blocks) if inherited_blocks is not None else tuple(root.block_ids)
    span = inherited_tokens if inherited_tokens is not None else root.token_len
    node = root
    # single-query chains fuse into one span (no zero-profit pack, packer.py:113-121)
    while not node.is_leaf and node.num_queries == 1:
        node = node.children[0]
        blocks += tuple(node.block_ids)
        span += node.token_len
    if node.is_leaf:
        return [CtaPack(query_ids=tuple(node.query_ids), block_ids=blocks, kv_len=span)] if span else []
    out, absorbed = [], set()
    for child in node.children:
        if child.is_leaf and child.token_len == 0:
            continue  # ends with the shared span: stays in this node's pack
        merge = 2 * (child.num_queries + _terminal(child)) > span
        if merge:
            out += tree_heuristic(child, blocks + tuple(child.block_ids), span + child.token_len)
            absorbed.update(child.subtree_queries())
        else:
            out += tree_heuristic(child, child.block_ids, child.token_len)
    rest = tuple(q for q in node.subtree_queries() if q not in absorbed)
    if rest and span > 0:
        out.append(CtaPack(query_ids=rest, block_ids=blocks, kv_len=span))
    return out


def pack_forest(forest: PrefixForest) -> list:
    """``tree_heuristic`` over every root (``packer.py:164-168``)."""
    return [p for r in forest.roots for p in tree_heuristic(r)]


__all__ = ["PrefixNode", "PrefixForest", "build_forest", "flatten_forest", "tree_heuristic", "pack_forest"]
