"""Block-table builders for the five BASELINE.json workloads (c1..c5).

Each workload is a list of rows; a row is a list of *segments* ``(key, tokens)``.
Segments with the same key are the same KV blocks (that is what "shared prefix"
means in a paged cache), block ids are handed out densely in first-use order,
and a row's last segment may end inside a block (partial last page).

c1 and c5 are exactly the reference's ``generate_workload`` outputs
(``/root/reference/pkg/src/prefixpack/workload.py:162-197``): level-major block
ids, every level length a multiple of the page.  c2..c4 follow SURVEY.md
Appendix C (one ``default_rng(0)`` consumed in the order c2 suffixes, c3
suffixes).  Checksums are asserted in the tests:
sum(kv_len) = 9,216 / 411,931 / 935,245 / 2,228,224 / 1,048,576 and distinct
tokens = 2,048 / 37,147 / 415,053 / 139,264 / 1,048,576.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    rows: list            # list[list[int]] block ids per query
    valid_last: list      # list[int] valid tokens in each row's last block
    block_size: int
    num_heads: int
    num_kv_heads: int
    head_dim: int
    description: str

    @property
    def batch(self) -> int:
        return len(self.rows)

    def seq_lens(self) -> list:
        bs = self.block_size
        return [(len(r) - 1) * bs + v for r, v in zip(self.rows, self.valid_last)]

    def max_blocks(self) -> int:
        return max(len(r) for r in self.rows)

    def num_pool_blocks(self) -> int:
        return 1 + max(max(r) for r in self.rows)

    def distinct_tokens(self) -> int:
        """Distinct KV tokens; a block used at several fill levels counts at its
        fullest use (``simulator.py:68-75``)."""
        best: dict = {}
        bs = self.block_size
        for r, v in zip(self.rows, self.valid_last):
            for i, b in enumerate(r):
                t = v if i == len(r) - 1 else bs
                if best.get(b, 0) < t:
                    best[b] = t
        return sum(best.values())

    def unique_kv_bytes(self, kv_dtype_bytes: int = 2) -> int:
        """Algorithmic HBM bytes of one layer: ``theoretical_min_kv_bytes``
        (``simulator.py:78-82``) = distinct tokens x KVH x d x 2 (K and V) x b."""
        return self.distinct_tokens() * self.num_kv_heads * self.head_dim * 2 * kv_dtype_bytes


def rows_from_segments(seg_rows, block_size: int = 16):
    """Materialise rows of ``(key, tokens)`` segments into block ids.

    A key always maps to the same blocks (first use decides the token count);
    ids are dense in first-use order."""
    next_block = 0
    seen: dict = {}
    rows, valid = [], []
    for segs in seg_rows:
        row: list = []
        last_tokens = 0
        for key, tokens in segs:
            if tokens <= 0:
                continue
            if key not in seen:
                n = -(-tokens // block_size)
                seen[key] = list(range(next_block, next_block + n))
                next_block += n
            row.extend(seen[key])
            last_tokens = tokens
        nblk = -(-last_tokens // block_size)
        rows.append(row)
        valid.append(last_tokens - block_size * (nblk - 1))
    return rows, valid


def generate_levels(level_counts, level_lengths, block_size: int = 16):
    """Same table as ``generate_workload`` (``workload.py:162-197``): level i has
    ``level_counts[i]`` nodes of ``level_lengths[i]`` tokens, ids level-major."""
    levels = len(level_counts)
    nxt = 0
    node_blocks = []
    for lv in range(levels):
        per = level_lengths[lv] // block_size
        this = []
        for _ in range(level_counts[lv]):
            this.append(list(range(nxt, nxt + per)))
            nxt += per
        node_blocks.append(this)
    batch = level_counts[-1]
    rows = []
    for q in range(batch):
        row = []
        for lv in range(levels):
            row.extend(node_blocks[lv][q * level_counts[lv] // batch])
        rows.append(row)
    return rows, [block_size] * batch


def _c2_c3_suffixes():
    rng = np.random.default_rng(0)
    suf2 = rng.integers(64, 513, size=64)
    suf3 = np.exp(rng.uniform(np.log(32), np.log(16384), size=128)).astype(int)
    return [int(x) for x in suf2], [int(x) for x in suf3]


def workload(name: str) -> Workload:
    """Build one of c1..c5 (BASELINE.json ``configs[0..4]``)."""
    bs = 16
    if name == "c1":
        rows, valid = generate_levels((1, 8), (1024, 128), bs)
        return Workload(name, rows, valid, bs, 32, 8, 128,
                        "8 decode queries sharing one 1024-token prefix + 128-token unique suffixes, 32q/8kv, d128")
    if name == "c2":
        suf2, _ = _c2_c3_suffixes()
        segs = [[("sys", 2048), (("doc", i // 16), 4096), (("u", i), suf2[i])] for i in range(64)]
        rows, valid = rows_from_segments(segs, bs)
        return Workload(name, rows, valid, bs, 32, 8, 128,
                        "2k system prompt -> 4 RAG docs of 4k -> 64 requests with 64-512 unique tokens, Llama-3-8B attention (32q/8kv, d128)")
    if name == "c3":
        _, suf3 = _c2_c3_suffixes()
        segs = [[("sys", 4096), (("u", i), suf3[i])] for i in range(128)]
        rows, valid = rows_from_segments(segs, bs)
        return Workload(name, rows, valid, bs, 32, 8, 128,
                        "batch 128, shared 4k prefix, log-uniform suffixes 32-16k tokens (long tail), 32q/8kv, d128")
    if name == "c4":
        segs = [[("sys", 8192), (("u", i), 512)] for i in range(256)]
        rows, valid = rows_from_segments(segs, bs)
        return Workload(name, rows, valid, bs, 64, 8, 128,
                        "Llama-3-70B attention (64q/8kv, d128), batch 256, 8k shared prefix + 512 unique tokens")
    if name == "c5":
        rows, valid = generate_levels((256,), (4096,), bs)
        return Workload(name, rows, valid, bs, 32, 8, 128,
                        "no-sharing control: batch 256, fully unique 4k contexts, 32q/8kv, d128")
    raise KeyError(name)


ALL = ("c1", "c2", "c3", "c4", "c5")
