"""Every query and every head of the full-size BASELINE configs, against a
float64 GPU restatement of ``full_attention`` (reference ``attention.py:70-102``)
on the same rounded inputs: c2 (bf16 and fp16), c3, c4, c5, c4's per-rank
head-shard shapes (8k shared prefix, B=256; H/KVH = 32/4, 16/2, 8/1), and the
opt-in pair-item schedule.  Tolerance: north_star 2e-3 abs + 1e-2 rel."""

import pytest
import torch

import paper_2511_22333_b200 as P
from paper_2511_22333_b200 import configs
from paper_2511_22333_b200.plan import PatPlan

from gpu_ref import check_close, full_attention_gpu, seeded_inputs

pytestmark = pytest.mark.gpu


def _run(w, dtype, num_heads=None, num_kv_heads=None, **plan_kw):
    H = num_heads or w.num_heads
    KVH = num_kv_heads or w.num_kv_heads
    q, kc, vc = seeded_inputs(w, dtype, num_heads=H, num_kv_heads=KVH)
    table = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
    plan = PatPlan.from_table(table, H, KVH, w.head_dim, **plan_kw)
    try:
        out = P.pat_attention(plan, q, kc, vc)
        torch.cuda.synchronize()
    finally:
        plan.close()
    ref = full_attention_gpu(q, kc, vc, w.rows, w.valid_last, w.block_size)
    return out, ref


@pytest.mark.parametrize("name,dtype", [("c2", torch.bfloat16), ("c2", torch.float16), ("c3", torch.bfloat16),
                                        ("c4", torch.bfloat16), ("c5", torch.bfloat16), ("c1", torch.float16)])
def test_full_config_every_query(name, dtype):
    w = configs.workload(name)
    out, ref = _run(w, dtype)
    err, mre = check_close(out, ref, f"{name} {dtype}")
    assert mre < 5e-3


@pytest.mark.parametrize("heads,kv_heads", [(32, 4), (16, 2), (8, 1)])
def test_c4_head_shard_shapes(heads, kv_heads):
    """The per-rank problem of c4 sharded 2/4/8 ways by kv heads (shard.py): same
    table, 64/8 * (8/n) query heads over 8/n kv heads."""
    w = configs.workload("c4")
    out, ref = _run(w, torch.bfloat16, num_heads=heads, num_kv_heads=kv_heads)
    check_close(out, ref, f"c4 shard {heads}/{kv_heads}")


@pytest.mark.parametrize("name", ["c2", "c4"])
def test_pair_items_every_query(name):
    """PAT_PLAN_PAIR_ITEMS: rows 0-127 and 128-255 of a wide pack on the two item
    pipelines of one CTA, reading one KV stream."""
    w = configs.workload(name)
    out, ref = _run(w, torch.bfloat16, pair_items=True)
    check_close(out, ref, f"{name} pair items")
