"""Scheduling paths on the GPU: the tcgen05 kernel's dynamic item counter is
re-armed between launches (repeat launches are bit-identical), the default
kernel choice (all-narrow plans on the streaming kernel) and the concurrent
two-kernel mode (explicit tc_min_rows: packs split across kernels on disjoint
SM shares) match the float64 oracle on sampled queries of full-size configs."""

import random

import numpy as np
import pytest
import torch

import paper_2511_22333_b200 as P
from paper_2511_22333_b200 import configs
from paper_2511_22333_b200.plan import PatPlan
from oracle import attn_oracle as AO

from test_gpu_parity import _close

pytestmark = pytest.mark.gpu


def _setup(name, seed=11, qscale=1.0):
    w = configs.workload(name)
    g = torch.Generator(device="cuda").manual_seed(seed)
    nb = w.num_pool_blocks()
    dt = torch.bfloat16
    kc = torch.randn(nb, w.block_size, w.num_kv_heads, w.head_dim, device="cuda", dtype=dt, generator=g)
    vc = torch.randn(nb, w.block_size, w.num_kv_heads, w.head_dim, device="cuda", dtype=dt, generator=g)
    q = torch.randn(w.batch, w.num_heads, w.head_dim, device="cuda", dtype=dt, generator=g) * qscale
    table = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
    return w, table, q, kc, vc


def _check_sampled(w, q, kc, vc, out, qids):
    for qi in qids:
        row = w.rows[qi]
        n = (len(row) - 1) * w.block_size + w.valid_last[qi]
        idx = torch.tensor(row, device="cuda")
        k = kc[idx].reshape(-1, w.num_kv_heads, w.head_dim)[:n].double().cpu().numpy()
        v = vc[idx].reshape(-1, w.num_kv_heads, w.head_dim)[:n].double().cpu().numpy()
        ref = AO.full_attention(q[qi:qi + 1].double().cpu().numpy(), [k], [v])[0]
        _close(out[qi].double().cpu().numpy(), ref)


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_repeat_launches_bit_identical(name):
    """Dynamic claims change which CTA runs which item, never the result."""
    w, table, q, kc, vc = _setup(name)
    plan = PatPlan.from_table(table, w.num_heads, w.num_kv_heads, w.head_dim)
    first = P.pat_attention(plan, q, kc, vc).clone()
    for _ in range(4):
        again = P.pat_attention(plan, q, kc, vc)
        torch.cuda.synchronize()
        assert torch.equal(again, first)
    plan.close()


@pytest.mark.parametrize("name", ["c5", "c3"])
def test_default_kernel_choice_vs_oracle(name):
    """c5 (no pack wider than 16 rows) runs on the streaming kernel, c3 on the
    tcgen05 kernel; both against the float64 oracle on sampled queries."""
    w, table, q, kc, vc = _setup(name)
    plan = PatPlan.from_table(table, w.num_heads, w.num_kv_heads, w.head_dim)
    inf = plan.info()
    assert inf.n_fwd_kernels == 1
    out = P.pat_attention(plan, q, kc, vc)
    torch.cuda.synchronize()
    rng = random.Random(5)
    _check_sampled(w, q, kc, vc, out, sorted(rng.sample(range(w.batch), 3)))
    plan.close()


@pytest.mark.parametrize("tc", [17, 65])
def test_concurrent_kernels_vs_oracle(tc):
    """Explicit tc_min_rows: narrow packs on the streaming kernel, wide ones on
    the tcgen05 kernel, forked streams on disjoint SM shares, one merge."""
    w, table, q, kc, vc = _setup("c2", qscale=2.0)
    plan = PatPlan.from_table(table, w.num_heads, w.num_kv_heads, w.head_dim, tc_min_rows=tc)
    assert plan.info().n_fwd_kernels >= 2
    out = P.pat_attention(plan, q, kc, vc)
    torch.cuda.synchronize()
    _check_sampled(w, q, kc, vc, out, [0, 17, 40, 63])
    plan.close()


def test_calibrated_cost_model_plans_vs_oracle():
    """The measured B200 profile (tools/calibrate.py) installed as the cost model
    re-chunks the plan; the layer still matches the oracle on sampled queries."""
    import os

    from paper_2511_22333_b200 import calibration as CAL

    saved = CAL.get_cost_model()
    try:
        CAL.load_profile(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                                      "b200_calibration.json"))
        w, table, q, kc, vc = _setup("c3", seed=5)
        plan = PatPlan.from_table(table, w.num_heads, w.num_kv_heads, w.head_dim)
        out = P.pat_attention(plan, q, kc, vc)
        torch.cuda.synchronize()
        _check_sampled(w, q, kc, vc, out, random.Random(5).sample(range(w.batch), 6))
        plan.close()
    finally:
        CAL.set_cost_model(saved)


def test_one_plan_two_streams_concurrently():
    """A plan is immutable after creation: the same plan launched on two streams at
    once (each with its own workspace and output) gives the serial result bit for
    bit -- the dynamic item counters live in the caller's workspace."""
    w = configs.workload("c2")
    table = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
    g = torch.Generator(device="cuda").manual_seed(21)
    nb = w.num_pool_blocks()
    kc = torch.randn(nb, 16, 8, 128, device="cuda", dtype=torch.bfloat16, generator=g)
    vc = torch.randn(nb, 16, 8, 128, device="cuda", dtype=torch.bfloat16, generator=g)
    qa = torch.randn(w.batch, 32, 128, device="cuda", dtype=torch.bfloat16, generator=g)
    qb = torch.randn(w.batch, 32, 128, device="cuda", dtype=torch.bfloat16, generator=g)
    plan = PatPlan.from_table(table, 32, 8, 128)
    ref_a = P.pat_attention(plan, qa, kc, vc).clone()
    ref_b = P.pat_attention(plan, qb, kc, vc).clone()
    torch.cuda.synchronize()
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    wsa = torch.empty(plan.workspace_bytes(), dtype=torch.uint8, device="cuda")
    wsb = torch.empty(plan.workspace_bytes(), dtype=torch.uint8, device="cuda")
    outs = []
    for _ in range(5):
        oa, ob = torch.empty_like(qa), torch.empty_like(qb)
        sa.wait_stream(torch.cuda.current_stream())
        sb.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(sa):
            P.pat_attention(plan, qa, kc, vc, out=oa, workspace=wsa, stream=sa)
        with torch.cuda.stream(sb):
            P.pat_attention(plan, qb, kc, vc, out=ob, workspace=wsb, stream=sb)
        outs.append((oa, ob))
    torch.cuda.synchronize()
    for oa, ob in outs:
        assert torch.equal(oa, ref_a) and torch.equal(ob, ref_b)
    plan.close()
