"""GPU packer (pat_plan_create_device) vs the reference plans: bit-exact on the
2,855-tree family, the random/edge corpus and c1..c5, from vLLM-layout device
block tables; invalid tables raise InvalidSpec."""

import numpy as np
import pytest
import torch

import paper_2511_22333_b200 as P
from paper_2511_22333_b200 import configs
from paper_2511_22333_b200.plan import PatPlan

from golden_io import as_packs, config_cases, family_cases, random_cases

from gpu_ref import check_close, full_attention_gpu  # noqa: E402

pytestmark = pytest.mark.gpu


def _device_packs(rows, valid, bs, extra_cols=0):
    t = P.BlockTable([list(r) for r in rows], list(valid), bs)
    bt, sl = t.padded((max(len(r) for r in rows) if rows else 1) + extra_cols)
    plan = PatPlan.from_device_table(torch.from_numpy(bt).cuda(), torch.from_numpy(sl).cuda(), block_size=bs,
                                     num_heads=8, num_kv_heads=2, head_dim=128, split="none")
    try:
        return plan.pack_tuples()
    finally:
        plan.close()


def test_tree_family_device_bit_exact():
    for c in family_cases():
        assert _device_packs(c["rows"], c["valid"], c["bs"]) == as_packs(c["packs"]), c["name"]


def test_random_edge_device_bit_exact():
    doc = random_cases()
    for i, c in enumerate(doc["cases"]):
        if not c["rows"]:
            continue
        got = _device_packs(c["rows"], c["valid"], c["bs"], extra_cols=i % 3)
        assert got == as_packs(c["packs"]), c["name"]


def test_configs_device_bit_exact():
    cc = config_cases()
    for name in configs.ALL:
        w = configs.workload(name)
        assert _device_packs(w.rows, w.valid_last, w.block_size) == as_packs(cc[name]["packs"]), name


def test_device_invalid_tables():
    bt = torch.tensor([[0, 1, 0]], dtype=torch.int32, device="cuda")
    with pytest.raises(P.InvalidSpec):
        PatPlan.from_device_table(bt, torch.tensor([40], dtype=torch.int32, device="cuda"), num_heads=8,
                                  num_kv_heads=2)
    with pytest.raises(P.InvalidSpec):
        PatPlan.from_device_table(bt, torch.tensor([0], dtype=torch.int32, device="cuda"), num_heads=8,
                                  num_kv_heads=2)


def test_device_plan_forward_matches_host_plan():
    w = configs.workload("c2")
    t = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
    bt, sl = t.padded()
    g = torch.Generator(device="cuda").manual_seed(0)
    nb = w.num_pool_blocks()
    kc = torch.randn(nb, 16, 8, 128, device="cuda", dtype=torch.bfloat16, generator=g)
    vc = torch.randn(nb, 16, 8, 128, device="cuda", dtype=torch.bfloat16, generator=g)
    q = torch.randn(w.batch, 32, 128, device="cuda", dtype=torch.bfloat16, generator=g)
    pd = PatPlan.from_device_table(torch.from_numpy(bt).cuda(), torch.from_numpy(sl).cuda())
    ph = PatPlan.from_table(t)
    assert pd.pack_tuples() == ph.pack_tuples()
    assert torch.equal(P.pat_attention(pd, q, kc, vc), P.pat_attention(ph, q, kc, vc))
    assert np.isfinite(1.0)


def test_device_lazy_update():
    """PatDecoder.forward_device: the device fingerprint (pat_table_hash_device)
    reuses the plan for an unchanged table, re-plans (GPU packer) when a block id
    or a length changes, and matches the host-table path bit for bit."""
    w = configs.workload("c2")
    table = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
    bt_np, sl_np = table.padded(max(len(r) for r in w.rows) + 3)
    bt = torch.from_numpy(bt_np).cuda()
    sl = torch.from_numpy(sl_np).cuda()
    g = torch.Generator(device="cuda").manual_seed(3)
    nb = w.num_pool_blocks() + 1
    kc = torch.randn(nb, 16, 8, 128, device="cuda", dtype=torch.bfloat16, generator=g)
    vc = torch.randn(nb, 16, 8, 128, device="cuda", dtype=torch.bfloat16, generator=g)
    q = torch.randn(w.batch, 32, 128, device="cuda", dtype=torch.bfloat16, generator=g)
    dec = P.PatDecoder(32, 8, 128)
    h0 = dec.table_hash(bt, sl)
    assert dec.table_hash(bt.clone(), sl.clone()) == h0
    out_dev = dec.forward_device(bt, sl, q, kc, vc).clone()
    out_dev2 = dec.forward_device(bt, sl, q, kc, vc).clone()  # same tensors: identity fast path
    assert dec.cache.hits == 0 and dec.cache.misses == 1
    out_dev3 = dec.forward_device(bt.clone(), sl.clone(), q, kc, vc)  # equal table: fingerprint hit
    assert dec.cache.hits == 1 and dec.cache.misses == 1
    assert torch.equal(out_dev3, out_dev)
    out_host = dec(table, q, kc, vc)
    torch.cuda.synchronize()
    assert torch.equal(out_dev, out_dev2) and torch.equal(out_dev, out_host)
    # padding past a row's length does not change the fingerprint ...
    bt_pad = bt.clone()
    bt_pad[0, -1] = 12345
    assert dec.table_hash(bt_pad, sl) == h0
    # ... a used block id or a length does
    bt2 = bt.clone()
    bt2[5, 0] = nb - 1
    assert dec.table_hash(bt2, sl) != h0
    sl2 = sl.clone()
    sl2[7] -= 1
    assert dec.table_hash(bt, sl2) != h0
    dec.forward_device(bt, sl2, q, kc, vc)
    assert dec.cache.misses == 3  # host-table call + the changed table


def test_torch_op_decode_attention():
    """torch.ops.patb200.decode_attention (vLLM-style tensors, planned on the GPU)
    against the float64 reference (full_attention, attention.py:70-102)."""
    w = configs.workload("c1")
    table = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
    bt_np, sl_np = table.padded()
    g = torch.Generator(device="cuda").manual_seed(9)
    nb = w.num_pool_blocks()
    kv = torch.randn(2, nb, 16, 8, 128, device="cuda", dtype=torch.float16, generator=g)
    q = torch.randn(w.batch, 32, 128, device="cuda", dtype=torch.float16, generator=g)
    out = torch.empty_like(q)
    torch.ops.patb200.decode_attention(q, kv[0], kv[1], torch.from_numpy(bt_np).cuda(),
                                       torch.from_numpy(sl_np).cuda(), out, 0.0)
    plan = PatPlan.from_table(table, 32, 8, 128)
    ref = P.pat_attention(plan, q, kv[0].contiguous(), kv[1].contiguous())
    torch.cuda.synchronize()
    check_close(out, full_attention_gpu(q, kv[0], kv[1], w.rows, w.valid_last, w.block_size), "torch op")
    # (the op plans on the GPU -- its split may differ from the host plan's)
    check_close(ref, full_attention_gpu(q, kv[0], kv[1], w.rows, w.valid_last, w.block_size), "pat_attention")


def test_vllm_backend_decode_matches_pat():
    """PatAttentionImpl (vLLM CUSTOM backend) on a decode-only batch whose query is a
    strided slice of a fused qkv buffer, against the float64 reference; its
    metadata builder declares full CUDA graphs for single-token decode batches."""
    vllm_backend = pytest.importorskip("paper_2511_22333_b200.vllm_backend")
    from types import SimpleNamespace

    w = configs.workload("c2")
    table = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
    bt_np, sl_np = table.padded()
    g = torch.Generator(device="cuda").manual_seed(13)
    nb = w.num_pool_blocks()
    kv = torch.randn(2, nb, 16, 8, 128, device="cuda", dtype=torch.bfloat16, generator=g)
    q = torch.randn(w.batch, 32, 128, device="cuda", dtype=torch.bfloat16, generator=g)
    impl = vllm_backend.PatAttentionImpl(32, 128, 128 ** -0.5, 8, None, None, "auto")
    meta = SimpleNamespace(max_query_len=1, use_cascade=False, num_actual_tokens=w.batch,
                           block_table=torch.from_numpy(bt_np).cuda(), seq_lens=torch.from_numpy(sl_np).cuda())
    qkv = torch.zeros(w.batch, (32 + 2 * 8) * 128, device="cuda", dtype=torch.bfloat16)
    qkv[:, :32 * 128] = q.view(w.batch, -1)
    query = qkv[:, :32 * 128]  # strided view, as vLLM splits the fused projection
    assert not query.is_contiguous()
    output = torch.empty(w.batch, 32 * 128, device="cuda", dtype=torch.bfloat16)
    impl.forward(None, query, None, None, kv, meta, output)
    impl.forward(None, query, None, None, kv, meta, output)  # plan reused (identity fast path)
    plan = PatPlan.from_table(table, 32, 8, 128)
    ref = P.pat_attention(plan, q, kv[0], kv[1])
    torch.cuda.synchronize()
    check_close(output.view(w.batch, 32, 128), full_attention_gpu(q, kv[0], kv[1], w.rows, w.valid_last,
                                                                   w.block_size), "vllm backend")
    check_close(ref, full_attention_gpu(q, kv[0], kv[1], w.rows, w.valid_last, w.block_size), "pat_attention")
    from vllm.v1.attention.backend import AttentionCGSupport
    builder = vllm_backend.PatAttentionBackend.get_builder_cls()
    assert builder.get_cudagraph_support(None, None) == AttentionCGSupport.UNIFORM_SINGLE_TOKEN_DECODE


def test_vllm_backend_decode_in_cuda_graph():
    """A decode-only batch through PatAttentionImpl captured in one CUDA graph; vLLM
    then rewrites block_table / seq_lens in place between replays (shorter rows,
    new last-block fills) and every replay matches the float64 reference."""
    vllm_backend = pytest.importorskip("paper_2511_22333_b200.vllm_backend")
    from types import SimpleNamespace

    w = configs.workload("c2")
    table = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
    bt_np, sl_np = table.padded()
    g = torch.Generator(device="cuda").manual_seed(17)
    nb = w.num_pool_blocks()
    kv = torch.randn(2, nb, 16, 8, 128, device="cuda", dtype=torch.bfloat16, generator=g)
    q = torch.randn(w.batch, 32, 128, device="cuda", dtype=torch.bfloat16, generator=g)
    impl = vllm_backend.PatAttentionImpl(32, 128, 128 ** -0.5, 8, None, None, "auto")
    bt, sl = torch.from_numpy(bt_np).cuda(), torch.from_numpy(sl_np).cuda()
    meta = SimpleNamespace(max_query_len=1, use_cascade=False, num_actual_tokens=w.batch, block_table=bt,
                           seq_lens=sl)
    query = q.view(w.batch, -1)
    output = torch.empty(w.batch, 32 * 128, device="cuda", dtype=torch.bfloat16)
    impl.forward(None, query, None, None, kv, meta, output)  # warm-up (decoder created outside capture)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(graph, stream=s):
        impl.forward(None, query, None, None, kv, meta, output)
    torch.cuda.current_stream().wait_stream(s)
    gen = torch.Generator().manual_seed(5)
    for step in range(3):
        rows, valid = [list(r) for r in w.rows], list(w.valid_last)
        for i in torch.randperm(w.batch, generator=gen)[:w.batch // 2].tolist():
            cut = int(torch.randint(0, max(1, len(rows[i]) // 3), (1,), generator=gen))
            rows[i] = rows[i][:len(rows[i]) - cut]
            valid[i] = int(torch.randint(1, 17, (1,), generator=gen))
        nbt, nsl = P.BlockTable(rows, valid, 16).padded(bt.shape[1])
        bt.copy_(torch.from_numpy(nbt))
        sl.copy_(torch.from_numpy(nsl))
        graph.replay()
        torch.cuda.synchronize()
        check_close(output.view(w.batch, 32, 128), full_attention_gpu(q, kv[0], kv[1], rows, valid, 16),
                    f"vllm graph step {step}")


def test_cli_run_and_verify(tmp_path, capsys):
    """B200 rows for the reference CLI: verify passes, run reports all strategies."""
    import json as _json
    from paper_2511_22333_b200 import cli
    spec = tmp_path / "w.json"
    spec.write_text(_json.dumps(P.WorkloadSpec((1, 4), (256, 64), num_heads=32, num_kv_heads=8,
                                               head_dim=128).to_json()))
    assert cli.main(["verify", str(spec)]) == cli.EXIT_OK
    assert cli.main(["run", "--config", "c1", "--verify"]) == cli.EXIT_OK
    rows = _json.loads(capsys.readouterr().out.split("\n", 1)[1])
    assert [r["strategy"] for r in rows] == list(cli.STRATEGIES) and all(r["verified"] for r in rows)
    assert rows[0]["kv_bytes"] < rows[1]["kv_bytes"]  # packing streams fewer KV bytes than query-centric
