"""Device-resident decoder (``pat_decoder``): fingerprint, GPU packer and device
scheduler on the stream with no host synchronisation.  Every query of c1..c5
against the float64 GPU reference; re-planning exactly when the table changes;
one CUDA graph replayed across in-place table rewrites (the vLLM full-graph
case); invalid tables reported by ``status``."""

import pytest
import torch

import paper_2511_22333_b200 as P
from paper_2511_22333_b200 import configs
from paper_2511_22333_b200.errors import InvalidSpec

from gpu_ref import check_close, full_attention_gpu, seeded_inputs

pytestmark = pytest.mark.gpu


def _table(w):
    t = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
    bt, sl = t.padded()
    return torch.from_numpy(bt).cuda(), torch.from_numpy(sl).cuda()


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_decoder_every_query(name):
    w = configs.workload(name)
    q, kc, vc = seeded_inputs(w, torch.bfloat16)
    bt, sl = _table(w)
    dec = P.PatDeviceDecoder(w.num_heads, w.num_kv_heads, w.head_dim, max_batch=w.batch,
                             max_blocks=bt.shape[1])
    out = dec.forward(bt, sl, q, kc, vc)
    torch.cuda.synchronize()
    check_close(out, full_attention_gpu(q, kc, vc, w.rows, w.valid_last, w.block_size), name)
    assert dec.status() == 1
    out2 = dec.forward(bt, sl, q, kc, vc)  # same table: no re-plan, same result
    torch.cuda.synchronize()
    assert dec.status() == 1 and torch.equal(out, out2)
    dec.close()


def test_decoder_graph_replays_across_table_rewrites():
    """Capture once; rewrite the block table / seq lens in place (a different
    prefix structure each time, same shapes) and replay: the device re-plans."""
    w = configs.workload("c2")
    bt0, sl0 = _table(w)
    B, mb = bt0.shape
    q, kc, vc = seeded_inputs(w, torch.bfloat16)
    dec = P.PatDeviceDecoder(w.num_heads, w.num_kv_heads, w.head_dim, max_batch=B, max_blocks=mb)
    bt, sl = bt0.clone(), sl0.clone()
    out = torch.empty_like(q)
    dec.forward(bt, sl, q, kc, vc, out=out)  # warm-up outside capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        dec.forward(bt, sl, q, kc, vc, out=out, stream=s)
    torch.cuda.current_stream().wait_stream(s)
    gen = torch.Generator().manual_seed(3)
    for step in range(4):
        rows, valid = [list(r) for r in w.rows], list(w.valid_last)
        if step:
            # shorten some rows (decode of a different batch composition) and
            # permute the unique suffix blocks of others
            for i in torch.randperm(B, generator=gen)[:B // 3].tolist():
                cut = int(torch.randint(1, max(2, len(rows[i]) // 2), (1,), generator=gen))
                rows[i] = rows[i][:len(rows[i]) - cut]
                valid[i] = int(torch.randint(1, 17, (1,), generator=gen))
        t = P.BlockTable(rows, valid, w.block_size)
        nbt, nsl = t.padded(mb)
        bt.copy_(torch.from_numpy(nbt))
        sl.copy_(torch.from_numpy(nsl))
        g.replay()
        torch.cuda.synchronize()
        check_close(out, full_attention_gpu(q, kc, vc, rows, valid, w.block_size), f"graph step {step}")
    assert dec.status() == 1 + 3  # the warm-up table, then three rewrites (step 0 reuses it)
    dec.close()


def test_decoder_invalid_table_reported():
    w = configs.workload("c1")
    bt, sl = _table(w)
    q, kc, vc = seeded_inputs(w, torch.float16)
    dec = P.PatDeviceDecoder(w.num_heads, w.num_kv_heads, w.head_dim, max_batch=w.batch, max_blocks=bt.shape[1])
    bt[2, 1] = bt[2, 0]  # a repeated block in row 2
    dec.forward(bt, sl, q, kc, vc)
    with pytest.raises(InvalidSpec):
        dec.status()
    dec.close()
