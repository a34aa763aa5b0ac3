"""One pass of every kernel family on small inputs, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool memcheck python tools/sanitize_run.py

tcgen05 forward (regular + transposed narrow items, bf16 and fp16), the
mma.sync streaming kernel (tc_min_rows = -1), the merge kernel, the GPU packer
and the device table hash.  Checks the outputs against the float64 GPU
reference so a silent corruption also fails the run."""

import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
import paper_2511_22333_b200 as P  # noqa: E402
from paper_2511_22333_b200 import configs  # noqa: E402
from gpu_ref import check_close, full_attention_gpu, seeded_inputs  # noqa: E402


def main():
    for name, dt, tc in [("c1", torch.bfloat16, 0), ("c1", torch.float16, 0), ("c1", torch.bfloat16, -1),
                         ("c2", torch.bfloat16, 0)]:
        w = configs.workload(name)
        q, kc, vc = seeded_inputs(w, dt)
        table = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
        plan = P.PatPlan.from_table(table, w.num_heads, w.num_kv_heads, w.head_dim, tc_min_rows=tc)
        out = P.pat_attention(plan, q, kc, vc)
        torch.cuda.synchronize()
        check_close(out, full_attention_gpu(q, kc, vc, w.rows, w.valid_last, w.block_size), f"{name} {dt} tc={tc}")
        plan.close()
        print("ok", name, dt, tc, flush=True)
    # GPU packer + device fingerprint (vLLM-style tables)
    w = configs.workload("c1")
    q, kc, vc = seeded_inputs(w, torch.float16)
    table = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
    bt, sl = table.padded()
    dec = P.PatDecoder(w.num_heads, w.num_kv_heads, w.head_dim)
    out = dec.forward_device(torch.from_numpy(bt).cuda(), torch.from_numpy(sl).cuda(), q, kc, vc)
    torch.cuda.synchronize()
    check_close(out, full_attention_gpu(q, kc, vc, w.rows, w.valid_last, w.block_size), "device packer")
    print("ok device packer", flush=True)


if __name__ == "__main__":
    main()
