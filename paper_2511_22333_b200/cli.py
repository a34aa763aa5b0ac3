"""B200 backend for the reference CLI's `run` / `verify` rows.

    python -m paper_2511_22333_b200.cli verify WORKLOAD.json [--seed 0] [--strategy packed] [--tol 1e-2]
    python -m paper_2511_22333_b200.cli run WORKLOAD.json [--strategies packed query_centric naive] [--verify]
    python -m paper_2511_22333_b200.cli run --config c2 ...

WORKLOAD.json is the reference WorkloadSpec format (``WorkloadSpec.from_json``);
``--config`` takes a BASELINE.json configuration instead.  Rows mirror
``prefixpack.cli.run_strategy`` (cli.py:91-138) with measured B200 numbers in
place of the simulator's: ``kv_bytes`` (KV bytes the plan streams),
``intermediate_bytes`` (fp32 partials written and read back), ``latency_us``
(one layer, CUDA events, L2 flushed), ``pack_count``, ``task_count`` (work
items).  Exit codes follow the reference (cli.py:24-27): 0 ok, 2 invalid
spec, 3 verification failed.  The verification reference is a float64
full-attention computed on the GPU from the same rounded inputs
(``full_attention`` + ``max_rel_error``, attention.py:70-102, 272-275)."""

from __future__ import annotations

import argparse
import json
import sys

import numpy as np
import torch

from .attention import pat_attention
from .errors import InvalidSpec
from .packer import baseline_query_centric, naive_per_node, pack_batch
from .plan import PatPlan
from .workload import BlockTable, WorkloadSpec, generate_workload

EXIT_OK = 0
EXIT_INVALID_SPEC = 2
EXIT_VERIFY_FAILED = 3
STRATEGIES = ("packed", "query_centric", "naive")


def _load(args):
    if args.config:
        from . import configs

        w = configs.workload(args.config)
        table = BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
        return table, w.num_heads, w.num_kv_heads, w.head_dim
    with open(args.workload) as fh:
        spec = WorkloadSpec.from_json(json.load(fh))
    return generate_workload(spec, args.seed), spec.num_heads, spec.num_kv_heads, spec.head_dim


def _plan(strategy, table, H, KVH, d):
    if strategy == "packed":
        return PatPlan.from_table(table, H, KVH, d), len(pack_batch(table).packs)
    part = baseline_query_centric(table) if strategy == "query_centric" else naive_per_node(table)
    units = [(p.query_ids, p.block_ids, p.kv_len) for p in part.packs]
    return PatPlan.from_units(table, units, H, KVH, d, split="native"), len(part.packs)


def _inputs(table, H, KVH, d, seed, dtype):
    g = torch.Generator(device="cuda").manual_seed(seed)
    nb = max(b for r in table.rows for b in r) + 1
    kc = torch.randn(nb, table.block_size, KVH, d, device="cuda", dtype=dtype, generator=g)
    vc = torch.randn(nb, table.block_size, KVH, d, device="cuda", dtype=dtype, generator=g)
    q = torch.randn(table.num_queries, H, d, device="cuda", dtype=dtype, generator=g)
    return q, kc, vc


def _reference(table, q, kc, vc):
    """float64 full attention per query (attention.py:70-102) on the GPU."""
    H, d = q.shape[1], q.shape[2]
    KVH = kc.shape[2]
    out = torch.empty(q.shape, dtype=torch.float64, device=q.device)
    for i, row in enumerate(table.rows):
        n = table.kv_len(i)
        idx = torch.tensor(row, device=q.device)
        k = kc[idx].reshape(-1, KVH, d)[:n].double()
        v = vc[idx].reshape(-1, KVH, d)[:n].double()
        qi = q[i].double().reshape(KVH, H // KVH, d)
        s = torch.einsum("kgd,tkd->kgt", qi, k) / d ** 0.5
        out[i] = torch.einsum("kgt,tkd->kgd", torch.softmax(s, dim=-1), v).reshape(H, d)
    return out


def _max_rel_error(x, ref) -> float:
    """attention.py:272-275: max |x - ref| / max |ref|."""
    return float((x - ref).abs().max() / ref.abs().max())


def run_strategy(strategy, table, H, KVH, d, seed, verify, tol, dtype=torch.bfloat16, iters=10):
    plan, npacks = _plan(strategy, table, H, KVH, d)
    inf = plan.info()
    q, kc, vc = _inputs(table, H, KVH, d, seed, dtype)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    out = pat_attention(plan, q, kc, vc)
    ts = []
    for _ in range(iters):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        pat_attention(plan, q, kc, vc, out=out)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    tok = KVH * d * 2 * 2
    pk = plan.packs()
    row = {"strategy": strategy, "backend": "b200",
           "kv_bytes": int(np.sum(pk.kv_len)) * tok,
           "intermediate_bytes": int(inf.n_slots) * H * (d + 1) * 4 * 2,
           "latency_us": round(float(np.median(ts)), 2), "pack_count": npacks, "task_count": int(inf.n_items),
           "verified": None}
    if verify:
        err = _max_rel_error(out.double(), _reference(table, q, kc, vc))
        row["verified"] = bool(err <= tol)
        row["max_rel_error"] = err
    plan.close()
    return row


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="patb200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("run", "verify"):
        p = sub.add_parser(name)
        p.add_argument("workload", nargs="?")
        p.add_argument("--config", default=None)
        p.add_argument("--seed", type=int, default=0)
        p.add_argument("--tol", type=float, default=1e-2)
    sub.choices["run"].add_argument("--strategies", nargs="+", default=list(STRATEGIES), choices=STRATEGIES)
    sub.choices["run"].add_argument("--verify", action="store_true")
    sub.choices["verify"].add_argument("--strategy", default="packed", choices=STRATEGIES)
    args = ap.parse_args(argv)
    try:
        if not args.config and not args.workload:
            raise InvalidSpec("a workload JSON or --config is required")
        table, H, KVH, d = _load(args)
    except (InvalidSpec, OSError, ValueError, KeyError) as exc:
        print(f"invalid workload spec: {exc}", file=sys.stderr)
        return EXIT_INVALID_SPEC
    if args.cmd == "verify":
        row = run_strategy(args.strategy, table, H, KVH, d, args.seed, True, args.tol)
        print(f"max relative error: {row['max_rel_error']:.3e} (tolerance {args.tol:.1e})")
        return EXIT_OK if row["verified"] else EXIT_VERIFY_FAILED
    rows = [run_strategy(s, table, H, KVH, d, args.seed, args.verify, args.tol) for s in args.strategies]
    print(json.dumps(rows, indent=1))
    return EXIT_VERIFY_FAILED if any(r["verified"] is False for r in rows) else EXIT_OK


if __name__ == "__main__":
    sys.exit(main())
