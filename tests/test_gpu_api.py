"""GPU side of the numerics API: ``cta_partial`` (the sm_100a forward kernel with
every partial exposed) folded with ``merge_partials`` reproduces the
reference's merged output and ``full_attention`` on the reference's own
fixtures (``tests/golden/api_surface.json.gz``)."""

import gzip
import json
import os

import numpy as np
import pytest
import torch

import paper_2511_22333_b200 as P

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
ATOL, RTOL = 2e-3, 1e-2


def test_cta_partial_fold_matches_reference():
    with gzip.open(os.path.join(HERE, "golden", "api_surface.json.gz"), "rt") as fh:
        cases = json.load(fh)["partials"]
    for c in cases:
        q, k, v, h = np.array(c["q"]), np.array(c["k"]), np.array(c["v"]), c["h"]
        a = P.cta_partial(q, k[:h], v[:h], dtype=torch.float16)
        b = P.cta_partial(q, k[h:], v[h:], dtype=torch.float16)
        nq, H, d = q.shape
        merged = np.stack([np.stack([P.merge_partials([a.at(i, j), b.at(i, j)]) for j in range(H)])
                           for i in range(nq)])
        for ref in (np.array(c["merged"]), np.array(c["full"])):
            err = np.abs(merged - ref)
            assert (err <= ATOL + RTOL * np.abs(ref)).all(), err.max()
        # a single partial normalises to the span's own attention output
        ref_a = np.array(c["a_ws"]) / np.array(c["a_sum"])[:, :, None]
        assert (np.abs(a.weighted_sum / a.exp_sum[:, :, None] - ref_a) <= ATOL + RTOL * np.abs(ref_a)).all()
        # the log-sum-exp representation equals the reference's m + ln(l)
        lse_ref = np.array(c["a_max"]) + np.log(np.array(c["a_sum"]))
        assert np.abs(a.max_score - lse_ref).max() < 2e-3
    full = P.full_attention(q, [k] * nq, [v] * nq)
    assert np.abs(full - np.array(cases[-1]["full"])).max() < 1e-9
