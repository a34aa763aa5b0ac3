"""Scheduler cost model (pat_set_cost_model / calibration.load_profile).  CPU only:
plans are built host-side, nothing runs on a GPU."""

import json
import os

import pytest

import paper_2511_22333_b200 as P
from paper_2511_22333_b200 import calibration as CAL
from paper_2511_22333_b200 import configs
from paper_2511_22333_b200.errors import InvalidSpec
from paper_2511_22333_b200.plan import PatPlan

PROFILE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                       "b200_calibration.json")


@pytest.fixture
def restore_model():
    saved = CAL.get_cost_model()
    yield
    CAL.set_cost_model(saved)


def _units(name):
    w = configs.workload(name)
    t = P.BlockTable([list(r) for r in w.rows], list(w.valid_last), w.block_size)
    plan = PatPlan.from_table(t, w.num_heads, w.num_kv_heads, w.head_dim, split="native", host_only=True)
    try:
        return plan.info().n_units
    finally:
        plan.close()


def test_default_model_is_the_measured_two_lane_constants():
    m = CAL.get_cost_model()
    assert (m.tc_item_ns, m.tc_item_row_ns, m.tc_step_ns, m.stream_item_ns, m.hbm_bytes_per_ns) == \
        (3600.0, 2000.0, 1440.0, 1500.0, 6500.0)


def test_set_get_roundtrip_and_validation(restore_model):
    m = CAL.CostModel(1400.0, 3300.0, 920.0, 1500.0, 5300.0)
    CAL.set_cost_model(m)
    assert CAL.get_cost_model() == m
    for bad in (CAL.CostModel(1.0, 0.0, 0.0, 1.0, 1.0), CAL.CostModel(1.0, 0.0, 1.0, 1.0, -5.0),
                CAL.CostModel(-1.0, 0.0, 1.0, 1.0, 1.0)):
        with pytest.raises(InvalidSpec):
            CAL.set_cost_model(bad)
    assert CAL.get_cost_model() == m


def test_item_cost_steers_the_native_split(restore_model):
    base = CAL.get_cost_model()
    # expensive item boundaries -> fewer, longer units; free boundaries -> at least as many
    CAL.set_cost_model(CAL.CostModel(200000.0, 0.0, base.tc_step_ns, base.stream_item_ns, base.hbm_bytes_per_ns))
    few = _units("c3")
    CAL.set_cost_model(CAL.CostModel(0.0, 0.0, base.tc_step_ns, base.stream_item_ns, base.hbm_bytes_per_ns))
    many = _units("c3")
    assert few < many


def test_profile_fit_matches_committed_calibration(restore_model):
    with open(PROFILE) as fh:
        prof = json.load(fh)
    m = CAL.model_from_profile(prof)
    f = prof["fits"]
    # the fitted model reproduces the 4-row and 128-row per-item costs
    assert m.tc_item_ns + m.tc_item_row_ns * 4 / 128 == pytest.approx(f["tcgen05_rows4"]["per_item_us"] * 1e3)
    assert m.tc_item_ns + m.tc_item_row_ns == pytest.approx(f["tcgen05_rows128"]["per_item_us"] * 1e3)
    assert 500 < m.tc_step_ns < 2000 and 3000 < m.hbm_bytes_per_ns < 8000
    assert CAL.load_profile(PROFILE) == CAL.get_cost_model()
