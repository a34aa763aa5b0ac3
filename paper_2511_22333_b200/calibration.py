"""Scheduler cost model: read / set it, or load a measured B200 profile.

The native KV split and the longest-first item order (`pat_schedule_host.cpp`)
estimate each work item with the model in ``include/pat.h``
(``pat_cost_model``).  ``tools/calibrate.py`` measures the per-tile and
per-item costs on the GPU and writes ``profiles/b200_calibration.json``;
``load_profile`` turns those fits into a model (the
B200 counterpart of the reference's A100 tile tables, ``tiles.py``)."""

from __future__ import annotations

import ctypes as C
import json
from dataclasses import asdict, dataclass

from . import _native as N


@dataclass
class CostModel:
    tc_item_ns: float
    tc_item_row_ns: float
    tc_step_ns: float
    stream_item_ns: float
    hbm_bytes_per_ns: float


def get_cost_model() -> CostModel:
    m = N.CostModel()
    N.check(N.lib().pat_get_cost_model(C.byref(m)), "pat_get_cost_model")
    return CostModel(*(getattr(m, f) for f, _ in N.CostModel._fields_))


def set_cost_model(model: CostModel) -> None:
    m = N.CostModel(**asdict(model))
    N.check(N.lib().pat_set_cost_model(C.byref(m)), "pat_set_cost_model")


def model_from_profile(profile: dict) -> CostModel:
    """Fit the model to a ``tools/calibrate.py`` profile: per-item cost of the
    4-row and 128-row tcgen05 items (intercept + per-row slope), per-tile cost,
    streaming per-item cost, and the bandwidth implied by the streaming kernel's
    per-tile cost (one 64-token d=128 tile per SM)."""
    f = profile["fits"]
    t4, t128 = f["tcgen05_rows4"], f["tcgen05_rows128"]
    row_ns = max(0.0, (t128["per_item_us"] - t4["per_item_us"]) * 1e3 * 128.0 / 124.0)
    item_ns = max(0.0, t4["per_item_us"] * 1e3 - row_ns * 4.0 / 128.0)
    step_ns = 1e3 * sum(f[k]["per_step_us"] for k in ("tcgen05_rows4", "tcgen05_rows32", "tcgen05_rows128")
                        if k in f) / sum(1 for k in ("tcgen05_rows4", "tcgen05_rows32", "tcgen05_rows128") if k in f)
    s4 = f["stream_rows4"]
    d = profile.get("heads", [32, 8, 128])[2]
    tile_bytes = 64.0 * d * 4
    bw = tile_bytes * profile["sms"] / (s4["per_step_us"] * 1e3)
    return CostModel(tc_item_ns=item_ns, tc_item_row_ns=row_ns, tc_step_ns=step_ns,
                     stream_item_ns=s4["per_item_us"] * 1e3, hbm_bytes_per_ns=bw)


def load_profile(path: str) -> CostModel:
    """Read a calibration profile and make it the process-wide cost model."""
    with open(path) as fh:
        model = model_from_profile(json.load(fh))
    set_cost_model(model)
    return model


__all__ = ["CostModel", "get_cost_model", "set_cost_model", "model_from_profile", "load_profile"]
