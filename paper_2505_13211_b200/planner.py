"""Planner host API over the C ABI: masks, scenarios, executor plans.

Mirrors the reference C ABI (/root/reference/proj/include/magiplan/magiplan.h)
one call per method; JSON formats are the reference's
(/root/reference/proj/docs/schema.md).
"""
from __future__ import annotations

import ctypes as C
import json
from typing import Any

from . import _lib


class Mask:
    """magiplan_mask handle: an AttnSlice composition."""

    def __init__(self, spec: dict | str):
        text = spec if isinstance(spec, str) else json.dumps(spec)
        h = C.c_void_p()
        _lib.check(_lib.lib().magiplan_mask_parse(text.encode(), C.byref(h)))
        self._h = h
        d = self.describe()
        self.seqlen_q, self.seqlen_k = d["seqlen_q"], d["seqlen_k"]
        self.slices = [(tuple(s["q"]), tuple(s["k"]), {"full": 0, "causal": 1, "inv_causal": 2,
                                                       "bi_causal": 3}[s["type"]]) for s in d["slices"]]

    def area(self, union: bool = False) -> int:
        out = C.c_int64()
        _lib.check(_lib.lib().magiplan_mask_area(self._h, _lib.COUNT_UNION if union else
                                                 _lib.COUNT_MULTIPLICITY, C.byref(out)))
        return out.value

    def is_allowed(self, q: int, k: int) -> bool:
        out = C.c_int()
        _lib.check(_lib.lib().magiplan_mask_is_allowed(self._h, q, k, C.byref(out)))
        return bool(out.value)

    def render(self) -> str:
        out = C.c_void_p()
        _lib.check(_lib.lib().magiplan_mask_render(self._h, C.byref(out)))
        return _lib.take_string(out)

    def describe(self) -> dict:
        out = C.c_void_p()
        _lib.check(_lib.lib().magiplan_mask_describe(self._h, C.byref(out)))
        return json.loads(_lib.take_string(out))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.lib().magiplan_mask_free(h)
            except Exception:  # noqa: BLE001
                pass


class Scenario:
    """magiplan_scenario handle: mask + workload + CP size + cost model."""

    def __init__(self, spec: dict | str, base_dir: str | None = None):
        text = spec if isinstance(spec, str) else json.dumps(spec)
        h = C.c_void_p()
        _lib.check(_lib.lib().magiplan_scenario_parse(
            text.encode(), base_dir.encode() if base_dir else None, C.byref(h)))
        self._h = h

    def set_seed(self, seed: int) -> None:
        _lib.check(_lib.lib().magiplan_scenario_set_seed(self._h, seed))

    def plan_text(self) -> str:
        out = C.c_void_p()
        _lib.check(_lib.lib().magiplan_scenario_plan(self._h, C.byref(out)))
        return _lib.take_string(out)

    def plan(self) -> dict:
        return json.loads(self.plan_text())

    def simulate_text(self, jobs: int = 1) -> str:
        out = C.c_void_p()
        _lib.check(_lib.lib().magiplan_scenario_simulate(self._h, jobs, C.byref(out)))
        return _lib.take_string(out)

    def exec_plan(self) -> dict:
        out = C.c_void_p()
        _lib.check(_lib.lib().magiplan_scenario_exec_plan(self._h, C.byref(out)))
        return json.loads(_lib.take_string(out))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.lib().magiplan_scenario_free(h)
            except Exception:  # noqa: BLE001
                pass


def debug_eval(op: str, **kwargs: Any):
    """Planner function access for parity tests (magiplan_debug_eval)."""
    out = C.c_void_p()
    req = json.dumps({"op": op, **kwargs})
    _lib.check(_lib.lib().magiplan_debug_eval(req.encode(), C.byref(out)))
    return json.loads(_lib.take_string(out))


def lognormal_lengths(count: int, median: float, sigma: float, max_length: int, seed: int) -> list[int]:
    return debug_eval("lognormal", count=count, median=median, sigma=sigma, max_length=max_length,
                      seed=seed)


def pack_run_text(config: dict | str, stream: str | None = None) -> str:
    """magiplan_pack_run: the online packing-and-padding report (reference
    proj/src/scenario.cpp:428-554). `stream` holds "id length" lines; None
    uses the config's log-normal generator."""
    text = config if isinstance(config, str) else json.dumps(config)
    out = C.c_void_p()
    _lib.check(_lib.lib().magiplan_pack_run(text.encode(), None if stream is None else stream.encode(),
                                            C.byref(out)))
    return _lib.take_string(out)


def pack_run(config: dict | str, stream: str | None = None) -> dict:
    return json.loads(pack_run_text(config, stream))


def pack_samples(lengths: list[int], max_length: int, bins: int, pool_capacity: int | None = None,
                 **packing: Any) -> list[list[int]]:
    """Pack a length list with the reference packer and return, per emitted
    bin, its sample lengths in bin order: the varlen document lists a packed
    FFA batch (config 4) is built from."""
    cfg = {"packing": {"max_length": max_length, "bins_per_iteration": bins,
                       "pool_capacity": pool_capacity or 4 * bins, **packing},
           "emit_bins": True}
    stream = "".join(f"{i} {n}\n" for i, n in enumerate(lengths))
    rep = pack_run(cfg, stream)
    return [[s["length"] for s in b["samples"]] for batch in rep["batches"] for b in batch["bins"]]


def packed_bin_masks(lengths: list[int], max_length: int, bins: int, pool_capacity: int | None = None,
                     causal_odd: bool = True, **packing: Any) -> list[dict]:
    """PnP packer -> FFA masks: every emitted bin becomes one
    max_length-token sequence whose documents are placed back to back, each
    attending only within itself (FULL, or CAUSAL for odd positions when
    ``causal_odd``, the config-4 convention); the unfilled tail is padding
    with no slice, so its rows give O = 0, LSE = -inf."""
    out = []
    for docs in pack_samples(lengths, max_length, bins, pool_capacity, **packing):
        sl, off = [], 0
        for i, n in enumerate(docs):
            sl.append({"q": [off, off + n], "k": [off, off + n],
                       "type": "causal" if causal_odd and i % 2 else "full"})
            off += n
        out.append({"seqlen_q": max_length, "seqlen_k": max_length, "slices": sl})
    return out
