"""Helpers turning the golden fixture (reference outputs) into arrays."""

from __future__ import annotations

import functools
import json
from pathlib import Path

import numpy as np

from paper_2605_10501_b200 import workload as W

GOLDEN = Path(__file__).resolve().parent / "golden" / "sched_golden.json"


@functools.lru_cache(maxsize=1)
def golden() -> dict:
    return json.loads(GOLDEN.read_text())


def cases(filter_fn=None):
    out = [c for c in golden()["cases"] if filter_fn is None or filter_fn(c)]
    return out


def product_graph(desc) -> W.SectionGraph:
    secs = [
        W.SectionSpec(s["id"], W.Role(s["role"]), W.ExecMode(s["exec_mode"]),
                      W.StructuralParams(*s["structural"]), tuple(s["submodules"]))
        for s in desc["sections"]
    ]
    return W.build_graph(secs, [W.Edge(a, b, float.fromhex(p)) for a, b, p in desc["edges"]])


def product_samples(case):
    return [
        W.SampleTiming(s["id"], *[float.fromhex(x) for x in s["t"]], activated_sections=frozenset(s["act"]))
        for s in case["samples"]
    ]


def configs(case):
    return {k: W.SectionConfig(*v) for k, v in case["configs"].items()}


def arrays(case, graph=None):
    """(times[6,B] f64, ids int32[B], act_mask uint32[B], tables)."""
    g = graph or product_graph(case["graph"])
    tab = g.tables
    t = np.array([[float.fromhex(x) for x in s["t"]] for s in case["samples"]], dtype=np.float64)
    times = np.ascontiguousarray(t.reshape(-1, 6).T) + 0.0
    ids = np.array([s["id"] for s in case["samples"]], dtype=np.int32)
    masks = np.array([tab.mask_of(s["act"]) for s in case["samples"]], dtype=np.uint32)
    return times, ids, masks, tab


def id_orders(case):
    """{(section, rank): tuple(ids)} from the fixture."""
    out = {}
    for key, ids in case["orders"].items():
        sec, r = key.rsplit("|", 1)
        out[(sec, int(r))] = tuple(ids)
    return out
