"""Executor model (simulator.py) vs the reference's simulate outputs, bit for bit (CPU)."""

import json

import pytest

from golden_cases import cases, configs, id_orders, product_graph, product_samples
from paper_2605_10501_b200 import errors as E
from paper_2605_10501_b200.scheduling import ExecPolicy, Schedule
from paper_2605_10501_b200.simulator import build_trace, export_trace, simulate

SIM = [c for c in cases() if "simulate" in c]


@pytest.mark.parametrize("case", SIM, ids=[c["name"] for c in SIM])
def test_simulate_matches_reference(case):
    g = product_graph(case["graph"])
    sched = Schedule(per_rank_orders=id_orders(case), batch=tuple(product_samples(case)),
                     policy=ExecPolicy(case["policy"]))
    ref = case["simulate"]
    if "error" in ref:
        with pytest.raises(getattr(E, ref["error"])):
            simulate(g, configs(case), sched)
        return
    rep, events = simulate(g, configs(case), sched)
    assert float.hex(rep.makespan) == ref["makespan"]
    assert float.hex(rep.critical_idle) == ref["critical_idle"]
    assert {str(k): float.hex(v) for k, v in rep.critical_idle_per_rank.items()} == ref["critical_idle_per_rank"]
    assert {k: float.hex(v) for k, v in rep.per_section_busy_time.items()} == ref["busy"]
    queues = {}
    for e in sorted(events, key=lambda e: (e.section, e.dp_rank, e.start, e.sample_id)):
        queues.setdefault(f"{e.section}|{e.dp_rank}", []).append([e.sample_id, e.phase, float.hex(e.start),
                                                                  float.hex(e.end)])
    assert queues == ref["queues"]


def test_fig8_zero_stall_and_trace(tmp_path):
    (case,) = [c for c in SIM if c["name"] == "example:vlm_fig8:interleaved"]
    g = product_graph(case["graph"])
    sched = Schedule(per_rank_orders=id_orders(case), batch=tuple(product_samples(case)))
    rep, events = simulate(g, configs(case), sched)
    assert rep.critical_idle == 0.0 and rep.makespan == 9.0
    tr = build_trace(events)
    assert {e["pid"] for e in tr["traceEvents"] if e["ph"] == "M"} == {0, 1}
    p1, p2 = tmp_path / "a.json", tmp_path / "b.json"
    export_trace(events, str(p1))
    export_trace(events, str(p2))
    assert p1.read_bytes() == p2.read_bytes()  # byte-stable
    assert json.loads(p1.read_text())["displayTimeUnit"] == "ms"


def test_comm_latency_monotone():
    (case,) = [c for c in SIM if c["name"] == "example:vlm_fig8:interleaved"]
    g = product_graph(case["graph"])
    sched = Schedule(per_rank_orders=id_orders(case), batch=tuple(product_samples(case)))
    base, _ = simulate(g, configs(case), sched)
    slow, _ = simulate(g, configs(case), sched, comm_model=lambda b: b / 1e9)
    assert slow.makespan >= base.makespan and len(slow.comm_events) > 0
