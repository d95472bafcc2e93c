"""Pin the oracle (and the host graph API) against the reference's own outputs.

The golden fixture was produced by running the reference implementation
(tests/golden/make_golden.py).  Everything here runs on CPU.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from golden_cases import arrays, cases, configs, golden, id_orders, product_graph, product_samples
from paper_2605_10501_b200 import errors as E
from paper_2605_10501_b200.workload import SIDE_CODE, Side

ALL = cases()
OK = [c for c in ALL if "error" not in c]
IDS = lambda cs: [c["name"] for c in cs]  # noqa: E731


def _resolved_indices(case, tab):
    """Reference resolved activations as section-index arrays."""
    idx = {sid: i for i, sid in enumerate(tab.section_ids)}
    up = np.array([-1 if r[0] is None else idx[r[0]] for r in case["resolved"]], dtype=np.int32)
    down = np.array([-1 if r[1] is None else idx[r[1]] for r in case["resolved"]], dtype=np.int32)
    return up, down


@pytest.mark.parametrize("case", ALL, ids=IDS(ALL))
def test_graph_tables_match_reference(case):
    g = product_graph(case["graph"])
    facts = case["facts"]
    assert {s.id: g.side(s.id).value for s in g.sections} == facts["sides"]
    assert {a.id: g.neighbor_toward_critical(a.id) for a in g.auxiliaries} == facts["neighbor"]
    assert [g.tables.section_ids[i] for i in g.tables.merge_order] == facts["merge_order"]
    assert list(g.topological_order()) == facts["topological_order"]


@pytest.mark.parametrize("case", ALL, ids=IDS(ALL))
def test_resolve_host_and_oracle(case):
    g = product_graph(case["graph"])
    times, ids, masks, tab = arrays(case, g)
    for s, ref in zip(product_samples(case), case["resolved"]):
        if isinstance(ref, dict):
            with pytest.raises(getattr(E, ref["error"])):
                g.resolve_activation(s)
        else:
            assert list(g.resolve_activation(s)) == ref
    first_err = next((r["error"] for r in case["resolved"] if isinstance(r, dict)), None)
    try:
        up, down = oracle.resolve(masks, times, tab.sub_owner, tab.side, tab.up_candidates, tab.down_candidates)
    except ValueError as exc:
        code, i = exc.args[0]
        assert E.DEVICE_CODES[code].__name__ == case["resolved"][i]["error"]
        return
    assert first_err is None
    ref_up, ref_down = _resolved_indices(case, tab)
    np.testing.assert_array_equal(up, ref_up)
    np.testing.assert_array_equal(down, ref_down)


@pytest.mark.parametrize("case", [c for c in ALL if "partition" in c], ids=IDS([c for c in ALL if "partition" in c]))
def test_oracle_partition_and_evals(case):
    g = product_graph(case["graph"])
    times, ids, masks, tab = arrays(case, g)
    up, down = _resolved_indices(case, tab)
    dp = configs(case)[g.critical.id].dp
    lists, _ = oracle.partition(times, ids, up, down, dp, len(tab.section_ids))
    got = {str(r): [int(ids[i]) for i in lst] for r, lst in enumerate(lists)}
    assert got == case["partition"]
    for r, lst in enumerate(lists):
        _, ev = oracle.schedule_rank(times, lst, case["policy"])
        assert ev == case["evals"][str(r)]


def oracle_schedule(case):
    g = product_graph(case["graph"])
    times, ids, masks, tab = arrays(case, g)
    up, down = _resolved_indices(case, tab)
    cf = configs(case)
    n = len(tab.section_ids)
    dp = [cf[s].dp for s in tab.section_ids]
    fan = [cf[s].fanout for s in tab.section_ids]
    out, ev = oracle.build_schedule(times, ids, up, down, n, tab.critical, dp, fan, tab.neighbor,
                                    tab.merge_order, case["policy"])
    return {(tab.section_ids[s], q): tuple(int(ids[i]) for i in o) for (s, q), o in out.items()}, times, ids


@pytest.mark.parametrize("case", OK, ids=IDS(OK))
def test_oracle_build_schedule_bitexact(case):
    got, times, ids = oracle_schedule(case)
    assert got == id_orders(case)
    crit = product_graph(case["graph"]).critical.id
    pos = {int(v): i for i, v in enumerate(ids)}
    for r, (mk, busy, span) in case["rank_metrics"].items():
        order = [pos[i] for i in got[(crit, int(r))]]
        m = oracle.rank_metrics(times, order, case["policy"])
        assert [float.hex(x) for x in m] == [mk, busy, span]


def test_oracle_fanout_violation():
    (case,) = [c for c in ALL if c["name"] == "err:fanout"]
    with pytest.raises(ValueError) as exc:
        oracle_schedule(case)
    assert exc.value.args[0][0] == 8


def test_known_answers():
    k = golden()["known"]
    fig8 = oracle.times_array([(0.1, 1, 0, 0, 2, 0.2), (0, 1, 0, 0, 2, 0), (0, 1, 0, 0, 2, 0), (0.2, 1, 0, 0, 2, 0.4)])
    # sort_initial is the seed order of schedule_rank; ids are 1..4
    order = sorted(range(4), key=lambda i: fig8[0, i])
    assert [i + 1 for i in order] == k["sort_initial"]
    one = oracle.times_array([(0, 1, 0, 0, 2, 0)])
    assert float.hex(oracle.rank_metrics(one, [0])[0]) == k["makespan_single_text"]
    img = oracle.times_array([(0.1, 1, 0, 0, 2, 0.2)])
    assert float.hex(oracle.rank_metrics(img, [0])[0]) == k["makespan_single_image"] == float.hex(3.3000000000000003)
    assert oracle.merge_fanout([["a1", "a2"], ["b1", "b2"]], 2) == k["merge"]
    assert oracle.merge_fanout([[1, 2, 3], [4], [], [5, 6]], 4) == k["merge_ragged"]


def test_eval_count_bound():
    for n, rec in golden()["evals"].items():
        n = int(n)
        assert rec["count"] == (n * (n + 1) // 2 if n > 1 else 0)
        if rec["samples"] is not None:
            t = oracle.times_array([[float.fromhex(x) for x in s["t"]] for s in rec["samples"]])
            order, ev = oracle.schedule_rank(t, list(range(n)))
            assert ev == rec["count"]
            assert [rec["samples"][i]["id"] for i in order] == rec["order"]
