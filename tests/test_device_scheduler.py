"""GPU parity: device scheduler kernels (K1-K5) vs the reference's golden outputs and the oracle.

Bit-exact: sample orders, partitions, evaluation counts, fp64 makespan / busy / span bits,
K1 6-tuples, and the error class the reference raises.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from golden_cases import arrays, cases, configs, golden, id_orders, product_graph, product_samples
from paper_2605_10501_b200 import errors as E
from paper_2605_10501_b200 import scheduling as S

pytestmark = pytest.mark.gpu

ALL = cases()
OK = [c for c in ALL if "error" not in c]
ERR = [c for c in ALL if "error" in c]
IDS = lambda cs: [c["name"] for c in cs]  # noqa: E731


@pytest.mark.parametrize("case", OK, ids=IDS(OK))
def test_build_schedule_matches_reference(case):
    g = product_graph(case["graph"])
    sched = S.build_schedule(g, configs(case), product_samples(case), case["policy"])
    assert dict(sched.per_rank_orders) == id_orders(case)


@pytest.mark.parametrize("case", OK, ids=IDS(OK))
def test_device_metrics_and_evals(case):
    """Critical-rank rank_metrics bits and EvalCounter totals from the plan kernels."""
    import torch

    g = product_graph(case["graph"])
    cf = configs(case)
    times, ids, masks, tab = arrays(case, g)
    B = times.shape[1]
    p = S.DevicePlanner(g, cf, case["policy"], max_batch=B)
    p.times[: 6 * B].copy_(torch.from_numpy(times.reshape(-1)))
    p.ids[:B].copy_(torch.from_numpy(ids))
    p.act[:B].copy_(torch.from_numpy(masks.view(np.int32)))
    p.plan_times(B)
    p.raise_errors(ids)
    m = p.metrics.view(-1, 3).cpu().numpy()
    for r, bits in case["rank_metrics"].items():
        assert [float.hex(float(x)) for x in m[int(r)]] == bits
    ev = p.evals.cpu().tolist()
    assert {str(r): v for r, v in enumerate(ev)} == case["evals"]


@pytest.mark.parametrize("case", ERR, ids=IDS(ERR))
def test_errors_match_reference(case):
    g = product_graph(case["graph"])
    with pytest.raises(getattr(E, case["error"])):
        S.build_schedule(g, configs(case), product_samples(case), case["policy"])


@pytest.mark.parametrize("case", [c for c in OK if c["name"].startswith(("example", "rand:g3"))][:12])
def test_partition_and_schedule_rank_api(case):
    g = product_graph(case["graph"])
    batch = product_samples(case)
    by_id = {s.sample_id: s for s in batch}
    crit = g.critical.id
    parts = S.partition_batch(batch, configs(case)[crit].dp, g)
    assert {str(r): [s.sample_id for s in v] for r, v in parts.items()} == case["partition"]
    for r, v in parts.items():
        c = S.EvalCounter()
        out = S.schedule_rank(v, case["policy"], c)
        assert tuple(s.sample_id for s in out) == id_orders(case)[(crit, r)]
        assert c.count == case["evals"][str(r)]
        mk = S.rank_metrics([by_id[i] for i in id_orders(case)[(crit, r)]], case["policy"])
        assert [float.hex(x) for x in (mk.makespan, mk.critical_busy, mk.critical_span)] == case["rank_metrics"][str(r)]


def test_known_answers():
    from paper_2605_10501_b200.workload import SampleTiming

    k = golden()["known"]
    assert float.hex(S.calculate_makespan([SampleTiming(0, 0, 1, 0, 0, 2, 0)])) == k["makespan_single_text"]
    assert float.hex(S.calculate_makespan([SampleTiming(0, 0.1, 1, 0, 0, 2, 0.2)])) == k["makespan_single_image"]
    assert S.merge_fanout([["a1", "a2"], ["b1", "b2"]], 2) == k["merge"]
    with pytest.raises(E.FanoutMismatch):
        S.merge_fanout([[1], [2]], 3)
    with pytest.raises(E.EmptyBatch):
        S.partition_batch([], 2)


def test_partition_without_graph():
    from paper_2605_10501_b200.workload import SampleTiming

    batch = [SampleTiming(i, 0.3 if i < 4 else 0.0, 1.0, 0, 0, 2.0, 0.3 if i < 4 else 0.0) for i in range(8)]
    parts = S.partition_batch(batch, 4)
    for r, v in parts.items():  # one image + one text per rank
        assert sorted(s.t_f_bc > 0 for s in v) == [False, True]


RECIPES = [c for c in OK if "tokens" in c]


@pytest.mark.parametrize("case", RECIPES, ids=IDS(RECIPES))
def test_k1_sample_times_bitexact(case):
    """Device 6-tuples from token counts == reference per_sample_times/derive_batch sums."""
    import torch

    from paper_2605_10501_b200 import recipes
    from paper_2605_10501_b200.costs import CostParams, cost_table

    g = product_graph(case["graph"])
    cf = configs(case)
    tab = g.tables
    B = len(case["samples"])
    params = {k: CostParams(float.fromhex(v[0]), float.fromhex(v[1]), float.fromhex(v[2]))
              for k, v in case["cost"].items()}
    tokens = np.zeros((len(tab.sub_names), B), dtype=np.int32)
    for name, tok in case["tokens"].items():
        tokens[tab.sub_names.index(name)] = tok
    p = S.DevicePlanner(g, cf, case["policy"], max_batch=B)
    p.ids[:B].copy_(torch.tensor([s["id"] for s in case["samples"]], dtype=torch.int32))
    p.plan_tokens(torch.from_numpy(cost_table(g, cf, params)).cuda(), torch.from_numpy(tokens).cuda(), B)
    p.raise_errors()
    got = p.times[: 6 * B].view(6, B).cpu().numpy()
    want = np.array([[float.fromhex(x) for x in s["t"]] for s in case["samples"]]).T
    assert [float.hex(float(x)) for x in got.reshape(-1)] == [float.hex(float(x)) for x in want.reshape(-1)]
    masks = p.act[:B].cpu().numpy().view(np.uint32)
    assert masks.tolist() == [tab.mask_of(s["act"]) for s in case["samples"]]
    per_rank = {(tab.section_ids[s], q): tuple(case["samples"][i]["id"] for i in o)
                for (s, q), o in p.host_orders().items()}
    assert per_rank == id_orders(case)


def _random_problem(rng, B, dp, fan, quant, with_dec=True, with_bac=True):
    from paper_2605_10501_b200.workload import Edge, ExecMode, Role, SectionSpec, StructuralParams, build_graph

    st = StructuralParams(64, 1, 1, 1, 64)
    g = build_graph([SectionSpec("enc", Role.AUXILIARY, ExecMode.FORWARD_BACKWARD, st),
                     SectionSpec("llm", Role.CRITICAL, ExecMode.FORWARD_BACKWARD, st),
                     SectionSpec("dec", Role.AUXILIARY, ExecMode.FORWARD_BACKWARD, st)],
                    [Edge("enc", "llm"), Edge("llm", "dec")])
    img = rng.random(B) < 0.5
    dec = (rng.random(B) < 0.3) & with_dec
    t = np.zeros((6, B))
    t[1] = rng.uniform(0.5, 3.0, B)
    t[4] = rng.uniform(0.0, 3.0, B)
    t[0] = np.where(img, rng.uniform(0.05, 2.0, B), 0.0)
    t[5] = np.where(img & with_bac, rng.uniform(0.0, 2.0, B), 0.0)
    t[2] = np.where(dec, rng.uniform(0.05, 1.0, B), 0.0)
    t[3] = np.where(dec, rng.uniform(0.0, 1.0, B), 0.0)
    if quant:
        t = np.round(t * 4) / 4
        t[1] = np.maximum(t[1], 0.25)
    from paper_2605_10501_b200.workload import SectionConfig

    cf = {"llm": SectionConfig(dp=dp), "enc": SectionConfig(dp=dp // fan, fanout=fan),
          "dec": SectionConfig(dp=dp)}
    return g, cf, np.ascontiguousarray(t), img, dec


@pytest.mark.parametrize("B,dp,with_bac,quant", [
    (1023, 1, True, True), (1023, 1, False, False), (2048, 4, True, False), (512, 2, False, True),
    (64, 1, False, True), (64, 1, True, False)])
def test_no_downstream_fast_path_vs_oracle(B, dp, with_bac, quant):
    """Interleaved ranks without a downstream stage run K3's branch-free recurrence (eval_nodown):
    orders, eval counts and metric bits == C oracle, with and without b_ac stages (the ub chain),
    continuous and quantised (tie-heavy) times, up to the per-rank maximum."""
    import torch

    rng = np.random.default_rng(B + dp + 7 * with_bac)
    g, cf, t, img, dec = _random_problem(rng, B, dp, 1, quant, with_dec=False, with_bac=with_bac)
    tab = g.tables
    masks = np.array([tab.mask_of(["enc"] if a else []) for a in img], dtype=np.uint32)
    p = S.DevicePlanner(g, cf, "interleaved", max_batch=B)
    p.times[: 6 * B].copy_(torch.from_numpy(t.reshape(-1)))
    p.ids[:B].copy_(torch.arange(B, dtype=torch.int32))
    p.act[:B].copy_(torch.from_numpy(masks.view(np.int32)))
    p.plan_times(B)
    p.raise_errors()
    up, down = oracle.resolve(masks, t, tab.sub_owner, tab.side, tab.up_candidates, tab.down_candidates)
    dps = [cf[s].dp for s in tab.section_ids]
    fans = [cf[s].fanout for s in tab.section_ids]
    want, ev = oracle.build_schedule(t, np.arange(B), up, down, len(dps), tab.critical, dps, fans, tab.neighbor,
                                     tab.merge_order, "interleaved")
    assert {k: v.tolist() for k, v in p.host_orders().items()} == want
    assert int(p.evals.sum().item()) == ev
    m = p.metrics.view(-1, 3).cpu().numpy()
    for r in range(dp):
        o = want[(tab.critical, r)]
        assert tuple(float.hex(float(x)) for x in m[r]) == tuple(float.hex(x) for x in
                                                                 oracle.rank_metrics(t, o, "interleaved"))


@pytest.mark.parametrize("B,dp,fan,policy,quant", [
    (4096, 8, 2, "interleaved", False),    # 512 samples per rank: max supported stress size
    (2046, 2, 2, "all-fwd-then-bwd", True),  # 1023 per rank: the per-rank maximum
    (1000, 1, 1, "interleaved", True),     # 1000 samples on one rank
    (777, 7, 7, "all-fwd-then-bwd", False),
])
def test_full_size_vs_oracle(B, dp, fan, policy, quant):
    """BASELINE-scale and stress sizes: device == C oracle bit-exactly."""
    import torch

    rng = np.random.default_rng(B + dp)
    g, cf, t, img, dec = _random_problem(rng, B, dp, fan, quant)
    tab = g.tables
    masks = np.array([tab.mask_of((["enc"] if a else []) + (["dec"] if b else [])) for a, b in zip(img, dec)],
                     dtype=np.uint32)
    p = S.DevicePlanner(g, cf, policy, max_batch=B)
    p.times[: 6 * B].copy_(torch.from_numpy(t.reshape(-1)))
    p.ids[:B].copy_(torch.arange(B, dtype=torch.int32))
    p.act[:B].copy_(torch.from_numpy(masks.view(np.int32)))
    p.plan_times(B)
    p.raise_errors()
    up, down = oracle.resolve(masks, t, tab.sub_owner, tab.side, tab.up_candidates, tab.down_candidates)
    dps = [cf[s].dp for s in tab.section_ids]
    fans = [cf[s].fanout for s in tab.section_ids]
    want, ev = oracle.build_schedule(t, np.arange(B), up, down, len(dps), tab.critical, dps, fans, tab.neighbor,
                                     tab.merge_order, policy)
    got = {k: v.tolist() for k, v in p.host_orders().items()}
    assert got == want
    assert int(p.evals.sum().item()) == ev
    m = p.metrics.view(-1, 3).cpu().numpy()
    for r in range(dp):
        o = want[(tab.critical, r)]
        assert tuple(float.hex(float(x)) for x in m[r]) == tuple(float.hex(x) for x in oracle.rank_metrics(t, o, policy))


def test_varlen_pack_and_pack_tokens():
    import torch

    from paper_2605_10501_b200 import _native as N

    rng = np.random.default_rng(0)
    for B, n, mbs in ((100, 37, 4), (3000, 2100, 3), (64, 64, 64)):
        lens = rng.integers(1, 500, B).astype(np.int32)
        order = rng.permutation(B)[:n].astype(np.int32)
        d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
        n_mb = -(-n // mbs)
        z = lambda k: torch.zeros(k, dtype=torch.int32, device="cuda")  # noqa: E731
        mb, off, tot, cu, start = z(n), z(n), z(n_mb), z(n_mb * (mbs + 1)), z(n_mb)
        dord, dlen = d(order), d(lens)
        N.check(N.lib().maestro_varlen_pack(N.ptr(dord), n, N.ptr(dlen), mbs, N.ptr(mb), N.ptr(off), N.ptr(tot),
                                            N.ptr(cu), N.ptr(start), N.stream_ptr()), "varlen")
        glob = np.concatenate([[0], np.cumsum(lens[order])[:-1]]).astype(np.int64)
        assert mb.cpu().numpy().tolist() == (np.arange(n) // mbs).tolist()
        assert off.cpu().numpy().tolist() == glob.tolist()
        cu_h = cu.cpu().numpy().reshape(n_mb, mbs + 1)
        for m in range(n_mb):
            ks = np.arange(m * mbs, min(n, (m + 1) * mbs))
            assert start[m].item() == glob[ks[0]]
            assert tot[m].item() == lens[order[ks]].sum()
            assert cu_h[m, : len(ks) + 1].tolist() == np.concatenate([[0], np.cumsum(lens[order[ks]])]).tolist()
        # pack token ids of the ordered samples
        L = int(lens.max())
        ids = rng.integers(0, 1 << 20, (B, L)).astype(np.int32)
        out = z(int(lens[order].sum()))
        N.check(N.lib().maestro_pack_tokens(N.ptr(d(ids)), L, N.ptr(dord), N.ptr(dlen), N.ptr(off), n, N.ptr(out),
                                            N.stream_ptr()), "pack")
        want = np.concatenate([ids[i, : lens[i]] for i in order])
        assert out.cpu().numpy().tolist() == want.tolist()


def test_scatter_rows_bitexact_and_bwd():
    import torch

    from paper_2605_10501_b200 import _native as N

    torch.manual_seed(0)
    d, n_src, n_dst = 768, 49 * 10, 4000
    src = torch.randn(n_src, d, device="cuda").to(torch.bfloat16)
    dst = torch.randn(n_dst, d, device="cuda").to(torch.bfloat16)
    dst_rows = torch.randperm(n_dst, device="cuda")[:n_src].to(torch.int32)
    src_rows = torch.arange(n_src, device="cuda", dtype=torch.int32)
    want = dst.clone()
    want[dst_rows.long()] = src[src_rows.long()]
    N.check(N.lib().maestro_scatter_rows_fwd(N.ptr(src), N.ptr(dst), N.ptr(src_rows), N.ptr(dst_rows), n_src, d,
                                             N.stream_ptr()), "scatter")
    assert torch.equal(dst, want)
    # backward: each src row gathers its (single) dst row -> exact copy; then a 2-to-1 segment map
    ddst = torch.randn(n_dst, d, device="cuda").to(torch.bfloat16)
    seg = torch.arange(n_src + 1, device="cuda", dtype=torch.int32)
    dsrc = torch.empty(n_src, d, device="cuda", dtype=torch.bfloat16)
    N.check(N.lib().maestro_gather_rows_bwd(N.ptr(ddst), N.ptr(dsrc), N.ptr(seg), N.ptr(dst_rows), n_src, d,
                                            N.stream_ptr()), "gather")
    assert torch.equal(dsrc, ddst[dst_rows.long()])
    seg2 = torch.arange(0, 2 * (n_src // 2) + 1, 2, device="cuda", dtype=torch.int32)
    dsrc2 = torch.empty(n_src // 2, d, device="cuda", dtype=torch.bfloat16)
    N.check(N.lib().maestro_gather_rows_bwd(N.ptr(ddst), N.ptr(dsrc2), N.ptr(seg2), N.ptr(dst_rows), n_src // 2, d,
                                            N.stream_ptr()), "gather2")
    ref = (ddst[dst_rows[0::2].long()].float() + ddst[dst_rows[1::2].long()].float()).to(torch.bfloat16)
    assert torch.equal(dsrc2, ref)
