"""planner.py vs the reference planner's own outputs (tests/golden/planner_golden.json).

CPU: the configuration search -- enumerate_configs, fit_auxiliary, verify_plan and solve(...,
evaluate=False): chosen configs, GPU counts, iteration times, slack and memory bit-exact (float.hex),
and the reference's error classes.  GPU: the full solve(), whose predicted iteration time is the
simulated makespan of the device-built schedule, also bit-exact.  Plus the B200 calibration helpers.
"""

import json
from pathlib import Path

import pytest

from golden_cases import product_graph, product_samples
from paper_2605_10501_b200 import errors as E
from paper_2605_10501_b200 import planner as PL
from paper_2605_10501_b200.costs import BatchProfile, CostParams
from paper_2605_10501_b200.scheduling import ExecPolicy
from paper_2605_10501_b200.workload import ClusterSpec, SectionConfig

GOLD = json.loads((Path(__file__).parent / "golden" / "planner_golden.json").read_text())
F = float.fromhex


def params(desc):
    return {k: CostParams(flops_per_token_fwd=F(p["f"]), peak_flops_per_gpu=F(p["peak"]), bwd_fwd_ratio=F(p["ratio"]),
                          bytes_per_param_weights=F(p["wb"]), bytes_per_param_optimizer=F(p["ob"]),
                          activation_bytes_per_token=F(p["act"]), live_microbatch_cap=F(p["cap"]),
                          parallel_efficiency={tuple(k2): F(v) for k2, v in p["par"]},
                          mbs_efficiency={m: F(v) for m, v in p["mbs_eff"]}) for k, p in desc.items()}


def solve_inputs(c):
    g = product_graph(c["graph"])
    o = c["options"]
    opts = PL.PlanOptions(cp_cap=o["cp_cap"], mbs_candidates=tuple(o["mbs"]), critical_gpu_budget=o["budget"],
                          policy=ExecPolicy(o["policy"]), seed=o["seed"])
    pr = c["profile"]
    batch = None if c["batch"] is None else product_samples({"samples": c["batch"]})
    return (g, ClusterSpec(c["cluster"][0], F(c["cluster"][1])), params(c["params"]),
            BatchProfile(pr["B"], pr["shares"], pr["tokens"]), opts, c["pinned"] or None, batch)


SOLVE = [c for c in GOLD if c["kind"] == "solve"]


def _check_plan(plan, want, full):
    assert {k: list(v.as_tuple()) for k, v in plan.configs().items()} == want["configs"]
    assert plan.total_gpus_used == want["total_gpus"]
    assert {k: float.hex(sp.iteration_time) for k, sp in plan.per_section.items()} == want["iteration"]
    assert {k: float.hex(sp.slack) for k, sp in plan.per_section.items()} == want["slack"]
    assert {k: float.hex(sp.memory.total) for k, sp in plan.per_section.items()} == want["memory"]
    if full:
        assert float.hex(plan.predicted_iteration_time) == want["makespan"]


@pytest.mark.parametrize("case", SOLVE, ids=[c["name"] for c in SOLVE])
def test_configuration_search_matches_reference(case):
    g, cl, par, prof, opts, pinned, batch = solve_inputs(case)
    if "error" in case:
        with pytest.raises(getattr(E, case["error"])):
            PL.solve(g, cl, par, prof, opts, pinned=pinned, explicit_batch=batch, evaluate=False)
        return
    _check_plan(PL.solve(g, cl, par, prof, opts, pinned=pinned, explicit_batch=batch, evaluate=False),
                case["plan"], full=False)


@pytest.mark.gpu
@pytest.mark.parametrize("case", [c for c in SOLVE if "error" not in c], ids=lambda c: c["name"])
def test_solve_matches_reference_makespan(case):
    g, cl, par, prof, opts, pinned, batch = solve_inputs(case)
    _check_plan(PL.solve(g, cl, par, prof, opts, pinned=pinned, explicit_batch=batch), case["plan"], full=True)


@pytest.mark.parametrize("case", [c for c in GOLD if c["kind"] == "enum"], ids=lambda c: c["name"])
def test_enumerate_configs_matches_reference(case):
    g = product_graph(case["graph"])
    sec = g.section(case["section"])
    (p,) = params(case["params"]).values()
    cands = PL.enumerate_configs(sec, ClusterSpec(case["cluster"][0], F(case["cluster"][1])), p, 2048)
    assert len(cands) == case["n"]
    assert [[list(c.config.as_tuple()), float.hex(c.step_time_per_sample), float.hex(c.memory.total)]
            for c in cands[:12]] == case["head"]


@pytest.mark.parametrize("case", [c for c in GOLD if c["kind"] == "fit"], ids=lambda c: c["name"])
def test_fit_auxiliary_matches_reference(case):
    g = product_graph(case["graph"])
    (p,) = params(case["params"]).values()
    if "error" in case:
        with pytest.raises(getattr(E, case["error"])):
            PL.fit_auxiliary(g.section("enc"), F(case["crit_time"]), 0.4, 6, p, 6, 80e9, 128, 512)
        return
    cfg, gpus = PL.fit_auxiliary(g.section("enc"), F(case["crit_time"]), 0.4, 6, p, 6, 80e9, 128, 512)
    assert list(cfg.as_tuple()) == case["config"] and gpus == case["gpus"]


def test_verify_plan_diagnostics_match_reference():
    (case,) = [c for c in GOLD if c["kind"] == "verify"]
    g = product_graph(case["graph"])
    cfgs = {k: SectionConfig(*v) for k, v in case["configs"].items()}
    got = PL.verify_plan(g, ClusterSpec(8, 80e9), params(case["params"]), cfgs, {"enc": 512, "llm": 2048, "dec": 64},
                         raise_on_violation=False)
    assert got == case["diagnostics"]
    with pytest.raises(E.FanoutViolation):
        PL.verify_plan(g, ClusterSpec(8, 80e9), params(case["params"]), cfgs, {"enc": 512, "llm": 2048, "dec": 64})


def test_b200_calibrated_plans():
    """Plans with B200-measured throughput: the tiny VLM fits 8 GPUs with a ViT that keeps pace;
    the KD graph cannot be placed on disjoint groups without stalling the student (the teacher's
    forward is ~2.4x the student's training FLOPs per sample while DP^teacher <= DP^student under the
    fan-out rule) -- which is why the executor's default layout co-locates the two sections."""
    from paper_2605_10501_b200 import recipes as R

    vlm = R.vlm_tiny(8, 64)
    par = {k: PL.b200_cost_params(p.flops_per_token_fwd, p.bwd_fwd_ratio, activation_bytes_per_token=2e5)
           for k, p in vlm.params.items()}
    plan = PL.solve(vlm.graph, PL.b200_cluster(8), par, BatchProfile(64, {"vit": 0.5}), evaluate=False)
    assert plan.total_gpus_used <= 8 and all(sp.slack >= 0 for sp in plan.per_section.values())
    assert all(sp.memory.total <= PL.B200_CLUSTER_MEM for sp in plan.per_section.values())
    kd = R.kd(8, 512, R.KD_SEQ, "disjoint")
    par = {k: PL.b200_cost_params(p.flops_per_token_fwd, p.bwd_fwd_ratio, activation_bytes_per_token=2e5)
           for k, p in kd.params.items()}
    with pytest.raises(E.CannotAvoidStall):
        PL.solve(kd.graph, PL.b200_cluster(8), par, BatchProfile(512, {"teacher": 1.0}), evaluate=False)


def test_fit_cost_params_recovers_the_cost_model():
    """Stage times generated by estimate_step_time (costs.py:105-123) with known knobs -> the fit
    returns those knobs; the fitted params then predict the stages exactly."""
    from paper_2605_10501_b200 import recipes as R
    from paper_2605_10501_b200.costs import CostParams, estimate_step_time
    from paper_2605_10501_b200.planner import StageSample, fit_cost_params
    from paper_2605_10501_b200.workload import SectionConfig

    g = R.kd_graph()
    true = {"student": CostParams(flops_per_token_fwd=3e9, peak_flops_per_gpu=9.1e14, bwd_fwd_ratio=2.3,
                                  mbs_efficiency={4: 0.8}),
            "teacher": CostParams(flops_per_token_fwd=5e9, peak_flops_per_gpu=1.2e15)}
    samples = []
    for sec in ("student", "teacher"):
        for mbs in (4, 8):
            for tok in (1024, 2048):
                f, b = estimate_step_time(g.section(sec), SectionConfig(mbs=mbs), true[sec], tok)
                samples.append(StageSample(sec, "fwd", mbs, tok, f))
                if b:
                    samples.append(StageSample(sec, "bwd", mbs, tok, b))
    fit = fit_cost_params(samples, {s: true[s].flops_per_token_fwd for s in true})
    assert abs(fit["student"].peak_flops_per_gpu / 9.1e14 - 1) < 1e-12
    assert abs(fit["student"].bwd_fwd_ratio - 2.3) < 1e-12
    assert abs(fit["student"].mbs_efficiency[4] - 0.8) < 1e-12
    assert abs(fit["teacher"].peak_flops_per_gpu / 1.2e15 - 1) < 1e-12
    for x in samples:
        f, b = estimate_step_time(g.section(x.section), SectionConfig(mbs=x.mbs), fit[x.section], x.tokens)
        assert abs((f if x.phase == "fwd" else b) / x.seconds - 1) < 1e-9
