"""Golden plans by running the REFERENCE planner (planner.py); build container only.

    python tests/golden/make_planner_golden.py   -> tests/golden/planner_golden.json

Cases: the three shipped example specs through solve() (as pipeline.run_optimize calls it), and
synthetic graphs through solve(), enumerate_configs(), fit_auxiliary() and verify_plan(), with the
reference's outputs (configs, GPU counts, iteration times / makespans as float.hex, candidate
lists, diagnostics) or the error class it raised.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
import make_golden as mg  # noqa: E402

from maestro import costs as rc  # noqa: E402
from maestro import planner as rp  # noqa: E402
from maestro import workload as rw  # noqa: E402
from maestro.examples import spec_path  # noqa: E402
from maestro.specfile import load_spec  # noqa: E402

H = float.hex


def params_desc(params):
    return {k: {"f": H(p.flops_per_token_fwd), "peak": H(p.peak_flops_per_gpu), "ratio": H(p.bwd_fwd_ratio),
                "wb": H(p.bytes_per_param_weights), "ob": H(p.bytes_per_param_optimizer),
                "act": H(p.activation_bytes_per_token), "cap": H(p.live_microbatch_cap),
                "par": [[list(k2), H(v)] for k2, v in p.parallel_efficiency.items()],
                "mbs_eff": [[m, H(v)] for m, v in p.mbs_efficiency.items()]} for k, p in params.items()}


def plan_desc(plan):
    return {"configs": {k: list(v.as_tuple()) for k, v in plan.configs().items()},
            "total_gpus": plan.total_gpus_used, "makespan": H(plan.predicted_iteration_time),
            "iteration": {k: H(sp.iteration_time) for k, sp in plan.per_section.items()},
            "slack": {k: H(sp.slack) for k, sp in plan.per_section.items()},
            "memory": {k: H(sp.memory.total) for k, sp in plan.per_section.items()}}


def solve_case(name, graph, cluster, params, profile, options=rp.PlanOptions(), pinned=None, batch=None):
    out = {"name": name, "kind": "solve", "graph": mg.graph_desc(graph),
           "cluster": [cluster.total_gpus, H(cluster.mem_per_gpu)], "params": params_desc(params),
           "profile": {"B": profile.global_batch_size, "shares": dict(profile.shares), "tokens": dict(profile.tokens)},
           "options": {"cp_cap": options.cp_cap, "mbs": list(options.mbs_candidates),
                       "budget": options.critical_gpu_budget, "policy": options.policy.value, "seed": options.seed},
           "pinned": {k: dict(v) for k, v in (pinned or {}).items()},
           "batch": None if batch is None else [mg.sample_desc(s) for s in batch]}
    try:
        out["plan"] = plan_desc(rp.solve(graph, cluster, params, profile, options, pinned=pinned,
                                         explicit_batch=batch))
    except Exception as e:  # noqa: BLE001
        out["error"] = type(e).__name__
    return out


def P(f, peak=3e14, ratio=2.0, act=2e5, **kw):
    return rc.CostParams(flops_per_token_fwd=f, peak_flops_per_gpu=peak, bwd_fwd_ratio=ratio,
                         activation_bytes_per_token=act, **kw)


def main():
    cases = []
    for ex in ("vlm_fig8", "distill_toy", "omni_toy"):
        spec = load_spec(spec_path(ex))
        cases.append(solve_case(f"example:{ex}", spec.graph, spec.cluster, spec.params_by_section,
                                spec.effective_profile(), pinned=spec.pinned, batch=spec.batch))
    g2, g3, g4, g5 = mg.g2(), mg.g3(), mg.g4(), mg.g5()
    for n, mem in ((8, 80e9), (16, 80e9), (4, 40e9), (32, 180e9)):
        cases.append(solve_case(f"g2:{n}x{mem:.0e}", g2, rw.ClusterSpec(n, mem),
                                {"enc": P(1.1e7), "llm": P(7.9e7)},
                                rc.BatchProfile(64, {"enc": 0.5}, {"llm": 1024, "enc": 512})))
        cases.append(solve_case(f"g3:{n}x{mem:.0e}", g3, rw.ClusterSpec(n, mem),
                                {"enc": P(2e7), "llm": P(1.4e9, ratio=2.5), "dec": P(5e6)},
                                rc.BatchProfile(128, {"enc": 0.3, "dec": 0.7}, {"llm": 2048})))
        cases.append(solve_case(f"g4:{n}x{mem:.0e}", g4, rw.ClusterSpec(n, mem),
                                {"image_enc": P(2e7), "audio_enc": P(1.5e7), "llm": P(1.4e10, peak=1.6e15)},
                                rc.BatchProfile(96, {"image_enc": 0.25, "audio_enc": 0.5})))
        cases.append(solve_case(f"g5:{n}x{mem:.0e}", g5, rw.ClusterSpec(n, mem),
                                {k: P(1e7 * (i + 1)) for i, k in enumerate(("pre", "enc", "llm", "dec"))},
                                rc.BatchProfile(33, {"pre": 1.0, "enc": 0.5, "dec": 0.25})))
    # budgets, pins, efficiencies, tiny memory (NoFeasibleConfig), slow aux (CannotAvoidStall)
    cases.append(solve_case("g2:budget", g2, rw.ClusterSpec(16, 80e9), {"enc": P(1.1e7), "llm": P(7.9e7)},
                            rc.BatchProfile(64, {"enc": 0.5}), rp.PlanOptions(critical_gpu_budget=6)))
    cases.append(solve_case("g2:pinned", g2, rw.ClusterSpec(16, 80e9), {"enc": P(1.1e7), "llm": P(7.9e7)},
                            rc.BatchProfile(64, {"enc": 0.5}), pinned={"llm": {"tp": 2}, "enc": {"mbs": 4}}))
    cases.append(solve_case("g2:eff", g2, rw.ClusterSpec(8, 80e9),
                            {"enc": P(1.1e7, mbs_efficiency={1: 0.5, 2: 0.7, 4: 0.9}),
                             "llm": P(7.9e7, parallel_efficiency={(2, 1, 1): 0.8, (1, 2, 1): 0.9})},
                            rc.BatchProfile(64, {"enc": 0.5})))
    cases.append(solve_case("g2:nomem", g2, rw.ClusterSpec(8, 1e6), {"enc": P(1.1e7), "llm": P(7.9e7)},
                            rc.BatchProfile(64, {"enc": 0.5})))
    cases.append(solve_case("g2:stall", g2, rw.ClusterSpec(2, 80e9), {"enc": P(5e10), "llm": P(1e6)},
                            rc.BatchProfile(64, {"enc": 1.0})))
    cases.append(solve_case("g3:alltoall", g3, rw.ClusterSpec(8, 80e9),
                            {"enc": P(2e7), "llm": P(1.4e9), "dec": P(5e6)}, rc.BatchProfile(16, {"enc": 1.0}),
                            rp.PlanOptions(mbs_candidates=(1, 2), cp_cap=4, policy=rw_policy_all())))
    # stage-level: enumerate_configs, fit_auxiliary, verify_plan
    secs = {s.id: s for s in g3.sections}
    for sid, f, n, mem in (("llm", 1.4e9, 8, 80e9), ("enc", 2e7, 4, 20e9), ("dec", 5e6, 16, 80e9)):
        rec = {"name": f"enum:{sid}:{n}", "kind": "enum", "graph": mg.graph_desc(g3), "section": sid,
               "cluster": [n, H(mem)], "params": params_desc({sid: P(f)})}
        try:
            cands = rp.enumerate_configs(secs[sid], rw.ClusterSpec(n, mem), P(f), 2048)
            rec["n"] = len(cands)
            rec["head"] = [[list(c.config.as_tuple()), H(c.step_time_per_sample), H(c.memory.total)] for c in cands[:12]]
        except Exception as e:  # noqa: BLE001
            rec["error"] = type(e).__name__
        cases.append(rec)
    for crit_t in (1e-3, 1e-1, 10.0):
        rec = {"name": f"fit:enc:{crit_t}", "kind": "fit", "graph": mg.graph_desc(g3), "crit_time": H(crit_t),
               "params": params_desc({"enc": P(2e7)})}
        try:
            cfg, gpus = rp.fit_auxiliary(secs["enc"], crit_t, 0.4, 6, P(2e7), 6, 80e9, 128, 512)
            rec["config"], rec["gpus"] = list(cfg.as_tuple()), gpus
        except Exception as e:  # noqa: BLE001
            rec["error"] = type(e).__name__
        cases.append(rec)
    bad = {"llm": rw.SectionConfig(dp=4, tp=3), "enc": rw.SectionConfig(dp=3, fanout=2),
           "dec": rw.SectionConfig(dp=2, fanout=1)}
    par = {"enc": P(2e7), "llm": P(1.4e9), "dec": P(5e6)}
    diags = rp.verify_plan(g3, rw.ClusterSpec(8, 80e9), par, bad, {"enc": 512, "llm": 2048, "dec": 64},
                           raise_on_violation=False)
    cases.append({"name": "verify:bad", "kind": "verify", "graph": mg.graph_desc(g3), "params": params_desc(par),
                  "configs": {k: list(v.as_tuple()) for k, v in bad.items()}, "diagnostics": diags})
    path = Path(__file__).with_name("planner_golden.json")
    path.write_text(json.dumps(cases, separators=(",", ":"), sort_keys=True))
    print(f"wrote {len(cases)} cases to {path}")


def rw_policy_all():
    from maestro.scheduling import ExecPolicy

    return ExecPolicy.ALL_FWD_THEN_BWD


if __name__ == "__main__":
    main()
