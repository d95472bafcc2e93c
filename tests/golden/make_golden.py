"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    python tests/golden/make_golden.py

Writes tests/golden/sched_golden.json.  Floats are stored as ``float.hex``
so fixtures pin the reference's fp64 bits.  Each case stores the inputs
(graph description, configs, 6-tuples, activations), the reference's
outputs (partition, per-rank orders, rank metrics, evaluation counts,
resolved activations, simulate's per-resource stage order and stall
metrics) or the error class the reference raised.
"""

from __future__ import annotations

import json
import math
import random
import sys
import time
from pathlib import Path

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from maestro import costs as rcosts  # noqa: E402
from maestro import errors as rerr  # noqa: E402
from maestro import scheduling as rs  # noqa: E402
from maestro import simulator as rsim  # noqa: E402
from maestro import workload as rw  # noqa: E402
from maestro.examples import spec_path  # noqa: E402
from maestro.pipeline import RunOptions, batch_for, run_optimize  # noqa: E402
from maestro.specfile import load_spec  # noqa: E402

from paper_2605_10501_b200 import recipes  # noqa: E402  (synthetic inputs only)

H = float.hex


def graph_desc(g) -> dict:
    return {
        "sections": [
            {
                "id": s.id,
                "role": s.role.value,
                "exec_mode": s.exec_mode.value,
                "submodules": list(s.submodules),
                "structural": [s.structural.hidden_dim, s.structural.num_heads, s.structural.num_layers,
                               s.structural.vocab_size, s.structural.max_seq_len, s.structural.param_count],
            }
            for s in g.sections
        ],
        "edges": [[e.src, e.dst, H(float(e.payload_bytes_per_sample))] for e in g.edges],
    }


def ref_graph(desc: dict):
    secs = [
        rw.SectionSpec(s["id"], rw.Role(s["role"]), rw.ExecMode(s["exec_mode"]),
                       rw.StructuralParams(*s["structural"]), tuple(s["submodules"]))
        for s in desc["sections"]
    ]
    edges = [rw.Edge(a, b, float.fromhex(p)) for a, b, p in desc["edges"]]
    return rw.build_graph(secs, edges)


def graph_facts(g) -> dict:
    sides = {s.id: g.side(s.id).value for s in g.sections}
    nb = {s.id: g.neighbor_toward_critical(s.id) for s in g.auxiliaries}
    order = []
    for aux in g.auxiliaries:
        hops, node = 0, aux.id
        while g.side(node) is not rw.Side.CRITICAL:
            node = g.neighbor_toward_critical(node)
            hops += 1
        order.append((hops, aux.id))
    return {"sides": sides, "neighbor": nb, "merge_order": [sid for _, sid in sorted(order)],
            "topological_order": list(g.topological_order())}


def sample_desc(s) -> dict:
    return {"id": s.sample_id, "t": [H(float(x)) for x in s.as_tuple()], "act": sorted(s.activated_sections)}


def run_case(name, g, configs, batch, policy, with_sim=True, extra=None) -> dict:
    case = {
        "name": name,
        "graph": graph_desc(g),
        "facts": graph_facts(g),
        "configs": {k: list(v.as_tuple()) for k, v in configs.items()},
        "policy": policy.value,
        "samples": [sample_desc(s) for s in batch],
    }
    if extra:
        case.update(extra)
    resolved = []
    for s in batch:
        try:
            resolved.append(list(g.resolve_activation(s)))
        except rerr.MaestroError as e:
            resolved.append({"error": type(e).__name__})
    case["resolved"] = resolved
    try:
        crit = g.critical.id
        parts = rs.partition_batch(batch, configs[crit].dp, g)
        case["partition"] = {str(r): [s.sample_id for s in v] for r, v in parts.items()}
        evals = {}
        for r, v in parts.items():
            c = rs.EvalCounter()
            rs.schedule_rank(v, policy, c)
            evals[str(r)] = c.count
        case["evals"] = evals
        sched = rs.build_schedule(g, configs, batch, policy)
    except rerr.MaestroError as e:
        case["error"] = type(e).__name__
        return case
    case["orders"] = {f"{sec}|{r}": list(o) for (sec, r), o in sorted(sched.per_rank_orders.items())}
    by_id = {s.sample_id: s for s in batch}
    metrics = {}
    for r in sched.ranks_of(crit):
        m = rs.rank_metrics([by_id[i] for i in sched.order_for(crit, r)], policy)
        metrics[str(r)] = [H(m.makespan), H(m.critical_busy), H(m.critical_span)]
    case["rank_metrics"] = metrics
    if with_sim:
        try:
            rep, events = rsim.simulate(g, configs, sched)
            queues: dict[str, list] = {}
            for e in sorted(events, key=lambda e: (e.section, e.dp_rank, e.start, e.sample_id)):
                queues.setdefault(f"{e.section}|{e.dp_rank}", []).append([e.sample_id, e.phase, H(e.start), H(e.end)])
            case["simulate"] = {
                "makespan": H(rep.makespan),
                "critical_idle": H(rep.critical_idle),
                "critical_idle_per_rank": {str(k): H(v) for k, v in rep.critical_idle_per_rank.items()},
                "busy": {k: H(v) for k, v in rep.per_section_busy_time.items()},
                "queues": queues,
            }
        except rerr.MaestroError as e:
            case["simulate"] = {"error": type(e).__name__}
    return case


# ----------------------------------------------------------------------------- graphs
def sec(id_, role="auxiliary", mode="forward_backward", subs=(), heads=16, layers=16, seq=4096):
    return rw.SectionSpec(id_, rw.Role(role), rw.ExecMode(mode),
                          rw.StructuralParams(1024, heads, layers, 1000, seq, 1000), tuple(subs))


def g2():
    return rw.build_graph([sec("enc"), sec("llm", "critical")], [rw.Edge("enc", "llm", 100.0)])


def g3():
    return rw.build_graph([sec("enc"), sec("llm", "critical"), sec("dec")],
                          [rw.Edge("enc", "llm", 100.0), rw.Edge("llm", "dec", 50.0)])


def g4():
    return rw.build_graph([sec("image_enc"), sec("audio_enc"), sec("llm", "critical")],
                          [rw.Edge("image_enc", "llm", 4.0), rw.Edge("audio_enc", "llm", 2.0)])


def g5():
    # two-hop upstream chain (pre -> enc -> llm) plus a downstream decoder
    return rw.build_graph([sec("pre"), sec("enc"), sec("llm", "critical"), sec("dec")],
                          [rw.Edge("pre", "enc", 1.0), rw.Edge("enc", "llm", 1.0), rw.Edge("llm", "dec", 1.0)])


def rand_time(rng, lo=0.0, hi=3.0):
    return rng.uniform(lo, hi)


def random_batch(rng, g, n, p_up=0.4, p_down=0.3, quantized=False, ids=None):
    ups = [s.id for s in g.auxiliaries if g.side(s.id) is rw.Side.UPSTREAM]
    downs = [s.id for s in g.auxiliaries if g.side(s.id) is rw.Side.DOWNSTREAM]
    names_up = []
    for u in ups:
        subs = g.section(u).submodules
        names_up.extend(subs if len(subs) > 1 else [u])
    out = []
    q = (lambda x: round(x * 10) / 10) if quantized else (lambda x: x)
    for i in range(n):
        t = [0.0] * 6
        act = set()
        t[1] = q(rng.uniform(0.5, 3.0)) or 0.5
        t[4] = q(rng.uniform(0.0, 3.0)) if rng.random() < 0.9 else 0.0
        if names_up and rng.random() < p_up:
            t[0] = q(rng.uniform(0.05, 2.0)) or 0.1
            t[5] = q(rng.uniform(0.0, 2.0)) if rng.random() < 0.8 else 0.0
            act.add(rng.choice(names_up))
        if downs and rng.random() < p_down:
            t[2] = q(rng.uniform(0.05, 1.5)) or 0.1
            t[3] = q(rng.uniform(0.0, 1.5)) if rng.random() < 0.8 else 0.0
            act.add(rng.choice(downs))
        sid = ids[i] if ids is not None else i
        out.append(rw.SampleTiming(sid, *t, activated_sections=frozenset(act)))
    return out


def cfgs(g, dp_crit, aux):  # aux: {id: (dp, fanout)}
    out = {g.critical.id: rw.SectionConfig(dp=dp_crit)}
    for k, (dp, f) in aux.items():
        out[k] = rw.SectionConfig(dp=dp, fanout=f)
    return out


def recipe_case(rec, name, policy=rs.ExecPolicy.INTERLEAVED, with_sim=True):
    """Cost-model 6-tuples computed by the REFERENCE per_sample_times (costs.py:182-200)."""
    g = ref_graph(graph_desc(rec.graph))
    configs = {k: rw.SectionConfig(*v.as_tuple()) for k, v in rec.configs.items()}
    params = {k: rcosts.CostParams(flops_per_token_fwd=p.flops_per_token_fwd,
                                   peak_flops_per_gpu=p.peak_flops_per_gpu,
                                   bwd_fwd_ratio=p.bwd_fwd_ratio) for k, p in rec.params.items()}
    crit = g.critical.id
    B = rec.batch
    n_crit = math.ceil(B / configs[crit].dp)
    counts = {a.id: int((rec.tokens[a.id] > 0).sum()) for a in g.auxiliaries}
    batch = []
    for i in range(B):
        t = {p: 0.0 for p in rw.PHASES}
        t["f_c"], t["b_c"] = rcosts.per_sample_times(g.critical, configs[crit], params[crit],
                                                     int(rec.tokens[crit][i]), n_crit)
        act = set()
        for a in g.auxiliaries:
            tok = int(rec.tokens[a.id][i])
            if tok <= 0:
                continue
            n_aux = math.ceil(counts[a.id] / configs[a.id].dp)
            fwd, bwd = rcosts.per_sample_times(a, configs[a.id], params[a.id], tok, n_aux)
            if g.side(a.id) is rw.Side.UPSTREAM:
                t["f_bc"] += fwd
                t["b_ac"] += bwd
            else:
                t["f_ac"] += fwd
                t["b_bc"] += bwd
            act.add(a.id)
        batch.append(rw.SampleTiming(i, **{f"t_{p}": v for p, v in t.items()}, activated_sections=frozenset(act)))
    extra = {"recipe": rec.name, "tokens": {k: v.tolist() for k, v in rec.tokens.items()},
             "cost": {k: [H(p.flops_per_token_fwd), H(p.peak_flops_per_gpu), H(p.bwd_fwd_ratio)]
                      for k, p in rec.params.items()}}
    return run_case(name, g, configs, batch, policy, with_sim=with_sim, extra=extra)


def main():
    t0 = time.time()
    cases = []
    # --- shipped examples (vlm_fig8, distill_toy, omni_toy) ------------------
    for ex in ("vlm_fig8", "distill_toy", "omni_toy"):
        spec = load_spec(spec_path(ex))
        opts = RunOptions()
        plan = run_optimize(spec, opts)
        batch = batch_for(spec, plan, opts)
        for pol in rs.ExecPolicy:
            cases.append(run_case(f"example:{ex}:{pol.value}", spec.graph, plan.configs(), batch, pol))
    # --- SPEC known answers -----------------------------------------------------
    fig8 = [rw.SampleTiming(1, 0.1, 1, 0, 0, 2, 0.2), rw.SampleTiming(2, 0, 1, 0, 0, 2, 0),
            rw.SampleTiming(3, 0, 1, 0, 0, 2, 0), rw.SampleTiming(4, 0.2, 1, 0, 0, 2, 0.4)]
    known = {
        "sort_initial": [s.sample_id for s in rs.sort_initial(fig8)],
        "makespan_single_text": H(rs.calculate_makespan([rw.SampleTiming(0, 0, 1, 0, 0, 2, 0)])),
        "makespan_single_image": H(rs.calculate_makespan([rw.SampleTiming(0, 0.1, 1, 0, 0, 2, 0.2)])),
        "merge": rs.merge_fanout([["a1", "a2"], ["b1", "b2"]], 2),
        "merge_ragged": rs.merge_fanout([[1, 2, 3], [4], [], [5, 6]], 4),
    }
    # --- random instances ---------------------------------------------------------
    rng = random.Random(20260518)
    layouts = {
        "g2": (g2, [(1, {"enc": (1, 1)}), (2, {"enc": (1, 2)}), (3, {"enc": (1, 3)}), (4, {"enc": (2, 2)}),
                    (6, {"enc": (2, 3)}), (7, {"enc": (1, 7)}), (8, {"enc": (4, 2)})]),
        "g3": (g3, [(1, {"enc": (1, 1), "dec": (1, 1)}), (2, {"enc": (1, 2), "dec": (2, 1)}),
                    (4, {"enc": (2, 2), "dec": (1, 4)}), (6, {"enc": (3, 2), "dec": (2, 3)})]),
        "g4": (g4, [(2, {"image_enc": (1, 2), "audio_enc": (2, 1)}), (4, {"image_enc": (2, 2), "audio_enc": (1, 4)})]),
        "g5": (g5, [(2, {"enc": (1, 2), "pre": (1, 1), "dec": (1, 2)}), (4, {"enc": (2, 2), "pre": (1, 2), "dec": (4, 1)})]),
    }
    for gname, (gf, lays) in layouts.items():
        g = gf()
        for dp, aux in lays:
            for B in (dp, 3 * dp + 1, 12 * dp + (dp // 2)):
                if B > 200:
                    continue
                for pol in rs.ExecPolicy:
                    for quant in (False, True):
                        batch = random_batch(rng, g, B, quantized=quant)
                        cases.append(run_case(f"rand:{gname}:dp{dp}:B{B}:{pol.value}:q{int(quant)}",
                                              g, cfgs(g, dp, aux), batch, pol, with_sim=B <= 60))
    # merged exclusive encoders (omni-style) with submodule-named activations
    gm = rw.colocate_exclusive_encoders(g4(), "image_enc", "audio_enc")
    for dp, f in ((1, 1), (2, 1), (4, 2)):
        for pol in rs.ExecPolicy:
            batch = random_batch(rng, gm, 8 * dp + 3)
            cases.append(run_case(f"rand:merged:dp{dp}:{pol.value}", gm,
                                  cfgs(gm, dp, {"image_enc+audio_enc": (dp // f, f)}), batch, pol))
    # arbitrary sample ids (not 0..B-1), heavy ties
    g = g2()
    for pol in rs.ExecPolicy:
        ids = rng.sample(range(1000, 5000), 40)
        batch = random_batch(rng, g, 40, quantized=True, ids=ids)
        cases.append(run_case(f"rand:ids:{pol.value}", g, cfgs(g, 4, {"enc": (2, 2)}), batch, pol))
        batch = [rw.SampleTiming(i, 0.5 if i % 2 else 0.0, 1.0, 0, 0, 2.0, 0.5 if i % 2 else 0.0,
                                 frozenset({"enc"}) if i % 2 else frozenset()) for i in range(24)]
        cases.append(run_case(f"ties:{pol.value}", g, cfgs(g, 3, {"enc": (1, 3)}), batch, pol))
    # --- error cases ------------------------------------------------------------------
    g = g4()
    both = [rw.SampleTiming(0, 0.2, 1, 0, 0, 2, 0.2, frozenset({"image_enc", "audio_enc"})),
            rw.SampleTiming(1, 0, 1, 0, 0, 2, 0)]
    cases.append(run_case("err:two_upstream", g, cfgs(g, 1, {"image_enc": (1, 1), "audio_enc": (1, 1)}),
                          both, rs.ExecPolicy.INTERLEAVED))
    undeclared = [rw.SampleTiming(0, 0.2, 1, 0, 0, 2, 0.2), rw.SampleTiming(1, 0, 1, 0, 0, 2, 0)]
    cases.append(run_case("err:undeclared", g, cfgs(g, 1, {"image_enc": (1, 1), "audio_enc": (1, 1)}),
                          undeclared, rs.ExecPolicy.INTERLEAVED))
    cases.append(run_case("err:both_merged", gm, cfgs(gm, 1, {"image_enc+audio_enc": (1, 1)}),
                          both, rs.ExecPolicy.INTERLEAVED))
    g = g2()
    ok = random_batch(rng, g, 8)
    cases.append(run_case("err:fanout", g, cfgs(g, 4, {"enc": (1, 2)}), ok, rs.ExecPolicy.INTERLEAVED))
    dup = [rw.SampleTiming(3, 0, 1, 0, 0, 2, 0), rw.SampleTiming(3, 0, 1, 0, 0, 2, 0)]
    cases.append(run_case("err:dup_ids", g, cfgs(g, 1, {"enc": (1, 1)}), dup, rs.ExecPolicy.INTERLEAVED))
    # --- recipes (cost-model 6-tuples from token counts) --------------------------------
    for n in (1, 2, 4, 8):
        cases.append(recipe_case(recipes.vlm_tiny(n, 64), f"recipe:vlm_tiny:{n}gpu:B64"))
    cases.append(recipe_case(recipes.vlm_tiny(8, 256, seed=1), "recipe:vlm_tiny:8gpu:B256", with_sim=False))
    cases.append(recipe_case(recipes.vlm_tiny(4, 128, seed=2), "recipe:vlm_tiny:4gpu:B128:afb",
                             rs.ExecPolicy.ALL_FWD_THEN_BWD, with_sim=False))
    for n in (1, 4, 8):
        cases.append(recipe_case(recipes.kd(n, 32), f"recipe:kd:{n}gpu:B32"))
    for n in (1, 4, 8):  # cfg 3 Qwen2.5-VL-7B shape
        cases.append(recipe_case(recipes.vlm_7b(n, 64), f"recipe:vlm_7b:{n}gpu:B64", with_sim=n > 1))
    for n in (2, 8):  # cfg 4 omni, 3-way mix schedules; 4-way (img+audio) is rejected by the reference
        cases.append(recipe_case(recipes.omni(n, 48, mix="3way"), f"recipe:omni3:{n}gpu:B48"))
    cases.append(recipe_case(recipes.omni(8, 48, mix="4way"), "recipe:omni4:8gpu:B48"))
    for n in (4, 8):  # cfg 5 Llama-3-8B -> 3.2-1B
        cases.append(recipe_case(recipes.kd_8b(n, 32), f"recipe:kd_8b:{n}gpu:B32"))
    # --- evaluation-count bound ---------------------------------------------
    evals = {}
    g = g3()
    for n in (1, 2, 3, 8, 50, 200):
        batch = random_batch(rng, g, n)
        c = rs.EvalCounter()
        order = rs.schedule_rank(batch, rs.ExecPolicy.INTERLEAVED, c)
        evals[str(n)] = {"count": c.count, "samples": [sample_desc(s) for s in batch] if n <= 50 else None,
                         "order": [s.sample_id for s in order] if n <= 50 else None}
    out = {"generator": "tests/golden/make_golden.py", "reference": REF, "known": known,
           "evals": evals, "cases": cases}
    path = ROOT / "tests" / "golden" / "sched_golden.json"
    path.write_text(json.dumps(out, separators=(",", ":"), sort_keys=True))
    print(f"{len(cases)} cases -> {path} ({path.stat().st_size / 1e6:.2f} MB) in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
