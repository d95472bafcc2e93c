"""Golden wire-format artifacts by running the REFERENCE spec parser and pipeline; build container only.

    python tests/golden/make_pipeline_golden.py   -> tests/golden/pipeline_golden.json

For each shipped example spec (`maestro-spec v1`, examples/*.yaml) and a few option sets, the
reference's `run_end2end` bundle as canonical JSON (plan `maestro-plan v1`, schedule
`maestro-schedule v1`, summary, report, trace), plus invalid-spec mutations with the
reference's `validate_document` diagnostics and `parse_spec` error (class, message, context).
The spec documents are stored parsed (plain dicts), so the GPU box never reads the reference.
"""

from __future__ import annotations

import copy
import json
import sys
from pathlib import Path

import yaml

sys.path.insert(0, str(Path(__file__).resolve().parent))
import make_golden  # noqa: E402,F401  (puts the reference package on sys.path)

from maestro import pipeline as rpl  # noqa: E402
from maestro.examples import NAMES, spec_text  # noqa: E402
from maestro.scheduling import ExecPolicy  # noqa: E402
from maestro.specfile import parse_spec  # noqa: E402

OPTIONS = {
    "default": rpl.RunOptions(),
    "fwd_then_bwd": rpl.RunOptions(policy=ExecPolicy.ALL_FWD_THEN_BWD),
    "linear100": rpl.RunOptions(comm="linear:100"),
    "seed3_earliest": rpl.RunOptions(seed=3, aux_execution="earliest-ready"),
    "bad_aux_mode": rpl.RunOptions(aux_execution="split"),
}


def mutations(doc):
    """(name, document) pairs that the reference rejects or diagnoses."""
    out = []

    def mut(name, f):
        d = copy.deepcopy(doc)
        f(d)
        out.append((name, d))

    mut("bad_version", lambda d: d.__setitem__("version", "maestro-spec v0"))
    mut("unknown_top", lambda d: d.__setitem__("extra", 1))
    mut("missing_cluster", lambda d: d.pop("cluster"))
    mut("bad_role", lambda d: d["sections"][0].__setitem__("role", "boss"))
    mut("bad_exec_mode", lambda d: d["sections"][0].__setitem__("exec_mode", "sideways"))
    mut("bad_structural", lambda d: d["sections"][0]["structural"].__setitem__("hidden_dim", 1.5))
    mut("unknown_structural", lambda d: d["sections"][0]["structural"].__setitem__("width", 3))
    mut("bad_preset", lambda d: d["sections"][0].__setitem__("cost", {"preset": "nope"}))
    mut("bad_cost_number", lambda d: d["sections"][0].__setitem__("cost", {"flops_per_token_fwd": "x"}))
    mut("zero_pin", lambda d: d["sections"][0].__setitem__("config", {"dp": 0}))
    mut("unknown_pin", lambda d: d["sections"][0].__setitem__("config", {"zz": 1}))
    mut("pin_fanout_violation", lambda d: [s.__setitem__("config", {**s.get("config", {}), "dp": 3, "fanout": 5})
                                           for s in d["sections"] if s["role"] == "auxiliary"])
    mut("pin_indivisible", lambda d: d["sections"][0].__setitem__("config", {"tp": 7}))
    mut("tiny_cluster", lambda d: d["cluster"].__setitem__("total_gpus", 1))
    mut("both_batch", lambda d: d["batch"].__setitem__("profile", {"global_batch_size": 4}))
    mut("profile_unknown_section", lambda d: d.__setitem__("batch", {"profile": {"global_batch_size": 4,
                                                                               "shares": {"nope": 0.5}}}))
    mut("profile_bad_share", lambda d: d.__setitem__("batch", {"profile": {"global_batch_size": 4,
                                                                         "shares": {d["sections"][0]["name"]: 2.0}}}))
    mut("profile_ok", lambda d: d.__setitem__("batch", {"profile": {"global_batch_size": 16}}))
    mut("duplicate_ids", lambda d: d["batch"].__setitem__("samples", d["batch"].get("samples", [{}])[:1] * 2)
        if "samples" in d["batch"] else None)
    mut("negative_time", lambda d: d["batch"]["samples"][0].__setitem__("t_f_c", -1) if "samples" in d["batch"]
        else None)
    mut("no_sections", lambda d: d.__setitem__("sections", []))
    mut("bad_transform", lambda d: d.__setitem__("transforms", [{"op": "fold"}]))
    mut("bad_edge_key", lambda d: d.__setitem__("edges", [{"from": "a", "to": "b", "w": 1}]))
    return out


def parse_outcome(doc):
    try:
        parse_spec(doc)
        return None
    except Exception as e:  # noqa: BLE001
        return {"class": type(e).__name__, "message": str(e),
                "context": {k: str(v) for k, v in sorted(getattr(e, "context", {}).items())}}


def main():
    cases = []
    for name in NAMES:
        doc = yaml.safe_load(spec_text(name))
        spec = parse_spec(doc, source=name)
        case = {"name": name, "doc": doc, "end2end": {}, "validate": rpl.validate_document(doc, name),
                "mutations": []}
        for oname, opts in OPTIONS.items():
            try:
                case["end2end"][oname] = rpl.canonical_json(rpl.run_end2end(spec, opts))
            except Exception as e:  # noqa: BLE001
                case["end2end"][oname] = {"error": type(e).__name__, "message": str(e)}
        for mname, mdoc in mutations(doc):
            rec = {"name": mname, "doc": mdoc, "validate": rpl.validate_document(mdoc, name),
                   "parse": parse_outcome(mdoc)}
            if mname == "profile_ok":  # derived batch (cost model at the plan's configs)
                rec["end2end"] = rpl.canonical_json(rpl.run_end2end(parse_spec(mdoc), rpl.RunOptions()))
            case["mutations"].append(rec)
        cases.append(case)
    out = Path(__file__).resolve().parent / "pipeline_golden.json"
    out.write_text(json.dumps({"cases": cases}, indent=1, sort_keys=True) + "\n")
    print(f"wrote {out} ({len(cases)} specs)")


if __name__ == "__main__" and "--random" not in sys.argv:
    main()


# --- randomised spec documents (graph shapes x clusters x pins x batch kinds) -------------------


def _section(name, role, mode, hidden, heads, layers, vocab, seq, params, preset=None, extra=None, pin=None):
    d = {"name": name, "role": role, "exec_mode": mode,
         "structural": {"hidden_dim": hidden, "num_heads": heads, "num_layers": layers, "vocab_size": vocab,
                        "max_seq_len": seq, "param_count": params}}
    cost = {}
    if preset:
        cost["preset"] = preset
    if extra:
        cost.update(extra)
    if cost:
        d["cost"] = cost
    if pin:
        d["config"] = pin
    return d


def random_docs(seed=0, n=24):
    import random

    rng = random.Random(seed)
    docs = []
    for i in range(n):
        kind = ["vlm", "kd", "enc_dec", "omni"][i % 4]
        gpus = rng.choice([4, 8, 16])
        pin_crit = rng.random() < 0.5
        crit_pin = {"dp": rng.choice([1, 2, 4]), "tp": 1, "pp": 1, "cp": 1, "mbs": rng.choice([1, 2])} if pin_crit else None
        secs, edges, transforms, subs_up = [], [], [], []
        crit = _section("llm", "critical", "forward_backward", 2048, 16, 16, 32000, 4096, 1_000_000_000,
                        preset="moe-backbone", pin=crit_pin)
        if kind == "vlm":
            secs = [_section("vit", "auxiliary", "forward_backward", 1024, 16, 24, 1, 8192, 300_000_000,
                             preset="vit-encoder"), crit]
            edges = [{"from": "vit", "to": "llm", "payload_bytes_per_sample": 4194304}]
            subs_up = ["vit"]
        elif kind == "kd":
            crit = _section("student", "critical", "forward_backward", 768, 12, 12, 32000, 2048, 125_000_000,
                            preset="moe-backbone", extra={"flops_per_token_fwd": 2.5e9}, pin=crit_pin)
            secs = [_section("teacher", "auxiliary", "forward_only", 2048, 32, 22, 32000, 2048, 1_100_000_000,
                             preset="frozen-teacher"), crit]
            edges = [{"from": "teacher", "to": "student", "payload_bytes_per_sample": 2048 * 32000 * 2}]
            transforms = [{"op": "colocate_output_layer", "teacher": "teacher", "student": "student",
                           "hidden_dim": 2048, "vocab_size": 32000}]
            subs_up = ["teacher"]
        elif kind == "enc_dec":
            secs = [_section("enc", "auxiliary", "forward_backward", 1024, 16, 12, 1, 4096, 200_000_000,
                             preset="vit-encoder"), crit,
                    _section("dec", "auxiliary", "forward_backward", 1024, 8, 8, 4096, 2048, 150_000_000,
                             preset="vit-encoder", extra={"flops_per_token_fwd": 1.5e9})]
            edges = [{"from": "enc", "to": "llm", "payload_bytes_per_sample": 2097152},
                     {"from": "llm", "to": "dec", "payload_bytes_per_sample": 1048576}]
            subs_up = ["enc", "dec"]
        else:
            secs = [_section("image_enc", "auxiliary", "forward_backward", 1024, 16, 24, 1, 8192, 300_000_000,
                             preset="vit-encoder"),
                    _section("audio_enc", "auxiliary", "forward_backward", 1024, 8, 16, 1, 4096, 200_000_000,
                             preset="vit-encoder", extra={"flops_per_token_fwd": 1.2e9}), crit]
            edges = [{"from": "image_enc", "to": "llm", "payload_bytes_per_sample": 4194304},
                     {"from": "audio_enc", "to": "llm", "payload_bytes_per_sample": 2097152}]
            transforms = [{"op": "colocate_exclusive_encoders", "a": "image_enc", "b": "audio_enc"}]
            subs_up = ["image_enc", "audio_enc"]
        doc = {"version": "maestro-spec v1", "sections": secs, "edges": edges,
               "cluster": {"total_gpus": gpus, "mem_per_gpu": 8.0e10}}
        if transforms:
            doc["transforms"] = transforms
        crit_name = crit["name"]
        if rng.random() < 0.5:  # explicit batch of random 6-tuples
            B = rng.randint(4, 24)
            samples = []
            for s in range(B):
                row = {"id": s, "t_f_c": round(rng.uniform(0.5, 2.0), 3), "t_b_c": round(rng.uniform(1.0, 4.0), 3)}
                if kind == "kd":
                    row.update(t_f_bc=round(rng.uniform(0.5, 1.5), 3), activates=["teacher"])
                elif kind == "enc_dec":
                    if rng.random() < 0.6:
                        row.update(t_f_bc=round(rng.uniform(0.1, 0.5), 3), t_b_ac=round(rng.uniform(0.2, 1.0), 3),
                                   activates=["enc"])
                    if rng.random() < 0.5:
                        row.update(t_f_ac=round(rng.uniform(0.1, 0.4), 3), t_b_bc=round(rng.uniform(0.1, 0.6), 3),
                                   activates=sorted(set(row.get("activates", [])) | {"dec"}))
                elif rng.random() < 0.6:
                    sub = rng.choice(subs_up)
                    row.update(t_f_bc=round(rng.uniform(0.1, 0.5), 3), t_b_ac=round(rng.uniform(0.2, 1.0), 3),
                               activates=[sub])
                samples.append(row)
            doc["batch"] = {"samples": samples}
        else:  # statistical profile, batch derived from the cost model at the plan's configs
            prof = {"global_batch_size": rng.choice([8, 16, 32])}
            if kind != "kd":
                live = subs_up if kind != "omni" else []
                if live:
                    prof["shares"] = {s: round(rng.uniform(0.2, 0.8), 2) for s in live}
                prof["tokens"] = {crit_name: rng.choice([1024, 2048, 4096])}
            doc["batch"] = {"profile": prof}
        docs.append((f"random_{i}_{kind}", doc))
    return docs


def random_cases():
    out = []
    for name, doc in random_docs():
        case = {"name": name, "doc": doc, "validate": rpl.validate_document(doc, name), "parse": parse_outcome(doc),
                "end2end": {}}
        if case["parse"] is None:
            spec = parse_spec(doc, source=name)
            for oname in ("default", "fwd_then_bwd"):
                try:
                    case["end2end"][oname] = rpl.canonical_json(rpl.run_end2end(spec, OPTIONS[oname]))
                except Exception as e:  # noqa: BLE001
                    case["end2end"][oname] = {"error": type(e).__name__, "message": str(e)}
        out.append(case)
    return out


if __name__ == "__main__" and "--random" in sys.argv:
    rc = random_cases()
    p = Path(__file__).resolve().parent / "pipeline_random_golden.json"
    p.write_text(json.dumps({"cases": rc}, indent=1, sort_keys=True) + "\n")
    print(f"wrote {p}: {len(rc)} cases, {sum(1 for c in rc if c['parse'] is None)} parsed")
