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


if __name__ == "__main__":
    main()
