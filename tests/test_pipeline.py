"""`maestro-spec v1` parsing, `maestro-plan v1` / `maestro-schedule v1` documents and the
optimize -> schedule -> simulate pipeline against the reference's own outputs
(tests/golden/pipeline_golden.json, made by tests/golden/make_pipeline_golden.py from the
reference's shipped example specs and invalid mutations of them).

CPU: spec parsing (accept / reject with the reference's class, message and field), diagnostics,
document round trips.  GPU: run_end2end (planner + device schedule + simulator) byte-identical to
the reference's canonical JSON bundle.
"""

import json
from pathlib import Path

import pytest

from paper_2605_10501_b200 import pipeline as P
from paper_2605_10501_b200.errors import MaestroError
from paper_2605_10501_b200.specfile import load_spec, parse_spec

GOLD = json.loads((Path(__file__).parent / "golden" / "pipeline_golden.json").read_text())
CASES = {c["name"]: c for c in GOLD["cases"]}
MUTATIONS = [(c["name"], m["name"]) for c in GOLD["cases"] for m in c["mutations"]]
OPTIONS = {
    "default": P.RunOptions(),
    "fwd_then_bwd": P.RunOptions(policy=P.ExecPolicy.ALL_FWD_THEN_BWD),
    "linear100": P.RunOptions(comm="linear:100"),
    "seed3_earliest": P.RunOptions(seed=3, aux_execution="earliest-ready"),
    "bad_aux_mode": P.RunOptions(aux_execution="split"),
}


def _mutation(spec, name):
    return next(m for m in CASES[spec]["mutations"] if m["name"] == name)


@pytest.mark.parametrize("name", sorted(CASES))
def test_examples_parse_and_validate(name):
    case = CASES[name]
    spec = parse_spec(case["doc"], source=name)
    assert spec.graph.critical is not None
    assert P.validate_document(case["doc"], name) == case["validate"]


@pytest.mark.parametrize("spec,mut", MUTATIONS)
def test_invalid_specs_match_reference(spec, mut):
    m = _mutation(spec, mut)
    assert P.validate_document(m["doc"], spec) == m["validate"]
    want = m["parse"]
    if want is None:
        parse_spec(m["doc"])
        return
    with pytest.raises(MaestroError) as ei:
        parse_spec(m["doc"])
    e = ei.value
    assert type(e).__name__ == want["class"]
    assert str(e) == want["message"]
    assert {k: str(v) for k, v in sorted(e.context.items())} == want["context"]


def test_load_spec_yaml_and_errors(tmp_path):
    import yaml

    p = tmp_path / "vlm.yaml"
    p.write_text(yaml.safe_dump(CASES["vlm_fig8"]["doc"]))
    spec = load_spec(p)
    assert spec.source == str(p) and len(spec.batch) == 12
    bad = tmp_path / "bad.yaml"
    bad.write_text("version: [unclosed\n")
    with pytest.raises(MaestroError, match="invalid YAML"):
        load_spec(bad)
    with pytest.raises(MaestroError, match="cannot read spec file"):
        load_spec(tmp_path / "missing.yaml")


@pytest.mark.parametrize("name", sorted(CASES))
def test_document_round_trips(name):
    """plan / schedule documents of the reference's bundle survive from_dict -> to_dict unchanged."""
    bundle = json.loads(CASES[name]["end2end"]["default"])
    plan = P.plan_from_dict(bundle["plan"])
    assert P.plan_to_dict(plan) == bundle["plan"]
    sched = P.schedule_from_dict(bundle["schedule"])
    assert P.schedule_to_dict(sched) == bundle["schedule"]
    assert P.canonical_json(P.schedule_to_dict(sched)) == P.canonical_json(bundle["schedule"])
    with pytest.raises(MaestroError, match="version mismatch"):
        P.schedule_from_dict({**bundle["schedule"], "version": "maestro-schedule v0"})
    with pytest.raises(MaestroError, match="version mismatch"):
        P.plan_from_dict({**bundle["plan"], "version": None})


def test_run_options_comm():
    assert P.RunOptions().comm_model() is None
    assert P.RunOptions(comm="linear:100").comm_model()(1e9) == 1e9 / 100e9
    for bad in ("linear", "linear:x", "linear:-1", "cubic:3"):
        with pytest.raises(MaestroError, match="bad comm spec"):
            P.RunOptions(comm=bad).comm_model()


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("opt", sorted(OPTIONS))
def test_end2end_bundle_matches_reference(name, opt):
    """plan + device schedule + summary + simulator report + trace, byte-identical."""
    want = CASES[name]["end2end"][opt]
    spec = parse_spec(CASES[name]["doc"], source=name)
    if isinstance(want, dict):  # the reference rejected the options
        with pytest.raises(Exception) as ei:
            P.run_end2end(spec, OPTIONS[opt])
        assert type(ei.value).__name__ == want["error"] and str(ei.value) == want["message"]
        return
    got = P.canonical_json(P.run_end2end(spec, OPTIONS[opt]))
    assert got == want


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_end2end_derived_batch_matches_reference(name):
    """A profile-only spec: the batch is derived from the cost model at the plan's configs."""
    m = _mutation(name, "profile_ok")
    want = m.get("end2end")
    if want is None:
        pytest.skip("no derived-batch bundle in the golden file")
    got = P.canonical_json(P.run_end2end(parse_spec(m["doc"]), P.RunOptions()))
    assert got == want


RANDOM = json.loads((Path(__file__).parent / "golden" / "pipeline_random_golden.json").read_text())["cases"]
RANDOM_IDS = [c["name"] for c in RANDOM]


@pytest.mark.parametrize("case", RANDOM, ids=RANDOM_IDS)
def test_random_specs_parse_and_validate(case):
    """24 generated spec documents (VLM, KD with a colocated head, encoder + decoder, omni with
    colocated encoders; explicit batches or profiles; pinned or free configs; 4-16 GPUs)."""
    assert P.validate_document(case["doc"], case["name"]) == case["validate"]
    spec = parse_spec(case["doc"], source=case["name"])
    assert spec.graph.critical is not None


@pytest.mark.gpu
@pytest.mark.parametrize("case", RANDOM, ids=RANDOM_IDS)
@pytest.mark.parametrize("opt", ["default", "fwd_then_bwd"])
def test_random_specs_end2end_match_reference(case, opt):
    want = case["end2end"][opt]
    spec = parse_spec(case["doc"], source=case["name"])
    if isinstance(want, dict):  # the reference's planner rejected the spec
        with pytest.raises(Exception) as ei:
            P.run_end2end(spec, OPTIONS[opt])
        assert type(ei.value).__name__ == want["error"] and str(ei.value) == want["message"]
        return
    assert P.canonical_json(P.run_end2end(spec, OPTIONS[opt])) == want
