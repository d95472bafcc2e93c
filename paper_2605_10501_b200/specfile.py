"""`maestro-spec v1` workload spec files (host side of the drop-in API).

Same document schema, defaults and error behaviour as the reference's spec loader
(``/root/reference/pkg/src/maestro/specfile.py:242-401``): a YAML (or JSON) mapping declaring
sections, data-flow edges, the cluster, colocation transforms, pinned per-section configs, cost
parameters (or shipped presets), and either an explicit sample batch or a statistical batch
profile.  Unknown fields are rejected with their path; every failure is a :class:`ParseError`
whose ``field`` context names the offending path, except cost-model validation, which raises the
cost model's own class (as the reference does).

The parser is table-driven here: each record type is a :class:`_Rec` view that checks its key
set once and converts fields by path, so the document walk reads top to bottom.  The result
feeds :mod:`.pipeline` (planner -> device schedule -> simulator).
"""

from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path
from typing import Any, Mapping, Optional

from .costs import BatchProfile, CostParams, preset
from .errors import MaestroError, ParseError
from .workload import (
    ClusterSpec,
    Edge,
    ExecMode,
    Role,
    SampleTiming,
    SectionGraph,
    SectionId,
    SectionSpec,
    StructuralParams,
    build_graph,
    colocate_exclusive_encoders,
    colocate_output_layer,
)

SCHEMA_VERSION = "maestro-spec v1"

# cost of a section that declares none (specfile.py:36-40)
_DEFAULT_COST = CostParams(flops_per_token_fwd=1.0e9, peak_flops_per_gpu=1.0e14, activation_bytes_per_token=0.0)

_COST_SCALARS = ("flops_per_token_fwd", "peak_flops_per_gpu", "bwd_fwd_ratio", "bytes_per_param_weights",
                 "bytes_per_param_optimizer", "activation_bytes_per_token", "live_microbatch_cap")
_STRUCTURAL = ("hidden_dim", "num_heads", "num_layers", "vocab_size", "max_seq_len")
_DEGREES = ("dp", "tp", "pp", "cp", "mbs", "fanout")
_PHASES = ("t_f_bc", "t_f_c", "t_f_ac", "t_b_bc", "t_b_c", "t_b_ac")


@dataclass(frozen=True)
class WorkloadSpec:
    """A parsed, validated spec: everything the pipeline needs (specfile.py:43-73)."""

    graph: SectionGraph
    cluster: ClusterSpec
    params_by_section: Mapping[SectionId, CostParams]
    pinned: Mapping[SectionId, Mapping[str, int]]
    batch: Optional[tuple[SampleTiming, ...]]
    profile: Optional[BatchProfile]
    source: str = "<dict>"

    def effective_profile(self) -> BatchProfile:
        """The declared profile, or the activation shares of the explicit batch."""
        if self.profile is not None:
            return self.profile
        assert self.batch is not None
        counts: dict[SectionId, int] = {}
        for sample in self.batch:
            for sid in self.graph.resolve_activation(sample):
                if sid is not None:
                    counts[sid] = counts.get(sid, 0) + 1
        n = len(self.batch)
        return BatchProfile(global_batch_size=n, shares={sid: c / n for sid, c in sorted(counts.items())})


class _Rec:
    """One mapping of the document at ``path``, with its key set checked on construction."""

    def __init__(self, raw: Any, path: str, allowed=None, required=()):
        if not isinstance(raw, dict):
            raise ParseError(f"{path}: expected a mapping, got {type(raw).__name__}", field=path)
        self.raw, self.path = raw, path
        if allowed is not None:
            allowed = set(allowed)
            unknown = set(raw) - allowed
            if unknown:
                raise ParseError(f"{path}: unknown field(s) {sorted(unknown)}; allowed: {sorted(allowed)}",
                                 field=path)
            missing = set(required) - set(raw)
            if missing:
                raise ParseError(f"{path}: missing required field(s) {sorted(missing)}", field=path)

    def __contains__(self, key: str) -> bool:
        return key in self.raw

    def __getitem__(self, key: str) -> Any:
        return self.raw[key]

    def get(self, key: str, default: Any = None) -> Any:
        return self.raw.get(key, default)

    def at(self, key: str) -> str:
        return f"{self.path}.{key}"

    def num(self, key: str, default: Any = None) -> float:
        return _number(self.raw.get(key, default), self.at(key))

    def int(self, key: str, default: Any = None) -> int:
        return _integer(self.raw.get(key, default), self.at(key))


def _number(value: Any, path: str) -> float:
    if isinstance(value, bool) or not isinstance(value, (int, float)):
        raise ParseError(f"{path}: expected a number, got {value!r}", field=path)
    return float(value)


def _integer(value: Any, path: str) -> int:
    if isinstance(value, bool) or not isinstance(value, int):
        raise ParseError(f"{path}: expected an integer, got {value!r}", field=path)
    return value


def _structural(raw: Any, path: str) -> StructuralParams:
    r = _Rec(raw, path, _STRUCTURAL + ("param_count",), _STRUCTURAL)
    return StructuralParams(*(r.int(k) for k in _STRUCTURAL), param_count=r.int("param_count", 0))


def _cost(raw: Any, path: str) -> CostParams:
    """Preset (or the default) overlaid with the declared fields (specfile.py:121-177)."""
    r = _Rec(raw, path, ("preset", "parallel_efficiency", "mbs_efficiency") + _COST_SCALARS)
    base = preset(r["preset"]) if "preset" in r else _DEFAULT_COST
    kw: dict[str, Any] = {k: getattr(base, k) for k in _COST_SCALARS}
    kw["parallel_efficiency"] = dict(base.parallel_efficiency)
    kw["mbs_efficiency"] = dict(base.mbs_efficiency)
    kw.update({k: r.num(k) for k in _COST_SCALARS if k in r})
    if "parallel_efficiency" in r:
        entries = r["parallel_efficiency"]
        if not isinstance(entries, list):
            raise ParseError(f"{path}.parallel_efficiency: expected a list of entries")
        table = {}
        for i, entry in enumerate(entries):
            e = _Rec(entry, f"{path}.parallel_efficiency[{i}]", ("tp", "pp", "cp", "factor"),
                     ("tp", "pp", "cp", "factor"))
            table[(e["tp"], e["pp"], e["cp"])] = e.num("factor")
        kw["parallel_efficiency"] = table
    if "mbs_efficiency" in r:
        m = _Rec(r["mbs_efficiency"], f"{path}.mbs_efficiency")
        kw["mbs_efficiency"] = {_integer(k, f"{path}.mbs_efficiency key"): _number(v, f"{path}.mbs_efficiency[{k}]")
                                for k, v in m.raw.items()}
    try:
        return CostParams(**kw)
    except MaestroError as exc:
        raise ParseError(f"{path}: {exc}", field=path)


def _pin(raw: Any, path: str) -> dict[str, int]:
    r = _Rec(raw, path, _DEGREES)
    pin = {k: r.int(k) for k in r.raw}
    for k, v in pin.items():
        if v < 1:
            raise ParseError(f"{path}.{k}: must be >= 1, got {v}", field=f"{path}.{k}")
    return pin


def _sample(raw: Any, index: int, path: str) -> SampleTiming:
    r = _Rec(raw, path, ("id", "activates") + _PHASES, ("t_f_c",))
    acts = r.get("activates", [])
    if not isinstance(acts, list) or not all(isinstance(a, str) for a in acts):
        raise ParseError(f"{path}.activates: expected a list of section/submodule names")
    try:
        return SampleTiming(sample_id=r.int("id", index), **{k: r.num(k, 0) for k in _PHASES},
                            activated_sections=frozenset(acts))
    except MaestroError as exc:
        raise ParseError(f"{path}: {exc}", field=path)


def _section(raw: Any, path: str) -> tuple[SectionSpec, Optional[CostParams], Optional[dict[str, int]]]:
    r = _Rec(raw, path, ("name", "role", "exec_mode", "structural", "submodules", "cost", "config"),
             ("name", "role", "exec_mode", "structural"))
    name = r["name"]
    if not isinstance(name, str) or not name:
        raise ParseError(f"{path}.name: expected a non-empty string")
    try:
        role = Role(r["role"])
    except ValueError:
        raise ParseError(f"{path}.role: expected 'critical' or 'auxiliary', got {r['role']!r}")
    try:
        mode = ExecMode(r["exec_mode"])
    except ValueError:
        raise ParseError(f"{path}.exec_mode: expected 'forward_only' or 'forward_backward', got {r['exec_mode']!r}")
    subs = r.get("submodules", [])
    if "submodules" in r and (not isinstance(subs, list) or not all(isinstance(x, str) for x in subs)):
        raise ParseError(f"{path}.submodules: expected a list of strings")
    spec = SectionSpec(id=name, role=role, exec_mode=mode, structural=_structural(r["structural"], r.at("structural")),
                       submodules=tuple(subs))
    cost = _cost(r["cost"], r.at("cost")) if "cost" in r else None
    pin = _pin(r["config"], r.at("config")) if "config" in r else None
    return spec, cost, pin


_TRANSFORMS = {
    # op -> (fields, apply(graph, record))
    "colocate_output_layer": (("teacher", "student", "hidden_dim", "vocab_size"),
                              lambda g, r: colocate_output_layer(g, r["teacher"], r["student"], r.int("hidden_dim"),
                                                                 r.int("vocab_size"))),
    "colocate_exclusive_encoders": (("a", "b"), lambda g, r: colocate_exclusive_encoders(g, r["a"], r["b"])),
}


def _transforms(graph: SectionGraph, raw: Any, path: str) -> SectionGraph:
    if raw is None:
        return graph
    if not isinstance(raw, list):
        raise ParseError(f"{path}: expected a list of transform records")
    for i, entry in enumerate(raw):
        where = f"{path}[{i}]"
        op = _Rec(entry, where).get("op")
        if op not in _TRANSFORMS:
            raise ParseError(f"{where}.op: unknown transform {op!r} "
                             "(known: colocate_output_layer, colocate_exclusive_encoders)", field=f"{where}.op")
        fields, apply = _TRANSFORMS[op]
        graph = apply(graph, _Rec(entry, where, ("op",) + fields, ("op",) + fields))
    return graph


def _batch(raw: Any, graph: SectionGraph):
    b = _Rec(raw, "spec.batch", ("samples", "profile"))
    if ("samples" in b) == ("profile" in b):
        raise ParseError("spec.batch: declare exactly one of 'samples' or 'profile'")
    if "samples" in b:
        rows = b["samples"]
        if not isinstance(rows, list) or not rows:
            raise ParseError("spec.batch.samples: expected a non-empty list")
        batch = tuple(_sample(x, i, f"spec.batch.samples[{i}]") for i, x in enumerate(rows))
        if len({s.sample_id for s in batch}) != len(batch):
            raise ParseError("spec.batch.samples: duplicate sample ids")
        for i, sample in enumerate(batch):
            try:
                graph.resolve_activation(sample)
            except MaestroError as exc:
                raise ParseError(f"spec.batch.samples[{i}]: {exc}")
        return batch, None
    p = _Rec(b["profile"], "spec.batch.profile", ("global_batch_size", "shares", "tokens"), ("global_batch_size",))
    shares = _Rec(p.get("shares", {}), "spec.batch.profile.shares")
    tokens = _Rec(p.get("tokens", {}), "spec.batch.profile.tokens")
    live = set(graph.section_ids)
    for sid in list(shares.raw) + list(tokens.raw):
        if sid not in live:
            raise ParseError(f"spec.batch.profile: unknown section '{sid}'", field="spec.batch.profile")
    try:
        profile = BatchProfile(global_batch_size=p.int("global_batch_size"),
                               shares={k: _number(v, f"spec.batch.profile.shares[{k}]") for k, v in shares.raw.items()},
                               tokens={k: _integer(v, f"spec.batch.profile.tokens[{k}]") for k, v in tokens.raw.items()})
    except MaestroError as exc:
        raise ParseError(f"spec.batch.profile: {exc}")
    return None, profile


def parse_spec(doc: Any, source: str = "<dict>") -> WorkloadSpec:
    """Validate a parsed YAML/JSON document into a :class:`WorkloadSpec` (specfile.py:242-401)."""
    top = _Rec(doc, "spec", ("version", "sections", "edges", "cluster", "transforms", "batch"),
               ("version", "sections", "cluster", "batch"))
    if top["version"] != SCHEMA_VERSION:
        raise ParseError(f"spec.version: expected '{SCHEMA_VERSION}', got {top['version']!r}", field="spec.version")
    if not isinstance(top["sections"], list) or not top["sections"]:
        raise ParseError("spec.sections: expected a non-empty list")
    sections, costs, pins = [], {}, {}
    for i, raw in enumerate(top["sections"]):
        spec, cost, pin = _section(raw, f"spec.sections[{i}]")
        sections.append(spec)
        if cost is not None:
            costs[spec.id] = cost
        if pin is not None:
            pins[spec.id] = pin
    edges = []
    for i, raw in enumerate(top.get("edges", []) or []):
        e = _Rec(raw, f"spec.edges[{i}]", ("from", "to", "payload_bytes_per_sample"), ("from", "to"))
        edges.append(Edge(src=e["from"], dst=e["to"], payload_bytes_per_sample=e.num("payload_bytes_per_sample", 0)))
    c = _Rec(top["cluster"], "spec.cluster", ("total_gpus", "mem_per_gpu"), ("total_gpus", "mem_per_gpu"))
    cluster = ClusterSpec(total_gpus=c.int("total_gpus"), mem_per_gpu=c.num("mem_per_gpu"))
    try:
        graph = _transforms(build_graph(sections, edges), top.get("transforms"), "spec.transforms")
    except ParseError:
        raise
    except MaestroError as exc:
        raise ParseError(f"spec: {exc}", field="spec")
    live = set(graph.section_ids)
    for name in pins:
        if name not in live:
            raise ParseError(f"spec: section '{name}' pins a config but a transform replaced it",
                             field="spec.transforms")
    # cost params of a section merged away by a transform carry over to the merged section
    params = {}
    for s in graph.sections:
        donors = [n for n in costs if n in s.submodules or s.id.startswith(f"{n}+")]
        params[s.id] = costs.get(s.id) or (costs[sorted(donors)[0]] if donors else _DEFAULT_COST)
    batch, profile = _batch(top["batch"], graph)
    return WorkloadSpec(graph=graph, cluster=cluster, params_by_section=params, pinned=pins, batch=batch,
                        profile=profile, source=source)


def load_spec(path: "str | Path") -> WorkloadSpec:
    """Parse a spec file from disk (YAML or JSON)."""
    import yaml

    p = Path(path)
    try:
        text = p.read_text(encoding="utf-8")
    except OSError as exc:
        raise ParseError(f"cannot read spec file {p}: {exc}", file=str(p))
    try:
        doc = yaml.safe_load(text)
    except yaml.YAMLError as exc:
        mark = getattr(exc, "problem_mark", None)
        where = f" at line {mark.line + 1}, column {mark.column + 1}" if mark else ""
        raise ParseError(f"invalid YAML in {p}{where}: {exc}", file=str(p))
    return parse_spec(doc, source=str(p))


__all__ = ["SCHEMA_VERSION", "WorkloadSpec", "parse_spec", "load_spec"]
