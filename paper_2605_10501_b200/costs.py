"""Cost model knobs that feed the device 6-tuple kernel (K1).

The reference derives per-sample 6-tuples from a roofline-style estimator
(``maestro/costs.py:105-200``) and sums them per side in ``derive_batch``
(``costs.py:230-299``).  Here the same arithmetic runs on the device, one
thread per sample, from the per-sample token counts of the step
(``csrc/plan.cu: plan_sample_times_kernel``).  This module holds the host-side
parameter objects and lowers them to the flat per-submodule cost table the
kernel reads.  The host only precomputes the per-section constant
``effective = peak * tp * cp * efficiency`` in exactly the reference's
left-to-right order, so the device result is bit-identical.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Mapping

import numpy as np

from .errors import InvalidConfig, InvalidDims
from .workload import SectionConfig, SectionGraph, SectionSpec


@dataclass(frozen=True)
class CostParams:
    """Time/memory model knobs of one section (costs.py:30-68)."""

    flops_per_token_fwd: float
    peak_flops_per_gpu: float
    bwd_fwd_ratio: float = 2.0
    parallel_efficiency: Mapping[tuple[int, int, int], float] = field(default_factory=dict)
    mbs_efficiency: Mapping[int, float] = field(default_factory=dict)
    bytes_per_param_weights: float = 2.0
    bytes_per_param_optimizer: float = 12.0
    activation_bytes_per_token: float = 0.0
    live_microbatch_cap: float = 4.0

    def __post_init__(self) -> None:
        if self.flops_per_token_fwd <= 0 or self.peak_flops_per_gpu <= 0:
            raise InvalidDims("flops_per_token_fwd and peak_flops_per_gpu must be positive")
        if self.bwd_fwd_ratio <= 0:
            raise InvalidDims("bwd_fwd_ratio must be positive")
        if self.parallel_efficiency.get((1, 1, 1), 1.0) != 1.0:
            raise InvalidDims("parallel_efficiency(1,1,1) must be 1")
        for eff in list(self.parallel_efficiency.values()) + list(self.mbs_efficiency.values()):
            if not 0 < eff <= 1:
                raise InvalidDims("efficiencies must lie in (0,1]")

    def efficiency(self, config: SectionConfig) -> float:
        par = self.parallel_efficiency.get((config.tp, config.pp, config.cp), 1.0)
        return par * self.mbs_efficiency.get(config.mbs, 1.0)


def check_config(section: SectionSpec, config: SectionConfig) -> None:
    if not config.divides(section.structural):
        s = section.structural
        raise InvalidConfig(
            f"config tp={config.tp} pp={config.pp} cp={config.cp} does not divide section "
            f"'{section.id}' structural params (heads={s.num_heads}, layers={s.num_layers}, "
            f"seq={s.max_seq_len})",
            section=section.id,
        )


def effective_rate(config: SectionConfig, params: CostParams) -> float:
    """``peak * tp * cp * efficiency`` with the reference's evaluation order (costs.py:121)."""
    return params.peak_flops_per_gpu * config.tp * config.cp * params.efficiency(config)


def estimate_step_time(section: SectionSpec, config: SectionConfig, params: CostParams,
                       tokens_per_sample: int) -> tuple[float, float]:
    """(forward, backward) time of one micro-batch of ``config.mbs`` samples (costs.py:105-123):
    mbs * tokens * flops_per_token / (peak * tp * cp * efficiency); backward = ratio x forward,
    or 0 for forward-only sections."""
    check_config(section, config)
    if tokens_per_sample <= 0:
        raise InvalidDims("tokens_per_sample must be positive")
    fwd = (config.mbs * tokens_per_sample * params.flops_per_token_fwd) / effective_rate(config, params)
    return fwd, (0.0 if section.forward_only else fwd * params.bwd_fwd_ratio)


def section_iteration_time(section: SectionSpec, config: SectionConfig, params: CostParams,
                           tokens_per_sample: int, samples_per_rank: int) -> float:
    """One DP rank's share of an iteration through a pp-deep pipeline (costs.py:159-179):
    (m + pp - 1) * (fwd + bwd) / pp with m = ceil(samples / mbs) micro-batches."""
    if samples_per_rank <= 0:
        return 0.0
    fwd, bwd = estimate_step_time(section, config, params, tokens_per_sample)
    m = math.ceil(samples_per_rank / config.mbs)
    return (m + config.pp - 1) * (fwd + bwd) / config.pp


@dataclass(frozen=True)
class MemoryEstimate:
    """Per-GPU bytes by component (costs.py:71-92)."""

    weights: float
    optimizer_state: float
    gradients: float
    activations: float

    @property
    def total(self) -> float:
        return self.weights + self.optimizer_state + self.gradients + self.activations

    def as_dict(self) -> dict[str, float]:
        return {"weights": self.weights, "optimizer_state": self.optimizer_state, "gradients": self.gradients,
                "activations": self.activations, "total": self.total}


def estimate_memory(section: SectionSpec, config: SectionConfig, params: CostParams,
                    tokens_per_sample: int) -> MemoryEstimate:
    """Per-GPU memory of one section under one config (costs.py:126-156): weights and optimizer
    state shard over tp*pp, activations over tp*cp; forward-only sections keep no optimizer state
    or gradients and at most ``live_microbatch_cap`` micro-batches of activations."""
    check_config(section, config)
    if tokens_per_sample <= 0:
        raise InvalidDims("tokens_per_sample must be positive")
    shard = config.tp * config.pp
    weights = section.structural.param_count * params.bytes_per_param_weights / shard
    if section.forward_only:
        opt = grads = 0.0
        live = min(config.mbs, params.live_microbatch_cap)
    else:
        opt = section.structural.param_count * params.bytes_per_param_optimizer / shard
        grads = weights
        live = float(config.mbs)
    act = live * tokens_per_sample * params.activation_bytes_per_token / (config.tp * config.cp)
    return MemoryEstimate(weights=weights, optimizer_state=opt, gradients=grads, activations=act)


def per_sample_times(section, config, params, tokens_per_sample, samples_per_rank):
    """Host twin of the device K1 arithmetic (costs.py:105-123, 182-200)."""
    if samples_per_rank <= 0:
        return 0.0, 0.0
    fwd, bwd = estimate_step_time(section, config, params, tokens_per_sample)
    m = math.ceil(samples_per_rank / config.mbs)
    scale = (m + config.pp - 1) / (m * config.pp * config.mbs)
    return fwd * scale, bwd * scale


# Row layout of the device cost table, one row per submodule bit (float64).
COST_COLS = ("flops_per_token_fwd", "effective", "bwd_fwd_ratio", "forward_only", "mbs", "pp", "dp", "owner")


def cost_table(graph: SectionGraph, configs: Mapping[str, SectionConfig],
               params_by_section: Mapping[str, CostParams],
               params_by_submodule: Mapping[str, CostParams] | None = None) -> np.ndarray:
    """Lower cost knobs to a ``[n_bits, 8]`` float64 table indexed by submodule bit.

    Merged exclusive encoders keep one config but may carry per-submodule
    ``CostParams`` (``params_by_submodule``), since a sample's time in the
    merged section is whichever submodule it activates (workload.py:520-523).
    """
    tab = graph.tables
    out = np.zeros((len(tab.sub_names), len(COST_COLS)), dtype=np.float64)
    for bit, name in enumerate(tab.sub_names):
        owner = tab.sub_owner[bit]
        sid = tab.section_ids[owner]
        spec, cfg = graph.section(sid), configs[sid]
        params = (params_by_submodule or {}).get(name) or params_by_section[sid]
        check_config(spec, cfg)
        out[bit] = (
            params.flops_per_token_fwd,
            effective_rate(cfg, params),
            params.bwd_fwd_ratio,
            1.0 if spec.forward_only else 0.0,
            cfg.mbs,
            cfg.pp,
            cfg.dp,
            owner,
        )
    return out


# --- batch synthesis (host; costs.py:206-299) ----------------------------------------------------


@dataclass(frozen=True)
class BatchProfile:
    """Statistical description of a global batch (costs.py:206-227): ``shares`` = fraction of
    samples activating each auxiliary, ``tokens`` = tokens per sample per section (default:
    the section's max_seq_len)."""

    global_batch_size: int
    shares: Mapping[str, float] = field(default_factory=dict)
    tokens: Mapping[str, int] = field(default_factory=dict)

    def __post_init__(self) -> None:
        from .errors import EmptyBatch

        if self.global_batch_size < 1:
            raise EmptyBatch("global_batch_size must be positive")
        for sid, share in self.shares.items():
            if not 0 <= share <= 1:
                raise InvalidDims(f"share for '{sid}' must lie in [0,1]", section=sid)

    def tokens_for(self, section: SectionSpec) -> int:
        return int(self.tokens.get(section.id, section.structural.max_seq_len))


def derive_batch(graph: SectionGraph, configs: Mapping[str, SectionConfig],
                 params_by_section: Mapping[str, CostParams], profile: BatchProfile, seed: int = 0):
    """Synthesise a global batch of 6-tuples from the cost model (costs.py:230-299).

    Host-side planning input, identical to the reference: membership of each auxiliary is the
    rounded share of the batch chosen by ``random.Random(seed)`` shuffles (the reference's own
    generator, so a given seed yields the same batch); per-sample times come from
    :func:`per_sample_times` at the rank's sample count, summed per side.  The device step path
    never uses this generator (its batches come from the token counts, csrc/plan.cu K1)."""
    import random

    from .workload import SampleTiming, Side

    crit = graph.critical
    b = profile.global_batch_size
    rng = random.Random(seed)
    member = {}
    for aux in graph.auxiliaries:
        count = min(b, round(profile.shares.get(aux.id, 0.0) * b))
        ids = list(range(b))
        rng.shuffle(ids)
        member[aux.id] = set(ids[:count])
    times = {crit.id: per_sample_times(crit, configs[crit.id], params_by_section[crit.id], profile.tokens_for(crit),
                                       math.ceil(b / configs[crit.id].dp))}
    for aux in graph.auxiliaries:
        n = len(member[aux.id])
        times[aux.id] = per_sample_times(aux, configs[aux.id], params_by_section[aux.id], profile.tokens_for(aux),
                                         math.ceil(n / configs[aux.id].dp) if n else 0)
    out = []
    fwd_c, bwd_c = times[crit.id]
    for i in range(b):
        up_f = up_b = down_f = down_b = 0.0
        act = set()
        for aux in graph.auxiliaries:
            if i not in member[aux.id]:
                continue
            f, bw = times[aux.id]
            if graph.side(aux.id) is Side.UPSTREAM:
                up_f += f
                up_b += bw
            else:
                down_f += f
                down_b += bw
            act.add(aux.id)
        out.append(SampleTiming(sample_id=i, t_f_bc=up_f, t_f_c=fwd_c, t_f_ac=down_f, t_b_bc=down_b, t_b_c=bwd_c,
                                t_b_ac=up_b, activated_sections=frozenset(act)))
    return out


# --- shipped presets (costs.py:300-373) --------------------------------------------------------
# The reference's calibrations of its documented workload archetypes, used by `maestro-spec v1`
# files (`cost: {preset: ...}`).  They assume 3e14 FLOP/s per GPU; planner.fit_cost_params
# replaces that with B200-measured rates.


def _eff(*rows):
    return {tuple(r[:3]): r[3] for r in rows}


PRESETS: dict[str, CostParams] = {
    "vit-encoder": CostParams(
        flops_per_token_fwd=2.4e9, peak_flops_per_gpu=3.0e14, bwd_fwd_ratio=2.0,
        parallel_efficiency=_eff((1, 1, 2, 0.97), (1, 1, 4, 0.93), (1, 1, 8, 0.88), (1, 1, 16, 0.80),
                                 (2, 1, 1, 0.95), (2, 1, 2, 0.92), (2, 1, 4, 0.88), (4, 1, 1, 0.90)),
        bytes_per_param_weights=2.0, bytes_per_param_optimizer=12.0, activation_bytes_per_token=4096.0),
    "moe-backbone": CostParams(
        flops_per_token_fwd=3.4e10, peak_flops_per_gpu=3.0e14, bwd_fwd_ratio=2.0,
        parallel_efficiency=_eff((2, 1, 1, 0.96), (4, 1, 1, 0.92), (8, 1, 1, 0.85), (2, 2, 1, 0.93),
                                 (4, 2, 1, 0.89), (4, 4, 1, 0.84), (8, 2, 1, 0.82), (8, 4, 1, 0.78),
                                 (2, 1, 2, 0.92), (4, 1, 2, 0.88), (2, 2, 2, 0.89)),
        bytes_per_param_weights=2.0, bytes_per_param_optimizer=12.0, activation_bytes_per_token=24576.0),
    "frozen-teacher": CostParams(
        flops_per_token_fwd=5.6e10, peak_flops_per_gpu=3.0e14, bwd_fwd_ratio=2.0,
        parallel_efficiency=_eff((2, 1, 1, 0.96), (4, 1, 1, 0.92), (8, 1, 1, 0.86), (2, 2, 1, 0.93),
                                 (4, 2, 1, 0.88), (1, 1, 2, 0.93), (1, 1, 4, 0.88), (2, 1, 2, 0.90)),
        mbs_efficiency={1: 0.35, 2: 0.62, 3: 0.80, 4: 0.91, 8: 1.0},
        bytes_per_param_weights=2.0, bytes_per_param_optimizer=0.0, activation_bytes_per_token=1024.0),
}


def preset(name: str) -> CostParams:
    """A shipped preset by name; unknown names raise InvalidDims listing the known ones."""
    if name not in PRESETS:
        raise InvalidDims(f"unknown cost preset '{name}' (known: {', '.join(sorted(PRESETS))})", preset=name)
    return PRESETS[name]
