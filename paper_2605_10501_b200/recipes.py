"""Section graphs, layouts and cost knobs of the BASELINE.json configs.

Each recipe builds the section graph through the public construction API
(workload.py mirror), picks per-section ``SectionConfig``s for a GPU count,
and describes the per-sample token counts the device 6-tuple kernel (K1)
consumes.  Model shapes are in :mod:`.transformer` (``SHAPES``).

cfg 1  tiny VLM: ViT-tiny encoder (upstream) -> 2-layer GPT backbone (critical)
cfg 2  KD: forward-only 1.1B teacher (upstream) -> 125M student (critical),
       teacher output layer colocated with the student (workload.py:471-514)
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .costs import CostParams
from .synthetic import vlm_batch
from .workload import (
    Edge,
    ExecMode,
    Role,
    SectionConfig,
    SectionGraph,
    SectionSpec,
    StructuralParams,
    build_graph,
    colocate_output_layer,
)

# peak used by the cost model: measured bf16 burst peak of this pool's B200 (MEASURED_PEAKS.json)
B200_PEAK_FLOPS = 1.6381e15


@dataclass(frozen=True)
class Recipe:
    name: str
    graph: SectionGraph
    configs: dict
    params: dict
    #: per-sample tokens per submodule-bit name: name -> int[B]
    tokens: dict
    batch: int
    extra: dict


# ----------------------------------------------------------------------------- cfg 1
VIT_PATCHES = 196          # 224^2 / 16^2
VIT_MERGED = 49            # 2x2 patch merge -> LLM tokens per image


def vlm_tiny_graph() -> SectionGraph:
    vit = SectionSpec("vit", Role.AUXILIARY, ExecMode.FORWARD_BACKWARD,
                      StructuralParams(192, 3, 12, 1, VIT_PATCHES, 5_300_000))
    llm = SectionSpec("llm", Role.CRITICAL, ExecMode.FORWARD_BACKWARD,
                      StructuralParams(768, 12, 2, 32768, 512, 64_500_000))
    return build_graph([vit, llm], [Edge("vit", "llm", VIT_MERGED * 768 * 2)])


VLM_LAYOUTS = {
    # n_gpus -> (llm dp, vit dp, vit fanout); 1 GPU = both sections co-resident
    1: (1, 1, 1),
    2: (1, 1, 1),
    4: (3, 1, 3),
    8: (6, 2, 3),
}


def vlm_tiny(n_gpus: int = 1, batch: int = 64, seed: int = 0) -> Recipe:
    g = vlm_tiny_graph()
    dp_llm, dp_vit, f_vit = VLM_LAYOUTS[n_gpus]
    configs = {"llm": SectionConfig(dp=dp_llm), "vit": SectionConfig(dp=dp_vit, fanout=f_vit)}
    params = {
        "vit": CostParams(flops_per_token_fwd=1.1e7, peak_flops_per_gpu=B200_PEAK_FLOPS),
        "llm": CostParams(flops_per_token_fwd=7.9e7, peak_flops_per_gpu=B200_PEAK_FLOPS),
    }
    b = vlm_batch(seed, batch)
    llm_tokens = b["text_len"] + np.where(b["has_image"], VIT_MERGED, 0)
    vit_tokens = np.where(b["has_image"], VIT_PATCHES, 0)
    return Recipe("vlm_tiny", g, configs, params,
                  {"llm": llm_tokens.astype(np.int32), "vit": vit_tokens.astype(np.int32)},
                  batch, dict(b))


# ----------------------------------------------------------------------------- cfg 2
KD_SEQ = 2048
KD_VOCAB = 32000
KD_TEACHER_HIDDEN = 2048


def kd_graph() -> SectionGraph:
    teacher = SectionSpec("teacher", Role.AUXILIARY, ExecMode.FORWARD_ONLY,
                          StructuralParams(KD_TEACHER_HIDDEN, 32, 22, KD_VOCAB, KD_SEQ, 1_100_000_000),
                          submodules=("teacher", "output_layer"))
    student = SectionSpec("student", Role.CRITICAL, ExecMode.FORWARD_BACKWARD,
                          StructuralParams(768, 12, 12, KD_VOCAB, KD_SEQ, 125_000_000))
    g = build_graph([teacher, student], [Edge("teacher", "student", KD_SEQ * KD_VOCAB * 2.0)])
    return colocate_output_layer(g, "teacher", "student", KD_TEACHER_HIDDEN, KD_VOCAB)


KD_LAYOUTS = {
    # disjoint GPU groups: n_gpus -> (student dp, teacher dp, teacher fanout); teacher ranks first
    1: (1, 1, 1),
    2: (1, 1, 1),
    4: (2, 2, 1),
    8: (4, 4, 1),
}


def kd_layout(n_gpus: int, layout: str = "colocated"):
    """(student dp, teacher dp, teacher fanout, colocated?) for a GPU count.

    "colocated": every GPU hosts one teacher and one student DP rank (handoff = CUDA event);
    "disjoint":  teacher and student on disjoint GPU groups (handoff = NCCL send/recv).
    The teacher is ~70% of the per-sample FLOPs, so with equal GPUs the disjoint split is
    teacher-bound and the colocated layout is the throughput-optimal plan on one node.
    """
    if layout == "colocated" or n_gpus == 1:
        return n_gpus, n_gpus, 1, True
    dp_s, dp_t, f = KD_LAYOUTS[n_gpus]
    return dp_s, dp_t, f, False


def kd(n_gpus: int = 1, batch: int = 64, seq: int = KD_SEQ, layout: str = "disjoint") -> Recipe:
    g = kd_graph()
    dp_s, dp_t, f_t, _ = kd_layout(n_gpus, layout)
    configs = {"student": SectionConfig(dp=dp_s), "teacher": SectionConfig(dp=dp_t, fanout=f_t)}
    # fwd FLOPs per token ~ 2 * params (+ attention); student includes the colocated teacher head
    params = {
        "teacher": CostParams(flops_per_token_fwd=2.0 * 0.97e9 + 4 * 22 * 2048 * seq / 2,
                              peak_flops_per_gpu=B200_PEAK_FLOPS),
        "student": CostParams(flops_per_token_fwd=2.0 * (1.13e8 + 2048 * KD_VOCAB) + 4 * 12 * 768 * seq / 2,
                              peak_flops_per_gpu=B200_PEAK_FLOPS),
    }
    tokens = {"student": np.full(batch, seq, np.int32), "teacher": np.full(batch, seq, np.int32)}
    return Recipe("kd", g, configs, params, tokens, batch, {})


RECIPES = {"vlm_tiny": vlm_tiny, "kd": kd}
