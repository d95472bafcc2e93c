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


# ----------------------------------------------------------------------------- cfg 3
QWEN_VIT_PARAMS = 630_000_000
QWEN_LLM_PARAMS = 7_600_000_000


def vlm_7b_graph() -> SectionGraph:
    vit = SectionSpec("vit", Role.AUXILIARY, ExecMode.FORWARD_BACKWARD,
                      StructuralParams(1280, 16, 32, 1, 16384, QWEN_VIT_PARAMS))
    llm = SectionSpec("llm", Role.CRITICAL, ExecMode.FORWARD_BACKWARD,
                      StructuralParams(3584, 28, 28, 152064, 8192, QWEN_LLM_PARAMS))
    return build_graph([vit, llm], [Edge("vit", "llm", 1024 * 3584 * 2.0)])


VLM7B_LAYOUTS = {1: (1, 1, 1), 2: (1, 1, 1), 4: (3, 1, 3), 8: (7, 1, 7)}


def vlm_7b(n_gpus: int = 8, batch: int = 64, seed: int = 0) -> Recipe:
    """cfg 3: Qwen2.5-VL-7B-shaped VLM; 50 % images with U{256..4096} patches (2x2 merge -> /4)."""
    from .synthetic import rand_int

    g = vlm_7b_graph()
    dp_llm, dp_vit, f_vit = VLM7B_LAYOUTS[n_gpus]
    configs = {"llm": SectionConfig(dp=dp_llm), "vit": SectionConfig(dp=dp_vit, fanout=f_vit)}
    params = {
        "vit": CostParams(flops_per_token_fwd=2.0 * QWEN_VIT_PARAMS, peak_flops_per_gpu=B200_PEAK_FLOPS),
        "llm": CostParams(flops_per_token_fwd=2.0 * QWEN_LLM_PARAMS, peak_flops_per_gpu=B200_PEAK_FLOPS),
    }
    b = vlm_batch(seed, batch, text_lo=256, text_hi=2048)
    patches = rand_int(seed, 7, np.arange(batch), 256, 4096).astype(np.int32) // 4 * 4
    vit_tokens = np.where(b["has_image"], patches, 0)
    llm_tokens = b["text_len"] + vit_tokens // 4
    return Recipe("vlm_7b", g, configs, params,
                  {"llm": llm_tokens.astype(np.int32), "vit": vit_tokens.astype(np.int32)}, batch, dict(b))


# ----------------------------------------------------------------------------- cfg 4
def omni_graph(parallel_upstream: bool = False) -> SectionGraph:
    img = SectionSpec("image_enc", Role.AUXILIARY, ExecMode.FORWARD_BACKWARD,
                      StructuralParams(1280, 16, 32, 1, 16384, QWEN_VIT_PARAMS))
    aud = SectionSpec("audio_enc", Role.AUXILIARY, ExecMode.FORWARD_BACKWARD,
                      StructuralParams(1280, 20, 32, 1, 1500, 640_000_000))
    llm = SectionSpec("llm", Role.CRITICAL, ExecMode.FORWARD_BACKWARD,
                      StructuralParams(3584, 28, 28, 152064, 8192, QWEN_LLM_PARAMS))
    dec = SectionSpec("audio_dec", Role.AUXILIARY, ExecMode.FORWARD_BACKWARD,
                      StructuralParams(1024, 16, 12, 4096, 4096, 300_000_000))
    return build_graph([img, aud, llm, dec], [Edge("image_enc", "llm", 1024 * 3584 * 2.0),
                                             Edge("audio_enc", "llm", 375 * 3584 * 2.0),
                                             Edge("llm", "audio_dec", 512 * 3584 * 2.0)],
                       parallel_upstream=parallel_upstream)


OMNI_LAYOUTS = {1: (1, 1, 1), 2: (2, 1, 2), 4: (4, 2, 2), 8: (8, 2, 4)}


def omni(n_gpus: int = 8, batch: int = 64, seed: int = 0, mix: str = "4way",
         parallel_upstream: bool = False) -> Recipe:
    """cfg 4: image + audio encoders (upstream), 7B backbone, audio decoder (downstream).

    mix "4way" = text / img / audio / img+audio in equal shares.  The img+audio class activates
    two upstream sections; the reference's 6-tuple model rejects it (ActivationError,
    workload.py:323-328) and so does the device resolver -- that is the parity-pinned behaviour.
    mix "3way" drops that class (text / img / audio) and schedules.  Audio samples also run the
    downstream audio decoder on 512 generated tokens.  ``parallel_upstream=True`` switches on this
    build's generalisation (workload.SectionGraph.parallel_upstream): the img+audio class runs
    both encoders in parallel and schedules with t_f_bc = max of the two.
    """
    from .synthetic import permutation

    g = omni_graph(parallel_upstream)
    dp_llm, dp_enc, f_enc = OMNI_LAYOUTS[n_gpus]
    configs = {"llm": SectionConfig(dp=dp_llm), "image_enc": SectionConfig(dp=dp_enc, fanout=f_enc),
               "audio_enc": SectionConfig(dp=dp_enc, fanout=f_enc), "audio_dec": SectionConfig(dp=dp_llm)}
    params = {
        "image_enc": CostParams(flops_per_token_fwd=2.0 * QWEN_VIT_PARAMS, peak_flops_per_gpu=B200_PEAK_FLOPS),
        "audio_enc": CostParams(flops_per_token_fwd=2.0 * 640_000_000, peak_flops_per_gpu=B200_PEAK_FLOPS),
        "llm": CostParams(flops_per_token_fwd=2.0 * QWEN_LLM_PARAMS, peak_flops_per_gpu=B200_PEAK_FLOPS),
        "audio_dec": CostParams(flops_per_token_fwd=2.0 * 300_000_000, peak_flops_per_gpu=B200_PEAK_FLOPS),
    }
    classes = 4 if mix == "4way" else 3
    perm = permutation(seed, 9, batch)
    cls = np.empty(batch, dtype=np.int64)
    cls[perm] = np.arange(batch) % classes  # 0 text, 1 img, 2 audio, 3 img+audio
    b = vlm_batch(seed, batch, text_lo=256, text_hi=2048)
    img = (cls == 1) | (cls == 3)
    aud = (cls == 2) | (cls == 3)
    img_tok = np.where(img, 4096, 0)
    aud_tok = np.where(aud, 1500, 0)
    llm_tok = b["text_len"] + img_tok // 4 + aud_tok // 4
    dec_tok = np.where(aud, 512, 0)
    return Recipe("omni", g, configs, params,
                  {"llm": llm_tok.astype(np.int32), "image_enc": img_tok.astype(np.int32),
                   "audio_enc": aud_tok.astype(np.int32), "audio_dec": dec_tok.astype(np.int32)},
                  batch, {"class": cls})


# ----------------------------------------------------------------------------- cfg 5
def kd_8b_graph() -> SectionGraph:
    teacher = SectionSpec("teacher", Role.AUXILIARY, ExecMode.FORWARD_ONLY,
                          StructuralParams(4096, 32, 32, 128256, 8192, 8_000_000_000),
                          submodules=("teacher", "output_layer"))
    student = SectionSpec("student", Role.CRITICAL, ExecMode.FORWARD_BACKWARD,
                          StructuralParams(2048, 32, 16, 128256, 8192, 1_240_000_000))
    g = build_graph([teacher, student], [Edge("teacher", "student", 8192 * 128256 * 2.0)])
    return colocate_output_layer(g, "teacher", "student", 4096, 128256)


KD8B_LAYOUTS = {1: (1, 1, 1), 2: (1, 1, 1), 4: (2, 2, 1), 8: (4, 4, 1)}


def kd_8b(n_gpus: int = 8, batch: int = 32, seq: int = 8192, layout: str = "disjoint") -> Recipe:
    """cfg 5: Llama-3-8B teacher -> Llama-3.2-1B student, 8k seq, disjoint GPU groups (the
    co-located layout puts a teacher and a student rank on every GPU, as for cfg 2)."""
    g = kd_8b_graph()
    if layout == "colocated" or n_gpus == 1:
        dp_s, dp_t, f_t = n_gpus, n_gpus, 1
    else:
        dp_s, dp_t, f_t = KD8B_LAYOUTS[n_gpus]
    configs = {"student": SectionConfig(dp=dp_s), "teacher": SectionConfig(dp=dp_t, fanout=f_t)}
    params = {
        "teacher": CostParams(flops_per_token_fwd=2.0 * 7.5e9 + 4 * 32 * 4096 * seq / 2,
                              peak_flops_per_gpu=B200_PEAK_FLOPS),
        "student": CostParams(flops_per_token_fwd=2.0 * (0.97e9 + 4096 * 128256) + 4 * 16 * 2048 * seq / 2,
                              peak_flops_per_gpu=B200_PEAK_FLOPS),
    }
    tokens = {"student": np.full(batch, seq, np.int32), "teacher": np.full(batch, seq, np.int32)}
    return Recipe("kd_8b", g, configs, params, tokens, batch, {})


RECIPES = {"vlm_tiny": vlm_tiny, "kd": kd, "vlm_7b": vlm_7b, "omni": omni, "kd_8b": kd_8b}
