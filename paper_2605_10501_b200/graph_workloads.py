"""Section graphs of BASELINE configs 3 and 4 (and KD) for the generic executor (graph_exec).

cfg 3  Qwen2.5-VL-7B shape: ViT (d 1280, 32 layers, 16 heads of 80 -> zero-padded 128-wide heads,
       SwiGLU 3420 -> padded 3456, 14x14 patches of 3*14*14 = 588 values padded to 640, 2x2
       merge = 4 consecutive patches) upstream of a Qwen2.5-7B-shaped backbone (d 3584, 28
       layers, GQA 28/4, head_dim 128, SwiGLU 18944, V 152064); 50 % images with U{256..4096}
       patches (recipes.vlm_7b).
cfg 4  omni: image encoder (the cfg 3 ViT) + audio encoder (Whisper-large-v3-encoder shape:
       d 1280, 32 layers, 20 heads of 64, 1500 frames of 128 mel bins, 4:1 -> 375 tokens)
       upstream, the 7B backbone, and an audio decoder downstream (d 1024, 12 layers, 16 heads,
       4096 audio codes) on the backbone's last 512 positions of audio samples; mix text / img /
       audio / img+audio (recipes.omni "4way"; the img+audio class activates two upstream
       sections, scheduled with this build's parallel-upstream generalisation).

``layers`` scales every stack's depth (reduced-depth runs keep the widths and sequence shapes:
one GPU cannot hold a 7.6B model with fp32 master weights, gradients and Adam moments plus
activations; the graph, the schedule and every kernel shape are the full model's).
"""

from __future__ import annotations

import dataclasses

import numpy as np
import torch

from . import recipes as R
from .costs import CostParams
from .graph_exec import (BackboneModule, DecoderModule, DownInput, EncoderModule, GraphBatch, SectionGraphExecutor,
                         TeacherModule, UpInput)
from .synthetic import rand_int
from .transformer import SHAPES, Shape
from .workload import SectionConfig

QWEN_VIT = Shape(d=1280, layers=32, heads=16, kv_heads=16, ffn=3456, vocab=8, head_dim=128, causal=False,
                 head_dim_true=80, ffn_true=3420)
QWEN_7B = Shape(d=3584, layers=28, heads=28, kv_heads=4, ffn=18944, vocab=152064, head_dim=128, rope_base=1e6)
WHISPER_ENC = Shape(d=1280, layers=32, heads=20, kv_heads=20, ffn=5120, vocab=8, head_dim=64, causal=False)
AUDIO_DEC = Shape(d=1024, layers=12, heads=16, kv_heads=16, ffn=4096, vocab=4096)
PATCH_DIM = 640    # 3 * 14 * 14 = 588 pixel values, zero-padded to a 16-byte-multiple row
MEL_DIM = 128
MERGE = 4

# tiny stand-ins with the same structure (tests)
TINY_VIT = Shape(d=128, layers=2, heads=2, kv_heads=2, ffn=256, vocab=8, head_dim=128, causal=False,
                 head_dim_true=80, ffn_true=200)
TINY_LLM = Shape(d=256, layers=2, heads=4, kv_heads=2, ffn=512, vocab=1024, head_dim=64)
TINY_AUD = Shape(d=128, layers=2, heads=2, kv_heads=2, ffn=256, vocab=8, head_dim=64, causal=False)
TINY_DEC = Shape(d=128, layers=2, heads=2, kv_heads=2, ffn=256, vocab=64, head_dim=64)


def depth(shape: Shape, layers: int | None) -> Shape:
    return shape if layers is None else dataclasses.replace(shape, layers=layers)


def _costs(graph, shapes: dict, seq: dict) -> dict:
    """Cost knobs per section: 2 x params + attention per token (recipes' convention)."""
    out = {}
    for sid, sh in shapes.items():
        out[sid] = CostParams(flops_per_token_fwd=sh.fwd_flops_per_token(seq[sid], with_head=False),
                              peak_flops_per_gpu=R.B200_PEAK_FLOPS)
    return out


def vlm7b_batch(B: int, seed: int, vocab: int, patch_dim: int, lo: int = 256, hi: int = 4096,
                text_lo: int = 256, text_hi: int = 2048, step: int = 0) -> GraphBatch:
    """cfg 3 batch: recipes.vlm_7b's modality mix and lengths (50 % images, U{lo..hi} patches
    rounded to the 2x2 merge, text U{text_lo..text_hi}), placeholders inside the text."""
    from .synthetic import vlm_batch

    b = vlm_batch(seed, B, text_lo=text_lo, text_hi=text_hi)
    patches = rand_int(seed, 7, np.arange(B), lo, hi).astype(np.int64) // MERGE * MERGE
    in_len = np.where(b["has_image"], patches, 0)
    rows = in_len // MERGE
    tl = b["text_len"].astype(np.int64)
    off = np.minimum(b["img_offset"].astype(np.int64), tl)
    lens = tl + rows
    ids, labels = _text(B, lens, off, rows, seed, vocab, step)
    g = np.random.default_rng(seed + 100 + step)
    feats = (g.standard_normal((int(in_len.sum()), patch_dim)) * 0.5).astype(np.float32)
    if patch_dim > 588:
        feats[:, 588:] = 0.0  # pad columns of the 3*14*14 patch vector
    return GraphBatch(lens=lens, ids=ids, labels=labels,
                      up={"vit": UpInput(in_len=in_len, rows=rows, dst_off=np.where(rows > 0, off, 0), feats=feats)})


def _text(B, lens, off, rows, seed, vocab, step):
    Lmax = int(lens.max())
    ids = np.full((B, Lmax), -1, dtype=np.int32)
    labels = np.full((B, Lmax), -1, dtype=np.int32)
    toks = rand_int(seed + 977 * step, 4, np.arange(B * Lmax), 0, vocab - 1).astype(np.int32).reshape(B, Lmax)
    for i in range(B):
        L = int(lens[i])
        seq = toks[i, :L].copy()
        o, r = int(off[i]), int(rows[i])
        seq[o:o + r] = -1
        ids[i, :L] = seq
        nxt = np.concatenate([seq[1:], [-1]])
        labels[i, :L] = np.where((seq >= 0) & (nxt >= 0), nxt, -1)
    return ids, labels


def omni_batch(B: int, seed: int, vocab: int, patch_dim: int, n_codes: int, img_patches: int = 4096,
               frames: int = 1500, dec_rows: int = 512, text_lo: int = 256, text_hi: int = 2048,
               mix: str = "3way", step: int = 0) -> GraphBatch:
    """cfg 4 batch: recipes.omni's classes (0 text, 1 image, 2 audio[, 3 image+audio]): image
    samples carry img_patches patches (-> /4 tokens), audio samples `frames` mel frames (-> /4
    tokens) and their last `dec_rows` backbone positions feed the audio decoder."""
    from .synthetic import permutation, vlm_batch

    classes = 4 if mix == "4way" else 3
    perm = permutation(seed, 9, B)
    cls = np.empty(B, dtype=np.int64)
    cls[perm] = np.arange(B) % classes
    b = vlm_batch(seed, B, text_lo=text_lo, text_hi=text_hi)
    img, aud = (cls == 1) | (cls == 3), (cls == 2) | (cls == 3)
    in_img, in_aud = np.where(img, img_patches, 0), np.where(aud, frames, 0)
    r_img, r_aud = in_img // MERGE, in_aud // MERGE
    tl = b["text_len"].astype(np.int64)
    tl = np.maximum(tl, np.where(aud, dec_rows, 0))  # audio samples: the decoder reads their last dec_rows positions
    lens = tl + r_img + r_aud
    off_i = np.minimum(b["img_offset"].astype(np.int64), tl)
    off_a = off_i + r_img  # audio tokens follow the image tokens
    ids = np.full((B, int(lens.max())), -1, dtype=np.int32)
    labels = np.full_like(ids, -1)
    toks = rand_int(seed + 977 * step, 4, np.arange(B * ids.shape[1]), 0, vocab - 1).astype(np.int32)
    toks = toks.reshape(B, -1)
    for i in range(B):
        L = int(lens[i])
        seq = toks[i, :L].copy()
        seq[off_i[i]: off_i[i] + r_img[i]] = -1
        seq[off_a[i]: off_a[i] + r_aud[i]] = -1
        ids[i, :L] = seq
        nxt = np.concatenate([seq[1:], [-1]])
        labels[i, :L] = np.where((seq >= 0) & (nxt >= 0), nxt, -1)
    g = np.random.default_rng(seed + 200 + step)
    fi = (g.standard_normal((int(in_img.sum()), patch_dim)) * 0.5).astype(np.float32)
    if patch_dim > 588:
        fi[:, 588:] = 0.0
    fa = (g.standard_normal((int(in_aud.sum()), MEL_DIM)) * 0.5).astype(np.float32)
    dr = np.where(aud, dec_rows, 0)
    tg = rand_int(seed + 31 * step, 11, np.arange(int(dr.sum())), 0, n_codes - 1).astype(np.int32)
    return GraphBatch(
        lens=lens, ids=ids, labels=labels,
        up={"image_enc": UpInput(in_len=in_img, rows=r_img, dst_off=np.where(img, off_i, 0), feats=fi),
            "audio_enc": UpInput(in_len=in_aud, rows=r_aud, dst_off=np.where(aud, off_a, 0), feats=fa)},
        down={"audio_dec": DownInput(rows=dr, src_off=np.where(aud, lens - dec_rows, 0), targets=tg)})


def vlm7b_executor(n_gpus: int = 1, layers: int | None = None, tiny: bool = False, mbs_llm: int = 1,
                   mbs_vit: int = 4, seed: int = 0, lr: float = 3e-4, policy="interleaved", dp_group=None,
                   max_pos: int = 8192):
    vit = TINY_VIT if tiny else depth(QWEN_VIT, layers)
    llm = TINY_LLM if tiny else depth(QWEN_7B, layers)
    pd = 128 if tiny else PATCH_DIM
    graph = R.vlm_7b_graph()
    configs = {"llm": SectionConfig(dp=n_gpus, mbs=mbs_llm), "vit": SectionConfig(dp=n_gpus, mbs=mbs_vit)}
    dev = torch.device("cuda", torch.cuda.current_device())
    mods = {"vit": EncoderModule(vit, pd, llm.d, MERGE, dev, seed + 11, max_pos=max_pos),
            "llm": BackboneModule(llm, dev, seed + 10, max_pos=max_pos)}
    costs = _costs(graph, {"vit": vit, "llm": llm}, {"vit": 4096, "llm": 4096})
    ex = SectionGraphExecutor(graph, configs, mods, costs, policy=policy, lr=lr, dp_group=dp_group)
    ex.shapes = {"vit": vit, "llm": llm}
    ex.patch_dim = pd
    return ex


def omni_executor(n_gpus: int = 1, layers: int | None = None, tiny: bool = False, mbs_llm: int = 1,
                  mbs_enc: int = 4, seed: int = 0, lr: float = 3e-4, policy="interleaved", dp_group=None,
                  max_pos: int = 8192):
    vit = TINY_VIT if tiny else depth(QWEN_VIT, layers)
    aud = TINY_AUD if tiny else depth(WHISPER_ENC, layers)
    llm = TINY_LLM if tiny else depth(QWEN_7B, layers)
    dec = TINY_DEC if tiny else depth(AUDIO_DEC, layers)
    pd = 128 if tiny else PATCH_DIM
    graph = R.omni_graph(parallel_upstream=True)  # img+audio samples: both encoders, in parallel
    configs = {"llm": SectionConfig(dp=n_gpus, mbs=mbs_llm), "image_enc": SectionConfig(dp=n_gpus, mbs=mbs_enc),
               "audio_enc": SectionConfig(dp=n_gpus, mbs=mbs_enc), "audio_dec": SectionConfig(dp=n_gpus, mbs=mbs_llm)}
    dev = torch.device("cuda", torch.cuda.current_device())
    mods = {"image_enc": EncoderModule(vit, pd, llm.d, MERGE, dev, seed + 11, max_pos=max_pos),
            "audio_enc": EncoderModule(aud, MEL_DIM, llm.d, MERGE, dev, seed + 12, max_pos=max_pos),
            "llm": BackboneModule(llm, dev, seed + 10, max_pos=max_pos),
            "audio_dec": DecoderModule(dec, llm.d, dev, seed + 13, max_pos=max_pos)}
    costs = _costs(graph, {"image_enc": vit, "audio_enc": aud, "llm": llm, "audio_dec": dec},
                   {"image_enc": 4096, "audio_enc": 1500, "llm": 4096, "audio_dec": 512})
    ex = SectionGraphExecutor(graph, configs, mods, costs, policy=policy, lr=lr, dp_group=dp_group)
    ex.shapes = {"image_enc": vit, "audio_enc": aud, "llm": llm, "audio_dec": dec}
    ex.patch_dim = pd
    return ex


def kd_executor(teacher: str = "test_tiny", student: str = "test_tiny", n_gpus: int = 1, mbs: int = 2,
                teacher_mbs: int = 2, seed: int = 0, lr: float = 3e-4, seq: int = 2048, policy="interleaved",
                dp_group=None):
    """The KD graph (recipes.kd_graph: teacher -> student, teacher head colocated with the student)
    on the generic executor, with KDExecutor's parameter seeds (tests compare the two)."""
    ts, ss = SHAPES[teacher], SHAPES[student]
    graph = R.kd_graph()
    configs = {"student": SectionConfig(dp=n_gpus, mbs=mbs), "teacher": SectionConfig(dp=n_gpus, mbs=teacher_mbs)}
    dev = torch.device("cuda", torch.cuda.current_device())
    g = torch.Generator(device=dev).manual_seed(seed + 3)
    t_head = (torch.randn(ts.vocab, ts.d, device=dev, generator=g) * 0.02).bfloat16()
    mods = {"teacher": TeacherModule(ts, dev, seed + 1, max_pos=seq),
            "student": BackboneModule(ss, dev, seed + 2, loss="kd", t_head=t_head, max_pos=seq)}
    costs = R.kd(n_gpus, 64, seq, "colocated").params
    ex = SectionGraphExecutor(graph, configs, mods, costs, policy=policy, lr=lr, dp_group=dp_group)
    ex.shapes = {"teacher": ts, "student": ss}
    return ex


def kd_batch(ids: np.ndarray) -> GraphBatch:
    """Text-only KD batch: every sample activates the teacher with its full sequence."""
    B, L = ids.shape
    lens = np.full(B, L, dtype=np.int64)
    return GraphBatch(lens=lens, ids=ids.astype(np.int32), labels=None,
                      up={"teacher": UpInput(in_len=lens.copy(), rows=lens.copy(), dst_off=np.zeros(B, np.int64))})
