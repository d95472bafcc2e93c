"""Counter-based synthetic batch generator (splitmix64).

The reference synthesises batches with ``random.Random`` (costs.py:245-253),
which cannot be reproduced on a device.  Every synthetic input of this repo
(modality mix, text lengths, image-placeholder offsets, token ids) is instead
a pure function of ``(seed, stream, index)`` through the splitmix64 finaliser,
implemented identically here (numpy, vectorised) and in
``csrc/common.cuh`` (``mix64``), so host and device draw the same values.
"""

from __future__ import annotations

import numpy as np

_M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
STREAM_MUL = 0xD1B54A32D192ED03


def mix64(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def rand_u64(seed: int, stream: int, index) -> np.ndarray:
    """splitmix64(seed*golden + stream*mul + index + 1), element-wise over ``index``."""
    base = (seed * GOLDEN + stream * STREAM_MUL + 1) & _M64
    idx = np.asarray(index, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return mix64(idx + np.uint64(base))


def rand_int(seed: int, stream: int, index, lo: int, hi: int) -> np.ndarray:
    """Integers in [lo, hi] (inclusive; modulo draw, deterministic)."""
    span = np.uint64(hi - lo + 1)
    return (rand_u64(seed, stream, index) % span).astype(np.int64) + lo


def permutation(seed: int, stream: int, n: int) -> np.ndarray:
    """Seeded permutation of range(n): argsort of per-index random keys (stable)."""
    return np.argsort(rand_u64(seed, stream, np.arange(n)), kind="stable")


# Streams (keep fixed: golden fixtures depend on them)
S_MODALITY, S_TEXT_LEN, S_IMG_OFFSET, S_TOKENS, S_PIXELS, S_WEIGHTS = 1, 2, 3, 4, 5, 6


def vlm_batch(seed: int, batch: int, text_lo: int = 64, text_hi: int = 448, image_frac: float = 0.5,
              max_offset: int = 16):
    """Modality mix + lengths of the tiny-VLM config (SURVEY §8d cfg 1).

    Returns dict with ``has_image`` (bool[B], exactly round(frac*B) images
    chosen by a seeded permutation), ``text_len`` (int[B], U{lo..hi}) and
    ``img_offset`` (int[B], text tokens before the image placeholders).
    """
    n_img = int(round(image_frac * batch))
    perm = permutation(seed, S_MODALITY, batch)
    has_image = np.zeros(batch, dtype=bool)
    has_image[perm[:n_img]] = True
    text_len = rand_int(seed, S_TEXT_LEN, np.arange(batch), text_lo, text_hi)
    off = rand_int(seed, S_IMG_OFFSET, np.arange(batch), 0, max_offset)
    img_offset = np.where(has_image, np.minimum(off, text_len), 0)
    return {"has_image": has_image, "text_len": text_len.astype(np.int32), "img_offset": img_offset.astype(np.int32)}


def token_ids(seed: int, stream_offset: int, n: int, vocab: int) -> np.ndarray:
    return rand_int(seed, S_TOKENS + 16 * stream_offset, np.arange(n), 0, vocab - 1).astype(np.int32)
