"""Launch accounting and per-kernel device timing (used by bench.py; off by default).

``launches`` counts kernel launches made through our C ABI (the driver cross-checks this
against the .so files actually loaded).  When timing is on (``start_timing``), the host
wrappers record (work, start_event, end_event) around every launch of a timed kind on the
launching stream: "gemm" (tcgen05 GEMM, work = 2MNK FLOPs), "attn_fwd" / "attn_bwd"
(work = algorithmic FLOPs when the caller states them, else 0) and "kd_loss" (work =
algorithmic bytes).  bench.py turns timing on only for a separate, serialised step outside the
headline timed region, so the events never perturb the measured throughput and the per-kernel
durations do not overlap (their sum is at most the step time).
"""

from __future__ import annotations

launches = 0
timing = None          # kind -> list of (work, e0, e1) while on
gemm_timing = None     # legacy alias: list of GEMM records while timing is on

# kernels launched per C-ABI call (default 1)
KERNELS_PER_CALL = {"build_schedule": 3}


def count(what: str) -> None:
    global launches
    launches += KERNELS_PER_CALL.get(what, 1)


def begin(kind: str, work: float = 0.0):
    """Start a timed launch of ``kind`` on the current stream (None when timing is off)."""
    if timing is None:
        return None
    import torch

    e0 = torch.cuda.Event(enable_timing=True)
    e0.record()
    return (kind, work, e0)


def end(tok) -> None:
    if tok is None or timing is None:
        return
    import torch

    kind, work, e0 = tok
    e1 = torch.cuda.Event(enable_timing=True)
    e1.record()
    timing.setdefault(kind, []).append((work, e0, e1))


def start_timing() -> None:
    global timing, gemm_timing
    timing = {}
    gemm_timing = timing.setdefault("gemm", [])


def stop_timing() -> dict:
    """-> {kind: (total work, total device ms, launches)} of the recorded launches."""
    global timing, gemm_timing
    rec, timing, gemm_timing = timing or {}, None, None
    return {k: (sum(w for w, _, _ in v), sum(a.elapsed_time(b) for _, a, b in v), len(v)) for k, v in rec.items()}


def start_gemm_timing() -> None:
    start_timing()


def stop_gemm_timing():
    """-> (total algorithmic FLOPs, total device ms, launches) of the recorded GEMMs."""
    return stop_timing().get("gemm", (0.0, 0.0, 0))
