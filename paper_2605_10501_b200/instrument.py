"""Launch accounting and per-GEMM device timing (used by bench.py; off by default).

``launches`` counts kernel launches made through our C ABI (the driver cross-checks this
against the .so files actually loaded).  When ``gemm_timing`` is a list, dense.gemm records
(flops, start_event, end_event) around every tcgen05 GEMM on the launching stream, so the
bench can report the dominant kernel's achieved TFLOP/s from CUDA events inside the timed
region.
"""

from __future__ import annotations

launches = 0
gemm_timing = None

# kernels launched per C-ABI call (default 1)
KERNELS_PER_CALL = {"build_schedule": 3}


def count(what: str) -> None:
    global launches
    launches += KERNELS_PER_CALL.get(what, 1)


def start_gemm_timing() -> None:
    global gemm_timing
    gemm_timing = []


def stop_gemm_timing():
    """-> (total algorithmic FLOPs, total device ms, launches) of the recorded GEMMs."""
    global gemm_timing
    rec, gemm_timing = gemm_timing or [], None
    flops = sum(f for f, _, _ in rec)
    ms = sum(a.elapsed_time(b) for _, a, b in rec)
    return flops, ms, len(rec)
