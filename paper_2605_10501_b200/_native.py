"""ctypes binding of the C ABI (``include/maestro_b200.h``) + device error decoding.

The native library is mandatory: importing a compute entry point without it
raises :class:`NativeError` (there is no CPU fallback anywhere in the
product).  Device buffers are torch tensors (torch owns allocations and
streams); kernels receive raw pointers and the current CUDA stream.
"""

from __future__ import annotations

import ctypes
from pathlib import Path

from . import errors as E
from . import instrument as _instrument
from .workload import MAX_SECTIONS, SectionConfig, SectionGraph

import os as _os

# MAESTRO_LIB_PATH: an alternative build of the same library (scripts/build_variant.py, kernel A/B
# experiments); the default is the in-tree build
LIB_PATH = Path(_os.environ.get("MAESTRO_LIB_PATH") or Path(__file__).resolve().parent / "_lib" / "libmaestro_b200.so")
MAX_DP = 64
MAX_BATCH = 4096
MAX_RANK_SAMPLES = 1023
ERR_CLEAN = 0x7FFFFFFFFFFFFFFF

_lib = None


class GraphStruct(ctypes.Structure):
    """maestro_graph_t (include/maestro_b200.h)."""

    S = MAX_SECTIONS
    _fields_ = [
        ("n_sections", ctypes.c_int32),
        ("n_bits", ctypes.c_int32),
        ("critical", ctypes.c_int32),
        ("n_up", ctypes.c_int32),
        ("n_down", ctypes.c_int32),
        ("n_aux", ctypes.c_int32),
        ("sub_owner", ctypes.c_int32 * 32),
        ("side", ctypes.c_int32 * S),
        ("up_cand", ctypes.c_int32 * S),
        ("down_cand", ctypes.c_int32 * S),
        ("neighbor", ctypes.c_int32 * S),
        ("merge_order", ctypes.c_int32 * S),
        ("dp", ctypes.c_int32 * S),
        ("fanout", ctypes.c_int32 * S),
        ("mbs", ctypes.c_int32 * S),
        ("sec_bits", ctypes.c_uint32 * S),
        ("crit_bit", ctypes.c_int32),
        ("par_up", ctypes.c_int32),
    ]


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise E.NativeError(
            f"native library {LIB_PATH} is missing; run `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    L = ctypes.CDLL(str(LIB_PATH))
    P, I32, I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    G = ctypes.POINTER(GraphStruct)
    sig = {
        "maestro_error_reset": [P, P],
        "maestro_sample_times": [G, P, P, I32, P, P, P, P],
        "maestro_partition": [G, P, P, P, I32, P, P, P, P, P, P, P],
        "maestro_wavefront": [P, I32, P, P, I32, I32, P, P, P, P],
        "maestro_rank_metrics": [P, I32, P, I32, I32, P, P],
        "maestro_fanout_merge": [G, I32, P, P, P, P, P, P],
        "maestro_build_schedule": [G, P, P, P, I32, I32, P, P, P, P, P, P, P],
        "maestro_varlen_pack": [P, I32, P, I32, P, P, P, P, P, P],
        "maestro_pack_tokens": [P, I32, P, P, P, I32, P, P],
        "maestro_scatter_rows_fwd": [P, P, P, P, I32, I32, P],
        "maestro_gather_rows_bwd": [P, P, P, P, I32, I32, P],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    L.maestro_schedule_workspace.argtypes = [I32, I32]
    L.maestro_schedule_workspace.restype = I64
    _lib = L
    return L


def extra_symbols(names):
    """Bind further entry points (other kernel families register theirs lazily)."""
    L = lib()
    for name, (args, res) in names.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    return L


def set_pdl(on: bool) -> bool:
    """Programmatic dependent launch of the step kernels on/off (maestro_set_pdl); returns the
    previous setting."""
    L = extra_symbols({"maestro_set_pdl": ([ctypes.c_int32], ctypes.c_int)})
    return bool(L.maestro_set_pdl(1 if on else 0))


def reserve_sms_for_comm(default: int = 16) -> int:
    """Cap the persistent kernels' grids below the SM count so NCCL point-to-point kernels that
    spin while waiting on another GPU never hold an SM a persistent CTA needs
    (maestro_set_sm_budget).  MAESTRO_NCCL_RESERVED_SMS overrides the reserve; returns the budget."""
    import os

    import torch

    reserve = int(os.environ.get("MAESTRO_NCCL_RESERVED_SMS", default))
    n = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    budget = max(2, n - reserve) if reserve > 0 else 0
    L = extra_symbols({"maestro_set_sm_budget": ([ctypes.c_int32], ctypes.c_int)})
    check(L.maestro_set_sm_budget(budget), "set_sm_budget")
    return budget


def check(rc: int, what: str) -> None:
    if rc != 0:
        raise E.NativeError(f"{what} failed with CUDA error {rc}")
    _instrument.count(what)


def ptr(t) -> int:
    return t.data_ptr()


def stream_ptr(stream=None) -> int:
    """cudaStream_t of ``stream`` or of the current stream.  The raw getter costs ~0.1 us against
    ~3 us for building a ``torch.cuda.Stream`` object per launch (measured; it is host overhead on
    every kernel launch of the launch-bound VLM step)."""
    import torch

    if stream is not None:
        return stream.cuda_stream
    return torch._C._cuda_getCurrentRawStream(torch.cuda.current_device())


def graph_struct(graph: SectionGraph, configs) -> GraphStruct:
    """Fill maestro_graph_t from the lowered graph + per-section configs."""
    t = graph.tables
    g = GraphStruct()
    n = len(t.section_ids)
    g.n_sections, g.n_bits, g.critical = n, len(t.sub_names), t.critical
    g.n_up, g.n_down, g.n_aux = len(t.up_candidates), len(t.down_candidates), len(t.merge_order)
    for b, o in enumerate(t.sub_owner):
        g.sub_owner[b] = o
        g.sec_bits[o] |= 1 << b
    for i, sid in enumerate(t.section_ids):
        cfg = configs.get(sid, SectionConfig()) if hasattr(configs, "get") else configs[sid]
        if cfg.dp > MAX_DP:
            raise E.InvalidDims(f"dp {cfg.dp} exceeds the device limit {MAX_DP}", section=sid)
        g.side[i], g.neighbor[i] = t.side[i], t.neighbor[i]
        g.dp[i], g.fanout[i], g.mbs[i] = cfg.dp, cfg.fanout, cfg.mbs
    for k, v in enumerate(t.up_candidates):
        g.up_cand[k] = v
    for k, v in enumerate(t.down_candidates):
        g.down_cand[k] = v
    for k, v in enumerate(t.merge_order):
        g.merge_order[k] = v
    g.crit_bit = t.sub_names.index(t.section_ids[t.critical])
    g.par_up = int(getattr(graph, "parallel_upstream", False))
    return g


def raise_device_error(word: int, ids=None, section_ids=None) -> None:
    """Decode the device error word and raise the reference's exception class."""
    if word == ERR_CLEAN:
        return
    code = (word >> 24) & 0xFF
    index = word & 0xFFFFFF
    cls = E.DEVICE_CODES.get(code, E.MaestroError)
    if cls is E.FanoutViolation:
        sec = section_ids[index] if section_ids is not None else index
        raise cls(f"DP x fanout != DP of the toward-critical neighbour for section '{sec}'", edge=str(sec))
    sample = int(ids[index]) if ids is not None and index < len(ids) else index
    messages = {
        E.NegativeTime: "t_f_c must be positive and every time finite and nonnegative",
        E.BothActivated: "sample activates two submodules colocated in one section",
        E.ActivationError: "sample's activated sections cannot be attributed on one side",
        E.InvalidDims: "tokens_per_sample must be positive",
        E.InconsistentSchedule: "duplicate sample ids in batch",
    }
    raise cls(f"sample {sample}: {messages.get(cls, 'device error')}", sample=sample)
