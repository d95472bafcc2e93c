"""CPU checks of the C-ABI boundary: the library loads and exports every declared symbol."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "maestro_b200.h"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^(?:int|int64_t|void)\s+(maestro_\w+)\(", text, flags=re.M)))


def test_header_declares_entry_points():
    names = declared()
    assert "maestro_build_schedule" in names and "maestro_wavefront" in names
    assert len(names) >= 10


def test_library_exports_every_declared_symbol():
    from paper_2605_10501_b200 import _native

    if not _native.LIB_PATH.exists():
        from paper_2605_10501_b200 import build_native

        build_native.build()
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    _native.lib()  # argtypes bind


def test_graph_struct_layout_matches_header():
    """sizeof(maestro_graph_t): 6 ints + sub_owner[32] + 9 arrays of 16 + crit_bit + par_up."""
    from paper_2605_10501_b200._native import GraphStruct

    assert ctypes.sizeof(GraphStruct) == 4 * (6 + 32 + 16 * 9 + 2)


def test_graph_tables_for_recipes():
    from paper_2605_10501_b200 import _native, recipes

    for rec in (recipes.vlm_tiny(4), recipes.kd(1)):
        gs = _native.graph_struct(rec.graph, rec.configs)
        t = rec.graph.tables
        assert gs.critical == t.critical and gs.n_bits == len(t.sub_names)
        assert t.sub_names[gs.crit_bit] == rec.graph.critical.id


def test_no_device_means_loud_failure():
    import torch

    from paper_2605_10501_b200 import errors, scheduling
    from paper_2605_10501_b200.workload import SampleTiming

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(errors.NativeError):
        scheduling.schedule_rank([SampleTiming(0, 0, 1), SampleTiming(1, 0, 1)])
