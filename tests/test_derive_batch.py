"""costs.derive_batch (host planning input) vs the reference's own outputs (CPU, bit-exact).

Fixtures: tests/golden/derive_golden.json from tests/golden/make_derive_golden.py, which ran the
reference derive_batch (costs.py:230-299) with the same graphs, configs, params, profiles and
seeds.  Times compared as float.hex; activated sets exactly; invalid profiles raise the same
error class.
"""

import json
from pathlib import Path

import pytest

from golden_cases import product_graph
from paper_2605_10501_b200 import costs as C
from paper_2605_10501_b200 import errors as E
from paper_2605_10501_b200.workload import SectionConfig

GOLD = json.loads((Path(__file__).parent / "golden" / "derive_golden.json").read_text())


@pytest.mark.parametrize("case", GOLD, ids=[c["name"] for c in GOLD])
def test_derive_batch_matches_reference(case):
    g = product_graph(case["graph"])
    cfg = {k: SectionConfig(*v) for k, v in case["configs"].items()}
    params = {k: C.CostParams(flops_per_token_fwd=float.fromhex(f), peak_flops_per_gpu=float.fromhex(p),
                              bwd_fwd_ratio=float.fromhex(r)) for k, (f, p, r) in case["params"].items()}
    pr = case["profile"]
    if "error" in case:
        with pytest.raises(getattr(E, case["error"])):
            C.derive_batch(g, cfg, params, C.BatchProfile(pr["B"], pr["shares"], pr["tokens"]), case["seed"])
        return
    batch = C.derive_batch(g, cfg, params, C.BatchProfile(pr["B"], pr["shares"], pr["tokens"]), case["seed"])
    got = [{"id": s.sample_id, "t": [float.hex(float(x)) for x in s.as_tuple()], "act": sorted(s.activated_sections)}
           for s in batch]
    assert got == case["samples"]
