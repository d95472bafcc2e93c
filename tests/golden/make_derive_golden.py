"""Golden batches from the REFERENCE derive_batch (costs.py:230-299); build container only.

    python tests/golden/make_derive_golden.py   -> tests/golden/derive_golden.json

Per case: the graph (make_golden.graph_desc), configs, cost params (float.hex), the batch
profile, the seed, and the reference's samples (6-tuples as float.hex + activated sections) or
the error class it raised.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
import make_golden as mg  # noqa: E402  (puts the reference and the repo on sys.path)

rw, rcosts = mg.rw, mg.rcosts
H = float.hex


def case(name, g, configs, params, profile, seed):
    out = {"name": name, "graph": mg.graph_desc(g), "configs": {k: list(v.as_tuple()) for k, v in configs.items()},
           "params": {k: [H(p.flops_per_token_fwd), H(p.peak_flops_per_gpu), H(p.bwd_fwd_ratio)]
                      for k, p in params.items()},
           "profile": {"B": profile["B"], "shares": profile.get("shares", {}), "tokens": profile.get("tokens", {})},
           "seed": seed}
    try:
        bp = rcosts.BatchProfile(profile["B"], profile.get("shares", {}), profile.get("tokens", {}))
        batch = rcosts.derive_batch(g, configs, params, bp, seed)
        out["samples"] = [mg.sample_desc(s) for s in batch]
    except Exception as e:  # noqa: BLE001
        out["error"] = type(e).__name__
    return out


def P(f, peak=3e14, ratio=2.0):
    return rcosts.CostParams(flops_per_token_fwd=f, peak_flops_per_gpu=peak, bwd_fwd_ratio=ratio)


def main():
    cases = []
    g2, g3, g4, g5 = mg.g2(), mg.g3(), mg.g4(), mg.g5()
    for seed in (0, 1, 17):
        cases.append(case(f"g2:s{seed}", g2, mg.cfgs(g2, 4, {"enc": (1, 4)}),
                          {"enc": P(1.1e7), "llm": P(7.9e7)}, {"B": 64, "shares": {"enc": 0.5}}, seed))
        cases.append(case(f"g3:s{seed}", g3, mg.cfgs(g3, 2, {"enc": (1, 2), "dec": (2, 1)}),
                          {"enc": P(1.1e7), "llm": P(7.9e7, ratio=2.5), "dec": P(3e6)},
                          {"B": 48, "shares": {"enc": 0.3, "dec": 0.7}, "tokens": {"llm": 2048, "enc": 512}}, seed))
        cases.append(case(f"g4:s{seed}", g4, mg.cfgs(g4, 3, {"image_enc": (1, 3), "audio_enc": (3, 1)}),
                          {"image_enc": P(2e7), "audio_enc": P(1.5e7), "llm": P(1.4e10, peak=1.6381e15)},
                          {"B": 96, "shares": {"image_enc": 0.25, "audio_enc": 0.75}}, seed))
        cases.append(case(f"g5:s{seed}", g5, mg.cfgs(g5, 2, {"pre": (1, 1), "enc": (1, 2), "dec": (1, 2)}),
                          {k: P(1e7 * (i + 1)) for i, k in enumerate(("pre", "enc", "llm", "dec"))},
                          {"B": 33, "shares": {"pre": 1.0, "enc": 0.5, "dec": 0.0}}, seed))
    # shares rounding at the edges; pipeline/mbs amortisation
    cfg = {"llm": rw.SectionConfig(dp=2, pp=2, mbs=4), "enc": rw.SectionConfig(dp=1, fanout=2, mbs=2)}
    cases.append(case("g2:pp-mbs", g2, cfg, {"enc": P(1e7), "llm": P(8e7)}, {"B": 10, "shares": {"enc": 0.25}}, 3))
    cases.append(case("g2:bad-share", g2, mg.cfgs(g2, 1, {"enc": (1, 1)}), {"enc": P(1e7), "llm": P(8e7)},
                      {"B": 4, "shares": {"enc": 1.5}}, 0))
    cases.append(case("g2:empty", g2, mg.cfgs(g2, 1, {"enc": (1, 1)}), {"enc": P(1e7), "llm": P(8e7)},
                      {"B": 0}, 0))
    path = Path(__file__).with_name("derive_golden.json")
    path.write_text(json.dumps(cases, separators=(",", ":"), sort_keys=True))
    print(f"wrote {len(cases)} cases to {path}")


if __name__ == "__main__":
    main()
