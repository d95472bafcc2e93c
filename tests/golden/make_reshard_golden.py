"""Golden reshard plans by running the REFERENCE (build container only; imports /root/reference).

    python tests/golden/make_reshard_golden.py   -> tests/golden/reshard_golden.json

Each case: the two layouts, the reference's transfer list (plan_reshard, mq.py:123-160) and a
checksum of each receiver shard produced by the reference's apply_plan (mq.py:163-174) on an
arange tensor; plus the reference's error class for invalid inputs.
"""

from __future__ import annotations

import json
import random
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from maestro import mq  # noqa: E402


def lay(d):
    return mq.ShardLayout(tuple(d["shape"]), d["tp"], d["cp"], d["tp_axis"], d["cp_axis"])


def case(src, dst):
    out = {"src": src, "dst": dst}
    try:
        s, d = lay(src), lay(dst)
        plan = mq.plan_reshard(s, d)
    except Exception as e:  # noqa: BLE001
        out["error"] = type(e).__name__
        return out
    out["transfers"] = [[list(t.sender), list(t.receiver), [list(x) for x in t.sender_slice],
                         [list(x) for x in t.receiver_slice]] for t in plan.transfers]
    full = np.arange(int(np.prod(src["shape"])), dtype=np.int64).reshape(src["shape"])
    shards = {r: s.shard(full, r) for r in s.ranks()}
    res = mq.apply_plan(plan, shards)
    out["receivers"] = {f"{r[0]},{r[1]}": [list(v.shape), int((v * (1 + np.arange(v.size).reshape(v.shape))).sum())]
                        for r, v in res.items()}
    return out


def L(shape, tp=1, cp=1, ta=0, ca=1):
    return {"shape": list(shape), "tp": tp, "cp": cp, "tp_axis": ta, "cp_axis": ca}


def main():
    cases = [
        case(L([8, 4], tp=2), L([8, 4])),                      # SPEC.md:427 gather halves
        case(L([8, 4]), L([8, 4], tp=2)),                      # scatter halves
        case(L([6, 6], tp=2, cp=3), L([6, 6], tp=3, cp=2)),
        case(L([2048, 2048]), L([2048, 2048])),                # KD handoff: identity
        case(L([12, 8, 4], tp=4, cp=2, ta=0, ca=2), L([12, 8, 4], tp=3, cp=1, ta=0, ca=2)),
        case(L([8, 4], tp=2), L([8, 6])),                      # IncompatibleShapes
        case(L([8, 4], tp=2, ta=0), L([8, 4], tp=2, ta=1)),    # axes disagree
    ]
    rng = random.Random(7)
    while len(cases) < 80:  # fuzz: M, N <= 4 on 2-3 d tensors
        nd = rng.choice([2, 3])
        ta, ca = rng.sample(range(nd), 2)
        degs = [rng.choice([1, 2, 3, 4]) for _ in range(4)]
        shape = [rng.choice([1, 2, 3]) for _ in range(nd)]
        for ax, a, b in ((ta, degs[0], degs[2]), (ca, degs[1], degs[3])):
            shape[ax] *= int(np.lcm(a, b))
        if int(np.prod(shape)) > 4096:
            continue
        cases.append(case(L(shape, degs[0], degs[1], ta, ca), L(shape, degs[2], degs[3], ta, ca)))
    for bad in ([L([0, 4]), L([8, 4])], [L([8, 4], tp=3), L([8, 4])], [L([8, 4], tp=2, cp=2, ta=0, ca=0), L([8, 4])]):
        try:
            lay(bad[0])
            cases.append({"layout": bad[0]})
        except Exception as e:  # noqa: BLE001
            cases.append({"layout": bad[0], "error": type(e).__name__})
    path = Path(__file__).with_name("reshard_golden.json")
    path.write_text(json.dumps(cases, separators=(",", ":"), sort_keys=True))
    print(f"wrote {len(cases)} cases to {path}")


if __name__ == "__main__":
    main()
