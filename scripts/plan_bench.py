"""Device plan (K1-K4) time vs the oracle's C port at the bench batches: KD (B = 64, 8 identical
samples... all equal lengths), VLM cfg 1 (B = 64 mixed), cfg 5 (B = 8); isolated on an idle GPU.
Prints JSON lines."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def breakdown(p, cost, tokens, B):
    """Device time of each plan launch (CUDA events between them), best of 10."""
    from paper_2605_10501_b200 import _native as N
    from paper_2605_10501_b200.scheduling import ctypes_ref

    L = N.lib()
    s = torch.cuda.current_stream().cuda_stream
    w = p.work.view(torch.int32)
    up, down, lpt, part, part_off = (w[i * B:] for i in range(5))
    crit = p.tables.critical
    W = N.MAX_DP + 1
    steps = [
        ("reset", lambda: L.maestro_error_reset(N.ptr(p.err), s)),
        ("k1_sample_times", lambda: L.maestro_sample_times(ctypes_ref(p.gs), N.ptr(cost), N.ptr(tokens), B, N.ptr(p.times),
                                                           N.ptr(p.act), N.ptr(p.err), s)),
        ("k2_partition", lambda: L.maestro_partition(ctypes_ref(p.gs), N.ptr(p.times), N.ptr(p.ids), N.ptr(p.act), B,
                                                     N.ptr(up), N.ptr(down), N.ptr(lpt), N.ptr(part), N.ptr(part_off),
                                                     N.ptr(p.err), s)),
        ("k3_wavefront", lambda: L.maestro_wavefront(N.ptr(p.times), B, N.ptr(part), N.ptr(part_off), p.dp_crit,
                                                     p.policy.code, N.ptr(p.orders[crit * B:]), N.ptr(p.metrics),
                                                     N.ptr(p.evals), s)),
        ("k4_fanout_merge", lambda: L.maestro_fanout_merge(ctypes_ref(p.gs), B, N.ptr(up), N.ptr(down), N.ptr(p.orders),
                                                           N.ptr(p.sec_off), N.ptr(p.err), s)),
    ]
    best = {k: 1e9 for k, _ in steps}
    for _ in range(10):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(steps) + 1)]
        torch.cuda.synchronize()
        ev[0].record()
        for i, (k, f) in enumerate(steps):
            if k == "k4_fanout_merge":  # critical offsets into sec_off (maestro_build_schedule does this in K4)
                p.sec_off.view(-1, W)[crit, : p.dp_crit + 1].copy_(part_off[: p.dp_crit + 1])
            N.check(f(), k)
            ev[i + 1].record()
        torch.cuda.synchronize()
        for i, (k, _) in enumerate(steps):
            best[k] = min(best[k], ev[i].elapsed_time(ev[i + 1]) * 1e3)
    return best


def main():
    import oracle
    from paper_2605_10501_b200 import recipes as R
    from paper_2605_10501_b200.costs import cost_table
    from paper_2605_10501_b200.scheduling import DevicePlanner

    for name, rec in [("kd_cfg2_B64", R.kd(1, 64)), ("vlm_cfg1_B64", R.vlm_tiny(1, 64)), ("kd_cfg5_B8", R.kd_8b(1, 8)),
                      ("vlm_cfg1_B256_dp4", R.vlm_tiny(4, 256)), ("omni4_B64_dp8", R.omni(8, 64, mix="4way", parallel_upstream=True))]:
        tab = rec.graph.tables
        B = rec.batch
        tok = np.zeros((len(tab.sub_names), B), dtype=np.int32)
        for b, n in enumerate(tab.sub_names):
            if n in rec.tokens:
                tok[b] = rec.tokens[n]
        cost = torch.from_numpy(cost_table(rec.graph, rec.configs, rec.params)).cuda()
        tokens = torch.from_numpy(tok).cuda()
        p = DevicePlanner(rec.graph, rec.configs, "interleaved", max_batch=B)
        p.ids[:B].copy_(torch.arange(B, dtype=torch.int32))
        ts = []
        for _ in range(12):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            p.plan_tokens(cost, tokens, B)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        p.raise_errors()
        tg = []
        for _ in range(12):  # the same plan replayed from a CUDA graph (one launch)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            p.plan_tokens_graphed(cost, tokens, B)
            e1.record()
            torch.cuda.synchronize()
            tg.append(e0.elapsed_time(e1))
        p.raise_errors()
        bd = breakdown(p, cost, tokens, B)
        times = p.times[: 6 * B].view(6, B).cpu().numpy()
        act = p.act[:B].cpu().numpy().view(np.uint32)
        dp = [rec.configs[s].dp for s in tab.section_ids]
        fan = [rec.configs[s].fanout for s in tab.section_ids]
        best = 1e9
        for _ in range(5):
            t0 = time.perf_counter()
            up, down = oracle.resolve(act, times, tab.sub_owner, tab.side, tab.up_candidates, tab.down_candidates,
                                      rec.graph.parallel_upstream)
            want, ev = oracle.build_schedule(times, np.arange(B), up, down, len(tab.section_ids), tab.critical, dp, fan,
                                             tab.neighbor, tab.merge_order)
            best = min(best, time.perf_counter() - t0)
        got = {k: list(v) for k, v in p.host_orders().items()}
        print(json.dumps({"case": name, "device_plan_us": min(ts[2:]) * 1e3, "device_plan_graph_us": min(tg[2:]) * 1e3, "cpu_port_us": best * 1e6,
                          "evals": ev, "orders_match": got == want,
                          "breakdown_us": bd}), flush=True)


if __name__ == "__main__":
    main()
