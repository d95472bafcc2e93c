"""Benchmark: training samples/s of the section-graph executor step (BASELINE.json metric).

Default workload (configs[1] of BASELINE.json): knowledge distillation, forward-only 1.1B teacher
(TinyLlama shape) -> 125M student, fused KL over the 32k vocabulary, seq 2048, 64 samples per
student DP rank, synthetic token ids, random-init weights.  Default layout (--layout colocated):
every GPU hosts a teacher and a student DP rank (handoff = CUDA event, student gradients
all-reduced over NCCL); --layout disjoint puts teacher and student on disjoint GPU groups with the
teacher hidden states handed over NVLink (mq.PeerTransport, or NCCL with MAESTRO_HANDOFF=nccl).

Other workloads (--workload): kd8b = configs[4] (Llama-3-8B -> Llama-3.2-1B, 8k seq, V 128256),
vlm = configs[0] (tiny VLM), section = the generic section-graph executor on cfg 3 / cfg 4 shapes
(--graph vlm7b|omni).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload ...]

Prints one JSON line (rank 0).  `value` is device-timed (CUDA events, max over ranks) with
inputs resident in HBM; `e2e` is the same metric through the public API (executor.step) timed by
the host wall clock, with the step inputs copied from pinned host memory and the loss read back
every step.  Per-kernel timing (roofline) comes from one extra, untimed step with the sections
serialised on one stream, so kernel durations never overlap and never perturb `value`.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "training samples/sec (device-timed, max over ranks) at 1/2/4/8 B200; section-stall %"
UNIT = "samples/s"

KD_PRESETS = {
    # workload -> (teacher shape, student shape, recipe, seq, batch/rank, student mbs, teacher mbs, vocab, label)
    "kd": ("kd_teacher_1b", "kd_student_125m", "kd", 2048, 64, 8, 16, 32000,
           "kd_cfg2: fwd-only 1.1B teacher (TinyLlama shape) -> 125M student, fused KL over 32k vocab, "
           "seq 2048, teacher head colocated with the student"),
    "kd8b": ("llama3_8b", "llama32_1b", "kd_8b", 8192, 8, 1, 2, 128256,
             "kd_cfg5: fwd-only Llama-3-8B-shaped teacher (hd128, GQA 32/8) -> Llama-3.2-1B-shaped student, "
             "fused KL over 128256 vocab, seq 8192, teacher head colocated with the student"),
}


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        for line in Path(self.path).read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[4:8]) if v.lower().startswith("active")})

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None

        sm = [num(r[0]) for r in rows if num(r[0]) is not None]
        pw = [num(r[2]) for r in rows if num(r[2]) is not None]
        loaded = [s for s, p in zip(sm, pw) if p is not None and p > 300] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": num(rows[0][1]), "reasons": reasons, "samples": len(rows),
                "power_w_max": max(pw) if pw else None}


# ---------------------------------------------------------------------------------------------- CPU leg
def cpu_schedule_baseline(planner, reps: int = 5):
    """The reference's CPU scheduler path (scheduling.py build_schedule) on the step's own 6-tuples,
    through the oracle's C port, single-threaded -- the CPU baseline for K1-K5.  The
    6-tuples and activation masks are read back from the device planner after the timed region;
    the device orders are compared with the oracle's (bit-exact parity on the benched batch)."""
    import numpy as np

    import oracle

    tab, B = planner.tables, planner.B
    times = planner.times[: 6 * B].view(6, B).cpu().numpy()
    act = planner.act[:B].cpu().numpy().view(np.uint32)
    dp = [planner.configs[s].dp for s in tab.section_ids]
    fan = [planner.configs[s].fanout for s in tab.section_ids]
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        up, down = oracle.resolve(act, times, tab.sub_owner, tab.side, tab.up_candidates, tab.down_candidates)
        want, evals = oracle.build_schedule(times, np.arange(B), up, down, len(tab.section_ids), tab.critical, dp,
                                            fan, tab.neighbor, tab.merge_order, planner.policy.value)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    got = {k: list(v) for k, v in planner.host_orders().items()}
    return {"ms": best * 1e3, "cores": 1, "makespan_evals": evals, "device_orders_match": got == want,
            "sample": f"build_schedule of the benched batch (B={B}), oracle/sched_oracle.c port of scheduling.py"}


def cpu_kd_step_sample(preset: str = "kd", reps: int = 1):
    """The oracle's fp32 CPU restatement of one KD training step (all host threads).

    kd: one full sample (2048 tokens, full depth).  kd8b: an 8B fp32 teacher and 8k tokens do not
    fit a bounded CPU sample, so one 8192-token sample runs through ONE teacher and ONE student
    layer at full width plus both full-vocab heads and the KL; the step time is extrapolated by the
    layer counts (t = t_heads + L_t t_teacher_layer + L_s t_student_layer).
    Returns (seconds per sample, threads, sample description)."""
    import dataclasses
    import math

    import torch

    from oracle import torch_ref as R
    from paper_2605_10501_b200.transformer import SHAPES

    torch.set_num_threads(os.cpu_count() or 1)
    tname, sname, _, seq, _, _, _, vocab, _ = KD_PRESETS[preset]
    t_full, s_full = SHAPES[tname], SHAPES[sname]
    g = torch.Generator().manual_seed(0)

    def flat(shape):
        n = sum(((math.prod(s) + 63) // 64 * 64) for _, s in shape.param_shapes())
        return torch.randn(n, generator=g) * 0.02

    def run(t_shape, s_shape):
        t_flat, s_flat = flat(t_shape), flat(s_shape)
        t_head = torch.randn(t_shape.vocab, t_shape.d, generator=g) * 0.02
        ids = torch.randint(0, vocab, (seq,), generator=g, dtype=torch.int32)
        cu = torch.tensor([0, seq], dtype=torch.int32)
        m, v = torch.zeros_like(s_flat), torch.zeros_like(s_flat)
        best = None
        for i in range(reps):
            t0 = time.perf_counter()
            _, grad = R.kd_step_reference(t_shape, s_shape, t_flat, s_flat, t_head, ids, cu, global_tokens=seq)
            R.adamw_reference(s_flat, grad, m, v, 3e-4, i + 1)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        return best

    if preset == "kd":
        sec = run(t_full, s_full)
        desc = ("1 sample of 2048 tokens: oracle/torch_ref.py fp32 KD step on the host CPU "
                "(teacher fwd + colocated head, student fwd/bwd, KL, AdamW)")
    else:
        one = lambda s: dataclasses.replace(s, layers=1)  # noqa: E731
        zero = lambda s: dataclasses.replace(s, layers=0)  # noqa: E731
        t1 = run(one(t_full), one(s_full))
        t0 = run(zero(t_full), zero(s_full))
        t_only = run(one(t_full), zero(s_full))
        tl, sl = t_only - t0, t1 - t_only
        sec = t0 + t_full.layers * tl + s_full.layers * sl
        desc = (f"1 sample of {seq} tokens through 1 teacher + 1 student layer at full width plus both "
                f"{vocab}-vocab heads and the KL (oracle/torch_ref.py fp32), extrapolated to "
                f"{t_full.layers} + {s_full.layers} layers: heads {t0:.2f} s, teacher layer {tl:.2f} s, "
                f"student layer {sl:.2f} s")
    return sec, torch.get_num_threads(), desc


def cpu_vlm_step_sample(batch: int = 8):
    """The oracle's fp32 CPU restatement of one VLM (cfg 1) step on a bounded batch."""
    import torch

    from oracle import torch_ref as R
    from paper_2605_10501_b200 import vlm
    from paper_2605_10501_b200.transformer import SHAPES

    torch.set_num_threads(os.cpu_count() or 1)
    ls, vs = SHAPES["vlm_gpt2l"], SHAPES["vit_tiny"]
    import math

    g = torch.Generator().manual_seed(0)

    def flat(shapes):
        n = sum(((math.prod(s) + 63) // 64 * 64) for _, s in shapes)
        return torch.randn(n, generator=g) * 0.02

    lf = flat(ls.param_shapes())
    vf = flat(vs.param_shapes() + [("patch_w", (vs.d, vlm.PATCH_DIM)), ("proj_w", (ls.d, 4 * vs.d))])
    hb = vlm.vlm_host_batch(batch, seed=0)
    t0 = time.perf_counter()
    R.vlm_step_reference(ls, vs, lf, vf, hb, vlm.merge_index())
    return (time.perf_counter() - t0) / batch, torch.get_num_threads()


def run_reference(args):
    """--impl reference: the CPU implementation of the path (the oracle's fp32 port; the reference
    itself is a planning/simulation toolkit with no training step), rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    secs, threads, desc = [], 1, ""
    for _ in range(args.warmup + args.steps):
        if args.workload == "vlm":
            t, threads = cpu_vlm_step_sample()
            desc = "8 samples per step: oracle/torch_ref.py fp32 VLM step (ViT-tiny, merge, projector, GPT, CE)"
        elif args.workload == "section":
            from paper_2605_10501_b200.graph_bench import _cpu_sample

            v, threads, desc = _cpu_sample(args.graph, args.layers or 4)
            t = 1.0 / v
        else:
            t, threads, desc = cpu_kd_step_sample(args.workload)
        secs.append(t)
    sec = statistics.mean(secs[args.warmup:]) if args.steps else secs[-1]
    value = 1.0 / sec
    if args.workload == "vlm":
        workload, seq, gb = "vlm_cfg1: ViT-tiny (d192 L12) -> 2-layer GPT (d768), 50/50 text/image", "64..497", 64
    elif args.workload == "section":
        workload, seq, gb = f"{args.graph} (generic section-graph executor)", "varlen", (args.batch_per_rank or 8) * args.gpus
    else:
        P = KD_PRESETS[args.workload]
        workload, seq, gb = P[8], P[3], (args.batch_per_rank or P[4]) * args.gpus
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload, "global_batch": gb, "seq_len": seq,
                   "parallelism": f"host CPU ({threads} threads); each step times a bounded sample"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------------- helpers
def fp64_probe():
    """Measured fp64 CUDA-core add throughput (adds/s) and dependent-add latency (s): the
    denominators of the scheduler kernels' roofline (maestro_fp64_probe)."""
    import ctypes

    import torch

    from paper_2605_10501_b200 import _native as N

    L = N.extra_symbols({"maestro_fp64_probe": ([ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                                 ctypes.c_void_p], ctypes.c_int)})
    out = torch.zeros(4096, dtype=torch.float64, device="cuda")
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    res = []
    for mode, iters, blocks in ((0, 4096, sms * 8), (1, 1 << 16, 1)):
        for rep in range(2):  # first launch warms up
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            N.check(L.maestro_fp64_probe(out.data_ptr(), mode, iters, blocks, N.stream_ptr()), "fp64_probe")
            e1.record()
            torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        res.append(blocks * 256 * 8 * iters / t if mode == 0 else t / iters)
    return res[0], res[1]


def scheduler_roofline(n_per_rank, plan_ms, ops_per_sample=8):
    """K3 (wavefront) work and critical path for ranks of n samples: insertion step k evaluates
    k+1 candidate orders of k+1 samples (one thread each), ~8 dependent fp64 ops per sample update."""
    add_rate, lat = fp64_probe()
    work = sum(ops_per_sample * sum((k + 1) ** 2 for k in range(1, n)) for n in n_per_rank)
    chain = max(ops_per_sample * sum(k + 1 for k in range(1, n)) for n in n_per_rank) * lat
    t = plan_ms / 1e3
    return {"fp64_add_rate_measured_Gps": add_rate / 1e9, "fp64_dep_add_latency_ns": lat * 1e9,
            "k3_fp64_ops": work, "achieved_fp64_Gops": work / t / 1e9 if t > 0 else None,
            "frac_of_fp64_throughput": (work / t) / add_rate if t > 0 else None,
            "critical_path_bound_us": chain * 1e6,
            "frac_of_latency_bound": chain / t if t > 0 else None,
            "note": "latency-bound: the wavefront recurrence is a dependent chain per candidate order"}


def p2p_bandwidth(ex, dist, nbytes=64 << 20, reps=4):
    """Measured NCCL point-to-point bandwidth on the handoff pairs (teacher rank -> student rank),
    GB/s on the receiver; the peak the handoff (C1) is reported against.  Disjoint layout only."""
    import torch

    buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    out = None
    for it in range(2):  # first pass warms the NCCL point-to-point channel
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        e0.record()
        for _ in range(reps):
            for dst in ex.roles["send_to"]:
                dist.send(buf, dst)
            for src in ex.roles["recv_from"]:
                dist.recv(buf, src)
        e1.record()
        torch.cuda.synchronize()
        if ex.roles["recv_from"] and it == 1:
            out = reps * nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9
    t = torch.tensor([out or 0.0], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def kernel_fractions(rec: dict, step_ms: float, peaks: dict, attn_flops=None, kd_bytes=None) -> dict:
    """Per-kernel roofline fractions from one serialised, untimed step (instrument.stop_timing):
    tensor-bound kernels against the measured sustained bf16 peak, K9 against measured HBM GB/s."""
    peak_t = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
    out = {}
    for kind in ("attn_fwd", "attn_bwd"):
        if kind in rec and attn_flops is not None:
            _, ms, n = rec[kind]
            fl = attn_flops[0 if kind == "attn_fwd" else 1]
            if ms > 0 and fl > 0:
                a = fl / (ms / 1e3) / 1e12
                out[kind] = {"achieved": a, "peak": peak_t, "unit": "TFLOP/s", "frac": a / peak_t,
                             "launches": n, "ms": ms, "share_of_step": ms / step_ms}
    if "kd_loss" in rec:
        by, ms, n = rec["kd_loss"]
        if ms > 0:
            a = by / (ms / 1e3) / 1e9
            out["kd_loss"] = {"achieved": a, "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": a / peaks["hbm_gbs"],
                              "launches": n, "ms": ms, "share_of_step": ms / step_ms}
    return out


def gemm_traffic(workload: str):
    """DRAM bytes per launch of the dominant GEMM at the benched shape, from the committed ncu
    --set full capture (profiles/r02_gemm_traffic.json, one entry per workload), or None."""
    p = ROOT / "profiles" / "r02_gemm_traffic.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text()).get(workload)
    return d


# ---------------------------------------------------------------------------------------------- KD leg
def run_kd(args):
    import torch

    tname, sname, recipe, seq, bpr, mbs, tmbs, vocab, workload = KD_PRESETS[args.workload]
    bpr = args.batch_per_rank or bpr
    mbs = args.mbs or mbs
    tmbs = args.teacher_mbs or tmbs
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")

    from paper_2605_10501_b200 import instrument
    from paper_2605_10501_b200.executor import KDExecutor, handoff_mode, synthetic_ids

    ex = KDExecutor(n_gpus=args.gpus, batch_per_rank=bpr, seq=seq, mbs=mbs, layout=args.layout, teacher_mbs=tmbs,
                    teacher=tname, student=sname, recipe=recipe)
    B = ex.batch
    ids_host = torch.from_numpy(synthetic_ids(B, seq, vocab)).pin_memory()
    ids_dev = ids_host.cuda()

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    p2p = p2p_bandwidth(ex, dist) if (dist is not None and not ex.colocated) else None
    for _ in range(args.warmup):
        ex.step(ids_dev, want_loss=False, plan_ahead=True)
    barrier()
    # ---- device-timed region (inputs resident in HBM); no per-kernel events inside it
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = instrument.launches
    main_stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stalls, busy, span, stats = [], 0.0, 0.0, []
    e0.record(main_stream)
    for _ in range(args.steps):  # step() does not synchronise: the host runs a step ahead
        stats.append(ex.step(ids_dev, want_loss=False, plan_ahead=True))
    e1.record(main_stream)
    barrier()
    for st in stats:  # lazy statistics, read after the timed region
        stalls.append(st.stall_frac)
        busy += st.critical_busy_ms
        span += st.critical_span_ms
    launches = instrument.launches - launches0
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], device="cuda")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    ms_per_step = ms / max(args.steps, 1)
    value = B * args.steps / (ms / 1e3)
    # ---- end-to-end through the public API, host wall clock: ids from pinned host memory every
    # step (H2D inside the step), the loss read back every step (D2H)
    barrier()
    w0 = time.perf_counter()
    losses, prev = [], None
    for _ in range(args.steps):
        st = ex.step(ids_host, want_loss=True, plan_ahead=True)
        if prev is not None:
            losses.append(prev.loss)  # the previous step's loss, read while this step runs
        prev = st
    losses.append(prev.loss)
    torch.cuda.synchronize()
    w1 = time.perf_counter()
    barrier()
    # ---- per-kernel timing: one extra step with the sections serialised on one stream (untimed),
    # after one serialised warm-up step (its different buffer lifetimes settle in the allocator)
    with ex.serialized():
        ex.step(ids_dev, want_loss=False)
    torch.cuda.synchronize()
    instrument.start_timing()
    with ex.serialized():
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        ex.step(ids_dev, want_loss=False)
        s1.record()
    torch.cuda.synchronize()
    rec = instrument.stop_timing()
    serial_ms = s0.elapsed_time(s1)
    g_flops, g_ms, g_n = rec.get("gemm", (0.0, 0.0, 0))
    # planner calibration: fit each section's CostParams (costs.py:105-123) to the
    # serialised step's measured stage times, then predict that step with the fitted model
    calib = None
    try:
        from paper_2605_10501_b200.costs import section_iteration_time
        from paper_2605_10501_b200.planner import fit_cost_params, kd_stage_samples

        samples = kd_stage_samples(ex)
        fpt = {k: v.flops_per_token_fwd for k, v in ex.recipe.params.items()}
        fit = fit_cost_params(samples, fpt, ex.recipe.params)
        pred = sum(section_iteration_time(ex.graph.section(sec), ex.configs[sec], fit[sec], seq,
                                          ex.batch // ex.configs[sec].dp) for sec in fit)
        calib = {"fitted": {k: {"effective_flops": v.peak_flops_per_gpu, "bwd_fwd_ratio": v.bwd_fwd_ratio}
                            for k, v in fit.items()},
                 "stages": len(samples), "predicted_sections_ms": pred * 1e3,
                 "measured_sections_ms": sum(x.seconds for x in samples) * 1e3,
                 "measured_serialized_step_ms": serial_ms,
                 "note": "planner.fit_cost_params on the serialised step's device stage times; the fitted "
                         "CostParams replace the presets' nominal 3e14 FLOP/s (costs.py:309,327,348)"}
    except Exception as exc:  # noqa: BLE001
        calib = {"error": repr(exc)}
    # the step's K1-K5 plan alone on an idle GPU (in the step it shares the SMs with the running
    # persistent kernels, so its in-step device time is mostly queueing)
    iso = []
    for _ in range(5):
        torch.cuda.synchronize()
        _, _, _, (p0, p1) = ex._plan_async(torch.cuda.current_stream())
        torch.cuda.synchronize()
        iso.append(p0.elapsed_time(p1))
    plan_iso_ms = min(iso)
    if dist is not None:  # loss lives on student ranks; report the first student rank's
        lt = torch.tensor([losses[-1] if losses and losses[-1] is not None else float("nan")], device="cuda")
        src = 0 if ex.colocated else ex.dp_t
        dist.broadcast(lt, src)
        losses = [float(lt.item())]
    t = torch.tensor([(w1 - w0) * 1e3], device="cuda")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_value = B * args.steps / (float(t.item()) / 1e3)
    # ---- stall: max and mean over critical ranks; per-section idle; scheduler; C2 all-reduce
    stall = torch.tensor([max(stalls) if stalls and ex.student is not None else 0.0,
                          (1 - busy / span) if span > 0 else 0.0], device="cuda")
    mean_stall = torch.tensor([sum(stalls) / len(stalls) if stalls and ex.student is not None else 0.0,
                               1.0 if ex.student is not None else 0.0], device="cuda")
    avg = lambda f: sum(f(x) for x in stats) / max(len(stats), 1)  # noqa: E731
    per_rank = torch.tensor([avg(lambda x: x.plan_ms), avg(lambda x: x.allreduce_ms),
                             avg(lambda x: x.step_ms - x.critical_busy_ms) if ex.student is not None else 0.0,
                             avg(lambda x: x.step_ms - x.teacher_busy_ms) if ex.teacher is not None else 0.0],
                            device="cuda")
    if dist is not None:
        dist.all_reduce(stall, op=dist.ReduceOp.MAX)
        dist.all_reduce(mean_stall, op=dist.ReduceOp.SUM)
        dist.all_reduce(per_rank, op=dist.ReduceOp.MAX)
    plan_ms, ar_ms, idle_s, idle_t = (float(x) for x in per_rank.tolist())
    n_sched = [ex.batch // ex.dp_s] * ex.dp_s + ([ex.batch // ex.dp_t] * ex.dp_t if ex.dp_t else [])
    grad_bytes = ex.student.p.grad.numel() * 4 if ex.student is not None else 0
    peaks, peak_kind = load_peaks()
    peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
    gemm_tflops = (g_flops / (g_ms / 1e3) / 1e12) if g_ms > 0 else None
    cpu = None
    if rank == 0 and args.gpus == 1 and not args.no_cpu_baseline:
        try:
            sec, threads, desc = cpu_kd_step_sample(args.workload)
            cpu = {"value": 1.0 / sec, "unit": UNIT, "cores": threads, "kind": "port", "sample": desc}
            try:
                cpu["scheduler"] = cpu_schedule_baseline(ex.planner)
            except Exception as exc:  # noqa: BLE001
                cpu["scheduler"] = {"error": repr(exc)}
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {exc}"}
    xcheck = None
    if ex.colocated or ex.student is not None:
        try:
            mk, cidle, span_x, midle = ex.crosscheck()
            xcheck = {"model_makespan_ms": mk * 1e3, "model_critical_idle_ms": cidle * 1e3,
                      "measured_critical_span_ms": span_x * 1e3, "measured_critical_idle_ms": midle * 1e3}
        except Exception as exc:  # noqa: BLE001
            xcheck = {"error": repr(exc)}
    if args.trace and rank == 0:
        from paper_2605_10501_b200.simulator import export_trace

        export_trace(ex.measured_events(), args.trace)
    sched_roof = None
    if rank == 0:
        try:
            sched_roof = scheduler_roofline(n_sched, plan_iso_ms)
        except Exception as exc:  # noqa: BLE001
            sched_roof = {"error": repr(exc)}
    if rank == 0:
        dp_s, dp_t = ex.dp_s, ex.dp_t
        transport = ("mq.PeerTransport: copy-engine puts over NVLink + stream memory-op signals"
                     if handoff_mode() == "nvlink" else "mq.DistTransport over NCCL point-to-point")
        traffic = gemm_traffic(args.workload)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {
                "workload": workload,
                "global_batch": B, "seq_len": seq, "micro_batch": mbs, "teacher_micro_batch": ex.mbs_t,
                "parallelism": (f"colocated teacher+student per GPU, student dp{dp_s} (grad all-reduce)"
                                if ex.colocated
                                else f"disjoint groups: teacher dp{dp_t} -> student dp{dp_s} (fanout 1, "
                                     f"{handoff_mode()} handoff)"),
                "l2": "inputs larger than L2 (teacher weights >= 2.2 GB, logits >= 1 GB per micro-batch)",
            },
            "section_stall_pct": 100.0 * float(stall[0].item()),
            "section_stall": {"max_pct": 100.0 * float(stall[0].item()),
                              "mean_pct": 100.0 * float(mean_stall[0].item()) / max(float(mean_stall[1].item()), 1.0),
                              "definition": "(critical span - critical busy) / critical span per student rank"},
            "section_idle_ms": {"student": idle_s, "teacher": idle_t,
                                "definition": "step time - section busy time, max over ranks"},
            "scheduler": {"device_us_per_step": plan_ms * 1e3, "isolated_us": plan_iso_ms * 1e3,
                          "share_of_step_pct": 100.0 * plan_ms / ms_per_step,
                          "makespan_evals_per_step": sum(n * (n + 1) // 2 for n in n_sched),
                          "placement": "K1-K5 of step k+1 on a side stream while step k runs (KDExecutor.step(plan_ahead=True))",
                          "roofline": sched_roof,
                          "note": "device_us_per_step: in-step, on a side stream next to the step's persistent kernels "
                                  "(mostly waiting for SMs); isolated_us: the same plan alone on an idle GPU "
                                  "(roofline computed on it)"},
            "grad_allreduce": ({"ms": ar_ms, "bytes": grad_bytes,
                                "overlapped": ex.gsync is not None,
                                "note": ("ms = the exposed tail after the student backward; the per-layer buckets "
                                         "run during the last micro-batch's backward (gradsync.GradSync)"
                                         if ex.gsync is not None else "ms = the whole all-reduce after the backward"),
                                "bus_GBps": (2 * (dp_s - 1) / dp_s * grad_bytes / (ar_ms / 1e3) / 1e9
                                             if ar_ms and ex.gsync is None else None)}
                               if dp_s > 1 else None),
            "handoff": (None if ex.colocated else
                        {"bytes_per_step": int(B // max(dp_s, 1) * seq * ex.tshape.d * 2),
                         "p2p_GBps_measured": p2p, "transport": transport}),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(B * seq * 4),
                    "d2h_bytes_per_step": ex.readback_bytes_per_step(),
                    "timing": "host wall clock (perf_counter) around the steps, synchronised at both ends"},
            "gpu_launches": launches // max(args.steps, 1),
            "roofline": {"bound": "tensor", "kernel": "maestro tcgen05 GEMM (csrc/gemm.cu)",
                         "achieved": gemm_tflops, "peak": peak, "unit": "TFLOP/s",
                         "frac": (gemm_tflops / peak) if gemm_tflops else None,
                         "traffic": traffic.get("traffic_bytes_per_launch") if traffic else None,
                         "traffic_source": traffic.get("source") if traffic else None,
                         "peak_kind": f"{peak_kind} bf16_tflops_sustained",
                         "launches_timed": g_n, "gemm_ms": g_ms, "serialized_step_ms": serial_ms,
                         "share_of_step": g_ms / serial_ms if serial_ms > 0 else None,
                         "note": "achieved = sum of 2MNK over every GEMM launch / sum of their CUDA-event "
                                 "durations, from one extra step with the sections serialised on one stream, "
                                 "outside the timed region (durations do not overlap: share_of_step <= 1)"},
            "kernels": kernel_fractions(rec, serial_ms, peaks, ex.attention_flops_per_step(),
                                        ex.kd_loss_bytes_per_step()),
            "model_tflops": ex.model_flops_per_step() * args.steps / (ms / 1e3) / 1e12,
            "simulator_crosscheck": xcheck,
            "planner_calibration": calib,
            "clocks": clk,
            "cpu_baseline": cpu,
            "loss": losses[-1] if losses else None,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------------------------------------- VLM leg
def run_vlm(args):
    """configs[0] (tiny VLM: ViT-tiny encoder -> 2-layer GPT, 50/50 text/image).  N=1: sections
    co-resident on one GPU; N>1: --layout colocated (both sections DP on every GPU) or disjoint
    (ViT / LLM groups, recipes.VLM_LAYOUTS, activation and gradient handoff through mq)."""
    import torch

    from paper_2605_10501_b200 import instrument
    from paper_2605_10501_b200.executor import handoff_mode
    from paper_2605_10501_b200.vlm import VLMExecutor, VLMGroupExecutor, vlm_host_batch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    mbs = args.mbs or 32
    bpr = args.batch_per_rank or 64
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        if args.layout == "colocated":
            ex = VLMExecutor(batch=bpr, mbs_llm=mbs, mbs_vit=args.vit_mbs, dp_group=dist.group.WORLD)
            layout = f"colocated vit+llm per GPU, both sections dp{world} (grad all-reduce)"
        else:
            ex = VLMGroupExecutor(world, batch_per_llm_rank=bpr, mbs_llm=mbs, mbs_vit=args.vit_mbs)
            layout = f"disjoint: vit dp{ex.dp_vit} (fanout {ex.f}) -> llm dp{ex.dp_llm}, {handoff_mode()} handoff (mq)"
    else:
        ex = VLMExecutor(batch=bpr, mbs_llm=mbs, mbs_vit=args.vit_mbs)
        layout = "colocated vit+llm"
    B = ex.batch
    hb = vlm_host_batch(B, seed=rank if (world > 1 and args.layout == "colocated") else 0)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # the VLM step is ~10 ms, so the sampler (200 ms period, ~100 ms start-up) already runs through
    # the warm-up steps to have samples under load
    clocks = ClockSampler(local)
    clocks.start()
    # the co-resident executor plans the next step's batch beside the current step (the batch of
    # step i+1 is known at step i, as with a prefetching loader)
    nxt = {"next_hb": hb}  # both executors plan the next batch beside the current step
    for _ in range(args.warmup):
        ex.step(hb, want_loss=False, **nxt)
    barrier()
    launches0 = instrument.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sts = []
    for _ in range(args.steps):
        sts.append(ex.step(hb, want_loss=False, **nxt))
    e1.record()
    barrier()
    launches = instrument.launches - launches0
    stalls = [x.stall_frac for x in sts]  # read after the timed region (lazy stats synchronise)
    clk = clocks.stop()
    t = torch.tensor([e0.elapsed_time(e1), max(stalls) if getattr(ex, "role", "llm") == "llm" else 0.0],
                     device="cuda")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t[0].item())
    B_all = B * world if (world > 1 and args.layout == "colocated") else B
    value = B_all * args.steps / (ms / 1e3)
    # ---- end-to-end, host wall clock: every step copies its inputs from pinned host memory and
    # the loss is read back every step
    barrier()
    w0 = time.perf_counter()
    losses = []
    for _ in range(args.steps):
        losses.append(ex.step(hb, want_loss=True, **nxt).loss)
    torch.cuda.synchronize()
    w1 = time.perf_counter()
    barrier()
    te = torch.tensor([(w1 - w0) * 1e3], device="cuda")
    if dist is not None:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = B_all * args.steps / (float(te.item()) / 1e3)
    # ---- per-kernel timing in one extra untimed step
    instrument.start_timing()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    ex.step(hb, want_loss=False, **nxt)
    s1.record()
    torch.cuda.synchronize()
    rec = instrument.stop_timing()
    serial_ms = s0.elapsed_time(s1)
    g_flops, g_ms, g_n = rec.get("gemm", (0.0, 0.0, 0))
    peaks, peak_kind = load_peaks()
    peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
    gt = g_flops / (g_ms / 1e3) / 1e12 if g_ms > 0 else None
    cpu = None
    if rank == 0 and args.gpus == 1 and not args.no_cpu_baseline:
        try:
            sec, threads = cpu_vlm_step_sample()
            cpu = {"value": 1.0 / sec, "unit": UNIT, "cores": threads, "kind": "port",
                   "sample": "8 samples: oracle/torch_ref.py fp32 VLM step on the host CPU"}
            try:
                cpu["scheduler"] = cpu_schedule_baseline(ex.planner)
            except Exception as exc:  # noqa: BLE001
                cpu["scheduler"] = {"error": repr(exc)}
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {exc}"}
    if rank == 0:
        from paper_2605_10501_b200.vlm import pinned_inputs

        pin = pinned_inputs(hb)
        h2d = sum(int(pin[k].numel() * pin[k].element_size()) for k in ("ids", "labels", "lens", "pixels"))
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": "vlm_cfg1: ViT-tiny (d192 L12) -> 2-layer GPT (d768), 50/50 text/image, "
                                   "wavefront schedule on device", "global_batch": B_all, "seq_len": "64..497",
                       "parallelism": layout, "micro_batch_llm": mbs, "micro_batch_vit": args.vit_mbs,
                       "l2": "inputs copied from pinned host memory every step (value and e2e alike)"},
            "section_stall_pct": 100.0 * float(t[1].item()),
            "gpu_launches": launches // max(args.steps, 1),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": (4 * (ex._h_orders.numel() + ex._h_off.numel()) + 8 + 4
                                           if hasattr(ex, "_h_orders") else None),
                    "timing": "host wall clock (perf_counter) around the steps, synchronised at both ends"},
            "roofline": {"bound": "tensor", "kernel": "maestro tcgen05 GEMM (csrc/gemm.cu)", "achieved": gt,
                         "peak": peak, "unit": "TFLOP/s", "frac": gt / peak if gt else None, "traffic": None,
                         "peak_kind": f"{peak_kind} bf16_tflops_sustained", "launches_timed": g_n,
                         "share_of_step": g_ms / serial_ms if serial_ms > 0 else None,
                         "note": "one extra untimed step; the tiny cfg 1 GEMMs (d 192/768) are launch-bound"},
            "model_tflops": ex.model_flops_per_step(hb) * (B_all // B) * args.steps / (ms / 1e3) / 1e12,
            "loss": losses[-1] if losses else None,
            "clocks": clk,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--batch-per-rank", type=int, default=None)
    ap.add_argument("--mbs", type=int, default=None,
                    help="student (KD) or LLM (VLM, default 32) micro-batch size")
    ap.add_argument("--vit-mbs", type=int, default=32,
                    help="VLM: ViT micro-batch (images); measured 8 -> 32 (with the LLM's): 1724 -> 4471 samples/s")
    ap.add_argument("--teacher-mbs", type=int, default=None,
                    help="teacher (forward-only) micro-batch size, a multiple of --mbs")
    ap.add_argument("--layout", default="colocated", choices=["colocated", "disjoint"])
    ap.add_argument("--trace", default=None, help="write the measured chrome trace of the last step here")
    ap.add_argument("--workload", default="kd", choices=["kd", "kd8b", "vlm", "section"],
                    help="kd = BASELINE configs[1] (default); kd8b = configs[4]; vlm = configs[0]; "
                         "section = generic section-graph executor (--graph)")
    ap.add_argument("--graph", default="vlm7b", choices=["vlm7b", "omni"],
                    help="--workload section: cfg 3 (vlm7b) or cfg 4 (omni) shapes")
    ap.add_argument("--layers", type=int, default=None, help="--workload section: layers per stack (reduced depth)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.workload == "vlm":
        run_vlm(args)
    elif args.workload == "section":
        from paper_2605_10501_b200.graph_bench import run_section

        run_section(args, METRIC, UNIT, ClockSampler, load_peaks)
    else:
        run_kd(args)


if __name__ == "__main__":
    main()
