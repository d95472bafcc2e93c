"""bench.py --workload section: the generic section-graph executor on cfg 3 (--graph vlm7b) and
cfg 4 (--graph omni) shapes, one JSON line with the contract's keys (value, e2e, roofline,
cpu_baseline, clocks, gpu_launches, section stall).

Depth: ``--layers L`` runs every stack at L layers (default 4) with the full widths, head layouts,
vocabulary and sequence-length distributions; a 7.6B backbone with fp32 master weights, gradients
and Adam moments does not fit one GPU next to its activations, so the line says which depth ran.
"""

from __future__ import annotations

import json
import os
import time


def _flops_per_step(ex, gb) -> float:
    """Algorithmic model FLOPs of one step (unpadded shapes; training = 3x forward)."""
    tot = 0.0
    for name, sh in ex.shapes.items():
        mod = ex.mod[name]
        mult = 3.0 if mod.trainable else 1.0
        if name == ex.crit:
            toks = gb.lens
            with_head = True
        elif name in gb.up:
            toks = gb.up[name].in_len
            with_head = False
        else:
            toks = gb.down[name].rows
            with_head = True
        for t in toks:
            t = int(t)
            if t:
                tot += mult * t * sh.fwd_flops_per_token(t, with_head=with_head)
    return tot


def _cpu_sample(graph: str, layers_full: int):
    """Oracle fp32 step on the host CPU, bounded: 2 samples at full width through 1 layer per stack
    and through 0 layers, extrapolated to `layers_full` layers per stack."""
    import dataclasses

    import torch

    from oracle import torch_ref as R

    from . import graph_workloads as W

    torch.set_num_threads(os.cpu_count() or 1)
    g = torch.Generator().manual_seed(0)

    def flat(shape, extra):
        import math

        n = sum(((math.prod(s) + 63) // 64 * 64) for _, s in list(shape.param_shapes()) + extra)
        return torch.randn(n, generator=g) * 0.02

    def run(L):
        d = lambda s: dataclasses.replace(s, layers=L)  # noqa: E731
        if graph == "vlm7b":
            vit, llm = d(W.QWEN_VIT), d(W.QWEN_7B)
            gb = W.vlm7b_batch(2, seed=1, vocab=llm.vocab, patch_dim=W.PATCH_DIM, lo=1024, hi=1024)  # 1 image + 1 text
            ups = {"vit": (vit, flat(vit, [("in_w", (vit.d, W.PATCH_DIM)), ("proj_w", (llm.d, 4 * vit.d))]),
                           W.PATCH_DIM, 4)}
            downs = {}
        else:
            vit, aud, llm, dec = d(W.QWEN_VIT), d(W.WHISPER_ENC), d(W.QWEN_7B), d(W.AUDIO_DEC)
            gb = W.omni_batch(3, seed=1, vocab=llm.vocab, patch_dim=W.PATCH_DIM, n_codes=dec.vocab)
            ups = {"image_enc": (vit, flat(vit, [("in_w", (vit.d, W.PATCH_DIM)), ("proj_w", (llm.d, 4 * vit.d))]),
                                 W.PATCH_DIM, 4),
                   "audio_enc": (aud, flat(aud, [("in_w", (aud.d, W.MEL_DIM)), ("proj_w", (llm.d, 4 * aud.d))]),
                                 W.MEL_DIM, 4)}
            downs = {"audio_dec": (dec, flat(dec, [("in_w", (dec.d, llm.d))]), llm.d)}
        crit = (llm, flat(llm, []))
        t0 = time.perf_counter()
        R.graph_step_reference(crit, ups, downs, gb)
        return time.perf_counter() - t0, gb.B

    t1, B = run(1)
    t0, _ = run(0)
    per = t0 + layers_full * (t1 - t0)
    return B / per, torch.get_num_threads(), (
        f"{B} samples of the {graph} workload (oracle/torch_ref.graph_step_reference, fp32) through 1 and 0 layers "
        f"per stack at full width, extrapolated to {layers_full} layers: {t0:.2f} s + {layers_full} x {t1 - t0:.2f} s")


def run_section(args, METRIC, UNIT, ClockSampler, load_peaks):
    import torch

    from . import graph_workloads as W
    from . import instrument

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    layers = args.layers or 4
    bpr = args.batch_per_rank or 8
    B = bpr * world
    if args.graph == "vlm7b":
        ex = W.vlm7b_executor(n_gpus=world, layers=layers, mbs_llm=args.mbs or 1, mbs_vit=4,
                              dp_group=dist.group.WORLD if dist else None)
        gb = W.vlm7b_batch(B, seed=0, vocab=W.QWEN_7B.vocab, patch_dim=W.PATCH_DIM)
        workload = (f"vlm7b_cfg3: Qwen2.5-VL-7B-shaped ViT (d1280, 16x80 heads padded to 128, SwiGLU 3420) -> "
                    f"Qwen2.5-7B-shaped backbone (d3584, GQA 28/4, V 152064) at {layers} layers per stack; "
                    f"50% images with U{{256..4096}} patches")
    else:
        ex = W.omni_executor(n_gpus=world, layers=layers, mbs_llm=args.mbs or 1, mbs_enc=4,
                             dp_group=dist.group.WORLD if dist else None)
        gb = W.omni_batch(B, seed=0, vocab=W.QWEN_7B.vocab, patch_dim=W.PATCH_DIM, n_codes=W.AUDIO_DEC.vocab)
        workload = (f"omni_cfg4: image encoder (cfg 3 ViT) + audio encoder (Whisper-large-v3 shape) -> 7B backbone "
                    f"-> audio decoder (d1024), text/img/audio mix, {layers} layers per stack")

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        ex.step(gb, want_loss=False)
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = instrument.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stalls = []
    e0.record()
    for _ in range(args.steps):
        stalls.append(ex.step(gb, want_loss=False).stall_frac)
    e1.record()
    barrier()
    launches = instrument.launches - launches0
    clk = clocks.stop()
    t = torch.tensor([e0.elapsed_time(e1), max(stalls)], device="cuda")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t[0].item())
    value = B * args.steps / (ms / 1e3)
    # e2e: host wall clock; every step uploads its inputs from host memory and reads the loss
    barrier()
    w0 = time.perf_counter()
    losses = [ex.step(gb, want_loss=True).loss for _ in range(args.steps)]
    torch.cuda.synchronize()
    w1 = time.perf_counter()
    te = torch.tensor([(w1 - w0) * 1e3], device="cuda")
    if dist is not None:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e = B * args.steps / (float(te.item()) / 1e3)
    # per-kernel timing on one extra untimed step
    instrument.start_timing()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    ex.step(gb, want_loss=False)
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
            v, cores, desc = _cpu_sample(args.graph, layers)
            cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": desc}
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {exc}"}
    if rank == 0:
        h2d = int(gb.lens.nbytes + gb.ids.nbytes + (gb.labels.nbytes if gb.labels is not None else 0)
                  + sum(u.feats.nbytes // 2 + 3 * u.in_len.nbytes for u in gb.up.values() if u.feats is not None)
                  + sum(d.targets.nbytes + 2 * d.rows.nbytes for d in gb.down.values()))
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": workload, "global_batch": B, "seq_len": f"{int(gb.lens.min())}..{int(gb.lens.max())}",
                       "layers_per_stack": layers, "parallelism": f"co-located: every section dp{world} (fan-out 1)",
                       "executor": "graph_exec.SectionGraphExecutor", "policy": ex.policy.value,
                       "l2": "inputs larger than L2 (weights and activations of 4-layer 7B-width stacks)"},
            "section_stall_pct": 100.0 * float(t[1].item()),
            "gpu_launches": launches // max(args.steps, 1),
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": None,
                    "timing": "host wall clock (perf_counter) around the steps, synchronised at both ends"},
            "roofline": {"bound": "tensor", "kernel": "maestro tcgen05 GEMM (csrc/gemm.cu)", "achieved": gt,
                         "peak": peak, "unit": "TFLOP/s", "frac": gt / peak if gt else None, "traffic": None,
                         "peak_kind": f"{peak_kind} bf16_tflops_sustained", "launches_timed": g_n,
                         "share_of_step": g_ms / serial_ms if serial_ms > 0 else None,
                         "note": "one extra untimed step; sections on separate streams may overlap"},
            "model_tflops": _flops_per_step(ex, gb) * args.steps / (ms / 1e3) / 1e12,
            "loss": losses[-1] if losses else None,
            "clocks": clk,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
