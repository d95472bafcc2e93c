"""Diagnostic: PeerTransport between two processes sharing cuda:0 (gloo group), with progress
prints and a traceback dump if a rank stalls.  Usage: python scripts/peer_same_gpu.py"""
import faulthandler
import os
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def worker(rank, port):
    import torch.distributed as dist
    from paper_2605_10501_b200 import mq

    log = open(ROOT / "gpurun_out" / f"peer_rank{rank}.log", "w", buffering=1)
    faulthandler.dump_traceback_later(90, exit=True, file=log)
    p = lambda *a: print(f"[{rank} {time.time():.2f}]", *a, file=log, flush=True)  # noqa: E731
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    torch.cuda.set_device(0)
    p("init")
    layout = mq.ShardLayout((64, 256))
    plan = mq.plan_reshard(layout, layout)
    g = torch.Generator().manual_seed(7)
    xs = [torch.randn(64, 256, generator=g).bfloat16() for _ in range(6)]
    if rank == 0:
        tx = mq.PeerTransport(peer=1, role="send", slot_bytes=64 * 256 * 2, slots=2)
        p("transport")
        ch = mq.Channel((0, 0), (0, 0), tx)
        for i, x in enumerate(xs):
            ch.push(x.cuda(), mq.MessageMeta((64, 256), 2, "teacher", (0, 0), 100 + i))
            p("pushed", i)
        torch.cuda.synchronize()
        p("synced")
        dist.barrier()
        tx.close()
    else:
        rx = mq.PeerTransport(peer=0, role="recv", slot_bytes=64 * 256 * 2, slots=2)
        p("transport")
        ep = mq.Endpoint((0, 0), plan, {(0, 0): mq.Channel((0, 0), (0, 0), rx)}, torch.bfloat16)
        s = torch.cuda.Stream()
        got = []
        with torch.cuda.stream(s):
            for i in range(len(xs)):
                got.append(ep.pull(validate=False)[0])
                p("pulled", i)
        torch.cuda.synchronize()
        p("synced", all(torch.equal(a.cpu(), b) for a, b in zip(got, xs)), [m.sample_id for m in ep.verify()])
        dist.barrier()
        rx.close()
    p("done")
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as tmp

    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    ctx = tmp.get_context("spawn")
    procs = [ctx.Process(target=worker, args=(r, 31777)) for r in range(2)]
    for q in procs:
        q.start()
    for q in procs:
        q.join(timeout=150)
        if q.is_alive():
            q.kill()
    print("exitcodes", [q.exitcode for q in procs])
