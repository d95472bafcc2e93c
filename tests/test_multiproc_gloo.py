"""N>1 host logic on CPU with gloo (world size 2, 4 and 8): every rank derives the same device-free
placement, the teacher->student handoff pairs match on both ends, payloads arrive intact in
schedule order, and the student DP all-reduce covers exactly the student ranks."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, layout, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_10501_b200.executor import rank_roles

        roles = rank_roles(rank, world, layout)
        everyone = [None] * world
        dist.all_gather_object(everyone, roles)
        # consistency: every send has a matching recv on the peer
        for r, ro in enumerate(everyone):
            for dst in ro["send_to"]:
                assert r in everyone[dst]["recv_from"]
        # handoff: teacher rank streams 3 micro-batches of "hidden states" to its student rank(s)
        n_mb, T, d = 3, 5, 4
        got = []
        for m in range(n_mb):
            for dst in roles["send_to"]:
                dist.send(torch.full((T, d), float(100 * rank + m)), dst)
            for src in roles["recv_from"]:
                buf = torch.empty(T, d)
                dist.recv(buf, src)
                got.append(float(buf[0, 0]))
        if roles["recv_from"]:
            assert got == [100.0 * roles["recv_from"][0] + m for m in range(n_mb)]
        # per-section gradient all-reduce over the student DP group only
        s_ranks = roles["student_ranks"]
        grp = dist.new_group(s_ranks)
        if roles["s_rank"] is not None:
            g = torch.tensor([float(rank + 1)])
            dist.all_reduce(g, group=grp)
            assert g.item() == sum(r + 1 for r in s_ranks)
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,layout", [(2, "disjoint"), (4, "disjoint"), (8, "disjoint"), (2, "colocated"),
                                          (4, "colocated"), (8, "colocated")])
def test_handoff_and_group_allreduce(world, layout):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, layout, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res


def _vlm_worker(rank, world, port, q):
    """VLM disjoint layouts (recipes.VLM_LAYOUTS: 2 = 1+1, 4 = ViT 1 (fan-out 3) + LLM 3, 8 = ViT 2
    (fan-out 3) + LLM 6): every LLM rank r pairs with ViT rank r // f (scheduling.py:366-369), the
    forward message reaches it and the gradient comes back; per-section all-reduce per group."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_10501_b200 import recipes as R

        dp_llm, dp_vit, f = R.VLM_LAYOUTS[world]
        assert dp_llm + dp_vit == world and dp_vit * f == dp_llm
        role = "vit" if rank < dp_vit else "llm"
        if role == "vit":
            peers = [dp_vit + r for r in range(dp_llm) if r // f == rank]
            for p in peers:
                dist.send(torch.full((3,), float(rank)), p)
            back = []
            for p in peers:
                b = torch.empty(3)
                dist.recv(b, p)
                back.append(float(b[0]))
            assert back == [float(p) for p in peers]
        else:
            r = rank - dp_vit
            b = torch.empty(3)
            dist.recv(b, r // f)
            assert float(b[0]) == r // f
            dist.send(torch.full((3,), float(rank)), r // f)
        groups = [dist.new_group(list(range(dp_vit))), dist.new_group(list(range(dp_vit, world)))]
        g = torch.tensor([1.0])
        dist.all_reduce(g, group=groups[0 if role == "vit" else 1])
        assert g.item() == (dp_vit if role == "vit" else dp_llm)
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_vlm_fanout_layouts(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_vlm_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res
