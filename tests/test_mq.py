"""Reshard message queue (paper_2605_10501_b200/mq.py) vs the reference mq.py semantics.

CPU: plans against the reference's own plan_reshard outputs (tests/golden/reshard_golden.json,
bit-exact integer boxes), the oracle against the reference's apply_plan checksums, the
control-header codec, slot accounting, and a 2-process gloo run of DistTransport.
GPU (-m gpu): device apply_plan / push / pull against the oracle, the SPEC.md:427-449 examples
(round trip, FIFO, SlotExhausted on the (budget+1)-th push, FragmentTimeout, M=2 -> N=1 gather)
and a fuzz of random M-to-N reshards.
"""

import json
import os
import random
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import reshard_ref as R
from paper_2605_10501_b200 import errors as E
from paper_2605_10501_b200 import mq

GOLD = json.loads((Path(__file__).parent / "golden" / "reshard_golden.json").read_text())
PLANS = [c for c in GOLD if "src" in c]
LAYOUTS = [c for c in GOLD if "layout" in c]


def lay(d):
    return mq.ShardLayout(tuple(d["shape"]), d["tp"], d["cp"], d["tp_axis"], d["cp_axis"])


def checksum(v: np.ndarray) -> int:
    return int((v.astype(np.int64) * (1 + np.arange(v.size).reshape(v.shape))).sum())


@pytest.mark.parametrize("case", PLANS, ids=[f"plan{i}" for i in range(len(PLANS))])
def test_plan_matches_reference(case):
    if "error" in case:
        with pytest.raises(getattr(E, case["error"])):
            mq.plan_reshard(lay(case["src"]), lay(case["dst"]))
        return
    plan = mq.plan_reshard(lay(case["src"]), lay(case["dst"]))
    got = [[list(t.sender), list(t.receiver), [list(x) for x in t.sender_slice], [list(x) for x in t.receiver_slice]]
           for t in plan.transfers]
    assert got == case["transfers"]
    # plan completeness (SPEC.md invariant): receiver slices tile each destination shard once
    for r in plan.dst.ranks():
        cover = np.zeros(plan.dst.shard_shape(r), dtype=np.int32)
        for t in plan.for_receiver(r):
            cover[tuple(slice(a, b) for a, b in t.receiver_slice)] += 1
        assert (cover == 1).all()


@pytest.mark.parametrize("case", LAYOUTS, ids=[f"layout{i}" for i in range(len(LAYOUTS))])
def test_layout_validation_matches_reference(case):
    if "error" in case:
        with pytest.raises(getattr(E, case["error"])):
            lay(case["layout"])
    else:
        lay(case["layout"])


@pytest.mark.parametrize("case", [c for c in PLANS if "error" not in c][:40])
def test_oracle_pinned_to_reference_apply(case):
    """Both oracle restatements reproduce the reference's apply_plan on an arange tensor."""
    s, d = case["src"], case["dst"]
    full = np.arange(int(np.prod(s["shape"])), dtype=np.int64).reshape(s["shape"])
    sb = R.boxes(s["shape"], s["tp"], s["cp"], s["tp_axis"], s["cp_axis"])
    db = R.boxes(d["shape"], d["tp"], d["cp"], d["tp_axis"], d["cp_axis"])
    shards = {r: full[tuple(slice(a, b) for a, b in bx)] for r, bx in sb.items()}
    by_transfers = R.apply_ref(case["transfers"], {r: [b - a for a, b in bx] for r, bx in db.items()}, shards)
    by_elements = R.element_oracle(full, sb, db) if full.size <= 512 else by_transfers
    for key, (shape, ck) in case["receivers"].items():
        r = tuple(int(x) for x in key.split(","))
        assert list(by_transfers[r].shape) == shape and checksum(by_transfers[r]) == ck
        assert checksum(by_elements[r]) == ck


def test_header_roundtrip():
    m = mq.MessageMeta((2048, 2048), 2, "teacher", (1, 2), 77, 5)
    assert mq._decode_header(mq._encode_header(m)) == m
    assert m.nbytes == 2048 * 2048 * 2


def test_slot_budget_backpressure():
    b = mq.SlotBudget(capacity_bytes=100)
    b.reserve(60)
    b.reserve(40)
    with pytest.raises(E.SlotExhausted) as ei:
        b.reserve(1)
    assert ei.value.context == {"reserved": 100, "request": 1}
    b.release(40)
    b.reserve(40)
    assert b.peak_bytes == 100


def _gloo_worker(rank, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        src = mq.ShardLayout((6, 4), tp=2)
        dst = mq.ShardLayout((6, 4))
        plan = mq.plan_reshard(src, dst)
        full = torch.arange(24, dtype=torch.float32).reshape(6, 4)
        if rank == 0:  # both senders live in process 0
            chans = {(s, (0, 0)): mq.Channel(s, (0, 0), mq.DistTransport(peer=1)) for s in src.ranks()}
            for sample in (3, 4):
                for s in src.ranks():
                    mq.push_tensor(plan, chans, s, src.shard(full * sample, s), "teacher", sample)
            for c in chans.values():
                c.transport.flush()
            q.put(("ok", None))
        else:
            chans = {s: mq.Channel(s, (0, 0), mq.DistTransport(peer=0)) for s in src.ranks()}
            ep = mq.Endpoint((0, 0), plan, chans, torch.float32)
            out = []
            for sample in (3, 4):
                t, meta = ep.pull(validate=True)
                out.append((meta.sample_id, meta.section_name, bool(torch.equal(t, full * sample))))
            q.put(("ok", out))
    except Exception as e:  # noqa: BLE001
        q.put(("err", repr(e)))
    finally:
        dist.destroy_process_group()


def test_dist_transport_gloo_two_processes():
    import torch.multiprocessing as tmp

    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + random.Random(os.getpid()).randint(0, 2000)
    procs = [ctx.Process(target=_gloo_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    try:
        res = [q.get(timeout=90) for _ in procs]
    finally:
        for p in procs:
            p.join(timeout=20)
            if p.is_alive():
                p.kill()
    assert all(r[0] == "ok" for r in res), res
    pulled = [r[1] for r in res if r[1] is not None][0]
    assert pulled == [(3, "teacher", True), (4, "teacher", True)]


# ----------------------------------------------------------------------------------- GPU


@pytest.mark.gpu
@pytest.mark.parametrize("case", [c for c in PLANS if "error" not in c], ids=lambda c: str(c["src"]["shape"]))
def test_device_apply_plan_matches_reference(case):
    s, d = lay(case["src"]), lay(case["dst"])
    plan = mq.plan_reshard(s, d)
    full = torch.arange(int(np.prod(s.tensor_shape)), dtype=torch.int64, device="cuda").reshape(s.tensor_shape)
    res = mq.apply_plan(plan, {r: s.shard(full, r) for r in s.ranks()})
    for key, (shape, ck) in case["receivers"].items():
        r = tuple(int(x) for x in key.split(","))
        v = res[r].cpu().numpy()
        assert list(v.shape) == shape and checksum(v) == ck


@pytest.mark.gpu
def test_push_pull_roundtrip_fifo_and_gather():
    src, dst = mq.ShardLayout((8, 4), tp=2), mq.ShardLayout((8, 4))
    plan = mq.plan_reshard(src, dst)
    chans, eps = mq.connect(plan, dtype=torch.bfloat16)
    a = torch.randn(8, 4, device="cuda").bfloat16()
    b = torch.randn(8, 4, device="cuda").bfloat16()
    for sample, t in ((10, a), (11, b)):  # two tensors: pulled in sequence order
        for s in src.ranks():
            mq.push_tensor(plan, chans, s, src.shard(t, s), "vit", sample)
    ep = eps[(0, 0)]
    ta, ma = ep.pull()
    tb, mb = ep.pull()
    torch.cuda.synchronize()
    assert torch.equal(ta, a) and torch.equal(tb, b)  # M=2 -> N=1: concatenation along tp_axis
    assert (ma.sample_id, mb.sample_id) == (10, 11) and ma.section_name == "vit"
    assert all(c.budget.reserved_bytes == 0 for c in chans.values())
    assert chans[((0, 0), (0, 0))].budget.peak_bytes == 2 * 4 * 4 * 2 * 2  # two senders x two tensors in flight


@pytest.mark.gpu
def test_slot_exhausted_on_budget_plus_one_push():
    plan = mq.plan_reshard(mq.ShardLayout((4, 4)), mq.ShardLayout((4, 4)))
    k = 3
    chans, eps = mq.connect(plan, dtype=torch.float32, slot_budget_bytes=k * 64)
    ch = chans[((0, 0), (0, 0))]
    x = torch.ones(4, 4, device="cuda")
    for i in range(k):
        mq.push_tensor(plan, chans, (0, 0), x * i, "s", i)
    with pytest.raises(E.SlotExhausted):
        mq.push_tensor(plan, chans, (0, 0), x, "s", k)
    t, m = eps[(0, 0)].pull()  # releasing one slot re-opens the budget
    assert m.sample_id == 0 and m.sequence_number == 0
    mq.push_tensor(plan, chans, (0, 0), x, "s", k)
    assert ch.budget.reserved_bytes == k * 64


@pytest.mark.gpu
def test_timeout_and_closed_channel():
    src, dst = mq.ShardLayout((8, 4), tp=2), mq.ShardLayout((8, 4))
    plan = mq.plan_reshard(src, dst)
    chans, eps = mq.connect(plan, timeout=0.05)
    x = torch.zeros(4, 4, device="cuda")
    mq.push_tensor(plan, chans, (0, 0), x, "s", 0)  # sender (1, 0) never pushes
    with pytest.raises(E.FragmentTimeout) as ei:
        eps[(0, 0)].pull()
    assert ei.value.context["sender"] == "(1, 0)"
    ch = chans[((1, 0), (0, 0))]
    ch.close()
    with pytest.raises(E.ChannelClosed):
        mq.push_tensor(plan, chans, (1, 0), x, "s", 0)


@pytest.mark.gpu
def test_mismatched_fragment_streams_rejected():
    src, dst = mq.ShardLayout((8, 4), tp=2), mq.ShardLayout((8, 4))
    plan = mq.plan_reshard(src, dst)
    chans, eps = mq.connect(plan)
    x = torch.zeros(4, 4, device="cuda")
    mq.push_tensor(plan, chans, (0, 0), x, "s", 0)
    mq.push_tensor(plan, chans, (1, 0), x, "s", 1)  # a different sample
    with pytest.raises(E.IncompatibleShapes):
        eps[(0, 0)].pull()


@pytest.mark.gpu
def test_fuzz_random_reshards_vs_element_oracle():
    """Random M, N <= 4 layouts on 2-4 d tensors: pull at every receiver == element oracle."""
    rng = random.Random(11)
    n_done = 0
    while n_done < 150:
        nd = rng.choice([2, 3, 4])
        ta, ca = rng.sample(range(nd), 2)
        d = [rng.choice([1, 2, 3, 4]) for _ in range(4)]
        shape = [rng.choice([1, 2, 5]) for _ in range(nd)]
        shape[ta] *= int(np.lcm(d[0], d[2]))
        shape[ca] *= int(np.lcm(d[1], d[3]))
        if int(np.prod(shape)) > 3000:
            continue
        src = mq.ShardLayout(tuple(shape), d[0], d[1], ta, ca)
        dst = mq.ShardLayout(tuple(shape), d[2], d[3], ta, ca)
        plan = mq.plan_reshard(src, dst)
        dtype = rng.choice([torch.float32, torch.bfloat16, torch.int64, torch.uint8])
        full = torch.randint(0, 100, tuple(shape), device="cuda").to(dtype)
        chans, eps = mq.connect(plan, dtype=dtype)
        for s in src.ranks():
            mq.push_tensor(plan, chans, s, src.shard(full, s), "x", n_done)
        sb = R.boxes(shape, d[0], d[1], ta, ca)
        db = R.boxes(shape, d[2], d[3], ta, ca)
        ref = R.element_oracle(full.cpu().float().numpy(), sb, db) if full.numel() <= 400 else None
        for r in dst.ranks():
            got, meta = eps[r].pull()
            want = dst.shard(full, r)
            assert torch.equal(got, want), (shape, d, r)
            if ref is not None:
                assert np.array_equal(got.cpu().float().numpy(), ref[r])
        n_done += 1


@pytest.mark.gpu
def test_identity_plan_is_zero_copy_and_box_copy_strided():
    plan = mq.plan_reshard(mq.ShardLayout((64, 2048)), mq.ShardLayout((64, 2048)))
    chans, eps = mq.connect(plan, dtype=torch.bfloat16)
    x = torch.randn(64, 2048, device="cuda").bfloat16()
    tok = chans[((0, 0), (0, 0))].push(x, mq.MessageMeta((64, 2048), 2, "teacher", (0, 0), 5), donate=True)
    y, _ = eps[(0, 0)].pull()
    assert tok == 0 and y.data_ptr() == x.data_ptr()
    # 5-d strided box copy (non-contiguous on both sides)
    a = torch.randn(3, 4, 5, 6, 7, device="cuda")
    b = torch.zeros(6, 8, 10, 12, 14, device="cuda")
    mq.box_copy(a.permute(0, 2, 1, 3, 4)[:, 1:4, :, ::2], b[1:4, 2:5, 3:7, 0:3, 5:12])
    torch.cuda.synchronize()
    assert torch.equal(b[1:4, 2:5, 3:7, 0:3, 5:12], a.permute(0, 2, 1, 3, 4)[:, 1:4, :, ::2])


@pytest.mark.gpu
@pytest.mark.timeout(60)
def test_peer_transport_ring_protocol_on_one_gpu():
    """PeerTransport's slot ring (flags, credits, copy-engine puts, stream memory ops) through an
    in-process pair: six messages through two slots, pushed on one stream and pulled on another,
    so later pushes wait (in-stream) for the receiver to release slots."""
    src = mq.ShardLayout((64, 256))
    plan = mq.plan_reshard(src, src)
    tx, rx = mq.PeerTransport.local_pair(slot_bytes=64 * 256 * 2, slots=2)
    ch_tx = mq.Channel((0, 0), (0, 0), tx)
    ch_rx = mq.Channel((0, 0), (0, 0), rx)
    ep = mq.Endpoint((0, 0), plan, {(0, 0): ch_rx}, torch.bfloat16)
    s_push, s_pull = torch.cuda.Stream(), torch.cuda.Stream()
    xs = [torch.randn(64, 256, device="cuda").bfloat16() for _ in range(6)]
    torch.cuda.synchronize()
    with torch.cuda.stream(s_push):
        for i, x in enumerate(xs):
            ch_tx.push(x, mq.MessageMeta((64, 256), 2, "teacher", (0, 0), 100 + i))
    got = []
    with torch.cuda.stream(s_pull):
        for _ in xs:
            got.append(ep.pull(validate=False)[0])
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(got, xs))
    assert [m.sample_id for m in ep.verify()] == [100 + i for i in range(6)]
    with pytest.raises(E.SlotExhausted):
        ch_tx.push(torch.zeros(65, 256, device="cuda").bfloat16(), mq.MessageMeta((65, 256), 2, "t", (0, 0), 0))
    rx.close()


def _peer_worker(rank, port, q):
    """Two processes on cuda:0: rank 0 pushes six messages through a two-slot PeerTransport ring
    (IPC-mapped slots, cross-process credits), rank 1 pulls them on its own stream."""
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        torch.cuda.set_device(0)
        layout = mq.ShardLayout((64, 256))
        plan = mq.plan_reshard(layout, layout)
        g = torch.Generator().manual_seed(7)
        xs = [torch.randn(64, 256, generator=g).bfloat16() for _ in range(6)]
        if rank == 0:
            tx = mq.PeerTransport(peer=1, role="send", slot_bytes=64 * 256 * 2, slots=2)
            ch = mq.Channel((0, 0), (0, 0), tx)
            for i, x in enumerate(xs):
                ch.push(x.cuda(), mq.MessageMeta((64, 256), 2, "teacher", (0, 0), 100 + i))
            torch.cuda.synchronize()
            dist.barrier()  # the receiver has copied everything out before the sender frees
            tx.close()
            q.put(("ok", None))
        else:
            rx = mq.PeerTransport(peer=0, role="recv", slot_bytes=64 * 256 * 2, slots=2)
            ep = mq.Endpoint((0, 0), plan, {(0, 0): mq.Channel((0, 0), (0, 0), rx)}, torch.bfloat16)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                got = [ep.pull(validate=False)[0] for _ in xs]
            torch.cuda.synchronize()
            ids = [m.sample_id for m in ep.verify()]
            ok = all(torch.equal(a.cpu(), b) for a, b in zip(got, xs))
            dist.barrier()
            rx.close()
            q.put(("ok", (ok, ids)))
    except Exception as e:  # noqa: BLE001
        q.put(("err", repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_peer_transport_two_processes_one_gpu():
    """The cross-process PeerTransport path (IPC handle exchange over the process group, slot
    ring in the receiver's memory, credits in the sender's) between two processes sharing one
    GPU, so it runs on a single-GPU box; the ring has two slots for six messages, so the sender's
    later puts wait in-stream for the receiver's credits."""
    import torch.multiprocessing as tmp

    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = 31500 + random.Random(os.getpid()).randint(0, 2000)
    procs = [ctx.Process(target=_peer_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    try:
        res = [q.get(timeout=180) for _ in procs]
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    assert all(r[0] == "ok" for r in res), res
    ok, ids = [r[1] for r in res if r[1] is not None][0]
    assert ok and ids == [100 + i for i in range(6)]
