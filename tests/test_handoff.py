"""K5b handoff (scatter) indices: device kernel == numpy oracle, bit-exact (north_star item 2)."""

import numpy as np
import pytest
import torch

from oracle import handoff_ref as H


def test_oracle_known_answer():
    """Two samples with images in a 3-sample consumer order, micro-batches of 2: rows land at the
    placeholder offset inside each micro-batch; producer rows follow the producer order."""
    lens = {0: 10, 1: 7, 2: 12}
    rows = np.array([3, 0, 2])
    dst_off = np.array([4, 0, 1])
    crit = [2, 1, 0]
    up = [0, 2]                       # producer order (fan-out merged)
    tok = H.varlen_offsets(crit, lens)  # [0, 12, 19]
    pos, src, dst = H.handoff_index(up, crit, tok, 2, rows, dst_off)
    assert pos.tolist() == [0, 2, 2, 5]
    assert src.tolist() == [3, 4, 0, 1, 2]          # sample 2 -> producer rows 3,4; sample 0 -> 0,1,2
    assert dst.tolist() == [1, 2, 4, 5, 6]          # mb0: 0 + 1; mb1 starts at sample 0: 0 + 4


def test_oracle_missing_producer_raises():
    with pytest.raises(KeyError):
        H.handoff_index([0], [0, 1], [0, 5], 2, np.array([1, 1]), np.array([0, 0]))


def _case(rng, B, mbs, p_img):
    lens = rng.integers(1, 600, B)
    has = rng.random(B) < p_img
    rows = np.where(has, rng.integers(1, 300, B), 0)
    rows = np.minimum(rows, lens)
    dst_off = np.array([rng.integers(0, lens[i] - rows[i] + 1) for i in range(B)])
    crit = rng.permutation(B)
    up = rng.permutation(np.nonzero(has)[0])
    return lens, rows, dst_off, crit, up


@pytest.mark.gpu
@pytest.mark.parametrize("B,mbs,p", [(1, 1, 1.0), (64, 8, 0.5), (300, 7, 0.3), (2048, 32, 0.9), (17, 4, 0.0)])
def test_device_matches_oracle(B, mbs, p):
    from paper_2605_10501_b200 import _native as N
    from paper_2605_10501_b200.handoff import handoff_index

    rng = np.random.default_rng(B * 31 + mbs)
    lens, rows, dst_off, crit, up = _case(rng, B, mbs, p)
    tok = H.varlen_offsets(crit, lens)
    want = H.handoff_index(up, crit, tok, mbs, rows, dst_off)
    d = lambda a: torch.tensor(np.asarray(a, dtype=np.int32), device="cuda")  # noqa: E731
    err = torch.full((1,), N.ERR_CLEAN, dtype=torch.int64, device="cuda")
    ix = handoff_index(d(up), d(crit), d(tok), mbs, d(rows), d(dst_off), int(rows.sum()), int(rows.sum()), err)
    R = int(want[0][-1])
    assert ix.pos.cpu().numpy().tolist() == want[0].tolist()
    assert ix.src[:R].cpu().numpy().tolist() == want[1].tolist()
    assert ix.dst[:R].cpu().numpy().tolist() == want[2].tolist()
    assert int(err.item()) == N.ERR_CLEAN


@pytest.mark.gpu
def test_scatter_range_moves_rows_and_back():
    from paper_2605_10501_b200.handoff import handoff_index, scatter_mb

    rng = np.random.default_rng(5)
    B, mbs, d = 40, 6, 256
    lens, rows, dst_off, crit, up = _case(rng, B, mbs, 0.6)
    tok = H.varlen_offsets(crit, lens)
    pos, src, dst = H.handoff_index(up, crit, tok, mbs, rows, dst_off)
    dv = lambda a: torch.tensor(np.asarray(a, dtype=np.int32), device="cuda")  # noqa: E731
    buf = torch.randn(int(rows.sum()), d, device="cuda").bfloat16()
    mb_rows = [int(pos[min(B, (m + 1) * mbs)] - pos[m * mbs]) for m in range(-(-B // mbs))]
    ix = handoff_index(dv(up), dv(crit), dv(tok), mbs, dv(rows), dv(dst_off), int(rows.sum()), max(mb_rows))
    for m in range(-(-B // mbs)):
        k0, k1 = m * mbs, min(B, (m + 1) * mbs)
        T = int(sum(lens[i] for i in crit[k0:k1]))
        x = torch.zeros(T, d, device="cuda", dtype=torch.bfloat16)
        scatter_mb(ix, m, buf, x)
        a, b = pos[k0], pos[k1]
        ref = torch.zeros_like(x)
        if b > a:
            ref[torch.from_numpy(dst[a:b]).long().cuda()] = buf[torch.from_numpy(src[a:b]).long().cuda()]
        assert torch.equal(x, ref)
        back = torch.zeros_like(buf)
        scatter_mb(ix, m, x, back, reverse=True)
        if b > a:
            sel = torch.from_numpy(src[a:b]).long().cuda()
            assert torch.equal(back[sel], buf[sel])
