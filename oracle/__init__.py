"""ORACLE -- test infrastructure only.

CPU restatement of the reference scheduler (``maestro/scheduling.py``) and of
the reference's activation resolution (``maestro/workload.py:297-355``), used
as the checker by ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs.  The product package never
imports this module.

Pinning: every function here is checked against golden vectors produced by
running the reference itself (``tests/golden/make_golden.py``); see
``tests/test_oracle_golden.py``.

The arithmetic lives in ``sched_oracle.c`` (plain C, no FP contraction) so
the port is fast enough to also serve as the CPU baseline.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "lib" / "libsched_oracle.so"
_lib = None

POLICIES = {"interleaved": 0, "all-fwd-then-bwd": 1}


def build() -> Path:
    """Compile the C oracle (checker only)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(_LIB_PATH))
        dp, ip, lp = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_longlong)
        L.oracle_rank_metrics.restype = ctypes.c_double
        L.oracle_rank_metrics.argtypes = [dp, ctypes.c_int, ip, ctypes.c_int, ctypes.c_int, dp, dp, dp]
        L.oracle_schedule_rank.restype = ctypes.c_longlong
        L.oracle_schedule_rank.argtypes = [dp, ctypes.c_int, ip, ctypes.c_int, ctypes.c_int, ip]
        L.oracle_partition.restype = ctypes.c_int
        L.oracle_partition.argtypes = [dp, ip, ip, ip, ctypes.c_int, ctypes.c_int, ctypes.c_int, ip, ip, ip, ip]
        L.oracle_build_schedule.restype = ctypes.c_int
        L.oracle_build_schedule.argtypes = [
            dp, ip, ip, ip, ctypes.c_int, ctypes.c_int, ctypes.c_int, ip, ip, ip, ip,
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ip, ip, ip, lp, ip,
        ]
        _lib = L
    return _lib


def _d(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _i(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))


def times_array(tuples) -> np.ndarray:
    """[B] 6-tuples -> phase-major float64 [6, B]; -0.0 canonicalised to +0.0."""
    t = np.ascontiguousarray(np.asarray(tuples, dtype=np.float64).reshape(-1, 6).T) + 0.0
    return np.ascontiguousarray(t)


def rank_metrics(times: np.ndarray, order, policy="interleaved"):
    """scheduling.py:81-152 -> (makespan, critical_busy, critical_span)."""
    B = times.shape[1]
    o = np.ascontiguousarray(order, dtype=np.int32)
    busy, span = np.zeros(1), np.zeros(1)
    scratch = np.zeros(2 * max(len(o), 1) + 2)
    mk = lib().oracle_rank_metrics(_d(times), B, _i(o), len(o), POLICIES[policy], _d(busy), _d(span), _d(scratch))
    return mk, float(busy[0]), float(span[0])


def schedule_rank(times: np.ndarray, order, policy="interleaved"):
    """scheduling.py:162-199 -> (new order of batch indices, evaluation count)."""
    B = times.shape[1]
    o = np.ascontiguousarray(order, dtype=np.int32)
    out = np.zeros(max(len(o), 1), dtype=np.int32)
    ev = lib().oracle_schedule_rank(_d(times), B, _i(o), len(o), POLICIES[policy], _i(out))
    return out[: len(o)].tolist(), int(ev)


def partition(times: np.ndarray, ids, up_sec, down_sec, dp: int, n_sec: int):
    """scheduling.py:202-264 -> (list of per-rank batch-index lists, LPT order)."""
    B = times.shape[1]
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    up = np.ascontiguousarray(up_sec, dtype=np.int32)
    down = np.ascontiguousarray(down_sec, dtype=np.int32)
    lists = np.zeros(max(B, 1), dtype=np.int32)
    offs = np.zeros(max(dp, 1), dtype=np.int32)
    cnts = np.zeros(max(dp, 1), dtype=np.int32)
    lpt = np.zeros(max(B, 1), dtype=np.int32)
    rc = lib().oracle_partition(_d(times), _i(ids), _i(up), _i(down), B, dp, max(n_sec, 1),
                                _i(lists), _i(offs), _i(cnts), _i(lpt))
    if rc:
        raise RuntimeError(f"oracle partition error {rc}")
    return [lists[offs[r]: offs[r] + cnts[r]].tolist() for r in range(dp)], lpt[:B].tolist()


def merge_fanout(lists, fanout):
    """scheduling.py:267-285 (pure Python; tiny)."""
    if fanout < 1 or len(lists) != fanout:
        raise ValueError("fanout mismatch")
    out = []
    for i in range(max((len(x) for x in lists), default=0)):
        for x in lists:
            if i < len(x):
                out.append(x[i])
    return out


MAX_SECTIONS = 16


def resolve(act_masks, times: np.ndarray, sub_owner, side, up_candidates, down_candidates,
            parallel_upstream: bool = False):
    """workload.py:297-355 over submodule bitmasks (bit order = sorted names).

    Returns (up_sec, down_sec) arrays of section indices (-1 = none) or raises
    ``ValueError((code, batch_index))`` with the reference's error: 2 =
    BothActivated, 3 = ActivationError.  ``parallel_upstream`` (extension, not in the
    reference): several upstream sections resolve to MAX_SECTIONS + their section mask.
    """
    B = times.shape[1]
    up_out = np.full(B, -1, dtype=np.int32)
    down_out = np.full(B, -1, dtype=np.int32)
    for i in range(B):
        m = int(act_masks[i])
        seen = {}
        ups, downs = [], []
        for bit in range(len(sub_owner)):
            if not (m >> bit) & 1:
                continue
            o = sub_owner[bit]
            if seen.setdefault(o, bit) != bit:
                raise ValueError((2, i))
            if side[o] == 0:
                ups.append(o)
            elif side[o] == 2:
                downs.append(o)
        if (len(set(ups)) > 1 and not parallel_upstream) or len(set(downs)) > 1:
            raise ValueError((3, i))
        up_t = times[0, i] + times[5, i]
        down_t = times[2, i] + times[3, i]
        for t_side, decl, pool, out in ((up_t, ups, up_candidates, up_out), (down_t, downs, down_candidates, down_out)):
            if t_side <= 0:
                continue
            if len(set(decl)) > 1:
                out[i] = MAX_SECTIONS + sum(1 << x for x in set(decl))
            elif decl:
                out[i] = decl[0]
            elif len(pool) == 1:
                out[i] = pool[0]
            else:
                raise ValueError((3, i))
    return up_out, down_out


def build_schedule(times, ids, up_sec, down_sec, n_sec, critical, dp, fanout, neighbor, merge_order,
                   policy="interleaved"):
    """scheduling.py:309-373 -> ({(section_index, rank): [batch indices]}, evals)."""
    B = times.shape[1]
    max_dp = max(dp)
    arr = lambda x: np.ascontiguousarray(x, dtype=np.int32)
    ids, up, down = arr(ids), arr(up_sec), arr(down_sec)
    dpa, fa, nba, mo = arr(dp), arr(fanout), arr(neighbor), arr(list(merge_order) or [0])
    orders = np.zeros(n_sec * B, dtype=np.int32)
    off = np.zeros(n_sec * max_dp, dtype=np.int32)
    cnt = np.zeros(n_sec * max_dp, dtype=np.int32)
    ev = ctypes.c_longlong(0)
    bad = ctypes.c_int(-1)
    rc = lib().oracle_build_schedule(
        _d(times), _i(ids), _i(up), _i(down), B, n_sec, critical, _i(dpa), _i(fa), _i(nba), _i(mo),
        len(merge_order), POLICIES[policy], max_dp, _i(orders), _i(off), _i(cnt), ctypes.byref(ev),
        ctypes.byref(bad),
    )
    if rc:
        raise ValueError((rc, bad.value))
    out = {}
    for s in range(n_sec):
        if s != critical and s not in merge_order:
            continue
        for q in range(dp[s]):
            o, c = off[s * max_dp + q], cnt[s * max_dp + q]
            out[(s, q)] = orders[s * B + o: s * B + o + c].tolist()
    return out, int(ev.value)


def sample_times(cost, tokens, sub_owner, side, crit_bit, parallel_upstream=False):
    """K1 restatement (costs.py:105-123 estimate_step_time, :182-200 per_sample_times, :264-286
    derive_batch's per-side sums) over the device cost table [n_bits, 8] and token counts
    [n_bits, B] -> (times [6, B] phase-major, activation masks [B]).  ``parallel_upstream``
    (extension, not in the reference): the upstream phases are the max over the activated
    upstream sections instead of their sum (identical when at most one is activated)."""
    cost = np.asarray(cost, dtype=np.float64)
    tokens = np.asarray(tokens, dtype=np.int64)
    n_bits, B = tokens.shape
    crit_owner = sub_owner[crit_bit]
    act = np.zeros(B, dtype=np.uint32)
    cnt = {}
    for i in range(B):
        secs = set()
        for b in range(n_bits):
            if sub_owner[b] == crit_owner:
                continue
            if tokens[b, i] > 0:
                act[i] |= np.uint32(1 << b)
                secs.add(sub_owner[b])
        for s_ in secs:
            cnt[s_] = cnt.get(s_, 0) + 1

    def pst(row, tok, n):
        fpt, eff, ratio, fwd_only, mbs, pp = row[0], row[1], row[2], row[3] != 0.0, int(row[4]), int(row[5])
        if n <= 0:
            return 0.0, 0.0
        fwd = float(mbs * int(tok)) * fpt / eff
        bwd = 0.0 if fwd_only else fwd * ratio
        m = (n + mbs - 1) // mbs
        sc = float(m + pp - 1) / float(m * pp * mbs)
        return fwd * sc, bwd * sc

    times = np.zeros((6, B), dtype=np.float64)
    crow = cost[crit_bit]
    dpc = int(crow[6])
    n_crit = (B + dpc - 1) // dpc
    for i in range(B):
        t = [0.0] * 6
        t[1], t[4] = pst(crow, tokens[crit_bit, i], n_crit)
        upf, upb = {}, {}
        for b in range(n_bits):
            if not (int(act[i]) >> b) & 1:
                continue
            s_ = sub_owner[b]
            row = cost[b]
            dps = int(row[6])
            n_aux = (cnt[s_] + dps - 1) // dps if cnt.get(s_, 0) > 0 else 0
            f, bw = pst(row, tokens[b, i], n_aux)
            if side[s_] == 0 and parallel_upstream:
                upf[s_] = upf.get(s_, 0.0) + f
                upb[s_] = upb.get(s_, 0.0) + bw
            elif side[s_] == 0:
                t[0] += f
                t[5] += bw
            else:
                t[2] += f
                t[3] += bw
        for s_ in sorted(upf):
            t[0] = upf[s_] if upf[s_] > t[0] else t[0]
            t[5] = upb[s_] if upb[s_] > t[5] else t[5]
        times[:, i] = [x + 0.0 for x in t]
    return times, act


def cpu_count() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
