"""ORACLE -- test infrastructure only.

numpy restatement of the K5b handoff (scatter) indices (csrc/handoff.cu): encoder output rows
are placed at each sample's placeholder rows inside the consumer's packed varlen stream -- the
paper's "4:1 downsampled visual tokens concatenated with the text tokens".
The reference has no data path, so this is unpinned by it; it is pinned to the reference's own
schedule semantics through the orders it consumes (scheduling.py:288-373) and to the cfg 1
executor's former host-side construction (vlm.py, round 1).  Never imported by the product.
"""

from __future__ import annotations

import numpy as np


def varlen_offsets(order, lens):
    """tok_off[k] = exclusive prefix of lens over the order (maestro_varlen_pack)."""
    l = np.asarray([lens[i] for i in order], dtype=np.int64)
    return np.concatenate([[0], np.cumsum(l)[:-1]]).astype(np.int64) if len(l) else np.zeros(0, np.int64)


def handoff_index(up_order, crit_order, tok_off, mbs, rows, dst_off):
    """-> (pos [n+1], src [R], dst [R]) exactly as maestro_handoff_index."""
    up_off = {}
    acc = 0
    for i in up_order:
        up_off[int(i)] = acc
        acc += int(rows[i])
    pos = [0]
    src, dst = [], []
    for k, i in enumerate(crit_order):
        i = int(i)
        nr = int(rows[i])
        if nr > 0:
            if i not in up_off:
                raise KeyError(f"sample {i} activated but absent from the producer order")
            first = (k // mbs) * mbs
            base = int(tok_off[k]) - int(tok_off[first]) + int(dst_off[i])
            src.extend(range(up_off[i], up_off[i] + nr))
            dst.extend(range(base, base + nr))
        pos.append(pos[-1] + nr)
    return np.asarray(pos, np.int32), np.asarray(src, np.int32), np.asarray(dst, np.int32)
