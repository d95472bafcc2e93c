"""M-to-N reshard message queue over device memory (the section handoff, C1).

Mirrors the reference API of ``maestro.mq`` (``/root/reference/pkg/src/maestro/mq.py``): the
same class/function names, argument meaning and errors -- ``ShardLayout`` (:39-96),
``Transfer``/``ReshardPlan`` (:99-120), ``plan_reshard`` (:123-160), ``apply_plan`` (:163-174),
``MessageMeta`` (:180-196), ``Transport`` (:199-209), ``SlotBudget`` (:326-352), ``Channel``
(:355-407), ``Endpoint`` (:410-497), ``connect`` (:500-523), ``push_tensor`` (:526-551).

What is B200-native here:

* payloads are torch CUDA tensors and never visit the host: ``Channel.push`` slices the
  sender's shard into a destination slot with the ``maestro_box_copy`` kernel on the pushing
  stream and returns immediately (the slot is reserved against the receiver's ``SlotBudget``
  first, exactly as the reference reserves before sending);
* ``DeviceTransport`` (in-process, any GPU of this process) hands the slot over with a CUDA
  event: ``pull`` makes the puller's stream wait on it -- ordering without a host sync;
* ``DistTransport`` moves (header, payload) pairs over ``torch.distributed`` point-to-point
  (NCCL over NVLink on the GPU box; gloo for the CPU tests).  The receiver knows each
  fragment's shape from the plan, so it posts both receives without blocking the host; the
  header (the control subchannel: magic, sequence, sample, sender position, element size,
  dims, section) is checked at ``pull(validate=True)`` or deferred to ``Endpoint.verify()``
  (the executor verifies once per step);
* ``Endpoint.pull`` gathers all fragments of the earliest logical tensor into the receiver's
  shard with one box copy per transfer; a plan whose single transfer covers the whole shard
  returns the slot itself (zero copy).

The reference's loopback-socket transport is networking and out of scope; the
``Transport`` plug-in point is kept, so one can be supplied through ``transport_factory``.
"""

from __future__ import annotations

import ctypes
import threading
from collections import deque
from dataclasses import dataclass, field
from itertools import product
from typing import Iterator, Optional

import numpy as np
import torch

from . import _native as N
from .errors import ChannelClosed, FragmentTimeout, IncompatibleShapes, InvalidDims, SlotExhausted

Rank = tuple[int, int]  # (tp_rank, cp_rank)
Box = tuple[tuple[int, int], ...]  # half-open (start, stop) per axis

_MAX_DIMS = 6
_bound = None


def _lib():
    global _bound
    if _bound is None:
        P, I32 = ctypes.c_void_p, ctypes.c_int32
        _bound = N.extra_symbols({"maestro_box_copy": ([P, P, P, P, P, I32, I32, P], ctypes.c_int)})
    return _bound


def _torch_dtype(dtype) -> torch.dtype:
    if isinstance(dtype, torch.dtype):
        return dtype
    return torch.from_numpy(np.empty(0, dtype=np.dtype(dtype))).dtype


def box_copy(src: torch.Tensor, dst: torch.Tensor) -> torch.Tensor:
    """dst[...] = src[...] for equally shaped (strided) device views, on the current stream."""
    if tuple(src.shape) != tuple(dst.shape):
        raise IncompatibleShapes(f"box copy shape {tuple(src.shape)} != {tuple(dst.shape)}")
    if src.dtype != dst.dtype:
        raise IncompatibleShapes(f"box copy dtype {src.dtype} != {dst.dtype}")
    if src.numel() == 0:
        return dst
    if not (src.is_cuda and dst.is_cuda):
        if src.is_cuda or dst.is_cuda:
            raise IncompatibleShapes("box copy between host and device memory")
        dst.copy_(src)  # host-resident payloads (gloo transport); device data never takes this path
        return dst
    shape, ss, ds = list(src.shape), list(src.stride()), list(dst.stride())
    # drop unit dims, then merge dims that are contiguous on both sides
    dims = [(n, a, b) for n, a, b in zip(shape, ss, ds) if n != 1] or [(1, 1, 1)]
    merged = [list(dims[0])]
    for n, a, b in dims[1:]:
        pn, pa, pb = merged[-1]
        if pa == a * n and pb == b * n:
            merged[-1] = [pn * n, a, b]
        else:
            merged.append([n, a, b])
    if len(merged) > _MAX_DIMS:
        raise InvalidDims(f"box copy supports at most {_MAX_DIMS} non-contiguous dims, got {len(merged)}")
    nd = len(merged)
    arr = lambda k: (ctypes.c_int64 * nd)(*[m[k] for m in merged])  # noqa: E731
    rc = _lib().maestro_box_copy(src.data_ptr(), arr(1), dst.data_ptr(), arr(2), arr(0), nd, src.element_size(),
                                 N.stream_ptr())
    N.check(rc, "box_copy")
    return dst


# --- layouts and plans ----------------------------------------------------------------------


@dataclass(frozen=True)
class ShardLayout:
    """How a logical tensor is split over a (TP, CP) grid (mq.py:39-96)."""

    tensor_shape: tuple[int, ...]
    tp: int = 1
    cp: int = 1
    tp_axis: int = 0
    cp_axis: int = 1

    def __post_init__(self) -> None:
        shape = tuple(int(d) for d in self.tensor_shape)
        object.__setattr__(self, "tensor_shape", shape)
        if not shape or min(shape) <= 0:
            raise InvalidDims(f"tensor_shape must be positive, got {shape}")
        if self.tp < 1 or self.cp < 1:
            raise InvalidDims("tp and cp degrees must be >= 1")
        for name, axis, deg in (("tp_axis", self.tp_axis, self.tp), ("cp_axis", self.cp_axis, self.cp)):
            if deg > 1 and not 0 <= axis < len(shape):
                raise InvalidDims(f"{name} {axis} out of range for {len(shape)}-d tensor")
        if self.tp > 1 and self.cp > 1 and self.tp_axis == self.cp_axis:
            raise InvalidDims("tp_axis and cp_axis must differ when both degrees exceed 1")
        for axis, deg, what in ((self.tp_axis, self.tp, "tp"), (self.cp_axis, self.cp, "cp")):
            if deg > 1 and shape[axis] % deg:
                raise InvalidDims(f"axis {axis} ({shape[axis]}) not divisible by {what}={deg}")

    def ranks(self) -> Iterator[Rank]:
        return iter(product(range(self.tp), range(self.cp)))

    def global_box(self, rank: Rank) -> Box:
        """Region of the logical tensor held by ``rank`` in global coordinates."""
        t, c = rank
        if not (0 <= t < self.tp and 0 <= c < self.cp):
            raise InvalidDims(f"rank {rank} outside {self.tp}x{self.cp} grid")
        box = [(0, d) for d in self.tensor_shape]
        for axis, deg, idx in ((self.tp_axis, self.tp, t), (self.cp_axis, self.cp, c)):
            if deg > 1:
                w = self.tensor_shape[axis] // deg
                box[axis] = (idx * w, idx * w + w)
        return tuple(box)

    def shard_shape(self, rank: Rank) -> tuple[int, ...]:
        return tuple(b - a for a, b in self.global_box(rank))

    def shard(self, tensor, rank: Rank):
        """View of ``rank``'s region (torch or numpy; no copy)."""
        if tuple(tensor.shape) != self.tensor_shape:
            raise IncompatibleShapes(f"tensor shape {tuple(tensor.shape)} != layout shape {self.tensor_shape}")
        return tensor[_slices(self.global_box(rank))]


def _slices(box: Box):
    return tuple(slice(a, b) for a, b in box)


@dataclass(frozen=True)
class Transfer:
    sender: Rank
    receiver: Rank
    sender_slice: Box  # local to the sender's shard
    receiver_slice: Box  # local to the receiver's shard


@dataclass(frozen=True)
class ReshardPlan:
    src: ShardLayout
    dst: ShardLayout
    transfers: tuple[Transfer, ...]

    def for_receiver(self, rank: Rank) -> tuple[Transfer, ...]:
        return tuple(t for t in self.transfers if t.receiver == rank)

    def for_sender(self, rank: Rank) -> tuple[Transfer, ...]:
        return tuple(t for t in self.transfers if t.sender == rank)

    def senders_of(self, receiver: Rank) -> tuple[Rank, ...]:
        return tuple(sorted({t.sender for t in self.transfers if t.receiver == receiver}))


def plan_reshard(src: ShardLayout, dst: ShardLayout) -> ReshardPlan:
    """Minimal point-to-point transfer set taking ``src`` sharding to ``dst`` (mq.py:123-160).

    One transfer per (sender, receiver) pair whose boxes intersect, receivers in ``dst.ranks()``
    order and senders in ``src.ranks()`` order; the receiver slices tile each destination shard
    exactly once (boxes of one layout are disjoint and cover the tensor)."""
    if src.tensor_shape != dst.tensor_shape:
        raise IncompatibleShapes(f"layouts disagree on tensor shape: {src.tensor_shape} vs {dst.tensor_shape}")
    if (src.tp_axis, src.cp_axis) != (dst.tp_axis, dst.cp_axis):
        raise IncompatibleShapes("layouts must agree on tp_axis/cp_axis "
                                 f"({src.tp_axis},{src.cp_axis}) vs ({dst.tp_axis},{dst.cp_axis})")
    sboxes = [(s, src.global_box(s)) for s in src.ranks()]
    out = []
    for r in dst.ranks():
        rbox = dst.global_box(r)
        for s, sbox in sboxes:
            lo = [max(a[0], b[0]) for a, b in zip(sbox, rbox)]
            hi = [min(a[1], b[1]) for a, b in zip(sbox, rbox)]
            if any(x >= y for x, y in zip(lo, hi)):
                continue
            out.append(Transfer(sender=s, receiver=r,
                                sender_slice=tuple((x - o[0], y - o[0]) for x, y, o in zip(lo, hi, sbox)),
                                receiver_slice=tuple((x - o[0], y - o[0]) for x, y, o in zip(lo, hi, rbox))))
    return ReshardPlan(src=src, dst=dst, transfers=tuple(out))


def apply_plan(plan: ReshardPlan, shards_by_sender: dict) -> dict:
    """Full reshard on device (mq.py:163-174): one box copy per transfer into each receiver's
    shard.  Shards are CUDA tensors; numpy shards are uploaded and the results returned as
    numpy (the reference's array type), still moved by the device kernel."""
    as_numpy = isinstance(next(iter(shards_by_sender.values())), np.ndarray)
    dev = torch.device("cuda", torch.cuda.current_device())
    shards = {k: (torch.from_numpy(np.ascontiguousarray(v)).to(dev) if as_numpy else v)
              for k, v in shards_by_sender.items()}
    sample = next(iter(shards.values()))
    out = {}
    for r in plan.dst.ranks():
        buf = torch.empty(plan.dst.shard_shape(r), dtype=sample.dtype, device=sample.device)
        for t in plan.for_receiver(r):
            box_copy(shards[t.sender][_slices(t.sender_slice)], buf[_slices(t.receiver_slice)])
        out[r] = buf
    if as_numpy:
        return {k: v.cpu().numpy() for k, v in out.items()}
    return out


# --- metadata and transports -------------------------------------------------------------------


@dataclass(frozen=True)
class MessageMeta:
    """Control-subchannel record identifying one fragment of one tensor (mq.py:180-196)."""

    tensor_shape: tuple[int, ...]
    element_size_bytes: int
    section_name: str
    sender_position: Rank
    sample_id: int
    sequence_number: int = -1  # assigned by the channel on push

    @property
    def nbytes(self) -> int:
        n = self.element_size_bytes
        for d in self.tensor_shape:
            n *= d
        return n


class Transport:
    """Moves (meta, payload) pairs from one sender to one receiver (mq.py:199-209).

    ``send(meta, payload)`` takes a device tensor that the channel owns from then on;
    ``recv(shape, dtype, timeout)`` returns a :class:`Fragment`."""

    def send(self, meta: MessageMeta, payload: torch.Tensor) -> None:
        raise NotImplementedError

    def recv(self, shape, dtype, timeout: Optional[float] = None) -> "Fragment":
        raise NotImplementedError

    def close(self) -> None:
        pass


@dataclass
class Fragment:
    """One received fragment: its payload, the event/work to order on, and its metadata (or
    the undecoded header when the transport defers the control check)."""

    payload: torch.Tensor
    meta: Optional[MessageMeta] = None
    event: Optional[torch.cuda.Event] = None
    works: tuple = ()
    header: Optional[torch.Tensor] = None

    def _wait_works(self) -> None:
        # each work is waited once (for NCCL: the current stream waits on the comm stream)
        works, self.works = self.works, ()
        for w in works:
            w.wait()

    def ready_on_current_stream(self) -> None:
        if self.event is not None:
            torch.cuda.current_stream(self.payload.device).wait_event(self.event)
        self._wait_works()

    def decoded(self) -> MessageMeta:
        if self.meta is None:
            self._wait_works()
            self.meta = _decode_header(self.header.cpu())
        return self.meta


class DeviceTransport(Transport):
    """In-process transport between streams/GPUs of one process: a FIFO of device slots, each
    published with a CUDA event recorded on the pushing stream."""

    def __init__(self) -> None:
        self._items: deque = deque()
        self._cond = threading.Condition()
        self._closed = False

    def send(self, meta: MessageMeta, payload: torch.Tensor) -> None:
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(payload.device))
        with self._cond:
            self._items.append(Fragment(payload=payload, meta=meta, event=ev))
            self._cond.notify_all()

    def recv(self, shape=None, dtype=None, timeout: Optional[float] = None) -> Fragment:
        with self._cond:
            if not self._items:
                if self._closed:
                    raise ChannelClosed("transport closed")
                self._cond.wait(timeout)
            if not self._items:
                raise TimeoutError
            return self._items.popleft()

    def pending(self) -> int:
        with self._cond:
            return len(self._items)

    def close(self) -> None:
        with self._cond:
            self._closed = True
            self._cond.notify_all()


# control header (little-endian int64 words): magic, seq, sample, tp, cp, esize, ndim,
# dims[6], section-name length, section name (64 bytes in 8 words)
_MAGIC = 0x4D535251
_HDR = 7 + _MAX_DIMS + 1 + 8


def _encode_header(meta: MessageMeta) -> torch.Tensor:
    name = meta.section_name.encode("utf-8")
    if len(meta.tensor_shape) > _MAX_DIMS or len(name) > 64:
        raise InvalidDims("fragment rank > 6 or section name > 64 bytes")
    words = [_MAGIC, meta.sequence_number, meta.sample_id, meta.sender_position[0], meta.sender_position[1],
             meta.element_size_bytes, len(meta.tensor_shape)]
    words += list(meta.tensor_shape) + [0] * (_MAX_DIMS - len(meta.tensor_shape))
    words.append(len(name))
    words += np.frombuffer(name.ljust(64, b"\0"), dtype="<i8").tolist()
    return torch.tensor(words, dtype=torch.int64)


def _decode_header(h: torch.Tensor) -> MessageMeta:
    w = h.tolist()
    if w[0] != _MAGIC:
        raise ChannelClosed(f"bad control magic 0x{w[0] & 0xffffffff:08x}")
    nd = w[6]
    name = np.array(w[7 + _MAX_DIMS + 1:], dtype="<i8").tobytes()[: w[7 + _MAX_DIMS]].decode("utf-8")
    return MessageMeta(tensor_shape=tuple(w[7: 7 + nd]), element_size_bytes=w[5], section_name=name,
                       sender_position=(w[3], w[4]), sample_id=w[2], sequence_number=w[1])


class DistTransport(Transport):
    """Point-to-point over ``torch.distributed`` (NCCL over NVLink on the box, gloo on CPU):
    header then payload.  ``peer`` is the other process's global rank."""

    def __init__(self, peer: int, group=None) -> None:
        import torch.distributed as dist

        self.dist, self.peer, self.group = dist, peer, group
        self._inflight: deque = deque()

    def send(self, meta: MessageMeta, payload: torch.Tensor) -> None:
        hdr = _encode_header(meta)
        if payload.is_cuda:  # pinned staging: a pageable upload would block the host on the stream
            hdr = hdr.pin_memory().to(payload.device, non_blocking=True)
        w1 = self.dist.isend(hdr, self.peer, group=self.group)
        w2 = self.dist.isend(payload, self.peer, group=self.group)
        self.last_works = (w1, w2)
        self._inflight.append((w1, w2, hdr, payload))  # keep buffers alive until completion
        while len(self._inflight) > 64:
            for w in self._inflight.popleft()[:2]:
                w.wait()

    def recv(self, shape, dtype, timeout: Optional[float] = None, device=None) -> Fragment:
        dev = device if device is not None else (torch.device("cuda", torch.cuda.current_device())
                                                 if torch.cuda.is_available() else torch.device("cpu"))
        hdr = torch.empty(_HDR, dtype=torch.int64, device=dev)
        payload = torch.empty(tuple(shape), dtype=_torch_dtype(dtype), device=dev)
        w1 = self.dist.irecv(hdr, self.peer, group=self.group)
        w2 = self.dist.irecv(payload, self.peer, group=self.group)
        return Fragment(payload=payload, works=(w1, w2), header=hdr)

    def flush(self) -> None:
        while self._inflight:
            for w in self._inflight.popleft()[:2]:
                w.wait()

    def close(self) -> None:
        self.flush()


_p2p = None


def _p2p_lib():
    global _p2p
    if _p2p is None:
        P, I64, U32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint32
        _p2p = N.extra_symbols({
            "maestro_device_alloc": ([I64, ctypes.POINTER(P)], ctypes.c_int),
            "maestro_device_free": ([P], ctypes.c_int),
            "maestro_ipc_get_handle": ([P, P], ctypes.c_int),
            "maestro_ipc_open_handle": ([P, ctypes.POINTER(P)], ctypes.c_int),
            "maestro_ipc_close": ([P], ctypes.c_int),
            "maestro_stream_wait_geq": ([P, P, U32], ctypes.c_int),
            "maestro_stream_write": ([P, P, U32], ctypes.c_int),
            "maestro_copy_async": ([P, P, I64, P], ctypes.c_int),
        })
    return _p2p


class PeerTransport(Transport):
    """One-sided NVLink transport between two processes of one node (csrc/p2p.cu).

    The receiver owns a ring of ``slots`` slots (a 256-byte control header + ``slot_bytes`` of
    payload each) and one flag word per slot; the sender owns one credit word.  Both are exported
    once through CUDA IPC.  Message i goes to slot i % slots.  Send, on the sender's stream:
    stream-wait credit >= i - slots + 1, copy header + payload into the peer slot (copy engine),
    stream-write the peer flag = i + 1.  Receive, on the receiver's stream: stream-wait flag >=
    i + 1, copy the payload out, stream-write the sender's credit = i + 1.  Nothing blocks the
    host and no kernel spins on the other GPU, so compute keeps every SM (compare DistTransport,
    whose NCCL kernels hold SMs while they wait for the peer).  The constructor is collective
    over the pair: both processes call it in the same order with the same sizes."""

    HEADER = 256

    def __init__(self, peer: int = -1, role: str = "send", slot_bytes: int = 64 << 20, slots: int = 4,
                 group=None, _local=None) -> None:
        L = _p2p_lib()
        self.role, self.slots = role, slots
        self.stride = self.HEADER + (slot_bytes + 255) // 256 * 256
        self.slot_bytes = slot_bytes
        self.seq = 0
        self._owned = []
        self._opened = []
        dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev

        def alloc(nbytes):
            ptr = ctypes.c_void_p()
            N.check(L.maestro_device_alloc(nbytes, ctypes.byref(ptr)), "device_alloc")
            self._owned.append(ptr.value)
            return ptr.value

        if _local is not None:  # in-process pair (tests): share the receiver's buffers directly
            self.flags, self.arena, self.credit = _local
            self.peer_flags, self.peer_arena, self.peer_credit = _local
            return
        import torch.distributed as dist

        # the 64-byte IPC handles travel over the pair's process group (host tensors under gloo,
        # e.g. two processes sharing one GPU; device tensors under NCCL)
        hdev = torch.device("cpu") if dist.get_backend(group) == "gloo" else dev

        def send_handle(ptr):
            h = (ctypes.c_ubyte * 64)()
            N.check(L.maestro_ipc_get_handle(ptr, h), "ipc_get_handle")
            dist.send(torch.tensor(list(h), dtype=torch.uint8, device=hdev), peer, group=group)

        def recv_handle():
            t = torch.empty(64, dtype=torch.uint8, device=hdev)
            dist.recv(t, peer, group=group)
            h = (ctypes.c_ubyte * 64)(*t.cpu().tolist())
            ptr = ctypes.c_void_p()
            N.check(L.maestro_ipc_open_handle(h, ctypes.byref(ptr)), "ipc_open_handle")
            self._opened.append(ptr.value)
            return ptr.value

        if role == "recv":
            base = alloc(256 + slots * self.stride)  # flags (slots x u32, padded) then the slot ring
            self.flags, self.arena = base, base + 256
            send_handle(base)
            self.peer_credit = recv_handle()
        else:
            self.credit = alloc(256)
            base = recv_handle()
            self.peer_flags, self.peer_arena = base, base + 256
            send_handle(self.credit)

    @classmethod
    def local_pair(cls, slot_bytes: int = 1 << 20, slots: int = 4):
        """(sender, receiver) in one process sharing one ring (single-GPU protocol tests)."""
        L = _p2p_lib()
        stride = cls.HEADER + (slot_bytes + 255) // 256 * 256
        ptr, cred = ctypes.c_void_p(), ctypes.c_void_p()
        N.check(L.maestro_device_alloc(256 + slots * stride, ctypes.byref(ptr)), "device_alloc")
        N.check(L.maestro_device_alloc(256, ctypes.byref(cred)), "device_alloc")
        bufs = (ptr.value, ptr.value + 256, cred.value)
        tx = cls(role="send", slot_bytes=slot_bytes, slots=slots, _local=bufs)
        rx = cls(role="recv", slot_bytes=slot_bytes, slots=slots, _local=bufs)
        rx._owned = [ptr.value, cred.value]
        return tx, rx

    def send(self, meta: MessageMeta, payload: torch.Tensor) -> None:
        L, st = _p2p_lib(), N.stream_ptr()
        nbytes = payload.numel() * payload.element_size()
        if nbytes > self.slot_bytes:
            raise SlotExhausted(f"fragment of {nbytes} B exceeds the {self.slot_bytes} B transport slot",
                                request=nbytes, reserved=self.slot_bytes)
        i, slot = self.seq, self.seq % self.slots
        if i >= self.slots:  # the receiver released this slot's previous message
            N.check(L.maestro_stream_wait_geq(st, self.credit, i - self.slots + 1), "stream_wait")
        hdr = _encode_header(meta).pin_memory().to(payload.device, non_blocking=True)
        dst = self.peer_arena + slot * self.stride
        N.check(L.maestro_copy_async(dst, hdr.data_ptr(), hdr.numel() * 8, st), "copy_async")
        N.check(L.maestro_copy_async(dst + self.HEADER, payload.data_ptr(), nbytes, st), "copy_async")
        N.check(L.maestro_stream_write(st, self.peer_flags + 4 * slot, i + 1), "stream_write")
        payload.record_stream(torch.cuda.current_stream(payload.device))
        hdr.record_stream(torch.cuda.current_stream(payload.device))
        self.last_works = ()
        self.seq += 1

    def recv(self, shape, dtype, timeout: Optional[float] = None) -> Fragment:
        L, st = _p2p_lib(), N.stream_ptr()
        i, slot = self.seq, self.seq % self.slots
        out = torch.empty(tuple(shape), dtype=_torch_dtype(dtype), device=self.device)
        nbytes = out.numel() * out.element_size()
        if nbytes > self.slot_bytes:
            raise SlotExhausted(f"fragment of {nbytes} B exceeds the {self.slot_bytes} B transport slot",
                                request=nbytes, reserved=self.slot_bytes)
        src = self.arena + slot * self.stride
        N.check(L.maestro_stream_wait_geq(st, self.flags + 4 * slot, i + 1), "stream_wait")
        hdr = torch.empty(_HDR, dtype=torch.int64, device=self.device)
        N.check(L.maestro_copy_async(hdr.data_ptr(), src, _HDR * 8, st), "copy_async")
        N.check(L.maestro_copy_async(out.data_ptr(), src + self.HEADER, nbytes, st), "copy_async")
        N.check(L.maestro_stream_write(st, self.peer_credit, i + 1), "stream_write")  # slot released
        self.seq += 1
        return Fragment(payload=out, header=hdr)

    def close(self) -> None:
        L = _p2p_lib()
        torch.cuda.synchronize()
        for p in self._opened:
            L.maestro_ipc_close(p)
        for p in self._owned:
            L.maestro_device_free(p)
        self._opened, self._owned = [], []


# --- slot accounting ---------------------------------------------------------------------------


@dataclass
class SlotBudget:
    """Destination-memory quota with explicit backpressure (mq.py:326-352): exhaustion raises
    SlotExhausted at push time, nothing is dropped; peak_bytes is the memory statistic."""

    capacity_bytes: Optional[int] = None
    reserved_bytes: int = 0
    peak_bytes: int = 0
    _lock: threading.Lock = field(default_factory=threading.Lock, repr=False)

    def reserve(self, nbytes: int) -> None:
        with self._lock:
            if self.capacity_bytes is not None and self.reserved_bytes + nbytes > self.capacity_bytes:
                raise SlotExhausted(f"slot budget exhausted: {self.reserved_bytes} + {nbytes} > "
                                    f"{self.capacity_bytes} bytes", reserved=self.reserved_bytes, request=nbytes)
            self.reserved_bytes += nbytes
            self.peak_bytes = max(self.peak_bytes, self.reserved_bytes)

    def release(self, nbytes: int) -> None:
        with self._lock:
            self.reserved_bytes -= nbytes


class Channel:
    """One sender -> one receiver path, FIFO by per-channel sequence number (mq.py:355-407).

    ``device`` is where the receiver's slots live (default: the current CUDA device)."""

    def __init__(self, sender: Rank, receiver: Rank, transport: Optional[Transport] = None,
                 budget: Optional[SlotBudget] = None, device=None) -> None:
        self.sender, self.receiver = sender, receiver
        self.transport = transport or DeviceTransport()
        self.budget = budget or SlotBudget()
        self.device = device
        self._next_seq = 0
        self._closed = False
        self._lock = threading.Lock()
        self._inflight: deque = deque()

    def push(self, fragment: torch.Tensor, meta: MessageMeta, donate: bool = False) -> int:
        """Reserve a destination slot, ship metadata and payload; returns the sequence number
        (acknowledgment token) without waiting for the receiver.

        The fragment is copied into a fresh slot on the pushing stream, so the caller may
        overwrite its buffer afterwards.  ``donate=True`` hands a contiguous buffer over instead
        (the caller promises not to write it again): no copy."""
        if self._closed:
            raise ChannelClosed(f"channel {self.sender}->{self.receiver} is closed")
        if tuple(fragment.shape) != tuple(meta.tensor_shape):
            raise IncompatibleShapes(f"fragment shape {tuple(fragment.shape)} != declared {meta.tensor_shape}")
        if fragment.element_size() != meta.element_size_bytes:
            raise IncompatibleShapes(f"fragment element size {fragment.element_size()} != declared "
                                     f"{meta.element_size_bytes}")
        nbytes = fragment.numel() * fragment.element_size()
        remote = isinstance(self.transport, (DistTransport, PeerTransport))
        if remote:  # the receiver's slots live in another process: count bytes in flight here
            self._reap()
        self.budget.reserve(nbytes)
        with self._lock:
            seq = self._next_seq
            self._next_seq += 1
        stamped = MessageMeta(tensor_shape=tuple(meta.tensor_shape), element_size_bytes=meta.element_size_bytes,
                              section_name=meta.section_name, sender_position=tuple(meta.sender_position),
                              sample_id=meta.sample_id, sequence_number=seq)
        if donate and fragment.is_contiguous() and (remote or self.device is None or fragment.device == self.device):
            slot = fragment
        else:
            dev = self.device if self.device is not None else fragment.device
            slot = torch.empty(tuple(fragment.shape), dtype=fragment.dtype, device=dev)
            if slot.device == fragment.device and fragment.is_cuda:
                box_copy(fragment, slot)
            else:  # cross-device (peer GPU) or host tensors (gloo tests)
                slot.copy_(fragment, non_blocking=True)
        self.transport.send(stamped, slot)
        if remote:
            self._inflight.append((self.transport.last_works, nbytes))
        return seq

    def _reap(self) -> None:
        """Release the budget of remote sends that have completed."""
        while self._inflight and all(w.is_completed() for w in self._inflight[0][0]):
            self.budget.release(self._inflight.popleft()[1])

    def close(self) -> None:
        self._closed = True
        self.transport.close()


class Endpoint:
    """Receiver side: gathers the earliest logical tensor from M channels (mq.py:410-497)."""

    def __init__(self, receiver: Rank, plan: ReshardPlan, channels: dict, dtype, timeout: Optional[float] = None,
                 device=None) -> None:
        self.receiver = receiver
        self.plan = plan
        self.channels = channels
        self.dtype = _torch_dtype(dtype)
        self.timeout = timeout
        self.device = device
        self.pulled_tensors = 0
        expected = plan.senders_of(receiver)
        missing = [r for r in expected if r not in channels]
        if missing:
            raise IncompatibleShapes(f"receiver {receiver} lacks channels from senders {missing}")
        self._expected = expected
        self._deferred: list = []

    def pull(self, timeout: Optional[float] = None, validate: bool = True):
        """Assemble this receiver's shard of the earliest logical tensor; returns (tensor, meta).

        Blocks (host) until every contributing sender's next fragment is available
        (FragmentTimeout names the missing sender).  The returned tensor is ready on the
        caller's current stream.  ``validate=False`` defers the cross-fragment control check
        of header-carrying transports to :meth:`verify`."""
        timeout = self.timeout if timeout is None else timeout
        shapes = {t.sender: tuple(b - a for a, b in t.receiver_slice) for t in self.plan.for_receiver(self.receiver)}
        frags = {}
        for s in self._expected:
            try:
                frags[s] = self.channels[s].transport.recv(shapes[s], self.dtype, timeout)
            except TimeoutError:
                raise FragmentTimeout(f"receiver {self.receiver} timed out waiting for sender {s}",
                                      receiver=str(self.receiver), sender=str(s)) from None
        if validate or all(f.meta is not None for f in frags.values()):
            self._check([f.decoded() for f in frags.values()])
        else:
            self._deferred.append(list(frags.values()))
        shape = self.plan.dst.shard_shape(self.receiver)
        for f in frags.values():
            f.ready_on_current_stream()
        transfers = self.plan.for_receiver(self.receiver)
        only = frags[transfers[0].sender].payload if len(transfers) == 1 else None
        if only is not None and tuple(only.shape) == tuple(shape) and only.is_contiguous():
            buf = only  # the slot is the shard (identity / 1:1 plans): zero copy
        else:
            dev = self.device if self.device is not None else next(iter(frags.values())).payload.device
            buf = torch.empty(shape, dtype=self.dtype, device=dev)
            for t in transfers:
                box_copy(frags[t.sender].payload, buf[_slices(t.receiver_slice)])
        for s in self._expected:
            if isinstance(self.channels[s].transport, DeviceTransport):  # in-process slots
                p = frags[s].payload
                self.channels[s].budget.release(p.numel() * p.element_size())
        self.pulled_tensors += 1
        first = next(iter(frags.values()))
        ref = first.meta
        summary = MessageMeta(tensor_shape=tuple(shape), element_size_bytes=buf.element_size(),
                              section_name=ref.section_name if ref else "", sender_position=self.receiver,
                              sample_id=ref.sample_id if ref else -1,
                              sequence_number=ref.sequence_number if ref else -1)
        return buf, summary

    def _check(self, metas) -> None:
        sections = {m.section_name for m in metas}
        samples = {m.sample_id for m in metas}
        if len(sections) > 1 or len(samples) > 1:
            raise IncompatibleShapes(f"fragment streams disagree: sections={sorted(sections)}, "
                                     f"samples={sorted(samples)}")

    def take_deferred(self) -> list:
        """Detach the deferred headers pulled so far (to verify them later with ``verify``)."""
        out, self._deferred = self._deferred, []
        return out

    def verify(self, deferred: list | None = None) -> list[MessageMeta]:
        """Decode and check deferred headers (one host sync): this endpoint's pending ones, or a
        list detached earlier by ``take_deferred``; returns their metadata."""
        lists = self._deferred if deferred is None else deferred
        out = []
        for frags in lists:
            metas = [f.decoded() for f in frags]
            self._check(metas)
            out.append(metas[0])
        if deferred is None:
            self._deferred.clear()
        return out


def connect(plan: ReshardPlan, dtype=torch.float32, slot_budget_bytes: Optional[int] = None,
            timeout: Optional[float] = None, transport_factory=None):
    """Wire up every point-to-point channel the plan needs (mq.py:500-523).

    Returns ({(sender, receiver): Channel}, {receiver: Endpoint}); each endpoint enforces one
    shared slot budget across its incoming channels.  ``transport_factory(sender, receiver)``
    (or a zero-argument factory) picks the transport; default :class:`DeviceTransport`."""
    channels, endpoints = {}, {}
    for r in plan.dst.ranks():
        budget = SlotBudget(capacity_bytes=slot_budget_bytes)
        incoming = {}
        for s in plan.senders_of(r):
            if transport_factory is None:
                tr = DeviceTransport()
            else:
                try:
                    tr = transport_factory(s, r)
                except TypeError:
                    tr = transport_factory()
            ch = Channel(s, r, tr, budget)
            channels[(s, r)] = ch
            incoming[s] = ch
        endpoints[r] = Endpoint(r, plan, incoming, dtype, timeout)
    return channels, endpoints


def push_tensor(plan: ReshardPlan, channels: dict, sender: Rank, shard: torch.Tensor, section_name: str,
                sample_id: int) -> list[int]:
    """Split a sender's shard per the plan and push each slice on its channel (mq.py:526-551)."""
    expected = plan.src.shard_shape(sender)
    if tuple(shard.shape) != expected:
        raise IncompatibleShapes(f"sender {sender} shard shape {tuple(shard.shape)} != layout shard {expected}")
    tokens = []
    for t in plan.for_sender(sender):
        view = shard[_slices(t.sender_slice)]
        meta = MessageMeta(tensor_shape=tuple(view.shape), element_size_bytes=shard.element_size(),
                           section_name=section_name, sender_position=sender, sample_id=sample_id)
        tokens.append(channels[(sender, t.receiver)].push(view, meta))
    return tokens
