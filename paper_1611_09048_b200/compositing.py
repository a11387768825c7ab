"""Visibility-ordered sort-last compositing (drop-in for insitu.compositing).

* ``binary_swap(transport, local_pixels, order)`` keeps the reference
  signature (compositing.py:107-181).  With an :class:`NvlinkTransport` it is
  one fused peer-memory kernel per rank (``isc_binary_swap``: pull partner
  half-span over NVLink + ``over`` + in-place write per round, then a direct
  store of the final 1/R span into rank 0's output); non-power-of-two world
  sizes use ``isc_direct_send`` (rank 0 folds every peer image straight out
  of peer memory, compositing.py:184-194).  With any other byte ``Transport``
  (e.g. the reference-style ``LocalFabric`` or ``TorchDistTransport``) the
  messages travel as bytes and the ``over`` runs on the GPU.
* ``composite_sequential`` / ``over_arrays`` run ``isc_composite_fold`` /
  ``isc_over`` on device tensors.
* ``visibility_order`` and ``over`` (4-tuples) are host utilities.
"""

from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _abi
from .errors import CompositeError
from .fields import GlobalVolume
from .scene import Camera

__all__ = ["CompositeError", "over", "over_arrays", "visibility_order", "composite_sequential",
           "CompositeMessage", "binary_swap", "binary_swap_local", "swap_schedule", "DeviceOps"]


def over(front: Sequence[float], back: Sequence[float]) -> tuple:
    """Premultiplied over on one RGBA 4-tuple (compositing.py:25-28)."""
    k = 1.0 - front[3]
    return tuple(float(front[c] + k * back[c]) for c in range(4))


def visibility_order(volume: GlobalVolume, camera: Camera) -> list:
    """Near-to-far rank permutation by nested slab distances (compositing.py:36-63)."""
    per_axis = []
    for a in range(3):
        width = volume.size[a] / volume.decomposition[a]
        c = camera.position[a]
        dist = [(max(i * width - c, 0.0, c - (i * width + width)), i) for i in range(volume.decomposition[a])]
        per_axis.append([i for _, i in sorted(dist)])
    return [volume.rank_of((bx, by, bz)) for bx in per_axis[0] for by in per_axis[1] for bz in per_axis[2]]


def swap_schedule(virtual: int, size: int, n_pixels: int):
    """Binary-swap plan for the rank at visibility position ``virtual``:
    [(partner_virtual, keep_span, give_span)] per round and the final span
    (compositing.py:133-167)."""
    lo, hi = 0, n_pixels
    plan = []
    r = 0
    while (1 << r) < size:
        bit = 1 << r
        mid = (lo + hi) // 2
        keep, give = ((mid, hi), (lo, mid)) if virtual & bit else ((lo, mid), (mid, hi))
        plan.append((virtual ^ bit, keep, give))
        lo, hi = keep
        r += 1
    return plan, (lo, hi)


class DeviceOps:
    """Device-side primitives used by the byte-transport swap path."""

    def __init__(self, device=None, stream=None):
        import torch
        from .device import require_cuda
        self.torch = torch
        self.device = device if device is not None else require_cuda()
        self.stream = stream

    def _s(self):
        from .device import stream_handle
        return C.c_void_p(stream_handle(self.stream))

    def as_flat(self, pixels):
        t = self.torch.as_tensor(pixels) if not isinstance(pixels, self.torch.Tensor) else pixels
        t = t.to(device=self.device, dtype=self.torch.float32).contiguous()
        return t.reshape(-1, 4)

    def to_bytes(self, span) -> bytes:
        return span.contiguous().cpu().numpy().astype("<f4", copy=False).tobytes()

    def from_array(self, arr: np.ndarray):
        return self.torch.from_numpy(np.array(arr, dtype=np.float32)).to(self.device)

    def over(self, front, back):
        front, back = front.contiguous(), back.contiguous()
        out = self.torch.empty_like(front)
        _abi.check(_abi.lib().isc_over(C.c_void_p(out.data_ptr()), C.c_void_p(front.data_ptr()),
                                       C.c_void_p(back.data_ptr()), front.shape[0], self._s()), "over")
        return out

    def fold(self, flats, order):
        out = self.torch.empty_like(flats[0])
        ptrs = (C.c_void_p * len(order))(*[flats[r].data_ptr() for r in order])
        _abi.check(_abi.lib().isc_composite_fold(C.c_void_p(out.data_ptr()), ptrs, len(order), out.shape[0],
                                                 self._s()), "composite_sequential")
        return out

    def empty(self, n):
        return self.torch.empty((n, 4), dtype=self.torch.float32, device=self.device)


def over_arrays(front, back):
    """Premultiplied over on (..., 4) device tensors (compositing.py:31-33)."""
    ops = DeviceOps()
    f, b = ops.as_flat(front), ops.as_flat(back)
    if f.shape != b.shape:
        raise CompositeError(f"shape mismatch: {tuple(f.shape)} vs {tuple(b.shape)}")
    shape = tuple(front.shape)
    return ops.over(f, b).reshape(shape)


def composite_sequential(images: Sequence, order: Sequence[int]):
    """Front-to-back fold in visibility order (compositing.py:66-77) on the GPU."""
    if not len(images):
        raise CompositeError("no images to composite")
    shape = tuple(images[0].shape)
    for img in images:
        if tuple(img.shape) != shape:
            raise CompositeError(f"image size mismatch: {tuple(img.shape)} vs {shape}")
    ops = DeviceOps()
    flats = [ops.as_flat(im) for im in images]
    return ops.fold(flats, list(order)).reshape(shape)


@dataclass(frozen=True)
class CompositeMessage:
    """Wire unit of the byte-transport path: 16-byte header ``<iiii`` (round,
    sender, span offset, span length) + float32 RGBA span (compositing.py:80-104,
    with float32 payload because images are float32 here)."""

    round_index: int
    sender: int
    span_offset: int
    span_length: int
    payload: np.ndarray

    HEADER = struct.Struct("<iiii")
    DTYPE = "<f4"

    def to_bytes(self) -> bytes:
        return (self.HEADER.pack(self.round_index, self.sender, self.span_offset, self.span_length)
                + np.ascontiguousarray(self.payload, dtype=self.DTYPE).tobytes())

    @staticmethod
    def from_bytes(data: bytes) -> "CompositeMessage":
        rnd, sender, off, length = CompositeMessage.HEADER.unpack_from(data)
        payload = np.frombuffer(data, dtype=CompositeMessage.DTYPE, offset=CompositeMessage.HEADER.size)
        if payload.size != length * 4:
            raise CompositeError(f"span/payload mismatch: span {length} pixels, {payload.size} scalars")
        return CompositeMessage(rnd, sender, off, length, payload.reshape(length, 4))


def _wire(rnd, sender, lo, hi, body: bytes) -> bytes:
    return CompositeMessage.HEADER.pack(rnd, sender, lo, hi - lo) + body


def _torch():
    import torch
    return torch


def binary_swap(transport, local_pixels, order: Sequence[int], *, ops: Optional[DeviceOps] = None):
    """Composite every rank's image; the full frame appears on rank 0
    (returned as a new (H, W, 4) float32 CUDA tensor), ``None`` elsewhere."""
    from .transport import NvlinkTransport
    if isinstance(transport, NvlinkTransport):
        return _swap_nvlink(transport, local_pixels, list(order))
    if transport.size == 1 and ops is None and getattr(local_pixels, "is_cuda", False) \
            and local_pixels.dtype == _torch().float32 and local_pixels.shape[-1] == 4:
        return local_pixels.clone(memory_format=_torch().contiguous_format)   # one rank: a copy (compositing.py:123)
    ops = ops or DeviceOps()
    shape = tuple(local_pixels.shape)
    flat = ops.as_flat(local_pixels)
    if transport.size == 1:
        return flat.clone().reshape(shape)
    return _swap_bytes(transport, flat, list(order), shape, ops)


def _swap_bytes(transport, flat, order, shape, ops):
    rank, size = transport.rank, transport.size
    n = flat.shape[0]
    if size & (size - 1):
        if rank != 0:
            transport.send(0, _wire(0, rank, 0, n, ops.to_bytes(flat)))
            return None
        flats = [None] * size
        flats[0] = flat
        for other in range(1, size):
            msg = CompositeMessage.from_bytes(transport.receive(other))
            flats[msg.sender] = ops.from_array(msg.payload)
        return ops.fold(flats, order).reshape(shape)
    v = order.index(rank)
    plan, (lo, hi) = swap_schedule(v, size, n)
    span_lo = 0
    mine = flat
    for r, (pv, keep, give) in enumerate(plan):
        partner = order[pv]
        transport.send(partner, _wire(r, rank, give[0], give[1], ops.to_bytes(mine[give[0] - span_lo:give[1] - span_lo])))
        msg = CompositeMessage.from_bytes(transport.receive(partner))
        if msg.round_index != r:
            raise CompositeError(f"round mismatch: expected {r}, got {msg.round_index} from rank {partner}")
        if msg.span_offset != keep[0] or msg.span_length != keep[1] - keep[0]:
            raise CompositeError("partner sent an unexpected span")
        kept = mine[keep[0] - span_lo:keep[1] - span_lo]
        theirs = ops.from_array(msg.payload)
        mine = ops.over(theirs, kept) if pv < v else ops.over(kept, theirs)
        span_lo = keep[0]
    rounds = len(plan)
    if rank != 0:
        transport.send(0, _wire(rounds, rank, lo, hi, ops.to_bytes(mine)))
        return None
    full = ops.empty(n)
    full[lo:hi] = mine
    for other in range(1, size):
        msg = CompositeMessage.from_bytes(transport.receive(other))
        if msg.round_index != rounds:
            raise CompositeError("stray swap-round message during collection")
        full[msg.span_offset:msg.span_offset + msg.span_length] = ops.from_array(msg.payload)
    return full.reshape(shape)


def _swap_nvlink(t, pixels, order):
    import torch
    from .device import stream_handle
    if len(order) != t.size or sorted(order) != list(range(t.size)):
        raise CompositeError("order must be a permutation of the ranks")
    shape = tuple(pixels.shape)
    if len(shape) != 3 or shape[2] != 4:
        raise CompositeError(f"expected (H, W, 4) pixels, got {shape}")
    h, w = shape[0], shape[1]
    if h * w != t.n_pixels:
        raise CompositeError(f"image has {h * w} pixels, transport arena holds {t.n_pixels}")
    if t.size == 1:
        return pixels.clone()
    canvas = t.canvas(h, w)
    if pixels.data_ptr() != canvas.data_ptr():
        canvas.copy_(pixels)
    s = stream_handle()
    # the epoch lives on the device (one bump per swap; the kernel reads it),
    # so a captured frame replays; the host counter keeps step with it
    t.epoch += 1
    _abi.check(_abi.lib().isc_swap_epoch_bump(C.c_void_p(t.flags[t.rank]), C.c_void_p(s)), "swap epoch")
    args = t.swap_args(order, epoch=0)
    fn = _abi.lib().isc_binary_swap if (t.size & (t.size - 1)) == 0 else _abi.lib().isc_direct_send
    _abi.check(fn(C.byref(args), C.c_void_p(s)), "binary_swap")
    _account(t, order)
    if not t.capturing:     # inside a CUDA-graph capture: FrameGraph.check() reads the error word
        t.check_errors(s)
    if t.rank == 0:
        return t.root_output(h, w).clone()
    return None


def binary_swap_local(group, images, order):
    """Binary swap / direct send for every rank of a :class:`LocalNvlinkGroup`
    from ONE host thread on ONE stream: the same ``isc_binary_swap`` kernel,
    launched per (stage, rank) in dependency order so no two ranks need to be
    co-resident (virtual ranks on a single GPU).  Returns rank 0's frame."""
    import torch
    from .device import stream_handle
    order = list(order)
    eps = group.endpoints
    size = group.size
    if len({ep.n_ctas for ep in eps}) != 1:
        raise CompositeError("every rank must cut the image into the same number of slices (n_ctas)")
    shape = tuple(images[0].shape)
    h, w = shape[0], shape[1]
    s = stream_handle()
    lib = _abi.lib()
    for r, ep in enumerate(eps):
        canvas = ep.canvas(h, w)
        canvas.copy_(images[r])
        ep.epoch += 1       # host and device epochs in step (launches below pass the host value)
        _abi.check(lib.isc_swap_epoch_bump(C.c_void_p(ep.flags[ep.rank]), C.c_void_p(s)), "swap epoch")
    if size == 1:
        return images[0].clone()
    if size & (size - 1):
        for r in list(range(1, size)) + [0]:
            a = eps[r].swap_args(order, finish=0)
            _abi.check(lib.isc_direct_send(C.byref(a), C.c_void_p(s)), "direct_send")
        for ep in eps:
            _account(ep, order)
        eps[0].status(s)
        return eps[0].root_output(h, w).clone()
    rounds = size.bit_length() - 1
    for r in range(size):   # stage 0: every image ready
        a = eps[r].swap_args(order, round_begin=0, round_end=0, collect=0, finish=0, publish_ready=1)
        _abi.check(lib.isc_binary_swap(C.byref(a), C.c_void_p(s)), "binary_swap")
    for rnd in range(rounds):
        for r in range(size):
            a = eps[r].swap_args(order, round_begin=rnd, round_end=rnd + 1, collect=0, finish=0, publish_ready=0)
            _abi.check(lib.isc_binary_swap(C.byref(a), C.c_void_p(s)), "binary_swap")
    for r in list(range(1, size)) + [0]:
        a = eps[r].swap_args(order, round_begin=rounds, round_end=rounds, collect=1, finish=1, publish_ready=0)
        _abi.check(lib.isc_binary_swap(C.byref(a), C.c_void_p(s)), "binary_swap")
    for ep in eps:
        _account(ep, order)
    for ep in eps:
        ep.status(s)
    return eps[0].root_output(h, w).clone()


def _account(t, order):
    """Bytes that crossed the link for this rank (float32 RGBA, 16 B/px)."""
    n, size = t.n_pixels, t.size
    if size & (size - 1):
        if t.rank == 0:
            t.received_bytes += (size - 1) * n * 16
        else:
            t.sent_bytes += n * 16
        return
    plan, (lo, hi) = swap_schedule(order.index(t.rank), size, n)
    for _, keep, give in plan:
        t.sent_bytes += (give[1] - give[0]) * 16
        t.received_bytes += (keep[1] - keep[0]) * 16
    if t.rank == 0:
        t.received_bytes += (n - (hi - lo)) * 16
    else:
        t.sent_bytes += (hi - lo) * 16
