"""Rank transports.

* ``Transport`` -- the reference protocol (transport.py:20-28).
* ``LocalFabric`` / ``LocalTransport`` / ``run_ranks`` -- in-process queues,
  one thread per rank, same semantics as transport.py:31-133 (kept for
  host-side control messages and tests).
* ``TorchDistTransport`` -- the same byte protocol over ``torch.distributed``
  point-to-point (gloo for host bytes), one process per GPU.
* ``NvlinkTransport`` -- the B200 data plane: every rank owns a device arena
  (image + root output + flag block) allocated by the native library, the
  arenas are cross-mapped (CUDA IPC between processes, plain pointers inside
  one process), and ``binary_swap`` runs as ONE fused peer-memory kernel per
  rank (``isc_binary_swap``).  Control bytes (handle exchange, scene
  broadcast) ride on a host transport it wraps.
"""

from __future__ import annotations

import ctypes as C
import queue
import threading
from typing import Callable, Optional, Protocol

from .errors import TransportError

__all__ = ["TransportError", "Transport", "LocalFabric", "LocalTransport", "run_ranks", "TorchDistTransport",
           "NvlinkTransport", "LocalNvlinkGroup"]


class Transport(Protocol):
    rank: int
    size: int

    def send(self, to: int, data: bytes) -> None: ...

    def receive(self, from_rank: int, timeout: Optional[float] = None) -> bytes: ...

    def broadcast_from_root(self, data: Optional[bytes]) -> bytes: ...


class LocalFabric:
    """FIFO queue per (src, dst) with byte counters (transport.py:31-71)."""

    def __init__(self, size: int, default_timeout: float = 120.0):
        self.size = size
        self.default_timeout = default_timeout
        self._queues = {(s, d): queue.Queue() for s in range(size) for d in range(size)}
        self._lock = threading.Lock()
        self.sent_bytes = [0] * size
        self.received_bytes = [0] * size

    def endpoint(self, rank: int) -> "LocalTransport":
        return LocalTransport(self, rank)

    def endpoints(self) -> list:
        return [LocalTransport(self, r) for r in range(self.size)]

    def reset_counters(self) -> None:
        with self._lock:
            self.sent_bytes = [0] * self.size
            self.received_bytes = [0] * self.size

    def _send(self, src: int, dst: int, data: bytes) -> None:
        if not 0 <= dst < self.size:
            raise TransportError(f"destination rank {dst} out of range")
        with self._lock:
            self.sent_bytes[src] += len(data)
        self._queues[(src, dst)].put(data)

    def _receive(self, src: int, dst: int, timeout: Optional[float]) -> bytes:
        try:
            data = self._queues[(src, dst)].get(timeout=self.default_timeout if timeout is None else timeout)
        except queue.Empty:
            raise TransportError(f"rank {dst} timed out waiting for rank {src}") from None
        with self._lock:
            self.received_bytes[dst] += len(data)
        return data


class _HostCollectives:
    """broadcast / gather written once on top of send / receive (transport.py:86-103)."""

    def broadcast_from_root(self, data: Optional[bytes] = None) -> bytes:
        if self.rank == 0:
            if data is None:
                raise TransportError("root must provide broadcast data")
            for other in range(1, self.size):
                self.send(other, data)
            return data
        return self.receive(0)

    def gather_to_root(self, data: bytes) -> Optional[list]:
        if self.rank != 0:
            self.send(0, data)
            return None
        return [data] + [self.receive(r) for r in range(1, self.size)]

    def all_gather(self, data: bytes) -> list:
        docs = self.gather_to_root(data)
        if self.rank == 0:
            import pickle
            blob = pickle.dumps(docs)
            self.broadcast_from_root(blob)
            return docs
        import pickle
        return pickle.loads(self.broadcast_from_root(None))


class LocalTransport(_HostCollectives):
    def __init__(self, fabric: LocalFabric, rank: int):
        self.fabric = fabric
        self.rank = rank
        self.size = fabric.size

    def send(self, to: int, data: bytes) -> None:
        self.fabric._send(self.rank, to, data)

    def receive(self, from_rank: int, timeout: Optional[float] = None) -> bytes:
        return self.fabric._receive(from_rank, self.rank, timeout)


def run_ranks(size: int, body: Callable, timeout: float = 300.0) -> list:
    """One thread per rank over a LocalFabric; first failure re-raised (transport.py:106-133)."""
    fabric = LocalFabric(size)
    results: list = [None] * size
    errors: list = []

    def runner(r: int):
        try:
            results[r] = body(fabric.endpoint(r))
        except BaseException as exc:  # noqa: BLE001
            errors.append((r, exc))

    threads = [threading.Thread(target=runner, args=(r,), daemon=True) for r in range(size)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout)
        if t.is_alive():
            raise TransportError("rank thread did not finish (deadlock?)")
    if errors:
        r, exc = errors[0]
        raise RuntimeError(f"rank {r} failed: {exc}") from exc
    return results


class TorchDistTransport(_HostCollectives):
    """Byte messages over torch.distributed point-to-point.

    Uses a gloo group for host bytes (so it also runs on CPU-only test
    machines); with an NCCL default group a gloo side group is created.
    Sends are posted asynchronously (isend) so the reference's
    send-then-receive exchange pattern cannot deadlock.
    """

    def __init__(self, group=None):
        import torch.distributed as dist
        self._dist = dist
        if group is None:
            group = dist.group.WORLD
            if dist.get_backend(group) != "gloo":
                group = dist.new_group(backend="gloo")
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self._pending: list = []
        self.sent_bytes = 0
        self.received_bytes = 0

    def _global(self, r: int) -> int:
        return self._dist.get_global_rank(self.group, r) if self.group is not self._dist.group.WORLD else r

    def send(self, to: int, data: bytes) -> None:
        import torch
        if not 0 <= to < self.size:
            raise TransportError(f"destination rank {to} out of range")
        head = torch.tensor([len(data)], dtype=torch.int64)
        body = torch.frombuffer(bytearray(data), dtype=torch.uint8) if data else torch.empty(0, dtype=torch.uint8)
        dst = self._global(to)
        self._pending.append((self._dist.isend(head, dst, group=self.group), head))
        if len(data):
            self._pending.append((self._dist.isend(body, dst, group=self.group), body))
        self.sent_bytes += len(data)

    def receive(self, from_rank: int, timeout: Optional[float] = None) -> bytes:
        import torch
        src = self._global(from_rank)
        head = torch.empty(1, dtype=torch.int64)
        self._dist.recv(head, src, group=self.group)
        n = int(head.item())
        body = torch.empty(n, dtype=torch.uint8)
        if n:
            self._dist.recv(body, src, group=self.group)
        self.received_bytes += n
        self._reap()
        return body.numpy().tobytes()

    def _reap(self) -> None:
        keep = []
        for work, buf in self._pending:
            if not work.is_completed():
                keep.append((work, buf))
        self._pending = keep

    def flush(self) -> None:
        for work, _ in self._pending:
            work.wait()
        self._pending = []


# --------------------------------------------------------------------------
# NVLink data plane


class _CudaArray:
    """Minimal __cuda_array_interface__ provider to view arena memory as a tensor."""

    def __init__(self, ptr: int, shape: tuple, typestr: str):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


class _Arena:
    """One rank's device arena: [image n*16 B | root output n*16 B | flags]."""

    def __init__(self, n_pixels: int, device_index: int):
        from . import _abi
        import torch
        self.n_pixels = n_pixels
        self.device_index = device_index
        self.flag_words = _abi.lib().isc_flag_words()
        self.image_bytes = n_pixels * 16
        total = 2 * self.image_bytes + self.flag_words * 8
        p = C.c_void_p()
        with torch.cuda.device(device_index):
            _abi.check(_abi.lib().isc_arena_alloc(total, C.byref(p)), "arena alloc")
        self.base = int(p.value)
        self.image_ptr = self.base
        self.out_ptr = self.base + self.image_bytes
        self.flags_ptr = self.base + 2 * self.image_bytes

    def tensor(self, ptr: int, shape: tuple):
        import torch
        return torch.as_tensor(_CudaArray(ptr, shape, "<f4"), device=f"cuda:{self.device_index}")

    def free(self):
        from . import _abi
        if self.base:
            import torch
            with torch.cuda.device(self.device_index):
                _abi.lib().isc_arena_free(C.c_void_p(self.base))
            self.base = 0


class NvlinkTransport(_HostCollectives):
    """Peer-memory compositing transport (one per rank).

    Collective constructor: every rank calls ``NvlinkTransport(host, n_pixels)``
    with the same ``n_pixels``; arenas are exchanged through the host
    transport ``host`` (CUDA IPC handles) -- or, for ranks living in one
    process, built by :class:`LocalNvlinkGroup`.  ``send`` / ``receive`` /
    ``broadcast_from_root`` delegate to ``host`` so this object satisfies the
    reference ``Transport`` protocol.
    """

    timeout_s: float = 30.0
    # True: every binary_swap synchronises its stream to check the spin-wait
    # error word (the reference raises from the call).  False: the word is
    # copied to pinned memory on the stream and checked on a later call or
    # at flush(), so the host keeps enqueueing frames (pipelined rendering).
    sync_errors: bool = True

    def __init__(self, host=None, n_pixels: int = 0, *, _local=None):
        from . import _abi
        import torch
        self.host = host
        self._abi = _abi
        if _local is not None:
            group, rank = _local
            self.rank, self.size = rank, group.size
            self.arena = group.arenas[rank]
            self.images = [a.image_ptr for a in group.arenas]
            self.flags = [a.flags_ptr for a in group.arenas]
            self.root_out = group.arenas[0].out_ptr
            self._opened = []
        else:
            self.rank, self.size = host.rank, host.size
            dev = torch.cuda.current_device()
            self.arena = _Arena(n_pixels, dev)
            buf = (C.c_char * _abi.IPC_HANDLE_BYTES)()
            _abi.check(_abi.lib().isc_ipc_handle(C.c_void_p(self.arena.base), buf), "ipc handle")
            mine = bytes(buf)
            handles = host.all_gather(mine)
            self._opened = []
            self.images, self.flags = [], []
            root_base = None
            for r, h in enumerate(handles):
                if r == self.rank:
                    base = self.arena.base
                else:
                    p = C.c_void_p()
                    hb = (C.c_char * _abi.IPC_HANDLE_BYTES).from_buffer_copy(h)
                    _abi.check(_abi.lib().isc_ipc_open(hb, C.byref(p)), f"ipc open rank {r}")
                    base = int(p.value)
                    self._opened.append(base)
                self.images.append(base)
                self.flags.append(base + 2 * self.arena.image_bytes)
                if r == 0:
                    root_base = base
            self.root_out = root_base + self.arena.image_bytes
        self.n_pixels = self.arena.n_pixels
        self.epoch = 0
        self._status_host = torch.zeros(1, dtype=torch.int64).pin_memory()   # allocated up front
        self._err_slots = [torch.zeros(1, dtype=torch.int64).pin_memory() for _ in range(4)]
        self._pending: list = []      # (event, slot) of deferred error checks
        self._next_slot = 0
        sms = _abi.lib().isc_device_sm_count(self.arena.device_index)
        self.n_ctas = max(1, sms if sms > 0 else 148)
        self.sent_bytes = 0
        self.received_bytes = 0

    # -- Transport protocol (control plane) --
    def send(self, to: int, data: bytes) -> None:
        self.host.send(to, data)

    def receive(self, from_rank: int, timeout: Optional[float] = None) -> bytes:
        return self.host.receive(from_rank, timeout)

    def canvas(self, height: int, width: int):
        """This rank's arena image as an (H, W, 4) float32 tensor: render into
        it (``render_local(..., out=canvas)``) and ``binary_swap`` needs no copy."""
        if height * width != self.n_pixels:
            raise TransportError(f"canvas of {height}x{width} px does not match the arena ({self.n_pixels} px)")
        return self.arena.tensor(self.arena.image_ptr, (height, width, 4))

    def root_output(self, height: int, width: int):
        if self.rank != 0:
            raise TransportError("only rank 0 holds the composited frame")
        return self.arena.tensor(self.arena.out_ptr, (height, width, 4))

    def swap_args(self, order, **kw):
        a = self._abi.SwapArgs()
        a.rank, a.size, a.n_ctas = self.rank, self.size, kw.get("n_ctas", self.n_ctas)
        a.round_begin = kw.get("round_begin", 0)
        a.round_end = kw.get("round_end", 64)
        a.collect = kw.get("collect", 1)
        a.finish = kw.get("finish", 1)
        a.publish_ready = kw.get("publish_ready", 1)
        a.n_pixels = self.n_pixels
        a.epoch = self.epoch
        a.timeout_ns = int(kw.get("timeout_s", self.timeout_s) * 1e9)
        for i in range(self.size):
            a.order[i] = int(order[i])
            a.image[i] = self.images[i]
            a.flags[i] = self.flags[i]
        a.root_out = self.root_out
        return a

    def status(self, stream_ptr: int) -> None:
        code = C.c_int32(0)
        self._abi.check(self._abi.lib().isc_swap_status(C.c_void_p(self.flags[self.rank]), C.c_void_p(stream_ptr),
                                                        C.c_void_p(self._status_host.data_ptr()), C.byref(code)),
                        "swap status")
        if code.value:
            raise TransportError(f"rank {self.rank}: peer did not arrive within {self.timeout_s}s "
                                 "(binary swap spin-wait timed out)")

    def check_errors(self, stream_ptr: int) -> None:
        """After a swap launch: synchronous check (``sync_errors``) or a
        deferred one -- the error word is copied into a pinned slot on the
        stream and examined once that copy has completed."""
        if self.sync_errors:
            self.status(stream_ptr)
            return
        import torch
        self._poll(block=len(self._pending) >= len(self._err_slots))
        slot = self._err_slots[self._next_slot]
        self._next_slot = (self._next_slot + 1) % len(self._err_slots)
        stream = torch.cuda.ExternalStream(stream_ptr)
        with torch.cuda.stream(stream):
            slot.copy_(self._error_word(), non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
        self._pending.append((ev, slot))

    def flush(self) -> None:
        """Wait for every deferred error check; raise if a swap timed out."""
        self._poll(block=True, all_=True)

    def _error_word(self):
        import torch
        flags = torch.as_tensor(_CudaArray(self.flags[self.rank], (16,), "<i8"),
                                device=f"cuda:{self.arena.device_index}")
        return flags[9:10]

    def _poll(self, block: bool, all_: bool = False) -> None:
        bad = False
        while self._pending:
            ev, slot = self._pending[0]
            if not ev.query():
                if not (block or all_):
                    break
                ev.synchronize()
                block = False
            self._pending.pop(0)
            bad = bad or int(slot.item()) != 0
        if bad:
            self._error_word().zero_()
            raise TransportError(f"rank {self.rank}: peer did not arrive within {self.timeout_s}s "
                                 "(binary swap spin-wait timed out)")

    def close(self) -> None:
        for p in self._opened:
            self._abi.lib().isc_ipc_close(C.c_void_p(p))
        self._opened = []


class LocalNvlinkGroup:
    """All ranks' arenas inside one process (threads or virtual ranks on one
    GPU).  ``devices[r]`` is rank r's CUDA device; peer access is enabled
    between distinct devices so the fused kernel can load peer memory."""

    def __init__(self, size: int, n_pixels: int, devices=None):
        from . import _abi
        import torch
        devices = list(devices) if devices is not None else [torch.cuda.current_device()] * size
        self.size = size
        self.devices = devices
        for d in set(devices):
            with torch.cuda.device(d):
                for p in set(devices) - {d}:
                    _abi.check(_abi.lib().isc_enable_peer_access(p), "peer access")
        self.arenas = [_Arena(n_pixels, d) for d in devices]
        self.fabric = LocalFabric(size)
        self.endpoints = [NvlinkTransport(self.fabric.endpoint(r), _local=(self, r)) for r in range(size)]

    def close(self):
        for a in self.arenas:
            a.free()
