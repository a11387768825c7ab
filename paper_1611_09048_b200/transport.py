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

import collections
import ctypes as C
import threading
import time
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
    """In-process rank fabric with the reference's semantics
    (transport.py:31-71): messages are delivered reliably and in order per
    (sender, receiver) pair, a receive gives up after a timeout with
    TransportError, and per-rank byte counters back the compositing balance
    checks.  Built on one condition-variable mailbox per receiving rank."""

    def __init__(self, size: int, default_timeout: float = 120.0):
        self.size = size
        self.default_timeout = default_timeout
        self._mail = [_Mailbox(size) for _ in range(size)]
        self._count_lock = threading.Lock()
        self.sent_bytes = [0] * size
        self.received_bytes = [0] * size

    def endpoint(self, rank: int) -> "LocalTransport":
        return LocalTransport(self, rank)

    def endpoints(self) -> list:
        return list(map(self.endpoint, range(self.size)))

    def reset_counters(self) -> None:
        with self._count_lock:
            self.sent_bytes = [0] * self.size
            self.received_bytes = [0] * self.size

    def _count(self, counters: list, rank: int, n: int) -> None:
        with self._count_lock:
            counters[rank] += n

    def _send(self, src: int, dst: int, data: bytes) -> None:
        if dst < 0 or dst >= self.size:
            raise TransportError(f"destination rank {dst} out of range")
        self._count(self.sent_bytes, src, len(data))
        self._mail[dst].put(src, data)

    def _receive(self, src: int, dst: int, timeout: Optional[float]) -> bytes:
        limit = self.default_timeout if timeout is None else timeout
        data = self._mail[dst].take(src, limit)
        if data is None:
            raise TransportError(f"rank {dst} timed out waiting for rank {src}")
        self._count(self.received_bytes, dst, len(data))
        return data


class _Mailbox:
    """Per-sender FIFOs of one receiving rank behind a single condition variable."""

    def __init__(self, senders: int):
        self._fifo = [collections.deque() for _ in range(senders)]
        self._cv = threading.Condition()

    def put(self, src: int, data: bytes) -> None:
        with self._cv:
            self._fifo[src].append(data)
            self._cv.notify_all()

    def take(self, src: int, timeout: float) -> Optional[bytes]:
        with self._cv:
            if not self._cv.wait_for(lambda: len(self._fifo[src]) > 0, timeout):
                return None
            return self._fifo[src].popleft()


class _HostCollectives:
    """broadcast / gather / all-gather written once on top of send / receive
    (the reference's LocalTransport collectives, transport.py:86-103)."""

    def broadcast_from_root(self, data: Optional[bytes] = None) -> bytes:
        if self.rank != 0:
            return self.receive(0)
        if data is None:
            raise TransportError("root must provide broadcast data")
        for dst in range(1, self.size):
            self.send(dst, data)
        return data

    def gather_to_root(self, data: bytes) -> Optional[list]:
        if self.rank == 0:
            return [data, *(self.receive(src) for src in range(1, self.size))]
        self.send(0, data)
        return None

    def all_gather(self, data: bytes) -> list:
        import pickle
        docs = self.gather_to_root(data)
        blob = self.broadcast_from_root(pickle.dumps(docs) if self.rank == 0 else None)
        return docs if self.rank == 0 else pickle.loads(blob)


class LocalTransport(_HostCollectives):
    """One rank's endpoint on a LocalFabric."""

    def __init__(self, fabric: LocalFabric, rank: int):
        self.fabric, self.rank, self.size = fabric, rank, fabric.size

    def send(self, to: int, data: bytes) -> None:
        self.fabric._send(self.rank, to, data)

    def receive(self, from_rank: int, timeout: Optional[float] = None) -> bytes:
        return self.fabric._receive(from_rank, self.rank, timeout)


def run_ranks(size: int, body: Callable, timeout: float = 300.0) -> list:
    """``body(endpoint)`` on one daemon thread per rank over a fresh
    LocalFabric; per-rank results in rank order.  A rank that is still running
    after ``timeout`` raises TransportError; otherwise the lowest failing
    rank's exception is re-raised (transport.py:106-133)."""
    fabric = LocalFabric(size)
    outcome: list = [None] * size          # ("ok", value) | ("err", exc)

    def runner(rank: int) -> None:
        try:
            outcome[rank] = ("ok", body(fabric.endpoint(rank)))
        except BaseException as exc:  # noqa: BLE001 -- surfaced below
            outcome[rank] = ("err", exc)

    threads = [threading.Thread(target=runner, args=(r,), daemon=True) for r in range(size)]
    for t in threads:
        t.start()
    deadline = time.monotonic() + timeout
    for t in threads:
        t.join(max(0.0, deadline - time.monotonic()))
        if t.is_alive():
            raise TransportError("rank thread did not finish (deadlock?)")
    for rank, (kind, val) in enumerate(outcome):
        if kind == "err":
            raise RuntimeError(f"rank {rank} failed: {val}") from val
    return [val for _, val in outcome]


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
            self._agreed_ctas = group.n_ctas
        else:
            self.rank, self.size = host.rank, host.size
            dev = torch.cuda.current_device()
            self.arena = _Arena(n_pixels, dev)
            buf = (C.c_char * _abi.IPC_HANDLE_BYTES)()
            _abi.check(_abi.lib().isc_ipc_handle(C.c_void_p(self.arena.base), buf), "ipc handle")
            sms = _abi.lib().isc_device_sm_count(dev)
            want = min(_abi.MAX_SWAP_CTAS, sms if sms > 0 else 148)
            # every rank must slice the image identically: agree on the
            # smallest grid any rank proposes (ranks may sit on different SKUs)
            docs = host.all_gather(want.to_bytes(4, "little") + bytes(buf))
            self._agreed_ctas = min(int.from_bytes(d[:4], "little") for d in docs)
            handles = [d[4:] for d in docs]
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
        self.capturing = False        # set by FrameGraph while a frame is captured
        self._status_host = torch.zeros(1, dtype=torch.int64).pin_memory()   # allocated up front
        self._err_slots = [torch.zeros(1, dtype=torch.int64).pin_memory() for _ in range(4)]
        self._pending: list = []      # (event, slot) of deferred error checks
        self._next_slot = 0
        # slices (= CTAs) of the swap kernel; equal on every rank by
        # construction.  Changing it is a collective decision: set the same
        # value on every rank.
        self.n_ctas = self._agreed_ctas
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
        a.epoch = kw.get("epoch", self.epoch)     # 0: the device-resident epoch (isc_swap_epoch_bump)
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
        deferred one -- the library copies the error word into a pinned slot
        on the swap's own stream (``isc_swap_error_async``, the same raw
        handle the kernel was launched on) and a torch event recorded on the
        current stream after it tells when the slot can be read."""
        if self.sync_errors:
            self.status(stream_ptr)
            return
        import torch
        cur = torch.cuda.current_stream()
        if int(cur.cuda_stream) != int(stream_ptr):
            raise TransportError("check_errors must run on the stream the swap was launched on")
        self._poll(block=len(self._pending) >= len(self._err_slots))
        slot = self._err_slots[self._next_slot]
        self._next_slot = (self._next_slot + 1) % len(self._err_slots)
        slot.zero_()
        self._abi.check(self._abi.lib().isc_swap_error_async(C.c_void_p(self.flags[self.rank]),
                                                             C.c_void_p(slot.data_ptr()), C.c_void_p(stream_ptr)),
                        "swap error copy")
        ev = torch.cuda.Event()
        ev.record(cur)
        self._pending.append((ev, slot))

    def flush(self) -> None:
        """Wait for every deferred error check; raise if a swap timed out."""
        self._poll(block=True, all_=True)

    def _error_word(self):
        import torch
        flags = torch.as_tensor(_CudaArray(self.flags[self.rank], (16,), "<i8"),
                                device=f"cuda:{self.arena.device_index}")
        return flags[self._abi.ERR_WORD:self._abi.ERR_WORD + 1]

    def reset(self) -> None:
        """Collective recovery after a TransportError: every rank drains its
        stream, zeroes its own flag block and restarts at epoch 1 behind two
        host barriers, so no rank polls a half-reset block.  (A timed-out
        CTA leaves its counters one short for good, so without a reset
        every later swap would time out too.)"""
        import torch
        from .device import stream_handle
        torch.cuda.synchronize(self.arena.device_index)
        self.host.all_gather(b"")
        s = stream_handle()
        self._abi.check(self._abi.lib().isc_swap_reset(C.c_void_p(self.flags[self.rank]), C.c_void_p(s)),
                        "swap reset")
        torch.cuda.synchronize(self.arena.device_index)
        self.host.all_gather(b"")
        self.epoch = 0
        self._pending = []

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
        sms = min(_abi.lib().isc_device_sm_count(d) for d in set(devices))
        self.n_ctas = min(_abi.MAX_SWAP_CTAS, sms if sms > 0 else 148)
        self.fabric = LocalFabric(size)
        self.endpoints = [NvlinkTransport(self.fabric.endpoint(r), _local=(self, r)) for r in range(size)]

    def set_n_ctas(self, n: int) -> None:
        """Slice count of every rank's swap (must be equal across ranks)."""
        for ep in self.endpoints:
            ep.n_ctas = n

    def reset(self) -> None:
        """Zero every rank's flag block and restart all ranks at epoch 1."""
        import torch
        from .device import stream_handle
        torch.cuda.synchronize()
        for ep in self.endpoints:
            with torch.cuda.device(ep.arena.device_index):
                _abi_check_reset(ep.flags[ep.rank], stream_handle())
            ep.epoch = 0
            ep._pending = []
        torch.cuda.synchronize()

    def close(self):
        for a in self.arenas:
            a.free()


def _abi_check_reset(flags_ptr: int, stream: int) -> None:
    from . import _abi
    _abi.check(_abi.lib().isc_swap_reset(C.c_void_p(flags_ptr), C.c_void_p(stream)), "swap reset")
