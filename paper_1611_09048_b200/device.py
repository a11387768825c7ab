"""Device plumbing shared by the render and composite wrappers: torch is used
for device memory and streams only; every computation goes through the C-ABI."""

from __future__ import annotations

import ctypes as C
import threading
from collections import OrderedDict

import numpy as np
import torch

from . import _abi

_DTYPES = {torch.float32: _abi.F32, torch.float64: _abi.F64, torch.float16: _abi.F16, torch.bfloat16: _abi.BF16}
DEVICE_DTYPES = frozenset(_DTYPES)   # dtypes the kernels read in place


_CUDA_OK = False


def require_cuda() -> torch.device:
    global _CUDA_OK
    if not _CUDA_OK:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1611_09048_b200 renders on a CUDA device (sm_100a); none is available "
                               "and there is no CPU fallback")
        _abi.lib()
        _CUDA_OK = True
    return torch.device("cuda", torch.cuda.current_device())


_RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream_handle(stream=None, device_index=None) -> int:
    """Raw cudaStream_t of ``stream`` (default: the current stream of
    ``device_index`` / the current device) -- without building a Stream
    object on the per-frame path."""
    if stream is not None:
        return int(stream.cuda_stream)
    if _RAW_STREAM is not None:
        return int(_RAW_STREAM(torch.cuda.current_device() if device_index is None else device_index))
    return int(torch.cuda.current_stream().cuda_stream)


def as_device_field(array, device: torch.device) -> torch.Tensor:
    """Zero-copy for CUDA tensors on ``device``; numpy / host tensors are staged
    (one H2D copy).  Integer arrays are converted to float32."""
    if isinstance(array, torch.Tensor):
        t = array
        if t.device != device:
            t = t.to(device, non_blocking=True)
    else:
        a = np.asarray(array)
        if a.dtype not in (np.float32, np.float64, np.float16):
            a = a.astype(np.float32)
        t = torch.from_numpy(np.ascontiguousarray(a)).to(device, non_blocking=False)
    if t.dtype not in _DTYPES:
        t = t.to(torch.float32)
    return t


def dtype_code(t: torch.Tensor) -> int:
    return _DTYPES[t.dtype]


class LutCache:
    """Device float32 LUTs keyed by content, so an unchanged transfer function
    is uploaded once and steering changes cost one 4 KB H2D copy."""

    _SLOTS = 8

    def __init__(self, capacity: int = 64):
        self._cache: "OrderedDict[tuple, torch.Tensor]" = OrderedDict()
        self._lock = threading.Lock()       # rank threads share one cache
        self.capacity = capacity
        self.uploads = 0
        self._staging = None                # pinned slots + the events of their last copies
        self._slot = 0

    def _upload(self, host: np.ndarray, device: torch.device) -> torch.Tensor:
        """Stream-ordered H2D copy through a ring of pinned staging slots (no
        stream synchronisation, no pinned allocation per upload)."""
        if device.type != "cuda" or host.shape != (256, 4):
            return torch.from_numpy(host).to(device)
        with self._lock:
            if self._staging is None:
                self._staging = [[torch.empty((256, 4), dtype=torch.float32).pin_memory(), None]
                                 for _ in range(self._SLOTS)]
            slot = self._staging[self._slot]
            self._slot = (self._slot + 1) % self._SLOTS
            if slot[1] is not None:
                slot[1].synchronize()       # that slot's previous copy (8 uploads ago)
            slot[0].numpy()[:] = host
            dev = torch.empty((256, 4), dtype=torch.float32, device=device)
            dev.copy_(slot[0], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            slot[1] = ev
        return dev

    def get(self, lut: np.ndarray, device: torch.device) -> torch.Tensor:
        host = np.ascontiguousarray(lut, dtype=np.float32)
        key = (device.index, host.tobytes())
        with self._lock:
            t = self._cache.get(key)
            if t is not None:
                self._cache.move_to_end(key)
                return t
        # pinned staging + stream-ordered copy: a pageable .to(device) would
        # synchronise the stream and stall the host behind the previous frame
        t = self._upload(host, device)
        with self._lock:
            self.uploads += 1
            self._cache[key] = t
            if len(self._cache) > self.capacity:
                self._cache.popitem(last=False)
        return t

    def clear(self) -> None:
        with self._lock:
            self._cache.clear()


LUTS = LutCache()


def ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def c_ptr(t) -> C.c_void_p:
    return C.c_void_p(ptr(t))
