"""ctypes binding of ``include/isaac_b200.h`` (libisaac_b200.so).

The structs below mirror the header field for field; ``check_layout()``
compares their sizes with the library's own ``isc_struct_size``.  Status
codes map onto the reference's exception classes (see the header).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ISC_LIB_PATH") or os.path.join(_HERE, "lib", "libisaac_b200.so")

ABI_VERSION = 4
MAX_SOURCES = 8
MAX_CLIP_PLANES = 8
MAX_CHAIN = 8
LUT_ENTRIES = 256
MAX_LUT_KINKS = 7
MAX_RANKS = 64
IPC_HANDLE_BYTES = 64
MAX_SWAP_CTAS = 1024
ERR_WORD = 9          # transport error word of a flag block (composite.cu kErrWord)

F32, F64, F16, BF16 = 0, 1, 2, 3
VOLUME, ISO = 0, 1
OPCODES = {"add": 1, "mul": 2, "pow": 3, "length": 4, "sum": 5, "sqrt": 6, "abs": 7, "neg": 8,
           "exp": 9, "log": 10, "min": 11, "max": 12}
TAKES_ARGUMENT = {"add", "mul", "pow", "min", "max"}
REDUCES = {"length", "sum"}


class ChainStep(C.Structure):
    _fields_ = [("op", C.c_int32), ("in_dim", C.c_int32), ("arg", C.c_float * 4), ("arg_d", C.c_double * 4)]


class Source(C.Structure):
    _fields_ = [
        ("data", C.c_void_p),
        ("stride", C.c_int64 * 4),
        ("dtype", C.c_int32),
        ("feature_dim", C.c_int32),
        ("has_guard", C.c_int32),
        ("mode", C.c_int32),
        ("iso_threshold", C.c_float),
        ("range_lo", C.c_float),
        ("range_hi", C.c_float),
        ("n_steps", C.c_int32),
        ("lut", C.c_void_p),
        ("steps", ChainStep * MAX_CHAIN),
        ("lut_linear", C.c_int32),
        ("lut_base", C.c_float * 4),
        ("lut_slope", C.c_float * 4),
        ("lut_kinks", C.c_int32),
        ("lut_kink_x", C.c_float * MAX_LUT_KINKS),
        ("lut_kink_dslope", (C.c_float * 4) * MAX_LUT_KINKS),
        ("iso_threshold_d", C.c_double),
        ("iso_exact", C.c_int32),
        ("step_ops", C.c_uint32),
    ]


class Camera(C.Structure):
    _fields_ = [
        ("origin", C.c_double * 3),
        ("fwd", C.c_double * 3),
        ("right", C.c_double * 3),
        ("up", C.c_double * 3),
        ("tan_half", C.c_double),
        ("aspect", C.c_double),
        ("width", C.c_int32),
        ("height", C.c_int32),
    ]


class ClipPlane(C.Structure):
    _fields_ = [("point", C.c_double * 3), ("normal", C.c_double * 3), ("f0", C.c_double)]


class RenderArgs(C.Structure):
    _fields_ = [
        ("camera", Camera),
        ("step", C.c_double),
        ("alpha_stop", C.c_double),
        ("interpolation", C.c_int32),
        ("n_sources", C.c_int32),
        ("n_clip", C.c_int32),
        ("guard_width", C.c_int32),
        ("brick_offset", C.c_int32 * 3),
        ("brick_size", C.c_int32 * 3),
        ("volume_size", C.c_int32 * 3),
        ("decomposition", C.c_int32 * 3),
        ("clip", ClipPlane * MAX_CLIP_PLANES),
        ("src", Source * MAX_SOURCES),
        ("out_rgba", C.c_void_p),
        ("out_stations", C.c_void_p),
        ("out_krange", C.c_void_p),
        ("out_t", C.c_void_p),
        ("out_hit", C.c_void_p),
        ("error_word", C.c_void_p),
        ("out_station_total", C.c_void_p),
        ("work_counter", C.c_void_p),
        ("ray_dirs", C.c_void_p),
        ("ray_intervals", C.c_void_p),
        ("no_layout", C.c_int32),
    ]


class SwapArgs(C.Structure):
    _fields_ = [
        ("rank", C.c_int32),
        ("size", C.c_int32),
        ("n_ctas", C.c_int32),
        ("round_begin", C.c_int32),
        ("round_end", C.c_int32),
        ("collect", C.c_int32),
        ("finish", C.c_int32),
        ("publish_ready", C.c_int32),
        ("n_pixels", C.c_int64),
        ("epoch", C.c_int64),
        ("timeout_ns", C.c_int64),
        ("order", C.c_int32 * MAX_RANKS),
        ("image", C.c_void_p * MAX_RANKS),
        ("flags", C.c_void_p * MAX_RANKS),
        ("root_out", C.c_void_p),
    ]


class ToyArgs(C.Structure):
    _fields_ = [
        ("global_size", C.c_int32 * 3),
        ("offset", C.c_int32 * 3),
        ("size", C.c_int32 * 3),
        ("guard", C.c_int32),
        ("step_index", C.c_int32),
        ("seed", C.c_int32),
        ("shear_speed", C.c_double),
        ("perturbation", C.c_double),
        ("dt", C.c_double),
        ("density", C.c_void_p),
        ("velocity", C.c_void_p),
    ]


_lib = None
_lock = threading.Lock()

_SIGNATURES = {
    "isc_abi_version": (C.c_int, []),
    "isc_last_error": (C.c_char_p, []),
    "isc_struct_size": (C.c_size_t, [C.c_int]),
    "isc_device_sm_count": (C.c_int, [C.c_int]),
    "isc_render_local": (C.c_int, [C.POINTER(RenderArgs), C.c_void_p]),
    "isc_ray_setup": (C.c_int, [C.POINTER(RenderArgs), C.c_void_p]),
    "isc_gradient_normals": (C.c_int, [C.POINTER(RenderArgs), C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                       C.c_void_p]),
    "isc_value_range": (C.c_int, [C.POINTER(Source), C.POINTER(C.c_int32), C.c_int32, C.c_void_p, C.c_void_p]),
    "isc_over": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "isc_composite_fold": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.c_int32, C.c_int64, C.c_void_p]),
    "isc_binary_swap": (C.c_int, [C.POINTER(SwapArgs), C.c_void_p]),
    "isc_direct_send": (C.c_int, [C.POINTER(SwapArgs), C.c_void_p]),
    "isc_flag_words": (C.c_int, []),
    "isc_swap_status": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int32)]),
    "isc_swap_reset": (C.c_int, [C.c_void_p, C.c_void_p]),
    "isc_swap_epoch_bump": (C.c_int, [C.c_void_p, C.c_void_p]),
    "isc_swap_error_async": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "isc_debug_occupy": (C.c_int, [C.c_int32, C.c_int32, C.c_int64, C.c_void_p]),
    "isc_arena_alloc": (C.c_int, [C.c_size_t, C.POINTER(C.c_void_p)]),
    "isc_arena_free": (C.c_int, [C.c_void_p]),
    "isc_ipc_handle": (C.c_int, [C.c_void_p, C.c_char * IPC_HANDLE_BYTES]),
    "isc_ipc_open": (C.c_int, [C.c_char * IPC_HANDLE_BYTES, C.POINTER(C.c_void_p)]),
    "isc_ipc_close": (C.c_int, [C.c_void_p]),
    "isc_enable_peer_access": (C.c_int, [C.c_int]),
    "isc_to_rgba8": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "isc_toy_fields": (C.c_int, [C.POINTER(ToyArgs), C.c_void_p]),
}

EXPORTED = tuple(_SIGNATURES)


class NativeLibraryMissing(RuntimeError):
    """The sm_100a library is not built; the product path has no fallback."""


def lib():
    """Load (once) and return the native library; raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryMissing(
                f"{LIB_PATH} not found -- build it with `python -m paper_1611_09048_b200.build_native` "
                "(there is no CPU fallback for the render/composite path)")
        handle = C.CDLL(LIB_PATH)
        for name, (res, argtypes) in _SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = argtypes
        if handle.isc_abi_version() != ABI_VERSION:
            raise NativeLibraryMissing("libisaac_b200.so ABI version mismatch; rebuild it")
        _lib = handle
        check_layout(handle)
        return _lib


def check_layout(handle=None):
    h = handle or lib()
    for which, st in enumerate((RenderArgs, Source, Camera, ClipPlane, ChainStep, SwapArgs, ToyArgs)):
        native = h.isc_struct_size(which)
        if native != C.sizeof(st):
            raise NativeLibraryMissing(f"struct {st.__name__}: ctypes {C.sizeof(st)} B != native {native} B")


_STATUS_TO_EXC = {
    1: errors.FieldError,
    2: errors.GuardContractError,
    3: errors.ChainError,
    4: errors.SceneError,
    5: errors.CompositeError,
    6: errors.TransportError,
    7: ValueError,
    8: errors.CudaError,
}


def check(status: int, what: str = "") -> None:
    if status == 0:
        return
    msg = lib().isc_last_error().decode("utf-8", "replace")
    exc = _STATUS_TO_EXC.get(status, RuntimeError)
    raise exc(f"{what}: {msg}" if what else msg)
