"""Brick rendering entry point: ``render_local`` over the sm_100a kernel.

Drop-in for ``insitu.raycast.render_local`` (raycast.py:492-541): same
arguments (a rank context exposing ``domain``, ``global_volume``,
``registry``, ``functor_registry``, ``limits``; a ``SceneState``; optional
``plans`` and ``station_recorder``) and the same result type, except that
``LocalImage.pixels`` is a CUDA float32 tensor (H, W, 4) of premultiplied
RGBA instead of a float64 numpy array.  All per-pixel work -- ray setup,
clipping, the station march, sampling, chains, classification, iso-surfaces
and front-to-back compositing -- runs in ``isc_render_local``; this module
only packs the argument block.

``station_recorder(k, pixel_ids)`` is honoured by replaying the per-pixel
station ranges the kernel reports (stations of a pixel are contiguous from
its k_lo), which reproduces the reference's callback sequence exactly.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import threading
import weakref
from dataclasses import dataclass
from typing import Callable, Optional, Sequence

import numpy as np
import torch

from . import _abi
from .device import DEVICE_DTYPES, LUTS, as_device_field, dtype_code, ptr, require_cuda, stream_handle
from .errors import FieldError, GuardContractError
from .fields import LocalDomain, SourceHandle, SourceRegistry
from .functors import ChainLimits, FunctorChain, FunctorRegistry, device_program, parse_chain
from .scene import ISO_MODE, Camera, RenderSettings, SceneState, TransferFunction

StationRecorder = Callable[[int, np.ndarray], None]

__all__ = ["LocalImage", "SourcePlan", "build_plans", "render_local", "RankContext", "pack_render_args",
           "ray_box_intersection", "ray_setup"]


class LocalImage:
    """One rank's partial image (raycast.py:38-50).  ``pixels`` is a CUDA
    float32 (H, W, 4) premultiplied tensor; ``stations`` is resolved lazily
    from the device station counters (one reduction + sync on first access)."""

    def __init__(self, width: int, height: int, pixels, order_key: int = 0, stations=0):
        self.width = width
        self.height = height
        self.pixels = pixels
        self.order_key = order_key
        self._stations = stations
        self.station_counts = None     # (H*W,) uint32 device tensor when kept
        self.krange = None             # (H*W, 4) int32 device tensor when kept
        self._error_word = None

    @property
    def stations(self) -> int:
        s = self._stations
        if callable(s):
            s = int(s())
            self._stations = s
        return s

    @stations.setter
    def stations(self, v):
        self._stations = v

    def check(self) -> "LocalImage":
        """Raise GuardContractError if the kernel saw a guard-contract violation."""
        if self._error_word is not None:
            n = int(self._error_word.item()) & 0xFFFFFFFF
            self._error_word = None
            if n:
                raise GuardContractError(f"{n} trilinear reads beyond the guard halo")
        return self

    @staticmethod
    def blank(width: int, height: int, order_key: int = 0) -> "LocalImage":
        dev = require_cuda()
        return LocalImage(width, height, torch.zeros((height, width, 4), device=dev), order_key)


@dataclass(frozen=True)
class SourcePlan:
    """Per-active-source render inputs (raycast.py:53-63)."""

    source_id: int
    handle: SourceHandle
    domain: LocalDomain
    chain: FunctorChain
    tf: TransferFunction
    mode: str
    iso_threshold: float


def build_plans(registry: SourceRegistry, functor_registry: FunctorRegistry, limits: ChainLimits,
                scene: SceneState) -> list:
    """Active sources in id order with parsed chains (raycast.py:66-93)."""
    known = set(registry.source_ids)
    plans = []
    for sid in sorted(scene.settings.active_set):
        if sid not in known:
            raise ValueError(f"active source id {sid} is not registered")
        handle = registry.render_handle(sid)
        chain = parse_chain(scene.chain_text(sid), functor_registry, limits, handle.descriptor.feature_dim)
        plans.append(SourcePlan(sid, handle, registry.domain, chain, scene.transfer_function(sid),
                                scene.settings.mode(sid), scene.settings.iso_threshold(sid)))
    return plans


@dataclass
class RankContext:
    """What ``render_local`` reads from a rank (runtime.py:263-281, subset)."""

    global_volume: object
    domain: LocalDomain
    registry: SourceRegistry
    functor_registry: FunctorRegistry
    limits: ChainLimits
    transport: object = None


def _strides(t: torch.Tensor):
    s = list(t.stride())
    return (s[0], s[1], s[2], s[3] if t.dim() == 4 else 1)


def pack_render_args(domain, volume, scene: SceneState, plans: Sequence[SourcePlan], device,
                     keep: list, analytic_lut: bool = True) -> _abi.RenderArgs:
    """Fill an ``isc_render_args`` block.  ``keep`` collects the tensors whose
    device pointers the block references (they must outlive the launch)."""
    a = _abi.RenderArgs()
    cam = scene.camera
    w, h = cam.image_size
    fwd, right, up = cam.basis()
    a.camera.origin[:] = [float(v) for v in cam.position]
    a.camera.fwd[:] = fwd.tolist()
    a.camera.right[:] = right.tolist()
    a.camera.up[:] = up.tolist()
    a.camera.tan_half = math.tan(cam.vertical_fov / 2.0)
    a.camera.aspect = w / h
    a.camera.width, a.camera.height = int(w), int(h)
    st = scene.settings
    a.step = float(st.step_length)
    a.alpha_stop = float(st.early_termination_alpha)
    a.interpolation = 1 if st.interpolation else 0
    a.guard_width = int(domain.guard_width)
    a.brick_offset[:] = [int(v) for v in domain.offset]
    a.brick_size[:] = [int(v) for v in domain.size]
    a.volume_size[:] = [int(v) for v in volume.size]
    a.decomposition[:] = [int(v) for v in volume.decomposition]
    if len(scene.clip_planes) > _abi.MAX_CLIP_PLANES:
        raise ValueError(f"at most {_abi.MAX_CLIP_PLANES} clip planes")
    origin = np.asarray(cam.position, dtype=np.float64)
    a.n_clip = len(scene.clip_planes)
    for i, plane in enumerate(scene.clip_planes):
        n = np.asarray(plane.normal)
        a.clip[i].point[:] = [float(v) for v in plane.point]
        a.clip[i].normal[:] = n.tolist()
        a.clip[i].f0 = float(np.dot(origin - np.asarray(plane.point), n))  # raycast.py:133
    if len(plans) > _abi.MAX_SOURCES:
        raise ValueError(f"at most {_abi.MAX_SOURCES} active sources per render")
    a.n_sources = len(plans)
    for i, plan in enumerate(plans):
        s = a.src[i]
        hnd = plan.handle
        array, guard = hnd.device_view(domain)
        t = as_device_field(array, device)
        dim = hnd.descriptor.feature_dim
        need = tuple(domain.size[a_] + 2 * guard for a_ in (2, 1, 0))
        if tuple(t.shape[:3]) != need:
            raise FieldError(f"source {hnd.descriptor.name!r}: array shape {tuple(t.shape)} does not match "
                             f"domain size + 2*guard {need}")
        if hnd.descriptor.has_guard and st.interpolation and guard < domain.guard_width:
            raise FieldError(f"source {hnd.descriptor.name!r} declares a guard of {guard} cells but the "
                             f"domain promises {domain.guard_width}")
        keep.append(t)
        sz, sy, sx, sc = _strides(t)
        # The kernel indexes with the domain guard; re-base the pointer when
        # the array carries a different halo width (fields.py:274-276).
        shift = (guard - domain.guard_width) * (sz + sy + sx)
        s.data = ptr(t) + shift * t.element_size()
        s.stride[:] = [sz, sy, sx, sc]
        s.dtype = dtype_code(t)
        s.feature_dim = dim
        s.has_guard = 1 if hnd.descriptor.has_guard else 0
        s.mode = _abi.ISO if plan.mode == ISO_MODE else _abi.VOLUME
        s.iso_threshold = float(plan.iso_threshold)
        s.iso_threshold_d = float(plan.iso_threshold)
        # float64 iso decisions: scalar sources whose chain is add / mul only
        # (exactly reproducible in the reference's float64 order)
        s.iso_exact = 1 if (dim == 1 and all(op in (_abi.OPCODES["add"], _abi.OPCODES["mul"])
                                             for op, _, _ in device_program(plan.chain))) else 0
        prog = device_program(plan.chain)
        lo, hi = (float(v) for v in plan.tf.value_range)
        if plan.mode != ISO_MODE:
            prog, lo, hi = fold_affine_tail(prog, lo, hi)
        s.range_lo, s.range_hi = lo, hi
        lut = LUTS.get(plan.tf.lut, device)
        keep.append(lut)
        s.lut = ptr(lut)
        pw = lut_analytic(plan.tf.lut) if analytic_lut else None
        if pw is not None:
            base, slope, kinks = pw
            s.lut_linear = 1
            s.lut_base[:] = [float(v) for v in base]
            s.lut_slope[:] = [float(v) for v in slope]
            s.lut_kinks = len(kinks)
            for k, (xk, d) in enumerate(kinks):
                s.lut_kink_x[k] = xk
                s.lut_kink_dslope[k][:] = [float(v) for v in d]
        s.n_steps = len(prog)
        for j, (op, in_dim, arg) in enumerate(prog):
            s.steps[j].op = op
            s.steps[j].in_dim = in_dim
            s.steps[j].arg[:] = [float(v) for v in arg]
            s.steps[j].arg_d[:] = [float(v) for v in arg]
            s.step_ops |= (op & 0xF) << (4 * j)
    return a


def fold_affine_tail(prog, lo: float, hi: float):
    """Fold the trailing scalar add / mul steps of a volume source's device
    program into its classification range.  The chain's last steps map the
    scalar v to v*M + A (functors.py:212-222); classify_array normalises
    (v*M + A - lo) / (hi - lo) (scene.py:139-152), which for M > 0 equals
    (v - lo') / (hi' - lo') with lo' = (lo - A) / M, hi' = lo' + (hi - lo) / M:
    the same value in real arithmetic (float32 rounding moves the LUT
    coordinate by a few ulps, far inside the 1e-3 image tolerance), two
    device steps fewer per sample.  Iso sources keep their chain: their sign
    tests follow the reference's float64 order exactly (march_multi.cu)."""
    add_op, mul_op = _abi.OPCODES["add"], _abi.OPCODES["mul"]
    j = len(prog)
    while j > 0 and prog[j - 1][0] in (add_op, mul_op) and prog[j - 1][1] == 1:
        j -= 1
    if j == len(prog):
        return prog, lo, hi
    m, a = 1.0, 0.0
    for op, _, arg in prog[j:]:
        c = float(arg[0])
        if op == mul_op:
            m, a = m * c, a * c
        else:
            a = a + c
    if not (math.isfinite(m) and math.isfinite(a) and m > 0.0):
        return prog, lo, hi
    lo2 = (lo - a) / m
    hi2 = lo2 + (hi - lo) / m
    if not (math.isfinite(lo2) and math.isfinite(hi2) and np.float32(lo2) < np.float32(hi2)):
        return prog, lo, hi
    return prog[:j], lo2, hi2


class _ArgsCache:
    """Packed launch blocks of recent (scene, plans, domain, volume) objects.
    A frame that re-renders the same immutable scene objects (a static view,
    the bench loop) reuses the 3 KB block instead of re-packing it; every
    reuse re-validates what the block points at: each source's device array
    (pointer, shape, strides, dtype, guard) and each transfer function's LUT
    bytes.  Entries hold only weak references to the key objects (an ``id``
    reused by a new object fails the identity check) and strong references to
    the LUT tensors the block points at -- never to simulation fields.
    Sources staged per frame (numpy, host samplers) are never cached."""

    def __init__(self, capacity: int = 16):
        self._entries: "dict" = {}
        self._lock = threading.Lock()
        self.capacity = capacity

    @staticmethod
    def _fingerprint(plans, domain, device):
        fp, fields = [], []
        for plan in plans:
            array, guard = plan.handle.device_view(domain)
            # only zero-copy sources: a CUDA tensor on the render device whose
            # dtype the kernels read directly.  Anything as_device_field would
            # convert or move (integer dtypes, another GPU) gets a fresh copy
            # per frame, and a block pointing at last frame's copy would read
            # freed (and stale) memory.
            if not (isinstance(array, torch.Tensor) and array.is_cuda and array.device == device
                    and array.dtype in DEVICE_DTYPES):
                return None, None
            fp.append((array.data_ptr(), tuple(array.shape), tuple(array.stride()), array.dtype, guard,
                       hash(np.ascontiguousarray(plan.tf.lut).tobytes())))
            fields.append(array)
        return tuple(fp), fields

    def get(self, key, objects, plans, domain, device):
        with self._lock:
            e = self._entries.get(key)
        if e is None or any(r() is not o for r, o in zip(e[3], objects)):
            return None
        fp, fields = self._fingerprint(plans, domain, device)
        if fp is None or fp != e[1]:
            return None
        return _abi.RenderArgs.from_buffer_copy(e[0]), list(e[2]) + fields

    def put(self, key, objects, plans, domain, device, args, keep):
        fp, _ = self._fingerprint(plans, domain, device)
        if fp is None:
            return
        try:
            refs = [weakref.ref(o) for o in objects]
        except TypeError:
            return
        luts = [t for t in keep if t.dtype == torch.float32 and tuple(t.shape) == (_abi.LUT_ENTRIES, 4)]
        with self._lock:
            if len(self._entries) >= self.capacity:
                self._entries.pop(next(iter(self._entries)))
            self._entries[key] = (bytes(args), fp, luts, refs)


_ARGS = _ArgsCache()
_LINE_CACHE: dict = {}
_LINE_LOCK = threading.Lock()


# Most slope changes classified analytically.  The launch block holds up to
# MAX_LUT_KINKS (7); measured on C4 / C2 (one B200), 4 kinks analytic 4.54 /
# 0.96 ms vs the shared-memory LUT 4.93 / 1.01, 6 kinks 4.95 / 1.09 -- no
# better than the LUT from 6 on.
ANALYTIC_MAX_KINKS = 5


def lut_analytic(lut: np.ndarray, max_kinks: int = ANALYTIC_MAX_KINKS, tol: float = 1e-12):
    """(base, slope, kinks) when the LUT lerp -- the piecewise-linear
    interpolant through (i, lut[i]), scene.py:139-152 -- changes slope at no
    more than ``max_kinks`` integer positions: then for x in [0, 255]
    lerp(x) = base + slope*x + sum_k dslope_k * max(x - x_k, 0) exactly
    (``kinks`` = [(x_k, dslope_k)]).  None otherwise (the kernel reads the LUT
    from shared memory).  A tf_from_points ramp with c control points has at
    most 2(c-2) kinks (one per interior point on an integer position, two
    when it falls between LUT samples).  Memoised on the LUT bytes (a
    transfer function changes only when steered)."""
    lut = np.asarray(lut, dtype=np.float64)
    key = (lut.tobytes(), max_kinks, tol)
    with _LINE_LOCK:
        if key in _LINE_CACHE:
            return _LINE_CACHE[key]
    res = _lut_analytic(lut, max_kinks, tol)
    with _LINE_LOCK:
        if len(_LINE_CACHE) > 256:
            _LINE_CACHE.clear()
        _LINE_CACHE[key] = res
    return res


def _lut_analytic(lut: np.ndarray, max_kinks: int, tol: float):
    seg = lut[1:] - lut[:-1]                       # slope of segment i = [i, i+1]
    change = np.abs(seg[1:] - seg[:-1]).max(axis=1) > tol
    at = np.nonzero(change)[0] + 1                 # segment i starts a new slope
    if at.size > max_kinks:
        return None
    base, slope = lut[0].copy(), seg[0].copy()
    kinks = [(float(i), seg[i] - seg[i - 1]) for i in at]
    x = np.arange(lut.shape[0], dtype=np.float64)[:, None]
    fit = base[None, :] + slope[None, :] * x
    for xk, d in kinks:
        fit = fit + d[None, :] * np.maximum(x - xk, 0.0)
    if np.abs(fit - lut).max() > 1e-9:
        return None
    return base, slope, kinks


def lut_line(lut: np.ndarray, tol: float = 1e-12):
    """(base, slope) if all 256 LUT entries lie on one straight run, else None."""
    res = lut_analytic(lut, 0, tol)
    return None if res is None else res[:2]


# analytic LUT forms instantiated per (element type, dim, early termination):
# LINE = 1 + kinks (march.cu launch_line); where up to 3 kinks are
# instantiated, 4..MAX_LUT_KINKS kinks take one variant with the count read
# at run time (LINE = MAX_LUT_KINKS + 1)
_LINE_MAX = {("float", 1, False): 4, ("float", 1, True): 4, ("float", 3, False): 2, ("float", 3, True): 2}
_LINE_RUNTIME = _abi.MAX_LUT_KINKS + 1


def _line_variant(kinks: int, elem: str, dim: int, et: bool) -> int:
    line = 1 + kinks
    top = _LINE_MAX.get((elem, dim, et), 1)
    if line <= top:
        return line
    return _LINE_RUNTIME if top >= 4 and line <= _LINE_RUNTIME else 0


def _aos3(arr) -> bool:
    """float3 field in the interleaved layout the AOS3 gather takes (march.cu aos3_layout)."""
    try:
        st = arr.stride()
        return (len(st) == 4 and st[3] == 1 and st[2] == 3 and st[1] % 2 == 0 and st[0] % 2 == 0
                and arr.data_ptr() % 8 == 0 and not os.environ.get("ISC_DISABLE_AOS3"))
    except (AttributeError, TypeError):
        return False


def _small_frame(image_size) -> bool:
    """march.cu small_frame: fewer 8x2 tiles than two per resident warp (4 CTAs
    of 8 warps per SM) -> 4 lanes per ray.  ISC_QUAD=0/1 forces it."""
    env = os.environ.get("ISC_QUAD")
    if env is not None:
        return env.strip() == "1"
    if image_size is None:
        return False
    import torch as _t
    w, h = image_size
    sms = _t.cuda.get_device_properties(_t.cuda.current_device()).multi_processor_count
    return ((w + 7) // 8) * ((h + 1) // 2) < 2 * sms * 4 * 8


def describe_kernel(plans: Sequence[SourcePlan], settings, analytic_lut: bool = True, image_size=None) -> str:
    """Name of the march kernel ``isc_render_local`` dispatches to for these
    plans (mirrors the library's dispatch; for reports and bench lines)."""
    import torch as _t
    interp = bool(settings.interpolation)
    et = settings.early_termination_alpha < 1.0
    if len(plans) == 1 and plans[0].mode != ISO_MODE:
        p = plans[0]
        dim = p.handle.descriptor.feature_dim
        arr, _ = p.handle.device_view(p.domain)
        dtype = getattr(arr, "dtype", None)
        f32 = dtype in (_t.float32, np.float32)
        guarded = interp and p.handle.descriptor.has_guard
        pw = lut_analytic(p.tf.lut) if analytic_lut else None
        if (dim == 1 and (f32 or guarded)) or (dim == 3 and f32 and guarded):
            elem = {_t.float32: "float", _t.float64: "double", _t.float16: "__half",
                    _t.bfloat16: "__nv_bfloat16"}.get(dtype, "float")
            line = 0
            if pw is not None and guarded:
                line = _line_variant(len(pw[2]), elem, dim, bool(et))
            aos3 = ",AOS3=1" if dim == 3 and _aos3(arr) else ""
            lanes = ",LANES=4" if (guarded and elem == "float" and dim == 1 and not et and line in (0, 1)
                                   and _small_frame(image_size)) else ""
            return (f"isc::march_fast_kernel<INTERP={int(interp)},GUARDED={int(guarded)},PAIRED=1,"
                    f"LINE={line},DIM={dim},ET={int(et)},T={elem}{aos3}{lanes}>")
    if (len(plans) == 2 and interp and not et and plans[0].mode == ISO_MODE and plans[1].mode != ISO_MODE
            and plans[0].handle.descriptor.feature_dim == 1 and plans[1].handle.descriptor.feature_dim in (1, 3)
            and all(p.handle.descriptor.has_guard for p in plans)
            and all(getattr(p.handle.device_view(p.domain)[0], "dtype", None) in (_t.float32, np.float32)
                    for p in plans)):
        # split render (march.cu launch_split): iso probe, then the volume pass
        pw = lut_analytic(plans[1].tf.lut) if analytic_lut else None
        dim = plans[1].handle.descriptor.feature_dim
        line = _line_variant(len(pw[2]), "float", dim, False) if pw is not None else 0
        chain = "1" if plans[0].chain.steps else "0"
        aos3 = ",AOS3=1" if dim == 3 and _aos3(plans[1].handle.device_view(plans[1].domain)[0]) else ""
        return (f"isc::iso_probe_kernel<CHAIN={chain}> (paired iso probe) + "
                f"isc::march_fast_kernel<INTERP=1,GUARDED=1,PAIRED=1,LINE={line},DIM={dim},ET=0,T=float{aos3}> "
                "(volume)")
    if 1 <= len(plans) <= 4:
        dims = [p.handle.descriptor.feature_dim for p in plans]
        if interp and all(p.handle.descriptor.has_guard for p in plans) and len(plans) <= 2 and \
                all(d in (1, 3) for d in dims):
            return f"isc::march_multi_fast_kernel<NS={len(plans)},DIMS={dims}>"
        return f"isc::march_multi_kernel<NS={len(plans)},INTERP={int(interp)}>"
    return f"isc::march_kernel<INTERP={int(interp)}>"


def render_local(rank_ctx, scene: SceneState, plans: Optional[Sequence[SourcePlan]] = None,
                 station_recorder: Optional[StationRecorder] = None, *, out: Optional[torch.Tensor] = None,
                 stream=None, check_errors: bool = True, keep_station_counts: bool = False,
                 keep_krange: bool = False, events=None, analytic_lut: bool = True) -> LocalImage:
    """Render the rank's brick into a partial image (raycast.py:492-541).

    ``out`` (optional) is a caller-owned CUDA float32 (H, W, 4) tensor to
    render into (e.g. an ``NvlinkTransport`` canvas, which saves the copy in
    ``binary_swap``).  ``check_errors=False`` skips the synchronising guard
    check; call ``LocalImage.check()`` later instead.  ``events`` = (start,
    end) CUDA events recorded around the kernel launch (bench timing).
    ``analytic_lut=False`` forces the shared-memory LUT lookup even for
    single-ramp transfer functions (see ``lut_line``).
    """
    device = require_cuda()
    domain, volume = rank_ctx.domain, rank_ctx.global_volume
    if plans is None:
        plans = build_plans(rank_ctx.registry, rank_ctx.functor_registry, rank_ctx.limits, scene)
    w, h = scene.camera.image_size
    keep: list = []
    objects = (scene, *plans, domain, volume)
    key = (tuple(id(o) for o in objects), analytic_lut, device.index)
    hit = _ARGS.get(key, objects, plans, domain, device)
    if hit is not None:
        args, kept = hit
        keep.extend(kept)
    else:
        args = pack_render_args(domain, volume, scene, plans, device, keep, analytic_lut)
        _ARGS.put(key, objects, plans, domain, device, args, keep)
    if out is None:
        out = torch.empty((h, w, 4), dtype=torch.float32, device=device)
    elif out.shape != (h, w, 4) or out.dtype != torch.float32 or not out.is_contiguous() or out.device != device:
        raise ValueError(f"out must be a contiguous float32 ({h}, {w}, 4) tensor on {device}")
    per_px = keep_station_counts or station_recorder is not None
    counts = torch.empty(h * w, dtype=torch.int32, device=device) if per_px else None
    kr = torch.empty((h * w, 4), dtype=torch.int32, device=device) if (keep_krange or station_recorder) else None
    stats = torch.empty(3, dtype=torch.int64, device=device)   # [stations, error word, tile counter]; zeroed by the library
    args.out_rgba = ptr(out)
    args.out_stations = ptr(counts) if counts is not None else None
    args.out_krange = ptr(kr) if kr is not None else None
    args.out_station_total = ptr(stats)
    args.error_word = ptr(stats) + 8
    args.work_counter = ptr(stats) + 16
    if events is not None:
        events[0].record(stream)
    _abi.check(_abi.lib().isc_render_local(C.byref(args), C.c_void_p(stream_handle(stream, device.index))),
               "render_local")
    if events is not None:
        events[1].record(stream)

    img = LocalImage(w, h, out)
    img._error_word = stats[1:2]
    img._stations = lambda: int(stats[0].item())
    taps = 8 if scene.settings.interpolation else 1
    for plan in plans:
        plan.handle.add_device_samples(stats[0], taps)
    img.station_counts = counts
    img.krange = kr
    if check_errors:
        img.check()
    if station_recorder is not None:
        _replay_stations(station_recorder, counts, kr)
    # tensors the launch reads (staged fields, LUTs) stay alive for the
    # allocator until this stream has passed the kernel
    if keep:
        run_stream = stream if stream is not None else torch.cuda.current_stream(device)
        for t in keep:
            t.record_stream(run_stream)
        keep.clear()
    return img


def ray_setup(rank_ctx, scene: SceneState, stream=None) -> dict:
    """Ray setup only (isc_ray_setup): per-pixel hit mask, brick interval and
    station ranges, for parity checks against the float64 reference."""
    device = require_cuda()
    w, h = scene.camera.image_size
    keep: list = []
    args = pack_render_args(rank_ctx.domain, rank_ctx.global_volume, scene, [], device, keep)
    hit = torch.empty(h * w, dtype=torch.uint8, device=device)
    tt = torch.empty((h * w, 2), dtype=torch.float64, device=device)
    kr = torch.empty((h * w, 4), dtype=torch.int32, device=device)
    args.out_hit, args.out_t, args.out_krange = ptr(hit), ptr(tt), ptr(kr)
    _abi.check(_abi.lib().isc_ray_setup(C.byref(args), C.c_void_p(stream_handle(stream))), "ray_setup")
    return {"hit": hit.bool(), "t_in": tt[:, 0], "t_out": tt[:, 1], "k_lo": kr[:, 0], "k_hi": kr[:, 1],
            "kg_lo": kr[:, 2], "kg_hi": kr[:, 3]}


def _replay_stations(recorder: StationRecorder, counts: torch.Tensor, kr: torch.Tensor) -> None:
    c = counts.cpu().numpy().astype(np.int64)
    lo = kr[:, 0].cpu().numpy().astype(np.int64)
    live = np.nonzero(c > 0)[0]
    if live.size == 0:
        return
    start = lo[live]
    stop = start + c[live]
    for k in range(int(start.min()), int(stop.max())):
        sel = live[(start <= k) & (k < stop)]
        if sel.size:
            recorder(k, sel)


class _RayListScene:
    """What pack_render_args reads from a scene, for ray-list launches: the
    camera supplies only the common origin (directions come from the list)."""

    def __init__(self, origin, n, settings):
        o = tuple(float(v) for v in origin)
        self.camera = Camera(o, (o[0], o[1], o[2] + 1.0), image_size=(max(int(n), 1), 1))
        self.settings = settings
        self.clip_planes = ()


class _WholeVolume:
    """Layout stand-in when the caller gives no GlobalVolume: the brick is the
    whole volume.  march_rays(volume=None) also sets ``no_layout`` so iso entry
    pairs are clamped into the guard reach (raycast.py:404-409)."""

    def __init__(self, domain):
        self.size = tuple(int(domain.offset[a]) + int(domain.size[a]) for a in range(3))
        self.decomposition = (1, 1, 1)


def march_rays(origin, dirs, local_interval, global_interval, plans: Sequence[SourcePlan], settings,
               station_recorder: Optional[StationRecorder] = None, volume=None):
    """March explicit rays on the device (raycast.py:291-381): every ray i
    marches the stations k in [ceil(max(t0_i,0)/step), ceil(max(t1_i,0)/step))
    from ``origin`` along ``dirs[i]`` (used as given).  Returns
    ((n, 4) float64 premultiplied RGBA, stations marched).  The same kernels
    as ``render_local`` run, in ray-list mode (isc_render_args.ray_dirs)."""
    device = require_cuda()
    d = np.asarray(dirs, dtype=np.float64).reshape(-1, 3)
    n = d.shape[0]
    if n == 0 or not plans:
        return np.zeros((n, 4)), 0
    t0 = np.asarray(local_interval[0], dtype=np.float64).reshape(-1)
    t1 = np.asarray(local_interval[1], dtype=np.float64).reshape(-1)
    g0 = np.asarray(global_interval[0], dtype=np.float64).reshape(-1)
    g1 = np.asarray(global_interval[1], dtype=np.float64).reshape(-1)
    domain = plans[0].domain
    vol = volume if volume is not None else _WholeVolume(domain)
    keep: list = []
    args = pack_render_args(domain, vol, _RayListScene(origin, n, settings), plans, device, keep)
    dirs_t = torch.from_numpy(np.ascontiguousarray(d)).to(device)
    iv_t = torch.from_numpy(np.ascontiguousarray(np.stack([t0, t1, g0, g1], axis=1))).to(device)
    out = torch.empty((1, n, 4), dtype=torch.float32, device=device)
    counts = torch.empty(n, dtype=torch.int32, device=device) if station_recorder is not None else None
    kr = torch.empty((n, 4), dtype=torch.int32, device=device) if station_recorder is not None else None
    stats = torch.zeros(3, dtype=torch.int64, device=device)
    args.ray_dirs, args.ray_intervals = ptr(dirs_t), ptr(iv_t)
    args.no_layout = 1 if volume is None else 0
    args.out_rgba = ptr(out)
    args.out_stations = ptr(counts) if counts is not None else None
    args.out_krange = ptr(kr) if kr is not None else None
    args.out_station_total = ptr(stats)
    args.error_word = ptr(stats) + 8
    args.work_counter = ptr(stats) + 16
    _abi.check(_abi.lib().isc_render_local(C.byref(args), C.c_void_p(stream_handle(None))), "march_rays")
    torch.cuda.current_stream().synchronize()
    if int(stats[1].item()):
        raise GuardContractError(f"{int(stats[1].item())} trilinear reads beyond the guard halo")
    if station_recorder is not None:
        _replay_stations(station_recorder, counts, kr)
    stations = int(stats[0].item())
    taps = 8 if settings.interpolation else 1
    for plan in plans:
        plan.handle.add_device_samples(stations, taps)
    return out.reshape(n, 4).double().cpu().numpy(), stations


def march_ray(origin, direction, interval, plans: Sequence[SourcePlan], settings, global_interval=None):
    """Single-ray convenience wrapper over :func:`march_rays` (raycast.py:471-489)."""
    gi = global_interval if global_interval is not None else interval
    rgba, _ = march_rays(origin, [direction], ([interval[0]], [interval[1]]), ([gi[0]], [gi[1]]), plans, settings)
    return rgba[0]


def gradient_normals(plan: SourcePlan, pos, view_dirs, interpolation: bool) -> np.ndarray:
    """Central-difference normals of the plan's chained scalar on the device
    (raycast.py:210-242, isc_gradient_normals); (n, 3) float64."""
    device = require_cuda()
    p = np.ascontiguousarray(np.asarray(pos, dtype=np.float64).reshape(-1, 3))
    v = np.ascontiguousarray(np.asarray(view_dirs, dtype=np.float64).reshape(-1, 3))
    n = p.shape[0]
    if n == 0:
        return np.zeros((0, 3))
    settings = RenderSettings(active_set=(plan.source_id,), interpolation=bool(interpolation))
    keep: list = []
    args = pack_render_args(plan.domain, _WholeVolume(plan.domain), _RayListScene((0.0, 0.0, 0.0), n, settings),
                            [plan], device, keep)
    p_t, v_t = torch.from_numpy(p).to(device), torch.from_numpy(v).to(device)
    out = torch.empty((n, 3), dtype=torch.float32, device=device)
    err = torch.zeros(1, dtype=torch.int32, device=device)
    args.error_word = ptr(err)
    _abi.check(_abi.lib().isc_gradient_normals(C.byref(args), C.c_void_p(ptr(p_t)), C.c_void_p(ptr(v_t)), n,
                                               C.c_void_p(ptr(out)), C.c_void_p(stream_handle(None))),
               "gradient_normals")
    torch.cuda.current_stream().synchronize()
    if int(err.item()):
        raise GuardContractError(f"{int(err.item())} trilinear reads beyond the guard halo")
    return out.double().cpu().numpy()


def gradient_normal(plan: SourcePlan, position, view_dir, interpolation: bool = True) -> np.ndarray:
    """Single-point wrapper over :func:`gradient_normals` (raycast.py:245-256)."""
    return gradient_normals(plan, [position], [view_dir], interpolation)[0]


def ray_box_intersection(origin, direction, box_lo, box_hi, clip_planes=()):
    """Host scalar utility (raycast.py:146-162): parametric interval of one ray
    in a cuboid after clipping, or None."""
    o = np.asarray(origin, dtype=np.float64)
    d = np.asarray(direction, dtype=np.float64)
    if not d.any():
        raise ValueError("ray direction must be non-zero")
    lo = np.asarray(box_lo, dtype=np.float64)
    hi = np.asarray(box_hi, dtype=np.float64)
    t0, t1 = -np.inf, np.inf
    for a in range(3):
        if d[a] == 0.0:
            if not lo[a] <= o[a] <= hi[a]:
                return None
            continue
        ta, tb = (lo[a] - o[a]) / d[a], (hi[a] - o[a]) / d[a]
        t0, t1 = max(t0, min(ta, tb)), min(t1, max(ta, tb))
    for plane in clip_planes:
        n = np.asarray(plane.normal)
        f0 = float(np.dot(o - np.asarray(plane.point), n))
        dn = float(d @ n)
        if dn > 0:
            t0 = max(t0, -f0 / dn)
        elif dn < 0:
            t1 = min(t1, -f0 / dn)
        elif f0 < 0:
            return None
    if t1 < t0:
        return None
    return (float(t0), float(t1))
