"""Per-frame pipeline around the hot path (the caller of render_local /
binary_swap): scene broadcast -> update_sources ->
render -> visibility order -> binary swap -> metadata merge -> background
encode/send on rank 0.

Mirrors ``insitu.runtime`` (runtime.py:36-388), including the root's
steering fold (``apply_steering`` over the context's inbox; the gateway and
websocket that fill the inbox are out of scope).  The B200 differences: the frame stays on the device until
``to_rgba8`` quantises it there (``isc_to_rgba8``), so 8.3 MB instead of 33 MB
per 1080p frame crosses PCIe, and that copy runs on a side stream while the
next frame renders (FrameStreamer overlap, runtime.py:187-249).
"""

from __future__ import annotations

import base64
import concurrent.futures
import ctypes as C
import dataclasses
import io
import json
import logging
import queue
import time
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from . import _abi
from .compositing import binary_swap, visibility_order
from .errors import ChainError
from .fields import update_sources
from .functors import parse_chain
from .scene import Camera, SceneState, clip_plane

log = logging.getLogger(__name__)
_log = log

RAW_RGBA8 = "raw-rgba8"
PNG = "png"

__all__ = ["RAW_RGBA8", "PNG", "CONTROL_ACTIONS", "SteeringResult", "apply_steering", "FrameAborted", "to_rgba8", "encode_frame", "decode_frame", "merge_metadata",
           "FrameStreamer", "FrameResult", "PipelineContext", "broadcast_scene", "frame_pipeline"]


class FrameAborted(Exception):
    def __init__(self, reason: str, controls: Optional[list] = None):
        super().__init__(reason)
        self.controls = controls or []


def to_rgba8(image, stream=None):
    """round(clip(rgba, 0, 1) * 255) as uint8 (runtime.py:66-67), on the device.
    Accepts a CUDA float32 (H, W, 4) tensor (or anything torch.as_tensor takes)."""
    import torch
    from .device import require_cuda, stream_handle
    dev = require_cuda()
    t = torch.as_tensor(image)
    t = t.to(device=dev, dtype=torch.float32).contiguous()
    if t.shape[-1] != 4:
        raise ValueError(f"expected (..., 4) RGBA, got {tuple(t.shape)}")
    out = torch.empty(t.shape, dtype=torch.uint8, device=dev)
    _abi.check(_abi.lib().isc_to_rgba8(C.c_void_p(t.data_ptr()), C.c_void_p(out.data_ptr()), t.numel() // 4,
                                       C.c_void_p(stream_handle(stream))), "to_rgba8")
    return out


def _png_bytes(rgba8: np.ndarray) -> bytes:
    from PIL import Image
    out = io.BytesIO()
    Image.fromarray(rgba8, mode="RGBA").save(out, format="PNG")
    return out.getvalue()


def _png_array(blob: bytes, width: int, height: int) -> np.ndarray:
    from PIL import Image
    return np.asarray(Image.open(io.BytesIO(blob)).convert("RGBA"))


# frame codecs of the reference's wire format (runtime.py:45-81): uint8
# (H, W, 4) frame <-> payload bytes; base64 on top for the message
_CODECS = {
    RAW_RGBA8: (lambda a: a.tobytes(),
                lambda blob, w, h: np.frombuffer(blob, dtype=np.uint8).reshape(h, w, 4)),
    PNG: (_png_bytes, _png_array),
}


def _codec(encoding: str):
    try:
        return _CODECS[encoding]
    except KeyError:
        raise ValueError(f"unknown frame encoding {encoding!r}") from None


def _encode_bytes(data: np.ndarray, encoding: str) -> str:
    return base64.b64encode(_codec(encoding)[0](data)).decode("ascii")


def encode_frame(image, encoding: str = RAW_RGBA8, quality: Optional[int] = None) -> str:
    """Quantise on the device, then base64 (raw) or PNG+base64 on the host (runtime.py:45-63)."""
    return _encode_bytes(to_rgba8(image).cpu().numpy(), encoding)


def decode_frame(data: str, width: int, height: int, encoding: str = RAW_RGBA8) -> np.ndarray:
    """Inverse of encode_frame (runtime.py:70-78)."""
    unpack = _codec(encoding)[1]
    return unpack(base64.b64decode(data), width, height)


def merge_metadata(per_rank_docs: Sequence[dict]) -> dict:
    """Rank-ordered merge; all-list keys concatenate, others keep the first (runtime.py:81-100)."""
    seen: dict = {}
    for doc in per_rank_docs:
        for k, v in (doc or {}).items():
            seen.setdefault(k, []).append(v)
    return {k: ([x for v in vs for x in v] if len(vs) > 1 and all(isinstance(v, list) for v in vs) else vs[0])
            for k, vs in seen.items()}


class FrameStreamer:
    """Root-side background encode + send, one frame in flight (runtime.py:187-249).

    ``submit`` quantises the frame on the device (``to_rgba8``), starts its
    D2H on a side stream and returns; a worker thread waits for the copy,
    encodes and calls ``sink(message)`` with the reference's message schema
    (``type``, ``step``, ``image: {width, height, encoding, data}``,
    ``metadata``, ``scene``: the scene echo, runtime.py:222-235).
    ``wait_previous`` is the single per-frame rendezvous; submitting while a
    frame is in flight raises, as in the reference.  ``encoder(data,
    encoding, quality)`` receives the already-quantised uint8 (H, W, 4)
    frame (the 8-bit quantisation runs on the GPU).
    """

    def __init__(self, sink: Callable[[dict], None],
                 encoder: Optional[Callable[[np.ndarray, str, Optional[int]], str]] = None,
                 encoding: str = RAW_RGBA8, quality: Optional[int] = None):
        import torch
        self.sink = sink
        self.encoder = encoder or (lambda data, enc, _q: _encode_bytes(data, enc))
        self.encoding = encoding
        self.quality = quality
        self.timeline: list = []
        # one background worker, at most one frame in flight: the future of
        # the frame being sent (its exception re-raised at the rendezvous)
        self._worker = concurrent.futures.ThreadPoolExecutor(max_workers=1, thread_name_prefix="frame-send")
        self._inflight: Optional[concurrent.futures.Future] = None
        self._stream = torch.cuda.Stream()
        self._host = None

    def mark(self, event: str, step: int) -> None:
        self.timeline.append((event, step, time.monotonic()))

    def wait_previous(self) -> None:
        job, self._inflight = self._inflight, None
        if job is not None:
            job.result()

    def submit(self, frame, step: int, metadata: dict, scene: SceneState) -> None:
        import torch
        if self._inflight is not None:
            raise RuntimeError("previous frame still in flight; wait_previous() first")
        q = to_rgba8(frame)
        ready = torch.cuda.Event()
        ready.record()
        if self._host is None or self._host.shape != q.shape:
            self._host = torch.empty(q.shape, dtype=torch.uint8).pin_memory()
        host = self._host
        self._stream.wait_event(ready)
        with torch.cuda.stream(self._stream):
            host.copy_(q, non_blocking=True)
            q.record_stream(self._stream)
        copied = torch.cuda.Event()
        copied.record(self._stream)
        message = {"type": "frame", "step": step,
                   "image": {"width": int(q.shape[1]), "height": int(q.shape[0]), "encoding": self.encoding},
                   "metadata": metadata, "scene": scene.to_json()}
        self._inflight = self._worker.submit(self._send, message, host, copied, step)

    def _send(self, message: dict, host, copied, step: int) -> None:
        self.mark("send_begin", step)
        try:
            copied.synchronize()            # the frame's D2H landed in pinned memory
            message["image"]["data"] = self.encoder(host.numpy(), self.encoding, self.quality)
            self.sink(message)
        finally:
            self.mark("send_end", step)

    def close(self) -> None:
        job, self._inflight = self._inflight, None
        if job is not None:
            concurrent.futures.wait([job])
        self._worker.shutdown(wait=True)


CONTROL_ACTIONS = ("pause", "resume", "step", "exit")


@dataclass
class SteeringResult:
    scene: SceneState
    controls: list
    dropped: int = 0
    unknown: int = 0


def _steer_camera(scene, m):
    cam = scene.camera
    return scene.bump(camera=Camera(position=tuple(m.get("position", cam.position)),
                                    look_at=tuple(m.get("look_at", cam.look_at)), up=tuple(m.get("up", cam.up)),
                                    vertical_fov=float(m.get("vertical_fov", cam.vertical_fov)),
                                    image_size=cam.image_size))


def _steer_keyed(field: str, key: str, value):
    """Fold for the per-source dict fields of the scene (chain texts,
    transfer-function points, value ranges): copy, set one entry, bump."""
    def fold(scene, m):
        table = dict(getattr(scene, field))
        table[int(m[key])] = value(m)
        return scene.bump(**{field: table})
    return fold


# one fold per steering action (runtime.py:129-178): scene -> new scene
_STEER = {
    "set_period": lambda sc, m: sc.bump(render_period=max(1, int(m["value"]))),
    "set_active_sources": lambda sc, m: sc.bump(settings=dataclasses.replace(
        sc.settings, active_set=tuple(sorted(int(i) for i in m["ids"])))),
    "set_functor_chain": _steer_keyed("chain_texts", "source_id", lambda m: str(m["text"])),
    "set_transfer_function": _steer_keyed("tf_points", "source_id",
                                          lambda m: [tuple(float(v) for v in p) for p in m["points"]]),
    "set_range": _steer_keyed("value_ranges", "source_id", lambda m: (float(m["min"]), float(m["max"]))),
    "set_camera": _steer_camera,
    "set_clip_planes": lambda sc, m: sc.bump(clip_planes=tuple(clip_plane(p["point"], p["normal"])
                                                               for p in m.get("planes", []))),
    "set_interpolation": lambda sc, m: sc.bump(settings=dataclasses.replace(sc.settings,
                                                                            interpolation=bool(m["value"]))),
}


def apply_steering(scene: SceneState, messages: Sequence[object]) -> SteeringResult:
    """Fold steering messages into the scene in arrival order, last writer
    wins per field (runtime.py:111-184).  pause / resume / step / exit are
    returned as control events; malformed messages (bad JSON, not an object,
    missing or mistyped fields) are dropped and counted; unknown actions are
    counted and ignored.  The scene lives on the host; what it drives on the
    device (LUTs, the packed launch block) is re-uploaded only for what a
    message changed (device.LutCache is keyed by LUT content)."""
    controls: list = []
    dropped = unknown = 0
    for raw in messages:
        msg = raw
        if isinstance(raw, (str, bytes)):
            try:
                msg = json.loads(raw)
            except (ValueError, UnicodeDecodeError):
                dropped += 1
                continue
        if not isinstance(msg, dict):
            dropped += 1
            continue
        action = msg.get("action")
        if action in CONTROL_ACTIONS:
            controls.append(msg)
            continue
        fold = _STEER.get(action)
        if fold is None:
            unknown += 1
            _log.warning("ignoring steering message with unknown action %r", action)
            continue
        try:
            scene = fold(scene, msg)
        except (KeyError, TypeError, ValueError) as exc:
            dropped += 1
            _log.warning("dropping malformed steering message %r: %s", msg, exc)
    return SteeringResult(scene, controls, dropped, unknown)


@dataclass
class FrameResult:
    step: int
    image: object
    metadata: dict
    controls: list
    render_seconds: float
    composite_seconds: float
    stations: int
    aborted: bool = False


@dataclass
class PipelineContext:
    """What one rank carries across frames (runtime.py:262-281).  Root only:
    ``inbox`` receives raw steering messages (folded by apply_steering at the
    start of each frame), ``error_sink`` gets the abort notice of a frame
    whose chain no longer parses; ``steer`` is an optional extra hook
    scene -> (scene, controls) run after the inbox fold."""

    transport: object
    global_volume: object
    domain: object
    registry: object
    functor_registry: object
    limits: object
    scene: SceneState
    streamer: Optional[FrameStreamer] = None
    metadata_hook: Optional[Callable[[int], dict]] = None
    steer: Optional[Callable[[SceneState], tuple]] = None    # root: scene -> (scene, controls)
    canvas: object = None
    inbox: "queue.Queue" = dataclasses.field(default_factory=queue.Queue)
    error_sink: Optional[Callable[[dict], None]] = None
    steering_dropped: int = 0
    steering_unknown: int = 0

    def drain_inbox(self) -> list:
        """Every steering message queued so far (non-blocking; later arrivals
        wait for the next frame)."""
        got = []
        for _ in range(self.inbox.qsize()):
            try:
                got.append(self.inbox.get_nowait())
            except queue.Empty:
                break
        return got

    @property
    def rank(self) -> int:
        return self.transport.rank

    @property
    def is_root(self) -> bool:
        return self.transport.rank == 0


def broadcast_scene(ctx: PipelineContext, scene: Optional[SceneState] = None, controls: Sequence = ()):
    """Root's scene (+ controls) to every rank as JSON bytes; a chain that no
    longer parses aborts the frame everywhere and keeps the previous scene
    (runtime.py:305-333)."""
    if ctx.is_root:
        env: dict = {"controls": list(controls)}
        try:
            for sid in scene.settings.active_set:
                parse_chain(scene.chain_text(sid), ctx.functor_registry, ctx.limits,
                            ctx.registry.descriptor(sid).feature_dim)
            env["scene"] = scene.to_json()
        except ChainError as exc:
            env["abort"] = str(exc)
            env["scene"] = ctx.scene.to_json()
        payload = json.dumps(env, sort_keys=True).encode("utf-8")
        ctx.transport.broadcast_from_root(payload)
    else:
        env = json.loads(ctx.transport.broadcast_from_root(None).decode("utf-8"))
    ctx.scene = SceneState.from_json(env["scene"])
    if "abort" in env:
        if ctx.is_root and getattr(ctx, "error_sink", None) is not None:
            ctx.error_sink({"type": "error", "error": env["abort"]})
        raise FrameAborted(env["abort"], list(env.get("controls", ())))
    return ctx.scene, list(env.get("controls", ()))


def frame_pipeline(ctx: PipelineContext, frame_payload: dict) -> Optional[FrameResult]:
    """One frame on this rank (runtime.py:336-388).  Rank 0 hands the frame to
    the streamer and returns while it is encoded/sent in the background."""
    import torch
    from .raycast import render_local
    step = int(frame_payload.get("step", 0))
    scene, controls = ctx.scene, []
    if ctx.is_root:
        if ctx.streamer is not None:
            ctx.streamer.wait_previous()
        steering = apply_steering(ctx.scene, ctx.drain_inbox())
        ctx.steering_dropped += steering.dropped
        ctx.steering_unknown += steering.unknown
        scene, controls = steering.scene, list(steering.controls)
        if ctx.steer is not None:
            scene, more = ctx.steer(scene)
            controls += list(more)
    try:
        scene, controls = broadcast_scene(ctx, scene, controls)
    except FrameAborted as abort:
        return FrameResult(step, None, {}, abort.controls, 0.0, 0.0, 0, aborted=True)
    update_sources(ctx.registry, scene.settings.active_set, frame_payload)
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    if ctx.is_root and ctx.streamer is not None:
        ctx.streamer.mark("render_begin", step)
    e0.record()
    out = ctx.canvas if ctx.canvas is not None and tuple(ctx.canvas.shape[:2]) == scene.camera.image_size[::-1] \
        else None
    image = render_local(ctx, scene, out=out)
    e1.record()
    order = visibility_order(ctx.global_volume, scene.camera)
    image.order_key = order.index(ctx.rank)
    full = binary_swap(ctx.transport, image.pixels, order)
    e2.record()
    e2.synchronize()
    render_s, comp_s = e0.elapsed_time(e1) / 1e3, e1.elapsed_time(e2) / 1e3
    doc = dict(ctx.metadata_hook(step) if ctx.metadata_hook is not None else {})
    doc.setdefault("render_ms", [render_s * 1000.0])
    gathered = ctx.transport.gather_to_root(json.dumps(doc).encode("utf-8"))
    metadata: dict = {}
    if ctx.is_root:
        metadata = merge_metadata([json.loads(d.decode("utf-8")) for d in gathered])
        if ctx.streamer is not None:
            ctx.streamer.submit(full, step, metadata, scene)
    return FrameResult(step, full if ctx.is_root else None, metadata, controls, render_s, comp_s, image.stations)


class FrameGraph:
    """A static view's frame (``render_local`` + ``binary_swap``) captured once
    as a CUDA graph and replayed per frame -- no host preparation, one graph
    launch per rank.  One rank (``LocalFabric`` of size 1 / no transport), or
    every rank of an ``NvlinkTransport``: the peer-memory swap keeps its
    epoch on the device (``isc_swap_epoch_bump``), so the captured swap
    replays; construction and every ``replay()`` are then collective (all
    ranks, same count, as ``binary_swap``).  Byte transports are not
    replayable.

    The fields are read in place at replay time (zero-copy, as every render);
    the scene, plans, transfer functions and the brick's device arrays must
    stay the ones captured.  ``replay()`` returns the frame tensor (rank 0;
    ``None`` on other ranks of a swap), which the next replay overwrites.
    ``check()`` raises the last replay's guard-contract error and any swap
    spin-wait timeout since the previous check.
    """

    def __init__(self, rank_ctx, scene: SceneState, warmup: int = 4):
        import torch
        from .raycast import build_plans, render_local
        from .transport import NvlinkTransport
        tr = rank_ctx.transport
        multi = tr is not None and getattr(tr, "size", 1) != 1
        if multi and not isinstance(tr, NvlinkTransport):
            raise ValueError("FrameGraph replays a multi-rank frame only over an NvlinkTransport "
                             "(byte transports run on the host)")
        self._tr = tr if multi else None
        self.plans = build_plans(rank_ctx.registry, rank_ctx.functor_registry, rank_ctx.limits, scene)
        w, h = scene.camera.image_size
        dev = torch.device("cuda", torch.cuda.current_device())
        self.canvas = tr.canvas(h, w) if multi else torch.empty((h, w, 4), dtype=torch.float32, device=dev)
        order = visibility_order(rank_ctx.global_volume, scene.camera)
        self._stream = torch.cuda.Stream()

        def frame():
            img = render_local(rank_ctx, scene, plans=self.plans, out=self.canvas, check_errors=False)
            self._last = img
            return binary_swap(tr, img.pixels, order) if tr is not None else img.pixels.clone()

        # warm-up on the capture stream: LUT uploads, launch block, launch-shape choice
        with torch.cuda.stream(self._stream):
            for _ in range(warmup):
                frame()
                self._stream.synchronize()
        self._last.check()
        if multi:
            tr.flush()
            tr.capturing = True
        try:
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph, stream=self._stream):
                self.frame = frame()
        finally:
            if multi:
                tr.capturing = False

    def replay(self):
        self.graph.replay()
        if self._tr is not None:
            self._tr.epoch += 1     # the replayed swap bumped the device epoch
        return self.frame

    def check(self) -> None:
        """Synchronise and raise GuardContractError / TransportError if a
        replay hit one (the errors of all replays since the last check)."""
        from .device import stream_handle
        self._last.check()          # replays run on the current stream; this reads after them
        if self._tr is not None:
            self._tr.status(stream_handle())
