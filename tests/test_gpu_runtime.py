"""GPU tests of the per-frame caller: device to_rgba8 / encode, FrameStreamer
overlap and frame_pipeline (runtime.py:45-388 restated)."""

import base64
import threading

import numpy as np
import pytest

from case_build import full_fields
from golden_io import cases, load

pytestmark = pytest.mark.gpu


def test_to_rgba8_bit_exact_vs_numpy():
    import torch
    from paper_1611_09048_b200.runtime import to_rgba8
    rng = np.random.default_rng(0)
    img = rng.uniform(-0.2, 1.2, (37, 53, 4)).astype(np.float32)
    img[0, :8, 0] = np.array([0.5, 1.5, 2.5, 127.5, 254.5, 0.49999997, 0.50000006, 1.0], np.float32) / 255.0
    want = (np.clip(img, 0.0, 1.0) * 255.0).round().astype(np.uint8)   # runtime.py:66-67 on the same f32
    got = to_rgba8(torch.from_numpy(img).cuda()).cpu().numpy()
    assert np.array_equal(got, want)


def test_encode_decode_round_trip():
    import torch
    from paper_1611_09048_b200.runtime import PNG, RAW_RGBA8, decode_frame, encode_frame, to_rgba8
    rng = np.random.default_rng(1)
    img = torch.from_numpy(rng.random((20, 30, 4), dtype=np.float32)).cuda()
    q = to_rgba8(img).cpu().numpy()
    for enc in (RAW_RGBA8, PNG):
        assert np.array_equal(decode_frame(encode_frame(img, enc), 30, 20, enc), q)
    assert base64.b64decode(encode_frame(img)) == q.tobytes()


def _pipeline_ctx(P, c, decomp, rank, transport, full, streamer=None):
    from product_build import product_ctx, product_scene
    from paper_1611_09048_b200.runtime import PipelineContext
    rc = product_ctx(c, decomp, rank, full)
    return PipelineContext(transport=transport, global_volume=rc.global_volume, domain=rc.domain,
                           registry=rc.registry, functor_registry=rc.functor_registry, limits=rc.limits,
                           scene=product_scene(c), streamer=streamer)


def test_frame_pipeline_single_rank_with_streamer():
    import paper_1611_09048_b200 as P
    from paper_1611_09048_b200.runtime import FrameStreamer, decode_frame, frame_pipeline, to_rgba8
    c = cases.case("multi")
    gold = load("render_multi.npz")
    full = full_fields(c)
    sent = []
    streamer = FrameStreamer(sent.append)
    ctx = _pipeline_ctx(P, c, (1, 1, 1), 0, P.LocalFabric(1).endpoint(0), full, streamer)
    results = [frame_pipeline(ctx, {"step": s}) for s in range(3)]
    streamer.wait_previous()
    assert [m["step"] for m in sent] == [0, 1, 2]
    frame = results[-1].image
    assert np.abs(frame.cpu().numpy() - gold["d111_composite"]).max() <= 1e-3
    w, h = c["camera"]["image_size"]
    msg = sent[-1]
    # the reference's frame message schema (runtime.py:222-235, harness FrameSink
    # reads message["image"][...], frontend FrameMessage protocol.ts:50-56)
    assert set(msg) == {"type", "step", "image", "metadata", "scene"} and msg["type"] == "frame"
    assert set(msg["image"]) == {"width", "height", "encoding", "data"}
    assert (msg["image"]["width"], msg["image"]["height"]) == (w, h) and msg["image"]["encoding"] == "raw-rgba8"
    assert P.SceneState.from_json(msg["scene"]).to_json() == ctx.scene.to_json()
    assert np.array_equal(decode_frame(msg["image"]["data"], w, h), to_rgba8(frame).cpu().numpy())
    ev = [e for e, _, _ in streamer.timeline]
    assert ev.count("send_end") == 3 and results[-1].stations > 0 and results[-1].render_seconds > 0


def test_frame_pipeline_two_ranks_byte_transport():
    """Two ranks (threads, LocalFabric bytes + GPU over) through frame_pipeline:
    rank 0's frame equals the reference's 2-brick composite."""
    import torch
    import paper_1611_09048_b200 as P
    from paper_1611_09048_b200.runtime import frame_pipeline
    c = cases.case("multi")
    gold = load("render_multi.npz")
    full = full_fields(c)
    fabric = P.LocalFabric(2)
    out = [None, None]
    errs = []

    def body(r):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                ctx = _pipeline_ctx(P, c, (2, 1, 1), r, fabric.endpoint(r), full)
                res = frame_pipeline(ctx, {"step": 7})
                out[r] = res
        except Exception as exc:  # noqa: BLE001
            errs.append(exc)

    ts = [threading.Thread(target=body, args=(r,)) for r in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(120)
    assert not errs, errs
    assert out[1].image is None and out[0].image is not None
    assert np.abs(out[0].image.cpu().numpy() - gold["d211_composite"]).max() <= 1e-3
    assert len(out[0].metadata["render_ms"]) == 2


def test_frame_graph_replay_matches_render():
    """A captured static-view frame replays bit-identically to render_local +
    binary_swap, and re-reads the field in place on every replay."""
    import numpy as np
    import torch
    import paper_1611_09048_b200 as P
    n = 24
    rng = np.random.default_rng(41)
    arr = torch.from_numpy(rng.random((n + 2,) * 3).astype(np.float32)).cuda()
    vol = P.GlobalVolume((n, n, n))
    dom = vol.local_domain(0, 1)
    reg = P.SourceRegistry(dom)
    reg.register_handle(P.array_backed_handle(P.SourceDescriptor("f", 1, has_guard=True), arr, 1))
    P.update_sources(reg, {0}, {})
    fr = P.default_registry()
    ctx = P.RankContext(vol, dom, reg, fr, fr.limits, P.LocalFabric(1).endpoint(0))
    scene = P.SceneState(camera=P.Camera((60.0, 41.0, -30.0), (12.0, 12.0, 12.0), image_size=(64, 40)),
                         tf_points={0: [(0.0, 0.0, 0.0, 0.0, 0.0), (1.0, 1.0, 0.5, 0.2, 0.6)]},
                         settings=P.RenderSettings(active_set=(0,), early_termination_alpha=1.0))
    g = P.FrameGraph(ctx, scene)
    want = P.render_local(ctx, scene).pixels.cpu().numpy()
    got = g.replay().cpu().numpy()
    assert np.array_equal(got, want)
    arr.mul_(0.5)                                   # the simulation advanced: replay sees the new values
    want2 = P.render_local(ctx, scene).pixels.cpu().numpy()
    got2 = g.replay().cpu().numpy()
    assert np.array_equal(got2, want2) and not np.array_equal(got2, got)


def test_bench_json_line_contract():
    """bench.py prints ONE JSON line with the driver's contract keys
    (metric / value / unit / n_gpus / steps / warmup / ms_per_step /
    higher_is_better / scaling / vs_baseline / dtype / data / config.workload,
    roofline, e2e with copy byte counts, gpu_launches, clocks)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--config", "c1", "--steps", "3",
                          "--warmup", "3", "--no-cpu-baseline", "--no-host-field-e2e"],
                         capture_output=True, text=True, timeout=300, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, lines
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["value"] > 0 and "workload" in d["config"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] and r["peak"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= 3
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
