"""Parity at the benchmark's full sizes (C4: 1024^3 float32, 1920x1080).

* decomposition invariance -- the reference's central oracle
  (test_raycast.py:307-343): 8 bricks rendered from zero-copy strided views
  of ONE field tensor and composited in visibility order equal the
  single-brick render (<= 1e-4), and the station totals partition exactly;
* a seeded sample of full-length rays (every ~10k-th pixel) against the CPU
  oracle (float64 reference restatement) at <= 1e-3, plus bit-exact per-pixel
  station counts.
"""

import math

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

N = 1024
W, H = 1920, 1080


def _field():
    import torch
    import bench
    import paper_1611_09048_b200 as P
    dom = P.GlobalVolume((N, N, N)).local_domain(0, 1)
    return bench.make_field_torch(N, dom, torch.device("cuda"))


def _scene(P):
    diag = math.sqrt(3.0 * N * N)
    return P.SceneState(camera=P.Camera((N * 1.4, N * 1.15, -0.8 * diag), (N / 2.0,) * 3, image_size=(W, H)),
                        tf_points={0: [(0.0, 0.0, 0.0, 0.0, 0.0), (1.0, 1.0, 1.0, 1.0, 1.0)]},
                        value_ranges={0: (-0.4, 2.4)},
                        settings=P.RenderSettings(active_set=(0,), early_termination_alpha=1.0))


def _ctx(P, vol, rank, full):
    dom = vol.local_domain(rank, 1)
    (ox, oy, oz), (sx, sy, sz) = dom.offset, dom.size
    view = full[oz:oz + sz + 2, oy:oy + sy + 2, ox:ox + sx + 2]          # zero-copy brick + guard
    reg = P.SourceRegistry(dom)
    reg.register_handle(P.array_backed_handle(P.SourceDescriptor("f", 1, has_guard=True), view, 1))
    P.update_sources(reg, {0}, {})
    fr = P.default_registry()
    return P.RankContext(vol, dom, reg, fr, fr.limits)


def test_c4_decomposition_invariance_full_size():
    import paper_1611_09048_b200 as P
    full = _field()
    scene = _scene(P)
    one = P.render_local(_ctx(P, P.GlobalVolume((N, N, N)), 0, full), scene)
    vol8 = P.GlobalVolume((N, N, N), (2, 2, 2))
    imgs = [P.render_local(_ctx(P, vol8, r, full), scene) for r in range(8)]
    comp = P.composite_sequential([im.pixels for im in imgs], P.visibility_order(vol8, scene.camera))
    assert float((comp - one.pixels).abs().max()) <= 1e-4
    assert sum(im.stations for im in imgs) == one.stations == 781957855


def test_c4_sampled_rays_vs_oracle():
    import paper_1611_09048_b200 as P
    from oracle import isaac_oracle as O
    full = _field()
    scene = _scene(P)
    img = P.render_local(_ctx(P, P.GlobalVolume((N, N, N)), 0, full), scene, keep_station_counts=True)
    rng = np.random.default_rng(2024)
    covered = np.nonzero(img.station_counts.cpu().numpy() > 0)[0]
    pix = np.sort(np.concatenate([rng.choice(covered, 200, replace=False),
                                  rng.choice(W * H, 40, replace=False)]))
    cam = scene.camera
    dirs = O.primary_rays(cam.position, cam.look_at, cam.up, cam.vertical_fov, W, H)[pix]
    src = O.Source(array=full.cpu().numpy(), offset=(0, 0, 0), size=(N, N, N), guard=1,
                   lut=O.lut_from_points(scene.tf_points[0]), value_range=(-0.4, 2.4))
    ref = O.render_rays(cam.position, dirs, O.Brick((0, 0, 0), (N, N, N), 1, (N, N, N)), [src])
    got = img.pixels.reshape(-1, 4)[pix].cpu().numpy()
    assert np.abs(got - ref.rgba).max() <= 1e-3
    counts = img.station_counts.cpu().numpy()[pix]
    assert np.array_equal(counts.astype(np.int64), ref.stations)
    assert ref.stations.sum() > 200_000


def _c3_scene(P, n):
    diag = math.sqrt(3.0 * n * n)
    cool = [(0.0, 0.0, 0.0, 0.0, 0.0), (0.6, 0.1, 0.7, 0.4, 0.3), (1.0, 0.7, 1.0, 0.9, 0.8)]
    return P.SceneState(camera=P.Camera((n * 1.4, n * 1.15, -0.8 * diag), (n / 2.0,) * 3, image_size=(W, H)),
                        tf_points={0: [(0.0, 0.0, 0.0, 0.0, 0.0), (1.0, 1.0, 1.0, 1.0, 1.0)], 1: cool},
                        value_ranges={0: (-0.4, 2.4), 1: (0.0, 6.0)},
                        chain_texts={0: "", 1: "length | mul(2) | add(0.1)"},
                        settings=P.RenderSettings(active_set=(0, 1), modes={0: "iso"}, iso_thresholds={0: 1.0},
                                                  early_termination_alpha=1.0))


def test_c2_clip_plane_decomposition_and_oracle():
    import torch
    import bench
    import paper_1611_09048_b200 as P
    from oracle import isaac_oracle as O
    n = 512
    full = bench.make_field_torch(n, P.GlobalVolume((n, n, n)).local_domain(0, 1), torch.device("cuda"))
    scene = bench.build_scene(P, bench.CONFIGS["c2"])
    ctx1 = _ctx_n(P, P.GlobalVolume((n, n, n)), 0, full)
    one = P.render_local(ctx1, scene, keep_station_counts=True)
    vol2 = P.GlobalVolume((n, n, n), (2, 1, 1))
    imgs = [P.render_local(_ctx_n(P, vol2, r, full), scene) for r in range(2)]
    comp = P.composite_sequential([im.pixels for im in imgs], P.visibility_order(vol2, scene.camera))
    assert float((comp - one.pixels).abs().max()) <= 1e-4
    assert sum(im.stations for im in imgs) == one.stations
    rng = np.random.default_rng(7)
    covered = np.nonzero(one.station_counts.cpu().numpy() > 0)[0]
    pix = np.sort(rng.choice(covered, 200, replace=False))
    cam = scene.camera
    dirs = O.primary_rays(cam.position, cam.look_at, cam.up, cam.vertical_fov, W, H)[pix]
    src = O.Source(array=full.cpu().numpy(), offset=(0, 0, 0), size=(n, n, n), guard=1,
                   lut=O.lut_from_points(scene.tf_points[0]), value_range=(-0.4, 2.4))
    planes = [(p.point, p.normal) for p in scene.clip_planes]
    ref = O.render_rays(cam.position, dirs, O.Brick((0, 0, 0), (n, n, n), 1, (n, n, n)), [src], planes=planes)
    assert np.abs(one.pixels.reshape(-1, 4)[pix].cpu().numpy() - ref.rgba).max() <= 1e-3
    assert np.array_equal(one.station_counts.cpu().numpy()[pix].astype(np.int64), ref.stations)


def test_c3_multi_source_iso_vs_oracle():
    import torch
    import bench
    import paper_1611_09048_b200 as P
    from oracle import isaac_oracle as O
    n = 512
    dom = P.GlobalVolume((n, n, n)).local_domain(0, 1)
    scal = bench.make_field_torch(n, dom, torch.device("cuda"))
    vec = bench.make_vector_field_torch(n, dom, torch.device("cuda"))
    reg = P.SourceRegistry(dom)
    reg.register_handle(P.array_backed_handle(P.SourceDescriptor("s", 1, has_guard=True), scal, 1))
    reg.register_handle(P.array_backed_handle(P.SourceDescriptor("v", 3, has_guard=True), vec, 1))
    P.update_sources(reg, {0, 1}, {})
    fr = P.default_registry()
    ctx = P.RankContext(P.GlobalVolume((n, n, n)), dom, reg, fr, fr.limits)
    scene = _c3_scene(P, n)
    img = P.render_local(ctx, scene, keep_station_counts=True)
    rng = np.random.default_rng(8)
    covered = np.nonzero(img.station_counts.cpu().numpy() > 0)[0]
    pix = np.sort(rng.choice(covered, 120, replace=False))
    cam = scene.camera
    dirs = O.primary_rays(cam.position, cam.look_at, cam.up, cam.vertical_fov, W, H)[pix]
    srcs = [O.Source(array=scal.cpu().numpy(), offset=(0, 0, 0), size=(n, n, n), guard=1,
                     lut=O.lut_from_points(scene.tf_points[0]), value_range=(-0.4, 2.4), mode="iso",
                     iso_threshold=1.0),
            O.Source(array=vec.cpu().numpy(), offset=(0, 0, 0), size=(n, n, n), guard=1,
                     steps=O.parse_steps("length | mul(2) | add(0.1)", 3), lut=O.lut_from_points(scene.tf_points[1]),
                     value_range=(0.0, 6.0))]
    ref = O.render_rays(cam.position, dirs, O.Brick((0, 0, 0), (n, n, n), 1, (n, n, n)), srcs)
    got = img.pixels.reshape(-1, 4)[pix].cpu().numpy()
    err = np.abs(got - ref.rgba).max(axis=1)
    # iso decisions are float64-exact (isc_source.iso_exact): no flipped pixel
    assert (err > 1e-3).sum() == 0, err.max()
    assert (img.station_counts.cpu().numpy()[pix].astype(np.int64) != ref.stations).sum() == 0


def _ctx_n(P, vol, rank, full):
    return _ctx(P, vol, rank, full)
