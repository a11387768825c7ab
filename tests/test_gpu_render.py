"""GPU parity: the sm_100a render path against the reference goldens and the oracle.

Tolerances (north star): float RGBA max-abs <= 1e-3 before 8-bit
quantisation; hit masks, station ranges and per-pixel station counts
bit-exact.  Colours are float32 on the device vs float64 in the reference.
"""

import numpy as np
import pytest

from case_build import full_fields, oracle_render
from golden_io import cases, decomp_key, load

pytestmark = pytest.mark.gpu

RGBA_TOL = 1e-3


def _torch():
    import torch
    return torch


@pytest.mark.parametrize("name", sorted(cases.RENDER_CASES))
def test_render_matches_reference_goldens(name):
    import paper_1611_09048_b200 as P
    from product_build import product_ctx, product_scene
    c = cases.case(name)
    gold = load(f"render_{name}.npz")
    scene = product_scene(c)
    full = full_fields(c)
    for decomp in c["decompositions"]:
        key = decomp_key(decomp)
        images = []
        for rank in range(int(np.prod(decomp))):
            p = f"{key}_r{rank}_"
            ctx = product_ctx(c, decomp, rank, full)
            rs = P.raycast.ray_setup(ctx, scene)
            assert np.array_equal(rs["hit"].cpu().numpy(), gold[p + "hit"]), (name, key, rank)
            hit = gold[p + "hit"]
            for k in ("k_lo", "k_hi", "kg_lo", "kg_hi"):
                got = rs[k].cpu().numpy()
                assert np.array_equal(got[hit], gold[p + k][hit]), (name, key, rank, k)
            tin = rs["t_in"].cpu().numpy()
            fin = np.isfinite(gold[p + "t_in"])
            np.testing.assert_allclose(tin[fin], gold[p + "t_in"][fin], rtol=4e-16, atol=0)
            img = P.render_local(ctx, scene, keep_station_counts=True)
            rgba = img.pixels.cpu().numpy().astype(np.float64)
            err = np.abs(rgba - gold[p + "rgba"]).max()
            assert err <= RGBA_TOL, (name, key, rank, err)
            counts = img.station_counts.cpu().numpy().astype(np.int64)
            want = gold[p + "stations"].astype(np.int64)
            # bit-exact on every pixel, iso and early-termination cases included
            assert np.array_equal(counts, want), (name, key, rank, int((counts != want).sum()))
            assert img.stations == int(counts.sum())
            images.append(img.pixels)
        order = P.visibility_order(P.GlobalVolume(tuple(c["size"]), tuple(decomp)), scene.camera)
        assert order == [int(v) for v in gold[key + "_order"]]
        comp = P.composite_sequential(images, order).cpu().numpy()
        assert np.abs(comp - gold[key + "_composite"]).max() <= RGBA_TOL


def test_render_matches_oracle_random_cameras():
    """Seeded random cameras / TFs on a random field, CUDA vs the oracle."""
    import paper_1611_09048_b200 as P
    from oracle import isaac_oracle as O
    torch = _torch()
    rng = np.random.default_rng(1234)
    n = 24
    field = rng.random((n + 2, n + 2, n + 2), dtype=np.float32)
    for trial in range(6):
        pos = tuple(float(v) for v in rng.uniform(-2 * n, 3 * n, 3))
        target = tuple(float(v) for v in rng.uniform(0.3 * n, 0.7 * n, 3))
        w, h = int(rng.integers(17, 70)), int(rng.integers(9, 50))
        step = float(rng.uniform(0.2, 1.3))
        interp = bool(trial % 3 != 2)
        pts = [(0.0, *rng.random(4)), (float(rng.uniform(0.2, 0.8)), *rng.random(4)), (1.0, *rng.random(4))]
        vol = P.GlobalVolume((n, n, n), (1, 1, 1))
        dom = vol.local_domain(0, 1)
        reg = P.SourceRegistry(dom)
        reg.register_handle(P.array_backed_handle(P.SourceDescriptor("f", 1, has_guard=True),
                                                  torch.from_numpy(field).cuda(), 1))
        P.update_sources(reg, {0}, {})
        fr = P.default_registry()
        ctx = P.RankContext(vol, dom, reg, fr, fr.limits)
        scene = P.SceneState(camera=P.Camera(pos, target, image_size=(w, h)), tf_points={0: pts},
                             value_ranges={0: (0.1, 0.9)},
                             settings=P.RenderSettings(active_set=(0,), interpolation=interp, step_length=step,
                                                       early_termination_alpha=1.0))
        got = P.render_local(ctx, scene).pixels.cpu().numpy()
        src = O.Source(array=field, offset=(0, 0, 0), size=(n, n, n), guard=1, lut=O.lut_from_points(pts),
                       value_range=(0.1, 0.9))
        ref = O.render_brick({"position": pos, "look_at": target, "width": w, "height": h},
                             O.Brick((0, 0, 0), (n, n, n), 1, (n, n, n)), [src], step=step, interp=interp)
        assert np.abs(got - ref.rgba).max() <= RGBA_TOL, trial


def test_station_recorder_replay_matches_oracle():
    import paper_1611_09048_b200 as P
    from product_build import product_ctx, product_scene
    c = cases.case("random_bricks")
    gold = load("render_random_bricks.npz")
    scene = product_scene(c)
    full = full_fields(c)
    for rank in range(8):
        want: dict = {}
        oracle_render(c, gold, (2, 2, 2), rank, recorder=lambda k, ids: [want.setdefault(int(i), []).append(k)
                                                                        for i in ids])
        got: dict = {}
        ctx = product_ctx(c, (2, 2, 2), rank, full)
        P.render_local(ctx, scene, station_recorder=lambda k, ids: [got.setdefault(int(i), []).append(k)
                                                                   for i in ids])
        assert got == want


def test_inactive_sources_never_touched():
    import paper_1611_09048_b200 as P
    from product_build import product_ctx, product_scene
    c = cases.case("multi")
    scene = product_scene(c)
    full = full_fields(c)
    for rank in range(2):
        ctx = product_ctx(c, (2, 1, 1), rank, full)
        P.render_local(ctx, scene)
        assert ctx.registry.handle(0).sample_count > 0
        assert ctx.registry.handle(1).sample_count > 0
        assert ctx.registry.handle(2).sample_count == 0


def test_sample_count_over_many_renders():
    """sample_count over a long render loop (device counters folded on the
    device every 64 renders, no host sync) = renders x stations x 8 taps."""
    import paper_1611_09048_b200 as P
    from product_build import product_ctx, product_scene
    c = cases.case("c1")
    scene = product_scene(c)
    ctx = product_ctx(c, (1, 1, 1), 0)
    h = ctx.registry.handle(0)
    h.sample_count = 0
    first = P.render_local(ctx, scene, check_errors=False)
    for _ in range(149):
        P.render_local(ctx, scene, check_errors=False)
    assert h.sample_count == 150 * first.stations * 8
    P.render_local(ctx, scene, check_errors=False)
    assert h.sample_count == 151 * first.stations * 8


def test_offscreen_is_transparent_and_energy_bound():
    import paper_1611_09048_b200 as P
    from product_build import product_ctx, product_scene
    c = cases.case("c1")
    ctx = product_ctx(c, (1, 1, 1), 0)
    scene = product_scene(c)
    away = P.SceneState(camera=P.Camera((32, 32, -100), (32, 32, -200), image_size=(40, 30)),
                        tf_points=scene.tf_points, value_ranges=scene.value_ranges, settings=scene.settings)
    assert float(P.render_local(ctx, away).pixels.abs().sum()) == 0.0
    px = P.render_local(ctx, scene).pixels
    assert bool((px[..., :3] <= px[..., 3:] + 1e-6).all())
    assert float(px[..., 3].max()) <= 1.0 + 1e-6 and float(px[..., 3].min()) >= 0.0


def test_guard_contract_violation_raises():
    import paper_1611_09048_b200 as P
    torch = _torch()
    n = 8
    vol = P.GlobalVolume((n, n, n))
    dom = vol.local_domain(0, 0)          # the domain promises no halo ...
    reg = P.SourceRegistry(dom)
    arr = torch.rand((n, n, n), device="cuda")
    reg.register_handle(P.array_backed_handle(P.SourceDescriptor("f", 1, has_guard=True), arr, 0))
    P.update_sources(reg, {0}, {})
    fr = P.default_registry()
    ctx = P.RankContext(vol, dom, reg, fr, fr.limits)
    scene = P.SceneState(camera=P.Camera((20.0, 17.0, -9.0), (4.0, 4.0, 4.0), image_size=(32, 24)),
                         settings=P.RenderSettings(active_set=(0,), early_termination_alpha=1.0))
    with pytest.raises(P.GuardContractError):   # ... but trilinear needs i0 + 1 == size
        P.render_local(ctx, scene)


@pytest.mark.parametrize("with_vector", [False, True])
def test_guard_tail_reached_only_if_marched(with_vector):
    """Guard contract on a brick whose far cells lack the halo (guard 0): rays
    that stop at an iso surface before the far face gather no bad corner and
    must not raise (the reference raises only on a gather it performs,
    fields.py:230-238); the same rays in volume mode reach the far face and
    must raise.  Covers the per-ray end-station proof of the specialised
    kernels (march_multi.cu / march.cu)."""
    import math
    import paper_1611_09048_b200 as P
    from oracle import isaac_oracle as O
    torch = _torch()
    n = 8
    z, y, x = np.meshgrid(*(np.arange(n, dtype=np.float64),) * 3, indexing="ij")
    scal = x.astype(np.float32)                        # iso at x = 2.5, reached from the x = 0 face
    vec = np.stack([x, y, z], axis=-1).astype(np.float32) * 0.1
    vol = P.GlobalVolume((n, n, n))
    dom = vol.local_domain(0, 0)
    cam = dict(position=(-50.0, 3.7, 3.3), look_at=(4.0, 3.7, 3.3), vertical_fov=math.radians(5.0),
               width=16, height=12)
    pts = [(0.0, 0.0, 0.0, 0.0, 0.0), (1.0, 1.0, 0.5, 0.2, 0.6)]

    def render(mode):
        reg = P.SourceRegistry(dom)
        reg.register_handle(P.array_backed_handle(P.SourceDescriptor("s", 1, has_guard=True),
                                                  torch.from_numpy(scal).cuda(), 0))
        active = (0,)
        if with_vector:
            reg.register_handle(P.array_backed_handle(P.SourceDescriptor("v", 3, has_guard=True),
                                                      torch.from_numpy(vec).cuda(), 0))
            active = (0, 1)
        P.update_sources(reg, set(active), {})
        fr = P.default_registry()
        scene = P.SceneState(
            camera=P.Camera(cam["position"], cam["look_at"], vertical_fov=cam["vertical_fov"],
                            image_size=(cam["width"], cam["height"])),
            tf_points={i: pts for i in active}, value_ranges={i: (0.0, 8.0) for i in active},
            chain_texts={0: "", 1: "length"} if with_vector else {0: ""},
            settings=P.RenderSettings(active_set=active, modes={0: mode}, iso_thresholds={0: 2.5},
                                      early_termination_alpha=1.0))
        return P.render_local(P.RankContext(vol, dom, reg, fr, fr.limits), scene).pixels.cpu().numpy()

    got = render("iso")
    srcs = [O.Source(scal, (0, 0, 0), (n, n, n), 0, lut=O.lut_from_points(pts), value_range=(0.0, 8.0),
                     mode="iso", iso_threshold=2.5)]
    if with_vector:
        srcs.append(O.Source(vec, (0, 0, 0), (n, n, n), 0, lut=O.lut_from_points(pts), value_range=(0.0, 8.0),
                             steps=O.parse_steps("length", 3)))
    ref = O.render_brick(cam, O.Brick((0, 0, 0), (n, n, n), 0, (n, n, n)), srcs)
    assert (ref.rgba[..., 3] == 1.0).all()            # every ray stopped on the surface
    assert np.abs(got - ref.rgba).max() <= 1e-3
    with pytest.raises(P.GuardContractError):
        render("volume")


def test_value_range_bit_exact():
    import paper_1611_09048_b200 as P
    from oracle import isaac_oracle as O
    torch = _torch()
    rng = np.random.default_rng(5)
    for dim, chain in ((1, ""), (1, "mul(-2) | add(0.25)"), (3, "length"), (3, "mul(1,2,3) | sum"),
                       (4, "add(0.5) | length | mul(3)")):
        arr = rng.standard_normal((14, 11, 19, dim) if dim > 1 else (14, 11, 19)).astype(np.float32)
        arr[3, 4, 5] = np.nan if dim == 1 else arr[3, 4, 5]
        dom = P.LocalDomain((0, 0, 0), (17, 9, 12), 1)
        h = P.array_backed_handle(P.SourceDescriptor("v", dim, has_guard=True), torch.from_numpy(arr).cuda(), 1)
        ch = P.parse_chain(chain, P.default_registry(), input_dim=dim)
        lo, hi = P.value_range(h, dom, ch)
        want = O.value_range(arr, 1, O.parse_steps(chain, dim))
        assert np.float32(lo) == want[0] and np.float32(hi) == want[1], chain
    # contiguous float32 rows take 16-byte loads: long rows (several partial
    # batches), a base pointer 4 bytes off 16-byte alignment, extremes placed
    # in the scalar head and tail of a row
    for width, off in ((300, 1), (1030, 0), (1030, 3), (7, 2)):
        big = torch.from_numpy(rng.standard_normal((6, 5, width + 2 + off)).astype(np.float32)).cuda()
        view = big[:, :, off:]                      # rows start `off` floats into the allocation
        view[2, 3, 1] = 50.0                        # first interior element of a row (head)
        view[4, 2, width] = -60.0                   # last interior element of a row (tail)
        dom = P.LocalDomain((0, 0, 0), (width, 3, 4), 1)
        h = P.array_backed_handle(P.SourceDescriptor("v", 1, has_guard=True), view, 1)
        lo, hi = P.value_range(h, dom, P.parse_chain("", P.default_registry(), input_dim=1))
        want = O.value_range(view.cpu().numpy(), 1, ())
        assert np.float32(lo) == want[0] == np.float32(-60.0) and np.float32(hi) == want[1] == np.float32(50.0), \
            (width, off)


def test_kernel_nan_pow_chain_is_transparent():
    import paper_1611_09048_b200 as P
    torch = _torch()
    n = 8
    vol = P.GlobalVolume((n, n, n))
    dom = vol.local_domain(0, 1)
    reg = P.SourceRegistry(dom)
    reg.register_handle(P.array_backed_handle(P.SourceDescriptor("f", 1, has_guard=True),
                                              torch.full((n + 2,) * 3, -2.0, device="cuda"), 1))
    P.update_sources(reg, {0}, {})
    fr = P.default_registry()
    ctx = P.RankContext(vol, dom, reg, fr, fr.limits)
    scene = P.SceneState(camera=P.Camera((4.0, 4.0, -20.0), (4.0, 4.0, 4.0), image_size=(16, 16)),
                         chain_texts={0: "pow(0.5)"},
                         tf_points={0: [(0.0, 1.0, 1.0, 1.0, 1.0), (1.0, 1.0, 1.0, 1.0, 1.0)]},
                         settings=P.RenderSettings(active_set=(0,), early_termination_alpha=1.0))
    assert float(P.render_local(ctx, scene).pixels.abs().sum()) == 0.0


def test_missing_device_op_raises_chain_error():
    import paper_1611_09048_b200 as P
    from product_build import product_ctx, product_scene
    c = cases.case("c1")
    ctx = product_ctx(c, (1, 1, 1), 0)
    ctx.functor_registry.register_functor(P.FunctorDescriptor("half", False, lambda d: d),
                                          {d: (lambda v, k: v / 2) for d in range(1, 5)})
    scene = product_scene(c)
    scene = P.SceneState(camera=scene.camera, tf_points=scene.tf_points, value_ranges=scene.value_ranges,
                         chain_texts={0: "half"}, settings=scene.settings)
    with pytest.raises(P.ChainError):
        P.render_local(ctx, scene)
    ctx.functor_registry.register_functor(P.FunctorDescriptor("sqrt", False, lambda d: d),
                                          {d: (lambda v, k: np.sqrt(v)) for d in range(1, 5)})
    scene = P.SceneState(camera=scene.camera, tf_points=scene.tf_points, value_ranges=scene.value_ranges,
                         chain_texts={0: "sqrt"}, settings=scene.settings)
    assert float(P.render_local(ctx, scene).pixels[..., 3].sum()) > 0


def _single_source_scene(P, n, pos, look, chain="", tf=None, rng=(0.0, 1.0), active=(0,), extra=0):
    tf = tf or [(0.0, 0.0, 0.1, 0.2, 0.0), (0.5, 0.9, 0.4, 0.1, 0.3), (1.0, 1.0, 1.0, 0.5, 0.8)]
    ids = list(range(1 + extra))
    return P.SceneState(camera=P.Camera(pos, look, image_size=(48, 32)),
                        tf_points={i: tf for i in ids}, value_ranges={i: rng for i in ids},
                        chain_texts={i: chain for i in ids},
                        settings=P.RenderSettings(active_set=tuple(active), early_termination_alpha=1.0))


@pytest.mark.parametrize("interp", [True, False])
@pytest.mark.parametrize("dtype", ["float64", "float16", "bfloat16"])
def test_other_dtypes(dtype, interp):
    """Non-float32 scalar fields: guarded trilinear takes the paired fast
    kernel with T = double / __half / __nv_bfloat16, nearest the generic
    any-dtype kernel; checked against the oracle on the values the kernel
    reads (converted to float32 on load)."""
    import paper_1611_09048_b200 as P
    from oracle import isaac_oracle as O
    torch = _torch()
    n = 20
    rng = np.random.default_rng(3)
    host = rng.random((n + 2, n + 2, n + 2)).astype(np.float32)
    t = torch.from_numpy(host).to(getattr(torch, dtype)).cuda()
    vals = t.float().cpu().numpy()               # what the kernel actually reads
    vol = P.GlobalVolume((n, n, n))
    dom = vol.local_domain(0, 1)
    reg = P.SourceRegistry(dom)
    reg.register_handle(P.array_backed_handle(P.SourceDescriptor("f", 1, has_guard=True), t, 1))
    P.update_sources(reg, {0}, {})
    fr = P.default_registry()
    ctx = P.RankContext(vol, dom, reg, fr, fr.limits)
    pos, look = (31.0, 27.0, -22.0), (10.0, 10.0, 10.0)
    scene = _single_source_scene(P, n, pos, look)
    if not interp:
        import dataclasses
        scene = P.SceneState(camera=scene.camera, tf_points=scene.tf_points, value_ranges=scene.value_ranges,
                             chain_texts=scene.chain_texts,
                             settings=dataclasses.replace(scene.settings, interpolation=False))
    got = P.render_local(ctx, scene).pixels.cpu().numpy()
    src = O.Source(array=vals.astype(np.float64), offset=(0, 0, 0), size=(n, n, n), guard=1,
                   lut=O.lut_from_points(scene.tf_points[0]), value_range=(0.0, 1.0))
    ref = O.render_brick({"position": pos, "look_at": look, "width": 48, "height": 32},
                         O.Brick((0, 0, 0), (n, n, n), 1, (n, n, n)), [src], interp=interp)
    assert np.abs(got - ref.rgba).max() <= RGBA_TOL


def test_generic_kernel_many_sources():
    """Six active sources (more than the multi kernel's 4) -> generic kernel."""
    import paper_1611_09048_b200 as P
    from oracle import isaac_oracle as O
    torch = _torch()
    n = 16
    rng = np.random.default_rng(4)
    arrays = [rng.random((n + 2, n + 2, n + 2)).astype(np.float32) * 0.4 for _ in range(6)]
    vol = P.GlobalVolume((n, n, n))
    dom = vol.local_domain(0, 1)
    reg = P.SourceRegistry(dom)
    for i, a in enumerate(arrays):
        reg.register_handle(P.array_backed_handle(P.SourceDescriptor(f"s{i}", 1, has_guard=True),
                                                  torch.from_numpy(a).cuda(), 1))
    P.update_sources(reg, set(range(6)), {})
    fr = P.default_registry()
    ctx = P.RankContext(vol, dom, reg, fr, fr.limits)
    pos, look = (25.0, 21.0, -17.0), (8.0, 8.0, 8.0)
    scene = _single_source_scene(P, n, pos, look, chain="mul(1.5) | add(0.05)", active=range(6), extra=5)
    got = P.render_local(ctx, scene).pixels.cpu().numpy()
    srcs = [O.Source(array=a, offset=(0, 0, 0), size=(n, n, n), guard=1, steps=O.parse_steps("mul(1.5) | add(0.05)", 1),
                     lut=O.lut_from_points(scene.tf_points[0]), value_range=(0.0, 1.0)) for a in arrays]
    ref = O.render_brick({"position": pos, "look_at": look, "width": 48, "height": 32},
                         O.Brick((0, 0, 0), (n, n, n), 1, (n, n, n)), srcs)
    assert np.abs(got - ref.rgba).max() <= RGBA_TOL


def test_zero_copy_strided_views():
    """A brick that is a strided view into a larger simulation buffer (padded
    rows, interleaved components) renders identically to a packed copy."""
    import paper_1611_09048_b200 as P
    torch = _torch()
    n = 18
    rng = np.random.default_rng(5)
    big = torch.from_numpy(rng.random((n + 2, n + 9, n + 7, 2)).astype(np.float32)).cuda()
    view = big[:, 3:n + 5, 1:n + 3, 1]               # (z, y, x) with non-unit x stride
    assert not view.is_contiguous()
    packed = view.contiguous()
    vol = P.GlobalVolume((n, n, n))
    dom = vol.local_domain(0, 1)
    imgs = []
    for arr in (view, packed):
        reg = P.SourceRegistry(dom)
        reg.register_handle(P.array_backed_handle(P.SourceDescriptor("f", 1, has_guard=True), arr, 1))
        P.update_sources(reg, {0}, {})
        fr = P.default_registry()
        ctx = P.RankContext(vol, dom, reg, fr, fr.limits)
        scene = _single_source_scene(P, n, (30.0, -9.0, 33.0), (9.0, 9.0, 9.0))
        imgs.append(P.render_local(ctx, scene).pixels.cpu().numpy())
    assert np.array_equal(imgs[0], imgs[1])


def test_numpy_and_sampler_sources_are_staged():
    """numpy arrays and Python samplers are materialised on the device per frame."""
    import paper_1611_09048_b200 as P
    torch = _torch()
    n = 12
    rng = np.random.default_rng(6)
    arr = rng.random((n + 2, n + 2, n + 2)).astype(np.float32)
    vol = P.GlobalVolume((n, n, n))
    dom = vol.local_domain(0, 1)
    scene = _single_source_scene(P, n, (20.0, 17.0, -14.0), (6.0, 6.0, 6.0))
    out = []
    for kind in ("torch", "numpy", "sampler"):
        reg = P.SourceRegistry(dom)
        if kind == "torch":
            reg.register_handle(P.array_backed_handle(P.SourceDescriptor("f", 1, has_guard=True),
                                                      torch.from_numpy(arr).cuda(), 1))
        elif kind == "numpy":
            reg.register_handle(P.array_backed_handle(P.SourceDescriptor("f", 1, has_guard=True), arr, 1))
        else:
            reg.register_source(P.SourceDescriptor("f", 1, has_guard=True), None,
                                batch_sampler=lambda x, y, z: arr[z + 1, y + 1, x + 1])
        P.update_sources(reg, {0}, {})
        fr = P.default_registry()
        out.append(P.render_local(P.RankContext(vol, dom, reg, fr, fr.limits), scene).pixels.cpu().numpy())
    assert np.array_equal(out[0], out[1]) and np.array_equal(out[0], out[2])


def test_analytic_single_ramp_classification_equals_lut_path():
    """A transfer function whose LUT is one straight run is classified as
    base + slope * x; the result matches the shared-memory LUT path and the
    oracle, and non-ramp TFs never take the shortcut."""
    import paper_1611_09048_b200 as P
    from paper_1611_09048_b200.raycast import lut_line
    from product_build import product_ctx, product_scene
    c = cases.case("c1")
    gold = load("render_c1.npz")
    ctx = product_ctx(c, (1, 1, 1), 0)
    scene = product_scene(c)
    assert lut_line(scene.transfer_function(0).lut) is not None
    fast = P.render_local(ctx, scene).pixels.cpu().numpy()
    lut = P.render_local(ctx, scene, analytic_lut=False).pixels.cpu().numpy()
    assert np.abs(fast - lut).max() <= 2e-6
    assert np.abs(fast - gold["d111_r0_rgba"]).max() <= RGBA_TOL
    warm = P.tf_from_points(cases.WARM_TF, (0.0, 1.0))
    assert lut_line(warm.lut) is None


@pytest.mark.parametrize("points", [
    [(0.0, 0.0, 0.1, 0.2, 0.0), (0.6, 0.9, 0.4, 0.1, 0.3), (1.0, 1.0, 1.0, 0.5, 0.8)],       # kink on a sample
    [(0.0, 0.0, 0.1, 0.2, 0.0), (0.37, 0.9, 0.4, 0.1, 0.3), (1.0, 1.0, 1.0, 0.5, 0.8)],      # between samples
    [(0.0, 0.0, 0.0, 0.0, 0.0), (0.2, 0.5, 0.1, 0.1, 0.05), (0.6, 0.1, 0.9, 0.3, 0.4), (1.0, 1.0, 1.0, 1.0, 0.9)],
    # 4 and 6 slope changes: the run-time kink count variant (LINE = ISC_MAX_LUT_KINKS + 1) and,
    # beyond ANALYTIC_MAX_KINKS, the shared-memory LUT
    [(0.0, 0.0, 0.0, 0.0, 0.0), (0.21, 0.5, 0.1, 0.1, 0.05), (0.63, 0.1, 0.9, 0.3, 0.4), (1.0, 1.0, 1.0, 1.0, 0.9)],
    [(0.0, 0.1, 0.0, 0.2, 0.0), (0.13, 0.6, 0.2, 0.1, 0.2), (0.47, 0.2, 0.8, 0.3, 0.05), (0.81, 0.9, 0.3, 0.7, 0.6),
     (1.0, 1.0, 1.0, 1.0, 0.9)],
])
@pytest.mark.parametrize("alpha_stop", [1.0, 0.95])
def test_piecewise_linear_tf_classified_analytically(points, alpha_stop):
    """tf_from_points LUTs with 1-5 slope changes take the analytic hinge form
    (base + slope x + sum dslope_k max(x - x_k, 0)), more take the LUT;
    images match the shared-memory LUT path and the CPU oracle."""
    import paper_1611_09048_b200 as P
    from oracle import isaac_oracle as O
    from paper_1611_09048_b200.raycast import describe_kernel, lut_analytic
    torch = _torch()
    n = 32
    rng = np.random.default_rng(77)
    field = rng.random((n + 2,) * 3).astype(np.float32)
    vol = P.GlobalVolume((n, n, n))
    dom = vol.local_domain(0, 1)
    reg = P.SourceRegistry(dom)
    reg.register_handle(P.array_backed_handle(P.SourceDescriptor("f", 1, has_guard=True),
                                              torch.from_numpy(field).cuda(), 1))
    P.update_sources(reg, {0}, {})
    fr = P.default_registry()
    ctx = P.RankContext(vol, dom, reg, fr, fr.limits)
    pos, look = (51.0, 40.0, -30.0), (15.0, 16.0, 17.0)
    scene = P.SceneState(camera=P.Camera(pos, look, image_size=(80, 60)), tf_points={0: points},
                         value_ranges={0: (0.1, 0.9)},
                         settings=P.RenderSettings(active_set=(0,), early_termination_alpha=alpha_stop))
    pw = lut_analytic(scene.transfer_function(0).lut)
    kinks = lut_analytic(scene.transfer_function(0).lut, max_kinks=7)[2]
    assert (pw is not None) == (len(kinks) <= 5) and 1 <= len(kinks) <= 7
    plans = P.build_plans(reg, fr, fr.limits, scene)
    line = 0 if pw is None else (1 + len(kinks) if len(kinks) <= 3 else 8)
    assert f"LINE={line}" in describe_kernel(plans, scene.settings)
    fast = P.render_local(ctx, scene).pixels.cpu().numpy()
    lut = P.render_local(ctx, scene, analytic_lut=False).pixels.cpu().numpy()
    # identical up to float32 rounding; with early termination a pixel may
    # stop one station apart where the alpha test sits on the threshold
    assert np.abs(fast - lut).max() <= (5e-6 if alpha_stop >= 1.0 else RGBA_TOL)
    src = O.Source(array=field, offset=(0, 0, 0), size=(n, n, n), guard=1, lut=O.lut_from_points(points),
                   value_range=(0.1, 0.9))
    ref = O.render_brick({"position": pos, "look_at": look, "width": 80, "height": 60},
                         O.Brick((0, 0, 0), (n, n, n), 1, (n, n, n)), [src], alpha_stop=alpha_stop)
    assert np.abs(fast - ref.rgba).max() <= RGBA_TOL


@pytest.mark.parametrize("multi", [False, True])
def test_screen_rect_culling_is_exact(multi):
    """Without per-pixel debug outputs the persistent kernels only schedule
    tiles inside the brick's projected screen rectangle (and clear the rest);
    the image must be bit-identical to the full-raster render (debug outputs
    requested), for every brick of a 2x2x2 decomposition and cameras outside,
    grazing and inside the volume."""
    import paper_1611_09048_b200 as P
    torch = _torch()
    n = 32
    rng = np.random.default_rng(17)
    full = rng.random((n + 2, n + 2, n + 2)).astype(np.float32)
    vec = rng.random((n + 2, n + 2, n + 2, 3)).astype(np.float32)
    vol = P.GlobalVolume((n, n, n), (2, 2, 2))
    cams = [((70.0, 50.0, -40.0), (16.0, 16.0, 16.0)), ((16.0, 90.0, 16.5), (16.0, 16.0, 16.0)),
            ((-3.0, 5.0, 4.0), (30.0, 20.0, 28.0)), ((15.0, 17.0, 14.0), (0.0, 40.0, 30.0)),
            ((8.0, 8.5, -1.5), (8.0, 8.0, 8.0))]  # brick 0 fills the image: rectangle == whole image
    for r in range(8):
        dom = vol.local_domain(r, 1)
        ox, oy, oz = dom.offset
        reg = P.SourceRegistry(dom)
        sl = np.s_[oz:oz + 18, oy:oy + 18, ox:ox + 18]
        reg.register_handle(P.array_backed_handle(P.SourceDescriptor("s", 1, has_guard=True),
                                                  torch.from_numpy(np.ascontiguousarray(full[sl])).cuda(), 1))
        reg.register_handle(P.array_backed_handle(P.SourceDescriptor("v", 3, has_guard=True),
                                                  torch.from_numpy(np.ascontiguousarray(vec[sl])).cuda(), 1))
        active = (0, 1) if multi else (0,)
        P.update_sources(reg, set(active), {})
        fr = P.default_registry()
        ctx = P.RankContext(vol, dom, reg, fr, fr.limits)
        for pos, look in cams:
            scene = P.SceneState(
                camera=P.Camera(pos, look, image_size=(64, 48)),
                tf_points={0: [(0.0, 0.0, 0.0, 0.0, 0.0), (1.0, 1.0, 0.5, 0.2, 0.6)],
                           1: [(0.0, 0.0, 0.0, 0.0, 0.0), (1.0, 0.2, 0.9, 1.0, 0.4)]},
                value_ranges={0: (0.0, 1.0), 1: (0.0, 2.0)}, chain_texts={0: "", 1: "length"},
                settings=P.RenderSettings(active_set=active, modes={0: "iso"} if multi else {},
                                          iso_thresholds={0: 0.5}, early_termination_alpha=1.0))
            # into a NaN-filled canvas: a pixel the culled launch neither
            # clears nor writes shows up as NaN (the canvas is left uncleared
            # when the rectangle is the whole image)
            canvas = torch.full((48, 64, 4), float("nan"), device="cuda")
            culled = P.render_local(ctx, scene, out=canvas).pixels.cpu().numpy()
            fullraster = P.render_local(ctx, scene, keep_station_counts=True).pixels.cpu().numpy()
            assert np.array_equal(culled, fullraster), (r, pos)


def test_early_termination_stops_before_a_bad_tail():
    """Early termination on the paired kernel: rays that saturate before the
    far face of a guard-0 brick gather no bad corner and must not raise; with
    early termination off the same rays reach the face and must raise
    (fields.py:230-238: the reference raises only on gathers it performs)."""
    import math
    import paper_1611_09048_b200 as P
    from oracle import isaac_oracle as O
    torch = _torch()
    n = 8
    z, y, x = np.meshgrid(*(np.arange(n, dtype=np.float64),) * 3, indexing="ij")
    field = (0.6 + 0.05 * np.sin(x + 2 * y + 3 * z)).astype(np.float32)
    vol = P.GlobalVolume((n, n, n))
    dom = vol.local_domain(0, 0)
    cam = dict(position=(-50.0, 3.7, 3.3), look_at=(4.0, 3.7, 3.3), vertical_fov=math.radians(5.0),
               width=16, height=12)
    pts = [(0.0, 0.0, 0.0, 0.0, 0.0), (1.0, 1.0, 0.5, 0.2, 1.0)]

    def render(alpha_stop):
        reg = P.SourceRegistry(dom)
        reg.register_handle(P.array_backed_handle(P.SourceDescriptor("s", 1, has_guard=True),
                                                  torch.from_numpy(field).cuda(), 0))
        P.update_sources(reg, {0}, {})
        fr = P.default_registry()
        scene = P.SceneState(
            camera=P.Camera(cam["position"], cam["look_at"], vertical_fov=cam["vertical_fov"],
                            image_size=(cam["width"], cam["height"])),
            tf_points={0: pts}, value_ranges={0: (0.0, 0.7)}, chain_texts={0: ""},
            settings=P.RenderSettings(active_set=(0,), early_termination_alpha=alpha_stop))
        img = P.render_local(P.RankContext(vol, dom, reg, fr, fr.limits), scene, keep_station_counts=True)
        return img.pixels.cpu().numpy(), img.station_counts.cpu().numpy()

    got, counts = render(0.99)
    ref = O.render_brick(cam, O.Brick((0, 0, 0), (n, n, n), 0, (n, n, n)),
                         [O.Source(field, (0, 0, 0), (n, n, n), 0, lut=O.lut_from_points(pts), value_range=(0.0, 0.7))],
                         alpha_stop=0.99)
    assert np.abs(got - ref.rgba).max() <= 1e-3
    assert (counts.reshape(-1).astype(np.int64) != ref.stations.reshape(-1)).sum() == 0, int((counts.reshape(-1).astype(np.int64) != ref.stations.reshape(-1)).sum())
    with pytest.raises(P.GuardContractError):
        render(1.0)


def test_occupancy_tuning_is_invisible():
    """The march kernels' online occupancy choice (two trial launches per
    key, then the faster) changes only how many persistent CTAs run: every
    render of a key is bit-identical, before, during and after the trials."""
    import paper_1611_09048_b200 as P
    torch = _torch()
    n = 40
    rng = np.random.default_rng(23)
    arr = torch.from_numpy(rng.random((n + 2, n + 2, n + 2)).astype(np.float32)).cuda()
    vol = P.GlobalVolume((n, n, n))
    dom = vol.local_domain(0, 1)
    reg = P.SourceRegistry(dom)
    reg.register_handle(P.array_backed_handle(P.SourceDescriptor("f", 1, has_guard=True), arr, 1))
    P.update_sources(reg, {0}, {})
    fr = P.default_registry()
    ctx = P.RankContext(vol, dom, reg, fr, fr.limits)
    scene = _single_source_scene(P, n, (70.0, 55.0, -31.0), (20.0, 20.0, 20.0))
    imgs = []
    for _ in range(5):
        imgs.append(P.render_local(ctx, scene).pixels.cpu().numpy())
        torch.cuda.synchronize()
    for im in imgs[1:]:
        assert np.array_equal(im, imgs[0])


def test_random_cameras_bricks_early_termination_vs_oracle():
    """Seeded random cameras on 2x1x1 / 2x2x2 decompositions, with and without
    early termination: every brick's partial image (screen-rectangle culled,
    paired kernel incl. its early-termination variant) against the oracle's
    render of the same brick."""
    import paper_1611_09048_b200 as P
    from oracle import isaac_oracle as O
    torch = _torch()
    rng = np.random.default_rng(4321)
    n = 24
    field = rng.random((n + 2, n + 2, n + 2), dtype=np.float32)
    for trial in range(6):
        decomp = [(2, 1, 1), (2, 2, 2), (1, 2, 1)][trial % 3]
        alpha_stop = [1.0, 0.95][trial % 2]
        pos = tuple(float(v) for v in rng.uniform(-2 * n, 3 * n, 3))
        target = tuple(float(v) for v in rng.uniform(0.3 * n, 0.7 * n, 3))
        w, h = int(rng.integers(17, 70)), int(rng.integers(9, 50))
        pts = [(0.0, *rng.random(4)), (float(rng.uniform(0.2, 0.8)), *rng.random(4)), (1.0, *rng.random(4))]
        vol = P.GlobalVolume((n, n, n), decomp)
        scene = P.SceneState(camera=P.Camera(pos, target, image_size=(w, h)), tf_points={0: pts},
                             value_ranges={0: (0.1, 0.9)},
                             settings=P.RenderSettings(active_set=(0,), early_termination_alpha=alpha_stop))
        for r in range(int(np.prod(decomp))):
            dom = vol.local_domain(r, 1)
            ox, oy, oz = dom.offset
            sx, sy, sz = dom.size
            arr = np.ascontiguousarray(field[oz:oz + sz + 2, oy:oy + sy + 2, ox:ox + sx + 2])
            reg = P.SourceRegistry(dom)
            reg.register_handle(P.array_backed_handle(P.SourceDescriptor("f", 1, has_guard=True),
                                                      torch.from_numpy(arr).cuda(), 1))
            P.update_sources(reg, {0}, {})
            fr = P.default_registry()
            got = P.render_local(P.RankContext(vol, dom, reg, fr, fr.limits), scene).pixels.cpu().numpy()
            src = O.Source(array=arr, offset=dom.offset, size=dom.size, guard=1, lut=O.lut_from_points(pts),
                           value_range=(0.1, 0.9))
            ref = O.render_brick({"position": pos, "look_at": target, "width": w, "height": h},
                                 O.Brick(dom.offset, dom.size, 1, (n, n, n), decomp), [src], alpha_stop=alpha_stop)
            err = np.abs(got - ref.rgba).max(axis=-1)
            # early termination: a float32 threshold test may end a ray one station apart
            assert (err > RGBA_TOL).sum() == 0, (trial, r, err.max(), int((err > RGBA_TOL).sum()))


def test_launch_block_cache_revalidates():
    """Re-rendering the same scene objects reuses the packed launch block, but
    a different field tensor behind the same handle (update_sources swapping
    arrays) or a steered transfer function is picked up: images match fresh
    renders."""
    import paper_1611_09048_b200 as P
    torch = _torch()
    n = 16
    rng = np.random.default_rng(31)
    a0 = torch.from_numpy(rng.random((n + 2,) * 3).astype(np.float32)).cuda()
    a1 = torch.from_numpy(rng.random((n + 2,) * 3).astype(np.float32)).cuda()
    vol = P.GlobalVolume((n, n, n))
    dom = vol.local_domain(0, 1)
    reg = P.SourceRegistry(dom)
    h = P.array_backed_handle(P.SourceDescriptor("f", 1, has_guard=True), a0, 1)
    reg.register_handle(h)
    P.update_sources(reg, {0}, {})
    fr = P.default_registry()
    ctx = P.RankContext(vol, dom, reg, fr, fr.limits)
    scene = _single_source_scene(P, n, (40.0, 30.0, -20.0), (8.0, 8.0, 8.0))
    plans = P.build_plans(reg, fr, fr.limits, scene)
    first = P.render_local(ctx, scene, plans=plans).pixels.cpu().numpy()
    again = P.render_local(ctx, scene, plans=plans).pixels.cpu().numpy()
    assert np.array_equal(first, again)
    h.array = a1                                   # the simulation swapped its buffer
    swapped = P.render_local(ctx, scene, plans=plans).pixels.cpu().numpy()
    h2 = P.array_backed_handle(P.SourceDescriptor("g", 1, has_guard=True), a1, 1)
    reg2 = P.SourceRegistry(dom)
    reg2.register_handle(h2)
    P.update_sources(reg2, {0}, {})
    fresh = P.render_local(P.RankContext(vol, dom, reg2, fr, fr.limits), scene).pixels.cpu().numpy()
    assert np.array_equal(swapped, fresh) and not np.array_equal(swapped, first)


def test_launch_block_not_cached_for_converted_fields():
    """An integer field is converted to a float32 copy per frame (as the
    reference casts every batch, fields.py:177); the launch block must not be
    reused across frames (it would point at the previous frame's freed copy),
    and an in-place update of the simulation's int array must show up."""
    import paper_1611_09048_b200 as P
    torch = _torch()
    n = 16
    rng = np.random.default_rng(37)
    ai = torch.from_numpy(rng.integers(0, 4, (n + 2,) * 3).astype(np.int32)).cuda()
    vol = P.GlobalVolume((n, n, n))
    dom = vol.local_domain(0, 1)
    reg = P.SourceRegistry(dom)
    reg.register_handle(P.array_backed_handle(P.SourceDescriptor("f", 1, has_guard=True), ai, 1))
    P.update_sources(reg, {0}, {})
    fr = P.default_registry()
    ctx = P.RankContext(vol, dom, reg, fr, fr.limits)
    scene = _single_source_scene(P, n, (40.0, 30.0, -20.0), (8.0, 8.0, 8.0))
    scene = P.SceneState(camera=scene.camera, tf_points=scene.tf_points, value_ranges={0: (0.0, 4.0)},
                         chain_texts=scene.chain_texts, settings=scene.settings)
    plans = P.build_plans(reg, fr, fr.limits, scene)

    def frame():
        img = P.render_local(ctx, scene, plans=plans).pixels.cpu().numpy()
        junk = [torch.full((n + 2,) * 3, 1e6, device="cuda") for _ in range(4)]   # reuse freed blocks
        del junk
        return img

    first = frame()
    assert np.array_equal(frame(), first)
    ai.add_(1)                                     # simulation updates its field in place
    after = frame()
    reg2 = P.SourceRegistry(dom)
    reg2.register_handle(P.array_backed_handle(P.SourceDescriptor("g", 1, has_guard=True), ai.float(), 1))
    P.update_sources(reg2, {0}, {})
    want = P.render_local(P.RankContext(vol, dom, reg2, fr, fr.limits), scene).pixels.cpu().numpy()
    assert np.array_equal(after, want) and not np.array_equal(after, first)


@pytest.mark.parametrize("seed", range(4))
def test_staged_gather_is_bit_identical(seed, monkeypatch):
    """Shared-memory brick staging (march_staged.cu, ISC_STAGE=1) reads the
    same corner values and does the same arithmetic as the direct gather:
    images and station totals are bit-identical, including chunks whose box
    overflows the warp's slice (far camera / long rays fall back to global)."""
    import paper_1611_09048_b200 as P
    torch = _torch()
    monkeypatch.setenv("ISC_QUAD", "0")    # the staging prototype is the 2-lanes-per-ray march
    rng = np.random.default_rng(900 + seed)
    n = int(rng.choice([24, 48, 96]))
    field = torch.from_numpy(rng.random((n + 2,) * 3).astype(np.float32)).cuda()
    vol = P.GlobalVolume((n, n, n), (2, 1, 1) if seed % 2 else (1, 1, 1))
    for rank in range(vol.rank_count):
        dom = vol.local_domain(rank, 1)
        (ox, oy, oz), (sx, sy, sz) = dom.offset, dom.size
        reg = P.SourceRegistry(dom)
        reg.register_handle(P.array_backed_handle(P.SourceDescriptor("f", 1, has_guard=True),
                                                  field[oz:oz + sz + 2, oy:oy + sy + 2, ox:ox + sx + 2], 1))
        P.update_sources(reg, {0}, {})
        fr = P.default_registry()
        ctx = P.RankContext(vol, dom, reg, fr, fr.limits)
        pos = tuple(float(v) for v in rng.uniform(-1.5 * n, 2.5 * n, 3))
        pts = [(0.0, 0.0, 0.0, 0.0, 0.0), (1.0, 1.0, 1.0, 1.0, 1.0)] if seed < 2 else \
            [(0.0, *rng.random(4)), (0.5, *rng.random(4)), (1.0, *rng.random(4))]
        scene = P.SceneState(camera=P.Camera(pos, (n / 2.0,) * 3, image_size=(97, 61)), tf_points={0: pts},
                             value_ranges={0: (0.1, 0.9)},
                             settings=P.RenderSettings(active_set=(0,), step_length=float(rng.choice([0.5, 0.3])),
                                                       early_termination_alpha=1.0))
        for analytic in (True, False):
            monkeypatch.delenv("ISC_STAGE", raising=False)
            ref = P.render_local(ctx, scene, analytic_lut=analytic)
            monkeypatch.setenv("ISC_STAGE", "1")
            got = P.render_local(ctx, scene, analytic_lut=analytic)
            monkeypatch.delenv("ISC_STAGE", raising=False)
            assert torch.equal(got.pixels, ref.pixels), (seed, rank, analytic)
            assert got.stations == ref.stations


def test_composite_user_functor_renders_like_its_expansion():
    """A user functor registered with device_chain renders exactly like the
    chain it expands to (same device op program)."""
    import paper_1611_09048_b200 as P
    from paper_1611_09048_b200.functors import FunctorDescriptor
    torch = _torch()
    n = 20
    rng = np.random.default_rng(5)
    vec = torch.from_numpy(rng.random((n + 2,) * 3 + (3,)).astype(np.float32)).cuda()
    vol = P.GlobalVolume((n, n, n))
    dom = vol.local_domain(0, 1)
    reg = P.SourceRegistry(dom)
    reg.register_handle(P.array_backed_handle(P.SourceDescriptor("v", 3, has_guard=True), vec, 1))
    P.update_sources(reg, {0}, {})
    fr = P.default_registry()
    ev = {d: (lambda v, c: np.sqrt(np.sum((v * c[None, :]) ** 2, axis=1, keepdims=True))) for d in range(1, 5)}
    fr.register_functor(FunctorDescriptor("scaled_norm", True, lambda d: 1), ev, device_chain="mul($) | length")
    ctx = P.RankContext(vol, dom, reg, fr, fr.limits)
    imgs = []
    for chain in ("scaled_norm(2) | add(0.1)", "mul(2) | length | add(0.1)"):
        scene = P.SceneState(camera=P.Camera((33.0, 27.0, -19.0), (10.0, 10.0, 10.0), image_size=(40, 30)),
                             tf_points={0: [(0.0, 0.0, 0.1, 0.2, 0.0), (1.0, 1.0, 0.6, 0.3, 0.5)]},
                             value_ranges={0: (0.0, 4.0)}, chain_texts={0: chain},
                             settings=P.RenderSettings(active_set=(0,), early_termination_alpha=1.0))
        imgs.append(P.render_local(ctx, scene).pixels)
    assert torch.equal(imgs[0], imgs[1]) and float(imgs[0][..., 3].max()) > 0


@pytest.mark.parametrize("iso_chain", ["", "mul(1.5) | add(-4.75)", "pow(2) | mul(0.1)"])
@pytest.mark.parametrize("probe", ["paired", "multi-probe", "single-kernel"])
def test_split_iso_volume_render_matches_oracle(probe, iso_chain, monkeypatch):
    """Iso source + volume source scenes render in two passes (iso probe,
    then the volume march stopped at each ray's hit, march.cu launch_split);
    the paired probe (default), the multi-source kernel as the probe
    (ISC_DISABLE_PAIRED_PROBE=1) and the single multi-source kernel
    (ISC_DISABLE_SPLIT=1) give the same station counts and images within
    float32 rounding, and all match the CPU oracle -- for an identity iso
    chain, an add / mul chain (float64 decisions) and a general chain; the
    culled render (no per-pixel outputs) equals the full-raster one."""
    import paper_1611_09048_b200 as P
    from oracle import isaac_oracle as O
    torch = _torch()
    if probe == "multi-probe":
        monkeypatch.setenv("ISC_DISABLE_PAIRED_PROBE", "1")
    if probe == "single-kernel":
        monkeypatch.setenv("ISC_DISABLE_SPLIT", "1")
    n = 28
    rng = np.random.default_rng(41)
    z, y, x = np.meshgrid(*(np.arange(-1, n + 1, dtype=np.float64),) * 3, indexing="ij")
    scal = np.sqrt((x - n / 2) ** 2 + (y - n / 2 + 0.3) ** 2 + (z - n / 2 - 0.2) ** 2).astype(np.float32)
    vec = rng.random((n + 2,) * 3 + (3,)).astype(np.float32)
    cool = [(0.0, 0.0, 0.0, 0.0, 0.0), (0.6, 0.1, 0.7, 0.4, 0.3), (1.0, 0.7, 1.0, 0.9, 0.8)]
    pos, look = (61.0, 47.0, -37.0), (14.0, 13.5, 14.5)
    for decomp in ((1, 1, 1), (2, 1, 1)):
        vol = P.GlobalVolume((n, n, n), decomp)
        for rank in range(vol.rank_count):
            dom = vol.local_domain(rank, 1)
            (ox, oy, oz), (sx, sy, sz) = dom.offset, dom.size
            sl = np.s_[oz:oz + sz + 2, oy:oy + sy + 2, ox:ox + sx + 2]
            reg = P.SourceRegistry(dom)
            reg.register_handle(P.array_backed_handle(P.SourceDescriptor("s", 1, has_guard=True),
                                                      torch.from_numpy(np.ascontiguousarray(scal[sl])).cuda(), 1))
            reg.register_handle(P.array_backed_handle(P.SourceDescriptor("v", 3, has_guard=True),
                                                      torch.from_numpy(np.ascontiguousarray(vec[sl])).cuda(), 1))
            P.update_sources(reg, {0, 1}, {})
            fr = P.default_registry()
            ctx = P.RankContext(vol, dom, reg, fr, fr.limits)
            scene = P.SceneState(camera=P.Camera(pos, look, image_size=(72, 54)),
                                 tf_points={0: [(0.0, 0.0, 0.0, 0.0, 0.0), (1.0, 1.0, 1.0, 1.0, 1.0)], 1: cool},
                                 value_ranges={0: (0.0, 20.0), 1: (0.0, 6.0)},
                                 chain_texts={0: iso_chain, 1: "length | mul(2) | add(0.1)"},
                                 settings=P.RenderSettings(active_set=(0, 1), modes={0: "iso"},
                                                           iso_thresholds={0: 9.5}, early_termination_alpha=1.0))
            img = P.render_local(ctx, scene, keep_station_counts=True)
            culled = P.render_local(ctx, scene)
            assert torch.equal(culled.pixels, img.pixels)
            srcs = [O.Source(np.ascontiguousarray(scal[sl]), dom.offset, dom.size, 1,
                             lut=O.lut_from_points(scene.tf_points[0]), value_range=(0.0, 20.0), mode="iso",
                             iso_threshold=9.5, steps=O.parse_steps(iso_chain, 1)),
                    O.Source(np.ascontiguousarray(vec[sl]), dom.offset, dom.size, 1, lut=O.lut_from_points(cool),
                             value_range=(0.0, 6.0), steps=O.parse_steps("length | mul(2) | add(0.1)", 3))]
            ref = O.render_brick({"position": pos, "look_at": look, "width": 72, "height": 54},
                                 O.Brick(dom.offset, dom.size, 1, (n, n, n), decomp), srcs)
            assert np.abs(img.pixels.cpu().numpy() - ref.rgba).max() <= RGBA_TOL
            assert np.array_equal(img.station_counts.cpu().numpy().astype(np.int64), ref.stations.reshape(-1))
