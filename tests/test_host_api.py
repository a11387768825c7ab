"""Host-side logic of the drop-in API (no GPU): the reference's own unit tests
for fields / functors / scene / compositing restated against
paper_1611_09048_b200, plus the render-argument packing and the device
op-program lowering.  Reference tests mirrored: test_fields.py,
test_functors.py, test_raycast.py (classify / ray-box), test_compositing.py
(visibility order, messages)."""

import math

import numpy as np
import pytest

import paper_1611_09048_b200 as P
from paper_1611_09048_b200 import _abi
from paper_1611_09048_b200.compositing import CompositeMessage, swap_schedule, visibility_order
from paper_1611_09048_b200.functors import device_program
from oracle import isaac_oracle as O


# ---- fields (test_fields.py) ------------------------------------------------

def ramp(size, guard):
    n = size + 2 * guard
    z, y, x = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    return (x + 10.0 * y + 100.0 * z).astype(np.float64)


def test_volume_layout_and_tiling():
    with pytest.raises(P.FieldError):
        P.GlobalVolume((10, 10, 10), (3, 1, 1))
    vol = P.GlobalVolume((8, 8, 8), (2, 2, 2))
    assert [vol.brick_coords(r) for r in (0, 1, 2, 4)] == [(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)]
    assert all(vol.rank_of(vol.brick_coords(r)) == r for r in range(8))
    for size, dec in [((4, 4, 4), (1, 1, 1)), ((4, 6, 2), (2, 3, 1)), ((8, 4, 4), (4, 2, 2))]:
        assert P.tile_check(P.GlobalVolume(size, dec))
    assert P.GlobalVolume((8, 8, 8), (2, 1, 1)).local_domain(1).offset == (4, 0, 0)


def test_guard_and_clamp_contract():
    dom = P.LocalDomain((0, 0, 0), (4, 4, 4), 1)
    h = P.array_backed_handle(P.SourceDescriptor("r", 1, has_guard=True), ramp(4, 1), 1)
    assert P.sample(h, dom, (-1, 0, 0), True).components == (0.0 + 10 + 100,)
    with pytest.raises(P.GuardContractError):
        P.sample(h, dom, (-2, 0, 0), True)
    nog = P.array_backed_handle(P.SourceDescriptor("n", 1, has_guard=False), ramp(4, 1), 1)
    assert P.sample(nog, dom, (-5, 9, 2), True).components == P.sample(nog, dom, (0, 3, 2)).components
    got = P.sample_many(nog, dom, np.array([-3, 7]), np.array([0, 0]), np.array([0, 0]))
    assert got.shape == (2, 1)


def test_registry_and_update_order():
    dom = P.LocalDomain((0, 0, 0), (2, 2, 2), 1)
    reg = P.SourceRegistry(dom)
    calls = []
    for name in ("a", "b", "c"):
        reg.register_source(P.SourceDescriptor(name, 1), lambda i, j, k: P.field_vector(1.0),
                            update_hook=lambda en, pl, name=name: calls.append((name, en)))
    with pytest.raises(P.DuplicateSourceError):
        reg.register_source(P.SourceDescriptor("a", 1), lambda i, j, k: P.field_vector(1.0))
    P.update_sources(reg, {0, 2}, {})
    assert calls == [("a", True), ("b", False), ("c", True)]

    def boom(en, pl):
        raise RuntimeError("bad")

    reg.register_source(P.SourceDescriptor("d", 1), lambda i, j, k: P.field_vector(1.0), update_hook=boom)
    with pytest.raises(P.SourceUpdateError, match="d"):
        P.update_sources(reg, {3}, {})


def test_snapshot_non_persistent_isolated():
    dom = P.LocalDomain((0, 0, 0), (3, 3, 3), 1)
    arr = ramp(3, 1)
    h = P.array_backed_handle(P.SourceDescriptor("np", 1, has_guard=True, persistent=False), arr, 1)
    snap = P.snapshot_non_persistent(h, dom)
    arr[...] = -1.0
    assert P.sample(snap, dom, (0, 0, 0)).components[0] == 111.0
    with pytest.raises(P.FieldError):
        P.snapshot_non_persistent(snap, dom)


def test_sampler_sources_materialise_for_the_device():
    dom = P.LocalDomain((0, 0, 0), (4, 3, 2), 1)
    h = P.SourceHandle(P.SourceDescriptor("an", 1, has_guard=True), None,
                       batch_sampler=lambda x, y, z: x + 10.0 * y + 100.0 * z)
    arr, g = h.device_view(dom)
    assert g == 1 and arr.shape == (4, 5, 6)
    assert arr[1, 1, 1] == 0.0 and arr[0, 0, 0] == -111.0
    assert h.sample_count == 0


# ---- functors (test_functors.py) -------------------------------------------

def test_parse_chain_grammar():
    reg = P.default_registry()
    c = P.parse_chain("mul(2,3,4) | add(1) | length", reg, input_dim=3)
    assert len(c.steps) == 3 and c.output_dim == 1 and c.steps[1].argument == (1.0, 1.0, 1.0)
    assert P.parse_chain("", reg, input_dim=3).output_dim == 3
    a = P.parse_chain("mul( 2 , 3 ,4)|add(1)  |length", reg, input_dim=3)
    assert [s.argument for s in a.steps] == [s.argument for s in c.steps]
    with pytest.raises(P.ChainError, match="unknown functor"):
        P.parse_chain("foo", reg, input_dim=1)
    with pytest.raises(P.ChainError, match="limit"):
        P.parse_chain("add(1)|add(1)|add(1)", reg, P.ChainLimits(max_length=2), input_dim=1)
    for bad in ("add(1,2)", "add", "length(2)"):
        with pytest.raises(P.ChainError):
            P.parse_chain(bad, reg, input_dim=3)
    assert [s.input_dim for s in P.parse_chain("length | add(3) | mul(2)", reg, input_dim=4).steps] == [4, 1, 1]


def test_eval_chain_known_answers():
    reg = P.default_registry()
    c = P.parse_chain("mul(2,3,4) | add(1) | length", reg, input_dim=3)
    assert P.eval_chain(c, P.field_vector(1, 1, 1)).components == (math.sqrt(50.0),)
    c = P.parse_chain("mul(0,1,0) | sum", reg, input_dim=3)
    assert P.eval_chain(c, P.field_vector(7, 9, 2)).components == (9.0,)
    assert math.isnan(P.eval_chain(P.parse_chain("pow(0.5)", reg), P.field_vector(-2.0)).components[0])


def test_registry_extension_and_device_ops():
    reg = P.default_registry()
    with pytest.raises(P.ChainError, match="already registered"):
        reg.register_functor(P.FunctorDescriptor("add", True, lambda d: d), {d: (lambda v, c: v) for d in range(1, 5)})
    with pytest.raises(P.ChainError, match="missing evaluators"):
        reg.register_functor(P.FunctorDescriptor("half", False, lambda d: d), {1: lambda v, c: v / 2})
    reg.register_functor(P.FunctorDescriptor("sqrt", False, lambda d: d), {d: (lambda v, c: np.sqrt(v)) for d in range(1, 5)})
    assert P.eval_chain(P.parse_chain("sqrt", reg), P.field_vector(9.0)).components == (3.0,)
    prog = device_program(P.parse_chain("sqrt | mul(2)", reg))
    assert [p[0] for p in prog] == [_abi.OPCODES["sqrt"], _abi.OPCODES["mul"]]
    reg.register_functor(P.FunctorDescriptor("halve", False, lambda d: d), {d: (lambda v, c: v / 2) for d in range(1, 5)})
    with pytest.raises(P.ChainError, match="device opcode"):
        device_program(P.parse_chain("halve", reg))
    reg.register_functor(P.FunctorDescriptor("scale", True, lambda d: d), {d: (lambda v, c: v * c) for d in range(1, 5)},
                         device_op="mul")
    assert device_program(P.parse_chain("scale(3)", reg))[0] == (_abi.OPCODES["mul"], 1, (3.0, 0.0, 0.0, 0.0))


def test_device_program_matches_float32_oracle_semantics():
    reg = P.default_registry()
    prog = device_program(P.parse_chain("mul(2) | add(0.5,1.5,-1) | length", reg, input_dim=3))
    assert [(op, dim) for op, dim, _ in prog] == [(2, 3), (1, 3), (4, 3)]
    assert prog[0][2] == (2.0, 2.0, 2.0, 0.0) and prog[1][2] == (0.5, 1.5, -1.0, 0.0)


# ---- scene (test_raycast.py classify / ray-box, scene JSON) ----------------

def test_classify_known_answers():
    lut = np.repeat(np.linspace(0, 1, 256)[:, None], 4, axis=1)
    tf = P.TransferFunction(lut, (10.0, 20.0))
    assert P.classify(tf, 10.0) == tuple(lut[0]) and P.classify(tf, 99.0) == tuple(lut[255])
    assert P.classify(tf, float("nan")) == (0.0, 0.0, 0.0, 0.0)
    with pytest.raises(P.SceneError):
        P.TransferFunction(lut, (1.0, 1.0))


def test_scene_json_round_trip_and_validation():
    s = P.SceneState(camera=P.Camera((1, 2, 3), (0, 0, 0), image_size=(32, 18)),
                     tf_points={0: [(0, 0, 0, 0, 0), (1, 1, 1, 1, 1)]}, value_ranges={0: (0.0, 2.0)},
                     chain_texts={0: "length"}, settings=P.RenderSettings(active_set=(0,), modes={0: "iso"}),
                     clip_planes=(P.clip_plane((0, 0, 0), (0, 0, 2)),))
    assert P.SceneState.from_bytes(s.to_bytes()) == s
    with pytest.raises(P.SceneError):
        P.Camera((0, 0, 0), (0, 0, 0))
    with pytest.raises(P.SceneError):
        P.RenderSettings(step_length=0)
    with pytest.raises(P.SceneError):
        P.ClipPlane((0, 0, 0), (0, 0, 2))


def test_ray_box_intersection_known_answers():
    from paper_1611_09048_b200.raycast import ray_box_intersection
    hit = ray_box_intersection((-1, 0.5, 0.5), (1, 0, 0), (0, 0, 0), (1, 1, 1))
    assert hit[1] - hit[0] == pytest.approx(1.0)
    assert ray_box_intersection((2.0, -1.0, 0.5), (0, 1, 0), (0, 0, 0), (1, 1, 1)) is None
    plane = P.clip_plane((0.5, 0.0, 0.0), (1.0, 0.0, 0.0))
    assert ray_box_intersection((-1, 0.5, 0.5), (1, 0, 0), (0, 0, 0), (1, 1, 1), [plane]) == pytest.approx((1.5, 2.0))
    with pytest.raises(ValueError):
        ray_box_intersection((0, 0, 0), (0, 0, 0), (0, 0, 0), (1, 1, 1))


def test_camera_basis_matches_oracle_bit_for_bit():
    cam = P.Camera((140.0, 115.0, -88.7), (50.0, 50.0, 50.0), image_size=(33, 17))
    f, r, u = cam.basis()
    of, orr, ou = O.camera_frame(cam.position, cam.look_at, cam.up)
    assert np.array_equal(f, of) and np.array_equal(r, orr) and np.array_equal(u, ou)
    assert np.array_equal(cam.ray_directions(), O.primary_rays(cam.position, cam.look_at, cam.up,
                                                               cam.vertical_fov, 33, 17))


# ---- compositing host logic (test_compositing.py) --------------------------

def test_visibility_order_cases():
    vol = P.GlobalVolume((8, 8, 8), (2, 1, 1))
    assert visibility_order(vol, P.Camera((-10, 4, 4), (4, 4, 4), image_size=(8, 8))) == [0, 1]
    assert visibility_order(vol, P.Camera((4.0, 4.0, -9.0), (4, 4, 4), image_size=(8, 8))) == [0, 1]
    vol8 = P.GlobalVolume((8, 8, 8), (2, 2, 2))
    assert visibility_order(vol8, P.Camera((6.0, 6.9, 1.2), (0, 0, 0), image_size=(8, 8)))[0] == 3
    rng = np.random.default_rng(0)
    for _ in range(50):
        pos = tuple(rng.uniform(-30, 46, 3))
        cam = P.Camera(pos, tuple(rng.uniform(4, 12, 3)), image_size=(8, 8))
        assert visibility_order(vol8, cam) == O.visibility_order((8, 8, 8), (2, 2, 2), pos)


def test_swap_schedule_matches_oracle():
    for size in (2, 4, 8, 16):
        order = list(np.random.default_rng(size).permutation(size))
        for rank in range(size):
            plan, fin = swap_schedule(order.index(rank), size, 1000003)
            oplan, ofin = O.swap_schedule(rank, size, order, 1000003)
            assert fin == ofin
            assert [(order[pv], k, g, pv < order.index(rank)) for pv, k, g in plan] == oplan


def test_composite_message_round_trip():
    payload = np.arange(12, dtype=np.float32).reshape(3, 4)
    back = CompositeMessage.from_bytes(CompositeMessage(2, 5, 7, 3, payload).to_bytes())
    assert (back.round_index, back.sender, back.span_offset, back.span_length) == (2, 5, 7, 3)
    assert np.array_equal(back.payload, payload)
    with pytest.raises(P.CompositeError):
        CompositeMessage.from_bytes(CompositeMessage(0, 0, 0, 3, np.zeros((3, 4))).to_bytes()[:-16])


def test_local_fabric_and_run_ranks():
    res = P.run_ranks(3, lambda t: t.broadcast_from_root(b"x" if t.rank == 0 else None))
    assert res == [b"x", b"x", b"x"]
    fab = P.LocalFabric(2, default_timeout=0.05)
    with pytest.raises(P.TransportError):
        fab.endpoint(0).receive(1)


# ---- render argument packing (no launch) -------------------------------------

def test_pack_render_args_on_host_tensors():
    import torch
    from paper_1611_09048_b200.raycast import build_plans, pack_render_args
    vol = P.GlobalVolume((16, 16, 16), (2, 1, 1))
    dom = vol.local_domain(1, 1)
    reg = P.SourceRegistry(dom)
    t = torch.zeros((18, 18, 10, 3))
    reg.register_handle(P.array_backed_handle(P.SourceDescriptor("v", 3, has_guard=True), t, 1))
    P.update_sources(reg, {0}, {})
    fr = P.default_registry()
    scene = P.SceneState(camera=P.Camera((40.0, 30.0, -20.0), (8.0, 8.0, 8.0), image_size=(20, 10)),
                         chain_texts={0: "length | mul(2) | add(0.1)"}, value_ranges={0: (0.0, 3.0)},
                         settings=P.RenderSettings(active_set=(0,), modes={0: "iso"}, iso_thresholds={0: 1.25}),
                         clip_planes=(P.clip_plane((8, 8, 8), (0.3, -0.5, 0.81)),))
    keep = []
    a = pack_render_args(dom, vol, scene, build_plans(reg, fr, fr.limits, scene), torch.device("cpu"), keep)
    assert (a.camera.width, a.camera.height) == (20, 10) and a.camera.aspect == 2.0
    assert list(a.brick_offset) == [8, 0, 0] and list(a.brick_size) == [8, 16, 16]
    s = a.src[0]
    assert list(s.stride) == [18 * 10 * 3, 10 * 3, 3, 1] and s.feature_dim == 3 and s.mode == _abi.ISO
    assert s.n_steps == 3 and s.steps[0].op == _abi.OPCODES["length"] and s.steps[1].in_dim == 1
    assert s.iso_threshold == 1.25 and (s.range_lo, s.range_hi) == (0.0, 3.0)
    n = np.asarray(scene.clip_planes[0].normal)
    assert a.n_clip == 1 and a.clip[0].f0 == float(np.dot(np.asarray((40.0, 30.0, -20.0)) - 8.0, n))
    with pytest.raises(P.FieldError):
        bad = P.SourceRegistry(dom)
        bad.register_handle(P.array_backed_handle(P.SourceDescriptor("w", 1, has_guard=True), torch.zeros((5, 5, 5)), 1))
        P.update_sources(bad, {0}, {})
        pack_render_args(dom, vol, P.SceneState(camera=scene.camera, settings=P.RenderSettings(active_set=(0,))),
                         build_plans(bad, fr, fr.limits, P.SceneState(camera=scene.camera,
                                                                      settings=P.RenderSettings(active_set=(0,)))),
                         torch.device("cpu"), [])


# ---- runtime host logic (runtime.py:81-100, 305-333) ------------------------

def test_merge_metadata_rules():
    from paper_1611_09048_b200.runtime import merge_metadata
    assert merge_metadata([{"a": 1}, {"a": 2}]) == {"a": 1}
    assert merge_metadata([{"v": [1]}, {"v": [2, 3]}]) == {"v": [1, 2, 3]}
    assert len(merge_metadata([{f"k{i}": i} for i in range(12)])) == 12
    doc = {"a": 1, "v": [1, 2], "o": {"x": 1}}
    assert merge_metadata([doc]) == doc


def test_broadcast_scene_aborts_on_bad_chain_everywhere():
    from paper_1611_09048_b200.runtime import FrameAborted, PipelineContext, broadcast_scene
    dom = P.LocalDomain((0, 0, 0), (4, 4, 4), 1)
    good = P.SceneState(camera=P.Camera((10, 10, -10), (2, 2, 2), image_size=(8, 8)), chain_texts={0: "add(1)"},
                        settings=P.RenderSettings(active_set=(0,)))
    bad = good.bump(chain_texts={0: "nosuch"})

    def body(t):
        reg = P.SourceRegistry(dom)
        reg.register_source(P.SourceDescriptor("f", 1), lambda i, j, k: P.field_vector(1.0))
        fr = P.default_registry()
        ctx = PipelineContext(t, None, dom, reg, fr, fr.limits, good)
        ok = broadcast_scene(ctx, good if t.rank == 0 else None)[0]
        try:
            broadcast_scene(ctx, bad if t.rank == 0 else None)
            return "no-abort"
        except FrameAborted:
            return (ok == good, ctx.scene == good)

    assert P.run_ranks(3, body) == [(True, True)] * 3


def test_station_cells_monotone_in_k():
    """The kernels check the guard contract at a ray's end stations only; that
    is exact because every axis of pos_k = o + (k*step)*d (float64,
    round-to-nearest, raycast.py:346) is monotone in k, so each cell index
    floor(pos_k) is too.  Checked on random rays, with positions evaluated
    exactly as numpy (and the device) evaluate them."""
    rng = np.random.default_rng(11)
    k = np.arange(0, 4000, dtype=np.float64)
    for _ in range(200):
        o = rng.uniform(-3000.0, 3000.0, 3)
        d = rng.normal(size=3)
        d /= np.sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2])
        step = float(rng.choice([0.5, 0.37, 1.0 / 3.0, 0.25]))
        pos = o[None, :] + (k * step)[:, None] * d[None, :]
        cells = np.floor(pos)
        for a in range(3):
            diff = np.diff(cells[:, a])
            assert (diff >= 0).all() or (diff <= 0).all()


def test_describe_kernel_mirrors_dispatch():
    """Bench lines name the kernel the library dispatches to (host mirror)."""
    import torch
    from paper_1611_09048_b200.raycast import build_plans, describe_kernel
    n = 8
    dom = P.GlobalVolume((n, n, n)).local_domain(0, 1)
    reg = P.SourceRegistry(dom)
    reg.register_handle(P.array_backed_handle(P.SourceDescriptor("s", 1, has_guard=True),
                                              torch.zeros((n + 2,) * 3), 1))
    reg.register_handle(P.array_backed_handle(P.SourceDescriptor("v", 3, has_guard=True),
                                              torch.zeros((n + 2,) * 3 + (3,)), 1))
    P.update_sources(reg, {0, 1}, {})
    fr = P.default_registry()
    linear = [(0.0, 0.0, 0.0, 0.0, 0.0), (1.0, 1.0, 1.0, 1.0, 1.0)]
    one = P.SceneState(camera=P.Camera((20.0, 17.0, -9.0), (4.0, 4.0, 4.0)), tf_points={0: linear},
                       settings=P.RenderSettings(active_set=(0,), early_termination_alpha=1.0))
    k = describe_kernel(build_plans(reg, fr, fr.limits, one), one.settings)
    assert k.startswith("isc::march_fast_kernel") and "LINE=1" in k and "ET=0" in k
    two = P.SceneState(camera=one.camera, chain_texts={1: "length"},
                       settings=P.RenderSettings(active_set=(0, 1), modes={0: "iso"}))
    assert describe_kernel(build_plans(reg, fr, fr.limits, two), two.settings).startswith(
        "isc::march_multi_fast_kernel<NS=2")
    split = P.SceneState(camera=one.camera, chain_texts={1: "length"},
                         settings=P.RenderSettings(active_set=(0, 1), modes={0: "iso"}, early_termination_alpha=1.0))
    k = describe_kernel(build_plans(reg, fr, fr.limits, split), split.settings)
    assert k.startswith("isc::iso_probe_kernel<CHAIN=0>") and "DIM=3" in k and "AOS3=1" in k


def test_lut_analytic_hinge_form_equals_lut_lerp():
    """The analytic transfer-function form (raycast.lut_analytic) equals the
    LUT lerp of scene.classify_array (scene.py:139-152) everywhere on
    [0, 255] for tf_from_points ramps with up to ANALYTIC_MAX_KINKS slope changes, and is
    refused (None) beyond that or for non-piecewise LUTs."""
    import numpy as np
    import paper_1611_09048_b200 as P
    from paper_1611_09048_b200.raycast import lut_analytic, lut_line
    rng = np.random.default_rng(3)
    seen = {k: 0 for k in range(8)}
    seen[None] = 0
    for trial in range(400):
        k = int(rng.integers(0, 6))
        mids = sorted(float(int(rng.integers(1, 255)) / 255.0) if rng.random() < 0.5 else float(rng.uniform(0.01, 0.99))
                      for _ in range(k))
        pts = [(0.0, *rng.random(4)), *[(t, *rng.random(4)) for t in mids], (1.0, *rng.random(4))]
        lut = P.tf_from_points(pts, (0.0, 1.0)).lut
        res = lut_analytic(lut, max_kinks=7)
        seen[None if res is None else len(res[2])] += 1
        x = np.concatenate([rng.uniform(0.0, 255.0, 2000), np.arange(256.0)])
        i = np.floor(x).astype(int)
        j = np.minimum(i + 1, 255)
        want = lut[i] + (x - i)[:, None] * (lut[j] - lut[i])
        if res is None:
            continue
        base, slope, kinks = res
        got = base[None, :] + slope[None, :] * x[:, None]
        for xk, d in kinks:
            got = got + d[None, :] * np.maximum(x - xk, 0.0)[:, None]
        # float64 rounding of the hinge sums (lut_analytic verifies <= 1e-9 at
        # the samples); far below the float32 the kernels evaluate it in
        assert np.abs(got - want).max() <= 1e-9, (pts, kinks)
    assert all(seen[c] > 10 for c in (0, 1, 2, 3, 4)) and seen[None] > 10, seen
    assert lut_line(P.tf_from_points([(0, 0, 0, 0, 0), (1, 1, 1, 1, 1)], (0, 1)).lut) is not None
    noisy = np.sin(np.linspace(0.0, 3.0, 256))[:, None] * np.ones((1, 4))
    assert lut_analytic(noisy) is None


def test_apply_steering_matches_reference_goldens():
    """runtime.apply_steering folds steering messages exactly as the
    reference (runtime.py:111-184): same resulting scene (JSON), control
    events, dropped and unknown counts, on 60 seeded sequences generated by
    the real reference (tests/golden/make_golden_steering.py)."""
    import json
    import logging
    import paper_1611_09048_b200 as P
    from paper_1611_09048_b200.runtime import apply_steering
    import os
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "steering.json")) as fh:
        gold = json.load(fh)
    logging.getLogger("paper_1611_09048_b200.runtime").setLevel(logging.ERROR)
    base = P.SceneState.from_json(gold["base"])
    for case in gold["cases"]:
        msgs = [m.encode() if b else m for m, b in zip(case["messages"], case["bytes"])]
        res = apply_steering(base, msgs)
        assert json.loads(json.dumps(res.scene.to_json())) == case["scene"]
        assert res.controls == case["controls"]
        assert (res.dropped, res.unknown) == (case["dropped"], case["unknown"])


def test_composite_user_functor_lowers_to_device_steps():
    """A user functor defined by a chain of device steps (register_functor(...,
    device_chain=...), $ = its constant) lowers inline into the kernel op
    program; the host evaluators still serve eval_chain."""
    import numpy as np
    import pytest
    import paper_1611_09048_b200 as P
    from paper_1611_09048_b200 import _abi
    from paper_1611_09048_b200.functors import FunctorDescriptor, device_program
    reg = P.default_registry()
    ev = {d: (lambda v, c: np.sqrt(np.sum((v * c[None, :]) ** 2, axis=1, keepdims=True))) for d in range(1, 5)}
    reg.register_functor(FunctorDescriptor("scaled_norm", True, lambda d: 1), ev, device_chain="mul($) | length")
    ch = P.parse_chain("scaled_norm(2) | add(1)", reg, None, 3)
    prog = device_program(ch)
    assert [op for op, _, _ in prog] == [_abi.OPCODES["mul"], _abi.OPCODES["length"], _abi.OPCODES["add"]]
    assert prog[0][2][:3] == (2.0, 2.0, 2.0) and prog[2][1] == 1
    out = P.eval_chain(ch, P.FieldVector((1.0, 2.0, 2.0)))
    assert abs(out.components[0] - 7.0) < 1e-12
    # a wrong domain map is caught when lowering; no device path at all raises
    reg.register_functor(FunctorDescriptor("bad", False, lambda d: d), {d: ev[d] for d in ev}, device_chain="length")
    with pytest.raises(P.ChainError):
        device_program(P.parse_chain("bad", reg, None, 3))
    reg.register_functor(FunctorDescriptor("host_only", False, lambda d: d), {d: (lambda v, c: v) for d in ev})
    with pytest.raises(P.ChainError):
        device_program(P.parse_chain("host_only", reg, None, 2))


def test_fold_affine_tail_preserves_normalised_value():
    """raycast.fold_affine_tail: a volume source's trailing scalar add / mul
    steps fold into its value range -- (f(v) - lo) / (hi - lo) is unchanged
    (float64, random chains); mul by a non-positive constant, non-scalar
    steps and chains without such a tail are left alone."""
    import math
    import numpy as np
    from paper_1611_09048_b200 import _abi
    from paper_1611_09048_b200.raycast import fold_affine_tail
    add, mul, length = _abi.OPCODES["add"], _abi.OPCODES["mul"], _abi.OPCODES["length"]
    rng = np.random.default_rng(5)
    v = rng.normal(0.0, 3.0, 1000)
    for _ in range(200):
        tail = [(int(rng.choice([add, mul])), 1, (float(rng.uniform(0.2, 3.0)), 0.0, 0.0, 0.0))
                for _ in range(int(rng.integers(1, 4)))]
        prog = [(length, 3, (0.0,) * 4)] + tail
        lo, hi = sorted(rng.uniform(-5, 5, 2))
        out, lo2, hi2 = fold_affine_tail(prog, lo, hi)
        assert out == prog[:1]
        f = v.copy()
        for op, _, arg in tail:
            f = f * arg[0] if op == mul else f + arg[0]
        assert np.allclose((f - lo) / (hi - lo), (v - lo2) / (hi2 - lo2), rtol=1e-9, atol=1e-9)
    neg = [(mul, 1, (-2.0, 0.0, 0.0, 0.0)), (add, 1, (1.0, 0.0, 0.0, 0.0))]
    assert fold_affine_tail(neg, 0.0, 1.0) == (neg, 0.0, 1.0)
    vec = [(mul, 3, (2.0, 2.0, 2.0, 0.0)), (length, 3, (0.0,) * 4)]
    assert fold_affine_tail(vec, 0.0, 1.0) == (vec, 0.0, 1.0)
    assert fold_affine_tail([], 0.0, 1.0) == ([], 0.0, 1.0)
    assert math.isclose(fold_affine_tail([(add, 1, (0.5, 0, 0, 0))], 0.0, 1.0)[1], -0.5)


def test_float_stop_threshold_equals_float64_test():
    """The kernels test early termination as w >= stop_f, stop_f =
    __double2float_ru(alpha_stop) (the smallest float >= alpha_stop), in
    place of the reference's float64 (double)w >= alpha_stop
    (raycast.py:377-380): the two agree for every float w."""
    import numpy as np
    rng = np.random.default_rng(5)
    alphas = np.concatenate([rng.random(2000), [0.99, 0.5, 1.0 - 2.0 ** -30, 2.0 ** -149, 0.1]])
    for a in alphas:
        t = np.float32(a)
        if float(t) < a:
            t = np.nextafter(t, np.float32(np.inf))
        w = np.array([np.nextafter(t, np.float32(-np.inf)), t, np.nextafter(t, np.float32(np.inf)), np.float32(a),
                      np.float32(np.nan)], dtype=np.float32)
        assert np.array_equal(w >= t, w.astype(np.float64) >= a), a


def test_frame_graph_refuses_byte_transports():
    """runtime.FrameGraph replays a multi-rank frame only over an
    NvlinkTransport (device-resident swap epoch); a byte transport with more
    than one rank is refused before any device work."""
    import pytest
    import paper_1611_09048_b200 as P
    vol = P.GlobalVolume((8, 8, 8), (2, 1, 1))
    dom = vol.local_domain(0, 1)
    reg = P.SourceRegistry(dom)
    fr = P.default_registry()
    ctx = P.RankContext(vol, dom, reg, fr, fr.limits, P.LocalFabric(2).endpoint(0))
    scene = P.SceneState(camera=P.Camera((30.0, 4.0, 4.0), (4.0, 4.0, 4.0), image_size=(8, 8)))
    with pytest.raises(ValueError, match="NvlinkTransport"):
        P.FrameGraph(ctx, scene)
