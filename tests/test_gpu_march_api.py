"""The reference's single-ray / explicit-ray API on the device:
``march_rays`` / ``march_ray`` (raycast.py:291-381, 471-489) and
``gradient_normal(s)`` (raycast.py:210-256), run through the same sm_100a
kernels as ``render_local`` (ray-list mode of isc_render_args, and
isc_gradient_normals).

The first two classes restate the reference's own known-answer tests
(test_raycast.py:129-172 TestMarch, 346-375 TestGradient) against this
package; the last compares explicit ray lists with the CPU oracle.
"""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _plan(fn, domain, dim=1, tf=None, mode="volume", iso=0.5, has_guard=False):
    """Sampler-backed plan, as the reference's analytic_plan (test_raycast.py:52-70)."""
    import paper_1611_09048_b200 as P
    desc = P.SourceDescriptor("analytic", dim, has_guard=has_guard, persistent=True)

    def batch(ix, iy, iz):
        return np.asarray(fn(ix, iy, iz), dtype=np.float64).reshape(len(ix), dim)

    handle = P.SourceHandle(desc, lambda i, j, k: P.FieldVector(tuple(batch(
        np.asarray([i]), np.asarray([j]), np.asarray([k]))[0])), batch_sampler=batch)
    return P.SourcePlan(source_id=0, handle=handle, domain=domain, chain=P.identity_chain(dim),
                        tf=tf if tf is not None else _grayscale(), mode=mode, iso_threshold=iso)


def _grayscale(value_range=(0.0, 1.0), alpha=None):
    import paper_1611_09048_b200 as P
    lut = np.empty((256, 4))
    t = np.linspace(0.0, 1.0, 256)
    for c in range(4):
        lut[:, c] = t
    if alpha is not None:
        lut[:, 3] = alpha
    return P.TransferFunction(lut, value_range)


class TestMarch:
    def test_transparent_tf_yields_zero(self):
        import paper_1611_09048_b200 as P
        dom = P.LocalDomain((0, 0, 0), (8, 8, 8), 0)
        plan = _plan(lambda x, y, z: np.ones(len(x)), dom, tf=_grayscale(alpha=0.0))
        out = P.march_ray((-1, 4, 4), (1, 0, 0), (0.0, 8.0), [plan],
                          P.RenderSettings(active_set=(0,), interpolation=False))
        assert tuple(out) == (0.0, 0.0, 0.0, 0.0)

    def test_homogeneous_alpha_accumulation(self):
        import paper_1611_09048_b200 as P
        a = 0.3
        dom = P.LocalDomain((0, 0, 0), (32, 32, 32), 0)
        plan = _plan(lambda x, y, z: np.full(len(x), 0.7), dom, tf=_grayscale(alpha=a))
        settings = P.RenderSettings(active_set=(0,), interpolation=False, step_length=0.1,
                                    early_termination_alpha=1.0)
        n_stations = 20
        t0, t1 = 0.05, 0.05 + 0.1 * n_stations
        out = P.march_ray((0, 16, 16), (1, 0, 0), (t0, t1), [plan], settings)
        assert out[3] == pytest.approx(1.0 - (1.0 - a) ** n_stations, abs=1e-5)

    def test_alpha_monotone_over_prefix_intervals(self):
        import paper_1611_09048_b200 as P
        dom = P.LocalDomain((0, 0, 0), (32, 32, 32), 0)
        plan = _plan(lambda x, y, z: (x % 7) / 7.0, dom)
        settings = P.RenderSettings(active_set=(0,), interpolation=False, step_length=0.5,
                                    early_termination_alpha=1.0)
        alphas = [P.march_ray((0, 9.3, 11.1), (1, 0, 0), (0.25, 0.25 + 0.5 * m), [plan], settings)[3]
                  for m in range(1, 30)]
        assert all(b >= a - 1e-7 for a, b in zip(alphas, alphas[1:]))

    def test_early_termination_stops_accumulation(self):
        import paper_1611_09048_b200 as P
        dom = P.LocalDomain((0, 0, 0), (32, 32, 32), 0)
        plan = _plan(lambda x, y, z: np.ones(len(x)), dom, tf=_grayscale(alpha=0.5))
        settings = P.RenderSettings(active_set=(0,), interpolation=False, step_length=0.5,
                                    early_termination_alpha=0.9)
        out = P.march_ray((0, 16, 16), (1, 0, 0), (0.0, 32.0), [plan], settings)
        assert out[3] == pytest.approx(1.0 - 0.5 ** 4)   # first accumulation >= 0.9


class TestGradient:
    def test_linear_ramp_normal_along_x(self):
        import paper_1611_09048_b200 as P
        dom = P.LocalDomain((0, 0, 0), (16, 16, 16), 0)
        plan = _plan(lambda x, y, z: x.astype(float), dom)
        n = P.gradient_normal(plan, (8.2, 8.0, 8.0), (0, 0, 1), interpolation=False)
        assert abs(abs(n[0]) - 1.0) < 1e-9
        assert abs(n[1]) < 1e-9 and abs(n[2]) < 1e-9

    def test_spherical_field_normal_is_radial(self):
        import paper_1611_09048_b200 as P
        center = np.array([32.0, 32.0, 32.0])
        dom = P.LocalDomain((0, 0, 0), (64, 64, 64), 0)

        def radial(x, y, z):
            return np.sqrt((x - center[0]) ** 2 + (y - center[1]) ** 2 + (z - center[2]) ** 2)

        plan = _plan(radial, dom)
        rng = np.random.default_rng(11)
        for _ in range(10):
            d = rng.normal(size=3)
            d /= np.linalg.norm(d)
            n = P.gradient_normal(plan, center + 20.0 * d, -d, interpolation=True)
            assert abs(float(np.dot(n, d))) > 1.0 - 1e-3

    def test_constant_field_falls_back_to_view_opposite(self):
        import paper_1611_09048_b200 as P
        dom = P.LocalDomain((0, 0, 0), (8, 8, 8), 0)
        plan = _plan(lambda x, y, z: np.full(len(x), 3.0), dom)
        n = P.gradient_normal(plan, (4, 4, 4), (0, 0, 1), interpolation=False)
        assert np.allclose(n, (0, 0, -1))


@pytest.mark.parametrize("mode", ["volume", "iso"])
def test_march_rays_matches_oracle(mode):
    """Random rays through a guarded 24^3 field with the slab intervals as the
    explicit intervals: device ray-list march == oracle render_rays (<= 1e-3),
    station totals equal."""
    import paper_1611_09048_b200 as P
    from oracle import isaac_oracle as O
    n = 24
    rng = np.random.default_rng(21)
    field = rng.random((n + 2, n + 2, n + 2)).astype(np.float32)
    z, y, x = np.meshgrid(*(np.arange(-1, n + 1, dtype=np.float64),) * 3, indexing="ij")
    if mode == "iso":
        field = np.sqrt((x - 12.0) ** 2 + (y - 11.0) ** 2 + (z - 12.5) ** 2).astype(np.float32)
    dom = P.LocalDomain((0, 0, 0), (n, n, n), 1)
    import torch
    handle = P.array_backed_handle(P.SourceDescriptor("f", 1, has_guard=True), torch.from_numpy(field).cuda(), 1)
    pts = [(0.0, 0.0, 0.1, 0.2, 0.0), (0.5, 0.9, 0.5, 0.1, 0.4), (1.0, 1.0, 0.9, 0.8, 0.9)]
    rng_v = (0.0, 1.0) if mode == "volume" else (0.0, 20.0)
    plan = P.SourcePlan(0, handle, dom, P.identity_chain(1), P.tf_from_points(pts, rng_v), mode, 7.5)
    origin = np.array([40.0, 31.0, -17.0])
    target = rng.uniform(2.0, n - 2.0, size=(300, 3))
    dirs = target - origin
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    t0, t1 = O.slab(origin, dirs, np.zeros(3), np.full(3, float(n)))
    settings = P.RenderSettings(active_set=(0,), modes={0: mode}, iso_thresholds={0: 7.5},
                                early_termination_alpha=1.0)
    got, stations = P.march_rays(origin, dirs, (t0, t1), (t0, t1), [plan], settings)
    src = O.Source(array=field, offset=(0, 0, 0), size=(n, n, n), guard=1, lut=O.lut_from_points(pts),
                   value_range=rng_v, mode=mode, iso_threshold=7.5)
    ref = O.render_rays(tuple(origin), dirs, O.Brick((0, 0, 0), (n, n, n), 1, (n, n, n)), [src])
    assert np.abs(got - ref.rgba).max() <= 1e-3
    assert stations == int(ref.stations.sum())


@pytest.mark.parametrize("thr", [3.0, 5.0, 6.5])
def test_march_rays_without_layout_clamps_iso_entry_pairs(thr):
    """march_rays(volume=None) with a guarded trilinear iso source: the
    reference clamps each entry pair's earlier station into the guard reach
    instead of testing reachability, and checks no exit pairs
    (raycast.py:396-418).  Golden from the real reference
    (tests/golden/make_golden_march.py), rays entering a brick through its
    upper y face; rays whose hit shading reads past the halo raise
    GuardContractError there and here."""
    import paper_1611_09048_b200 as P
    from golden_io import load
    torch = pytest.importorskip("torch")
    gold = load("march_nolayout.npz")
    off, size, g = tuple(int(v) for v in gold["offset"]), tuple(int(v) for v in gold["size"]), int(gold["guard"])
    dom = P.LocalDomain(off, size, g)
    handle = P.array_backed_handle(P.SourceDescriptor("d", 1, has_guard=True),
                                   torch.from_numpy(gold["field"]).cuda(), g)
    plan = P.SourcePlan(source_id=0, handle=handle, domain=dom, chain=P.identity_chain(1),
                        tf=P.TransferFunction(gold["tf_lut"], (0.0, 12.0)), mode="iso", iso_threshold=thr)
    settings = P.RenderSettings(active_set=(0,), modes={0: "iso"}, iso_thresholds={0: thr}, interpolation=True,
                                step_length=0.5, early_termination_alpha=1.0)
    raised = gold[f"raised_{thr}"]
    ok = ~raised
    rgba, stations = P.march_rays(gold["origin"], gold["dirs"][ok], (gold["t0"][ok], gold["t1"][ok]),
                                  (gold["g0"][ok], gold["g1"][ok]), [plan], settings)
    assert np.abs(rgba - gold[f"rgba_{thr}"][ok]).max() <= 1e-3
    assert stations == int(gold[f"stations_{thr}"][ok].sum())
    for i in np.nonzero(raised)[0]:
        sl = slice(i, i + 1)
        with pytest.raises(P.GuardContractError):
            P.march_rays(gold["origin"], gold["dirs"][sl], (gold["t0"][sl], gold["t1"][sl]),
                         (gold["g0"][sl], gold["g1"][sl]), [plan], settings)
