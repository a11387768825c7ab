"""Golden vectors for the explicit-ray API without a volume layout:
``march_rays(..., volume=None)`` of the REAL reference (raycast.py:291-381)
with a guarded trilinear iso source, where entry pairs are clamped into the
guard reach (raycast.py:404-409) instead of tested for reachability, and no
exit pairs are checked.

Run in the build container only:  ``python tests/golden/make_golden_march.py``
-> ``tests/golden/march_nolayout.npz`` (committed; read by
tests/test_gpu_march_api.py).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from insitu import fields as ref_fields  # noqa: E402
from insitu import functors as ref_fun  # noqa: E402
from insitu import raycast as ref_ray  # noqa: E402
from insitu import scene as ref_scene  # noqa: E402


def field(n_x, n_y, n_z, g, offset):
    """Smooth scalar over the brick + guard: a sphere-distance field whose
    iso surfaces cross brick faces (values depend on global coordinates)."""
    z, y, x = np.meshgrid(*(np.arange(-g, n + g, dtype=np.float64) + o
                            for n, o in ((n_z, offset[2]), (n_y, offset[1]), (n_x, offset[0]))), indexing="ij")
    return np.sqrt((x - 7.3) ** 2 + (y - 8.1) ** 2 + (z - 7.7) ** 2).astype(np.float32)


def main():
    rng = np.random.default_rng(2024)
    g = 1
    # the lower-y brick of a 16^3 volume decomposed (1, 2, 1); rays enter it
    # through its upper y face, where the guard does not reach (reach ends at
    # offset + size + g - 1), so every entry pair's earlier station is clamped
    offset, size = (0, 0, 0), (16, 8, 16)
    arr = field(*size, g, offset)
    dom = ref_fields.LocalDomain(offset, size, g)
    desc = ref_fields.SourceDescriptor("d", 1, has_guard=True)
    handle = ref_fields.array_backed_handle(desc, arr, g)
    tf = ref_scene.tf_from_points([(0.0, 0.0, 0.0, 0.0, 0.0), (1.0, 0.9, 0.6, 0.3, 0.7)], (0.0, 12.0))
    chain = ref_fun.parse_chain("", ref_fun.default_registry(), ref_fun.ChainLimits(), 1)
    out = {"field": arr, "offset": np.asarray(offset), "size": np.asarray(size), "guard": np.asarray(g)}
    n = 300
    origin = np.array([7.6, 31.0, 8.25])
    target = rng.uniform([1.0, 0.5, 1.0], [15.0, 7.5, 15.0], (n, 3))
    dirs = target - origin
    dirs /= np.linalg.norm(dirs, axis=1)[:, None]
    lo, hi = np.asarray(offset, np.float64), np.asarray(offset, np.float64) + np.asarray(size, np.float64)
    t0, t1 = ref_ray._ray_box_intervals(origin, dirs, lo, hi)
    g0, g1 = ref_ray._ray_box_intervals(origin, dirs, np.zeros(3), np.full(3, 16.0))
    for thr in (3.0, 5.0, 6.5):
        plan = ref_ray.SourcePlan(source_id=0, handle=handle, domain=dom, chain=chain, tf=tf, mode="iso",
                                  iso_threshold=thr)
        settings = ref_scene.RenderSettings(active_set=(0,), modes={0: "iso"}, iso_thresholds={0: thr},
                                            interpolation=True, step_length=0.5, early_termination_alpha=1.0)
        # one call per ray: the reference raises GuardContractError for the
        # whole batch when any ray's hit shading reads past the halo, so
        # record per ray either its colour or that it raised
        rgba = np.zeros((n, 4))
        raised = np.zeros(n, dtype=bool)
        stations = np.zeros(n, dtype=np.int64)
        for i in range(n):
            sl = slice(i, i + 1)
            try:
                rgba[i], stations[i] = ref_ray.march_rays(origin, dirs[sl], (t0[sl], t1[sl]), (g0[sl], g1[sl]),
                                                          [plan], settings, volume=None)
            except ref_fields.GuardContractError:
                raised[i] = True
        out[f"rgba_{thr}"] = rgba
        out[f"raised_{thr}"] = raised
        out[f"stations_{thr}"] = stations
        # the same rays WITH the layout (exact entry pairs + forward exit
        # pairs): must differ somewhere, or this case would not pin the clamp
        vol = ref_fields.GlobalVolume((16, 16, 16), (1, 2, 1))
        ok = ~raised
        with_layout, _ = ref_ray.march_rays(origin, dirs[ok], (t0[ok], t1[ok]), (g0[ok], g1[ok]), [plan],
                                            settings, volume=vol)
        print(thr, "raised:", int(raised.sum()), "rays differing from the layout-aware march:",
              int((np.abs(with_layout - rgba[ok]).max(axis=1) > 1e-6).sum()), "of", int(ok.sum()))
    out.update(origin=origin, dirs=dirs, t0=t0, t1=t1, g0=g0, g1=g1, tf_lut=tf.lut)
    np.savez_compressed(os.path.join(HERE, "march_nolayout.npz"), **out)
    print("wrote march_nolayout.npz")


if __name__ == "__main__":
    main()
