"""Render / composite cases shared by ``make_golden.py`` (reference side) and the
parity tests (oracle and CUDA side).  Plain data only."""

from __future__ import annotations

import math

LINEAR_TF = [(0.0, 0.0, 0.0, 0.0, 0.0), (1.0, 1.0, 1.0, 1.0, 1.0)]
WARM_TF = [(0.0, 0.05, 0.05, 0.25, 0.0), (0.45, 0.1, 0.45, 0.85, 0.35),
           (0.75, 0.95, 0.65, 0.2, 0.7), (1.0, 1.0, 0.95, 0.75, 0.95)]
COOL_TF = [(0.0, 0.0, 0.0, 0.0, 0.0), (0.6, 0.1, 0.7, 0.4, 0.3), (1.0, 0.7, 1.0, 0.9, 0.8)]


def harness_camera(n, image_size):
    """The reference harness camera (harness.py:80-85) for a cube of edge n."""
    diag = math.sqrt(3.0 * n * n)
    return {"position": [n * 1.4, n * 1.15, -0.8 * diag], "look_at": [n / 2.0] * 3,
            "up": [0.0, 1.0, 0.0], "vertical_fov": math.radians(45.0),
            "image_size": list(image_size)}


def test_camera(n, image_size):
    """The reference tests' default camera (test_raycast.py:211-221)."""
    return {"position": [n * 1.3, n * 1.6, -1.1 * n], "look_at": [n / 2.0] * 3,
            "up": [0.0, 1.0, 0.0], "vertical_fov": math.radians(45.0),
            "image_size": list(image_size)}


def src(field, *, chain="", tf=LINEAR_TF, rng=(0.0, 1.0), mode="volume", iso=0.5, has_guard=True):
    return {"field": field, "chain": chain, "tf_points": [list(p) for p in tf],
            "range": list(rng), "mode": mode, "iso": iso, "has_guard": has_guard}


RENDER_CASES = {
    # configs[0] of BASELINE.json: 64^3 f32, 256x256, trilinear, linear TF.
    "c1": dict(size=[64, 64, 64], decompositions=[[1, 1, 1]], camera=harness_camera(64, (256, 256)),
               sources=[src("smooth", rng=(0.0, 2.4))], active=[0]),
    "random_bricks": dict(size=[32, 32, 32], decompositions=[[1, 1, 1], [2, 2, 2]],
                          camera=harness_camera(32, (128, 96)),
                          sources=[src("random", rng=(0.0, 1.0), tf=WARM_TF)], active=[0]),
    "clip": dict(size=[32, 32, 32], decompositions=[[1, 1, 1], [2, 1, 1]],
                 camera=test_camera(32, (120, 80)),
                 sources=[src("smooth", rng=(0.3, 2.3), tf=WARM_TF)], active=[0],
                 planes=[[[16.0, 16.0, 16.0], [0.3, -0.5, 0.81]]]),
    "nearest": dict(size=[24, 24, 24], decompositions=[[1, 1, 1], [1, 2, 1]],
                    camera=test_camera(24, (64, 48)), interp=False,
                    sources=[src("random7", rng=(0.0, 1.0), tf=COOL_TF)], active=[0]),
    "multi": dict(size=[32, 32, 32], decompositions=[[1, 1, 1], [2, 1, 1], [2, 2, 2]],
                  camera=harness_camera(32, (96, 54)),
                  sources=[src("smooth", rng=(0.0, 2.4), tf=WARM_TF, mode="iso", iso=1.9),
                           src("vector", chain="length | mul(2) | add(0.1)", rng=(0.0, 3.0), tf=COOL_TF),
                           src("random", rng=(0.0, 1.0))],
                  active=[0, 1]),
    "iso_face": dict(size=[16, 16, 16], decompositions=[[1, 1, 1], [2, 1, 1]],
                     camera=test_camera(16, (64, 36)),
                     sources=[src("linear_x", rng=(0.0, 24.0), mode="iso", iso=8.0)], active=[0]),
    "iso_sphere": dict(size=[16, 16, 16], decompositions=[[1, 1, 1], [2, 1, 1]],
                       camera=test_camera(16, (64, 36)),
                       sources=[src("sphere_l", rng=(0.0, 24.0), tf=WARM_TF, mode="iso", iso=4.0)],
                       active=[0]),
    "early": dict(size=[32, 32, 32], decompositions=[[1, 1, 1]], camera=harness_camera(32, (64, 64)),
                  alpha_stop=0.9, sources=[src("random", rng=(0.0, 1.0))], active=[0]),
    "noguard": dict(size=[24, 24, 24], decompositions=[[1, 1, 1], [2, 1, 1]],
                    camera=test_camera(24, (64, 40)),
                    sources=[src("smooth", rng=(0.0, 2.4), has_guard=False)], active=[0]),
    "pow_nan": dict(size=[24, 24, 24], decompositions=[[1, 1, 1]], camera=test_camera(24, (48, 32)),
                    sources=[src("random", chain="add(-0.5) | pow(0.5) | mul(2)", rng=(0.0, 1.0),
                                 tf=WARM_TF)], active=[0]),
    "axis_odd": dict(size=[16, 16, 16], decompositions=[[1, 1, 1], [1, 1, 2]],
                     camera={"position": [8.0, 8.0, -40.0], "look_at": [8.0, 8.0, 8.0],
                             "up": [0.0, 1.0, 0.0], "vertical_fov": math.radians(30.0),
                             "image_size": [33, 17]},
                     sources=[src("smooth", rng=(0.0, 2.4))], active=[0]),
    "inside": dict(size=[24, 24, 24], decompositions=[[1, 1, 1], [2, 2, 1]],
                   camera={"position": [12.3, 11.8, 12.1], "look_at": [0.0, 3.0, 24.0],
                           "up": [0.0, 1.0, 0.0], "vertical_fov": math.radians(60.0),
                           "image_size": [48, 36]},
                   sources=[src("random", rng=(0.0, 1.0), tf=WARM_TF)], active=[0]),
    "vec_iso_multi": dict(size=[16, 16, 16], decompositions=[[1, 1, 1], [2, 2, 2]],
                          camera=harness_camera(16, (40, 30)), step=0.37,
                          sources=[src("random_vec3", chain="sum", rng=(0.0, 3.0), tf=WARM_TF),
                                   src("sphere_c", rng=(0.0, 24.0), tf=COOL_TF, mode="iso", iso=20.0)],
                          active=[0, 1]),
    # single float3 source in volume mode (the paired vector march): LUT and
    # analytic (single-ramp) classification
    "vec_volume": dict(size=[24, 24, 24], decompositions=[[1, 1, 1], [2, 1, 1]],
                       camera=harness_camera(24, (48, 32)),
                       sources=[src("vector", chain="length | mul(2) | add(0.1)", rng=(0.0, 3.0), tf=COOL_TF)],
                       active=[0]),
    "vec_linear": dict(size=[20, 20, 20], decompositions=[[1, 1, 1], [1, 2, 1]],
                       camera=test_camera(20, (40, 30)),
                       sources=[src("random_vec3", chain="sum", rng=(0.0, 3.0))], active=[0]),
}

DEFAULTS = dict(step=0.5, alpha_stop=1.0, interp=True, planes=[], guard=1)


def case(name):
    c = dict(DEFAULTS)
    c.update(RENDER_CASES[name])
    return c


COMPOSITE_CASES = {
    "swap2": dict(ranks=2, shape=[13, 9], seed=102),
    "swap4": dict(ranks=4, shape=[13, 9], seed=104),
    "swap8": dict(ranks=8, shape=[16, 16], seed=108),
    "swap16": dict(ranks=16, shape=[13, 9], seed=116),
    "direct3": dict(ranks=3, shape=[6, 7], seed=203),
    "direct6": dict(ranks=6, shape=[6, 7], seed=206),
}
