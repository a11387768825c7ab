"""Build oracle inputs for a golden case (shared by CPU and GPU parity tests)."""

from __future__ import annotations

import numpy as np

from golden_io import brick_of, gfields
from oracle import isaac_oracle as O


def full_fields(c):
    return {i: gfields.make(s["field"], tuple(c["size"]), c["guard"]) for i, s in enumerate(c["sources"])}


def oracle_camera(c):
    cam = c["camera"]
    return {"position": cam["position"], "look_at": cam["look_at"], "up": cam["up"],
            "vertical_fov": cam["vertical_fov"], "width": cam["image_size"][0],
            "height": cam["image_size"][1]}


def oracle_sources(c, full, decomp, rank, planes_normal=None):
    size = tuple(c["size"])
    g = c["guard"]
    out = []
    for i in c["active"]:
        s = c["sources"][i]
        local, off, lsize = gfields.brick_slice(full[i], size, decomp, rank, g)
        dim = 1 if local.ndim == 3 else local.shape[3]
        out.append(O.Source(array=local, offset=off, size=lsize, guard=g, has_guard=s["has_guard"],
                            steps=O.parse_steps(s["chain"], dim), lut=O.lut_from_points(s["tf_points"]),
                            value_range=tuple(s["range"]), mode=s["mode"], iso_threshold=s["iso"]))
    return out


def oracle_planes(c, golden):
    normals = golden["planes_normalized"]
    return [(p, tuple(normals[j])) for j, (p, _) in enumerate(c["planes"])]


def oracle_render(c, golden, decomp, rank, recorder=None):
    full = full_fields(c)
    off, lsize = brick_of(c["size"], decomp, rank)
    brick = O.Brick(offset=off, size=lsize, guard=c["guard"], volume_size=tuple(c["size"]),
                    decomposition=tuple(decomp))
    return O.render_brick(oracle_camera(c), brick, oracle_sources(c, full, decomp, rank), step=c["step"],
                          alpha_stop=c["alpha_stop"], interp=c["interp"],
                          planes=oracle_planes(c, golden), recorder=recorder)
