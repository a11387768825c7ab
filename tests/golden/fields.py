"""Deterministic synthetic fields shared by the golden generator and the tests.

Only IEEE-exact numpy operations (+, -, *, PCG64 draws) are used, so the same
float32 arrays come out on any host -- the golden vectors made here in the
build container stay valid on the GPU box.
"""

from __future__ import annotations

import numpy as np


def lattice(size, guard, offset=(0, 0, 0)):
    """Global integer coordinates (z, y, x order) over a brick plus guard."""
    sx, sy, sz = size
    ox, oy, oz = offset
    z = np.arange(oz - guard, oz + sz + guard, dtype=np.float64)
    y = np.arange(oy - guard, oy + sy + guard, dtype=np.float64)
    x = np.arange(ox - guard, ox + sx + guard, dtype=np.float64)
    return np.meshgrid(z, y, x, indexing="ij")


def smooth(size, guard, n=None, offset=(0, 0, 0)):
    """Smooth polynomial bump in [~0, ~2.3] over the global volume of edge n."""
    z, y, x = lattice(size, guard, offset)
    n = float(n if n is not None else max(size))
    u, v, w = x / n, y / n, z / n
    f = 1.0 + 3.0 * (u * (1.0 - u)) * (1.0 + 0.5 * v) - 1.5 * (w - 0.5) * (w - 0.5) + 0.25 * u * v * w
    return f.astype(np.float32)


def random_field(size, guard, seed=0, dim=1):
    sx, sy, sz = size
    shape = (sz + 2 * guard, sy + 2 * guard, sx + 2 * guard) + ((dim,) if dim > 1 else ())
    return np.random.default_rng(seed).random(shape, dtype=np.float32)


def linear_x(size, guard, offset=(0, 0, 0)):
    z, y, x = lattice(size, guard, offset)
    return x.astype(np.float32)


def sphere(size, guard, center, offset=(0, 0, 0)):
    """Squared distance from ``center`` (exact in float64 for integer lattices)."""
    z, y, x = lattice(size, guard, offset)
    cx, cy, cz = center
    return ((x - cx) * (x - cx) + (y - cy) * (y - cy) + (z - cz) * (z - cz)).astype(np.float32)


def vector(size, guard, n=None, offset=(0, 0, 0)):
    """float3 field: three differently scaled copies of ``smooth``."""
    base = smooth(size, guard, n, offset).astype(np.float64)
    z, y, x = lattice(size, guard, offset)
    n = float(n if n is not None else max(size))
    out = np.stack([base - 1.0, 0.5 * base * (y / n), (x / n) - (z / n)], axis=-1)
    return out.astype(np.float32)


def brick_slice(full, size, decomposition, rank, guard):
    """The rank's (z, y, x[, d]) slice of a global-plus-guard array (x-fastest ranks)."""
    dx, dy, dz = decomposition
    bx, by, bz = rank % dx, (rank // dx) % dy, rank // (dx * dy)
    lx, ly, lz = size[0] // dx, size[1] // dy, size[2] // dz
    ox, oy, oz = bx * lx, by * ly, bz * lz
    g = guard
    return np.ascontiguousarray(full[oz:oz + lz + 2 * g, oy:oy + ly + 2 * g, ox:ox + lx + 2 * g]), \
        (ox, oy, oz), (lx, ly, lz)


MAKERS = {
    "smooth": lambda size, guard: smooth(size, guard),
    "random": lambda size, guard: random_field(size, guard, seed=0),
    "random7": lambda size, guard: random_field(size, guard, seed=7),
    "linear_x": lambda size, guard: linear_x(size, guard),
    "sphere_c": lambda size, guard: sphere(size, guard, (size[0] / 2 + 0.25, size[1] / 2, size[2] / 2)),
    "sphere_l": lambda size, guard: sphere(size, guard, (size[0] / 4 + 0.5, size[1] / 2, size[2] / 2)),
    "vector": lambda size, guard: vector(size, guard),
    "random_vec3": lambda size, guard: random_field(size, guard, seed=3, dim=3),
}


def make(name, size, guard=1):
    return MAKERS[name](tuple(size), guard)
