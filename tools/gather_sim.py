"""Gather-footprint model of the march kernels on the C4 view (numpy, no GPU).

For a warp's 32 samples laid out as (rays across x) x (rays across y) x
(consecutive stations per ray), counts per trilinear corner request:
  * distinct 32-byte sectors of the (z, y, x) float32 field (what one LDG
    request makes the L1 process; ~4 sectors per L1 wavefront measured), and
  * shared-memory wavefronts (worst bank multiplicity) if the same corners
    were read from a brick staged in shared memory,
and, for the staging alternative, the floats a CTA would have to stage per
sample for an axis-aligned box around a screen tile's rays over a chunk of
stations.  Used in DESIGN.md to choose the warp shape and to argue against
box staging for oblique views.

    python tools/gather_sim.py
"""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import isaac_oracle as O  # noqa: E402

N, W, H = 1024, 1920, 1080
PITCH = N + 2


def setup():
    diag = math.sqrt(3 * N * N)
    pos = np.array((N * 1.4, N * 1.15, -0.8 * diag))
    dirs = O.primary_rays(tuple(pos), (N / 2,) * 3, (0.0, 1.0, 0.0), math.radians(45.0), W, H).reshape(H, W, 3)
    ti, to = O.slab(pos, dirs.reshape(-1, 3), np.zeros(3), np.full(3, float(N)))
    return pos, dirs, ti.reshape(H, W), to.reshape(H, W)


def warp_points(pos, dirs, px, py, k, tw, th, ns):
    pts = [pos + ((k + s) * 0.5) * dirs[py + j, px + i] for j in range(th) for i in range(tw) for s in range(ns)]
    return np.array(pts)


def main(trials=300):
    pos, dirs, ti, to = setup()
    rng = np.random.default_rng(0)
    print("warp shape (rays x, rays y, stations)   sectors/request   smem wavefronts/request (row pad 40)")
    for shape in ((8, 2, 2), (8, 4, 1), (16, 2, 1), (4, 4, 2), (8, 1, 4), (4, 2, 4), (4, 1, 8)):
        secs, banks = [], []
        for _ in range(trials):
            py, px = rng.integers(300, 700), rng.integers(700, 1200)
            k = int((ti[py, px] + to[py, px]) / 2 / 0.5)
            c = np.floor(warp_points(pos, dirs, px, py, k, *shape)).astype(np.int64)
            lo = c.min(0)
            for dz in (0, 1):
                for dy in (0, 1):
                    for dx in (0, 1):
                        cc = c + np.array([dx, dy, dz])
                        addr = (cc[:, 2] * PITCH + cc[:, 1]) * PITCH + cc[:, 0] + PITCH * PITCH + PITCH + 1
                        secs.append(len(np.unique(addr // 8)))
                        sa = np.unique(((cc[:, 2] - lo[2]) * 64 + (cc[:, 1] - lo[1])) * 40 + (cc[:, 0] - lo[0]))
                        banks.append(np.bincount(sa % 32, minlength=32).max())
        print(f"{str(shape):40s} {np.mean(secs):8.2f}          {np.mean(banks):8.2f}")
    print("\nbox staging: floats staged per sample (tile of rays, chunk of stations, AABB of the chunk)")
    for tile, chunk in ((8, 16), (8, 32), (16, 32), (16, 64)):
        per = []
        for _ in range(trials // 10):
            py, px = rng.integers(300, 700), rng.integers(700, 1200)
            k = int((ti[py, px] + to[py, px]) / 2 / 0.5)
            pts = np.concatenate([warp_points(pos, dirs, px, py, k, tile, tile, 1),
                                  warp_points(pos, dirs, px, py, k + chunk, tile, tile, 1)])
            ext = np.floor(pts.max(0)) - np.floor(pts.min(0)) + 2
            per.append(float(np.prod(ext)) / (tile * tile * chunk))
        print(f"tile {tile}x{tile}, {chunk} stations: {np.mean(per):6.1f} floats/sample "
              f"({4 * np.mean(per):5.1f} B/sample through L2)")


if __name__ == "__main__":
    main()
