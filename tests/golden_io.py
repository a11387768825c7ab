"""Loading helpers for the committed golden vectors (tests/golden/)."""

from __future__ import annotations

import json
import os
import sys

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
if GOLDEN not in sys.path:
    sys.path.insert(0, GOLDEN)

import cases  # noqa: E402
import fields as gfields  # noqa: E402


def manifest():
    with open(os.path.join(GOLDEN, "manifest.json")) as fh:
        return json.load(fh)


def load(fname):
    with np.load(os.path.join(GOLDEN, fname)) as z:
        return {k: z[k] for k in z.files}


def decomp_key(decomp):
    return "d" + "".join(str(v) for v in decomp)


def brick_of(size, decomp, rank):
    dx, dy, dz = decomp
    bx, by, bz = rank % dx, (rank // dx) % dy, rank // (dx * dy)
    lsize = (size[0] // dx, size[1] // dy, size[2] // dz)
    return (bx * lsize[0], by * lsize[1], bz * lsize[2]), lsize
