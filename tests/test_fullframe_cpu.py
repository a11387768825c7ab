"""The whole-frame CPU renderer of the full-size GPU parity tests
(tests/fullframe_cpu.py) agrees with itself across its two back ends: the
reference (baseline/_ref) and the oracle port give identical images and
per-pixel station counts on a small multi-source frame with an iso surface,
a float3 chain and a clip plane.  Skipped when baseline/_ref is absent."""

import numpy as np
import pytest

from fullframe_cpu import reference_available, render_frame


@pytest.mark.skipif(not reference_available(), reason="reference not installed in baseline/_ref")
def test_reference_and_oracle_frames_agree():
    n = 24
    rng = np.random.default_rng(0)
    z, y, x = np.meshgrid(*(np.arange(-1, n + 1, dtype=np.float64),) * 3, indexing="ij")
    s = np.sqrt((x - n / 2) ** 2 + (y - n / 2 + 0.3) ** 2 + (z - n / 2) ** 2).astype(np.float32)
    v = rng.random((n + 2, n + 2, n + 2, 3)).astype(np.float32)
    srcs = [dict(array=s, dim=1, tf=[(0, 0, 0, 0, 0), (1, 1, 1, 1, 1)], range=(0, 20.0), mode="iso", iso=7.0),
            dict(array=v, dim=3, tf=[(0, 0, 0, 0, 0), (0.6, 0.1, 0.7, 0.4, 0.3), (1, 0.7, 1, 0.9, 0.8)],
                 range=(0, 6.0), chain="length | mul(2) | add(0.1)")]
    cam = dict(position=(35.0, 31.0, -22.0), look_at=(12.0, 12.0, 12.0), size=(48, 36))
    planes = [((12, 12, 12), (0.3, -0.5, 0.81))]
    a, ca, ka = render_frame(srcs, cam, n=n, planes=planes, cores=2)
    b, cb, kb = render_frame(srcs, cam, n=n, planes=planes, cores=2, prefer="oracle")
    assert (ka, kb) == ("reference", "oracle")
    assert np.abs(a - b).max() <= 1e-12
    assert np.array_equal(ca, cb) and ca.sum() > 1000
