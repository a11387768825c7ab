"""Whole-frame CPU renders for the full-size parity tests (test only).

The frame is split into interleaved row chunks rendered by one worker
process per host core (fork; workers only touch numpy).  Two renderers:

* ``"reference"`` -- the reference itself (insitu 0.1.0 pip-installed into
  baseline/_ref): render_local's body (raycast.py:508-541)
  on the chunk's rays, with the reference's station recorder for per-pixel
  station counts;
* ``"oracle"`` -- oracle/isaac_oracle.py render_rays (pinned to the
  reference by the committed goldens), when baseline/_ref is absent.

Returns the (H*W, 4) float64 RGBA, the (H*W,) per-pixel station counts and
the renderer used.
"""

from __future__ import annotations

import math
import multiprocessing as mp
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
_G: dict = {}


def reference_available() -> bool:
    if not os.path.isdir(os.path.join(REF, "insitu")):
        return False
    if REF not in sys.path:
        sys.path.insert(0, REF)
    try:
        import insitu.raycast  # noqa: F401
        return True
    except Exception:  # noqa: BLE001
        return False


def _setup_reference(sources, camera, settings, planes, n):
    import insitu.fields as rf
    import insitu.functors as rfn
    import insitu.raycast as rr
    import insitu.scene as rs
    vol = rf.GlobalVolume((n, n, n), (1, 1, 1))
    dom = vol.local_domain(0, 1)
    reg = rf.SourceRegistry(dom)
    for i, s in enumerate(sources):
        reg.register_handle(rf.array_backed_handle(rf.SourceDescriptor(f"s{i}", s["dim"], has_guard=True),
                                                   s["array"], 1))
    active = tuple(range(len(sources)))
    rf.update_sources(reg, set(active), {})
    scene = rs.SceneState(
        camera=rs.Camera(position=camera["position"], look_at=camera["look_at"], image_size=camera["size"]),
        tf_points={i: s["tf"] for i, s in enumerate(sources)},
        value_ranges={i: s["range"] for i, s in enumerate(sources)},
        chain_texts={i: s.get("chain", "") for i, s in enumerate(sources)},
        settings=rs.RenderSettings(active_set=active, modes={i: s.get("mode", "volume") for i, s in enumerate(sources)},
                                   iso_thresholds={i: s.get("iso", 0.5) for i, s in enumerate(sources)},
                                   interpolation=True, step_length=settings["step"],
                                   early_termination_alpha=settings["alpha_stop"]),
        clip_planes=tuple(rs.clip_plane(p, q) for p, q in planes))
    plans = rr.build_plans(reg, rfn.default_registry(), rfn.ChainLimits(), scene)
    origin = np.asarray(scene.camera.position, dtype=np.float64)
    _G.update(kind="reference", rr=rr, plans=plans, scene=scene, volume=vol, dom=dom, origin=origin,
              dirs=scene.camera.ray_directions())


def _setup_oracle(sources, camera, settings, planes, n):
    from oracle import isaac_oracle as O
    srcs = [O.Source(array=s["array"], offset=(0, 0, 0), size=(n, n, n), guard=1, lut=O.lut_from_points(s["tf"]),
                     value_range=s["range"], mode=s.get("mode", "volume"), iso_threshold=s.get("iso", 0.5),
                     steps=O.parse_steps(s["chain"], s["dim"]) if s.get("chain") else [])
            for s in sources]
    w, h = camera["size"]
    dirs = O.primary_rays(camera["position"], camera["look_at"], (0.0, 1.0, 0.0), math.radians(45.0), w, h)
    _G.update(kind="oracle", O=O, srcs=srcs, brick=O.Brick((0, 0, 0), (n, n, n), 1, (n, n, n)), dirs=dirs,
              origin=np.asarray(camera["position"], dtype=np.float64), planes=planes, settings=settings)


def _chunk(rows):
    w = _G["w"]
    sel = np.concatenate([np.arange(r * w, (r + 1) * w) for r in rows])
    dirs = _G["dirs"][sel]
    o = _G["origin"]
    if _G["kind"] == "oracle":
        st = _G["settings"]
        res = _G["O"].render_rays(o, dirs, _G["brick"], _G["srcs"], step=st["step"], alpha_stop=st["alpha_stop"],
                                  planes=_G["planes"])
        return sel, res.rgba, res.stations
    rr, scene, dom, vol = _G["rr"], _G["scene"], _G["dom"], _G["volume"]
    lo = np.asarray(dom.offset, np.float64)
    hi = lo + np.asarray(dom.size, np.float64)
    t0, t1 = rr._apply_clip_planes(o, dirs, *rr._ray_box_intervals(o, dirs, lo, hi), scene.clip_planes)
    g0, g1 = rr._apply_clip_planes(o, dirs, *rr._ray_box_intervals(o, dirs, np.zeros(3),
                                                                    np.asarray(vol.size, np.float64)),
                                   scene.clip_planes)
    hit = (t1 > np.maximum(t0, 0.0)) & (t1 > 0.0)
    idx = np.nonzero(hit)[0]
    rgba = np.zeros((sel.size, 4))
    counts = np.zeros(sel.size, dtype=np.int64)
    if idx.size:
        per = np.zeros(idx.size, dtype=np.int64)

        def rec(k, sub):
            np.add.at(per, sub, 1)

        out, _ = rr.march_rays(o, dirs[idx], (t0[idx], t1[idx]), (g0[idx], g1[idx]), _G["plans"],
                               scene.settings, rec, volume=vol)
        rgba[idx] = out
        counts[idx] = per
    return sel, rgba, counts


def render_frame(sources, camera, settings=None, planes=(), n=None, cores=None, prefer="reference"):
    settings = settings or {"step": 0.5, "alpha_stop": 1.0}
    w, h = camera["size"]
    kind = "reference" if prefer == "reference" and reference_available() else "oracle"
    (_setup_reference if kind == "reference" else _setup_oracle)(sources, camera, settings, planes, n)
    _G["w"] = w
    cores = cores or os.cpu_count() or 1
    parts = cores * 4
    chunks = [list(range(i, h, parts)) for i in range(parts) if i < h]
    rgba = np.zeros((w * h, 4))
    counts = np.zeros(w * h, dtype=np.int64)
    with mp.get_context("fork").Pool(cores) as pool:
        for sel, c_rgba, c_counts in pool.imap_unordered(_chunk, chunks):
            rgba[sel] = c_rgba
            counts[sel] = c_counts
    return rgba, counts, kind
