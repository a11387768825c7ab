"""Time the march kernel alone (CUDA events, field resident) for one BASELINE
config: python tools/time_march.py [--config c4] [--reps 20].  With
ISC_LIB_PATH set it times that library build (A/B experiments)."""
import argparse
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1611_09048_b200 as P  # noqa: E402
from paper_1611_09048_b200.raycast import describe_kernel  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--lut", action="store_true", help="force the shared-memory LUT path")
    ap.add_argument("--alpha", type=float, default=None, help="early_termination_alpha (default: the config's 1.0)")
    ap.add_argument("--opacity", type=float, default=None, help="scale the transfer function's alpha ramp")
    ap.add_argument("--dtype", default="float32", help="field element type (float32, float16, bfloat16)")
    ap.add_argument("--points", default=None, help="transfer-function control points of source 0 as JSON, "
                                                   "e.g. '[[0,0,0,0,0],[0.37,1,0.5,0.2,0.4],[1,1,1,1,1]]'")
    ap.add_argument("--volume-only", action="store_true", help="every source in volume mode (no iso)")
    ap.add_argument("--active", default=None, help="comma-separated source ids to render (C3: 0 = iso scalar, "
                                                   "1 = float3 chain)")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    n = cfg["n"]
    vol = P.GlobalVolume((n,) * 3, (1, 1, 1))
    dom = vol.local_domain(0, 1)
    field = bench.make_field_torch(n, dom, "cuda")
    if args.dtype != "float32":
        field = field.to(getattr(torch, args.dtype))
    reg = P.SourceRegistry(dom)
    reg.register_handle(P.array_backed_handle(P.SourceDescriptor("density", 1, has_guard=True), field, 1))
    active = {0}
    if cfg.get("multi"):
        reg.register_handle(P.array_backed_handle(P.SourceDescriptor("velocity", 3, has_guard=True),
                                                  bench.make_vector_field_torch(n, dom, "cuda"), 1))
        active = {0, 1}
    P.update_sources(reg, active, {})
    fr = P.default_registry()
    ctx = P.RankContext(vol, dom, reg, fr, fr.limits)
    scene = bench.build_scene(P, cfg)
    if args.opacity is not None:
        pts = {k: [(p[0], p[1], p[2], p[3], p[4] * args.opacity) for p in v] for k, v in scene.tf_points.items()}
        scene = P.SceneState(camera=scene.camera, tf_points=pts, value_ranges=scene.value_ranges,
                             chain_texts=scene.chain_texts, clip_planes=scene.clip_planes, settings=scene.settings)
    if args.volume_only:
        import dataclasses
        scene = P.SceneState(camera=scene.camera, tf_points=scene.tf_points, value_ranges=scene.value_ranges,
                             chain_texts=scene.chain_texts, clip_planes=scene.clip_planes,
                             settings=dataclasses.replace(scene.settings, modes={}))
    if args.points is not None:
        pts = [tuple(float(v) for v in p) for p in json.loads(args.points)]
        scene = P.SceneState(camera=scene.camera, tf_points={**scene.tf_points, 0: pts},
                             value_ranges=scene.value_ranges, chain_texts=scene.chain_texts,
                             clip_planes=scene.clip_planes, settings=scene.settings)
    if args.active is not None:
        import dataclasses
        ids = tuple(int(v) for v in args.active.split(","))
        scene = P.SceneState(camera=scene.camera, tf_points=scene.tf_points, value_ranges=scene.value_ranges,
                             chain_texts=scene.chain_texts, clip_planes=scene.clip_planes,
                             settings=dataclasses.replace(scene.settings, active_set=ids))
    if args.alpha is not None:
        import dataclasses
        scene = P.SceneState(camera=scene.camera, tf_points=scene.tf_points, value_ranges=scene.value_ranges,
                             chain_texts=scene.chain_texts, clip_planes=scene.clip_planes,
                             settings=dataclasses.replace(scene.settings, early_termination_alpha=args.alpha))
    w, h = cfg["image"]
    out = torch.empty((h, w, 4), dtype=torch.float32, device="cuda")
    plans = P.build_plans(reg, fr, fr.limits, scene)
    kw = dict(plans=plans, out=out, check_errors=False)
    if args.lut:
        kw["analytic_lut"] = False
    for _ in range(3):
        img = P.render_local(ctx, scene, **kw)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.reps)]
    for e in evs:
        P.render_local(ctx, scene, events=e, **kw)
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in evs)
    res = {"lib": os.environ.get("ISC_LIB_PATH", "default"), "config": args.config, "alpha": args.alpha,
           "kernel": describe_kernel(plans, scene.settings, analytic_lut=not args.lut,
                                     image_size=scene.camera.image_size),
           "dtype": args.dtype,
           "median_ms": round(ms[len(ms) // 2], 4),
           "min_ms": round(ms[0], 4), "stations": int(img.stations)}
    chk = out.double().sum().item()
    res["checksum"] = round(chk, 3)
    res["digest"] = hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest()[:16]  # bit-identity across A/B builds
    print(json.dumps(res))


if __name__ == "__main__":
    main()
