"""Per-brick march time of a BASELINE config decomposed as at N GPUs, all
bricks rendered one after another on ONE GPU (contiguous per-rank brick
arrays as bench.py allocates them, or --views: strided views of one field):
predicts the strong-scaling frame time (max over bricks) and its imbalance.

    python tools/brick_times.py [--config c4] [--n 8]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1611_09048_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--n", type=int, default=8)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--rank", type=int, default=-1, help="only this brick (for ncu)")
    ap.add_argument("--views", action="store_true", help="bricks as strided views of one field")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    n = cfg["n"]
    full_vol = P.GlobalVolume((n,) * 3)
    field = bench.make_field_torch(n, full_vol.local_domain(0, 1), "cuda")
    vol = P.GlobalVolume((n,) * 3, bench.DECOMP[args.n])
    scene = bench.build_scene(P, cfg)
    w, h = cfg["image"]
    out = torch.empty((h, w, 4), dtype=torch.float32, device="cuda")
    res = []
    for r in range(args.n):
        if args.rank >= 0 and r != args.rank:
            continue
        dom = vol.local_domain(r, 1)
        ox, oy, oz = dom.offset
        sx, sy, sz = dom.size
        view = field[oz:oz + sz + 2, oy:oy + sy + 2, ox:ox + sx + 2]
        if not args.views:      # as bench.py: each rank owns a contiguous brick array
            view = view.contiguous()
        reg = P.SourceRegistry(dom)
        reg.register_handle(P.array_backed_handle(P.SourceDescriptor("density", 1, has_guard=True), view, 1))
        P.update_sources(reg, {0}, {})
        fr = P.default_registry()
        ctx = P.RankContext(vol, dom, reg, fr, fr.limits)
        plans = P.build_plans(reg, fr, fr.limits, scene)
        for _ in range(5):      # the library's launch-shape choice: a repeat + up to three trials
            img = P.render_local(ctx, scene, plans=plans, out=out, check_errors=False)
            torch.cuda.synchronize()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.reps)]
        for e in evs:
            P.render_local(ctx, scene, plans=plans, out=out, check_errors=False, events=e)
        torch.cuda.synchronize()
        ms = sorted(a.elapsed_time(b) for a, b in evs)[args.reps // 2]
        res.append({"rank": r, "ms": round(ms, 4), "stations": int(img.stations)})
        del view, reg, ctx, plans
    mx = max(x["ms"] for x in res)
    mean = sum(x["ms"] for x in res) / len(res)
    print(json.dumps({"config": args.config, "n": args.n, "bricks": res, "max_ms": round(mx, 4),
                      "mean_ms": round(mean, 4), "imbalance": round(mx / mean, 3)}))


if __name__ == "__main__":
    main()
