"""C5 weak-scaling prediction from ONE B200: 512^3 float32 per GPU, bricks
(1,1,1) / (2,1,1) / (2,2,1) / (2,2,2), 3840x2160, the 26-direction camera
orbit of bench.py.  Every brick of every N is rendered on
this GPU for every orbit view (its own contiguous field, as bench.py
allocates it per rank); per view the predicted N-GPU frame time is the
slowest brick plus the modelled binary-swap cost, and weak-scaling
efficiency is reported two ways: T_1 / T_N (the frame time as GPUs and
volume grow together at a fixed 4K image; the rays get longer, the screen
share of a brick shrinks) and the throughput efficiency (samples/s of N GPUs
over N x the 1-GPU samples/s; 1.0 = linear).

Swap model (per rank, 16 B/px float32 RGBA, binary swap): a rank pulls
n/2 + n/4 + ... = n(1 - 1/N) pixels over NVLink and stores its final n/N
span into rank 0's frame; at the --nvlink-gbps per-direction rate plus
log2(N) flag hand-offs of --handoff-us each.  Launch-shape trials are off
(ISC_DISABLE_TUNE), as for the orbit in bench.py (no view repeats).

    python tools/weak_scaling.py [--reps 3] [--nvlink-gbps 750] [--views 26]
"""
import argparse
import json
import math
import os
import sys

os.environ.setdefault("ISC_DISABLE_TUNE", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1611_09048_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--views", type=int, default=26)
    ap.add_argument("--nvlink-gbps", type=float, default=750.0)
    ap.add_argument("--handoff-us", type=float, default=3.0)
    ap.add_argument("--gpus", default="1,2,4,8")
    args = ap.parse_args()
    cfg = bench.CONFIGS["c5"]
    w, h = cfg["image"]
    out = torch.empty((h, w, 4), dtype=torch.float32, device="cuda")
    report = {"config": "c5", "image": [w, h], "per_gpu_volume": [cfg["n"]] * 3, "nvlink_gbps": args.nvlink_gbps,
              "handoff_us": args.handoff_us, "runs": []}
    base = None
    for N in [int(v) for v in args.gpus.split(",")]:
        decomp = bench.DECOMP[N]
        size = tuple(cfg["n"] * decomp[a] for a in range(3))
        n = size[0]
        vol = P.GlobalVolume(size, decomp)
        scene0 = bench.build_scene(P, cfg, n)
        views = [bench.orbit_scene(P, scene0, n, d) for d in bench.ORBIT[: args.views]]
        per_view = [[0.0] * N for _ in views]
        stations = [[0] * N for _ in views]
        for r in range(N):
            dom = vol.local_domain(r, 1)
            field = bench.make_field_torch(n, dom, "cuda")
            reg = P.SourceRegistry(dom)
            reg.register_handle(P.array_backed_handle(P.SourceDescriptor("density", 1, has_guard=True), field, 1))
            P.update_sources(reg, {0}, {})
            fr = P.default_registry()
            ctx = P.RankContext(vol, dom, reg, fr, fr.limits)
            for vi, sc in enumerate(views):
                plans = P.build_plans(reg, fr, fr.limits, sc)
                img = P.render_local(ctx, sc, plans=plans, out=out, check_errors=False)
                evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                       for _ in range(args.reps)]
                for e in evs:
                    P.render_local(ctx, sc, plans=plans, out=out, check_errors=False, events=e)
                torch.cuda.synchronize()
                per_view[vi][r] = sorted(a.elapsed_time(b) for a, b in evs)[args.reps // 2]
                stations[vi][r] = int(img.stations)
            del field, reg, ctx
            torch.cuda.empty_cache()
        npx = w * h
        swap_ms = 0.0
        if N > 1:
            pulled = npx * (1.0 - 1.0 / N) * 16 + npx / N * 16
            swap_ms = pulled / (args.nvlink_gbps * 1e9) * 1e3 + math.log2(N) * args.handoff_us * 1e-3
        frame = [max(t) + swap_ms for t in per_view]
        mean_brick = [sum(t) / N for t in per_view]
        t_mean = sum(frame) / len(frame)
        run = {"n_gpus": N, "decomposition": list(decomp), "volume": list(size),
               "frame_ms_mean": round(t_mean, 4), "frame_ms_worst_view": round(max(frame), 4),
               "render_max_brick_ms_mean": round(sum(max(t) for t in per_view) / len(per_view), 4),
               "imbalance_mean": round(sum(max(t) / m for t, m in zip(per_view, mean_brick)) / len(per_view), 3),
               "swap_ms_model": round(swap_ms, 4),
               "swap_share_of_frame": round(swap_ms / t_mean, 4),
               "samples_per_frame_mean": int(sum(sum(s) for s in stations) / len(stations)),
               "frames_per_s": round(1000.0 / t_mean, 2)}
        rate = run["samples_per_frame_mean"] / t_mean
        if base is None:
            base = (t_mean, rate)
        run["frame_time_ratio_1_over_n"] = round(base[0] / t_mean, 4)
        # samples/s of N GPUs over N x the 1-GPU samples/s: the per-GPU
        # throughput kept at scale (1.0 = linear)
        run["throughput_efficiency"] = round(rate / (N * base[1]), 4)
        report["runs"].append(run)
        print(json.dumps(run), flush=True)
    print(json.dumps(report))


if __name__ == "__main__":
    main()
