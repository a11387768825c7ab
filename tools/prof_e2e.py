"""Host profile of the bench e2e loop for one config (cProfile, top entries)."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1611_09048_b200 as P  # noqa: E402
from paper_1611_09048_b200.device import LUTS  # noqa: E402
from paper_1611_09048_b200.runtime import to_rgba8  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
n = cfg["n"]
vol = P.GlobalVolume((n,) * 3)
dom = vol.local_domain(0, 1)
reg = P.SourceRegistry(dom)
reg.register_handle(P.array_backed_handle(P.SourceDescriptor("d", 1, has_guard=True),
                                          bench.make_field_torch(n, dom, "cuda"), 1))
P.update_sources(reg, {0}, {})
fr = P.default_registry()
ctx = P.RankContext(vol, dom, reg, fr, fr.limits)
scene = bench.build_scene(P, cfg)
w, h = cfg["image"]
canvas = torch.empty((h, w, 4), device="cuda")
payload = scene.to_bytes()
tr = P.LocalFabric(1).endpoint(0)
order = P.visibility_order(vol, scene.camera)
host = torch.empty((h, w, 4), dtype=torch.uint8).pin_memory()


def one(clear=True, rgba8=True):
    sc = P.SceneState.from_bytes(payload)
    if clear:
        LUTS.clear()
    img = P.render_local(ctx, sc, out=canvas, check_errors=False)
    full = P.binary_swap(tr, img.pixels, order)
    if rgba8:
        host.copy_(to_rgba8(full), non_blocking=True)


for variant in [dict(), dict(clear=False), dict(rgba8=False)]:
    for _ in range(3):
        one(**variant)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        one(**variant)
    torch.cuda.synchronize()
    print(variant, "ms/frame", round((time.perf_counter() - t0) / 20 * 1e3, 3), flush=True)
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    one()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)

# the bench's own e2e loop on the same objects
import torch.distributed as dist  # noqa: E402
for steps in (10, 10):
    res = bench.run_e2e(P, torch, dist, ctx, scene, tr, canvas, order, 0, 1, torch.device("cpu"), steps)
    print("bench.run_e2e", res["ms_per_step"], flush=True)

# host-side cost of one bench step (render_local + binary_swap, no sync)
plans = P.build_plans(reg, fr, fr.limits, scene)
for _ in range(5):
    P.render_local(ctx, scene, plans=plans, out=canvas, check_errors=False)
torch.cuda.synchronize()
ts = []
for _ in range(50):
    t0 = time.perf_counter()
    img = P.render_local(ctx, scene, plans=plans, out=canvas, check_errors=False)
    full = P.binary_swap(tr, img.pixels, order)
    ts.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
ts.sort()
print("host us per step: median", round(ts[25] * 1e6, 1), "p90", round(ts[45] * 1e6, 1), flush=True)
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    img = P.render_local(ctx, scene, plans=plans, out=canvas, check_errors=False)
    full = P.binary_swap(tr, img.pixels, order)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
