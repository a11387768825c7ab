"""Per-pixel station counts of the C3 frame (for warp-utilisation models)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1611_09048_b200 as P  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
n = cfg["n"]
vol = P.GlobalVolume((n,) * 3)
dom = vol.local_domain(0, 1)
reg = P.SourceRegistry(dom)
reg.register_handle(P.array_backed_handle(P.SourceDescriptor("s", 1, has_guard=True),
                                          bench.make_field_torch(n, dom, "cuda"), 1))
active = {0}
if cfg.get("multi"):
    reg.register_handle(P.array_backed_handle(P.SourceDescriptor("v", 3, has_guard=True),
                                              bench.make_vector_field_torch(n, dom, "cuda"), 1))
    active = {0, 1}
P.update_sources(reg, active, {})
fr = P.default_registry()
img = P.render_local(P.RankContext(vol, dom, reg, fr, fr.limits), bench.build_scene(P, cfg), keep_station_counts=True,
                     keep_krange=True)
w, h = cfg["image"]
kr = img.krange.cpu().numpy()
np.savez_compressed(os.path.join(ROOT, "gpurun_out", f"counts_{sys.argv[1] if len(sys.argv) > 1 else 'c3'}.npz"),
                    stations=img.station_counts.cpu().numpy().reshape(h, w), k_lo=kr[:, 0].reshape(h, w),
                    k_hi=kr[:, 1].reshape(h, w))
print("ok", img.stations)
