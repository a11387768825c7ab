"""Build product-side (paper_1611_09048_b200) rank contexts for a golden case."""

from __future__ import annotations

import paper_1611_09048_b200 as P
from case_build import full_fields
from golden_io import gfields


def product_scene(c):
    cam = c["camera"]
    srcs = c["sources"]
    return P.SceneState(
        camera=P.Camera(position=tuple(cam["position"]), look_at=tuple(cam["look_at"]), up=tuple(cam["up"]),
                        vertical_fov=cam["vertical_fov"], image_size=tuple(cam["image_size"])),
        tf_points={i: [tuple(p) for p in s["tf_points"]] for i, s in enumerate(srcs)},
        value_ranges={i: tuple(s["range"]) for i, s in enumerate(srcs)},
        chain_texts={i: s["chain"] for i, s in enumerate(srcs)},
        settings=P.RenderSettings(active_set=tuple(c["active"]),
                                  modes={i: s["mode"] for i, s in enumerate(srcs)},
                                  iso_thresholds={i: s["iso"] for i, s in enumerate(srcs)},
                                  interpolation=c["interp"], step_length=c["step"],
                                  early_termination_alpha=c["alpha_stop"]),
        clip_planes=tuple(P.clip_plane(p, n) for p, n in c["planes"]))


def product_ctx(c, decomp, rank, full=None, device="cuda"):
    import torch
    full = full if full is not None else full_fields(c)
    size = tuple(c["size"])
    g = c["guard"]
    volume = P.GlobalVolume(size, tuple(decomp))
    domain = volume.local_domain(rank, g)
    reg = P.SourceRegistry(domain)
    for i, s in enumerate(c["sources"]):
        local, _, _ = gfields.brick_slice(full[i], size, tuple(decomp), rank, g)
        dim = 1 if local.ndim == 3 else local.shape[3]
        t = torch.from_numpy(local).to(device)
        reg.register_handle(P.array_backed_handle(
            P.SourceDescriptor(f"s{i}", dim, has_guard=s["has_guard"], persistent=True), t, g))
    fr = P.default_registry()
    ctx = P.RankContext(global_volume=volume, domain=domain, registry=reg, functor_registry=fr,
                        limits=fr.limits)
    P.update_sources(reg, set(c["active"]), {})
    return ctx
