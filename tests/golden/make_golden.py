"""Generate golden vectors by running the REAL reference (``/root/reference``).

Run in the build container only (the reference does not exist on the GPU
box):  ``python tests/golden/make_golden.py`` (all) or
``python tests/golden/make_golden.py --only name,name`` (render cases).  Outputs ``tests/golden/*.npz``
plus ``manifest.json``; those files are committed and are what the tests read.

Every array here comes out of the reference's own public or module-level
functions -- ``render_local`` over ``array_backed_handle`` registries,
``_ray_box_intervals`` / ``_apply_clip_planes`` for the ray setup,
``binary_swap`` over ``LocalFabric`` threads, ``eval_chain_array``,
``classify_array`` and ``tf_from_points``.
"""

from __future__ import annotations

import json
import os
import random
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, HERE)

from insitu import compositing as ref_comp  # noqa: E402
from insitu import fields as ref_fields  # noqa: E402
from insitu import functors as ref_fun  # noqa: E402
from insitu import raycast as ref_ray  # noqa: E402
from insitu import scene as ref_scene  # noqa: E402
from insitu.transport import LocalFabric  # noqa: E402

import cases  # noqa: E402
import fields as gfields  # noqa: E402


def build_scene(c):
    cam = c["camera"]
    srcs = c["sources"]
    camera = ref_scene.Camera(position=tuple(cam["position"]), look_at=tuple(cam["look_at"]),
                              up=tuple(cam["up"]), vertical_fov=cam["vertical_fov"],
                              image_size=tuple(cam["image_size"]))
    settings = ref_scene.RenderSettings(
        active_set=tuple(c["active"]),
        modes={i: s["mode"] for i, s in enumerate(srcs)},
        iso_thresholds={i: s["iso"] for i, s in enumerate(srcs)},
        interpolation=c["interp"], step_length=c["step"],
        early_termination_alpha=c["alpha_stop"])
    planes = tuple(ref_scene.clip_plane(p, n) for p, n in c["planes"])
    return ref_scene.SceneState(
        camera=camera,
        tf_points={i: [tuple(p) for p in s["tf_points"]] for i, s in enumerate(srcs)},
        value_ranges={i: tuple(s["range"]) for i, s in enumerate(srcs)},
        chain_texts={i: s["chain"] for i, s in enumerate(srcs)},
        settings=settings, clip_planes=planes)


def render_case(name):
    c = cases.case(name)
    scene = build_scene(c)
    g = c["guard"]
    size = tuple(c["size"])
    full = {i: gfields.make(s["field"], size, g) for i, s in enumerate(c["sources"])}
    out = {"planes_normalized": np.asarray([p.normal for p in scene.clip_planes]).reshape(-1, 3)}
    t0 = time.time()
    for decomp in c["decompositions"]:
        volume = ref_fields.GlobalVolume(size, tuple(decomp))
        key = "d" + "".join(str(v) for v in decomp)
        images = []
        for rank in range(volume.rank_count):
            domain = volume.local_domain(rank, g)
            registry = ref_fields.SourceRegistry(domain)
            for i, s in enumerate(c["sources"]):
                local, _, _ = gfields.brick_slice(full[i], size, decomp, rank, g)
                dim = 1 if local.ndim == 3 else local.shape[3]
                registry.register_handle(ref_fields.array_backed_handle(
                    ref_fields.SourceDescriptor(f"s{i}", dim, has_guard=s["has_guard"],
                                                persistent=True), local, g))

            class Ctx:
                pass

            ctx = Ctx()
            ctx.domain = domain
            ctx.global_volume = volume
            ctx.registry = registry
            ctx.functor_registry = ref_fun.default_registry()
            ctx.limits = ctx.functor_registry.limits
            ref_fields.update_sources(registry, set(c["active"]), {})
            w, h = scene.camera.image_size
            per_px = np.zeros(w * h, np.int64)

            def rec(k, pix, per_px=per_px):
                np.add.at(per_px, pix, 1)

            img = ref_ray.render_local(ctx, scene, station_recorder=rec)
            assert img.stations == per_px.sum()
            # Ray setup through the reference's own helpers (raycast.py:510-523).
            origin = np.asarray(scene.camera.position, dtype=np.float64)
            dirs = scene.camera.ray_directions()
            lo = np.asarray(domain.offset, dtype=np.float64)
            hi = lo + np.asarray(domain.size, dtype=np.float64)
            ti, to = ref_ray._ray_box_intervals(origin, dirs, lo, hi)
            ti, to = ref_ray._apply_clip_planes(origin, dirs, ti, to, scene.clip_planes)
            gi, go = ref_ray._ray_box_intervals(origin, dirs, np.zeros(3),
                                                np.asarray(volume.size, dtype=np.float64))
            gi, go = ref_ray._apply_clip_planes(origin, dirs, gi, go, scene.clip_planes)
            hit = (to > np.maximum(ti, 0.0)) & (to > 0.0)
            k = {n_: np.zeros(w * h, np.int64) for n_ in ("k_lo", "k_hi", "kg_lo", "kg_hi")}
            step = scene.settings.step_length
            r = np.nonzero(hit)[0]
            k["k_lo"][r] = np.ceil(np.maximum(ti[r], 0.0) / step)
            k["k_hi"][r] = np.ceil(np.maximum(to[r], 0.0) / step)
            k["kg_lo"][r] = np.ceil(np.maximum(gi[r], 0.0) / step)
            k["kg_hi"][r] = np.ceil(np.maximum(go[r], 0.0) / step)
            p = f"{key}_r{rank}_"
            out[p + "rgba"] = img.pixels
            out[p + "stations"] = per_px.astype(np.int32)
            out[p + "hit"] = hit
            out[p + "t_in"] = ti
            out[p + "t_out"] = to
            for n_, v in k.items():
                out[p + n_] = v.astype(np.int32)
            images.append(img.pixels)
        order = ref_comp.visibility_order(volume, scene.camera)
        out[key + "_order"] = np.asarray(order, np.int32)
        out[key + "_composite"] = ref_comp.composite_sequential(images, order)
    print(f"  {name}: {time.time() - t0:.1f}s", flush=True)
    return out


def random_premultiplied(rng, shape):
    a = rng.uniform(0.0, 1.0, tuple(shape) + (1,))
    c = rng.uniform(0.0, 1.0, tuple(shape) + (3,)) * a
    return np.concatenate([c, a], axis=-1)


def composite_case(name):
    c = cases.COMPOSITE_CASES[name]
    rng = np.random.default_rng(c["seed"])
    R = c["ranks"]
    images = [random_premultiplied(rng, c["shape"]) for _ in range(R)]
    order = [int(v) for v in rng.permutation(R)]
    fabric = LocalFabric(R)
    results = [None] * R

    def body(rank):
        results[rank] = ref_comp.binary_swap(fabric.endpoint(rank), images[rank], order)

    threads = [threading.Thread(target=body, args=(r,)) for r in range(R)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(60)
    return {"images": np.stack(images), "order": np.asarray(order, np.int32),
            "result": results[0], "sent": np.asarray(fabric.sent_bytes, np.int64),
            "received": np.asarray(fabric.received_bytes, np.int64),
            "sequential": ref_comp.composite_sequential(images, order)}


def chain_goldens(count=400, batch=6, seed=20161117):
    """Random chains in the reference tests' grammar (test_functors.py:134-158)."""
    reg = ref_fun.default_registry()
    rng = random.Random(seed)
    nrng = np.random.default_rng(seed)
    takes = {"add": True, "mul": True, "pow": True, "length": False, "sum": False}
    texts, dims, ins, outs, odims = [], [], [], [], []
    while len(texts) < count:
        dim = rng.randint(1, 4)
        parts = []
        cur = dim
        for _ in range(rng.randint(0, 5)):
            nm = rng.choice(sorted(takes))
            if takes[nm]:
                n_args = rng.choice([1, cur])
                parts.append(f"{nm}({','.join(str(round(rng.uniform(-2, 2), 3)) for _ in range(n_args))})")
            else:
                parts.append(nm)
                cur = 1
        text = " | ".join(parts)
        chain = ref_fun.parse_chain(text, reg, input_dim=dim)
        vals = np.round(nrng.uniform(-10, 10, (batch, dim)), 3)
        res = ref_fun.eval_chain_array(chain, vals)
        pad_in = np.full((batch, 4), np.nan)
        pad_in[:, :dim] = vals
        pad_out = np.full((batch, 4), np.nan)
        pad_out[:, :res.shape[1]] = res
        texts.append(text)
        dims.append(dim)
        odims.append(res.shape[1])
        ins.append(pad_in)
        outs.append(pad_out)
    return {"dims": np.asarray(dims, np.int32), "out_dims": np.asarray(odims, np.int32),
            "inputs": np.stack(ins), "outputs": np.stack(outs)}, texts


def classify_goldens(seed=99):
    rng = np.random.default_rng(seed)
    tfs = [cases.LINEAR_TF, cases.WARM_TF, cases.COOL_TF, [(0.5, 1.0, 0.0, 0.0, 0.7)], []]
    ranges = [(0.0, 1.0), (-2.0, 3.5), (10.0, 20.0), (0.0, 100.0), (-1e-3, 1e-3)]
    out = {}
    values = np.concatenate([rng.uniform(-5, 25, 2000), [np.nan, np.inf, -np.inf, 0.0, 1.0, 0.42, 42.0]])
    out["values"] = values
    for i, (pts, rg) in enumerate(zip(tfs, ranges)):
        tf = ref_scene.tf_from_points(pts, rg)
        out[f"lut{i}"] = tf.lut
        out[f"range{i}"] = np.asarray(rg)
        out[f"rgba{i}"] = ref_scene.classify_array(tf, values)
    return out, [[list(p) for p in t] for t in tfs]


def toy_goldens():
    """Reference harness fields (ToyState) and whole harness frames (run)."""
    from insitu import harness as H
    out = {}
    cfg = H.HarnessConfig(size=(24, 16, 20), ranks=(2, 1, 1), image_size=(40, 30))
    vol = cfg.volume()
    for rank in range(2):
        dom = vol.local_domain(rank, 1)
        st = H.ToyState(cfg, dom)
        for step in (0, 3):
            st.step_index = step
            st.refresh()
            st.fill_scratch()
            out[f"r{rank}_s{step}_density"] = st.density.copy()
            out[f"r{rank}_s{step}_velocity"] = st.velocity.copy()
            out[f"r{rank}_s{step}_scratch"] = st.scratch.copy()
    frames = {}
    run_cfg = H.HarnessConfig(size=(32, 32, 32), ranks=(2, 1, 1), steps=3, image_size=(72, 40),
                              active_sources=(0, 2))
    H.run(run_cfg, frame_hook=lambda step, img: frames.__setitem__(step, np.array(img)))
    for step, img in frames.items():
        out[f"frame_s{step}"] = img
    return out


def main():
    if len(sys.argv) > 2 and sys.argv[1] == "--only":
        # regenerate the named render cases only (manifest entries updated in place)
        with open(os.path.join(HERE, "manifest.json")) as fh:
            manifest = json.load(fh)
        for name in sys.argv[2].split(","):
            np.savez_compressed(os.path.join(HERE, f"render_{name}.npz"), **render_case(name))
            manifest["render"][name] = f"render_{name}.npz"
        with open(os.path.join(HERE, "manifest.json"), "w") as fh:
            json.dump(manifest, fh, indent=1)
        print("done")
        return
    manifest = {"reference": "/root/reference/pkg/src/insitu (insitu 0.1.0)",
                "numpy": np.__version__, "render": {}, "composite": {}}
    print("render cases:")
    for name in cases.RENDER_CASES:
        np.savez_compressed(os.path.join(HERE, f"render_{name}.npz"), **render_case(name))
        manifest["render"][name] = f"render_{name}.npz"
    print("composite cases:")
    for name in cases.COMPOSITE_CASES:
        np.savez_compressed(os.path.join(HERE, f"composite_{name}.npz"), **composite_case(name))
        manifest["composite"][name] = f"composite_{name}.npz"
    arrays, texts = chain_goldens()
    np.savez_compressed(os.path.join(HERE, "chains.npz"), **arrays)
    manifest["chains"] = {"file": "chains.npz", "texts": texts}
    arrays, tf_points = classify_goldens()
    np.savez_compressed(os.path.join(HERE, "classify.npz"), **arrays)
    manifest["classify"] = {"file": "classify.npz", "tf_points": tf_points}
    np.savez_compressed(os.path.join(HERE, "toy.npz"), **toy_goldens())
    manifest["toy"] = {"file": "toy.npz", "fields_config": {"size": [24, 16, 20], "ranks": [2, 1, 1]},
                       "run_config": {"size": [32, 32, 32], "ranks": [2, 1, 1], "steps": 3,
                                      "image_size": [72, 40], "active_sources": [0, 2]}}
    with open(os.path.join(HERE, "manifest.json"), "w") as fh:
        json.dump(manifest, fh, indent=1)
    print("done")


if __name__ == "__main__":
    main()
