"""Max errors of the CUDA path vs the reference goldens, per case (GPU)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1611_09048_b200 as P  # noqa: E402
from case_build import full_fields  # noqa: E402
from golden_io import cases, decomp_key, load  # noqa: E402
from product_build import product_ctx, product_scene  # noqa: E402

rows = []
for name in sorted(cases.RENDER_CASES):
    c = cases.case(name)
    gold = load(f"render_{name}.npz")
    scene = product_scene(c)
    full = full_fields(c)
    for decomp in c["decompositions"]:
        key = decomp_key(decomp)
        errs, st_mis, hit_mis, k_mis, npx = [], 0, 0, 0, 0
        for rank in range(int(np.prod(decomp))):
            p = f"{key}_r{rank}_"
            ctx = product_ctx(c, decomp, rank, full)
            rs = P.raycast.ray_setup(ctx, scene)
            hit = gold[p + "hit"]
            hit_mis += int((rs["hit"].cpu().numpy() != hit).sum())
            for k in ("k_lo", "k_hi", "kg_lo", "kg_hi"):
                k_mis += int((rs[k].cpu().numpy()[hit] != gold[p + k][hit]).sum())
            img = P.render_local(ctx, scene, keep_station_counts=True)
            errs.append(float(np.abs(img.pixels.cpu().numpy().astype(np.float64) - gold[p + "rgba"]).max()))
            st_mis += int((img.station_counts.cpu().numpy() != gold[p + "stations"]).sum())
            npx += hit.size
        rows.append({"case": name, "decomp": key, "max_abs_rgba": max(errs), "hit_mismatch": hit_mis,
                     "krange_mismatch": k_mis, "station_count_mismatch": st_mis, "pixels": npx})
        print(json.dumps(rows[-1]), flush=True)
