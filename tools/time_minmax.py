"""Time the normalisation kernel (isc_value_range) on a BASELINE config's
field: python tools/time_minmax.py [--config c2] (ISC_LIB_PATH for A/B)."""
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
    ap.add_argument("--config", default="c2")
    args = ap.parse_args()
    n = bench.CONFIGS[args.config]["n"]
    dom = P.GlobalVolume((n,) * 3).local_domain(0, 1)
    reg = P.SourceRegistry(dom)
    reg.register_handle(P.array_backed_handle(P.SourceDescriptor("density", 1, has_guard=True),
                                              bench.make_field_torch(n, dom, "cuda"), 1))
    P.update_sources(reg, {0}, {})
    res = bench.time_normalisation(P, torch, reg, dom, bench.peak_hbm()[0], reps=20)
    res["lib"] = os.environ.get("ISC_LIB_PATH", "default")
    res["config"] = args.config
    print(json.dumps(res))


if __name__ == "__main__":
    main()
