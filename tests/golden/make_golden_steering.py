"""Golden vectors for the steering fold: the REAL reference's
``insitu.runtime.apply_steering`` (runtime.py:111-184) over seeded random
message sequences (valid, malformed JSON, non-objects, unknown actions,
missing / mistyped fields, control actions).

Run in the build container only:  ``python tests/golden/make_golden_steering.py``
-> ``tests/golden/steering.json`` (committed; read by tests/test_host_api.py).
"""

from __future__ import annotations

import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from insitu import runtime as rt  # noqa: E402
from insitu import scene as rs  # noqa: E402


def random_message(rng: random.Random):
    kind = rng.randrange(16)
    sid = rng.randrange(3)
    if kind == 0:
        return "{not json"
    if kind == 1:
        return rng.choice([7, [1, 2], None, "[]"])
    if kind == 2:
        return {"action": rng.choice(["pause", "resume", "step", "exit"]), "n": rng.randrange(5)}
    if kind == 3:
        return {"action": "frobnicate"}
    if kind == 4:
        return json.dumps({"action": "set_period", "value": rng.choice([0, 1, 3, "4", "x"])})
    if kind == 5:
        return {"action": "set_active_sources", "ids": rng.sample([0, 1, 2], rng.randrange(1, 4))}
    if kind == 6:
        return {"action": "set_functor_chain", "source_id": sid, "text": rng.choice(["", "mul(2)", "length | add(1)"])}
    if kind == 7:
        pts = [[0.0, rng.random(), rng.random(), rng.random(), rng.random()],
               [1.0, rng.random(), rng.random(), rng.random(), rng.random()]]
        return {"action": "set_transfer_function", "source_id": sid, "points": pts}
    if kind == 8:
        return {"action": "set_range", "source_id": sid, "min": rng.uniform(-1, 0), "max": rng.uniform(1, 2)}
    if kind == 9:
        return {"action": "set_range", "source_id": sid, "min": "low"}
    if kind == 10:
        m = {"action": "set_camera"}
        if rng.random() < 0.7:
            m["position"] = [rng.uniform(-50, 50) for _ in range(3)]
        if rng.random() < 0.5:
            m["look_at"] = [rng.uniform(0, 10) for _ in range(3)]
        if rng.random() < 0.3:
            m["vertical_fov"] = rng.uniform(0.3, 1.3)
        return json.dumps(m)
    if kind == 11:
        return {"action": "set_clip_planes", "planes": [{"point": [rng.random() * 10 for _ in range(3)],
                                                         "normal": [rng.uniform(-1, 1) for _ in range(3)]}
                                                        for _ in range(rng.randrange(3))]}
    if kind == 12:
        return {"action": "set_interpolation", "value": rng.random() < 0.5}
    if kind == 13:
        return {"action": "set_functor_chain", "text": "mul(2)"}         # missing source_id
    if kind == 14:
        return b'{"action": "set_period", "value": 2}'
    return {"action": "set_clip_planes", "planes": [{"point": [0, 0]}]}   # malformed plane


def base_scene():
    return rs.SceneState(camera=rs.Camera(position=(40.0, 30.0, -20.0), look_at=(8.0, 8.0, 8.0), image_size=(64, 48)),
                         tf_points={0: [(0.0, 0, 0, 0, 0), (1.0, 1, 1, 1, 1)]}, value_ranges={0: (0.0, 1.0)},
                         chain_texts={0: ""})


def main():
    rng = random.Random(11)
    cases = []
    for _ in range(60):
        msgs = [random_message(rng) for _ in range(rng.randrange(0, 9))]
        res = rt.apply_steering(base_scene(), msgs)
        enc = [m.decode() if isinstance(m, bytes) else m for m in msgs]
        cases.append({"messages": enc, "bytes": [isinstance(m, bytes) for m in msgs],
                      "scene": res.scene.to_json(), "controls": res.controls, "dropped": res.dropped,
                      "unknown": res.unknown})
    with open(os.path.join(HERE, "steering.json"), "w") as fh:
        json.dump({"base": base_scene().to_json(), "cases": cases}, fh, indent=0)
    print(f"wrote steering.json ({len(cases)} cases)")


if __name__ == "__main__":
    main()
