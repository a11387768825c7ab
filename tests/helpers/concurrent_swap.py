"""R virtual ranks on one GPU, one host thread + stream each, all swap kernels
live at once (the multi-GPU execution model).  Run with
CUDA_DEVICE_MAX_CONNECTIONS=32 so no two ranks' streams share a hardware queue
(on a real box each rank owns its GPU, so this aliasing cannot occur).
Prints one JSON line: max error vs the oracle fold and per-rank failures."""
import json
import os
import sys
import threading

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1611_09048_b200 as P  # noqa: E402
from oracle import isaac_oracle as O  # noqa: E402

R, epochs = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(R)
h, w = 37, 29
host = []
for _ in range(R):
    a = rng.uniform(0, 1, (h, w, 1))
    host.append(np.concatenate([rng.uniform(0, 1, (h, w, 3)) * a, a], axis=2))
order = [int(v) for v in rng.permutation(R)]
want = O.composite_in_order(host, order)
grp = P.LocalNvlinkGroup(R, h * w)
results, errors = [None] * R, []
# Everything that could cudaMalloc happens before any swap kernel spins: on
# ONE device a first-time allocation in one rank's thread may implicitly
# synchronise the device while another rank's kernel is waiting for it (with
# one GPU per process -- the real deployment -- that cannot couple ranks).
imgs = [torch.from_numpy(host[r].astype(np.float32)).cuda() for r in range(R)]
warm = [torch.empty((h, w, 4), device="cuda") for _ in range(4 * R)]
del warm
torch.cuda.synchronize()


def body(r):
    try:
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            ep = grp.endpoints[r]
            ep.n_ctas, ep.timeout_s = 2, 10.0
            img = imgs[r]
            for _ in range(epochs):
                out = P.binary_swap(ep, img, order)
            results[r] = None if out is None else out.cpu().numpy()
    except Exception as exc:  # noqa: BLE001
        errors.append(f"rank {r}: {exc}")


threads = [threading.Thread(target=body, args=(r,)) for r in range(R)]
for t in threads:
    t.start()
for t in threads:
    t.join(120)
err = float(np.abs(results[0] - want).max()) if results[0] is not None else None
print(json.dumps({"err": err, "errors": errors, "others_none": all(x is None for x in results[1:])}))
grp.close()
