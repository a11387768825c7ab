"""Run under torchrun with every rank on cuda:0 (one GPU): the real
process-per-rank path -- gloo host transport, CUDA IPC arena exchange,
fused peer-memory binary swap / direct send -- against a reference golden.
Ranks time-share the GPU, so spin-waits rely on context time-slicing.
Rank 0 prints one JSON line."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))
import paper_1611_09048_b200 as P  # noqa: E402
from golden_io import load  # noqa: E402

name = sys.argv[1]
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
gold = load(f"composite_{name}.npz")
assert len(gold["images"]) == world, (name, world)
order = [int(v) for v in gold["order"]]
img = torch.from_numpy(gold["images"][rank].astype(np.float32)).cuda()
h, w = img.shape[:2]
host = P.TorchDistTransport()
t = P.NvlinkTransport(host, h * w)
t.timeout_s = 60.0
errs = []
for e in range(epochs):
    out = P.binary_swap(t, img, order)
    if rank == 0:
        errs.append(float(np.abs(out.cpu().numpy() - gold["result"]).max()))
    else:
        assert out is None
dist.barrier()
t.close()
if rank == 0:
    print(json.dumps({"name": name, "world": world, "max_err": max(errs), "epochs": epochs,
                      "sent": t.sent_bytes, "received": t.received_bytes}))
dist.destroy_process_group()
