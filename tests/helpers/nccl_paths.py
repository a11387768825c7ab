"""torchrun --nproc-per-node 1 on one GPU: the NCCL-backed code paths that
multi-GPU runs take -- normalize.reduce_range (MIN/MAX all-reduce on device
tensors), TorchDistTransport (a gloo side group under an NCCL default group)
carrying NvlinkTransport's arena exchange, binary_swap at world size 1.
Prints one JSON line."""
import json
import math
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import paper_1611_09048_b200 as P  # noqa: E402

torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
assert dist.get_backend() == "nccl"
rng = np.random.default_rng(3)
arr = rng.standard_normal((10, 9, 12)).astype(np.float32)
dom = P.LocalDomain((0, 0, 0), (10, 7, 8), 1)
h = P.array_backed_handle(P.SourceDescriptor("v", 1, has_guard=True), torch.from_numpy(arr).cuda(), 1)
ch = P.parse_chain("", P.default_registry(), input_dim=1)
local = P.value_range(h, dom, ch)
reduced = P.value_range(h, dom, ch, group=True)
from paper_1611_09048_b200.normalize import reduce_range  # noqa: E402
empty = reduce_range(math.nan, math.nan, group=True)
t = P.NvlinkTransport(P.TorchDistTransport(), 6 * 4)
img = torch.rand((4, 6, 4), device="cuda")
out = P.binary_swap(t, img, [0])
dist.barrier()
print(json.dumps({"local": list(local), "reduced": list(reduced), "empty_is_nan": all(math.isnan(v) for v in empty),
                  "swap_equal": bool(torch.equal(out, img))}))
t.close()
dist.destroy_process_group()
