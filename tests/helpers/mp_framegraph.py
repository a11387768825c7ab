"""Run under torchrun with every rank on cuda:0: each rank owns one brick of
a (world, 1, 1) decomposition and an NvlinkTransport (CUDA IPC arenas); a
static view is captured as a multi-rank FrameGraph (render + peer-memory
binary swap with the device-resident epoch) and replayed.  Rank 0 checks
every replayed frame against render_local + binary_swap (bit-identical),
including plain swaps interleaved after the replays (host and device epochs
must stay in step), and prints one JSON line."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
import paper_1611_09048_b200 as P  # noqa: E402

replays = int(sys.argv[1]) if len(sys.argv) > 1 else 5
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
n = 24
rng = np.random.default_rng(9)
full = rng.random((n + 2, n + 2, n * world + 2)).astype(np.float32)     # (z, y, x) with a 1-cell guard
vol = P.GlobalVolume((n * world, n, n), (world, 1, 1))
dom = vol.local_domain(rank, 1)
ox = dom.offset[0]
brick = torch.from_numpy(np.ascontiguousarray(full[:, :, ox:ox + n + 2])).cuda()
reg = P.SourceRegistry(dom)
reg.register_handle(P.array_backed_handle(P.SourceDescriptor("f", 1, has_guard=True), brick, 1))
P.update_sources(reg, {0}, {})
fr = P.default_registry()
w, h = 64, 40
t = P.NvlinkTransport(P.TorchDistTransport(), w * h)
t.timeout_s = 60.0
ctx = P.RankContext(vol, dom, reg, fr, fr.limits, t)
scene = P.SceneState(camera=P.Camera((n * world * 2.5, 41.0, -30.0), (n * world / 2.0, 12.0, 12.0), image_size=(w, h)),
                     tf_points={0: [(0.0, 0.0, 0.0, 0.0, 0.0), (1.0, 1.0, 0.5, 0.2, 0.6)]},
                     settings=P.RenderSettings(active_set=(0,), early_termination_alpha=1.0))
order = P.visibility_order(vol, scene.camera)


def plain():
    img = P.render_local(ctx, scene, out=t.canvas(h, w))
    out = P.binary_swap(t, img.pixels, order)
    return None if out is None else out.cpu().numpy()


want = plain()
g = P.FrameGraph(ctx, scene)
same = []
for i in range(replays):
    f = g.replay()
    if rank == 0:
        same.append(bool(np.array_equal(f.cpu().numpy(), want)))
    else:
        assert f is None
    if i == 1:   # a plain swap between replays: the epochs stay in step
        again = plain()
        if rank == 0:
            same.append(bool(np.array_equal(again, want)))
g.check()
after = plain()
t.flush()
dist.barrier()
if rank == 0:
    same.append(bool(np.array_equal(after, want)))
    print(json.dumps({"world": world, "replays": replays, "all_identical": all(same), "checks": len(same),
                      "epoch": t.epoch, "nonzero": float(np.abs(want).sum())}))
t.close()
dist.destroy_process_group()
