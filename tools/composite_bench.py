"""Microbenchmark of the fused binary-swap kernel on ONE GPU: R virtual ranks
(arenas in local HBM, launched stage by stage on one stream), 1080p and 4K.
This measures the kernel's memory efficiency; on a real box the partner
loads go over NVLink (770 GB/s measured per direction) instead of HBM."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1611_09048_b200 as P  # noqa: E402
from paper_1611_09048_b200.compositing import binary_swap_local, swap_schedule  # noqa: E402


def traffic(R, n):
    """HBM bytes the swap moves for all ranks (16 B/px): per round read own keep
    + partner keep span, write keep span; collect: read final span + write it."""
    tot = 0
    for v in range(R):
        plan, (lo, hi) = swap_schedule(v, R, n)
        for _, keep, _ in plan:
            tot += 3 * 16 * (keep[1] - keep[0])
        tot += 2 * 16 * (hi - lo)
    return tot


for (w, h) in ((1920, 1080), (3840, 2160)):
    for R in (2, 4, 8):
        imgs = [torch.rand((h, w, 4), device="cuda") * 0.5 for _ in range(R)]
        grp = P.LocalNvlinkGroup(R, w * h)
        order = list(range(R))[::-1]
        for _ in range(3):
            binary_swap_local(grp, imgs, order)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        a.record()
        for _ in range(reps):
            binary_swap_local(grp, imgs, order)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        tb = traffic(R, w * h)
        print(json.dumps({"image": [w, h], "ranks": R, "ms_all_ranks_sequential": round(ms, 4),
                          "hbm_bytes": tb, "GBps": round(tb / (ms * 1e-3) / 1e9, 1),
                          "note": "includes canvas copy-in (R*16 B/px) and root clone (16 B/px)"}), flush=True)
        grp.close()
