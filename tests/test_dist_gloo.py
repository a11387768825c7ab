"""Multi-process (world size 2 and 4, gloo, CPU) coverage of the N>1 host
path: TorchDistTransport bytes, broadcast / gather, and the binary-swap /
direct-send message schedule of ``binary_swap`` over a byte transport.  The
per-pixel ``over`` is injected (the oracle's) because kernels need a GPU; the
GPU tests cover the same schedule with the CUDA ``over``."""

import os
import pickle
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class OracleOps:
    """Host stand-in for compositing.DeviceOps (test only)."""

    def as_flat(self, pixels):
        return np.ascontiguousarray(pixels, dtype=np.float64).reshape(-1, 4)

    def to_bytes(self, span):
        return np.ascontiguousarray(span, dtype="<f4").tobytes()

    def from_array(self, arr):
        return np.asarray(arr, dtype=np.float64)

    def over(self, front, back):
        from oracle import isaac_oracle as O
        return O.over(front, back)

    def fold(self, flats, order):
        from oracle import isaac_oracle as O
        return O.composite_in_order(flats, order)

    def empty(self, n):
        return np.empty((n, 4))


def _worker(rank, world, port, out_dir, images, order):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1611_09048_b200.compositing import _swap_bytes
    from paper_1611_09048_b200.transport import TorchDistTransport
    from test_dist_gloo import OracleOps
    t = TorchDistTransport()
    res = {}
    # point to point in both directions + collectives
    peer = (rank + 1) % world
    t.send(peer, f"hello from {rank}".encode())
    res["p2p"] = t.receive((rank - 1) % world).decode()
    res["bcast"] = t.broadcast_from_root(b"scene-bytes" if rank == 0 else None)
    res["gather"] = t.gather_to_root(str(rank).encode())
    res["allgather"] = t.all_gather(bytes([rank]))
    ops = OracleOps()
    flat = ops.as_flat(images[rank])
    out = _swap_bytes(t, flat, list(order), tuple(images[rank].shape), ops)
    res["frame"] = None if out is None else np.asarray(out)
    res["sent"], res["received"] = t.sent_bytes, t.received_bytes
    t.flush()
    dist.barrier()
    dist.destroy_process_group()
    with open(os.path.join(out_dir, f"r{rank}.pkl"), "wb") as fh:
        pickle.dump(res, fh)


@pytest.mark.parametrize("world", [2, 4, 3])
def test_gloo_transport_and_swap_schedule(tmp_path, world):
    import torch.multiprocessing as mp
    from oracle import isaac_oracle as O
    rng = np.random.default_rng(world)
    images = []
    for _ in range(world):
        a = rng.uniform(0, 1, (9, 7, 1))
        images.append(np.concatenate([rng.uniform(0, 1, (9, 7, 3)) * a, a], axis=2))
    order = [int(v) for v in rng.permutation(world)]
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), images, order), nprocs=world, join=True)
    res = [pickle.load(open(tmp_path / f"r{r}.pkl", "rb")) for r in range(world)]
    for r in range(world):
        assert res[r]["p2p"] == f"hello from {(r - 1) % world}"
        assert res[r]["bcast"] == b"scene-bytes"
        assert res[r]["allgather"] == [bytes([q]) for q in range(world)]
    assert res[0]["gather"] == [str(q).encode() for q in range(world)]
    want = O.composite_in_order(images, order)
    assert np.abs(res[0]["frame"] - want).max() <= 1e-6   # float32 wire payload
    assert all(res[r]["frame"] is None for r in range(1, world))
    if world & (world - 1) == 0:
        image_bytes = images[0][..., 0].size * 16
        for r in range(world):   # balance bound (test_compositing.py:193-214), control bytes excluded
            assert res[r]["sent"] <= 2 * image_bytes + 256


def test_bench_gpus_flag_launches_that_many_ranks():
    """``python bench.py --gpus N`` outside torchrun starts N ranks itself (the
    driver's scaling run must not silently measure one rank)."""
    import json
    import subprocess
    import sys
    bench = os.path.join(ROOT, "bench.py")
    for n, decomp in ((2, [2, 1, 1]), (4, [2, 2, 1])):
        out = subprocess.run([sys.executable, bench, "--gpus", str(n), "--dry-run"], capture_output=True,
                             text=True, timeout=300)
        assert out.returncode == 0, out.stderr[-2000:]
        line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
        assert line["n_gpus"] == n and line["ranks_seen"] == n
        assert line["rank_sum"] == n * (n - 1) // 2
        assert line["decomposition"] == decomp


def _range_worker(rank, world, port, out_dir, ranges):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1611_09048_b200.normalize import reduce_range
    got = reduce_range(*ranges[rank], group=True)
    with open(os.path.join(out_dir, f"range{rank}.pkl"), "wb") as fh:
        pickle.dump(got, fh)
    dist.destroy_process_group()


@pytest.mark.parametrize("ranges,want", [
    ([(0.5, 2.0), (-1.25, 0.75), (0.0, 3.5)], (-1.25, 3.5)),
    ([(float("nan"), float("nan")), (0.25, 0.5), (0.125, 0.375)], (0.125, 0.5)),   # an empty brick
    ([(float("nan"), float("nan"))] * 3, None),                                      # nothing anywhere
])
def test_value_range_group_reduction(tmp_path, ranges, want):
    """Cross-rank auto range (normalize.value_range(group=...)): every rank
    gets the global (min, max) of the per-brick ranges, empty bricks ignored,
    over a 3-rank gloo group."""
    import math
    import torch.multiprocessing as mp
    world = len(ranges)
    mp.spawn(_range_worker, args=(world, _free_port(), str(tmp_path), ranges), nprocs=world, join=True)
    for r in range(world):
        with open(tmp_path / f"range{r}.pkl", "rb") as fh:
            got = pickle.load(fh)
        if want is None:
            assert all(math.isnan(v) for v in got)
        else:
            assert got == want


def test_bench_reference_arm_contract():
    """`bench.py --impl reference` (runs on host cores, no GPU): one JSON line
    with impl "reference", the metric / unit of the GPU arm, a cpu_baseline
    naming what ran (the reference from baseline/_ref, else the oracle port)
    and an e2e block with zero copy bytes; steps x ms_per_step is the timed
    wall clock."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "3", "--ref-step-s", "0.3"], capture_output=True, text=True, timeout=600,
                         cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, lines
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "frames/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 2
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    c = d["consistency"]
    assert abs(c["timed_seconds"] - c["steps_x_ms_per_step_s"]) <= 0.05 * c["timed_seconds"] + 0.01
