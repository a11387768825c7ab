"""GPU parity for sort-last compositing: fused peer-memory binary swap, direct
send, byte-transport swap and the fold kernel against the reference goldens
(binary_swap over LocalFabric threads, compositing.py:107-194).

float32 images vs the reference's float64: tolerance 1e-6 (the reference
tests' own swap-vs-sequential bound, test_compositing.py:173).
"""

import threading

import numpy as np
import pytest

from golden_io import cases, load

pytestmark = pytest.mark.gpu
TOL = 1e-6


def _images(gold):
    import torch
    return [torch.from_numpy(im.astype(np.float32)).cuda() for im in gold["images"]]


@pytest.mark.parametrize("name", sorted(cases.COMPOSITE_CASES))
def test_peer_memory_swap_sequential_launch(name):
    import paper_1611_09048_b200 as P
    from paper_1611_09048_b200.compositing import binary_swap_local
    gold = load(f"composite_{name}.npz")
    imgs = _images(gold)
    order = [int(v) for v in gold["order"]]
    h, w = imgs[0].shape[:2]
    grp = P.LocalNvlinkGroup(len(imgs), h * w)
    try:
        for ep in grp.endpoints:
            ep.n_ctas = 3
        for _ in range(3):   # epochs advance; result must be stable
            out = binary_swap_local(grp, imgs, order).cpu().numpy()
            assert np.abs(out - gold["result"]).max() <= TOL
        R = len(imgs)
        image_bytes = h * w * 16
        if R & (R - 1) == 0:   # binary swap balance bound (test_compositing.py:193-214), per epoch
            for ep in grp.endpoints:
                assert ep.sent_bytes <= 3 * 2 * image_bytes and ep.received_bytes <= 3 * 2 * image_bytes
    finally:
        grp.close()


@pytest.mark.parametrize("ranks", [2, 4, 8, 3, 6])
def test_peer_memory_swap_concurrent_ranks(ranks):
    """Every rank on its own host thread + stream, all kernels live at once and
    order themselves through the flag protocol (the multi-GPU execution model,
    here with all ranks sharing one device), over 3 epochs.  Runs in a child
    process with CUDA_DEVICE_MAX_CONNECTIONS=32 so the ranks' streams do not
    alias onto one hardware queue (a single-GPU artefact)."""
    import json
    import os
    import subprocess
    import sys
    helper = os.path.join(os.path.dirname(os.path.abspath(__file__)), "helpers", "concurrent_swap.py")
    env = dict(os.environ, CUDA_DEVICE_MAX_CONNECTIONS="32")
    out = subprocess.run([sys.executable, helper, str(ranks), "3"], env=env, capture_output=True, text=True,
                         timeout=240)
    assert out.returncode == 0, out.stderr[-2000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert not res["errors"], res["errors"]
    assert res["err"] is not None and res["err"] <= TOL
    assert res["others_none"]


@pytest.mark.parametrize("name", ["swap2", "swap8", "direct3", "direct6"])
def test_byte_transport_swap_gpu_over(name):
    import paper_1611_09048_b200 as P
    gold = load(f"composite_{name}.npz")
    imgs = _images(gold)
    order = [int(v) for v in gold["order"]]
    fabric = P.LocalFabric(len(imgs))
    res = [None] * len(imgs)

    def body(r):
        res[r] = P.binary_swap(fabric.endpoint(r), imgs[r], order)

    threads = [threading.Thread(target=body, args=(r,)) for r in range(len(imgs))]
    for t in threads:
        t.start()
    for t in threads:
        t.join(60)
    assert np.abs(res[0].cpu().numpy() - gold["result"]).max() <= TOL
    image_bytes = imgs[0].numel() * 4
    if len(imgs) & (len(imgs) - 1) == 0:
        for r in range(len(imgs)):
            assert fabric.sent_bytes[r] <= 2 * image_bytes
            assert fabric.received_bytes[r] <= 2 * image_bytes


def test_fold_and_over_kernels():
    import torch
    import paper_1611_09048_b200 as P
    gold = load("composite_swap4.npz")
    imgs = _images(gold)
    order = [int(v) for v in gold["order"]]
    assert np.abs(P.composite_sequential(imgs, order).cpu().numpy() - gold["sequential"]).max() <= TOL
    f = torch.tensor([[0.5, 0.0, 0.0, 0.5]], device="cuda")
    b = torch.tensor([[0.0, 0.0, 0.5, 0.5]], device="cuda")
    assert P.over_arrays(f, b).cpu().tolist() == [[0.5, 0.0, 0.25, 0.75]]


def test_swap_timeout_surfaces_as_transport_error():
    import torch
    import paper_1611_09048_b200 as P
    grp = P.LocalNvlinkGroup(2, 64)
    try:
        ep = grp.endpoints[0]
        ep.timeout_s = 0.2
        ep.n_ctas = 1
        with pytest.raises(P.TransportError):
            P.binary_swap(ep, torch.zeros((8, 8, 4), device="cuda"), [0, 1])   # rank 1 never arrives
    finally:
        grp.close()


@pytest.mark.parametrize("name,world", [("swap2", 2), ("swap4", 4), ("direct3", 3)])
def test_multi_process_ipc_swap(name, world):
    """Process-per-rank with CUDA IPC arenas (torchrun, all ranks on one GPU)."""
    import json
    import os
    import socket
    import subprocess
    import sys
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    helper = os.path.join(os.path.dirname(os.path.abspath(__file__)), "helpers", "mp_swap.py")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={port}", helper, name, "3"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=400)
    assert out.returncode == 0, out.stderr[-3000:]
    res = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert res["max_err"] <= TOL


def test_swap_timeout_deferred_check():
    """sync_errors=False: the swap returns without synchronising; the timed-out
    spin-wait surfaces as TransportError at flush()."""
    import torch
    import paper_1611_09048_b200 as P
    grp = P.LocalNvlinkGroup(2, 64)
    try:
        ep = grp.endpoints[0]
        ep.timeout_s = 0.2
        ep.n_ctas = 1
        ep.sync_errors = False
        P.binary_swap(ep, torch.zeros((8, 8, 4), device="cuda"), [0, 1])   # rank 1 never arrives
        with pytest.raises(P.TransportError):
            ep.flush()
        ep.flush()   # the error word was cleared: nothing pending
    finally:
        grp.close()
