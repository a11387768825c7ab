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


def _over_np(front, back):
    return front + (np.float32(1.0) - front[:, 3:4]) * back


@pytest.mark.parametrize("order,hog", [([0, 1], False), ([1, 0], False), ([0, 1], True)])
def test_swap_needs_no_coresident_grid(order, hog):
    """The swap kernel must make progress with any subset of its CTAs
    resident (in situ the simulation's kernels share the GPU, and CTAs are
    only guaranteed to run eventually, not together).  Rank 0 runs the real
    kernel with the maximum slice count (1024 CTAs of 512 threads: far more
    than the 4 x 148 that fit on a B200 at once), while rank 1 is played by
    a host thread that serves slices in index order -- the partner is
    independent of this GPU's SM residency, as on a multi-GPU box.  Arenas
    live in pinned host memory (device-accessible under unified
    addressing).  A design with a grid-wide barrier deadlocks here; the
    per-slice protocol completes and matches the composite.  With ``hog``, a
    stand-in for the simulation's kernels (isc_debug_occupy: one 1024-thread
    CTA on half the SMs, spinning 0.3 s) holds the GPU from another stream
    when the swap is launched."""
    import ctypes as C
    import threading
    import time
    import torch
    from paper_1611_09048_b200 import _abi
    lib = _abi.lib()
    n, parts = 48 * 1024 + 77, _abi.MAX_SWAP_CTAS
    words = lib.isc_flag_words()
    ctrl = 16
    rng = np.random.default_rng(5)
    host = []
    for _ in range(2):
        a = rng.uniform(0, 1, (n, 1)).astype(np.float32)
        host.append(np.concatenate([rng.uniform(0, 1, (n, 3)).astype(np.float32) * a, a], axis=1))
    img = [torch.from_numpy(h.copy()).pin_memory() for h in host]
    flags = [torch.zeros(words, dtype=torch.int64).pin_memory() for _ in range(2)]
    root = torch.zeros((n, 4), dtype=torch.float32).pin_memory()
    args = _abi.SwapArgs()
    args.rank, args.size, args.n_ctas = 0, 2, parts
    args.round_begin, args.round_end, args.collect, args.finish, args.publish_ready = 0, 64, 1, 1, 1
    args.n_pixels, args.epoch, args.timeout_ns = n, 1, int(20e9)
    for i in range(2):
        args.order[i] = order[i]
        args.image[i] = img[i].data_ptr()
        args.flags[i] = flags[i].data_ptr()
    args.root_out = root.data_ptr()
    va, vb = order.index(0), order.index(1)
    fa, fb = flags[0].numpy(), flags[1].numpy()
    a_img, b_img, out = img[0].numpy(), img[1].numpy(), root.numpy()
    failure = []

    def word(stage, sl):
        return ctrl + stage * parts + sl

    def wait(arr, idx, deadline):
        while arr[idx] < 1:
            if time.monotonic() > deadline:
                raise TimeoutError(f"flag {idx} never set")

    def partner():          # rank 1: compositing.py:145-181 on each slice, in slice order
        try:
            deadline = time.monotonic() + 60.0
            per = (n + parts - 1) // parts
            fb[word(0, 0):word(0, parts)] = 1                # image ready
            for sl in range(parts):
                lo, hi = min(n, per * sl), min(n, per * sl + per)
                mid = (lo + hi) // 2
                k0, k1 = (mid, hi) if vb & 1 else (lo, mid)
                wait(fa, word(0, sl), deadline)
                mine, theirs = b_img[k0:k1], a_img[k0:k1]
                b_img[k0:k1] = _over_np(theirs, mine) if va < vb else _over_np(mine, theirs)
                fb[word(1, sl)] = 1
                out[k0:k1] = b_img[k0:k1]
                fb[word(2, sl)] = 1
            for sl in range(parts):                          # rank 0 has read our half
                wait(fa, word(1, sl), deadline)
        except BaseException as exc:  # noqa: BLE001
            failure.append(exc)

    stream = torch.cuda.Stream()
    hog_stream = torch.cuda.Stream()
    if hog:
        sms = lib.isc_device_sm_count(torch.cuda.current_device())
        _abi.check(lib.isc_debug_occupy(max(sms // 2, 1), 1024, int(3e8), C.c_void_p(hog_stream.cuda_stream)),
                   "occupy")
    t = threading.Thread(target=partner, daemon=True)
    t.start()
    _abi.check(lib.isc_binary_swap(C.byref(args), C.c_void_p(stream.cuda_stream)), "binary_swap")
    stream.synchronize()
    hog_stream.synchronize()
    t.join(90)
    assert not failure, failure
    assert int(fa[_abi.ERR_WORD]) == 0, "rank 0 timed out waiting"
    front, back = (host[0], host[1]) if order == [0, 1] else (host[1], host[0])
    assert np.abs(out - _over_np(front, back)).max() <= TOL


def test_swap_recovers_after_timeout_with_reset():
    """A timed-out swap leaves counters short; reset() restores the group."""
    import torch
    import paper_1611_09048_b200 as P
    from paper_1611_09048_b200.compositing import binary_swap_local
    gold = load("composite_swap4.npz")
    imgs = _images(gold)
    order = [int(v) for v in gold["order"]]
    h, w = imgs[0].shape[:2]
    grp = P.LocalNvlinkGroup(len(imgs), h * w)
    try:
        grp.set_n_ctas(4)
        ep = grp.endpoints[0]
        ep.timeout_s = 0.2
        with pytest.raises(P.TransportError):
            P.binary_swap(ep, imgs[0], order)            # the other ranks never arrive
        grp.reset()
        for _ in range(2):
            out = binary_swap_local(grp, imgs, order).cpu().numpy()
            assert np.abs(out - gold["result"]).max() <= TOL
    finally:
        grp.close()


def test_slice_count_must_agree():
    import paper_1611_09048_b200 as P
    from paper_1611_09048_b200.compositing import binary_swap_local
    gold = load("composite_swap2.npz")
    imgs = _images(gold)
    h, w = imgs[0].shape[:2]
    grp = P.LocalNvlinkGroup(2, h * w)
    try:
        grp.endpoints[1].n_ctas = 7
        with pytest.raises(P.CompositeError):
            binary_swap_local(grp, imgs, [0, 1])
    finally:
        grp.close()


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
        torch.cuda.synchronize()
        diag = (int(ep._error_word().item()), [int(s.item()) for s in ep._err_slots], len(ep._pending),
                [int(v) for v in torch.as_tensor(P.transport._CudaArray(ep.flags[1], (32,), "<i8"), device="cuda")
                 .cpu().tolist()])
        with pytest.raises(P.TransportError, match="did not arrive"):
            try:
                ep.flush()
            except P.TransportError:
                raise
            else:
                raise AssertionError(f"no TransportError: {diag}")
        ep.flush()   # the error word was cleared: nothing pending
    finally:
        grp.close()


@pytest.mark.parametrize("world", [2, 4])
def test_multi_rank_frame_graph_replays(world):
    """A static view captured as a multi-rank FrameGraph (render + fused
    peer-memory swap; the swap reads its epoch from the device) replays
    bit-identically to render_local + binary_swap, with plain swaps
    interleaved (torchrun, process per rank, all on one GPU)."""
    import json
    import os
    import socket
    import subprocess
    import sys
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    helper = os.path.join(os.path.dirname(os.path.abspath(__file__)), "helpers", "mp_framegraph.py")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={port}", helper, "5"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=400)
    assert out.returncode == 0, out.stderr[-3000:]
    res = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert res["all_identical"] and res["checks"] == 7 and res["nonzero"] > 0, res


def test_nccl_backed_paths_world_one():
    """The NCCL-default-group code paths of a multi-GPU run, exercised at world
    size 1 on this GPU (NCCL needs one GPU per rank): the MIN/MAX all-reduce of
    the auto value range on device tensors, the gloo side group of
    TorchDistTransport under NCCL, the IPC arena exchange and binary_swap."""
    import json
    import os
    import socket
    import subprocess
    import sys
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    helper = os.path.join(os.path.dirname(os.path.abspath(__file__)), "helpers", "nccl_paths.py")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr=127.0.0.1", f"--master-port={port}", helper]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-3000:]
    res = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert res["local"] == res["reduced"] and res["empty_is_nan"] and res["swap_equal"], res
