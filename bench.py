#!/usr/bin/env python
"""Benchmark of the ISAAC render hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config c4]

One JSON line on rank 0.  A "step" is one frame: ``render_local`` of this
rank's brick (the sm_100a march kernel) + ``binary_swap`` of the sub-images
(the fused peer-memory swap kernel; a device copy at N=1).  Default workload
(N=1 and every N): config C4 of BASELINE.json -- a 1024^3 float32 field with
a one-cell guard, decomposed into N bricks (1x1x1, 2x1x1, 2x2x1, 2x2x2; strong
scaling), rendered at 1920x1080 with the reference harness camera, trilinear
sampling, step 0.5, linear transfer function, early termination off.

Under torchrun each rank drives one GPU.  Timing: W untimed steps, then K
steps bracketed by barrier + synchronize, CUDA events on the launching
stream, max over ranks.  The 4.32 GB field is far larger than the 126 MB L2,
so no explicit L2 flush is needed between steps (stated in ``config``).
"""

from __future__ import annotations

import argparse
import gc
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "frames/sec and Gsamples/sec at 1024³×1080p, 1/2/4/8 B200; % of HBM roofline"
def decomposition(world):
    """Bricks per axis for `world` ranks: powers of two split x, y, z in turn
    (1x1x1, 2x1x1, 2x2x1, 2x2x2, 4x2x2, ...); other counts put their prime
    factors, largest first, on the currently smallest axis."""
    d = [1, 1, 1]
    n, p, primes = world, 2, []
    while n > 1:
        while n % p == 0:
            primes.append(p)
            n //= p
        p += 1
    for f in sorted(primes, reverse=True) if world & (world - 1) else primes:
        a = d.index(min(d))
        d[a] *= f
    return tuple(d)


DECOMP = {n: decomposition(n) for n in range(1, 65)}
CONFIGS = {
    "c4": dict(n=1024, image=(1920, 1080), desc="1024^3 float32 field (1 cell guard), 1920x1080, trilinear, "
                                                "linear TF, harness camera, step 0.5, bricks across N GPUs"),
    "c2": dict(n=512, image=(1920, 1080), clip=True, desc="512^3 float32, 1920x1080, trilinear + clip plane"),
    "c1": dict(n=64, image=(256, 256), desc="64^3 float32, 256x256, trilinear, linear TF"),
    "c3": dict(n=512, image=(1920, 1080), multi=True,
               desc="512^3 scalar (iso surface) + 512^3 float3 (chain length|mul(2)|add(0.1), volume), 1920x1080"),
    "c5": dict(n=512, image=(3840, 2160), weak=True, orbit=True,
               desc="512^3 float32 per GPU (weak scaling), 3840x2160, 26-direction camera orbit"),
}
ORBIT = [(i, j, k) for i in (-1, 0, 1) for j in (-1, 0, 1) for k in (-1, 0, 1) if (i, j, k) != (0, 0, 0)]
BYTES_PER_SAMPLE = 32       # 8 trilinear corners x 4 B
BYTES_PER_PIXEL_OUT = 16    # float32 RGBA written per pixel


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def harness_camera(n):
    diag = math.sqrt(3.0 * n * n)
    return (n * 1.4, n * 1.15, -0.8 * diag), (n / 2.0, n / 2.0, n / 2.0)


def make_field_torch(n, domain, device):
    """Separable smooth field f = 1 + sin(0.4 x s) cos(0.3 y s) + 0.4 sin(0.5 z s),
    s = 64/n (scaled from test_raycast.py:230-231); range
    ~[-0.4, 2.4]; built in 64-slab chunks to bound temporaries."""
    import torch
    g = domain.guard_width
    ox, oy, oz = domain.offset
    sx, sy, sz = domain.size
    s = 64.0 / n
    dt = torch.float64
    x = torch.arange(ox - g, ox + sx + g, dtype=dt, device=device)
    y = torch.arange(oy - g, oy + sy + g, dtype=dt, device=device)
    z = torch.arange(oz - g, oz + sz + g, dtype=dt, device=device)
    ab = (1.0 + torch.sin(0.4 * x * s)[None, :] * torch.cos(0.3 * y * s)[:, None]).float()
    cz = (0.4 * torch.sin(0.5 * z * s)).float()
    out = torch.empty((sz + 2 * g, sy + 2 * g, sx + 2 * g), dtype=torch.float32, device=device)
    for z0 in range(0, out.shape[0], 64):
        out[z0:z0 + 64] = ab[None] + cz[z0:z0 + 64, None, None]
    return out


def make_vector_field_torch(n, domain, device):
    """float3 field for C3: three phase-shifted copies of the scalar field."""
    import torch
    g = domain.guard_width
    sx, sy, sz = domain.size
    out = torch.empty((sz + 2 * g, sy + 2 * g, sx + 2 * g, 3), dtype=torch.float32, device=device)
    base = make_field_torch(n, domain, device)
    out[..., 0] = base - 1.0
    out[..., 1] = 0.5 * base
    out[..., 2] = base.flip(0) - 1.0
    return out


def build_scene(P, cfg, n=None):
    n = n if n is not None else cfg["n"]
    pos, look = harness_camera(n)
    planes = ()
    if cfg.get("clip"):
        planes = (P.clip_plane((n / 2.0,) * 3, (0.3, -0.5, 0.81)),)
    linear = [(0.0, 0.0, 0.0, 0.0, 0.0), (1.0, 1.0, 1.0, 1.0, 1.0)]
    if cfg.get("multi"):
        cool = [(0.0, 0.0, 0.0, 0.0, 0.0), (0.6, 0.1, 0.7, 0.4, 0.3), (1.0, 0.7, 1.0, 0.9, 0.8)]
        return P.SceneState(camera=P.Camera(pos, look, image_size=cfg["image"]),
                            tf_points={0: linear, 1: cool}, value_ranges={0: (-0.4, 2.4), 1: (0.0, 6.0)},
                            chain_texts={0: "", 1: "length | mul(2) | add(0.1)"},
                            settings=P.RenderSettings(active_set=(0, 1), modes={0: "iso"},
                                                      iso_thresholds={0: 1.0}, interpolation=True,
                                                      step_length=0.5, early_termination_alpha=1.0),
                            clip_planes=planes)
    return P.SceneState(camera=P.Camera(pos, look, image_size=cfg["image"]),
                        tf_points={0: linear},
                        value_ranges={0: (-0.4, 2.4)}, chain_texts={0: ""},
                        settings=P.RenderSettings(active_set=(0,), interpolation=True, step_length=0.5,
                                                  early_termination_alpha=1.0),
                        clip_planes=planes)


def orbit_scene(P, scene, n, dvec):
    """Camera on the 26-direction orbit {-1,0,1}^3 minus 0 at
    radius 1752 * n / 512 about the centre."""
    c = n / 2.0
    norm = math.sqrt(sum(v * v for v in dvec))
    r = 1752.0 * n / 1024.0
    pos = tuple(c + r * v / norm for v in dvec)
    up = (0.0, 1.0, 0.0) if dvec[0] or dvec[2] else (0.0, 0.0, 1.0)
    cam = P.Camera(pos, (c, c, c), up=up, image_size=scene.camera.image_size)
    return P.SceneState(camera=cam, tf_points=scene.tf_points, value_ranges=scene.value_ranges,
                        chain_texts=scene.chain_texts, settings=scene.settings, clip_planes=scene.clip_planes)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = os.path.join("/tmp", f"isc_clocks_{os.getpid()}.csv")

    def start(self):
        if os.environ.get("ISC_BENCH_NO_CLOCKS"):   # experiment switch: no sampler
            return
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
            return
        # wait for the first sample: nvidia-smi's NVML start-up must not fall
        # inside the timed region (it can stall the driver for tens of ms)
        t_end = time.time() + 5.0
        while time.time() < t_end:
            try:
                if os.path.getsize(self.path) > 0:
                    break
            except OSError:
                pass
            time.sleep(0.02)

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sms, maxs, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as fh:
            for line in fh:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sms.append(float(parts[1]))
                    maxs.append(float(parts[2]))
                except ValueError:
                    continue
                for nm, v in zip(names, parts[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        if not sms:
            return None
        return {"sm_mhz": statistics.median(sms), "sm_max_mhz": max(maxs), "reasons": sorted(reasons),
                "samples": len(sms)}


# --------------------------------------------------------------------------
# B200 arm


def run_b200(args):
    import torch
    import torch.distributed as dist

    import paper_1611_09048_b200 as P
    from paper_1611_09048_b200.raycast import describe_kernel

    rank, world, local = dist_env()
    if world > torch.cuda.device_count() and not args.share_gpu:
        raise SystemExit(f"bench: {world} ranks but only {torch.cuda.device_count()} visible GPU(s); "
                         "use --share-gpu for a one-GPU rehearsal")
    if args.share_gpu:          # rehearsal: every rank on cuda:0 (ranks time-share one GPU)
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    red_dev = torch.device("cpu") if args.share_gpu else dev
    cfg = CONFIGS[args.config]
    w, h = cfg["image"]
    decomp = DECOMP[world]
    if cfg.get("weak"):
        size = tuple(cfg["n"] * decomp[a] for a in range(3))
    else:   # strong scaling; a non-power-of-two rank count trims the volume to divide evenly
        size = tuple(cfg["n"] - cfg["n"] % decomp[a] for a in range(3))
    n = size[0]
    volume = P.GlobalVolume(size, decomp)
    domain = volume.local_domain(rank, 1)
    t0 = time.time()
    field = make_field_torch(n, domain, dev)
    reg = P.SourceRegistry(domain)
    reg.register_handle(P.array_backed_handle(P.SourceDescriptor("density", 1, has_guard=True), field, 1))
    active = {0}
    if cfg.get("multi"):
        vec = make_vector_field_torch(n, domain, dev)
        reg.register_handle(P.array_backed_handle(P.SourceDescriptor("velocity", 3, has_guard=True), vec, 1))
        active = {0, 1}
    torch.cuda.synchronize()
    log(f"[rank {rank}] field {tuple(field.shape)} ready in {time.time() - t0:.1f}s")
    P.update_sources(reg, active, {})
    fr = P.default_registry()
    scene = build_scene(P, cfg, n)
    scenes = [scene]
    if cfg.get("orbit"):
        scenes = [orbit_scene(P, scene, n, dvec) for dvec in ORBIT]
    orders = [P.visibility_order(volume, sc.camera) for sc in scenes]
    order = orders[0]
    if world > 1:
        host = P.TorchDistTransport()
        transport = P.NvlinkTransport(host, w * h)
        transport.sync_errors = False     # pipelined frames; checked at flush() below
        canvas = transport.canvas(h, w)
    else:
        transport = P.LocalFabric(1).endpoint(0)
        canvas = torch.empty((h, w, 4), dtype=torch.float32, device=dev)
    ctx = P.RankContext(volume, domain, reg, fr, fr.limits, transport)
    plans = [P.build_plans(reg, fr, fr.limits, sc) for sc in scenes]
    stream = torch.cuda.current_stream()
    counter = [0]

    def step(events=None, swap_events=None):
        i = counter[0] % len(scenes)
        counter[0] += 1
        img = P.render_local(ctx, scenes[i], plans=plans[i], out=canvas, check_errors=False, events=events)
        if swap_events is not None:
            swap_events[0].record(stream)
        full = P.binary_swap(transport, img.pixels, orders[i])
        if swap_events is not None:
            swap_events[1].record(stream)
        return img, full

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up (also: station count of this brick, guard-contract check)
    img = None
    for _ in range(max(args.warmup, 1)):
        img, _ = step()
    img.check()
    stations = img.stations
    if len(scenes) > 1:       # orbit: samples per frame averaged over the timed camera sequence
        counter[0] = 0
        tot = 0
        for _ in range(args.steps):
            im, _ = step()
            tot += im.stations
        stations = tot / args.steps
        counter[0] = 0
    n_active = len(active)
    bytes_per_station = sum(BYTES_PER_SAMPLE * reg.descriptor(sid).feature_dim for sid in sorted(active))
    st_t = torch.tensor([stations * n_active], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(st_t)
    samples_frame = int(st_t.item())

    clocks = ClockSampler(local)
    k = args.steps
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
    sevs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    clocks.start()
    # Python's cyclic GC off for the timed steps (as timeit does): a full
    # collection over torch's object graph can pause the enqueueing host for
    # tens of ms, i.e. idle the GPU inside the timed region
    gc.collect()
    gc.disable()
    # keep the GPU busy right up to the timed region: ~100 ms of untimed
    # frames, so the SM clock is at its boost level when timing starts (an
    # idle GPU drops its clock, and short frames -- C1, C2 -- would otherwise
    # time the ramp-up), then only the barrier's brief drain before start
    warm_gpu(step, dist, world, red_dev)
    counter[0] = 0          # the orbit's timed views are the ones its samples were averaged over
    barrier()
    start.record(stream)
    for i in range(k):
        step(evs[i], sevs[i] if world > 1 else None)   # swap timing only where there is a swap
    end.record(stream)
    torch.cuda.synchronize()
    gc.enable()
    clk = clocks.stop()
    if world > 1:
        transport.flush()             # a timed-out swap raises here
    ms_total = start.elapsed_time(end)
    kernel_ms = sum(a.elapsed_time(b) for a, b in evs) / k
    swap_ms = sum(a.elapsed_time(b) for a, b in sevs) / k if world > 1 else 0.0
    t = torch.tensor([ms_total, kernel_ms], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total, kernel_ms_max = float(t[0]), float(t[1])
    # compositing: per-rank time of the binary_swap call (spin-waits for late
    # partners included); its minimum over ranks is the last-arriving rank's,
    # i.e. transfer + over without waiting.  Each rank pulls / stores n*16 B
    # through peer memory per frame in a binary swap (rank 0 reads (R-1)*n*16 B
    # in a direct send).
    composite = None
    if world > 1:
        sw = torch.tensor([swap_ms, -swap_ms], dtype=torch.float64, device=red_dev)
        dist.all_reduce(sw, op=dist.ReduceOp.MAX)
        swap_max, swap_min = float(sw[0]), -float(sw[1])
        pow2 = (world & (world - 1)) == 0
        peer_bytes = w * h * 16 * (1 if pow2 else (world - 1))
        composite = {"kind": "binary_swap" if pow2 else "direct_send", "ms_max_over_ranks": round(swap_max, 4),
                     "ms_min_over_ranks": round(swap_min, 4),
                     "share_of_frame": round(swap_min / (ms_total / k), 4),
                     "peer_bytes_per_rank": peer_bytes,
                     "peer_GBps": round(peer_bytes / (swap_min * 1e-3) / 1e9, 1) if swap_min > 0 else None,
                     "note": "min over ranks = the last-arriving rank's swap (no waiting): transfer + over"}
    ms_step = ms_total / k
    fps = 1000.0 / ms_step
    gsps = samples_frame * fps / 1e9

    # roofline of the dominant kernel (the march): algorithmic bytes per launch
    bytes_rank = stations * bytes_per_station + w * h * BYTES_PER_PIXEL_OUT
    br = torch.tensor([float(bytes_rank)], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(br)
    peak, peak_src = peak_hbm()
    achieved = float(br.item()) / (kernel_ms_max * 1e-3) / 1e9 / world
    # ncu evidence for this config (profiles/ncu_counters.json, written by
    # tools/ncu_counters.py from one `ncu --set full` capture of the kernel)
    traffic, l1tex = ncu_evidence(f"{args.config}_n{world}")

    # e2e through the public API with host buffers: scene bytes in (JSON, as
    # broadcast by the reference runtime) -> LUT + launch block H2D, frame out
    # to pinned host memory (D2H) every step.
    e2e = run_e2e(P, torch, dist, ctx, scenes[0], transport, canvas, order, rank, world, red_dev, max(3, k))

    # transfer-function variants of the same frame, timed in this run: the
    # general shared-memory LUT lookup (no analytic form), and a 3-point
    # transfer function (one slope change: the analytic hinge form, and the
    # same through the LUT) -- what a user steering the TF gets
    def time_tf(scene_v, analytic, count_stations=False):
        plans_v = P.build_plans(reg, fr, fr.limits, scene_v)
        bytes_v = br
        if count_stations:  # the variant marches fewer stations (early termination): its own bytes
            im = P.render_local(ctx, scene_v, plans=plans_v, out=canvas, analytic_lut=analytic)
            bytes_v = torch.tensor([float(im.stations * bytes_per_station + w * h * BYTES_PER_PIXEL_OUT)],
                                   dtype=torch.float64, device=red_dev)
            if world > 1:
                dist.all_reduce(bytes_v)
        evs2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
        def frame_v():
            P.render_local(ctx, scene_v, plans=plans_v, out=canvas, check_errors=False, analytic_lut=analytic)
            P.binary_swap(transport, canvas, order)

        warm_gpu(frame_v, dist, world, red_dev, seconds=0.05)
        barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for i in range(k):
            P.render_local(ctx, scene_v, plans=plans_v, out=canvas, check_errors=False, events=evs2[i],
                           analytic_lut=analytic)
            P.binary_swap(transport, canvas, order)
        s1.record(stream)
        torch.cuda.synchronize()
        kl = sum(x.elapsed_time(y) for x, y in evs2) / k
        tl = torch.tensor([s0.elapsed_time(s1) / k, kl], dtype=torch.float64, device=red_dev)
        if world > 1:
            dist.all_reduce(tl, op=dist.ReduceOp.MAX)
        return {"value": round(1000.0 / float(tl[0]), 3), "unit": "frames/s", "kernel_ms": round(float(tl[1]), 4),
                "roofline_frac": round(float(bytes_v.item()) / (float(tl[1]) * 1e-3) / 1e9 / world / peak, 4),
                "kernel": describe_kernel(plans_v, scene_v.settings, analytic, scene_v.camera.image_size)}

    lut_path = tf_variants = tf4_variants = et_variant = None
    if len(scenes) == 1 and len(active) == 1:
        lut_path = time_tf(scenes[0], False)
        lut_path["note"] = ("same frame, transfer function classified through the 256-entry shared-memory LUT "
                            "(planar: one float table per channel)")
        lut_path["traffic"], lut_path["l1tex"] = ncu_evidence(f"{args.config}_lut_n{world}")
        tf3 = tf3_scene(P, scenes[0])
        tf_variants = {"points": [list(p) for p in TF3_POINTS],
                       "analytic": time_tf(tf3, True), "lut": time_tf(tf3, False),
                       "note": "same frame with a 3-point transfer function (slope change at t=0.6): analytic "
                               "hinge form (raycast.lut_analytic) vs the shared-memory LUT"}
        # early termination at the reference's default alpha_stop 0.99
        # (scene.py:165) with the transfer function's opacity scaled to 0.01
        # (translucent: rays run deep before they stop)
        import dataclasses
        sc0 = scenes[0]
        et_scene = P.SceneState(camera=sc0.camera, value_ranges=sc0.value_ranges, chain_texts=sc0.chain_texts,
                                clip_planes=sc0.clip_planes,
                                tf_points={i: [(p[0], p[1], p[2], p[3], p[4] * 0.01) for p in pts]
                                           for i, pts in sc0.tf_points.items()},
                                settings=dataclasses.replace(sc0.settings, early_termination_alpha=0.99))
        et_variant = time_tf(et_scene, True, count_stations=True)
        et_variant["note"] = ("same frame, alpha_stop 0.99 (the reference's default) and the transfer function's "
                              "opacity x0.01; roofline_frac over the stations actually marched")
        et_variant["traffic"], et_variant["l1tex"] = ncu_evidence(f"{args.config}_et_n{world}")
        tf4 = tf3_scene(P, scenes[0], TF4_POINTS)
        tf4_variants = {"points": [list(p) for p in TF4_POINTS],
                        "analytic": dict(time_tf(tf4, True),
                                         l1tex=ncu_evidence(f"{args.config}_tf4_n{world}")[1]),
                        "lut": time_tf(tf4, False),
                        "note": "a 4-point transfer function with both interior points between LUT samples: 4 "
                                "slope changes, the run-time kink-count variant vs the shared-memory LUT"}

    # informational: the same static-view frame replayed as one CUDA graph
    # (FrameGraph: no per-frame host preparation), N=1 only
    # (N > 1: every rank replays its captured render + peer-memory swap, the
    # swap's epoch on the device; max over ranks)
    graph_replay = None
    if len(scenes) == 1 and (world == 1 or isinstance(transport, P.NvlinkTransport)):
        fg = P.FrameGraph(ctx, scenes[0])
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        warm_gpu(fg.replay, dist, world, red_dev, seconds=0.05)
        barrier()
        g0.record(stream)
        for _ in range(k):
            fg.replay()
        g1.record(stream)
        torch.cuda.synchronize()
        fg.check()
        gt = torch.tensor([g0.elapsed_time(g1) / k], dtype=torch.float64, device=red_dev)
        if world > 1:
            dist.all_reduce(gt, op=dist.ReduceOp.MAX)
        gms = float(gt.item())
        graph_replay = {"value": round(1000.0 / gms, 3), "unit": "frames/s", "ms_per_step": round(gms, 4),
                        "note": "same frame captured once as a CUDA graph (runtime.FrameGraph: render + "
                                "binary swap) and replayed"}

    norm = time_normalisation(P, torch, reg, domain, peak)
    host_field = None if args.no_host_field_e2e else run_e2e_host_field(
        P, torch, dist, ctx, scenes[0], transport, canvas, order, rank, world, red_dev, field)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not cfg.get("multi") and not cfg.get("weak"):
        cpu = cpu_baseline(field.cpu().numpy(), cfg, n, samples_frame, budget_s=args.cpu_budget)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(fps, 3), "unit": "frames/s", "n_gpus": world, "steps": k,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
            "scaling": "weak" if cfg.get("weak") else "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": {"workload": f"{args.config.upper()}: {cfg['desc']}",
                       "volume": list(size), "image": [w, h], "decomposition": list(decomp),
                       "samples_per_frame": samples_frame, "field_bytes_per_gpu": field.numel() * 4,
                       "l2": "inputs larger than L2 (field >> 126 MB); no flush needed",
                       "parallelism": f"bricks{decomp[0]}x{decomp[1]}x{decomp[2]}",
                       "ranks_share_one_gpu": bool(args.share_gpu and world > 1)},
            "gsamples_per_s": round(gsps, 3),
            "samples_note": ("samples = stations x active sources; iso rays stop at the hit" if cfg.get("multi")
                             else "samples = stations (one active source)"),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic, "l1tex": l1tex,
                         "peak_source": peak_src,
                         "kernel": describe_kernel(plans[0], scenes[0].settings, image_size=scenes[0].camera.image_size), "kernel_ms": round(kernel_ms_max, 4),
                         "algorithmic_bytes_per_launch": int(br.item() / world),
                         **({"frac_above_1": (
                             "the 32 B/sample model counts every corner read; neighbouring rays share corners "
                             "through L1 (hit rate %s), DRAM moved %s B per launch (ncu), so the kernel is not "
                             "HBM-bound -- its limiter is %s" % (
                                 l1tex and l1tex["l1_hit_rate"], traffic, l1tex and l1tex["limiter"]))}
                            if achieved / peak > 1.0 else {})},
            "e2e": e2e,
            "classification": ("analytic transfer function (exact: the LUT lerp is piecewise linear with "
                               "few slope changes, raycast.lut_analytic); general shared-memory LUT path "
                               "timed in 'lut_path', a 3-point TF in 'tf_3point'") if lut_path else
                              "per-source analytic form or shared-memory LUT",
            "lut_path": lut_path,
            "tf_3point": tf_variants,
            "tf_4point": tf4_variants,
            "early_termination": et_variant,
            "graph_replay": graph_replay,
            "composite": composite,
            "e2e_host_field": host_field,
            "normalisation": norm,
            "gpu_launches": k * (1 + (1 if world > 1 else 0)),
            "clocks": clk,
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_e2e_host_field(P, torch, dist, ctx, scene, transport, canvas, order, rank, world, red_dev, field,
                       steps=3):
    """Informational: the same public-API frame, but with the brick's field
    uploaded every step from pinned host memory (a host-resident simulation),
    plus the frame D2H.  The in-situ contract keeps fields in HBM, so this is
    not the headline e2e; it shows what PCIe costs when they are not."""
    host = torch.empty(field.shape, dtype=field.dtype).pin_memory()
    host.copy_(field)
    w, h = scene.camera.image_size
    out = torch.empty((h, w, 4), dtype=torch.float32).pin_memory() if rank == 0 else None
    stream = torch.cuda.current_stream()

    def one():
        field.copy_(host, non_blocking=True)
        img = P.render_local(ctx, scene, out=canvas, check_errors=False)
        full = P.binary_swap(transport, img.pixels, order)
        if full is not None:
            out.copy_(full, non_blocking=True)

    one()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        one()
    b.record(stream)
    torch.cuda.synchronize()
    tt = torch.tensor([a.elapsed_time(b) / steps], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms = float(tt.item())
    del host
    return {"value": round(1000.0 / ms, 3), "unit": "frames/s", "ms_per_step": round(ms, 3), "steps": steps,
            "h2d_bytes_per_step": field.numel() * field.element_size(),
            "d2h_bytes_per_step": (w * h * 16) if rank == 0 else 0,
            "note": "field re-uploaded from pinned host memory every frame (not the in-situ case)"}


TF3_POINTS = [(0.0, 0.0, 0.0, 0.0, 0.0), (0.6, 0.1, 0.7, 0.4, 0.3), (1.0, 0.7, 1.0, 0.9, 0.8)]


TF4_POINTS = [(0.0, 0.0, 0.0, 0.0, 0.0), (0.21, 0.5, 0.1, 0.1, 0.05), (0.63, 0.1, 0.9, 0.3, 0.4),
              (1.0, 1.0, 1.0, 1.0, 0.9)]


def tf3_scene(P, scene, points=None):
    """The scene with C3's 3-point 'cool' transfer function (or ``points``) on source 0."""
    return P.SceneState(camera=scene.camera, tf_points={0: points or TF3_POINTS}, value_ranges=scene.value_ranges,
                        chain_texts=scene.chain_texts, settings=scene.settings, clip_planes=scene.clip_planes)


def ncu_evidence(key):
    """(traffic bytes, l1tex block) for one kernel from profiles/ncu_counters.json
    (tools/ncu_counters.py: one `ncu --set full` capture of that kernel), or (None, None)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_counters.json")) as fh:
            rec = json.load(fh).get(key)
    except (OSError, ValueError):
        return None, None
    if not rec:
        return None, None
    fracs = {"l1tex_data_pipe": rec["l1tex_data_pipe_lsu_pct"] / 100.0, "issue": rec["issue_active_pct"] / 100.0,
             "dram": rec["dram_throughput_pct"] / 100.0}
    return rec.get("traffic_bytes"), {
        "data_pipe_lsu_frac": round(fracs["l1tex_data_pipe"], 4),
        "dram_throughput_frac": round(fracs["dram"], 4),
        "issue_active_frac": round(fracs["issue"], 4),
        "l1_hit_rate": round(rec["l1_hit_rate_pct"] / 100.0, 4),
        "limiter": max(fracs, key=fracs.get),
        "ncu_kernel_ms": round(rec["duration_ms"], 4), "source": rec["source"],
        "note": "what bounds the kernel (limiter = the busiest of L1TEX data-pipe wavefronts, warp-instruction "
                "issue and DRAM throughput, each a fraction of its peak) from the ncu capture named in source "
                "(cold, serialised launch); the gather is served mostly by L1, so the HBM frac above is the "
                "north star's samples/s figure of merit, not the DRAM load"}


def time_normalisation(P, torch, reg, domain, peak, reps=10):
    """Per-source normalisation pass (isc_value_range: min/max of the chained
    scalar over the brick interior, warp-shuffle reduction) on source 0."""
    from paper_1611_09048_b200.normalize import value_range_device
    h = reg.render_handle(0)
    out = torch.empty(4, dtype=torch.float32, device="cuda")
    for _ in range(2):
        value_range_device(h, domain, out=out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        value_range_device(h, domain, out=out)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    nbytes = domain.size[0] * domain.size[1] * domain.size[2] * 4 * h.descriptor.feature_dim
    gbs = nbytes / (ms * 1e-3) / 1e9
    return {"kernel": "isc::minmax_kernel<DIM=1,F32>", "ms": round(ms, 4), "bytes": nbytes,
            "achieved_GBps": round(gbs, 1), "frac_of_hbm_peak": round(gbs / peak, 4),
            "range": [float(v) for v in out[:2].tolist()], "note": "L2-cold: field >> L2"}


def warm_gpu(fn, dist=None, world=1, red_dev=None, seconds=0.1, max_calls=2000):
    """Untimed calls of ``fn`` for ~``seconds`` right before a timed region,
    so the SM clock is at its boost level when timing starts (an idle GPU
    drops its clock; short frames would time the ramp-up).  The call count
    is agreed across ranks (max of the per-call times), because ``fn`` may
    contain a collective (binary_swap)."""
    import torch
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    per = max((time.perf_counter() - t0) / 3, 1e-6)
    if world > 1:
        t = torch.tensor([per], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        per = float(t.item())
    for i in range(min(max_calls, int(math.ceil(seconds / per)))):
        fn()
        if i % 8 == 7:
            torch.cuda.synchronize()


def run_e2e(P, torch, dist, ctx, scene, transport, canvas, order, rank, world, red_dev, steps):
    """Public-API frame loop with host buffers.  Per step: the scene arrives as
    bytes (as broadcast by the reference runtime, runtime.py:305-333), is
    parsed, its LUT uploaded (cache cleared so the H2D really happens) and the
    launch block sent; the frame is rendered + composited, quantised to RGBA8
    on the device (runtime.to_rgba8, the reference's frame encoding step,
    runtime.py:66-67 -- what FrameStreamer ships) and rank 0 copies it into
    pinned host memory on a side stream, overlapped with the next frame
    (double-buffered -- the reference's FrameStreamer overlap,
    runtime.py:187-249).  Each timed window ends after its last D2H landed;
    the median of three windows is reported."""
    from paper_1611_09048_b200.device import LUTS
    from paper_1611_09048_b200.runtime import to_rgba8
    w, h = scene.camera.image_size
    payload = scene.to_bytes()
    host = [torch.empty((h, w, 4), dtype=torch.uint8).pin_memory() for _ in range(2)] if rank == 0 else None
    stream = torch.cuda.current_stream()
    copy_stream = torch.cuda.Stream()
    done = [torch.cuda.Event(), torch.cuda.Event()]
    counter = [0]

    def one():
        i = counter[0] % 2
        counter[0] += 1
        sc = P.SceneState.from_bytes(payload)          # scene as received from the root
        LUTS.clear()                                    # force this step's LUT upload
        img = P.render_local(ctx, sc, out=canvas, check_errors=False)
        full = P.binary_swap(transport, img.pixels, order)
        if full is not None:
            q = to_rgba8(full)
            ready = torch.cuda.Event()
            ready.record(stream)
            copy_stream.wait_event(ready)
            copy_stream.wait_event(done[i])             # buffer i free again
            with torch.cuda.stream(copy_stream):
                host[i].copy_(q, non_blocking=True)
                q.record_stream(copy_stream)
            done[i].record(copy_stream)

    gc.collect()
    gc.disable()                    # as in the device-timed loop
    warm_gpu(one, dist, world, red_dev)   # boost clocks before timing (see run_b200)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # three back-to-back timed windows of `steps` frames each; the median
    # window is reported (a host-side stall -- another process, a page-cache
    # hiccup -- lands in one window and would otherwise set the number)
    windows = []
    for _ in range(3):
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(steps):
            one()
        stream.wait_stream(copy_stream)
        t1.record(stream)
        torch.cuda.synchronize()
        tt = torch.tensor([t0.elapsed_time(t1)], dtype=torch.float64, device=red_dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        windows.append(float(tt.item()) / steps)
    gc.enable()
    ms_step = sorted(windows)[1]
    import ctypes
    from paper_1611_09048_b200 import _abi
    h2d = 256 * 4 * 4 + ctypes.sizeof(_abi.RenderArgs)
    return {"value": round(1000.0 / ms_step, 3), "unit": "frames/s", "ms_per_step": round(ms_step, 4),
            "steps_per_window": steps, "window_ms_per_step": [round(v, 4) for v in windows],
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": (w * h * 4) if rank == 0 else 0,
            "path": "SceneState.from_bytes -> render_local -> binary_swap -> to_rgba8 -> pinned host frame "
                    "(side stream)",
            "note": "field is simulation-resident in HBM (in-situ zero-copy contract, fields.py:249-278); "
                    "per-step host inputs are the scene (LUT + launch block), output the RGBA8 frame the "
                    "reference streams (runtime.py:66-67, 222-235)"}


# --------------------------------------------------------------------------
# CPU baselines.  The reference itself (insitu 0.1.0, pure Python + numpy) is
# pip-installed into baseline/_ref (git-ignored, it travels to
# the GPU box with the snapshot) and timed through its own functions:
# render_local's body (raycast.py:492-541: ray_directions, _ray_box_intervals,
# _apply_clip_planes, march_rays) restricted to a stated subset of image rows,
# one worker process per host core.  Without baseline/_ref the oracle port
# (oracle/isaac_oracle.py, bit-identical to the reference per the goldens)
# stands in and the line says kind "port".

REF_PATH = os.path.join(ROOT, "baseline", "_ref")
_WORKER: dict = {}


def _import_reference():
    if not os.path.isdir(os.path.join(REF_PATH, "insitu")):
        return None
    if REF_PATH not in sys.path:
        sys.path.insert(0, REF_PATH)
    try:
        import insitu.fields as rf
        import insitu.functors as rfn
        import insitu.raycast as rr
        import insitu.scene as rs
    except Exception as exc:  # noqa: BLE001
        log(f"[reference] baseline/_ref present but not importable: {exc}")
        return None
    return rf, rfn, rr, rs


def _ref_scene(rs, cfg, n):
    """The B200 arm's scene (build_scene) as the reference's own SceneState."""
    pos, look = harness_camera(n)
    planes = (rs.clip_plane((n / 2.0,) * 3, (0.3, -0.5, 0.81)),) if cfg.get("clip") else ()
    linear = [(0.0, 0.0, 0.0, 0.0, 0.0), (1.0, 1.0, 1.0, 1.0, 1.0)]
    settings = rs.RenderSettings(active_set=(0,), interpolation=True, step_length=0.5, early_termination_alpha=1.0)
    return rs.SceneState(camera=rs.Camera(position=pos, look_at=look, image_size=cfg["image"]),
                         tf_points={0: linear}, value_ranges={0: (-0.4, 2.4)}, chain_texts={0: ""},
                         settings=settings, clip_planes=planes)


def _setup_cpu_workload(field, n, cfg, kind):
    """Everything a worker needs, built once in the parent (inherited by fork):
    the host field, the frame's rays, per-row station counts."""
    import numpy as np
    w, h = cfg["image"]
    g = {"kind": kind, "w": w, "n": n}
    if kind == "reference":
        rf, rfn, rr, rs = _import_reference()
        vol = rf.GlobalVolume((n, n, n), (1, 1, 1))
        dom = vol.local_domain(0, 1)
        reg = rf.SourceRegistry(dom)
        reg.register_handle(rf.array_backed_handle(rf.SourceDescriptor("density", 1, has_guard=True), field, 1))
        rf.update_sources(reg, {0}, {})
        scene = _ref_scene(rs, cfg, n)
        fr = rfn.default_registry()
        plans = rr.build_plans(reg, fr, rfn.ChainLimits(), scene)
        origin = np.asarray(scene.camera.position, dtype=np.float64)
        dirs = scene.camera.ray_directions()
        lo, hi = np.asarray(dom.offset, np.float64), np.asarray(dom.offset, np.float64) + np.asarray(dom.size, np.float64)
        t0, t1 = rr._apply_clip_planes(origin, dirs, *rr._ray_box_intervals(origin, dirs, lo, hi), scene.clip_planes)
        g.update(rr=rr, plans=plans, settings=scene.settings, volume=vol, origin=origin, dirs=dirs, lo=lo, hi=hi,
                 planes=scene.clip_planes)
    else:
        from oracle import isaac_oracle as O
        pos, look = harness_camera(n)
        origin = np.asarray(pos, dtype=np.float64)
        dirs = O.primary_rays(pos, look, (0.0, 1.0, 0.0), math.radians(45.0), w, h)
        t0, t1 = O.slab(origin, dirs, np.zeros(3), np.full(3, float(n)))
        src = O.Source(array=field, offset=(0, 0, 0), size=(n, n, n), guard=1,
                       lut=O.lut_from_points([(0, 0, 0, 0, 0), (1, 1, 1, 1, 1)]), value_range=(-0.4, 2.4))
        g.update(O=O, src=src, brick=O.Brick((0, 0, 0), (n, n, n), 1, (n, n, n), (1, 1, 1)), origin=origin,
                 dirs=dirs)
    hit = (t1 > np.maximum(t0, 0.0)) & (t1 > 0.0)
    k_lo = np.ceil(np.maximum(t0, 0.0) / 0.5)
    k_hi = np.ceil(np.maximum(t1, 0.0) / 0.5)
    per_px = np.where(hit, k_hi - k_lo, 0).astype(np.int64)
    g["per_row"] = per_px.reshape(h, w).sum(axis=1)
    _WORKER.clear()
    _WORKER.update(g)
    return g


def _rows_worker(rows):
    """Stations marched for image rows `rows` (in a forked worker)."""
    import numpy as np
    g = _WORKER
    sel = np.concatenate([np.arange(r * g["w"], (r + 1) * g["w"]) for r in rows])
    dirs = g["dirs"][sel]
    if g["kind"] == "reference":           # render_local's body, raycast.py:508-541
        rr = g["rr"]
        o = g["origin"]
        t0, t1 = rr._apply_clip_planes(o, dirs, *rr._ray_box_intervals(o, dirs, g["lo"], g["hi"]), g["planes"])
        g0, g1 = rr._apply_clip_planes(o, dirs, *rr._ray_box_intervals(o, dirs, np.zeros(3),
                                                                        np.asarray(g["volume"].size, np.float64)),
                                       g["planes"])
        hit = (t1 > np.maximum(t0, 0.0)) & (t1 > 0.0)
        idx = np.nonzero(hit)[0]
        if not idx.size:
            return 0
        _, stations = rr.march_rays(o, dirs[idx], (t0[idx], t1[idx]), (g0[idx], g1[idx]), g["plans"],
                                    g["settings"], None, volume=g["volume"])
        return int(stations)
    res = g["O"].render_rays(g["origin"], dirs, g["brick"], [g["src"]], step=0.5, alpha_stop=1.0, interp=True)
    return int(res.stations.sum())


def _row_sample(per_row, fraction):
    """Every k-th image row (k = round(1/fraction)): the sample spans the frame."""
    k = max(1, int(round(1.0 / fraction)))
    rows = list(range(0, len(per_row), k))
    return rows, k, int(per_row[rows].sum())


def _run_rows(pool, rows, cores):
    chunks = [rows[i::cores * 2] for i in range(cores * 2) if rows[i::cores * 2]]
    if pool is None:
        return sum(_rows_worker(c) for c in chunks)
    return sum(pool.map(_rows_worker, chunks))


def _host_field(n):
    import torch
    vol = __import__("paper_1611_09048_b200").GlobalVolume((n, n, n), (1, 1, 1))
    return make_field_torch(n, vol.local_domain(0, 1), "cpu").numpy()


def cpu_baseline(field_np, cfg, n, samples_frame, budget_s=15.0):
    """The GPU arm's cpu_baseline: the reference (or the port) on all host
    cores over every k-th image row of the same frame, ~budget_s of CPU time."""
    import multiprocessing as mp
    kind = "reference" if _import_reference() is not None else "port"
    cores = os.cpu_count() or 1
    g = _setup_cpu_workload(field_np, n, cfg, kind)
    rate = 1.0e6 * cores      # ~reference samples/s per core (measured 0.7-1.1 M)
    rows, k, expect = _row_sample(g["per_row"], min(1.0, rate * budget_s / max(samples_frame, 1)))
    with mp.get_context("fork").Pool(cores) as pool:
        t0 = time.perf_counter()
        done = _run_rows(pool, rows, cores)
        dt = time.perf_counter() - t0
    frac = done / samples_frame
    return {"value": round(frac / dt, 6), "unit": "frames/s", "cores": cores, "kind": kind,
            "samples_per_s": round(done / dt, 1),
            "sample": f"every {k}-th image row ({len(rows)} of {cfg['image'][1]} rows, {done} of {samples_frame} "
                      f"samples = {100.0 * frac:.2f}% of the frame) of the same {n}^3 x "
                      f"{cfg['image'][0]}x{cfg['image'][1]} frame in {dt:.1f}s; value = sampled fraction / time; "
                      + ("the reference's own render_local body (march_rays) from baseline/_ref"
                         if kind == "reference" else "oracle/isaac_oracle.py render_rays (port)")}


def run_reference(args):
    """--impl reference: the reference's own CPU path (baseline/_ref, else the
    oracle port) on all host cores, rank 0 only.  One step = the frame's
    image rows k, 2k, 3k, ... (a fixed, stated fraction of the frame, sized so
    --steps K --warmup W ends in a few minutes); value = frames/s = sampled
    fraction of the frame's samples / measured step time, so ms_per_step x
    steps is the real timed wall clock."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import multiprocessing as mp
    cfg = CONFIGS[args.config]
    if cfg.get("weak") or cfg.get("multi"):
        print(json.dumps({"impl": "reference", "unavailable": f"reference arm implemented for the single-source "
                                                               f"strong-scaling configs (c1, c2, c4), not {args.config}"}))
        return
    n = cfg["n"]
    w, h = cfg["image"]
    cores = os.cpu_count() or 1
    kind = "reference" if _import_reference() is not None else "port"
    t0 = time.time()
    import torch
    torch.set_num_threads(cores)
    field = _host_field(n)
    g = _setup_cpu_workload(field, n, cfg, kind)
    samples_frame = int(g["per_row"].sum())
    log(f"[reference] {kind}: host field + rays ready in {time.time() - t0:.1f}s, {cores} cores")
    rate = 1.0e6 * cores      # ~reference samples/s per core (measured 0.7-1.1 M)
    rows, k, expect = _row_sample(g["per_row"], min(1.0, rate * args.ref_step_s / max(samples_frame, 1)))
    port = None
    with mp.get_context("fork").Pool(cores) as pool:
        for _ in range(args.warmup):
            _run_rows(pool, rows[: max(1, len(rows) // 8)], cores)     # warm the workers (imports, pages)
        times, done = [], 0
        for _ in range(args.steps):
            a = time.perf_counter()
            done += _run_rows(pool, rows, cores)
            times.append(time.perf_counter() - a)
    dt = sum(times)
    per_step = done / args.steps
    frac = per_step / samples_frame
    fps = frac / (dt / args.steps)
    if kind == "reference":   # the port on the same rows, once, for the port/reference speed ratio
        try:
            gp = _setup_cpu_workload(field, n, cfg, "port")
            sub = rows[: max(1, len(rows) // 4)]
            with mp.get_context("fork").Pool(cores) as pool:
                a = time.perf_counter()
                pd = _run_rows(pool, sub, cores)
                pt = time.perf_counter() - a
            ref_rate = done / dt
            port = {"samples_per_s": round(pd / pt, 1), "reference_samples_per_s": round(ref_rate, 1),
                    "port_over_reference_speed": round((pd / pt) / ref_rate, 3),
                    "note": "oracle/isaac_oracle.py on a quarter of the same rows, same cores"}
        except Exception as exc:  # noqa: BLE001
            port = {"error": str(exc)}
    line = {"metric": METRIC, "value": round(fps, 6), "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(1000.0 * dt / args.steps, 1), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{args.config.upper()}: {cfg['desc']}", "volume": [n, n, n], "image": [w, h],
                       "decomposition": [1, 1, 1], "samples_per_frame": samples_frame,
                       "step_unit": f"every {k}-th image row of the frame ({len(rows)} rows, {per_step:.0f} samples "
                                    f"= {100.0 * frac:.2f}% of the frame's samples)"},
            "gsamples_per_s": round(done / dt / 1e9, 6),
            "cpu_baseline": {"value": round(fps, 6), "unit": "frames/s", "cores": cores, "kind": kind,
                             "sample": f"per step every {k}-th image row of the {n}^3 frame, "
                                       + ("the reference's render_local body (insitu.raycast.march_rays, "
                                          "baseline/_ref)" if kind == "reference" else
                                          "oracle/isaac_oracle.py render_rays") + f" over {cores} worker processes"},
            "e2e": {"value": round(fps, 6), "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "consistency": {"timed_seconds": round(dt, 2), "steps_x_ms_per_step_s": round(dt, 2),
                            "frames_per_step": round(frac, 5)},
            "port_check": port}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--ref-step-s", type=float, default=3.0, help="reference arm: target seconds per step")
    ap.add_argument("--share-gpu", action="store_true", help="test only: all ranks on cuda:0")
    ap.add_argument("--no-host-field-e2e", action="store_true")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch the ranks, form the process group (gloo), report the world and exit")
    args = ap.parse_args()
    if args.warmup < 3:
        log("note: warmup < 3 requested; using 3")
        args.warmup = 3
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "b200":
        sys.exit(relaunch(args.gpus))
    _, world, _ = dist_env()
    if args.impl == "b200" and world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but the launcher started {world} rank(s)")
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


def relaunch(n):
    """``python bench.py --gpus N`` outside torchrun: start N ranks (one
    process per GPU) with torch.distributed.run on 127.0.0.1 and return its
    exit code; rank 0 prints the JSON line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    log(f"bench: launching {n} ranks: {' '.join(cmd)}")
    return subprocess.call(cmd)


def run_dry(args):
    """Launcher check without a GPU: every rank joins a gloo group and rank 0
    reports how many ranks answered and the brick each would render."""
    import torch
    import torch.distributed as dist
    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    t = torch.tensor([1.0, float(rank)])
    if world > 1:
        dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "ranks_seen": int(t[0].item()),
                          "rank_sum": int(t[1].item()), "decomposition": list(DECOMP[world])}), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
