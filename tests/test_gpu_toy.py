"""GPU harness field generator (isc_toy_fields) and the harness's own
three-source scene through frame_pipeline, against goldens produced by the
reference harness (ToyState fields, harness.run frames)."""

import threading

import numpy as np
import pytest

from golden_io import load, manifest

pytestmark = pytest.mark.gpu


def test_toy_fields_match_reference_harness():
    import paper_1611_09048_b200 as P
    from paper_1611_09048_b200.toy import HarnessConfig, ToyState
    gold = load(manifest()["toy"]["file"])
    cfg = HarnessConfig(size=(24, 16, 20), ranks=(2, 1, 1), image_size=(40, 30))
    vol = cfg.volume()
    for rank in range(2):
        st = ToyState(cfg, vol.local_domain(rank, 1))
        for step in (0, 3):
            st.step_index = step
            st.refresh()
            st.fill_scratch()
            for name in ("density", "velocity", "scratch"):
                got = getattr(st, name).cpu().numpy().astype(np.float64)
                want = gold[f"r{rank}_s{step}_{name}"]
                assert got.shape == want.shape
                assert np.abs(got - want).max() <= 2e-6, (rank, step, name)
    assert isinstance(P, object)


def test_harness_frames_match_reference_run():
    """harness.run(size 32^3, ranks 2x1x1, 3 steps, sources 0 + 2) restated on
    the GPU: ToyState fields, non-persistent current snapshotted per frame,
    frame_pipeline over a byte transport, composited on rank 0."""
    import torch
    import paper_1611_09048_b200 as P
    from paper_1611_09048_b200.runtime import PipelineContext, frame_pipeline
    from paper_1611_09048_b200.toy import HarnessConfig, ToyState, build_registry, default_scene
    gold = load(manifest()["toy"]["file"])
    cfg = HarnessConfig(size=(32, 32, 32), ranks=(2, 1, 1), image_size=(72, 40), active_sources=(0, 2))
    vol = cfg.volume()
    fabric = P.LocalFabric(2)
    frames, errs = {}, []

    def body(rank):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                dom = vol.local_domain(rank, 1)
                st = ToyState(cfg, dom)
                reg = build_registry(st, dom)
                fr = P.default_registry()
                ctx = PipelineContext(fabric.endpoint(rank), vol, dom, reg, fr, fr.limits, default_scene(cfg))
                for _ in range(3):
                    st.advance()
                    res = frame_pipeline(ctx, {"step": st.step_index})
                    if rank == 0:
                        frames[st.step_index] = res.image.cpu().numpy()
        except Exception as exc:  # noqa: BLE001
            errs.append(exc)

    ts = [threading.Thread(target=body, args=(r,)) for r in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(180)
    assert not errs, errs
    for step in (1, 2, 3):
        want = gold[f"frame_s{step}"]
        assert want[..., 3].max() > 0.5
        assert np.abs(frames[step] - want).max() <= 1e-3, step
