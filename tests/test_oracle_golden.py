"""Pin the CPU oracle against golden vectors produced by the real reference.

These run without a GPU.  The oracle must reproduce the reference
bit-for-bit on the machine that made the goldens (float64, same evaluation
order); we allow 1e-12 on colours and a few ulps on t only where the clip
plane BLAS dot may pick a different kernel on another host CPU.
"""

import math

import numpy as np
import pytest

from case_build import oracle_render
from golden_io import cases, decomp_key, load, manifest
from oracle import isaac_oracle as O

RENDER = sorted(cases.RENDER_CASES)


@pytest.mark.parametrize("name", RENDER)
def test_render_matches_reference(name):
    c = cases.case(name)
    gold = load(f"render_{name}.npz")
    for decomp in c["decompositions"]:
        key = decomp_key(decomp)
        images = []
        for rank in range(int(np.prod(decomp))):
            p = f"{key}_r{rank}_"
            res = oracle_render(c, gold, decomp, rank)
            assert np.array_equal(res.hit, gold[p + "hit"]), (name, key, rank)
            for k in ("k_lo", "k_hi", "kg_lo", "kg_hi"):
                assert np.array_equal(getattr(res, k), gold[p + k].astype(np.int64)), (name, k)
            assert np.array_equal(res.stations, gold[p + "stations"].astype(np.int64))
            finite = np.isfinite(gold[p + "t_in"])
            assert np.array_equal(finite, np.isfinite(res.t_in))
            np.testing.assert_allclose(res.t_in[finite], gold[p + "t_in"][finite], rtol=4e-16, atol=0)
            np.testing.assert_allclose(res.rgba, gold[p + "rgba"], rtol=0, atol=1e-12)
            images.append(res.rgba)
        order = O.visibility_order(c["size"], decomp, c["camera"]["position"])
        assert order == list(gold[key + "_order"])
        np.testing.assert_allclose(O.composite_in_order(images, order), gold[key + "_composite"],
                                   rtol=0, atol=1e-12)


def test_goldens_are_not_trivial():
    # Guard against a generator bug producing blank fixtures.
    for name in RENDER:
        gold = load(f"render_{name}.npz")
        tot = sum(float(v[..., 3].sum()) for k, v in gold.items() if k.endswith("_rgba"))
        assert tot > 0, name
    iso = load("render_iso_face.npz")
    assert (iso["d111_r0_rgba"][..., 3] > 0.5).sum() > 20


@pytest.mark.parametrize("name", sorted(cases.COMPOSITE_CASES))
def test_composite_matches_reference(name):
    gold = load(f"composite_{name}.npz")
    images = list(gold["images"])
    order = [int(v) for v in gold["order"]]
    full, sent, recv = O.binary_swap_emulated(images, order)
    np.testing.assert_allclose(full, gold["result"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(O.composite_in_order(images, order), gold["sequential"], atol=1e-15)
    assert list(sent) == list(gold["sent"])
    assert list(recv) == list(gold["received"])


def test_chains_match_reference():
    m = manifest()["chains"]
    gold = load(m["file"])
    for i, text in enumerate(m["texts"]):
        dim = int(gold["dims"][i])
        steps = O.parse_steps(text, dim)
        got = O.run_chain(steps, gold["inputs"][i][:, :dim])
        want = gold["outputs"][i][:, :int(gold["out_dims"][i])]
        assert got.shape == want.shape, text
        both_nan = np.isnan(got) & np.isnan(want)
        assert np.array_equal(got[~both_nan], want[~both_nan]), text


def test_classify_and_lut_match_reference():
    m = manifest()["classify"]
    gold = load(m["file"])
    for i, pts in enumerate(m["tf_points"]):
        lut = O.lut_from_points(pts)
        assert np.array_equal(lut, gold[f"lut{i}"])
        lo, hi = gold[f"range{i}"]
        assert np.array_equal(O.classify(lut, lo, hi, gold["values"]), gold[f"rgba{i}"])


# Closed-form known answers from the reference tests (test_raycast.py,
# test_compositing.py, test_functors.py), re-asserted on the oracle.

def test_known_answers_ray_box():
    o = np.asarray([-1.0, 0.5, 0.5])
    d = np.asarray([[1.0, 0.0, 0.0]])
    ti, to = O.slab(o, d, np.zeros(3), np.ones(3))
    assert to[0] - ti[0] == pytest.approx(1.0)
    plane = ((0.5, 0.0, 0.0), (1.0, 0.0, 0.0))
    ti, to = O.clip(o, d, ti, to, [plane])
    assert (ti[0], to[0]) == pytest.approx((1.5, 2.0))
    ti, to = O.slab(np.asarray([2.0, -1.0, 0.5]), np.asarray([[0.0, 1.0, 0.0]]), np.zeros(3), np.ones(3))
    assert to[0] < ti[0]


def test_known_answers_over_and_classify():
    got = O.over(np.asarray([0.5, 0.0, 0.0, 0.5]), np.asarray([0.0, 0.0, 0.5, 0.5]))
    assert tuple(got) == (0.5, 0.0, 0.25, 0.75)
    lut = np.repeat(np.linspace(0.0, 1.0, 256)[:, None], 4, axis=1)
    assert tuple(O.classify(lut, 0.0, 1.0, np.asarray([np.nan]))[0]) == (0.0, 0.0, 0.0, 0.0)
    mid = O.classify(lut, 0.0, 1.0, np.asarray([0.5]))[0]
    assert mid == pytest.approx((lut[127] + lut[128]) / 2.0, abs=1e-12)


def test_known_answers_chain():
    steps = O.parse_steps("mul(2,3,4) | add(1) | length", 3)
    assert O.run_chain(steps, np.asarray([[1.0, 1.0, 1.0]]))[0, 0] == math.sqrt(50.0)
    steps = O.parse_steps("mul(0,1,0) | sum", 3)
    assert O.run_chain(steps, np.asarray([[7.0, 9.0, 2.0]]))[0, 0] == 9.0


def test_homogeneous_alpha_accumulation():
    # A_N = 1 - (1 - a)^N (test_raycast.py:139-151), through render_brick with
    # a constant field, nearest sampling and a 1-pixel camera looking down +x.
    n = 32
    arr = np.full((n, n, n), 0.7, np.float32)
    lut = np.zeros((256, 4))
    lut[:, 3] = 0.3
    src = O.Source(array=arr, offset=(0, 0, 0), size=(n, n, n), guard=0, has_guard=False, lut=lut)
    brick = O.Brick((0, 0, 0), (n, n, n), 0, (n, n, n))
    cam = {"position": (-1.0, 16.0, 16.0), "look_at": (16.0, 16.0, 16.0), "width": 1, "height": 1}
    res = O.render_brick(cam, brick, [src], step=0.1, alpha_stop=1.0, interp=False)
    m = int(res.stations[0])
    assert res.rgba[0, 0, 3] == pytest.approx(1.0 - 0.7 ** m, abs=1e-9)
    res = O.render_brick(cam, brick, [src], step=0.1, alpha_stop=0.9, interp=False)
    assert res.rgba[0, 0, 3] == pytest.approx(1.0 - 0.7 ** 7, abs=1e-12)


def test_guard_contract_raises():
    arr = np.zeros((6, 6, 6), np.float32)
    src = O.Source(array=arr, offset=(0, 0, 0), size=(4, 4, 4), guard=1)
    with pytest.raises(O.OracleGuardError):
        O.fetch(src, np.asarray([5]), np.asarray([0]), np.asarray([0]), True)
    v = O.fetch(src, np.asarray([9]), np.asarray([-3]), np.asarray([0]), False)
    assert v.shape == (1, 1)


def test_value_range_float32_exact():
    rng = np.random.default_rng(3)
    arr = rng.standard_normal((10, 12, 14, 3)).astype(np.float32)
    lo, hi = O.value_range(arr, 1, O.parse_steps("length", 3))
    core = arr[1:-1, 1:-1, 1:-1].reshape(-1, 3)
    l32 = np.sqrt((core[:, 0] * core[:, 0] + core[:, 1] * core[:, 1]) + core[:, 2] * core[:, 2])
    assert lo == l32.min() and hi == l32.max()
