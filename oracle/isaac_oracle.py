"""CPU oracle for the ISAAC rendering hot path -- TEST INFRASTRUCTURE ONLY.

This module is the *checker*, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` may import it.  The product path
(``paper_1611_09048_b200``) never routes through here and fails loudly when
its CUDA library is missing.

It is a float64 numpy restatement of the reference algorithm
(``/root/reference/pkg/src/insitu``), written against plain arrays instead of
the reference's classes so it can travel to the GPU box (where
``/root/reference`` does not exist).  Every function cites the reference
file:line it restates.  Evaluation order of every float64 expression follows
the reference so results are bit-identical to it on the same machine; the
only BLAS-dependent expression is the clip-plane dot ``dirs @ n``
(``raycast.py:134``), which we also compute with ``@`` so that it picks the
same OpenBLAS kernel the reference would.

Parity pinning: ``tests/test_oracle_golden.py`` checks this module against
golden vectors produced by running the real reference
(``tests/golden/make_golden.py``) and against the reference tests'
closed-form known answers.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

LUT_ENTRIES = 256


class OracleGuardError(Exception):
    """Mirror of ``fields.GuardContractError`` (fields.py:32-33)."""


# ---------------------------------------------------------------------------
# Camera and primary rays  (scene.py:46-70)


def camera_frame(position, look_at, up):
    """Unit (forward, right, up) -- scene.py:46-53."""
    f = np.subtract(look_at, position, dtype=np.float64)
    f /= np.linalg.norm(f)
    r = np.cross(f, np.asarray(up, dtype=np.float64))
    r /= np.linalg.norm(r)
    u = np.cross(r, f)
    return f, r, u


def primary_rays(position, look_at, up, vertical_fov, width, height):
    """(H*W, 3) unit ray directions, row-major, y = 0 at the top -- scene.py:55-70.

    Per component: d = (fwd + xs*right) + ys*up, then divided by
    sqrt((dx*dx + dy*dy) + dz*dz).
    """
    f, r, u = camera_frame(position, look_at, up)
    tan_half = math.tan(vertical_fov / 2.0)
    aspect = width / height
    col = (np.arange(width, dtype=np.float64) + 0.5) / width * 2.0 - 1.0
    row = 1.0 - (np.arange(height, dtype=np.float64) + 0.5) / height * 2.0
    sx = col * tan_half * aspect          # (W,)
    sy = row * tan_half                   # (H,)
    d = np.empty((height, width, 3))
    for c in range(3):
        d[:, :, c] = (f[c] + sx[None, :] * r[c]) + sy[:, None] * u[c]
    length = np.sqrt((d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2])
    d /= length[..., None]
    return d.reshape(-1, 3)


# ---------------------------------------------------------------------------
# Ray / box / clip planes  (raycast.py:100-143)


def slab(origin, dirs, lo, hi):
    """Slab-test interval, parallel rays via +-inf -- raycast.py:100-120."""
    n = dirs.shape[0]
    t_in = np.full(n, -np.inf)
    t_out = np.full(n, np.inf)
    for a in range(3):
        o = origin[a]
        d = dirs[:, a]
        with np.errstate(divide="ignore", invalid="ignore"):
            ta = (lo[a] - o) / d
            tb = (hi[a] - o) / d
        near = np.minimum(ta, tb)
        far = np.maximum(ta, tb)
        flat = d == 0.0
        inside = (o >= lo[a]) & (o <= hi[a])
        near = np.where(flat, -np.inf if inside else np.inf, near)
        far = np.where(flat, np.inf if inside else -np.inf, far)
        t_in = np.maximum(t_in, near)
        t_out = np.minimum(t_out, far)
    return t_in, t_out


def clip(origin, dirs, t_in, t_out, planes):
    """Intersect with each plane's kept half-space -- raycast.py:123-143.

    ``planes``: sequence of (point, unit normal).  ``f0`` uses np.dot and
    ``dn`` uses ``@`` exactly as the reference does (BLAS ddot / dgemv).
    """
    for point, normal in planes:
        nv = np.asarray(normal, dtype=np.float64)
        f0 = np.dot(origin - np.asarray(point, dtype=np.float64), nv)
        dn = dirs @ nv
        with np.errstate(divide="ignore", invalid="ignore"):
            tc = -f0 / dn
        t_in = np.where(dn > 0, np.maximum(t_in, tc), t_in)
        t_out = np.where(dn < 0, np.minimum(t_out, tc), t_out)
        t_out = np.where((dn == 0) & (f0 < 0), -np.inf, t_out)
    return t_in, t_out


def hit_mask(t_in, t_out):
    """raycast.py:522."""
    return (t_out > np.maximum(t_in, 0.0)) & (t_out > 0.0)


def station_range(t_in, t_out, step):
    """Half-open global station range [k_lo, k_hi) -- raycast.py:316-324."""
    lo = np.ceil(np.maximum(t_in, 0.0) / step).astype(np.int64)
    hi = np.ceil(np.maximum(t_out, 0.0) / step).astype(np.int64)
    return lo, hi


# ---------------------------------------------------------------------------
# Transfer functions  (scene.py:113-152)


def lut_from_points(points):
    """256-entry RGBA LUT by np.interp of (t, r, g, b, a) points -- scene.py:113-126."""
    pts = sorted((tuple(float(v) for v in p) for p in points), key=lambda p: p[0])
    if not pts:
        pts = [(0.0, 0.0, 0.0, 0.0, 0.0), (1.0, 1.0, 1.0, 1.0, 1.0)]
    knots = np.asarray([p[0] for p in pts])
    grid = np.linspace(0.0, 1.0, LUT_ENTRIES)
    lut = np.empty((LUT_ENTRIES, 4))
    for c in range(4):
        lut[:, c] = np.interp(grid, knots, np.asarray([p[c + 1] for p in pts]))
    return lut


def classify(lut, lo, hi, values):
    """Straight RGBA lookup with linear interpolation -- scene.py:139-152."""
    bad = ~np.isfinite(values)
    with np.errstate(invalid="ignore"):
        t = np.clip((values - lo) / (hi - lo), 0.0, 1.0)
    t = np.where(bad, 0.0, t)
    x = t * (LUT_ENTRIES - 1)
    i0 = np.floor(x).astype(np.intp)
    i1 = np.minimum(i0 + 1, LUT_ENTRIES - 1)
    w = (x - i0)[:, None]
    out = lut[i0] * (1.0 - w) + lut[i1] * w
    if bad.any():
        out[bad] = 0.0
    return out


def over(front, back):
    """Premultiplied over, C = C_f + (1 - A_f) C_b -- compositing.py:25-33."""
    return front + (1.0 - front[..., 3:4]) * back


# ---------------------------------------------------------------------------
# Functor chains  (functors.py:102-147, 212-240)

# name -> (takes_argument, output dim given input dim, float64 evaluator)
_BUILTIN_OPS = {
    "add": (True, lambda d: d, lambda v, c: v + c[None, :]),
    "mul": (True, lambda d: d, lambda v, c: v * c[None, :]),
    "length": (False, lambda d: 1, lambda v, c: np.sqrt(np.sum(v * v, axis=1, keepdims=True))),
    "sum": (False, lambda d: 1, lambda v, c: np.sum(v, axis=1, keepdims=True)),
    "pow": (True, lambda d: d, None),
}
# Device ops beyond the five built-ins, for user-registered functors.
_EXTRA_OPS = {
    "sqrt": (False, lambda d: d, lambda v, c: np.sqrt(v)),
    "abs": (False, lambda d: d, lambda v, c: np.abs(v)),
    "neg": (False, lambda d: d, lambda v, c: -v),
    "exp": (False, lambda d: d, lambda v, c: np.exp(v)),
    "log": (False, lambda d: d, lambda v, c: np.log(v)),
    "min": (True, lambda d: d, lambda v, c: np.minimum(v, c[None, :])),
    "max": (True, lambda d: d, lambda v, c: np.maximum(v, c[None, :])),
}


def _pow64(v, c):
    with np.errstate(invalid="ignore", divide="ignore", over="ignore"):
        return np.power(v, c[None, :])


def run_chain(steps, values):
    """Apply [(op, args or None), ...] to (m, dim) float64 -- functors.py:212-222."""
    out = values
    with np.errstate(invalid="ignore", divide="ignore", over="ignore"):
        for op, args in steps:
            const = None if args is None else np.asarray(args, dtype=np.float64)
            if op == "pow":
                out = _pow64(out, const)
                continue
            table = _BUILTIN_OPS if op in _BUILTIN_OPS else _EXTRA_OPS
            out = table[op][2](out, const)
    return out


def parse_steps(text, input_dim, max_length=5):
    """Minimal parser for the chain grammar (functors.py:150-205): returns
    [(op, broadcast args or None)].  Test helper; errors raise ValueError."""
    text = text.strip()
    if not text:
        return []
    parts = text.split("|")
    if len(parts) > max_length:
        raise ValueError("chain too long")
    dim = input_dim
    steps = []
    for part in parts:
        part = part.strip()
        if "(" in part:
            name, rest = part.split("(", 1)
            args = tuple(float(t) for t in rest.rstrip(")").split(","))
        else:
            name, args = part, None
        name = name.strip()
        takes, dmap, _ = {**_BUILTIN_OPS, **_EXTRA_OPS}[name]
        if takes:
            args = args * dim if len(args) == 1 else args
            if len(args) != dim:
                raise ValueError("bad argument count")
        steps.append((name, args))
        dim = dmap(dim)
    return steps


# ---------------------------------------------------------------------------
# Field sampling  (fields.py:218-246, raycast.py:169-199)


@dataclass
class Source:
    """One active source for the oracle (a SourcePlan restated, raycast.py:53-63)."""

    array: np.ndarray            # (z, y, x) or (z, y, x, dim) incl. guard halo
    offset: tuple                # brick offset in global cells (x, y, z)
    size: tuple                  # brick size (x, y, z)
    guard: int                   # domain guard width
    has_guard: bool = True
    steps: list = field(default_factory=list)   # chain [(op, args)]
    lut: Optional[np.ndarray] = None             # (256, 4) float64
    value_range: tuple = (0.0, 1.0)
    mode: str = "volume"
    iso_threshold: float = 0.5

    @property
    def dim(self):
        return 1 if self.array.ndim == 3 else self.array.shape[3]


def fetch(src: Source, ix, iy, iz, interp: bool):
    """Guard/clamp read of integer local indices -> (m, dim) float64 -- fields.py:218-246, 274-276."""
    sx, sy, sz = src.size
    if src.has_guard and interp:
        g = src.guard
        outside = ((ix < -g) | (ix >= sx + g) | (iy < -g) | (iy >= sy + g)
                   | (iz < -g) | (iz >= sz + g))
        if outside.any():
            raise OracleGuardError(f"{int(outside.sum())} indices beyond guard halo")
    else:
        ix = np.clip(ix, 0, sx - 1)
        iy = np.clip(iy, 0, sy - 1)
        iz = np.clip(iz, 0, sz - 1)
    g = src.guard
    vals = np.asarray(src.array[iz + g, iy + g, ix + g], dtype=np.float64)
    return vals[:, None] if vals.ndim == 1 else vals


def field_values(src: Source, local, interp: bool):
    """Trilinear (8 corners, dx fastest, weight (wx*wy)*wz) or nearest -- raycast.py:169-199."""
    base = np.floor(local).astype(np.intp)
    if not interp:
        return fetch(src, base[:, 0], base[:, 1], base[:, 2], False)
    frac = local - base
    acc = np.zeros((local.shape[0], src.dim))
    for cz in (0, 1):
        wz = frac[:, 2] if cz else 1.0 - frac[:, 2]
        for cy in (0, 1):
            wy = frac[:, 1] if cy else 1.0 - frac[:, 1]
            for cx in (0, 1):
                wx = frac[:, 0] if cx else 1.0 - frac[:, 0]
                v = fetch(src, base[:, 0] + cx, base[:, 1] + cy, base[:, 2] + cz, True)
                acc += (wx * wy * wz)[:, None] * v
    return acc


def scalar_at(src: Source, pos, interp: bool):
    """Global positions -> chained first-component scalars -- raycast.py:169-179, functors.py:239-240."""
    local = pos - np.asarray(src.offset, dtype=np.float64)
    return run_chain(src.steps, field_values(src, local, interp))[:, 0]


def _reachable(lo_corner, size, guard, pos):
    """raycast.py:270-278 and 463-468 (offset/size may be per row)."""
    lo = lo_corner - guard
    hi = lo_corner + size + guard - 1
    return ((pos >= lo) & (pos < hi)).all(axis=1)


def _owner_brick(vol_size, decomp, pos):
    """(offset, size) of the brick holding each position -- raycast.py:281-288."""
    bsize = np.asarray([vol_size[a] / decomp[a] for a in range(3)])
    cell = np.clip(np.floor(pos / bsize[None, :]), 0, np.asarray(decomp)[None, :] - 1)
    return cell * bsize[None, :], np.broadcast_to(bsize, pos.shape)


def surface_normals(src: Source, pos, view, interp: bool):
    """Central differences of the chained scalar, clamped stencil -- raycast.py:202-242."""
    g = src.guard if (src.has_guard and interp) else 0
    lo = np.asarray(src.offset, dtype=np.float64) - g
    hi = lo + np.asarray(src.size, dtype=np.float64) + 2 * g - 1 - 1e-9
    grad = np.empty_like(pos)
    for a in range(3):
        up = pos.copy()
        dn = pos.copy()
        up[:, a] = np.clip(pos[:, a] + 1.0, lo[a], hi[a])
        dn[:, a] = np.clip(pos[:, a] - 1.0, lo[a], hi[a])
        width = up[:, a] - dn[:, a]
        width[width == 0.0] = 1.0
        grad[:, a] = (scalar_at(src, up, interp) - scalar_at(src, dn, interp)) / width
    mag = np.sqrt((grad[:, 0] * grad[:, 0] + grad[:, 1] * grad[:, 1]) + grad[:, 2] * grad[:, 2])
    flat = mag < 1e-12
    with np.errstate(invalid="ignore", divide="ignore"):
        nrm = grad / mag[:, None]
    if flat.any():
        v = view[flat]
        vm = np.sqrt((v[:, 0] * v[:, 0] + v[:, 1] * v[:, 1]) + v[:, 2] * v[:, 2])
        nrm[flat] = -v / vm[:, None]
    return nrm


# ---------------------------------------------------------------------------
# The brick render  (raycast.py:291-381, 384-468, 492-541)


@dataclass
class Brick:
    offset: tuple
    size: tuple
    guard: int
    volume_size: tuple
    decomposition: tuple = (1, 1, 1)


@dataclass
class RenderResult:
    rgba: np.ndarray           # (H, W, 4) float64 premultiplied
    stations: np.ndarray       # (H*W,) int64 stations marched per pixel
    hit: np.ndarray            # (H*W,) bool
    t_in: np.ndarray
    t_out: np.ndarray
    k_lo: np.ndarray           # (H*W,) int64, 0 where not hit
    k_hi: np.ndarray
    kg_lo: np.ndarray
    kg_hi: np.ndarray

    @property
    def total_stations(self) -> int:
        return int(self.stations.sum())


def render_brick(camera: dict, brick: Brick, sources: Sequence[Source], *, step=0.5,
                 alpha_stop=1.0, interp=True, planes=(), recorder: Optional[Callable] = None,
                 dirs: Optional[np.ndarray] = None) -> RenderResult:
    """One brick's partial image -- raycast.py:492-541 with march_rays (291-381).

    ``camera``: dict(position, look_at, up, vertical_fov, width, height).
    ``sources``: the active sources in source-id order.
    """
    w, h = camera["width"], camera["height"]
    if dirs is None:
        dirs = primary_rays(camera["position"], camera["look_at"], camera.get("up", (0.0, 1.0, 0.0)),
                            camera.get("vertical_fov", math.radians(45.0)), w, h)
    res = render_rays(camera["position"], dirs, brick, sources, step=step, alpha_stop=alpha_stop,
                      interp=interp, planes=planes, recorder=recorder)
    res.rgba = res.rgba.reshape(h, w, 4)
    return res


def render_rays(position, dirs, brick: Brick, sources: Sequence[Source], *, step=0.5, alpha_stop=1.0,
                interp=True, planes=(), recorder: Optional[Callable] = None) -> RenderResult:
    """The per-ray body of :func:`render_brick` for an arbitrary ray list
    (``rgba`` comes back flat, (n, 4))."""
    origin = np.asarray(position, dtype=np.float64)
    lo = np.asarray(brick.offset, dtype=np.float64)
    hi = lo + np.asarray(brick.size, dtype=np.float64)
    t_in, t_out = clip(origin, dirs, *slab(origin, dirs, lo, hi), planes)
    g_in, g_out = clip(origin, dirs, *slab(origin, dirs, np.zeros(3),
                                            np.asarray(brick.volume_size, dtype=np.float64)), planes)
    hit = hit_mask(t_in, t_out)
    npx = dirs.shape[0]
    k_lo = np.zeros(npx, np.int64)
    k_hi = np.zeros(npx, np.int64)
    kg_lo = np.zeros(npx, np.int64)
    kg_hi = np.zeros(npx, np.int64)
    rays = np.nonzero(hit)[0]
    k_lo[rays], k_hi[rays] = station_range(t_in[rays], t_out[rays], step)
    kg_lo[rays], kg_hi[rays] = station_range(g_in[rays], g_out[rays], step)
    image = np.zeros((npx, 4))
    per_px = np.zeros(npx, np.int64)
    if rays.size:
        rgba, cnt = _march(origin, dirs[rays], k_lo[rays], k_hi[rays], kg_lo[rays], kg_hi[rays],
                           brick, sources, step, alpha_stop, interp,
                           None if recorder is None else (lambda k, sub: recorder(k, rays[sub])))
        image[rays] = rgba
        per_px[rays] = cnt
    return RenderResult(image, per_px, hit, t_in, t_out, k_lo, k_hi, kg_lo, kg_hi)


def _march(origin, dirs, k_lo, k_hi, kg_lo, kg_hi, brick, sources, step, alpha_stop, interp, recorder):
    n = dirs.shape[0]
    acc = np.zeros((n, 4))
    done = np.zeros(n, bool)
    count = np.zeros(n, np.int64)
    iso_state = {i: np.full(n, np.nan) for i, s in enumerate(sources) if s.mode == "iso"}
    if n == 0 or not (k_lo < k_hi).any():
        return acc, count
    gate_alpha = alpha_stop < 1.0
    for k in range(int(k_lo.min()), int(k_hi.max())):
        live = np.nonzero(~done & (k >= k_lo) & (k < k_hi))[0]
        if live.size == 0:
            continue
        count[live] += 1
        if recorder is not None:
            recorder(k, live)
        d = dirs[live]
        pos = origin[None, :] + (k * step) * d
        colour = np.zeros((live.size, 4))
        stop = np.zeros(live.size, bool)
        for i, src in enumerate(sources):
            s = scalar_at(src, pos, interp)
            if src.mode == "iso":
                got, tau, back_off = _iso_pairs(src, iso_state[i], k, pos, s, live, d, origin, step,
                                                k_lo, k_hi, kg_lo, kg_hi, brick, interp)
                if got.any():
                    dh = d[got]
                    where = pos[got] + (tau[got] + back_off[got])[:, None] * step * dh
                    nrm = surface_normals(src, where, dh, interp)
                    shade = np.abs((nrm[:, 0] * dh[:, 0] + nrm[:, 1] * dh[:, 1]) + nrm[:, 2] * dh[:, 2])
                    tint = classify(src.lut, src.value_range[0], src.value_range[1],
                                    np.full(int(got.sum()), src.iso_threshold))
                    layer = np.empty((int(got.sum()), 4))
                    layer[:, :3] = tint[:, :3] * shade[:, None]
                    layer[:, 3] = 1.0
                    colour[got] = over(colour[got], layer)
                    stop |= got
            else:
                c = classify(src.lut, src.value_range[0], src.value_range[1], s)
                layer = np.empty_like(c)
                layer[:, :3] = c[:, :3] * c[:, 3:4]
                layer[:, 3] = c[:, 3]
                colour = over(colour, layer)
        acc[live] = over(acc[live], colour)
        finished = stop
        if gate_alpha:
            finished = finished | (acc[live, 3] >= alpha_stop)
        done[live] |= finished
    return acc, count


def _iso_pairs(src, prev_all, k, pos, s_now, live, d, origin, step, k_lo, k_hi, kg_lo, kg_hi,
               brick, interp):
    """Sign-change ownership across bricks -- raycast.py:384-460."""
    m = live.size
    thr = src.iso_threshold
    exact = src.has_guard and interp
    off = np.asarray(src.offset, dtype=np.float64)
    size = np.asarray(src.size, dtype=np.float64)
    g = src.guard
    got = np.zeros(m, bool)
    tau = np.zeros(m)
    back_off = np.zeros(m)
    before = prev_all[live]

    entry = (k == k_lo[live]) & (k - 1 >= kg_lo[live])
    if entry.any():
        p_prev = origin[None, :] + ((k - 1) * step) * d[entry]
        v = np.full(int(entry.sum()), np.nan)
        ok = _reachable(off, size, g, p_prev) if exact else np.ones(p_prev.shape[0], bool)
        if ok.any():
            v[ok] = scalar_at(src, p_prev[ok], interp)
        before[entry] = v

    a = before - thr
    b = s_now - thr
    crossing = np.isfinite(a) & ((a < 0) != (b < 0))
    if crossing.any():
        den = a[crossing] - b[crossing]
        with np.errstate(divide="ignore", invalid="ignore"):
            tau[crossing] = np.where(den != 0.0, a[crossing] / den, 1.0)
        back_off[crossing] = -1.0
        got |= crossing

    if exact:
        tail = (k == k_hi[live] - 1) & (k + 1 < kg_hi[live]) & ~got
        if tail.any():
            p_next = origin[None, :] + ((k + 1) * step) * d[tail]
            mine = _reachable(off, size, g, p_next)
            n_off, n_size = _owner_brick(brick.volume_size, brick.decomposition, p_next)
            theirs = _reachable(n_off, n_size, g, pos[tail])
            ask = mine & ~theirs
            if ask.any():
                rows = np.nonzero(tail)[0][ask]
                c = scalar_at(src, p_next[ask], interp) - thr
                here = b[rows]
                flip = (here < 0) != (c < 0)
                if flip.any():
                    r = rows[flip]
                    den = here[flip] - c[flip]
                    with np.errstate(divide="ignore", invalid="ignore"):
                        tau[r] = np.where(den != 0.0, here[flip] / den, 1.0)
                    back_off[r] = 0.0
                    got[r] = True
    prev_all[live] = s_now
    return got, tau, back_off


# ---------------------------------------------------------------------------
# Sort-last compositing  (compositing.py:36-194)


def visibility_order(volume_size, decomposition, camera_position):
    """Nested-slab near-to-far brick order, x outermost -- compositing.py:36-63."""
    per_axis = []
    for a in range(3):
        width = volume_size[a] / decomposition[a]
        c = camera_position[a]
        keyed = sorted((max(i * width - c, 0.0, c - (i * width + width)), i)
                       for i in range(decomposition[a]))
        per_axis.append([i for _, i in keyed])
    dx, dy, _ = decomposition
    return [bx + by * dx + bz * dx * dy
            for bx in per_axis[0] for by in per_axis[1] for bz in per_axis[2]]


def composite_in_order(images, order):
    """Front-to-back fold -- compositing.py:66-77."""
    out = np.zeros_like(images[0])
    for r in order:
        out = over(out, images[r])
    return out


def swap_schedule(rank, size, order, n_pixels):
    """Per-round (partner, keep span, give span, partner_in_front) -- compositing.py:133-167."""
    v = list(order).index(rank)
    lo, hi = 0, n_pixels
    plan = []
    for r in range(size.bit_length() - 1):
        bit = 1 << r
        pv = v ^ bit
        mid = (lo + hi) // 2
        if v & bit:
            keep, give = (mid, hi), (lo, mid)
        else:
            keep, give = (lo, mid), (mid, hi)
        plan.append((order[pv], keep, give, pv < v))
        lo, hi = keep
    return plan, (lo, hi)


def binary_swap_emulated(images, order):
    """Lock-step emulation of every rank's binary swap + collection.

    Returns (full image on rank 0, sent_bytes per rank, received_bytes per
    rank) with the reference's wire format (16-byte header + float64 span,
    compositing.py:80-104).  Non-power-of-two sizes use direct send
    (compositing.py:184-194).
    """
    size = len(images)
    shape = images[0].shape
    flat = [np.asarray(im, dtype=np.float64).reshape(-1, 4) for im in images]
    n = flat[0].shape[0]
    sent = [0] * size
    recv = [0] * size
    if size == 1:
        return images[0].copy(), sent, recv
    if size & (size - 1):
        for r in range(1, size):
            sent[r] += 16 + n * 32
            recv[0] += 16 + n * 32
        return composite_in_order(flat, order).reshape(shape), sent, recv
    plans = {r: swap_schedule(r, size, order, n) for r in range(size)}
    state = {r: (0, n, flat[r]) for r in range(size)}
    for rnd in range(size.bit_length() - 1):
        nxt = {}
        for r in range(size):
            partner, keep, give, partner_front = plans[r][0][rnd]
            lo, hi, mine = state[r]
            plo, phi, theirs = state[partner]
            incoming = theirs[keep[0] - plo: keep[1] - plo]
            kept = mine[keep[0] - lo: keep[1] - lo]
            sent[r] += 16 + (give[1] - give[0]) * 32
            recv[r] += 16 + (keep[1] - keep[0]) * 32
            merged = over(incoming, kept) if partner_front else over(kept, incoming)
            nxt[r] = (keep[0], keep[1], merged)
        state = nxt
    full = np.empty((n, 4))
    for r in range(size):
        lo, hi, mine = state[r]
        full[lo:hi] = mine
        if r:
            sent[r] += 16 + (hi - lo) * 32
            recv[0] += 16 + (hi - lo) * 32
    return full.reshape(shape), sent, recv


# ---------------------------------------------------------------------------
# Per-source normalisation (no reference function; north-star addition)


def _chain32(steps, v):
    """float32 chain in the device's operation order (no FMA contraction)."""
    v = v.astype(np.float32)
    with np.errstate(invalid="ignore", divide="ignore", over="ignore"):
        for op, args in steps:
            c = None if args is None else np.asarray(args, dtype=np.float32)[None, :]
            if op == "add":
                v = v + c
            elif op == "mul":
                v = v * c
            elif op == "pow":
                v = np.power(v, c)
            elif op in ("length", "sum"):
                acc = v[:, :1] * v[:, :1] if op == "length" else v[:, :1].copy()
                for j in range(1, v.shape[1]):
                    acc = acc + (v[:, j:j + 1] * v[:, j:j + 1] if op == "length" else v[:, j:j + 1])
                v = np.sqrt(acc) if op == "length" else acc
            elif op == "sqrt":
                v = np.sqrt(v)
            elif op == "abs":
                v = np.abs(v)
            elif op == "neg":
                v = -v
            elif op == "exp":
                v = np.exp(v)
            elif op == "log":
                v = np.log(v)
            elif op == "min":
                v = np.minimum(v, c)
            elif op == "max":
                v = np.maximum(v, c)
            else:
                raise ValueError(op)
    return v


def value_range(array, guard, steps=(), chunk=1 << 22):
    """(min, max) of the float32-chained first component over the brick
    interior (guard excluded), NaNs ignored; (nan, nan) if none finite-or-inf."""
    g = guard
    core = array[g:array.shape[0] - g, g:array.shape[1] - g, g:array.shape[2] - g]
    dim = 1 if core.ndim == 3 else core.shape[3]
    flat = core.reshape(-1, dim)
    lo, hi = np.float32(np.nan), np.float32(np.nan)
    for s in range(0, flat.shape[0], chunk):
        v = _chain32(list(steps), flat[s:s + chunk])[:, 0]
        v = v[~np.isnan(v)]
        if v.size:
            a, b = v.min(), v.max()
            lo = a if np.isnan(lo) else min(lo, a)
            hi = b if np.isnan(hi) else max(hi, b)
    return np.float32(lo), np.float32(hi)
