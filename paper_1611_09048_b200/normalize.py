"""Per-source normalisation: device min/max of the chained scalar.

No reference function exists for this -- value ranges are scene state in the
reference (scene.py:188, set by steering runtime.py:154-157 or hard-coded by
the harness harness.py:104).  The north star adds an automatic range: the
(min, max) of the float32-chained first component over each brick interior,
reduced across ranks.  ``isc_value_range`` is one streaming warp-shuffle
reduction over the field; min/max are exact operations, so the result is
bit-identical to the oracle and independent of the decomposition.
"""

from __future__ import annotations

import ctypes as C
import math
from typing import Iterable, Optional

import torch

from . import _abi
from .device import as_device_field, dtype_code, ptr, require_cuda, stream_handle
from .errors import FieldError
from .functors import FunctorChain, FunctorRegistry, default_registry, device_program, parse_chain

__all__ = ["value_range", "value_range_device", "reduce_range", "auto_value_ranges"]


def _source_struct(array, guard_arr: int, guard_dom: int, feature_dim: int, chain: Optional[FunctorChain],
                   device, keep: list) -> _abi.Source:
    t = as_device_field(array, device)
    keep.append(t)
    s = _abi.Source()
    st = list(t.stride())
    sz, sy, sx, sc = st[0], st[1], st[2], (st[3] if t.dim() == 4 else 1)
    shift = (guard_arr - guard_dom) * (sz + sy + sx)
    s.data = ptr(t) + shift * t.element_size()
    s.stride[:] = [sz, sy, sx, sc]
    s.dtype = dtype_code(t)
    s.feature_dim = feature_dim
    s.range_lo, s.range_hi = 0.0, 1.0
    prog = device_program(chain) if chain is not None else []
    s.n_steps = len(prog)
    for j, (op, in_dim, arg) in enumerate(prog):
        s.steps[j].op, s.steps[j].in_dim = op, in_dim
        s.steps[j].arg[:] = [float(v) for v in arg]
        s.steps[j].arg_d[:] = [float(v) for v in arg]
        s.step_ops |= (op & 0xF) << (4 * j)
    return s


def value_range_device(handle, domain, chain: Optional[FunctorChain] = None, *, out=None, stream=None):
    """Asynchronous form: launches ``isc_value_range`` and returns the (4,)
    float32 device tensor whose first two entries become (min, max)."""
    device = require_cuda()
    array, guard = handle.device_view(domain) if hasattr(handle, "device_view") else (handle, domain.guard_width)
    dim = handle.descriptor.feature_dim if hasattr(handle, "descriptor") else (1 if array.dim() == 3 else array.shape[3])
    need = tuple(domain.size[a] + 2 * guard for a in (2, 1, 0))
    if tuple(array.shape[:3]) != need:
        raise FieldError(f"array shape {tuple(array.shape)} does not match domain size + 2*guard {need}")
    keep: list = []
    src = _source_struct(array, guard, 0, dim, chain, device, keep)
    out = out if out is not None else torch.empty(4, dtype=torch.float32, device=device)
    size = (C.c_int32 * 3)(*[int(v) for v in domain.size])
    _abi.check(_abi.lib().isc_value_range(C.byref(src), size, 0, C.c_void_p(out.data_ptr()),
                                          C.c_void_p(stream_handle(stream))), "value_range")
    return out


def value_range(handle, domain, chain: Optional[FunctorChain] = None, *, group=None, stream=None):
    """(min, max) of the chained scalar of ``handle`` over ``domain``'s interior.

    With ``group`` (a torch.distributed process group, or True for WORLD) the
    per-rank results are all-reduced (MIN / MAX) so every rank gets the global
    range.  NaN samples are ignored; (nan, nan) if a brick has no value.
    """
    out = value_range_device(handle, domain, chain, stream=stream)
    lo, hi = out[:2].tolist()
    if group is not None:
        return reduce_range(lo, hi, group)
    return (lo, hi)


def reduce_range(lo: float, hi: float, group=True):
    """Global (min, max) over the ranks of ``group`` (True = WORLD) from each
    rank's brick range; a rank whose brick has no value passes (nan, nan)
    and is ignored; (nan, nan) if no rank has a value.  One MIN/MAX
    all-reduce pair on a float32 pair (NCCL on the GPU, gloo on the host)."""
    import torch.distributed as dist
    g = None if group is True else group
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(g) == "nccl" else torch.device("cpu")
    lo_t = torch.tensor([math.inf if math.isnan(lo) else lo], dtype=torch.float32, device=dev)
    hi_t = torch.tensor([-math.inf if math.isnan(hi) else hi], dtype=torch.float32, device=dev)
    dist.all_reduce(lo_t, op=dist.ReduceOp.MIN, group=g)
    dist.all_reduce(hi_t, op=dist.ReduceOp.MAX, group=g)
    glo, ghi = float(lo_t.item()), float(hi_t.item())
    if math.isinf(glo) and glo > 0:
        return (math.nan, math.nan)
    return (glo, ghi)


def auto_value_ranges(scene, rank_ctx, source_ids: Optional[Iterable[int]] = None, *, group=None,
                      functor_registry: Optional[FunctorRegistry] = None):
    """Return ``scene`` with value_ranges replaced by the measured ranges of the
    given (default: active) sources, through each source's own chain."""
    reg = functor_registry or getattr(rank_ctx, "functor_registry", None) or default_registry()
    ranges = dict(scene.value_ranges)
    sids = list(scene.settings.active_set if source_ids is None else source_ids)
    for sid in sids:
        handle = rank_ctx.registry.render_handle(sid)
        chain = parse_chain(scene.chain_text(sid), reg, None, handle.descriptor.feature_dim)
        lo, hi = value_range(handle, rank_ctx.domain, chain, group=group)
        if not (lo < hi):
            hi = lo + 1.0 if math.isfinite(lo) else 1.0
            lo = lo if math.isfinite(lo) else 0.0
        ranges[sid] = (lo, hi)
    return scene.bump(value_ranges=ranges)
