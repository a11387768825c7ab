"""The reference harness's analytic shear-flow simulation on the GPU
(SURVEY.md §8(f) row 3): ``ToyState`` / ``build_registry`` / ``default_scene``
(harness.py:47-220) with the fields computed by ``isc_toy_fields`` into CUDA
tensors, so the harness's own three-source workload (density, float3
velocity, non-persistent current = density * velocity) renders at full scale
through the zero-copy registry.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

from . import _abi
from .fields import SourceDescriptor, SourceRegistry, array_backed_handle
from .scene import Camera, RenderSettings, SceneState

GUARD = 1

__all__ = ["ToyParameters", "HarnessConfig", "default_scene", "ToyState", "build_registry"]


@dataclass(frozen=True)
class ToyParameters:
    """harness.py:50-55"""

    shear_speed: float = 0.5
    perturbation: float = 0.08
    seed: int = 7
    dt: float = 0.5


@dataclass
class HarnessConfig:
    """The render-relevant subset of harness.HarnessConfig (harness.py:58-77)."""

    size: tuple = (64, 64, 64)
    ranks: tuple = (2, 2, 2)
    image_size: tuple = (480, 270)
    active_sources: tuple = (0,)
    interpolation: bool = True
    step_length: float = 0.5
    period: int = 1
    params: ToyParameters = field(default_factory=ToyParameters)

    def volume(self):
        from .fields import GlobalVolume
        return GlobalVolume(tuple(self.size), tuple(self.ranks))


_WARM = [(0.0, 0.05, 0.05, 0.25, 0.0), (0.45, 0.1, 0.45, 0.85, 0.35), (0.75, 0.95, 0.65, 0.2, 0.7),
         (1.0, 1.0, 0.95, 0.75, 0.95)]
_COOL = [(0.0, 0.0, 0.0, 0.0, 0.0), (0.6, 0.1, 0.7, 0.4, 0.3), (1.0, 0.7, 1.0, 0.9, 0.8)]


def default_scene(config: HarnessConfig) -> SceneState:
    """The harness's default scene (harness.py:80-116)."""
    sx, sy, sz = config.size
    diag = math.sqrt(sx * sx + sy * sy + sz * sz)
    return SceneState(
        camera=Camera(position=(sx * 1.4, sy * 1.15, -0.8 * diag), look_at=(sx / 2.0, sy / 2.0, sz / 2.0),
                      up=(0.0, 1.0, 0.0), image_size=tuple(config.image_size)),
        tf_points={0: _WARM, 1: _COOL, 2: _COOL},
        value_ranges={0: (0.4, 1.7), 1: (-1.0, 1.0), 2: (-1.5, 1.5)},
        chain_texts={0: "", 1: "length", 2: "length"},
        settings=RenderSettings(active_set=tuple(config.active_sources), interpolation=config.interpolation,
                                step_length=config.step_length, early_termination_alpha=1.0),
        render_period=config.period)


class ToyState:
    """Per-rank analytic fields over the brick plus guard, resident on the GPU."""

    def __init__(self, config: HarnessConfig, domain, device=None):
        import torch
        from .device import require_cuda
        self.params = config.params
        self.global_size = tuple(config.size)
        self.domain = domain
        self.step_index = 0
        self.device = device or require_cuda()
        sx, sy, sz = domain.size
        shape = (sz + 2 * GUARD, sy + 2 * GUARD, sx + 2 * GUARD)
        self.density = torch.empty(shape, dtype=torch.float32, device=self.device)
        self.velocity = torch.empty(shape + (3,), dtype=torch.float32, device=self.device)
        self.scratch = torch.empty(shape + (3,), dtype=torch.float32, device=self.device)
        self.refresh()

    def refresh(self) -> None:
        from .device import stream_handle
        a = _abi.ToyArgs()
        a.global_size[:] = list(self.global_size)
        a.offset[:] = list(self.domain.offset)
        a.size[:] = list(self.domain.size)
        a.guard = GUARD
        a.step_index = self.step_index
        a.seed = int(self.params.seed)
        a.shear_speed, a.perturbation, a.dt = self.params.shear_speed, self.params.perturbation, self.params.dt
        a.density = self.density.data_ptr()
        a.velocity = self.velocity.data_ptr()
        _abi.check(_abi.lib().isc_toy_fields(C.byref(a), C.c_void_p(stream_handle())), "toy fields")

    def advance(self) -> None:
        self.step_index += 1
        self.refresh()

    def fill_scratch(self) -> None:
        self.scratch.copy_(self.density[..., None] * self.velocity)

    def density_sum(self) -> float:
        g = GUARD
        return float(self.density[g:-g, g:-g, g:-g].double().sum())


def build_registry(state: ToyState, domain) -> SourceRegistry:
    """density, velocity (persistent) and current (non-persistent, filled by
    its update hook from a shared scratch buffer) -- harness.py:197-220."""
    registry = SourceRegistry(domain)
    registry.register_handle(array_backed_handle(SourceDescriptor("density", 1, has_guard=True, persistent=True),
                                                 state.density, GUARD))
    registry.register_handle(array_backed_handle(SourceDescriptor("velocity", 3, has_guard=True, persistent=True),
                                                 state.velocity, GUARD))

    def current_update(enabled: bool, payload: object) -> None:
        if enabled:
            state.fill_scratch()

    registry.register_handle(array_backed_handle(SourceDescriptor("current", 3, has_guard=True, persistent=False),
                                                 state.scratch, GUARD, update_hook=current_update))
    return registry
